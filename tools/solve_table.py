"""Solve-time table for BASELINE configs 1..5 on one GPU, with a breakdown."""
import sys, time, json, ctypes as C
sys.path.insert(0, '.')
from paper_1301_5914_b200 import (_native as N, discretize, PhysicalParams, SolverConfig, assemble_rhs,
                                  make_operator, gmres_solve, solvation_energy)
from paper_1301_5914_b200.surfaces import baseline_config
lib = N.load()
rows = []
for idx in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]:
    t0 = time.perf_counter(); cfg = baseline_config(idx); tgen = time.perf_counter() - t0
    scfg = SolverConfig(workers=1, restart=cfg.restart, tolerance=cfg.tol)
    t0 = time.perf_counter(); prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, scfg); tdisc = time.perf_counter() - t0
    for rep in range(2):
        lib.hobi_timing_reset(prob.handle)
        t0 = time.perf_counter(); b = assemble_rhs(prob); trhs = time.perf_counter() - t0
        t0 = time.perf_counter()
        with make_operator(prob, scfg) as op:
            sol = gmres_solve(op, b, scfg)
        tg = time.perf_counter() - t0
        t0 = time.perf_counter(); e = solvation_energy(prob, sol); te = time.perf_counter() - t0
    ms = C.c_double(0); nl = C.c_int64(0); al = C.c_int64(0)
    lib.hobi_timing(prob.handle, C.byref(ms), C.byref(nl), C.byref(al))
    r = dict(config=cfg.name, nv=cfg.mesh.n_vertices, nf=cfg.mesh.n_faces, nc=len(cfg.charges), gen_s=tgen, discretize_s=tdisc,
             rhs_s=trhs, gmres_s=tg, energy_s=te, iterations=sol.iterations, matvecs=sol.matvecs,
             sweep_ms_total=ms.value, launches=al.value, residual=sol.residual, energy=e)
    rows.append(r)
    print(json.dumps(r), flush=True)
