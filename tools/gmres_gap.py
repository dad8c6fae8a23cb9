import sys, time
sys.path.insert(0, '.')
from paper_1301_5914_b200 import discretize, PhysicalParams, SolverConfig, assemble_rhs, make_operator, gmres_solve
from paper_1301_5914_b200.surfaces import baseline_config
for idx in (3, 4, 4, 4):
    cfg = baseline_config(idx)
    scfg = SolverConfig(workers=1, restart=cfg.restart)
    prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, scfg)
    b = assemble_rhs(prob)
    for rep in range(3):
        t0 = time.perf_counter()
        with make_operator(prob, scfg) as op:
            sol = gmres_solve(op, b, scfg)
        print(idx, rep, time.perf_counter() - t0, flush=True)
