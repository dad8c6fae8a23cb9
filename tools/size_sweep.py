"""Throughput against problem size: sweep pairs/s (device events) and the
host-buffer matvec time for BASELINE configs 1-5 and config 5's surface at L8."""
import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, '.')
from paper_1301_5914_b200 import _native as N, discretize, PhysicalParams, SolverConfig, matvec_hobi
from paper_1301_5914_b200.surfaces import baseline_config
lib = N.load()
print("| config | N_v | N_f | pairs/matvec | sweep ms | sweep pairs/s | matvec ms (host buffers) |")
print("|---|---|---|---|---|---|---|")
for idx, lv in ((1, None), (2, None), (3, None), (4, None), (5, None), (5, 8)):
    cfg = baseline_config(idx, level=lv)
    prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, SolverConfig(workers=1))
    u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
    matvec_hobi(prob, u)
    matvec_hobi(prob, u)  # small problems: this call captures the host-buffer graph
    reps = 20 if cfg.mesh.n_faces <= 81920 else 3
    t0 = time.perf_counter()
    for _ in range(reps):
        matvec_hobi(prob, u)
    wall = (time.perf_counter() - t0) / reps * 1e3
    # sweep time from device events: resident-input applications (graph replays carry no event pairs)
    out, step_ms = np.empty_like(u), np.empty(reps)
    lib.hobi_timing_reset(prob.handle)
    N.check(lib.hobi_bench(prob.handle, N.dptr(u), N.dptr(out), reps, 0, 0, N.dptr(step_ms)))
    ms, nl = C.c_double(0), C.c_int64(0)
    lib.hobi_timing(prob.handle, C.byref(ms), C.byref(nl), None)
    pairs = C.c_double(0)
    lib.hobi_pairs_per_matvec(prob.handle, C.byref(pairs))
    sweep = ms.value / reps
    print(f"| {cfg.name} | {cfg.mesh.n_vertices} | {cfg.mesh.n_faces} | {pairs.value:.3e} | {sweep:.3f} | "
          f"{pairs.value / sweep * 1e3:.3e} | {wall:.3f} |", flush=True)
    prob.close()
