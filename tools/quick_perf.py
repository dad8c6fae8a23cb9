"""Scratch: time the matvec at configs 3-5 through the C ABI (device timing)."""
import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, '.')
from paper_1301_5914_b200 import _native as N, discretize, PhysicalParams, SolverConfig, matvec_hobi
from paper_1301_5914_b200.surfaces import baseline_config
lib = N.load()
t = C.c_double(0); lib.hobi_probe_fp64_tflops(0, 300.0, C.byref(t)); print('fp64 probe TF/s', t.value, flush=True)
for idx in [int(a) for a in sys.argv[1:]] or [3, 4]:
    cfg = baseline_config(idx)
    t0 = time.time()
    prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, SolverConfig(workers=1))
    print(cfg.name, 'discretize', time.time() - t0, flush=True)
    u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
    for _ in range(2): matvec_hobi(prob, u)
    lib.hobi_timing_reset(prob.handle)
    reps = 5
    t0 = time.time()
    for _ in range(reps): matvec_hobi(prob, u)
    wall = (time.time() - t0) / reps
    ms = C.c_double(0); nl = C.c_int64(0); al = C.c_int64(0)
    lib.hobi_timing(prob.handle, C.byref(ms), C.byref(nl), C.byref(al))
    pairs = C.c_double(0); lib.hobi_pairs_per_matvec(prob.handle, C.byref(pairs))
    sweep = ms.value / nl.value
    print(f'{cfg.name}: pairs {pairs.value:.3e} sweep {sweep:.3f} ms -> {pairs.value/sweep*1e3:.3e} pairs/s; wall {wall*1e3:.2f} ms; frac(96 flop/pair of {t.value:.1f}) {pairs.value/sweep*1e3*96/(t.value*1e12):.3f}', flush=True)
