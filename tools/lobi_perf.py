import sys, ctypes as C, numpy as np
import os; os.environ.setdefault("HOBI_MATVEC_GRAPH", "0")  # event-timed sweeps need the plain host path
sys.path.insert(0, '.')
from paper_1301_5914_b200 import _native as N, discretize, PhysicalParams, SolverConfig, matvec_lobi, matvec_hobi
from paper_1301_5914_b200.surfaces import baseline_config
lib = N.load()
cfg = baseline_config(4)
for scheme, mv in (("lobi", matvec_lobi), ("hobi", matvec_hobi)):
    prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, SolverConfig(scheme=scheme, workers=1))
    u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
    mv(prob, u)
    lib.hobi_timing_reset(prob.handle)
    for _ in range(4): mv(prob, u)
    ms = C.c_double(0); nl = C.c_int64(0)
    lib.hobi_timing(prob.handle, C.byref(ms), C.byref(nl), None)
    pairs = C.c_double(0); lib.hobi_pairs_per_matvec(prob.handle, C.byref(pairs))
    t = ms.value / 4
    print(scheme, f"{t:.3f} ms per matvec sweep, {pairs.value/t*1e3:.3e} pairs/s, pairs {pairs.value:.3e}")
