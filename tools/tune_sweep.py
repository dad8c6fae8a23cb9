"""Scratch: time every sweep variant on a config (device time of the sweep kernel)."""
import sys, ctypes as C
import os; os.environ.setdefault("HOBI_MATVEC_GRAPH", "0")  # event-timed sweeps need the plain host path
import numpy as np
sys.path.insert(0, '.')
from paper_1301_5914_b200 import _native as N, discretize, PhysicalParams, SolverConfig, matvec_hobi
from paper_1301_5914_b200.surfaces import baseline_config
lib = N.load()
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = baseline_config(idx)
prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, SolverConfig(workers=1))
h = prob.handle
u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
n = C.c_int(0); name = C.create_string_buffer(64)
lib.hobi_sweep_variant(h, -1, C.byref(n), name, 64)
pairs = C.c_double(0); lib.hobi_pairs_per_matvec(h, C.byref(pairs))
ref = None
for v in range(n.value):
    N.check(lib.hobi_sweep_variant(h, v, None, name, 64))
    out = matvec_hobi(prob, u)
    if ref is None: ref = out
    same = np.array_equal(out, ref)
    lib.hobi_timing_reset(h)
    for _ in range(4): matvec_hobi(prob, u)
    ms = C.c_double(0); nl = C.c_int64(0)
    lib.hobi_timing(h, C.byref(ms), C.byref(nl), None)
    t = ms.value / nl.value
    print(f'{v:2d} {name.value.decode():24s} {t:8.3f} ms  {pairs.value/t*1e3:.4e} pairs/s  bitwise-same={same}', flush=True)
