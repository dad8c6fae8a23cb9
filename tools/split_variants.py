"""Scratch: per-rank sweep time for a p-way split under each tiling variant."""
import sys, ctypes as C
import numpy as np
sys.path.insert(0, '.')
from paper_1301_5914_b200 import _native as N, discretize, PhysicalParams, SolverConfig, partition_targets
from paper_1301_5914_b200.surfaces import baseline_config
lib = N.load()
cfg = baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, SolverConfig(workers=1))
u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
n = prob.n_collocation
name = C.create_string_buffer(64)
for v in (7, 4, 6, 3):
    N.check(lib.hobi_sweep_variant(prob.handle, v, None, name, 64))
    row = []
    for p in (1, 4, 8):
        lo, hi = partition_targets(n, p)[0]
        ms = np.zeros(3)
        N.check(lib.hobi_bench_rows(prob.handle, N.dptr(u), lo, hi, 3, 1, N.dptr(ms)))
        row.append(float(np.median(ms)))
    print(f"{name.value.decode():22s}", "  ".join(f"p={p}: {t:8.3f} ms eff {row[0]/(p*t)*100:5.1f}%" for p, t in zip((1, 4, 8), row)), flush=True)
