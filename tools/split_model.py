"""Per-rank compute time of a p-way row split, measured on one GPU
(hobi_bench_rows over each rank's range), for configs 4 and 5.  The
slowest rank bounds the step; efficiency = T1 / (p * max_r T_r)."""
import sys, json
import numpy as np
sys.path.insert(0, '.')
from paper_1301_5914_b200 import _native as N, discretize, PhysicalParams, SolverConfig, partition_targets
from paper_1301_5914_b200.surfaces import baseline_config
lib = N.load()
res = {}
for idx in [int(a) for a in sys.argv[1:]] or [4, 5]:
    cfg = baseline_config(idx)
    prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, SolverConfig(workers=1))
    u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
    n = prob.n_collocation
    t1 = None
    for p in (1, 2, 4, 8):
        worst = 0.0
        ranks = partition_targets(n, p)
        for r, (lo, hi) in enumerate(ranks if p <= 2 else [ranks[0], ranks[-1]]):
            ms = np.zeros(3)
            N.check(lib.hobi_bench_rows(prob.handle, N.dptr(u), lo, hi, 3, 1, N.dptr(ms)))
            worst = max(worst, float(np.median(ms)))
        if p == 1: t1 = worst
        eff = t1 / (p * worst)
        print(f'C{idx} p={p}: slowest rank {worst:.3f} ms  compute-only efficiency {eff*100:.1f}%', flush=True)
        res[f'C{idx}_p{p}'] = {'rank_ms': worst, 'efficiency': eff}
print(json.dumps(res))
