"""One-off parity evidence at config 5 (L7, 327,680 triangles): sampled rows of
the GPU matvec against the oracle's _apply_range restatement."""
import sys, time
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import hobi_oracle as O
from paper_1301_5914_b200 import discretize, PhysicalParams, SolverConfig, matvec_hobi
from paper_1301_5914_b200.surfaces import baseline_config
cfg = baseline_config(5)
t = time.time()
prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, SolverConfig(workers=1))
u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
full = matvec_hobi(prob, u)
print('gpu matvec done', time.time() - t, flush=True)
o = O.discretize(cfg.mesh.vertices, cfg.mesh.normals, cfg.mesh.faces, cfg.eps1, cfg.eps2, cfg.kappa, check=False)
print('oracle discretize', time.time() - t, flush=True)
T = prob.n_collocation
worst = 0.0
for lo in (0, 40000, 81921, 120000, T - 24):
    r1, r2 = O.rows(o, u, lo, lo + 24)
    e = max(np.linalg.norm(full[lo:lo + 24] - r1) / np.linalg.norm(r1),
            np.linalg.norm(full[T + lo:T + lo + 24] - r2) / np.linalg.norm(r2))
    worst = max(worst, e)
    print(f'rows [{lo},{lo+24}) rel err {e:.2e}', flush=True)
print(f'C5 sampled rows: max relative L2 error {worst:.2e} (gate 1e-10)')
