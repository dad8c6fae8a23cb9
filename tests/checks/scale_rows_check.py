"""Index-arithmetic check beyond the BASELINE sizes: config 5's surface at a
finer icosphere level (default 8: 1,310,720 triangles, 5.2M regular points,
3.4e12 pairs per matvec).  Full GPU matvec, then sampled row blocks against the
oracle's _apply_range restatement.  Usage: python tests/checks/scale_rows_check.py [level]"""
import sys, time
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import hobi_oracle as O
from paper_1301_5914_b200 import discretize, PhysicalParams, SolverConfig, matvec_hobi
from paper_1301_5914_b200.surfaces import baseline_config
level = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = baseline_config(5, level=level)
t = time.time()
prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, SolverConfig(workers=1))
print(f'{cfg.name}: {cfg.mesh.n_vertices} vertices, {cfg.mesh.n_faces} faces; discretize {time.time() - t:.1f} s', flush=True)
u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
matvec_hobi(prob, u)
t = time.time()
full = matvec_hobi(prob, u)
dt = time.time() - t
pairs = float(cfg.mesh.n_vertices) * cfg.mesh.n_faces * 4
print(f'gpu matvec {dt:.2f} s = {pairs / dt:.3e} pairs/s (host-buffer call)', flush=True)
o = O.discretize(cfg.mesh.vertices, cfg.mesh.normals, cfg.mesh.faces, cfg.eps1, cfg.eps2, cfg.kappa, check=False)
T = prob.n_collocation
worst = 0.0
for lo in (0, T // 3, T // 2 + 1, T - 24):
    r1, r2 = O.rows(o, u, lo, lo + 24)
    e = max(np.linalg.norm(full[lo:lo + 24] - r1) / np.linalg.norm(r1),
            np.linalg.norm(full[T + lo:T + lo + 24] - r2) / np.linalg.norm(r2))
    worst = max(worst, e)
    print(f'rows [{lo},{lo+24}) rel err {e:.2e}', flush=True)
print(f'L{level} sampled rows: max relative L2 error {worst:.2e} (gate 1e-10)')
