"""Is the oracle port a fair stand-in for the reference's CPU path?  Times the
unmodified reference (pbbem, from /root/reference -- build container only)
and the oracle port on the same rows of the same config-3 matvec, serial and
with the fork pool over all cores, and checks they agree.  Usage (repo root):
python tests/checks/cpu_baseline_fidelity.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
sys.path.insert(0, "/root/reference/pkg/src")
import hobi_oracle as O  # noqa: E402
import pbbem  # noqa: E402
from paper_1301_5914_b200.surfaces import baseline_config  # noqa: E402

cfg = baseline_config(3)
m = cfg.mesh
params = pbbem.PhysicalParams(eps1=cfg.eps1, eps2=cfg.eps2, kappa=cfg.kappa)
charges = pbbem.ChargeSystem(positions=cfg.charges.positions, charges=cfg.charges.charges)
mesh = pbbem.FlatMesh(vertices=m.vertices, normals=m.normals, faces=m.faces)
t = time.perf_counter()
ref = pbbem.discretize(mesh, params, charges, pbbem.SolverConfig(workers=1))
print(f"reference discretize {time.perf_counter() - t:.1f} s")
o = O.discretize(m.vertices, m.normals, m.faces, cfg.eps1, cfg.eps2, cfg.kappa, check=False)
u = np.random.default_rng(0).standard_normal(2 * m.n_vertices)
nsrc = m.n_faces * 4
rows = 512
from pbbem.solver import _apply_range  # noqa: E402

t = time.perf_counter()
r_ref = _apply_range(ref, u, 0, rows)
t_ref = time.perf_counter() - t
t = time.perf_counter()
r_or = O.rows(o, u, 0, rows)
t_or = time.perf_counter() - t
a = np.concatenate(r_ref) if isinstance(r_ref, tuple) else np.asarray(r_ref)
b = np.concatenate(r_or)
print(f"serial, rows [0,{rows}) x {nsrc} sources: reference {rows * nsrc / t_ref:.3e} pairs/s, "
      f"port {rows * nsrc / t_or:.3e} pairs/s, rel diff {np.linalg.norm(a - b) / np.linalg.norm(a):.1e}")
w = os.cpu_count()
with pbbem.make_operator(ref, pbbem.SolverConfig(workers=w)) as op:
    op(u)
    t = time.perf_counter()
    y_ref = op(u)
    t_ref = time.perf_counter() - t
with O.PoolOperator(o, w) as op:
    op(u)
    t = time.perf_counter()
    y_or = op(u)
    t_or = time.perf_counter() - t
pairs = m.n_vertices * nsrc
print(f"fork pool x{w}, full matvec ({pairs:.3e} pairs): reference {pairs / t_ref:.3e} pairs/s, "
      f"port {pairs / t_or:.3e} pairs/s, rel diff {np.linalg.norm(y_ref - y_or) / np.linalg.norm(y_ref):.1e}")
