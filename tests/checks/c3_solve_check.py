"""One-off parity evidence at BASELINE config 3 (L5 star surface, 20,480
curved triangles, 500 charges, restart 20, tol 1e-6; `python
tests/checks/c3_solve_check.py 4` runs config 4, about an hour of oracle time): the full GPU solve
through the public API against a full oracle solve (the reference algorithm
restated in numpy, fork pool over all host cores) on the same seeded inputs —
GMRES iteration and matvec counts, surface potential, normal derivative and
solvation energy (north-star gate: 1e-8 relative at equal tolerance)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'oracle')
import hobi_oracle as O  # noqa: E402
from paper_1301_5914_b200 import PhysicalParams, SolverConfig, solvation_energy, solve  # noqa: E402
from paper_1301_5914_b200.surfaces import baseline_config  # noqa: E402

cfg = baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
scheme = sys.argv[2] if len(sys.argv) > 2 else "hobi"  # "lobi": the flat one-point scheme (f1)
m = cfg.mesh
t0 = time.time()
prob, sol = solve(m, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges,
                  SolverConfig(workers=1, restart=cfg.restart, tolerance=cfg.tol, scheme=scheme))
e_gpu = solvation_energy(prob, sol)
t_gpu = time.time() - t0
print(f"scheme {scheme}: GPU solve: {sol.iterations} its, residual {sol.residual:.3e}, E {e_gpu:.12f} kcal/mol, {t_gpu:.2f} s",
      flush=True)
t0 = time.time()
o = O.discretize(m.vertices, m.normals, m.faces, cfg.eps1, cfg.eps2, cfg.kappa,
                 cfg.charges.positions, cfg.charges.charges, scheme=scheme, check=False)
workers = os.cpu_count() or 1
phi, dphi, its, rel, nmv = O.solve(o, tol=cfg.tol, restart=cfg.restart, workers=workers)
e_ref = O.energy(o, phi, dphi)
t_ref = time.time() - t0
print(f"oracle solve ({workers} workers): {its} its, {nmv} matvecs, residual {rel:.3e}, E {e_ref:.12f} kcal/mol, "
      f"{t_ref:.1f} s", flush=True)
ep = np.linalg.norm(sol.phi - phi) / np.linalg.norm(phi)
ed = np.linalg.norm(sol.dphi_dn - dphi) / np.linalg.norm(dphi)
ee = abs(e_gpu - e_ref) / abs(e_ref)
print(f"iterations {sol.iterations} vs {its}; phi rel L2 {ep:.2e}, dphi/dn rel L2 {ed:.2e}, energy rel {ee:.2e} "
      f"(gate 1e-8); oracle/GPU wall time {t_ref / t_gpu:.0f}x")
assert sol.iterations == its and max(ep, ed, ee) <= 1e-8
