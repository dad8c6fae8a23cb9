"""Targeted accuracy check of the sweep at small screening (kappa*R << 1),
where K1 = W1 (e^{-kr} - 1)/r needs expm1-grade relative accuracy: u with a
zero phi block makes the first output block a pure K1 sum; er ~ 1 removes
the K2 term that would otherwise dominate.  GPU vs oracle, relative L2.
The energy column is the error relative to the energy's own magnitude scale
0.5 * 4 pi * kcal * sum_k |q_k phi_reac(x_k)|: with net-neutral charges and
kr << 1 the leading O(kappa) parts of the per-charge potentials cancel in the
sum, so the energy itself is ill-conditioned (reference and device alike).
"""
import sys
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import hobi_oracle as O
from paper_1301_5914_b200 import (PhysicalParams, SolverConfig, SurfaceSolution, discretize,
                                  matvec_hobi, solvation_energy)
from paper_1301_5914_b200.surfaces import StarShape

shape = StarShape.from_seed(12.0, seed=5)
mesh = shape.surface(2)
charges = shape.interior_charges(20, seed=6)
rng = np.random.default_rng(0)
worst = 0.0
print("| kappa | eps2/eps1 | u | matvec block 1 | matvec block 2 | energy (vs its scale) |")
print("|---|---|---|---|---|---|")
for kap in (1e-12, 1e-9, 1e-6, 1e-3):
    for e2 in (40.0, 1.0 + 1e-6, 1.0):
        prob = discretize(mesh, PhysicalParams(1.0, e2, kap), charges, SolverConfig())
        o = O.discretize(mesh.vertices, mesh.normals, mesh.faces, 1.0, e2, kap, charges.positions, charges.charges)
        T = prob.n_collocation
        for kind in ("phi=0", "mixed"):
            u = rng.standard_normal(2 * T)
            if kind == "phi=0":
                u[:T] = 0.0
            g, r = matvec_hobi(prob, u), O.matvec(o, u)
            e1 = np.linalg.norm(g[:T] - r[:T]) / max(np.linalg.norm(r[:T]), 1e-300)
            e2b = np.linalg.norm(g[T:] - r[T:]) / max(np.linalg.norm(r[T:]), 1e-300)
            phi, dphi = u[:T].copy(), u[T:].copy()
            er_ = O.energy(o, phi, dphi)
            eg = solvation_energy(prob, SurfaceSolution(phi, dphi, "hobi", 0, 0.0))
            wp, wd = O.source_weights(o, u)
            src, snrm = o.reg_pos.reshape(-1, 3), o.reg_nrm.reshape(-1, 3)
            scale = 0.0
            for pos, qk in zip(o.qpos, o.q):
                k1, k2, _, _ = O.k1234(pos[None, :] - src, snrm, snrm, o.eps1, o.eps2, o.kappa)
                scale += abs(qk * float((k1 * wd + k2 * wp).sum()))
            scale *= 0.5 * O.FOUR_PI * O.KCAL
            ee = abs(eg - er_) / max(scale, 1e-300)
            worst = max(worst, e1, e2b, ee)
            print(f"| {kap:g} | {e2:.7g} | {kind} | {e1:.1e} | {e2b:.1e} | {ee:.1e} |", flush=True)
        prob.close()
print(f"\nworst relative error {worst:.2e}")
