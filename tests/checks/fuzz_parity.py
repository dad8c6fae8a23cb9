"""Parameter-space sweep of GPU-vs-oracle parity (seeded, for profiles/):
random star surfaces, eps1/eps2 (including eps2 < eps1 and eps2 ~ eps1),
kappa from 0 through 1e-12 to 5, vectors with a zero phi or dphi block,
HOBI and LOBI; matvec, RHS and energy relative errors per case.
Usage: python tests/checks/fuzz_parity.py [n_cases]"""
import sys
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import hobi_oracle as O
from paper_1301_5914_b200 import (PhysicalParams, SolverConfig, SurfaceSolution, assemble_rhs, discretize,
                                  matvec_hobi, matvec_lobi, solvation_energy)
from paper_1301_5914_b200.surfaces import StarShape

def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - b) / nb) if nb else float(np.linalg.norm(a))

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
worst = {"matvec": 0.0, "rhs": 0.0, "energy": 0.0, "lobi": 0.0}
print("| seed | level | N_f | eps1 | eps2 | kappa | u | matvec | RHS | energy | LOBI matvec |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for seed in range(1000, 1000 + n):
    rng = np.random.default_rng(seed)
    shape = StarShape.from_seed(float(rng.uniform(2, 60)), seed=seed, amplitude=float(rng.uniform(0.02, 0.25)))
    level = int(rng.integers(1, 4))
    mesh = shape.surface(level)
    charges = shape.interior_charges(int(rng.integers(1, 60)), seed=seed + 7)
    e1 = float(rng.uniform(0.5, 10))
    e2 = float(rng.choice([rng.uniform(1, 100), e1 * (1 + 1e-6), rng.uniform(0.2, 1.0) * e1]))
    kap = float(rng.choice([0.0, 1e-12, rng.uniform(1e-4, 0.05), rng.uniform(0.05, 1.0), rng.uniform(1, 5)]))
    prob = discretize(mesh, PhysicalParams(e1, e2, kap), charges, SolverConfig())
    o = O.discretize(mesh.vertices, mesh.normals, mesh.faces, e1, e2, kap, charges.positions, charges.charges)
    u = rng.standard_normal(prob.n_unknowns)
    kind = str(rng.choice(["mixed", "phi=0", "dphi=0"]))
    T = prob.n_collocation
    if kind == "phi=0":
        u[:T] = 0.0
    elif kind == "dphi=0":
        u[T:] = 0.0
    em = rel(matvec_hobi(prob, u), O.matvec(o, u))
    er = rel(assemble_rhs(prob), O.rhs(o))
    phi, dphi = rng.standard_normal(T), rng.standard_normal(T)
    e_ref = O.energy(o, phi, dphi)
    e_gpu = solvation_energy(prob, SurfaceSolution(phi, dphi, "hobi", 0, 0.0))
    ee = abs(e_gpu - e_ref) / max(abs(e_ref), 1e-300)
    pl = discretize(mesh, PhysicalParams(e1, e2, kap), charges, SolverConfig(scheme="lobi"))
    ol = O.discretize(mesh.vertices, mesh.normals, mesh.faces, e1, e2, kap, scheme="lobi")
    ul = rng.standard_normal(pl.n_unknowns)
    el = rel(matvec_lobi(pl, ul), O.matvec(ol, ul))
    for k, v in (("matvec", em), ("rhs", er), ("energy", ee), ("lobi", el)):
        worst[k] = max(worst[k], v)
    print(f"| {seed} | {level} | {mesh.n_faces} | {e1:.3g} | {e2:.6g} | {kap:.3g} | {kind} | {em:.1e} | {er:.1e} | {ee:.1e} | {el:.1e} |",
          flush=True)
    prob.close(); pl.close()
print()
print("worst: " + ", ".join(f"{k} {v:.2e}" for k, v in worst.items()) + " (gates: matvec 1e-10, energy 1e-8)")
