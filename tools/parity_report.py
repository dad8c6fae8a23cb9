"""Parity summary against the reference goldens (measured errors, for profiles/)."""
import os, sys
import numpy as np
sys.path.insert(0, '.')
from paper_1301_5914_b200 import (ChargeSystem, FlatMesh, PhysicalParams, SolverConfig, discretize, matvec_hobi,
                                  matvec_lobi, assemble_rhs, make_operator, gmres_solve, solvation_energy, TriangleRule)

def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))

print("| golden | N_v | N_f | caches | matvec rel L2 | RHS rel L2 | its (ref) | matvecs (ref) | phi rel L2 | dphi rel L2 | E rel diff |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for name in ("sphere_l1_mixed", "star_l2", "star_l3", "c1", "c2", "uv_sphere", "star_l1_duffy6", "star_l2_rule9", "star_l2_lobi"):
    g = dict(np.load(os.path.join("tests", "golden", name + ".npz")))
    scheme = str(g.get("scheme", "hobi"))
    kw = {"duffy_points": int(g.get("duffy", 4))}
    if "rule_points" in g:
        kw["regular_rule"] = TriangleRule(g["rule_points"], g["rule_weights"], "custom", int(g["rule_degree"]))
    restart = int(g["restart"]) if "restart" in g else 100
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    cfg = SolverConfig(scheme=scheme, workers=1, restart=restart, **kw)
    prob = discretize(mesh, PhysicalParams(*g["params"]), ChargeSystem(g["qpos"], g["q"]), cfg)
    caches = "-"
    if "reg_pos" in g:
        caches = "bit-exact" if all(np.array_equal(getattr(prob, k), g[k]) for k in
                                    ("reg_pos", "reg_nrm", "reg_w", "duf_pos", "duf_nrm", "duf_w")) else "DIFF"
    mv = (matvec_hobi if scheme == "hobi" else matvec_lobi)(prob, g["u"])
    row = [name, str(prob.n_collocation if scheme == "hobi" else mesh.n_vertices), str(mesh.n_faces), caches,
           f"{rel(mv, g['Au']):.1e}", f"{rel(assemble_rhs(prob), g['rhs']):.1e}"]
    if "phi" in g:
        with make_operator(prob, cfg) as op:
            sol = gmres_solve(op, assemble_rhs(prob), cfg)
        e = solvation_energy(prob, sol)
        row += [f"{sol.iterations} ({int(g['iterations'])})", f"{sol.matvecs} ({int(g['matvecs'])})",
                f"{rel(sol.phi, g['phi']):.1e}", f"{rel(sol.dphi_dn, g['dphi']):.1e}",
                f"{abs(e - float(g['energy'])) / abs(float(g['energy'])):.1e}"]
    else:
        row += ["-"] * 5
    print("| " + " | ".join(row) + " |", flush=True)
