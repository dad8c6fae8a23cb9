"""Capacity run: a full solve on config 5's surface one level finer (L8:
655,362 vertices, 1,310,720 curved triangles, 3.4e12 pairs per matvec) with
config 5's 10,000 charges, one GPU."""
import sys, time, json
sys.path.insert(0, '.')
from paper_1301_5914_b200 import (PhysicalParams, SolverConfig, assemble_rhs, discretize, gmres_solve,
                                  make_operator, solvation_energy)
from paper_1301_5914_b200.surfaces import baseline_config
level = int(sys.argv[1]) if len(sys.argv) > 1 else 8
t0 = time.perf_counter()
cfg = baseline_config(5, level=level)
t1 = time.perf_counter()
scfg = SolverConfig(workers=1, restart=cfg.restart, tolerance=cfg.tol)
prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, scfg)
t2 = time.perf_counter()
b = assemble_rhs(prob)
t3 = time.perf_counter()
with make_operator(prob, scfg) as op:
    sol = gmres_solve(op, b, scfg)
t4 = time.perf_counter()
e = solvation_energy(prob, sol)
t5 = time.perf_counter()
print(json.dumps({"config": cfg.name, "n_vertices": cfg.mesh.n_vertices, "n_faces": cfg.mesh.n_faces,
                  "n_charges": len(cfg.charges), "pairs_per_matvec": cfg.mesh.n_vertices * cfg.mesh.n_faces * 4.0,
                  "surface_s": t1 - t0, "discretize_s": t2 - t1, "rhs_s": t3 - t2, "gmres_s": t4 - t3,
                  "energy_s": t5 - t4, "iterations": sol.iterations, "matvecs": sol.matvecs,
                  "residual": sol.residual, "energy_kcal_mol": e}))
