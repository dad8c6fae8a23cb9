"""Scratch: reproduce bench.py's sequence and trace the GMRES solve timing."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_1301_5914_b200 import _native as N, discretize, PhysicalParams, SolverConfig, assemble_rhs, make_operator, gmres_solve, solvation_energy
from paper_1301_5914_b200.surfaces import baseline_config
lib = N.load()
cfg = baseline_config(4)
scfg = SolverConfig(workers=1, restart=cfg.restart, tolerance=cfg.tol)
prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, scfg)
h = prob.handle
u = np.random.default_rng(0).standard_normal(prob.n_unknowns); out = np.empty_like(u)
ms = np.zeros(10)
N.check(lib.hobi_bench(h, N.dptr(u), N.dptr(out), 5, 0, 1, N.dptr(ms)))
N.check(lib.hobi_bench(h, N.dptr(u), N.dptr(out), 5, 1, 1, N.dptr(ms)))
for rep in range(4):
    t0 = time.perf_counter(); b = assemble_rhs(prob); t1 = time.perf_counter()
    with make_operator(prob, scfg) as op:
        sol = gmres_solve(op, b, scfg)
    t2 = time.perf_counter(); e = solvation_energy(prob, sol); t3 = time.perf_counter()
    print(f"rep {rep}: rhs {t1-t0:.4f} gmres {t2-t1:.4f} energy {t3-t2:.4f}", flush=True)
