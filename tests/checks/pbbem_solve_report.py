"""Measured errors of the GPU solve against the pbbem solve fixtures
(tests/golden/c{3,4}_solve.npz, made by tests/golden/make_scale_golden.py):
matvec, RHS, GMRES counts, potentials and energy.  Needs a B200.

    python tests/checks/pbbem_solve_report.py 3 4 3lobi 4lobi
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from scale_hash import input_hash  # noqa: E402

from paper_1301_5914_b200 import (PhysicalParams, SolverConfig, assemble_rhs, discretize, gmres_solve,  # noqa: E402
                                  make_operator, matvec_hobi, matvec_lobi, solvation_energy)
from paper_1301_5914_b200.surfaces import baseline_config  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


for arg in sys.argv[1:] or ["3", "4"]:
    index, scheme = int(arg[0]), ("lobi" if arg.endswith("lobi") else "hobi")
    tag = "" if scheme == "hobi" else "_lobi"
    fx = dict(np.load(os.path.join(ROOT, "tests", "golden", f"c{index}_solve{tag}.npz")))
    cfg = baseline_config(index)
    assert input_hash(cfg) == str(fx["input_sha256"])
    scfg = SolverConfig(workers=1, restart=cfg.restart, tolerance=cfg.tol, scheme=scheme)
    prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, scfg)
    u = np.random.default_rng(int(fx["u_seed"])).standard_normal(2 * prob.n_collocation)
    e_mv = rel((matvec_hobi if scheme == "hobi" else matvec_lobi)(prob, u), fx["Au"])
    b = assemble_rhs(prob)
    t0 = time.perf_counter()
    with make_operator(prob, scfg) as op:
        sol = gmres_solve(op, b, scfg)
    e = solvation_energy(prob, sol)
    dt = time.perf_counter() - t0
    print(f"config {index} {scheme}: matvec {e_mv:.2e}, rhs {rel(b, fx['rhs']):.2e}, "
          f"iterations {sol.iterations} (pbbem {int(fx['iterations'])}), matvecs {sol.matvecs} "
          f"(pbbem {int(fx['matvecs'])}), phi {rel(sol.phi, fx['phi']):.2e}, "
          f"dphi {rel(sol.dphi_dn, fx['dphi']):.2e}, energy {e!r} vs {float(fx['energy'])!r} "
          f"({abs(e - float(fx['energy'])) / abs(float(fx['energy'])):.1e}), "
          f"GPU solve+energy {dt:.3f} s vs pbbem solve {float(fx['reference_solve_seconds']):.0f} s on "
          f"{int(fx['reference_workers'])} workers", flush=True)
    prob.close()
