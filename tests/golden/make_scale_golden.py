"""Reference-generated fixtures at the BASELINE sizes (configs 3, 4, 5).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_scale_golden.py c3 c4rows c5rows
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_scale_golden.py c4solve
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_scale_golden.py c4lobirows c5lobirows

Every output array comes from the unmodified reference package ``pbbem``
(``solver.discretize``, ``solver._apply_range`` -- the row-range unit its fork
pool runs, ``solver.py:278-367`` -- ``kernels.source_terms_at``, and for config
3 the full ``make_operator`` / ``assemble_rhs`` / ``gmres_solve`` /
``solvation_energy`` chain, ``solver.py:393-402,475-614``).  The meshes are far
too large to commit, so each fixture stores a SHA-256 of the mesh and charge
arrays that ``paper_1301_5914_b200.surfaces.baseline_config`` generates; the
GPU tests regenerate the mesh, check the hash, and only then compare.

Row blocks (configs 4 and 5): 5 blocks of 24 rows spread over [0, N_v) of both
equation blocks for a seeded u = default_rng(0).standard_normal(2 N_v), plus the
right-hand side at the same rows.  Config 5's full right-hand side would need
~39 GB in the reference (kernels.py:166), so only its rows are taken.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from pbbem import kernels as rk  # noqa: E402
from pbbem import solver as rs  # noqa: E402
from pbbem.mesh import ChargeSystem as RCharges  # noqa: E402
from pbbem.mesh import FlatMesh as RMesh  # noqa: E402

from paper_1301_5914_b200.surfaces import baseline_config  # noqa: E402

sys.path.insert(0, HERE)
from scale_hash import input_hash  # noqa: E402

ROWS = 24


def row_blocks(nv: int) -> list[int]:
    return [0, nv // 5, nv // 2 + 7, (4 * nv) // 5 - 3, nv - ROWS]


_PROB = None


def _rows_task(args):
    u, lo = args
    return rs._apply_range(_PROB, u, lo, lo + ROWS)


def _problem(cfg, workers, scheme="hobi"):
    params = rk.PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa)
    scfg = rs.SolverConfig(scheme=scheme, workers=workers, restart=cfg.restart, tolerance=cfg.tol)
    t0 = time.time()
    prob = rs.discretize(RMesh(vertices=cfg.mesh.vertices, normals=cfg.mesh.normals, faces=cfg.mesh.faces),
                         params, RCharges(positions=cfg.charges.positions, charges=cfg.charges.charges), scfg)
    print(f"  discretize {time.time() - t0:.0f} s", flush=True)
    return prob, scfg


def rows_case(index, workers=5, scheme="hobi"):
    global _PROB
    t0 = time.time()
    cfg = baseline_config(index)
    print(f"c{index}rows ({scheme}): N_v={cfg.mesh.n_vertices} N_f={cfg.mesh.n_faces}", flush=True)
    prob, _ = _problem(cfg, 1, scheme)
    _PROB = prob
    nv = prob.n_collocation  # N_v for hobi, N_f for lobi
    u = np.random.default_rng(0).standard_normal(2 * nv)
    starts = row_blocks(nv)
    with mp.get_context("fork").Pool(min(workers, len(starts))) as pool:
        parts = pool.map(_rows_task, [(u, lo) for lo in starts])
    idx = np.concatenate([np.arange(lo, lo + ROWS) for lo in starts])
    s1, s2 = rk.source_terms_at(prob.colloc_pos[idx], prob.colloc_nrm[idx], prob.charges)
    out = dict(input_sha256=np.array(input_hash(cfg)), config=np.array(index), u_seed=np.array(0),
               rows=idx, Au_phi=np.concatenate([p[0] for p in parts]),
               Au_dphi=np.concatenate([p[1] for p in parts]),
               rhs_phi=s1 / cfg.eps1, rhs_dphi=s2 / cfg.eps1,
               params=np.array([cfg.eps1, cfg.eps2, cfg.kappa]), scheme=np.array(scheme),
               generated_by=np.array("pbbem solver._apply_range + kernels.source_terms_at"))
    tag = "" if scheme == "hobi" else "_" + scheme
    np.savez_compressed(os.path.join(HERE, f"c{index}_rows{tag}.npz"), **out)
    print(f"c{index}rows ({scheme}): {time.time() - t0:.0f} s", flush=True)


def solve_case(index, workers=8, name=None, scheme="hobi"):
    t0 = time.time()
    cfg = baseline_config(index)
    nv = cfg.mesh.n_vertices
    print(f"c{index}solve ({scheme}): N_v={nv} N_f={cfg.mesh.n_faces} workers={workers}", flush=True)
    prob, scfg = _problem(cfg, workers, scheme)
    u = np.random.default_rng(0).standard_normal(2 * prob.n_collocation)
    count = [0]
    with rs.make_operator(prob, scfg) as op:
        t1 = time.time()
        Au = op(u)
        print(f"  matvec {time.time() - t1:.0f} s", flush=True)
        rhs = rs.assemble_rhs(prob)

        def apply(v):
            count[0] += 1
            t2 = time.time()
            y = op(v)
            print(f"  matvec {count[0]} {time.time() - t2:.0f} s", flush=True)
            return y

        t1 = time.time()
        sol = rs.gmres_solve(apply, rhs, scfg)
        solve_s = time.time() - t1
    energy = rs.solvation_energy(prob, sol)
    out = dict(input_sha256=np.array(input_hash(cfg)), config=np.array(index), u_seed=np.array(0),
               Au=Au, rhs=rhs, phi=sol.phi, dphi=sol.dphi_dn, iterations=np.array(sol.iterations),
               residual=np.array(sol.residual), matvecs=np.array(count[0]), restart=np.array(cfg.restart),
               tol=np.array(cfg.tol), energy=np.array(energy),
               params=np.array([cfg.eps1, cfg.eps2, cfg.kappa]), scheme=np.array(scheme),
               reference_solve_seconds=np.array(solve_s), reference_workers=np.array(workers),
               generated_by=np.array("pbbem make_operator/assemble_rhs/gmres_solve/solvation_energy"))
    tag = "" if scheme == "hobi" else "_" + scheme
    np.savez_compressed(os.path.join(HERE, name or f"c{index}_solve{tag}.npz"), **out)
    print(f"c{index}solve: its={sol.iterations} matvecs={count[0]} E={energy!r} "
          f"solve {solve_s:.0f} s, total {time.time() - t0:.0f} s", flush=True)


def main():
    jobs = {"c3": lambda: solve_case(3), "c4rows": lambda: rows_case(4), "c5rows": lambda: rows_case(5),
            "c4lobirows": lambda: rows_case(4, scheme="lobi"), "c5lobirows": lambda: rows_case(5, scheme="lobi"),
            "c4solve": lambda: solve_case(4, workers=int(os.environ.get("WORKERS", "6"))),
            "c3lobisolve": lambda: solve_case(3, workers=int(os.environ.get("WORKERS", "6")), scheme="lobi"),
            "c4lobisolve": lambda: solve_case(4, workers=int(os.environ.get("WORKERS", "6")), scheme="lobi")}
    for name in sys.argv[1:] or ["c3", "c4rows", "c5rows"]:
        jobs[name]()


if __name__ == "__main__":
    main()
