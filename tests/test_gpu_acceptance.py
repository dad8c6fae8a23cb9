"""The reference's release-gate scenarios (ref tests/test_acceptance.py), run
through the GPU path and pinned to the numbers the reference itself printed
for them (ref pkg/test_output.txt:358-367).  Printed values carry 4-5
significant digits, so each comparison allows half a unit of the last printed
digit; iteration counts must be equal.  Criteria 6, 7 and 10 concern the host
quadrature tables, closed-form kernel checks and MSMS text round trip (covered
by tests/test_oracle_golden.py, test_host.py and test_msms.py), not the device
path.
"""
from functools import lru_cache

import numpy as np
import pytest

from paper_1301_5914_b200 import (ChargeSystem, PhysicalParams, SolverConfig, assemble_rhs,
                                  convergence_order, discretize, gmres_solve, icosahedral_sphere,
                                  make_operator, matvec_hobi, matvec_lobi, solvation_energy,
                                  surface_potential_error)
from paper_1301_5914_b200.kirkwood import SphereProblem, kirkwood_series

pytestmark = pytest.mark.gpu

BORN = (PhysicalParams(1.0, 80.0, 0.0), ChargeSystem([[0.0, 0.0, 0.0]], [1.0]), 2.0)
ECC = (PhysicalParams(1.0, 80.0, 1.0), ChargeSystem([[0.5, 0.0, 0.0]], [1.0]), 1.0)


def _close(x, printed: str):
    """x agrees with a value printed as `printed` (half a unit of its last digit)."""
    mant = printed.split("e")[0]
    decimals = len(mant.split(".")[1]) if "." in mant else 0
    exp = int(printed.split("e")[1]) if "e" in printed else 0
    return abs(x - float(printed)) <= 0.5 * 10.0 ** (exp - decimals) * (1 + 1e-9)


@lru_cache(maxsize=None)
def _run(family: str, scheme: str, level: int, workers: int = 1):
    params, charges, radius = BORN if family == "born" else ECC
    cfg = SolverConfig(scheme=scheme, workers=workers)
    prob = discretize(icosahedral_sphere(level, radius), params, charges, cfg)
    with make_operator(prob, cfg) as op:
        sol = gmres_solve(op, assemble_rhs(prob), cfg)
    ks = kirkwood_series(SphereProblem(radius=radius, params=params, charges=charges), n_terms=40)
    assert ks.converged
    e_phi = surface_potential_error(sol.phi, ks.phi(prob.colloc_pos))
    out = dict(energy=solvation_energy(prob, sol), e_phi=e_phi, iterations=sol.iterations,
               n_faces=prob.mesh.n_faces, vector=sol.vector.copy())
    prob.close()
    return out


def test_criterion_01_born_energy():
    assert _close(_run("born", "hobi", 3)["energy"], "-81.98086")


def test_criterion_02_born_trace_error():
    assert _close(_run("born", "hobi", 3)["e_phi"], "3.870e-05")
    assert _close(_run("born", "hobi", 4)["e_phi"], "1.868e-05")


def test_criterion_03_observed_orders():
    # the reference fails its own gate here (hobi 0.482 < 1.2); the GPU path
    # must reproduce the same observed orders, not a different answer
    for scheme, printed in (("hobi", "0.482"), ("lobi", "0.557")):
        lo, hi = _run("born", scheme, 2), _run("born", scheme, 4)
        order = convergence_order(lo["n_faces"], hi["n_faces"], lo["e_phi"], hi["e_phi"])
        assert _close(order, printed), (scheme, order)


def test_criterion_04_eccentric_charge():
    h3, h4 = _run("ecc", "hobi", 3), _run("ecc", "hobi", 4)
    l3, l4 = _run("ecc", "lobi", 3), _run("ecc", "lobi", 4)
    assert _close(h4["e_phi"], "4.061e-04")
    assert _close(l4["e_phi"], "1.151e-02")
    assert _close(h3["e_phi"] / h4["e_phi"], "3.79")
    assert _close(l3["e_phi"] / l4["e_phi"], "2.56")


def test_criterion_05_identity_medium():
    params = PhysicalParams(4.0, 4.0, 0.0)
    charges = ChargeSystem([[0.3, 0.1, -0.2]], [1.0])
    rng = np.random.default_rng(11)
    for scheme, apply_fn in (("hobi", matvec_hobi), ("lobi", matvec_lobi)):
        prob = discretize(icosahedral_sphere(2, 2.0), params, charges,
                          SolverConfig(scheme=scheme, workers=1))
        for _ in range(10):
            u = rng.standard_normal(prob.n_unknowns)
            assert np.array_equal(apply_fn(prob, u), u)  # reference: max |Au - u| = 0.0
        prob.close()


def test_criterion_08_split_determinism():
    ref = _run("born", "hobi", 3)["vector"]
    for w in (2, 4, 8):
        assert np.array_equal(_run("born", "hobi", 3, workers=w)["vector"], ref)


def test_criterion_09_gmres_iterations():
    its = {
        ("born", "hobi"): [6, 6, 3], ("born", "lobi"): [8, 9, 9],
        ("ecc", "hobi"): [15, 15], ("ecc", "lobi"): [16, 16],
    }
    for (family, scheme), expect in its.items():
        levels = (2, 3, 4) if family == "born" else (3, 4)
        assert [_run(family, scheme, lv)["iterations"] for lv in levels] == expect, (family, scheme)
