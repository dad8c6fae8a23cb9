"""Analytic Kirkwood validator against the reference's
kirkwood_series / kirkwood_centered outputs (tests/golden/kirkwood.npz): the
product's host coefficients (kirkwood_coefficients) with the numpy Legendre
sums of oracle/kirkwood_host.py; the device sums are tests/test_gpu_kirkwood.py."""

import numpy as np
import pytest

from conftest import golden
from paper_1301_5914_b200 import ChargeSystem, PhysicalParams
from kirkwood_host import kirkwood_series_host, legendre_table
from paper_1301_5914_b200.kirkwood import NotCenteredError, SphereProblem, bessel_log_derivative, kirkwood_centered


@pytest.mark.parametrize("tag", ["c2", "ecc", "lap"])
def test_series_matches_reference(tag):
    g = golden("kirkwood")
    v = g[tag + "_in"]
    e1, e2, kap, a = v[-4:]
    nq = (v.size - 4) // 4
    pos, q = v[: 3 * nq].reshape(nq, 3), v[3 * nq: 4 * nq]
    ks = kirkwood_series_host(SphereProblem(a, PhysicalParams(e1, e2, kap), ChargeSystem(pos, q)), 40)
    assert ks.energy == pytest.approx(float(g[tag + "_energy"]), rel=1e-12)
    pts = a / 2.0 * g["points"]
    for name, fn in (("_phi", ks.phi), ("_dphi", ks.dphi_dn)):
        ref = g[tag + name]
        assert np.abs(fn(pts) - ref).max() <= 1e-12 * np.abs(ref).max()
    assert ks.tail_ratio == pytest.approx(float(g[tag + "_tail"][0]), rel=1e-9, abs=1e-300)
    assert ks.converged == bool(g[tag + "_tail"][1])


def test_centered_closed_form_and_series_agree():
    g = golden("kirkwood")
    sph = SphereProblem(2.0, PhysicalParams(1.0, 80.0, 0.1257), ChargeSystem([[0, 0, 0]], [1.0]))
    e, phi, dphi = kirkwood_centered(sph)
    assert np.allclose([e, phi(np.array([0, 0, 2.0])), dphi(np.array([0, 0, 2.0]))], g["centered"],
                       rtol=1e-14, atol=0)
    ks = kirkwood_series_host(sph, 10)
    assert ks.energy == pytest.approx(e, rel=1e-12)
    with pytest.raises(NotCenteredError):
        kirkwood_centered(SphereProblem(2.0, sph.params, ChargeSystem([[0, 0, 0.5]], [1.0])))
    with pytest.raises(ValueError, match="not strictly"):
        SphereProblem(2.0, sph.params, ChargeSystem([[0, 0, 2.0]], [1.0]))


def test_special_functions():
    x = np.linspace(-1, 1, 7)
    p = legendre_table(4, x)
    assert np.allclose(p[2], 0.5 * (3 * x**2 - 1)) and np.allclose(p[4], (35 * x**4 - 30 * x**2 + 3) / 8)
    assert np.array_equal(bessel_log_derivative(3, 0.0), [-1.0, -2.0, -3.0, -4.0])
    # k_1(x) = e^{-x}(1+x)/x^2  =>  x k_1'/k_1 = -(x^2 + 2x + 2)/(1 + x)
    x0 = 0.7
    assert bessel_log_derivative(2, x0)[1] == pytest.approx(-(x0 * x0 + 2 * x0 + 2) / (1 + x0), rel=1e-14)
