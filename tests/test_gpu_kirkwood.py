"""f4 on the device: kirkwood_series' Legendre sums (csrc/hobi_kirkwood.cu)
against the reference's own outputs (tests/golden/kirkwood.npz, made by
pbbem.kirkwood.kirkwood_series) and against the numpy sums of
oracle/kirkwood_host.py."""

import ctypes as C

import numpy as np
import pytest

from conftest import golden
from kirkwood_host import kirkwood_series_host
from paper_1301_5914_b200 import ChargeSystem, PhysicalParams
from paper_1301_5914_b200.kirkwood import SphereProblem, kirkwood_series

pytestmark = pytest.mark.gpu


def _problem(g, tag):
    v = g[tag + "_in"]
    e1, e2, kap, a = v[-4:]
    nq = (v.size - 4) // 4
    pos, q = v[: 3 * nq].reshape(nq, 3), v[3 * nq: 4 * nq]
    return SphereProblem(a, PhysicalParams(e1, e2, kap), ChargeSystem(pos, q)), a


@pytest.mark.parametrize("tag", ["c2", "ecc", "lap"])
def test_device_series_matches_reference(tag):
    g = golden("kirkwood")
    sph, a = _problem(g, tag)
    ks = kirkwood_series(sph, 40)
    assert ks.energy == pytest.approx(float(g[tag + "_energy"]), rel=1e-12)
    pts = a / 2.0 * g["points"]
    for name, fn in (("_phi", ks.phi), ("_dphi", ks.dphi_dn)):
        ref = g[tag + name]
        assert np.abs(fn(pts) - ref).max() <= 1e-12 * np.abs(ref).max(), name
    assert ks.converged == bool(g[tag + "_tail"][1])
    host = kirkwood_series_host(sph, 40)
    assert abs(ks.energy - host.energy) <= 1e-13 * abs(host.energy)
    assert np.abs(ks.phi(pts) - host.phi(pts)).max() <= 1e-13 * np.abs(host.phi(pts)).max()
    assert ks.phi(pts[3]) == pytest.approx(ks.phi(pts)[3], rel=0, abs=0)  # single point


def test_device_series_many_points_and_charges():
    """Config-5-sized evaluation (L7 icosphere vertices, 200 charges): the device
    sums agree with the numpy sums everywhere."""
    from paper_1301_5914_b200.mesh import icosahedral_sphere
    from paper_1301_5914_b200.surfaces import sphere_charges

    pts = icosahedral_sphere(7, 2.0).vertices
    ch = sphere_charges(200, 1.2, 77)
    sph = SphereProblem(2.0, PhysicalParams(1.0, 80.0, 0.1257), ch)
    dev = kirkwood_series(sph, 40)
    host = kirkwood_series_host(sph, 40)
    sub = pts[::97]
    for f, h in ((dev.phi, host.phi), (dev.dphi_dn, host.dphi_dn)):
        ref = h(sub)
        assert np.abs(f(pts)[::97] - ref).max() <= 1e-12 * np.abs(ref).max()
    assert dev.energy == pytest.approx(host.energy, rel=1e-12)


def test_device_series_rejects_bad_sizes():
    from paper_1301_5914_b200 import _native as N

    lib = N.load()
    z = np.zeros(3)
    assert lib.hobi_kirkwood_traces(0, N.dptr(z), 1, N.dptr(z), N.dptr(z), 1, N.dptr(z), N.dptr(z), 0,
                                    N.dptr(z), N.dptr(z)) == N.HOBI_ERR_VALUE
    assert lib.hobi_kirkwood_energy_terms(0, N.dptr(z), N.dptr(z), -1, N.dptr(z), N.dptr(z), 3,
                                          N.dptr(z)) == N.HOBI_ERR_VALUE
