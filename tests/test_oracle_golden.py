"""Pin the oracle (oracle/hobi_oracle.py) against the reference's own outputs.

The golden .npz files were produced by running the unmodified reference
package (tests/golden/make_golden.py); the frozen numbers are the reference
test-suite's known answers (pbbem tests/test_solver.py:375-403).  CPU only.
"""

import numpy as np
import pytest

import hobi_oracle as O
from conftest import golden, rel_l2


def _disc(g, scheme="hobi", charges=True):
    e1, e2, k = g["params"]
    if charges:
        return O.discretize(g["vertices"], g["normals"], g["faces"], e1, e2, k, g["qpos"], g["q"],
                            scheme=scheme)
    return O.discretize(g["vertices"], g["normals"], g["faces"], e1, e2, k, scheme=scheme)


@pytest.mark.parametrize("name", ["sphere_l1_mixed", "star_l2", "uv_sphere"])
def test_oracle_caches_bit_exact(name):
    g = golden(name)
    p = _disc(g)
    for key in ("reg_pos", "reg_nrm", "reg_w", "duf_pos", "duf_nrm", "duf_w", "reg_bary", "duf_bary"):
        assert np.array_equal(getattr(p, key), g[key]), key
    for key in ("pair_vertex", "pair_face", "pair_gverts", "pair_starts"):
        assert np.array_equal(getattr(p, key), g[key]), key


@pytest.mark.parametrize("name", ["sphere_l1_mixed", "star_l2", "star_l3", "c1", "c2", "uv_sphere"])
def test_oracle_matvec_and_rhs(name):
    g = golden(name)
    p = _disc(g)
    assert rel_l2(O.matvec(p, g["u"]), g["Au"]) <= 1e-14
    assert rel_l2(O.rhs(p), g["rhs"]) <= 1e-15


@pytest.mark.parametrize("name", ["star_l2", "c1", "uv_sphere"])
def test_oracle_solve_and_energy(name):
    g = golden(name)
    p = _disc(g)
    phi, dphi, its, rel, nmv = O.solve(p, restart=int(g["restart"]), workers=1)
    assert its == int(g["iterations"]) and nmv == int(g["matvecs"])
    assert rel_l2(phi, g["phi"]) <= 1e-12 and rel_l2(dphi, g["dphi"]) <= 1e-12
    e = O.energy(p, phi, dphi)
    assert abs(e - float(g["energy"])) <= 1e-12 * abs(float(g["energy"]))


def test_oracle_frozen_born_energies():
    """pbbem tests/test_solver.py:375-403 known answers, both schemes."""
    from paper_1301_5914_b200.mesh import icosahedral_sphere

    m = icosahedral_sphere(2, 2.0)
    for scheme, ref in (("hobi", -81.98131581725495), ("lobi", -86.3199784371863)):
        p = O.discretize(m.vertices, m.normals, m.faces, 1.0, 80.0, 0.0, [[0, 0, 0]], [1.0],
                         scheme=scheme)
        phi, dphi, its, _, _ = O.solve(p, workers=1)
        assert O.energy(p, phi, dphi) == pytest.approx(ref, rel=1e-9)


def test_oracle_identity_medium():
    g = golden("star_l2")
    rng = np.random.default_rng(0)
    for scheme in ("hobi", "lobi"):
        p = O.discretize(g["vertices"], g["normals"], g["faces"], 3.0, 3.0, 0.0, scheme=scheme)
        u = rng.standard_normal(2 * p.n_colloc)
        assert np.abs(O.matvec(p, u) - u).max() == 0.0


def test_oracle_lobi_against_naive_loop():
    """LOBI blocked sweep vs an explicit double loop (pbbem test_solver.py:168-197)."""
    from paper_1301_5914_b200.mesh import icosahedral_sphere

    m = icosahedral_sphere(0)
    e1, e2, kap = 2.0, 80.0, 0.5
    p = O.discretize(m.vertices, m.normals, m.faces, e1, e2, kap, scheme="lobi")
    t = p.n_colloc
    er = e2 / e1
    u = np.random.default_rng(1).standard_normal(2 * t)
    exp = np.empty(2 * t)
    for i in range(t):
        o1 = 0.5 * (1.0 + er) * u[i]
        o2 = 0.5 * (1.0 + 1.0 / er) * u[t + i]
        for j in range(t):
            if j == i:
                continue
            k1, k2, k3, k4 = O.k1234(p.colloc_pos[i] - p.colloc_pos[j], p.colloc_nrm[i],
                                     p.colloc_nrm[j], e1, e2, kap)
            o1 -= (k1 * u[t + j] + k2 * u[j]) * p.area[j]
            o2 -= (k3 * u[t + j] + k4 * u[j]) * p.area[j]
        exp[i], exp[t + i] = o1, o2
    assert np.abs(O.matvec(p, u) - exp).max() <= 1e-13 * np.abs(exp).max()


def test_oracle_kernels_match_reference():
    g = golden("kernels")
    for tag in "abcd":
        e1, e2, kap = g["params_" + tag]
        got = np.stack(O.k1234(g["d"], g["nx"], g["ny"], e1, e2, kap))
        assert np.array_equal(got, g["K_" + tag]) or np.abs(got - g["K_" + tag]).max() <= 1e-15 * np.abs(
            g["K_" + tag]).max()


def test_oracle_degenerate_face_message():
    g = golden("degenerate")
    with pytest.raises(O.OracleGeometryError) as info:
        O.discretize(g["vertices"], g["normals"], g["faces"], 1.0, 80.0, 0.0, check=False)
    assert str(g["message"]).endswith(str(info.value))


def test_oracle_row_split_bitwise():
    g = golden("star_l3")
    p = _disc(g, charges=False)
    u = g["u"]
    full = O.matvec(p, u)
    T = p.n_colloc
    for w in (2, 5):
        parts = [O.rows(p, u, lo, hi) for lo, hi in O.partition(T, w)]
        got = np.concatenate([np.concatenate([a for a, _ in parts]), np.concatenate([b for _, b in parts])])
        assert np.array_equal(got, full)


@pytest.mark.parametrize("name", ["star_l1_duffy6", "star_l2_rule9"])
def test_oracle_quadrature_variants(name):
    g = golden(name)
    rule = (g["rule_points"], g["rule_weights"]) if "rule_points" in g else None
    p = O.discretize(g["vertices"], g["normals"], g["faces"], *g["params"], g["qpos"], g["q"],
                     duffy_n=int(g["duffy"]), rule=rule)
    for key in ("reg_pos", "reg_nrm", "reg_w", "duf_pos", "duf_nrm", "duf_w"):
        assert np.array_equal(getattr(p, key), g[key]), key
    assert rel_l2(O.matvec(p, g["u"]), g["Au"]) <= 1e-14


def test_oracle_lobi_solve():
    g = golden("star_l2_lobi")
    p = _disc(g, scheme="lobi")
    assert rel_l2(O.matvec(p, g["u"]), g["Au"]) <= 1e-14
    phi, dphi, its, _, nmv = O.solve(p, restart=int(g["restart"]), workers=1)
    assert its == int(g["iterations"]) and nmv == int(g["matvecs"])
    assert abs(O.energy(p, phi, dphi) - float(g["energy"])) <= 1e-12 * abs(float(g["energy"]))
