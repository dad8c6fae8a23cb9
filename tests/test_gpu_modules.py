"""GPU parity of the function-level module surfaces (``geometry``, ``kernels``)
the reference exposes beside its solver API (pbbem/geometry.py, kernels.py):
the same device functions the precompute runs, called through
``hobi_geometry_*`` / ``hobi_kernel_values`` / ``hobi_source_terms``, against
the reference-made goldens (bit-exact for geometry) and the numpy oracle.
"""

import os
import sys

import numpy as np
import pytest

from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1301_5914_b200")
from paper_1301_5914_b200 import ChargeSystem, FlatMesh, PhysicalParams, icosahedral_sphere  # noqa: E402
from paper_1301_5914_b200 import geometry as G  # noqa: E402
from paper_1301_5914_b200 import kernels as K  # noqa: E402
from paper_1301_5914_b200 import _native as N  # noqa: E402
from paper_1301_5914_b200.quadrature import duffy_rule, gauss_radau_rule, integrate_element  # noqa: E402

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import hobi_oracle as O  # noqa: E402


def _triples(g):
    v, n, f = g["vertices"], g["normals"], g["faces"]
    return v[f], n[f]  # (nf, 3, 3) each


def test_frames_at_reproduces_reference_caches_bitwise():
    """nodes_from_vertex_data + frames_at (geometry.py:261-302, 342-359) through
    the module functions = the reference's regular-rule caches, bit for bit."""
    g = golden("star_l2")
    vp, vn = _triples(g)
    pos, nrm, bad, _ = G.nodes_for_triangles(vp, vn)
    assert bad == -1
    rule = gauss_radau_rule()
    fp, fn, jac = G.frames_at(pos, nrm, rule.points)
    assert np.array_equal(fp, g["reg_pos"])
    assert np.array_equal(fn, g["reg_nrm"])
    assert np.array_equal(jac * rule.weights[None, :], g["reg_w"])


def test_nodes_match_oracle_bitwise_and_keep_vertices():
    g = golden("star_l2")
    vp, vn = _triples(g)
    pos, nrm, _, _ = G.nodes_for_triangles(vp, vn)
    op, on, code = O.curved_nodes(vp[:, 0], vn[:, 0], vp[:, 1], vn[:, 1], vp[:, 2], vn[:, 2])
    assert not code.any()
    assert np.array_equal(pos, op) and np.array_equal(nrm, on)
    one_p, one_n = G.nodes_from_vertex_data(vp[7, 0], vn[7, 0], vp[7, 1], vn[7, 1], vp[7, 2], vn[7, 2])
    assert np.array_equal(one_p, pos[7]) and np.array_equal(one_n, nrm[7])
    for local, k in zip(G.VERTEX_LOCAL, range(3)):  # vertex nodes keep the inputs bitwise
        assert np.array_equal(one_p[local], vp[7, k]) and np.array_equal(one_n[local], vn[7, k])


def test_fit_arc_endpoints_tangents_and_errors():
    """fit_arc (geometry.py:46-84): interpolates the endpoints, tangents are
    orthogonal to the endpoint normals; the three degenerate inputs raise with
    the reference's messages."""
    p0, p1 = np.array([1.0, 0.0, 0.0]), np.array([0.0, 1.0, 0.0])
    arc = G.fit_arc(p0, p0, p1, p1)  # quarter of the unit circle
    assert np.array_equal(G.arc_point(arc, 0.0), p0)
    assert np.allclose(G.arc_point(arc, 1.0), p1, atol=1e-15)
    assert abs(np.dot(G.arc_velocity(arc, 0.0), p0)) < 1e-15
    assert abs(np.dot(G.arc_velocity(arc, 1.0), p1)) < 1e-14
    mid = G.arc_point(arc, 0.5)
    assert abs(np.linalg.norm(mid) - 1.0) < 2e-3  # fourth-order accurate circle
    n, straight = G.arc_normal(arc, 0.5, mid)
    assert not straight and np.allclose(n, mid / np.linalg.norm(mid), atol=1e-3)
    with pytest.raises(G.DegenerateArcError, match="arc endpoints coincide"):
        G.fit_arc(p0, p0, p0, p0)
    with pytest.raises(G.DegenerateArcError, match="nearly parallel to the chord"):
        G.fit_arc([0, 0, 0], [0, 0, 1.0], [0, 0, 1.0], [0, 1.0, 0])
    line = G.fit_arc([0, 0, 0], [0, 0, 1.0], [1.0, 0, 0], [0, 0, 1.0])
    ref = np.array([0.0, 0.0, 1.0])
    n, straight = G.arc_normal(line, 0.3, ref)
    assert straight and np.array_equal(n, ref)


def test_degenerate_face_message_matches_reference():
    g = golden("degenerate")
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    kind, _, message = str(g["message"]).partition(": ")  # "DegenerateArcError: face 0: ..."
    assert kind == "DegenerateArcError"
    face = int(message.split(":")[0].split()[1])
    with pytest.raises(G.DegenerateArcError) as info:
        G.build_curved_element(mesh, face)
    assert str(info.value) == message
    with pytest.raises(IndexError):
        G.build_curved_element(mesh, mesh.n_faces)


def test_element_frame_and_integrate_element():
    """element_frame (geometry.py:323-339) agrees with frames_at; the curved
    level-2 sphere area converges on 4 pi r^2 (ref tests/test_quadrature.py)."""
    mesh = icosahedral_sphere(2, radius=2.0)
    elem = G.build_curved_element(mesh, 5)
    rule = gauss_radau_rule()
    fp, fn, jac = G.frames_at(elem.nodes[None], elem.node_normals[None], rule.points)
    many = G.element_frames(elem, rule.points)
    assert all(np.array_equal(many[q].position, fp[0, q]) and many[q].jacobian == jac[0, q] for q in range(4))
    for q, (r, s) in enumerate(rule.points):
        fr = G.element_frame(elem, r, s)
        # one point at a time the basis row comes from a (1, 10) product instead of
        # the (m, 10) one (entries differ by ~4e-15) -- as it does in the reference
        assert np.allclose(fr.position, fp[0, q], rtol=0, atol=1e-13)
        assert np.allclose(fr.normal, fn[0, q], rtol=0, atol=1e-13)
        assert fr.jacobian == pytest.approx(jac[0, q], rel=1e-13)
        cr = np.cross(fr.d_dr, fr.d_ds)
        assert abs(np.linalg.norm(cr) - fr.jacobian) <= 1e-15 * fr.jacobian
    area = sum(integrate_element(G.build_curved_element(mesh, f), lambda fr: 1.0, rule)
               for f in range(mesh.n_faces))
    assert abs(area - 16.0 * np.pi) / (16.0 * np.pi) < 1e-5
    flat = G.CurvedElement(nodes=np.c_[G.REFERENCE_NODES, np.zeros(10)],
                           node_normals=np.tile([0.0, 0.0, 1.0], (10, 1)), vertex_ids=(0, 1, 2))
    assert integrate_element(flat, lambda fr: 1.0, duffy_rule(4)) == pytest.approx(0.5, abs=1e-15)
    with pytest.raises(G.DegenerateElementError):
        G.element_frame(G.CurvedElement(nodes=np.zeros((10, 3)), node_normals=flat.node_normals,
                                        vertex_ids=(0, 1, 2)), 0.2, 0.2)


def test_kernel_values_module_matches_reference_table():
    """kernels.kernel_values_d / kernel_values / kernel_block against the
    reference-made table (kernels.py:88-141), broadcasting included."""
    g = golden("kernels")
    for tag in "abcd":
        e1, e2, kap = g[f"params_{tag}"]
        prm = PhysicalParams(e1, e2, kap)
        k = np.stack(K.kernel_values_d(g["d"], g["nx"], g["ny"], prm))
        raw = np.empty_like(k)  # the C entry test_gpu_parity.py pins to the reference table
        N.check(N.load().hobi_kernel_values(0, N.dptr(N.f64(g["d"])), N.dptr(N.f64(g["nx"])),
                                            N.dptr(N.f64(g["ny"])), k.shape[1], e1, e2, kap, N.dptr(raw)))
        assert np.array_equal(k, raw)
        ref = g[f"K_{tag}"]
        for i, tol in ((0, 1e-14), (1, 1e-13), (2, 1e-13)):
            assert (rel_l2(k[i], ref[i]) <= tol) if ref[i].any() else (not k[i].any())
    prm = PhysicalParams(2.0, 80.0, 0.3)
    x = g["d"][:6].reshape(2, 3, 3)
    kb = K.kernel_values(x, g["nx"][0], np.zeros(3) - 5.0, g["ny"][0], prm)  # broadcast (2,3,3) with (3,)
    assert all(a.shape == (2, 3) for a in kb)
    one = K.kernel_block(x[1, 2], g["nx"][0], np.zeros(3) - 5.0, g["ny"][0], prm)
    assert one == tuple(float(a[1, 2]) for a in kb)  # same elementwise operations, bitwise
    with pytest.raises(K.SingularityError):
        K.kernel_block([1, 2, 3], g["nx"][0], [1, 2, 3], g["ny"][0], prm)
    zero = K.kernel_values_d(g["d"][:5], g["nx"][:5], g["ny"][:5], PhysicalParams(4.0, 4.0, 0.0))
    assert all(not a.any() for a in zero)  # identity medium: every kernel vanishes


def test_source_terms_module():
    """kernels.source_terms_at / source_terms (kernels.py:144-178)."""
    g = golden("star_l2")
    charges = ChargeSystem(g["qpos"], g["q"])
    s1, s2 = K.source_terms_at(g["vertices"], g["normals"], charges)
    d = g["vertices"][:, None, :] - g["qpos"][None, :, :]
    r = np.linalg.norm(d, axis=2)
    ref1 = (g["q"] / (K.FOUR_PI * r)).sum(axis=1)
    ref2 = (-g["q"] * np.einsum("mki,mi->mk", d, g["normals"]) / (K.FOUR_PI * r**3)).sum(axis=1)
    assert rel_l2(s1, ref1) <= 1e-14 and rel_l2(s2, ref2) <= 1e-13
    e1 = float(g["params"][0])
    assert rel_l2(np.concatenate([s1, s2]) / e1, g["rhs"]) <= 1e-13  # solver.py:393-402
    a, b = K.source_terms(g["vertices"][3], g["normals"][3], charges)
    assert (a, b) == (s1[3], s2[3])
    assert K.source_terms([1.0, 0, 0], [1.0, 0, 0], ChargeSystem(np.zeros((0, 3)), np.zeros(0))) == (0.0, 0.0)
    one = ChargeSystem([[0.0, 0.0, 0.0]], [1.0])
    a, b = K.source_terms([0.0, 0.0, 2.0], [0.0, 0.0, 1.0], one)
    assert a == pytest.approx(1.0 / (8.0 * np.pi), rel=1e-15) and b == pytest.approx(-1.0 / (16.0 * np.pi), rel=1e-15)
    with pytest.raises(K.SingularityError, match="surface point 1 coincides with charge 0"):
        K.source_terms_at(np.array([[1.0, 0, 0], [0.5, 0.5, 0.5]]), np.array([[1.0, 0, 0], [1.0, 0, 0]]),
                          ChargeSystem([[0.5, 0.5, 0.5]], [1.0]))
    assert K.g0([0, 0, 0], [0, 0, 2]) == pytest.approx(1.0 / (8.0 * np.pi), rel=1e-15)
    assert K.g_kappa([0, 0, 0], [0, 1, 0], 0.0) == K.g0([0, 0, 0], [0, 1, 0])
