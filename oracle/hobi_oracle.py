"""CPU oracle for the HOBI-PB boundary-integral hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the reference package ``pbbem``'s algorithm
for the path the B200 build accelerates (arXiv 1301.5914):
curved-element geometry precompute, the HOBI matvec (regular sweep + Duffy swap +
diagonal), the right-hand side, restarted GMRES and the solvation energy.  Every
function cites the reference file:line it follows (paths relative to
``/root/reference/pkg/src/pbbem``).

Status: parity PINNED.  ``tests/test_oracle_golden.py`` checks this restatement
against golden vectors produced by running the reference itself in the build
container (``tests/golden/make_golden.py``), plus the reference's own frozen
known answers (``test_solver.py:375-403``).

Who may use it: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs, and only as the checker or the timed CPU
baseline.  The product package ``paper_1301_5914_b200`` never imports it.

The restatement is deliberately vectorised differently from the reference (all
faces x rotations at once instead of a per-face Python loop, counting sort instead
of lexsort) so it is an independent implementation of the same arithmetic.
"""

from __future__ import annotations

import math
import multiprocessing
import os
from dataclasses import dataclass

import numpy as np

FOUR_PI = 4.0 * math.pi  # kernels.py:27
KCAL = 332.0716  # kernels.py:33
TARGET_BLOCK = 48  # solver.py:45


class OracleGeometryError(ValueError):
    """Mirrors geometry.DegenerateArcError (geometry.py:24-25)."""


class OracleNonConvergence(RuntimeError):
    """Mirrors solver.GmresNonConvergence (solver.py:50-55)."""

    def __init__(self, message, best_residual):
        super().__init__(message)
        self.best_residual = best_residual


# ----------------------------------------------------------------------------
# quadrature rules (quadrature.py:68-116)


def conical_rule():
    """4-point conical product rule, quadrature.py:68-87: (r_i, (1-r_i) t_j), w = a_i/2."""
    s6, s3 = math.sqrt(6.0), math.sqrt(3.0)
    radial = [((4.0 - s6) / 10.0, (9.0 + s6) / 36.0), ((4.0 + s6) / 10.0, (9.0 - s6) / 36.0)]
    trans = [0.5 - 0.5 / s3, 0.5 + 0.5 / s3]
    pts = np.array([(r, (1.0 - r) * t) for r, _ in radial for t in trans])
    wts = np.array([0.5 * a for _, a in radial for _ in trans])
    return pts, wts


def duffy_points(n):
    """n x n Gauss-Legendre on the square pushed through r=(1-y)x, s=yx (quadrature.py:90-116)."""
    g, gw = np.polynomial.legendre.leggauss(n)
    g = 0.5 * (g + 1.0)
    gw = 0.5 * gw
    xx = np.repeat(g, n)
    yy = np.tile(g, n)
    wx = np.repeat(gw, n)
    wy = np.tile(gw, n)
    pts = np.stack([(1.0 - yy) * xx, yy * xx], axis=1)
    return pts, wx * wy * xx


def linear_weights(pts):
    """(1-r-s, r, s) at reference points, solver.py:158-162."""
    return np.stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]], axis=1)


# ----------------------------------------------------------------------------
# cubic Lagrange basis on the 10-node triangle (geometry.py:127-205)

NODE_RS = np.array(
    [[0, 0], [1 / 3, 0], [0, 1 / 3], [1, 0], [2 / 3, 0], [0, 2 / 3],
     [2 / 3, 1 / 3], [1 / 3, 2 / 3], [0, 1], [1 / 3, 1 / 3]],
    dtype=float,
)
POWERS = [(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2), (3, 0), (2, 1), (1, 2), (0, 3)]


def _mono(pts, dr=0, ds=0):
    r, s = pts[:, 0], pts[:, 1]
    cols = []
    for i, j in POWERS:
        if (dr and i == 0) or (ds and j == 0):
            cols.append(np.zeros_like(r))
            continue
        c = (i if dr else 1.0) * (j if ds else 1.0)
        cols.append(c * r ** (i - dr) * s ** (j - ds))
    return np.stack(cols, axis=1)


BASIS_COEF = np.linalg.inv(_mono(NODE_RS))  # geometry.py:169-183


def basis_tables(pts):
    """(N, dN/dr, dN/ds) at the rule points, each (m, 10)  (geometry.py:197-205)."""
    return _mono(pts) @ BASIS_COEF, _mono(pts, dr=1) @ BASIS_COEF, _mono(pts, ds=1) @ BASIS_COEF


# ----------------------------------------------------------------------------
# curved nodes from vertex data, vectorised over many (face, rotation) slots


def _dot(a, b):
    return a[..., 0] * b[..., 0] + a[..., 1] * b[..., 1] + a[..., 2] * b[..., 2]


def _norm(a):
    return np.sqrt(_dot(a, a))


def _fma(a, b, c):
    """Correctly rounded a*b+c emulated with error-free transforms (Dekker/Knuth)."""
    p = a * b
    t = 134217729.0 * a
    ah = t - (t - a)
    t = 134217729.0 * b
    bh = t - (t - b)
    ep = ((ah * bh - p) + ah * (b - bh) + (a - ah) * bh) + (a - ah) * (b - bh)
    s = p + c
    bb = s - p
    es = (p - (s - bb)) + (c - bb)
    return s + (ep + es)


def _bdot(a, b):
    """np.dot / np.linalg.norm of single 3-vectors go through BLAS ddot, which rounds as
    fma(z, z', fma(y, y', x*x')); the per-face geometry (geometry.py:46-121, 252-258)
    uses exactly those calls, so the restatement reproduces that rounding."""
    return _fma(a[..., 2], b[..., 2], _fma(a[..., 1], b[..., 1], a[..., 0] * b[..., 0]))


def _bnorm(a):
    return np.sqrt(_bdot(a, a))


class _Fail:
    """First-failure bookkeeping per slot: code 0 = ok (messages geometry.py:63,70,257)."""

    MESSAGES = {
        1: "arc endpoints coincide",
        2: "endpoint normal is nearly parallel to the chord",
        3: "endpoint normals are antiparallel",
    }

    def __init__(self, n):
        self.code = np.zeros(n, dtype=np.int64)

    def flag(self, mask, code):
        self.code[(self.code == 0) & mask] = code


def _hermite_arc(p0, n0, p1, n1, fail):
    """fit_arc, geometry.py:46-84; returns the power-basis coefficients (c0..c3)."""
    chord = p1 - p0
    clen = _bnorm(chord)
    fail.flag(clen < 1e-300, 1)
    t0 = chord - _bdot(chord, n0)[:, None] * n0
    t1 = chord - _bdot(chord, n1)[:, None] * n1
    l0 = _bnorm(t0)
    l1 = _bnorm(t1)
    fail.flag((l0 < 1e-12 * clen) | (l1 < 1e-12 * clen), 2)
    with np.errstate(divide="ignore", invalid="ignore"):
        t0 = t0 / l0[:, None]
        t1 = t1 / l1[:, None]
        c2t = np.clip(_bdot(t0, t1), -1.0, 1.0)
        mag = 2.0 * clen / (1.0 + np.sqrt(0.5 * (1.0 + c2t)))
    m0 = mag[:, None] * t0
    m1 = mag[:, None] * t1
    return (p0, m0, -3.0 * p0 + 3.0 * p1 - 2.0 * m0 - m1, 2.0 * p0 - 2.0 * p1 + m0 + m1)


def _arc_at(c, t):
    return c[0] + t * (c[1] + t * (c[2] + t * c[3]))  # geometry.py:87-88


def _arc_nrm(c, t, ref):
    """arc_normal, geometry.py:99-121 (curvature direction, signed by ref)."""
    v = c[1] + t * (2.0 * c[2] + t * (3.0 * c[3]))
    a = 2.0 * c[2] + 6.0 * t * c[3]
    v2 = _bdot(v, v)
    with np.errstate(divide="ignore", invalid="ignore"):
        k = (a - (_bdot(v, a) / v2)[:, None] * v) / np.sqrt(v2)[:, None]
        kl = _bnorm(k)
        n = k / kl[:, None]
    n = np.where((_bdot(n, ref) < 0.0)[:, None], -n, n)
    straight = (v2 < 1e-300) | ~(kl >= 1e-12)
    return np.where(straight[:, None], ref, n)


def _blend(n0, n1, t, fail):
    """_blend_reference, geometry.py:252-258."""
    ref = (1.0 - t) * n0 + t * n1
    ln = _bnorm(ref)
    fail.flag(ln < 1e-12, 3)
    with np.errstate(divide="ignore", invalid="ignore"):
        return ref / ln[:, None]


def curved_nodes(x1, n1, x2, n2, x3, n3):
    """nodes_from_vertex_data (geometry.py:261-302) for S slots at once.

    Returns node positions (S, 10, 3), node normals (S, 10, 3) and the per-slot
    failure code (0 = fine).
    """
    S = x1.shape[0]
    fail = _Fail(S)
    P = np.empty((S, 10, 3))
    N = np.empty((S, 10, 3))
    P[:, 0], N[:, 0] = x1, n1
    P[:, 3], N[:, 3] = x2, n2
    P[:, 8], N[:, 8] = x3, n3
    e12 = _hermite_arc(x1, n1, x2, n2, fail)
    e13 = _hermite_arc(x1, n1, x3, n3, fail)
    third = 1.0 / 3.0
    for slot, t in ((1, third), (4, 2 * third)):
        P[:, slot] = _arc_at(e12, t)
        N[:, slot] = _arc_nrm(e12, t, _blend(n1, n2, t, fail))
    for slot, t in ((2, third), (5, 2 * third)):
        P[:, slot] = _arc_at(e13, t)
        N[:, slot] = _arc_nrm(e13, t, _blend(n1, n3, t, fail))
    y1, y2 = _arc_at(e12, 1.0), _arc_at(e13, 1.0)
    ny1, ny2 = _arc_nrm(e12, 1.0, n2), _arc_nrm(e13, 1.0, n3)
    far = _hermite_arc(y1, ny1, y2, ny2, fail)
    for slot, t in ((6, third), (7, 2 * third)):
        P[:, slot] = _arc_at(far, t)
        N[:, slot] = _arc_nrm(far, t, _blend(ny1, ny2, t, fail))
    mid = _hermite_arc(P[:, 4], N[:, 4], P[:, 5], N[:, 5], fail)
    P[:, 9] = _arc_at(mid, 0.5)
    N[:, 9] = _arc_nrm(mid, 0.5, _blend(N[:, 4], N[:, 5], 0.5, fail))
    return P, N, fail.code


def frames(P, N, pts):
    """frames_at, geometry.py:342-359: positions, oriented unit normals, Jacobians."""
    B, Br, Bs = basis_tables(pts)
    pos = np.einsum("mk,eki->emi", B, P)
    xr = np.einsum("mk,eki->emi", Br, P)
    xs = np.einsum("mk,eki->emi", Bs, P)
    cr = np.cross(xr, xs)
    jac = _norm(cr)
    nrm = cr / jac[..., None]
    hint = np.einsum("mk,eki->emi", B, N)
    flip = _dot(nrm, hint) < 0.0
    nrm = np.where(flip[..., None], -nrm, nrm)
    return pos, nrm, jac


# ----------------------------------------------------------------------------
# mesh validation (mesh.py:50-89)


def validate_mesh(vertices, normals, faces):
    """Returns None or an error string, in the reference's check order."""
    ln = _norm(normals)
    bad = np.nonzero(np.abs(ln - 1.0) > 1e-12)[0]
    if bad.size:
        return f"normal {bad[0]} has length {ln[bad[0]]!r}, expected 1"
    nv = vertices.shape[0]
    if faces.size and (faces.min() < 0 or faces.max() >= nv):
        j = np.nonzero(((faces < 0) | (faces >= nv)).any(axis=1))[0][0]
        return f"face {j} references a vertex outside [0, {nv})"
    x = vertices[faces]
    geo = np.cross(x[:, 1] - x[:, 0], x[:, 2] - x[:, 0])
    dots = _dot(geo, normals[faces].mean(axis=1))
    flipped = np.nonzero(dots <= 0.0)[0]
    if flipped.size:
        return f"face {flipped[0]} is oriented against its vertex normals"
    e = np.sort(np.concatenate([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]]), axis=1)
    uniq, cnt = np.unique(e, axis=0, return_counts=True)
    bad = np.nonzero(cnt != 2)[0]
    if bad.size:
        i, j = uniq[bad[0]]
        return (f"mesh is not closed: edge ({i}, {j}) belongs to {cnt[bad[0]]} "
                f"face(s), expected 2")
    return None


# ----------------------------------------------------------------------------
# discretisation caches (solver.py:165-266)


@dataclass
class Problem:
    vertices: np.ndarray
    normals: np.ndarray
    faces: np.ndarray
    eps1: float
    eps2: float
    kappa: float
    qpos: np.ndarray
    q: np.ndarray
    scheme: str = "hobi"
    reg_pos: np.ndarray = None
    reg_nrm: np.ndarray = None
    reg_w: np.ndarray = None
    reg_bary: np.ndarray = None
    pair_vertex: np.ndarray = None
    pair_face: np.ndarray = None
    pair_gverts: np.ndarray = None
    pair_starts: np.ndarray = None
    duf_pos: np.ndarray = None
    duf_nrm: np.ndarray = None
    duf_w: np.ndarray = None
    duf_bary: np.ndarray = None
    area: np.ndarray = None
    colloc_pos: np.ndarray = None
    colloc_nrm: np.ndarray = None

    @property
    def n_colloc(self):
        return self.colloc_pos.shape[0]


def incident_pairs(faces, nv):
    """Pair tables of solver.py:229-243 via a stable counting sort by vertex.

    Slot p = 3 f + k couples vertex faces[f, k] with face f; the reference
    lexsorts by (vertex, face), which for slots enumerated in face order is a
    stable bucket sort on the vertex id.
    """
    nf = faces.shape[0]
    vert = faces.reshape(-1)
    order = np.argsort(vert, kind="stable")
    starts = np.zeros(nv + 1, dtype=np.int64)
    np.cumsum(np.bincount(vert, minlength=nv), out=starts[1:])
    rot = np.stack([faces, np.roll(faces, -1, axis=1), np.roll(faces, -2, axis=1)], axis=1)
    face_of = np.repeat(np.arange(nf, dtype=np.int64), 3)
    return order, vert[order], face_of[order], rot.reshape(-1, 3)[order], starts


def discretize(vertices, normals, faces, eps1, eps2, kappa, qpos=None, q=None,
               scheme="hobi", duffy_n=4, check=True, rule=None):
    """Build the caches of solver.py:165-266 (HOBI) or the flat LOBI ones (:177-186)."""
    vertices = np.asarray(vertices, dtype=float)
    normals = np.asarray(normals, dtype=float)
    faces = np.asarray(faces, dtype=np.int64)
    qpos = np.zeros((0, 3)) if qpos is None else np.asarray(qpos, float).reshape(-1, 3)
    q = np.zeros(0) if q is None else np.asarray(q, float).reshape(-1)
    if check:
        msg = validate_mesh(vertices, normals, faces)
        if msg:
            raise ValueError(msg)
    prob = Problem(vertices, normals, faces, float(eps1), float(eps2), float(kappa), qpos, q,
                   scheme=scheme)
    corners = vertices[faces]
    cr = np.cross(corners[:, 1] - corners[:, 0], corners[:, 2] - corners[:, 0])
    two_a = _norm(cr)
    prob.area = 0.5 * two_a
    if scheme == "lobi":
        prob.colloc_pos = corners.mean(axis=1)
        prob.colloc_nrm = cr / two_a[:, None]
        return prob
    nf, nv = faces.shape[0], vertices.shape[0]
    rot = np.stack([faces, np.roll(faces, -1, axis=1), np.roll(faces, -2, axis=1)], axis=1)
    idx = rot.reshape(-1, 3)  # slot 3f+k -> (local 1, local 2, local 3) vertex ids
    P, N, code = curved_nodes(vertices[idx[:, 0]], normals[idx[:, 0]],
                              vertices[idx[:, 1]], normals[idx[:, 1]],
                              vertices[idx[:, 2]], normals[idx[:, 2]])
    bad = np.nonzero(code)[0]
    if bad.size:
        s = bad[0]
        raise OracleGeometryError(f"face {s // 3}: {_Fail.MESSAGES[int(code[s])]}")
    P = P.reshape(nf, 3, 10, 3)
    N = N.reshape(nf, 3, 10, 3)
    rpts, rwts = conical_rule() if rule is None else (np.asarray(rule[0], float), np.asarray(rule[1], float))
    dpts, dwts = duffy_points(duffy_n)
    prob.reg_pos, prob.reg_nrm, jac = frames(P[:, 0], N[:, 0], rpts)
    prob.reg_w = rwts[None, :] * jac
    dpos, dnrm, djac = frames(P.reshape(-1, 10, 3), N.reshape(-1, 10, 3), dpts)
    order, pv, pf, pg, starts = incident_pairs(faces, nv)
    prob.duf_pos, prob.duf_nrm = dpos[order], dnrm[order]
    prob.duf_w = (dwts[None, :] * djac)[order]
    prob.pair_vertex, prob.pair_face, prob.pair_gverts, prob.pair_starts = pv, pf, pg, starts
    prob.reg_bary = linear_weights(rpts)
    prob.duf_bary = linear_weights(dpts)
    prob.colloc_pos, prob.colloc_nrm = vertices, normals
    return prob


# ----------------------------------------------------------------------------
# kernels (kernels.py:99-130, 159-178)


def k1234(d, nx, ny, eps1, eps2, kappa):
    """K1..K4 of kernels.py:99-130 from displacements d = x - y."""
    er = eps2 / eps1
    r2 = _dot(d, d)
    r = np.sqrt(r2)
    kr = kappa * r
    e = np.exp(-kr)
    m = np.expm1(-kr)
    a = m + kr * e
    b = 3.0 * m + kr * e * (3.0 + kr)
    dny, dnx, nn = _dot(d, ny), _dot(d, nx), _dot(nx, ny)
    i3 = 1.0 / (FOUR_PI * r2 * r)
    return (-m / (FOUR_PI * r),
            dny * i3 * ((er - 1.0) + er * a),
            -dnx * i3 * ((1.0 - 1.0 / er) - a / er),
            (-b * dnx * dny / r2 + a * nn) * i3)


def rhs(prob):
    """assemble_rhs (solver.py:393-402) over source_terms_at (kernels.py:159-178)."""
    x, n = prob.colloc_pos, prob.colloc_nrm
    t = x.shape[0]
    if prob.q.size == 0:
        return np.zeros(2 * t)
    s1 = np.empty(t)
    s2 = np.empty(t)
    for lo in range(0, t, 256):  # bounded transients instead of one (t, nc, 3) block
        hi = min(lo + 256, t)
        d = x[lo:hi, None, :] - prob.qpos[None, :, :]
        r2 = _dot(d, d)
        if (r2 < 1e-300).any():
            i, k = np.argwhere(r2 < 1e-300)[0]
            raise ZeroDivisionError(f"surface point {lo + i} coincides with charge {k}")
        r = np.sqrt(r2)
        s1[lo:hi] = (prob.q / (FOUR_PI * r)).sum(axis=1)
        s2[lo:hi] = (-prob.q * _dot(d, n[lo:hi, None, :]) / (FOUR_PI * r2 * r)).sum(axis=1)
    return np.concatenate([s1, s2]) / prob.eps1


def _lin(vals, bary):
    return vals[..., 0, None] * bary[:, 0] + vals[..., 1, None] * bary[:, 1] + vals[..., 2, None] * bary[:, 2]


def source_weights(prob, u):
    """Interpolated, weighted source strengths on the regular points (solver.py:318-324)."""
    T = prob.n_colloc
    phi, dphi = u[:T], u[T:]
    wp = (prob.reg_w * _lin(phi[prob.faces], prob.reg_bary)).reshape(-1)
    wd = (prob.reg_w * _lin(dphi[prob.faces], prob.reg_bary)).reshape(-1)
    return wp, wd


def rows(prob, u, lo, hi):
    """Rows [lo, hi) of both blocks: _apply_range, solver.py:278-367."""
    T = prob.n_colloc
    par = (prob.eps1, prob.eps2, prob.kappa)
    er = prob.eps2 / prob.eps1
    phi, dphi = u[:T], u[T:]
    n = hi - lo
    acc1 = np.zeros(n)
    acc2 = np.zeros(n)
    xt, nt = prob.colloc_pos[lo:hi], prob.colloc_nrm[lo:hi]
    if prob.scheme == "lobi":  # solver.py:296-315
        wp, wd = prob.area * phi, prob.area * dphi
        src, snrm = prob.colloc_pos, prob.colloc_nrm
        for s in range(0, n, TARGET_BLOCK):
            e = min(s + TARGET_BLOCK, n)
            d = xt[s:e, None, :] - src[None, :, :]
            own = np.arange(s, e)
            d[own - s, lo + own] = (1.0, 0.0, 0.0)
            ks = k1234(d, nt[s:e, None, :], snrm[None, :, :], *par)
            for k in ks:
                k[own - s, lo + own] = 0.0
            acc1[s:e] = (ks[0] * wd + ks[1] * wp).sum(axis=1)
            acc2[s:e] = (ks[2] * wd + ks[3] * wp).sum(axis=1)
        return 0.5 * (1.0 + er) * phi[lo:hi] - acc1, 0.5 * (1.0 + 1.0 / er) * dphi[lo:hi] - acc2
    wp, wd = source_weights(prob, u)
    src = prob.reg_pos.reshape(-1, 3)
    snrm = prob.reg_nrm.reshape(-1, 3)
    for s in range(0, n, TARGET_BLOCK):  # regular sweep, solver.py:325-334
        e = min(s + TARGET_BLOCK, n)
        ks = k1234(xt[s:e, None, :] - src[None, :, :], nt[s:e, None, :], snrm[None, :, :], *par)
        acc1[s:e] = (ks[0] * wd + ks[1] * wp).sum(axis=1)
        acc2[s:e] = (ks[2] * wd + ks[3] * wp).sum(axis=1)
    p0, p1 = int(prob.pair_starts[lo]), int(prob.pair_starts[hi])
    if p1 > p0:  # Duffy swap, solver.py:336-363
        pv = prob.pair_vertex[p0:p1]
        pf = prob.pair_face[p0:p1]
        px = prob.colloc_pos[pv][:, None, :]
        pn = prob.colloc_nrm[pv][:, None, :]
        phq = _lin(phi[prob.faces[pf]], prob.reg_bary)
        dpq = _lin(dphi[prob.faces[pf]], prob.reg_bary)
        ks = k1234(px - prob.reg_pos[pf], pn, prob.reg_nrm[pf], *par)
        r1 = (ks[0] * prob.reg_w[pf] * dpq + ks[1] * prob.reg_w[pf] * phq).sum(axis=1)
        r2 = (ks[2] * prob.reg_w[pf] * dpq + ks[3] * prob.reg_w[pf] * phq).sum(axis=1)
        gv = prob.pair_gverts[p0:p1]
        ks = k1234(px - prob.duf_pos[p0:p1], pn, prob.duf_nrm[p0:p1], *par)
        wpd = prob.duf_w[p0:p1] * _lin(phi[gv], prob.duf_bary)
        wdd = prob.duf_w[p0:p1] * _lin(dphi[gv], prob.duf_bary)
        d1 = (ks[0] * wdd + ks[1] * wpd).sum(axis=1)
        d2 = (ks[2] * wdd + ks[3] * wpd).sum(axis=1)
        acc1 += np.bincount(pv - lo, weights=d1 - r1, minlength=n)
        acc2 += np.bincount(pv - lo, weights=d2 - r2, minlength=n)
    return 0.5 * (1.0 + er) * phi[lo:hi] - acc1, 0.5 * (1.0 + 1.0 / er) * dphi[lo:hi] - acc2


def matvec(prob, u):
    """_full_matvec, solver.py:370-376."""
    u = np.asarray(u, dtype=float)
    T = prob.n_colloc
    if u.shape != (2 * T,):
        raise ValueError(f"expected vector of length {2 * T}, got shape {u.shape}")
    a, b = rows(prob, u, 0, T)
    return np.concatenate([a, b])


def partition(n, w):
    """partition_targets, solver.py:405-418."""
    if w < 1:
        raise ValueError(f"n_workers must be >= 1, got {w}")
    if n < 0:
        raise ValueError(f"n_targets must be >= 0, got {n}")
    q, extra = divmod(n, w)
    out, lo = [], 0
    for i in range(w):
        hi = lo + q + (1 if i < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


_POOL_PROBLEM = {}


def _pool_rows(key, u, lo, hi):
    return rows(_POOL_PROBLEM[key], u, lo, hi)


class PoolOperator:
    """Fork-pool row split of solver.py:432-472 (the reference's CPU parallel path)."""

    def __init__(self, prob, workers=None):
        self.prob = prob
        self.workers = workers or os.cpu_count() or 1
        self.ranges = partition(prob.n_colloc, self.workers)
        self.key = id(self)
        _POOL_PROBLEM[self.key] = prob
        self.pool = None
        if self.workers > 1 and prob.n_colloc > 0:
            self.pool = multiprocessing.get_context("fork").Pool(self.workers)

    def rows(self, u, lo, hi):
        """Rows [lo, hi) split over the pool (used for bounded CPU-baseline samples)."""
        if self.pool is None:
            return rows(self.prob, u, lo, hi)
        parts = self.pool.starmap(_pool_rows, [(self.key, u, a, b) for a, b in partition(hi - lo, self.workers)
                                               for a, b in [(lo + a, lo + b)]])
        return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])

    def __call__(self, u):
        a, b = self.rows(np.asarray(u, float), 0, self.prob.n_colloc)
        return np.concatenate([a, b])

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None
        _POOL_PROBLEM.pop(self.key, None)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def gmres(apply, b, tol=1e-6, restart=100, max_it=1000):
    """Restarted GMRES(m) with MGS and Givens, solver.py:484-560.

    Returns (x, iterations, relative residual, matvec count).
    """
    b = np.asarray(b, dtype=float)
    n = b.size
    if n % 2:
        raise ValueError("vector length must be even: (phi, dphi/dn) halves")
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return np.zeros(n), 0, 0.0, 0
    x = np.zeros(n)
    its = 0
    nmv = 0
    best = np.inf
    while True:
        r = b - apply(x)
        nmv += 1
        rel = float(np.linalg.norm(r)) / nb
        best = min(best, rel)
        if rel <= tol:
            return x, its, rel, nmv
        if its >= max_it:
            raise OracleNonConvergence(f"no convergence in {its} iterations", best)
        beta = float(np.linalg.norm(r))
        V = np.zeros((restart + 1, n))
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        V[0] = r / beta
        g[0] = beta
        j = 0
        while j < restart and its < max_it:
            w = apply(V[j])
            nmv += 1
            for i in range(j + 1):
                H[i, j] = float(V[i] @ w)
                w = w - H[i, j] * V[i]
            H[j + 1, j] = float(np.linalg.norm(w))
            if H[j + 1, j] > 1e-300:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                hi_, hn = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * hi_ + sn[i] * hn
                H[i + 1, j] = -sn[i] * hi_ + cs[i] * hn
            den = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j] = H[j, j] / den
            sn[j] = H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            j += 1
            if abs(g[j]) / nb <= tol:
                break
        y = np.linalg.solve(np.triu(H[:j, :j]), g[:j]) if j else np.zeros(0)
        x = x + V[:j].T @ y


def energy(prob, phi, dphi):
    """solvation_energy, solver.py:581-614 (kcal/mol)."""
    if prob.q.size == 0:
        return 0.0
    if prob.scheme == "hobi":
        u = np.concatenate([phi, dphi])
        wp, wd = source_weights(prob, u)
        src, snrm = prob.reg_pos.reshape(-1, 3), prob.reg_nrm.reshape(-1, 3)
    else:
        wp, wd = prob.area * phi, prob.area * dphi
        src, snrm = prob.colloc_pos, prob.colloc_nrm
    tot = 0.0
    for pos, qk in zip(prob.qpos, prob.q):
        k1, k2, _, _ = k1234(pos[None, :] - src, snrm, snrm, prob.eps1, prob.eps2, prob.kappa)
        tot += qk * float((k1 * wd + k2 * wp).sum())
    return 0.5 * FOUR_PI * KCAL * tot


def solve(prob, tol=1e-6, restart=100, max_it=1000, workers=1):
    """solve(), solver.py:563-574, on an already discretised problem."""
    b = rhs(prob)
    with PoolOperator(prob, workers) as op:
        x, its, rel, nmv = gmres(op, b, tol, restart, max_it)
    T = prob.n_colloc
    return x[:T], x[T:], its, rel, nmv
