"""The reference's ``pbbem.geometry`` module surface on the device.

Every function that does geometry arithmetic -- ``fit_arc`` (geometry.py:46-84),
``arc_normal`` (:99-121), ``nodes_from_vertex_data`` (:261-302),
``element_frame`` (:323-339), ``frames_at`` (:342-359) -- calls the device
functions that ``hobi_create``'s precompute runs (``csrc/hobi_geometry.cu``),
batched behind ``hobi_geometry_*`` in the C ABI, so what these return is what
the solver's caches hold, bit for bit.  The cubic Lagrange basis tables are
the host constants of ``quadrature.py`` (they are uploaded to the device, not
computed there), and ``arc_point`` / ``arc_velocity`` / ``arc_acceleration``
evaluate the returned cubic's coefficients (geometry.py:87-96).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .mesh import FlatMesh
from .quadrature import REFERENCE_NODES, shape_tables

VERTEX_LOCAL = (0, 3, 8)  # local node ids of the three triangle vertices (geometry.py:142)

_ARC_MESSAGES = ("", "arc endpoints coincide", "endpoint normal is nearly parallel to the chord",
                 "endpoint normals are antiparallel")


class DegenerateArcError(ValueError):
    """An edge arc could not be fitted (geometry.py:24-25)."""


class DegenerateElementError(ValueError):
    """An element's surface Jacobian vanished (geometry.py:28-29)."""


@dataclass(frozen=True)
class CubicArc:
    """x(t) = c0 + c1 t + c2 t^2 + c3 t^3 on [0, 1] (geometry.py:36-43)."""

    c0: np.ndarray
    c1: np.ndarray
    c2: np.ndarray
    c3: np.ndarray


def _row(v) -> np.ndarray:
    return N.f64(np.asarray(v, dtype=float).reshape(1, 3))


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def fit_arc(p0, n0, p1, n1, device: int = 0) -> CubicArc:
    """Cubic arc between two surface points with outward unit normals."""
    N.require_device()
    coef = np.empty((1, 4, 3))
    code = np.zeros(1, dtype=np.intc)
    N.check(N.load().hobi_geometry_fit_arcs(device, N.dptr(_row(p0)), N.dptr(_row(n0)), N.dptr(_row(p1)),
                                            N.dptr(_row(n1)), 1, N.dptr(coef), _iptr(code)))
    if code[0]:
        raise DegenerateArcError(_ARC_MESSAGES[int(code[0])])
    return CubicArc(*(coef[0, k].copy() for k in range(4)))


def arc_point(arc: CubicArc, t: float) -> np.ndarray:
    return arc.c0 + t * (arc.c1 + t * (arc.c2 + t * arc.c3))


def arc_velocity(arc: CubicArc, t: float) -> np.ndarray:
    return arc.c1 + t * (2.0 * arc.c2 + t * (3.0 * arc.c3))


def arc_acceleration(arc: CubicArc, t: float) -> np.ndarray:
    return 2.0 * arc.c2 + 6.0 * t * arc.c3


def arc_normal(arc: CubicArc, t: float, reference, device: int = 0):
    """(unit normal from the arc's curvature, signed like `reference`; True
    where the arc is locally straight and `reference` itself comes back)."""
    N.require_device()
    coef = N.f64(np.stack([arc.c0, arc.c1, arc.c2, arc.c3]).reshape(1, 4, 3))
    tt = N.f64(np.array([t], dtype=float))
    out = np.empty((1, 3))
    flag = np.zeros(1, dtype=np.intc)
    N.check(N.load().hobi_geometry_arc_normals(device, N.dptr(coef), N.dptr(tt), N.dptr(_row(reference)), 1,
                                               N.dptr(out), _iptr(flag)))
    return out[0].copy(), bool(flag[0])


# ---------------------------------------------------------------------------
# cubic Lagrange basis on the 10-node reference triangle (geometry.py:127-205)


def shape_matrix(pts) -> np.ndarray:
    """(m, 2) -> (m, 10) basis values."""
    return shape_tables(np.asarray(pts, dtype=float).reshape(-1, 2))[0]


def shape_gradient_matrices(pts):
    """(m, 2) -> (dN/dr, dN/ds), each (m, 10)."""
    t = shape_tables(np.asarray(pts, dtype=float).reshape(-1, 2))
    return t[1], t[2]


def shape_functions(r: float, s: float) -> np.ndarray:
    return shape_matrix([[r, s]])[0]


def shape_gradients(r: float, s: float) -> np.ndarray:
    """(10, 2): (dN/dr, dN/ds) at (r, s)."""
    g_r, g_s = shape_gradient_matrices([[r, s]])
    return np.stack([g_r[0], g_s[0]], axis=-1)


# ---------------------------------------------------------------------------
# curved elements


@dataclass(frozen=True)
class CurvedElement:
    """10-node cubic element: positions, unit normals, source vertex ids (geometry.py:212-230)."""

    nodes: np.ndarray
    node_normals: np.ndarray
    vertex_ids: tuple

    def __post_init__(self):
        pos = np.array(self.nodes, dtype=float).reshape(10, 3)
        nrm = np.array(self.node_normals, dtype=float).reshape(10, 3)
        if np.abs(np.linalg.norm(nrm, axis=1) - 1.0).max() > 1e-12:
            raise ValueError("node normals must be unit length")
        pos.setflags(write=False)
        nrm.setflags(write=False)
        object.__setattr__(self, "nodes", pos)
        object.__setattr__(self, "node_normals", nrm)
        object.__setattr__(self, "vertex_ids", tuple(int(i) for i in self.vertex_ids))


@dataclass(frozen=True)
class SurfaceFrame:
    """Local geometry at one point of an element (geometry.py:233-241)."""

    position: np.ndarray
    d_dr: np.ndarray
    d_ds: np.ndarray
    normal: np.ndarray
    jacobian: float


def rs_to_uv(r: float, s: float):
    """u = r + s, v = s/(r + s) (geometry.py:244-249)."""
    u = r + s
    return (0.0, 0.0) if u == 0.0 else (u, s / u)


def nodes_for_triangles(vertex_pos, vertex_nrm, device: int = 0):
    """Batched nodes_from_vertex_data: (n, 3, 3) vertex positions and normals
    -> (n, 10, 3) node positions and normals, plus (first degenerate triple or
    -1, its message)."""
    N.require_device()
    vp = N.f64(np.asarray(vertex_pos, dtype=float).reshape(-1, 3, 3))
    vn = N.f64(np.asarray(vertex_nrm, dtype=float).reshape(-1, 3, 3))
    n = vp.shape[0]
    pos, nrm = np.empty((n, 10, 3)), np.empty((n, 10, 3))
    bad, code = np.full(1, -1, dtype=np.int64), np.zeros(1, dtype=np.intc)
    N.check(N.load().hobi_geometry_nodes(device, N.dptr(vp), N.dptr(vn), n, N.dptr(pos), N.dptr(nrm),
                                         N.iptr(bad), _iptr(code)))
    return pos, nrm, int(bad[0]), _ARC_MESSAGES[int(code[0])]


def nodes_from_vertex_data(x1, n1, x2, n2, x3, n3):
    """The 10 node positions and normals of one curved element from its three
    vertices; vertex nodes keep the inputs bitwise."""
    pos, nrm, bad, msg = nodes_for_triangles(np.stack([np.asarray(v, dtype=float) for v in (x1, x2, x3)]),
                                             np.stack([np.asarray(v, dtype=float) for v in (n1, n2, n3)]))
    if bad >= 0:
        raise DegenerateArcError(msg)
    return pos[0], nrm[0]


def build_curved_element(mesh: FlatMesh, face_index: int) -> CurvedElement:
    """Curved cubic element of one face (geometry.py:305-320)."""
    if not 0 <= face_index < mesh.n_faces:
        raise IndexError(f"face index {face_index} outside [0, {mesh.n_faces})")
    ids = tuple(int(i) for i in mesh.faces[face_index])
    try:
        nodes, normals = nodes_from_vertex_data(*(a for i in ids for a in (mesh.vertices[i], mesh.normals[i])))
    except DegenerateArcError as exc:
        raise DegenerateArcError(f"face {face_index}: {exc}") from None
    return CurvedElement(nodes=nodes, node_normals=normals, vertex_ids=ids)


def _frames(node_pos, node_nrm, pts, tangents: bool, device: int = 0):
    N.require_device()
    node_pos = N.f64(np.asarray(node_pos, dtype=float).reshape(-1, 10, 3))
    node_nrm = N.f64(np.asarray(node_nrm, dtype=float).reshape(-1, 10, 3))
    pts = np.asarray(pts, dtype=float).reshape(-1, 2)
    ne, m = node_pos.shape[0], pts.shape[0]
    shape = N.f64(shape_tables(pts))
    pos, nrm, jac = np.empty((ne, m, 3)), np.empty((ne, m, 3)), np.empty((ne, m))
    d_dr = np.empty((ne, m, 3)) if tangents else None
    d_ds = np.empty((ne, m, 3)) if tangents else None
    N.check(N.load().hobi_geometry_frames(device, N.dptr(node_pos), N.dptr(node_nrm), ne, N.dptr(shape), m,
                                          N.dptr(pos), N.dptr(nrm), N.dptr(jac),
                                          N.dptr(d_dr) if tangents else None,
                                          N.dptr(d_ds) if tangents else None))
    return pos, nrm, jac, d_dr, d_ds


def frames_at(node_pos, node_nrm, pts):
    """Frames of many elements at the same reference points: (n_e, 10, 3) x 2,
    (m, 2) -> positions (n_e, m, 3), oriented unit normals (n_e, m, 3),
    Jacobians (n_e, m)."""
    return _frames(node_pos, node_nrm, pts, False)[:3]


def element_frames(elem: CurvedElement, pts):
    """SurfaceFrame at each of the (m, 2) reference points of one element."""
    pts = np.asarray(pts, dtype=float).reshape(-1, 2)
    pos, nrm, jac, d_dr, d_ds = _frames(elem.nodes, elem.node_normals, pts, True)
    frames = []
    for q in range(pts.shape[0]):
        if jac[0, q] < 1e-14:
            raise DegenerateElementError(f"vanishing Jacobian at (r, s) = ({pts[q, 0]}, {pts[q, 1]})")
        frames.append(SurfaceFrame(position=pos[0, q], d_dr=d_dr[0, q], d_ds=d_ds[0, q], normal=nrm[0, q],
                                   jacobian=float(jac[0, q])))
    return frames


def element_frame(elem: CurvedElement, r: float, s: float) -> SurfaceFrame:
    """Position, tangents, oriented unit normal and Jacobian at (r, s)."""
    return element_frames(elem, [[r, s]])[0]


__all__ = ["REFERENCE_NODES", "VERTEX_LOCAL", "CubicArc", "CurvedElement", "SurfaceFrame",
           "DegenerateArcError", "DegenerateElementError", "arc_acceleration", "arc_normal", "arc_point",
           "arc_velocity", "build_curved_element", "element_frame", "element_frames", "fit_arc",
           "frames_at", "nodes_for_triangles", "nodes_from_vertex_data", "rs_to_uv", "shape_functions",
           "shape_gradient_matrices", "shape_gradients", "shape_matrix"]
