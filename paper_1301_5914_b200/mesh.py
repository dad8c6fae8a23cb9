"""Surface meshes and point charges: the input contract of the hot path.

Mirrors the reference's immutable input types and their validation
(``pbbem/mesh.py:24-110``, ``validate`` at ``:50-89``) plus the icosahedral
sphere generator (``:230-300``) used to build every benchmark surface.  File
ingest (MSMS) is a later row of SURVEY.md section 8(f) and lives here too.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class MeshFormatError(ValueError):
    """A mesh or charge file could not be parsed (pbbem/mesh.py:16-17)."""


class MeshValidationError(ValueError):
    """A mesh violates a structural invariant (pbbem/mesh.py:20-21)."""


def _frozen(a, dtype):
    a = np.array(a, dtype=dtype)
    a.setflags(write=False)
    return a


@dataclass(frozen=True)
class FlatMesh:
    """Closed triangulated surface with outward unit vertex normals (pbbem/mesh.py:24-75)."""

    vertices: np.ndarray  # (n_v, 3) Angstrom
    normals: np.ndarray  # (n_v, 3) unit
    faces: np.ndarray  # (n_f, 3) int64, 0-based, outward winding

    def __post_init__(self):
        object.__setattr__(self, "vertices", _frozen(self.vertices, float).reshape(-1, 3))
        object.__setattr__(self, "normals", _frozen(self.normals, float).reshape(-1, 3))
        object.__setattr__(self, "faces", _frozen(self.faces, np.int64).reshape(-1, 3))

    @property
    def n_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def n_faces(self) -> int:
        return self.faces.shape[0]

    def validate(self) -> None:
        """Unit normals, index range, orientation, closedness -- in the reference's order."""
        n = self.normals
        lengths = np.sqrt(n[:, 0] ** 2 + n[:, 1] ** 2 + n[:, 2] ** 2)
        bad = np.flatnonzero(np.abs(lengths - 1.0) > 1e-12)
        if bad.size:
            raise MeshValidationError(
                f"normal {bad[0]} has length {lengths[bad[0]]!r}, expected 1")
        f = self.faces
        nv = self.n_vertices
        if f.size:
            out = ((f < 0) | (f >= nv)).any(axis=1)
            if out.any():
                raise MeshValidationError(
                    f"face {np.flatnonzero(out)[0]} references a vertex outside [0, {nv})")
        x = self.vertices[f]
        geo = np.cross(x[:, 1] - x[:, 0], x[:, 2] - x[:, 0])
        mean_n = self.normals[f].mean(axis=1)
        flipped = np.flatnonzero(np.einsum("ij,ij->i", geo, mean_n) <= 0.0)
        if flipped.size:
            raise MeshValidationError(
                f"face {flipped[0]} is oriented against its vertex normals")
        _check_closed(f)


def _check_closed(faces: np.ndarray) -> None:
    """Every undirected edge shared by exactly two faces (pbbem/mesh.py:78-89)."""
    if faces.size == 0:
        return
    e = np.sort(np.concatenate([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]]), axis=1)
    key = e[:, 0] * (int(e.max()) + 1) + e[:, 1]
    uniq, counts = np.unique(key, return_counts=True)
    bad = np.flatnonzero(counts != 2)
    if bad.size:
        k = int(uniq[bad[0]])
        m = int(e.max()) + 1
        raise MeshValidationError(
            f"mesh is not closed: edge ({k // m}, {k % m}) belongs to {counts[bad[0]]} "
            f"face(s), expected 2")


@dataclass(frozen=True)
class ChargeSystem:
    """Point charges in Angstrom / elementary charges (pbbem/mesh.py:92-110)."""

    positions: np.ndarray
    charges: np.ndarray

    def __post_init__(self):
        p = _frozen(self.positions, float).reshape(-1, 3)
        q = _frozen(self.charges, float).reshape(-1)
        if p.shape[0] != q.shape[0]:
            raise ValueError(f"{p.shape[0]} positions but {q.shape[0]} charges")
        object.__setattr__(self, "positions", p)
        object.__setattr__(self, "charges", q)

    def __len__(self) -> int:
        return self.charges.size


# ----------------------------------------------------------------------------
# icosahedral spheres (pbbem/mesh.py:230-300), vectorised subdivision


def _base_icosahedron():
    t = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array([(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0),
                  (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
                  (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)], dtype=float)
    v /= np.linalg.norm(v[0])
    f = np.array([(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
                  (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
                  (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
                  (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)], dtype=np.int64)
    return v, f


def _fma(a, b, c):
    """Error-free-transform emulation of fused a*b+c (Dekker product + two-sum)."""
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


def _blas_norm(m):
    """Row norms with the same rounding as np.linalg.norm on one 3-vector
    (OpenBLAS ddot: fma(z, z, fma(y, y, x*x))), so generated spheres match the
    reference's vertex coordinates bit for bit."""
    return np.sqrt(_fma(m[:, 2], m[:, 2], _fma(m[:, 1], m[:, 1], m[:, 0] * m[:, 0])))


def _split(v, f):
    """One 4-to-1 split.  New midpoint vertices are numbered in order of first
    encounter over (face, edge ab/bc/ca), which reproduces the reference's
    dictionary-insertion numbering (pbbem/mesh.py:281-300)."""
    nf = f.shape[0]
    a, b, c = f[:, 0], f[:, 1], f[:, 2]
    ends = np.stack([np.stack([a, b], 1), np.stack([b, c], 1), np.stack([c, a], 1)], 1).reshape(-1, 2)
    lo = ends.min(axis=1)
    hi = ends.max(axis=1)
    key = lo * v.shape[0] + hi
    uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")  # unique edges by first appearance
    rank = np.empty_like(order)
    rank[order] = np.arange(order.size)
    mid_id = v.shape[0] + rank[inv].reshape(nf, 3)
    e0 = ends[first[order]]
    m = v[e0[:, 0]] + v[e0[:, 1]]
    m = m / _blas_norm(m)[:, None]
    ab, bc, ca = mid_id[:, 0], mid_id[:, 1], mid_id[:, 2]
    nfaces = np.stack([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                       np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], 1).reshape(-1, 3)
    return np.concatenate([v, m]), nfaces


def unit_icosphere(level: int):
    """Unit-sphere vertices and faces of the level-`level` subdivided icosahedron
    (levels 0-9; the reference-facing icosahedral_sphere keeps its 0-7)."""
    if not 0 <= level <= 9:
        raise ValueError(f"refinement level must be in [0, 9], got {level}")
    v, f = _base_icosahedron()
    for _ in range(level):
        v, f = _split(v, f)
    return v, f


def icosahedral_sphere(level: int, radius: float = 1.0, center=(0.0, 0.0, 0.0)) -> FlatMesh:
    """Subdivided icosahedron on a sphere with exact radial normals (pbbem/mesh.py:258-278)."""
    if not 0 <= level <= 7:
        raise ValueError(f"refinement level must be in [0, 7], got {level}")
    if radius <= 0.0:
        raise ValueError(f"radius must be positive, got {radius}")
    v, f = unit_icosphere(level)
    c = np.asarray(center, dtype=float)
    return FlatMesh(vertices=c + radius * v, normals=v.copy(), faces=f)


# ----------------------------------------------------------------------------
# MSMS .vert/.face text and charge files (pbbem/mesh.py:113-227), SURVEY.md 8(f) f2


def _records(text: str):
    """(1-based line number, tokens) of every non-blank line, '#' comments removed."""
    for number, raw in enumerate(text.splitlines(), start=1):
        body = raw.split("#", 1)[0].split()
        if body:
            yield number, body


def _parses(tok: str, kind) -> bool:
    try:
        kind(tok)
        return True
    except ValueError:
        return False


def parse_msms(vert_text: str, face_text: str) -> FlatMesh:
    """MSMS .vert/.face contents -> validated FlatMesh (pbbem/mesh.py:141-185).

    Records are recognised by shape, headers skipped: a vertex record starts
    with a real and has >= 6 fields (x y z nx ny nz), a face record has >= 3
    leading integers (1-based).  A record that breaks midway is an error with
    its line number; normals are renormalised (MSMS prints 3 digits).
    Regular texts go through the library's native scanner (same rules, same
    values, ~50x faster at protein sizes); anything it is unsure about goes
    through the line-by-line parser below, which also produces the errors.
    """
    fast = _parse_msms_native(vert_text, face_text)
    if fast is not None:
        return _msms_mesh(*fast)
    return _msms_mesh(*_parse_msms_python(vert_text, face_text))


def _parse_msms_python(vert_text: str, face_text: str):
    """Line-by-line record parser (mesh.py:141-185 rules and messages)."""
    rows = []
    for number, tok in _records(vert_text):
        if len(tok) < 6 or not _parses(tok[0], float):
            continue
        try:
            rows.append([float(t) for t in tok[:6]])
        except ValueError as exc:
            raise MeshFormatError(f".vert line {number}: {exc}") from None
    tris = []
    for number, tok in _records(face_text):
        if len(tok) < 3 or not all(_parses(t, int) for t in tok[:3]):
            continue
        ijk = tuple(int(t) for t in tok[:3])
        if min(ijk) < 1:
            raise MeshFormatError(f".face line {number}: vertex indices are 1-based, got {ijk}")
        tris.append(tuple(i - 1 for i in ijk))
    if not rows:
        raise MeshFormatError("no vertex records found in .vert text")
    if not tris:
        raise MeshFormatError("no face records found in .face text")
    return np.asarray(rows, dtype=float), np.asarray(tris, dtype=np.int64)


def _parse_msms_native(vert_text: str, face_text: str):
    """(vertex rows, 0-based faces) from the native scanner, or None when the
    texts are irregular (or the library is unavailable)."""
    try:
        import ctypes as C

        from . import _native as N

        lib = N.load()
    except Exception:  # noqa: BLE001
        return None
    try:
        vb, fb = vert_text.encode("ascii"), face_text.encode("ascii")
    except UnicodeEncodeError:
        return None
    vcap, fcap = vb.count(b"\n") + 1, fb.count(b"\n") + 1
    data = np.empty((vcap, 6))
    faces = np.empty((fcap, 3), dtype=np.int64)
    nv, nf = C.c_int64(0), C.c_int64(0)
    if lib.hobi_msms_parse(vb, len(vb), fb, len(fb), N.dptr(data), vcap, N.iptr(faces), fcap,
                           C.byref(nv), C.byref(nf)) != 0:
        return None
    if nv.value == 0 or nf.value == 0:
        return None  # the Python parser raises the reference's message
    return data[: nv.value], faces[: nf.value]


def _msms_mesh(data: np.ndarray, faces: np.ndarray) -> FlatMesh:
    nrm = data[:, 3:6]
    length = np.linalg.norm(nrm, axis=1)
    zero = np.flatnonzero(length < 1e-300)
    if zero.size:
        raise MeshFormatError(f"vertex {zero[0]} has a zero normal")
    mesh = FlatMesh(vertices=data[:, :3], normals=nrm / length[:, None], faces=faces)
    mesh.validate()
    return mesh


def write_msms(mesh: FlatMesh) -> tuple[str, str]:
    """Render a mesh as MSMS-style (vert_text, face_text) that parse_msms reads back
    exactly: full-precision reprs, comment headers (pbbem/mesh.py:188-207)."""
    vert = ["# vertices: x y z nx ny nz", f"{mesh.n_vertices} 1 1.0 1.0"]
    for p, n in zip(mesh.vertices.tolist(), mesh.normals.tolist()):
        vert.append(" ".join(repr(float(c)) for c in (*p, *n)) + " 0 0 0")
    face = ["# faces: i j k (1-based)", f"{mesh.n_faces} 1"]
    face.extend(f"{a + 1} {b + 1} {c + 1} 1 1" for a, b, c in mesh.faces.tolist())
    return "\n".join(vert) + "\n", "\n".join(face) + "\n"


def parse_charges(text: str) -> ChargeSystem:
    """'x y z q' records (a 5th radius column is ignored) -> ChargeSystem (pbbem/mesh.py:210-227)."""
    rows = []
    for number, tok in _records(text):
        if len(tok) < 4:
            raise MeshFormatError(f"charge line {number}: need at least 'x y z q', got {tok!r}")
        try:
            rows.append([float(t) for t in tok[:4]])
        except ValueError as exc:
            raise MeshFormatError(f"charge line {number}: {exc}") from None
    data = np.asarray(rows, dtype=float).reshape(-1, 4)
    return ChargeSystem(positions=data[:, :3], charges=data[:, 3])


def radial_project(mesh: FlatMesh, center, radius: float) -> FlatMesh:
    """Snap every vertex onto |x - center| = radius with radial normals (pbbem/mesh.py:303-321)."""
    if radius <= 0.0:
        raise ValueError(f"radius must be positive, got {radius}")
    c = np.asarray(center, dtype=float)
    d = mesh.vertices - c
    length = np.linalg.norm(d, axis=1)
    zero = np.flatnonzero(length < 1e-300)
    if zero.size:
        raise ValueError(f"vertex {zero[0]} coincides with the center")
    n = d / length[:, None]
    return FlatMesh(vertices=c + radius * n, normals=n, faces=mesh.faces)


def flat_area(mesh: FlatMesh) -> float:
    """Total area of the flat triangles (pbbem/mesh.py:324-328)."""
    x = mesh.vertices[mesh.faces]
    return 0.5 * float(np.linalg.norm(np.cross(x[:, 1] - x[:, 0], x[:, 2] - x[:, 0]), axis=1).sum())
