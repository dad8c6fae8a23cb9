"""MSMS .vert/.face and charge-file ingest against the
reference's own writer/reader outputs (tests/golden/msms.npz)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import golden
from paper_1301_5914_b200 import (FlatMesh, MeshFormatError, flat_area, icosahedral_sphere,
                                  parse_charges, parse_msms, radial_project, write_msms)


@pytest.fixture(scope="module")
def g():
    return golden("msms")


def test_writer_matches_reference_text(g):
    vert, face = write_msms(FlatMesh(g["vertices"], g["normals"], g["faces"]))
    assert vert == str(g["vert_text"]) and face == str(g["face_text"])


def test_round_trip_is_exact(g):
    m = parse_msms(str(g["vert_text"]), str(g["face_text"]))
    assert np.array_equal(m.vertices, g["vertices"])
    assert np.array_equal(m.faces, g["faces"])
    assert np.abs(m.normals - g["normals"]).max() <= 1e-15


def test_msms_headers_comments_three_digit_normals(g):
    m = parse_msms(str(g["messy_vert"]), str(g["messy_face"]))
    assert np.array_equal(m.vertices, g["parsed_vertices"])
    assert np.array_equal(m.normals, g["parsed_normals"])
    assert np.array_equal(m.faces, g["parsed_faces"])


def test_malformed_inputs_raise_like_reference(g):
    cases = (("1.0 0.0 0.0 0.6 0.6 0.6\n2.0 nope 0.0 0.6 0.6 0.6\n", "1 1 1\n"),
             ("1.0 0.0 0.0 0.6 0.6 0.6\n" * 3, "0 1 2\n"),
             ("1 0 0 0 0 0\n" * 3, "1 2 3\n"), ("# nothing\n", "1 2 3\n"),
             ("1.0 0.0 0.0 0.6 0.6 0.6\n", "# none\n"))
    for (v, f), expect in zip(cases, g["errors"]):
        with pytest.raises(MeshFormatError) as info:
            parse_msms(v, f)
        assert f"MeshFormatError: {info.value}" == str(expect)


def test_charges(g):
    c = parse_charges(str(g["charges_text"]))
    assert np.array_equal(c.positions, g["charges_pos"]) and np.array_equal(c.charges, g["charges_q"])
    with pytest.raises(MeshFormatError, match="charge line 1"):
        parse_charges("1 2 3\n")
    with pytest.raises(MeshFormatError, match="charge line 2"):
        parse_charges("0 0 0 1\n1 2 x 4\n")
    assert len(parse_charges("# empty\n")) == 0


@settings(max_examples=20, deadline=None)
@given(level=st.integers(0, 3), radius=st.floats(0.5, 40.0))
def test_round_trip_property(level, radius):
    m = icosahedral_sphere(level, radius)
    back = parse_msms(*write_msms(m))
    assert np.array_equal(back.vertices, m.vertices) and np.array_equal(back.faces, m.faces)


def test_radial_project_and_area():
    m = icosahedral_sphere(2, 3.0)
    p = radial_project(m, (0, 0, 0), 2.0)
    assert np.allclose(np.linalg.norm(p.vertices, axis=1), 2.0)
    assert np.abs(radial_project(p, (0, 0, 0), 2.0).vertices - p.vertices).max() <= 1e-14
    a2, a3 = flat_area(icosahedral_sphere(2, 1.0)), flat_area(icosahedral_sphere(3, 1.0))
    assert a2 < a3 < 4 * np.pi
    with pytest.raises(ValueError, match="coincides"):
        radial_project(FlatMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.eye(3), [[0, 1, 2]]), (0, 0, 0), 1.0)


def _both(v, f):
    from paper_1301_5914_b200.mesh import _parse_msms_native, _parse_msms_python

    fast = _parse_msms_native(v, f)
    try:
        slow = _parse_msms_python(v, f)
    except MeshFormatError:
        slow = None
    return fast, slow


def test_native_scanner_matches_line_parser(g):
    """The library's one-pass scanner (parse_msms's fast path) reads exactly
    what the line-by-line parser reads: reference texts, messy headers and
    comments, CRLF line ends, and a written icosphere."""
    cases = [(str(g["vert_text"]), str(g["face_text"])), (str(g["messy_vert"]), str(g["messy_face"])),
             write_msms(icosahedral_sphere(3, 2.0))]
    cases.append(tuple(t.replace("\n", "\r\n") for t in cases[0]))
    for v, f in cases:
        fast, slow = _both(v, f)
        assert fast is not None and slow is not None
        assert np.array_equal(fast[0], slow[0]) and np.array_equal(fast[1], slow[1])


def test_native_scanner_defers_when_unsure():
    """Whatever the two readers could disagree on, or the line parser would
    reject, the scanner hands back to the line parser."""
    ok = "1.0 0.0 0.0 0.6 0.6 0.6\n2.0 0.0 0.0 0.6 0.6 0.6\n3.0 1.0 0.0 0.6 0.6 0.6\n"
    face = "1 2 3\n"
    for v, f in ((ok.replace("2.0", "2_0"), face), (ok.replace("2.0", "0x2p0"), face),
                 (ok.replace("\n", "\r", 1), face), (ok + "4.0 0 0 0.6 0.6 0.6 é\n", face),
                 (ok.replace("3.0", "nan(7)"), face), (ok, "1 2 3_0\n"), (ok, "0 1 2\n"),
                 (ok.replace("0.0 0.0 0.6", "0.0 x 0.6", 1), face), (ok, "1 2 99999999999999999999\n")):
        from paper_1301_5914_b200.mesh import _parse_msms_native

        assert _parse_msms_native(v, f) is None, (v, f)


_word = st.sampled_from(["1.5", "-2", "+.5", "3e2", "1e-400", "inf", "-Infinity", "nan", "abc", "#", "# c",
                         "0", "07", "2.", ".", "-", "e5", "1e", "12", "x1"])


@settings(max_examples=200, deadline=None)
@given(lines=st.lists(st.lists(_word, min_size=0, max_size=9), min_size=0, max_size=12),
       flines=st.lists(st.lists(st.sampled_from(["1", "2", "3", "4", "0", "-1", "+2", "2.0", "a", "#"]),
                                min_size=0, max_size=5), min_size=0, max_size=8))
def test_native_scanner_property(lines, flines):
    v = "\n".join(" ".join(l) for l in lines)
    f = "\n".join(" ".join(l) for l in flines)
    fast, slow = _both(v, f)
    if fast is not None:  # whenever the scanner answers, it answers like the line parser
        assert slow is not None
        assert np.array_equal(fast[0], slow[0], equal_nan=True) and np.array_equal(fast[1], slow[1])
