"""CPU tests of the host-side logic: input types and validation, generators,
quadrature constants, partitioning, config validation, and the fail-loud rule."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import golden
from paper_1301_5914_b200 import (ChargeSystem, FlatMesh, MeshValidationError, PhysicalParams,
                                  SolverConfig, duffy_rule, gauss_radau_rule, icosahedral_sphere,
                                  partition_targets, surface_potential_error, convergence_order)
from paper_1301_5914_b200.quadrature import BASIS_COEF, REFERENCE_NODES, shape_tables
from paper_1301_5914_b200.surfaces import StarShape, baseline_config


def test_icosphere_matches_reference_bitwise():
    g = golden("c1")  # the reference's icosahedral_sphere(3, 2.0) arrays
    m = icosahedral_sphere(3, 2.0)
    assert np.array_equal(m.vertices, g["vertices"])
    assert np.array_equal(m.normals, g["normals"])
    assert np.array_equal(m.faces, g["faces"])
    for lv in range(6):
        m = icosahedral_sphere(lv)
        assert m.n_faces == 20 * 4**lv and m.n_vertices == m.n_faces // 2 + 2
        m.validate()


def test_mesh_validation_messages():
    m = icosahedral_sphere(1)
    bad_n = m.normals.copy()
    bad_n[3] *= 1.01
    with pytest.raises(MeshValidationError, match="normal 3 has length"):
        FlatMesh(m.vertices, bad_n, m.faces).validate()
    f = m.faces.copy()
    f[5, 1] = 999
    with pytest.raises(MeshValidationError, match="face 5 references a vertex outside"):
        FlatMesh(m.vertices, m.normals, f).validate()
    f = m.faces.copy()
    f[7] = f[7][::-1]
    with pytest.raises(MeshValidationError, match="face 7 is oriented against"):
        FlatMesh(m.vertices, m.normals, f).validate()
    with pytest.raises(MeshValidationError, match="not closed"):
        FlatMesh(m.vertices, m.normals, m.faces[:-1]).validate()


def test_inputs_are_immutable():
    m = icosahedral_sphere(0)
    with pytest.raises(ValueError):
        m.vertices[0, 0] = 1.0
    c = ChargeSystem([[0, 0, 0]], [1.0])
    with pytest.raises(ValueError):
        c.charges[0] = 2.0
    with pytest.raises(ValueError, match="positions but"):
        ChargeSystem([[0, 0, 0]], [1.0, 2.0])


def test_rules_match_reference_constants():
    g = golden("sphere_l1_mixed")
    r = gauss_radau_rule()
    assert r.name == "conical-radau-4" and r.degree == 3 and len(r) == 4
    bary = np.stack([1 - r.points[:, 0] - r.points[:, 1], r.points[:, 0], r.points[:, 1]], 1)
    assert np.array_equal(bary, g["reg_bary"])
    d = duffy_rule(4)
    assert d.degree == 6 and len(d) == 16
    dbary = np.stack([1 - d.points[:, 0] - d.points[:, 1], d.points[:, 0], d.points[:, 1]], 1)
    assert np.array_equal(dbary, g["duf_bary"])
    for n in range(1, 9):
        assert abs(duffy_rule(n).weights.sum() - 0.5) < 1e-14


def test_cubic_basis_is_lagrange():
    N, Nr, Ns = shape_tables(REFERENCE_NODES)
    assert np.abs(N - np.eye(10)).max() < 1e-13
    assert np.abs(N.sum(axis=1) - 1).max() < 1e-13
    assert np.abs(Nr.sum(axis=1)).max() < 1e-12 and np.abs(Ns.sum(axis=1)).max() < 1e-12
    assert BASIS_COEF.shape == (10, 10)


def test_partition_examples():
    assert partition_targets(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert partition_targets(3, 5) == [(0, 1), (1, 2), (2, 3), (3, 3), (3, 3)]
    assert partition_targets(0, 2) == [(0, 0), (0, 0)]
    with pytest.raises(ValueError):
        partition_targets(5, 0)
    with pytest.raises(ValueError):
        partition_targets(-1, 2)


@settings(max_examples=60, deadline=None)
@given(n=st.integers(0, 300), w=st.integers(1, 17))
def test_partition_property(n, w):
    r = partition_targets(n, w)
    assert len(r) == w and r[0][0] == 0 and r[-1][1] == n
    sizes = [hi - lo for lo, hi in r]
    assert max(sizes) - min(sizes) <= 1 and all(a[1] == b[0] for a, b in zip(r, r[1:]))


def test_config_and_params_validation():
    with pytest.raises(ValueError, match="scheme"):
        SolverConfig(scheme="dense")
    with pytest.raises(ValueError, match="tolerance"):
        SolverConfig(tolerance=1.5)
    with pytest.raises(ValueError, match="restart"):
        SolverConfig(restart=0)
    with pytest.raises(ValueError, match="max_iterations"):
        SolverConfig(max_iterations=0)
    with pytest.raises(ValueError, match="workers"):
        SolverConfig(workers=0)
    assert SolverConfig(workers=3).worker_count() == 3
    with pytest.raises(ValueError, match="eps1"):
        PhysicalParams(0.0, 80.0, 0.1)
    with pytest.raises(ValueError, match="kappa"):
        PhysicalParams(1.0, 80.0, -0.1)
    assert PhysicalParams(2.0, 80.0, 0.1).eps == 2.0 / 80.0


def test_error_metrics():
    assert surface_potential_error([1.0, 2.0], [1.0, 2.5]) == pytest.approx(0.2)
    with pytest.raises(ZeroDivisionError):
        surface_potential_error([1.0], [0.0])
    assert convergence_order(10, 40, 1e-2, 1e-4) == pytest.approx(np.log(100) / np.log(4))


@pytest.mark.parametrize("index", [3, 4])
def test_star_surfaces_are_valid(index):
    cfg = baseline_config(index, level=3)
    cfg.mesh.validate()
    q = cfg.charges
    assert abs(q.charges.sum()) < 1e-9
    shape = StarShape.from_seed({3: 16.0, 4: 30.0}[index], seed=3)
    u = q.positions / np.linalg.norm(q.positions, axis=1)[:, None]
    p, _ = shape.perturbation(u)
    assert np.all(np.linalg.norm(q.positions, axis=1) < 0.8 * shape.radius * (1 + p))


def test_star_normals_are_surface_normals():
    shape = StarShape.from_seed(16.0, seed=3)
    rng = np.random.default_rng(1)
    u = rng.standard_normal((100, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    p, gp = shape.perturbation(u)
    n = u - gp / (1 + p)[:, None]
    n /= np.linalg.norm(n, axis=1)[:, None]

    def X(v):
        v = v / np.linalg.norm(v, axis=1)[:, None]
        q, _ = shape.perturbation(v)
        return (16 * (1 + q))[:, None] * v

    t = np.cross(u, [0.3, 0.5, 0.8])
    t /= np.linalg.norm(t, axis=1)[:, None]
    for tt in (t, np.cross(u, t)):
        d = (X(u + 1e-6 * tt) - X(u - 1e-6 * tt)) / 2e-6
        assert np.abs(np.einsum("ij,ij->i", d, n)).max() < 1e-7 * np.linalg.norm(d, axis=1).max()


def test_config_table():
    c1 = baseline_config(1)
    assert (c1.mesh.n_vertices, c1.mesh.n_faces, c1.restart) == (642, 1280, 10)
    c2 = baseline_config(2)
    assert c2.mesh.n_faces == 5120 and len(c2.charges) == 8
    assert np.all(np.abs(c2.charges.charges) == 1.0)
    assert np.all(np.linalg.norm(c2.charges.positions, axis=1) < 1.2)


def test_cli_restart_flag_is_honoured_even_at_100():
    from paper_1301_5914_b200.cli import _restart, build_parser

    assert _restart(None, None) == 100
    assert _restart(None, 4) == 20  # BASELINE config 4's restart
    assert _restart(100, 4) == 100  # an explicit --restart 100 wins over the config
    assert _restart(7, None) == 7
    args = build_parser().parse_args(["solve", "--config", "4"])
    assert args.restart is None


def test_module_surface_matches_the_reference_package():
    """Every public name of every pbbem module (tests/golden/pbbem_api.json, read
    from the reference sources by make_api_surface.py) exists in the same-named
    module here, every public function takes the reference's positional
    parameters in the reference's order (extra trailing ones must have
    defaults), and every record class has the reference's fields: the drop-in
    surface, checked without a GPU."""
    import dataclasses
    import importlib
    import inspect
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pbbem_api.json")
    with open(path) as fh:
        api = json.load(fh)
    assert set(api["names"]) == {"cli", "geometry", "kernels", "kirkwood", "mesh", "quadrature", "report",
                                 "solver"}
    problems = []
    for module, names in api["names"].items():
        mod = importlib.import_module("paper_1301_5914_b200." + module)
        problems += [f"{module}.{n} missing" for n in names if not hasattr(mod, n)]
        for fn, ref in api["signatures"].get(module, {}).items():
            params = [p for p in inspect.signature(getattr(mod, fn)).parameters.values()
                      if p.kind in (p.POSITIONAL_ONLY, p.POSITIONAL_OR_KEYWORD)]
            if [p.name for p in params[:len(ref)]] != ref:
                problems.append(f"{module}.{fn}{[p.name for p in params]} != {ref}")
            problems += [f"{module}.{fn}: extra parameter {p.name} has no default" for p in params[len(ref):]
                         if p.default is inspect.Parameter.empty]
        for cls, ref in api["fields"].get(module, {}).items():
            ours = getattr(mod, cls)
            if dataclasses.is_dataclass(ours):
                have = [f.name for f in dataclasses.fields(ours)]
                if have[:len(ref)] != ref:
                    problems.append(f"{module}.{cls} fields {have} != {ref}")
            else:  # DiscretizedProblem: device-backed, caches exported on first access
                src = inspect.getsource(ours)
                problems += [f"{module}.{cls}.{f} missing" for f in ref
                             if not (hasattr(ours, f) or f"self.{f}" in src or f'"{f}"' in src)]
    assert not problems, problems
