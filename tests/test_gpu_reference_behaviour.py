"""Behaviour the reference's own solver tests pin (ref tests/test_solver.py),
re-run through the GPU path: discretisation bookkeeping, the singular-face
partition, closed-form and symmetry properties of the device RHS, and the
accuracy ordering of the two schemes.  Numeric gates are the reference's."""
import numpy as np
import pytest

from paper_1301_5914_b200 import (ChargeSystem, FlatMesh, MeshValidationError, PhysicalParams,
                                  SolverConfig, assemble_rhs, discretize, icosahedral_sphere, solvation_energy,
                                  solve, surface_potential_error)
from paper_1301_5914_b200.kirkwood import SphereProblem, kirkwood_centered

pytestmark = pytest.mark.gpu

WATER = PhysicalParams(1.0, 80.0, 0.0)
CENTERED = ChargeSystem([[0.0, 0.0, 0.0]], [1.0])
NONE = ChargeSystem(np.zeros((0, 3)), np.zeros(0))


def test_discretize_counts_and_collocation():
    """ref test_solver.py:80-95."""
    mesh = icosahedral_sphere(1, 2.0)
    hobi = discretize(mesh, WATER, CENTERED, SolverConfig(scheme="hobi"))
    assert hobi.n_collocation == mesh.n_vertices and hobi.n_unknowns == 2 * mesh.n_vertices
    assert np.array_equal(hobi.colloc_pos, mesh.vertices)
    assert np.array_equal(hobi.colloc_nrm, mesh.normals)
    assert len(hobi.elements) == mesh.n_faces
    lobi = discretize(mesh, WATER, CENTERED, SolverConfig(scheme="lobi"))
    assert lobi.n_collocation == mesh.n_faces
    assert np.abs(lobi.colloc_pos - mesh.vertices[mesh.faces].mean(axis=1)).max() <= 1e-15
    assert np.abs(np.linalg.norm(lobi.colloc_nrm, axis=1) - 1.0).max() <= 1e-12


def test_discretize_rejects_open_mesh():
    """ref test_solver.py:98-105: an open surface never reaches the device."""
    v = np.array([[1.0, 1.0, 1.0], [1.0, -1.0, -1.0], [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]]) / np.sqrt(3.0)
    faces = np.array([[0, 1, 2], [0, 3, 1], [0, 2, 3]])
    with pytest.raises(MeshValidationError):
        discretize(FlatMesh(v, v.copy(), faces), WATER, CENTERED, SolverConfig())


def test_singular_faces_partition():
    """ref test_solver.py:117-133: the device pair table lists exactly the
    faces incident to each vertex, face-ordered; LOBI has none."""
    mesh = icosahedral_sphere(0)
    prob = discretize(mesh, WATER, NONE, SolverConfig(scheme="hobi"))
    for v in range(mesh.n_vertices):
        got = prob.singular_faces(v)
        assert np.array_equal(np.sort(got), np.nonzero((mesh.faces == v).any(axis=1))[0])
        assert np.array_equal(got, np.sort(got))
    lobi = discretize(mesh, WATER, NONE, SolverConfig(scheme="lobi"))
    with pytest.raises(ValueError):
        lobi.singular_faces(0)


def test_rhs_centred_charge_closed_form():
    """ref test_solver.py:204-213: S1/eps1 = 1/(8 pi eps1), S2/eps1 = -1/(16 pi eps1) at radius 2."""
    mesh = icosahedral_sphere(1, 2.0)
    for eps1 in (1.0, 4.0):
        prob = discretize(mesh, PhysicalParams(eps1, 80.0, 0.0), CENTERED, SolverConfig())
        rhs = assemble_rhs(prob)
        t = prob.n_collocation
        assert rhs.shape == (2 * t,)
        assert np.abs(rhs[:t] - 1.0 / (8.0 * np.pi * eps1)).max() <= 1e-14
        assert np.abs(rhs[t:] + 1.0 / (16.0 * np.pi * eps1)).max() <= 1e-14


def test_rhs_mirror_antisymmetry():
    """ref test_solver.py:216-233: a +/- pair mirrored in z makes the source odd."""
    mesh = icosahedral_sphere(1, 2.0)
    prob = discretize(mesh, WATER, ChargeSystem([[0, 0, 0.6], [0, 0, -0.6]], [1.0, -1.0]), SolverConfig())
    rhs = assemble_rhs(prob)
    t = prob.n_collocation
    index = {tuple(np.round(v, 9)): i for i, v in enumerate(prob.colloc_pos)}
    mirror = np.array([index[tuple(np.round(v * [1, 1, -1], 9))] for v in prob.colloc_pos])
    scale = np.abs(rhs).max()
    assert np.abs(rhs[:t][mirror] + rhs[:t]).max() <= 1e-12 * scale
    assert np.abs(rhs[t:][mirror] + rhs[t:]).max() <= 1e-12 * scale


def test_hobi_beats_lobi_and_refinement_helps():
    """ref test_solver.py:406-426: HOBI's trace error is < 1/100 of LOBI's on
    the same mesh, and refining HOBI moves the energy towards the closed form."""
    sphere = SphereProblem(radius=2.0, params=WATER, charges=CENTERED)
    _, exact_phi, _ = kirkwood_centered(sphere)
    hp, hs = solve(icosahedral_sphere(2, 2.0), WATER, CENTERED, SolverConfig(scheme="hobi", workers=1))
    lp, ls = solve(icosahedral_sphere(2, 2.0), WATER, CENTERED, SolverConfig(scheme="lobi", workers=1))
    err_h = surface_potential_error(hs.phi, exact_phi(hp.colloc_pos))
    err_l = surface_potential_error(ls.phi, exact_phi(lp.colloc_pos))
    assert err_h < err_l / 100.0
    exact = -81.98017625
    fp, fs = solve(icosahedral_sphere(3, 2.0), WATER, CENTERED, SolverConfig(scheme="hobi", workers=1))
    assert abs(solvation_energy(fp, fs) - exact) < abs(solvation_energy(hp, hs) - exact)


def test_zero_charge_lobi_solve_is_trivial():
    """ref test_solver.py:429-436."""
    prob, sol = solve(icosahedral_sphere(1), WATER, NONE, SolverConfig(scheme="lobi", workers=1))
    assert np.all(sol.vector == 0.0) and sol.iterations == 0
    assert solvation_energy(prob, sol) == 0.0
