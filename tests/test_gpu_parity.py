"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (tests/golden, produced by running pbbem itself) and the numpy oracle.

Tolerances (north star, BASELINE.json): matvec <= 1e-10 relative L2 (we hold
1e-12); potentials and energy <= 1e-8 relative at equal GMRES tolerance;
geometry caches bit-exact (the device geometry replays numpy's rounding).
"""

import numpy as np
import pytest

from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1301_5914_b200")
from paper_1301_5914_b200 import (  # noqa: E402
    ChargeSystem,
    DegenerateArcError,
    FlatMesh,
    GmresNonConvergence,
    PhysicalParams,
    SolverConfig,
    apply_rows,
    assemble_rhs,
    discretize,
    gmres_solve,
    make_operator,
    matvec_hobi,
    matvec_lobi,
    solvation_energy,
    solve,
)
from paper_1301_5914_b200.solver import SurfaceSolution  # noqa: E402
from paper_1301_5914_b200 import _native as N  # noqa: E402

MATVEC_TOL = 1e-12
SOLVE_TOL = 1e-8


def _problem(g, scheme="hobi", **kw):
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    e1, e2, k = g["params"]
    charges = ChargeSystem(g["qpos"], g["q"])
    return discretize(mesh, PhysicalParams(e1, e2, k), charges,
                      SolverConfig(scheme=scheme, workers=1, **kw))


def test_kernel_values_match_reference():
    """Device kernel_values_d vs kernels.kernel_values_d (kernels.py:99-130)."""
    g = golden("kernels")
    n = g["d"].shape[0]
    for tag in "abcd":
        e1, e2, kap = g["params_" + tag]
        k = np.empty((4, n))
        N.check(N.load().hobi_kernel_values(0, N.dptr(N.f64(g["d"])), N.dptr(N.f64(g["nx"])),
                                            N.dptr(N.f64(g["ny"])), n, e1, e2, kap, N.dptr(k)))
        ref = g["K_" + tag]
        d, nx, ny = g["d"], g["nx"], g["ny"]
        r2 = np.einsum("ij,ij->i", d, d)
        r = np.sqrt(r2)
        kr = kap * r
        a = np.expm1(-kr) + kr * np.exp(-kr)
        b = 3.0 * np.expm1(-kr) + kr * np.exp(-kr) * (3.0 + kr)
        dnx, dny = np.einsum("ij,ij->i", d, nx), np.einsum("ij,ij->i", d, ny)
        inv3 = 1.0 / (4.0 * np.pi * r2 * r)
        # a, b are O((kr)^2) cancellations (kernels.py:117-120): any implementation's
        # rounding in them is ~ulp/kr relative, then K4 adds the cancellation
        # between its two terms; bound the error by the terms' magnitudes.
        cond = 1.0 + 1.0 / np.maximum(kr, 1e-300)
        k4_scale = (np.abs(b * dnx * dny / r2) + np.abs(a * np.einsum("ij,ij->i", nx, ny))) * inv3
        bound = [1e-14 * np.abs(ref[0]), 1e-13 * np.abs(ref[1]), 1e-13 * np.abs(ref[2]),
                 4e-15 * cond * k4_scale]
        for i in range(4):
            nz = ref[i] != 0.0
            assert np.all(k[i][~nz] == 0.0)  # identity medium / kappa=0: exact zeros
            err = np.abs(k[i] - ref[i])
            assert np.all(err[nz] <= bound[i][nz]), (tag, i, (err[nz] / bound[i][nz]).max())


@pytest.mark.parametrize("name", ["sphere_l1_mixed", "star_l2", "uv_sphere"])
def test_geometry_caches_bit_exact(name):
    g = golden(name)
    prob = _problem(g)
    for key in ("reg_pos", "reg_nrm", "reg_w", "duf_pos", "duf_nrm", "duf_w"):
        got, ref = getattr(prob, key), g[key]
        assert got.shape == ref.shape
        assert np.array_equal(got, ref), (key, np.abs(got - ref).max())
    for key in ("pair_vertex", "pair_face", "pair_gverts", "pair_starts"):
        assert np.array_equal(getattr(prob, key), g[key]), key


@pytest.mark.parametrize("name", ["sphere_l1_mixed", "star_l2", "star_l3", "c1", "c2", "uv_sphere"])
def test_matvec_matches_reference(name):
    g = golden(name)
    prob = _problem(g)
    got = matvec_hobi(prob, g["u"])
    assert rel_l2(got, g["Au"]) <= MATVEC_TOL


@pytest.mark.parametrize("name", ["sphere_l1_mixed", "star_l2", "star_l3", "c1", "c2", "uv_sphere"])
def test_rhs_matches_reference(name):
    g = golden(name)
    prob = _problem(g)
    assert rel_l2(assemble_rhs(prob), g["rhs"]) <= 1e-14


@pytest.mark.parametrize("name", ["star_l2", "star_l3", "c1", "c2", "uv_sphere"])
def test_solve_matches_reference(name):
    g = golden(name)
    prob = _problem(g, restart=int(g["restart"]))
    cfg = SolverConfig(workers=1, restart=int(g["restart"]))
    with make_operator(prob, cfg) as op:
        sol = gmres_solve(op, assemble_rhs(prob), cfg)
    assert sol.iterations == int(g["iterations"])
    assert sol.matvecs == int(g["matvecs"])
    assert rel_l2(sol.phi, g["phi"]) <= SOLVE_TOL
    assert rel_l2(sol.dphi_dn, g["dphi"]) <= SOLVE_TOL
    e = solvation_energy(prob, sol)
    assert abs(e - float(g["energy"])) <= SOLVE_TOL * abs(float(g["energy"]))
    if "kirkwood_energy" in g:  # analytic sphere answer, HOBI discretisation error ~1e-3
        assert abs(e - float(g["kirkwood_energy"])) <= 5e-3 * abs(float(g["kirkwood_energy"]))


def test_identity_medium_is_exact_identity():
    """eps1 = eps2, kappa = 0: every kernel vanishes, operator == I bitwise (test_solver.py:138-148)."""
    g = golden("star_l2")
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    rng = np.random.default_rng(0)
    for scheme, apply in (("hobi", matvec_hobi), ("lobi", matvec_lobi)):
        prob = discretize(mesh, PhysicalParams(3.0, 3.0, 0.0), ChargeSystem(np.zeros((0, 3)), []),
                          SolverConfig(scheme=scheme))
        for _ in range(5):
            u = rng.standard_normal(prob.n_unknowns)
            assert np.abs(apply(prob, u) - u).max() == 0.0


def test_row_split_bitwise_deterministic():
    """Any partition of rows reproduces the unsplit operator bitwise (test_solver.py:333-359)."""
    g = golden("star_l3")
    prob = _problem(g)
    u = g["u"]
    full = matvec_hobi(prob, u)
    T = prob.n_collocation
    for workers in (2, 3, 4, 8, 700):
        with make_operator(prob, SolverConfig(workers=workers)) as op:
            assert np.array_equal(op(u), full), workers
        from paper_1301_5914_b200 import partition_targets

        parts = [apply_rows(prob, u, lo, hi) for lo, hi in partition_targets(T, workers)]
        assert np.array_equal(np.concatenate([p[0] for p in parts]), full[:T])
        assert np.array_equal(np.concatenate([p[1] for p in parts]), full[T:])


def test_degenerate_face_reported_like_reference():
    g = golden("degenerate")
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    with pytest.raises(DegenerateArcError) as info:
        discretize(mesh, PhysicalParams(1.0, 80.0, 0.0), ChargeSystem(np.zeros((0, 3)), []),
                   SolverConfig(scheme="hobi"))
    assert f"DegenerateArcError: {info.value}" == str(g["message"])


def test_gmres_host_callable_paths():
    """gmres_solve on arbitrary callables (test_solver.py:246-297)."""
    rng = np.random.default_rng(3)
    a = np.eye(8) + 0.3 * rng.standard_normal((8, 8))
    b = rng.standard_normal(8)
    sol = gmres_solve(lambda v: a @ v, b, SolverConfig(tolerance=1e-12, workers=1))
    assert np.abs(sol.vector - np.linalg.solve(a, b)).max() <= 1e-9
    assert sol.iterations <= 8 and sol.residual <= 1e-12
    rng = np.random.default_rng(4)
    a = np.eye(12) + 0.1 * rng.standard_normal((12, 12))
    b = rng.standard_normal(12)
    sol = gmres_solve(lambda v: a @ v, b, SolverConfig(tolerance=1e-12, restart=3, max_iterations=500))
    assert np.abs(a @ sol.vector - b).max() <= 1e-10 and sol.iterations > 3
    b = np.array([1.0, -2.0, 0.5, 3.0])
    sol = gmres_solve(lambda v: v, b, SolverConfig())
    assert np.array_equal(sol.vector, b) and sol.iterations == 1
    sol = gmres_solve(lambda v: v, np.zeros(6), SolverConfig())
    assert np.all(sol.vector == 0.0) and sol.iterations == 0 and sol.residual == 0.0
    with pytest.raises(ValueError, match="even"):
        gmres_solve(lambda v: v, np.ones(5), SolverConfig())
    rng = np.random.default_rng(5)
    a = np.eye(20) + 2.5 * rng.standard_normal((20, 20))
    with pytest.raises(GmresNonConvergence) as info:
        gmres_solve(lambda v: a @ v, rng.standard_normal(20),
                    SolverConfig(tolerance=1e-14, max_iterations=3))
    assert 0.0 < info.value.best_residual <= 1.0


def test_gmres_matches_oracle_gmres_on_dense():
    import hobi_oracle as O

    rng = np.random.default_rng(9)
    a = np.eye(40) + 0.05 * rng.standard_normal((40, 40))
    b = rng.standard_normal(40)
    x, its, rel, nmv = O.gmres(lambda v: a @ v, b, tol=1e-10, restart=7, max_it=400)
    sol = gmres_solve(lambda v: a @ v, b, SolverConfig(tolerance=1e-10, restart=7, max_iterations=400))
    assert sol.iterations == its and sol.matvecs == nmv
    assert rel_l2(sol.vector, x) <= 1e-12


def test_lobi_matches_oracle():
    import hobi_oracle as O

    g = golden("star_l2")
    prob = _problem(g, scheme="lobi")
    o = O.discretize(g["vertices"], g["normals"], g["faces"], *g["params"], scheme="lobi")
    rng = np.random.default_rng(2)
    u = rng.standard_normal(prob.n_unknowns)
    assert rel_l2(matvec_lobi(prob, u), O.matvec(o, u)) <= MATVEC_TOL
    assert rel_l2(assemble_rhs(prob), O.rhs(O.discretize(
        g["vertices"], g["normals"], g["faces"], *g["params"], g["qpos"], g["q"], scheme="lobi"))) <= 1e-14


def test_born_sphere_frozen_energy():
    """Known answer of the reference test-suite (test_solver.py:375-392)."""
    from paper_1301_5914_b200 import icosahedral_sphere

    water = PhysicalParams(1.0, 80.0, 0.0)
    prob, sol = solve(icosahedral_sphere(2, 2.0), water, ChargeSystem([[0.0, 0.0, 0.0]], [1.0]),
                      SolverConfig(workers=1))
    assert solvation_energy(prob, sol) == pytest.approx(-81.98131581725495, rel=1e-9)
    assert 4 <= sol.iterations <= 9
    from paper_1301_5914_b200 import surface_potential_error
    from paper_1301_5914_b200.kirkwood import SphereProblem, kirkwood_centered

    _, exact_phi, _ = kirkwood_centered(SphereProblem(2.0, water, ChargeSystem([[0.0, 0.0, 0.0]], [1.0])))
    assert surface_potential_error(sol.phi, exact_phi(prob.colloc_pos)) == pytest.approx(7.105e-5, rel=0.05)
    prob, sol = solve(icosahedral_sphere(2, 2.0), water, ChargeSystem([[0.0, 0.0, 0.0]], [1.0]),
                      SolverConfig(scheme="lobi", workers=1))
    assert solvation_energy(prob, sol) == pytest.approx(-86.3199784371863, rel=1e-9)


@pytest.mark.parametrize("index", [3, 4, 5])
def test_large_config_rows_vs_oracle(index):
    """Configs 3-5 at full size (config 5: 327,680 triangles, 2.1e11 pairs per
    matvec): sampled rows against the oracle's _apply_range."""
    import hobi_oracle as O
    from paper_1301_5914_b200.surfaces import baseline_config

    cfg = baseline_config(index)
    prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges,
                      SolverConfig(workers=1))
    o = O.discretize(cfg.mesh.vertices, cfg.mesh.normals, cfg.mesh.faces, cfg.eps1, cfg.eps2,
                     cfg.kappa, check=False)
    u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
    full = matvec_hobi(prob, u)
    T = prob.n_collocation
    for lo in (0, T // 2, T - 37):
        hi = lo + 37
        r1, r2 = O.rows(o, u, lo, hi)
        assert rel_l2(full[lo:hi], r1) <= MATVEC_TOL
        assert rel_l2(full[T + lo:T + hi], r2) <= MATVEC_TOL


def test_sphere_solves_against_kirkwood():
    """Configs 1-2 validated against the analytic series."""
    from paper_1301_5914_b200 import surface_potential_error
    from paper_1301_5914_b200.kirkwood import SphereProblem, kirkwood_series
    from paper_1301_5914_b200.surfaces import baseline_config

    errs = []
    for level in (2, 3, 4):
        cfg = baseline_config(1, level=level)
        params = PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa)
        prob, sol = solve(cfg.mesh, params, cfg.charges, SolverConfig(restart=cfg.restart, workers=1))
        ks = kirkwood_series(SphereProblem(2.0, params, cfg.charges), 40)
        errs.append(surface_potential_error(sol.phi, ks.phi(prob.colloc_pos)))
        assert abs(solvation_energy(prob, sol) - ks.energy) <= 1e-2 * abs(ks.energy)
    assert errs[0] > errs[1] > errs[2] and errs[1] < 1e-4  # refinement converges
    cfg = baseline_config(2)
    params = PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa)
    prob, sol = solve(cfg.mesh, params, cfg.charges, SolverConfig(restart=cfg.restart, workers=1))
    ks = kirkwood_series(SphereProblem(2.0, params, cfg.charges), 40)
    assert ks.converged
    assert surface_potential_error(sol.phi, ks.phi(prob.colloc_pos)) < 5e-3
    assert abs(solvation_energy(prob, sol) - ks.energy) <= 5e-3 * abs(ks.energy)


@pytest.mark.parametrize("name", ["star_l1_duffy6", "star_l2_rule9"])
def test_quadrature_variants_bit_exact_caches_and_matvec(name):
    """SolverConfig.duffy_points / regular_rule other than the defaults (solver.py:67-68)."""
    from paper_1301_5914_b200 import TriangleRule

    g = golden(name)
    kw = {"duffy_points": int(g["duffy"])}
    if "rule_points" in g:
        kw["regular_rule"] = TriangleRule(g["rule_points"], g["rule_weights"], "custom",
                                          int(g["rule_degree"]))
    prob = _problem(g, **kw)
    for key in ("reg_pos", "reg_nrm", "reg_w", "duf_pos", "duf_nrm", "duf_w"):
        assert np.array_equal(getattr(prob, key), g[key]), key
    assert rel_l2(matvec_hobi(prob, g["u"]), g["Au"]) <= MATVEC_TOL
    if "phi" in g:
        cfg = SolverConfig(workers=1, restart=int(g["restart"]), **kw)
        with make_operator(prob, cfg) as op:
            sol = gmres_solve(op, assemble_rhs(prob), cfg)
        assert sol.iterations == int(g["iterations"])
        assert rel_l2(sol.phi, g["phi"]) <= SOLVE_TOL
        e = solvation_energy(prob, sol)
        assert abs(e - float(g["energy"])) <= SOLVE_TOL * abs(float(g["energy"]))


def test_lobi_solve_matches_reference():
    g = golden("star_l2_lobi")
    prob = _problem(g, scheme="lobi")
    assert rel_l2(matvec_lobi(prob, g["u"]), g["Au"]) <= MATVEC_TOL
    cfg = SolverConfig(scheme="lobi", workers=1, restart=int(g["restart"]))
    with make_operator(prob, cfg) as op:
        sol = gmres_solve(op, assemble_rhs(prob), cfg)
    assert sol.iterations == int(g["iterations"]) and sol.matvecs == int(g["matvecs"])
    assert rel_l2(sol.phi, g["phi"]) <= SOLVE_TOL
    e = solvation_energy(prob, sol)
    assert abs(e - float(g["energy"])) <= SOLVE_TOL * abs(float(g["energy"]))


def test_gpu_operator_nonconvergence_and_empty_charges():
    g = golden("star_l2")
    prob = _problem(g)
    cfg = SolverConfig(workers=1, tolerance=1e-14, max_iterations=3, restart=2)
    with make_operator(prob, cfg) as op:
        with pytest.raises(GmresNonConvergence) as info:
            gmres_solve(op, assemble_rhs(prob), cfg)
    assert 0.0 < info.value.best_residual < 1.0
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    empty = discretize(mesh, PhysicalParams(*g["params"]), ChargeSystem(np.zeros((0, 3)), []),
                       SolverConfig())
    assert np.all(assemble_rhs(empty) == 0.0)
    with make_operator(empty, SolverConfig()) as op:
        sol = gmres_solve(op, assemble_rhs(empty), SolverConfig())
    assert sol.iterations == 0 and np.all(sol.vector == 0.0)
    assert solvation_energy(empty, sol) == 0.0


def test_rhs_singularity_reported():
    from paper_1301_5914_b200 import SingularityError

    g = golden("star_l2")
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    prob = discretize(mesh, PhysicalParams(*g["params"]),
                      ChargeSystem([[0.0, 0.0, 0.0], g["vertices"][5]], [1.0, 1.0]), SolverConfig())
    with pytest.raises(SingularityError, match="surface point 5 coincides with charge 1"):
        assemble_rhs(prob)


def test_wrong_length_and_scheme_mismatch():
    g = golden("star_l2")
    prob = _problem(g)
    with pytest.raises(ValueError, match="length"):
        matvec_hobi(prob, np.zeros(prob.n_unknowns + 2))
    with pytest.raises(ValueError):
        matvec_lobi(prob, np.zeros(prob.n_unknowns))


def test_repeated_runs_and_all_sweep_variants_bitwise_identical():
    """Race canary (compute-sanitizer is closed on this pool): the same matvec
    repeated, and under every sweep tiling variant, must agree bit for bit --
    a data race or an order-dependent reduction would show up here first."""
    import ctypes as C

    g = golden("star_l3")
    prob = _problem(g)
    ref = matvec_hobi(prob, g["u"])
    for _ in range(10):
        assert np.array_equal(matvec_hobi(prob, g["u"]), ref)
    lib = N.load()
    n = C.c_int(0)
    lib.hobi_sweep_variant(prob.handle, -1, C.byref(n), None, 0)
    for v in range(n.value):
        N.check(lib.hobi_sweep_variant(prob.handle, v, None, None, 0))
        assert np.array_equal(matvec_hobi(prob, g["u"]), ref), v


def test_sweep_frame_invariance(monkeypatch):
    """The sweep runs in a rotated frame with target normals held as
    (n_x/n_z, n_y/n_z) (csrc/hobi_sweep.cu, Physics::q).  Distances and dot
    products do not depend on the frame: the matvec and the energy computed in
    different frames of the sequence agree to rounding, and each matches the
    reference golden."""
    g = golden("star_l3")
    out = []
    for k in (0, 3, 7):
        monkeypatch.setenv("HOBI_SWEEP_FRAME", str(k))
        prob = _problem(g)
        au = matvec_hobi(prob, g["u"])
        assert np.linalg.norm(au - g["Au"]) / np.linalg.norm(g["Au"]) <= 1e-12, k
        sol = SurfaceSolution(np.asarray(g["phi"], float), np.asarray(g["dphi"], float), "hobi", 0, 0.0)
        assert abs(solvation_energy(prob, sol) - float(g["energy"])) <= 1e-10 * abs(float(g["energy"]))
        out.append((au, solvation_energy(prob, sol)))
        prob.close()
    for au, e in out[1:]:
        assert np.linalg.norm(au - out[0][0]) / np.linalg.norm(out[0][0]) <= 1e-14
        assert abs(e - out[0][1]) <= 1e-13 * abs(out[0][1])


def test_sweep_frame_retry(monkeypatch):
    """Context creation tries the frames of the sequence until every target
    normal has a nonzero z component (csrc/hobi_sweep.cu prepare_targets);
    the HOBI_TEST_FRAME_REJECT hook rejects the first frames: the retry lands
    on a later frame with the same results, and rejecting all of them is a
    clean error, not a wrong answer."""
    g = golden("star_l3")
    monkeypatch.setenv("HOBI_TEST_FRAME_REJECT", "5")
    prob = _problem(g)
    au = matvec_hobi(prob, g["u"])
    assert np.linalg.norm(au - g["Au"]) / np.linalg.norm(g["Au"]) <= 1e-12
    prob.close()
    monkeypatch.setenv("HOBI_TEST_FRAME_REJECT", "8")
    with pytest.raises(Exception, match="no sweep frame"):
        _problem(g)


def test_elements_are_the_rotation0_nodes():
    """problem.elements (solver.py:208-215): node 0/3/8 are the face's vertices bitwise."""
    g = golden("star_l2")
    prob = _problem(g)
    els = prob.elements
    assert len(els) == prob.mesh.n_faces
    for f in (0, 17, len(els) - 1):
        a, b, c = g["faces"][f]
        e = els[f]
        assert e.vertex_ids == (a, b, c)
        assert np.array_equal(e.nodes[[0, 3, 8]], g["vertices"][[a, b, c]])
        assert np.abs(np.linalg.norm(e.node_normals, axis=1) - 1).max() < 1e-12


def test_rhs_and_energy_splits_are_bitwise_identical():
    """The row-split RHS and charge-split energy (emulated ranks on one GPU:
    same slot layout and permutations as the NCCL path) reproduce the
    unsplit results bit for bit, including ranks that own no charge."""
    g = golden("star_l3")
    prob = _problem(g)
    b0 = assemble_rhs(prob)
    cfg = SolverConfig(workers=1, restart=int(g["restart"]))
    with make_operator(prob, cfg) as op:
        sol = gmres_solve(op, b0, cfg)
    e0 = solvation_energy(prob, sol)
    lib = N.load()
    for ranks in (2, 3, 7, 64):
        N.check(lib.hobi_emulate_ranks(prob.handle, ranks))
        assert np.array_equal(assemble_rhs(prob), b0), ranks
        assert solvation_energy(prob, sol) == e0, ranks
        assert np.array_equal(matvec_hobi(prob, g["u"]), matvec_hobi(_problem(g), g["u"]))
    N.check(lib.hobi_emulate_ranks(prob.handle, 1))


def test_extreme_screening_lengths_against_oracle():
    """kappa far from the configs: tiny (coordinates scaled by kappa would
    underflow -> Laplace instantiation) and large (exp underflow branch)."""
    import hobi_oracle as O

    g = golden("star_l2")
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    u = g["u"]
    for kap in (1e-150, 1e-35, 1e-25, 1e-9, 2.0, 50.0):
        prob = discretize(mesh, PhysicalParams(2.0, 80.0, kap), ChargeSystem(np.zeros((0, 3)), []),
                          SolverConfig())
        o = O.discretize(g["vertices"], g["normals"], g["faces"], 2.0, 80.0, kap)
        assert rel_l2(matvec_hobi(prob, u), O.matvec(o, u)) <= MATVEC_TOL, kap


def test_problem_from_reference_caches():
    """The reference's own DiscretizedProblem caches (golden fields) uploaded as
    they are: the operator equals the device-geometry operator bit for bit
    (the caches are bitwise the same) and the reference's A u."""
    from types import SimpleNamespace

    from paper_1301_5914_b200.solver import problem_from_caches

    g = golden("star_l2")
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    ref = SimpleNamespace(mesh=mesh, params=PhysicalParams(*g["params"]),
                          charges=ChargeSystem(g["qpos"], g["q"]), scheme="hobi",
                          **{k: g[k] for k in ("reg_pos", "reg_nrm", "reg_w", "reg_bary", "duf_pos",
                                               "duf_nrm", "duf_w", "duf_bary", "pair_vertex",
                                               "pair_face", "pair_gverts", "pair_starts")})
    up = problem_from_caches(ref)
    assert np.array_equal(matvec_hobi(up, g["u"]), matvec_hobi(_problem(g), g["u"]))
    assert rel_l2(matvec_hobi(up, g["u"]), g["Au"]) <= MATVEC_TOL
    assert rel_l2(assemble_rhs(up), g["rhs"]) <= 1e-14
    cfg = SolverConfig(workers=1, restart=int(g["restart"]))
    with make_operator(up, cfg) as op:
        sol = gmres_solve(op, assemble_rhs(up), cfg)
    assert sol.iterations == int(g["iterations"])
    assert abs(solvation_energy(up, sol) - float(g["energy"])) <= SOLVE_TOL * abs(float(g["energy"]))


@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_random_surfaces_against_oracle(seed):
    """Seeded random star surfaces / parameters / vectors: device caches are
    bitwise the oracle's (which is bitwise the reference's), matvec and RHS to
    1e-12, LOBI too."""
    import hobi_oracle as O
    from paper_1301_5914_b200.surfaces import StarShape

    rng = np.random.default_rng(seed)
    shape = StarShape.from_seed(float(rng.uniform(5, 40)), seed=seed, amplitude=float(rng.uniform(0.05, 0.2)))
    mesh = shape.surface(int(rng.integers(1, 4)))
    charges = shape.interior_charges(int(rng.integers(1, 40)), seed=seed + 100)
    e1, e2, kap = float(rng.uniform(1, 8)), float(rng.uniform(2, 90)), float(rng.choice([0.0, rng.uniform(0.01, 1.0)]))
    prob = discretize(mesh, PhysicalParams(e1, e2, kap), charges, SolverConfig())
    o = O.discretize(mesh.vertices, mesh.normals, mesh.faces, e1, e2, kap, charges.positions, charges.charges)
    for key in ("reg_pos", "reg_nrm", "reg_w", "duf_pos", "duf_nrm", "duf_w"):
        assert np.array_equal(getattr(prob, key), getattr(o, key)), key
    u = rng.standard_normal(prob.n_unknowns)
    assert rel_l2(matvec_hobi(prob, u), O.matvec(o, u)) <= MATVEC_TOL
    assert rel_l2(assemble_rhs(prob), O.rhs(o)) <= 1e-13
    pl = discretize(mesh, PhysicalParams(e1, e2, kap), charges, SolverConfig(scheme="lobi"))
    ol = O.discretize(mesh.vertices, mesh.normals, mesh.faces, e1, e2, kap, scheme="lobi")
    ul = rng.standard_normal(pl.n_unknowns)
    assert rel_l2(matvec_lobi(pl, ul), O.matvec(ol, ul)) <= MATVEC_TOL


@pytest.mark.parametrize("kappa", [1e-12, 1e-9, 1e-6])
def test_small_screening_keeps_expm1_accuracy(kappa):
    """kappa*R << 1 with a zero phi block: the first output block is a pure
    K1 sum, K1 = W1 (e^{-kr} - 1)/r, so e^{-kr} - 1 must keep expm1's relative
    accuracy (an exp-only formulation lost up to 1e-6 here).  The same with
    eps2 ~ eps1, where K2 no longer dominates mixed vectors."""
    import hobi_oracle as O

    g = golden("star_l2")
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    rng = np.random.default_rng(17)
    for e2 in (40.0, 1.0 + 1e-6):
        prob = discretize(mesh, PhysicalParams(1.0, e2, kappa), ChargeSystem(np.zeros((0, 3)), []),
                          SolverConfig())
        o = O.discretize(g["vertices"], g["normals"], g["faces"], 1.0, e2, kappa)
        T = prob.n_collocation
        u = rng.standard_normal(2 * T)
        u[:T] = 0.0
        got, ref = matvec_hobi(prob, u), O.matvec(o, u)
        assert rel_l2(got[:T], ref[:T]) <= 1e-13, (e2, rel_l2(got[:T], ref[:T]))
        assert rel_l2(got[T:], ref[T:]) <= 1e-13
        prob.close()


def test_concurrent_creation_with_different_rules():
    """Contexts built concurrently from threads with different quadrature rules
    (rule tables live in device constant memory) still get bitwise the
    reference's caches."""
    import threading

    from paper_1301_5914_b200 import TriangleRule

    g9, g4 = golden("star_l2_rule9"), golden("star_l2")
    rule9 = TriangleRule(g9["rule_points"], g9["rule_weights"], "custom", int(g9["rule_degree"]))
    errors = []

    def build(g, kw):
        try:
            for _ in range(4):
                prob = _problem(g, **kw)
                for key in ("reg_pos", "reg_w", "duf_pos", "duf_w"):
                    if not np.array_equal(getattr(prob, key), g[key]):
                        errors.append(key)
                prob.close()
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    kw9 = {"regular_rule": rule9, "duffy_points": int(g9["duffy"])}
    threads = [threading.Thread(target=build, args=(g, kw)) for g, kw in ((g9, kw9), (g4, {})) * 2]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_lobi_self_mask_tiles_bitwise_across_splits():
    """LOBI on the tuned tiles: only source tiles that overlap a work item's
    target rows take the self-masked path.  Row splits move every tile
    boundary (and the remainder onto 128-row tiles), so equal bits across
    splits show the masked and unmasked paths agree; level 4 is checked
    against the oracle."""
    import hobi_oracle as O
    from paper_1301_5914_b200 import _native as N
    from paper_1301_5914_b200.surfaces import StarShape

    shape = StarShape.from_seed(14.0, seed=8)
    mesh5 = shape.surface(5)  # 20,480 faces: wide-tile path
    prob = discretize(mesh5, PhysicalParams(2.0, 80.0, 0.1257), ChargeSystem(np.zeros((0, 3)), []),
                      SolverConfig(scheme="lobi"))
    u = np.random.default_rng(23).standard_normal(prob.n_unknowns)
    ref = matvec_lobi(prob, u)
    lib = N.load()
    for p in (2, 3, 7):
        N.check(lib.hobi_emulate_ranks(prob.handle, p))
        assert np.array_equal(matvec_lobi(prob, u), ref), p
    N.check(lib.hobi_emulate_ranks(prob.handle, 1))
    prob.close()
    mesh4 = shape.surface(4)
    p4 = discretize(mesh4, PhysicalParams(2.0, 80.0, 0.1257), ChargeSystem(np.zeros((0, 3)), []),
                    SolverConfig(scheme="lobi"))
    o4 = O.discretize(mesh4.vertices, mesh4.normals, mesh4.faces, 2.0, 80.0, 0.1257, scheme="lobi")
    u4 = np.random.default_rng(24).standard_normal(p4.n_unknowns)
    assert rel_l2(matvec_lobi(p4, u4), O.matvec(o4, u4)) <= MATVEC_TOL
    p4.close()


@pytest.mark.parametrize("scheme,staged", [("hobi", False), ("lobi", False), ("hobi", True)])
def test_single_process_group_operator_bitwise(scheme, staged, monkeypatch):
    """The single-process multi-GPU group (workers -> GPUs without torchrun):
    replicas on the problem's device stand in for peers (members are ordered
    by events only, so sharing a device is legal).  Fused path: every member's
    epilogue stores its rows into the leader's output; staged path: slots are
    copied over.  The group matvec and GMRES solve are bitwise one context's."""
    from paper_1301_5914_b200.solver import GpuOperator

    if staged:  # members without peer access stage their rows and copy them over
        monkeypatch.setenv("HOBI_GROUP_STAGED", "1")
    g = golden("star_l3")
    prob = _problem(g, scheme=scheme)
    cfg = SolverConfig(workers=1, restart=int(g["restart"]), scheme=scheme)
    u = np.random.default_rng(31).standard_normal(prob.n_unknowns)
    mv = matvec_hobi if scheme == "hobi" else matvec_lobi
    ref = mv(prob, u)
    b = assemble_rhs(prob)
    with make_operator(prob, cfg) as op:
        sol_ref = gmres_solve(op, b, cfg)
    dev = prob.device
    for devices in ([dev, dev], [dev, dev, dev]):
        with GpuOperator(prob, len(devices), devices=devices) as op:
            assert op.group is not None
            assert np.array_equal(op(u), ref), devices
            sol = gmres_solve(op, b, cfg)
        assert sol.iterations == sol_ref.iterations and np.array_equal(sol.vector, sol_ref.vector)
    assert np.array_equal(mv(prob, u), ref)  # the problem itself is untouched
    op = GpuOperator(prob, 2, devices=[dev, dev])
    prob.close()
    op.close()  # releasing the group after its leader is gone is safe


def test_c_abi_one_call_solve_matches_python_path():
    """hobi_solve (RHS + GMRES + energy in one C call, for C/C++ integrators)
    equals the Python solve path bit for bit and the reference's golden."""
    import ctypes as C

    from paper_1301_5914_b200 import _native as N

    g = golden("star_l2")
    prob = _problem(g)
    cfg = SolverConfig(workers=1, restart=int(g["restart"]))
    with make_operator(prob, cfg) as op:
        sol = gmres_solve(op, assemble_rhs(prob), cfg)
    e_py = solvation_energy(prob, sol)
    T = prob.n_collocation
    phi, dphi, e = np.empty(T), np.empty(T), C.c_double(0)
    its, res, mv = C.c_int(0), C.c_double(0), C.c_int(0)
    q, qp = N.f64(g["q"]), N.f64(g["qpos"])
    N.check(N.load().hobi_solve(prob.handle, N.dptr(qp), N.dptr(q), q.size, cfg.tolerance, cfg.restart,
                                cfg.max_iterations, N.dptr(phi), N.dptr(dphi), C.byref(e), C.byref(its),
                                C.byref(res), C.byref(mv)))
    assert its.value == sol.iterations == int(g["iterations"]) and mv.value == sol.matvecs
    assert np.array_equal(phi, sol.phi) and np.array_equal(dphi, sol.dphi_dn)
    assert e.value == e_py
    assert abs(e.value - float(g["energy"])) <= SOLVE_TOL * abs(float(g["energy"]))


def test_c_abi_argument_errors():
    """Bad arguments come back as status codes with a message, never a crash:
    out-of-range faces, oversized rules, kappa*extent beyond the table range,
    group members of different problems, P2P open before its handle."""
    import ctypes as C

    from paper_1301_5914_b200 import _native as N

    lib = N.load()
    g = golden("star_l2")
    v, n = N.f64(g["vertices"]), N.f64(g["normals"])
    f = N.i64(g["faces"]).copy()
    rule = np.zeros((1, 2)); w = np.ones(1); sh = np.zeros((3, 1, 10))
    ctx = C.c_void_p()

    def create(faces, nq=1, kappa=0.1):
        return lib.hobi_create(0, N.dptr(v), N.dptr(n), v.shape[0], N.iptr(faces), faces.shape[0], 1.0, 80.0,
                               kappa, N.dptr(N.f64(np.zeros((nq, 2)))), N.dptr(N.f64(np.ones(nq))),
                               N.dptr(N.f64(np.zeros((3, nq, 10)))), nq, N.dptr(N.f64(rule)), N.dptr(N.f64(w)),
                               N.dptr(N.f64(sh)), 1, C.byref(ctx))

    bad = f.copy()
    bad[3, 1] = v.shape[0]
    assert create(bad) == N.HOBI_ERR_VALUE and "references a vertex outside" in N.last_error()
    assert create(f, nq=17) == N.HOBI_ERR_VALUE and "1..16" in N.last_error()
    assert create(f, kappa=1e12) == N.HOBI_ERR_VALUE and "supported range" in N.last_error()
    a = _problem(g)
    b = _problem(golden("star_l3"))
    members = (C.c_void_p * 2)(a.handle, b.handle)
    grp = C.c_void_p()
    assert lib.hobi_group_create(members, 2, C.byref(grp)) == N.HOBI_ERR_VALUE
    assert "same problem" in N.last_error()
    handles = (C.c_ubyte * 64)()
    assert lib.hobi_comm_p2p_open(a.handle, handles, 1, 0) == N.HOBI_ERR_STATE


def test_no_device_memory_leak_across_lifecycles():
    """Create / use / close contexts, emulated splits, groups and workspaces
    many times: device memory returns to where it started."""
    import torch

    from paper_1301_5914_b200.solver import GpuOperator

    g = golden("star_l3")

    def cycle():
        prob = _problem(g)
        u = np.random.default_rng(1).standard_normal(prob.n_unknowns)
        matvec_hobi(prob, u)
        cfg = SolverConfig(workers=1, restart=int(g["restart"]))
        with make_operator(prob, cfg) as op:
            sol = gmres_solve(op, assemble_rhs(prob), cfg)
        solvation_energy(prob, sol)
        with GpuOperator(prob, 3) as op:  # emulated split
            op(u)
        with GpuOperator(prob, 2, devices=[prob.device] * 2) as op:  # group with a replica
            gmres_solve(op, assemble_rhs(prob), cfg)
        prob.close()

    cycle()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(15):
        cycle()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 16 << 20, (free0 - free1) / 2**20  # < 16 MiB drift (allocator granularity)


def test_concurrent_contexts_from_threads():
    """Different contexts driven from different threads at once (each has its
    own streams and workspaces) give the sequential results bit for bit."""
    import threading

    names = ["star_l2", "star_l3", "c1", "uv_sphere"]
    probs = {n: _problem(golden(n)) for n in names}
    us = {n: np.random.default_rng(7).standard_normal(p.n_unknowns) for n, p in probs.items()}
    ref = {n: matvec_hobi(probs[n], us[n]) for n in names}
    errors = []

    def run(n):
        try:
            for _ in range(5):
                if not np.array_equal(matvec_hobi(probs[n], us[n]), ref[n]):
                    errors.append(n)
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    threads = [threading.Thread(target=run, args=(n,)) for n in names]  # one thread per context
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_c_host_example_matches_python_path(tmp_path):
    """examples/c_solve.c -- a plain C program on the C ABI with the built-in
    default rules (hobi_create_default + hobi_solve) -- reproduces the Python
    path's solve bit for bit (same caches, same GMRES, same energy)."""
    import os
    import shutil
    import subprocess

    from paper_1301_5914_b200 import _native as N
    from paper_1301_5914_b200 import icosahedral_sphere, solve

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "c_solve")
    libdir = os.path.dirname(N.LIB_PATH)
    subprocess.run([cc, "-std=c99", "-I", os.path.join(root, "include"), os.path.join(root, "examples", "c_solve.c"),
                    "-L", libdir, "-lhobi", f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    mesh = icosahedral_sphere(2, 2.0)
    params = PhysicalParams(1.0, 80.0, 0.1257)
    charges = ChargeSystem([[0.1, -0.2, 0.3], [-0.4, 0.0, 0.2]], [1.0, -0.5])
    blob = (np.array([mesh.n_vertices, mesh.n_faces, 2], dtype=np.int64).tobytes()
            + np.array([params.eps1, params.eps2, params.kappa]).tobytes()
            + N.f64(mesh.vertices).tobytes() + N.f64(mesh.normals).tobytes()
            + N.i64(mesh.faces).tobytes() + N.f64(charges.positions).tobytes() + N.f64(charges.charges).tobytes())
    (tmp_path / "problem.bin").write_bytes(blob)
    out = subprocess.run([exe, str(tmp_path / "problem.bin")], capture_output=True, text=True, check=True)
    its, mvs, res, e_hex = out.stdout.split()
    prob, sol = solve(mesh, params, charges, SolverConfig(workers=1))
    assert int(its) == sol.iterations and int(mvs) == sol.matvecs
    assert float.fromhex(e_hex) == solvation_energy(prob, sol)


def test_operator_out_buffer():
    """op(u, out=buf) writes into the caller's array (e.g. pinned memory) and
    returns it; wrong dtype / shape / a read-only array are rejected."""
    g = golden("star_l2")
    prob = _problem(g)
    with make_operator(prob, SolverConfig(workers=1)) as op:
        ref = op(g["u"])
        buf = np.empty_like(ref)
        assert op(g["u"], out=buf) is buf and np.array_equal(buf, ref)
        for bad in (np.empty(ref.size, dtype=np.float32), np.empty(ref.size + 2), np.empty((2, ref.size // 2))):
            with pytest.raises(ValueError, match="out must be"):
                op(g["u"], out=bad)
        ro = np.empty_like(ref)
        ro.setflags(write=False)
        with pytest.raises(ValueError, match="out must be"):
            op(g["u"], out=ro)


@pytest.mark.parametrize("restart", [1, 2, 3, 5])
def test_short_restart_cycles_match_oracle_gmres(restart):
    """Restart lengths down to 1 (every cycle a true-residual restart,
    solver.py:509-560): iterations, matvec counts and the solution follow the
    oracle's GMRES on the oracle's operator."""
    import hobi_oracle as O

    g = golden("star_l2")
    prob = _problem(g)
    o = O.discretize(g["vertices"], g["normals"], g["faces"], *g["params"], g["qpos"], g["q"])
    b = assemble_rhs(prob)
    x, its, rel, nmv = O.gmres(lambda v: O.matvec(o, v), O.rhs(o), tol=1e-6, restart=restart, max_it=2000)
    cfg = SolverConfig(workers=1, restart=restart, max_iterations=2000)
    with make_operator(prob, cfg) as op:
        sol = gmres_solve(op, b, cfg)
    assert sol.iterations == its and sol.matvecs == nmv
    assert rel_l2(sol.vector, x) <= 1e-9
