"""Generate the golden fixtures under tests/golden/ by running the REFERENCE itself.

Run once in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array in the .npz files comes out of the unmodified reference package
``pbbem`` (solver.discretize / matvec_hobi / assemble_rhs / gmres_solve /
solvation_energy, kernels.kernel_values_d, kirkwood.kirkwood_series); the
inputs (meshes, charges, seeded vectors) come from this repo's generators and
are stored alongside so the fixtures are self-contained on the GPU box.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from pbbem import kernels as rk  # noqa: E402
from pbbem import solver as rs  # noqa: E402
from pbbem.kirkwood import SphereProblem, kirkwood_series  # noqa: E402
from pbbem.mesh import ChargeSystem as RCharges  # noqa: E402
from pbbem.mesh import FlatMesh as RMesh  # noqa: E402

from paper_1301_5914_b200.surfaces import StarShape, baseline_config  # noqa: E402


def _ref_mesh(m):
    return RMesh(vertices=m.vertices, normals=m.normals, faces=m.faces)


def _ref_charges(c):
    return RCharges(positions=c.positions, charges=c.charges)


def _counted(op):
    count = [0]

    def apply(v):
        count[0] += 1
        return op(v)

    return apply, count


def case(name, mesh, charges, eps1, eps2, kappa, *, restart=None, caches=False, solve=False,
         kirkwood_radius=None, u_seed=7, workers=8, scheme="hobi", duffy=4, rule=None):
    t0 = time.time()
    params = rk.PhysicalParams(eps1, eps2, kappa)
    extra = {} if rule is None else {"regular_rule": rule}
    cfg = rs.SolverConfig(scheme=scheme, workers=workers, restart=restart or 100, duffy_points=duffy,
                          **extra)
    prob = rs.discretize(_ref_mesh(mesh), params, _ref_charges(charges), cfg)
    out = dict(vertices=mesh.vertices, normals=mesh.normals, faces=mesh.faces,
               qpos=charges.positions, q=charges.charges,
               params=np.array([eps1, eps2, kappa]))
    u = np.random.default_rng(u_seed).standard_normal(prob.n_unknowns)
    with rs.make_operator(prob, cfg) as op:
        out["u"] = u
        out["Au"] = op(u)
        out["rhs"] = rs.assemble_rhs(prob)
        if solve:
            apply, count = _counted(op)
            sol = rs.gmres_solve(apply, out["rhs"], cfg)
            out["phi"], out["dphi"] = sol.phi, sol.dphi_dn
            out["iterations"] = np.array(sol.iterations)
            out["residual"] = np.array(sol.residual)
            out["matvecs"] = np.array(count[0])
            out["restart"] = np.array(cfg.restart)
            out["energy"] = np.array(rs.solvation_energy(prob, sol))
    out["duffy"] = np.array(duffy)
    out["scheme"] = np.array(scheme)
    if rule is not None:
        out["rule_points"], out["rule_weights"] = rule.points, rule.weights
        out["rule_degree"] = np.array(rule.degree)
    if caches:
        for k in ("reg_pos", "reg_nrm", "reg_w", "reg_bary", "pair_vertex", "pair_face",
                  "pair_gverts", "pair_starts", "duf_pos", "duf_nrm", "duf_w", "duf_bary"):
            out[k] = getattr(prob, k)
    if kirkwood_radius is not None:
        sph = SphereProblem(radius=kirkwood_radius, params=params, charges=_ref_charges(charges))
        ks = kirkwood_series(sph, n_terms=40)
        out["kirkwood_energy"] = np.array(ks.energy)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: N_v={mesh.n_vertices} N_f={mesh.n_faces} {time.time() - t0:.1f}s", flush=True)


def kernel_table():
    """kernels.kernel_values_d on random pairs, incl. near-coincident and kappa = 0."""
    rng = np.random.default_rng(11)
    n = 4000
    d = rng.standard_normal((n, 3)) * np.exp(rng.uniform(np.log(1e-3), np.log(60.0), n))[:, None]
    nx = rng.standard_normal((n, 3))
    nx /= np.linalg.norm(nx, axis=1)[:, None]
    ny = rng.standard_normal((n, 3))
    ny /= np.linalg.norm(ny, axis=1)[:, None]
    out = dict(d=d, nx=nx, ny=ny)
    for tag, (e1, e2, kap) in {"a": (1.0, 80.0, 0.1257), "b": (2.0, 80.0, 0.5),
                               "c": (4.0, 80.0, 0.0), "d": (3.0, 3.0, 0.0)}.items():
        ks = rk.kernel_values_d(d, nx, ny, rk.PhysicalParams(e1, e2, kap))
        out["params_" + tag] = np.array([e1, e2, kap])
        out["K_" + tag] = np.stack(ks, axis=0)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    print("kernels: done", flush=True)


def degenerate_case():
    """The reference's first-failing-face error (test_solver.py:109-115 octahedron)."""
    verts = np.array([[1.0, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]])
    faces = np.array([[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4], [2, 0, 5], [1, 2, 5],
                      [3, 1, 5], [0, 3, 5]])
    normals = verts.copy()
    normals[0] = np.array([-1.0, 1.0, 0.0]) / np.sqrt(2.0)
    try:
        rs.discretize(RMesh(vertices=verts, normals=normals, faces=faces),
                      rk.PhysicalParams(1.0, 80.0, 0.0),
                      RCharges(positions=np.zeros((0, 3)), charges=np.zeros(0)),
                      rs.SolverConfig(scheme="hobi"))
        msg = ""
    except Exception as exc:  # noqa: BLE001
        msg = f"{type(exc).__name__}: {exc}"
    np.savez_compressed(os.path.join(HERE, "degenerate.npz"), vertices=verts, normals=normals,
                        faces=faces, message=np.array(msg))
    print("degenerate:", msg, flush=True)


def msms_case():
    """The reference's MSMS writer/reader and charge parser on a curved mesh plus
    malformed inputs (mesh.py:141-227): texts, parsed arrays, error messages."""
    from pbbem import mesh as rm

    star = StarShape.from_seed(16.0, seed=3).surface(2)
    ref = rm.FlatMesh(vertices=star.vertices, normals=star.normals, faces=star.faces)
    vert, face = rm.write_msms(ref)
    # MSMS-style headers, comments, 3-digit normals, extra columns
    messy_vert = "# MSMS vertices\n#faces #sphere density probe_r\n%d 1 1.50 1.40\n" % star.n_vertices
    for p, n in zip(star.vertices, star.normals):
        messy_vert += "%.6f %.6f %.6f %.3f %.3f %.3f 0 %d 2\n" % (*p, *n, 7)
    messy_face = "# MSMS faces\n%d 1 1.50 1.40\n" % star.n_faces + "".join(
        "%d %d %d 1 4  # tri\n" % tuple(f + 1) for f in star.faces)
    parsed = rm.parse_msms(messy_vert, messy_face)
    errors = []
    for v, f in (("1.0 0.0 0.0 0.6 0.6 0.6\n2.0 nope 0.0 0.6 0.6 0.6\n", "1 1 1\n"),
                 ("1.0 0.0 0.0 0.6 0.6 0.6\n" * 3, "0 1 2\n"),
                 ("1 0 0 0 0 0\n" * 3, "1 2 3\n"), ("# nothing\n", "1 2 3\n"),
                 ("1.0 0.0 0.0 0.6 0.6 0.6\n", "# none\n")):
        try:
            rm.parse_msms(v, f)
            errors.append("")
        except Exception as exc:  # noqa: BLE001
            errors.append(f"{type(exc).__name__}: {exc}")
    charges_txt = "# x y z q r\n1.5 -2 0.25 0.5 1.8\n\n-1e-3 0 4 -0.25\n  2 2 2 1  # ion\n"
    ch = rm.parse_charges(charges_txt)
    np.savez_compressed(os.path.join(HERE, "msms.npz"), vertices=star.vertices, normals=star.normals,
                        faces=star.faces, vert_text=np.array(vert), face_text=np.array(face),
                        messy_vert=np.array(messy_vert), messy_face=np.array(messy_face),
                        parsed_vertices=parsed.vertices, parsed_normals=parsed.normals,
                        parsed_faces=parsed.faces, errors=np.array(errors),
                        charges_text=np.array(charges_txt), charges_pos=ch.positions, charges_q=ch.charges)
    print("msms: done", flush=True)


def kirkwood_case():
    """kirkwood_series / kirkwood_centered of the reference (kirkwood.py:159-263)."""
    from pbbem.kirkwood import kirkwood_centered

    c2 = baseline_config(2)
    pts = c2.mesh.vertices
    out = {"points": pts}
    cases = {
        "c2": (c2.charges.positions, c2.charges.charges, 1.0, 80.0, 0.1257, 2.0),
        "ecc": (np.array([[0.0, 0.0, 1.7]]), np.array([1.0]), 2.0, 80.0, 0.5, 2.0),
        "lap": (c2.charges.positions[:3], np.array([1.0, -0.5, 0.25]), 4.0, 80.0, 0.0, 2.0),
    }
    for tag, (pos, q, e1, e2, kap, a) in cases.items():
        sph = SphereProblem(radius=a, params=rk.PhysicalParams(e1, e2, kap),
                            charges=RCharges(positions=pos, charges=q))
        ks = kirkwood_series(sph, n_terms=40)
        out[tag + "_in"] = np.concatenate([pos.ravel(), q, [e1, e2, kap, a]])
        out[tag + "_energy"] = np.array(ks.energy)
        out[tag + "_phi"] = ks.phi(a / 2.0 * pts)
        out[tag + "_dphi"] = ks.dphi_dn(a / 2.0 * pts)
        out[tag + "_tail"] = np.array([ks.tail_ratio, float(ks.converged)])
    sph = SphereProblem(radius=2.0, params=rk.PhysicalParams(1.0, 80.0, 0.1257),
                        charges=RCharges(positions=[[0.0, 0.0, 0.0]], charges=[1.0]))
    e, phi, dphi = kirkwood_centered(sph)
    out["centered"] = np.array([e, phi(np.array([0.0, 0.0, 2.0])), dphi(np.array([0.0, 0.0, 2.0]))])
    np.savez_compressed(os.path.join(HERE, "kirkwood.npz"), **out)
    print("kirkwood: done", flush=True)


def variants_case():
    """Other quadrature choices and the LOBI solve (SolverConfig knobs, solver.py:58-68)."""
    from pbbem.quadrature import duffy_rule

    star = StarShape.from_seed(16.0, seed=3)
    few = star.interior_charges(20, seed=5)
    case("star_l1_duffy6", star.surface(1), few, 2.0, 80.0, 0.5, caches=True, duffy=6)
    case("star_l2_rule9", star.surface(2), few, 4.0, 80.0, 0.1257, caches=True, duffy=3,
         rule=duffy_rule(3), solve=True, restart=15)
    case("star_l2_lobi", star.surface(2), few, 2.0, 80.0, 0.1257, solve=True, restart=20, scheme="lobi")


def uv_sphere(n_lat, n_lon, radius):
    """Latitude-longitude sphere: pole vertices of valence n_lon, skinny polar
    triangles -- a mesh family unlike the icospheres (valence 5/6)."""
    verts = [(0.0, 0.0, 1.0)]
    for i in range(1, n_lat):
        th = np.pi * i / n_lat
        for j in range(n_lon):
            ph = 2 * np.pi * j / n_lon + (0.5 * np.pi / n_lon if i % 2 else 0.0)
            verts.append((np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)))
    verts.append((0.0, 0.0, -1.0))
    verts = np.asarray(verts)
    ring = lambda i, j: 1 + (i - 1) * n_lon + (j % n_lon)  # noqa: E731
    faces = [(0, ring(1, j), ring(1, j + 1)) for j in range(n_lon)]
    for i in range(1, n_lat - 1):
        for j in range(n_lon):
            a, b, c, d = ring(i, j), ring(i, j + 1), ring(i + 1, j), ring(i + 1, j + 1)
            faces += [(a, c, d), (a, d, b)]
    south = len(verts) - 1
    faces += [(south, ring(n_lat - 1, j + 1), ring(n_lat - 1, j)) for j in range(n_lon)]
    faces = np.asarray(faces, dtype=np.int64)
    x = verts[faces]
    geo = np.cross(x[:, 1] - x[:, 0], x[:, 2] - x[:, 0])
    flip = np.einsum("ij,ij->i", geo, x.mean(axis=1)) < 0
    faces[flip] = faces[flip][:, ::-1]
    from paper_1301_5914_b200.mesh import FlatMesh

    return FlatMesh(vertices=radius * verts, normals=verts, faces=faces)


def uv_case():
    mesh = uv_sphere(10, 16, 2.0)
    rng = np.random.default_rng(21)
    pos = rng.uniform(-0.8, 0.8, size=(6, 3))
    from paper_1301_5914_b200.mesh import ChargeSystem

    charges = ChargeSystem(positions=pos, charges=rng.choice([-1.0, 1.0], 6))
    case("uv_sphere", mesh, charges, 2.0, 80.0, 0.3, restart=15, caches=True, solve=True,
         kirkwood_radius=2.0)


def main():
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[name]()
        return
    msms_case()
    kirkwood_case()
    variants_case()
    uv_case()
    kernel_table()
    degenerate_case()
    star = StarShape.from_seed(16.0, seed=3)
    few = star.interior_charges(50, seed=4)
    from paper_1301_5914_b200.mesh import ChargeSystem, icosahedral_sphere

    centred = ChargeSystem(positions=[[0.0, 0.0, 0.0]], charges=[1.0])
    case("sphere_l1_mixed", icosahedral_sphere(1, 2.0), centred, 2.0, 80.0, 0.5, caches=True)
    case("star_l2", star.surface(2), few, 2.0, 80.0, 0.1257, restart=20, caches=True, solve=True)
    case("star_l3", star.surface(3), few, 2.0, 80.0, 0.1257, restart=20, solve=True)
    c1 = baseline_config(1)
    case("c1", c1.mesh, c1.charges, c1.eps1, c1.eps2, c1.kappa, restart=c1.restart, solve=True,
         kirkwood_radius=2.0)
    c2 = baseline_config(2)
    case("c2", c2.mesh, c2.charges, c2.eps1, c2.eps2, c2.kappa, restart=c2.restart, solve=True,
         kirkwood_radius=2.0)


if __name__ == "__main__":
    main()
