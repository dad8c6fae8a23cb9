"""Host-side mirror of the reference solver API over the B200 C-ABI library.

Same names, arguments, return types and error behaviour as
``pbbem/solver.py`` (cited per function), but every array operation on the
hot path -- geometry precompute, matvec, right-hand side, GMRES, energy --
runs in hand-written sm_100a kernels behind ``libhobi.so``.  There is no CPU
fallback: without the library or a CUDA device the calls raise.

Parallelism: ``SolverConfig.workers`` keeps its meaning of "number of row
partitions".  Under ``torch.distributed`` with world size > 1 (one process
per GPU, e.g. torchrun) the partitions are the ranks and every matvec ends in
one NCCL allgather over NVLink; in a single process a workers > 1 operator
emulates the same split on one GPU.  Either way rows are bitwise identical to
the unsplit operator (solver.py:12-17).
"""

from __future__ import annotations

import ctypes as C
import os
import sys
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .geometry import CurvedElement, DegenerateArcError
from .mesh import ChargeSystem, FlatMesh
from .physics import FOUR_PI, KCAL_MOL_PER_E2_ANG, PhysicalParams, SingularityError
from .quadrature import TriangleRule, barycentric, duffy_rule, gauss_radau_rule, shape_tables

SCHEMES = ("hobi", "lobi")


class GmresNonConvergence(RuntimeError):
    """GMRES hit its iteration budget; carries the best residual (solver.py:50-55)."""

    def __init__(self, message: str, best_residual: float):
        super().__init__(message)
        self.best_residual = best_residual


@dataclass(frozen=True)
class SolverConfig:
    """Solver knobs (solver.py:58-87); ``workers`` = row partitions (GPU ranks)."""

    scheme: str = "hobi"
    tolerance: float = 1e-6
    restart: int = 100
    max_iterations: int = 1000
    workers: int | None = None
    regular_rule: TriangleRule = field(default_factory=gauss_radau_rule)
    duffy_points: int = 4

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise ValueError(f"scheme must be one of {SCHEMES}, got {self.scheme!r}")
        if not 0.0 < self.tolerance < 1.0:
            raise ValueError(f"tolerance must be in (0, 1), got {self.tolerance}")
        if self.restart < 1:
            raise ValueError(f"restart must be >= 1, got {self.restart}")
        if self.max_iterations < 1:
            raise ValueError(f"max_iterations must be >= 1, got {self.max_iterations}")
        if self.workers is not None and self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")

    def worker_count(self) -> int:
        if self.workers is not None:
            return self.workers
        return _world()[1]


@dataclass(frozen=True)
class SurfaceSolution:
    """Solved surface traces plus diagnostics (solver.py:90-102)."""

    phi: np.ndarray
    dphi_dn: np.ndarray
    scheme: str
    iterations: int
    residual: float

    @property
    def vector(self) -> np.ndarray:
        return np.concatenate([self.phi, self.dphi_dn])


def _world():
    """(rank, world_size, local_rank) of an initialised torch.distributed job.

    A job that never imported torch cannot have initialised torch.distributed,
    so torch (seconds to import) is only consulted when already loaded."""
    if "torch" not in sys.modules:
        return 0, 1, 0
    try:
        import torch.distributed as dist
    except Exception:  # noqa: BLE001
        return 0, 1, 0
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1, 0
    return dist.get_rank(), dist.get_world_size(), int(os.environ.get("LOCAL_RANK", dist.get_rank()))


def _dist_initialized() -> bool:
    if "torch" not in sys.modules:
        return False
    try:
        import torch.distributed as dist
    except Exception:  # noqa: BLE001
        return False
    return dist.is_available() and dist.is_initialized()


def _device_index() -> int:
    if "HOBI_DEVICE" in os.environ:
        return int(os.environ["HOBI_DEVICE"])
    return _world()[2]


class _Handle:
    """Owns one native context (device caches live as long as this object)."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr:
            try:
                N.load().hobi_destroy(self.ptr)
            except Exception:  # noqa: BLE001
                pass
            self.ptr = None


def _raise(status: int):
    if status == N.HOBI_OK:
        return
    msg = N.last_error()
    if status == N.HOBI_ERR_DEGENERATE_ARC:
        raise DegenerateArcError(msg)
    if status == N.HOBI_ERR_SINGULARITY:
        raise SingularityError(msg)
    if status == N.HOBI_ERR_VALUE:
        raise ValueError(msg)
    raise N.NativeError(status, msg)


class DiscretizedProblem:
    """Device-resident discretisation (solver.py:105-155).

    The reference's cache arrays are exposed as read-only properties copied
    back from HBM on first access (the device copies are what the kernels
    read).  ``n_collocation``, ``n_unknowns`` and ``singular_faces`` behave as
    in the reference.
    """

    _CACHE = ("reg_pos", "reg_nrm", "reg_w", "duf_pos", "duf_nrm", "duf_w", "pair_vertex",
              "pair_face", "pair_gverts", "pair_starts")

    def __init__(self, mesh, params, charges, scheme, handle, rule, duffy, rank_info):
        self.mesh = mesh
        self.params = params
        self.charges = charges
        self.scheme = scheme
        self._h = handle
        self._rule = rule
        self._duffy = duffy
        self._cache = {}
        self.rank, self.world = rank_info
        self.device = _device_index()
        x = mesh.vertices[mesh.faces]
        cr = np.cross(x[:, 1] - x[:, 0], x[:, 2] - x[:, 0])
        two = np.linalg.norm(cr, axis=1)
        self.area = 0.5 * two  # flat areas, both schemes (solver.py:184, 265)
        if scheme == "hobi":
            self.colloc_pos = mesh.vertices
            self.colloc_nrm = mesh.normals
            self.reg_bary = barycentric(rule.points)
            self.duf_bary = barycentric(duffy.points)
        else:
            self.colloc_pos = x.mean(axis=1)
            self.colloc_nrm = cr / two[:, None]
            self.reg_bary = self.duf_bary = None

    @property
    def handle(self):
        if not self._h.ptr:
            raise ValueError("problem has been closed")
        return self._h.ptr

    def close(self):
        """Free the device caches (and the NCCL communicator) now rather than at GC."""
        self._h.__del__()

    @property
    def n_collocation(self) -> int:
        return self.colloc_pos.shape[0]

    @property
    def n_unknowns(self) -> int:
        return 2 * self.n_collocation

    def _export(self):
        if "reg_pos" in self._cache or self.scheme != "hobi":
            return
        nf, nq, nd = self.mesh.n_faces, len(self._rule), len(self._duffy)
        out = {
            "reg_pos": np.empty((nf, nq, 3)), "reg_nrm": np.empty((nf, nq, 3)), "reg_w": np.empty((nf, nq)),
            "duf_pos": np.empty((3 * nf, nd, 3)), "duf_nrm": np.empty((3 * nf, nd, 3)),
            "duf_w": np.empty((3 * nf, nd)), "pair_vertex": np.empty(3 * nf, np.int64),
            "pair_face": np.empty(3 * nf, np.int64), "pair_gverts": np.empty((3 * nf, 3), np.int64),
            "pair_starts": np.empty(self.mesh.n_vertices + 1, np.int64),
        }
        _raise(N.load().hobi_export_caches(
            self.handle, *(N.dptr(out[k]) for k in self._CACHE[:6]),
            *(N.iptr(out[k]) for k in self._CACHE[6:])))
        for a in out.values():
            a.setflags(write=False)
        self._cache.update(out)

    def __getattr__(self, name):
        if name in DiscretizedProblem._CACHE:
            if self.scheme != "hobi":
                return None
            self._export()
            return self._cache[name]
        raise AttributeError(name)

    @property
    def elements(self):
        """Rotation-0 curved element per face (solver.py:208-215), from the device nodes."""
        if self.scheme != "hobi":
            return ()
        if "elements" not in self._cache:
            nf = self.mesh.n_faces
            pos, nrm = np.empty((nf, 10, 3)), np.empty((nf, 10, 3))
            _raise(N.load().hobi_export_nodes(self.handle, N.dptr(pos), N.dptr(nrm)))
            self._export()
            faces = self.mesh.faces
            self._cache["elements"] = tuple(
                CurvedElement(nodes=pos[f], node_normals=nrm[f], vertex_ids=tuple(int(v) for v in faces[f]))
                for f in range(nf))
        return self._cache["elements"]

    def singular_faces(self, vertex: int) -> np.ndarray:
        """Faces treated singularly for this vertex, face-ordered (solver.py:150-155)."""
        if self.scheme != "hobi":
            raise ValueError("singular partition exists only for scheme 'hobi'")
        lo, hi = self.pair_starts[vertex], self.pair_starts[vertex + 1]
        return self.pair_face[lo:hi]


def _create_handle(mesh: FlatMesh, params: PhysicalParams, scheme: str, rule, duffy, dev: int) -> "_Handle":
    """One native context of the problem on device `dev`."""
    lib = N.load()
    v, n, f = N.f64(mesh.vertices), N.f64(mesh.normals), N.i64(mesh.faces)
    ctx = C.c_void_p()
    if scheme == "hobi":
        rpts, rw, rsh = N.f64(rule.points), N.f64(rule.weights), N.f64(shape_tables(rule.points))
        dpts, dw, dsh = N.f64(duffy.points), N.f64(duffy.weights), N.f64(shape_tables(duffy.points))
        st = lib.hobi_create(dev, N.dptr(v), N.dptr(n), mesh.n_vertices, N.iptr(f), mesh.n_faces,
                             params.eps1, params.eps2, params.kappa, N.dptr(rpts), N.dptr(rw),
                             N.dptr(rsh), len(rule), N.dptr(dpts), N.dptr(dw), N.dptr(dsh), len(duffy),
                             C.byref(ctx))
    else:
        st = lib.hobi_create_lobi(dev, N.dptr(v), N.dptr(n), mesh.n_vertices, N.iptr(f), mesh.n_faces,
                                  params.eps1, params.eps2, params.kappa, C.byref(ctx))
    _raise(st)
    return _Handle(ctx.value)


def discretize(mesh: FlatMesh, params: PhysicalParams, charges: ChargeSystem,
               config: SolverConfig) -> DiscretizedProblem:
    """Validate the mesh and build every cache on the GPU (solver.py:165-266)."""
    mesh.validate()
    N.require_device()
    dev = _device_index()
    rule = config.regular_rule
    duffy = duffy_rule(config.duffy_points)
    handle = _create_handle(mesh, params, config.scheme, rule, duffy, dev)
    rank, world, _ = _world()
    # HOBI_FORCE_NCCL=1 runs the collective path even for a one-rank job (test hook)
    if world > 1 or (_dist_initialized() and os.environ.get("HOBI_FORCE_NCCL") == "1"):
        from .distributed import init_nccl_comm

        try:
            init_nccl_comm(handle.ptr, rank, world, _device_index())
        except N.NativeError as exc:
            _raise(exc.status)
    return DiscretizedProblem(mesh, params, charges, config.scheme, handle, rule, duffy, (rank, world))


def problem_from_caches(reference_problem, config: SolverConfig | None = None) -> DiscretizedProblem:
    """Device problem from an already discretised reference problem.

    ``reference_problem`` is any object with the fields of the reference's
    DiscretizedProblem (solver.py:119-140: mesh, params, charges, reg_pos,
    reg_nrm, reg_w, reg_bary, duf_pos, duf_nrm, duf_w, duf_bary, pair_vertex,
    pair_face, pair_gverts, pair_starts) -- e.g. pbbem's own.  The caches are
    uploaded as they are (no device geometry), so an installation can keep its
    discretize and run only the operator, RHS, GMRES and energy here.
    """
    rp = reference_problem
    if getattr(rp, "scheme", "hobi") != "hobi":
        raise ValueError("caches exist only for scheme 'hobi'")
    N.require_device()
    config = config or SolverConfig()
    m = rp.mesh
    v, n, f = N.f64(m.vertices), N.f64(m.normals), N.i64(m.faces)
    arr = {k: N.f64(getattr(rp, k)) for k in ("reg_pos", "reg_nrm", "reg_w", "reg_bary", "duf_pos",
                                               "duf_nrm", "duf_w", "duf_bary")}
    ints = {k: N.i64(getattr(rp, k)) for k in ("pair_vertex", "pair_face", "pair_gverts", "pair_starts")}
    nq, nd = arr["reg_w"].shape[1], arr["duf_w"].shape[1]
    ctx = C.c_void_p()
    p = rp.params
    _raise(N.load().hobi_create_from_caches(
        _device_index(), N.dptr(v), N.dptr(n), m.n_vertices, N.iptr(f), m.n_faces, p.eps1, p.eps2,
        p.kappa, N.dptr(arr["reg_pos"]), N.dptr(arr["reg_nrm"]), N.dptr(arr["reg_w"]),
        N.dptr(arr["reg_bary"]), nq, N.dptr(arr["duf_pos"]), N.dptr(arr["duf_nrm"]),
        N.dptr(arr["duf_w"]), N.dptr(arr["duf_bary"]), nd, N.iptr(ints["pair_vertex"]),
        N.iptr(ints["pair_face"]), N.iptr(ints["pair_gverts"]), N.iptr(ints["pair_starts"]),
        C.byref(ctx)))
    handle = _Handle(ctx.value)
    rank, world, _ = _world()
    if world > 1:
        from .distributed import init_nccl_comm

        init_nccl_comm(handle.ptr, rank, world, _device_index())
    mesh = FlatMesh(m.vertices, m.normals, m.faces)
    charges = ChargeSystem(rp.charges.positions, rp.charges.charges)
    prob = DiscretizedProblem(mesh, p, charges, "hobi", handle, _rule_of(arr["reg_bary"]),
                              _rule_of(arr["duf_bary"]), (rank, world))
    prob.reg_bary, prob.duf_bary = arr["reg_bary"], arr["duf_bary"]
    return prob


def _rule_of(bary):
    """A stand-in rule with the uploaded points (sizes and bookkeeping only)."""
    pts = np.clip(np.asarray(bary)[:, 1:3], 0.0, 1.0)
    return TriangleRule(pts, np.full(len(pts), 0.5 / len(pts)), "uploaded", 0)


def _as_vector(problem, u):
    u = N.f64(u)
    T = problem.n_collocation
    if u.shape != (2 * T,):
        raise ValueError(f"expected vector of length {2 * T}, got shape {u.shape}")
    return u


def _out_vector(u: np.ndarray, out):
    if out is None:
        return np.empty_like(u)
    if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.shape == u.shape
            and out.flags.c_contiguous and out.flags.writeable):
        raise ValueError(f"out must be a writable contiguous float64 array of shape {u.shape}")
    return out


def _full_matvec(problem: DiscretizedProblem, u, out=None) -> np.ndarray:
    u = _as_vector(problem, u)
    out = _out_vector(u, out)
    _raise(N.load().hobi_matvec(problem.handle, N.dptr(u), N.dptr(out)))
    return out


def matvec_hobi(problem: DiscretizedProblem, u) -> np.ndarray:
    """Vertex-collocated curved-element operator (solver.py:379-383)."""
    if problem.scheme != "hobi":
        raise ValueError(f"problem was discretized for scheme {problem.scheme!r}")
    return _full_matvec(problem, u)


def matvec_lobi(problem: DiscretizedProblem, u) -> np.ndarray:
    """Centroid-collocated flat-element operator (solver.py:386-390)."""
    if problem.scheme != "lobi":
        raise ValueError(f"problem was discretized for scheme {problem.scheme!r}")
    return _full_matvec(problem, u)


def apply_rows(problem: DiscretizedProblem, u, lo: int, hi: int):
    """Rows [lo, hi) of both blocks (_apply_range, solver.py:278-367)."""
    u = _as_vector(problem, u)
    o1 = np.empty(max(hi - lo, 0))
    o2 = np.empty(max(hi - lo, 0))
    _raise(N.load().hobi_matvec_rows(problem.handle, N.dptr(u), lo, hi, N.dptr(o1), N.dptr(o2)))
    return o1, o2


def assemble_rhs(problem: DiscretizedProblem) -> np.ndarray:
    """(S1, S2)/eps1 at the collocation points (solver.py:393-402)."""
    q = N.f64(problem.charges.charges)
    p = N.f64(problem.charges.positions)
    b = np.empty(problem.n_unknowns)
    _raise(N.load().hobi_rhs(problem.handle, N.dptr(p), N.dptr(q), q.size, N.dptr(b)))
    return b


def partition_targets(n_targets: int, n_workers: int) -> list[tuple[int, int]]:
    """Contiguous ranges, sizes within 1 (solver.py:405-418)."""
    if n_workers < 1:
        raise ValueError(f"n_workers must be >= 1, got {n_workers}")
    if n_targets < 0:
        raise ValueError(f"n_targets must be >= 0, got {n_targets}")
    base, extra = divmod(n_targets, n_workers)
    out, lo = [], 0
    for w in range(n_workers):
        hi = lo + base + (1 if w < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


class GpuOperator:
    """Callable matvec with the reference operator protocol (solver.py:432-472).

    ``workers`` > 1 is the reference's row split (solver.py:405-477).  In a
    single process with at least ``workers`` visible GPUs the rows run on that
    many GPUs (``devices``, default 0..workers-1 with the problem's device
    first): every extra device gets a replica context and the native group
    operator gathers the rows over peer copies.  With fewer GPUs the split is
    emulated on the problem's GPU (same gather layout and permutation as the
    NCCL path) and a ``RuntimeWarning`` says so; ``placement`` reports which
    of the three ran.  Either way the result is bitwise that of one GPU.
    ``devices`` may repeat a device (replicas sharing it) -- the test hook for
    the group path on a one-GPU machine.
    """

    def __init__(self, problem: DiscretizedProblem, workers: int = 1, devices=None):
        self._problem = problem
        self._closed = False
        self._emulated = False
        self._group = None
        self._replicas = []
        self._workers = 1
        lib = N.load()
        if problem.world != 1 or problem.n_collocation == 0:
            return
        if devices is None and workers > 1 and N.device_count() >= workers:
            others = [d for d in range(N.device_count()) if d != problem.device]
            devices = [problem.device] + others[: workers - 1]
        if devices is not None and len(devices) > 1:
            devices = list(devices)
            if devices[0] != problem.device:
                raise ValueError(f"devices[0] must be the problem's device {problem.device}")
            for d in devices[1:]:
                self._replicas.append(_create_handle(problem.mesh, problem.params, problem.scheme,
                                                     problem._rule, problem._duffy, int(d)))
            members = (C.c_void_p * len(devices))(problem.handle, *[h.ptr for h in self._replicas])
            grp = C.c_void_p()
            _raise(lib.hobi_group_create(members, len(devices), C.byref(grp)))
            self._group = grp.value
        elif workers > 1:
            import warnings

            warnings.warn(f"workers={workers} but only {N.device_count()} GPU(s) visible: the {workers}-way "
                          f"row split is emulated on GPU {problem.device} (same rows, one device)",
                          RuntimeWarning, stacklevel=3)
            _raise(lib.hobi_emulate_ranks(problem.handle, workers))
            self._emulated = True
        self._workers = workers

    @property
    def placement(self) -> dict:
        """How the rows run: ``mode`` is "single", "group" (one process, one
        context per device, ``devices`` lists them), "emulated" (a workers-way
        split on one GPU) or "ranks" (torch.distributed, one process per GPU)."""
        if self._problem.world != 1:
            return {"mode": "ranks", "workers": self._problem.world, "devices": [self._problem.device]}
        if self._group is not None:
            n = len(self._replicas) + 1
            devs = (C.c_int * n)()
            N.check(N.load().hobi_group_info(self._group, None, devs, None, None, None))
            return {"mode": "group", "workers": n, "devices": list(devs)}
        if self._emulated:
            return {"mode": "emulated", "workers": self._workers, "devices": [self._problem.device]}
        return {"mode": "single", "workers": 1, "devices": [self._problem.device]}

    @property
    def member_handles(self) -> list:
        """Native contexts of a group (leader first); [problem.handle] otherwise."""
        return [self._problem.handle] + [h.ptr for h in self._replicas]

    @property
    def problem(self):
        return self._problem

    @property
    def group(self):
        """Native multi-GPU group handle, or None."""
        return self._group

    def __call__(self, u, out=None) -> np.ndarray:
        """A u (solver.py:447-459).  `out` (extension): a float64 array to
        write into, e.g. pinned host memory for the fastest copies."""
        if self._closed:
            raise ValueError("operator is closed")
        if self._group is None:
            return _full_matvec(self._problem, u, out)
        u = _as_vector(self._problem, u)
        out = _out_vector(u, out)
        _raise(N.load().hobi_group_matvec(self._group, N.dptr(u), N.dptr(out)))
        return out

    def close(self):
        if self._closed:
            return
        if self._group is not None:
            N.load().hobi_group_destroy(self._group)
            self._group = None
        for h in self._replicas:
            h.__del__()
        self._replicas = []
        if self._emulated:
            _raise(N.load().hobi_emulate_ranks(self._problem.handle, 1))
        self._closed = True

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def make_operator(problem: DiscretizedProblem, config: SolverConfig) -> GpuOperator:
    """Matvec closure honouring config.workers (solver.py:475-477)."""
    return GpuOperator(problem, config.worker_count())


def gmres_solve(apply, b, config: SolverConfig) -> SurfaceSolution:
    """Restarted GMRES, true-residual restarts (solver.py:484-560), device-resident.

    With a GpuOperator the whole solve runs in HBM (native matvec); any other
    callable is applied through a host callback inside the same device GMRES.
    """
    b = N.f64(b)
    n = b.size
    if n % 2:
        raise ValueError("vector length must be even: (phi, dphi/dn) halves")
    N.require_device()
    lib = N.load()
    x = np.empty(n)
    its, mv = C.c_int(0), C.c_int(0)
    res, best = C.c_double(0.0), C.c_double(0.0)
    if isinstance(apply, GpuOperator) and apply.group is not None:
        st = lib.hobi_group_gmres(apply.group, N.dptr(b), config.tolerance, config.restart,
                                  config.max_iterations, N.dptr(x), C.byref(its), C.byref(res),
                                  C.byref(best), C.byref(mv))
    elif isinstance(apply, GpuOperator):
        st = lib.hobi_gmres(apply.problem.handle, N.dptr(b), config.tolerance, config.restart,
                            config.max_iterations, N.dptr(x), C.byref(its), C.byref(res), C.byref(best),
                            C.byref(mv))
    else:
        err = []

        def _cb(_user, src, dst, m):
            try:
                vin = np.ctypeslib.as_array(src, shape=(m,)).copy()
                vout = np.asarray(apply(vin), dtype=float).reshape(m)
                np.ctypeslib.as_array(dst, shape=(m,))[:] = vout
                return 0
            except Exception as exc:  # noqa: BLE001
                err.append(exc)
                return 1

        cb = N.APPLY_FN(_cb)
        st = lib.hobi_gmres_host_operator(_device_index(), n, cb, None, N.dptr(b), config.tolerance,
                                          config.restart, config.max_iterations, N.dptr(x),
                                          C.byref(its), C.byref(res), C.byref(best), C.byref(mv))
        if err:
            raise err[0]
    if st == N.HOBI_ERR_NONCONVERGENCE:
        raise GmresNonConvergence(N.last_error(), best_residual=best.value)
    _raise(st)
    half = n // 2
    sol = SurfaceSolution(phi=x[:half], dphi_dn=x[half:], scheme=config.scheme,
                          iterations=its.value, residual=res.value)
    object.__setattr__(sol, "matvecs", mv.value)
    return sol


def solve(mesh: FlatMesh, params: PhysicalParams, charges: ChargeSystem,
          config: SolverConfig) -> tuple[DiscretizedProblem, SurfaceSolution]:
    """Discretize, assemble, and solve in one call (solver.py:563-574)."""
    problem = discretize(mesh, params, charges, config)
    b = assemble_rhs(problem)
    with make_operator(problem, config) as op:
        solution = gmres_solve(op, b, config)
    return problem, solution


def solvation_energy(problem: DiscretizedProblem, solution: SurfaceSolution) -> float:
    """Reaction-field energy in kcal/mol (solver.py:581-614)."""
    if len(problem.charges) == 0:
        return 0.0
    q = N.f64(problem.charges.charges)
    p = N.f64(problem.charges.positions)
    phi, dphi = N.f64(solution.phi), N.f64(solution.dphi_dn)
    e = C.c_double(0.0)
    _raise(N.load().hobi_energy(problem.handle, N.dptr(p), N.dptr(q), q.size, N.dptr(phi),
                                N.dptr(dphi), C.byref(e)))
    return float(e.value)


def surface_potential_error(numerical, exact) -> float:
    """max_i |num_i - exact_i| / max_i |exact_i| (solver.py:617-628)."""
    numerical = np.asarray(numerical, dtype=float)
    exact = np.asarray(exact, dtype=float)
    if numerical.shape != exact.shape:
        raise ValueError(f"shape mismatch: {numerical.shape} vs {exact.shape}")
    scale = float(np.abs(exact).max())
    if scale == 0.0:
        raise ZeroDivisionError("exact vector is identically zero")
    return float(np.abs(numerical - exact).max()) / scale


def convergence_order(coarse_mesh: float, fine_mesh: float, coarse_error: float,
                      fine_error: float) -> float:
    """Observed order log(e_c/e_f) / |log(m_c/m_f)| (solver.py:631-655)."""
    for name, value in (("coarse_mesh", coarse_mesh), ("fine_mesh", fine_mesh),
                        ("coarse_error", coarse_error), ("fine_error", fine_error)):
        if not value > 0.0:
            raise ValueError(f"{name} must be positive, got {value}")
    if coarse_mesh == fine_mesh:
        raise ValueError("mesh parameters must differ")
    return float(np.log(coarse_error / fine_error) / abs(np.log(coarse_mesh / fine_mesh)))


__all__ = [
    "DegenerateArcError", "DiscretizedProblem", "GmresNonConvergence", "GpuOperator", "SCHEMES",
    "SolverConfig", "SurfaceSolution", "apply_rows", "assemble_rhs", "convergence_order",
    "discretize", "gmres_solve", "make_operator", "problem_from_caches", "matvec_hobi", "matvec_lobi", "partition_targets",
    "solvation_energy", "solve", "surface_potential_error", "FOUR_PI", "KCAL_MOL_PER_E2_ANG",
]
