#!/usr/bin/env python
"""HOBI-PB boundary-integral matvec on B200: the bench contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

--gpus N always means N GPUs (plan_launch): under torchrun WORLD_SIZE must
equal N (one process per GPU, NCCL / fused peer-store gather); without a
launcher and N > 1 one process drives N GPUs through the native group
operator (csrc/hobi_group.cu).  Fewer than N visible GPUs, or a WORLD_SIZE
other than N, exits with status 2 -- never a smaller run under an N label.

A step is one application of the HOBI operator (SURVEY.md 8(a) rows a11-a14:
source weights, all-pairs regular sweep, Duffy swap, diagonal, and for N > 1
the gather of the row split: epilogue peer stores over NVLink once a start-up
check matches ncclAllGather bit for bit, else ncclAllGather) to a seeded u on BASELINE.json config 4
(star surface, icosphere level 6, 81,920 triangles, row-sharded at 1/2/4/8
GPUs).  The unit of work is one regular pair (target vertex, source regular
quadrature point): N_v * 4 N_f = 1.342e10 pairs per step.

`value`   : pairs/s, u resident in HBM, device time (CUDA events on the
            library's stream), L2 flushed between steps, max over ranks.
`e2e`     : the same through the call a user makes -- the operator protocol
            op(u, out=...) on pinned host arrays (H2D of u, matvec, D2H of A u
            inside every call), wall clock, max over ranks; `e2e.device_events`
            is the pinned host-buffer C-ABI step timed with CUDA events.
`roofline`: the all-pairs sweep kernel, 96 canonical FP64 flops per pair
             over its event-timed duration (the slowest GPU's
            for N > 1), against the FP64 DFMA peak measured on every GPU in
            the same run (MEASURED_PEAKS.json has none); `traffic` is the
            committed ncu capture only while its stamp matches the sweep
            sources.
`multi_gpu`: N > 1 only -- devices, row ranges, per-GPU compute and sweep ms,
            exchange bytes per matvec and the step time not spent computing.
`solve`   : one full GMRES solve of the config (restart 20, tol 1e-6) through
            the public API (wall clock, includes every matvec).
`cpu_baseline`: the numpy restatement of the reference (oracle/, a "port")
            on a bounded row sample of the same workload, fork pool over all
            cores.  `--impl reference` times the unmodified reference
            (pbbem pip-installed under baseline/_ref, which travels with the
            repo) on the same kind of sample, falling back to the port.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BIE matvec pair-interactions/s (FP64) and GMRES solve time at 1/2/4/8 B200"
FLOPS_PER_PAIR = 96  # SURVEY.md 8(d) canonical accounting
# FP64 instructions the default sweep executes per pair (24 DFMA + 12 DMUL + 7 DADD;
# SASS count, checked against the built library by tests/test_cabi.py)
FP64_INSTR_PER_PAIR = 43


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=4, help="BASELINE.json config (1-based)")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=0, help="rows per CPU sample (0 = auto)")
    ap.add_argument("--gather", choices=("auto", "nccl", "p2p"), default=os.environ.get("HOBI_GATHER", "auto"),
                    help="N>1 row gather: fused epilogue + NVLink peer stores when a start-up check "
                         "matches the NCCL gather (auto), always (p2p), or ncclAllGather (nccl)")
    return ap.parse_args()


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class LaunchError(SystemExit):
    """--gpus N cannot be honoured: exit non-zero with the reason, never a
    silently smaller run."""

    def __init__(self, msg):
        super().__init__(2)
        self.msg = msg


def plan_launch(gpus: int, env, visible) -> str:
    """How `--gpus N` runs: "torchrun" (one process per GPU, WORLD_SIZE from
    the launcher, which must equal N), "group" (N > 1 without a launcher: one
    process drives N GPUs through the native group operator) or "single".
    `visible` is a callable returning the visible GPU count (asked only when
    it matters).  Raises LaunchError when N cannot be honoured."""
    if gpus < 1:
        raise LaunchError(f"--gpus must be >= 1, got {gpus}")
    if "WORLD_SIZE" in env:
        world = int(env["WORLD_SIZE"])
        if world != gpus:
            raise LaunchError(f"--gpus {gpus} but the launcher started WORLD_SIZE={world} ranks")
        return "torchrun" if world > 1 or env.get("HOBI_FORCE_NCCL") == "1" else "single"
    if gpus == 1:
        return "single"
    if env.get("HOBI_BENCH_GROUP_SHARED") == "1":
        return "group-shared"  # test hook: N group members on GPU 0, labelled as such
    n = visible()
    if n < gpus:
        raise LaunchError(f"--gpus {gpus} requested but only {n} GPU(s) are visible; "
                          "refusing to report a smaller run under an N-GPU label")
    return "group"


def _workload(cfg, nv, nf, nq, n_gpus):
    """`config` of the JSON line; identical for both arms at the same --gpus."""
    return {
        "workload": f"BASELINE config {cfg.name}: {nv} vertices, {nf} curved cubic triangles, "
                    f"{len(cfg.charges)} charges, eps {cfg.eps1:g}/{cfg.eps2:g}, kappa {cfg.kappa}",
        "pairs_per_step": float(nv) * nf * nq,
        "n_vertices": nv, "n_faces": nf, "quad_points_per_face": nq,
        "duffy_points": 16, "gmres_restart": cfg.restart, "gmres_tol": cfg.tol,
        "l2": "512 MiB scratch write between timed steps (inputs < L2)",
        "parallelism": "single GPU" if n_gpus == 1 else f"row split over {n_gpus} GPUs (partition_targets)",
    }


class _Clocks:
    """Sample SM clock and throttle reasons every 50 ms (NVML) during a region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, indices):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            # CUDA ordinal -> NVML handle honouring CUDA_VISIBLE_DEVICES
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = [int(x) for x in vis.split(",")] if vis and all(x.strip().isdigit() for x in vis.split(",")) else None
            self._h = [pynvml.nvmlDeviceGetHandleByIndex(phys[i] if phys else i) for i in indices]
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h[0], pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            for h in self._h:
                try:
                    self.samples.append(self._nv.nvmlDeviceGetClockInfo(h, self._nv.NVML_CLOCK_SM))
                    self.reasons |= self._nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:  # noqa: BLE001
                    pass
            time.sleep(0.05)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        if not self._nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        r = [name for bit, name in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": r, "samples": len(self.samples)}


def _cpu_sample(cfg, u, rows_hint, target_s=15.0):
    """Oracle (numpy port of the reference) on rows [0, R) of the workload, fork pool."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hobi_oracle as O

    m = cfg.mesh
    prob = O.discretize(m.vertices, m.normals, m.faces, cfg.eps1, cfg.eps2, cfg.kappa, check=False)
    workers = os.cpu_count() or 1
    nsrc = prob.reg_pos.shape[0] * prob.reg_pos.shape[1]
    with O.PoolOperator(prob, workers) as op:
        rows = rows_hint or max(workers, 16)
        t0 = time.perf_counter()
        op.rows(u, 0, rows)
        dt = time.perf_counter() - t0
        if not rows_hint:  # calibrate to ~target_s of CPU work
            rows = int(min(prob.n_colloc, max(workers * 4, rows * target_s / max(dt, 1e-3))))
            t0 = time.perf_counter()
            op.rows(u, 0, rows)
            dt = time.perf_counter() - t0
    return {"pairs": float(rows) * nsrc, "seconds": dt, "rows": rows, "workers": workers}


def _reference_rows(cfg, workers):
    """The reference's own row-range unit on a fork pool of `workers`.

    Prefers the unmodified reference package installed under baseline/_ref
    (pip install --no-deps --target baseline/_ref of the reference's pkg/):
    pbbem.solver.discretize, then its _Operator fork pool running
    _range_task / _apply_range (solver.py:278-367, 424-459) over the sampled
    rows split with its own partition_targets -- kind "reference".  Without
    that install, the numpy restatement under oracle/ (kind "port").
    Returns (rows(u, lo, hi), close(), kind, label, setup_seconds)."""
    t0 = time.perf_counter()
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    m = cfg.mesh
    if os.path.isdir(os.path.join(ref_dir, "pbbem")):
        sys.path.insert(0, ref_dir)
        from pbbem import kernels as rk
        from pbbem import mesh as rm
        from pbbem import solver as rs

        prob = rs.discretize(rm.FlatMesh(vertices=m.vertices, normals=m.normals, faces=m.faces),
                             rk.PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa),
                             rm.ChargeSystem(positions=cfg.charges.positions, charges=cfg.charges.charges),
                             rs.SolverConfig(scheme="hobi", workers=workers))
        op = rs._Operator(prob, workers)

        def rows(u, lo, hi):
            if op._pool is None:
                return rs._apply_range(prob, u, lo, hi)
            parts = rs.partition_targets(hi - lo, workers)
            return op._pool.starmap(rs._range_task, [(op._token, u, lo + a, lo + b) for a, b in parts])

        return (rows, op.close, "reference",
                f"unmodified pbbem (baseline/_ref) _Operator fork pool of {workers} workers, _range_task",
                time.perf_counter() - t0)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hobi_oracle as O

    prob = O.discretize(m.vertices, m.normals, m.faces, cfg.eps1, cfg.eps2, cfg.kappa, check=False)
    op = O.PoolOperator(prob, workers)
    op.__enter__()
    return (op.rows, lambda: op.__exit__(None, None, None), "port",
            f"oracle/hobi_oracle.py (numpy port of the reference) fork pool of {workers} workers",
            time.perf_counter() - t0)


def run_reference(a):
    """--impl reference: the reference's CPU implementation of the path on the
    host cores (unmodified pbbem from baseline/_ref, else the oracle port),
    rank 0 only."""
    rank, world, _ = _dist()
    if rank != 0:
        return 0
    from paper_1301_5914_b200.surfaces import baseline_config

    cfg = baseline_config(a.config)
    nv, nf, nq = cfg.mesh.n_vertices, cfg.mesh.n_faces, 4
    u = np.random.default_rng(0).standard_normal(2 * nv)
    workers = os.cpu_count() or 1
    rows = a.cpu_rows or max(2 * workers, 256)
    nsrc = nf * nq
    times = []
    run_rows, close, kind, label, setup_s = _reference_rows(cfg, workers)
    try:
        for i in range(a.warmup + a.steps):
            lo = (i * rows) % max(1, nv - rows)
            t0 = time.perf_counter()
            run_rows(u, lo, lo + rows)
            dt = time.perf_counter() - t0
            if i >= a.warmup:
                times.append(dt)
    finally:
        close()
    total = sum(times)
    value = a.steps * rows * nsrc / total
    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * total / a.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _workload(cfg, nv, nf, nq, a.gpus), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": workers, "kind": kind,
                         "sample": f"{rows} target rows x {nsrc} sources per step (rows rotate), {label}; "
                                   f"setup (discretize) {setup_s:.1f} s untimed"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


class _RankRunner:
    """One process per GPU (single GPU, or torchrun ranks over NCCL)."""

    def __init__(self, a, use_dist, lib, N, prob, world, rank):
        self.a, self.use_dist, self.lib, self.N = a, use_dist, lib, N
        self.prob, self.world, self.rank = prob, world, rank
        self.handles = [prob.handle]
        self.devices = [int(os.environ["HOBI_DEVICE"])]
        nv = prob.n_collocation
        base, extra = divmod(nv, world)
        lo = rank * base + min(rank, extra)
        self.ranges = [(lo, lo + base + (1 if rank < extra else 0))]

    def barrier(self):
        if self.use_dist:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(self, x):
        if not self.use_dist:
            return x
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather_all(self, obj):
        if not self.use_dist:
            return [obj]
        import torch.distributed as dist

        box = [None] * self.world
        dist.all_gather_object(box, obj)
        return box

    def bench(self, up, op, steps, mode, ms):
        self.N.check(self.lib.hobi_bench(self.prob.handle, up, op, steps, mode, 1, self.N.dptr(ms)))

    def op(self, make_operator, scfg):
        return make_operator(self.prob, scfg)


class _GroupRunner(_RankRunner):
    """One process driving N GPUs through the native group operator."""

    def __init__(self, a, lib, N, prob, op, shared=False):
        self.a, self.use_dist, self.lib, self.N = a, False, lib, N
        self.prob, self.world, self.rank = prob, a.gpus, 0
        self.group_op = op
        pl = op.placement
        distinct = 1 if shared else a.gpus
        if pl["mode"] != "group" or pl["workers"] != a.gpus or len(set(pl["devices"])) != distinct:
            raise LaunchError(f"group operator did not place {a.gpus} GPUs: {pl}")
        self.handles = op.member_handles
        self.devices = pl["devices"]
        n = a.gpus
        lo, hi, direct = (C.c_int64 * n)(), (C.c_int64 * n)(), (C.c_int * n)()
        N.check(lib.hobi_group_info(op.group, None, None, lo, hi, direct))
        self.ranges = list(zip(lo, hi))
        self.direct = list(direct)

    def gather_all(self, obj):
        return [obj]

    def bench(self, up, op, steps, mode, ms):
        self.N.check(self.lib.hobi_group_bench(self.group_op.group, up, op, steps, mode, 1, self.N.dptr(ms)))

    def op(self, make_operator, scfg):
        return self.group_op


# the default config-4 sweep instantiation, sweep_kernel<kScreened, FULL, !SELF, R=7, MINB=2, UNROLL=3, STEP>
MAIN_SWEEP = "sweep_kernelILi1ELb1ELb0ELi7ELi2ELi3ELb1E"


def _sweep_source_hash(lib_path=None):
    """SHA-256 of the main sweep kernel's SASS in the built library: stamps the
    committed ncu traffic capture, which stays valid exactly as long as the
    kernel's machine code is unchanged.  None if cuobjdump is unavailable."""
    import hashlib
    import re
    import shutil
    import subprocess

    lib_path = lib_path or os.path.join(ROOT, "paper_1301_5914_b200", "libhobi.so")
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    try:
        dump = subprocess.run([tool, "-sass", lib_path], capture_output=True, text=True, timeout=300).stdout
    except Exception:  # noqa: BLE001
        return None
    for block in dump.split("Function : ")[1:]:
        name, _, body = block.partition("\n")
        if MAIN_SWEEP not in name:
            continue
        lines = []
        for ln in body.splitlines():
            t = ln.strip()
            if t.startswith("....") or t.startswith("Fatbin"):
                break
            if t:
                lines.append(re.sub(r"\s+", " ", t))
        return hashlib.sha256("\n".join(lines).encode()).hexdigest()
    return None


def _committed_traffic(config, world):
    """ncu dram bytes of one sweep launch from profiles/sweep_traffic.json, only
    if it was captured on this config/GPU count from the current sweep sources."""
    tfile = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    try:
        t = json.load(open(tfile))
    except Exception:  # noqa: BLE001
        return None, "no committed ncu capture"
    stamp = _sweep_source_hash()
    if stamp is None:
        return None, "cannot read the sweep kernel's SASS (cuobjdump unavailable)"
    if t.get("sweep_sass_sha256") != stamp:
        return None, "committed ncu capture is stale (the sweep kernel's SASS changed since)"
    if t.get("config") != config or t.get("n_gpus", 1) != world:
        return None, f"committed ncu capture is for config {t.get('config')} on {t.get('n_gpus', 1)} GPU(s)"
    return t["bytes_per_launch"], t.get("source")


def run_ours(a):
    rank, world, local = _dist()
    os.environ["HOBI_GATHER"] = a.gather
    from paper_1301_5914_b200 import _native as N

    mode = plan_launch(a.gpus, os.environ, N.device_count)
    use_dist = mode == "torchrun"
    if use_dist:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group(backend="nccl", device_id=torch.device("cuda", local))
    shared = mode == "group-shared"
    if shared:
        mode = "group"
    if mode == "group":
        os.environ["HOBI_DEVICE"] = "0"
        local = 0
    os.environ.setdefault("HOBI_DEVICE", str(local))
    from paper_1301_5914_b200 import (PhysicalParams, SolverConfig, assemble_rhs, discretize,
                                      gmres_solve, make_operator, solvation_energy)
    from paper_1301_5914_b200.solver import GpuOperator
    from paper_1301_5914_b200.surfaces import baseline_config

    lib = N.load()
    cfg = baseline_config(a.config)
    params = PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa)
    scfg = SolverConfig(workers=1, restart=cfg.restart, tolerance=cfg.tol)
    prob = discretize(cfg.mesh, params, cfg.charges, scfg)
    if mode == "group":
        devs = [0] * a.gpus if shared else None
        run = _GroupRunner(a, lib, N, prob, GpuOperator(prob, workers=a.gpus, devices=devs), shared)
        world = a.gpus
    else:
        run = _RankRunner(a, use_dist, lib, N, prob, world, rank)
    nv, nf, nq = cfg.mesh.n_vertices, cfg.mesh.n_faces, 4
    pairs_step = float(nv) * nf * nq
    peaks = []
    for d in sorted(set(run.devices)):
        pk = C.c_double(0.0)
        N.check(lib.hobi_probe_fp64_tflops(d, 300.0, C.byref(pk)))
        peaks.append(pk.value)
    u = np.random.default_rng(0).standard_normal(2 * nv)
    out = np.empty_like(u)
    barrier, max_over_ranks = run.barrier, run.max_over_ranks

    # --- value: HBM-resident operator applications ---------------------------
    ms = np.zeros(max(a.warmup, a.steps, 1))
    run.bench(N.dptr(u), N.dptr(out), a.warmup, 0, ms)
    barrier()
    for h in run.handles:
        N.check(lib.hobi_timing_reset(h))
    with _Clocks(sorted(set(run.devices))) as clocks:
        run.bench(N.dptr(u), N.dptr(out), a.steps, 0, ms)
    barrier()
    launches_total, members = 0, []
    for h, (lo, hi) in zip(run.handles, run.ranges):
        sweep_ms, sweep_n, launches = C.c_double(0), C.c_int64(0), C.c_int64(0)
        N.check(lib.hobi_timing(h, C.byref(sweep_ms), C.byref(sweep_n), C.byref(launches)))
        launches_total += int(launches.value)
        members.append({"rows": [int(lo), int(hi)], "sweep_ms": sweep_ms.value / max(sweep_n.value, 1),
                        "sweep_launches_per_step": sweep_n.value / max(a.steps, 1)})
    total_ms = max_over_ranks(float(ms[: a.steps].sum()))
    value = a.steps * pairs_step / (total_ms * 1e-3)
    ngroups, nspad = C.c_int(0), C.c_int64(0)
    N.check(lib.hobi_sweep_layout(prob.handle, C.byref(ngroups), C.byref(nspad)))
    # per-GPU sweep: canonical flops of its rows over its own event-timed launches
    for m in members:
        lo, hi = m["rows"]
        m["pairs"] = float(hi - lo) * nf * nq
        m["achieved_tflops"] = m["pairs"] * FLOPS_PER_PAIR / (m["sweep_ms"] * 1e-3) * 1e-12 if m["sweep_ms"] else 0.0
    all_members = [m for part in run.gather_all(members) for m in part]
    worst = max(all_members, key=lambda m: m["sweep_ms"])
    lo0, hi0 = members[0]["rows"]
    # per launch: source records (80 B) + this rank's targets (48 B) + the fixed
    # per-group partial sums (2 doubles per row per group) that keep row sums
    # independent of the split
    algo_bytes = 80.0 * nspad.value + 48.0 * (hi0 - lo0) + 16.0 * ngroups.value * (hi0 - lo0)

    # --- e2e device events: host buffers (pinned) through the C ABI ------------
    try:
        import torch

        hu = torch.from_numpy(u).pin_memory()
        ho = torch.empty_like(hu).pin_memory()
        up = C.cast(C.c_void_p(hu.data_ptr()), C.POINTER(C.c_double))
        op_ = C.cast(C.c_void_p(ho.data_ptr()), C.POINTER(C.c_double))
        pinned = True
    except Exception:  # noqa: BLE001
        up, op_, pinned = N.dptr(u), N.dptr(out), False
    ms2 = np.zeros(max(a.warmup, a.steps, 1))
    run.bench(up, op_, a.warmup, 1, ms2)
    barrier()
    run.bench(up, op_, a.steps, 1, ms2)
    barrier()
    e2e_ms = max_over_ranks(float(ms2[: a.steps].sum()))
    e2e = a.steps * pairs_step / (e2e_ms * 1e-3)

    # --- the call a user makes: the operator protocol on host numpy arrays
    # (solver.py:447-459), wall clock per synchronous call, L2 flushed between
    # calls outside the timed window -------------------------------------------
    flush = []
    try:
        import torch

        for d in sorted(set(run.devices)):
            flush.append(torch.empty(64 << 20, dtype=torch.float64, device=f"cuda:{d}"))
    except Exception:  # noqa: BLE001
        flush = []
    api_wall = []
    u_api, out_api = u, None
    if pinned:  # the step's input and result live in pinned host memory (views of hu / ho)
        u_api, out_api = hu.numpy(), ho.numpy()
    op_api = run.op(make_operator, scfg)
    for _ in range(a.warmup):
        op_api(u_api, out=out_api)
    barrier()
    for _ in range(a.steps):
        for f in flush:
            f.fill_(1.0)
        if flush:
            for d in sorted(set(run.devices)):
                torch.cuda.synchronize(d)
        t0 = time.perf_counter()
        op_api(u_api, out=out_api)
        api_wall.append(time.perf_counter() - t0)
    if op_api is not getattr(run, "group_op", None):
        op_api.close()
    api_ms = max_over_ranks(1e3 * float(sum(api_wall)))
    api = a.steps * pairs_step / (api_ms * 1e-3)

    # --- multi-GPU exchange: per-GPU compute alone vs the whole step ----------
    multi = None
    if world > 1:
        compute = []
        for h, (lo, hi) in zip(run.handles, run.ranges):
            msr = np.zeros(3)
            N.check(lib.hobi_bench_rows(h, N.dptr(u), lo, hi, 3, 1, N.dptr(msr)))
            compute.append(float(np.median(msr)))
        slowest = max_over_ranks(max(compute))
        step = total_ms / a.steps
        if mode == "group":
            xbytes = 16.0 * nv * (world - 1) + 16.0 * (nv - (run.ranges[0][1] - run.ranges[0][0]))
            how = ("one process, one context per GPU (csrc/hobi_group.cu): iterate peer-copied "
                   "to every member, each member's epilogue kernel stores its rows straight into "
                   "device 0's output over NVLink peer memory"
                   + ("" if all(run.direct) else " (some members staged: no peer access)"))
            gather_mode = "group peer stores" if all(run.direct) else "group staged copies"
        else:
            p2p_on = C.c_int(0)
            N.check(lib.hobi_comm_info(prob.handle, None, None, C.byref(p2p_on)))
            xbytes = 16.0 * nv * (world - 1)
            gather_mode = "fused epilogue + NVLink peer stores" if p2p_on.value else "ncclAllGather"
            how = f"one process per GPU (torchrun), {gather_mode}, --gather {a.gather}"
        ranks_info = run.gather_all({"device": run.devices, "rows": [list(r) for r in run.ranges],
                                     "compute_ms": compute})
        multi = {"mode": mode, "gather": gather_mode, "how": how,
                 "devices": [d for r in ranks_info for d in r["device"]],
                 "rows": [x for r in ranks_info for x in r["rows"]],
                 "compute_ms_per_gpu": [x for r in ranks_info for x in r["compute_ms"]],
                 "sweep_ms_per_gpu": [m["sweep_ms"] for m in all_members],
                 "step_ms": step,
                 "exchange_ms": max(step - slowest, 0.0),
                 "exchange_bytes_per_matvec": xbytes,
                 "exchange_GBps": xbytes / max(step - slowest, 1e-6) * 1e-6,
                 "note": "exchange_ms = device step time minus the slowest GPU's compute-only "
                         "time for its rows (hobi_bench_rows); it includes the stream/event "
                         "synchronisation, not only bytes in flight"}

    # --- solve through the public API ------------------------------------------
    solve = None
    if not a.no_solve:
        times = []
        for _ in range(2):  # the first solve of a process also pays one-time allocations and graph capture
            barrier()
            t0 = time.perf_counter()
            b = assemble_rhs(prob)
            op = run.op(make_operator, scfg)
            sol = gmres_solve(op, b, scfg)
            if op is not getattr(run, "group_op", None):
                op.close()
            energy = solvation_energy(prob, sol)
            barrier()
            times.append(max_over_ranks(time.perf_counter() - t0))
        solve = {"seconds": times[1], "first_seconds": times[0], "iterations": sol.iterations,
                 "matvecs": sol.matvecs, "residual": sol.residual, "energy_kcal_mol": energy,
                 "includes": "rhs + GMRES(restart %d, tol %g) + energy, wall clock; second of two solves "
                             "(first_seconds: the process's first)" % (cfg.restart, cfg.tol)}

    # one-GPU model of the p-way row split: the slowest of the first and last
    # rank's compute (everything before the gather), device-timed; labelled a
    # model -- measured multi-GPU numbers come from --gpus N runs of this file
    split_model = None
    if world == 1:
        split_model = {"what": "MODEL, not a multi-GPU run: slowest-rank compute of a p-way split "
                               "timed on this one GPU (no collective)"}
        t1 = None
        for p in (1, 2, 4, 8):
            worst_ms = 0.0
            for r in ((0,) if p == 1 else (0, p - 1)):
                base, extra = divmod(nv, p)
                rlo = r * base + min(r, extra)
                rhi = rlo + base + (1 if r < extra else 0)
                msr = np.zeros(3)
                N.check(lib.hobi_bench_rows(prob.handle, N.dptr(u), rlo, rhi, 3, 1, N.dptr(msr)))
                worst_ms = max(worst_ms, float(np.median(msr)))
            t1 = worst_ms if p == 1 else t1
            split_model[str(p)] = {"rank_ms": worst_ms, "efficiency": t1 / (p * worst_ms)}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        s = _cpu_sample(cfg, u, a.cpu_rows)
        cpu = {"value": s["pairs"] / s["seconds"], "unit": "pairs/s", "cores": s["workers"],
               "kind": "port",
               "sample": f"rows [0, {s['rows']}) of the same matvec ({s['pairs']:.3e} pairs, "
                         f"{s['seconds']:.1f} s), oracle/hobi_oracle.py fork pool"}
        # the full workload does not fit the CPU budget: extrapolated from the
        # measured per-pair rate, labelled as such
        rate = cpu["value"]
        cpu["extrapolated"] = {"matvec_s": pairs_step / rate,
                               "note": "extrapolated from the measured per-pair rate, not run"}
        if solve:
            cpu["extrapolated"]["solve_s"] = solve["matvecs"] * pairs_step / rate

    traffic, traffic_src = _committed_traffic(a.config, world)
    # executed-instruction view of the same launches: FP64 lane-ops per clock
    # per SM against the pipe's 64 (the canonical-flop frac above is the headline)
    clk = clocks.summary()
    pipe = None
    sms = C.c_int(0)
    if clk.get("sm_mhz") and lib.hobi_device_sms(run.devices[0], C.byref(sms)) == 0:
        m0 = members[0]
        ops = FP64_INSTR_PER_PAIR * m0["pairs"] / (m0["sweep_ms"] * 1e-3) / (sms.value * clk["sm_mhz"] * 1e6)
        pipe = {"instr_per_pair": FP64_INSTR_PER_PAIR, "lane_ops_per_clk_per_sm": ops,
                "frac_of_64": ops / 64.0, "sms": sms.value, "sm_mhz": clk["sm_mhz"], "gpu": run.devices[0]}
    peak_all = run.gather_all(peaks)
    peak_total = float(sum(p for part in peak_all for p in part))
    # whole-job sweep rate: every GPU's pairs over the slowest GPU's sweep time
    achieved = pairs_step * FLOPS_PER_PAIR / (worst["sweep_ms"] * 1e-3) * 1e-12
    launches_total = int(sum(run.gather_all(launches_total)))  # every GPU's kernels
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _workload(cfg, nv, nf, nq, world),
            "e2e": {"value": api, "unit": "pairs/s", "h2d_bytes_per_step": 16 * nv * (1 if mode == "group" else world),
                    "d2h_bytes_per_step": 16 * nv * (1 if mode == "group" else world),
                    "ms_per_step": api_ms / a.steps,
                    "pinned": pinned,
                    "how": "wall clock of the public operator call op(u, out=...) on host arrays "
                           "(make_operator, solver.py:447-459), "
                           + ("pinned " if pinned else "pageable ")
                           + "H2D + matvec + D2H inside each call, max over ranks; L2 flushed between "
                           "calls" + ("" if flush else " (flush unavailable)"),
                    "device_events": {"value": e2e, "ms_per_step": e2e_ms / a.steps, "pinned": pinned,
                                      "how": "bench mode 1: pinned H2D + matvec + D2H between "
                                             "CUDA events on the (leader's) library stream"}},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak_total, "unit": "TFLOP/s",
                         "frac": achieved / peak_total, "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_bytes": algo_bytes,
                         "kernel": "sweep_kernel<kScreened,FULL>", "flops_per_pair": FLOPS_PER_PAIR,
                         "avg_launch_ms": worst["sweep_ms"], "pairs_per_launch": worst["pairs"],
                         "per_gpu": [{"rows": m["rows"], "sweep_ms": m["sweep_ms"],
                                      "achieved_tflops": m["achieved_tflops"]} for m in all_members],
                         "peak_source": "DFMA probe on each GPU in this run (hobi_probe_fp64_tflops), "
                                        "summed over GPUs; MEASURED_PEAKS.json has no FP64 entry",
                         "fp64_pipe": pipe},
            "gpu_launches": launches_total,
            "clocks": clk,
            "solve": solve,
            "multi_gpu": multi,
            "split_model": split_model,
            "cpu_baseline": cpu,
        }
        if shared:
            line["n_gpus"] = 1
            line["test_hook"] = (f"HOBI_BENCH_GROUP_SHARED=1: {a.gpus} group members share GPU 0 -- exercises "
                                 f"the {a.gpus}-way group code path, NOT an {a.gpus}-GPU measurement")
        print(json.dumps(line), flush=True)
    if mode == "group":
        run.group_op.close()
    prob.close()  # release the device context and its NCCL communicator before torch's
    if use_dist:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    a = _args()
    if a.impl == "reference":
        return run_reference(a)
    try:
        return run_ours(a)
    except LaunchError as exc:
        print(f"bench.py: {exc.msg}", file=sys.stderr, flush=True)
        return 2


if __name__ == "__main__":
    sys.exit(main())
