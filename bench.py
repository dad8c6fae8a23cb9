#!/usr/bin/env python
"""HOBI-PB boundary-integral matvec on B200: the bench contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

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
             over its event-timed duration, against the FP64
            DFMA peak measured in the same run (MEASURED_PEAKS.json has none).
`solve`   : one full GMRES solve of the config (restart 20, tol 1e-6) through
            the public API (wall clock, includes every matvec).
`cpu_baseline`: the numpy restatement of the reference (oracle/, a "port";
            the reference itself is Python and cannot travel to the box) on a
            bounded row sample of the same workload, fork pool over all cores.
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


def _workload(cfg, nv, nf, nq):
    return {
        "workload": f"BASELINE config {cfg.name}: {nv} vertices, {nf} curved cubic triangles, "
                    f"{len(cfg.charges)} charges, eps {cfg.eps1:g}/{cfg.eps2:g}, kappa {cfg.kappa}",
        "pairs_per_step": float(nv) * nf * nq,
        "n_vertices": nv, "n_faces": nf, "quad_points_per_face": nq,
        "duffy_points": 16, "gmres_restart": cfg.restart, "gmres_tol": cfg.tol,
        "l2": "512 MiB scratch write between timed steps (inputs < L2)",
    }


class _Clocks:
    """Sample SM clock and throttle reasons every 50 ms (NVML) during a region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                self.reasons |= self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
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


def run_reference(a):
    """--impl reference: the reference algorithm on host cores (oracle port), rank 0 only."""
    rank, world, _ = _dist()
    if rank != 0:
        return 0
    from paper_1301_5914_b200.surfaces import baseline_config

    cfg = baseline_config(a.config)
    nv, nf, nq = cfg.mesh.n_vertices, cfg.mesh.n_faces, 4
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hobi_oracle as O

    u = np.random.default_rng(0).standard_normal(2 * nv)
    m = cfg.mesh
    prob = O.discretize(m.vertices, m.normals, m.faces, cfg.eps1, cfg.eps2, cfg.kappa, check=False)
    workers = os.cpu_count() or 1
    rows = a.cpu_rows or max(2 * workers, 256)
    nsrc = nf * nq
    times = []
    with O.PoolOperator(prob, workers) as op:
        for i in range(a.warmup + a.steps):
            lo = (i * rows) % max(1, nv - rows)
            t0 = time.perf_counter()
            op.rows(u, lo, lo + rows)
            dt = time.perf_counter() - t0
            if i >= a.warmup:
                times.append(dt)
    total = sum(times)
    value = a.steps * rows * nsrc / total
    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * total / a.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _workload(cfg, nv, nf, nq), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": workers, "kind": "port",
                         "sample": f"{rows} target rows x {nsrc} sources per step (rows rotate), "
                                   f"oracle/hobi_oracle.py fork pool of {workers} workers"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(a):
    rank, world, local = _dist()
    os.environ["HOBI_GATHER"] = a.gather
    if world != a.gpus:
        a.gpus = world
    use_dist = world > 1 or ("RANK" in os.environ and os.environ.get("HOBI_FORCE_NCCL") == "1")
    if use_dist:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group(backend="nccl", device_id=torch.device("cuda", local))
    os.environ.setdefault("HOBI_DEVICE", str(local))
    from paper_1301_5914_b200 import (PhysicalParams, SolverConfig, assemble_rhs, discretize,
                                      gmres_solve, make_operator, solvation_energy)
    from paper_1301_5914_b200 import _native as N
    from paper_1301_5914_b200.surfaces import baseline_config

    lib = N.load()
    cfg = baseline_config(a.config)
    params = PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa)
    scfg = SolverConfig(workers=1, restart=cfg.restart, tolerance=cfg.tol)
    prob = discretize(cfg.mesh, params, cfg.charges, scfg)
    h = prob.handle
    nv, nf, nq = cfg.mesh.n_vertices, cfg.mesh.n_faces, 4
    pairs_step = float(nv) * nf * nq
    peak = C.c_double(0.0)
    N.check(lib.hobi_probe_fp64_tflops(int(os.environ["HOBI_DEVICE"]), 300.0, C.byref(peak)))
    u = np.random.default_rng(0).standard_normal(2 * nv)
    out = np.empty_like(u)
    lo, hi = (0, nv)
    if world > 1:
        base, extra = divmod(nv, world)
        lo = rank * base + min(rank, extra)
        hi = lo + base + (1 if rank < extra else 0)

    def barrier():
        if use_dist:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(x):
        if not use_dist:
            return x
        import torch
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # --- value: HBM-resident operator applications ---------------------------
    ms = np.zeros(max(a.warmup, a.steps))
    N.check(lib.hobi_bench(h, N.dptr(u), N.dptr(out), a.warmup, 0, 1, N.dptr(ms)))
    barrier()
    N.check(lib.hobi_timing_reset(h))
    with _Clocks(int(os.environ["HOBI_DEVICE"])) as clocks:
        N.check(lib.hobi_bench(h, N.dptr(u), N.dptr(out), a.steps, 0, 1, N.dptr(ms)))
    barrier()
    sweep_ms, sweep_n, launches = C.c_double(0), C.c_int64(0), C.c_int64(0)
    N.check(lib.hobi_timing(h, C.byref(sweep_ms), C.byref(sweep_n), C.byref(launches)))
    total_ms = max_over_ranks(float(ms[: a.steps].sum()))
    value = a.steps * pairs_step / (total_ms * 1e-3)
    sweep_avg = sweep_ms.value / max(sweep_n.value, 1)
    local_pairs = float(hi - lo) * nf * nq
    achieved = local_pairs * FLOPS_PER_PAIR / (sweep_avg * 1e-3) * 1e-12
    ngroups, nspad = C.c_int(0), C.c_int64(0)
    N.check(lib.hobi_sweep_layout(h, C.byref(ngroups), C.byref(nspad)))
    # per launch: source records (80 B) + this rank's targets (48 B) + the fixed
    # per-group partial sums (2 doubles per row per group) that keep row sums
    # independent of the split
    algo_bytes = 80.0 * nspad.value + 48.0 * (hi - lo) + 16.0 * ngroups.value * (hi - lo)

    # --- e2e: host buffers (pinned) through the C ABI, copies inside ------------
    try:
        import torch

        hu = torch.from_numpy(u).pin_memory()
        ho = torch.empty_like(hu).pin_memory()
        up = C.cast(C.c_void_p(hu.data_ptr()), C.POINTER(C.c_double))
        op_ = C.cast(C.c_void_p(ho.data_ptr()), C.POINTER(C.c_double))
        pinned = True
    except Exception:  # noqa: BLE001
        up, op_, pinned = N.dptr(u), N.dptr(out), False
    ms2 = np.zeros(max(a.warmup, a.steps))
    N.check(lib.hobi_bench(h, up, op_, a.warmup, 1, 1, N.dptr(ms2)))
    barrier()
    N.check(lib.hobi_bench(h, up, op_, a.steps, 1, 1, N.dptr(ms2)))
    barrier()
    e2e_ms = max_over_ranks(float(ms2[: a.steps].sum()))
    e2e = a.steps * pairs_step / (e2e_ms * 1e-3)

    # --- the call a user makes: the operator protocol on host numpy arrays
    # (solver.py:447-459), wall clock per synchronous call, L2 flushed between
    # calls outside the timed window -------------------------------------------
    flush = None
    try:
        import torch

        flush = torch.empty(64 << 20, dtype=torch.float64, device=f"cuda:{os.environ['HOBI_DEVICE']}")
    except Exception:  # noqa: BLE001
        flush = None
    api_wall = []
    u_api, out_api = u, None
    if pinned:  # the step's input and result live in pinned host memory (views of hu / ho)
        u_api, out_api = hu.numpy(), ho.numpy()
    with make_operator(prob, scfg) as op_api:
        for _ in range(a.warmup):
            op_api(u_api, out=out_api)
        barrier()
        for _ in range(a.steps):
            if flush is not None:
                flush.fill_(1.0)
                torch.cuda.synchronize()
            t0 = time.perf_counter()
            op_api(u_api, out=out_api)
            api_wall.append(time.perf_counter() - t0)
    api_ms = max_over_ranks(1e3 * float(sum(api_wall)))
    api = a.steps * pairs_step / (api_ms * 1e-3)

    # --- solve through the public API ------------------------------------------
    solve = None
    if not a.no_solve:
        barrier()
        t0 = time.perf_counter()
        b = assemble_rhs(prob)
        with make_operator(prob, scfg) as op:
            sol = gmres_solve(op, b, scfg)
        energy = solvation_energy(prob, sol)
        barrier()
        dt = max_over_ranks(time.perf_counter() - t0)
        solve = {"seconds": dt, "iterations": sol.iterations, "matvecs": sol.matvecs,
                 "residual": sol.residual, "energy_kcal_mol": energy,
                 "includes": "rhs + GMRES(restart %d, tol %g) + energy, wall clock" % (cfg.restart, cfg.tol)}

    # one-GPU model of the p-way row split: the slowest of the first and last
    # rank's compute (everything before the gather), device-timed; labelled a
    # model -- the real multi-GPU numbers come from torchrun runs of this file
    split_model = None
    if world == 1:
        split_model = {"what": "slowest-rank compute of a p-way split timed on this GPU (no collective)"}
        t1 = None
        for p in (1, 2, 4, 8):
            worst = 0.0
            for r in ((0,) if p == 1 else (0, p - 1)):
                base, extra = divmod(nv, p)
                rlo = r * base + min(r, extra)
                rhi = rlo + base + (1 if r < extra else 0)
                msr = np.zeros(3)
                N.check(lib.hobi_bench_rows(h, N.dptr(u), rlo, rhi, 3, 1, N.dptr(msr)))
                worst = max(worst, float(np.median(msr)))
            t1 = worst if p == 1 else t1
            split_model[str(p)] = {"rank_ms": worst, "efficiency": t1 / (p * worst)}

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

    traffic = None
    tfile = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if os.path.exists(tfile):
        try:
            t = json.load(open(tfile))
            if t.get("config") == a.config and t.get("n_gpus", 1) == world:
                traffic = t["bytes_per_launch"]
        except Exception:  # noqa: BLE001
            traffic = None
    # executed-instruction view of the same launches: FP64 lane-ops per clock
    # per SM against the pipe's 64 (the canonical-flop frac above is the headline)
    clk = clocks.summary()
    pipe = None
    sms = C.c_int(0)
    if clk.get("sm_mhz") and lib.hobi_device_sms(int(os.environ["HOBI_DEVICE"]), C.byref(sms)) == 0:
        ops = FP64_INSTR_PER_PAIR * local_pairs / (sweep_avg * 1e-3) / (sms.value * clk["sm_mhz"] * 1e6)
        pipe = {"instr_per_pair": FP64_INSTR_PER_PAIR, "lane_ops_per_clk_per_sm": ops,
                "frac_of_64": ops / 64.0, "sms": sms.value, "sm_mhz": clk["sm_mhz"]}
    if rank == 0:
        conf = _workload(cfg, nv, nf, nq)
        p2p_on = C.c_int(0)
        N.check(lib.hobi_comm_info(h, None, None, C.byref(p2p_on)))
        conf["parallelism"] = (f"row split x{world} + " + ("fused epilogue/NVLink peer-store gather"
                                                            if p2p_on.value else "NCCL allgather")
                               + f" (--gather {a.gather})") if world > 1 else "single GPU"
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": total_ms / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": conf,
            "e2e": {"value": api, "unit": "pairs/s", "h2d_bytes_per_step": 16 * nv * world,
                    "d2h_bytes_per_step": 16 * nv * world, "ms_per_step": api_ms / a.steps,
                    "pinned": pinned,
                    "how": "wall clock of the public operator call op(u, out=...) on host arrays "
                           "(make_operator, solver.py:447-459), "
                           + ("pinned " if pinned else "pageable ")
                           + "H2D + matvec + D2H inside each call, max over ranks; L2 flushed between "
                           "calls" + ("" if flush is not None else " (flush unavailable)"),
                    "device_events": {"value": e2e, "ms_per_step": e2e_ms / a.steps, "pinned": pinned,
                                      "how": "hobi_bench mode 1: pinned H2D + matvec + D2H between "
                                             "CUDA events on the library stream"}},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                         "frac": achieved / peak.value, "traffic": traffic,
                         "algorithmic_bytes": algo_bytes,
                         "kernel": "sweep_kernel<kScreened,FULL>", "flops_per_pair": FLOPS_PER_PAIR,
                         "avg_launch_ms": sweep_avg, "pairs_per_launch": local_pairs,
                         "peak_source": "DFMA probe in this run (hobi_probe_fp64_tflops); "
                                        "MEASURED_PEAKS.json has no FP64 entry",
                         "fp64_pipe": pipe},
            "gpu_launches": int(launches.value),
            "clocks": clk,
            "solve": solve,
            "split_model": split_model,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    prob.close()  # release the device context and its NCCL communicator before torch's
    if use_dist:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    a = _args()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
