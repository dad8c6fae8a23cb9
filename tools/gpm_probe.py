"""Probe: NVML GPM (GPU Performance Monitoring) counters around a run of
config-C matvecs, outside any profiler.  Prints FP64 pipe utilisation, DRAM
bandwidth utilisation, PCIe and NVLink byte rates over the window, next to
the event-timed sweep numbers.

    python tools/gpm_probe.py [config] [steps]
"""

import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pynvml as nv  # noqa: E402

METRICS = {
    "sm_util": nv.NVML_GPM_METRIC_SM_UTIL,
    "sm_occupancy": nv.NVML_GPM_METRIC_SM_OCCUPANCY,
    "fp64_util": nv.NVML_GPM_METRIC_FP64_UTIL,
    "fp32_util": nv.NVML_GPM_METRIC_FP32_UTIL,
    "integer_util": nv.NVML_GPM_METRIC_INTEGER_UTIL,
    "dfma_tensor_util": nv.NVML_GPM_METRIC_DFMA_TENSOR_UTIL,
    "dram_bw_util": nv.NVML_GPM_METRIC_DRAM_BW_UTIL,
    "pcie_tx_per_sec": nv.NVML_GPM_METRIC_PCIE_TX_PER_SEC,
    "pcie_rx_per_sec": nv.NVML_GPM_METRIC_PCIE_RX_PER_SEC,
    "nvlink_tx_per_sec": nv.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC,
    "nvlink_rx_per_sec": nv.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC,
}


def metrics(h, s1, s2):
    mg = nv.c_nvmlGpmMetricsGet_t()
    mg.version = nv.NVML_GPM_METRICS_GET_VERSION
    mg.numMetrics = len(METRICS)
    mg.sample1, mg.sample2 = s1, s2
    for i, mid in enumerate(METRICS.values()):
        mg.metrics[i].metricId = mid
    nv.nvmlGpmMetricsGet(mg)
    out = {}
    for i, k in enumerate(METRICS):
        m = mg.metrics[i]
        out[k] = None if m.nvmlReturn != 0 else float(m.value)
    return out


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    sup = nv.nvmlGpmQueryDeviceSupport(h)
    print("gpm supported:", sup.isSupportedDevice)
    bus = nv.nvmlDeviceGetMemoryBusWidth(h)
    mclk = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_MEM)
    for attempt in ("before CUDA init", "streaming on"):
        if attempt == "streaming on":
            try:
                nv.nvmlGpmSetStreamingEnabled(h, 1)
            except nv.NVMLError as e:
                print("set streaming:", e)
        try:
            a = nv.nvmlGpmSampleAlloc()
            nv.nvmlGpmSampleGet(h, a)
            time.sleep(0.2)
            b = nv.nvmlGpmSampleAlloc()
            nv.nvmlGpmSampleGet(h, b)
            print(attempt, "ok", metrics(h, a, b))
        except nv.NVMLError as e:
            print(attempt, "failed:", e)
    print("bus width", bus, "mem max MHz", mclk, "=> DDR peak GB/s", 2 * mclk * 1e6 * bus / 8 / 1e9)

    from paper_1301_5914_b200 import PhysicalParams, SolverConfig, discretize
    from paper_1301_5914_b200 import _native as N
    from paper_1301_5914_b200.surfaces import baseline_config

    lib = N.load()
    cf = baseline_config(cfg_id)
    prob = discretize(cf.mesh, PhysicalParams(cf.eps1, cf.eps2, cf.kappa), cf.charges,
                      SolverConfig(workers=1, restart=cf.restart))
    nv_, nf = cf.mesh.n_vertices, cf.mesh.n_faces
    u = np.random.default_rng(0).standard_normal(2 * nv_)
    out = np.empty_like(u)
    ms = np.zeros(steps)
    N.check(lib.hobi_bench(prob.handle, N.dptr(u), N.dptr(out), 3, 0, 0, N.dptr(ms)))
    for label, flush in (("no flush", 0), ("idle", None)):
        s1, s2 = nv.nvmlGpmSampleAlloc(), nv.nvmlGpmSampleAlloc()
        N.check(lib.hobi_timing_reset(prob.handle))
        nv.nvmlGpmSampleGet(h, s1)
        t0 = time.perf_counter()
        if flush is None:
            time.sleep(0.5)
        else:
            N.check(lib.hobi_bench(prob.handle, N.dptr(u), N.dptr(out), steps, 0, flush, N.dptr(ms)))
        wall = time.perf_counter() - t0
        nv.nvmlGpmSampleGet(h, s2)
        m = metrics(h, s1, s2)
        nv.nvmlGpmSampleFree(s1)
        nv.nvmlGpmSampleFree(s2)
        sweep_ms, sweep_n, launches = C.c_double(0), C.c_int64(0), C.c_int64(0)
        N.check(lib.hobi_timing(prob.handle, C.byref(sweep_ms), C.byref(sweep_n), C.byref(launches)))
        rec = {"window": label, "wall_s": wall, "event_ms_sum": float(ms.sum()) if flush is not None else 0,
               "sweep_ms_avg": sweep_ms.value / max(sweep_n.value, 1), "launches": launches.value, **m}
        print(json.dumps(rec))
    prob.close()


if __name__ == "__main__":
    main()
