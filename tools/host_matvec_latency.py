"""Host-buffer operator latency on the small configs: wall clock of op(u) on
numpy arrays, median of 200 calls.  Run once per mode:
    python tools/host_matvec_latency.py            # graph replay (default)
    HOBI_MATVEC_GRAPH=0 python tools/host_matvec_latency.py"""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1301_5914_b200 import PhysicalParams, SolverConfig, discretize, make_operator
from paper_1301_5914_b200.surfaces import baseline_config

mode = "plain" if os.environ.get("HOBI_MATVEC_GRAPH") == "0" else "graph"
for idx in (1, 2, 3):
    cfg = baseline_config(idx)
    sc = SolverConfig(workers=1, restart=cfg.restart)
    prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, sc)
    u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
    with make_operator(prob, sc) as op:
        for _ in range(5):
            op(u)
        ts = []
        for _ in range(200):
            t0 = time.perf_counter()
            op(u)
            ts.append(time.perf_counter() - t0)
    ts = np.array(ts) * 1e6
    print(f"{mode} C{idx}: median {np.median(ts):.1f} us, min {ts.min():.1f} us, p90 {np.percentile(ts, 90):.1f} us")
