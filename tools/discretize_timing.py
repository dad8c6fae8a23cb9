"""Where discretize() spends its time (host validation, library create,
first-call CUDA start-up): python tools/discretize_timing.py [configs...]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

from paper_1301_5914_b200 import PhysicalParams, SolverConfig, discretize
from paper_1301_5914_b200 import _native as N
from paper_1301_5914_b200.surfaces import baseline_config

for c in [int(a) for a in sys.argv[1:]] or [3, 4, 5]:
    t = time.perf_counter()
    cfg = baseline_config(c)
    t_mesh = time.perf_counter() - t
    prm = PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa)
    sc = SolverConfig(workers=1, restart=cfg.restart)
    for rep in range(3):
        t0 = time.perf_counter()
        cfg.mesh.validate()
        t1 = time.perf_counter()
        prob = discretize(cfg.mesh, prm, cfg.charges, sc)
        t2 = time.perf_counter()
        prob.close() if hasattr(prob, "close") else None
        print(f"config {c} rep {rep}: mesh build {t_mesh:.3f} s, validate {t1 - t0:.3f} s, "
              f"discretize (validate + create) {t2 - t1:.3f} s")
