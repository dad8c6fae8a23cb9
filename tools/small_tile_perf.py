"""Device time of the sweep on small problems for every kernel family that
uses the 128-row tile: HOBI / LOBI x screened / kappa = 0 on level-3 and -4
spheres, plus the energy sweep.  python tools/small_tile_perf.py"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1301_5914_b200 import (ChargeSystem, PhysicalParams, SolverConfig, _native as N, discretize,
                                  icosahedral_sphere, solvation_energy)
from paper_1301_5914_b200.solver import SurfaceSolution

lib = N.load()
rng = np.random.default_rng(1)
for level in (3, 4):
    mesh = icosahedral_sphere(level, 2.0)
    qpos = rng.uniform(-0.5, 0.5, (64, 3))
    charges = ChargeSystem(qpos, rng.standard_normal(64))
    for scheme in ("hobi", "lobi"):
        for kappa in (0.1257, 0.0):
            prob = discretize(mesh, PhysicalParams(1.0, 80.0, kappa), charges, SolverConfig(scheme=scheme, workers=1))
            u = rng.standard_normal(prob.n_unknowns)
            out, ms = np.empty_like(u), np.empty(50)
            N.check(lib.hobi_bench(prob.handle, N.dptr(u), N.dptr(out), 5, 0, 0, N.dptr(ms)))
            lib.hobi_timing_reset(prob.handle)
            N.check(lib.hobi_bench(prob.handle, N.dptr(u), N.dptr(out), 50, 0, 0, N.dptr(ms)))
            sw, nl = C.c_double(0), C.c_int64(0)
            lib.hobi_timing(prob.handle, C.byref(sw), C.byref(nl), None)
            n = prob.n_collocation
            sol = SurfaceSolution(u[:n], u[n:], scheme, 0, 0.0)
            solvation_energy(prob, sol)
            t0 = time.perf_counter()
            for _ in range(20):
                solvation_energy(prob, sol)
            te = (time.perf_counter() - t0) / 20 * 1e6
            print(f"L{level} {scheme} kappa={kappa}: sweep {sw.value / max(nl.value, 1) * 1e3:7.1f} us, "
                  f"matvec step {np.median(ms) * 1e3:7.1f} us, energy call {te:7.1f} us", flush=True)
            prob.close()
