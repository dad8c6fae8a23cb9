"""Device-driven GMRES cycles (a CUDA graph with a WHILE conditional node:
operator application, MGS and the Givens update/stopping test per step, no
host round trip) against the host-paced loop (HOBI_GMRES_GRAPH=0): same
kernels, same rotation arithmetic (glibc hypot restated on the device), so
iteration counts, residuals and solutions must agree bit for bit -- and the
iteration counts must equal the reference's."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import sys, json, numpy as np
sys.path.insert(0, {root!r})
from paper_1301_5914_b200 import (ChargeSystem, FlatMesh, PhysicalParams, SolverConfig, assemble_rhs,
                                  discretize, gmres_solve, make_operator, solvation_energy)
from paper_1301_5914_b200.surfaces import baseline_config
from paper_1301_5914_b200 import _native as N
out = {{}}
cases = []
for name in ("c1", "c2", "star_l2", "star_l3", "uv_sphere", "star_l2_lobi"):
    g = dict(np.load({root!r} + "/tests/golden/" + name + ".npz"))
    scheme = str(g["scheme"]) if "scheme" in g else "hobi"
    cases.append((name, FlatMesh(g["vertices"], g["normals"], g["faces"]), PhysicalParams(*g["params"]),
                  ChargeSystem(g["qpos"], g["q"]), int(g["restart"]), scheme))
for idx in (3, 4):  # n = 20484: the single-CTA MGS; n = 81924: the cooperative MGS inside the graph
    cf = baseline_config(idx)
    cases.append((f"c{{idx}}", cf.mesh, PhysicalParams(cf.eps1, cf.eps2, cf.kappa), cf.charges, cf.restart, "hobi"))
for name, mesh, params, charges, restart, scheme in cases:
    cfg = SolverConfig(workers=1, restart=restart, scheme=scheme)
    prob = discretize(mesh, params, charges, cfg)
    for rep in range(2):  # the second solve replays the cached graph
        N.check(N.load().hobi_timing_reset(prob.handle))  # no stale instrumentation events
        with make_operator(prob, cfg) as op:
            sol = gmres_solve(op, assemble_rhs(prob), cfg)
        N.check(N.load().hobi_timing_reset(prob.handle))
    out[name] = sol.vector
    out[name + "_meta"] = np.array([sol.iterations, sol.matvecs, sol.residual, solvation_energy(prob, sol)])
    prob.close()
np.savez(sys.argv[1], **out)
"""


def _run(tmp_path, graph):
    path = os.path.join(tmp_path, f"sol_{graph}.npz")
    env = dict(os.environ, PYTHONPATH=ROOT, HOBI_GMRES_GRAPH="1" if graph else "0")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), path], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(path))


def test_graph_cycles_bitwise_equal_host_loop(tmp_path):
    from conftest import golden

    g = _run(tmp_path, True)
    h = _run(tmp_path, False)
    for name in [k for k in g if not k.endswith("_meta")]:
        assert np.array_equal(g[name], h[name]), name
        assert np.array_equal(g[name + "_meta"], h[name + "_meta"]), name
        if name != "c4":  # config 3: the pbbem solve fixture (tests/golden/c3_solve.npz)
            ref = golden("c3_solve" if name == "c3" else name)
            assert int(g[name + "_meta"][0]) == int(ref["iterations"]), name
            assert int(g[name + "_meta"][1]) == int(ref["matvecs"]), name
