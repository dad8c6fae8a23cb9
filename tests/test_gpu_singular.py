"""The warp-per-pair Duffy swap (singular_warp_kernel) against the serial
one-thread-per-pair kernel it replaced: identical operations in identical
order, so matvecs must agree bit for bit -- on the default 4 + 16-point rules
and on a 6x6 Duffy rule (4 + 36 terms: lanes loop past 32)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_1301_5914_b200 import ChargeSystem, FlatMesh, PhysicalParams, SolverConfig, discretize, matvec_hobi
out = {{}}
for name in ("star_l2", "star_l1_duffy6", "uv_sphere", "c2"):
    g = dict(np.load({root!r} + "/tests/golden/" + name + ".npz"))
    duffy = int(g["duffy"]) if "duffy" in g else 4
    prob = discretize(FlatMesh(g["vertices"], g["normals"], g["faces"]), PhysicalParams(*g["params"]),
                      ChargeSystem(g["qpos"], g["q"]), SolverConfig(workers=1, duffy_points=duffy))
    out[name] = matvec_hobi(prob, g["u"])
    prob.close()
np.savez(sys.argv[1], **out)
"""


def _run(tmp_path, serial):
    path = os.path.join(tmp_path, f"mv_{int(serial)}.npz")
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("HOBI_SINGULAR_SERIAL", None)
    if serial:
        env["HOBI_SINGULAR_SERIAL"] = "1"
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), path], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(path))


def test_warp_singular_kernel_bitwise_equals_serial(tmp_path):
    warp = _run(tmp_path, False)
    serial = _run(tmp_path, True)
    for name in warp:
        assert np.array_equal(warp[name], serial[name]), name
        g = golden(name)
        assert np.linalg.norm(warp[name] - g["Au"]) <= 1e-12 * np.linalg.norm(g["Au"]), name
