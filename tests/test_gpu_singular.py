"""The three Duffy-swap kernels (solver.py:336-363).

* warp-per-pair literal kernel (singular_warp_kernel, HOBI_SINGULAR=warp)
  against the serial one-thread-per-pair literal kernel: identical operations
  in identical order, so matvecs agree bit for bit;
* the default thread-per-term kernel (singular_fast_kernel: the sweep's
  rsqrt/expm1 arithmetic, numpy's summation order) against the literal one:
  the matvec within 1e-14 relative (L2) and the reference goldens within 1e-12.

Default 4 + 16-point rules, and a 6x6 Duffy rule (4 + 36 terms: the warp
kernel's lanes loop past 32, the fast kernel packs 6 pairs per block)."""

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


def _run(tmp_path, kind, variant=None):
    path = os.path.join(tmp_path, f"mv_{kind}_{variant}.npz")
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("HOBI_SINGULAR_VARIANT", None)
    env["HOBI_SINGULAR"] = kind
    if variant is not None:
        env["HOBI_SINGULAR_VARIANT"] = str(variant)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), path], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(path))


def test_warp_singular_kernel_bitwise_equals_serial(tmp_path):
    warp = _run(tmp_path, "warp")
    serial = _run(tmp_path, "serial")
    for name in warp:
        assert np.array_equal(warp[name], serial[name]), name
        g = golden(name)
        assert np.linalg.norm(warp[name] - g["Au"]) <= 1e-12 * np.linalg.norm(g["Au"]), name


def test_fast_singular_kernel_matches_literal(tmp_path):
    fast = _run(tmp_path, "fast")
    warp = _run(tmp_path, "warp")
    for name in fast:
        rel = np.linalg.norm(fast[name] - warp[name]) / np.linalg.norm(warp[name])
        assert rel <= 1e-14, (name, rel)
        g = golden(name)
        assert np.linalg.norm(fast[name] - g["Au"]) <= 1e-12 * np.linalg.norm(g["Au"]), name


def test_fast_singular_tilings_bitwise_identical(tmp_path):
    """Every block tiling of the default-rule kernel (HOBI_SINGULAR_VARIANT
    1-8: pairs and threads per block, registers; the default is 4) does the
    same operations per term and the same row sums: bitwise equal matvecs."""
    base = _run(tmp_path, "fast")
    for v in range(1, 9):
        other = _run(tmp_path, "fast", v)
        for name in base:
            assert np.array_equal(base[name], other[name]), (v, name)
