"""Small host-buffer applications replay one captured graph (hobi_matvec,
csrc/hobi_api.cu): results must be bitwise those of the plain path."""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from conftest import golden
from paper_1301_5914_b200 import ChargeSystem, FlatMesh, PhysicalParams, SolverConfig, discretize, matvec_hobi, matvec_lobi
out = {}
for name, scheme in (("star_l2", "hobi"), ("c1", "hobi"), ("star_l2_lobi", "lobi")):
    g = golden(name)
    e1, e2, k = g["params"]
    prob = discretize(FlatMesh(g["vertices"], g["normals"], g["faces"]), PhysicalParams(e1, e2, k),
                      ChargeSystem(g["qpos"], g["q"]), SolverConfig(scheme=scheme, workers=1))
    mv = matvec_hobi if scheme == "hobi" else matvec_lobi
    rng = np.random.default_rng(5)
    for rep in range(4):  # call 0: plain path; call 1 captures; calls 2-3 replay
        u = rng.standard_normal(prob.n_unknowns)
        out[f"{name}_{rep}"] = mv(prob, u)
    out[name + "_golden"] = mv(prob, g["u"])
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, graph):
    path = tmp_path / f"mv_{graph}.npz"
    env = dict(os.environ, HOBI_MATVEC_GRAPH=graph)
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT, str(path)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return dict(np.load(path))


def test_graph_replay_is_bitwise_the_plain_path(tmp_path):
    a, b = _run(tmp_path, "1"), _run(tmp_path, "0")
    assert a.keys() == b.keys() and len(a) == 15
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    for name in ("star_l2", "c1", "star_l2_lobi"):
        g = golden(name)
        err = np.linalg.norm(a[name + "_golden"] - g["Au"]) / np.linalg.norm(g["Au"])
        assert err <= 1e-12, (name, err)
