"""The reference-generated scale fixtures (tests/golden/make_scale_golden.py)
store a SHA-256 of the generated BASELINE meshes instead of the meshes: the
generator must still reproduce those inputs exactly (CPU check; the GPU
comparison is tests/test_gpu_scale_golden.py)."""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN

sys.path.insert(0, GOLDEN)


@pytest.mark.parametrize("name,index", [("c3_solve", 3), ("c4_rows", 4), ("c5_rows", 5), ("c4_rows_lobi", 4),
                                        ("c5_rows_lobi", 5), ("c4_solve", 4), ("c3_solve_lobi", 3),
                                        ("c4_solve_lobi", 4)])
def test_fixture_inputs_are_reproduced(name, index):
    from scale_hash import input_hash

    from paper_1301_5914_b200.surfaces import baseline_config

    path = os.path.join(GOLDEN, name + ".npz")
    if name == "c4_solve_lobi" and not os.path.exists(path):
        pytest.skip("config-4 LOBI pbbem solve fixture not generated yet")
    fx = np.load(path)
    cfg = baseline_config(index)
    assert input_hash(cfg) == str(fx["input_sha256"])
    assert np.array_equal(fx["params"], [cfg.eps1, cfg.eps2, cfg.kappa])
    assert int(fx["config"]) == index
