"""bench.py's reference arm runs on CPU: check its JSON line carries the
contract's keys (the GPU arm is exercised by the driver and `-m gpu` runs)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def test_reference_arm_json_line():
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "2",
                        "--warmup", "1", "--cpu-rows", "64"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["dtype"] == "f64"
    installed = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "pbbem"))
    assert d["cpu_baseline"]["kind"] == ("reference" if installed else "port")
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("BASELINE config C1")


def test_reference_arm_nonzero_ranks_exit_quietly():
    env = dict(os.environ, PYTHONPATH=ROOT, RANK="3", WORLD_SIZE="4", LOCAL_RANK="3")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "4"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_plan_launch_never_downgrades():
    sys.path.insert(0, ROOT)
    import bench

    none = lambda: 0  # noqa: E731
    one = lambda: 1  # noqa: E731
    eight = lambda: 8  # noqa: E731
    assert bench.plan_launch(1, {}, none) == "single"
    assert bench.plan_launch(2, {}, eight) == "group"
    assert bench.plan_launch(8, {}, eight) == "group"
    assert bench.plan_launch(4, {"WORLD_SIZE": "4", "RANK": "1"}, none) == "torchrun"
    assert bench.plan_launch(1, {"WORLD_SIZE": "1", "RANK": "0"}, none) == "single"
    assert bench.plan_launch(1, {"WORLD_SIZE": "1", "RANK": "0", "HOBI_FORCE_NCCL": "1"}, none) == "torchrun"
    assert bench.plan_launch(2, {"HOBI_BENCH_GROUP_SHARED": "1"}, one) == "group-shared"
    for gpus, env, vis in ((2, {}, one), (8, {}, none), (2, {"WORLD_SIZE": "4"}, eight),
                           (4, {"WORLD_SIZE": "1"}, eight), (0, {}, eight)):
        with pytest.raises(bench.LaunchError) as exc:
            bench.plan_launch(gpus, env, vis)
        assert exc.value.code == 2 and exc.value.msg


def test_more_gpus_than_visible_exits_nonzero():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["PYTHONPATH"] = ROOT
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "1"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, (r.returncode, r.stdout, r.stderr)
    assert r.stdout.strip() == "" and "refusing" in r.stderr


def test_both_arms_share_config():
    sys.path.insert(0, ROOT)
    import bench
    from paper_1301_5914_b200.surfaces import baseline_config

    cfg = baseline_config(1)
    for n in (1, 2, 8):
        c = bench._workload(cfg, 642, 1280, 4, n)
        assert c == bench._workload(cfg, 642, 1280, 4, n) and ("GPU" in c["parallelism"])
