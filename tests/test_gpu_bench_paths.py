"""bench.py's multi-GPU code paths on the one GPU this build has: the
single-process group path (`--gpus 2` with the HOBI_BENCH_GROUP_SHARED test
hook: both members on GPU 0) and the torchrun path (one rank with a one-rank
NCCL communicator).  Checks the JSON line's fields, not speed."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

ARGS = ["--config", "2", "--steps", "2", "--warmup", "1", "--no-cpu-baseline"]


def _line(cmd, env):
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def _env(**extra):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(PYTHONPATH=ROOT, **extra)
    return env


def test_group_path_line():
    d = _line([sys.executable, "bench.py", "--gpus", "2", *ARGS], _env(HOBI_BENCH_GROUP_SHARED="1"))
    assert d["n_gpus"] == 1 and "NOT an 2-GPU measurement" in d["test_hook"]
    mg = d["multi_gpu"]
    assert mg["mode"] == "group" and mg["devices"] == [0, 0]
    nv = d["config"]["n_vertices"]
    assert mg["rows"] == [[0, nv // 2 + nv % 2], [nv // 2 + nv % 2, nv]]
    assert len(mg["compute_ms_per_gpu"]) == 2 and mg["exchange_bytes_per_matvec"] > 0
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["solve"]["iterations"] == 17
    assert len(d["roofline"]["per_gpu"]) == 2


def test_torchrun_path_line():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    d = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
               "--master-addr", "127.0.0.1", f"--master-port={port}", "bench.py", "--gpus", "1", *ARGS],
              _env(HOBI_FORCE_NCCL="1"))
    assert d["n_gpus"] == 1 and d["config"]["parallelism"] == "single GPU"
    assert d["value"] > 0 and d["solve"]["iterations"] == 17 and d["gpu_launches"] > 0
    single = _line([sys.executable, "bench.py", *ARGS], _env())
    assert set(single) == set(d)
