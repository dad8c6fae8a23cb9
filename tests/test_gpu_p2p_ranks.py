"""The multi-rank fused P2P gather across real processes.

2 and 3 processes share cuda:0, each a rank with a P2P-only communicator:
they exchange CUDA IPC handles of their receive areas, every rank's epilogue
kernel stores its rows into every other process's area and bumps that
process's arrival counters, and the gathered A u must be bitwise the
one-context operator's over many epochs (both buffer parities), then a
replicated GMRES solve through the same operator must equal the one-context
solve on every rank.  Phases are host-ordered (tests/_p2p_rank_worker.py), so
no kernel waits for another process's kernel.  A stalled peer is caught by
the wait kernel's watchdog instead of hanging the GPU."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

WORKER = os.path.join(ROOT, "tests", "_p2p_rank_worker.py")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, tmp_path, *extra):
    port = _port()
    env = dict(os.environ, PYTHONPATH=ROOT, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen([sys.executable, WORKER, str(r), str(world), str(port), str(tmp_path), *extra],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out)
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, f"rank {r} failed:\n{out[-3000:]}"
    return [json.load(open(os.path.join(tmp_path, f"rank{r}.json"))) for r in range(world)]


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_p2p_gather_bitwise(world, tmp_path):
    res = _run(world, tmp_path)
    for r in res:
        assert r["comm"] == [world, r["rank"], 1]
        assert r["phase1_first_rejected"]
        assert r["epochs"] == 7 and all(r["bitwise"]), r
        assert r["golden_rel"] <= 1e-12
        its, its0, its_ref = r["gmres_iterations"]
        assert its == its0 == its_ref
        assert r["gmres_bitwise"], r["gmres_rel"]
        assert r["ranks_agree"]


def test_multiprocess_p2p_stalled_peer_hits_watchdog(tmp_path):
    res = _run(2, tmp_path, "stall")
    r0 = res[0]
    assert all(r0["bitwise"]) and r0["gmres_bitwise"]
    assert r0["stall_status"] == 6, r0  # HOBI_ERR_NCCL: collective failure
    assert "did not arrive" in r0["stall_message"]
    assert 1.5 <= r0["stall_seconds"] < 60.0
