"""World-size-2 tests of the row-split path on CPU (gloo): every rank computes
its partition_targets range (with the oracle standing in for the per-rank GPU
sweep), packs it in the [2][m] slot layout, all-gathers, and unpacks with the
same index map the CUDA permutation kernel uses.  The result must equal the
unsplit operator bitwise, and replicated GMRES must agree on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT
from paper_1301_5914_b200 import distributed as D


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_dir):
    import sys

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hobi_oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = dict(np.load(os.path.join(GOLDEN, "star_l2.npz")))
    p = O.discretize(g["vertices"], g["normals"], g["faces"], *g["params"], g["qpos"], g["q"])
    n = p.n_colloc
    m = D.slot_size(n, world)
    lo, hi = D.row_range(n, world, rank)

    def apply(u):
        r1, r2 = O.rows(p, u, lo, hi)
        send = torch.from_numpy(D.pack_rows(r1, r2, m))
        recv = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(recv, send)
        return D.unpack_gathered(torch.stack(recv).numpy(), n, world)

    out = apply(g["u"])
    ok = np.array_equal(out, O.matvec(p, g["u"]))
    # unique-id style broadcast of 128 opaque bytes (as init_nccl_comm does)
    box = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    ok &= box[0] == bytes(range(128))
    x, its, rel, nmv = O.gmres(apply, O.rhs(p), tol=1e-6, restart=int(g["restart"]))
    np.save(os.path.join(result_dir, f"x{rank}.npy"), x)
    with open(os.path.join(result_dir, f"ok{rank}"), "w") as f:
        f.write(f"{int(ok)} {its} {nmv}")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_split_allgather_gloo(tmp_path, world):
    mp.spawn(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    g = dict(np.load(os.path.join(GOLDEN, "star_l2.npz")))
    xs = [np.load(tmp_path / f"x{r}.npy") for r in range(world)]
    for r in range(world):
        ok, its, nmv = open(tmp_path / f"ok{r}").read().split()
        assert ok == "1"
        assert int(its) == int(g["iterations"]) and int(nmv) == int(g["matvecs"])
        assert np.array_equal(xs[r], xs[0])  # replicated GMRES is bitwise identical
    assert np.linalg.norm(xs[0][: xs[0].size // 2] - g["phi"]) <= 1e-12 * np.linalg.norm(g["phi"])


@pytest.mark.parametrize("n,world", [(10, 3), (7, 8), (162, 4), (5, 1)])
def test_layout_round_trip(n, world):
    m = D.slot_size(n, world)
    u = np.arange(2 * n, dtype=float)
    slots = []
    for r in range(world):
        lo, hi = D.row_range(n, world, r)
        slots.append(D.pack_rows(u[lo:hi], u[n + lo:n + hi], m))
    assert np.array_equal(D.unpack_gathered(np.stack(slots), n, world), u)
    owners = D.owner_of(np.arange(n), n, world)
    for r in range(world):
        lo, hi = D.row_range(n, world, r)
        assert np.all(owners[lo:hi] == r)


def _agree_worker(rank, world, port, result_dir):
    """_all_true: the step agreement of the auto gather check."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = [D._all_true(True), D._all_true(rank != 1), D._all_true(False)]
    with open(os.path.join(result_dir, f"agree{rank}"), "w") as f:
        f.write(" ".join(str(int(r)) for r in res))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_step_agreement_gloo(tmp_path):
    """Every rank reaches the same decision even when one rank's local check
    fails -- so no rank proceeds into a P2P collective the others skip."""
    world = 3
    mp.spawn(_agree_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert open(tmp_path / f"agree{r}").read() == "1 0 0"
