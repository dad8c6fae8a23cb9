"""Row-split plumbing for one-process-per-GPU runs.

The reference splits target rows into contiguous ranges
(``partition_targets``, solver.py:405-418), computes each range in a worker
and concatenates the two half-vectors (solver.py:447-459).  Here every rank
owns one range on its GPU; after the sweep each rank's rows sit in a
``[2][m]`` send slot (m = ceil(n / nranks)), one ``ncclAllGather`` fills the
rank-major ``[nranks][2][m]`` receive buffer, and a permutation kernel
rebuilds ``out[0:n] ++ out[n:2n]``.  This module is the host-side statement of
that layout (the CUDA permutation kernel in csrc/hobi_sweep.cu implements the
same index map) plus the NCCL unique-id exchange over torch.distributed.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np


def row_range(n: int, nranks: int, rank: int) -> tuple[int, int]:
    """partition_targets(n, nranks)[rank] (solver.py:405-418)."""
    base, extra = divmod(n, nranks)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def slot_size(n: int, nranks: int) -> int:
    return -(-n // nranks)


def owner_of(v: np.ndarray, n: int, nranks: int) -> np.ndarray:
    """Rank owning row v -- the closed form used by permute_kernel."""
    base, extra = divmod(n, nranks)
    cut = extra * (base + 1)
    v = np.asarray(v, dtype=np.int64)
    return np.where(v < cut, v // (base + 1), extra + (v - cut) // max(base, 1))


def pack_rows(phi_rows: np.ndarray, dphi_rows: np.ndarray, m: int) -> np.ndarray:
    """This rank's send slot [2][m] (tail padded with zeros)."""
    slot = np.zeros((2, m))
    slot[0, : phi_rows.size] = phi_rows
    slot[1, : dphi_rows.size] = dphi_rows
    return slot


def unpack_gathered(recv: np.ndarray, n: int, nranks: int) -> np.ndarray:
    """[nranks][2][m] gathered slots -> (phi rows ++ dphi rows), length 2n."""
    recv = np.asarray(recv).reshape(nranks, 2, -1)
    v = np.arange(n)
    r = owner_of(v, n, nranks)
    lo = np.array([row_range(n, nranks, k)[0] for k in range(nranks)])[r]
    return np.concatenate([recv[r, 0, v - lo], recv[r, 1, v - lo]])


def init_nccl_comm(handle, rank: int, world: int, device: int | None = None) -> None:
    """Create the library's NCCL communicator: rank 0 draws the unique id,
    torch.distributed broadcasts the 128 bytes, every rank joins.  The row
    gather is then chosen by HOBI_GATHER: "auto" (default) switches to the
    fused epilogue + NVLink peer-store path when a start-up check shows it
    reproduces the NCCL gather bit for bit on every rank, "p2p" switches
    unconditionally, "nccl" keeps ncclAllGather."""
    import torch.distributed as dist

    from . import _native as N

    if device is not None and dist.get_backend() == "nccl":
        # torch's NCCL collectives run on torch's current device: make it this
        # rank's GPU, or every rank would broadcast from device 0
        import torch

        if torch.cuda.current_device() != device:
            torch.cuda.set_device(device)

    lib = N.load()
    uid = (C.c_ubyte * 128)()
    if rank == 0:
        N.check(lib.hobi_comm_unique_id(uid))
    box = [bytes(uid) if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    uid = (C.c_ubyte * 128).from_buffer_copy(box[0])
    N.check(lib.hobi_comm_init(handle, uid, world, rank))
    mode = os.environ.get("HOBI_GATHER", "auto")
    if mode == "p2p":
        init_p2p_gather(handle, rank, world)
    elif mode == "auto" and world > 1:
        init_p2p_gather_checked(handle, rank, world)


def _all_true(ok: bool) -> bool:
    """Logical AND of `ok` over all ranks (every rank calls it)."""
    import torch
    import torch.distributed as dist

    flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                        device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return int(flag.item()) == 1


def init_p2p_gather_checked(handle, rank: int, world: int) -> bool:
    """Default multi-rank gather: switch to the fused epilogue + peer-store
    gather only when every rank opened its peers' buffers and the P2P gather
    reproduces the NCCL gather bit for bit on every rank (one seeded matvec
    each way); otherwise stay on ncclAllGather.  Every step that can fail is
    agreed on by all ranks before the next collective step, so a failure on
    one rank never leaves the others waiting.  Returns whether P2P is active."""
    import numpy as np

    from . import _native as N

    lib = N.load()
    nc, nr = C.c_int64(0), C.c_int64(0)
    N.check(lib.hobi_size(handle, C.byref(nc), C.byref(nr)))
    u = np.random.default_rng(20251019).standard_normal(2 * nc.value)
    ref, got = np.empty_like(u), np.empty_like(u)
    N.check(lib.hobi_matvec(handle, N.dptr(u), N.dptr(ref)))  # NCCL gather
    ok = _all_true(init_p2p_gather(handle, rank, world, strict=False))
    if ok:
        local = lib.hobi_matvec(handle, N.dptr(u), N.dptr(got)) == N.HOBI_OK and np.array_equal(got, ref)
        ok = _all_true(local)
    if not ok:
        info = C.c_int(0)
        N.check(lib.hobi_comm_info(handle, None, None, C.byref(info)))
        if info.value:
            N.check(lib.hobi_comm_p2p_disable(handle))
    return ok


def init_p2p_gather(handle, rank: int, world: int, strict: bool = True) -> bool:
    """Exchange the CUDA IPC handles of every rank's receive area (rank order)
    and switch the operator's gather to peer stores from the epilogue.  Every
    rank takes part in the exchange even if its own handle failed; with
    strict=False failures return False instead of raising."""
    from . import _native as N

    lib = N.load()
    mine = (C.c_ubyte * 64)()
    ok = lib.hobi_comm_p2p_handle(handle, mine) == N.HOBI_OK
    if world > 1:
        import torch.distributed as dist

        allh = [None] * world
        dist.all_gather_object(allh, (ok, bytes(mine)))
    else:
        allh = [(ok, bytes(mine))]
    if not all(o for o, _ in allh):
        if strict:
            raise RuntimeError("P2P gather: a rank could not export its receive buffer")
        return False
    buf = (C.c_ubyte * (64 * world)).from_buffer_copy(b"".join(h for _, h in allh))
    st = lib.hobi_comm_p2p_open(handle, buf, world, rank)
    if st != N.HOBI_OK:
        if strict:
            N.check(st)
        return False
    return True
