"""The NCCL gather path on one GPU: a one-rank communicator (HOBI_FORCE_NCCL=1)
runs the same send slot -> ncclAllGather -> permutation kernel sequence as an
8-way split does, and must reproduce the plain operator bitwise."""

import ctypes as C

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def test_single_rank_nccl_gather_path(monkeypatch):
    pytest.importorskip("torch")
    import torch  # noqa: F401  (loads libnccl.so.2 into the process, as under torchrun)

    from paper_1301_5914_b200 import (ChargeSystem, FlatMesh, PhysicalParams, SolverConfig,
                                      discretize, gmres_solve, make_operator, matvec_hobi,
                                      assemble_rhs)
    from paper_1301_5914_b200 import _native as N

    g = golden("star_l3")
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    params = PhysicalParams(*g["params"])
    charges = ChargeSystem(g["qpos"], g["q"])
    plain = discretize(mesh, params, charges, SolverConfig(workers=1))
    ref = matvec_hobi(plain, g["u"])
    prob = discretize(mesh, params, charges, SolverConfig(workers=1))
    lib = N.load()
    uid = (C.c_ubyte * 128)()
    N.check(lib.hobi_comm_unique_id(uid))
    monkeypatch.setenv("HOBI_FORCE_NCCL", "1")
    N.check(lib.hobi_comm_init(prob.handle, uid, 1, 0))
    out = matvec_hobi(prob, g["u"])
    assert np.array_equal(out, ref)
    cfg = SolverConfig(workers=1, restart=int(g["restart"]))
    with make_operator(prob, cfg) as op:
        sol = gmres_solve(op, assemble_rhs(prob), cfg)
    assert sol.iterations == int(g["iterations"])


def test_single_rank_p2p_fused_gather(monkeypatch):
    """Fused epilogue + peer-store gather (HOBI_GATHER=p2p path) with one rank:
    the kernel stores into the (own) receive area, bumps the arrival counter
    and the wait kernel releases -- bitwise equal to the plain operator over
    many epochs (both buffer parities) and through a full GMRES solve."""
    from paper_1301_5914_b200 import (ChargeSystem, FlatMesh, PhysicalParams, SolverConfig,
                                      discretize, gmres_solve, make_operator, matvec_hobi,
                                      assemble_rhs)
    from paper_1301_5914_b200 import _native as N
    from paper_1301_5914_b200.distributed import init_p2p_gather

    g = golden("star_l3")
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    params = PhysicalParams(*g["params"])
    charges = ChargeSystem(g["qpos"], g["q"])
    plain = discretize(mesh, params, charges, SolverConfig(workers=1))
    ref = matvec_hobi(plain, g["u"])
    prob = discretize(mesh, params, charges, SolverConfig(workers=1))
    lib = N.load()
    uid = (C.c_ubyte * 128)()
    N.check(lib.hobi_comm_init(prob.handle, uid, 1, 0))
    init_p2p_gather(prob.handle, 0, 1)
    for _ in range(5):
        assert np.array_equal(matvec_hobi(prob, g["u"]), ref)
    cfg = SolverConfig(workers=1, restart=int(g["restart"]))
    with make_operator(prob, cfg) as op:
        sol = gmres_solve(op, assemble_rhs(prob), cfg)
    assert sol.iterations == int(g["iterations"])
    with make_operator(plain, cfg) as op:
        sol0 = gmres_solve(op, assemble_rhs(plain), cfg)
    assert np.array_equal(sol.vector, sol0.vector)


def test_p2p_missing_peer_times_out_instead_of_hanging(monkeypatch):
    """A peer whose rows never arrive (test hook: wait for one arrival more than
    any rank sends) must not wedge the GPU: the wait kernel's watchdog gives up
    after HOBI_P2P_TIMEOUT_MS and the call reports a collective failure."""
    import time

    from paper_1301_5914_b200 import ChargeSystem, FlatMesh, PhysicalParams, SolverConfig, discretize, matvec_hobi
    from paper_1301_5914_b200 import _native as N
    from paper_1301_5914_b200.distributed import init_p2p_gather

    g = golden("star_l2")
    prob = discretize(FlatMesh(g["vertices"], g["normals"], g["faces"]), PhysicalParams(*g["params"]),
                      ChargeSystem(g["qpos"], g["q"]), SolverConfig(workers=1))
    lib = N.load()
    uid = (C.c_ubyte * 128)()
    N.check(lib.hobi_comm_init(prob.handle, uid, 1, 0))
    monkeypatch.setenv("HOBI_P2P_TIMEOUT_MS", "300")
    monkeypatch.setenv("HOBI_P2P_TEST_MISSING_ARRIVALS", "1")
    init_p2p_gather(prob.handle, 0, 1)
    t0 = time.monotonic()
    with pytest.raises(RuntimeError, match="did not arrive"):
        matvec_hobi(prob, g["u"])
    assert time.monotonic() - t0 < 30.0
    prob.close()


@pytest.mark.parametrize("break_p2p", [False, True])
def test_auto_gather_startup_check(monkeypatch, tmp_path, break_p2p):
    """HOBI_GATHER=auto: the P2P gather is switched on only after it matches
    the NCCL gather bit for bit; a P2P path whose arrivals never complete
    (test hook + short watchdog) is detected and every rank stays on NCCL."""
    torch = pytest.importorskip("torch")
    import torch.distributed as dist

    from paper_1301_5914_b200 import ChargeSystem, FlatMesh, PhysicalParams, SolverConfig, discretize, matvec_hobi
    from paper_1301_5914_b200 import _native as N
    from paper_1301_5914_b200.distributed import init_p2p_gather_checked

    g = golden("star_l3")
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    params, charges = PhysicalParams(*g["params"]), ChargeSystem(g["qpos"], g["q"])
    ref = matvec_hobi(discretize(mesh, params, charges, SolverConfig(workers=1)), g["u"])
    prob = discretize(mesh, params, charges, SolverConfig(workers=1))
    lib = N.load()
    uid = (C.c_ubyte * 128)()
    N.check(lib.hobi_comm_unique_id(uid))
    monkeypatch.setenv("HOBI_FORCE_NCCL", "1")
    N.check(lib.hobi_comm_init(prob.handle, uid, 1, 0))
    if break_p2p:
        monkeypatch.setenv("HOBI_P2P_TIMEOUT_MS", "300")
        monkeypatch.setenv("HOBI_P2P_TEST_MISSING_ARRIVALS", "1")
    dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    try:
        active = init_p2p_gather_checked(prob.handle, 0, 1)
    finally:
        dist.destroy_process_group()
    info = C.c_int(-1)
    N.check(lib.hobi_comm_info(prob.handle, None, None, C.byref(info)))
    assert active == (not break_p2p) and info.value == int(active)
    assert np.array_equal(matvec_hobi(prob, g["u"]), ref)  # P2P or NCCL, same bits
    prob.close()
