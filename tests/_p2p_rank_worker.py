"""One rank of the multi-process P2P gather test (tests/test_gpu_p2p_ranks.py).

Every rank is a separate process on cuda:0.  Ranks join a gloo group
(127.0.0.1), build the same problem, split rows with a P2P-only communicator
(hobi_comm_init_p2p: NCCL refuses two ranks on one device), exchange their
receive areas' CUDA IPC handles (distributed.init_p2p_gather) and apply the
operator through hobi_matvec_p2p_phase: phase 0 (rows + peer stores +
arrival counters), a gloo barrier, phase 1 (gather released, copied out).
The barrier means no kernel ever waits for another process's kernel -- the
wait kernel finds every arrival already in place -- which is the only safe
way to run ranks that exchange data on one time-sliced GPU
(/opt/skills/guides/B200_PROFILING.md).  A replicated GMRES solve then runs
through the same two-phase operator.  Results go to a JSON file per rank.

    python tests/_p2p_rank_worker.py RANK WORLD PORT OUTDIR [stall]
"""

import ctypes as C
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def main():
    rank, world, port, outdir = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    stall = len(sys.argv) > 5 and sys.argv[5] == "stall"
    os.environ["HOBI_DEVICE"] = "0"
    os.environ["HOBI_P2P_TIMEOUT_MS"] = "2000"
    from paper_1301_5914_b200 import (ChargeSystem, FlatMesh, PhysicalParams, SolverConfig, assemble_rhs,
                                      discretize, gmres_solve, make_operator, matvec_hobi)
    from paper_1301_5914_b200 import _native as N
    from paper_1301_5914_b200.distributed import init_p2p_gather

    g = dict(np.load(os.path.join(HERE, "golden", "star_l3.npz")))
    mesh = FlatMesh(g["vertices"], g["normals"], g["faces"])
    params = PhysicalParams(*g["params"])
    charges = ChargeSystem(g["qpos"], g["q"])
    cfg = SolverConfig(workers=1, restart=int(g["restart"]))
    plain = discretize(mesh, params, charges, cfg)
    prob = discretize(mesh, params, charges, cfg)
    # the gloo group comes after discretize: under an initialised world > 1
    # discretize would build an NCCL communicator, which refuses two ranks on
    # one device -- these ranks use the P2P-only communicator instead
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    lib = N.load()
    N.check(lib.hobi_comm_init_p2p(prob.handle, world, rank))
    init_p2p_gather(prob.handle, rank, world)
    info = [C.c_int(-1) for _ in range(3)]
    N.check(lib.hobi_comm_info(prob.handle, *(C.byref(x) for x in info)))
    n = prob.n_unknowns
    res = {"rank": rank, "world": world, "comm": [x.value for x in info], "epochs": 0, "bitwise": [],
           "max_abs_diff": 0.0}

    def apply(u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.empty(n)
        N.check(lib.hobi_matvec_p2p_phase(prob.handle, N.dptr(u), None, 0))
        dist.barrier()  # every rank's rows are in every receive area
        N.check(lib.hobi_matvec_p2p_phase(prob.handle, None, N.dptr(out), 1))
        return out

    # phase order is enforced
    res["phase1_first_rejected"] = lib.hobi_matvec_p2p_phase(prob.handle, None, None, 1) == N.HOBI_ERR_STATE
    rng = np.random.default_rng(100)
    for k in range(7):  # both buffer parities, several times over
        u = rng.standard_normal(n) if k else g["u"]
        got = apply(u)
        ref = matvec_hobi(plain, u)
        res["bitwise"].append(bool(np.array_equal(got, ref)))
        res["max_abs_diff"] = max(res["max_abs_diff"], float(np.max(np.abs(got - ref))))
        res["epochs"] += 1
        if k == 0:
            res["golden_rel"] = float(np.linalg.norm(got - g["Au"]) / np.linalg.norm(g["Au"]))

    # replicated GMRES through the two-phase operator (host-callback GMRES)
    b = assemble_rhs(prob)
    sol = gmres_solve(apply, b, cfg)
    with make_operator(plain, cfg) as op:
        sol0 = gmres_solve(op, assemble_rhs(plain), cfg)
    res["gmres_iterations"] = [sol.iterations, sol0.iterations, int(g["iterations"])]
    res["gmres_bitwise"] = bool(np.array_equal(sol.vector, sol0.vector))
    res["gmres_rel"] = float(np.linalg.norm(sol.vector - sol0.vector) / np.linalg.norm(sol0.vector))
    phis = [None] * world
    dist.all_gather_object(phis, sol.vector.tobytes())
    res["ranks_agree"] = all(p == phis[0] for p in phis)

    if stall:
        # rank 1 stops sending; rank 0's next gather must give up (watchdog),
        # not wedge the GPU.  The stalled rank does no GPU work meanwhile.
        flag = os.path.join(outdir, "release")
        if rank == 1:
            dist.barrier()
            t0 = time.monotonic()
            while not os.path.exists(flag) and time.monotonic() - t0 < 120:
                time.sleep(0.05)
        else:
            dist.barrier()
            u = rng.standard_normal(n)
            out = np.empty(n)
            N.check(lib.hobi_matvec_p2p_phase(prob.handle, N.dptr(u), None, 0))
            t0 = time.monotonic()
            st = lib.hobi_matvec_p2p_phase(prob.handle, None, N.dptr(out), 1)
            res["stall_status"] = st
            res["stall_message"] = N.last_error()
            res["stall_seconds"] = time.monotonic() - t0
            open(flag, "w").close()
    with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)
    prob.close()
    plain.close()
    # no collective after a stall: the group's state is not trusted any more
    if not stall:
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
