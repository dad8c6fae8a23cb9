"""Small end-to-end case for compute-sanitizer: geometry, matvec (hobi + lobi),
row-split emulation, one-rank P2P gather, RHS, GMRES, energy."""
import ctypes as C
import os
import sys
import numpy as np
sys.path.insert(0, '.')
from paper_1301_5914_b200 import (ChargeSystem, FlatMesh, PhysicalParams, SolverConfig, discretize, matvec_hobi,
                                  matvec_lobi, assemble_rhs, make_operator, gmres_solve, solvation_energy)
from paper_1301_5914_b200 import _native as N
from paper_1301_5914_b200.distributed import init_p2p_gather
g = dict(np.load('tests/golden/star_l2.npz'))
mesh = FlatMesh(g['vertices'], g['normals'], g['faces'])
params = PhysicalParams(*g['params'])
ch = ChargeSystem(g['qpos'], g['q'])
for scheme in ('hobi', 'lobi'):
    cfg = SolverConfig(scheme=scheme, restart=20, workers=3)
    prob = discretize(mesh, params, ch, cfg)
    u = g['u'] if scheme == 'hobi' else np.random.default_rng(0).standard_normal(prob.n_unknowns)
    (matvec_hobi if scheme == 'hobi' else matvec_lobi)(prob, u)
    with make_operator(prob, cfg) as op:
        sol = gmres_solve(op, assemble_rhs(prob), cfg)
    print(scheme, sol.iterations, solvation_energy(prob, sol))
prob = discretize(mesh, PhysicalParams(1.0, 80.0, 0.0), ch, SolverConfig())
matvec_hobi(prob, g['u'])
prob = discretize(mesh, params, ch, SolverConfig())
uid = (C.c_ubyte * 128)()
N.check(N.load().hobi_comm_init(prob.handle, uid, 1, 0))
init_p2p_gather(prob.handle, 0, 1)
for _ in range(3):
    matvec_hobi(prob, g['u'])
print('sanitize case ok')
