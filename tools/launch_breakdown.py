"""Scratch: one solve of a config with per-kernel device times via the GMRES trace."""
import sys
sys.path.insert(0, '.')
from paper_1301_5914_b200 import discretize, PhysicalParams, SolverConfig, assemble_rhs, make_operator, gmres_solve
from paper_1301_5914_b200.surfaces import baseline_config
idx = int(sys.argv[1])
cfg = baseline_config(idx)
scfg = SolverConfig(workers=1, restart=cfg.restart)
prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, scfg)
b = assemble_rhs(prob)
for _ in range(2):
    with make_operator(prob, scfg) as op:
        sol = gmres_solve(op, b, scfg)
print(sol.iterations)
