"""Group-operator overhead on one GPU: config-4 matvec through one context vs
a group whose members are replicas on the same device (peer copies become
device copies; the rows of both members share the GPU)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_1301_5914_b200 import PhysicalParams, SolverConfig, discretize, matvec_hobi
from paper_1301_5914_b200.solver import GpuOperator
from paper_1301_5914_b200.surfaces import baseline_config
cfg = baseline_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
prob = discretize(cfg.mesh, PhysicalParams(cfg.eps1, cfg.eps2, cfg.kappa), cfg.charges, SolverConfig(workers=1))
u = np.random.default_rng(0).standard_normal(prob.n_unknowns)
def timeit(f, n=5):
    f(); t = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t) / n * 1e3
t1 = timeit(lambda: matvec_hobi(prob, u))
print(f"{cfg.name}: one context {t1:.3f} ms per host-buffer matvec")
for k in (2, 4, 8):
    with GpuOperator(prob, k, devices=[prob.device] * k) as op:
        tk = timeit(lambda: op(u))
    print(f"group of {k} replicas on one GPU: {tk:.3f} ms ({100 * (tk / t1 - 1):+.2f} %)")
