import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
from conftest import golden
from paper_1301_5914_b200 import _native as N
g = golden("kernels"); n = g["d"].shape[0]
r = np.linalg.norm(g["d"], axis=1)
for tag in "abcd":
    e1, e2, kap = g["params_" + tag]
    k = np.empty((4, n))
    N.check(N.load().hobi_kernel_values(0, N.dptr(N.f64(g["d"])), N.dptr(N.f64(g["nx"])), N.dptr(N.f64(g["ny"])), n, e1, e2, kap, N.dptr(k)))
    ref = g["K_" + tag]
    for i in range(4):
        den = np.abs(ref[i]); m = den > 0
        rel = np.zeros(n); rel[m] = np.abs(k[i]-ref[i])[m]/den[m]
        j = np.argmax(rel)
        print(tag, i, 'max rel %.2e at r=%.3e (kr=%.2e)' % (rel.max(), r[j], kap*r[j]), 'n_ne', (k[i]!=ref[i]).sum(), 'zeros-ok', np.all(k[i][~m]==0))
