"""Host (numpy) Legendre sums of the Kirkwood series -- TEST INFRASTRUCTURE ONLY.

The product evaluates kirkwood_series' O(N_points x N_c x n_terms) sums on the
device (paper_1301_5914_b200/kirkwood.py -> csrc/hobi_kirkwood.cu).  This
module restates those sums in numpy over the product's host coefficients
(``kirkwood_coefficients``), so the CPU suite can pin the coefficient code
against the reference's outputs (tests/golden/kirkwood.npz, made by
``pbbem.kirkwood.kirkwood_series``) and the GPU suite can check the device sums
against an independent evaluation.  Follows ``pbbem/kirkwood.py``:
legendre_all (:59-71), the energy loop (:180-188), the traces (:193-203).

Status: parity PINNED (tests/test_kirkwood.py).  Who may use it: tests only;
the product package never imports it.
"""

from __future__ import annotations

import numpy as np

from paper_1301_5914_b200.kirkwood import (KirkwoodSolution, SphereProblem, _directions,
                                           kirkwood_coefficients)
from paper_1301_5914_b200.physics import FOUR_PI, KCAL_MOL_PER_E2_ANG


def legendre_table(nmax: int, x) -> np.ndarray:
    """P_0..P_nmax(x) by the three-term recurrence (kirkwood.py:59-71);
    shape (nmax+1,) + x.shape."""
    x = np.asarray(x, dtype=float)
    out = np.empty((nmax + 1,) + x.shape)
    out[0] = 1.0
    if nmax >= 1:
        out[1] = x
    for n in range(1, nmax):
        out[n + 1] = ((2 * n + 1) * x * out[n] - n * out[n - 1]) / (n + 1)
    return out


def kirkwood_series_host(problem: SphereProblem, n_terms: int = 40) -> KirkwoodSolution:
    """kirkwood_series with the Legendre sums in numpy."""
    c = kirkwood_coefficients(problem, n_terms)
    q = problem.charges.charges
    nmax = c.nmax
    # E = 1/2 sum_j q_j phi_reac(y_j): P_n(u_j . u_k) for all charge pairs at once
    pn = legendre_table(nmax, np.clip(c.units @ c.units.T, -1.0, 1.0)) if len(q) else np.zeros((nmax + 1, 0, 0))
    energy = 0.0
    for j in range(len(q)):
        energy += 0.5 * q[j] * float((c.reac * c.rpow[j][None, :] * pn[:, :, j].T).sum())
    energy *= FOUR_PI * KCAL_MOL_PER_E2_ANG

    def trace(coef):
        def evaluate(points):
            pts = np.asarray(points, dtype=float)
            single = pts.ndim == 1
            pts = pts.reshape(-1, 3)
            _, rad = _directions(pts)
            cos = rad @ c.units.T  # (m, nc)
            cos[:, c.rho == 0.0] = 1.0
            out = np.einsum("kn,nmk->m", coef, legendre_table(nmax, cos))
            return out[0] if single else out

        return evaluate

    return KirkwoodSolution(energy=energy, phi=trace(c.coef_phi), dphi_dn=trace(c.coef_dphi),
                            tail_ratio=c.tail_ratio, converged=c.tail_ratio <= 0.99, n_terms=n_terms)
