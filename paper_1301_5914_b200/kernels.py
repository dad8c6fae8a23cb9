"""The reference's ``pbbem.kernels`` module surface on the device.

``kernel_values_d`` / ``kernel_values`` / ``kernel_block`` (kernels.py:88-141)
run the literal K1..K4 transcription of ``csrc/hobi_literal.cu``
(``hobi_kernel_values``); ``source_terms_at`` / ``source_terms``
(kernels.py:144-178) run the right-hand-side kernel at arbitrary points
(``hobi_source_terms``).  The all-pairs sweep does not go through this module:
it evaluates the same kernels in its fused form (``csrc/hobi_fastmath.cuh``).
``g0`` / ``g_kappa`` are the scalar closed forms (kernels.py:66-81).
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as N
from .mesh import ChargeSystem
from .physics import FOUR_PI, KCAL_MOL_PER_E2_ANG, PhysicalParams, SingularityError

__all__ = ["FOUR_PI", "KCAL_MOL_PER_E2_ANG", "PhysicalParams", "SingularityError", "g0", "g_kappa",
           "kernel_values", "kernel_values_d", "kernel_block", "source_terms", "source_terms_at"]


def _distance(x, y) -> float:
    d = np.asarray(x, dtype=float) - np.asarray(y, dtype=float)
    return math.sqrt(float(np.dot(d, d)))


def g0(x, y) -> float:
    """1/(4 pi |x-y|) (kernels.py:66-72)."""
    r = _distance(x, y)
    if r < 1e-300:
        raise SingularityError("g0 evaluated at coincident points")
    return 1.0 / (FOUR_PI * r)


def g_kappa(x, y, kappa: float) -> float:
    """exp(-kappa |x-y|)/(4 pi |x-y|) (kernels.py:75-81)."""
    r = _distance(x, y)
    if r < 1e-300:
        raise SingularityError("g_kappa evaluated at coincident points")
    return math.exp(-kappa * r) / (FOUR_PI * r)


def kernel_values_d(d, nx, ny, params: PhysicalParams, device: int = 0):
    """K1..K4 from displacements d = x - y, all broadcastable (..., 3)
    (kernels.py:99-130), evaluated on the device."""
    d, nx, ny = np.broadcast_arrays(np.asarray(d, dtype=float), np.asarray(nx, dtype=float),
                                    np.asarray(ny, dtype=float))
    if d.shape[-1] != 3:
        raise ValueError(f"last axis must have length 3, got shape {d.shape}")
    shape = d.shape[:-1]
    n = int(np.prod(shape, dtype=np.int64))
    k = np.empty((4, n))
    if n:
        N.require_device()
        dd, dx, dy = (N.f64(a.reshape(n, 3)) for a in (d, nx, ny))
        N.check(N.load().hobi_kernel_values(device, N.dptr(dd), N.dptr(dx), N.dptr(dy), n,
                                            params.eps1, params.eps2, params.kappa, N.dptr(k)))
    return tuple(k[i].reshape(shape) for i in range(4))


def kernel_values(x, nx, y, ny, params: PhysicalParams, device: int = 0):
    """K1..K4 over broadcastable (..., 3) points (kernels.py:88-96); the caller
    excludes coincident pairs."""
    return kernel_values_d(np.asarray(x, dtype=float) - np.asarray(y, dtype=float), nx, ny, params, device)


def kernel_block(x, nx, y, ny, params: PhysicalParams):
    """Scalar (K1, K2, K3, K4) of one pair, coincidence checked (kernels.py:133-141)."""
    d = np.asarray(x, dtype=float) - np.asarray(y, dtype=float)
    if float(np.dot(d, d)) < 1e-300:
        raise SingularityError("kernel_block evaluated at coincident points")
    k1, k2, k3, k4 = kernel_values_d(d, nx, ny, params)
    return float(k1), float(k2), float(k3), float(k4)


def source_terms_at(points, normals, charges: ChargeSystem, device: int = 0):
    """(S1, S2) at many surface points, (m, 3) -> two (m,) (kernels.py:159-178)."""
    points = N.f64(np.asarray(points, dtype=float))
    normals = N.f64(np.asarray(normals, dtype=float))
    m = points.shape[0]
    s1, s2 = np.zeros(m), np.zeros(m)
    nc = len(charges)
    if m == 0 or nc == 0:
        return s1, s2
    N.require_device()
    qpos, q = N.f64(charges.positions), N.f64(charges.charges)
    try:
        N.check(N.load().hobi_source_terms(device, N.dptr(points), N.dptr(normals), m, N.dptr(qpos),
                                           N.dptr(q), nc, N.dptr(s1), N.dptr(s2)))
    except N.NativeError as e:
        if e.status == N.HOBI_ERR_SINGULARITY:
            raise SingularityError(str(e)) from None
        raise
    return s1, s2


def source_terms(x, nx, charges: ChargeSystem):
    """(S1, S2) at one surface point (kernels.py:144-156)."""
    s1, s2 = source_terms_at(np.asarray(x, dtype=float).reshape(1, 3),
                             np.asarray(nx, dtype=float).reshape(1, 3), charges)
    return float(s1[0]), float(s2[0])
