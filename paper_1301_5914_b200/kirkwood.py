"""Analytic Kirkwood solutions for charges inside a dielectric sphere.

The validator that follows a solve for configs 1-2,
restated from the reference (``pbbem/kirkwood.py:59-263``): Laplace
harmonics inside, modified spherical Bessel functions k_n(kappa r) outside,
matched by continuity of phi and eps dphi/dr at r = a.  Vectorised over
charges and evaluation points (the reference loops over charges).

The O(N_c x n_terms) coefficients (the Bessel log-derivative recurrence,
the reaction coefficients, the trace rows) are computed here on the host, as
the reference computes them (``kirkwood_coefficients``); the
O(N_points x N_c x n_terms) Legendre sums -- the surface traces
(kirkwood.py:193-203) and the charge-charge energy (kirkwood.py:180-188) --
run in sm_100a kernels (csrc/hobi_kirkwood.cu) behind the C ABI and raise
without a device, like every other product path.  The numpy form of those
sums is test infrastructure, outside this package (tests/test_kirkwood.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .mesh import ChargeSystem
from .physics import FOUR_PI, KCAL_MOL_PER_E2_ANG, PhysicalParams


class NotCenteredError(ValueError):
    """The closed form was asked about an eccentric or multi-charge system."""


class SeriesDivergenceError(ValueError):
    """The requested truncation cannot converge for this geometry (kirkwood.py:30-31;
    part of the module's surface, raised by neither implementation)."""


@dataclass(frozen=True)
class SphereProblem:
    """Sphere of `radius` at the origin with strictly interior charges."""

    radius: float
    params: PhysicalParams
    charges: ChargeSystem

    def __post_init__(self):
        if not self.radius > 0.0:
            raise ValueError(f"radius must be positive, got {self.radius}")
        if len(self.charges):
            rho = np.linalg.norm(self.charges.positions, axis=1)
            bad = np.flatnonzero(rho >= self.radius - 1e-9)
            if bad.size:
                raise ValueError(f"charge {bad[0]} at distance {rho[bad[0]]} is not strictly "
                                 f"inside the sphere of radius {self.radius}")


def legendre_all(nmax: int, x) -> np.ndarray:
    """P_0..P_nmax at x by the three-term recurrence, shape (nmax+1,) + x.shape
    (kirkwood.py:59-71).  Host helper; the series sums run the same
    recurrence on the device (csrc/hobi_kirkwood.cu)."""
    x = np.asarray(x, dtype=float)
    out = np.zeros((nmax + 1,) + x.shape)
    out[0] = 1.0
    if nmax >= 1:
        out[1] = x
    for n in range(1, nmax):
        out[n + 1] = ((2 * n + 1) * x * out[n] - n * out[n - 1]) / (n + 1)
    return out


def modified_spherical_kn(nmax: int, x: float) -> np.ndarray:
    """k_0..k_nmax at x > 0 with k_0 = exp(-x)/x, by the upward recurrence
    k_{n+1} = k_{n-1} + (2n+1)/x k_n (stable upward; kirkwood.py:74-89)."""
    if x <= 0.0:
        raise ValueError(f"argument must be positive, got {x}")
    out = np.empty(nmax + 1)
    out[0] = np.exp(-x) / x
    if nmax >= 1:
        out[1] = out[0] * (1.0 + 1.0 / x)
    for n in range(1, nmax):
        out[n + 1] = out[n - 1] + ((2 * n + 1) / x) * out[n]
    return out


def bessel_log_derivative(nmax: int, x: float) -> np.ndarray:
    """x k_n'(x)/k_n(x), n = 0..nmax, through tau_n = k_n/k_{n-1} (never overflows);
    x = 0 is the Laplace limit -(n+1) (kirkwood.py:92-110)."""
    if x < 0.0:
        raise ValueError(f"argument must be nonnegative, got {x}")
    if x == 0.0:
        return -np.arange(1.0, nmax + 2.0)
    out = np.empty(nmax + 1)
    out[0] = -(1.0 + x)
    tau = 1.0 + 1.0 / x
    for n in range(1, nmax + 1):
        out[n] = -x / tau - (n + 1)
        tau = 1.0 / tau + (2 * n + 1) / x
    return out


@dataclass(frozen=True)
class KirkwoodSolution:
    energy: float
    phi: Callable[[np.ndarray], np.ndarray]
    dphi_dn: Callable[[np.ndarray], np.ndarray]
    tail_ratio: float
    converged: bool
    n_terms: int


def _directions(v):
    r = np.linalg.norm(v, axis=1)
    with np.errstate(invalid="ignore", divide="ignore"):
        u = np.where(r[:, None] > 0.0, v / r[:, None], 0.0)
    return r, u


def _gpu_traces(coef_phi, coef_dphi, units, rho, nmax):
    """Both traces at a set of points through hobi_kirkwood_traces (one launch)."""
    from . import _native as N
    from .solver import _device_index, _raise

    units, rho = N.f64(units), N.f64(rho)
    c1, c2 = N.f64(coef_phi), N.f64(coef_dphi)
    nc = rho.size

    def evaluate(points):
        pts = N.f64(points)
        single = pts.ndim == 1
        pts = np.ascontiguousarray(pts.reshape(-1, 3))
        m = pts.shape[0]
        phi, dphi = np.empty(m), np.empty(m)
        N.require_device()
        _raise(N.load().hobi_kirkwood_traces(_device_index(), N.dptr(pts), m, N.dptr(units), N.dptr(rho), nc,
                                             N.dptr(c1), N.dptr(c2), nmax + 1, N.dptr(phi), N.dptr(dphi)))
        return (phi[0], dphi[0]) if single else (phi, dphi)

    return evaluate


def _gpu_energy(units, q, reac, rpow, nmax):
    from . import _native as N
    from .solver import _device_index, _raise

    q = N.f64(q)
    terms = np.empty(q.size)
    if q.size:
        N.require_device()
        _raise(N.load().hobi_kirkwood_energy_terms(_device_index(), N.dptr(N.f64(units)), N.dptr(q), q.size,
                                                   N.dptr(N.f64(reac)), N.dptr(N.f64(rpow)), nmax + 1,
                                                   N.dptr(terms)))
    energy = 0.0
    for t in terms:  # charge order, like the reference's loop over j
        energy += float(t)
    return energy


@dataclass(frozen=True)
class KirkwoodCoefficients:
    """Per-charge multipole data of kirkwood_series (kirkwood.py:159-178)."""

    nmax: int
    rho: np.ndarray        # |y_k|
    units: np.ndarray      # y_k / |y_k| (0 for a charge at the centre)
    rpow: np.ndarray       # rho_k^n, (N_c, nmax+1)
    reac: np.ndarray       # reaction-field coefficients, (N_c, nmax+1)
    coef_phi: np.ndarray   # trace rows of phi, (N_c, nmax+1)
    coef_dphi: np.ndarray  # trace rows of dphi/dn, (N_c, nmax+1)
    tail_ratio: float


def kirkwood_coefficients(problem: SphereProblem, n_terms: int = 40) -> KirkwoodCoefficients:
    """The O(N_c x n_terms) part of kirkwood_series, on the host as the
    reference computes it; the truncation check is its tail ratio."""
    if n_terms < 1:
        raise ValueError(f"n_terms must be >= 1, got {n_terms}")
    nmax = n_terms - 1
    a, p = problem.radius, problem.params
    q = problem.charges.charges
    rho, units = _directions(problem.charges.positions)
    n = np.arange(nmax + 1, dtype=float)
    ell = bessel_log_derivative(nmax, p.kappa * a)
    with np.errstate(divide="ignore", invalid="ignore"):
        rpow = np.where(rho[:, None] > 0.0, rho[:, None] ** n[None, :], 0.0)
    rpow[:, 0] = 1.0
    alpha = q[:, None] * rpow / (FOUR_PI * p.eps1)
    reac = alpha * (a ** -(2 * n + 1.0) * (p.eps2 * ell + (n + 1) * p.eps1) / (n * p.eps1 - p.eps2 * ell))
    coef_phi = alpha * a ** -(n + 1.0) + reac * a**n
    coef_dphi = -(n + 1.0) * alpha * a ** -(n + 2.0) + n * reac * a ** (n - 1.0)
    if nmax >= 1 and len(q):
        last, prev = np.abs(coef_phi[:, nmax]), np.abs(coef_phi[:, nmax - 1])
        tail = float(np.where(last > 0.0, last / np.maximum(prev, 1e-300), 0.0).max())
    else:
        tail = 1.0 if np.abs(coef_phi).max(initial=0.0) > 0.0 else 0.0
    return KirkwoodCoefficients(nmax, rho, units, rpow, reac, coef_phi, coef_dphi, tail)


def kirkwood_series(problem: SphereProblem, n_terms: int = 40) -> KirkwoodSolution:
    """Multipole solution for arbitrary interior charges (kirkwood.py:159-220):
    coefficients on the host, the energy and the traces on the device (no
    CPU fallback: raises without one)."""
    c = kirkwood_coefficients(problem, n_terms)
    q = problem.charges.charges
    energy = _gpu_energy(c.units, q, c.reac, c.rpow, c.nmax) * (FOUR_PI * KCAL_MOL_PER_E2_ANG)
    both = _gpu_traces(c.coef_phi, c.coef_dphi, c.units, c.rho, c.nmax)
    return KirkwoodSolution(energy=energy, phi=lambda points: both(points)[0],
                            dphi_dn=lambda points: both(points)[1], tail_ratio=c.tail_ratio,
                            converged=c.tail_ratio <= 0.99, n_terms=n_terms)


def kirkwood_centered(problem: SphereProblem):
    """Closed form for one charge at the centre (kirkwood.py:223-263):
    returns (E_sol, phi(points), dphi_dn(points)) with constant traces."""
    if len(problem.charges) != 1:
        raise NotCenteredError(f"closed form needs exactly one centered charge, got "
                               f"{len(problem.charges)}; use kirkwood_series")
    if float(np.linalg.norm(problem.charges.positions[0])) > 1e-12:
        raise NotCenteredError("closed form needs the charge at the center; use kirkwood_series")
    a, p = problem.radius, problem.params
    q = float(problem.charges.charges[0])
    screen = 1.0 + p.kappa * a
    energy = KCAL_MOL_PER_E2_ANG * q * q / (2.0 * a) * (1.0 / (p.eps2 * screen) - 1.0 / p.eps1)

    def const(value):
        def fn(points):
            pts = np.asarray(points, dtype=float)
            return value if pts.ndim == 1 else np.full(pts.shape[0], value)

        return fn

    return (energy, const(q / (FOUR_PI * p.eps2 * a * screen)),
            const(-q / (FOUR_PI * p.eps1 * a * a)))
