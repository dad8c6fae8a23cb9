"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved: configs 1-2 are icosphere
spheres with interior charges, configs 3-5 a star-shaped "globular molecule"

    r(u) = R0 * (1 + p(u)),   p(u) = 0.15 * s * sum_{l=2..6, m=-l..l} a_lm Y_lm(u)

with a_lm ~ N(0, 1)/(l+1) drawn from ``default_rng(surface_seed)`` in (l, m)
order, and ``s = min(1, 0.3 / max|0.15 * sum|)`` over the directions of a
level-6 icosphere (the "normalised so that max|perturbation| <= 0.3" clause,
read as "scale down only if the cap binds").  Y_lm are orthonormal real
spherical harmonics with the Condon-Shortley phase (m > 0: sqrt2*Re, m < 0:
sqrt2*Im of |m|).  Vertices are an icosphere radially mapped onto r(u); vertex
normals are the analytic gradient of the implicit surface |x| - r(x/|x|),
``n ~ u - grad_S p(u) / (1 + p(u))``, evaluated through real solid harmonics so
the poles need no special case.  Charges are uniform inside 0.8 r(u) by
rejection, q ~ N(0, 0.4) re-centred to net zero.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .mesh import ChargeSystem, FlatMesh, icosahedral_sphere, unit_icosphere


def _solid_harmonics(u, lmax):
    """Real solid harmonics R_lm(u) = |u|^l Y_lm(u/|u|) and their gradients.

    Returns dict (l, m) -> (value (n,), gradient (n, 3)).  Uses
    (x + i y)^m for the azimuthal part and the associated-Legendre recurrence
    on q_l^m = r^(l-m) P_l^(m)(z/r) (a polynomial in z and r^2).
    """
    x, y, z = u[:, 0], u[:, 1], u[:, 2]
    n = u.shape[0]
    zero = np.zeros(n)
    ex = np.stack([np.ones(n), zero, zero], 1)
    ey = np.stack([zero, np.ones(n), zero], 1)
    ez = np.stack([zero, zero, np.ones(n)], 1)
    r2 = x * x + y * y + z * z
    gr2 = 2.0 * u
    # C_m + i S_m = (x + i y)^m with gradients
    C = [np.ones(n)]
    S = [np.zeros(n)]
    gC = [np.zeros((n, 3))]
    gS = [np.zeros((n, 3))]
    for m in range(1, lmax + 1):
        C.append(x * C[-1] - y * S[-1])
        S.append(x * S[-1] + y * C[-2])
        gC.append(m * (C[m - 1][:, None] * ex - S[m - 1][:, None] * ey))
        gS.append(m * (S[m - 1][:, None] * ex + C[m - 1][:, None] * ey))
    out = {}
    for m in range(0, lmax + 1):
        dfact = 1.0
        for k in range(1, 2 * m, 2):
            dfact *= k
        q = {m: (np.full(n, dfact), np.zeros((n, 3)))}
        if m + 1 <= lmax:
            q0, g0 = q[m]
            q[m + 1] = ((2 * m + 1) * z * q0, (2 * m + 1) * (z[:, None] * g0 + q0[:, None] * ez))
        for l in range(m + 2, lmax + 1):
            q1, g1 = q[l - 1]
            q2, g2 = q[l - 2]
            val = ((2 * l - 1) * z * q1 - (l + m - 1) * r2 * q2) / (l - m)
            grad = ((2 * l - 1) * (z[:, None] * g1 + q1[:, None] * ez)
                    - (l + m - 1) * (r2[:, None] * g2 + q2[:, None] * gr2)) / (l - m)
            q[l] = (val, grad)
        for l in range(max(m, 2), lmax + 1):
            norm = math.sqrt((2 * l + 1) / (4 * math.pi) * math.factorial(l - m) / math.factorial(l + m))
            sign = -1.0 if m % 2 else 1.0  # Condon-Shortley
            ql, gql = q[l]
            if m == 0:
                out[(l, 0)] = (norm * ql, norm * gql)
                continue
            c = math.sqrt(2.0) * norm * sign
            out[(l, m)] = (c * C[m] * ql, c * (gC[m] * ql[:, None] + C[m][:, None] * gql))
            out[(l, -m)] = (c * S[m] * ql, c * (gS[m] * ql[:, None] + S[m][:, None] * gql))
    return out


@dataclass(frozen=True)
class StarShape:
    """Star-shaped radius function r(u) = R0 (1 + p(u)) on unit directions u."""

    radius: float
    coeffs: tuple  # ((l, m, a_lm), ...)
    scale: float  # 0.15 * s

    @staticmethod
    def from_seed(radius: float, seed: int, amplitude: float = 0.15, cap: float = 0.3):
        rng = np.random.default_rng(seed)
        coeffs = []
        for l in range(2, 7):
            for m in range(-l, l + 1):
                coeffs.append((l, m, float(rng.standard_normal()) / (l + 1)))
        shape = StarShape(radius, tuple(coeffs), amplitude)
        probe, _ = unit_icosphere(6)
        peak = float(np.abs(shape.perturbation(probe)[0]).max())
        s = 1.0 if peak <= cap else cap / peak
        return StarShape(radius, tuple(coeffs), amplitude * s)

    def perturbation(self, u):
        """p(u) and its tangential gradient on the unit sphere, for unit rows u."""
        sh = _solid_harmonics(u, 6)
        f = np.zeros(u.shape[0])
        g = np.zeros_like(u)
        for l, m, a in self.coeffs:
            v, gv = sh[(l, m)]
            f += a * v
            g += a * (gv - l * v[:, None] * u)  # degree-0 extension: tangential part
        return self.scale * f, self.scale * g

    def surface(self, level: int) -> FlatMesh:
        u, faces = unit_icosphere(level)
        p, gp = self.perturbation(u)
        verts = (self.radius * (1.0 + p))[:, None] * u
        nrm = u - gp / (1.0 + p)[:, None]
        nrm /= np.sqrt(np.einsum("ij,ij->i", nrm, nrm))[:, None]
        return FlatMesh(vertices=verts, normals=nrm, faces=faces)

    def interior_charges(self, count: int, seed: int, frac: float = 0.8, sigma: float = 0.4):
        rng = np.random.default_rng(seed)
        rmax = frac * self.radius * (1.0 + 0.3)
        pts = []
        while len(pts) < count:
            cand = rng.uniform(-rmax, rmax, size=(4 * count, 3))
            rho = np.sqrt(np.einsum("ij,ij->i", cand, cand))
            ok = rho > 0.0
            cand, rho = cand[ok], rho[ok]
            p, _ = self.perturbation(cand / rho[:, None])
            inside = rho < frac * self.radius * (1.0 + p)
            pts.extend(cand[inside][: count - len(pts)])
        pos = np.asarray(pts[:count])
        q = rng.normal(0.0, sigma, size=count)
        q -= q.mean()
        return ChargeSystem(positions=pos, charges=q)


def sphere_charges(count: int, radius: float, seed: int) -> ChargeSystem:
    """`count` charges of seeded sign +-1, uniform in the ball |x| < radius (config 2)."""
    rng = np.random.default_rng(seed)
    pts = []
    while len(pts) < count:
        c = rng.uniform(-radius, radius, size=3)
        if float(np.sqrt(c @ c)) < radius:
            pts.append(c)
    signs = rng.choice([-1.0, 1.0], size=count)
    return ChargeSystem(positions=np.asarray(pts), charges=signs)


@dataclass(frozen=True)
class Config:
    name: str
    mesh: FlatMesh
    charges: ChargeSystem
    eps1: float
    eps2: float
    kappa: float
    restart: int
    tol: float = 1e-6
    sphere_radius: float | None = None  # set for the analytic-Kirkwood spheres


def baseline_config(index: int, level: int | None = None) -> Config:
    """BASELINE.json configs[index - 1] (1-based, as SURVEY.md names them C1..C5).

    ``level`` overrides the icosphere level (used by tests to shrink a config).
    """
    if index == 1:
        lv = 3 if level is None else level
        return Config("C1 Kirkwood sphere L%d" % lv, icosahedral_sphere(lv, 2.0),
                      ChargeSystem(positions=[[0.0, 0.0, 0.0]], charges=[1.0]),
                      1.0, 80.0, 0.1257, 10, sphere_radius=2.0)
    if index == 2:
        lv = 4 if level is None else level
        return Config("C2 off-centre sphere L%d" % lv, icosahedral_sphere(lv, 2.0),
                      sphere_charges(8, 1.2, 1234), 1.0, 80.0, 0.1257, 10, sphere_radius=2.0)
    table = {3: (5, 16.0, 500, 2.0), 4: (6, 30.0, 2000, 4.0), 5: (7, 50.0, 10000, 1.0)}
    if index not in table:
        raise ValueError(f"config index must be 1..5, got {index}")
    lv0, r0, nc, eps1 = table[index]
    lv = lv0 if level is None else level
    shape = StarShape.from_seed(r0, seed=3)
    return Config(f"C{index} star R0={r0:g} L{lv}", shape.surface(lv),
                  shape.interior_charges(nc, seed=4), eps1, 80.0, 0.1257, 20)
