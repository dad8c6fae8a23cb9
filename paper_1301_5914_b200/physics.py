"""Physical parameters and unit constants (pbbem/kernels.py:27-63)."""

from __future__ import annotations

import math
from dataclasses import dataclass

FOUR_PI = 4.0 * math.pi
KCAL_MOL_PER_E2_ANG = 332.0716  # e^2/(4 pi eps0 Angstrom) in kcal/mol


class SingularityError(ValueError):
    """Evaluation point coincides with a source point (kernels.py:36-37)."""


@dataclass(frozen=True)
class PhysicalParams:
    """Interior/exterior dielectric and inverse Debye length (kernels.py:40-63).

    The kernels use er = eps2/eps1 and the right-hand side is divided by eps1
    (kernels.py:11-16, solver.py:393-402) -- the code's convention, not the
    paper's eps = eps1/eps2 (kept here for reporting only).
    """

    eps1: float
    eps2: float
    kappa: float

    def __post_init__(self):
        if not self.eps1 > 0.0:
            raise ValueError(f"eps1 must be positive, got {self.eps1}")
        if not self.eps2 > 0.0:
            raise ValueError(f"eps2 must be positive, got {self.eps2}")
        if not self.kappa >= 0.0:
            raise ValueError(f"kappa must be nonnegative, got {self.kappa}")

    @property
    def eps(self) -> float:
        return self.eps1 / self.eps2
