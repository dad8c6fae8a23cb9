"""B200-native HOBI-PB: the dense boundary-integral matvec of arXiv 1301.5914
and everything around it on the device (geometry, singular swap, sources,
GMRES, energy, NCCL row split), behind the reference package's Python API
(``pbbem``).  Kernels: ``csrc/`` -> ``libhobi.so`` (sm_100a);
C ABI: ``include/hobi.h``.
"""

from . import geometry, kernels  # noqa: F401  (pbbem.geometry / pbbem.kernels on the device)
from .mesh import (ChargeSystem, FlatMesh, MeshFormatError, MeshValidationError, flat_area,
                   icosahedral_sphere, parse_charges, parse_msms, radial_project, write_msms)
from .physics import FOUR_PI, KCAL_MOL_PER_E2_ANG, PhysicalParams, SingularityError
from .kirkwood import SphereProblem, kirkwood_centered, kirkwood_series
from .quadrature import TriangleRule, duffy_rule, gauss_radau_rule
from .report import RunReport, ScalingRow
from .solver import (
    DegenerateArcError,
    DiscretizedProblem,
    GmresNonConvergence,
    GpuOperator,
    SolverConfig,
    SurfaceSolution,
    apply_rows,
    assemble_rhs,
    convergence_order,
    discretize,
    gmres_solve,
    make_operator,
    matvec_hobi,
    matvec_lobi,
    partition_targets,
    solvation_energy,
    solve,
    surface_potential_error,
)

__version__ = "0.1.0"

__all__ = [
    "ChargeSystem", "DegenerateArcError", "DiscretizedProblem", "FOUR_PI", "FlatMesh",
    "GmresNonConvergence", "GpuOperator", "KCAL_MOL_PER_E2_ANG", "MeshFormatError",
    "MeshValidationError", "PhysicalParams", "SingularityError", "SolverConfig", "SurfaceSolution",
    "TriangleRule", "apply_rows", "assemble_rhs", "convergence_order", "discretize", "duffy_rule",
    "gauss_radau_rule", "gmres_solve", "icosahedral_sphere", "make_operator", "matvec_hobi",
    "matvec_lobi", "partition_targets", "solvation_energy", "solve", "surface_potential_error",
    "flat_area", "parse_charges", "parse_msms", "radial_project", "write_msms",
    "SphereProblem", "kirkwood_centered", "kirkwood_series", "RunReport", "ScalingRow",
]
