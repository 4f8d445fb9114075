"""B200-native hot path of arXiv 2408.03571: GMRES + two-level Bezier-Schwarz for 2-D Helmholtz.

Public names mirror the reference package ``helmdd`` (``__init__.py:5-37``) for
the operators on the hot path; the arithmetic runs in ``libhelmb200.so``
(hand-written sm_100a CUDA kernels behind a C ABI, ``include/helmb200.h``).
"""

from .discretization import (
    CoarseSpace,
    Decomposition,
    Grid,
    Partition,
    build_focs,
    build_hocs,
    extend,
    extend_max,
    max_overlap_layers,
    partition,
)
from .fdm_setup import SingularMatrixError
from .gmres import GmresConfig, SolveReport, gmres, gmres_multi
from .operators import (
    HelmholtzOperator,
    HelmholtzProblem,
    SchwarzPreconditioner,
    assemble,
    coarse_correct,
    galerkin,
)

__all__ = [
    "CoarseSpace",
    "Decomposition",
    "GmresConfig",
    "Grid",
    "HelmholtzOperator",
    "HelmholtzProblem",
    "Partition",
    "SchwarzPreconditioner",
    "SingularMatrixError",
    "SolveReport",
    "assemble",
    "build_focs",
    "build_hocs",
    "coarse_correct",
    "extend",
    "extend_max",
    "galerkin",
    "gmres",
    "gmres_multi",
    "max_overlap_layers",
    "partition",
]

__version__ = "0.1.0"
