"""B200-native Randomly Pivoted LU (arXiv 2601.22344) — the RPLU pivot loop.

Drop-in for the hot entry points of the reference package ``rplu`` 0.1.0
(``pkg/src/rplu/__init__.py:14-36`` re-exports): the same names, signatures,
exception classes and uniform-stream consumption, computed by hand-written
sm_100a kernels in ``librplu_b200.so`` (C ABI: ``include/rplu_b200.h``).

There is no CPU fallback: without the built extension or a CUDA device the
entry points raise.
"""

__version__ = "0.1.0"

from .accessors import CallableOperator, CapabilityError, DenseMatrix, MatrixAccessor, materialize
from .cauchy import (CauchyLikeMatrix, StructuredPivotTrace, exact_row_norms,
                     generator_schur_update, loewner_build, structured_eliminate)
from .dense_pivots import EliminationTrace, PivotRule, eliminate
from .lowmem_cur import (CurBuildInfo, CurFactorization, core_extend, cur_build, residual_column,
                         residual_row)
from .operators import GaussianKernelOperator
from .precond import GmresResult, SmwPreconditioner, device_callable, gmres, smw_build
from .rational import BarycentricRational, SampleSet, aaa, bary_eval, cur_aaa
from .rng import RngState, sample_index
from . import errors, sweep  # noqa: F401  (§8(f2) error evaluation / sweep harness)
from .treebounds import (CoincidentPointsError, InteractionPlan, PointQuadtree, build_plan,
                         certified_upper_bounds)

__all__ = [
    "CallableOperator", "CapabilityError", "DenseMatrix", "MatrixAccessor", "materialize",
    "CauchyLikeMatrix", "StructuredPivotTrace", "exact_row_norms", "generator_schur_update",
    "structured_eliminate", "loewner_build",
    "EliminationTrace", "PivotRule", "eliminate",
    "CurBuildInfo", "CurFactorization", "core_extend", "cur_build", "residual_column",
    "residual_row", "GaussianKernelOperator",
    "RngState", "sample_index",
    "CoincidentPointsError", "InteractionPlan", "PointQuadtree", "build_plan",
    "certified_upper_bounds",
    "BarycentricRational", "SampleSet", "aaa", "bary_eval", "cur_aaa",
    "GmresResult", "SmwPreconditioner", "device_callable", "gmres", "smw_build",
]
