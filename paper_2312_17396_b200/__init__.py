"""B200-native mixed-precision Paterson-Stockmeyer evaluation of matrix
polynomials (arXiv 2312.17396): a drop-in for the hot path of the reference
package ``mpps`` (pkg/src/mpps/__init__.py:28-45 names).

Host side (this package): the reference's entry points, plan and report
records and a bit-exact precision planner.  Device side: the sm_100a kernels
of ``_lib/libmpps_b200.so`` behind the C-ABI in ``include/mpps_b200.h``.
"""

from .precision import (BOUND_CTX, DD, FP32, FP64, LATTICE, NORM_CTX, QD,
                        DimensionError, MatBatch, PrecisionCtx,
                        UnsupportedPrecisionError, format_for_digits)
from .coefficients import (CoefficientSeries, eval_coeff, make_series,
                           pade_exp_coeffs, series_from_json, series_to_json,
                           taylor_cos_coeffs, taylor_exp_coeffs)
from .planner import (EvaluationPlan, cost_ratio, default_block_size,
                      plan_precisions, snap_to_lattice)
from .bounds import (BoundInputs, BoundInvalidError, extra_squarings, gamma,
                     tau_sequence, thm21_bound)
from .engine import (BatchReport, EvaluationReport, cos_argument, horner_mixed, plan_only, ps_mixed_pade,
                     ps_fixed, ps_mixed_exp, ps_mixed_general, submit_mixed_exp, submit_mixed_general,
                     PendingEvaluation)

from .complexmat import ComplexMatBatch
from .expm import expm_ss
from . import ops, summa, pipeline, matio, harness
from .harness import compare, reference_eval, relative_error
from .matio import matrix_from_csv, matrix_from_json, matrix_to_csv, matrix_to_json

__version__ = "0.1.0"

__all__ = [
    "BOUND_CTX", "NORM_CTX", "DimensionError", "PrecisionCtx", "MatBatch",
    "UnsupportedPrecisionError", "format_for_digits", "FP32", "FP64", "DD", "QD", "LATTICE",
    "CoefficientSeries", "eval_coeff", "make_series", "pade_exp_coeffs",
    "series_from_json", "series_to_json", "taylor_cos_coeffs", "taylor_exp_coeffs",
    "EvaluationPlan", "EvaluationReport", "BatchReport", "cost_ratio", "cos_argument",
    "default_block_size", "horner_mixed", "plan_only", "plan_precisions",
    "ps_fixed", "ps_mixed_exp", "ps_mixed_general", "submit_mixed_exp", "submit_mixed_general",
    "PendingEvaluation", "snap_to_lattice",
    "BoundInputs", "BoundInvalidError", "extra_squarings", "gamma",
    "tau_sequence", "thm21_bound", "expm_ss", "ops", "summa", "ps_mixed_pade",
    "ComplexMatBatch", "harness", "reference_eval", "relative_error", "compare", "matio", "matrix_to_json", "matrix_from_json", "matrix_to_csv", "matrix_from_csv",
]
