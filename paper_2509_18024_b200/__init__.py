"""B200-native core-elements ALS (arXiv 2509.18024): a drop-in for the
reference package's ``core`` method path (``coreals.fit_core`` and its
sketch / update / predict entry points), running every half-sweep as
hand-written sm_100a CUDA kernels behind the C ABI in include/coreals_b200.h.
"""

from .als import FactorPair, FitReport, SolverConfig, init_factors, predict, predict_entries, predict_full
from .core import SparseSketch, ces_sketch, fit, fit_core, fit_fast_core, sketch_budget, update_item_core, update_user_core
from .driver import fit_method
from .errors import ConfigError, DataError, NumericalError
from .metrics import EvalResult, evaluate, hit_at_k, ndcg_at_k, prmse, relevance_threshold, rmse
from . import serialize
from .ratings import DeviceRatingMatrix, RatingMatrix, build_rating_matrix, read_ratings_csv, write_ratings_csv

__all__ = [
    "FactorPair", "FitReport", "SolverConfig", "init_factors", "predict", "predict_entries", "predict_full",
    "SparseSketch", "ces_sketch", "fit", "fit_core", "fit_fast_core", "sketch_budget", "update_item_core", "update_user_core",
    "fit_method", "ConfigError", "DataError", "NumericalError", "RatingMatrix", "DeviceRatingMatrix",
    "build_rating_matrix", "read_ratings_csv", "write_ratings_csv", "serialize",
    "EvalResult", "evaluate", "hit_at_k", "ndcg_at_k", "prmse", "relevance_threshold", "rmse",
]

__version__ = "0.1.0"
