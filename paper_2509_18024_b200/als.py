"""Types and helpers shared with the reference's ALS module.

Mirrors the public types of /root/reference/pkg/src/coreals/als.py
(FactorPair :40-59, SolverConfig :62-95, FitReport :98-112, init_factors
:117-131, predict/predict_entries/predict_full :134-157) so callers of the
reference keep working.  Only method "core" is implemented on the GPU by this
package; the other reference methods are outside its scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError

__all__ = [
    "FactorPair", "SolverConfig", "FitReport", "init_factors",
    "predict", "predict_entries", "predict_full", "METHODS",
]

METHODS = ("full", "core", "fast_core", "unif", "blev")
INIT_SCHEMES = ("uniform", "normal")

#: relative diagonal jitter applied once when a Gram factorization fails (als.py:37)
JITTER_SCALE = 1e-10


@dataclass
class FactorPair:
    """Dense user factors (n_users, n_f) and item factors (n_items, n_f), float64 on the host."""

    user_factors: np.ndarray
    item_factors: np.ndarray

    def __post_init__(self):
        self.user_factors = np.ascontiguousarray(self.user_factors, dtype=np.float64)
        self.item_factors = np.ascontiguousarray(self.item_factors, dtype=np.float64)
        if self.user_factors.ndim != 2 or self.item_factors.ndim != 2 \
                or self.user_factors.shape[1] != self.item_factors.shape[1]:
            raise ConfigError("factor matrices must be 2-d with a common rank")

    @property
    def n_f(self):
        return int(self.user_factors.shape[1])

    def copy(self):
        return FactorPair(self.user_factors.copy(), self.item_factors.copy())


@dataclass
class SolverConfig:
    """Method selection and hyperparameters for one fit (validation as als.py:80-95)."""

    method: str = "full"
    n_f: int = 10
    lam: float = 0.1
    rate: float = 1.0
    max_iters: int = 50
    tol: float = 0.01
    seed: int = 0
    init_scheme: str = "uniform"
    diagnostics: bool = False

    def __post_init__(self):
        self.method = str(self.method).lower()
        if self.method not in METHODS:
            raise ConfigError(f"unknown method {self.method!r}; expected one of {METHODS}")
        if self.n_f < 1:
            raise ConfigError("n_f must be >= 1")
        if self.lam < 0:
            raise ConfigError("lambda must be >= 0")
        if not 0.0 < self.rate <= 1.0:
            raise ConfigError("rate must be in (0, 1]")
        if self.max_iters < 0:
            raise ConfigError("max_iters must be >= 0")
        if not self.tol > 0:
            raise ConfigError("tol must be > 0")
        if self.init_scheme not in INIT_SCHEMES:
            raise ConfigError(f"unknown init_scheme {self.init_scheme!r}")


@dataclass
class FitReport:
    """Per-iteration traces, timings, and flags from one fit (als.py:98-112)."""

    method: str
    objective_trace: np.ndarray
    rmse_trace: np.ndarray
    iters_run: int
    wall_clock_total: float
    sketch_time: float
    solve_time: float
    converged: bool
    skipped_users: int = 0
    skipped_items: int = 0
    diagnostics: list = field(default_factory=list)


def init_factors(R, cfg):
    """Seeded initial factors exactly as the reference draws them (als.py:117-131):
    item rows i.i.d. (uniform on (0, 1/sqrt(n_f)) or normal), user rows zero."""
    rng = np.random.default_rng(cfg.seed)
    scale = 1.0 / np.sqrt(cfg.n_f)
    if cfg.init_scheme == "uniform":
        M = rng.uniform(0.0, scale, size=(R.n_items, cfg.n_f))
    else:
        M = rng.normal(0.0, scale / np.sqrt(cfg.n_f), size=(R.n_items, cfg.n_f))
    U = np.zeros((R.n_users, cfg.n_f))
    return FactorPair(U, M)


def predict(F, i, j):
    """Predicted rating for one (user, item) cell (als.py:134-140)."""
    if not 0 <= i < F.user_factors.shape[0]:
        raise IndexError(f"user index {i} out of range")
    if not 0 <= j < F.item_factors.shape[0]:
        raise IndexError(f"item index {j} out of range")
    return float(F.user_factors[i] @ F.item_factors[j])


def _device_factors(F):
    """FactorPair rows as float64 CUDA tensors (the reference's precision, als.py:40-49)."""
    from . import _lib
    torch = _lib.require_cuda()
    dev = torch.device("cuda")
    U = torch.from_numpy(np.ascontiguousarray(F.user_factors, dtype=np.float64)).to(dev)
    M = torch.from_numpy(np.ascontiguousarray(F.item_factors, dtype=np.float64)).to(dev)
    return torch, dev, U, M


def predict_entries_device(F, users, items):
    """predict_entries with the scores left on the device (float64 CUDA tensor, flat);
    the evaluation metrics rank them there (metrics.py)."""
    from . import _lib
    users = np.asarray(users, dtype=np.int64)
    items = np.asarray(items, dtype=np.int64)
    if users.shape != items.shape:
        raise ValueError("users and items must have the same shape")
    torch, dev, U, M = _device_factors(F)
    if users.size == 0:
        return torch.empty(0, dtype=torch.float64, device=dev)
    if users.min() < 0 or users.max() >= U.shape[0] or items.min() < 0 or items.max() >= M.shape[0]:
        raise IndexError("entry index out of range")
    uu = torch.from_numpy(users.reshape(-1)).to(dev)
    ii = torch.from_numpy(items.reshape(-1)).to(dev)
    out = torch.empty(users.size, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    nf = F.n_f
    _lib.check(_lib.load().cals_predict_entries_f64(U.data_ptr(), M.data_ptr(), nf, nf, nf, uu.data_ptr(),
                                                    ii.data_ptr(), users.size, out.data_ptr(), st),
               "cals_predict_entries_f64")
    return out


def predict_entries(F, users, items, chunk=1 << 18):
    """Predicted ratings for parallel index arrays (als.py:143-152), evaluated on
    the GPU by the float64 gather-dot kernel (cals_predict_entries_f64) on the
    FactorPair's float64 rows, so scores match the reference's einsum up to the
    summation order (rankings in the evaluation metrics depend on them)."""
    users = np.asarray(users, dtype=np.int64)
    if users.size == 0:
        if users.shape != np.asarray(items).shape:
            raise ValueError("users and items must have the same shape")
        return np.empty(0, dtype=np.float64)
    return predict_entries_device(F, users, items).cpu().numpy().reshape(users.shape)


def predict_full(F, block_rows=1 << 16):
    """Dense reconstruction U @ M^T (als.py:155-157) in float64 on the GPU
    (cals_predict_full_f64, a register-tiled kernel), in blocks of user rows so the
    device holds at most block_rows x n_items outputs at a time."""
    from . import _lib
    torch, dev, U, M = _device_factors(F)
    n_u, n_i, nf = U.shape[0], M.shape[0], F.n_f
    out = np.empty((n_u, n_i), dtype=np.float64)
    if n_u == 0 or n_i == 0:
        return out
    st = torch.cuda.current_stream().cuda_stream
    L = _lib.load()
    for r0 in range(0, n_u, block_rows):
        r1 = min(n_u, r0 + block_rows)
        blk = torch.empty((r1 - r0, n_i), dtype=torch.float64, device=dev)
        _lib.check(L.cals_predict_full_f64(U[r0:r1].data_ptr(), M.data_ptr(), r1 - r0, n_i, nf, nf, nf,
                                           blk.data_ptr(), n_i, st), "cals_predict_full_f64")
        out[r0:r1] = blk.cpu().numpy()
    return out
