"""Core-elements subsampling for ALS on B200: the drop-in for the reference's
``coreals.core`` hot path (/root/reference/pkg/src/coreals/core.py).

Public entry points keep the reference's names, arguments, return types and
error behaviour:

  sketch_budget(n, rate)                       core.py:48-54
  SparseSketch                                 core.py:57-92
  ces_sketch(X, rate)                          core.py:95-115   (GPU selection kernel)
  update_user_core / update_item_core          core.py:134-162  (GPU solve, float64)
  fit_core(R, cfg, init_u, init_m, items_first) core.py:301-312 (GPU half-sweeps)

Numerics: ratings and factors are fp32 on the device (the reference is
float64); selections are bit-exact with the reference on the same fp32
inputs, per-row solutions agree to ~1e-6 relative, and the returned
FactorPair is float64 like the reference's.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .als import FactorPair, FitReport, SolverConfig, init_factors
from .errors import ConfigError, DataError, NumericalError

__all__ = [
    "SparseSketch", "ces_sketch", "sketch_budget",
    "update_user_core", "update_item_core", "fit_core",
]


def sketch_budget(n, rate):
    """Retained entries per column: max(1, floor(n * rate + 1e-9)), capped at n (core.py:48-54)."""
    return min(int(n), max(1, int(np.floor(n * rate + 1e-9))))


@dataclass(frozen=True)
class SparseSketch:
    """Per-column retained entries of a dense slice, column-compressed (core.py:57-92)."""

    n_rows: int
    n_cols: int
    col_ptr: np.ndarray
    rows: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self):
        return int(self.rows.size)

    @property
    def kept_per_column(self):
        return np.diff(self.col_ptr)

    @property
    def complete(self):
        return self.nnz == self.n_rows * self.n_cols

    def column(self, c):
        lo, hi = self.col_ptr[c], self.col_ptr[c + 1]
        return self.rows[lo:hi], self.vals[lo:hi]

    def to_dense(self):
        out = np.zeros((self.n_rows, self.n_cols))
        cols = np.repeat(np.arange(self.n_cols), self.kept_per_column)
        out[self.rows, cols] = self.vals
        return out


_F64_RANK_MAX_N = 8192  # exact-rank float64 kernel up to this slice height (O(n^2) per column)


def ces_sketch(X, rate):
    """Top-|value| sketch of each column (core.py:95-115), selected on the GPU.

    Per column keep s = max(1, floor(n*rate)) entries of largest |x|, ties to
    the smallest row; rows are emitted strictly-above-threshold first, then
    tied, each in row order, exactly as the reference emits them.  Selection
    runs on the float64 values (exact ranks) unless the slice is tall and
    fp32-representable, where the fp32 sample-select kernel of the fit is used
    (same order: fp32 -> fp64 is exact and monotone).
    """
    X64 = np.ascontiguousarray(X, dtype=np.float64)
    if X64.ndim != 2 or X64.shape[0] < 1:
        raise DataError("ces_sketch expects a non-empty 2-d slice")
    if not 0.0 < rate <= 1.0:
        raise ConfigError(f"rate must be in (0, 1], got {rate}")
    torch = _lib.require_cuda()
    n, p = X64.shape
    s = sketch_budget(n, rate)
    dev = torch.device("cuda")
    L = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    rows = torch.empty(p * s, dtype=torch.int32, device=dev)
    X32 = X64.astype(np.float32)
    if n <= _F64_RANK_MAX_N or not np.array_equal(X32.astype(np.float64), X64):
        Xd = torch.from_numpy(X64).to(dev)
        ws = torch.empty(max(n * p, 256), dtype=torch.uint8, device=dev)
        _lib.check(L.cals_ces_sketch_f64(Xd.data_ptr(), n, p, s, rows.data_ptr(), ws.data_ptr(), ws.numel(), st),
                   "cals_ces_sketch_f64")
    else:
        Xd = torch.from_numpy(X32).to(dev)
        vals = torch.empty(p * s, dtype=torch.float32, device=dev)
        wsb = int(L.cals_ces_sketch_workspace_bytes(n, p))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        _lib.check(L.cals_ces_sketch(Xd.data_ptr(), n, p, s, rows.data_ptr(), vals.data_ptr(), ws.data_ptr(), wsb,
                                     st), "cals_ces_sketch")
    rows_h = rows.cpu().numpy()
    cols = np.repeat(np.arange(p), s)
    return SparseSketch(n_rows=n, n_cols=p, col_ptr=np.arange(p + 1, dtype=np.int64) * s,
                        rows=rows_h, vals=X64[rows_h, cols])


def update_user_core(M_slice, sketch, y, lam, n_count, context=""):
    """Sketched ridge update for one row (core.py:134-157), solved on the GPU in
    float64: (X*^T X + lam*n I) u = X*^T y; a complete sketch takes the SPD path."""
    X = np.ascontiguousarray(M_slice, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    if X.ndim != 2 or sketch.n_rows != X.shape[0] or sketch.n_cols != X.shape[1]:
        raise DataError("sketch shape does not match the slice")
    if y.size != X.shape[0]:
        raise DataError("response length does not match the slice height")
    torch = _lib.require_cuda()
    n, p = X.shape
    if p > _lib.CALS_MAX_NF:
        raise ConfigError(f"slice width {p} exceeds the supported maximum {_lib.CALS_MAX_NF}")
    dev = torch.device("cuda")
    Xd = torch.from_numpy(X).to(dev)
    yd = torch.from_numpy(y).to(dev)
    cp = torch.from_numpy(np.ascontiguousarray(sketch.col_ptr, dtype=np.int64)).to(dev)
    rw = torch.from_numpy(np.ascontiguousarray(sketch.rows, dtype=np.int32) if sketch.nnz else np.zeros(1, np.int32)).to(dev)
    w = torch.empty(p, dtype=torch.float64, device=dev)
    stt = torch.empty(1, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.load().cals_update_core(Xd.data_ptr(), n, p, cp.data_ptr(), rw.data_ptr(), yd.data_ptr(),
                                            float(lam) * float(n_count), int(sketch.complete), w.data_ptr(),
                                            stt.data_ptr(), st), "cals_update_core")
    if int(stt.item()) == _lib.CALS_ROW_SINGULAR:
        if sketch.complete:
            raise NumericalError(f"singular Gram matrix after jitter retry {context}")
        raise NumericalError(f"singular sketched system after jitter retry {context}")
    return w.cpu().numpy()


def update_item_core(U_slice, sketch, y, lam, n_count, context=""):
    """Sketched ridge update for one item row (same math as the user side, core.py:160-162)."""
    return update_user_core(U_slice, sketch, y, lam, n_count, context)


def _host(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def _raise_for(status, side, engine_side, it):
    st, row = status
    if st != _lib.CALS_ROW_SINGULAR:
        return
    full = engine_side.complete_row(row)
    if full:  # exact SPD row (core.py:206-207 -> als.py:197, no context passed)
        raise NumericalError("singular Gram matrix after jitter retry ")
    raise NumericalError(f"singular sketched system after jitter retry ({side} {row}, iteration {it})")


def fit_core(R, cfg, *, init_u=None, init_m=None, items_first=False, engine=None):
    """Alternating fit with one element sketch per regression slice (core.py:301-312),
    every half-sweep running on the GPU.

    Same semantics as the reference: seeded init (or init_u / init_m
    overrides), rows without ratings skipped and warned, fused residual in the
    second half-sweep, objective rss + lam*(sum n_i |u_i|^2 + sum n_j |m_j|^2),
    relative RMSE sqrt(rss/ssq), convergence on |d obj|/obj_prev < tol.
    ``cfg.diagnostics`` (the reference's slow instrumented CPU path) is not
    offered: it is warned about and ignored, as fit_fast_core does (core.py:319-322).
    """
    if cfg.method != "core":
        raise ConfigError(f"fit_core handles method 'core', got {cfg.method!r}")
    if cfg.diagnostics:
        warnings.warn("per-regression diagnostics are not available on the GPU path; ignoring the flag",
                      stacklevel=2)
        cfg = replace(cfg, diagnostics=False)
    return _fit_gpu(R, cfg, cfg.rate, init_u, init_m, items_first, engine)


def fit(R, cfg, *, init_u=None, init_m=None, items_first=False, engine=None):
    """Exact full-sample ALS (method 'full', als.py:326-336) on the GPU.

    Every regression is the exact ridge X^T X + lam*n_i*I (als.py:200-205) --
    the same kernels with a complete budget (s_i = n_i: no selection, identity
    kept-row lists, the SPD elimination with the reference's Cholesky failure
    point and jitter retry, als.py:184-197).  Reference semantics otherwise as
    fit_core; the report's sketch_time is 0 as in _FullSweeper.
    """
    if cfg.method != "full":
        raise ConfigError(f"als.fit handles method 'full', got {cfg.method!r}")
    return _fit_gpu(R, cfg, 1.0, init_u, init_m, items_first, engine)


def fit_fast_core(R, cfg, *, init_u=None, init_m=None, items_first=False, engine=None):
    """Alternating fit sketching each whole factor matrix once per half-iteration
    (method 'fast_core', core.py:314-324) on the GPU: per half-sweep one
    whole-source element sketch (ces_sketch of the full source, core.py:276-286),
    then every regression's Gram sums the slice rows that sketch kept for each
    column, an empty column falling back to the slice's first largest-|x| row
    (gram_rhs_rowsketch, _kernels.py:172-216), solved by LU (or the exact SPD
    row when the sketch is complete).  ``cfg.diagnostics`` is warned about and
    ignored, as the reference does (core.py:319-322).
    """
    if cfg.method != "fast_core":
        raise ConfigError(f"fit_fast_core handles method 'fast_core', got {cfg.method!r}")
    if cfg.diagnostics:
        warnings.warn("per-regression diagnostics are only instrumented for method 'core'; ignoring the flag",
                      stacklevel=2)
        cfg = replace(cfg, diagnostics=False)
    if engine is None:
        from .engine import CoreEngine
        engine = CoreEngine(R, cfg.n_f, cfg.rate, cfg.lam, fast=True)
    return _fit_gpu(R, cfg, cfg.rate, init_u, init_m, items_first, engine)


def _fit_gpu(R, cfg, rate, init_u, init_m, items_first, engine):
    start = time.perf_counter()
    torch = _lib.require_cuda()
    from .engine import CoreEngine

    # init_factors draws only the item rows (user rows start at zero, als.py:117-131),
    # so an explicit init_m needs no draw at all, and zero user rows need no upload
    M0 = (init_factors(R, cfg).item_factors if init_m is None
          else np.ascontiguousarray(init_m, dtype=np.float64))
    U0 = None if init_u is None else np.ascontiguousarray(init_u, dtype=np.float64)
    if (U0 is not None and U0.shape != (R.n_users, cfg.n_f)) or M0.shape != (R.n_items, cfg.n_f):
        raise ConfigError("initial factor shapes do not match the rating matrix")

    row_counts = np.diff(_host(R.row_ptr))
    col_counts = np.diff(_host(R.col_ptr))
    skipped_u = int(np.count_nonzero(row_counts == 0))
    skipped_m = int(np.count_nonzero(col_counts == 0))
    if skipped_u or skipped_m:
        warnings.warn(
            f"{skipped_u} user(s) and {skipped_m} item(s) have no training ratings; "
            "their factor rows are left at initialization", stacklevel=2)
    active_u = row_counts > 0
    if active_u.any() and cfg.n_f > int(row_counts[active_u].min()):
        warnings.warn(
            f"n_f={cfg.n_f} exceeds the smallest user rating count; "
            "the penalty term is doing the disambiguation", stacklevel=2)

    eng = engine if engine is not None else CoreEngine(R, cfg.n_f, rate, cfg.lam)
    eng.set_factors(U0, M0)
    if U0 is None:
        eng.zero_factors("user")
    ssq = eng.ssq
    obj_trace, rmse_trace = [], []
    converged = False
    first = "item" if items_first else "user"
    second = "user" if items_first else "item"
    sides = eng._side  # side objects by name (built lazily by the engine)
    prev = [None]

    def consume(t):
        """obj/rmse of iteration t (als.py:299-307); True when converged there."""
        terms = eng.terms(t)
        _raise_for(terms.status_first, first, sides(first), t)
        _raise_for(terms.status_second, second, sides(second), t)
        obj = terms.rss + (cfg.lam * terms.pen if cfg.lam != 0.0 else 0.0)
        obj_trace.append(obj)
        rmse_trace.append(np.sqrt(terms.rss / ssq) if ssq > 0 else 0.0)
        done = False
        if prev[0] is not None:
            rel = abs(obj - prev[0]) / max(prev[0], np.finfo(np.float64).tiny)
            done = rel < cfg.tol
        prev[0] = obj
        return done

    # selection time (core.py:193-195,208-219): event time of the standalone selection
    # kernels, collected through the native per-kernel timer unless the caller runs it.
    # Iterations 0 and 1 run eagerly under the timer; from iteration 2 on the engine
    # replays CUDA graphs (no per-kernel events inside a graph), each counted at
    # iteration 1's selection time (the same launches on data of the same shape).
    own_timer = not _lib.profile_enabled()
    sel_ms = [0.0, 0.0]  # iteration 0, iteration 1
    graph_iters = 0

    def selection_ms():
        return sum(ms for k, (_, ms) in _lib.profile_collect().items() if k in _lib.SELECTION_KERNELS)

    if own_timer:
        _lib.profile_enable(True)
        _lib.profile_collect()
    t0 = time.perf_counter()
    try:
        for it in range(cfg.max_iters):
            if own_timer and it == 1:
                torch.cuda.current_stream().synchronize()
                sel_ms[0] = selection_ms()
            eng.step(first)  # iteration it; its first half also yields the residual of it-1
            if own_timer and it == 1:
                torch.cuda.current_stream().synchronize()
                sel_ms[1] = selection_ms()
                _lib.profile_enable(False)
            if own_timer and it >= 2:
                graph_iters += 1
            if it >= 1 and consume(it - 1):
                converged = True
                eng.rewind()  # the factors of iteration it-1 are the result
                break
        if not converged and eng.iters_done > 0:
            eng.finish(first)
            converged = consume(eng.iters_done - 1)
        torch.cuda.current_stream().synchronize()
    except BaseException:
        if own_timer:  # (a NumericalError mid-fit must not leave the timer running)
            _lib.profile_enable(False)
            _lib.profile_collect()
        raise
    t_loop = time.perf_counter() - t0
    sketch_s = 0.0
    if own_timer:
        if _lib.profile_enabled():  # stopped before iteration 1 ended: the timer is still on
            sel_ms[0] += selection_ms()
            _lib.profile_enable(False)
        _lib.profile_collect()
        sketch_s = (sel_ms[0] + sel_ms[1] * (1 + graph_iters)) / 1e3
    iters = eng.iters_done
    U, M = eng.factors_host()
    report = FitReport(
        method=cfg.method,
        objective_trace=np.asarray(obj_trace),
        rmse_trace=np.asarray(rmse_trace),
        iters_run=iters,
        wall_clock_total=time.perf_counter() - start,
        sketch_time=sketch_s,
        solve_time=max(t_loop - sketch_s, 0.0),  # iteration wall - sketch time (als.py:294-298)
        converged=converged,
        skipped_users=skipped_u,
        skipped_items=skipped_m,
        diagnostics=[],
    )
    return FactorPair(U, M), report
