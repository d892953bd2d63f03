"""Device-resident sweep engine: the GPU replacement for the reference's
alternating loop (/root/reference/pkg/src/coreals/als.py:243-323) driving the
core sweeper (core.py:173-223).

Ratings live on the device as CSR (users) + CSC (items) with int64 pointers,
int32 indices and fp32 values; factors are fp32 row-major.  One half-sweep is
one call into libcoreals_b200.so (``cals_core_half_sweep``), enqueued on the
current torch stream.  The host only reads back, once per iteration, the
objective terms and a status word.
"""

from __future__ import annotations

import ctypes
import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigError, NumericalError

__all__ = ["DeviceSide", "CoreEngine"]


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class DeviceSide:
    """One side of the rating matrix (CSR over users or CSC over items) on the
    device, with its static schedule (budgets, tiers) and workspace."""

    def __init__(self, ptr, idx, val, n_src, n_f, rate, device, row_begin=0, row_end=None):
        torch = _lib.require_cuda()
        L = _lib.load()
        ptr_dev = ptr if torch.is_tensor(ptr) else None
        ptr = np.ascontiguousarray(ptr.cpu().numpy() if torch.is_tensor(ptr) else ptr, dtype=np.int64)
        n_rows = ptr.size - 1
        self.n_rows = n_rows
        self.n_src = int(n_src)
        self.n_f = int(n_f)
        self.device = device
        counts = np.diff(ptr).astype(np.int64)
        if row_end is None:
            row_end = n_rows
        # rows outside [row_begin, row_end) are another rank's shard: no work here
        sched = counts.copy()
        sched[:row_begin] = 0
        sched[row_end:] = 0
        self.counts = counts
        budget = np.empty(n_rows, np.int32)
        small = np.empty(n_rows, np.int32)
        big = np.empty(n_rows, np.int32)
        tile_ptr = np.zeros(n_rows + 1, np.int64)
        cand_ptr = np.zeros(n_rows + 1, np.int64)
        meta = _lib.cals_plan()
        rc = L.cals_plan_build(sched.ctypes.data, n_rows, self.n_f, float(rate), budget.ctypes.data,
                               small.ctypes.data, big.ctypes.data, tile_ptr.ctypes.data, cand_ptr.ctypes.data,
                               ctypes.byref(meta))
        _lib.check(rc, "cals_plan_build")
        self.budget_host = budget
        self.small_host = small[:meta.n_small].copy()
        self.big_host = big[:meta.n_big].copy()
        nnz = int(ptr[-1])
        def t(a, dt):
            if torch.is_tensor(a):
                return a.to(device=device, dtype=dt).contiguous()
            return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)

        self.ptr = t(ptr_dev if ptr_dev is not None else ptr, torch.int64)
        self.idx = t(idx, torch.int32)
        self.val = t(val, torch.float32)
        self.budget = t(budget, torch.int32)
        self.small = t(self.small_host if meta.n_small else np.zeros(1, np.int32), torch.int32)
        self.big = t(self.big_host if meta.n_big else np.zeros(1, np.int32), torch.int32)
        self.tile_ptr = t(tile_ptr[:meta.n_big + 1], torch.int64)
        self.cand_ptr = t(cand_ptr[:meta.n_big + 1], torch.int64)
        meta.budget = self.budget.data_ptr()
        meta.small_rows = self.small.data_ptr()
        meta.big_rows = self.big.data_ptr()
        meta.big_tile_ptr = self.tile_ptr.data_ptr()
        meta.big_cand_ptr = self.cand_ptr.data_ptr()
        self.plan = meta
        self.side = _lib.cals_side(self.ptr.data_ptr(), self.idx.data_ptr(), self.val.data_ptr(), n_rows, nnz)
        self.ws_bytes = int(L.cals_workspace_bytes(ctypes.byref(meta)))
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=device)
        self.status = torch.zeros(n_rows, dtype=torch.int32, device=device)
        self.rss_rows = torch.zeros(n_rows, dtype=torch.float64, device=device)
        self.summary = torch.zeros(1, dtype=torch.int64, device=device)
        self.nnz = nnz

    def half_sweep(self, source, target, lam, want_rss, thr_keys=None, stream=None):
        torch = _lib.require_cuda()
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        L = _lib.load()
        rc = L.cals_core_half_sweep(
            ctypes.byref(self.side), ctypes.byref(self.plan), source.data_ptr(), source.shape[0],
            source.stride(0), self.n_f, float(lam), target.data_ptr(), target.stride(0),
            self.rss_rows.data_ptr() if want_rss else None,
            thr_keys.data_ptr() if thr_keys is not None else None,
            self.status.data_ptr(), self.summary.data_ptr(), self.ws.data_ptr(), self.ws.numel(), stream)
        _lib.check(rc, "cals_core_half_sweep")


def decode_summary(word: int):
    """(status, row) from the packed status word; status 0 means all rows ok."""
    word = int(word) & 0xFFFFFFFFFFFFFFFF
    st = word >> 32
    row = 0xFFFFFFFF - (word & 0xFFFFFFFF)
    return st, (row if st else -1)


@dataclass
class IterationTerms:
    rss: float
    pen_u: float
    pen_m: float
    status_first: tuple
    status_second: tuple


class CoreEngine:
    """Device state for one fit: both sides, both factor matrices, scratch."""

    def __init__(self, R, n_f, rate, lam, device=None, user_range=None, item_range=None):
        torch = _lib.require_cuda()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        self.n_f, self.rate, self.lam = int(n_f), float(rate), float(lam)
        if self.n_f > _lib.CALS_MAX_NF:
            raise ConfigError(f"n_f={n_f} exceeds the supported maximum {_lib.CALS_MAX_NF}")
        self.n_users, self.n_items = int(R.n_users), int(R.n_items)
        ur = user_range or (0, self.n_users)
        ir = item_range or (0, self.n_items)
        self.user = DeviceSide(R.row_ptr, R.row_items, R.row_vals, self.n_items, n_f, rate, device, *ur)
        self.item = DeviceSide(R.col_ptr, R.col_users, R.col_vals, self.n_users, n_f, rate, device, *ir)
        self.U = torch.zeros((self.n_users, self.n_f), dtype=torch.float32, device=device)
        self.M = torch.zeros((self.n_items, self.n_f), dtype=torch.float32, device=device)
        self.red_ws = torch.empty(4096, dtype=torch.uint8, device=device)
        self.scalars = torch.zeros(3, dtype=torch.float64, device=device)
        vals = R.row_vals if torch.is_tensor(R.row_vals) else torch.from_numpy(np.asarray(R.row_vals))
        vals = vals.to(device=device, dtype=torch.float64)
        self.ssq = float(torch.dot(vals, vals).item()) if vals.numel() else 0.0

    def set_factors(self, U=None, M=None):
        torch = _lib.require_cuda()
        if U is not None:
            self.U.copy_(torch.as_tensor(np.asarray(U, dtype=np.float32)).to(self.device))
        if M is not None:
            self.M.copy_(torch.as_tensor(np.asarray(M, dtype=np.float32)).to(self.device))

    def half(self, side, want_rss=False, thr_keys=None):
        if side == "user":
            self.user.half_sweep(self.M, self.U, self.lam, want_rss, thr_keys)
        else:
            self.item.half_sweep(self.U, self.M, self.lam, want_rss, thr_keys)

    def objective_terms(self, rss_side, stream=None):
        """Enqueue rss (sum of the fused residual rows) and both penalty sums."""
        torch = _lib.require_cuda()
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        L = _lib.load()
        ws, nb = self.red_ws.data_ptr(), self.red_ws.numel()
        s = self.user if rss_side == "user" else self.item
        _lib.check(L.cals_sum_f64(s.rss_rows.data_ptr(), s.n_rows, self.scalars.data_ptr(), ws, nb, stream),
                   "cals_sum_f64")
        _lib.check(L.cals_weighted_sqnorm(self.U.data_ptr(), self.n_users, self.n_f, self.U.stride(0),
                                          self.user.ptr.data_ptr(), self.scalars.data_ptr() + 8, ws, nb, stream),
                   "cals_weighted_sqnorm")
        _lib.check(L.cals_weighted_sqnorm(self.M.data_ptr(), self.n_items, self.n_f, self.M.stride(0),
                                          self.item.ptr.data_ptr(), self.scalars.data_ptr() + 16, ws, nb, stream),
                   "cals_weighted_sqnorm")

    def iterate(self, first="user"):
        """One ALS iteration (both half-sweeps + fused RSS) -> IterationTerms.
        The only device->host traffic: 3 doubles and 2 status words."""
        torch = _lib.require_cuda()
        second = "item" if first == "user" else "user"
        self.half(first, want_rss=False)
        s1 = (self.user if first == "user" else self.item).summary.clone()
        self.half(second, want_rss=True)
        s2 = (self.user if second == "user" else self.item).summary
        self.objective_terms(second)
        host = torch.cat([self.scalars, s1.view(torch.float64), s2.view(torch.float64)]).cpu()
        rss, pu, pm = (float(x) for x in host[:3])
        w1 = int(host[3:4].view(torch.int64).item())
        w2 = int(host[4:5].view(torch.int64).item())
        return IterationTerms(rss, pu, pm, decode_summary(w1), decode_summary(w2))

    def factors_host(self):
        return self.U.double().cpu().numpy(), self.M.double().cpu().numpy()
