"""Device-resident sweep engine: the GPU replacement for the reference's
alternating loop (/root/reference/pkg/src/coreals/als.py:243-323) driving the
core sweeper (core.py:173-223).

Ratings live on the device as CSR (users) + CSC (items) with int64 pointers,
int32 indices and fp32 values; factors are fp32 row-major with rows padded to
16 bytes, double-buffered (a half-sweep reads the current buffer and writes
the other one).  One half-sweep is one call into libcoreals_b200.so
(``cals_core_half_sweep``) on the current torch stream.

Objective bookkeeping.  The reference fuses the residual of iteration t into
its second half-sweep (als.py:287-288).  Here it rides on the FIRST
half-sweep of iteration t+1, whose staged slices hold exactly the rows the
residual needs (each rating against the previous iteration's rows), so it
costs no extra memory traffic; the last iteration's residual is one extra
gather pass (``cals_residual``).  obj(t) therefore becomes available one
half-sweep later; thanks to the double buffers the factors of iteration t are
still intact when the host decides to stop there.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import threading

import numpy as np

from . import _lib, hostio
from .errors import ConfigError

__all__ = ["DeviceSide", "CoreEngine", "IterationTerms"]


def _budget(n, rate):
    """sketch_budget (core.py:48-54) for one count."""
    s = int(np.floor(np.float64(n) * np.float64(rate) + 1e-9))
    return max(1, min(s, int(n)))


class DeviceSide:
    """One side of the rating matrix (CSR over users or CSC over items) on the
    device, with its static schedule (budgets, tiers) and workspace."""

    def complete_row(self, row):
        """Whether (global) row's sketch is complete (s_i == n_i: the exact SPD row,
        core.py:206-207)."""
        loc = int(row) - self.row0
        if self.fast:
            return int(self.budget_host[loc]) == int(self.counts[loc])
        return _budget(int(self.counts[loc]), self.rate) == int(self.counts[loc])

    def __init__(self, ptr, idx, val, n_src, n_f, rate, device, row_begin=0, row_end=None, fast=False, ptr_dev=None):
        torch = _lib.require_cuda()
        L = _lib.load()
        if ptr_dev is None and torch.is_tensor(ptr):
            ptr_dev = ptr
        ptr = np.ascontiguousarray(ptr.cpu().numpy() if torch.is_tensor(ptr) else ptr, dtype=np.int64)
        n_all = ptr.size - 1
        if row_end is None:
            row_end = n_all
        row_begin, row_end = int(row_begin), int(row_end)
        # a shard: only rows [row_begin, row_end) and their ratings live on this
        # device -- a rebased pointer block and views of the index / value arrays; the kernels
        # see a side of row_end - row_begin rows, and every per-row output pointer (target
        # rows, thresholds) is offset by row_begin, so results land at the global rows
        self.row0 = row_begin
        if (row_begin, row_end) != (0, n_all):
            base, end = int(ptr[row_begin]), int(ptr[row_end])
            idx = idx[base:end]
            val = val[base:end]
            if ptr_dev is not None:
                ptr_dev = (ptr_dev[row_begin:row_end + 1] - base).contiguous()
            ptr = ptr[row_begin:row_end + 1] - base
            row_begin, row_end = 0, ptr.size - 1
        n_rows = ptr.size - 1
        self.n_rows = n_rows
        self.n_src = int(n_src)
        self.n_f = int(n_f)
        self.rate = float(rate)
        self.device = device
        counts = np.diff(ptr).astype(np.int64)
        if row_end is None:
            row_end = n_rows
        self.row_range = (int(row_begin), int(row_end))
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
        self.fast = bool(fast)
        if self.fast:
            # method 'fast_core': one whole-source sketch per half-sweep; every row a work-item row
            self.fast_s = _budget(self.n_src, rate)
            complete = int(self.fast_s >= self.n_src)
            rc = L.cals_plan_build_fast(sched.ctypes.data, n_rows, self.n_f, complete, budget.ctypes.data,
                                        big.ctypes.data, tile_ptr.ctypes.data, cand_ptr.ctypes.data,
                                        ctypes.byref(meta))
            _lib.check(rc, "cals_plan_build_fast")
        else:
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
            return hostio.upload(a, dt, device)

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
        self.tile_ptr_host = np.ascontiguousarray(tile_ptr[:meta.n_big + 1])
        self.cand_ptr_host = np.ascontiguousarray(cand_ptr[:meta.n_big + 1])
        # work item -> big row (saves each item a binary search over tile_ptr)
        tp = self.tile_ptr_host
        self.tile_row = t(np.repeat(np.arange(meta.n_big, dtype=np.int32), np.diff(tp)) if meta.n_big
                          else np.zeros(1, np.int32), torch.int32)
        meta.big_tile_row = self.tile_row.data_ptr()
        meta.big_tile_ptr_host = self.tile_ptr_host.ctypes.data
        meta.big_cand_ptr_host = self.cand_ptr_host.ctypes.data
        self.plan = meta
        self.side = _lib.cals_side(self.ptr.data_ptr(), self.idx.data_ptr(), self.val.data_ptr(), n_rows, nnz)
        self.ws_bytes = int(L.cals_workspace_bytes(ctypes.byref(meta)))
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=device)
        self.status = torch.zeros(n_rows, dtype=torch.int32, device=device)
        self.rss_rows = torch.zeros(n_rows, dtype=torch.float64, device=device)
        self.pen_rows = torch.zeros(n_rows, dtype=torch.float64, device=device)
        self.summary = torch.zeros(1, dtype=torch.int64, device=device)
        self.nnz = nnz
        if self.fast:
            self.gwords = (self.n_f + 31) // 32
            self.fast_thr = torch.zeros(self.n_f, dtype=torch.int64, device=device)
            self.gmask = torch.zeros(max(self.n_src, 1) * self.gwords, dtype=torch.int32, device=device)
            self.fast_ws = torch.empty(int(L.cals_fast_sketch_workspace_bytes(self.n_f)), dtype=torch.uint8,
                                       device=device)

    def half_sweep(self, source, target, target_old=None, want_rss=False, thr_keys=None, lam=0.0, stream=None):
        torch = _lib.require_cuda()
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        L = _lib.load()
        if self.fast:
            if self.plan.n_big:
                _lib.check(L.cals_fast_sketch(source.data_ptr(), self.n_src, source.stride(0), self.n_f, self.fast_s,
                                              self.fast_thr.data_ptr(), self.gmask.data_ptr(), self.fast_ws.data_ptr(),
                                              self.fast_ws.numel(), stream), "cals_fast_sketch")
            _lib.check(L.cals_fast_half_sweep(
                ctypes.byref(self.side), ctypes.byref(self.plan), source.data_ptr(), source.shape[0], source.stride(0),
                self.n_f, float(lam), self.gmask.data_ptr(), self._rows_ptr(target), target.stride(0),
                self._rows_ptr(target_old) if target_old is not None else None,
                target_old.stride(0) if target_old is not None else 0,
                self.rss_rows.data_ptr() if want_rss else None,
                self.pen_rows.data_ptr(), self.status.data_ptr(), self.summary.data_ptr(), self.ws.data_ptr(),
                self.ws.numel(), stream), "cals_fast_half_sweep")
            self._globalize_summary(stream)
            return
        rc = L.cals_core_half_sweep(
            ctypes.byref(self.side), ctypes.byref(self.plan), source.data_ptr(), source.shape[0],
            source.stride(0), self.n_f, float(lam), self._rows_ptr(target), target.stride(0),
            self._rows_ptr(target_old) if target_old is not None else None,
            target_old.stride(0) if target_old is not None else 0,
            self.rss_rows.data_ptr() if want_rss else None, self.pen_rows.data_ptr(),
            self._rows_ptr(thr_keys) if thr_keys is not None else None,
            self.status.data_ptr(), self.summary.data_ptr(), self.ws.data_ptr(), self.ws.numel(), stream)
        _lib.check(rc, "cals_core_half_sweep")
        self._globalize_summary(stream)

    def index_bytes(self):
        """Device bytes of this side's index (pointers, row ids, ratings)."""
        return int(self.ptr.numel() * 8 + self.idx.numel() * 4 + self.val.numel() * 4)

    def _rows_ptr(self, t):
        """Address of global row row0 of a per-row array (a shard's first row)."""
        return t.data_ptr() + self.row0 * t.stride(0) * t.element_size()

    def _globalize_summary(self, stream):
        """The status word names a shard-local row: make it the global row (word - row0:
        the low half stores 0xFFFFFFFF - row), so ranks' words compare under MAX."""
        if self.row0:
            torch = _lib.require_cuda()
            with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
                self.summary.sub_((self.summary != 0).to(torch.int64) * self.row0)

    def residual(self, source, rows_w, stream=None):
        torch = _lib.require_cuda()
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        # this side's rows (a shard holds only its own), against their global target rows
        _lib.check(_lib.load().cals_residual(ctypes.byref(self.side), source.data_ptr(), source.stride(0), self.n_f,
                                             self._rows_ptr(rows_w), rows_w.stride(0), self.rss_rows.data_ptr(),
                                             stream),
                   "cals_residual")


def decode_summary(word: int):
    """(status, row) from the packed status word; status 0 means all rows ok."""
    word = int(word) & 0xFFFFFFFFFFFFFFFF
    st = word >> 32
    row = 0xFFFFFFFF - (word & 0xFFFFFFFF)
    return st, (row if st else -1)


@dataclass
class IterationTerms:
    """Objective terms of one completed iteration."""

    rss: float
    pen: float  # sum_i n_i |u_i|^2 + sum_j n_j |m_j|^2 (multiply by lam)
    status_first: tuple
    status_second: tuple


class CoreEngine:
    """Device state for one fit: both sides, double-buffered factors, scratch.

    The loop fit_core runs (pipelined, one host read per iteration):
        eng.set_factors(U0, M0)
        for t in range(max_iters):
            eng.step(first)                 # iteration t (+ residual of t-1)
            if t: terms = eng.terms(t - 1)  # host read overlaps iteration t's second half
        eng.finish(first); terms = eng.terms(max_iters - 1)
    """

    def __init__(self, R, n_f, rate, lam, device=None, user_range=None, item_range=None, fast=False):
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
        # each side (plan + uploads) is built on first use, so the second side's
        # host->device copies overlap the first half-sweep already on the GPU
        self._side_args = {
            "user": (R.row_ptr, R.row_items, R.row_vals, self.n_items, n_f, rate, device, *ur, fast),
            "item": (R.col_ptr, R.col_users, R.col_vals, self.n_users, n_f, rate, device, *ir, fast),
        }
        self._sides = {}
        # a host matrix ships its CSR only: the CSC (item side) is built from the
        # device CSR (csrc/index.cu) on a side stream, beside the first half-sweep
        # (a shard holds a CSR row block only, so its CSC block comes from the host index)
        self._csc_on_device = not torch.is_tensor(R.col_ptr) and tuple(ir) == (0, self.n_items) and \
            tuple(ur) == (0, self.n_users)
        self._user_ready = None
        # factor rows padded to a multiple of 4 floats (16-byte gathers); padding stays zero
        self.ld = (self.n_f + 3) // 4 * 4
        self.Ub = [torch.zeros((self.n_users, self.ld), dtype=torch.float32, device=device) for _ in range(2)]
        self.Mb = [torch.zeros((self.n_items, self.ld), dtype=torch.float32, device=device) for _ in range(2)]
        self.cu = self.cm = 0
        self.red_ws = torch.empty(4096, dtype=torch.uint8, device=device)
        # per iteration parity: [rss, pen_user, pen_item, status_first, status_second]
        self.slots = torch.zeros((2, 5), dtype=torch.float64, device=device)
        self.host_slots = torch.zeros((2, 5), dtype=torch.float64).pin_memory()
        self.events = [torch.cuda.Event(), torch.cuda.Event()]
        # sum of squared ratings in float64 (relative RMSE denominator): on the
        # device for device data, else on the host in a background thread
        vals = R.row_vals
        if torch.is_tensor(vals):
            v = vals.to(device=device, dtype=torch.float64)
            self._ssq = float(torch.dot(v, v).item()) if v.numel() else 0.0
            self._ssq_thread = None
        else:
            v = np.asarray(vals, dtype=np.float64)
            self._ssq = None
            self._ssq_box = [0.0]
            self._ssq_thread = threading.Thread(
                target=lambda: self._ssq_box.__setitem__(0, float(np.dot(v, v)) if v.size else 0.0), daemon=True)
            self._ssq_thread.start()
        self.iters_done = 0
        self._s1 = torch.zeros(1, dtype=torch.int64, device=device)
        # CUDA-graph replay of iterations t >= 1 (see step); the sharded engine turns it off
        # (its exchange is a collective between half-sweeps)
        self.use_graphs = True
        self._graphs, self._graph_after, self._graph_failed = {}, {}, set()

    @property
    def ssq(self):
        if self._ssq is None:
            self._ssq_thread.join()
            self._ssq = self._ssq_box[0]
        return self._ssq

    def _side(self, name):
        s = self._sides.get(name)
        if s is None:
            if name == "item" and self._csc_on_device:
                s = self._device_csc_side()
            else:
                s = DeviceSide(*self._side_args[name])
            self._sides[name] = s
            if name == "user":
                torch = _lib.require_cuda()
                self._user_ready = torch.cuda.Event()
                self._user_ready.record(torch.cuda.current_stream(self.device))
        return s

    def _device_csc_side(self):
        """Item side from the device CSR: the transpose waits only for the user
        side's uploads (not for a half-sweep already enqueued behind them)."""
        torch = _lib.require_cuda()
        from .ratings import csr_to_csc_device
        u = self.user
        side_st = torch.cuda.Stream(self.device)
        side_st.wait_event(self._user_ready)
        with torch.cuda.stream(side_st):
            cp, ci, cv = csr_to_csc_device(u.ptr, u.idx, u.val, self.n_users, self.n_items)
        torch.cuda.current_stream(self.device).wait_stream(side_st)
        host_ptr, _, _, *rest = self._side_args["item"]
        return DeviceSide(host_ptr, ci, cv, *rest, ptr_dev=cp)

    @property
    def user(self):
        return self._side("user")

    @property
    def item(self):
        return self._side("item")

    # -- factor buffers ------------------------------------------------------
    @property
    def U(self):
        return self.Ub[self.cu]

    @property
    def M(self):
        return self.Mb[self.cm]

    @property
    def U_view(self):
        return self.U[:, :self.n_f]

    @property
    def M_view(self):
        return self.M[:, :self.n_f]

    def set_factors(self, U=None, M=None):
        """Initial factors into BOTH buffers (rows without ratings never change)."""
        torch = _lib.require_cuda()
        if U is not None:
            u = U.to(self.device, torch.float32) if torch.is_tensor(U) else hostio.upload(np.asarray(U), torch.float32,
                                                                                         self.device)
            for b in self.Ub:
                b[:, :self.n_f].copy_(u)
        if M is not None:
            m = M.to(self.device, torch.float32) if torch.is_tensor(M) else hostio.upload(np.asarray(M), torch.float32,
                                                                                         self.device)
            for b in self.Mb:
                b[:, :self.n_f].copy_(m)
        self.iters_done = 0

    def zero_factors(self, side):
        """Zero rows for one side in both buffers (the reference's user init)."""
        for b in (self.Ub if side == "user" else self.Mb):
            b.zero_()
        self.iters_done = 0

    def _exchange(self, side):  # all-gather of the new rows (sharded engine)
        pass

    def _reduce_scalars(self, parity, cols):  # all-reduce of objective terms (sharded engine)
        pass

    def half(self, side, rss=False, thr_keys=None):
        """One half-sweep into the other buffer; rss: fused residual of the old rows."""
        if side == "user":
            new = self.Ub[1 - self.cu]
            self.user.half_sweep(self.M, new, self.U, rss, thr_keys, self.lam)
            self.cu = 1 - self.cu
        else:
            new = self.Mb[1 - self.cm]
            self.item.half_sweep(self.U, new, self.M, rss, thr_keys, self.lam)
            self.cm = 1 - self.cm
        self._exchange(side)

    def undo_half(self, side):
        """Make the buffer before the last half-sweep of `side` current again (its rows
        are untouched: half-sweeps write the other buffer)."""
        if side == "user":
            self.cu = 1 - self.cu
        else:
            self.cm = 1 - self.cm

    def _sum(self, src, dst_ptr):
        torch = _lib.require_cuda()
        st = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(_lib.load().cals_sum_f64(src.data_ptr(), src.numel(), dst_ptr, self.red_ws.data_ptr(),
                                            self.red_ws.numel(), st), "cals_sum_f64")

    def _publish(self, t):
        self.host_slots[t % 2].copy_(self.slots[t % 2], non_blocking=True)
        self.events[t % 2].record()

    def step(self, first="user"):
        """Enqueue iteration t = iters_done; its first half also yields the
        residual of iteration t-1, which is then published to the host.

        From t = 1 on, an iteration is a fixed sequence of launches on fixed
        buffers that depends only on t's parity (which factor buffer is current,
        which objective slot is written), so with ``use_graphs`` it is captured
        once per parity as a CUDA graph and replayed: one launch per iteration
        instead of a few dozen (the small configs are launch-bound)."""
        t = self.iters_done
        if self.use_graphs and t > 0:
            key = (first, t % 2, self.cu, self.cm)
            g = self._graphs.get(key)
            if g is None and key not in self._graph_failed:
                g = self._capture(first, key)
            if g is not None:
                g.replay()
                self.cu, self.cm = self._graph_after[key]
                self._publish(t - 1)
                self.iters_done = t + 1
                return
        self._step_body(first, t)
        if t > 0:
            self._publish(t - 1)
        self.iters_done = t + 1

    def _step_body(self, first, t):
        """The device work of iteration t (no host reads, no publication)."""
        second = "item" if first == "user" else "user"
        sf = self._side(first)
        self.half(first, rss=t > 0)
        ss = self._side(second)  # built here on the first step: overlaps the first half-sweep
        if t > 0:
            self._sum(sf.rss_rows, self.slots[(t - 1) % 2, 0:1].data_ptr())
            self._reduce_scalars((t - 1) % 2, (0,))
        self._s1.copy_(sf.summary)
        self.half(second, rss=False)
        cur = self.slots[t % 2]
        self._sum(self.user.pen_rows, cur[1:2].data_ptr())
        self._sum(self.item.pen_rows, cur[2:3].data_ptr())
        cur[3:4].copy_(self._s1.view(_lib.require_cuda().float64))
        cur[4:5].copy_(ss.summary.view(_lib.require_cuda().float64))
        self._reduce_scalars(t % 2, (1, 2, 3, 4))

    def _capture(self, first, key):
        """Capture iteration t's device work (t >= 1, parity key[1]) as a CUDA graph.
        The capture runs nothing; the factor-buffer flips it implies are recorded and
        undone so replay() applies them.  A capture failure (e.g. a kernel profile
        scope recording events) leaves this parity on the eager path."""
        torch = _lib.require_cuda()
        if _lib.profile_enabled():
            return None
        cu, cm, done = self.cu, self.cm, self.iters_done
        g = torch.cuda.CUDAGraph()
        try:
            torch.cuda.synchronize(self.device)
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                self._step_body(first, done)
        except RuntimeError:
            self._graph_failed.add(key)
            self.cu, self.cm = cu, cm
            torch.cuda.synchronize(self.device)
            return None
        self._graph_after[key] = (self.cu, self.cm)
        self.cu, self.cm = cu, cm
        self._graphs[key] = g
        return g

    def finish(self, first="user"):
        """Residual of the last iteration: one gather pass over the first side."""
        t = self.iters_done - 1
        if t < 0:
            return
        sf = self.user if first == "user" else self.item
        src, rows = (self.M, self.U) if first == "user" else (self.U, self.M)
        sf.residual(src, rows)
        self._sum(sf.rss_rows, self.slots[t % 2, 0:1].data_ptr())
        self._reduce_scalars(t % 2, (0,))
        self._publish(t)

    def terms(self, t):
        """Host copy of iteration t's objective terms (waits until published)."""
        self.events[t % 2].synchronize()
        h = self.host_slots[t % 2].numpy().copy()
        w = h[3:5].view(np.int64)
        return IterationTerms(float(h[0]), float(h[1] + h[2]), decode_summary(int(w[0])), decode_summary(int(w[1])))

    def iterate(self, first="user"):
        """One iteration together with its own residual (synchronous form used
        by tests and the benchmark's per-step timing)."""
        self.step(first)
        self.finish(first)
        return self.terms(self.iters_done - 1)

    def rewind(self):
        """Make the previous buffers current again (drop the last step's rows)."""
        self.cu, self.cm = 1 - self.cu, 1 - self.cm
        self.iters_done -= 1

    def factors_host(self):
        # widen on the device: the float64 copy-out is cheaper than a host conversion
        return hostio.download_f64(self.U_view), hostio.download_f64(self.M_view)
