"""Row sharding across GPUs of one node.

Rows of a half-sweep are independent given a read-only source snapshot
(SPEC.md:178,282), so each rank solves a contiguous, nnz-balanced block of
rows of each side against its full replica of the source factors, then the
updated blocks are all-gathered (one collective per half-sweep) so every rank
again holds the full target matrix.  The fused residual is a scalar
all-reduce.  Ratings never move: a rank only holds its CSR row block and CSC
column block.

The exchange helpers are backend-agnostic (NCCL on GPUs, gloo on CPU for the
host-logic tests).  Each rank's DeviceSide holds only its CSR row block and CSC
column block (rebased pointers, views of the rating arrays), plus full fp32
replicas of both factor matrices (the gathers touch arbitrary source rows).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["nnz_balanced_ranges", "allgather_rows", "ShardedEngine"]


def nnz_balanced_ranges(ptr, world):
    """Contiguous row ranges [(r0, r1)] per rank with ~equal nnz (+1 per row,
    so empty-heavy tails still spread)."""
    ptr = np.asarray(ptr.cpu().numpy() if torch.is_tensor(ptr) else ptr, dtype=np.int64)
    n = ptr.size - 1
    work = ptr + np.arange(n + 1, dtype=np.int64)  # nnz + row count prefix
    total = work[-1]
    cuts = [0]
    for q in range(1, world):
        cuts.append(int(np.searchsorted(work, q * total / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[q]), int(cuts[q + 1])) for q in range(world)]


def allgather_rows(F, ranges, rank, group=None, scratch=None):
    """All-gather-v of row blocks: after the call every rank's F holds every rank's
    rows F[r0:r1].

    Every block is broadcast by its owner straight into the block's own rows of F
    on every rank (rows are contiguous in the row-major factor matrix), so no rank
    stages a send buffer or scatters a receive buffer; NCCL runs the broadcasts
    back to back on its stream over NVLink.  CUDA tensors under a host backend
    (gloo: several ranks on one device, functional tests only) go through one
    host copy."""
    world = len(ranges)
    if world == 1:
        return F
    backend = dist.get_backend(group)
    if F.is_cuda and backend != "nccl":
        host = F.cpu()
        _broadcast_blocks(host, ranges, group)
        F.copy_(host)
        return scratch
    _broadcast_blocks(F, ranges, group)
    return scratch


def _broadcast_blocks(F, ranges, group):
    works = []
    for q, (q0, q1) in enumerate(ranges):
        if q1 > q0:
            src = q if group is None else dist.get_global_rank(group, q)
            works.append(dist.broadcast(F[q0:q1], src=src, group=group, async_op=True))
    for w in works:
        w.wait()


class ShardedEngine:
    """Factory returning a CoreEngine restricted to this rank's row blocks,
    with the per-half-sweep exchange and the objective all-reduce hooked in."""

    def __new__(cls, R, n_f, rate, lam, rank, world, group=None, device=None, fast=False):
        from .engine import CoreEngine

        user_ranges = nnz_balanced_ranges(R.row_ptr, world)
        item_ranges = nnz_balanced_ranges(R.col_ptr, world)

        class _Sharded(CoreEngine):
            def _exchange(self, side):
                if side == "user":
                    self._scratch = allgather_rows(self.U, user_ranges, rank, group, self._scratch)
                else:
                    self._scratch = allgather_rows(self.M, item_ranges, rank, group, self._scratch)

            def _reduce_scalars(self, parity, cols):
                row = self.slots[parity]
                sums = [c for c in cols if c <= 2]
                maxes = [c for c in cols if c >= 3]
                host = dist.get_backend(group) != "nccl"  # gloo: reduce host copies
                if sums:
                    t = row[sums[0]:sums[-1] + 1].clone()
                    t = t.cpu() if host else t
                    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
                    row[sums[0]:sums[-1] + 1].copy_(t)
                if maxes:
                    t = row[maxes[0]:maxes[-1] + 1].view(torch.int64).clone()
                    t = t.cpu() if host else t
                    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
                    row[maxes[0]:maxes[-1] + 1].copy_(t.view(torch.float64).to(row.device))

        eng = _Sharded(R, n_f, rate, lam, device=device, user_range=user_ranges[rank], item_range=item_ranges[rank],
                       fast=fast)
        eng._scratch = None
        eng.use_graphs = False  # the exchange between half-sweeps is a collective: eager launches
        eng.rank, eng.world, eng.group = rank, world, group
        eng.user_ranges, eng.item_ranges = user_ranges, item_ranges
        return eng
