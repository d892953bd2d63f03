"""Row sharding across GPUs of one node.

Rows of a half-sweep are independent given a read-only source snapshot
(SPEC.md:178,282), so each rank solves a contiguous, nnz-balanced block of
rows of each side against its full replica of the source factors, then the
updated blocks are all-gathered (one collective per half-sweep) so every rank
again holds the full target matrix.  The fused residual is a scalar
all-reduce.  Ratings never move: a rank only needs its CSR row block and CSC
column block (it keeps the whole index here for simplicity of the planner).

The exchange helpers are backend-agnostic (NCCL on GPUs, gloo on CPU for the
host-logic tests).
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
    """All-gather-v of row blocks: after the call every rank's F holds every
    rank's rows F[r0:r1].  Blocks are padded to the largest one so a single
    all_gather_into_tensor moves everything."""
    world = len(ranges)
    if world == 1:
        return F
    maxr = max(r1 - r0 for r0, r1 in ranges)
    nf = F.shape[1]
    if scratch is None or scratch.numel() < (world + 1) * maxr * nf:
        scratch = torch.empty((world + 1) * maxr * nf, dtype=F.dtype, device=F.device)
    send = scratch[:maxr * nf].view(maxr, nf)
    recv = scratch[maxr * nf:(world + 1) * maxr * nf].view(world, maxr, nf)
    r0, r1 = ranges[rank]
    send[:r1 - r0].copy_(F[r0:r1])
    dist.all_gather_into_tensor(recv.view(-1), send.view(-1), group=group)
    for q, (q0, q1) in enumerate(ranges):
        if q != rank and q1 > q0:
            F[q0:q1].copy_(recv[q, :q1 - q0])
    return scratch


class ShardedEngine:
    """CoreEngine restricted to this rank's row blocks + the per-half-sweep
    exchange.  Same iterate() contract as CoreEngine."""

    def __init__(self, R, n_f, rate, lam, rank, world, group=None, device=None):
        from .engine import CoreEngine

        self.rank, self.world, self.group = rank, world, group
        self.user_ranges = nnz_balanced_ranges(R.row_ptr, world)
        self.item_ranges = nnz_balanced_ranges(R.col_ptr, world)
        self.eng = CoreEngine(R, n_f, rate, lam, device=device, user_range=self.user_ranges[rank],
                              item_range=self.item_ranges[rank])
        self._scratch = None

    def __getattr__(self, name):
        return getattr(self.eng, name)

    def _exchange(self, side):
        if side == "user":
            self._scratch = allgather_rows(self.eng.U, self.user_ranges, self.rank, self.group, self._scratch)
        else:
            self._scratch = allgather_rows(self.eng.M, self.item_ranges, self.rank, self.group, self._scratch)

    def iterate(self, first="user"):
        from .engine import IterationTerms, decode_summary

        e = self.eng
        second = "item" if first == "user" else "user"
        e.half(first, want_rss=False)
        self._exchange(first)
        s1 = (e.user if first == "user" else e.item).summary.clone()
        e.half(second, want_rss=True)
        self._exchange(second)
        s2 = (e.user if second == "user" else e.item).summary
        e.objective_terms(second)
        rss = e.scalars[:1].clone()
        dist.all_reduce(rss, op=dist.ReduceOp.SUM, group=self.group)
        words = torch.stack([s1[0], s2[0]])
        dist.all_reduce(words, op=dist.ReduceOp.MAX, group=self.group)
        host = torch.cat([rss, e.scalars[1:3], words.view(torch.float64)]).cpu()
        w = host[3:5].view(torch.int64)
        return IterationTerms(float(host[0]), float(host[1]), float(host[2]),
                              decode_summary(int(w[0])), decode_summary(int(w[1])))
