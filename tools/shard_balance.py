"""Per-rank cost of the row-sharded half-sweeps, measured on ONE GPU (tool).

For N ranks, each rank's engine (CoreEngine restricted to that rank's user and
item row blocks -- exactly what ShardedEngine builds) runs iterations alone
on the device; the sharded iteration time is the max over ranks plus the
all-gathers.  This projects strong scaling without N GPUs (no rank waits on
another, so nothing here depends on concurrent kernels).

usage: python tools/shard_balance.py [CONFIG] [N ...]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import shard, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = args[0] if args else "large"
Ns = [int(a) for a in args[1:]] or [2, 4, 8]
spec = synth.CONFIGS[cfg]
n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
d = synth.generate(cfg, device="cuda")
M0 = synth.init_m(d.n_items, n_f)


REF = None  # (U, M) after two full iterations: every rank sees the all-gathered factors


def time_iter(eng, reps=2):
    if REF is None:
        eng.set_factors(np.zeros((d.n_users, n_f), np.float32), M0)
    else:
        eng.set_factors(*REF)
    eng.step("user")  # warm (builds both sides)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.step("user")
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


eng1 = CoreEngine(d, n_f, rate, lam)
t1 = time_iter(eng1)
REF = (eng1.U_view.contiguous(), eng1.M_view.contiguous())
t1 = time_iter(eng1)
del eng1
out = {"config": cfg, "balance": "nnz_balanced_ranges", "t1_ms": t1, "runs": []}
print(f"1 rank: {t1:.1f} ms/iter", flush=True)
for N in Ns:
    ur = shard.nnz_balanced_ranges(d.row_ptr, N)
    ir = shard.nnz_balanced_ranges(d.col_ptr, N)
    per = []
    for r in range(N):
        eng = CoreEngine(d, n_f, rate, lam, user_range=ur[r], item_range=ir[r])
        per.append(time_iter(eng))
        del eng
        torch.cuda.empty_cache()
    # all-gathers: (N-1)/N of each factor matrix per half-sweep at ~700 GB/s effective NVLink
    ag_ms = ((d.n_users + d.n_items) * n_f * 4 * (N - 1) / N) / 700e9 * 1e3
    tN = max(per) + ag_ms
    out["runs"].append({"n": N, "per_rank_ms": per, "max_ms": max(per), "mean_ms": float(np.mean(per)),
                        "allgather_ms_est": ag_ms, "speedup": t1 / tN})
    print(f"{N} ranks: per-rank {[round(x, 1) for x in per]} max {max(per):.1f} mean {np.mean(per):.1f} "
          f"-> projected speedup {t1 / tN:.2f}x", flush=True)
print(json.dumps(out))
