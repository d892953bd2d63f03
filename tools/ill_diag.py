"""Per-row error vs the oracle of ONE item half-sweep of the large config at a later
iteration, under several float64-deferral ratios (tuning ill_ratio), from the same state."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
from paper_2509_18024_b200 import synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402
from test_full_size import half, sample_rows, sub_csr  # noqa: E402

cfg, warm = sys.argv[1], int(sys.argv[2])
spec = synth.CONFIGS[cfg]
n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
d = synth.generate(cfg, device="cuda")
eng = CoreEngine(d, n_f, rate, lam)
eng.set_factors(np.zeros((d.n_users, n_f), np.float32), synth.init_m(d.n_items, n_f))
for _ in range(warm):
    eng.step("user")
eng.finish("user")
U = eng.U_view.contiguous().float().cpu().numpy()
ptr = d.col_ptr.cpu().numpy()
cnt = np.diff(ptr)
rows = sample_rows(cnt, np.random.default_rng(7), n_longest=16, n_random=100, per_decile=5)
sp, si, sv = sub_csr(ptr, d.col_users, d.col_vals, rows)
want = np.zeros((rows.size, n_f))
_, _, ko = oracle.core_half_sweep(sp, si, sv, U.astype(np.float64), n_f, lam, rate, want, want_keys=True,
                                  threads=os.cpu_count())
scale = np.maximum(np.abs(want).max(axis=1), 1e-2)
for ratio in sys.argv[3:] or ["default"]:
    if ratio != "default":
        from paper_2509_18024_b200 import _lib
        _lib.set_tuning(ill_ratio=float(ratio))
    outs = []
    for rep in range(2):
        tgt, keys = half(eng, "item", U)
        gk = keys[torch.from_numpy(rows).to(keys.device)].cpu().numpy().view(np.uint64)
        bad = (gk != ko).any(axis=1)
        if bad.any():
            print("KEY MISMATCH rows", rows[bad][:10], "n", cnt[rows[bad]][:10], "cols", (gk != ko).sum(axis=1)[bad][:10],
                  flush=True)
        got = tgt[torch.from_numpy(rows).to(tgt.device)].double().cpu().numpy()
        outs.append(got)
    err = np.abs(outs[0] - want).max(axis=1) / scale
    same = bool(np.array_equal(outs[0], outs[1]))
    line = [f"ratio {ratio}: deterministic {same}"]
    for lo, hi in [(0, 1e3), (1e3, 1e4), (1e4, 1e5), (1e5, 1e7)]:
        m = (cnt[rows] >= lo) & (cnt[rows] < hi)
        if m.any():
            line.append(f"[{lo:.0e},{hi:.0e}) max {err[m].max():.2e} med {np.median(err[m]):.2e}")
    print(" | ".join(line), flush=True)
