"""Per-row factor error vs the oracle on the wide config's item side (debug tool)."""
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

cfg = sys.argv[1] if len(sys.argv) > 1 else "wide"
spec = synth.CONFIGS[cfg]
n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
d = synth.generate(cfg, device="cuda")
eng = CoreEngine(d, n_f, rate, lam)
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 0
side = sys.argv[3] if len(sys.argv) > 3 else "item"
eng.set_factors(np.zeros((d.n_users, n_f), np.float32), synth.init_m(d.n_items, n_f))
for _ in range(warm):  # full iterations first: factors of a later iteration
    eng.step("user")
if warm:
    eng.finish("user")
    U, M = eng.U_view.contiguous(), eng.M_view.contiguous()
    if side == "item":
        source = U.float().cpu().numpy()
    else:
        source = M.float().cpu().numpy()
else:
    source = synth.init_m(d.n_items, n_f)
    if side == "item":
        U, _ = half(eng, "user", source)
        source = U.float().cpu().numpy()
tgt, keys = half(eng, side, source)
ptr = (d.col_ptr if side == "item" else d.row_ptr).cpu().numpy()
cnt = np.diff(ptr)
rng = np.random.default_rng(7)
rows = sample_rows(cnt, rng, n_longest=16, n_random=100, per_decile=5)
sp, si, sv = sub_csr(ptr, *((d.col_users, d.col_vals) if side == "item" else (d.row_items, d.row_vals)), rows)
want = np.zeros((rows.size, n_f))
oracle.core_half_sweep(sp, si, sv, source.astype(np.float64), n_f, lam, rate, want, threads=os.cpu_count())
got = tgt[torch.from_numpy(rows).to(tgt.device)].double().cpu().numpy()
scale = np.maximum(np.abs(want).max(axis=1), 1e-2)
err = np.abs(got - want).max(axis=1) / scale
o = np.argsort(-err)
print("U stats: mean|u|", float(np.abs(source).mean()), "max|u|", float(np.abs(source).max()))
for j in o[:25]:
    print(f"row {rows[j]:8d} n {cnt[rows[j]]:8d} err {err[j]:.3e} max|w| {np.abs(want[j]).max():.3e}")
print("err by n decile:")
for lo, hi in [(0, 1e3), (1e3, 1e4), (1e4, 1e5), (1e5, 1e6), (1e6, 1e8)]:
    m = (cnt[rows] >= lo) & (cnt[rows] < hi)
    if m.any():
        print(f"  n in [{lo:.0e}, {hi:.0e}): rows {m.sum()} max err {err[m].max():.3e} median {np.median(err[m]):.3e}")
