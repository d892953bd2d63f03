"""Kernel profile of one rank's engine at N ranks on one GPU (debug tool).
usage: python tools/shard_prof.py CONFIG N RANK"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, shard, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402
cfg, N, R = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
spec = synth.CONFIGS[cfg]
d = synth.generate(cfg, device="cuda")
ur, ir = shard.nnz_balanced_ranges(d.row_ptr, N), shard.nnz_balanced_ranges(d.col_ptr, N)
eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"], user_range=ur[R], item_range=ir[R])
eng.set_factors(np.zeros((d.n_users, spec["n_f"]), np.float32), synth.init_m(d.n_items, spec["n_f"]))
eng.step("user"); torch.cuda.synchronize()
for side in ("user", "item"):
    s = eng.user if side == "user" else eng.item
    p = s.plan
    print(side, "rows", s.row_range, "n_small", p.n_small, "n_big", p.n_big, "tiles", p.n_big_tiles, "cand", p.big_cand_total,
          "item_rows", p.item_rows, "ws GB", s.ws_bytes / 1e9)
_lib.profile_enable(True); _lib.profile_collect()
for side in ("user", "item"):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); eng.half(side); b.record(); torch.cuda.synchronize()
    print(side, "half ms", a.elapsed_time(b))
    for k, v in sorted(_lib.profile_collect().items(), key=lambda kv: -kv[1][1]):
        print("   ", k, v)
# selection counters of the item half (see cals_debug_stats)
st = torch.zeros(16, dtype=torch.int64, device="cuda")
_lib.load().cals_debug_stats(st.data_ptr())
eng.half("item"); torch.cuda.synchronize()
_lib.load().cals_debug_stats(None)
names = ["columns", "fallback", "candidates", "after_prenarrow", "select_rounds", "rows", "big_columns",
         "big_fallback", "small_over", "small_miss", "final_over", "big_miss_above", "big_miss_below",
         "big_overflow", "big_fallback_n"]
print({n: int(v) for n, v in zip(names, st.cpu().tolist())})
print("refined rows (item half):", int(st[15].item()))
