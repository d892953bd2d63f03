"""Selection statistics of one iteration on a synthetic config (debug)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "medium"
spec = synth.CONFIGS[cfg]
d = synth.generate(cfg, device="cuda")
eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
eng.set_factors(np.zeros((d.n_users, spec["n_f"])), synth.init_m(d.n_items, spec["n_f"]))
for it in range(2):
    eng.step("user")
st = torch.zeros(16, dtype=torch.int64, device="cuda")
for s in ("user", "item"):
    st.zero_()
    _lib.load().cals_debug_stats(st.data_ptr())
    eng.half(s)
    torch.cuda.synchronize()
    _lib.load().cals_debug_stats(None)
    v = st.cpu().numpy()
    print(cfg, s, "rows(small, table)", v[0], "fallback", v[1], "cand/col", v[2] / max(v[0], 1),
          "small over", v[8], "small miss", v[9], "final over", v[10], "big cols", v[6], "big fallback", v[7],
          "miss above/below/overflow", v[11], v[12], v[13], "mean n of fallbacks", v[14] / max(v[7], 1))
for side in (eng.user, eng.item):
    c = side.counts[side.counts > 0]
    print("rows", c.size, "n mean", round(float(c.mean()), 1), "max", c.max(), "small", side.plan.n_small,
          "big", side.plan.n_big, "segs", list(side.plan.small_seg), list(side.plan.small_seg_maxn))
for side in (eng.user, eng.item):
    if side.plan.n_big:
        c = side.counts[side.counts > 0]
        big = np.sort(c)[-side.plan.n_big:]
        print("big rows n quantiles (0,.5,.9,.99,1):", np.quantile(big, [0, .5, .9, .99, 1]).astype(int),
              "big nnz share", round(float(big.sum() / c.sum()), 3), "tiles", side.plan.n_big_tiles,
              "cand", side.plan.big_cand_total)
_lib.profile_enable(True)
for s in ("user", "item"):
    for _ in range(2):
        eng.half(s)
    torch.cuda.synchronize()
    _lib.profile_collect()
    eng.half(s)
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    print(s, "half-sweep kernels (ms):", {k: round(v[1], 3) if isinstance(v, tuple) else v for k, v in prof.items()})
_lib.profile_enable(False)
