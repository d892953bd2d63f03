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
_lib.load().cals_debug_stats(st.data_ptr())
eng.step("user")
torch.cuda.synchronize()
_lib.load().cals_debug_stats(None)
v = st.cpu().numpy()
print(cfg, "rows(small, table)", v[0], "fallback", v[1], "cand/col", v[2] / max(v[0], 1),
      "small over", v[8], "small miss", v[9], "final over", v[10], "big cols", v[6], "big fallback", v[7])
for side in (eng.user, eng.item):
    c = side.counts[side.counts > 0]
    print("rows", c.size, "n mean", round(float(c.mean()), 1), "max", c.max(), "small", side.plan.n_small,
          "big", side.plan.n_big, "segs", list(side.plan.small_seg), list(side.plan.small_seg_maxn))
