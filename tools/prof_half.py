"""One half-sweep of a synthetic config, for ncu captures (debug tool).

usage: python tools/prof_half.py CONFIG SIDE [WARM]
Runs WARM full iterations (default 1) and then one SIDE half-sweep.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

cfg, side = sys.argv[1], sys.argv[2]
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 1
spec = synth.CONFIGS[cfg]
d = synth.generate(cfg, device="cuda")
eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
eng.set_factors(np.zeros((d.n_users, spec["n_f"])), synth.init_m(d.n_items, spec["n_f"]))
for _ in range(warm):
    eng.step("user")
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("target")
eng.half(side)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
