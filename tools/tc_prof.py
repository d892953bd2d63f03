"""A scaled large config (same row-length law, ~60M ratings) for profiling the tiled tier:
two iterations after one warm-up."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

d = synth.generate("large", device="cuda", n_users=125_000, n_items=25_000, nnz=62_500_000)
spec = synth.CONFIGS["large"]
eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
eng.set_factors(np.zeros((d.n_users, spec["n_f"]), np.float32), synth.init_m(d.n_items, spec["n_f"]))
for _ in range(3):
    eng.step("user")
torch.cuda.synchronize()
print("ok", d.nnz)
