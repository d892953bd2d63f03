"""The full wide config (BASELINE.json configs[4]: 10M x 1M, 2B ratings, n_f = 128) on ONE GPU (tool):
generation, one iteration with the kernel profile, and the stratified-row oracle check of test_full_size."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

spec = synth.CONFIGS["wide"]
t = time.perf_counter()
d = synth.generate("wide", device="cuda")
torch.cuda.synchronize()
print("generated", d.nnz, "ratings", d.n_users, "x", d.n_items, f"{time.perf_counter() - t:.1f}s",
      "max user", int((d.row_ptr[1:] - d.row_ptr[:-1]).max()), "max item", int((d.col_ptr[1:] - d.col_ptr[:-1]).max()),
      "mem GB", torch.cuda.memory_allocated() / 1e9, flush=True)
eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
eng.set_factors(np.zeros((d.n_users, spec["n_f"]), np.float32), synth.init_m(d.n_items, spec["n_f"]))
t = time.perf_counter()
eng.step("user")
torch.cuda.synchronize()
print(f"first iteration (incl. side builds) {time.perf_counter() - t:.1f}s mem GB {torch.cuda.max_memory_allocated() / 1e9:.1f}",
      flush=True)
_lib.profile_enable(True)
_lib.profile_collect()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.step("user")
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"iteration {ms:.0f} ms -> {d.nnz / (ms / 1e3) / 1e9:.3f} G ratings/s/iter", flush=True)
for k, v in sorted(_lib.profile_collect().items(), key=lambda kv: -kv[1][1]):
    print("   ", k, v)
