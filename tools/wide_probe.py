"""Scaled-down 'wide' config (n_f = 128) on one GPU: per-kernel times (debug tool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.05
spec = dict(synth.CONFIGS["wide"])
over = dict(n_users=int(spec["n_users"] * scale), n_items=int(spec["n_items"] * scale))
t = time.perf_counter()
d = synth.generate("wide", device="cuda", nnz_target=int(spec["nnz"] * scale), **over)
torch.cuda.synchronize()
print("generated", d.nnz, "ratings", d.n_users, "x", d.n_items, f"{time.perf_counter() - t:.1f}s", flush=True)
eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
eng.set_factors(np.zeros((d.n_users, spec["n_f"])), synth.init_m(d.n_items, spec["n_f"]))
eng.step("user")
torch.cuda.synchronize()
_lib.profile_enable(True)
_lib.profile_collect()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.step("user")
e1.record()
torch.cuda.synchronize()
prof = _lib.profile_collect()
ms = e0.elapsed_time(e1)
print(f"iteration {ms:.1f} ms  {d.nnz / ms * 1e3 / 1e9:.3f} G ratings/s", flush=True)
print({k: round(v[1], 1) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])})
