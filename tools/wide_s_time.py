"""Event-timed iteration and per-kernel profile of a synth config (default wide_s: the wide config's
row-length distributions and rank at 1/100 scale) -- tool for the n_f = 128 path."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

if os.environ.get("CALS_LIB"):  # A/B runs: another build of the library (tool only)
    _lib.LIB_PATH = os.path.abspath(os.environ["CALS_LIB"])
cfg = sys.argv[1] if len(sys.argv) > 1 else "wide_s"
spec = synth.CONFIGS[cfg]
d = synth.generate(cfg, device="cuda")
for var in sys.argv[2:] or ["default"]:
    kw = {} if var == "default" else {k: float(v) if "." in v else int(v) for k, v in (t.split("=") for t in var.split(","))}
    _lib.set_tuning(**kw)
    eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
    eng.use_graphs = False  # eager launches: the per-kernel event profile below needs them
    eng.set_factors(np.zeros((d.n_users, spec["n_f"]), np.float32), synth.init_m(d.n_items, spec["n_f"]))
    for _ in range(3):
        eng.step("user")
    torch.cuda.synchronize()
    stats = torch.zeros(16, dtype=torch.int64, device="cuda")
    _lib.load().cals_debug_stats(stats.data_ptr())
    _lib.profile_enable(True)
    _lib.profile_collect()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.step("user")
    e1.record()
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    _lib.profile_enable(False)
    _lib.load().cals_debug_stats(None)
    ms = e0.elapsed_time(e1)
    print(f"{cfg} {var}: iteration {ms:.1f} ms ({d.nnz / ms / 1e6:.3f} G ratings/s/iter); float64-pass systems "
          f"{int(stats[15])} of {d.n_users + d.n_items}; "
          + ", ".join(f"{k} {v[1]:.1f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:8]), flush=True)
    del eng
    _lib.set_tuning()
