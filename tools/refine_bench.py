"""float64 solve throughput at a given rank: the medium config's data with n_f = NF, every
system through the float64 pass (n_f > 64), rows rebuilding from the slice or (rf_slice_max=0)
from the stored equations; event-timed kernels of one iteration after two warm-ups."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 128
d = synth.generate("medium", device="cuda")
spec = synth.CONFIGS["medium"]
for var in sys.argv[2:] or ["default"]:
    kw = {} if var == "default" else {k: int(v) for k, v in (t.split("=") for t in var.split(","))}
    _lib.set_tuning(serial_tiers=1, **kw)
    eng = CoreEngine(d, nf, spec["rate"], spec["lam"])
    eng.set_factors(np.zeros((d.n_users, nf), np.float32), synth.init_m(d.n_items, nf))
    for _ in range(2):
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
    _lib.profile_enable(False)
    ms = e0.elapsed_time(e1)
    systems = d.n_users + d.n_items
    rk = prof.get("refine_kernel", (0, 0.0))
    print(f"n_f {nf} {var}: iteration {ms:.1f} ms; refine {rk[1]:.1f} ms for ~{systems} systems "
          f"({rk[1] * 1e3 / systems:.2f} us/system); "
          + ", ".join(f"{k} {v[1]:.1f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:5]), flush=True)
    del eng
    _lib.set_tuning()
