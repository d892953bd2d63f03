"""Full-size config, one iteration (user half, then item half), timing each half with
CUDA events; under ncu, -k big_gram_tc -s N picks a launch of either side."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
_lib.set_tuning(**{k: int(v) for k, v in (a.split("=") for a in sys.argv[3:])})
spec = synth.CONFIGS[cfg]
d = synth.generate(cfg, device="cuda")
eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
eng.set_factors(np.zeros((d.n_users, spec["n_f"]), np.float32), synth.init_m(d.n_items, spec["n_f"]))
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    for side in ("user", "item"):
        _lib.profile_enable(True)
        _lib.profile_collect()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.half(side)
        e1.record()
        torch.cuda.synchronize()
        prof = _lib.profile_collect()
        print(it, side, round(e0.elapsed_time(e1), 2), "ms", {k: (c, round(v, 2)) for k, (c, v) in
                                                           sorted(prof.items(), key=lambda kv: -kv[1][1])[:12]},
              flush=True)
