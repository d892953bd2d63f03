"""Tier statistics of a config's plan (staged / tiled rows, work items, slice rows per side)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
d = synth.generate(cfg, device="cuda")
spec = synth.CONFIGS[cfg]
eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
for name in ("user", "item"):
    s = getattr(eng, name)
    cnt = s.counts
    big = s.big_host
    small = s.small_host
    print(f"{cfg} {name}: rows {cnt.size} staged {small.size} ({int(cnt[small].sum())} ratings) tiled {big.size} "
          f"({int(cnt[big].sum())} ratings, {s.plan.n_big_tiles} work items, "
          f"{int(((cnt[big] + 63) // 64).sum())} chunks of 64); max n {int(cnt.max())}", flush=True)
