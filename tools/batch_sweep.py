"""Tiled-tier batch-size sweep on a full-size config (tool): candidate-key and
work-item budgets per batch (cals_debug_big_batch) against the iteration time.
usage: python tools/batch_sweep.py [config] [cand_log2:tile_log2 ...]"""
import gc
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
points = sys.argv[2:] or ["0:0", "28:0", "29:17", "30:18"]
spec = synth.CONFIGS[cfg]
d = synth.generate(cfg, device="cuda")
L = _lib.load()
for p in points:
    c, t = (int(x) for x in p.split(":"))
    L.cals_debug_big_batch((1 << c) if c else 0, (1 << t) if t else 0)
    eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
    eng.set_factors(np.zeros((d.n_users, spec["n_f"]), np.float32), synth.init_m(d.n_items, spec["n_f"]))
    for _ in range(2):
        eng.iterate()
    torch.cuda.synchronize()
    ms = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.step()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    ws = (eng.user.ws_bytes + eng.item.ws_bytes) / 1e9
    print(f"cand 2^{c} tiles 2^{t}: iteration {np.median(ms):.1f} ms ({[round(x, 1) for x in ms]}), "
          f"workspace {ws:.1f} GB", flush=True)
    del eng
    gc.collect()
    torch.cuda.empty_cache()
