"""Per-kernel event-timed breakdown of full iterations of a config under several
tuning variants (one process, one dataset):  python tools/phase_prof.py large
"default" "serial_tiers=1" "cand=29" ...   Each variant: 2 (or $WARM) warm-up + 2 timed iterations."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

if os.environ.get("CALS_LIB"):  # A/B runs: another build of the library (tool only)
    _lib.LIB_PATH = os.path.abspath(os.environ["CALS_LIB"])
cfg = sys.argv[1]
spec = synth.CONFIGS[cfg]
d = synth.generate(cfg, device="cuda")
M0 = synth.init_m(d.n_items, spec["n_f"])
L = _lib.load()
for var in sys.argv[2:]:
    kw = {}
    cand = 0
    for tok in var.split(","):
        if tok == "default":
            continue
        k, v = tok.split("=")
        if k == "cand":
            cand = 1 << int(v)
        else:
            kw[k] = float(v) if "." in v else int(v)
    _lib.set_tuning(**kw)
    L.cals_debug_big_batch(cand, 0)
    eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
    eng.set_factors(np.zeros((d.n_users, spec["n_f"]), np.float32), M0)
    eng.use_graphs = False  # eager launches: the event profile needs them
    for _ in range(int(os.environ.get("WARM", "2"))):  # WARM=8: factors of a later iteration
        eng.step("user")
    torch.cuda.synchronize()
    stats = torch.zeros(16, dtype=torch.int64, device="cuda")
    L.cals_debug_stats(stats.data_ptr())
    _lib.profile_enable(True)
    _lib.profile_collect()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        eng.step("user")
    e1.record()
    torch.cuda.synchronize()
    prof = _lib.profile_collect()
    _lib.profile_enable(False)
    L.cals_debug_stats(None)
    print("float64-pass systems per iteration:", int(stats[15]) // 2, flush=True)
    ms = e0.elapsed_time(e1) / 2
    ks = {k: (c // 2, round(v / 2, 2)) for k, (c, v) in sorted(prof.items(), key=lambda kv: -kv[1][1])}
    print(json.dumps({"variant": var, "ms_per_iter": round(ms, 2), "kernels(launches, ms per iter)": ks}), flush=True)
    del eng
    torch.cuda.empty_cache()
    L.cals_debug_big_batch(0, 0)
    _lib.set_tuning()
