"""How many systems a half-sweep defers to the float64 solve (debug tool).
usage: python tools/refine_count.py CONFIG [WARM]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402
cfg = sys.argv[1]; warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = synth.CONFIGS[cfg]
d = synth.generate(cfg, device="cuda")
eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
eng.set_factors(np.zeros((d.n_users, spec["n_f"]), np.float32), synth.init_m(d.n_items, spec["n_f"]))
for _ in range(warm):
    eng.step("user")
torch.cuda.synchronize()
for side in ("user", "item"):
    st = torch.zeros(16, dtype=torch.int64, device="cuda")
    _lib.load().cals_debug_stats(st.data_ptr())
    _lib.profile_enable(True); _lib.profile_collect()
    eng.half(side); torch.cuda.synchronize()
    prof = _lib.profile_collect(); _lib.profile_enable(False)
    _lib.load().cals_debug_stats(None)
    rows = d.n_users if side == "user" else d.n_items
    print(side, "rows", rows, "refined", int(st[15]), "refine ms", prof.get("refine_kernel"), "solve ms", prof.get("solve_kernel"), flush=True)
