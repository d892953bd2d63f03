"""Timeline of one CTA of the tensor-core Gram (tc_debug 3) on a full-size config: per-chunk
compute / MMA timestamps and per-item epilogue timestamps, in SM cycles."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_18024_b200 import _lib, synth  # noqa: E402

_lib.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_trace", "libcoreals_trace.so")
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "large"
side = sys.argv[2] if len(sys.argv) > 2 else "user"
launch = int(sys.argv[3]) if len(sys.argv) > 3 else 0
spec = synth.CONFIGS[cfg]
d = synth.generate(cfg, device="cuda")
eng = CoreEngine(d, spec["n_f"], spec["rate"], spec["lam"])
eng.set_factors(np.zeros((d.n_users, spec["n_f"]), np.float32), synth.init_m(d.n_items, spec["n_f"]))
for _ in range(int(sys.argv[4]) if len(sys.argv) > 4 else 1):
    eng.half("user")
    eng.half("item")
buf = torch.zeros(49152, dtype=torch.int64, device="cuda")
L = _lib.load()
buf[49149] = launch
L.cals_debug_stats(buf.data_ptr())
_lib.set_tuning(tc_debug=8 | int(os.environ.get("TC_DBG", "0")), serial_tiers=1)
eng.half(side)
torch.cuda.synchronize()
L.cals_debug_stats(None)
_lib.set_tuning()
T = buf.cpu().numpy().astype(np.int64)
ch = T[:32768].reshape(4096, 8)
n = int((ch[:, 0] > 0).sum())
ch = ch[:n]
t0 = ch[0, 0]
print(f"{side}: launch {launch}: chunks traced {n} (CTA 0)")
print("chunk item | top->data | data->digits_done | empty_wait | ->full_arrive(w15) | mma_full_wait_done | mma_tmem_ok")
for j in list(range(0, min(n, 40))) + list(range(max(40, n - 10), n)):
    r = ch[j] - t0
    print(f"{j:5d} {ch[j,6]:4d} | {r[0]:9d} {ch[j,1]-ch[j,0]:6d} {ch[j,2]-ch[j,1]:6d} {ch[j,3]-ch[j,2]:6d} "
          f"{ch[j,7]-ch[j,0]:6d} | {r[4]:9d} {ch[j,5]-ch[j,4]:6d}")
d_top = np.diff(ch[:, 0])
print("cycles per chunk (compute warp 0): median", np.median(d_top), "mean", d_top.mean())
items = ch[:, 6]
bnd = np.nonzero(np.diff(items))[0] + 1
gap_at_item = d_top[bnd - 1] if bnd.size else np.array([0])
print(f"  items in trace {items.max() - items.min() + 1}, chunks per item {n / max(1, items.max() - items.min() + 1):.1f}; "
      f"top->top at item boundaries median {np.median(gap_at_item)} vs inside {np.median(np.delete(d_top, bnd - 1)) if bnd.size else 0}")
print("  MMA tmem-wait at item starts: median", np.median(ch[bnd, 5] - ch[bnd, 4]) if bnd.size else 0,
      "mean", (ch[bnd, 5] - ch[bnd, 4]).mean() if bnd.size else 0)
print("  issue (after data wait) median", np.median(ch[:, 7] - ch[:, 1]), " digit math median", np.median(ch[:, 2] - ch[:, 7]))
print("  data wait median", np.median(ch[:, 1] - ch[:, 0]), " digits median", np.median(ch[:, 2] - ch[:, 1]),
      " empty wait median", np.median(ch[:, 3] - ch[:, 2]), " mean", (ch[:, 3] - ch[:, 2]).mean())
e = T[32768:32768 + 8192].reshape(1024, 8)
ne = int((e[:, 0] > 0).sum())
e = e[:ne]
print(f"epilogue items {ne}: wait item_done median {np.median(e[:,1]-e[:,0])}, tmem_full wait {np.median(e[:,2]-e[:,1])},"
      f" drain {np.median(e[:,3]-e[:,2])}, exceptions {np.median(e[:,4]-e[:,3])} (max {(e[:,4]-e[:,3]).max()}),"
      f" writes {np.median(e[:,5]-e[:,4])}; items with exception work > 5000 cycles: {int(((e[:,4]-e[:,3]) > 5000).sum())}")
sch = T[40960:40960 + 8192]
ns = int((sch > 0).sum())
print(f"scheduler items {ns}: publish gap median {np.median(np.diff(sch[:ns])) if ns > 1 else 0}")
