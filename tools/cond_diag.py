"""Where the fp32 factor error of long rows comes from (debug tool): for the worst
item rows of the large config at a later iteration, rebuild the sketched normal
equations in float64 with numpy and compare solutions under controlled fp32
roundings: (a) G rounded to fp32, float64 solve; (b) float64 G, float32 LU;
(c) fp32 accumulation in chunked order; and the GPU row."""
import os
import sys

import numpy as np
import scipy.linalg as sla
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
from paper_2509_18024_b200 import synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402
from test_full_size import half  # noqa: E402

cfg, warm = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("large", 5)
spec = synth.CONFIGS[cfg]
n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
d = synth.generate(cfg, device="cuda")
eng = CoreEngine(d, n_f, rate, lam)
eng.set_factors(np.zeros((d.n_users, n_f), np.float32), synth.init_m(d.n_items, n_f))
for _ in range(warm):
    eng.step("user")
eng.finish("user")
U = eng.U_view.contiguous().float().cpu().numpy()
tgt, _ = half(eng, "item", U)
ptr = d.col_ptr.cpu().numpy()
cnt = np.diff(ptr)
rng = np.random.default_rng(3)
lo_n, hi_n = (float(sys.argv[3]), float(sys.argv[4])) if len(sys.argv) > 4 else (1e4, 1e5)
cand = np.flatnonzero((cnt >= lo_n) & (cnt < hi_n))
rows = rng.choice(cand, min(6, cand.size), replace=False)
chunked = hi_n <= 1e5
U64 = U.astype(np.float64)
for i in rows:
    lo, hi = ptr[i], ptr[i + 1]
    idx = d.col_users[lo:hi].cpu().numpy().astype(np.int64)
    y = d.col_vals[lo:hi].double().cpu().numpy()
    X = U64[idx]
    n = X.shape[0]
    s = max(1, min(n, int(np.floor(n * rate + 1e-9))))
    G = np.zeros((n_f, n_f)); b = np.zeros(n_f); G32 = np.zeros((n_f, n_f), np.float32); b32 = np.zeros(n_f, np.float32)
    for c in range(n_f):
        a = np.abs(X[:, c])
        order = np.lexsort((np.arange(n), -a))[:s]  # |x| desc, row asc
        keep = np.sort(order)
        Xk = X[keep]
        G[c] = X[keep, c] @ Xk
        b[c] = X[keep, c] @ y[keep]
        # fp32 sequential accumulation in 16384-row items, items summed in fp64 (the tiled tier)
        acc = np.zeros(n_f + 1)
        for i0 in (range(0, n, 16384) if chunked else []):
            kk = keep[(keep >= i0) & (keep < i0 + 16384)]
            part = np.zeros(n_f + 1, np.float32)
            xc = X[kk, c].astype(np.float32)
            rowsXY = np.concatenate([Xk[(keep >= i0) & (keep < i0 + 16384)], y[kk, None]], 1).astype(np.float32)
            for t in range(kk.size):
                part += xc[t] * rowsXY[t]
            acc += part.astype(np.float64)
        G32[c] = acc[:n_f]; b32[c] = acc[n_f]
    G += lam * n * np.eye(n_f)
    G32 = (G32.astype(np.float64) + lam * n * np.eye(n_f))
    w = np.linalg.solve(G, b)
    sc = max(np.abs(w).max(), 1e-2)
    wa = np.linalg.solve(G.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64))
    lu = sla.lu_factor(G.astype(np.float32)); wb = sla.lu_solve(lu, b.astype(np.float32)).astype(np.float64)
    wc = np.linalg.solve(G32, b32.astype(np.float64))
    wg = tgt[i].double().cpu().numpy()
    cond = np.linalg.cond(G)
    print(f"row {i} n {n} cond {cond:.2e} | G->fp32 {np.abs(wa-w).max()/sc:.1e} | fp32 LU {np.abs(wb-w).max()/sc:.1e} "
          f"| fp32 chunked acc {np.abs(wc-w).max()/sc:.1e} | GPU {np.abs(wg-w).max()/sc:.1e}", flush=True)
