"""Tiled-tier Gram paths (tensor-core integer vs float64 SIMT) against the float64
oracle on one half-sweep with long rows (n_f 64 and 48): factor error per path."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2509_18024_b200 as cb  # noqa: E402
from paper_2509_18024_b200 import _lib  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

rng = np.random.default_rng(3)
for n_f, outliers in ((64, 0), (48, 0), (40, 0), (64, 40)):
    n_u, n_i = 30000, 300
    mask = rng.random((n_u, n_i)) < 0.02
    mask[:, :5] = rng.random((n_u, 5)) < 0.9   # 5 long item rows (~27k ratings: two work items)
    u, i = np.nonzero(mask)
    v = (rng.normal(size=u.size) * 2 + 3).astype(np.float32).astype(np.float64)
    R = cb.RatingMatrix(u, i, v, n_users=n_u, n_items=n_i)
    U = (rng.normal(size=(n_u, n_f)) * 0.3).astype(np.float32)
    if outliers:  # heavy-tailed source rows (past the digit range: the float64 exception path)
        U[rng.choice(n_u, outliers, replace=False)] *= np.float32(1e4)
    want = np.zeros((n_i, n_f))
    _, st, ko = oracle.core_half_sweep(R.col_ptr, R.col_users, R.col_vals, U.astype(np.float64), n_f, 0.05, 0.1,
                                       want, want_keys=True, threads=os.cpu_count())
    act = np.diff(R.col_ptr) > 0
    for path in (0, 1):
        _lib.set_tuning(gram_path=path)
        eng = CoreEngine(R, n_f, 0.1, 0.05)
        eng.set_factors(U=U, M=np.zeros((n_i, n_f), np.float32))
        keys = torch.zeros((n_i, n_f), dtype=torch.int64, device="cuda")
        eng.half("item", thr_keys=keys)
        torch.cuda.synchronize()
        got = eng.M_view.double().cpu().numpy()
        kk = keys.cpu().numpy().view(np.uint64)
        err = np.abs(got - want).max(axis=1) / np.maximum(np.abs(want).max(axis=1), 1e-2)
        print(f"n_f {n_f} outliers {outliers} path {'tc' if path == 0 else 'f64'}: big rows {eng.item.plan.n_big} tiles "
              f"{eng.item.plan.n_big_tiles}; keys equal {bool((kk[act] == ko[act]).all())}; "
              f"max err {err[act].max():.2e} (long rows {err[:5].max():.2e})", flush=True)
    _lib.set_tuning()
