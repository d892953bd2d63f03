"""n_f > 64 solve (fp32 LU + float64 iterative refinement, csrc/sweep_solve_ir.cu): per-row factor error vs
the oracle and the share of systems handed to the float64 pass, for the default path and the float64 elimination (ill_ratio = 0)
settings, on (a) the ill-conditioned test matrix of tests/test_gpu_parity.py and (b) a synth config's user
side at a later iteration (debug / calibration tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
import paper_2509_18024_b200 as cb  # noqa: E402
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402
from test_gpu_parity import gpu_half, random_matrix  # noqa: E402

VARIANTS = [dict(), dict(ill_ratio=0.0),
            dict(ill_ratio=0.0, rf_slice_max=0)]


def errs(got, want):
    scale = np.maximum(np.abs(want).max(axis=1), 1e-2)
    return np.abs(got - want).max(axis=1) / scale


def run(tag, make_engine, side, source, rows_of, want):
    for var in VARIANTS:
        _lib.set_tuning(**var)
        eng = make_engine()
        stats = torch.zeros(16, dtype=torch.int64, device="cuda")
        _lib.load().cals_debug_stats(stats.data_ptr())
        got, _ = gpu_half(eng, side, source)
        _lib.load().cals_debug_stats(None)
        e = errs(got[rows_of], want)
        print(f"{tag} {var}: refined {int(stats[15])} of {got.shape[0]}; err max {e.max():.2e} p99 {np.quantile(e, 0.99):.2e} "
              f"median {np.median(e):.2e}; rows over 1e-4: {(e > 1e-4).sum()}", flush=True)
        del eng
    _lib.set_tuning()


n_f = 128
u, i, v = random_matrix(n_f + 50, 3000, 400, 0.04, heavy_items=6, heavy_density=0.9)
R = cb.RatingMatrix(u, i, v, n_users=3000, n_items=400)
rng = np.random.default_rng(3)
base = rng.normal(0.0, 3.0, (400, 1))
M0 = (base + 0.05 * rng.normal(0.0, 3.0, (400, n_f))).astype(np.float32)
want = np.zeros((3000, n_f))
oracle.core_half_sweep(R.row_ptr, R.row_items, R.row_vals, M0.astype(np.float64), n_f, 0.01, 0.1, want, threads=os.cpu_count())
act = np.flatnonzero(np.diff(R.row_ptr) > 0)
run("ill-test user", lambda: CoreEngine(R, n_f, 0.1, 0.01), "user", M0, act, want[act])

cfg = sys.argv[1] if len(sys.argv) > 1 else "wide_s"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = synth.CONFIGS[cfg]
n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
d = synth.generate(cfg, device="cuda")
eng = CoreEngine(d, n_f, rate, lam)
eng.set_factors(np.zeros((d.n_users, n_f), np.float32), synth.init_m(d.n_items, n_f))
for _ in range(warm):
    eng.step("user")
eng.finish("user")
M = eng.M_view.float().cpu().numpy().copy()
U = eng.U_view.float().cpu().numpy().copy()
del eng
for side, source, ptr, idx, val in (("user", M, d.row_ptr, d.row_items, d.row_vals), ("item", U, d.col_ptr, d.col_users, d.col_vals)):
    ptr = ptr.cpu().numpy()
    cnt = np.diff(ptr)
    rs = np.random.default_rng(5)
    rows = np.unique(np.concatenate([rs.choice(np.flatnonzero(cnt > 0), 1500, replace=False), np.argsort(-cnt)[:8]]))
    idx_h, val_h = idx.cpu().numpy(), val.cpu().numpy()
    sp = np.zeros(rows.size + 1, np.int64)
    sp[1:] = np.cumsum(cnt[rows])
    si = np.concatenate([idx_h[ptr[r]:ptr[r + 1]] for r in rows])
    sv = np.concatenate([val_h[ptr[r]:ptr[r + 1]] for r in rows]).astype(np.float64)
    want = np.zeros((rows.size, n_f))
    oracle.core_half_sweep(sp, si, sv, source.astype(np.float64), n_f, lam, rate, want, threads=os.cpu_count())
    run(f"{cfg} {side} (iteration {warm})", lambda: CoreEngine(d, n_f, rate, lam), side, source, rows, want)
