"""Parity on the BASELINE.json configs at their stated sizes and iteration counts
(north_star: selected index sets exact per half-sweep, factors within 1e-4,
final training RMSE within 1e-3 after the fixed number of iterations).

* config 1 (small: 1000 x 800, n_f 5, 10 iterations) against the REAL
  reference: ``tests/golden/config1.npz`` holds the reference's 10-iteration
  fit and its trajectory run half-sweep by half-sweep from fp32 input
  snapshots.  The GPU is fed the same 20 snapshots: every
  half-sweep's threshold keys must be equal and its factors within 1e-4.
* configs 2 and 3 (medium 10M / n_f 16 / 10 iterations, power-law 25M / n_f 32
  / 15 iterations): the whole fit against the float64 oracle (pinned to the
  reference by test_oracle_golden) on identical device-generated data; final
  RMSE within 1e-3 and the objective trace within 1e-3 relative, plus every
  row of the half-sweeps of iterations 1, 5 and the last re-run by the oracle
  from the GPU's own input snapshot (keys exact, factors 1e-4).
* config 4 (large, 500M, n_f 64): after 2, 5 and 9 iterations -- the
  ill-conditioned regime of long rows -- both half-sweeps from the GPU's state
  vs the oracle on a stratified row sample that includes every row above
  100k ratings.
"""

import os

import numpy as np
import pytest
import torch

import oracle
from conftest import load_golden

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected only on GPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2509_18024_b200 as cb  # noqa: E402
from paper_2509_18024_b200 import synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402
from test_full_size import sample_rows, sub_csr  # noqa: E402

FACTOR_TOL = 1e-4
RMSE_TOL = 1e-3
THREADS = max(1, os.cpu_count() or 1)


def rel_err_rows(got, want):
    scale = np.maximum(np.abs(want).max(axis=1), 1e-2)
    return float((np.abs(got - want).max(axis=1) / scale).max()) if got.size else 0.0


def keys_from_rows(ptr, idx, source32, rows_k):
    """Threshold keys (abs_bits(x) << 32 | 0xFFFFFFFF - k) from the slice row k of each
    (row, column) threshold element (-1: empty row -> key 0)."""
    n_rows, n_f = rows_k.shape
    keys = np.zeros((n_rows, n_f), np.uint64)
    act = rows_k[:, 0] >= 0
    r = np.flatnonzero(act)
    k = rows_k[act].astype(np.int64)
    src_rows = idx[ptr[r][:, None] + k]
    x = source32[src_rows, np.arange(n_f)[None, :]].astype(np.float32)
    bits = x.view(np.uint32).astype(np.uint64) & np.uint64(0x7FFFFFFF)
    keys[act] = (bits << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - k.astype(np.uint64))
    return keys


def gpu_half(eng, side, source32, keep=None):
    """One GPU half-sweep from an fp32 source snapshot -> (target f64, keys u64)."""
    n_rows = eng.n_users if side == "user" else eng.n_items
    keys = torch.zeros((n_rows, eng.n_f), dtype=torch.int64, device=eng.device)
    if side == "user":
        eng.set_factors(M=source32, U=keep)
    else:
        eng.set_factors(U=source32, M=keep)
    eng.half(side, rss=False, thr_keys=keys)
    torch.cuda.synchronize()
    tgt = (eng.U_view if side == "user" else eng.M_view).double().cpu().numpy()
    return tgt, keys.cpu().numpy().view(np.uint64)


def config1_matrix(g):
    n_u, n_m = int(g["n_users"]), int(g["n_items"])
    mask = np.unpackbits(g["mask"])[: n_u * n_m].reshape(n_u, n_m).astype(bool)
    u, i = np.nonzero(mask)
    return cb.RatingMatrix(u, i, g["vals"].astype(np.float64), n_users=n_u, n_items=n_m)


def test_config1_every_half_sweep_vs_reference():
    g = load_golden("config1.npz")
    R = config1_matrix(g)
    n_f, lam, rate, iters = int(g["n_f"]), float(g["lam"]), float(g["rate"]), int(g["iters"])
    eng = CoreEngine(R, n_f, rate, lam)
    act_u = np.diff(R.row_ptr) > 0
    act_m = np.diff(R.col_ptr) > 0
    src = g["M0"]
    worst = 0.0
    for t in range(iters):
        U, ku = gpu_half(eng, "user", src)
        want_ku = keys_from_rows(R.row_ptr, R.row_items, src, g[f"ku{t}"].astype(np.int32))
        np.testing.assert_array_equal(ku[act_u], want_ku[act_u], err_msg=f"user keys, iteration {t}")
        eu = rel_err_rows(U[act_u], g[f"Ut{t}"][act_u])
        U32 = g[f"Ut{t}"].astype(np.float32)
        M, km = gpu_half(eng, "item", U32)
        want_km = keys_from_rows(R.col_ptr, R.col_users, U32, g[f"km{t}"].astype(np.int32))
        np.testing.assert_array_equal(km[act_m], want_km[act_m], err_msg=f"item keys, iteration {t}")
        em = rel_err_rows(M[act_m], g[f"Mt{t}"][act_m])
        assert eu <= FACTOR_TOL and em <= FACTOR_TOL, (t, eu, em)
        worst = max(worst, eu, em)
        src = g[f"Mt{t}"].astype(np.float32)
    print(f"config 1: 20 half-sweeps, keys exact, worst factor rel err {worst:.2e}")


def test_config1_fit_rmse_vs_reference():
    g = load_golden("config1.npz")
    R = config1_matrix(g)
    cfg = cb.SolverConfig(method="core", n_f=int(g["n_f"]), lam=float(g["lam"]), rate=float(g["rate"]),
                          max_iters=int(g["iters"]), tol=1e-15)
    F, rep = cb.fit_core(R, cfg, init_m=g["M0"])
    assert rep.iters_run == int(g["iters"]) and not rep.converged
    assert abs(rep.rmse_trace[-1] - g["rmseN"][-1]) <= RMSE_TOL
    np.testing.assert_allclose(rep.rmse_trace, g["rmseN"], atol=RMSE_TOL)
    np.testing.assert_allclose(rep.objective_trace, g["objN"], rtol=1e-3)


def _device_csr_csc(data):
    csr = (data.row_ptr.cpu().numpy(), data.row_items.cpu().numpy(), data.row_vals.double().cpu().numpy())
    csc = (data.col_ptr.cpu().numpy(), data.col_users.cpu().numpy(), data.col_vals.double().cpu().numpy())
    return csr, csc


@pytest.mark.parametrize("config", ["medium", "powerlaw"])
def test_config_fit_vs_oracle(config):
    spec = synth.CONFIGS[config]
    n_f, lam, rate, iters = spec["n_f"], spec["lam"], spec["rate"], spec["iters"]
    data = synth.generate(config, device="cuda", seed=0)
    csr, csc = _device_csr_csc(data)
    M0 = synth.init_m(data.n_items, n_f)
    n_u = data.n_users
    # (a) end to end: the fit through the public API vs the oracle's fit from the same start
    cfg = cb.SolverConfig(method="core", n_f=n_f, lam=lam, rate=rate, max_iters=iters, tol=1e-15)
    F, rep = cb.fit_core(data, cfg, init_m=M0)
    _, _, orep = oracle.fit_core(csr, csc, n_f, lam, rate, iters, 1e-15, np.zeros((n_u, n_f)),
                                 M0.astype(np.float64), threads=THREADS)
    assert rep.iters_run == orep.iters_run == iters
    assert abs(rep.rmse_trace[-1] - orep.rmse_trace[-1]) <= RMSE_TOL, (rep.rmse_trace[-1], orep.rmse_trace[-1])
    np.testing.assert_allclose(rep.objective_trace, orep.objective_trace, rtol=1e-3)
    # (b) injection: the GPU's own input snapshots of iterations 1, 5 and the last, every row
    eng = CoreEngine(data, n_f, rate, lam)
    eng.set_factors(np.zeros((n_u, n_f), np.float32), M0)
    check_at = {1, 5, iters}
    for t in range(1, iters + 1):
        if t in check_at:
            for side, (ptr, idx, val) in (("user", csr), ("item", csc)):
                src = (eng.M_view if side == "user" else eng.U_view).contiguous().float().cpu().numpy()
                keys = torch.zeros(((n_u if side == "user" else data.n_items), n_f), dtype=torch.int64,
                                   device=eng.device)
                eng.half(side, rss=False, thr_keys=keys)
                torch.cuda.synchronize()
                got = (eng.U_view if side == "user" else eng.M_view).double().cpu().numpy()
                want = np.zeros((ptr.size - 1, n_f))
                _, st, ko = oracle.core_half_sweep(ptr, idx, val, src.astype(np.float64), n_f, lam, rate, want,
                                                   want_keys=True, threads=THREADS)
                act = np.diff(ptr) > 0
                np.testing.assert_array_equal(keys.cpu().numpy().view(np.uint64)[act], ko[act],
                                              err_msg=f"{config} iteration {t} {side}: keys")
                err = rel_err_rows(got[act], want[act])
                assert err <= FACTOR_TOL, f"{config} iteration {t} {side}: factor rel err {err:.2e}"
        else:
            eng.half("user")
            eng.half("item")
    del eng, data
    torch.cuda.empty_cache()


def test_large_later_iterations_both_sides():
    """Config 4 after 2, 5 and 9 iterations (long rows at cond ~1e4..1e6): one half-sweep
    per side from the GPU's state vs the oracle on a stratified sample with every row
    above 100k ratings."""
    spec = synth.CONFIGS["large"]
    n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
    data = synth.generate("large", device="cuda", seed=0)
    eng = CoreEngine(data, n_f, rate, lam)
    eng.set_factors(np.zeros((data.n_users, n_f), np.float32), synth.init_m(data.n_items, n_f))
    rng = np.random.default_rng(11)
    sides = {"user": (data.row_ptr, data.row_items, data.row_vals),
             "item": (data.col_ptr, data.col_users, data.col_vals)}
    ptr_h = {s: sides[s][0].cpu().numpy() for s in sides}
    done = 0
    report = []
    for t in (2, 5, 9):
        while done < t:
            eng.half("user")
            eng.half("item")
            done += 1
        for side in ("user", "item"):
            ptr = ptr_h[side]
            cnt = np.diff(ptr)
            rows = sample_rows(cnt, rng, n_longest=8, n_random=150, per_decile=8)
            rows = np.union1d(rows, np.flatnonzero(cnt > 100_000))
            src = (eng.M_view if side == "user" else eng.U_view).contiguous().float().cpu().numpy()
            keys = torch.zeros((ptr.size - 1, n_f), dtype=torch.int64, device=eng.device)
            eng.half(side, rss=False, thr_keys=keys)
            torch.cuda.synchronize()
            tgt = eng.U_view if side == "user" else eng.M_view
            sel = torch.from_numpy(rows).to(tgt.device)
            got = tgt[sel].double().cpu().numpy()
            gk = keys[sel].cpu().numpy().view(np.uint64)
            eng.undo_half(side)  # keep the trajectory: the loop re-runs this half-sweep
            sp, si, sv = sub_csr(ptr, sides[side][1], sides[side][2], rows)
            want = np.zeros((rows.size, n_f))
            _, st, ko = oracle.core_half_sweep(sp, si, sv, src.astype(np.float64), n_f, lam, rate, want,
                                               want_keys=True, threads=THREADS)
            np.testing.assert_array_equal(gk, ko, err_msg=f"large iteration {t} {side}: keys")
            err = np.abs(got - want).max(axis=1) / np.maximum(np.abs(want).max(axis=1), 1e-2)
            wr = int(np.argmax(err))
            report.append(f"it {t} {side}: rows {rows.size} (>100k: {(cnt[rows] > 100_000).sum()}) "
                          f"max {err.max():.2e} median {np.median(err):.2e}; worst row {rows[wr]} n {cnt[rows[wr]]} "
                          f"|w| {np.abs(want[wr]).max():.3g} status {int(eng.user.status[rows[wr]] if side == 'user' else eng.item.status[rows[wr]])}")
            assert err.max() <= FACTOR_TOL, report[-1]
    print("\n".join(report))
    del eng, data
    torch.cuda.empty_cache()
