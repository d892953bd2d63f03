"""Parity at BASELINE.json's full sizes (configs 2-5: medium 10M, power-law 25M,
large 500M, wide 2B ratings at n_f = 128 -- the 8-GPU config, which fits one
B200's 180 GB) on a stratified row sample, as SURVEY 8c.1-2 prescribe for
sizes the float64 oracle cannot sweep whole: one GPU half-sweep per side (the
item side fed the GPU's own user factors), then the oracle (a restatement of
core.py:199-223, pinned to the reference's fixtures) on the sampled rows with
the same fp32 source -- every longest row, random rows, and rows from each
length decile.  Bars as in test_gpu_parity: threshold keys (hence the kept
index sets) bit-exact, factor rows within 1e-4."""

import os

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected only on GPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2509_18024_b200 import synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402

FACTOR_TOL = 1e-4


def sample_rows(counts, rng, n_longest=8, n_random=200, per_decile=10):
    active = np.flatnonzero(counts > 0)
    order = active[np.argsort(counts[active], kind="stable")]
    pick = set(order[-n_longest:].tolist())
    pick.update(rng.choice(active, min(n_random, active.size), replace=False).tolist())
    for d in np.array_split(order, 10):
        if d.size:
            pick.update(rng.choice(d, min(per_decile, d.size), replace=False).tolist())
    return np.array(sorted(pick), dtype=np.int64)


def sub_csr(ptr, idx, val, rows):
    """Host CSR of the sampled rows only (their slices gathered on the device)."""
    lo = ptr[rows]
    cnt = ptr[rows + 1] - lo
    sub_ptr = np.zeros(rows.size + 1, np.int64)
    np.cumsum(cnt, out=sub_ptr[1:])
    pos = torch.from_numpy(np.repeat(lo - sub_ptr[:-1], cnt) + np.arange(sub_ptr[-1])).to(idx.device)
    return sub_ptr, idx[pos].cpu().numpy(), val[pos].double().cpu().numpy()


def half(eng, side, source):
    n_rows = eng.n_users if side == "user" else eng.n_items
    keys = torch.zeros((n_rows, eng.n_f), dtype=torch.int64, device=eng.device)
    if side == "user":
        eng.set_factors(M=source)
    else:
        eng.set_factors(U=source)
    eng.half(side, rss=False, thr_keys=keys)
    torch.cuda.synchronize()
    tgt = (eng.U_view if side == "user" else eng.M_view).contiguous()
    return tgt, keys


@pytest.mark.parametrize("config", ["medium", "powerlaw", "large", "wide"])
def test_full_size_config_stratified_rows(config):
    spec = synth.CONFIGS[config]
    n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
    data = synth.generate(config, device="cuda", seed=0)
    eng = CoreEngine(data, n_f, rate, lam)
    rng = np.random.default_rng(7)
    source = synth.init_m(data.n_items, n_f)
    threads = max(1, os.cpu_count() or 1)
    for side in ("user", "item"):
        ptr_d, idx_d, val_d = ((data.row_ptr, data.row_items, data.row_vals) if side == "user"
                               else (data.col_ptr, data.col_users, data.col_vals))
        tgt, keys = half(eng, side, source)
        ptr = ptr_d.cpu().numpy()
        rows = sample_rows(np.diff(ptr), rng)
        sp, si, sv = sub_csr(ptr, idx_d, val_d, rows)
        src64 = np.asarray(source, np.float32).astype(np.float64)
        want = np.zeros((rows.size, n_f))
        _, st, ko = oracle.core_half_sweep(sp, si, sv, src64, n_f, lam, rate, want, want_keys=True,
                                           threads=threads)
        assert (st == 0).all()
        got_keys = keys[torch.from_numpy(rows).to(keys.device)].cpu().numpy().view(np.uint64)
        np.testing.assert_array_equal(got_keys, ko, err_msg=f"{config} {side}: selection keys")
        got = tgt[torch.from_numpy(rows).to(tgt.device)].double().cpu().numpy()
        scale = np.maximum(np.abs(want).max(axis=1), 1e-2)
        err = float((np.abs(got - want).max(axis=1) / scale).max())
        assert err <= FACTOR_TOL, f"{config} {side}: factor rel err {err:.3e}"
        # the longest rows are in the sample (the tiled tier's giant rows)
        assert int(np.diff(ptr).max()) == int(np.diff(sp).max())
        source = tgt.float().cpu().numpy()  # the item side is fed the GPU's own user rows
    del eng, data
    torch.cuda.empty_cache()
