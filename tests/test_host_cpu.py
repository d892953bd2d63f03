"""CPU-only tests: the C ABI loads and exports every declared symbol, the host
planner and budget rule match the oracle, the host types validate like the
reference's, and the product path refuses to run without a GPU."""

import ctypes
import re
import os

import numpy as np
import pytest
import torch

import oracle
from conftest import ROOT, csr_csc, load_golden
import paper_2509_18024_b200 as cb
from paper_2509_18024_b200 import _lib
from paper_2509_18024_b200.synth import CONFIGS, generate

HEADER = os.path.join(ROOT, "include", "coreals_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(cals_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    names = declared_symbols()
    assert len(names) >= 12
    for name in names:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert b"sm_100a" in L.cals_build_info()


def test_shared_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_budget_host_matches_oracle(rng):
    L = _lib.load()
    counts = np.concatenate([np.arange(0, 300), rng.integers(1, 10**6, size=2000)]).astype(np.int64)
    for rate in (0.3, 0.2, 0.1, 0.05, 0.7, 0.999, 1.0, 0.1 + 0.2, 1e-4):
        out = np.empty(counts.size, np.int32)
        assert L.cals_budget_host(counts.ctypes.data, counts.size, rate, out.ctypes.data) == 0
        want = oracle.budget_array(counts, rate)
        np.testing.assert_array_equal(out[counts > 0], want[counts > 0])
        for n in (10, 7, 3, 1000):
            assert cb.sketch_budget(n, rate) == oracle.budget(n, rate)


def _plan(counts, n_f, rate):
    L = _lib.load()
    n = counts.size
    budget = np.empty(n, np.int32)
    small = np.empty(n, np.int32)
    big = np.empty(n, np.int32)
    tile_ptr = np.zeros(n + 1, np.int64)
    cand_ptr = np.zeros(n + 1, np.int64)
    meta = _lib.cals_plan()
    rc = L.cals_plan_build(counts.ctypes.data, n, n_f, rate, budget.ctypes.data, small.ctypes.data,
                           big.ctypes.data, tile_ptr.ctypes.data, cand_ptr.ctypes.data, ctypes.byref(meta))
    assert rc == 0
    return meta, budget, small[:meta.n_small], big[:meta.n_big], tile_ptr[:meta.n_big + 1], cand_ptr[:meta.n_big + 1]


@pytest.mark.parametrize("n_f", [1, 5, 16, 32, 64, 128])
def test_planner_partitions_rows(rng, n_f):
    counts = np.concatenate([np.zeros(7), rng.integers(1, 400, 500), rng.integers(1000, 200000, 40)]).astype(np.int64)
    rng.shuffle(counts)
    meta, budget, small, big, tile_ptr, cand_ptr = _plan(counts, n_f, 0.2)
    # every non-empty row exactly once, empty rows skipped (als.py:252-259)
    got = np.sort(np.concatenate([small, big]))
    np.testing.assert_array_equal(got, np.flatnonzero(counts > 0))
    # descending length order within each tier; segments cover the small list
    assert np.all(np.diff(counts[small]) <= 0) and np.all(np.diff(counts[big]) <= 0)
    assert meta.small_seg[0] == 0 and meta.small_seg[3] == meta.n_small
    for g in range(3):
        seg = small[meta.small_seg[g]:meta.small_seg[g + 1]]
        if seg.size:
            assert counts[seg].max() == meta.small_seg_maxn[g]
    if big.size:
        assert counts[big].min() > counts[small].max()
        items = np.diff(tile_ptr)
        np.testing.assert_array_equal(items, (counts[big] + meta.item_rows - 1) // meta.item_rows)
        caps = np.diff(cand_ptr) // n_f
        assert np.all(caps >= 64)
    assert _lib.load().cals_workspace_bytes(ctypes.byref(meta)) > 0


def test_solver_config_validation():
    with pytest.raises(cb.ConfigError):
        cb.SolverConfig(method="nope")
    for bad in (dict(n_f=0), dict(lam=-1), dict(rate=0.0), dict(rate=1.5), dict(max_iters=-1), dict(tol=0)):
        with pytest.raises(cb.ConfigError):
            cb.SolverConfig(method="core", **bad)
    assert issubclass(cb.ConfigError, ValueError) and issubclass(cb.NumericalError, RuntimeError)


def test_rating_matrix_layout_matches_reference_index():
    g = load_golden("fit_small.npz")
    R = cb.RatingMatrix(g["users"], g["items"], g["vals"], n_users=int(g["n_users"]), n_items=int(g["n_items"]))
    csr, csc = csr_csc(g["users"], g["items"], g["vals"], int(g["n_users"]), int(g["n_items"]))
    for a, b in zip((R.row_ptr, R.row_items, R.row_vals, R.col_ptr, R.col_users, R.col_vals), csr + csc):
        np.testing.assert_array_equal(a, b)
    with pytest.raises(cb.DataError):
        cb.RatingMatrix([0, 0], [1, 1], [1.0, 2.0])
    with pytest.raises(cb.DataError):
        cb.RatingMatrix([0], [1], [np.nan])
    with pytest.raises(cb.DataError):
        cb.RatingMatrix([0], [5], [1.0], n_users=1, n_items=3)


def test_driver_dispatch_scope():
    g = load_golden("fit_rate1.npz")
    R = cb.RatingMatrix(g["users"], g["items"], g["vals"])
    for m in ("unif", "blev"):  # outside this package: the reference keeps serving them
        with pytest.raises(cb.ConfigError):
            cb.fit_method(R, cb.SolverConfig(method=m))
    with pytest.raises(cb.ConfigError):
        cb.fit_core(R, cb.SolverConfig(method="full"))
    with pytest.raises(cb.ConfigError):
        cb.fit(R, cb.SolverConfig(method="core", rate=0.5))
    from paper_2509_18024_b200 import driver
    assert driver._DISPATCH == {"core": cb.fit_core, "full": cb.fit, "fast_core": cb.fit_fast_core}
    with pytest.raises(cb.ConfigError):
        cb.fit_fast_core(R, cb.SolverConfig(method="core", rate=0.5))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_product_path_fails_loudly_without_gpu():
    g = load_golden("fit_rate1.npz")
    R = cb.RatingMatrix(g["users"], g["items"], g["vals"])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cb.fit_core(R, cb.SolverConfig(method="core", n_f=4, rate=0.5, max_iters=1))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cb.ces_sketch(np.ones((4, 2)), 0.5)


def test_synthetic_generators_small_shapes():
    d = generate("small", device="cpu")
    assert (d.n_users, d.n_items) == (1000, 800)
    assert abs(d.nnz - 160_000) < 3000
    assert int(d.row_ptr[-1]) == d.nnz == int(d.col_ptr[-1])
    # CSR sorted by (user, item), CSC by (item, user)
    u, i, v = d.coo()
    key = u * d.n_items + i
    assert bool((key[1:] > key[:-1]).all())
    p = generate("powerlaw", device="cpu", n_users=3000, n_items=800, nnz=200_000)
    cnt = (p.row_ptr[1:] - p.row_ptr[:-1])
    assert int(cnt.min()) >= 20 and int(cnt.max()) <= 800
    vals = torch.unique(p.row_vals)
    assert set(vals.tolist()) <= {x / 2 for x in range(1, 11)}
    assert CONFIGS["large"]["nnz"] == 500_000_000
