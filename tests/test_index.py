"""Device dual index (csrc/index.cu) against the reference RatingMatrix
(ratings.py:54-92): exact arrays on the reference's own fixture
(tests/golden/index_cases.npz, made by tests/golden/make_golden.py), the
reference's duplicate / range / non-finite errors, edge shapes, and fits on a
device-built matrix equal fits on the host matrix.  Integer work: bit-exact."""

import numpy as np
import pytest
import torch

from conftest import csr_csc, load_golden

import paper_2509_18024_b200 as cb


def test_host_rating_matrix_matches_index_fixture():
    g = load_golden("index_cases.npz")
    R = cb.RatingMatrix(g["users"], g["items"], g["vals"].astype(np.float64), n_users=int(g["n_users"]),
                        n_items=int(g["n_items"]))
    np.testing.assert_array_equal(R.row_ptr, g["row_ptr"])
    np.testing.assert_array_equal(R.row_items, g["row_items"])
    np.testing.assert_array_equal(R.row_vals.astype(np.float32), g["row_vals"])
    np.testing.assert_array_equal(R.col_ptr, g["col_ptr"])
    np.testing.assert_array_equal(R.col_users, g["col_users"])
    np.testing.assert_array_equal(R.col_vals.astype(np.float32), g["col_vals"])
    cases = {"dup_simple": ([3, 1, 3, 0], [2, 4, 2, 9]), "dup_two": ([9, 2, 5, 2, 9, 5], [1, 8, 3, 8, 1, 3]),
             "dup_many": ([4] * 40 + [1, 1], [7] * 40 + [0, 0])}
    for name, msg in zip(g["dup_names"], g["dup_msgs"]):
        u, i = cases[str(name)]
        with pytest.raises(cb.DataError, match=f"^{str(msg).replace('(', '[(]').replace(')', '[)]')}$"):
            cb.RatingMatrix(u, i, np.ones(len(u)))


gpu = pytest.mark.gpu
needs_cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


def _np(t):
    return t.cpu().numpy()


def _assert_same(D, users, items, vals, n_users, n_items):
    (rp, ri, rv), (cp, cu, cv) = csr_csc(users, items, vals, n_users, n_items)
    np.testing.assert_array_equal(_np(D.row_ptr), rp)
    np.testing.assert_array_equal(_np(D.row_items), ri)
    np.testing.assert_array_equal(_np(D.row_vals), rv.astype(np.float32))
    np.testing.assert_array_equal(_np(D.col_ptr), cp)
    np.testing.assert_array_equal(_np(D.col_users), cu)
    np.testing.assert_array_equal(_np(D.col_vals), cv.astype(np.float32))


@gpu
@needs_cuda
def test_device_index_matches_reference_fixture():
    g = load_golden("index_cases.npz")
    D = cb.DeviceRatingMatrix(g["users"], g["items"], g["vals"], n_users=int(g["n_users"]),
                              n_items=int(g["n_items"]))
    for f in ("row_ptr", "row_items", "row_vals", "col_ptr", "col_users", "col_vals"):
        np.testing.assert_array_equal(_np(getattr(D, f)), g[f], err_msg=f)
    cases = {"dup_simple": ([3, 1, 3, 0], [2, 4, 2, 9]), "dup_two": ([9, 2, 5, 2, 9, 5], [1, 8, 3, 8, 1, 3]),
             "dup_many": ([4] * 40 + [1, 1], [7] * 40 + [0, 0])}
    for name, msg in zip(g["dup_names"], g["dup_msgs"]):
        u, i = cases[str(name)]
        with pytest.raises(cb.DataError) as e:
            cb.DeviceRatingMatrix(u, i, np.ones(len(u)))
        assert str(e.value) == str(msg)


@gpu
@needs_cuda
def test_device_index_errors_and_edges():
    with pytest.raises(cb.DataError, match="negative entry index"):
        cb.DeviceRatingMatrix([0, -1], [1, 1], [1.0, 2.0])
    with pytest.raises(cb.DataError, match="out of range"):
        cb.DeviceRatingMatrix([0], [5], [1.0], n_users=1, n_items=3)
    with pytest.raises(cb.DataError, match=r"non-finite rating at entry 1: \(2, 0\)"):
        cb.DeviceRatingMatrix([0, 2], [1, 0], [1.0, np.inf])
    with pytest.raises(cb.DataError, match="equal length"):
        cb.DeviceRatingMatrix([0, 1], [1], [1.0])
    # empty matrix with a declared shape
    D = cb.DeviceRatingMatrix(np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0), n_users=3, n_items=2)
    assert D.n_entries == 0 and _np(D.row_ptr).tolist() == [0, 0, 0, 0] and _np(D.col_ptr).tolist() == [0, 0, 0]
    # single entry, shape inferred
    D = cb.DeviceRatingMatrix([4], [2], [0.5])
    assert (D.n_users, D.n_items) == (5, 3)
    _assert_same(D, [4], [2], [0.5], 5, 3)
    # one pair repeated past a whole secondary block (16384): the overflow path names it
    u = np.array([7] * 20000 + [3, 3, 9])
    i = np.array([1] * 20000 + [5, 6, 0])
    with pytest.raises(cb.DataError, match=r"\(7, 1\)$"):
        cb.DeviceRatingMatrix(u, i, np.ones(u.size))
    # the first duplicate in (user, item) order wins even when found in different segment tiers
    u = np.array([9] * 50 + [2, 2] + list(range(100)))
    i = np.array([30000] * 50 + [40000, 40000] + [0] * 100)
    with pytest.raises(cb.DataError, match=r"\(2, 40000\)$"):
        cb.DeviceRatingMatrix(u, i, np.ones(u.size))


@gpu
@needs_cuda
@pytest.mark.parametrize("seed,n_users,n_items,nnz", [(0, 300, 200, 5000), (1, 70000, 50000, 600000),
                                                      (2, 5, 100000, 90000)])
def test_device_index_random(seed, n_users, n_items, nnz):
    rng = np.random.default_rng(seed)
    # power-law items (hot columns spanning several secondary blocks), random order
    items = np.minimum((rng.pareto(1.1, nnz * 2) * 50).astype(np.int64), n_items - 1)
    users = rng.integers(0, n_users, nnz * 2)
    key = users * n_items + items
    _, first = np.unique(key, return_index=True)
    sel = rng.permutation(np.sort(first))[:nnz]
    users, items = users[sel], items[sel]
    vals = rng.normal(size=users.size).astype(np.float32).astype(np.float64)
    D = cb.DeviceRatingMatrix(users, items, vals, n_users=n_users, n_items=n_items)
    _assert_same(D, users, items, vals, n_users, n_items)
    H = D.to_host()
    assert H.n_entries == users.size and H.row_vals.dtype == np.float64
    # CSR -> CSC from a host matrix (the fit's upload path)
    R = cb.RatingMatrix(users, items, vals, n_users=n_users, n_items=n_items)
    D2 = cb.DeviceRatingMatrix.from_host(R)
    for f in ("col_ptr", "col_users", "col_vals"):
        np.testing.assert_array_equal(_np(getattr(D2, f)), np.asarray(getattr(R, f)).astype(
            np.float32 if f == "col_vals" else getattr(R, f).dtype), err_msg=f)


@gpu
@needs_cuda
def test_fit_on_device_matrix_equals_host_matrix():
    g = load_golden("fit_small.npz")
    kw = dict(n_users=int(g["n_users"]), n_items=int(g["n_items"]))
    R = cb.RatingMatrix(g["users"], g["items"], g["vals"], **kw)
    D = cb.DeviceRatingMatrix(g["users"], g["items"], g["vals"], **kw)
    cfg = cb.SolverConfig(method="core", n_f=5, lam=0.1, rate=0.3, max_iters=3, tol=1e-15)
    M0 = np.asarray(g["M0"], np.float64) if "M0" in g else None
    Fh, rh = cb.fit_core(R, cfg, init_m=M0)
    Fd, rd = cb.fit_core(D, cfg, init_m=M0)
    np.testing.assert_array_equal(Fh.user_factors, Fd.user_factors)
    np.testing.assert_array_equal(Fh.item_factors, Fd.item_factors)
    np.testing.assert_allclose(rh.rmse_trace, rd.rmse_trace, rtol=1e-12)  # ssq summed on host vs device
    assert cb.rmse(D, Fd) == pytest.approx(cb.rmse(R, Fh), rel=1e-12)
