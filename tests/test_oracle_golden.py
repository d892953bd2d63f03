"""Pin the CPU oracle (oracle/coreals_oracle.c) against fixtures produced by
the real reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle
from conftest import csr_csc, load_golden


def test_budget_known_answers():
    g = load_golden("sketch_cases.npz")
    for (n, r), want in zip(g["budget_cases"], g["budget_want"]):
        assert oracle.budget(int(n), float(r)) == int(want)
    # core.py:48-54 edge cases named in SURVEY 8(a) a2
    assert oracle.budget(10, 0.7) == 7
    assert oracle.budget(7, 0.01) == 1
    assert oracle.budget(3, 0.999) == 2


def test_selection_matches_reference_ces_sketch():
    g = load_golden("sketch_cases.npz")
    for i in range(int(g["n_cases"])):
        X, rate = g[f"X{i}"], float(g[f"rate{i}"])
        sk = oracle.ces_sketch(X, rate)
        # exact emission order too (strict-then-tied, row order): _kernels.py:86-96
        assert np.array_equal(sk.rows, g[f"rows{i}"]), i
        assert np.array_equal(sk.col_ptr, g[f"colptr{i}"]), i


def test_threshold_key_encodes_reference_tie_rule():
    # three tied |2.0| values, s=2 -> rows 0 and 1 (test_core.py:52-55)
    col = np.array([2.0, -2.0, 2.0, 1.0])
    keys = oracle.keys_of(col)
    top2 = set(np.argsort(-keys.astype(np.float64), kind="stable")[:2].tolist())
    assert top2 == {0, 1}
    assert keys[0] > keys[1] > keys[2] > keys[3]
    # +0 and -0 tie; denormals order as magnitudes
    k = oracle.keys_of(np.array([-0.0, 0.0, 1e-40, -2e-40]))
    assert k[0] > k[1] and k[3] > k[2] > k[0]


def test_update_core_matches_reference():
    g = load_golden("update_cases.npz")
    for i in range(int(g["n_cases"])):
        X, y = g[f"X{i}"], g[f"y{i}"]
        lam = float(g[f"lam{i}"])
        w, st = oracle.update_core(X, g[f"colptr{i}"], g[f"rows{i}"], y, lam, X.shape[0])
        if int(g[f"ok{i}"]) == 0:
            assert st == oracle.ORC_SINGULAR
            continue
        want = g[f"w{i}"]
        assert st != oracle.ORC_SINGULAR
        assert np.abs(w - want).max() <= 1e-9 * max(1.0, np.abs(want).max()), i


@pytest.mark.parametrize("name", ["small", "medium", "ties_wide", "rate1"])
def test_half_sweeps_and_fit_match_reference(name):
    g = load_golden(f"fit_{name}.npz")
    n_f, lam, rate = int(g["n_f"]), float(g["lam"]), float(g["rate"])
    csr, csc = csr_csc(g["users"], g["items"], g["vals"], int(g["n_users"]), int(g["n_items"]))
    # user half-sweep from M0 (SURVEY 8c.1 injection), exact selection keys
    U = np.zeros((int(g["n_users"]), n_f))
    _, st, keys = oracle.core_half_sweep(*csr, g["M0"], n_f, lam, rate, U, want_keys=True)
    assert not np.any(st == oracle.ORC_SINGULAR)
    active = np.diff(csr[0]) > 0
    assert np.array_equal(keys[active], g["thr_user"][active])
    assert np.abs(U - g["U1"]).max() <= 1e-10 * max(1.0, np.abs(g["U1"]).max())
    # item half-sweep from the fp32 snapshot of U1
    M = g["M0"].copy()
    rss, st, keys = oracle.core_half_sweep(*csc, g["U1_f32"], n_f, lam, rate, M, want_rss=True,
                                           want_keys=True)
    active = np.diff(csc[0]) > 0
    assert np.array_equal(keys[active], g["thr_item"][active])
    # empty items keep their init, which differs between the two calls
    assert np.abs(M[active] - g["M1_from_U1"][active]).max() <= 1e-10 * max(1.0, np.abs(M).max())
    # end-to-end fit trace (als.py:293-308)
    U0 = np.zeros((int(g["n_users"]), n_f))
    U, M, rep = oracle.fit_core(csr, csc, n_f, lam, rate, int(g["iters"]), 1e-15, U0, g["M0"])
    np.testing.assert_allclose(rep.objective_trace, g["objN"], rtol=1e-9)
    np.testing.assert_allclose(rep.rmse_trace, g["rmseN"], rtol=1e-9)
    np.testing.assert_allclose(U, g["UN"], rtol=1e-7, atol=1e-9)


def test_oracle_rate1_matches_reference_full_als():
    """The reference's exact ALS (method 'full') is the rate-1 collapse of the
    core estimator (test_acceptance.py:54-73): the oracle at rate 1 reproduces
    the reference's `als.fit` fixture."""
    g = load_golden("fit_full.npz")
    n_f, lam = int(g["n_f"]), float(g["lam"])
    csr, csc = csr_csc(g["users"], g["items"], g["vals"], int(g["n_users"]), int(g["n_items"]))
    U0 = np.zeros((int(g["n_users"]), n_f))
    U, M, rep = oracle.fit_core(csr, csc, n_f, lam, 1.0, int(g["iters"]), 1e-15, U0, g["M0"])
    np.testing.assert_allclose(rep.objective_trace, g["objN"], rtol=1e-9)
    np.testing.assert_allclose(rep.rmse_trace, g["rmseN"], rtol=1e-9)
    np.testing.assert_allclose(U, g["UN"], rtol=1e-7, atol=1e-9)
    np.testing.assert_allclose(M, g["MN"], rtol=1e-7, atol=1e-9)


@pytest.mark.parametrize("name", ["small", "sparse_ties", "rate1"])
def test_oracle_fast_core_matches_reference(name):
    """Method 'fast_core' (whole-matrix sketch + row-sketched Gram with the
    empty-column fallback): the oracle reproduces the reference's fixtures."""
    g = load_golden(f"fast_{name}.npz")
    n_f, lam, rate = int(g["n_f"]), float(g["lam"]), float(g["rate"])
    csr, csc = csr_csc(g["users"], g["items"], g["vals"], int(g["n_users"]), int(g["n_items"]))
    U = np.zeros((int(g["n_users"]), n_f))
    oracle.fast_half_sweep(*csr, g["M0"], n_f, lam, rate, U)
    act = np.diff(csr[0]) > 0
    np.testing.assert_allclose(U[act], g["U1"][act], rtol=1e-8, atol=1e-9)
    M = g["M0"].astype(np.float64).copy()
    oracle.fast_half_sweep(*csc, g["U1_f32"], n_f, lam, rate, M)
    act = np.diff(csc[0]) > 0
    np.testing.assert_allclose(M[act], g["M1_from_U1"][act], rtol=1e-8, atol=1e-9)
    U0 = np.zeros((int(g["n_users"]), n_f))
    U, M, rep = oracle.fit_fast_core(csr, csc, n_f, lam, rate, int(g["iters"]), 1e-15, U0, g["M0"])
    np.testing.assert_allclose(rep.objective_trace, g["objN"], rtol=1e-9)
    np.testing.assert_allclose(U, g["UN"], rtol=1e-7, atol=1e-9)


def test_multithreaded_oracle_is_deterministic():
    g = load_golden("fit_medium.npz")
    n_f, lam, rate = int(g["n_f"]), float(g["lam"]), float(g["rate"])
    csr, _ = csr_csc(g["users"], g["items"], g["vals"], int(g["n_users"]), int(g["n_items"]))
    U1 = np.zeros((int(g["n_users"]), n_f))
    U4 = np.zeros_like(U1)
    oracle.core_half_sweep(*csr, g["M0"], n_f, lam, rate, U1, threads=1)
    oracle.core_half_sweep(*csr, g["M0"], n_f, lam, rate, U4, threads=4)
    assert np.array_equal(U1, U4)
