import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def csr_csc(users, items, vals, n_users, n_items):
    """Reference RatingMatrix index layout (ratings.py:74-92) in numpy."""
    users = np.asarray(users, np.int64)
    items = np.asarray(items, np.int64)
    vals = np.asarray(vals, np.float64)
    o = np.lexsort((items, users))
    row_ptr = np.zeros(n_users + 1, np.int64)
    np.cumsum(np.bincount(users, minlength=n_users), out=row_ptr[1:])
    o2 = np.lexsort((users, items))
    col_ptr = np.zeros(n_items + 1, np.int64)
    np.cumsum(np.bincount(items, minlength=n_items), out=col_ptr[1:])
    return ((row_ptr, items[o].astype(np.int32), vals[o]),
            (col_ptr, users[o2].astype(np.int32), vals[o2]))


@pytest.fixture(autouse=True)
def _table_on_small_sides():
    """The production path skips the quantile table on sides below 2^20 ratings
    (qtab_min_nnz); the parity tests run at sizes far below that, so by default they
    build it anyway (the path every full-size config takes).  A test that wants the
    production setting asks for qtab_min_nnz=0 through `tuning`."""
    from paper_2509_18024_b200 import _lib

    try:
        _lib.load(build_if_missing=False)
    except (RuntimeError, OSError):  # no native library: nothing to tune
        yield
        return
    saved = _lib.TUNING_DEFAULTS["qtab_min_nnz"]
    _lib.TUNING_DEFAULTS["qtab_min_nnz"] = 1
    prev = _lib.set_tuning()
    yield
    _lib.TUNING_DEFAULTS["qtab_min_nnz"] = saved
    _lib.set_tuning(**prev)


@pytest.fixture
def tuning():
    """Explicit native tuning for one test (cals_set_tuning), restored afterwards."""
    from paper_2509_18024_b200 import _lib

    prev = []

    def set_(**fields):
        old = _lib.set_tuning(**fields)
        if not prev:
            prev.append(old)

    yield set_
    if prev:
        _lib.set_tuning(**prev[0])
