"""On-disk formats against files the reference wrote and read
(tests/golden/make_golden.py io_cases): CAMX factor container
(serialize.py:14-47) and ratings CSV (ratings.py:161-183, 253-291)."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN, load_golden

import paper_2509_18024_b200 as cb
from paper_2509_18024_b200 import serialize


def test_camx_matches_reference_bytes(tmp_path):
    g = load_golden("io_cases.npz")
    ref = os.path.join(GOLDEN, "factors.camx")
    np.testing.assert_array_equal(serialize.read_matrix(ref), g["F"])
    out = tmp_path / "f.camx"
    serialize.write_matrix(out, g["F"])
    assert out.read_bytes() == open(ref, "rb").read()


def test_camx_errors(tmp_path):
    p = tmp_path / "bad.camx"
    p.write_bytes(b"CAM")
    with pytest.raises(cb.DataError, match="truncated header"):
        serialize.read_matrix(p)
    data = open(os.path.join(GOLDEN, "factors.camx"), "rb").read()
    p.write_bytes(b"XAMX" + data[4:])
    with pytest.raises(cb.DataError, match="bad magic"):
        serialize.read_matrix(p)
    p.write_bytes(data[:4] + (2).to_bytes(4, "little") + data[8:])
    with pytest.raises(cb.DataError, match="unsupported container version 2"):
        serialize.read_matrix(p)
    p.write_bytes(data[:-8])
    with pytest.raises(cb.DataError, match="truncated payload"):
        serialize.read_matrix(p)
    with pytest.raises(cb.DataError, match="2-d"):
        serialize.write_matrix(p, np.zeros(3))
    serialize.write_matrix_csv(tmp_path / "m.csv", np.arange(6.0).reshape(2, 3) / 7)
    np.testing.assert_array_equal(serialize.read_matrix_csv(tmp_path / "m.csv"), np.arange(6.0).reshape(2, 3) / 7)


def _same_as_reference(R, g):
    for f in ("row_ptr", "row_items", "row_vals", "col_ptr", "col_users", "col_vals"):
        a = getattr(R, f)
        a = a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
        np.testing.assert_array_equal(a.astype(g[f].dtype), g[f], err_msg=f)
    assert list(np.asarray(R.user_ids).astype(str)) == list(g["user_ids"])
    assert list(np.asarray(R.item_ids).astype(str)) == list(g["item_ids"])


def test_ratings_csv_matches_reference(tmp_path):
    g = load_golden("io_cases.npz")
    R = cb.read_ratings_csv(os.path.join(GOLDEN, "ratings.csv"))
    _same_as_reference(R, g)
    out = tmp_path / "w.csv"
    cb.write_ratings_csv(out, R)
    assert out.read_text() == open(os.path.join(GOLDEN, "ratings_written.csv")).read()


def test_ratings_csv_errors(tmp_path):
    p = tmp_path / "r.csv"
    p.write_text("u,i,r\n1,2,3\n")
    with pytest.raises(cb.DataError, match="expected header"):
        cb.read_ratings_csv(p)
    p.write_text("user,item,rating\n1,2\n")
    with pytest.raises(cb.DataError, match=r":2: expected at least 3 fields, got 2"):
        cb.read_ratings_csv(p)
    p.write_text("user,item,rating\n1,2,3\n1,3,abc\n")
    with pytest.raises(cb.DataError, match=r":3: bad rating 'abc'"):
        cb.read_ratings_csv(p)
    p.write_text("user,item,rating\n1,2,3\n1,2,4\n")
    with pytest.raises(cb.DataError, match=r"duplicate \(user, item\) pair: \(1, 2\)"):
        cb.read_ratings_csv(p)


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_ratings_csv_device_index_matches_reference():
    g = load_golden("io_cases.npz")
    D = cb.read_ratings_csv(os.path.join(GOLDEN, "ratings.csv"), device="cuda")
    assert isinstance(D, cb.DeviceRatingMatrix)
    _same_as_reference(D, g)
