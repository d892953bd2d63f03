"""Host rating-matrix model with the reference's dual index.

Same constructor, validation and fields as
/root/reference/pkg/src/coreals/ratings.py:32-143 (RatingMatrix): CSR over
users (row_ptr int64, row_items int32, row_vals f64, sorted by (user, item))
and CSC over items (col_ptr, col_users, col_vals, sorted by (item, user)).
A reference ``coreals.RatingMatrix`` instance is accepted anywhere this
class is (duck-typed on those fields).
"""

from __future__ import annotations

import numpy as np

from .errors import DataError

__all__ = ["RatingMatrix"]


class RatingMatrix:
    __slots__ = (
        "n_users", "n_items", "user_ids", "item_ids",
        "row_ptr", "row_items", "row_vals",
        "col_ptr", "col_users", "col_vals",
    )

    def __init__(self, users, items, values, n_users=None, n_items=None, user_ids=None, item_ids=None):
        users = np.ascontiguousarray(users, dtype=np.int64)
        items = np.ascontiguousarray(items, dtype=np.int64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        if not (users.shape == items.shape == values.shape) or users.ndim != 1:
            raise DataError("users, items, values must be 1-d arrays of equal length")
        if users.size and (users.min() < 0 or items.min() < 0):
            raise DataError("negative entry index")
        self.n_users = int(n_users) if n_users is not None else (int(users.max()) + 1 if users.size else 0)
        self.n_items = int(n_items) if n_items is not None else (int(items.max()) + 1 if items.size else 0)
        if users.size and (users.max() >= self.n_users or items.max() >= self.n_items):
            raise DataError("entry index out of range for declared shape")
        bad = ~np.isfinite(values)
        if bad.any():
            k = int(np.flatnonzero(bad)[0])
            raise DataError(f"non-finite rating at entry {k}: ({users[k]}, {items[k]})")
        self.user_ids = None if user_ids is None else np.asarray(user_ids)
        self.item_ids = None if item_ids is None else np.asarray(item_ids)

        # one int64 sort key per entry instead of a two-key lexsort
        key = users * max(self.n_items, 1) + items
        order = np.argsort(key, kind="stable")
        ks = key[order]
        dup = ks[1:] == ks[:-1]
        if dup.any():
            k = int(np.flatnonzero(dup)[0])
            u, i = int(users[order[k]]), int(items[order[k]])
            u_lab = self.user_ids[u] if self.user_ids is not None else u
            i_lab = self.item_ids[i] if self.item_ids is not None else i
            raise DataError(f"duplicate (user, item) pair: ({u_lab}, {i_lab})")
        ru, ri, rv = users[order], items[order], values[order]
        self.row_ptr = np.zeros(self.n_users + 1, dtype=np.int64)
        np.cumsum(np.bincount(ru, minlength=self.n_users), out=self.row_ptr[1:])
        self.row_items = ri.astype(np.int32)
        self.row_vals = rv
        order2 = np.argsort(ri * max(self.n_users, 1) + ru, kind="stable")
        self.col_ptr = np.zeros(self.n_items + 1, dtype=np.int64)
        np.cumsum(np.bincount(ri, minlength=self.n_items), out=self.col_ptr[1:])
        self.col_users = ru[order2].astype(np.int32)
        self.col_vals = rv[order2]

    @classmethod
    def from_csr_csc(cls, n_users, n_items, row_ptr, row_items, row_vals, col_ptr, col_users, col_vals):
        """Wrap already-built dual indexes (e.g. from the synthetic generators)."""
        self = object.__new__(cls)
        self.n_users, self.n_items = int(n_users), int(n_items)
        self.user_ids = self.item_ids = None
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.row_items = np.ascontiguousarray(row_items, dtype=np.int32)
        self.row_vals = np.asarray(row_vals)
        self.col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int64)
        self.col_users = np.ascontiguousarray(col_users, dtype=np.int32)
        self.col_vals = np.asarray(col_vals)
        return self

    @property
    def n_entries(self):
        return int(self.row_vals.size)

    @property
    def row_counts(self):
        return np.diff(self.row_ptr)

    @property
    def col_counts(self):
        return np.diff(self.col_ptr)

    def user_slice(self, i):
        if not 0 <= i < self.n_users:
            raise IndexError(f"user index {i} out of range [0, {self.n_users})")
        lo, hi = self.row_ptr[i], self.row_ptr[i + 1]
        return self.row_items[lo:hi], self.row_vals[lo:hi]

    def item_slice(self, j):
        if not 0 <= j < self.n_items:
            raise IndexError(f"item index {j} out of range [0, {self.n_items})")
        lo, hi = self.col_ptr[j], self.col_ptr[j + 1]
        return self.col_users[lo:hi], self.col_vals[lo:hi]

    def entries(self):
        users = np.repeat(np.arange(self.n_users, dtype=np.int64), self.row_counts)
        return users, self.row_items.astype(np.int64), np.asarray(self.row_vals, dtype=np.float64).copy()

    def transpose(self):
        users, items, vals = self.entries()
        return RatingMatrix(items, users, vals, n_users=self.n_items, n_items=self.n_users,
                            user_ids=self.item_ids, item_ids=self.user_ids)

    def __repr__(self):
        return f"RatingMatrix({self.n_users} users x {self.n_items} items, {self.n_entries} observed)"
