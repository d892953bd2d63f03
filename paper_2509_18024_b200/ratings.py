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

__all__ = ["RatingMatrix", "DeviceRatingMatrix", "coo_to_csr_device", "csr_to_csc_device", "build_rating_matrix",
           "read_ratings_csv", "write_ratings_csv"]


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


# ---------------------------------------------------------------------------
# Device dual index (csrc/index.cu): the reference's two host lexsorts
# (ratings.py:74-92) as one device primitive, "group by key, order by
# secondary" -- exact integer work, identical arrays.
# ---------------------------------------------------------------------------

def _index_ws(torch, n_keys, n_sec, nnz, device):
    from . import _lib
    nbytes = int(_lib.load().cals_index_workspace_bytes(int(n_keys), int(n_sec), int(nnz)))
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)


def coo_to_csr_device(keys, secs, vals, n_keys, n_sec):
    """(keys, secs, vals) device tensors (int32, int32, float32) -> (ptr int64
    [n_keys + 1], idx int32 ascending per key, val float32, dup) where dup is
    None or the first duplicated (key, sec) pair in (key, sec) order."""
    from . import _lib
    torch = _lib.require_cuda()
    dev = keys.device
    nnz = int(keys.numel())
    keys = keys.to(torch.int32).contiguous()
    secs = secs.to(device=dev, dtype=torch.int32).contiguous()
    vals = vals.to(device=dev, dtype=torch.float32).contiguous()
    ptr = torch.empty(int(n_keys) + 1, dtype=torch.int64, device=dev)
    idx = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    val = torch.empty(max(nnz, 1), dtype=torch.float32, device=dev)
    dup = torch.empty(1, dtype=torch.int64, device=dev)
    ws = _index_ws(torch, n_keys, n_sec, nnz, dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.load().cals_coo_to_csr(keys.data_ptr(), secs.data_ptr(), vals.data_ptr(), nnz, int(n_keys),
                                           int(n_sec), ptr.data_ptr(), idx.data_ptr(), val.data_ptr(),
                                           dup.data_ptr(), ws.data_ptr(), ws.numel(), st), "cals_coo_to_csr")
    d = int(dup.item()) & 0xFFFFFFFFFFFFFFFF
    pair = None if d == 0xFFFFFFFFFFFFFFFF else (d >> 32, d & 0xFFFFFFFF)
    return ptr, idx[:nnz], val[:nnz], pair


def csr_to_csc_device(ptr, idx, val, n_rows, n_cols):
    """Dual (column-major) index of a device CSR: (col_ptr int64, col_idx int32
    rows ascending per column, col_val float32) -- ratings.py:86-92."""
    from . import _lib
    torch = _lib.require_cuda()
    dev = idx.device
    nnz = int(idx.numel())
    col_ptr = torch.empty(int(n_cols) + 1, dtype=torch.int64, device=dev)
    col_idx = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    col_val = torch.empty(max(nnz, 1), dtype=torch.float32, device=dev)
    ws = _index_ws(torch, n_cols, n_rows, nnz, dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(_lib.load().cals_csr_to_csc(ptr.data_ptr(), idx.data_ptr(), val.data_ptr(), int(n_rows), int(n_cols),
                                           nnz, col_ptr.data_ptr(), col_idx.data_ptr(), col_val.data_ptr(),
                                           ws.data_ptr(), ws.numel(), st), "cals_csr_to_csc")
    return col_ptr, col_idx[:nnz], col_val[:nnz]


class DeviceRatingMatrix:
    """RatingMatrix whose dual index lives on a CUDA device.

    Same constructor arguments, validation, error messages and field names as
    the reference RatingMatrix (ratings.py:32-143); the fields are torch
    tensors (int64 pointers, int32 indices, float32 ratings -- the values the
    GPU solver consumes; ratings must be float32-representable for the fit to
    see exactly the reference's inputs).  The index is built on the device
    (csrc/index.cu) instead of by two host lexsorts.  Accepted by fit_core /
    fit / fit_fast_core and the metrics like a host RatingMatrix.
    """

    __slots__ = (
        "n_users", "n_items", "user_ids", "item_ids",
        "row_ptr", "row_items", "row_vals",
        "col_ptr", "col_users", "col_vals",
    )

    def __init__(self, users, items, values, n_users=None, n_items=None, user_ids=None, item_ids=None,
                 device=None):
        from . import _lib
        torch = _lib.require_cuda()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())

        def dev(a, dt):
            return (a if torch.is_tensor(a) else torch.as_tensor(np.asarray(a))).to(device=device, dtype=dt)

        users, items, values = dev(users, torch.int64), dev(items, torch.int64), dev(values, torch.float64)
        if not (users.shape == items.shape == values.shape) or users.dim() != 1:
            raise DataError("users, items, values must be 1-d arrays of equal length")
        n = int(users.numel())
        if n and (int(users.min()) < 0 or int(items.min()) < 0):
            raise DataError("negative entry index")
        self.n_users = int(n_users) if n_users is not None else (int(users.max()) + 1 if n else 0)
        self.n_items = int(n_items) if n_items is not None else (int(items.max()) + 1 if n else 0)
        if n and (int(users.max()) >= self.n_users or int(items.max()) >= self.n_items):
            raise DataError("entry index out of range for declared shape")
        if max(self.n_users, self.n_items) > np.iinfo(np.int32).max:
            raise DataError("matrix shape exceeds the int32 index range of the device index")
        bad = ~torch.isfinite(values)
        if n and bool(bad.any()):
            k = int(torch.nonzero(bad)[0, 0])
            raise DataError(f"non-finite rating at entry {k}: ({int(users[k])}, {int(items[k])})")
        self.user_ids = None if user_ids is None else np.asarray(user_ids)
        self.item_ids = None if item_ids is None else np.asarray(item_ids)
        self.row_ptr, self.row_items, self.row_vals, pair = coo_to_csr_device(
            users.to(torch.int32), items.to(torch.int32), values.to(torch.float32), self.n_users, self.n_items)
        if pair is not None:
            u, i = pair
            u_lab = self.user_ids[u] if self.user_ids is not None else u
            i_lab = self.item_ids[i] if self.item_ids is not None else i
            raise DataError(f"duplicate (user, item) pair: ({u_lab}, {i_lab})")
        self.col_ptr, self.col_users, self.col_vals = csr_to_csc_device(
            self.row_ptr, self.row_items, self.row_vals, self.n_users, self.n_items)

    @classmethod
    def from_host(cls, R, device=None):
        """Device copy of a host RatingMatrix: the CSR is uploaded, the CSC is
        built on the device (half the host->device bytes)."""
        from . import _lib
        torch = _lib.require_cuda()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self = object.__new__(cls)
        self.n_users, self.n_items = int(R.n_users), int(R.n_items)
        self.user_ids, self.item_ids = getattr(R, "user_ids", None), getattr(R, "item_ids", None)

        def up(a, dt):
            return (a if torch.is_tensor(a) else torch.from_numpy(np.ascontiguousarray(a))).to(device=device,
                                                                                             dtype=dt)

        self.row_ptr = up(R.row_ptr, torch.int64)
        self.row_items = up(R.row_items, torch.int32)
        self.row_vals = up(R.row_vals, torch.float32)
        self.col_ptr, self.col_users, self.col_vals = csr_to_csc_device(
            self.row_ptr, self.row_items, self.row_vals, self.n_users, self.n_items)
        return self

    def to_host(self):
        """Host RatingMatrix (float64 ratings) with the same dual index."""
        return RatingMatrix.from_csr_csc(
            self.n_users, self.n_items, self.row_ptr.cpu().numpy(), self.row_items.cpu().numpy(),
            self.row_vals.cpu().double().numpy(), self.col_ptr.cpu().numpy(), self.col_users.cpu().numpy(),
            self.col_vals.cpu().double().numpy())

    @property
    def n_entries(self):
        return int(self.row_vals.numel())

    @property
    def row_counts(self):
        return np.diff(self.row_ptr.cpu().numpy())

    @property
    def col_counts(self):
        return np.diff(self.col_ptr.cpu().numpy())

    def user_slice(self, i):
        if not 0 <= i < self.n_users:
            raise IndexError(f"user index {i} out of range [0, {self.n_users})")
        lo, hi = int(self.row_ptr[i]), int(self.row_ptr[i + 1])
        return self.row_items[lo:hi], self.row_vals[lo:hi]

    def item_slice(self, j):
        if not 0 <= j < self.n_items:
            raise IndexError(f"item index {j} out of range [0, {self.n_items})")
        lo, hi = int(self.col_ptr[j]), int(self.col_ptr[j + 1])
        return self.col_users[lo:hi], self.col_vals[lo:hi]

    def __repr__(self):
        return f"DeviceRatingMatrix({self.n_users} users x {self.n_items} items, {self.n_entries} observed)"


# ---------------------------------------------------------------------------
# Ratings CSV (ratings.py:161-183, 253-291 of the reference): the same header,
# error messages and id remapping (np.unique order of the external ids), with
# the dual index optionally built on the device.
# ---------------------------------------------------------------------------

def build_rating_matrix(triples, device=None):
    """(user_id, item_id, rating) triples -> RatingMatrix with external ids
    remapped to dense indices in sorted-id order (ratings.py:161-181);
    ``device`` (e.g. "cuda") builds a DeviceRatingMatrix instead."""
    triples = list(triples)
    if not triples:
        raise DataError("no rating triples supplied")
    raw_u = np.asarray([t[0] for t in triples])
    raw_i = np.asarray([t[1] for t in triples])
    vals = np.asarray([float(t[2]) for t in triples], dtype=np.float64)
    user_ids, users = np.unique(raw_u, return_inverse=True)
    item_ids, items = np.unique(raw_i, return_inverse=True)
    cls = RatingMatrix if device is None else DeviceRatingMatrix
    kw = {} if device is None else {"device": device}
    return cls(users, items, vals, n_users=len(user_ids), n_items=len(item_ids), user_ids=user_ids,
               item_ids=item_ids, **kw)


def read_ratings_csv(path, device=None):
    """Rating-triple CSV with header ``user,item,rating[,date]`` (ratings.py:253-276)."""
    import csv

    triples = []
    with open(path, "r", encoding="utf-8", newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None or [h.strip().lower() for h in header[:3]] != ["user", "item", "rating"]:
            raise DataError(f"{path}: expected header 'user,item,rating[,date]', got {header}")
        for lineno, row in enumerate(reader, start=2):
            if not row:
                continue
            if len(row) < 3:
                raise DataError(f"{path}:{lineno}: expected at least 3 fields, got {len(row)}")
            try:
                rating = float(row[2])
            except ValueError as exc:
                raise DataError(f"{path}:{lineno}: bad rating {row[2]!r}") from exc
            triples.append((row[0], row[1], rating))
    return build_rating_matrix(triples, device=device)


def write_ratings_csv(path, R):
    """Observed entries as ``user,item,rating`` in row-major order, external ids if
    present, shortest round-trip decimals (ratings.py:284-291)."""
    import csv

    def host(a, dt):
        return np.asarray(a.cpu().numpy() if hasattr(a, "cpu") else a, dtype=dt)

    counts = np.diff(host(R.row_ptr, np.int64))
    users = np.repeat(np.arange(R.n_users, dtype=np.int64), counts)
    items = host(R.row_items, np.int64)
    vals = host(R.row_vals, np.float64)
    u_lab = R.user_ids[users] if R.user_ids is not None else users
    i_lab = R.item_ids[items] if R.item_ids is not None else items
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["user", "item", "rating"])
        for u, i, v in zip(u_lab, i_lab, vals):
            w.writerow([u, i, repr(float(v))])
