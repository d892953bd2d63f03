"""Generate golden fixtures by running the REAL reference package.

Run in the build container only (the reference is not on the GPU box):

    cd /tmp && NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python /root/repo/tests/golden/make_golden.py

The reference is imported read-only from /root/reference/pkg/src; numba's
cache is redirected to /tmp so nothing is written into the reference tree.
Outputs (committed): tests/golden/*.npz.  All inputs are fp32-representable
(float32 arrays upcast to float64) so the same fixtures serve the fp32 GPU
path: the reference sees exactly the values the GPU sees.
"""

import os
import sys
import warnings

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import coreals  # noqa: E402
from coreals import RatingMatrix, SolverConfig, ces_sketch, fit_core, update_user_core  # noqa: E402
from coreals.als import fit as fit_full  # noqa: E402
from coreals.core import fit_fast_core  # noqa: E402
from coreals.core import sketch_budget  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def sketch_cases():
    """ces_sketch on adversarial columns: Gaussian, 0.1-rounded ties, signed
    zeros, fp32 denormals, all-equal, sorted (core.py:95-115)."""
    rng = np.random.default_rng(20250918)
    Xs, rates, rows, cps = [], [], [], []
    fams = ["gauss", "round", "zeros", "denorm", "equal", "sorted"]
    for t in range(240):
        fam = fams[t % len(fams)]
        n = int(rng.integers(1, 300))
        p = int(rng.integers(1, 6))
        X = rng.normal(size=(n, p))
        if fam == "round":
            X = np.round(X, 1)
        elif fam == "zeros":
            X[rng.random(size=X.shape) < 0.3] = 0.0
            X[rng.random(size=X.shape) < 0.2] = -0.0
        elif fam == "denorm":
            X = X * 1e-39
        elif fam == "equal":
            X = np.sign(X) * 0.5
        elif fam == "sorted":
            X = np.sort(np.abs(X), axis=0)
        X = f32(X)
        rate = float(rng.choice([0.02, 0.05, 0.1, 0.2, 0.3, 0.5, 0.7, 0.999, 1.0, rng.uniform(0.01, 1)]))
        sk = ces_sketch(X, rate)
        Xs.append(X)
        rates.append(rate)
        rows.append(sk.rows.astype(np.int32))
        cps.append(sk.col_ptr)
    out = {"n_cases": len(Xs)}
    for i in range(len(Xs)):
        out[f"X{i}"] = Xs[i]
        out[f"rate{i}"] = rates[i]
        out[f"rows{i}"] = rows[i]
        out[f"colptr{i}"] = cps[i]
    budgets = [(10, 0.7), (7, 0.01), (3, 0.999), (5, 0.2), (1000, 0.3), (20, 0.05), (99, 0.1 + 0.2)]
    out["budget_cases"] = np.array([[n, r] for n, r in budgets], dtype=np.float64)
    out["budget_want"] = np.array([sketch_budget(n, r) for n, r in budgets], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "sketch_cases.npz"), **out)


def update_cases():
    """update_user_core (core.py:134-157) on sketched and complete slices."""
    rng = np.random.default_rng(7)
    out = {}
    n_cases = 120
    for i in range(n_cases):
        n = int(rng.integers(1, 60))
        p = int(rng.integers(1, 9))
        X = f32(rng.normal(size=(n, p)))
        y = f32(rng.normal(size=n))
        rate = float(rng.choice([0.1, 0.3, 0.5, 1.0]))
        lam = float(rng.choice([0.0, 0.05, 0.2])) if n >= p else 0.2
        sk = ces_sketch(X, rate)
        if lam == 0.0:
            # lam = 0 only where the sketched Gram is well conditioned; a
            # numerically singular system has no reproducible solution
            G = sk.to_dense().T @ X
            if np.linalg.cond(G) > 1e6:
                lam = 0.05
        try:
            w = update_user_core(X, sk, y, lam, n)
            ok = 1
        except coreals.NumericalError:
            w = np.full(p, np.nan)
            ok = 0
        out[f"X{i}"] = X
        out[f"y{i}"] = y
        out[f"rate{i}"] = rate
        out[f"lam{i}"] = lam
        out[f"w{i}"] = w
        out[f"ok{i}"] = ok
        out[f"rows{i}"] = sk.rows.astype(np.int32)
        out[f"colptr{i}"] = sk.col_ptr
    out["n_cases"] = n_cases
    np.savez_compressed(os.path.join(OUT, "update_cases.npz"), **out)


def make_matrix(seed, n_users, n_items, density, n_f_true, noise, ties=False):
    rng = np.random.default_rng(seed)
    mask = rng.random((n_users, n_items)) < density
    # every user and item keeps >= 1 rating except a couple of deliberate empties
    users, items = np.nonzero(mask)
    Ut = rng.normal(size=(n_users, n_f_true))
    Vt = rng.normal(size=(n_items, n_f_true))
    vals = np.einsum("ef,ef->e", Ut[users], Vt[items]) + noise * rng.normal(size=users.size)
    if ties:
        vals = np.round(vals * 2) / 2
    return users.astype(np.int64), items.astype(np.int64), f32(vals)


def fit_case(name, seed, n_users, n_items, density, n_f, lam, rate, iters, ties=False,
             drop_user=None, drop_item=None):
    users, items, vals = make_matrix(seed, n_users, n_items, density, max(2, n_f // 2), 0.5, ties)
    keep = np.ones(users.size, bool)
    if drop_user is not None:
        keep &= users != drop_user
    if drop_item is not None:
        keep &= items != drop_item
    users, items, vals = users[keep], items[keep], vals[keep]
    R = RatingMatrix(users, items, vals, n_users=n_users, n_items=n_items)
    rng = np.random.default_rng(seed + 1)
    M0 = rng.normal(0.0, 0.1, size=(n_items, n_f))
    if ties:
        M0 = np.round(M0, 2)
    M0 = f32(M0)
    cfg1 = SolverConfig(method="core", n_f=n_f, lam=lam, rate=rate, max_iters=1, tol=1e-15)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        F1, rep1 = fit_core(R, cfg1, init_m=M0)
        # item half from a fp32 snapshot of U1 (the GPU's input injection)
        U1 = f32(F1.user_factors)
        F1b, _ = fit_core(R, cfg1, init_u=U1, items_first=True)
        cfgN = SolverConfig(method="core", n_f=n_f, lam=lam, rate=rate, max_iters=iters, tol=1e-15)
        FN, repN = fit_core(R, cfgN, init_m=M0)

    def thr(side_ptr, side_idx, source):
        T = np.zeros((side_ptr.size - 1, n_f), dtype=np.uint64)
        for i in range(side_ptr.size - 1):
            lo, hi = side_ptr[i], side_ptr[i + 1]
            if hi == lo:
                continue
            X = source[side_idx[lo:hi]]
            sk = ces_sketch(X, rate)
            for c in range(n_f):
                r, v = sk.column(c)
                bits = np.abs(v).astype(np.float32).view(np.uint32).astype(np.uint64) & np.uint64(0x7FFFFFFF)
                k = (bits << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - r.astype(np.uint64))
                T[i, c] = k.min()
        return T

    np.savez_compressed(
        os.path.join(OUT, f"fit_{name}.npz"),
        users=users, items=items, vals=vals, n_users=n_users, n_items=n_items,
        n_f=n_f, lam=lam, rate=rate, iters=iters, M0=M0,
        U1=F1.user_factors, M1_from_U1=F1b.item_factors, U1_f32=U1,
        obj1=rep1.objective_trace, rmse1=rep1.rmse_trace,
        objN=repN.objective_trace, rmseN=repN.rmse_trace, UN=FN.user_factors, MN=FN.item_factors,
        thr_user=thr(R.row_ptr, R.row_items, M0), thr_item=thr(R.col_ptr, R.col_users, U1),
        skipped_users=repN.skipped_users, skipped_items=repN.skipped_items,
    )


def full_case(name, seed, n_users, n_items, density, n_f, lam, iters, drop_user=None):
    """The reference's exact ALS (method 'full', als.py:326-336)."""
    users, items, vals = make_matrix(seed, n_users, n_items, density, max(2, n_f // 2), 0.5)
    if drop_user is not None:
        keep = users != drop_user
        users, items, vals = users[keep], items[keep], vals[keep]
    R = RatingMatrix(users, items, vals, n_users=n_users, n_items=n_items)
    M0 = f32(np.random.default_rng(seed + 1).normal(0.0, 0.1, size=(n_items, n_f)))
    cfg = SolverConfig(method="full", n_f=n_f, lam=lam, max_iters=iters, tol=1e-15)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        F, rep = fit_full(R, cfg, init_m=M0)
    np.savez_compressed(
        os.path.join(OUT, f"fit_{name}.npz"),
        users=users, items=items, vals=vals, n_users=n_users, n_items=n_items, n_f=n_f, lam=lam, iters=iters,
        M0=M0, objN=rep.objective_trace, rmseN=rep.rmse_trace, UN=F.user_factors, MN=F.item_factors,
        skipped_users=rep.skipped_users, skipped_items=rep.skipped_items,
    )


def fast_case(name, seed, n_users, n_items, density, n_f, lam, rate, iters, drop_user=None, ties=False):
    """The reference's whole-matrix sketch variant (method 'fast_core', core.py:255-324):
    per-half-sweep global ces_sketch of the source, row-sketched Gram with the
    empty-slice-column fallback (_kernels.py:172-216).  One-iteration factors
    (from M0, and the item half from a fp32 snapshot of U1) plus N-iteration traces."""
    users, items, vals = make_matrix(seed, n_users, n_items, density, max(2, n_f // 2), 0.5, ties)
    if drop_user is not None:
        keep = users != drop_user
        users, items, vals = users[keep], items[keep], vals[keep]
    R = RatingMatrix(users, items, vals, n_users=n_users, n_items=n_items)
    M0 = np.random.default_rng(seed + 1).normal(0.0, 0.1, size=(n_items, n_f))
    if ties:
        M0 = np.round(M0, 2)
    M0 = f32(M0)
    cfg1 = SolverConfig(method="fast_core", n_f=n_f, lam=lam, rate=rate, max_iters=1, tol=1e-15)
    cfgN = SolverConfig(method="fast_core", n_f=n_f, lam=lam, rate=rate, max_iters=iters, tol=1e-15)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        F1, rep1 = fit_fast_core(R, cfg1, init_m=M0)
        U1 = f32(F1.user_factors)
        F1b, _ = fit_fast_core(R, cfg1, init_u=U1, items_first=True)
        FN, repN = fit_fast_core(R, cfgN, init_m=M0)
    np.savez_compressed(
        os.path.join(OUT, f"fast_{name}.npz"),
        users=users, items=items, vals=vals, n_users=n_users, n_items=n_items, n_f=n_f, lam=lam, rate=rate,
        iters=iters, M0=M0, U1=F1.user_factors, U1_f32=U1, M1_from_U1=F1b.item_factors,
        objN=repN.objective_trace, rmseN=repN.rmse_trace, UN=FN.user_factors, MN=FN.item_factors,
        skipped_users=repN.skipped_users, skipped_items=repN.skipped_items,
    )


def metric_cases():
    """The reference's evaluation metrics (metrics.py:64-160) on a fitted model:
    train RMSE, held-out PRMSE, hit@k and NDCG@k (with and without an explicit
    relevance threshold), for the device-side evaluation path."""
    from coreals import metrics
    users, items, vals = make_matrix(9, 150, 120, 0.3, 4, 0.5)
    rng = np.random.default_rng(10)
    test = rng.random(users.size) < 0.2
    R = RatingMatrix(users[~test], items[~test], vals[~test], n_users=150, n_items=120)
    M0 = f32(np.random.default_rng(11).normal(0.0, 0.1, size=(120, 6)))
    cfg = SolverConfig(method="core", n_f=6, lam=0.1, rate=0.3, max_iters=4, tol=1e-15)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        F, _ = fit_core(R, cfg, init_m=M0)
    held = (users[test], items[test], vals[test])
    np.savez_compressed(
        os.path.join(OUT, "metrics.npz"),
        users=users[~test], items=items[~test], vals=vals[~test], n_users=150, n_items=120,
        hu=held[0], hi=held[1], hr=held[2], U=F.user_factors, M=F.item_factors,
        rmse=metrics.rmse(R, F), prmse=metrics.prmse(held, F),
        thr95=metrics.relevance_threshold(held[2], 95.0),
        hit5=metrics.hit_at_k(held, F, 5), hit3_t0=metrics.hit_at_k(held, F, 3, threshold=0.0),
        hit1_p80=metrics.hit_at_k(held, F, 1, percentile=80.0), hit2_t1=metrics.hit_at_k(held, F, 2, threshold=1.0),
        ndcg10=metrics.ndcg_at_k(held, F, 10), ndcg3=metrics.ndcg_at_k(held, F, 3),
    )


def index_cases():
    """RatingMatrix dual index (ratings.py:54-92) on a shuffled COO with a
    heavy item (rated by users spanning several 16384-id blocks), a heavy user,
    empty rows/columns, plus the DataError messages of duplicate inputs."""
    rng = np.random.default_rng(11)
    n_users, n_items = 40000, 9000
    u_heavy = rng.choice(n_users, 20000, replace=False)            # item 7: 20000 raters
    i_heavy = rng.choice(np.setdiff1d(np.arange(n_items), [7]), 5000, replace=False)  # user 123: 5000 items
    ru = rng.integers(0, n_users, 12000)
    ri = rng.integers(0, n_items, 12000)
    users = np.concatenate([u_heavy, np.full(5000, 123), ru])
    items = np.concatenate([np.full(20000, 7), i_heavy, ri])
    key = users * n_items + items
    _, first = np.unique(key, return_index=True)
    keep = np.sort(first)
    users, items = users[keep], items[keep]
    users[users == 5] = 6          # user 5: empty row
    items[items == 11] = 12        # item 11: empty column
    key = users * n_items + items
    _, first = np.unique(key, return_index=True)
    users, items = users[np.sort(first)], items[np.sort(first)]
    perm = rng.permutation(users.size)
    users, items = users[perm], items[perm]
    vals = f32(np.round(rng.normal(3.0, 1.0, users.size), 1))
    R = RatingMatrix(users, items, vals, n_users=n_users, n_items=n_items)
    dups = {}
    for name, (du, di) in {
        "dup_simple": ([3, 1, 3, 0], [2, 4, 2, 9]),
        "dup_two": ([9, 2, 5, 2, 9, 5], [1, 8, 3, 8, 1, 3]),   # (2,8) named, not (5,3) or (9,1)
        "dup_many": ([4] * 40 + [1, 1], [7] * 40 + [0, 0]),    # first pair (1,0)
    }.items():
        try:
            RatingMatrix(np.array(du), np.array(di), np.ones(len(du)))
        except coreals.DataError as e:
            dups[name] = str(e)
    np.savez_compressed(os.path.join(OUT, "index_cases.npz"), users=users.astype(np.int32),
                        items=items.astype(np.int32), vals=vals.astype(np.float32), n_users=n_users,
                        n_items=n_items, row_ptr=R.row_ptr, row_items=R.row_items,
                        row_vals=R.row_vals.astype(np.float32), col_ptr=R.col_ptr, col_users=R.col_users,
                        col_vals=R.col_vals.astype(np.float32),
                        dup_names=np.array(list(dups)), dup_msgs=np.array(list(dups.values())))


def io_cases():
    """CAMX factor container and ratings CSV written/read by the reference
    (serialize.py:14-47, ratings.py:253-291): the files and what the reference
    reads back from them."""
    from coreals import serialize
    from coreals.ratings import read_ratings_csv, write_ratings_csv
    rng = np.random.default_rng(21)
    F = rng.normal(size=(5, 3))
    serialize.write_matrix(os.path.join(OUT, "factors.camx"), F)
    # string ids (sorted lexicographically by the reference: "u10" < "u2"), a date column
    rows = ["user,item,rating,date"]
    users = ["u2", "u10", "u2", "alice", "u10", "bob"]
    items = ["i1", "i1", "i3", "i3", "x", "i1"]
    vals = ["4.5", "3", "1e0", "2.25", "5", "0.5"]
    for u, i, v in zip(users, items, vals):
        rows.append(f"{u},{i},{v},2020-01-0{len(u)}")
    path = os.path.join(OUT, "ratings.csv")
    with open(path, "w") as fh:
        fh.write("\n".join(rows) + "\n")
    R = read_ratings_csv(path)
    write_ratings_csv(os.path.join(OUT, "ratings_written.csv"), R)
    np.savez_compressed(os.path.join(OUT, "io_cases.npz"), F=F, row_ptr=R.row_ptr, row_items=R.row_items,
                        row_vals=R.row_vals, col_ptr=R.col_ptr, col_users=R.col_users, col_vals=R.col_vals,
                        user_ids=np.asarray(R.user_ids).astype(str), item_ids=np.asarray(R.item_ids).astype(str))


def fast_cases():
    fast_case("small", 5, 200, 150, 0.2, 8, 0.1, 0.3, 4)
    # sparse slices (empty sketched columns -> fallback), ties, an empty user
    fast_case("sparse_ties", 6, 300, 120, 0.05, 16, 0.05, 0.1, 3, drop_user=2, ties=True)
    fast_case("rate1", 7, 60, 50, 0.4, 4, 0.1, 1.0, 3)


# ---------------------------------------------------------------------------
# Round 2: the BASELINE config 1 at its stated size, the reference's loop
# semantics (items_first / init_u / tol convergence / seeded init) and its
# acceptance cases c1, c6, c10 plus test_imaging's short-row restoration.
# ---------------------------------------------------------------------------

def _thr_rows(ptr, idx, source, n_f, rate):
    """Per (row, column) the slice row of the sketch threshold element: the
    last kept element of ces_sketch (core.py:95-115) in key order, i.e. the
    kept element with the smallest (|x|, -row) key.  -1 for empty rows.  The
    threshold key is (abs_bits(x) << 32) | (0xFFFFFFFF - k) of that element."""
    n_rows = ptr.size - 1
    out = np.full((n_rows, n_f), -1, dtype=np.int32)
    for i in range(n_rows):
        lo, hi = ptr[i], ptr[i + 1]
        if hi == lo:
            continue
        X = source[idx[lo:hi]]
        sk = ces_sketch(X, rate)
        for c in range(n_f):
            r, v = sk.column(c)
            bits = np.abs(v).astype(np.float32).view(np.uint32).astype(np.uint64) & np.uint64(0x7FFFFFFF)
            k = (bits << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - r.astype(np.uint64))
            out[i, c] = int(r[int(np.argmin(k))])
    return out


def config1_case():
    """BASELINE configs[0] exactly: U* 1000x5, V* 800x5 i.i.d. N(0,1), R = U* V*^T +
    N(0, 0.5^2), Bernoulli(0.2) mask, n_f 5, lam 0.1, rate 0.3, 10 iterations,
    M0 ~ N(0, 0.1^2) seed 0.  Values are fp32 (upcast for the reference).
    Besides the plain 10-iteration fit, the reference is run half-sweep by
    half-sweep along its own trajectory with every input snapshot rounded to
    fp32 (SURVEY 8c.1 injection): a GPU test feeds the same snapshots and
    compares all 20 half-sweeps (threshold rows exactly, factors to 1e-4)."""
    rng = np.random.default_rng(2025)
    n_u, n_m, r, n_f, lam, rate, iters = 1000, 800, 5, 5, 0.1, 0.3, 10
    Ut = rng.normal(size=(n_u, r))
    Vt = rng.normal(size=(n_m, r))
    mask = rng.random((n_u, n_m)) < 0.2
    users, items = np.nonzero(mask)
    vals = f32(np.einsum("ef,ef->e", Ut[users], Vt[items]) + 0.5 * rng.normal(size=users.size))
    R = RatingMatrix(users, items, vals, n_users=n_u, n_items=n_m)
    M0 = f32(np.random.default_rng(0).normal(0.0, 0.1, size=(n_m, n_f)))
    cfgN = SolverConfig(method="core", n_f=n_f, lam=lam, rate=rate, max_iters=iters, tol=1e-15)
    cfg1 = SolverConfig(method="core", n_f=n_f, lam=lam, rate=rate, max_iters=1, tol=1e-15)
    out = {}
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        FN, repN = fit_core(R, cfgN, init_m=M0)
        src = M0
        for t in range(iters):
            Fu, _ = fit_core(R, cfg1, init_m=src)                       # user half from the M snapshot
            U32 = f32(Fu.user_factors)
            Fm, _ = fit_core(R, cfg1, init_u=U32, items_first=True)      # item half from the U snapshot
            out[f"Ut{t}"] = Fu.user_factors
            out[f"Mt{t}"] = Fm.item_factors
            out[f"ku{t}"] = _thr_rows(R.row_ptr, R.row_items, src, n_f, rate).astype(np.int16)
            out[f"km{t}"] = _thr_rows(R.col_ptr, R.col_users, U32, n_f, rate).astype(np.int16)
            src = f32(Fm.item_factors)
    np.savez_compressed(
        os.path.join(OUT, "config1.npz"), mask=np.packbits(mask), vals=vals.astype(np.float32), n_users=n_u,
        n_items=n_m, n_f=n_f, lam=lam, rate=rate, iters=iters, M0=M0.astype(np.float32),
        objN=repN.objective_trace, rmseN=repN.rmse_trace, UN=FN.user_factors, MN=FN.item_factors, **out)


def semantics_case():
    """Loop semantics of _alternate (als.py:243-323) through fit_core: items_first with
    init_u, a tol-converged fit (iters_run / converged / traces / the factors of the
    converged iteration), the seeded default init, init_u on a user-first fit."""
    users, items, vals = make_matrix(12, 200, 150, 0.3, 4, 0.5)
    R = RatingMatrix(users, items, vals, n_users=200, n_items=150)
    rng = np.random.default_rng(13)
    n_f, lam, rate = 8, 0.1, 0.3
    M0 = f32(rng.normal(0.0, 0.1, size=(150, n_f)))
    U0 = f32(rng.normal(0.0, 0.1, size=(200, n_f)))
    out = dict(users=users, items=items, vals=vals, n_users=200, n_items=150, n_f=n_f, lam=lam, rate=rate,
               M0=M0, U0=U0)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg3 = SolverConfig(method="core", n_f=n_f, lam=lam, rate=rate, max_iters=3, tol=1e-15)
        F, rep = fit_core(R, cfg3, init_u=U0, init_m=M0, items_first=True)
        out.update(if_obj=rep.objective_trace, if_rmse=rep.rmse_trace, if_U=F.user_factors, if_M=F.item_factors)
        F, rep = fit_core(R, cfg3, init_u=U0, init_m=M0)
        out.update(iu_obj=rep.objective_trace, iu_U=F.user_factors, iu_M=F.item_factors)
        cfgt = SolverConfig(method="core", n_f=n_f, lam=lam, rate=rate, max_iters=60, tol=2e-3)
        F, rep = fit_core(R, cfgt, init_m=M0)
        out.update(tol_obj=rep.objective_trace, tol_rmse=rep.rmse_trace, tol_iters=rep.iters_run,
                   tol_conv=rep.converged, tol_U=F.user_factors, tol_M=F.item_factors)
        cfgs = SolverConfig(method="core", n_f=n_f, lam=lam, rate=rate, max_iters=3, tol=1e-15, seed=7)
        F, rep = fit_core(R, cfgs)
        out.update(seed_obj=rep.objective_trace, seed_rmse=rep.rmse_trace)
    np.savez_compressed(os.path.join(OUT, "semantics.npz"), **out)


def acceptance_cases():
    """The reference acceptance criteria c1 (rate-1 collapse, 20 seeds,
    pkg/tests/test_acceptance.py:54-73), c6 (convergence regime, :195-209; the
    first 12 of its 40 seeds) and c10 (image restoration, :414-429), and
    test_imaging.py:84-95 (n_f 50 on rows shorter than n_f).  Inputs come from
    the reference's own generators, values rounded to fp32; the initial item
    factors are the reference's seeded init rounded to fp32 and passed
    explicitly to both sides."""
    import itertools
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import random_matrix  # reference test helper (generator wrapper)
    from test_acceptance import _rank50_image
    from coreals import GrayImage, mask_image, restore  # noqa: F401
    from coreals.als import init_factors

    def f32R(R):
        u, i, v = R.entries()
        return RatingMatrix(u, i, f32(v), n_users=R.n_users, n_items=R.n_items)

    out = {}
    combos = list(itertools.product(["normal", "lognormal", "t4"], [0.4, 0.7]))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for seed in range(20):
            dist, alpha = combos[seed % len(combos)]
            n_u, n_m = 80 + 11 * (seed % 5), 70 + 7 * (seed % 4)
            R0, _ = random_matrix(seed, n_users=n_u, n_items=n_m, alpha=alpha, dist=dist, n_f=5)
            R = f32R(R0)
            kw = dict(n_f=5, lam=0.1, rate=1.0, max_iters=4, tol=1e-12, seed=seed)
            M0 = f32(init_factors(R, SolverConfig(method="full", **kw)).item_factors)
            _, rf = fit_full(R, SolverConfig(method="full", **kw), init_m=M0)
            u, i, v = R.entries()
            out.update({f"c1_u{seed}": u.astype(np.int32), f"c1_i{seed}": i.astype(np.int32),
                        f"c1_v{seed}": v.astype(np.float32), f"c1_shape{seed}": np.array([n_u, n_m]),
                        f"c1_M0{seed}": M0.astype(np.float32), f"c1_obj{seed}": rf.objective_trace})
        for j, seed in enumerate(range(12)):
            R = f32R(random_matrix(200 + seed, n_users=300, n_items=300, alpha=0.4, dist="normal", n_f=20)[0])
            cfg = SolverConfig(method="core", n_f=20, lam=0.1, rate=0.25, max_iters=50, tol=0.01, seed=seed)
            M0 = f32(init_factors(R, cfg).item_factors)
            F, rep = fit_core(R, cfg, init_m=M0)
            u, i, v = R.entries()
            out.update({f"c6_key{j}": (u * 300 + i).astype(np.int32), f"c6_v{j}": v.astype(np.float32),
                        f"c6_M0{j}": M0.astype(np.float32), f"c6_obj{j}": rep.objective_trace,
                        f"c6_iters{j}": rep.iters_run, f"c6_conv{j}": rep.converged})
        for seed in (1, 2, 3):
            img = GrayImage(f32(_rank50_image(seed).pixels))
            masked = mask_image(img, 0.6, seed=seed)
            common = dict(n_f=50, lam=0.01, max_iters=5, tol=1e-15, seed=seed)
            M0 = f32(init_factors(masked, SolverConfig(method="full", **common)).item_factors)
            res = {}
            for meth, rate in (("full", 1.0), ("core", 0.15)):
                cfg = SolverConfig(method=meth, rate=rate, **common)
                F, rep = (fit_full if meth == "full" else fit_core)(masked, cfg, init_m=M0)
                pred = np.clip(F.user_factors @ F.item_factors.T, 0.0, 1.0)
                mse = float(np.mean((pred - img.pixels) ** 2))
                res[meth] = (min(10.0 * np.log10(1.0 / mse), 100.0), rep.objective_trace)
            u, i, _ = masked.entries()
            out.update({f"c10_img{seed}": img.pixels.astype(np.float32), f"c10_key{seed}": (u * 256 + i).astype(np.int32),
                        f"c10_M0{seed}": M0.astype(np.float32),
                        f"c10_psnr_full{seed}": res["full"][0], f"c10_psnr_core{seed}": res["core"][0],
                        f"c10_obj_full{seed}": res["full"][1], f"c10_obj_core{seed}": res["core"][1]})
        img = GrayImage(f32(np.random.default_rng(5).uniform(size=(96, 96))))
        masked = mask_image(img, 0.6, seed=5)
        cfg = SolverConfig(method="core", n_f=50, lam=0.01, rate=0.15, max_iters=5, tol=1e-12, seed=1)
        M0 = f32(init_factors(masked, cfg).item_factors)
        F, rep = fit_core(masked, cfg, init_m=M0)
        u, i, _ = masked.entries()
        out.update(img96=img.pixels.astype(np.float32), img96_key=(u * 96 + i).astype(np.int32),
                   img96_M0=M0.astype(np.float32), img96_obj=rep.objective_trace, img96_iters=rep.iters_run,
                   img96_U=F.user_factors, img96_M=F.item_factors)
    np.savez_compressed(os.path.join(OUT, "acceptance.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["full"]:
        full_case("full", 4, 120, 90, 0.3, 8, 0.1, 4, drop_user=7)
        sys.exit(0)
    if sys.argv[1:] == ["fast"]:
        fast_cases()
        sys.exit(0)
    if sys.argv[1:] == ["io"]:
        io_cases()
        sys.exit(0)
    if sys.argv[1:] == ["index"]:
        index_cases()
        sys.exit(0)
    if sys.argv[1:] == ["r02"]:
        config1_case()
        semantics_case()
        acceptance_cases()
        sys.exit(0)
    if sys.argv[1:] == ["metrics"]:
        metric_cases()
        sys.exit(0)
    sketch_cases()
    update_cases()
    # config-1 shape scaled down (BASELINE configs[0]: n_f=5, lam=0.1, r=0.3)
    fit_case("small", 0, 300, 240, 0.2, 5, 0.1, 0.3, 5)
    # medium-like rank (n_f=16, lam=0.05, r=0.2), dense enough for long rows
    fit_case("medium", 1, 160, 120, 0.5, 16, 0.05, 0.2, 4)
    # n_f=32 with rows shorter than n_f, empty user/item, ties in data and factors
    fit_case("ties_wide", 2, 90, 70, 0.15, 32, 0.05, 0.2, 3, ties=True, drop_user=3, drop_item=5)
    # rate 1: every row takes the exact SPD path
    fit_case("rate1", 3, 50, 40, 0.4, 4, 0.1, 1.0, 3)
    # exact ALS (method 'full')
    full_case("full", 4, 120, 90, 0.3, 8, 0.1, 4, drop_user=7)
    fast_cases()
    metric_cases()
    index_cases()
    io_cases()
    print("golden fixtures written to", OUT)
