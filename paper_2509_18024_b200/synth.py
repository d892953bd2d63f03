"""Seeded synthetic rating matrices with the shapes and distributions of the
five BASELINE.json configs (no public dataset is involved).

Generation runs on the given torch device (the GPU for the big configs) and
returns both indexes -- CSR over users sorted by (user, item) and CSC over
items sorted by (item, user), the reference RatingMatrix layout
(ratings.py:74-92) -- with int64 pointers, int32 indices and fp32 values.
This is data preparation, not part of the timed hot path.

  small     1000 x 800, Bernoulli(0.2) mask, rank-5 N(0,1) truth + N(0,0.5^2)
  medium    20000 x 10000, Bernoulli(0.05), rank-16 truth + N(0,0.3^2)
  powerlaw  162541 x 59047, 25M: lognormal(4.0,1.2) user counts clipped to
            [20, n_items], Zipf(1.1) item popularity, rank-32 truth +
            N(0,0.5^2) mapped x -> 2.75 + z (z standardised) and quantised to
            {0.5, 1.0, ..., 5.0}
  large     1e6 x 2e5, 500M: lognormal(5.5,1.0) users, Zipf(1.05) items,
            rank-64 truth + N(0,0.3^2)
  wide      1e7 x 1e6, 2B: lognormal(4.5,1.3) users, Zipf(1.0) items,
            rank-128 truth + N(0,0.3^2)
Factor init for every config: M0 ~ N(0, 0.1^2) from numpy default_rng(0),
cast to fp32; U0 = 0 (als.py:130).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

CONFIGS = {
    "small": dict(n_users=1000, n_items=800, kind="bernoulli", density=0.2, rank=5, noise=0.5,
                  n_f=5, lam=0.1, rate=0.3, iters=10),
    "medium": dict(n_users=20000, n_items=10000, kind="bernoulli", density=0.05, rank=16, noise=0.3,
                   n_f=16, lam=0.05, rate=0.2, iters=10),
    "powerlaw": dict(n_users=162541, n_items=59047, kind="powerlaw", nnz=25_000_000, zipf=1.1, mu=4.0, sigma=1.2,
                     min_count=20, rank=32, noise=0.5, quantize=True, n_f=32, lam=0.05, rate=0.2, iters=15),
    "large": dict(n_users=1_000_000, n_items=200_000, kind="powerlaw", nnz=500_000_000, zipf=1.05, mu=5.5,
                  sigma=1.0, min_count=1, rank=64, noise=0.3, n_f=64, lam=0.02, rate=0.1, iters=10),
    "wide": dict(n_users=10_000_000, n_items=1_000_000, kind="powerlaw", nnz=2_000_000_000, zipf=1.0, mu=4.5,
                 sigma=1.3, min_count=1, rank=128, noise=0.3, n_f=128, lam=0.01, rate=0.05, iters=5),
    # wide at 1/100 scale (same row-length distributions and rank): profiling and parity runs of the
    # n_f = 128 path that finish in seconds
    "wide_s": dict(n_users=100_000, n_items=10_000, kind="powerlaw", nnz=20_000_000, zipf=1.0, mu=4.5,
                   sigma=1.3, min_count=1, rank=128, noise=0.3, n_f=128, lam=0.01, rate=0.05, iters=5),
}


@dataclass
class SynthData:
    name: str
    n_users: int
    n_items: int
    row_ptr: torch.Tensor
    row_items: torch.Tensor
    row_vals: torch.Tensor
    col_ptr: torch.Tensor
    col_users: torch.Tensor
    col_vals: torch.Tensor
    spec: dict

    @property
    def nnz(self):
        return int(self.row_items.numel())

    def rating_matrix(self):
        """Host RatingMatrix (numpy) holding the same entries (values as float64)."""
        from .ratings import RatingMatrix
        return RatingMatrix.from_csr_csc(
            self.n_users, self.n_items, self.row_ptr.cpu().numpy(), self.row_items.cpu().numpy(),
            self.row_vals.cpu().numpy().astype(np.float64), self.col_ptr.cpu().numpy(),
            self.col_users.cpu().numpy(), self.col_vals.cpu().numpy().astype(np.float64))

    def coo(self):
        users = torch.repeat_interleave(torch.arange(self.n_users, device=self.row_ptr.device),
                                        self.row_ptr[1:] - self.row_ptr[:-1])
        return users, self.row_items.long(), self.row_vals


def init_m(n_items, n_f, seed=0):
    """M0 ~ N(0, 0.1^2), numpy default_rng(seed), fp32 (BASELINE configs[0])."""
    return np.random.default_rng(seed).normal(0.0, 0.1, size=(n_items, n_f)).astype(np.float32)


def _ptr_from_sorted(keys_major, n):
    counts = torch.bincount(keys_major, minlength=n)
    ptr = torch.zeros(n + 1, dtype=torch.int64, device=keys_major.device)
    ptr[1:] = torch.cumsum(counts, 0)
    return ptr


def _finish(name, spec, users, items, vals, n_users, n_items):
    """users/items/vals sorted by (user, item) -> SynthData with both indexes."""
    row_ptr = _ptr_from_sorted(users, n_users)
    if users.is_cuda and users.numel() > (1 << 30):
        # past ~1G ratings: the CSC from the device dual index (csrc/index.cu, exact; a torch argsort of the keys needs 4x the memory)
        from .ratings import csr_to_csc_device
        row_items, row_vals = items.to(torch.int32), vals.float()
        del users, items, vals
        col_ptr, col_users, col_vals = csr_to_csc_device(row_ptr, row_items, row_vals, n_users, n_items)
        return SynthData(name, n_users, n_items, row_ptr, row_items, row_vals, col_ptr, col_users, col_vals, spec)
    key2 = items.long() * n_users + users.long()
    order = torch.argsort(key2)
    col_ptr = _ptr_from_sorted(items[order], n_items)
    return SynthData(name, n_users, n_items, row_ptr, items.to(torch.int32), vals.float(), col_ptr,
                     users[order].to(torch.int32), vals[order].float(), spec)


def _truth_values(users, items, Ut, Vt, noise, gen, chunk=1 << 24):
    out = torch.empty(users.numel(), dtype=torch.float32, device=users.device)
    for lo in range(0, users.numel(), chunk):
        hi = min(lo + chunk, users.numel())
        u = Ut[users[lo:hi]]
        v = Vt[items[lo:hi]]
        t = (u * v).sum(1)
        t += noise * torch.randn(hi - lo, generator=gen, device=users.device)
        out[lo:hi] = t
    return out


def _bernoulli(name, spec, device, seed):
    g = torch.Generator(device=device).manual_seed(seed)
    nu, ni, p, r = spec["n_users"], spec["n_items"], spec["density"], spec["rank"]
    Ut = torch.randn(nu, r, generator=g, device=device)
    Vt = torch.randn(ni, r, generator=g, device=device)
    us, its = [], []
    step = max(1, (1 << 26) // ni)
    for lo in range(0, nu, step):
        hi = min(nu, lo + step)
        mask = torch.rand(hi - lo, ni, generator=g, device=device) < p
        u, i = torch.nonzero(mask, as_tuple=True)
        us.append(u + lo)
        its.append(i)
    users = torch.cat(us)
    items = torch.cat(its)
    vals = _truth_values(users, items, Ut, Vt, spec["noise"], g)
    return _finish(name, spec, users, items, vals, nu, ni)


def _powerlaw(name, spec, device, seed, nnz_target=None):
    g = torch.Generator(device=device).manual_seed(seed)
    nu, ni, r = spec["n_users"], spec["n_items"], spec["rank"]
    target = int(nnz_target or spec["nnz"])
    lo_c, hi_c = spec["min_count"], ni
    raw = torch.exp(spec["mu"] + spec["sigma"] * torch.randn(nu, generator=g, device=device, dtype=torch.float64))
    counts = raw.clamp(lo_c, hi_c)
    for _ in range(6):
        counts = (counts * (target / counts.sum())).clamp(lo_c, hi_c)
    counts = torch.floor(counts + torch.rand(nu, generator=g, device=device, dtype=torch.float64)).long()
    counts = counts.clamp(lo_c, hi_c)
    # Zipf(s) popularity over item ranks, ranks mapped to ids by a random permutation
    ranks = torch.arange(1, ni + 1, device=device, dtype=torch.float64)
    pmf = ranks.pow(-spec["zipf"])
    cdf = torch.cumsum(pmf, 0)
    cdf /= cdf[-1].clone()
    perm = torch.randperm(ni, generator=g, device=device)

    def draw(user_ids):
        u = torch.rand(user_ids.numel(), generator=g, device=device, dtype=torch.float64)
        k = torch.searchsorted(cdf, u).clamp_max(ni - 1)
        return perm[k]

    if target > (1 << 30):
        return _powerlaw_blocked(name, spec, device, g, counts, draw)
    users = torch.repeat_interleave(torch.arange(nu, device=device), counts)
    items = draw(users)
    for _ in range(8):
        key = torch.unique(users * ni + items)
        users, items = key // ni, key % ni
        have = torch.bincount(users, minlength=nu)
        deficit = (counts - have).clamp_min(0)
        need = int(deficit.sum())
        if need == 0:
            break
        extra_u = torch.repeat_interleave(torch.arange(nu, device=device), deficit * 2)
        users = torch.cat([users, extra_u])
        items = torch.cat([items, draw(extra_u)])
    key = torch.unique(users * ni + items)
    users, items = key // ni, key % ni
    # drop overshoot at random (random priority within each user), keep (user, item) order
    have = torch.bincount(users, minlength=nu)
    if bool((have > counts).any()):
        pri = torch.rand(users.numel(), generator=g, device=device)
        order = torch.argsort(users.double() * 2.0 + pri.double())
        users_o = users[order]
        start = torch.zeros(nu + 1, dtype=torch.int64, device=device)
        start[1:] = torch.cumsum(have, 0)
        pos = torch.arange(users_o.numel(), device=device) - start[users_o]
        keep = order[pos < counts[users_o]]
        keep, _ = torch.sort(keep)
        users, items = users[keep], items[keep]
    Ut = torch.randn(nu, r, generator=g, device=device)
    Vt = torch.randn(ni, r, generator=g, device=device)
    vals = _truth_values(users, items, Ut, Vt, spec["noise"], g)
    if spec.get("quantize"):
        z = vals / float(np.sqrt(r + spec["noise"] ** 2))
        vals = torch.clamp(torch.round((2.75 + z) * 2.0) / 2.0, 0.5, 5.0)
    return _finish(name, spec, users, items, vals, nu, ni)


def _powerlaw_blocked(name, spec, device, g, counts, draw):
    """The power-law construction of _powerlaw over blocks of users (each block's
    draws stay far below torch's 2^31-element sort limit): per block, draw,
    dedupe, top up deficits, then drop overshoot at random -- the same steps,
    block-local (every step is per user, so blocks are independent)."""
    nu, ni, r = spec["n_users"], spec["n_items"], spec["rank"]
    us, its = [], []
    cum = torch.cumsum(counts, 0)
    lo = 0
    while lo < nu:
        base = int(cum[lo - 1]) if lo else 0
        hi = int(torch.searchsorted(cum, torch.tensor(base + (1 << 28), device=device, dtype=cum.dtype)))
        hi = min(nu, max(hi, lo + 1))
        c = counts[lo:hi]
        n = hi - lo
        users = torch.repeat_interleave(torch.arange(n, device=device), c)
        items = draw(users)
        for _ in range(8):
            key = torch.unique(users * ni + items)
            users, items = key // ni, key % ni
            have = torch.bincount(users, minlength=n)
            deficit = (c - have).clamp_min(0)
            if int(deficit.sum()) == 0:
                break
            extra_u = torch.repeat_interleave(torch.arange(n, device=device), deficit * 2)
            users = torch.cat([users, extra_u])
            items = torch.cat([items, draw(extra_u)])
        key = torch.unique(users * ni + items)
        users, items = key // ni, key % ni
        have = torch.bincount(users, minlength=n)
        if bool((have > c).any()):
            pri = torch.rand(users.numel(), generator=g, device=device)
            order = torch.argsort(users.double() * 2.0 + pri.double())
            users_o = users[order]
            start = torch.zeros(n + 1, dtype=torch.int64, device=device)
            start[1:] = torch.cumsum(have, 0)
            pos = torch.arange(users_o.numel(), device=device) - start[users_o]
            keep = order[pos < c[users_o]]
            keep, _ = torch.sort(keep)
            users, items = users[keep], items[keep]
        us.append((users + lo).to(torch.int32))
        its.append(items.to(torch.int32))
        lo = hi
    users = torch.cat(us)
    items = torch.cat(its)
    del us, its
    Ut = torch.randn(nu, r, generator=g, device=device)
    Vt = torch.randn(ni, r, generator=g, device=device)
    vals = _truth_values(users, items, Ut, Vt, spec["noise"], g)
    return _finish(name, spec, users, items, vals, nu, ni)


def generate(name, device="cuda", seed=0, nnz_target=None, **overrides):
    """Generate config `name` (optionally scaled by overrides such as
    n_users / n_items / nnz) on `device`."""
    spec = dict(CONFIGS[name])
    spec.update(overrides)
    device = torch.device(device)
    if spec["kind"] == "bernoulli":
        return _bernoulli(name, spec, device, seed)
    return _powerlaw(name, spec, device, seed, nnz_target)
