"""Multi-process (world_size 2, gloo, CPU) test of the row-sharding host logic:
nnz-balanced partition + all-gather-v of the updated rows after each
half-sweep.  The per-rank compute is the CPU oracle restricted to the rank's
rows (the CUDA kernels need a GPU); the exchanged result must equal a
single-process half-sweep bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import csr_csc, load_golden
from paper_2509_18024_b200.shard import allgather_rows, nnz_balanced_ranges


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = load_golden("fit_medium.npz")
    n_f, lam, rate = int(g["n_f"]), float(g["lam"]), float(g["rate"])
    csr, csc = csr_csc(g["users"], g["items"], g["vals"], int(g["n_users"]), int(g["n_items"]))
    ur = nnz_balanced_ranges(csr[0], world)
    ir = nnz_balanced_ranges(csc[0], world)
    U = torch.zeros((int(g["n_users"]), n_f), dtype=torch.float64)
    M = torch.from_numpy(g["M0"].astype(np.float64).copy())
    rss_total = 0.0
    for side in ("user", "item"):
        ptr, idx, val = csr if side == "user" else csc
        src, tgt = (M, U) if side == "user" else (U, M)
        r0, r1 = (ur if side == "user" else ir)[rank]
        rows = np.arange(r0, r1, dtype=np.int32)
        t = tgt.numpy()
        rss, _, _ = oracle.core_half_sweep(ptr, idx, val, src.numpy(), n_f, lam, rate, t,
                                           want_rss=(side == "item"), rows=rows)
        allgather_rows(tgt, ur if side == "user" else ir, rank)
        if side == "item":
            r = torch.tensor([float(rss[r0:r1].sum())], dtype=torch.float64)
            dist.all_reduce(r)
            rss_total = float(r.item())
    if rank == 0:
        np.savez(out_path, U=U.numpy(), M=M.numpy(), rss=rss_total, ur=np.array(ur), ir=np.array(ir))
    dist.barrier()
    dist.destroy_process_group()


def test_nnz_balanced_ranges_cover_rows():
    ptr = np.concatenate([[0], np.cumsum(np.random.default_rng(0).integers(0, 50, 1000))])
    for world in (1, 2, 3, 8):
        rr = nnz_balanced_ranges(ptr, world)
        assert rr[0][0] == 0 and rr[-1][1] == 1000
        assert all(rr[q][1] == rr[q + 1][0] for q in range(world - 1))
        work = [(ptr[b] - ptr[a]) + (b - a) for a, b in rr]
        assert max(work) - min(work) <= 2 * 50 + 2


def test_two_rank_sharded_iteration_matches_single_process(tmp_path):
    out = str(tmp_path / "rank0.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    g = load_golden("fit_medium.npz")
    n_f, lam, rate = int(g["n_f"]), float(g["lam"]), float(g["rate"])
    csr, csc = csr_csc(g["users"], g["items"], g["vals"], int(g["n_users"]), int(g["n_items"]))
    U = np.zeros((int(g["n_users"]), n_f))
    M = g["M0"].astype(np.float64).copy()
    oracle.core_half_sweep(*csr, M, n_f, lam, rate, U)
    rss, _, _ = oracle.core_half_sweep(*csc, U, n_f, lam, rate, M, want_rss=True)
    assert got["ur"][0][1] == got["ur"][1][0]  # two non-empty contiguous shards
    np.testing.assert_array_equal(got["U"], U)
    np.testing.assert_array_equal(got["M"], M)
    assert float(got["rss"]) == pytest.approx(float(rss.sum()), rel=1e-12)
