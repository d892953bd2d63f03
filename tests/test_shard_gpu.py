"""The sharded engine end to end on real kernels: 2 and 3 ranks (gloo, host-staged
exchange) sharing cuda:0 run full iterations of ShardedEngine; the gathered
factors must equal a single-process CoreEngine run bit for bit (rows are
independent within a half-sweep, each computed by the same kernels), the
all-reduced objective terms must agree to fp64 rounding, and each rank must hold
only its shard of the index (~1/N of the CSR and CSC bytes)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _matrix():
    rng = np.random.default_rng(11)
    n_u, n_i = 4000, 700
    mask = rng.random((n_u, n_i)) < 0.03
    mask[:, :4] = rng.random((n_u, 4)) < 0.7  # long item rows: the tiled tier at n_f = 32
    u, i = np.nonzero(mask)
    v = (np.einsum("ef,ef->e", rng.normal(size=(n_u, 6))[u], rng.normal(size=(n_i, 6))[i])
         + 0.3 * rng.normal(size=u.size)).astype(np.float32).astype(np.float64)
    M0 = rng.normal(0, 0.1, (n_i, 32)).astype(np.float32)
    return u, i, v, n_u, n_i, M0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path, bytes_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2509_18024_b200 as cb
    from paper_2509_18024_b200.shard import ShardedEngine
    u, i, v, n_u, n_i, M0 = _matrix()
    R = cb.RatingMatrix(u, i, v, n_users=n_u, n_items=n_i)
    eng = ShardedEngine(R, 32, 0.2, 0.05, rank, world, device=torch.device("cuda", 0))
    eng.set_factors(np.zeros((n_u, 32)), M0)
    terms = [eng.iterate() for _ in range(2)]
    np.save(bytes_path.format(rank), np.array([eng.user.index_bytes(), eng.item.index_bytes()]))
    if rank == 0:
        U, M = eng.factors_host()
        np.savez(out_path, U=U, M=M, rss=[t.rss for t in terms], pen=[t.pen for t in terms])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_engine_matches_single_process(tmp_path, world):
    import paper_2509_18024_b200 as cb
    from paper_2509_18024_b200.engine import CoreEngine
    out = str(tmp_path / "rank0.npz")
    bpath = str(tmp_path / "bytes{}.npy")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out, bpath)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    got = np.load(out)
    u, i, v, n_u, n_i, M0 = _matrix()
    R = cb.RatingMatrix(u, i, v, n_users=n_u, n_items=n_i)
    eng = CoreEngine(R, 32, 0.2, 0.05)
    assert eng.item.plan.n_big > 0
    eng.set_factors(np.zeros((n_u, 32)), M0)
    terms = [eng.iterate() for _ in range(2)]
    U, M = eng.factors_host()
    np.testing.assert_array_equal(got["U"], U)
    np.testing.assert_array_equal(got["M"], M)
    np.testing.assert_allclose(got["rss"], [t.rss for t in terms], rtol=1e-12)
    np.testing.assert_allclose(got["pen"], [t.pen for t in terms], rtol=1e-12)
    # per-rank index: its shard only (nnz-balanced blocks; pointers add one entry per row)
    full = np.array([eng.user.index_bytes(), eng.item.index_bytes()], dtype=np.float64)
    per_rank = np.array([np.load(bpath.format(r)) for r in range(world)], dtype=np.float64)
    assert np.allclose(per_rank.sum(axis=0), full, rtol=0.01)
    assert (per_rank / full <= 1.0 / world + 0.1).all(), per_rank / full
