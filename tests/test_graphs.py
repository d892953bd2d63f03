"""CUDA-graph replay of ALS iterations (CoreEngine.step, t >= 1): the replayed
iterations must equal the eager launches bit for bit (same kernels, same buffers,
fixed reduction trees), on both tiers, both loop orders and through fit_core,
including the convergence rewind that flips the factor buffers between graphs
(als.py:303-307)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected only on GPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2509_18024_b200 as cb  # noqa: E402
from paper_2509_18024_b200 import synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402


def _matrix(seed, n_u=700, n_i=400, p=0.08, long_items=3):
    rng = np.random.default_rng(seed)
    mask = rng.random((n_u, n_i)) < p
    mask[:, :long_items] = rng.random((n_u, long_items)) < 0.9  # tiled-tier rows at n_f >= 16
    u, i = np.nonzero(mask)
    v = rng.normal(size=u.size).astype(np.float32).astype(np.float64)
    return cb.RatingMatrix(u, i, v, n_users=n_u, n_items=n_i), rng


def _run(R, n_f, rate, lam, M0, iters, graphs, first="user"):
    eng = CoreEngine(R, n_f, rate, lam)
    eng.use_graphs = graphs
    U0 = np.zeros((R.n_users, n_f)) if first == "user" else np.random.default_rng(1).normal(0, 0.1, (R.n_users, n_f))
    eng.set_factors(U0, M0)
    terms = []
    for _ in range(iters):
        eng.step(first)
        if eng.iters_done > 1:
            terms.append(eng.terms(eng.iters_done - 2))
    eng.finish(first)
    terms.append(eng.terms(eng.iters_done - 1))
    torch.cuda.synchronize()
    return eng, terms


@pytest.mark.parametrize("n_f,rate,first", [(5, 0.3, "user"), (16, 0.2, "item"), (64, 0.1, "user")])
def test_graph_replay_equals_eager(n_f, rate, first):
    R, rng = _matrix(n_f)
    M0 = rng.normal(0, 0.1, (R.n_items, n_f)).astype(np.float32)
    e_eager, t_eager = _run(R, n_f, rate, 0.05, M0, 5, False, first)
    e_graph, t_graph = _run(R, n_f, rate, 0.05, M0, 5, True, first)
    assert len(e_graph._graphs) == 2, "both parities should have been captured and replayed"
    assert not e_graph._graph_failed
    assert torch.equal(e_eager.U_view, e_graph.U_view)
    assert torch.equal(e_eager.M_view, e_graph.M_view)
    for a, b in zip(t_eager, t_graph):
        assert a.rss == b.rss and a.pen == b.pen
        assert a.status_first == b.status_first and a.status_second == b.status_second


def test_fit_core_graphs_and_rewind():
    """fit_core replays graphs; a tol stop rewinds the buffers (the next parity's graph
    sees the flipped buffers) and still returns the converged iteration's factors."""
    d = synth.generate("small", device="cuda", seed=0)
    R = d.rating_matrix()
    M0 = synth.init_m(R.n_items, 5)
    cfg = cb.SolverConfig(method="core", n_f=5, lam=0.1, rate=0.3, max_iters=10, tol=1e-15)
    F, rep = cb.fit_core(R, cfg, init_m=M0)
    assert 0.0 <= rep.sketch_time <= rep.wall_clock_total
    eng = CoreEngine(R, 5, 0.3, 0.1)
    eng.use_graphs = False
    Fe, rep_e = cb.core._fit_gpu(R, cfg, cfg.rate, None, M0, False, eng)
    assert np.array_equal(rep.rmse_trace, rep_e.rmse_trace)
    assert np.array_equal(F.user_factors, Fe.user_factors) and np.array_equal(F.item_factors, Fe.item_factors)
    cfg2 = cb.SolverConfig(method="core", n_f=5, lam=0.1, rate=0.3, max_iters=30, tol=1e-3)
    F2, rep2 = cb.fit_core(R, cfg2, init_m=M0)
    assert rep2.converged and rep2.iters_run < 30
    assert np.isfinite(F2.user_factors).all() and np.isfinite(F2.item_factors).all()
