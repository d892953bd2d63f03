"""bench.py's N > 1 code path (torchrun, ShardedEngine, max-over-ranks timing,
sharded e2e) run functionally with two ranks on one device (gloo backend,
host-staged exchange): exits 0, prints one tagged line, and its objective
matches the single-rank run of the same config."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out):
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def test_bench_two_ranks_functional():
    env = dict(os.environ, CALS_BENCH_BACKEND="gloo")
    args = ["bench.py", "--config", "small", "--steps", "2", "--warmup", "3", "--no-cpu"]
    r2 = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                         "--master-addr", "127.0.0.1", "--master-port", "29541", *args, "--gpus", "2"],
                        cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r2.returncode == 0, r2.stderr[-3000:]
    two = _last_json(r2.stdout)
    r1 = subprocess.run([sys.executable, *args], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r1.returncode == 0, r1.stderr[-3000:]
    one = _last_json(r1.stdout)
    assert two["n_gpus"] == 2 and "functional_only" in two and "functional_only" not in one
    assert two["rmse_prev_iter"] == pytest.approx(one["rmse_prev_iter"], rel=1e-12)
    assert two["e2e"]["iters"] == one["e2e"]["iters"] == 10  # e2e: a whole fit of the config (small: 10 iterations)
