#!/usr/bin/env python
"""Benchmark: observed ratings processed per second per core-elements ALS
iteration (BASELINE.json metric) on 1..8 B200s.

A "step" is one full ALS iteration of fit_core over the workload: the user
half-sweep, its all-gather (N > 1), the item half-sweep with the fused
residual, its all-gather, and the objective terms (rss + penalty) read back
to the host -- exactly what fit_core does per iteration.  value = nnz * K / T
with T the max over ranks of the CUDA-event time of the K timed steps; inputs
are device resident and L2 is flushed (a 512 MiB write) before every timed
step, outside its events.

Extra keys: roofline (dominant kernel, algorithmic bytes / its event-timed
duration vs the measured HBM copy bandwidth), cpu_baseline (the float64 C
oracle port on one host core, bounded sample), e2e (fit_core through the
public API from host numpy arrays, copies included), clocks, gpu_launches.

--impl reference times the reference algorithm's CPU path (the oracle port;
the reference itself is Python+numba and does not travel to the GPU box) with
all host threads on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CONFIG = "large"
METRIC = "observed ratings processed/sec per ALS iteration"
UNIT = "ratings/s/iter"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 5 for large, more on the small configs so the timed region "
                         "lasts long enough for the clock sampler: DEFAULT_STEPS)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--method", default="core", choices=["core", "full", "fast_core"],
                    help="estimator (core = the BASELINE metric; full / fast_core for comparison lines)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    if args.steps is None:  # the CPU arm's steps are bounded samples of seconds each: 5 everywhere
        args.steps = DEFAULT_STEPS.get(args.config, 5) if args.impl == "ours" else 5
    return args


# default timed steps per workload: the small configs take 0.2-20 ms per iteration, and nvidia-smi
# delivers a sample every ~20 ms, so their timed region is stretched to ~1 s of iterations
DEFAULT_STEPS = {"small": 2000, "medium": 300, "powerlaw": 50, "large": 5, "wide": 2}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.perf_counter()  # nvidia-smi needs a few hundred ms to deliver its first sample
            while not self.samples and time.perf_counter() - t0 < 3.0:
                time.sleep(0.01)
            self.samples.clear()  # keep only samples taken while the timed region runs
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for s in self.samples for j in range(4) if s[2 + j].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def algorithmic_bytes(counts, n_f):
    """each observed rating gathers its fp32 factor row plus int32
    index and fp32 value; each solved row reads its pointer and writes its row."""
    counts = np.asarray(counts, np.int64)
    act = counts > 0
    return float(counts.sum() * (4 * n_f + 8) + act.sum() * (4 * n_f + 8))


def tier_bytes(side, n_f):
    c = side.counts
    small = algorithmic_bytes(c[side.small_host], n_f) if side.small_host.size else 0.0
    big = algorithmic_bytes(c[side.big_host], n_f) if side.big_host.size else 0.0
    return small, big


def measured_compute_peaks():
    """Microbenchmarked compute peaks of this pool's B200s (tools/peaks.cu ->
    profiles/r02_peaks.json): FFMA2 fp32, DFMA fp64, tcgen05 kind::i8."""
    p = os.path.join(ROOT, "profiles", "r02_peaks.json")
    if not os.path.exists(p):
        return {}
    with open(p) as fh:
        d = json.load(fh)
    return {"ffma2_tflops": d.get("ffma2_tflops"), "dfma_tflops": d.get("dfma_tflops"),
            "i8_tops": (d.get("i8_ss_m128_n256") or {}).get("tops")}


def compute_terms(core, n_f, prof, steps):
    """Pipe utilisation of the contraction kernels next to the HBM term: the
    tensor-core Gram's executed int8 MMA work (3 MMAs of M=128 N=144 K=32 per 32
    slice rows of the tiled tier) and its algorithmic Gram flops (2 n_f (n_f + 1)
    s_i per row), and the solve's LU flops (2/3 n_f^3 per row) on FFMA."""
    peaks = measured_compute_peaks()
    out = {"peaks_measured": peaks}
    ks, alg = 0, 0.0
    n_sys = 0
    for side in (core.user, core.item):
        c = side.counts
        big = side.big_host
        if big.size:
            ks += int(((c[big] + 31) // 32).sum())
            b = side.budget_host[big].astype(np.float64)
            alg += float((2.0 * n_f * (n_f + 1) * b).sum())
        n_sys += int((c > 0).sum())
    tc = prof.get("big_gram_tc_kernel")
    if tc and tc[1] > 0 and ks:
        ops = ks * 3 * 2 * 128 * 144 * 32 * steps
        t = tc[1] / 1e3
        out["big_gram_tc_kernel"] = {
            "pipe": "tensor (tcgen05 kind::i8)", "executed_tops": ops / t / 1e12,
            "peak_tops": peaks.get("i8_tops"),
            "frac": (ops / t / 1e12 / peaks["i8_tops"]) if peaks.get("i8_tops") else None,
            "algorithmic_tflops": alg * steps / t / 1e12,
            "note": "dense digit MMAs (1/rate x the sketched work, 4 int8 levels); algorithmic = sparse float64 Gram"}
    sv = prof.get("solve_kernel")
    if sv and sv[1] > 0:
        fl = n_sys * (2.0 / 3.0 * n_f ** 3 + 2.0 * n_f ** 2) * steps
        out["solve_kernel"] = {"pipe": "fp32 FMA (SIMT)", "achieved_tflops": fl / (sv[1] / 1e3) / 1e12,
                               "peak_tflops": peaks.get("ffma2_tflops"),
                               "frac": (fl / (sv[1] / 1e3) / 1e12 / peaks["ffma2_tflops"])
                               if peaks.get("ffma2_tflops") else None}
    return out


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def stratified_cpu_rate(R, spec, M0, threads, seconds, seed=0, n_strata=8):
    """Time the reference algorithm's CPU path (the float64 C oracle port) on a bounded
    sample of one full iteration and extrapolate to the whole workload.

    Per side, rows (n > 0) are ordered by length and cut into n_strata strata holding
    equal shares of the ratings; each stratum gets an equal slice of the time budget,
    its largest rows first (so every side's giant rows are in the sample: one per
    thread in stratum 0) and then random rows of the stratum.  The side's time is
    sum_s nnz_s * (t_s / sampled_nnz_s).  Returns (ratings/s/iter, details)."""
    import oracle

    n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
    rng = np.random.default_rng(seed)
    # the item half-sweep's source: user rows as a user half-sweep leaves them (nonzero; an
    # all-zero source would make every key tie and the reference's quickselect quadratic)
    U = np.random.default_rng(12345).normal(0.0, 0.3, (R.n_users, n_f)).astype(np.float32).astype(np.float64)
    M = M0.astype(np.float64)
    est_s, wall, sampled = 0.0, 0.0, 0
    per_stratum = seconds / (2.0 * n_strata)
    for side in ("user", "item"):
        ptr, idx, val = (R.row_ptr, R.row_items, R.row_vals) if side == "user" else (R.col_ptr, R.col_users, R.col_vals)
        src, tgt = (M, U.copy()) if side == "user" else (U, M.copy())
        counts = np.diff(ptr)
        order = np.argsort(-counts, kind="stable")
        order = order[counts[order] > 0].astype(np.int32)
        cum = np.cumsum(counts[order])
        total = int(cum[-1]) if cum.size else 0
        cuts = np.searchsorted(cum, np.linspace(0, total, n_strata + 1)[1:-1], side="right")
        bounds = [0, *[int(c) for c in cuts], order.size]
        for s in range(n_strata):
            lo, hi = bounds[s], bounds[s + 1]
            if hi <= lo:
                continue
            rows_s = order[lo:hi]
            head = rows_s[:threads]
            tail = rng.permutation(rows_s[threads:])
            seq = np.concatenate([head, tail])
            nnz_s = int(counts[rows_s].sum())
            done, t_s, pos = 0, 0.0, 0
            chunk = max(threads, 1)
            while pos < seq.size and (t_s < per_stratum or done == 0):
                sl = seq[pos:pos + chunk]
                t0 = time.perf_counter()
                oracle.core_half_sweep(ptr, idx, val, src, n_f, lam, rate, tgt, want_rss=(side == "item"), rows=sl,
                                       threads=threads)
                t_s += time.perf_counter() - t0
                done += int(counts[sl].sum())
                pos += sl.size
                chunk = min(chunk * 2, 64 * max(threads, 1))
            est_s += nnz_s * (t_s / done)
            print(f"  [cpu sample] {side} stratum {s}: {done} of {nnz_s} ratings in {t_s:.2f} s", file=sys.stderr,
                  flush=True)
            wall += t_s
            sampled += done
    value = float(len(R.row_vals)) / est_s if est_s > 0 else 0.0
    return value, {"estimated_s_per_iter": est_s, "sample_wall_s": wall, "sampled_ratings": sampled,
                   "strata": n_strata}


def cpu_baseline_port(data_host, spec, M0, seconds):
    """The float64 C oracle (a restatement of the reference algorithm) on ONE host core,
    on a stratified sample of one iteration (stratified_cpu_rate)."""
    value, det = stratified_cpu_rate(data_host, spec, M0, 1, seconds)
    return {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "cpu_model": cpu_model(),
            "sample": (f"nnz-stratified row sample of one user + one item half-sweep (8 strata per side, largest rows "
                       f"first), {det['sampled_ratings']} slice ratings in {det['sample_wall_s']:.1f} s measured; "
                       f"float64 C oracle port, 1 thread; extrapolated {det['estimated_s_per_iter']:.0f} s per "
                       f"iteration")}


def run_reference(args):
    """--impl reference: the reference algorithm's CPU path (the float64 C oracle port; the
    reference itself is Python+numba and does not travel to the GPU box) with all host
    threads; each step is a bounded nnz-stratified sample of one full iteration
    (stratified_cpu_rate), extrapolated to the whole workload (labelled as such)."""
    import torch

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2509_18024_b200 import synth

    spec = dict(synth.CONFIGS[args.config])
    data = synth.generate(args.config, device="cuda" if torch.cuda.is_available() else "cpu")
    R = data.rating_matrix()
    M0 = synth.init_m(R.n_items, spec["n_f"]).astype(np.float64)
    threads = os.cpu_count() or 1
    n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
    budget = max(8.0, 120.0 / max(args.steps + args.warmup, 1))
    rates, walls, ests, sampled = [], [], [], []
    for step in range(args.warmup + args.steps):
        v, det = stratified_cpu_rate(R, spec, M0, threads, budget, seed=step)
        if step >= args.warmup:
            rates.append(v)
            walls.append(det["sample_wall_s"])
            ests.append(det["estimated_s_per_iter"])
            sampled.append(det["sampled_ratings"])
    value = float(np.median(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": data.nnz / value * 1e3,
        "ms_per_step_is": "extrapolated from the stratified sample (see cpu_baseline)",
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "nnz": data.nnz, "n_users": R.n_users, "n_items": R.n_items,
                   "n_f": n_f, "lam": lam, "rate": rate},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
                         "sample": (f"per step an nnz-stratified row sample of both half-sweeps (8 strata per side, "
                                    f"largest rows first), {budget:.0f} s budget of {threads}-thread float64 C "
                                    f"oracle work; measured sample wall {np.median(walls):.1f} s over "
                                    f"{int(np.median(sampled))} ratings per step, extrapolated "
                                    f"{np.median(ests):.1f} s per full iteration")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


T_START = time.perf_counter()


def phase(msg):
    """Progress on stderr (the JSON line stays the only stdout)."""
    print(f"[bench {time.perf_counter() - T_START:7.1f}s] {msg}", file=sys.stderr, flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # CALS_BENCH_BACKEND=gloo: functional check of the N > 1 code path with several ranks on one
    # device (host-staged exchange); never a measurement -- the line is tagged "functional_only"
    backend = os.environ.get("CALS_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2509_18024_b200 import _lib, synth
    from paper_2509_18024_b200.engine import CoreEngine
    from paper_2509_18024_b200.shard import ShardedEngine

    spec = dict(synth.CONFIGS[args.config])
    n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
    t_gen = time.perf_counter()
    data = synth.generate(args.config, device=dev, seed=0)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    M0 = synth.init_m(data.n_items, n_f)
    phase(f"generated {args.config}")
    index_line = device_index_check(data, dev)
    phase("device index checked")
    eff_rate = 1.0 if args.method == "full" else rate  # full ALS = complete budgets on every row
    eng = (ShardedEngine(data, n_f, eff_rate, lam, rank, world, device=dev, fast=args.method == "fast_core")
           if world > 1 else CoreEngine(data, n_f, eff_rate, lam, device=dev, fast=args.method == "fast_core"))
    eng.set_factors(np.zeros((data.n_users, n_f), np.float32), M0)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    for _ in range(args.warmup):
        eng.step("user")
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream(dev)
    times = []
    # timed steps run as the fit runs them: iterations t >= 1 replay a CUDA graph per parity
    # (CoreEngine.step; the sharded engine stays eager) -- captured here, before the timed region
    eng.step("user")
    eng.step("user")
    torch.cuda.synchronize()
    graphs = len(getattr(eng, "_graphs", {}))
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng.step("user")  # iteration t, its first half fusing the residual of t-1
            terms = eng.terms(eng.iters_done - 2)  # the host read fit_core does every iteration
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    # per-kernel event times (roofline, launch count) from the same number of eager steps right
    # after the timed ones: profile scopes record events around every launch, so they are kept
    # out of the timed region
    _lib.profile_enable(True)
    _lib.profile_collect()
    use_graphs = getattr(eng, "use_graphs", False)
    eng.use_graphs = False
    for _ in range(args.steps):
        flush.fill_(1)
        eng.step("user")
        eng.terms(eng.iters_done - 2)
    torch.cuda.synchronize()
    eng.use_graphs = use_graphs
    prof = _lib.profile_collect()
    _lib.profile_enable(False)
    total_ms = float(sum(times))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    nnz = data.nnz
    value = nnz * args.steps / (total_ms / 1e3)

    e2e_line = None
    if not args.no_e2e:
        # a whole fit of the workload as its config states it (large: 10 iterations), from host arrays
        phase("timed steps done; e2e fit")
        e2e_line = e2e(data, spec, M0, spec["iters"], rank, world, args.method)
        phase("e2e done")
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    hbm, peak_kind = measured_peaks()
    core = eng  # ShardedEngine is a CoreEngine restricted to this rank's rows
    sb_u, bb_u = tier_bytes(core.user, n_f)
    sb_i, bb_i = tier_bytes(core.item, n_f)
    kbytes = {"small_gram_kernel": (sb_u + sb_i) * args.steps, "big_gram_kernel": (bb_u + bb_i) * args.steps,
              "big_gram_tc_kernel": (bb_u + bb_i) * args.steps, "big_scan2_kernel": (bb_u + bb_i) * args.steps,
              "fast_gram_kernel": (bb_u + bb_i) * args.steps}
    dom = max(prof.items(), key=lambda kv: kv[1][1]) if prof else ("none", (0, 0.0))
    dom_name, (dom_cnt, dom_ms) = dom
    dom_bytes = kbytes.get(dom_name)
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_bytes and dom_ms > 0 else None
    b_iter = algorithmic_bytes(np.diff(data.row_ptr.cpu().numpy()), n_f) + algorithmic_bytes(
        np.diff(data.col_ptr.cpu().numpy()), n_f)
    gpu_launches = sum(c for c, _ in prof.values())
    compute = compute_terms(core, n_f, prof, args.steps)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get(args.config, {}).get(dom_name, {}).get("dram_bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": args.config, "method": args.method, "nnz": nnz, "n_users": data.n_users,
                   "n_items": data.n_items,
                   "n_f": n_f, "lam": lam, "rate": rate, "parallelism": f"row-shard x{world}",
                   "l2": "512 MiB flush before every timed step (outside its events)",
                   "init": "M0 ~ N(0, 0.1^2) numpy seed 0, fp32; U0 = 0"},
        "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
                     "alg_bytes_per_launch": (dom_bytes / dom_cnt) if dom_bytes and dom_cnt else None,
                     "peak_kind": peak_kind,
                     "launches": dom_cnt, "kernel_ms_total": dom_ms,
                     "step_alg_bytes": b_iter,
                     "step_frac": (b_iter / (hbm * 1e9)) / (total_ms / 1e3 / args.steps),
                     "compute": compute},
        "kernels": {k: {"launches": c, "ms": ms} for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1])},
        "gpu_launches": gpu_launches,
        "cuda_graphs": {"replayed": graphs > 0, "graphs": graphs,
                        "note": "timed iterations replay one captured graph per parity; kernel times and the "
                                "launch count come from as many eager steps run after the timed region"},
        "clocks": clk.summary(),
        "rmse_prev_iter": float(np.sqrt(terms.rss / core.ssq)),
        "setup_s": {"generate": t_gen},
        "device_index": index_line,
    }
    if not args.no_cpu and world == 1:
        R_host = data.rating_matrix()
        phase("cpu baseline")
        line["cpu_baseline"] = cpu_baseline_port(R_host, spec, M0, args.cpu_seconds)
        phase("cpu baseline done")
    else:
        line["cpu_baseline"] = None
    if e2e_line is not None:
        line["e2e"] = e2e_line
    if backend != "nccl":
        line["functional_only"] = f"{backend} backend, ranks share a device: not a measurement"
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    print(json.dumps(line), flush=True)


def device_index_check(data, dev):
    """The dual index built on the device (csrc/index.cu) from the workload's
    CSR: its time, and that it equals the generator's CSC exactly (a full-size
    parity property of ratings.py:86-92)."""
    import torch

    from paper_2509_18024_b200.ratings import csr_to_csc_device

    csr_to_csc_device(data.row_ptr, data.row_items, data.row_vals, data.n_users, data.n_items)  # warm
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cp, ci, cv = csr_to_csc_device(data.row_ptr, data.row_items, data.row_vals, data.n_users, data.n_items)
    e1.record()
    torch.cuda.synchronize()
    same = bool(torch.equal(cp, data.col_ptr) and torch.equal(ci, data.col_users) and torch.equal(cv, data.col_vals))
    del cp, ci, cv
    # COO (shuffled) -> CSR, the RatingMatrix constructor's sort (ratings.py:74-82)
    from paper_2509_18024_b200.ratings import coo_to_csr_device

    users = torch.repeat_interleave(torch.arange(data.n_users, device=dev, dtype=torch.int32),
                                    data.row_ptr[1:] - data.row_ptr[:-1])
    perm = torch.randperm(data.nnz, device=dev, generator=torch.Generator(device=dev).manual_seed(5))
    ku, ki, kv = users[perm], data.row_items[perm], data.row_vals[perm]
    del users, perm
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    rp, ri, rv, dup = coo_to_csr_device(ku, ki, kv, data.n_users, data.n_items)
    e3.record()
    torch.cuda.synchronize()
    same_csr = dup is None and bool(torch.equal(rp, data.row_ptr) and torch.equal(ri, data.row_items)
                                    and torch.equal(rv, data.row_vals))
    del ku, ki, kv, rp, ri, rv
    torch.cuda.empty_cache()
    return {"csr_to_csc_ms": e0.elapsed_time(e1), "equals_reference_order": same,
            "ratings_per_s": data.nnz / (e0.elapsed_time(e1) / 1e3),
            "coo_to_csr_ms": e2.elapsed_time(e3), "coo_equals_reference_order": same_csr}


E2E_FITS = 3  # timed whole fits of the e2e leg (median reported)


def e2e(data, spec, M0, steps, rank=0, world=1, method="core"):
    """fit_core through the public API from host (numpy) arrays: H2D of the
    CSR and the init, `steps` iterations (the config's own count), D2H of both
    factor matrices.
    With N > 1 ranks every rank runs fit_core on its row shard (ShardedEngine,
    NCCL all-gather per half-sweep); wall = max over ranks."""
    import warnings

    import torch
    import torch.distributed as dist

    import paper_2509_18024_b200 as cb
    from paper_2509_18024_b200.shard import ShardedEngine

    R = data.rating_matrix()
    rate = 1.0 if method == "full" else spec["rate"]
    cfg = cb.SolverConfig(method=method, n_f=spec["n_f"], lam=spec["lam"], rate=rate, max_iters=steps, tol=1e-15)
    cfg1 = cb.SolverConfig(method=method, n_f=spec["n_f"], lam=spec["lam"], rate=rate, max_iters=1, tol=1e-15)
    fit = {"core": cb.fit_core, "full": cb.fit, "fast_core": cb.fit_fast_core}[method]
    dev = torch.device("cuda", torch.cuda.current_device())

    def engine():
        if world == 1:
            return None  # the fit builds its own engine
        return ShardedEngine(R, spec["n_f"], rate, spec["lam"], rank, world, device=dev, fast=method == "fast_core")

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        fit(R, cfg1, init_m=M0, engine=engine())  # warm
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # three whole fits, each from the host arrays (nothing of a previous fit is reused: every fit
        # uploads, plans, iterates and copies back); the median wall is reported, all three are listed
        walls = []
        for _ in range(E2E_FITS):
            t0 = time.perf_counter()
            F, rep = fit(R, cfg, init_m=M0, engine=engine())  # sides (and their H2D) built inside
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            if world > 1:
                w = torch.tensor([wall], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
                dist.all_reduce(w, op=dist.ReduceOp.MAX)
                wall = float(w.item())
            walls.append(wall)
    wall = sorted(walls)[len(walls) // 2]
    nnz = R.n_entries
    n_f = spec["n_f"]
    # copied tensors: the CSR only (int64 pointers, int32 indices, values narrowed to fp32 by torch's
    # host-side conversion before the copy) -- the CSC is built on the device (csrc/index.cu) -- and the
    # fp32 item init (user rows start at zero on the device); back: float64 factors and 5 float64
    # objective terms per iteration (per rank at N > 1: each rank uploads the full CSR)
    h2d = (R.row_ptr.nbytes + nnz * 4 + nnz * 4 + R.n_items * n_f * 4) * world
    d2h = ((R.n_users + R.n_items) * n_f * 8 + rep.iters_run * 5 * 8) * world
    return {"value": nnz * rep.iters_run / wall, "unit": UNIT, "h2d_bytes_per_step": h2d / rep.iters_run,
            "d2h_bytes_per_step": d2h / rep.iters_run, "wall_s": wall, "wall_s_all_fits": walls,
            "iters": rep.iters_run,
            "how": f"paper_2509_18024_b200.{fit.__name__}(RatingMatrix of numpy arrays) incl. plan, H2D of the CSR "
                   "(pageable), the CSC built on the device beside the first user half-sweep, all iterations, D2H of float64 "
                   "factors; per-step bytes amortised over the fit; median wall of 3 fits" + (
                       f"; {world} ranks, ShardedEngine, max wall over ranks" if world > 1 else "")}


if __name__ == "__main__":
    main()
