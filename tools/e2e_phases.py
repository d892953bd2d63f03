"""Phase timing of the e2e fit_core path on the large config (debug tool).

Synchronises at phase boundaries, so the sum exceeds the overlapped e2e wall;
it shows what each phase costs on its own."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_2509_18024_b200 as cb
from paper_2509_18024_b200 import synth, engine as E

cfgname = sys.argv[1] if len(sys.argv) > 1 else "large"
d = synth.generate(cfgname, device="cuda")
spec = synth.CONFIGS[cfgname]
t = time.perf_counter(); R = d.rating_matrix(); print(f"host RatingMatrix (not timed in e2e) {time.perf_counter()-t:.3f}s", flush=True)
M0 = synth.init_m(R.n_items, spec["n_f"])

def timed(name, fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{name:40s} {time.perf_counter() - t:.3f}s", flush=True)
    return r

orig = E.DeviceSide.__init__
def patched(self, *a, **k):
    torch.cuda.synchronize(); t = time.perf_counter(); orig(self, *a, **k); torch.cuda.synchronize()
    print(f"  DeviceSide({self.n_rows} rows) {time.perf_counter() - t:.3f}s", flush=True)
E.DeviceSide.__init__ = patched
for rep in range(2):
    print("--- rep", rep)
    eng = timed("CoreEngine()", lambda: E.CoreEngine(R, spec["n_f"], spec["rate"], spec["lam"]))
    timed("set_factors", lambda: eng.set_factors(None, M0))
    timed("user side", lambda: eng.user)
    timed("item side (device CSC)", lambda: eng.item)
    timed("ssq", lambda: eng.ssq)
    for i in range(2):
        timed(f"step {i}", lambda: eng.step("user"))
    timed("finish+terms", lambda: (eng.finish("user"), eng.terms(eng.iters_done - 1)))
    timed("factors_host", lambda: eng.factors_host())
    cfg = cb.SolverConfig(method="core", n_f=spec["n_f"], lam=spec["lam"], rate=spec["rate"], max_iters=5, tol=1e-15)
    timed("fit_core 5 iters (e2e)", lambda: cb.fit_core(R, cfg, init_m=M0))
    del eng
