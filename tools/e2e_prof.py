import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
from paper_2509_18024_b200 import synth
import paper_2509_18024_b200 as cb
from paper_2509_18024_b200.engine import CoreEngine
d = synth.generate("large", device="cuda")
R = d.rating_matrix()
print("vals dtype", R.row_vals.dtype, R.row_items.dtype, flush=True)
torch.cuda.synchronize()
for rep in range(2):
    t = time.perf_counter()
    v = torch.from_numpy(R.row_vals).to(device="cuda", dtype=torch.float32); torch.cuda.synchronize()
    t1 = time.perf_counter()
    i = torch.from_numpy(R.row_items).to(device="cuda"); torch.cuda.synchronize()
    t2 = time.perf_counter()
    v32 = R.row_vals.astype(np.float32); t3 = time.perf_counter()
    print(f"vals f64->cuda f32 {t1-t:.3f}s  idx i32 {t2-t1:.3f}s  host astype f32 {t3-t2:.3f}s", flush=True)
t = time.perf_counter(); eng = CoreEngine(R, 64, 0.1, 0.02); torch.cuda.synchronize(); print("engine", time.perf_counter() - t, flush=True)
t = time.perf_counter(); M0 = synth.init_m(R.n_items, 64); eng.set_factors(np.zeros((R.n_users, 64)), M0); torch.cuda.synchronize(); print("set_factors", time.perf_counter() - t, flush=True)
t = time.perf_counter(); eng.step("user"); torch.cuda.synchronize(); print("step", time.perf_counter() - t, flush=True)
t = time.perf_counter(); U, M = eng.factors_host(); print("factors_host", time.perf_counter() - t, flush=True)
