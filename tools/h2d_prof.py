"""Host->device upload strategies for large numpy arrays (debug tool)."""
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 500_000_000
a = np.random.default_rng(0).random(n)  # float64, 4 GB
b = a.astype(np.float32)
torch.cuda.init()
cudart = torch.cuda.cudart()
for rep in range(2):
    t = time.perf_counter(); d = torch.from_numpy(a).to("cuda", torch.float32); torch.cuda.synchronize()
    print(f"f64 -> cuda f32 via .to: {time.perf_counter() - t:.3f}s", flush=True)
    t = time.perf_counter(); d = torch.from_numpy(b).to("cuda"); torch.cuda.synchronize()
    print(f"f32 pageable .to: {time.perf_counter() - t:.3f}s", flush=True)
    dst = torch.empty(n, dtype=torch.float32, device="cuda")
    src = torch.from_numpy(b)
    def cp(i, k=8):
        s = slice(i * n // k, (i + 1) * n // k)
        dst[s].copy_(src[s])
    t = time.perf_counter()
    with ThreadPoolExecutor(8) as ex:
        list(ex.map(cp, range(8)))
    torch.cuda.synchronize(); print(f"f32 pageable 8 threads: {time.perf_counter() - t:.3f}s", flush=True)
    t = time.perf_counter()
    rc = cudart.cudaHostRegister(b.ctypes.data, b.nbytes, 0)
    t1 = time.perf_counter()
    dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    cudart.cudaHostUnregister(b.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {t1 - t:.3f}s (rc {rc}) copy {t2 - t1:.3f}s unregister {t3 - t2:.3f}s", flush=True)
    t = time.perf_counter(); c = a.astype(np.float32); print(f"host astype {time.perf_counter() - t:.3f}s", flush=True)
