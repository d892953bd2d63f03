"""Host <-> device transfers of the fit's large arrays through pinned staging.

A pageable ``tensor.to("cuda")`` of a multi-GB numpy array runs at a fraction
of PCIe/C2C bandwidth (the driver stages it through small bounce buffers), and
a float64 -> float32 narrowing runs as a separate host pass first.  Here the
array moves in chunks: each chunk is narrowed straight into a pinned buffer
(one pass, torch's parallel host copy) while the previous chunk's async copy
runs on a copy stream; two pinned buffers from torch's caching host allocator
alternate, guarded by events.  Results go back the same way: the device widens
to float64 and the copy lands in pinned memory owned by the returned array.
"""

from __future__ import annotations

import numpy as np

_CHUNK_BYTES = 64 << 20


def upload(a, dtype, device):
    """numpy array (any dtype) -> contiguous device tensor of `dtype`."""
    import torch

    src = torch.from_numpy(np.ascontiguousarray(a)).reshape(-1)
    n = src.numel()
    out = torch.empty(n, dtype=dtype, device=device)
    if n == 0:
        return out.reshape(a.shape)
    esz = torch.empty(0, dtype=dtype).element_size()
    chunk = max(1, _CHUNK_BYTES // esz)
    if n <= chunk:
        return src.to(device=device, dtype=dtype).reshape(a.shape)
    bufs = [torch.empty(chunk, dtype=dtype, pin_memory=True) for _ in range(2)]
    done = [None, None]
    cur = torch.cuda.current_stream(device)
    cs = torch.cuda.Stream(device)
    cs.wait_stream(cur)  # `out` was allocated on the current stream
    for i, lo in enumerate(range(0, n, chunk)):
        hi = min(n, lo + chunk)
        b = i & 1
        if done[b] is not None:
            done[b].synchronize()  # the copy that last read this buffer finished
        bufs[b][:hi - lo].copy_(src[lo:hi])  # narrowing + staging in one host pass
        with torch.cuda.stream(cs):
            out[lo:hi].copy_(bufs[b][:hi - lo], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        done[b] = ev
    cur.wait_stream(cs)
    for e in done:
        if e is not None:
            e.synchronize()  # pinned buffers go back to the cache only when idle
    return out.reshape(a.shape)


def download_f64(t):
    """Device tensor -> float64 numpy array: widened on the device, copied out in chunks
    through two pinned staging buffers (torch's host allocator caches them across calls;
    pinning a result-sized buffer per call costs more than the copy itself: 0.31 s for the
    614 MB of the 500M config's factors) into an ordinary numpy array, the host copy of
    one chunk overlapping the device read of the next."""
    import torch

    d = t.to(torch.float64).contiguous().reshape(-1)
    n = d.numel()
    out = np.empty(tuple(t.shape), dtype=np.float64)
    if n == 0:
        return out
    dst = torch.from_numpy(out).reshape(-1)
    chunk = max(1, _CHUNK_BYTES // 8)
    if n <= chunk:
        dst.copy_(d)
        return out
    bufs = [torch.empty(chunk, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    cur = torch.cuda.current_stream(d.device)
    cs = torch.cuda.Stream(d.device)
    cs.wait_stream(cur)  # `d` was produced on the current stream
    spans = [(lo, min(n, lo + chunk)) for lo in range(0, n, chunk)]
    evs = [None, None]

    def start(i):
        lo, hi = spans[i]
        with torch.cuda.stream(cs):
            bufs[i & 1][:hi - lo].copy_(d[lo:hi], non_blocking=True)
            evs[i & 1] = torch.cuda.Event()
            evs[i & 1].record(cs)

    start(0)
    for i, (lo, hi) in enumerate(spans):
        evs[i & 1].synchronize()
        if i + 1 < len(spans):
            start(i + 1)  # the other buffer: its previous host copy finished in the last round
        dst[lo:hi].copy_(bufs[i & 1][:hi - lo])
    cur.wait_stream(cs)  # `d` is released on the current stream only after the reads
    return out
