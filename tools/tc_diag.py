"""Large config after `warm` iterations: the user half-sweep with the tensor-core Gram vs
the float64 SIMT Gram vs the oracle on a stratified row sample; source column stats."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_2509_18024_b200 import _lib, synth  # noqa: E402
from paper_2509_18024_b200.engine import CoreEngine  # noqa: E402
from test_full_size import sample_rows, sub_csr  # noqa: E402

cfg, warm = sys.argv[1], int(sys.argv[2])
traj = int(sys.argv[3]) if len(sys.argv) > 3 else 1  # Gram path of the warm-up trajectory
spec = synth.CONFIGS[cfg]
n_f, lam, rate = spec["n_f"], spec["lam"], spec["rate"]
d = synth.generate(cfg, device="cuda")
_lib.set_tuning(gram_path=traj)
eng = CoreEngine(d, n_f, rate, lam)
eng.set_factors(np.zeros((d.n_users, n_f), np.float32), synth.init_m(d.n_items, n_f))
for t in range(warm):
    eng.half("user")
    eng.half("item")
    st_u = eng.user.status.cpu().numpy()
    st_i = eng.item.status.cpu().numpy()
    print(f"iteration {t}: status counts user {np.bincount(st_u, minlength=3).tolist()} item "
          f"{np.bincount(st_i, minlength=3).tolist()}", flush=True)
M = eng.M_view.contiguous().float().cpu().numpy()
am = np.abs(M)
print("source M: col max", np.round(am.max(0)[:8], 4), "col median", np.round(np.median(am, 0)[:8], 5),
      "max/median ratio max", float((am.max(0) / np.maximum(np.median(am, 0), 1e-30)).max()), flush=True)
ptr = d.row_ptr.cpu().numpy()
cnt = np.diff(ptr)
rows = sample_rows(cnt, np.random.default_rng(11), n_longest=8, n_random=150, per_decile=8)
if len(sys.argv) > 4:
    rows = np.union1d(rows, np.array([int(x) for x in sys.argv[4].split(",")]))
sp, si, sv = sub_csr(ptr, d.row_items, d.row_vals, rows)
want = np.zeros((rows.size, n_f))
_, _, ko = oracle.core_half_sweep(sp, si, sv, M.astype(np.float64), n_f, lam, rate, want, want_keys=True,
                                  threads=os.cpu_count())
scale = np.maximum(np.abs(want).max(axis=1), 1e-2)
for path in (1, 0):
    _lib.set_tuning(gram_path=path)
    keys = torch.zeros((d.n_users, n_f), dtype=torch.int64, device="cuda")
    eng.half("user", thr_keys=keys)
    torch.cuda.synchronize()
    got = eng.U_view[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    eng.undo_half("user")
    gk = keys[torch.from_numpy(rows).cuda()].cpu().numpy().view(np.uint64)
    err = np.abs(got - want).max(axis=1) / scale
    worst = np.argsort(-err)[:5]
    print(f"path {'tc' if path == 0 else 'f64'}: keys equal {bool((gk == ko).all())}, max err {err.max():.2e}; "
          f"worst rows {rows[worst].tolist()} n {cnt[rows[worst]].tolist()} err {np.round(err[worst], 6).tolist()} "
          f"|w| {np.round(np.abs(want[worst]).max(1), 4).tolist()}", flush=True)
