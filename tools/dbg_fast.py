import os, sys, warnings
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import numpy as np
import oracle, paper_2509_18024_b200 as cb
from conftest import load_golden, csr_csc
g = load_golden("fast_sparse_ties.npz")
R = cb.RatingMatrix(g["users"], g["items"], g["vals"], n_users=int(g["n_users"]), n_items=int(g["n_items"]))
n_f, lam, rate = int(g["n_f"]), float(g["lam"]), float(g["rate"])
print("golden obj", g["objN"], "rmse", g["rmseN"])
csr, csc = csr_csc(g["users"], g["items"], g["vals"], int(g["n_users"]), int(g["n_items"]))
U, M, rep = oracle.fit_fast_core(csr, csc, n_f, lam, rate, int(g["iters"]), 1e-15, np.zeros((R.n_users, n_f)), g["M0"])
print("oracle obj", rep.objective_trace, rep.rmse_trace)
cfg = cb.SolverConfig(method="fast_core", n_f=n_f, lam=lam, rate=rate, max_iters=int(g["iters"]), tol=1e-15)
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    F, rp = cb.fit_method(R, cfg, init_m=g["M0"])
print("gpu obj", rp.objective_trace, rp.rmse_trace)
print("U diff", np.abs(F.user_factors - g["UN"]).max(), "M diff", np.abs(F.item_factors - g["MN"]).max())
cfg1 = cb.SolverConfig(method="fast_core", n_f=n_f, lam=lam, rate=rate, max_iters=1, tol=1e-15)
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    F1, r1 = cb.fit_method(R, cfg1, init_m=g["M0"])
print("1-iter gpu", r1.objective_trace, "U1 diff", np.abs(F1.user_factors - g["U1"]).max())
