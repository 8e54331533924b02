"""Replay one fuzz case (normsq) and print the failing points: phi, iters on both sides."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import oracle
import paper_1605_01799_b200 as hb
import torch
seed = int(sys.argv[1])
rng = np.random.default_rng(seed)
kind = rng.choice(["diag", "diag", "union", "normsq", "ella", "dense", "distance", "maxh"])
lam = float(rng.choice([1.0, 1.0, 0.5, 2.0])); M = int(rng.integers(1, 400))
n = int(rng.integers(1, 65)); j = str(rng.choice(["l1sq", "linfsq"])); h = str(rng.choice(["l1", "wl1", "l2", "linf"]))
w = rng.uniform(0.5, 1.5, n).astype(np.float32) if h == "wl1" else None
X = rng.uniform(-10, 10, (M, n)).astype(np.float32)
t = rng.uniform(0, 10, M).astype(np.float32)
print("case", lam, M, n, j, h)
d = lambda a: None if a is None else torch.as_tensor(a).cuda()
for mi in (1000, 20000):
    g = hb.eval_normsq(d(X), d(t), j, 0.0, h, d(w), lam=lam, max_iter=mi)
    o = oracle.eval_normsq(X, t, j, 0.0, h, w, lam=lam, max_iter=mi)
    pg, gg, ig = (a.cpu().numpy() for a in g)
    dphi = np.abs(pg - o[0]) / np.maximum(1, np.abs(o[0]))
    idx = np.argsort(-dphi)[:6]
    print("max_iter", mi, hb.last_kernel())
    for i in idx:
        print(f"  pt {i}: t={t[i]:.4g} phi_g={pg[i]:.6g} phi_o={o[0][i]:.6g} rel={dphi[i]:.3g} it_g={ig[i]} it_o={o[2][i]}")
