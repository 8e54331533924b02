#!/usr/bin/env python
"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  usage: compute-sanitizer --tool <t> python tools/sanitize_run.py [family...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1605_01799_b200 as hb  # noqa: E402
from paper_1605_01799_b200 import inputs  # noqa: E402

dev = lambda a: None if a is None else torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32).cuda()


def diag(name, M, n=None):
    wl = inputs.config(name, M=M, n=n)
    X, t = inputs.points(wl)
    t = t.copy(); t[0] = 0.0; t[1] = -1.0
    r = hb.eval_diag(dev(X), dev(t), dev(wl.D), dev(wl.c), wl.gamma, wl.h, dev(wl.w))
    torch.cuda.synchronize()
    return hb.last_kernel(), r


def union(M, want_y=True):
    wl = inputs.config("c5", M=M)
    X, t = inputs.points(wl)
    r = hb.eval_union(dev(X), dev(t), dev(wl.Dk), dev(wl.Ck), dev(wl.gammak), "l2", want_y=want_y)
    torch.cuda.synchronize()
    return hb.last_kernel(), r


def dense(M):
    wl = inputs.config("c4", M=M)
    X, t = inputs.points(wl)
    t = t.copy(); t[0] = 0.0
    plan = hb.DensePlan(wl.Q, wl.Lam)
    r = hb.eval_dense(dev(X), dev(t), plan, wl.gamma, "l1")
    torch.cuda.synchronize()
    return hb.last_kernel(), r


FAMILIES = {
    "tm": lambda: diag("c3", 600),                   # hopf_diag_tm_kernel (n = 1000)
    "tmg": lambda: diag("c2", 3000),                 # hopf_diag_tmg_kernel (n = 100, bulk rows)
    "reg": lambda: diag("c2", 3000, n=90),           # hopf_diag_kernel (n = 90: unaligned rows)
    "tmu": lambda: union(1200),                      # hopf_union_tmg_kernel (C5)
    "union_reg": lambda: diag("c1", 500),            # thread-per-point register kernel (n = 8)
    "dense": lambda: dense(1200),                    # hopf_dense_tc3_kernel + SIMT fix-up
}

if __name__ == "__main__":
    torch.cuda.set_device(0)
    names = sys.argv[1:] or list(FAMILIES)
    for nm in names:
        k, _ = FAMILIES[nm]()
        print(f"{nm}: {k} ok", flush=True)
