#!/usr/bin/env python
"""Round timeline of the dense tensor-core kernel (K3) from a timing-only build.

Build with HOPF_EXTRA_NVCC_FLAGS=-DHOPF_TC3_TRACE (clock64 stamps of rounds 200..215 of CTA 0,
dense_tc3.cu), run one C4 evaluation, print per-round cycle offsets relative to the MMA
completion the epilogue waited for.  usage: python tools/tc3_trace.py [M]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1605_01799_b200 as hb  # noqa: E402
from paper_1605_01799_b200 import inputs  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
wl = inputs.config("c4", M=M)
X, t = inputs.points(wl, 0, M)
X = torch.as_tensor(X, dtype=torch.float32).cuda()
t = torch.as_tensor(t, dtype=torch.float32).cuda()
plan = hb.DensePlan(wl.Q, wl.Lam, wl.lam)
for _ in range(2):
    hb.eval_dense(X, t, plan, wl.gamma, wl.h, None, wl.max_iter, wl.tol)
torch.cuda.synchronize()
buf = np.zeros((16, 40), dtype=np.int64)
rc = hb.lib().hopf_tc3_trace_dump(ctypes.c_void_p(buf.ctypes.data))
assert rc == 0
names = {0: "mma:s0rdy", 1: "mma:s1rdy", 2: "mma:s2rdy", 3: "mma:s3rdy", 4: "mma:issued",
         8: "w0:red", 9: "w0:mmawake", 10: "w0:arr0", 11: "w0:arr1", 12: "w0:arr2", 13: "w0:arr3",
         14: "w0:end", 24: "w15:red", 25: "w15:mmawake", 26: "w15:arr0", 27: "w15:arr1",
         28: "w15:arr2", 29: "w15:arr3", 30: "w15:end"}
for r in range(1, 15):
    base = buf[r, 9]
    row = {v: int(buf[r, k] - base) for k, v in names.items()}
    period = int(buf[r + 1, 9] - buf[r, 9])
    print(f"round {200 + r}: period {period:5d} | " + " ".join(f"{k}={v}" for k, v in row.items()))
