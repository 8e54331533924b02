"""Randomised parity sweep (GPU vs the fp64 oracle) over the diag / union / NEXT entry points.

    python tools/fuzz_gpu.py [seconds]
Each case draws n, M, H kind, lambda, D, c, w, t (with zeros) at random and applies the parity
checks of tests/test_gpu_parity.py.  Prints one line per case; exits non-zero on a failure."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import oracle  # noqa: E402
import paper_1605_01799_b200 as hb  # noqa: E402
import test_gpu_parity as T  # noqa: E402


def case(rng):
    kind = rng.choice(["diag", "diag", "union", "normsq", "ella"])
    lam = float(rng.choice([1.0, 1.0, 0.5, 2.0]))
    M = int(rng.integers(1, 400))
    if kind == "diag":
        n = int(rng.integers(1, 1025))
        h = str(rng.choice(["l1", "wl1", "l2", "ell", "linf"]))
        D = rng.uniform(0.3, 3.0, n).astype(np.float32)
        c = rng.normal(size=n).astype(np.float32) if rng.random() < 0.5 else None
        w = rng.uniform(0.3, 2.0, n).astype(np.float32)
        X = (rng.normal(size=(M, n)) * rng.uniform(0.5, 4)).astype(np.float32)
        t = rng.uniform(0, 3, M).astype(np.float32)
        t[rng.random(M) < 0.05] = 0.0
        g = hb.eval_diag(T.dev(X), T.dev(t), T.dev(D), T.dev(c), -0.5, h, T.dev(w), lam=lam)
        o = oracle.eval_diag(X, t, D, c, -0.5, h, w, lam=lam)
        T.check(*g, *o, iters_slack=3, frac_exact=0.8 if M >= 50 else 0.0)
        return f"diag n={n} M={M} h={h} lam={lam}"
    if kind == "union":
        n = int(rng.integers(1, 257))
        K = int(rng.integers(1, 17))
        h = str(rng.choice(["l1", "wl1", "l2"]))
        Ck = (rng.standard_normal((K, n)) * 2).astype(np.float32)
        Dk = (rng.uniform(0.5, 2.0, (K, n)) ** 2).astype(np.float32)
        gk = np.full(K, -0.5, np.float32)
        w = rng.uniform(0.5, 1.5, n).astype(np.float32)
        X = (rng.standard_normal((M, n)) * 2).astype(np.float32)
        t = rng.uniform(0, 2, M).astype(np.float32)
        wy = h == "l2"
        r = hb.eval_union(T.dev(X), T.dev(t), T.dev(Dk), T.dev(Ck), T.dev(gk), h,
                          T.dev(w) if h == "wl1" else None, lam=lam, want_y=wy, want_phik=True)
        o = oracle.eval_union(X, t, Dk, Ck, gk, h, w if h == "wl1" else None, lam=lam, want_y=wy)
        T.check_union(r[0], r[1], r[2], r[3] if wy else None, r[4], r[5], o, t)
        return f"union n={n} K={K} M={M} h={h} lam={lam}"
    if kind == "normsq":
        n = int(rng.integers(1, 65))
        j = str(rng.choice(["l1sq", "linfsq"]))
        h = str(rng.choice(["l1", "wl1", "l2", "linf"]))
        w = rng.uniform(0.5, 1.5, n).astype(np.float32) if h == "wl1" else None
        X = rng.uniform(-10, 10, (M, n)).astype(np.float32)
        t = rng.uniform(0, 10, M).astype(np.float32)
        T.check_normsq(hb, X, t, j, h, w, lam=lam)
        return f"normsq n={n} M={M} J={j} h={h} lam={lam}"
    n = int(rng.integers(1, 129))
    B = rng.normal(size=(n, n))
    Q, _ = np.linalg.qr(B)
    A = (Q * rng.uniform(0.3, 3.0, n)) @ Q.T
    A = 0.5 * (A + A.T)
    D = rng.uniform(0.5, 2.0, n).astype(np.float32)
    X = (rng.normal(size=(M, n)) * 3).astype(np.float32)
    t = rng.uniform(0, 3, M).astype(np.float32)
    Qf, Lf = T._spectral(A)
    g = hb.eval_diag_A(T.dev(X), T.dev(t), T.dev(D), None, 0.0, T.dev(Qf), T.dev(Lf), lam=lam)
    o = oracle.eval_diag_A(X, t, D, None, 0.0, A, lam=lam)
    T.check(*g, *o, iters_slack=4, frac_exact=0.7 if M >= 50 else 0.0)   # fraction: a statistic
    return f"ellA n={n} M={M} lam={lam}"


if __name__ == "__main__":
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    rng = np.random.default_rng(int(time.time()) % 100000)
    t0, k = time.time(), 0
    while time.time() - t0 < secs:
        desc = case(rng)
        k += 1
        print("ok", desc, flush=True)
    print(f"fuzz: {k} cases passed")
