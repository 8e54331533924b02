"""Seeded synthetic workloads (BASELINE.json ``configs`` and the paper's protocol).

This module holds only random-number generation and the config table — none of
the method's arithmetic.  Both the product path (bench, GPU tests) and the fp64
oracle consume the buffers it returns, so they see identical fp32 inputs.

Counter-style chunking: point rows are generated in fixed chunks of
``CHUNK`` points, chunk ``j`` drawn from ``numpy.random.default_rng([seed, stream, j])``.
A rank that owns global rows [r0, r1) regenerates exactly the same values as a
single process would, for any world size.

Laws (BASELINE.json configs; readings R15/R16 in DESIGN.md):
  C1  n=8,    M=1024,  X~U[-3,3],  t~U[0.1,2], D=1, c=0, gamma=0,  H=l1
  C2  n=100,  M=1e6,   X~N(0,4I),  t~U[0,1],   D_i=exp(U[ln1/2,ln2]), w_i~U[0.5,1.5], gamma=-1/2, H=wl1
  C3  n=1000, M=1e5,   X~N(0,I),   t~U[0,2],   D from the C2 law, gamma=-1/2, H=l2
  C4  n=256,  M=4e6,   X~N(0,I),   t~U[0.1,1], A=Q diag(Lam) Q^T, Q Haar, Lam~logU[0.1,10], gamma=0, H=l1
  C5  n=64, K=16, M=5e5, X~N(0,25I), t~U[0,2], c_k~N(0,25I), a_ki~U[0.5,2], D_k=a_k^2, gamma_k=-1/2, H=l2
  P   paper protocol: n in {4,8,12,16}, x~U[-10,10]^n, t~U[0,10],
      J=1/2||.||^2 (D=1) or 1/2<.,D^{-1}.> with D_ii = 1+(i-1)/(n-1), H in {l1, l2}
"""
from __future__ import annotations

import concurrent.futures as cf
import os
from dataclasses import dataclass, field

import numpy as np

CHUNK = 4096
SEED_BASE = 1605017990
_STREAM_X, _STREAM_T, _STREAM_PARAMS = 1, 2, 3


@dataclass
class Workload:
    """One configuration: problem parameters (fp32 where the GPU consumes them)."""
    name: str
    n: int
    M: int
    h: str                      # "l1" | "wl1" | "l2" | "ell" | "linf"
    kind: str                   # "diag" | "dense" | "union" | "distance" | "maxh" | "normsq"
    seed: int
    x_law: tuple                # ("uniform", lo, hi) | ("normal", std)
    t_law: tuple                # ("uniform", lo, hi)
    D: np.ndarray | None = None        # [n] f32 (diag)
    c: np.ndarray | None = None        # [n] f32 or None (diag)
    gamma: float = 0.0
    w: np.ndarray | None = None        # [n] f32 (wl1)
    Q: np.ndarray | None = None        # [n,n] f64 (dense)
    Lam: np.ndarray | None = None      # [n] f64 (dense)
    Dk: np.ndarray | None = None       # [K,n] f32 (union)
    Ck: np.ndarray | None = None       # [K,n] f32 (union)
    gammak: np.ndarray | None = None   # [K] f32 (union)
    lam: float = 1.0
    max_iter: int = 1000
    tol: float = 1e-8
    meta: dict = field(default_factory=dict)

    @property
    def K(self) -> int:
        return 0 if self.Dk is None else self.Dk.shape[0]


def _gen_chunk(seed, stream, j, rows, n, law):
    rng = np.random.default_rng([seed, stream, j])
    if law[0] == "uniform":
        a = rng.random((rows, n), dtype=np.float32)
        return (law[1] + (law[2] - law[1]) * a).astype(np.float32)
    return (rng.standard_normal((rows, n), dtype=np.float32) * np.float32(law[1]))


def _rows(seed, stream, law, n, r0, r1, out=None, threads=None):
    """Rows [r0, r1) of an M x n array drawn chunk-by-chunk (deterministic in r0, r1)."""
    if out is None:
        out = np.empty((r1 - r0, n), dtype=np.float32)
    if r1 <= r0:
        return out
    j0, j1 = r0 // CHUNK, (r1 - 1) // CHUNK + 1

    def job(j):
        a = _gen_chunk(seed, stream, j, CHUNK, n, law)
        lo, hi = max(r0, j * CHUNK), min(r1, (j + 1) * CHUNK)
        out[lo - r0:hi - r0] = a[lo - j * CHUNK:hi - j * CHUNK]

    nthreads = threads or min(16, os.cpu_count() or 1)
    if j1 - j0 == 1 or nthreads == 1:
        for j in range(j0, j1):
            job(j)
    else:
        with cf.ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(job, range(j0, j1)))
    return out


def points(wl: Workload, r0: int = 0, r1: int | None = None, out_x=None, out_t=None):
    """(X[r1-r0, n], t[r1-r0]) fp32 for global rows [r0, r1) of the workload."""
    r1 = wl.M if r1 is None else r1
    X = _rows(wl.seed, _STREAM_X, wl.x_law, wl.n, r0, r1, out_x)
    tt = _rows(wl.seed, _STREAM_T, wl.t_law, 1, r0, r1,
               None if out_t is None else out_t.reshape(-1, 1))
    return X, tt.reshape(-1)


def _loguniform(rng, lo, hi, size):
    return np.exp(rng.uniform(np.log(lo), np.log(hi), size))


def haar_orthogonal(rng, n):
    """Haar-random orthogonal Q: QR of a Gaussian with the signs of diag(R) folded in."""
    G = rng.standard_normal((n, n))
    Q, R = np.linalg.qr(G)
    return Q * np.sign(np.diag(R))


def config(name: str, M: int | None = None, n: int | None = None, seed: int | None = None,
           h: str | None = None) -> Workload:
    """Workload by name: c1..c5, or p<n>_<j>_<h> (paper protocol, j in {id, diag})."""
    name = name.lower()
    if name == "c1":
        n = n or 8
        wl = Workload("c1", n, M or 1024, h or "l1", "diag", seed or SEED_BASE + 1,
                      ("uniform", -3.0, 3.0), ("uniform", 0.1, 2.0),
                      D=np.ones(n, np.float32), gamma=0.0)
        return wl
    if name == "c2h":
        # NEXT-4: C2's J and points with H = min(sum w_j |p_j|, 1.2 ||p||_2, 0.8 ||p||_1)
        wl = config("c2", M=M, n=n, seed=seed)
        wl.name, wl.kind = "c2h", "maxh"
        wl.maxh = (["wl1", "l2", "l1"], np.array([1.0, 1.2, 0.8], np.float32),
                   np.stack([wl.w, np.ones_like(wl.w), np.ones_like(wl.w)]).astype(np.float32))
        return wl
    if name.startswith("t5") or name.startswith("t3") or name.startswith("t2"):
        # NEXT-3: the paper's Tables 2, 3 and 5 protocol: x ~ U[-10,10]^n,
        # t ~ U[0,10], lambda = 1, tol 1e-8.  t5[_n]: J = 1/2||.||_1^2, H = ||.||_inf (Table 5's
        # scaling setup, n = 16 by default); t3_<n>_<h>: J = 1/2||.||_1^2; t2_<n>_<h>:
        # J = 1/2||.||_inf^2
        body = name.split("_")
        n = n or (int(body[1]) if len(body) > 1 else 16)
        hh = h or (body[2] if len(body) > 2 else ("linf" if name.startswith("t5") else "l1"))
        wl = Workload(name, n, M or 1_000_000, hh, "normsq", seed or SEED_BASE + 200 + n,
                      ("uniform", -10.0, 10.0), ("uniform", 0.0, 10.0), gamma=0.0)
        wl.jk = "linfsq" if name.startswith("t2") else "l1sq"
        if hh == "wl1":
            wl.w = (1.0 + np.arange(n) / max(n - 1, 1)).astype(np.float32)   # the paper's D_ii
        return wl
    if name.startswith("t4a"):
        # NEXT-2, Table 4's ||y||_A column: J = 1/2<., D^{-1}.>,
        # D_ii = 1 + (i-1)/(n-1), H = sqrt(<p, A p>) with A_ii = 2, A_ij = 1; x ~ U[-10,10]^n,
        # t ~ U[0,10].  t4a[_n], n = 16 by default.
        body = name.split("_")
        n = n or (int(body[1]) if len(body) > 1 else 16)
        D = (1.0 + np.arange(n) / max(n - 1, 1)).astype(np.float32)
        wl = Workload(name, n, M or 1_000_000, "A", "ella", seed or SEED_BASE + 300 + n,
                      ("uniform", -10.0, 10.0), ("uniform", 0.0, 10.0), D=D, gamma=0.0)
        wl.A = np.ones((n, n)) + np.eye(n)
        return wl
    if name == "c2e":
        # NEXT-2: C2's J and points with H(p) = sqrt(<p, diag(w) p>), w = C2's weights
        wl = config("c2", M=M, n=n, seed=seed, h="ell")
        wl.name = "c2e"
        return wl
    if name == "c2i":
        # NEXT-2: C2's J and points with H(p) = ||p||_inf
        wl = config("c2", M=M, n=n, seed=seed, h="linf")
        wl.name = "c2i"
        return wl
    if name in ("c2", "c3"):
        num = 2 if name == "c2" else 3
        n = n or (100 if num == 2 else 1000)
        seed = seed or SEED_BASE + num
        rng = np.random.default_rng([seed, _STREAM_PARAMS])
        D = _loguniform(rng, 0.5, 2.0, n).astype(np.float32)
        if num == 2:
            w = rng.uniform(0.5, 1.5, n).astype(np.float32)
            if name == "c2":
                return Workload("c2", n, M or 1_000_000, h or "wl1", "diag", seed,
                                ("normal", 2.0), ("uniform", 0.0, 1.0), D=D, w=w, gamma=-0.5)
        return Workload("c3", n, M or 100_000, h or "l2", "diag", seed,
                        ("normal", 1.0), ("uniform", 0.0, 2.0), D=D, gamma=-0.5)
    if name == "c4":
        n = n or 256
        seed = seed or SEED_BASE + 4
        rng = np.random.default_rng([seed, _STREAM_PARAMS])
        Q = haar_orthogonal(rng, n)
        Lam = _loguniform(rng, 0.1, 10.0, n)
        return Workload("c4", n, M or 4_000_000, h or "l1", "dense", seed,
                        ("normal", 1.0), ("uniform", 0.1, 1.0), Q=Q, Lam=Lam, gamma=0.0)
    if name in ("c5", "c5d"):
        n = n or 64
        K = 16
        seed = seed or SEED_BASE + 5
        rng = np.random.default_rng([seed, _STREAM_PARAMS])
        Ck = (rng.standard_normal((K, n)) * 5.0).astype(np.float32)
        a = rng.uniform(0.5, 2.0, (K, n))
        Dk = (a * a).astype(np.float32)
        gk = np.full(K, -0.5, np.float32)
        if name == "c5d":   # NEXT-1: distance / projection to the C5 union (same sets and y law)
            return Workload("c5d", n, M or 100_000, "l2", "distance", seed,
                            ("normal", 5.0), ("uniform", 0.0, 2.0), Dk=Dk, Ck=Ck, gammak=gk)
        return Workload("c5", n, M or 500_000, h or "l2", "union", seed,
                        ("normal", 5.0), ("uniform", 0.0, 2.0), Dk=Dk, Ck=Ck, gammak=gk)
    if name.startswith("p"):
        # p<n>_<id|diag>_<l1|l2>
        body = name[1:].split("_")
        n = int(body[0])
        jk = body[1] if len(body) > 1 else "id"
        hh = body[2] if len(body) > 2 else (h or "l1")
        if jk == "id":
            D = np.ones(n, np.float32)
        else:
            D = (1.0 + np.arange(n) / (n - 1)).astype(np.float32)
        return Workload(name, n, M or 1_000_000, hh, "diag", seed or SEED_BASE + 100 + n,
                        ("uniform", -10.0, 10.0), ("uniform", 0.0, 10.0), D=D, gamma=0.0)
    raise KeyError(name)


CONFIG_NAMES = ("c1", "c2", "c3", "c4", "c5", "c5d", "c2h", "c2e", "c2i", "t5", "t4a")
