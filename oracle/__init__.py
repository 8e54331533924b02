"""fp64 CPU oracle for the Hopf-formula split Bregman path — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1605_01799_b200``) never imports it and shares no code with it.

* ``hopf_oracle.c`` — the split Bregman iteration (3.4a)-(3.4c) of PAPER.md
  P:832-844 with the stopping rule of P:1595-1601, step by step in fp64.
* ``exact.py`` — independent references the oracle is pinned to (closed forms,
  secular equation, box-QP Hopf-Lax solve, duality certificate, brute force).

The shared library is compiled from the C source on first use (gcc -O2, no
fast-math, OpenMP over points) into ``oracle/_build/libhopf_oracle.so``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "hopf_oracle.c"
_BUILD = _HERE / "_build"
_LIB_PATH = _BUILD / "libhopf_oracle.so"

H_L1, H_WL1, H_L2, H_ELL, H_LINF = 0, 1, 2, 3, 4
H_KINDS = {"l1": H_L1, "wl1": H_WL1, "l2": H_L2, "ell": H_ELL, "linf": H_LINF}
INVALID = np.iinfo(np.int32).min

_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle with gcc (fp64, -O2, IEEE: no -ffast-math)."""
    _BUILD.mkdir(exist_ok=True)
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB_PATH.with_suffix(f".{os.getpid()}.tmp")
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
               "-ffp-contract=off", "-o", str(tmp), str(_SRC), "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(str(build()))
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int32)
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_diag.argtypes = [i64, i32, dp, dp, dp, dp, f64, i32, dp, f64, i32, f64,
                                    dp, dp, ip, i32]
        lib.oracle_dense.argtypes = [i64, i32, dp, dp, dp, dp, dp, f64, i32, dp, f64, i32, f64,
                                     dp, dp, ip, i32]
        lib.oracle_union.argtypes = [i64, i32, i32, dp, dp, dp, dp, dp, i32, dp, f64, i32, f64,
                                     dp, dp, ip, dp, ip, dp, i32]
        lib.oracle_distance_union.argtypes = [i64, i32, i32, dp, dp, dp, dp, f64, i32, f64, i32,
                                              f64, dp, dp, dp, dp, ip, ip, i32]
        lib.oracle_maxh.argtypes = [i64, i32, dp, dp, dp, dp, f64, i32, ip, dp, dp, f64, i32, f64,
                                    dp, dp, ip, ip, i32]
        lib.oracle_normsq.argtypes = [i64, i32, dp, dp, i32, f64, i32, dp, f64, i32, f64, dp, dp,
                                      ip, i32]
        lib.oracle_diag_A.argtypes = [i64, i32, dp, dp, dp, dp, f64, dp, dp, dp, f64, i32, f64, dp,
                                      dp, ip, i32]
        for f in (lib.oracle_diag, lib.oracle_dense, lib.oracle_union, lib.oracle_distance_union,
                  lib.oracle_maxh, lib.oracle_normsq, lib.oracle_diag_A):
            f.restype = ctypes.c_int
        lib.oracle_threads.argtypes = [i32]
        lib.oracle_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def threads(nthreads: int = 0) -> int:
    """Number of OpenMP threads the oracle uses for ``nthreads`` (0 = all cores)."""
    return _load().oracle_threads(nthreads)


def _d(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a, shape=None):
    if a is None:
        return None
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


def _hk(h):
    return H_KINDS[h] if isinstance(h, str) else int(h)


def eval_diag(X, t, D, c=None, gamma=0.0, h="l1", w=None, lam=1.0, max_iter=1000, tol=1e-8,
              nthreads=0):
    """phi, grad, iters for J(x)=1/2<x-c,D^{-1}(x-c)>+gamma."""
    X = _f64(X)
    M, n = X.shape
    t = _f64(t, (M,))
    D = _f64(D, (n,))
    c = _f64(c, (n,)) if c is not None else None
    w = _f64(w, (n,)) if w is not None else None
    phi = np.empty(M)
    grad = np.empty((M, n))
    iters = np.empty(M, dtype=np.int32)
    rc = _load().oracle_diag(M, n, _d(X), _d(t), _d(D), _d(c), float(gamma), _hk(h), _d(w),
                             float(lam), int(max_iter), float(tol), _d(phi), _d(grad),
                             iters.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_diag rejected its arguments (rc={rc})")
    return phi, grad, iters


def dense_matrices(Q, Lam, lam=1.0):
    """fp64 A = Q diag(Lam) Q^T, A^{-1}, and M_lambda = (A^{-1}+lam I)^{-1}
    = Q diag(Lam/(1+lam Lam)) Q^T (quadratic prox)."""
    Q = np.asarray(Q, dtype=np.float64)
    Lam = np.asarray(Lam, dtype=np.float64)
    A = (Q * Lam) @ Q.T
    Ainv = (Q / Lam) @ Q.T
    Ml = (Q * (Lam / (1.0 + lam * Lam))) @ Q.T
    sym = lambda S: 0.5 * (S + S.T)
    return sym(A), sym(Ainv), sym(Ml)


def eval_dense(X, t, Q, Lam, gamma=0.0, h="l1", w=None, lam=1.0, max_iter=1000, tol=1e-8,
               nthreads=0):
    """phi, grad, iters for J(x)=1/2<x,Ax>+gamma, A = Q diag(Lam) Q^T."""
    X = _f64(X)
    M, n = X.shape
    t = _f64(t, (M,))
    w = _f64(w, (n,)) if w is not None else None
    A, Ainv, Ml = dense_matrices(Q, Lam, lam)
    phi = np.empty(M)
    grad = np.empty((M, n))
    iters = np.empty(M, dtype=np.int32)
    rc = _load().oracle_dense(M, n, _d(X), _d(t), _d(Ml), _d(A), _d(Ainv), float(gamma), _hk(h),
                              _d(w), float(lam), int(max_iter), float(tol), _d(phi), _d(grad),
                              iters.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                              int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_dense rejected its arguments (rc={rc})")
    return phi, grad, iters


def eval_union(X, t, Dk, Ck, gammak, h="l2", w=None, lam=1.0, max_iter=1000, tol=1e-8,
               want_y=True, nthreads=0):
    """phi, grad, iters, Y, kstar, phi_k for J = min_k J_k."""
    X = _f64(X)
    M, n = X.shape
    Dk = _f64(Dk)
    K = Dk.shape[0]
    Dk = Dk.reshape(K, n)
    Ck = _f64(Ck, (K, n))
    gammak = _f64(gammak, (K,))
    t = _f64(t, (M,))
    w = _f64(w, (n,)) if w is not None else None
    phi = np.empty(M)
    grad = np.empty((M, n))
    iters = np.empty(M, dtype=np.int32)
    Y = np.empty((M, n)) if want_y else None
    kstar = np.empty(M, dtype=np.int32)
    phik = np.empty((M, K))
    ip = ctypes.POINTER(ctypes.c_int32)
    rc = _load().oracle_union(M, n, K, _d(X), _d(t), _d(Dk), _d(Ck), _d(gammak), _hk(h), _d(w),
                              float(lam), int(max_iter), float(tol), _d(phi), _d(grad),
                              iters.ctypes.data_as(ip), _d(Y), kstar.ctypes.data_as(ip),
                              _d(phik), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_union rejected its arguments (rc={rc})")
    return phi, grad, iters, Y, kstar, phik


def distance_union(Yq, Dk, Ck, gammak, lam=1.0, max_iter=1000, tol=1e-8, max_newton=50,
                   stol=1e-6, nthreads=0):
    """dist, proj, psi, grad, kstar, newton for Omega = union_k {L_k <= 0}: Newton in s on
    psi(y, s) = 0 with psi = min_k psi_k."""
    Yq = _f64(Yq)
    M, n = Yq.shape
    Dk = _f64(Dk)
    K = Dk.shape[0]
    Dk = Dk.reshape(K, n)
    Ck = _f64(Ck, (K, n))
    gammak = _f64(gammak, (K,))
    dist = np.empty(M)
    proj = np.empty((M, n))
    psi = np.empty(M)
    grad = np.empty((M, n))
    kstar = np.empty(M, dtype=np.int32)
    newton = np.empty(M, dtype=np.int32)
    ip = ctypes.POINTER(ctypes.c_int32)
    rc = _load().oracle_distance_union(M, n, K, _d(Yq), _d(Dk), _d(Ck), _d(gammak), float(lam),
                                       int(max_iter), float(tol), int(max_newton), float(stol),
                                       _d(dist), _d(proj), _d(psi), _d(grad),
                                       kstar.ctypes.data_as(ip), newton.ctypes.data_as(ip),
                                       int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_distance_union rejected its arguments (rc={rc})")
    return dist, proj, psi, grad, kstar, newton


def eval_maxh(X, t, D, c, gamma, kinds, a, W=None, lam=1.0, max_iter=1000, tol=1e-8, nthreads=0):
    """phi = max_i phi_i for H = min_i a_i H_{kind_i}; returns phi, grad, iters, istar."""
    X = _f64(X)
    M, n = X.shape
    D = _f64(D, (n,))
    c = _f64(c, (n,)) if c is not None else None
    t = _f64(t, (M,))
    K = len(kinds)
    kinds = np.ascontiguousarray([_hk(k) for k in kinds], dtype=np.int32)
    a = _f64(a, (K,))
    W = _f64(W, (K, n)) if W is not None else None
    phi = np.empty(M)
    grad = np.empty((M, n))
    iters = np.empty(M, dtype=np.int32)
    istar = np.empty(M, dtype=np.int32)
    ip = ctypes.POINTER(ctypes.c_int32)
    rc = _load().oracle_maxh(M, n, _d(X), _d(t), _d(D), _d(c), float(gamma), K,
                             kinds.ctypes.data_as(ip), _d(W), _d(a), float(lam), int(max_iter),
                             float(tol), _d(phi), _d(grad), iters.ctypes.data_as(ip),
                             istar.ctypes.data_as(ip), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_maxh rejected its arguments (rc={rc})")
    return phi, grad, iters, istar


J_KINDS = {"l1sq": 0, "linfsq": 1}


def eval_normsq(X, t, j, gamma=0.0, h="l1", w=None, lam=1.0, max_iter=1000, tol=1e-8, nthreads=0):
    """NEXT-3: J = 1/2||.||_1^2 (j="l1sq") or 1/2||.||_inf^2 (j="linfsq") plus gamma, any H
    (P:1488-1555).  Returns phi, grad, iters."""
    X = _f64(X)
    M, n = X.shape
    t = _f64(t, (M,))
    w = _f64(w, (n,)) if w is not None else None
    phi = np.empty(M)
    grad = np.empty((M, n))
    iters = np.empty(M, dtype=np.int32)
    ip = ctypes.POINTER(ctypes.c_int32)
    rc = _load().oracle_normsq(M, n, _d(X), _d(t), J_KINDS[j], float(gamma), _hk(h), _d(w),
                               float(lam), int(max_iter), float(tol), _d(phi), _d(grad),
                               iters.ctypes.data_as(ip), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_normsq rejected its arguments (rc={rc})")
    return phi, grad, iters


def eval_diag_A(X, t, D, c, gamma, A, lam=1.0, max_iter=1000, tol=1e-8, nthreads=0):
    """NEXT-2: diagonal J with H(p) = sqrt(<p, A p>), A SPD [n,n].  The spectral
    form A = Q diag(Lam) Q^T the paper's projection needs is computed here in fp64 (numpy eigh);
    returns phi, grad, iters."""
    X = _f64(X)
    M, n = X.shape
    t = _f64(t, (M,))
    D = _f64(D, (n,))
    c = _f64(c, (n,)) if c is not None else None
    A = _f64(A, (n, n))
    Lam, Q = np.linalg.eigh(A)
    Q = np.ascontiguousarray(Q)
    Lam = np.ascontiguousarray(Lam)
    phi = np.empty(M)
    grad = np.empty((M, n))
    iters = np.empty(M, dtype=np.int32)
    ip = ctypes.POINTER(ctypes.c_int32)
    rc = _load().oracle_diag_A(M, n, _d(X), _d(t), _d(D), _d(c), float(gamma), _d(Q), _d(Lam),
                               _d(A), float(lam), int(max_iter), float(tol), _d(phi), _d(grad),
                               iters.ctypes.data_as(ip), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_diag_A rejected its arguments (rc={rc})")
    return phi, grad, iters
