"""paper_1605_01799_b200 — B200-native batched Hopf-formula evaluator (arXiv 1605.01799).

Thin Python binding over the C ABI of ``libhopf.so`` (include/hopf.h): argument
marshalling only.  Every step of the split Bregman path runs in the library's sm_100a
kernels; PyTorch provides device memory (``data_ptr()``) and streams.  There is no
CPU fallback: if the extension is missing this module raises on import of ``lib()``.
"""
from __future__ import annotations

import contextlib
import ctypes
from pathlib import Path

__all__ = ["lib", "eval_diag", "eval_union", "eval_dense", "DensePlan", "eval_diag_host", "eval_normsq", "eval_diag_A",
           "HopfError", "H_KINDS", "INVALID"]

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libhopf.so"
H_KINDS = {"l1": 0, "wl1": 1, "l2": 2, "ell": 3, "linf": 4}
INVALID = -(2 ** 31)
_lib = None


class HopfError(RuntimeError):
    def __init__(self, code: int, where: str, detail: str):
        super().__init__(f"{where} failed with code {code}: {detail}")
        self.code = code


def lib():
    """The loaded libhopf.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1605_01799_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
        L.hopf_eval_diag.argtypes = [i64, i32, vp, vp, vp, vp, f32, ctypes.c_int, vp, f32, i32, f32,
                                     vp, vp, vp, vp]
        L.hopf_eval_normsq.argtypes = [i64, i32, vp, vp, ctypes.c_int, f32, ctypes.c_int, vp, f32,
                                       i32, f32, vp, vp, vp, vp]
        L.hopf_eval_diag_A.argtypes = [i64, i32, vp, vp, vp, vp, f32, vp, vp, f32, i32, f32, vp, vp,
                                       vp, vp]
        L.hopf_eval_union.argtypes = [i64, i32, i32, vp, vp, vp, vp, vp, ctypes.c_int, vp, f32, i32,
                                      f32, vp, vp, vp, vp, vp, vp, vp]
        L.hopf_dense_plan_create.argtypes = [i32, vp, vp, f32, ctypes.POINTER(vp)]
        L.hopf_dense_plan_destroy.argtypes = [vp]
        L.hopf_eval_dense.argtypes = [i64, i32, vp, vp, vp, f32, ctypes.c_int, vp, f32, i32, f32,
                                      vp, vp, vp, vp]
        L.hopf_eval_diag_host.argtypes = [i64, i32, vp, vp, vp, vp, f32, ctypes.c_int, vp, f32, i32,
                                          f32, vp, vp, vp]
        L.hopf_eval_maxh.argtypes = [i64, i32, vp, vp, vp, vp, f32, i32, vp, vp, vp, f32, i32, f32,
                                     vp, vp, vp, vp, vp]
        L.hopf_distance_union.argtypes = [i64, i32, i32, vp, vp, vp, vp, f32, i32, f32, i32, f32,
                                          vp, vp, vp, vp, vp, vp, vp]
        for f in (L.hopf_eval_diag, L.hopf_eval_union, L.hopf_dense_plan_create,
                  L.hopf_dense_plan_destroy, L.hopf_eval_dense, L.hopf_eval_diag_host,
                  L.hopf_distance_union, L.hopf_eval_maxh, L.hopf_eval_normsq, L.hopf_eval_diag_A):
            f.restype = ctypes.c_int
        L.hopf_last_error.restype = ctypes.c_char_p
        L.hopf_strerror.restype = ctypes.c_char_p
        L.hopf_strerror.argtypes = [ctypes.c_int]
        L.hopf_last_launch_count.restype = ctypes.c_int32
        L.hopf_set_iteration_counter.argtypes = [vp]
        L.hopf_set_iteration_counter.restype = ctypes.c_int
        L.hopf_last_kernel.restype = ctypes.c_char_p
        L.hopf_last_launch_config.restype = ctypes.c_int32
        L.hopf_last_launch_config.argtypes = [ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
        L.hopf_version.restype = ctypes.c_int32
        _lib = L
    return _lib


def _check(rc: int, where: str):
    if rc != 0:
        L = lib()
        raise HopfError(rc, where, (L.hopf_last_error() or b"").decode() or
                        L.hopf_strerror(rc).decode())


def set_iteration_counter(counter) -> None:
    """Point the library's solve-iteration counter at a device int64 tensor (or None)."""
    _check(lib().hopf_set_iteration_counter(None if counter is None else counter.data_ptr()),
           "hopf_set_iteration_counter")


def last_kernel() -> str:
    """Name of the main kernel the most recent call launched on this thread."""
    return (lib().hopf_last_kernel() or b"").decode()


def last_launch_count() -> int:
    return int(lib().hopf_last_launch_count())


def _ptr(tensor, dtype_name, numel=None, name="tensor"):
    """Device pointer of a contiguous CUDA tensor (validates dtype/size/device)."""
    import torch
    if tensor is None:
        return None
    if not isinstance(tensor, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    want = {"f32": torch.float32, "i32": torch.int32, "f64": torch.float64}[dtype_name]
    if tensor.dtype != want:
        raise TypeError(f"{name} must be {want}, got {tensor.dtype}")
    if not tensor.is_cuda:
        raise ValueError(f"{name} must live on a CUDA device")
    if not tensor.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and tensor.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {tensor.numel()}")
    return tensor.data_ptr()


def _host(tensor, dtype_name, numel, name):
    """Validate a HOST tensor handed to hopf_eval_diag_host (dtype, size, contiguity): the library
    copies exactly numel elements to / from its address."""
    import torch
    if not isinstance(tensor, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    want = {"f32": torch.float32, "i32": torch.int32}[dtype_name]
    if tensor.dtype != want:
        raise TypeError(f"{name} must be {want}, got {tensor.dtype}")
    if tensor.is_cuda:
        raise ValueError(f"{name} must be a host tensor (eval_diag_host)")
    if not tensor.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if tensor.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {tensor.numel()}")
    return tensor.data_ptr()


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


@contextlib.contextmanager
def _device_of(*tensors, stream=None):
    """Run the enclosed library call with the tensors' device as the current CUDA device.

    Every tensor (None entries skipped) and the stream must live on that device: the library
    launches on the current device, so a foreign-device pointer would fault."""
    import torch
    ts = [x for x in tensors if x is not None]
    dev = ts[0].device
    for x in ts[1:]:
        if x.device != dev:
            raise ValueError(f"all tensors must live on {dev}, got one on {x.device}")
    if stream is not None and stream.device != dev:
        raise ValueError(f"stream is on {stream.device}, the tensors on {dev}")
    with torch.cuda.device(dev):
        yield


def _outputs(M, n, device, out):
    import torch
    if out is not None:
        return out
    phi = torch.empty(M, dtype=torch.float32, device=device)
    grad = torch.empty((M, n), dtype=torch.float32, device=device)
    iters = torch.empty(M, dtype=torch.int32, device=device)
    return phi, grad, iters


def eval_diag(X, t, D, c=None, gamma=0.0, h="l1", w=None, lam=1.0, max_iter=1000, tol=1e-8,
              out=None, stream=None):
    """hopf_eval_diag: J(x) = 1/2<x-c, D^{-1}(x-c)> + gamma, H in {l1, wl1, l2, ell, linf}.

    X [M,n], t [M], D [n], c [n]|None, w [n]|None: float32 CUDA tensors.
    Returns (phi [M], grad [M,n], iters [M] int32)."""
    M, n = X.shape
    phi, grad, iters = _outputs(M, n, X.device, out)
    with _device_of(X, t, D, c, w, phi, grad, iters, stream=stream):
        rc = lib().hopf_eval_diag(M, n, _ptr(X, "f32", M * n, "X"), _ptr(t, "f32", M, "t"),
                                  _ptr(D, "f32", n, "D"), _ptr(c, "f32", n, "c"), float(gamma),
                                  H_KINDS[h], _ptr(w, "f32", n, "w"), float(lam), int(max_iter),
                                  float(tol), _ptr(phi, "f32", M, "phi"), _ptr(grad, "f32", M * n, "grad"),
                                  _ptr(iters, "i32", M, "iters"), _stream(stream))
    _check(rc, "hopf_eval_diag")
    return phi, grad, iters


def eval_union(X, t, Dk, Ck, gammak, h="l2", w=None, lam=1.0, max_iter=1000, tol=1e-8,
               want_y=True, want_kstar=True, want_phik=False, out=None, stream=None):
    """hopf_eval_union: J = min_k J_k.  Returns (phi, grad, iters, Y|None, kstar|None, phik|None)."""
    import torch
    M, n = X.shape
    K = Dk.shape[0]
    phi, grad, iters = _outputs(M, n, X.device, out)
    Y = torch.empty((M, n), dtype=torch.float32, device=X.device) if want_y else None
    ks = torch.empty(M, dtype=torch.int32, device=X.device) if want_kstar else None
    pk = torch.empty((M, K), dtype=torch.float32, device=X.device) if want_phik else None
    with _device_of(X, t, Dk, Ck, gammak, w, phi, grad, iters, Y, ks, pk, stream=stream):
        rc = lib().hopf_eval_union(M, n, K, _ptr(X, "f32", M * n, "X"), _ptr(t, "f32", M, "t"),
                                   _ptr(Dk, "f32", K * n, "Dk"), _ptr(Ck, "f32", K * n, "Ck"),
                                   _ptr(gammak, "f32", K, "gammak"), H_KINDS[h], _ptr(w, "f32", n, "w"),
                                   float(lam), int(max_iter), float(tol), _ptr(phi, "f32", M, "phi"),
                                   _ptr(grad, "f32", M * n, "grad"), _ptr(iters, "i32", M, "iters"),
                                   _ptr(Y, "f32", M * n, "Y"), _ptr(ks, "i32", M, "kstar"),
                                   _ptr(pk, "f32", M * K, "phik"), _stream(stream))
    _check(rc, "hopf_eval_union")
    return phi, grad, iters, Y, ks, pk


def eval_diag_A(X, t, D, c, gamma, Q, Lam, lam=1.0, max_iter=1000, tol=1e-8, out=None,
                stream=None):
    """hopf_eval_diag_A (NEXT-2): diagonal J, H(p) = sqrt(<p, A p>), A = Q diag(Lam) Q^T given in
    spectral form (Q [n,n] eigenvectors as columns, Lam [n]; float32 CUDA tensors)."""
    M, n = X.shape
    phi, grad, iters = _outputs(M, n, X.device, out)
    with _device_of(X, t, D, c, Q, Lam, phi, grad, iters, stream=stream):
        rc = lib().hopf_eval_diag_A(M, n, _ptr(X, "f32", M * n, "X"), _ptr(t, "f32", M, "t"),
                                    _ptr(D, "f32", n, "D"), _ptr(c, "f32", n, "c"), float(gamma),
                                    _ptr(Q, "f32", n * n, "Q"), _ptr(Lam, "f32", n, "Lam"), float(lam),
                                    int(max_iter), float(tol), _ptr(phi, "f32", M, "phi"),
                                    _ptr(grad, "f32", M * n, "grad"), _ptr(iters, "i32", M, "iters"),
                                    _stream(stream))
    _check(rc, "hopf_eval_diag_A")
    return phi, grad, iters


J_KINDS = {"l1sq": 0, "linfsq": 1}


def eval_normsq(X, t, j, gamma=0.0, h="l1", w=None, lam=1.0, max_iter=1000, tol=1e-8, out=None,
                stream=None):
    """hopf_eval_normsq (NEXT-3): J = 1/2||.||_1^2 (j="l1sq") or 1/2||.||_inf^2 (j="linfsq") plus
    gamma, H in {l1, wl1, l2, linf}.  Returns (phi [M], grad [M,n], iters [M] int32)."""
    M, n = X.shape
    phi, grad, iters = _outputs(M, n, X.device, out)
    with _device_of(X, t, w, phi, grad, iters, stream=stream):
        rc = lib().hopf_eval_normsq(M, n, _ptr(X, "f32", M * n, "X"), _ptr(t, "f32", M, "t"),
                                    J_KINDS[j], float(gamma), H_KINDS[h], _ptr(w, "f32", n, "w"),
                                    float(lam), int(max_iter), float(tol), _ptr(phi, "f32", M, "phi"),
                                    _ptr(grad, "f32", M * n, "grad"), _ptr(iters, "i32", M, "iters"),
                                    _stream(stream))
    _check(rc, "hopf_eval_normsq")
    return phi, grad, iters


def eval_maxh(X, t, D, c, gamma, kinds, a, W=None, lam=1.0, max_iter=1000, tol=1e-8, out=None,
              stream=None):
    """hopf_eval_maxh: phi = max_i phi_i for H = min_i a_i H_{kind_i}.

    kinds: K names from H_KINDS ("l1", "wl1", "l2", "ell", "linf"); a: K scales > 0 (host);
    W [K, n] float32 CUDA tensor, row i used by "wl1" / "ell" members (else may be None).
    Returns (phi, grad, iters, istar) with istar the winning member (-1 on invalid points)."""
    import numpy as np
    import torch
    M, n = X.shape
    K = len(kinds)
    phi, grad, iters = _outputs(M, n, X.device, out)
    ist = torch.empty(M, dtype=torch.int32, device=X.device)
    hk = np.ascontiguousarray([H_KINDS[k] if isinstance(k, str) else int(k) for k in kinds], dtype=np.int32)
    av = np.ascontiguousarray(a, dtype=np.float32)
    if av.shape != (K,):
        raise ValueError("a must have one scale per Hamiltonian")
    with _device_of(X, t, D, c, W, phi, grad, iters, ist, stream=stream):
        rc = lib().hopf_eval_maxh(M, n, _ptr(X, "f32", M * n, "X"), _ptr(t, "f32", M, "t"),
                                  _ptr(D, "f32", n, "D"), _ptr(c, "f32", n, "c"), float(gamma), K,
                                  hk.ctypes.data, av.ctypes.data, _ptr(W, "f32", K * n, "W"),
                                  float(lam), int(max_iter), float(tol), _ptr(phi, "f32", M, "phi"),
                                  _ptr(grad, "f32", M * n, "grad"), _ptr(iters, "i32", M, "iters"),
                                  _ptr(ist, "i32", M, "istar"), _stream(stream))
    _check(rc, "hopf_eval_maxh")
    return phi, grad, iters, ist


def distance_union(Y, Dk, Ck, gammak, lam=1.0, max_iter=1000, tol=1e-8, max_newton=50,
                   stol=1e-5, stream=None):
    """hopf_distance_union: distance and closest point to the union of the sets
    {L_k <= 0} by Newton in s on psi(y,s) = 0.
    Returns (dist, proj, psi, grad, kstar, newton)."""
    import torch
    M, n = Y.shape
    K = Dk.shape[0]
    dev = Y.device
    dist = torch.empty(M, dtype=torch.float32, device=dev)
    proj = torch.empty((M, n), dtype=torch.float32, device=dev)
    psi = torch.empty(M, dtype=torch.float32, device=dev)
    grad = torch.empty((M, n), dtype=torch.float32, device=dev)
    ks = torch.empty(M, dtype=torch.int32, device=dev)
    nn = torch.empty(M, dtype=torch.int32, device=dev)
    with _device_of(Y, Dk, Ck, gammak, dist, proj, psi, grad, ks, nn, stream=stream):
        rc = lib().hopf_distance_union(M, n, K, _ptr(Y, "f32", M * n, "Y"), _ptr(Dk, "f32", K * n, "Dk"),
                                       _ptr(Ck, "f32", K * n, "Ck"), _ptr(gammak, "f32", K, "gammak"),
                                       float(lam), int(max_iter), float(tol), int(max_newton),
                                       float(stol), _ptr(dist, "f32", M, "dist"),
                                       _ptr(proj, "f32", M * n, "proj"), _ptr(psi, "f32", M, "psi"),
                                       _ptr(grad, "f32", M * n, "grad"), _ptr(ks, "i32", M, "kstar"),
                                       _ptr(nn, "i32", M, "newton"), _stream(stream))
    _check(rc, "hopf_distance_union")
    return dist, proj, psi, grad, ks, nn


class DensePlan:
    """hopf_dense_plan for J(x) = 1/2<x, Q diag(Lam) Q^T x> (built in fp64 on the host)."""

    def __init__(self, Q, Lam, lam=1.0):
        import numpy as np
        Q = np.ascontiguousarray(np.asarray(Q, dtype=np.float64))
        Lam = np.ascontiguousarray(np.asarray(Lam, dtype=np.float64))
        n = Lam.shape[0]
        if Q.shape != (n, n):
            raise ValueError("Q must be n x n")
        self.n, self.lam = n, float(lam)
        h = ctypes.c_void_p()
        rc = lib().hopf_dense_plan_create(n, Q.ctypes.data, Lam.ctypes.data, float(lam),
                                          ctypes.byref(h))
        _check(rc, "hopf_dense_plan_create")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().hopf_dense_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def eval_dense(X, t, plan: DensePlan, gamma=0.0, h="l1", w=None, max_iter=1000, tol=1e-8,
               out=None, stream=None):
    """hopf_eval_dense with a DensePlan.  Returns (phi, grad, iters)."""
    M, n = X.shape
    phi, grad, iters = _outputs(M, n, X.device, out)
    with _device_of(X, t, w, phi, grad, iters, stream=stream):
        rc = lib().hopf_eval_dense(M, n, _ptr(X, "f32", M * n, "X"), _ptr(t, "f32", M, "t"), plan._h,
                                   float(gamma), H_KINDS[h], _ptr(w, "f32", n, "w"), float(plan.lam),
                                   int(max_iter), float(tol), _ptr(phi, "f32", M, "phi"),
                                   _ptr(grad, "f32", M * n, "grad"), _ptr(iters, "i32", M, "iters"),
                                   _stream(stream))
    _check(rc, "hopf_eval_dense")
    return phi, grad, iters


def eval_diag_host(X, t, D, c=None, gamma=0.0, h="l1", w=None, lam=1.0, max_iter=1000, tol=1e-8,
                   out=None):
    """hopf_eval_diag_host: HOST (ideally pinned) X, t in and phi, grad, iters out; D/c/w on device.
    Copies are pipelined inside the library.  Returns host tensors (phi, grad, iters)."""
    import torch
    if X.dim() != 2:
        raise ValueError("X must be 2-D [M, n]")
    M, n = X.shape
    if out is None:
        out = (torch.empty(M, dtype=torch.float32, pin_memory=True),
               torch.empty((M, n), dtype=torch.float32, pin_memory=True),
               torch.empty(M, dtype=torch.int32, pin_memory=True))
    phi, grad, iters = out
    _host(X, "f32", M * n, "X")
    _host(t, "f32", M, "t")
    _host(phi, "f32", M, "phi")
    _host(grad, "f32", M * n, "grad")
    _host(iters, "i32", M, "iters")
    dev = D.device
    for a in (c, w):
        if a is not None and a.device != dev:
            raise ValueError(f"D, c and w must live on one device, got {a.device} and {dev}")
    with torch.cuda.device(dev):
        rc = lib().hopf_eval_diag_host(M, n, X.data_ptr(), t.data_ptr(), _ptr(D, "f32", n, "D"),
                                       _ptr(c, "f32", n, "c"), float(gamma), H_KINDS[h],
                                       _ptr(w, "f32", n, "w"), float(lam), int(max_iter), float(tol),
                                       phi.data_ptr(), grad.data_ptr(), iters.data_ptr())
    _check(rc, "hopf_eval_diag_host")
    return phi, grad, iters
