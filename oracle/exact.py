"""Independent exact references that pin the split Bregman oracle — TEST INFRASTRUCTURE.

None of these run the paper's iteration; each is a *plain definition* of the
same quantity, so a dropped term, a wrong sign, a transposed operand or an index
slip in ``hopf_oracle.c`` makes one of them disagree.

Hopf formula (1.2)/(3.3), P:135-142 / P:815-818:
    phi(x,t) = max_v { <x,v> - J*(v) - t H(v) },  grad phi = the unique maximiser.
Hopf-Lax formula, P:640-646 and P:749-752 (H = support function of C):
    phi(x,t) = min { J(z) : (x - z)/t in C },      grad phi = grad J(z*).
C is the box prod_i [-w_i, w_i] for H = sum_i w_i |p_i|, the unit ball for H = ||p||_2.
"""
from __future__ import annotations

import itertools

import numpy as np


# --------------------------------------------------------------------------- diag, l1
def diag_wl1_closed(x, t, D, c=None, gamma=0.0, w=None):
    """Separable closed form for J = 1/2<x-c,D^{-1}(x-c)> + gamma, H = sum w_i|p_i|.

    The ellipsoid/l1 computation of P:209-263 (a_i^2 = D_i; alpha_i = t w_i):
    the Hopf objective decouples into 1-D problems 1/2 D_i v_i^2 + t w_i |v_i| - xt_i v_i
    whose minimiser is shrink_1(xt_i, t w_i)/D_i, giving
        grad_i = sign(xt_i) max(|xt_i| - t w_i, 0) / D_i
        phi    = gamma + sum_i 1/2 max(|xt_i| - t w_i, 0)^2 / D_i.
    """
    x = np.asarray(x, np.float64)
    D = np.asarray(D, np.float64)
    xt = x - (0.0 if c is None else np.asarray(c, np.float64))
    w = np.ones_like(D) if w is None else np.asarray(w, np.float64)
    t = np.asarray(t, np.float64)[..., None]
    s = np.maximum(np.abs(xt) - t * w, 0.0)
    grad = np.sign(xt) * s / D
    phi = gamma + 0.5 * np.sum(s * s / D, axis=-1)
    return phi, grad


# --------------------------------------------------------------------------- diag, l2
def diag_l2_secular(x, t, D, c=None, gamma=0.0, iters=200):
    """Exact phi, grad for J = 1/2<x-c,D^{-1}(x-c)> + gamma, H = ||.||_2.

    Optimality of the Hopf objective (3.3): D v + t v/||v|| = xt for v != 0, i.e.
    v_i = xt_i/(D_i + mu) with mu = t/||v|| > 0 the root of
        g(mu) = mu^2 sum_i xt_i^2/(D_i+mu)^2 - t^2      (strictly increasing, 0 -> ||xt||^2 - t^2).
    v = 0 iff ||xt|| <= t.  phi = <xt,v> - 1/2<v,Dv> - t||v|| + gamma
                                = gamma + 1/2 sum_i D_i xt_i^2/(D_i+mu)^2.
    D = I reduces to the sphere formula of P:306-310 (mu = t/(||x||-t)).
    Solved by fp64 bisection on the bracket [t Dmin/(|xt|-t), t Dmax/(|xt|-t)].
    """
    x = np.atleast_2d(np.asarray(x, np.float64))
    D = np.asarray(D, np.float64)
    xt = x - (0.0 if c is None else np.asarray(c, np.float64))
    t = np.broadcast_to(np.asarray(t, np.float64), (x.shape[0],))
    r = np.linalg.norm(xt, axis=1)
    phi = np.full(x.shape[0], float(gamma))
    grad = np.zeros_like(xt)
    for p in range(x.shape[0]):
        if not r[p] > t[p]:
            continue
        lo = t[p] * D.min() / (r[p] - t[p])
        hi = t[p] * D.max() / (r[p] - t[p])
        xp = xt[p]
        for _ in range(iters):
            mid = 0.5 * (lo + hi)
            g = mid * mid * np.sum(xp * xp / (D + mid) ** 2) - t[p] ** 2
            if g > 0:
                hi = mid
            else:
                lo = mid
        mu = 0.5 * (lo + hi)
        grad[p] = xp / (D + mu)
        phi[p] = gamma + 0.5 * np.sum(D * xp * xp / (D + mu) ** 2)
    return phi, grad


# --------------------------------------------------------------------------- dense
def box_qp_hopf_lax(x, t, A, w=None, gamma=0.0, sweeps=20000, tol=1e-15):
    """phi = min { 1/2<z,Az> + gamma : |x_i - z_i| <= t w_i } by projected Gauss-Seidel.

    Hopf-Lax for H = sum w_i |p_i| (C = box, P:465-496 with P:640-646).
    grad phi = A z* (grad phi = grad H*(...) in dJ(z*)).  Independent of
    split Bregman: exact coordinate minimisation of a strongly convex quadratic over a box.
    """
    x = np.asarray(x, np.float64)
    A = np.asarray(A, np.float64)
    n = x.size
    w = np.ones(n) if w is None else np.asarray(w, np.float64)
    lo, hi = x - t * w, x + t * w
    z = np.clip(np.zeros(n), lo, hi)
    g = A @ z
    diag = np.diag(A).copy()
    for _ in range(sweeps):
        zmax = 0.0
        for i in range(n):
            zi = min(max(z[i] - g[i] / diag[i], lo[i]), hi[i])
            dz = zi - z[i]
            if dz != 0.0:
                g += A[:, i] * dz
                z[i] = zi
                zmax = max(zmax, abs(dz))
        if zmax <= tol:
            break
    g = A @ z
    return 0.5 * z @ g + gamma, g, z


def dual_lower_bound(x, t, v, Ainv, w=None, gamma=0.0, h="l1"):
    """L(v) = <x,v> - J*(v) - t H(v) <= phi(x,t) for every v (weak duality of (3.3))."""
    x, v = np.asarray(x, np.float64), np.asarray(v, np.float64)
    Hv = np.linalg.norm(v) if h == "l2" else np.sum((1.0 if w is None else w) * np.abs(v))
    return x @ v - 0.5 * v @ (Ainv @ v) + gamma - t * Hv


def primal_upper_bound(x, t, v, A, Ainv, w=None, gamma=0.0):
    """U(z) = J(z) >= phi(x,t) for the Hopf-Lax-feasible z = x - clip(x - A^{-1}v, -tw, tw)."""
    x, v = np.asarray(x, np.float64), np.asarray(v, np.float64)
    ww = np.ones_like(x) if w is None else np.asarray(w, np.float64)
    z = x - np.clip(x - Ainv @ v, -t * ww, t * ww)
    return 0.5 * z @ (A @ z) + gamma


def box_qp_bruteforce(x, t, A, w=None, gamma=0.0):
    """Exhaustive KKT active-set enumeration (3^n sets) of the box QP, n <= 8.

    For every assignment of each coordinate to {lower bound, upper bound, free}
    solve the equality-constrained QP and keep the feasible point with the
    smallest J.  Brute force: no iteration, no tolerance.
    """
    x = np.asarray(x, np.float64)
    A = np.asarray(A, np.float64)
    n = x.size
    w = np.ones(n) if w is None else np.asarray(w, np.float64)
    lo, hi = x - t * w, x + t * w
    best, bestz = np.inf, None
    for pattern in itertools.product((0, 1, 2), repeat=n):
        pat = np.array(pattern)
        z = np.where(pat == 0, lo, np.where(pat == 1, hi, 0.0))
        free = pat == 2
        if free.any():
            fixed = ~free
            rhs = -A[np.ix_(free, fixed)] @ z[fixed]
            z[free] = np.linalg.solve(A[np.ix_(free, free)], rhs)
            if np.any(z[free] < lo[free] - 1e-12) or np.any(z[free] > hi[free] + 1e-12):
                continue
        val = 0.5 * z @ (A @ z)
        if val < best:
            best, bestz = val, z
    return best + gamma, A @ bestz, bestz


# --------------------------------------------------------------------------- brute force n <= 2
def hopf_lax_grid_2d(x, t, J, h="l2", w=None, m=801):
    """phi(x,t) = min_{p in C} J(x - t p) on a fine grid over C (n = 2), plus a local refine.

    C = unit disc (H = l2) or the box [-w1,w1]x[-w2,w2] (H = weighted l1), P:465-496,
    P:640-646.  J is any callable on an (k,2) array (e.g. a union min_k J_k).
    """
    x = np.asarray(x, np.float64)
    w = np.ones(2) if w is None else np.asarray(w, np.float64)

    def cands(c0, half, mm):
        g = np.linspace(-1.0, 1.0, mm)
        P = np.stack(np.meshgrid(c0[0] + half[0] * g, c0[1] + half[1] * g), -1).reshape(-1, 2)
        if h == "l2":
            nr = np.linalg.norm(P, axis=1)
            P = np.where(nr[:, None] > 1.0, P / np.maximum(nr, 1e-300)[:, None], P)
        else:
            P = np.clip(P, -w, w)
        return P

    P = cands(np.zeros(2), w if h != "l2" else np.ones(2), m)
    vals = J(x[None, :] - t * P)
    best = np.argmin(vals)
    p0, v0 = P[best], vals[best]
    half = (w if h != "l2" else np.ones(2)) * (4.0 / (m - 1))
    for _ in range(6):
        P = cands(p0, half, 81)
        vals = J(x[None, :] - t * P)
        k = np.argmin(vals)
        if vals[k] <= v0:
            p0, v0 = P[k], vals[k]
        half = half / 10.0
    return float(v0), x - t * p0


def hopf_dual_grid_2d(x, t, Jstar, Hfun, radius, m=801):
    """phi = -min_v {J*(v) + t H(v) - <x,v>} on a grid |v_i| <= radius (n = 2), refined.

    The Hopf formula (3.3) itself, minimised by exhaustive search.  Returns (phi, argmin v).
    """
    x = np.asarray(x, np.float64)

    def obj(V):
        return Jstar(V) + t * Hfun(V) - V @ x

    c0 = np.zeros(2)
    half = radius
    best_v, best = None, np.inf
    mm = m
    for _ in range(7):
        g = np.linspace(-1.0, 1.0, mm)
        V = np.stack(np.meshgrid(c0[0] + half * g, c0[1] + half * g), -1).reshape(-1, 2)
        vals = obj(V)
        k = np.argmin(vals)
        if vals[k] <= best:
            best, best_v = vals[k], V[k]
        c0 = best_v
        half = half * 8.0 / (mm - 1)
        mm = 81
    return float(-best), best_v


# --------------------------------------------------------------------------- union
def union_exact(x, t, Dk, Ck, gammak, h="l2", w=None):
    """phi = min_k phi_k with each phi_k from the exact single-set form
    (translation: J_k(x) = J_0(x - c_k) => phi_k(x,t) = phi_0(x - c_k, t)).
    Returns phi, grad of the lowest-index minimiser, kstar, phi_k."""
    x = np.atleast_2d(np.asarray(x, np.float64))
    K = len(gammak)
    phik = np.empty((x.shape[0], K))
    grads = []
    for k in range(K):
        if h == "l2":
            p, g = diag_l2_secular(x, t, Dk[k], Ck[k], gammak[k])
        else:
            p, g = diag_wl1_closed(x, t, Dk[k], Ck[k], gammak[k], w)
        phik[:, k] = p
        grads.append(g)
    kstar = np.argmin(phik, axis=1)
    grad = np.stack([grads[k][i] for i, k in enumerate(kstar)])
    return phik[np.arange(x.shape[0]), kstar], grad, kstar, phik


# --------------------------------------------------------------------------- distance (NEXT-1)
def ellipsoid_projection(y, c, D, gamma=-0.5, iters=200):
    """Euclidean projection of y onto E = {z : 1/2 <z-c, D^{-1}(z-c)> + gamma <= 0} (gamma < 0).

    Plain definition, no Hopf formula: minimise 1/2||z - y||^2 subject to
    sum_i (z_i - c_i)^2 / D_i <= r2, r2 = -2 gamma.  For y outside E the KKT condition
    z - y + mu D^{-1}(z - c) = 0 gives z_i - c_i = (y_i - c_i) D_i / (D_i + mu), with mu > 0 the
    root of sum_i (y_i - c_i)^2 D_i / (D_i + mu)^2 = r2 (left side strictly decreasing in mu);
    bisection to full precision.  Returns (distance, z)."""
    y = np.asarray(y, np.float64)
    c = np.asarray(c, np.float64)
    D = np.asarray(D, np.float64)
    r2 = -2.0 * gamma
    yt = y - c
    if np.sum(yt * yt / D) <= r2:
        return 0.0, y.copy()
    f = lambda mu: np.sum(yt * yt * D / (D + mu) ** 2) - r2
    lo, hi = 0.0, 1.0
    while f(hi) > 0:
        hi *= 2.0
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if f(mid) > 0:
            lo = mid
        else:
            hi = mid
    mu = 0.5 * (lo + hi)
    z = c + yt * D / (D + mu)
    return float(np.linalg.norm(z - y)), z


def union_distance_exact(y, Dk, Ck, gammak):
    """dist(y, union_k E_k) = min_k dist(y, E_k); the projection and member of the minimiser
    (lowest k on ties)."""
    best = (np.inf, None, -1)
    for k in range(len(gammak)):
        d, z = ellipsoid_projection(y, Ck[k], Dk[k], gammak[k])
        if d < best[0]:
            best = (d, z, k)
    return best


# --------------------------------------------------------------------------- ellipsoidal H (NEXT-2)
def diag_ell_secular(x, t, D, W, c=None, gamma=0.0, iters=200):
    """J = 1/2<x-c, D^{-1}(x-c)> + gamma, H(p) = sqrt(<p, W p>) (W, D diagonal > 0).

    Plain definition: the maximiser v of <xt,v> - 1/2<v,Dv> - t ||v||_W satisfies
    xt - D v = t W v / s with s = ||v||_W > 0, so v_i = xt_i s / (D_i s + t W_i) and
    h(s) = sum_i W_i xt_i^2 / (D_i s + t W_i)^2 = 1 (h strictly decreasing); v = 0 when
    h(0+) = sum_i xt_i^2 / (t^2 W_i) <= 1.  Bisection on s.  Returns (phi, grad)."""
    xt = np.asarray(x, np.float64) - (0.0 if c is None else np.asarray(c, np.float64))
    D = np.asarray(D, np.float64)
    W = np.asarray(W, np.float64)
    if t <= 0 or np.sum(xt * xt / (t * t * W)) <= 1.0:
        v = np.zeros_like(xt) if t > 0 else xt / D
        phi = gamma + (0.5 * np.sum(xt * xt / D) if t <= 0 else 0.0)
        return phi, v
    h = lambda s: np.sum(W * xt * xt / (D * s + t * W) ** 2) - 1.0
    lo, hi = 0.0, 1.0
    while h(hi) > 0:
        hi *= 2.0
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if h(mid) > 0:
            lo = mid
        else:
            hi = mid
    s = 0.5 * (lo + hi)
    v = xt * s / (D * s + t * W)
    phi = xt @ v - 0.5 * v @ (D * v) - t * np.sqrt(v @ (W * v)) + gamma
    return float(phi), v


# --------------------------------------------------------------------------- l_inf H (NEXT-2)
def diag_linf_bisection(x, t, D, c=None, gamma=0.0, iters=200):
    """J = 1/2<x-c, D^{-1}(x-c)> + gamma, H = ||.||_inf.

    Plain definition: phi = max_v <xt,v> - 1/2<v,Dv> - t max_i |v_i|.  For a fixed level
    s = max_i |v_i| the maximiser is v_i = clamp(xt_i / D_i, -s, s); the remaining objective
    g(s) = sum_i [1/2 D_i v_i^2 - xt_i v_i] + t s is convex in s >= 0 with derivative
    g'(s) = t - sum_{|xt_i|/D_i > s} (|xt_i| - D_i s), increasing: s* = 0 if g'(0) >= 0, else
    the root of g' by bisection.  Returns (phi, grad = v*)."""
    xt = np.asarray(x, np.float64) - (0.0 if c is None else np.asarray(c, np.float64))
    D = np.asarray(D, np.float64)
    if t <= 0:
        return 0.5 * np.sum(xt * xt / D) + gamma, xt / D
    a = np.abs(xt) / D
    gp = lambda s: t - np.sum(np.where(a > s, np.abs(xt) - D * s, 0.0))
    if gp(0.0) >= 0:
        s = 0.0
    else:
        lo, hi = 0.0, float(a.max())
        for _ in range(iters):
            mid = 0.5 * (lo + hi)
            if gp(mid) < 0:
                lo = mid
            else:
                hi = mid
        s = 0.5 * (lo + hi)
    v = np.clip(xt / D, -s, s)
    phi = xt @ v - 0.5 * v @ (D * v) - t * (np.abs(v).max() if v.size else 0.0) + gamma
    return float(phi), v


# --------------------------------------------------------------------------- NEXT-3 references
def normsq_hopf_lax(x, t, j, h):
    """Closed forms / 1-D searches for J = 1/2||.||_p^2 (p = 1: j="l1sq", p = inf: j="linfsq")
    from the Hopf-Lax formula phi = min_y J(y) + t L((x - y)/t), L = H* the indicator of the
    dual unit ball — no split Bregman, no prox:
      l1sq,   H = l1  : y = shrink_1(x, t) coordinatewise, phi = 1/2 (sum max(|x_i| - t, 0))^2
      l1sq,   H = linf: ||x - y||_1 <= t removes t of l1 mass, phi = 1/2 max(||x||_1 - t, 0)^2
      linfsq, H = l1  : phi = 1/2 (max_i max(|x_i| - t, 0))^2
      linfsq, H = l2  : phi = 1/2 s^2, s the least level with dist_2(x, [-s, s]^n) <= t
                        (bisection on sum max(|x_i| - s, 0)^2 = t^2)
    Returns phi only (grad is not unique for linfsq)."""
    x = np.asarray(x, np.float64)
    if j == "l1sq" and h == "l1":
        return 0.5 * np.sum(np.maximum(np.abs(x) - t, 0.0)) ** 2
    if j == "l1sq" and h == "linf":
        return 0.5 * max(np.abs(x).sum() - t, 0.0) ** 2
    if j == "linfsq" and h == "l1":
        return 0.5 * max(np.abs(x).max() - t, 0.0) ** 2
    if j == "linfsq" and h == "l2":
        a = np.abs(x)
        f = lambda s: np.sum(np.maximum(a - s, 0.0) ** 2) - t * t
        if f(0.0) <= 0:
            return 0.0
        lo, hi = 0.0, float(a.max())
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            if f(mid) > 0:
                lo = mid
            else:
                hi = mid
        return 0.5 * (0.5 * (lo + hi)) ** 2
    raise KeyError((j, h))
