"""Pins of the fp64 oracle (oracle/hopf_oracle.c) to things other than itself.

Each test compares the split Bregman oracle with a plain definition of the same
quantity from the paper (closed forms, the secular equation, Hopf-Lax box QP,
weak-duality certificates, exhaustive search, PDE invariants).  A dropped term,
a wrong sign, a wrong index or a transposed operand in the oracle fails at least
one of them.  "tight" runs use tol = 1e-26 on the squared norms so the iterate
is at the fixed point to fp64 precision; "paper" runs use tol = 1e-8.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import exact
from paper_1605_01799_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")
TIGHT = dict(tol=1e-26, max_iter=200000)


def _diag_case(case):
    n = case["n"]
    D = np.broadcast_to(np.asarray(case["D"], float), (n,)).copy()
    return n, D


@pytest.mark.parametrize("case", json.load(open(GOLD))["cases"], ids=lambda c: c["name"])
def test_golden_paper_examples(case):
    n, D = _diag_case(case)
    X = np.asarray(case["x"], float)[None, :]
    t = np.asarray([case["t"]])
    for kw in (TIGHT, dict(tol=1e-8, max_iter=1000)):
        phi, g, it = oracle.eval_diag(X, t, D, None, case["gamma"], case["h"], **kw)
        assert it[0] >= 1
        assert abs(phi[0] - case["phi"]) <= 1e-9, (phi, case)
        np.testing.assert_allclose(g[0], case["grad"], atol=1e-9 if kw is TIGHT else 2e-4)


def test_c1_closed_form_and_three_iterations():
    """C1: J = 1/2||x||^2, H = l1: phi = 1/2 sum max(|x_i|-t,0)^2, grad = shrink_1(x,t)
    (P:248-263 with a_i = 1, constant dropped).  With lambda = 1 the iteration is exact
    after two steps and the paper's test fires at k = 3 (v1 = x, d1 = d2 = shrink, v2 = v3 = d1)."""
    wl = inputs.config("c1")
    X, t = inputs.points(wl)
    phi, g, it = oracle.eval_diag(X, t, wl.D, None, wl.gamma, "l1")
    pe, ge = exact.diag_wl1_closed(X, t, wl.D)
    assert np.all(it == 3)
    np.testing.assert_allclose(phi, pe, rtol=0, atol=1e-12)
    np.testing.assert_allclose(g, ge, rtol=0, atol=1e-12)
    # same for H = l2 (shrink_2): exact after two steps as well
    phi2, g2, it2 = oracle.eval_diag(X, t, wl.D, None, 0.0, "l2")
    pe2, ge2 = exact.diag_l2_secular(X, t, wl.D)
    assert np.all(it2 == 3)
    np.testing.assert_allclose(phi2, pe2, atol=1e-12)
    np.testing.assert_allclose(g2, ge2, atol=1e-12)


def test_c2_weighted_l1_ellipsoid_closed_form():
    wl = inputs.config("c2")
    X, t = inputs.points(wl, 0, 400)
    pe, ge = exact.diag_wl1_closed(X, t, wl.D, None, wl.gamma, wl.w)
    phi, g, it = oracle.eval_diag(X, t, wl.D, None, wl.gamma, "wl1", wl.w, **TIGHT)
    np.testing.assert_allclose(phi, pe, atol=1e-11)
    np.testing.assert_allclose(g, ge, atol=1e-10)
    # the paper's tolerance: within the north_star parity budget of the exact answer
    phi, g, it = oracle.eval_diag(X, t, wl.D, None, wl.gamma, "wl1", wl.w)
    assert np.all(it > 0)
    assert np.max(np.abs(phi - pe) / np.maximum(1, np.abs(pe))) < 1e-6
    assert np.max(np.abs(g - ge)) < 1e-3


def test_c3_l2_secular_equation():
    wl = inputs.config("c3")
    X, t = inputs.points(wl, 0, 40)
    pe, ge = exact.diag_l2_secular(X, t, wl.D, None, wl.gamma)
    phi, g, it = oracle.eval_diag(X, t, wl.D, None, wl.gamma, "l2", **TIGHT)
    np.testing.assert_allclose(phi, pe, atol=1e-11)
    np.testing.assert_allclose(g, ge, atol=1e-10)
    phi, g, it = oracle.eval_diag(X, t, wl.D, None, wl.gamma, "l2")
    assert np.all(it > 0)
    assert np.max(np.abs(g - ge)) < 1e-3


@pytest.mark.parametrize("lam", [0.5, 2.0])
@pytest.mark.parametrize("h", ["wl1", "l2"])
def test_lambda_does_not_move_the_fixed_point(lam, h):
    """Any lambda > 0 converges to the same minimiser."""
    rng = np.random.default_rng(7)
    n, M = 12, 30
    D = rng.uniform(0.3, 3.0, n)
    c = rng.normal(size=n)
    w = rng.uniform(0.5, 1.5, n)
    X = rng.normal(scale=2.0, size=(M, n))
    t = rng.uniform(0.0, 2.0, M)
    phi, g, it = oracle.eval_diag(X, t, D, c, 0.3, h, w, lam=lam, **TIGHT)
    if h == "l2":
        pe, ge = exact.diag_l2_secular(X, t, D, c, 0.3)
    else:
        pe, ge = exact.diag_wl1_closed(X, t, D, c, 0.3, w)
    np.testing.assert_allclose(phi, pe, atol=1e-10)
    np.testing.assert_allclose(g, ge, atol=1e-9)


def test_dense_identity_rotation_reduces_to_separable():
    """Q = I: A = diag(Lam) => grad_i = Lam_i shrink_1(x,t)_i, phi = 1/2 sum Lam_i max(|x_i|-t,0)^2."""
    rng = np.random.default_rng(3)
    n, M = 16, 50
    Lam = np.exp(rng.uniform(np.log(0.1), np.log(10), n))
    X = rng.normal(size=(M, n))
    t = rng.uniform(0.1, 1.0, M)
    phi, g, it = oracle.eval_dense(X, t, np.eye(n), Lam, **TIGHT)
    pe, ge = exact.diag_wl1_closed(X, t, 1.0 / Lam)
    np.testing.assert_allclose(phi, pe, atol=1e-10)
    np.testing.assert_allclose(g, ge, atol=1e-9)


def test_dense_against_box_qp_bruteforce():
    """Random rotation, n = 5: exhaustive 3^n active-set enumeration of the Hopf-Lax box QP."""
    rng = np.random.default_rng(11)
    n = 5
    Q = inputs.haar_orthogonal(rng, n)
    Lam = np.exp(rng.uniform(np.log(0.1), np.log(10), n))
    A = (Q * Lam) @ Q.T
    X = rng.normal(size=(12, n))
    t = rng.uniform(0.1, 1.0, 12)
    w = rng.uniform(0.5, 1.5, n)
    for h, ww in (("l1", None), ("wl1", w)):
        phi, g, it = oracle.eval_dense(X, t, Q, Lam, 0.25, h, ww, **TIGHT)
        for p in range(X.shape[0]):
            pb, gb, _ = exact.box_qp_bruteforce(X[p], t[p], A, ww, 0.25)
            assert abs(phi[p] - pb) < 1e-10
            np.testing.assert_allclose(g[p], gb, atol=1e-8)


def test_dense_t0_branch_initial_value():
    """Dense t = 0 branch (reading R6; (1.1b) P:95-98, Hopf needs t > 0 P:106-107):
    phi(x,0) = J(x) = 1/2<x,Ax> + gamma and grad = A x, with A = Q diag(Lam) Q^T.
    Pinned three ways, none of which is the oracle's own branch:
      (i)  the n = 5 Hopf-Lax box QP at t = 0 by 3^n KKT enumeration (the box is the point x),
      (ii) continuity: the split Bregman branch at t = 1e-9 (itself pinned by the certificate
           and brute-force tests) agrees with the t = 0 branch,
      (iii) Q = I reduces to the separable closed form at t = 0.
    A mistake such as A^{-1} for A, a dropped 1/2 or a dropped gamma fails each of them."""
    rng = np.random.default_rng(41)
    for n in (5, 24):
        Q = inputs.haar_orthogonal(rng, n)
        Lam = np.exp(rng.uniform(np.log(0.1), np.log(10), n))
        X = rng.normal(size=(8, n))
        gamma = 0.375
        phi0, g0, it0 = oracle.eval_dense(X, np.zeros(8), Q, Lam, gamma, "l1")
        assert np.all(it0 == 0)
        if n == 5:
            A = (Q * Lam) @ Q.T
            for p in range(8):
                pb, gb, _ = exact.box_qp_bruteforce(X[p], 0.0, A, None, gamma)
                assert abs(phi0[p] - pb) < 1e-12
                np.testing.assert_allclose(g0[p], gb, atol=1e-12)
        phie, ge, ite = oracle.eval_dense(X, np.full(8, 1e-9), Q, Lam, gamma, "l1", **TIGHT)
        assert np.all(ite > 0)
        np.testing.assert_allclose(phi0, phie, atol=1e-7 * (1 + np.abs(phie)).max())
        np.testing.assert_allclose(g0, ge, atol=1e-7)
    Lam = np.exp(rng.uniform(np.log(0.1), np.log(10), 9))
    X = rng.normal(size=(6, 9))
    phi0, g0, _ = oracle.eval_dense(X, np.zeros(6), np.eye(9), Lam, -0.25, "wl1",
                                    rng.uniform(0.5, 1.5, 9))
    pe, ge = exact.diag_wl1_closed(X, np.zeros(6), 1.0 / Lam, None, -0.25)
    np.testing.assert_allclose(phi0, pe, atol=1e-12)
    np.testing.assert_allclose(g0, ge, atol=1e-12)


def test_dense_c4_duality_certificate():
    """C4 law at n = 256: L(v) <= phi <= U(z) with a certified gap, and the box-QP
    coordinate-descent Hopf-Lax solve agrees."""
    wl = inputs.config("c4")
    X, t = inputs.points(wl, 0, 6)
    A, Ainv, Ml = oracle.dense_matrices(wl.Q, wl.Lam)
    phi, g, it = oracle.eval_dense(X, t, wl.Q, wl.Lam, **TIGHT)
    lmax = wl.Lam.max()
    for p in range(X.shape[0]):
        L = exact.dual_lower_bound(X[p], t[p], g[p], Ainv)
        U = exact.primal_upper_bound(X[p], t[p], g[p], A, Ainv)
        assert L - 1e-9 <= phi[p] <= U + 1e-9
        assert U - L < 1e-9
        # ||v - v*||^2 <= 2 lambda_max(A) (U - L) (strong convexity of J*)
    pq, gq, _ = exact.box_qp_hopf_lax(X[0], t[0], A, sweeps=4000, tol=1e-14)
    assert abs(pq - phi[0]) < 1e-8
    np.testing.assert_allclose(gq, g[0], atol=1e-6)
    # paper tolerance: within budget
    phi8, g8, it8 = oracle.eval_dense(X, t, wl.Q, wl.Lam)
    assert np.all(it8 > 0)
    assert np.max(np.abs(g8 - g)) < 1e-3
    assert np.max(np.abs(phi8 - phi) / np.maximum(1, np.abs(phi))) < 1e-6


def test_union_c5_secular_and_closest_point():
    wl = inputs.config("c5")
    X, t = inputs.points(wl, 0, 30)
    Dk, Ck, gk = wl.Dk.astype(float), wl.Ck.astype(float), wl.gammak.astype(float)
    pe, ge, kse, pke = exact.union_exact(X, t, Dk, Ck, gk, "l2")
    phi, g, it, Y, ks, pk = oracle.eval_union(X, t, Dk, Ck, gk, "l2", **TIGHT)
    np.testing.assert_allclose(pk, pke, atol=1e-10)
    np.testing.assert_allclose(phi, pe, atol=1e-10)
    assert np.array_equal(ks, kse)
    np.testing.assert_allclose(g, ge, atol=1e-9)
    # closest / Hopf-Lax point: ||x - y|| = t and J_k*(y) = phi when grad != 0
    for p in range(X.shape[0]):
        k = ks[p]
        Jy = 0.5 * np.sum((Y[p] - Ck[k]) ** 2 / Dk[k]) + gk[k]
        if np.linalg.norm(g[p]) > 0:
            assert abs(np.linalg.norm(X[p] - Y[p]) - t[p]) < 1e-9
            assert abs(Jy - phi[p]) < 1e-8
        else:
            np.testing.assert_allclose(Y[p], Ck[k])


def test_union_fig4_fixture():
    """Fig. 4: J = min(1/2||x||^2 - <b,x>, 1/2||x||^2 + <b,x>), b = 1^8, H = l1.
    Branch k is D = 1, c = +-b, gamma = -1/2||b||^2; closed form per branch; iters = 3."""
    n = 8
    b = np.ones(n)
    Dk = np.ones((2, n))
    Ck = np.stack([b, -b])
    gk = np.full(2, -0.5 * b @ b)
    rng = np.random.default_rng(5)
    X = rng.uniform(-20, 20, (200, n))
    t = rng.uniform(0, 15, 200)
    phi, g, it, Y, ks, pk = oracle.eval_union(X, t, Dk, Ck, gk, "l1", want_y=False)
    for k in range(2):
        pe, _ = exact.diag_wl1_closed(X, t, Dk[k], Ck[k], gk[k])
        np.testing.assert_allclose(pk[:, k], pe, atol=1e-10)
    np.testing.assert_allclose(phi, pk.min(axis=1), atol=0)
    assert np.all((it == 3) | (it == 0))


@pytest.mark.parametrize("h", ["l1", "wl1", "l2"])
def test_bruteforce_n2_hopf_and_hopf_lax(h):
    """n = 2: the oracle matches (i) the Hopf formula (3.3) minimised by exhaustive grid search
    over v and (ii) the Hopf-Lax formula min_{z in x - tC} J(z) by grid search (north_star)."""
    rng = np.random.default_rng(19)
    D = np.array([0.7, 1.8])
    c = np.array([0.3, -0.4])
    w = np.array([0.6, 1.4]) if h == "wl1" else np.ones(2)
    gamma = -0.5
    for _ in range(6):
        x = rng.normal(scale=2.0, size=2)
        t = rng.uniform(0.2, 1.5)
        phi, g, it = oracle.eval_diag(x[None], np.array([t]), D, c, gamma, h, w, **TIGHT)
        Jstar = lambda V: 0.5 * np.sum(D * V * V, axis=1) + V @ c - gamma
        Hf = (lambda V: np.linalg.norm(V, axis=1)) if h == "l2" else (lambda V: np.abs(V) @ w)
        pd, vd = exact.hopf_dual_grid_2d(x, t, Jstar, Hf, radius=10.0)
        J = lambda Z: 0.5 * np.sum((Z - c) ** 2 / D, axis=1) + gamma
        pl, _ = exact.hopf_lax_grid_2d(x, t, J, "l2" if h == "l2" else "box", w)
        assert abs(phi[0] - pd) < 1e-7, (phi, pd)
        assert abs(phi[0] - pl) < 1e-7, (phi, pl)
        np.testing.assert_allclose(g[0], vd, atol=1e-4)


def test_bruteforce_n2_union_hopf_lax():
    """Union of two ellipses in n = 2: min_k phi_k equals Hopf-Lax with J = min_k J_k."""
    rng = np.random.default_rng(23)
    Dk = np.array([[0.5, 2.0], [1.5, 0.7]])
    Ck = np.array([[2.0, 0.0], [-1.0, 1.5]])
    gk = np.array([-0.5, -0.5])
    J = lambda Z: np.min(np.stack([0.5 * np.sum((Z - Ck[k]) ** 2 / Dk[k], axis=1) + gk[k]
                                   for k in range(2)]), axis=0)
    for _ in range(6):
        x = rng.normal(scale=3.0, size=2)
        t = rng.uniform(0.2, 1.5)
        phi, g, it, Y, ks, pk = oracle.eval_union(x[None], np.array([t]), Dk, Ck, gk, "l2", **TIGHT)
        pl, yl = exact.hopf_lax_grid_2d(x, t, J, "l2")
        assert abs(phi[0] - pl) < 1e-7
        if np.linalg.norm(g[0]) > 0:
            np.testing.assert_allclose(Y[0], yl, atol=1e-4)


def test_union_zero_gradient_closest_point_is_centre():
    """Reading R18: grad phi = 0 (||x - c_k*|| <= t) => y = c_k*, the Hopf-Lax minimiser
    argmin_{||z - x|| <= t} min_k J_k(z).  Pinned to (i) the n = 2 Hopf-Lax grid
    argmin and (ii) at n = 64 to the defining properties of that minimiser: y is feasible
    (||x - y|| <= t) and attains phi (min_k J_k(y) = phi), which returning x (or any other point
    than the centre) violates because J_k is strictly convex with its minimum gamma_k at c_k."""
    # (i) n = 2, three ellipses with distinct levels (no ties), points inside a ball around a centre
    Dk = np.array([[0.5, 2.0], [1.5, 0.7], [1.0, 1.0]])
    Ck = np.array([[2.0, 0.0], [-1.0, 1.5], [0.5, -2.0]])
    gk = np.array([-0.5, -0.8, -0.3])
    J = lambda Z: np.min(np.stack([0.5 * np.sum((Z - Ck[k]) ** 2 / Dk[k], axis=1) + gk[k]
                                   for k in range(3)]), axis=0)
    rng = np.random.default_rng(43)
    hits = 0
    for _ in range(12):
        k = rng.integers(3)
        x = Ck[k] + rng.normal(scale=0.3, size=2)
        t = np.linalg.norm(x - Ck[k]) + rng.uniform(0.05, 0.6)
        phi, g, it, Y, ks, pk = oracle.eval_union(x[None], np.array([t]), Dk, Ck, gk, "l2", **TIGHT)
        pl, yl = exact.hopf_lax_grid_2d(x, t, J, "l2")
        assert abs(phi[0] - pl) < 1e-7
        if np.all(g[0] == 0):
            hits += 1
            np.testing.assert_allclose(Y[0], yl, atol=1e-4)
            np.testing.assert_allclose(Y[0], Ck[ks[0]], atol=0)
            assert abs(phi[0] - gk[ks[0]]) < 1e-12
    assert hits >= 6
    # (ii) n = 64 with C5's sets: points near a centre, t beyond the distance
    wl = inputs.config("c5")
    Dk, Ck, gk = wl.Dk.astype(float), wl.Ck.astype(float), wl.gammak.astype(float)
    gk = gk - 0.05 * np.arange(len(gk))          # distinct levels: a unique winner
    K, n = Dk.shape
    X = Ck[np.arange(20) % K] + rng.normal(scale=0.2, size=(20, n))
    t = np.linalg.norm(X - Ck[np.arange(20) % K], axis=1) + 0.5
    phi, g, it, Y, ks, pk = oracle.eval_union(X, t, Dk, Ck, gk, "l2")
    Jk = lambda z: min(0.5 * np.sum((z - Ck[k]) ** 2 / Dk[k]) + gk[k] for k in range(K))
    zero = np.all(g == 0, axis=1)
    assert zero.sum() >= 10
    for p in np.nonzero(zero)[0]:
        assert np.linalg.norm(X[p] - Y[p]) <= t[p] + 1e-12
        assert abs(Jk(Y[p]) - phi[p]) < 1e-12
        assert abs(phi[p] - min(pk[p])) == 0


def test_dense_and_union_status_codes_and_ties():
    """Status conventions of the ABI on the dense and union branches, and the union
    tie rule R19 (lowest k wins): a duplicated set can never win over its first copy."""
    rng = np.random.default_rng(47)
    n = 6
    Q = inputs.haar_orthogonal(rng, n)
    Lam = np.exp(rng.uniform(np.log(0.1), np.log(10), n))
    X = rng.normal(size=(4, n))
    X[2, 1] = np.inf
    t = np.array([0.5, -0.1, 0.5, 0.3])
    phi, g, it = oracle.eval_dense(X, t, Q, Lam, 0.0, "l1", max_iter=2)
    assert it[0] == -2 and np.isfinite(phi[0]) and np.all(np.isfinite(g[0]))
    assert it[1] == oracle.INVALID and np.isnan(phi[1]) and np.all(np.isnan(g[1]))
    assert it[2] == oracle.INVALID
    # not converged after 2 iterations: outputs are the Hopf objective at the last d (R1, R2)
    A = (Q * Lam) @ Q.T
    L = exact.dual_lower_bound(X[0], t[0], g[0], np.linalg.inv(A))
    assert abs(phi[0] - L) < 1e-12
    Dk = np.stack([np.full(n, 1.3), np.full(n, 0.8), np.full(n, 1.3)])
    Ck = np.stack([np.zeros(n), np.ones(n), np.zeros(n)])      # set 2 duplicates set 0
    gk = np.array([-0.5, -0.5, -0.5])
    Xu = rng.normal(scale=0.5, size=(40, n))
    tu = rng.uniform(0.1, 1.0, 40)
    tu[5] = np.nan
    phi, g, it, Y, ks, pk = oracle.eval_union(Xu, tu, Dk, Ck, gk, "l2")
    assert ks[5] == -1 and it[5] == oracle.INVALID and np.isnan(phi[5]) and np.all(np.isnan(Y[5]))
    ok = np.arange(40) != 5
    assert np.all(ks[ok] != 2)
    assert np.array_equal(pk[ok, 0], pk[ok, 2])
    assert np.all(ks[ok] == np.argmin(pk[ok], axis=1))


def test_invariants_initial_value_monotone_fd_gradient_pde():
    """phi(x,0+) = J(x); t -> phi nonincreasing (dphi/dt = -H(grad) <= 0);
    grad = central differences of phi in x; PDE residual dphi/dt + H(grad phi) = 0."""
    rng = np.random.default_rng(29)
    n = 6
    D = rng.uniform(0.5, 2.0, n)
    w = rng.uniform(0.5, 1.5, n)
    gamma = -0.5
    for h in ("wl1", "l2"):
        Hf = (lambda p: np.linalg.norm(p)) if h == "l2" else (lambda p: np.abs(p) @ w)
        for _ in range(5):
            x = rng.normal(scale=2.0, size=n)
            J = 0.5 * np.sum(x * x / D) + gamma
            ev = lambda X, T: oracle.eval_diag(np.atleast_2d(X), np.atleast_1d(T), D, None,
                                               gamma, h, w, **TIGHT)
            assert abs(ev(x, 1e-9)[0][0] - J) < 1e-7
            assert ev(x, 0.0)[2][0] == 0 and abs(ev(x, 0.0)[0][0] - J) < 1e-12
            ts = np.linspace(0.05, 3.0, 12)
            ph = ev(np.repeat(x[None], 12, 0), ts)[0]
            assert np.all(np.diff(ph) <= 1e-12)
            t = 0.7
            phi, g, _ = ev(x, t)
            hs = 1e-5
            E = np.eye(n) * hs
            fd = (ev(x[None] + E, np.full(n, t))[0] - ev(x[None] - E, np.full(n, t))[0]) / (2 * hs)
            np.testing.assert_allclose(fd, g[0], atol=1e-6)
            dt = (ev(x, t + hs)[0][0] - ev(x, t - hs)[0][0]) / (2 * hs)
            assert abs(dt + Hf(g[0])) < 1e-6


def test_status_codes_nonconvergence_and_invalid():
    X = np.array([[3.0, -1.0], [1.0, 2.0], [np.nan, 0.0], [1.0, 1.0]])
    t = np.array([0.5, -1.0, 0.5, 0.0])
    D = np.array([1.3, 0.6])
    phi, g, it = oracle.eval_diag(X, t, D, None, 0.0, "l2", max_iter=2)
    assert it[0] == -2 and np.isfinite(phi[0])           # not converged in 2 iterations
    assert it[1] == oracle.INVALID and np.isnan(phi[1])  # t < 0
    assert it[2] == oracle.INVALID and np.all(np.isnan(g[2]))
    assert it[3] == 0 and abs(phi[3] - 0.5 * np.sum(X[3] ** 2 / D)) < 1e-15


# ----------------------------------------------------------------- distance mode (NEXT-1)
def test_distance_sphere_closed_form():
    """Newton in s on psi(y,s) = 0 for a ball: dist = ||y-c|| - r and
    pi(y) = c + r (y-c)/||y-c|| exactly (radial symmetry); interior points return 0, y."""
    rng = np.random.default_rng(11)
    n = 7
    r = 1.7
    c = rng.normal(size=n)
    Y = c + rng.normal(size=(40, n)) * 3.0
    Y[0] = c + 0.3 * r * np.eye(n)[0]          # interior
    D, C, g = np.full((1, n), r * r), c[None], np.array([-0.5])
    dist, proj, psi, grad, ks, nn = oracle.distance_union(Y, D, C, g, tol=1e-14, stol=1e-12)
    rho = np.linalg.norm(Y - c, axis=1)
    out = rho > r
    np.testing.assert_allclose(dist[out], rho[out] - r, rtol=1e-9, atol=1e-9)
    exp = c + r * (Y - c) / rho[:, None]
    np.testing.assert_allclose(proj[out], exp[out], atol=1e-8)
    assert dist[0] == 0.0 and nn[0] == 0 and np.array_equal(proj[0], Y[0])
    assert np.all(nn[out] >= 1)
    # the same on the 2-D unit circle: (3,0) -> (1,0) at 2, (3,4) -> (0.6,0.8) at 4
    d2, p2, *_ = oracle.distance_union(np.array([[3.0, 0.0], [3.0, 4.0]]), np.ones((1, 2)),
                                       np.zeros((1, 2)), np.array([-0.5]), tol=1e-14, stol=1e-12)
    np.testing.assert_allclose(d2, [2.0, 4.0], atol=1e-10)
    np.testing.assert_allclose(p2, [[1.0, 0.0], [0.6, 0.8]], atol=1e-9)


def test_distance_union_matches_exact_projection():
    """Against the plain definition: projection on each ellipsoid by its KKT secular equation
    (bisection, no Hopf formula), minimum over the members."""
    rng = np.random.default_rng(12)
    n, K = 12, 5
    Dk = rng.uniform(0.5, 2.0, (K, n)) ** 2
    Ck = rng.normal(0, 4, (K, n))
    gk = -0.5 * rng.uniform(0.5, 1.5, K)       # scaled ellipsoids: r^2 = -2 gamma
    Y = rng.normal(0, 4, (30, n))
    dist, proj, psi, grad, ks, nn = oracle.distance_union(Y, Dk, Ck, gk, tol=1e-14, stol=1e-12)
    for i in range(len(Y)):
        de, z, k = exact.union_distance_exact(Y[i], Dk, Ck, gk)
        assert abs(dist[i] - de) <= 1e-9 * max(1.0, de)
        np.testing.assert_allclose(proj[i], z, atol=1e-7 * max(1.0, de))
        assert ks[i] == k
        if de > 0:
            # invariants: ||y - pi|| = dist, pi on the boundary of the winner (L_k(pi) = 0)
            assert abs(np.linalg.norm(Y[i] - proj[i]) - dist[i]) <= 1e-9 * max(1.0, de)
            Lk = 0.5 * np.sum((proj[i] - Ck[k]) ** 2 / Dk[k]) + gk[k]
            assert abs(Lk) <= 1e-7
            assert abs(psi[i]) <= 1e-8


# ----------------------------------------------------------------- max over min of H (NEXT-4)
def test_maxh_closed_form_mixed_kinds():
    """J = 1/2||x||^2, H = min(||.||_1, c ||.||_2): phi = max(phi_1, phi_2) with the
    closed forms phi_1 = 1/2 sum max(|x_j| - t, 0)^2 (P:248-263 with a = 1) and
    phi_2 = 1/2 max(||x|| - c t, 0)^2; grad = the winner's."""
    rng = np.random.default_rng(31)
    n, M, cc = 6, 400, 1.7
    X = rng.uniform(-3, 3, (M, n))
    t = rng.uniform(0.1, 1.5, M)
    phi, grad, it, ist = oracle.eval_maxh(X, t, np.ones(n), None, 0.0, ["l1", "l2"], [1.0, cc],
                                          tol=1e-14, max_iter=5000)
    s1 = np.maximum(np.abs(X) - t[:, None], 0.0)
    p1 = 0.5 * np.sum(s1 * s1, axis=1)
    g1 = np.sign(X) * s1
    r = np.linalg.norm(X, axis=1)
    m2 = np.maximum(r - cc * t, 0.0)
    p2 = 0.5 * m2 * m2
    g2 = X * (m2 / r)[:, None]
    exp = np.maximum(p1, p2)
    np.testing.assert_allclose(phi, exp, rtol=1e-9, atol=1e-9)
    win2 = p2 > p1 + 1e-9
    win1 = p1 > p2 + 1e-9
    assert np.all(ist[win2] == 1) and np.all(ist[win1] == 0)
    np.testing.assert_allclose(grad[win1], g1[win1], atol=1e-6)
    np.testing.assert_allclose(grad[win2], g2[win2], atol=1e-6)


def test_maxh_matches_hopf_formula_with_min_hamiltonian_2d():
    """n = 2: the Hopf formula with the nonconvex H = min_i H_i minimised by exhaustive search
    (no split Bregman, no max identity) equals the oracle's max_i phi_i."""
    D = np.array([0.7, 1.6])
    w = np.array([[1.0, 1.0], [0.4, 1.8]])
    kinds, a = ["wl1", "wl1", "l2"], [1.0, 1.0, 1.3]
    W = np.stack([w[0], w[1], np.ones(2)])
    Jstar = lambda V: 0.5 * (V * V) @ D
    Hmin = lambda V: np.minimum(np.minimum(np.abs(V) @ w[0], np.abs(V) @ w[1]),
                                1.3 * np.linalg.norm(V, axis=1))
    rng = np.random.default_rng(32)
    X = rng.uniform(-3, 3, (6, 2))
    t = rng.uniform(0.2, 1.2, 6)
    phi, grad, it, ist = oracle.eval_maxh(X, t, D, None, 0.0, kinds, a, W, tol=1e-14, max_iter=5000)
    for i in range(len(X)):
        ref, vbest = exact.hopf_dual_grid_2d(X[i], t[i], Jstar, Hmin, 8.0)
        assert abs(phi[i] - ref) <= 1e-6 * max(1.0, abs(ref)), (i, phi[i], ref)
        np.testing.assert_allclose(grad[i], vbest, atol=1e-3)


# ----------------------------------------------------------------- ellipsoidal-norm H (NEXT-2)
def test_ell_hamiltonian_matches_secular_reference():
    """H(p) = sqrt(<p, W p>) (Moreau + projection on the dual ellipsoid by Newton
    on mu from mu_0 = 0): against the plain optimality condition solved by bisection."""
    rng = np.random.default_rng(41)
    n, M = 9, 60
    D = np.exp(rng.uniform(np.log(0.5), np.log(2.0), n))
    W = np.exp(rng.uniform(np.log(0.3), np.log(3.0), n))
    c = rng.normal(size=n)
    X = rng.normal(0, 2, (M, n))
    t = rng.uniform(0.05, 2.0, M)
    t[0] = 0.0
    X[1] = c + 0.01   # inside t W-ball: grad 0
    phi, grad, it = oracle.eval_diag(X, t, D, c, -0.5, "ell", W, tol=1e-22, max_iter=20000)
    for i in range(M):
        pe, ge = exact.diag_ell_secular(X[i], t[i], D, W, c, -0.5)
        assert abs(phi[i] - pe) <= 1e-9 * max(1.0, abs(pe)), i
        np.testing.assert_allclose(grad[i], ge, atol=1e-6)
    assert it[0] == 0 and np.all(grad[1] == 0.0)


def test_ell_with_identity_weights_is_l2():
    """W = I: ||.||_W = ||.||_2, the prox by ellipsoid projection must reproduce shrink_2."""
    rng = np.random.default_rng(42)
    n, M = 12, 200
    D = np.exp(rng.uniform(np.log(0.5), np.log(2.0), n))
    X = rng.normal(0, 1.5, (M, n))
    t = rng.uniform(0.1, 2.0, M)
    a = oracle.eval_diag(X, t, D, None, -0.5, "ell", np.ones(n))
    b = oracle.eval_diag(X, t, D, None, -0.5, "l2")
    np.testing.assert_allclose(a[0], b[0], rtol=1e-7, atol=1e-7)
    np.testing.assert_allclose(a[1], b[1], atol=1e-5)
    assert np.mean(np.abs(a[2] - b[2]) <= 1) > 0.95


def test_maxh_ell_member_is_time_scaled_ell_solve():
    """a ||p||_W with a single Hamiltonian: the ellipsoidal solve at time a t (t a H = (a t) H)."""
    rng = np.random.default_rng(43)
    n, M = 7, 40
    D = rng.uniform(0.5, 2.0, n)
    W = rng.uniform(0.5, 1.5, (1, n))
    X = rng.normal(0, 2, (M, n))
    t = rng.uniform(0.1, 1.0, M)
    m = oracle.eval_maxh(X, t, D, None, 0.3, ["ell"], np.array([1.7]), W)
    d = oracle.eval_diag(X, 1.7 * t, D, None, 0.3, "ell", W[0])
    np.testing.assert_array_equal(m[0], d[0])
    np.testing.assert_array_equal(m[1], d[1])
    assert np.all(m[3] == 0)


# ----------------------------------------------------------------- l_inf H (NEXT-2)
def test_linf_hamiltonian_matches_bisection_reference():
    """H = ||.||_inf (Moreau + projection on the l1 ball by sorted breakpoints and
    interpolation): against the plain level-set maximisation solved by bisection."""
    rng = np.random.default_rng(51)
    n, M = 10, 80
    D = np.exp(rng.uniform(np.log(0.5), np.log(2.0), n))
    c = rng.normal(size=n)
    X = rng.normal(0, 3, (M, n))
    t = rng.uniform(0.05, 4.0, M)
    t[0] = 0.0
    X[1] = c + 0.01          # ||x - c||_1 small: grad 0
    X[2, 3] = X[2, 4]        # duplicate breakpoints
    phi, grad, it = oracle.eval_diag(X, t, D, c, 0.25, "linf", None, tol=1e-22, max_iter=20000)
    for i in range(M):
        pe, ge = exact.diag_linf_bisection(X[i], t[i], D, c, 0.25)
        assert abs(phi[i] - pe) <= 1e-9 * max(1.0, abs(pe)), i
        np.testing.assert_allclose(grad[i], ge, atol=1e-6)
    assert it[0] == 0 and np.all(grad[1] == 0.0)


def test_linf_in_one_dimension_is_l1():
    """n = 1: ||.||_inf = ||.||_1 = |.|; the l1-ball projection must reproduce shrink_1."""
    rng = np.random.default_rng(52)
    X = rng.normal(0, 3, (300, 1))
    t = rng.uniform(0.0, 3.0, 300)
    a = oracle.eval_diag(X, t, np.array([0.7]), None, 0.0, "linf")
    b = oracle.eval_diag(X, t, np.array([0.7]), None, 0.0, "l1")
    np.testing.assert_allclose(a[0], b[0], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(a[1], b[1], atol=1e-12)
    np.testing.assert_array_equal(a[2], b[2])


def test_linf_isotropic_hopf_lax_closed_form():
    """J = 1/2||.||^2, H = ||.||_inf: Hopf-Lax with L = H* = indicator of the unit l1 ball gives
    phi(x,t) = 1/2 min_{||x - y||_1 <= t} ||y||^2, i.e. y = x - pi_{tB1}(x) with pi the Euclidean
    projection on the l1 ball of radius t, here found by sorting (Duchi et al.'s formula: the
    largest k with |x|_(k) > (sum_{j<=k} |x|_(j) - t)/k), not the oracle's breakpoint search."""
    rng = np.random.default_rng(53)
    n, M = 6, 100
    X = rng.normal(0, 3, (M, n))
    t = rng.uniform(0.1, 8.0, M)
    phi, grad, _ = oracle.eval_diag(X, t, np.ones(n), None, 0.0, "linf", None, tol=1e-24,
                                    max_iter=20000)
    for i in range(M):
        x, tt = X[i], t[i]
        if np.abs(x).sum() <= tt:
            y = np.zeros(n)
        else:
            a = np.sort(np.abs(x))[::-1]
            cs = np.cumsum(a)
            k = max(j for j in range(1, n + 1) if a[j - 1] > (cs[j - 1] - tt) / j)
            theta = (cs[k - 1] - tt) / k
            p = np.sign(x) * np.maximum(np.abs(x) - theta, 0.0)
            y = x - p
        assert abs(phi[i] - 0.5 * y @ y) <= 1e-9 * max(1.0, phi[i])
        np.testing.assert_allclose(grad[i], y, atol=1e-6)   # grad phi = grad J(y) = y


# ----------------------------------------------------------------- NEXT-3 (non-quadratic J)
@pytest.mark.parametrize("j,h", [("l1sq", "l1"), ("l1sq", "linf"), ("linfsq", "l1"), ("linfsq", "l2")])
def test_normsq_hopf_lax_closed_forms(j, h):
    """J = 1/2||.||_1^2 or 1/2||.||_inf^2 (Tables 2-3, 5): phi against the Hopf-Lax
    closed forms / 1-D searches of exact.normsq_hopf_lax; grad satisfies the Hopf optimality
    (the objective at grad equals phi)."""
    rng = np.random.default_rng(61 + len(j) + len(h))
    n, M = 6, 120
    X = rng.uniform(-10, 10, (M, n))
    t = rng.uniform(0.0, 10.0, M)
    t[0] = 0.0
    phi, grad, it = oracle.eval_normsq(X, t, j, 0.0, h, tol=1e-24, max_iter=50000)
    for i in range(M):
        pe = exact.normsq_hopf_lax(X[i], t[i], j, h)
        assert abs(phi[i] - pe) <= 1e-7 * max(1.0, pe), (i, phi[i], pe)
    assert it[0] == 0
    # grad attains the Hopf sup: <x,g> - J*(g) - t H(g) = phi (J* of the dual norm)
    js = (np.abs(grad).max(axis=1) if j == "l1sq" else np.abs(grad).sum(axis=1))
    hv = {"l1": np.abs(grad).sum(axis=1), "linf": np.abs(grad).max(axis=1),
          "l2": np.linalg.norm(grad, axis=1)}[h]
    obj = np.einsum("ij,ij->i", X, grad) - 0.5 * js ** 2 - t * hv
    np.testing.assert_allclose(obj[1:], phi[1:], rtol=1e-7, atol=1e-7)


def test_normsq_t0_and_subgradients():
    """t = 0: J(x) and the minimal-norm subgradient (reading R30)."""
    X = np.array([[3.0, -1.0, 0.0, 2.0], [-2.0, 2.0, 1.0, 0.5]])
    t = np.zeros(2)
    p1, g1, i1 = oracle.eval_normsq(X, t, "l1sq")
    np.testing.assert_allclose(p1, [18.0, 15.125])
    np.testing.assert_allclose(g1[0], [6.0, -6.0, 0.0, 6.0])
    p2, g2, _ = oracle.eval_normsq(X, t, "linfsq")
    np.testing.assert_allclose(p2, [4.5, 2.0])
    np.testing.assert_allclose(g2[0], [3.0, 0.0, 0.0, 0.0])
    np.testing.assert_allclose(g2[1], [-1.0, 1.0, 0.0, 0.0])
    assert np.all(i1 == 0)


@pytest.mark.parametrize("j", ["l1sq", "linfsq"])
def test_normsq_bruteforce_n2(j):
    """n = 2, H = l2 and weighted l1: the Hopf formula maximised by brute force on a fine grid."""
    rng = np.random.default_rng(71)
    X = rng.uniform(-3, 3, (12, 2))
    t = rng.uniform(0.2, 2.0, 12)
    g = np.linspace(-6, 6, 1201)
    V1, V2 = np.meshgrid(g, g, indexing="ij")
    js = (np.maximum(np.abs(V1), np.abs(V2)) if j == "l1sq" else np.abs(V1) + np.abs(V2))
    w = np.array([0.7, 1.3])
    for h in ("l2", "wl1"):
        phi, _, _ = oracle.eval_normsq(X, t, j, 0.0, h, w, tol=1e-20, max_iter=50000)
        Hv = np.hypot(V1, V2) if h == "l2" else w[0] * np.abs(V1) + w[1] * np.abs(V2)
        for i in range(len(X)):
            obj = X[i, 0] * V1 + X[i, 1] * V2 - 0.5 * js ** 2 - t[i] * Hv
            assert abs(obj.max() - phi[i]) <= 2e-3 * max(1.0, abs(phi[i])), (h, i)


# ----------------------------------------------------------------- ||.||_A, full SPD A (NEXT-2)
def _paper_A(n):
    """The paper's A: A_ii = 2, A_ij = 1."""
    return np.ones((n, n)) + np.eye(n)


def test_ellA_diagonal_A_is_ell():
    """A = diag(w): the rotated projection must reproduce the diagonal ellipsoid solve."""
    rng = np.random.default_rng(81)
    n, M = 7, 100
    w = rng.uniform(0.5, 2.0, n)
    D = rng.uniform(0.5, 2.0, n)
    X = rng.normal(0, 2, (M, n))
    t = rng.uniform(0, 2, M)
    a = oracle.eval_diag_A(X, t, D, None, 0.1, np.diag(w))
    b = oracle.eval_diag(X, t, D, None, 0.1, "ell", w)
    np.testing.assert_allclose(a[0], b[0], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(a[1], b[1], atol=1e-7)


def test_ellA_isotropic_J_rotation_invariance():
    """J = 1/2||.||^2 is rotation invariant, so phi_A(x) = phi_W(Q^T x) with W = eig(A) and
    grad_A = Q grad_W (the ellipsoid solve in the eigenbasis), for the paper's A."""
    rng = np.random.default_rng(82)
    n, M = 8, 60
    A = _paper_A(n)
    Lam, Q = np.linalg.eigh(A)
    X = rng.uniform(-10, 10, (M, n))
    t = rng.uniform(0, 10, M)
    a = oracle.eval_diag_A(X, t, np.ones(n), None, 0.0, A, tol=1e-20, max_iter=20000)
    b = oracle.eval_diag(X @ Q, t, np.ones(n), None, 0.0, "ell", Lam, tol=1e-20, max_iter=20000)
    np.testing.assert_allclose(a[0], b[0], rtol=1e-8, atol=1e-8)
    np.testing.assert_allclose(a[1], b[1] @ Q.T, atol=1e-6)


def test_ellA_bruteforce_n2():
    """n = 2: the Hopf formula with H = sqrt(<p, A p>) maximised by brute force on a grid."""
    rng = np.random.default_rng(83)
    A = np.array([[2.0, 0.7], [0.7, 1.0]])
    D = np.array([0.8, 1.5])
    X = rng.uniform(-3, 3, (10, 2))
    t = rng.uniform(0.2, 2.0, 10)
    phi, _, _ = oracle.eval_diag_A(X, t, D, None, 0.0, A, tol=1e-20, max_iter=50000)
    g = np.linspace(-6, 6, 1201)
    V1, V2 = np.meshgrid(g, g, indexing="ij")
    Hv = np.sqrt(A[0, 0] * V1 ** 2 + 2 * A[0, 1] * V1 * V2 + A[1, 1] * V2 ** 2)
    for i in range(len(X)):
        obj = X[i, 0] * V1 + X[i, 1] * V2 - 0.5 * (D[0] * V1 ** 2 + D[1] * V2 ** 2) - t[i] * Hv
        assert abs(obj.max() - phi[i]) <= 2e-3 * max(1.0, abs(phi[i])), i
