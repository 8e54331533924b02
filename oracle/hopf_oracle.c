/*
 * hopf_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU implementation of the split Bregman
 * evaluation of the Hopf formula (Darbon & Osher, arXiv 1605.01799).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It shares no code, header, table or
 * constant generator with the CUDA product path (paper_1605_01799_b200/csrc).
 *
 * Citations are PAPER.md line numbers ("P:n") with the equation label.
 *
 *   Hopf formula (1.2)/(3.3), P:135-142, P:815-818:
 *       phi(x,t) = -min_v { J*(v) + t H(v) - <x,v> }
 *   Split Bregman (3.4a)-(3.4c), lambda, v0=d0=x, b0=0 at P:842-844:
 *       v^{k+1} = argmin_v J*(v) - <x,v> + lambda/2 ||d^k - v - b^k||^2
 *       d^{k+1} = argmin_d t H(d) + lambda/2 ||d - v^{k+1} - b^k||^2
 *       b^{k+1} = b^k + v^{k+1} - d^{k+1}
 *   Stopping rule, P:1595-1601 (squared l2 norms, all three, every iteration):
 *       ||v^k-v^{k-1}||^2 <= tol  and ||d^k-d^{k-1}||^2 <= tol and ||d^k-v^k||^2 <= tol
 *   shrink_1 (soft threshold), P:239-247 (sign(0)=+1 at P:1322);
 *   shrink_2.
 *   Quadratic prox.
 *   Min over initial data (union).
 *   Closest point y = x - t grad/||grad||.
 *   Distance to a union (NEXT-1): Newton in s on psi(y,s) = 0 (eq. Newton_zero,
 *   P:1096-1108) with d psi/dt = -||grad psi||, psi = min_k psi_k
 *   for the union, pi_Omega(y) = y - s grad/||grad||.
 *
 * Readings of the paper: R1 grad := d at stop,
 * R2 phi := Hopf objective at d, R3 tol on squared norms, R5 shifted problems
 * solved centred at x - c with v0 = d0 = x - c, R6 t == 0 answered by J(x),
 * R8 shrink at the threshold -> 0, R18 y := c_k* when grad == 0, R19 lowest k
 * wins ties.
 *
 * Initial data handled:
 *   diag : J(x) = 1/2 <x-c, D^{-1}(x-c)> + gamma,  J*(v) = 1/2<v,Dv> + <c,v> - gamma
 *   dense: J(x) = 1/2 <x, A x> + gamma,            J*(v) = 1/2<v,A^{-1}v> - gamma
 * Hamiltonians: H_L1 (sum |p_i|), H_WL1 (sum w_i |p_i|), H_L2 (||p||_2).
 *
 * Per-point status in iters[i] (same convention as the product ABI):
 *   k >= 1 converged at iteration k; 0: t == 0; -max_iter: not converged;
 *   INT32_MIN: invalid point (t < 0 or non-finite input), phi/grad = NaN.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_H_L1 0
#define ORACLE_H_WL1 1
#define ORACLE_H_L2 2
#define ORACLE_H_ELL 3 /* NEXT-2: H(p) = sqrt(<p, W p>), W = diag(w) > 0 */
#define ORACLE_H_LINF 4 /* NEXT-2: H(p) = ||p||_inf */

/* ---------------- prox of t/lambda * H (3.4b) ---------------------------- */

/* shrink_1 with per-coordinate threshold alpha_i. */
static void shrink1(int n, const double *u, const double *alpha, double *out) {
  for (int i = 0; i < n; i++) {
    double a = fabs(u[i]) - alpha[i];
    double s = (u[i] >= 0.0) ? 1.0 : -1.0; /* sign(0) = +1 */
    out[i] = (a > 0.0) ? s * a : 0.0;      /* |u_i| <= alpha -> 0 */
  }
}

/* shrink_2: u/||u|| * max(||u|| - alpha, 0); 0 if u == 0. */
static void shrink2(int n, const double *u, double alpha, double *out) {
  double r2 = 0.0;
  for (int i = 0; i < n; i++) r2 += u[i] * u[i];
  double r = sqrt(r2);
  if (r == 0.0 || r - alpha <= 0.0) {
    for (int i = 0; i < n; i++) out[i] = 0.0;
    return;
  }
  double f = (r - alpha) / r;
  for (int i = 0; i < n; i++) out[i] = u[i] * f;
}

/* prox of tau ||.||_W, W = diag(w) (NEXT-2): Moreau gives
 * prox(u) = u - tau Pi_E(u / tau) with E = {y : <y, W^{-1} y> <= 1} the dual ball (semi-axes
 * d_i = sqrt(w_i)); outside E, Pi_E(z)_i = d_i^2 z_i / (d_i^2 + mu) with mu the root of
 * sum_i d_i^2 z_i^2 / (d_i^2 + mu)^2 = 1, found as the paper does: Newton on
 * mu -> sum_i d_i^2 z_i^2 / (d_i^2 + mu) + mu from mu_0 = 0, stopping at |mu_{k+1} - mu_k| <= 1e-8. */
static void prox_ell(int n, const double *u, double tau, const double *w, double *out) {
  if (!(tau > 0.0)) { memcpy(out, u, sizeof(double) * n); return; }
  double q = 0.0;
  for (int i = 0; i < n; i++) { double z = u[i] / tau; q += z * z / w[i]; }
  if (q <= 1.0) { for (int i = 0; i < n; i++) out[i] = 0.0; return; }
  double mu = 0.0;
  for (int it = 0; it < 1000; it++) {
    double f1 = 0.0, f2 = 0.0;
    for (int i = 0; i < n; i++) {
      double z = u[i] / tau, e = w[i] + mu;
      f1 += w[i] * z * z / (e * e);
      f2 += w[i] * z * z / (e * e * e);
    }
    double mn = mu - (1.0 - f1) / (2.0 * f2);   /* Newton on the derivative 1 - f1 */
    int done = fabs(mn - mu) <= 1e-8;
    mu = mn;
    if (done) break;
  }
  for (int i = 0; i < n; i++) out[i] = u[i] - tau * (w[i] * (u[i] / tau) / (w[i] + mu));
}

static int cmp_double(const void *a, const void *b) {
  const double x = *(const double *)a, y = *(const double *)b;
  return (x > y) - (x < y);
}
/* ||shrink_1(z, mu)||_1 = sum_i max(|z_i| - mu, 0)   (h of P:1410-1413) */
static double h_linf(int n, const double *z, double mu) {
  double s = 0.0;
  for (int i = 0; i < n; i++) s += fmax(fabs(z[i]) - mu, 0.0);
  return s;
}
/* prox of tau ||.||_inf: Moreau, prox(u) = u - tau pi_C(u / tau), C the unit l1
 * ball (the dual ball of l_inf).  For z = u / tau outside C: pi_C(z) = shrink_1(z, mu) with
 * ||shrink_1(z, mu)||_1 = 1 (eq. condition_mu_linfty); h(mu) = ||shrink_1(z, mu)||_1 is piecewise
 * affine and decreasing with breakpoints B = {0} U {|z_i|}: sort them increasingly (l_0 = 0 <=
 * l_1 <= ... <= l_n), search j with h(l_j) >= 1 > h(l_{j+1}) (binary search), and interpolate
 * on the affine piece.  sort_buf: n doubles. */
static void prox_linf(int n, const double *u, double tau, double *sort_buf, double *out) {
  if (!(tau > 0.0)) { memcpy(out, u, sizeof(double) * n); return; }
  double l1 = 0.0;
  for (int i = 0; i < n; i++) l1 += fabs(u[i] / tau);
  if (l1 <= 1.0) { for (int i = 0; i < n; i++) out[i] = 0.0; return; }   /* z in C: pi = z */
  double *z = out;   /* out holds z = u / tau until the end */
  for (int i = 0; i < n; i++) { z[i] = u[i] / tau; sort_buf[i] = fabs(z[i]); }
  qsort(sort_buf, (size_t)n, sizeof(double), cmp_double);
  /* breakpoint k: l_0 = 0, l_k = sort_buf[k-1]; h(l_0) = ||z||_1 > 1, h(l_n) = 0 < 1 */
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (h_linf(n, z, sort_buf[mid - 1]) >= 1.0) lo = mid; else hi = mid;
  }
  const double la = lo == 0 ? 0.0 : sort_buf[lo - 1], lb = sort_buf[hi - 1];
  const double ha = h_linf(n, z, la), hb = h_linf(n, z, lb);
  const double mu = la + (ha - 1.0) * (lb - la) / (ha - hb);
  for (int i = 0; i < n; i++) {
    const double a = fabs(z[i]) - mu;
    const double pi = a > 0.0 ? (z[i] >= 0.0 ? a : -a) : 0.0;   /* shrink_1(z, mu) */
    out[i] = u[i] - tau * pi;
  }
}

static void prox_tH(int n, int h, const double *u, double t, const double *w,
                    double lambda, double *alpha_buf, double *out) {
  if (h == ORACLE_H_ELL) {
    prox_ell(n, u, t / lambda, w, out);
  } else if (h == ORACLE_H_LINF) {
    prox_linf(n, u, t / lambda, alpha_buf, out);
  } else if (h == ORACLE_H_L2) {
    shrink2(n, u, t / lambda, out);
  } else {
    for (int i = 0; i < n; i++)
      alpha_buf[i] = t * (h == ORACLE_H_WL1 ? w[i] : 1.0) / lambda;
    shrink1(n, u, alpha_buf, out);
  }
}

static double H_of(int n, int h, const double *p, const double *w) {
  double s = 0.0;
  if (h == ORACLE_H_ELL) {
    for (int i = 0; i < n; i++) s += w[i] * p[i] * p[i];
    return sqrt(s);
  }
  if (h == ORACLE_H_L2) {
    for (int i = 0; i < n; i++) s += p[i] * p[i];
    return sqrt(s);
  }
  if (h == ORACLE_H_LINF) {
    for (int i = 0; i < n; i++) s = fmax(s, fabs(p[i]));
    return s;
  }
  for (int i = 0; i < n; i++) s += (h == ORACLE_H_WL1 ? w[i] : 1.0) * fabs(p[i]);
  return s;
}

static double sqdist(int n, const double *a, const double *b) {
  double s = 0.0;
  for (int i = 0; i < n; i++) {
    double e = a[i] - b[i];
    s += e * e;
  }
  return s;
}

static int point_invalid(int n, const double *x, double t) {
  if (!isfinite(t) || t < 0.0) return 1;
  for (int i = 0; i < n; i++)
    if (!isfinite(x[i])) return 1;
  return 0;
}

/* ---------------- one point, diagonal J ---------------------------------- */
/* Solves the problem centred at xt = x - c (reading R5), returns iters.
 * v-update (3.4a) with J*(v) = 1/2<v,Dv> + <c,v> - gamma: setting the gradient
 * D v + c - x - lambda (d - b - v) to zero gives
 *     v = (D + lambda I)^{-1} (x - c + lambda (d - b)). */
static int solve_diag_point(int n, const double *x, double t, const double *D,
                            const double *c, double gamma, int h, const double *w,
                            double lambda, int max_iter, double tol, double *phi,
                            double *grad, double *ws) {
  double *xt = ws, *v = ws + n, *d = ws + 2 * n, *b = ws + 3 * n;
  double *vp = ws + 4 * n, *dp = ws + 5 * n, *u = ws + 6 * n, *al = ws + 7 * n;
  if (point_invalid(n, x, t)) {
    *phi = NAN;
    for (int i = 0; i < n; i++) grad[i] = NAN;
    return INT32_MIN;
  }
  for (int i = 0; i < n; i++) xt[i] = x[i] - (c ? c[i] : 0.0);
  if (t == 0.0) { /* reading R6: phi(x,0) = J(x), grad = grad J(x) (1.1b) */
    double J = gamma;
    for (int i = 0; i < n; i++) {
      J += 0.5 * xt[i] * xt[i] / D[i];
      grad[i] = xt[i] / D[i];
    }
    *phi = J;
    return 0;
  }
  /* v^0 = d^0 = x, b^0 = 0, in centred coordinates (R5). */
  for (int i = 0; i < n; i++) {
    v[i] = xt[i];
    d[i] = xt[i];
    b[i] = 0.0;
  }
  int iters = -max_iter;
  for (int k = 1; k <= max_iter; k++) {
    memcpy(vp, v, sizeof(double) * n);
    memcpy(dp, d, sizeof(double) * n);
    /* (3.4a) */
    for (int i = 0; i < n; i++) v[i] = (xt[i] + lambda * (d[i] - b[i])) / (D[i] + lambda);
    /* (3.4b): d = prox_{(t/lambda) H}(v + b) */
    for (int i = 0; i < n; i++) u[i] = v[i] + b[i];
    prox_tH(n, h, u, t, w, lambda, al, d);
    /* (3.4c) */
    for (int i = 0; i < n; i++) b[i] = b[i] + v[i] - d[i];
    /* stopping rule P:1597-1601 */
    if (sqdist(n, v, vp) <= tol && sqdist(n, d, dp) <= tol && sqdist(n, d, v) <= tol) {
      iters = k;
      break;
    }
  }
  /* grad := d (R1); phi := -(J*(d) + t H(d) - <x,d>) (R2, (3.3)) */
  double xd = 0.0, dDd = 0.0;
  for (int i = 0; i < n; i++) {
    xd += xt[i] * d[i];
    dDd += d[i] * D[i] * d[i];
    grad[i] = d[i];
  }
  *phi = xd - 0.5 * dDd - t * H_of(n, h, d, w) + gamma;
  return iters;
}

static int nthreads_or_default(int nthreads) {
#ifdef _OPENMP
  return nthreads > 0 ? nthreads : omp_get_max_threads();
#else
  (void)nthreads;
  return 1;
#endif
}

int oracle_threads(int nthreads) { return nthreads_or_default(nthreads); }

/* Batched diagonal-J evaluation. X: [M*n] row-major, t: [M]. */
int oracle_diag(int64_t M, int n, const double *X, const double *t, const double *D,
                const double *c, double gamma, int h, const double *w, double lambda,
                int max_iter, double tol, double *phi, double *grad, int32_t *iters,
                int nthreads) {
  if (M < 0 || n < 1 || !D || lambda <= 0.0 || max_iter < 1 || tol < 0.0) return -1;
  if ((h == ORACLE_H_WL1 || h == ORACLE_H_ELL) && !w) return -1;
  if (h < 0 || h > ORACLE_H_LINF) return -1;
  int nt = nthreads_or_default(nthreads);
#pragma omp parallel num_threads(nt)
  {
    double *ws = (double *)malloc(sizeof(double) * 8 * (size_t)n);
#pragma omp for schedule(dynamic, 64)
    for (int64_t p = 0; p < M; p++)
      iters[p] = solve_diag_point(n, X + p * n, t[p], D, c, gamma, h, w, lambda, max_iter,
                                  tol, phi + p, grad + p * n, ws);
    free(ws);
  }
  return 0;
}

/* ---------------- one point, dense SPD J --------------------------------- */
/* v-update (3.4a) with J*(v) = 1/2<v,A^{-1}v> - gamma:
 *     (A^{-1} + lambda I) v = x + lambda (d - b)  =>  v = M_lambda (x + lambda(d-b)),
 * M_lambda = (A^{-1} + lambda I)^{-1} = P (I + ...)^{-1} P^T form of P:1336-1347,
 * supplied precomputed in fp64 by the caller (oracle/__init__.py). */
static int solve_dense_point(int n, const double *x, double t, const double *Ml,
                             const double *A, const double *Ainv, double gamma, int h,
                             const double *w, double lambda, int max_iter, double tol,
                             double *phi, double *grad, double *ws) {
  double *v = ws, *d = ws + n, *b = ws + 2 * n, *vp = ws + 3 * n, *dp = ws + 4 * n;
  double *u = ws + 5 * n, *al = ws + 6 * n, *r = ws + 7 * n;
  if (point_invalid(n, x, t)) {
    *phi = NAN;
    for (int i = 0; i < n; i++) grad[i] = NAN;
    return INT32_MIN;
  }
  if (t == 0.0) { /* R6: J(x) = 1/2<x,Ax> + gamma, grad J = A x */
    double J = gamma;
    for (int i = 0; i < n; i++) {
      double s = 0.0;
      for (int j = 0; j < n; j++) s += A[(size_t)i * n + j] * x[j];
      grad[i] = s;
      J += 0.5 * x[i] * s;
    }
    *phi = J;
    return 0;
  }
  for (int i = 0; i < n; i++) {
    v[i] = x[i];
    d[i] = x[i];
    b[i] = 0.0;
  }
  int iters = -max_iter;
  for (int k = 1; k <= max_iter; k++) {
    memcpy(vp, v, sizeof(double) * n);
    memcpy(dp, d, sizeof(double) * n);
    for (int j = 0; j < n; j++) r[j] = x[j] + lambda * (d[j] - b[j]);
    for (int i = 0; i < n; i++) { /* (3.4a) */
      double s = 0.0;
      for (int j = 0; j < n; j++) s += Ml[(size_t)i * n + j] * r[j];
      v[i] = s;
    }
    for (int i = 0; i < n; i++) u[i] = v[i] + b[i];
    prox_tH(n, h, u, t, w, lambda, al, d);                   /* (3.4b) */
    for (int i = 0; i < n; i++) b[i] = b[i] + v[i] - d[i]; /* (3.4c) */
    if (sqdist(n, v, vp) <= tol && sqdist(n, d, dp) <= tol && sqdist(n, d, v) <= tol) {
      iters = k;
      break;
    }
  }
  double xd = 0.0, dAd = 0.0;
  for (int i = 0; i < n; i++) {
    double s = 0.0;
    for (int j = 0; j < n; j++) s += Ainv[(size_t)i * n + j] * d[j];
    xd += x[i] * d[i];
    dAd += d[i] * s;
    grad[i] = d[i];
  }
  *phi = xd - 0.5 * dAd - t * H_of(n, h, d, w) + gamma;
  return iters;
}

int oracle_dense(int64_t M, int n, const double *X, const double *t, const double *Ml,
                 const double *A, const double *Ainv, double gamma, int h, const double *w,
                 double lambda, int max_iter, double tol, double *phi, double *grad,
                 int32_t *iters, int nthreads) {
  if (M < 0 || n < 1 || !Ml || !A || !Ainv || lambda <= 0.0 || max_iter < 1 || tol < 0.0)
    return -1;
  if ((h == ORACLE_H_WL1 || h == ORACLE_H_ELL) && !w) return -1;
  if (h < 0 || h > ORACLE_H_LINF) return -1;
  int nt = nthreads_or_default(nthreads);
#pragma omp parallel num_threads(nt)
  {
    double *ws = (double *)malloc(sizeof(double) * 8 * (size_t)n);
#pragma omp for schedule(dynamic, 16)
    for (int64_t p = 0; p < M; p++)
      iters[p] = solve_dense_point(n, X + p * n, t[p], Ml, A, Ainv, gamma, h, w, lambda,
                                   max_iter, tol, phi + p, grad + p * n, ws);
    free(ws);
  }
  return 0;
}

/* ---------------- union of K diagonal initial data ----------- */
/* phi = min_k phi_k (lowest k on ties, R19); grad = grad of the winner;
 * y = x - t grad/||grad|| (P:757-761 for H = l2), c_k* if grad = 0 (R18).
 * Y is only defined for H = l2 (returns -1 otherwise when Y is requested). */
int oracle_union(int64_t M, int n, int K, const double *X, const double *t, const double *Dk,
                 const double *Ck, const double *gammak, int h, const double *w,
                 double lambda, int max_iter, double tol, double *phi, double *grad,
                 int32_t *iters, double *Y, int32_t *kstar, double *phik, int nthreads) {
  if (M < 0 || n < 1 || K < 1 || !Dk || !Ck || !gammak || lambda <= 0.0 || max_iter < 1 ||
      tol < 0.0)
    return -1;
  if ((h == ORACLE_H_WL1 || h == ORACLE_H_ELL) && !w) return -1;
  if (h < 0 || h > ORACLE_H_LINF) return -1;
  if (Y && h != ORACLE_H_L2) return -1;
  int nt = nthreads_or_default(nthreads);
#pragma omp parallel num_threads(nt)
  {
    double *ws = (double *)malloc(sizeof(double) * 8 * (size_t)n);
    double *g = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 16)
    for (int64_t p = 0; p < M; p++) {
      const double *x = X + p * n;
      double best = INFINITY;
      int bestk = -1, bestit = 0;
      double *gout = grad + p * n;
      for (int k = 0; k < K; k++) {
        double ph;
        int it = solve_diag_point(n, x, t[p], Dk + (size_t)k * n, Ck + (size_t)k * n,
                                  gammak[k], h, w, lambda, max_iter, tol, &ph, g, ws);
        if (phik) phik[p * K + k] = ph;
        if (it == INT32_MIN) { /* invalid point: every phi_k is NaN (ABI convention) */
          if (phik) for (int k2 = 0; k2 < K; k2++) phik[p * K + k2] = NAN;
          bestk = -1; bestit = INT32_MIN; break;
        }
        if (ph < best) { /* strict: lowest k wins ties (R19) */
          best = ph;
          bestk = k;
          bestit = it;
          memcpy(gout, g, sizeof(double) * n);
        }
      }
      if (bestk < 0) {
        phi[p] = NAN;
        for (int i = 0; i < n; i++) gout[i] = NAN;
        iters[p] = INT32_MIN;
        if (kstar) kstar[p] = -1;
        if (Y) for (int i = 0; i < n; i++) Y[p * n + i] = NAN;
        continue;
      }
      phi[p] = best;
      iters[p] = bestit;
      if (kstar) kstar[p] = bestk;
      if (Y) {
        double gn = 0.0;
        for (int i = 0; i < n; i++) gn += gout[i] * gout[i];
        gn = sqrt(gn);
        for (int i = 0; i < n; i++)
          Y[p * n + i] = (gn > 0.0) ? x[i] - t[p] * gout[i] / gn : Ck[(size_t)bestk * n + i];
      }
    }
    free(g);
    free(ws);
  }
  return 0;
}

/* ---------------- distance / projection to a union (NEXT-1) -------------- */
/* Evaluates psi(y,s) = min_k psi_k(y,s) and its gradient (the winner's) with the
 * union routine above (split Bregman per set; s == 0 answered by L(y), R6). */
static double union_psi(int n, int K, const double *y, double s, const double *Dk,
                        const double *Ck, const double *gammak, double lambda, int max_iter,
                        double tol, double *g, double *gk, double *ws, int *kbest) {
  double best = INFINITY;
  *kbest = -1;
  for (int k = 0; k < K; k++) {
    double ph;
    int it = solve_diag_point(n, y, s, Dk + (size_t)k * n, Ck + (size_t)k * n, gammak[k],
                              ORACLE_H_L2, NULL, lambda, max_iter, tol, &ph, gk, ws);
    if (it == INT32_MIN) { *kbest = -1; return NAN; }
    if (ph < best) { /* strict: lowest k wins ties (R19) */
      best = ph;
      *kbest = k;
      memcpy(g, gk, sizeof(double) * n);
    }
  }
  return best;
}

/* Closest point and distance from y to Omega = union_k {L_k <= 0}, L_k(y) =
 * 1/2 <y-c_k, D_k^{-1}(y-c_k)> + gamma_k, by the paper's procedure:
 *   s_0 = 0 (psi(y,0) = L(y), grad L(y): reading R24), then
 *   s_{l+1} = s_l + psi(y,s_l) / ||grad_x psi(y,s_l)||           (eq. Newton_zero)
 stopping when the Newton correction |s_{l+1} - s_l| <= stol max(1, s_l) or after max_newton
 * evaluations, the result being the last evaluated s (reading R26); otherwise a step that
 * leaves the bracket (lo, hi) (psi(lo) > 0 >= psi(hi)) is replaced by bisection (R25):
 *   dist = s, proj = y - s grad/||grad||, psi = psi(y,s), grad, kstar,
 *   newton = number of union evaluations at s > 0 (0 for y in Omega: dist 0, proj y).
 * A point whose psi is non-finite gets NaN outputs and newton = INT32_MIN. */
int oracle_distance_union(int64_t M, int n, int K, const double *Yq, const double *Dk,
                          const double *Ck, const double *gammak, double lambda, int max_iter,
                          double tol, int max_newton, double stol, double *dist, double *proj,
                          double *psi, double *grad, int32_t *kstar, int32_t *newton,
                          int nthreads) {
  if (M < 0 || n < 1 || K < 1 || !Yq || !Dk || !Ck || !gammak || lambda <= 0.0 ||
      max_iter < 1 || tol < 0.0 || max_newton < 1 || !(stol >= 0.0))
    return -1;
  int nt = nthreads_or_default(nthreads);
#pragma omp parallel num_threads(nt)
  {
    double *ws = (double *)malloc(sizeof(double) * 8 * (size_t)n);
    double *gk = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 4)
    for (int64_t p = 0; p < M; p++) {
      const double *y = Yq + p * n;
      double *g = grad + p * n;
      int kb;
      double s = 0.0;
      double ps = union_psi(n, K, y, 0.0, Dk, Ck, gammak, lambda, max_iter, tol, g, gk, ws, &kb);
      int nn = 0, bad = !(ps == ps) || kb < 0;
      if (!bad && ps > 0.0) {
        double lo = 0.0, hi = INFINITY;
        for (int l = 1; l <= max_newton; l++) {
          double gn = 0.0;
          for (int i = 0; i < n; i++) gn += g[i] * g[i];
          gn = sqrt(gn);
          if (!(gn > 0.0)) break;
          double sn = s + ps / gn;                       /* eq. Newton_zero */
          if (fabs(sn - s) <= stol * fmax(1.0, s)) break; /* R26 */
          /* R25: a step that leaves the open bracket (lo, hi) is replaced by bisection; with
           * psi(s) > 0 the step is > 0, so this only happens once hi is finite */
          if (!(sn > lo && sn < hi)) sn = 0.5 * (lo + hi);
          s = sn;
          ps = union_psi(n, K, y, s, Dk, Ck, gammak, lambda, max_iter, tol, g, gk, ws, &kb);
          nn = l;
          if (!(ps == ps) || kb < 0) { bad = 1; break; }
          if (ps > 0.0) lo = s; else hi = s;
        }
      }
      if (bad) {
        dist[p] = NAN; psi[p] = NAN; kstar[p] = -1; newton[p] = INT32_MIN;
        for (int i = 0; i < n; i++) { g[i] = NAN; proj[p * n + i] = NAN; }
        continue;
      }
      dist[p] = s;
      psi[p] = ps;
      kstar[p] = kb;
      newton[p] = nn;
      double gn = 0.0;
      for (int i = 0; i < n; i++) gn += g[i] * g[i];
      gn = sqrt(gn);
      for (int i = 0; i < n; i++)
        proj[p * n + i] = (s > 0.0 && gn > 0.0) ? y[i] - s * g[i] / gn : y[i];
    }
    free(gk);
    free(ws);
  }
  return 0;
}

/* ---------------- max over a min of Hamiltonians (NEXT-4) --------- */
/* H = min_i a_i H_{kind_i}(.; w_i) with one diagonal J: phi = max_i phi_i, each phi_i
 * the split Bregman solve with H_i (its prox threshold t a_i w_ij / lambda, its t H_i(d) term in
 * (3.3)); grad = grad of the winner; the lowest i wins ties (as R19).  kinds[K], a[K] host
 * arrays, W [K*n] weights (rows used for ORACLE_H_WL1 / ORACLE_H_ELL only). */
int oracle_maxh(int64_t M, int n, const double *X, const double *t, const double *D,
                const double *c, double gamma, int K, const int32_t *kinds, const double *W,
                const double *a, double lambda, int max_iter, double tol, double *phi,
                double *grad, int32_t *iters, int32_t *istar, int nthreads) {
  if (M < 0 || n < 1 || K < 1 || !D || !kinds || !a || lambda <= 0.0 || max_iter < 1 || tol < 0.0)
    return -1;
  for (int i = 0; i < K; i++) {
    if (kinds[i] < 0 || kinds[i] > ORACLE_H_LINF || !(a[i] > 0.0)) return -1;
    if ((kinds[i] == ORACLE_H_WL1 || kinds[i] == ORACLE_H_ELL) && !W) return -1;
  }
  int nt = nthreads_or_default(nthreads);
#pragma omp parallel num_threads(nt)
  {
    double *ws = (double *)malloc(sizeof(double) * 8 * (size_t)n);
    double *g = (double *)malloc(sizeof(double) * (size_t)n);
    double *wa = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp for schedule(dynamic, 16)
    for (int64_t p = 0; p < M; p++) {
      const double *x = X + p * n;
      double best = -INFINITY;
      int besti = -1, bestit = 0;
      for (int i = 0; i < K; i++) {
        /* H_i = a_i H_kind(.; w_i): an l1 / weighted l1 with weights a_i w_ij, or a_i ||.||_2
         * (the l2 solve with t H_i = (a_i t) ||.||_2), or a_i ||.||_{W_i} (the ellipsoidal solve
         * at time a_i t) */
        double ph, ti = t[p];
        const double *wi = NULL;
        int h = kinds[i];
        if (h == ORACLE_H_L2) {
          ti = t[p] * a[i];
        } else if (h == ORACLE_H_ELL) {
          ti = t[p] * a[i];
          wi = W + (size_t)i * n;
        } else if (h == ORACLE_H_LINF) {
          ti = t[p] * a[i];
        } else {
          for (int j = 0; j < n; j++) wa[j] = a[i] * (h == ORACLE_H_WL1 ? W[(size_t)i * n + j] : 1.0);
          wi = wa;
          h = ORACLE_H_WL1;
        }
        int it = solve_diag_point(n, x, ti, D, c, gamma, h, wi, lambda, max_iter, tol, &ph, g, ws);
        if (it == INT32_MIN) { besti = -1; bestit = INT32_MIN; break; }
        if (ph > best) { /* strict: lowest i wins ties */
          best = ph;
          besti = i;
          bestit = it;
          memcpy(grad + p * n, g, sizeof(double) * n);
        }
      }
      if (besti < 0) {
        phi[p] = NAN;
        for (int j = 0; j < n; j++) grad[p * n + j] = NAN;
        iters[p] = INT32_MIN;
        if (istar) istar[p] = -1;
        continue;
      }
      phi[p] = best;
      iters[p] = bestit;
      if (istar) istar[p] = besti;
    }
    free(wa);
    free(g);
    free(ws);
  }
  return 0;
}

/* ---------------- non-quadratic initial data (NEXT-3) ------------ */
/* J = 1/2 ||.||_1^2 (ORACLE_J_L1SQ) or 1/2 ||.||_inf^2 (ORACLE_J_LINFSQ), plus gamma; any H.
 * (J*: 1/2||.||_inf^2 and 1/2||.||_1^2 respectively.) */
#define ORACLE_J_L1SQ 0
#define ORACLE_J_LINFSQ 1

/* beta >= 0 with beta = alpha ||shrink_1(z, beta)||_1 (eq. optimality_beta_l1_2): g(beta) =
 * alpha h(beta) - beta is decreasing and piecewise affine with breakpoints {0} U {|z_i|}: sort
 * them, search the bracketing pair g(l_j) >= 0 > g(l_{j+1}) (binary search), interpolate
 * (P:1513-1537).  z = 0 gives 0.  sort_buf: n doubles. */
static double beta_l1sq(int n, const double *z, double alpha, double *sort_buf) {
  double l1 = 0.0;
  for (int i = 0; i < n; i++) { sort_buf[i] = fabs(z[i]); l1 += sort_buf[i]; }
  if (l1 == 0.0) return 0.0;
  qsort(sort_buf, (size_t)n, sizeof(double), cmp_double);
  /* breakpoint k: l_0 = 0, l_k = sort_buf[k-1]; g(l_0) = alpha ||z||_1 > 0, g(l_n) = -max|z| < 0 */
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    const double l = sort_buf[mid - 1];
    if (alpha * h_linf(n, z, l) - l >= 0.0) lo = mid; else hi = mid;
  }
  const double la = lo == 0 ? 0.0 : sort_buf[lo - 1], lb = sort_buf[hi - 1];
  const double ga = alpha * h_linf(n, z, la) - la, gb = alpha * h_linf(n, z, lb) - lb;
  return la + ga * (lb - la) / (ga - gb);
}
/* prox_{(alpha/2)||.||_1^2}(z) = shrink_1(z, beta) (eq. prox_l1_2_with_beta) */
static void prox_l1sq(int n, const double *z, double alpha, double *sort_buf, double *out) {
  const double beta = beta_l1sq(n, z, alpha, sort_buf);
  for (int i = 0; i < n; i++) {
    const double a = fabs(z[i]) - beta;
    out[i] = a > 0.0 ? (z[i] >= 0.0 ? a : -a) : 0.0;
  }
}
/* prox_{(alpha/2)||.||_inf^2}(z) = z - alpha prox_{(1/(2 alpha))||.||_1^2}(z / alpha)  (Moreau,
 * P:1549-1555; the printed form z - prox_{(alpha/2)||.||_1^2}(z) is this at alpha = 1, the
 * paper's lambda; reading R29).  zs: n doubles of scratch. */
static void prox_linfsq(int n, const double *z, double alpha, double *sort_buf, double *zs,
                        double *out) {
  for (int i = 0; i < n; i++) zs[i] = z[i] / alpha;
  prox_l1sq(n, zs, 1.0 / alpha, sort_buf, out);
  for (int i = 0; i < n; i++) out[i] = z[i] - alpha * out[i];
}
static double l1norm(int n, const double *p) {
  double s = 0.0;
  for (int i = 0; i < n; i++) s += fabs(p[i]);
  return s;
}
static double linfnorm(int n, const double *p) {
  double s = 0.0;
  for (int i = 0; i < n; i++) s = fmax(s, fabs(p[i]));
  return s;
}

static int solve_normsq_point(int n, const double *x, double t, int jk, double gamma, int h,
                              const double *w, double lambda, int max_iter, double tol,
                              double *phi, double *grad, double *ws) {
  double *v = ws, *d = ws + n, *b = ws + 2 * n, *vp = ws + 3 * n, *dp = ws + 4 * n;
  double *u = ws + 5 * n, *al = ws + 6 * n, *z = ws + 7 * n, *zs = ws + 8 * n;
  if (point_invalid(n, x, t)) {
    *phi = NAN;
    for (int i = 0; i < n; i++) grad[i] = NAN;
    return INT32_MIN;
  }
  if (t == 0.0) {
    /* R6 with R30: phi = J(x); grad = the minimal-norm element of dJ(x):
     * 1/2||x||_1^2: ||x||_1 sign(x_i) (0 where x_i = 0);
     * 1/2||x||_inf^2: ||x||_inf sign(x_i) / m on the m maximal |x_i|, 0 elsewhere */
    if (jk == ORACLE_J_L1SQ) {
      const double s = l1norm(n, x);
      for (int i = 0; i < n; i++) grad[i] = x[i] > 0.0 ? s : (x[i] < 0.0 ? -s : 0.0);
      *phi = 0.5 * s * s + gamma;
    } else {
      const double s = linfnorm(n, x);
      int m = 0;
      for (int i = 0; i < n; i++) m += (fabs(x[i]) == s);
      for (int i = 0; i < n; i++)
        grad[i] = (s > 0.0 && fabs(x[i]) == s) ? (x[i] > 0.0 ? s : -s) / m : 0.0;
      *phi = 0.5 * s * s + gamma;
    }
    return 0;
  }
  for (int i = 0; i < n; i++) { v[i] = x[i]; d[i] = x[i]; b[i] = 0.0; }
  int iters = -max_iter;
  for (int k = 1; k <= max_iter; k++) {
    memcpy(vp, v, sizeof(double) * n);
    memcpy(dp, d, sizeof(double) * n);
    /* (3.4a): v = argmin J*(v) - <x,v> + lambda/2 ||d - v - b||^2, i.e. the prox of
     * (1/lambda) J* at z = d - b + x/lambda */
    for (int i = 0; i < n; i++) z[i] = d[i] - b[i] + x[i] / lambda;
    if (jk == ORACLE_J_L1SQ) prox_linfsq(n, z, 1.0 / lambda, al, zs, v);   /* J* = 1/2||.||_inf^2 */
    else prox_l1sq(n, z, 1.0 / lambda, al, v);                              /* J* = 1/2||.||_1^2 */
    for (int i = 0; i < n; i++) u[i] = v[i] + b[i];
    prox_tH(n, h, u, t, w, lambda, al, d);
    for (int i = 0; i < n; i++) b[i] = b[i] + v[i] - d[i];
    if (sqdist(n, v, vp) <= tol && sqdist(n, d, dp) <= tol && sqdist(n, d, v) <= tol) {
      iters = k;
      break;
    }
  }
  double xd = 0.0;
  for (int i = 0; i < n; i++) { xd += x[i] * d[i]; grad[i] = d[i]; }
  const double js = jk == ORACLE_J_L1SQ ? linfnorm(n, d) : l1norm(n, d);
  *phi = xd - 0.5 * js * js - t * H_of(n, h, d, w) + gamma;
  return iters;
}

int oracle_normsq(int64_t M, int n, const double *X, const double *t, int jk, double gamma,
                  int h, const double *w, double lambda, int max_iter, double tol, double *phi,
                  double *grad, int32_t *iters, int nthreads) {
  if (M < 0 || n < 1 || lambda <= 0.0 || max_iter < 1 || tol < 0.0) return -1;
  if (jk != ORACLE_J_L1SQ && jk != ORACLE_J_LINFSQ) return -1;
  if ((h == ORACLE_H_WL1 || h == ORACLE_H_ELL) && !w) return -1;
  if (h < 0 || h > ORACLE_H_LINF) return -1;
  int nt = nthreads_or_default(nthreads);
#pragma omp parallel num_threads(nt)
  {
    double *ws = (double *)malloc(sizeof(double) * 9 * (size_t)n);
#pragma omp for schedule(dynamic, 64)
    for (int64_t p = 0; p < M; p++)
      iters[p] = solve_normsq_point(n, X + p * n, t[p], jk, gamma, h, w, lambda, max_iter, tol,
                                    phi + p, grad + p * n, ws);
    free(ws);
  }
  return 0;
}

/* ---------------- H = ||.||_A with a full SPD A (NEXT-2) ------------------- */
/* prox of tau ||.||_A: u - tau pi_{E_A}(u / tau) (Moreau), pi_{E_A}(w) = P pi_{E_D}(P^T w) with
 * A = P D P^T; pi_{E_D} by prox_ell's Newton on mu (the diagonal case, with
 * w = D).  Q [n*n] row-major, columns = eigenvectors; Lam [n] eigenvalues. */
static void prox_ellA(int n, const double *u, double tau, const double *Q, const double *Lam,
                      double *s1, double *s2, double *out) {
  for (int i = 0; i < n; i++) {        /* s1 = Q^T u */
    double a = 0.0;
    for (int k = 0; k < n; k++) a += Q[(size_t)k * n + i] * u[k];
    s1[i] = a;
  }
  prox_ell(n, s1, tau, Lam, s2);       /* prox of tau ||.||_Lam in the eigenbasis */
  for (int i = 0; i < n; i++) {        /* out = Q s2 */
    double a = 0.0;
    for (int k = 0; k < n; k++) a += Q[(size_t)i * n + k] * s2[k];
    out[i] = a;
  }
}

static int solve_diagA_point(int n, const double *x, double t, const double *D, const double *c,
                             double gamma, const double *Q, const double *Lam, const double *A,
                             double lambda, int max_iter, double tol, double *phi, double *grad,
                             double *ws) {
  double *xt = ws, *v = ws + n, *d = ws + 2 * n, *b = ws + 3 * n;
  double *vp = ws + 4 * n, *dp = ws + 5 * n, *u = ws + 6 * n, *s1 = ws + 7 * n, *s2 = ws + 8 * n;
  if (point_invalid(n, x, t)) {
    *phi = NAN;
    for (int i = 0; i < n; i++) grad[i] = NAN;
    return INT32_MIN;
  }
  for (int i = 0; i < n; i++) xt[i] = x[i] - (c ? c[i] : 0.0);
  if (t == 0.0) {
    double J = gamma;
    for (int i = 0; i < n; i++) { J += 0.5 * xt[i] * xt[i] / D[i]; grad[i] = xt[i] / D[i]; }
    *phi = J;
    return 0;
  }
  for (int i = 0; i < n; i++) { v[i] = xt[i]; d[i] = xt[i]; b[i] = 0.0; }
  int iters = -max_iter;
  for (int k = 1; k <= max_iter; k++) {
    memcpy(vp, v, sizeof(double) * n);
    memcpy(dp, d, sizeof(double) * n);
    for (int i = 0; i < n; i++) v[i] = (xt[i] + lambda * (d[i] - b[i])) / (D[i] + lambda);  /* (3.4a) */
    for (int i = 0; i < n; i++) u[i] = v[i] + b[i];
    prox_ellA(n, u, t / lambda, Q, Lam, s1, s2, d);                                         /* (3.4b) */
    for (int i = 0; i < n; i++) b[i] = b[i] + v[i] - d[i];                                  /* (3.4c) */
    if (sqdist(n, v, vp) <= tol && sqdist(n, d, dp) <= tol && sqdist(n, d, v) <= tol) {
      iters = k;
      break;
    }
  }
  double xd = 0.0, dDd = 0.0, dAd = 0.0;
  for (int i = 0; i < n; i++) {
    xd += xt[i] * d[i];
    dDd += d[i] * D[i] * d[i];
    for (int j = 0; j < n; j++) dAd += d[i] * A[(size_t)i * n + j] * d[j];
    grad[i] = d[i];
  }
  *phi = xd - 0.5 * dDd - t * sqrt(fmax(dAd, 0.0)) + gamma;
  return iters;
}

int oracle_diag_A(int64_t M, int n, const double *X, const double *t, const double *D,
                  const double *c, double gamma, const double *Q, const double *Lam,
                  const double *A, double lambda, int max_iter, double tol, double *phi,
                  double *grad, int32_t *iters, int nthreads) {
  if (M < 0 || n < 1 || !D || !Q || !Lam || !A || lambda <= 0.0 || max_iter < 1 || tol < 0.0)
    return -1;
  int nt = nthreads_or_default(nthreads);
#pragma omp parallel num_threads(nt)
  {
    double *ws = (double *)malloc(sizeof(double) * 9 * (size_t)n);
#pragma omp for schedule(dynamic, 64)
    for (int64_t p = 0; p < M; p++)
      iters[p] = solve_diagA_point(n, X + p * n, t[p], D, c, gamma, Q, Lam, A, lambda, max_iter,
                                   tol, phi + p, grad + p * n, ws);
    free(ws);
  }
  return 0;
}
