// diag_kernel.cuh — register-resident split Bregman kernels for diagonal J (K1/K2) and the
// min-over-K-sets union kernel (K4).  sm_100a, FP32 SIMT.
//
// Paper: Hopf formula (3.3) P:815-818; split Bregman (3.4a)-(3.4c) P:832-844; stopping rule
// P:1595-1601; shrink_1 P:239-247; shrink_2 P:279-287; quadratic prox P:901-906, P:1336-1347;
// Moreau / prox = I - projection P:924-992; union (min over initial data) P:628-667;
// closest point y = x - t grad/||grad|| P:1049-1051.
//
// Execution model.  A "group" of G lanes (G in {1,2,4,8,16,32}) owns one point; lane l of the
// group owns coordinates i = l + G*j, j < CPL (CPL = coordinates per lane, compile time), so
// every per-point vector lives in registers (x_hat, kappa, d, b, v_prev: 5*CPL floats) and
// the per-point sums (||u||^2 for shrink_2, the three stopping sums, phi) are xor-shuffle
// reductions inside the group.  Padded coordinates (i >= n) hold zeros, which the iteration
// maps to zeros, so they never contribute.  Grids are persistent (SMs x resident blocks);
// groups take points p = gid, gid + ngroups, ...  When a group's point stops (paper test or
// max_iter) the warp runs the finalize/refill branch: that group writes phi, grad, iters and
// immediately loads its next point while the other groups of the warp keep iterating, so a
// finished point stops costing cycles after one pass of the branch (per-point masking with
// in-place refill instead of lockstep batches).
//
// Per coordinate and iteration (exact rearrangement of (3.4a)-(3.4c)):
//   a = d - b;  v = x_hat + kappa*a          (3.4a), kappa = lambda/(D+lambda), x_hat = (x-c)/(D+lambda)
//   u = v + b;                               argument of (3.4b)
//   l1/wl1:  b' = clamp(u, -tau_i, tau_i);  d' = u - b'          shrink_1 via Moreau
//   l2:      s = max(0, 1 - tau/||u||);     d' = s u;  b' = u - d'   shrink_2
//   (3.4c): b + v - d' = u - d' = b'  (identical in exact arithmetic; the clamp form is also
//   bit-identical to sign(u) max(|u|-tau,0) in IEEE arithmetic)
//   test:  ||v - v_prev||^2, ||d' - d||^2, ||d' - v||^2 = ||b - b'||^2  <= tol
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hopf {

enum { HK_L1 = 0, HK_WL1 = 1, HK_L2 = 2 };

struct DiagParams {
  int64_t M;
  int n;
  const float *X, *t;
  const float *D, *c, *w;  // diag: D[n], c[n] or null; union: D = Dj[K*n], c = C[K*n]
  const float *gk;         // union: gamma[K]
  float gamma;
  float lambda;
  int max_iter;
  float tol;
  int K;  // 0 = plain diag
  float *phi, *grad;
  int *iters;
  float *Y;
  int *kstar;
  float *phik;
};

template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int G>
__device__ __forceinline__ bool group_any(bool f) {
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  if (G == 32) return bal != 0u;
  const int lane = threadIdx.x & 31;
  const unsigned gm = ((1u << G) - 1u) << (lane & ~(G - 1));
  return (bal & gm) != 0u;
}

__device__ __forceinline__ bool finite_f(float x) { return fabsf(x) <= 3.402823466e38f; }

// One kernel template for the diagonal and the union entry points.
//   UNION = false: K1/K2 (set constants once per kernel, one solve per point)
//   UNION = true : K4 (K solves per point, running arg-min, optional Y/kstar/phik)
template <int G, int CPL, int HK, bool UNION>
__global__ void __launch_bounds__(256) hopf_diag_kernel(const DiagParams p) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int n = p.n;
  const float lam = p.lambda, tol = p.tol;
  // slots j < jmax of this lane hold real coordinates (i = gl + G*j < n)
  const int jmax = (n - gl + G - 1) / G;

  // Per-slot registers.
  float xh[CPL], kap[CPL], d[CPL], b[CPL], vp[CPL];
  float tau[HK == HK_WL1 ? CPL : 1];
  float xr[UNION ? CPL : 1];   // union: the raw point x (sets translate it by c_k)
  float bd[UNION ? CPL : 1];   // union: grad of the best set so far

  // Kernel-lifetime constant of the diag path: kappa_i = lambda/(D_i+lambda).
  if (!UNION) {
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      const int i = gl + G * j;
      kap[j] = (j < jmax) ? __fdividef(lam, __ldg(p.D + i) + lam) : 0.f;
    }
  }

  int64_t pt = gid;
  bool have = pt < p.M;
  int it = 0;       // iterations of the current solve
  int kset = 0;     // union: current set
  float tt = 0.f;   // t of the current point
  float tauS = 0.f; // scalar threshold t/lambda
  int spec = 0;     // 0 normal, 1 t == 0, 2 invalid
  float best = 0.f;
  int bestk = -1, bestit = 0;

  // ---- load the point (x, t) into registers; detect t == 0 / invalid ------------------------
  auto load_point = [&](bool active) {
    bool bad = false;
    if (active) {
      tt = __ldg(p.t + pt);
      bad = !(tt >= 0.f) || !finite_f(tt);
      const float *xrow = p.X + pt * (int64_t)n;
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const int i = gl + G * j;
        const float xv = (j < jmax) ? __ldg(xrow + i) : 0.f;
        bad |= !finite_f(xv);
        if (UNION) xr[j] = xv; else xh[j] = xv;
      }
    }
    bad = group_any<G>(bad);
    if (active) {
      spec = bad ? 2 : (tt == 0.f ? 1 : 0);
      tauS = tt / lam;
    }
  };

  // ---- set up one solve: centred start v0 = d0 = x - c, b0 = 0 (reading R5) -------
  auto setup_solve = [&]() {
    const float *Dp = UNION ? p.D + (size_t)kset * n : p.D;
    const float *cp = UNION ? p.c + (size_t)kset * n : p.c;
    // stage D, c (and w) into the registers of d, b (tau) that are re-initialised below
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      const int i = gl + G * j;
      d[j] = (j < jmax) ? __ldg(Dp + i) : 1.f;
      b[j] = (cp && j < jmax) ? __ldg(cp + i) : 0.f;
      if (HK == HK_WL1) tau[j] = (j < jmax) ? __ldg(p.w + i) : 0.f;
    }
    const float tl = tt / lam;
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      const float xv = UNION ? xr[j] : xh[j];
      const float xt = (j < jmax) ? xv - b[j] : 0.f;
      const float dinv = __fdividef(1.f, d[j] + lam);
      if (UNION) kap[j] = (j < jmax) ? lam * dinv : 0.f;
      if (HK == HK_WL1) tau[j] *= tl;
      xh[j] = xt * dinv;
      d[j] = xt;
      b[j] = 0.f;
      vp[j] = xt;
    }
    it = 0;
  };

  load_point(have);
  if (have) {
    setup_solve();
    if (UNION) { best = __int_as_float(0x7f800000); bestk = -1; bestit = 0; }
  } else {
#pragma unroll
    for (int j = 0; j < CPL; j++) { xh[j] = 0.f; d[j] = 0.f; b[j] = 0.f; vp[j] = 0.f; if (UNION) kap[j] = 0.f; }
  }

  while (__any_sync(0xffffffffu, have)) {
    // ================= one split Bregman iteration (all lanes, branch-free) ==================
    // Register reuse: after (3.4a) b[j] holds u = v + b (b itself is no longer needed: the
    // new b is u - d' and the test term d' - v needs only d' and v = vp[j]).
    float sv = 0.f, sd = 0.f, sb = 0.f;
    if (HK == HK_L2) {
      float r2 = 0.f;
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const float a = d[j] - b[j];
        const float v = fmaf(kap[j], a, xh[j]);   // (3.4a)
        const float dv = v - vp[j];
        sv = fmaf(dv, dv, sv);
        vp[j] = v;
        b[j] = v + b[j];                           // u, argument of (3.4b)
        r2 = fmaf(b[j], b[j], r2);
      }
      r2 = group_sum<G>(r2);
      const float r = sqrtf(r2);
      const float s = (r > tauS) ? (r - tauS) / r : 0.f;   // shrink_2 factor
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const float u = b[j];
        const float dn = s * u;                    // (3.4b) shrink_2
        const float dd = dn - d[j];
        sd = fmaf(dd, dd, sd);
        const float dmv = dn - vp[j];              // d^k - v^k
        sb = fmaf(dmv, dmv, sb);
        d[j] = dn;
        b[j] = u - dn;                             // (3.4c): b + v - d' = u - d'
      }
    } else {
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const float a = d[j] - b[j];
        const float v = fmaf(kap[j], a, xh[j]);   // (3.4a)
        const float dv = v - vp[j];
        sv = fmaf(dv, dv, sv);
        vp[j] = v;
        const float u = v + b[j];
        const float tj = (HK == HK_WL1) ? tau[j] : tauS;
        const float bn = fminf(fmaxf(u, -tj), tj); // projection on the box [-tau, tau] (Moreau)
        const float dn = u - bn;                   // (3.4b) shrink_1; (3.4c) b' = u - d' = bn
        const float dd = dn - d[j];
        sd = fmaf(dd, dd, sd);
        const float dmv = dn - v;                  // d^k - v^k
        sb = fmaf(dmv, dmv, sb);
        d[j] = dn;
        b[j] = bn;
      }
    }
    sv = group_sum<G>(sv);
    sd = group_sum<G>(sd);
    sb = group_sum<G>(sb);
    it++;
    const bool conv = (sv <= tol) && (sd <= tol) && (sb <= tol);
    const bool done = have && (spec != 0 || conv || it >= p.max_iter);

    if (__any_sync(0xffffffffu, done)) {
      // ============ finalize (all lanes compute; done groups store and refill) ===============
      // phi = <x - c, d> - 1/2 <d, D d> - t H(d) + gamma   ((3.3) at d, reading R2)
      // t == 0: phi = J(x) = 1/2 <x-c, D^{-1}(x-c)> + gamma, grad = D^{-1}(x-c) (reading R6)
      const float *Dp = UNION ? p.D + (size_t)kset * n : p.D;
      const float *cp = UNION ? p.c + (size_t)kset * n : p.c;
      const float *xrow = p.X + pt * (int64_t)n;
      float q = 0.f, hsum = 0.f;
      if (done && spec != 2) {
        // the solve state of a done group is dead: stage x - c in vp and D in xh
#pragma unroll
        for (int j = 0; j < CPL; j++) {
          const int i = gl + G * j;
          if (j < jmax) {
            const float xv = UNION ? xr[j] : __ldg(xrow + i);
            vp[j] = cp ? xv - __ldg(cp + i) : xv;
            xh[j] = __ldg(Dp + i);
          }
        }
#pragma unroll
        for (int j = 0; j < CPL; j++) {
          if (j < jmax) {
            const float xt = vp[j], Dv = xh[j];
            if (spec == 1) {
              d[j] = __fdividef(xt, Dv);   // grad J(x)
              q = fmaf(0.5f * xt, d[j], q);
            } else {
              q = fmaf(xt, d[j], q);
              q = fmaf(-0.5f * Dv * d[j], d[j], q);
              if (HK == HK_L2) hsum = fmaf(d[j], d[j], hsum);
              else if (HK == HK_WL1) hsum = fmaf(__ldg(p.w + gl + G * j), fabsf(d[j]), hsum);
              else hsum += fabsf(d[j]);
            }
          }
        }
      }
      q = group_sum<G>(q);
      hsum = group_sum<G>(hsum);
      const float gam = UNION ? __ldg(p.gk + kset) : p.gamma;
      float phiv;
      if (spec == 1) phiv = q + gam;
      else phiv = q - tt * (HK == HK_L2 ? sqrtf(hsum) : hsum) + gam;
      int status = (spec == 1) ? 0 : (conv ? it : -p.max_iter);
      if (spec == 2) { phiv = __int_as_float(0x7fc00000); status = INT32_MIN; }

      bool point_done = done;
      if (UNION) {
        if (done) {
          if (p.phik && gl == 0) p.phik[pt * p.K + kset] = phiv;
          if (phiv < best) {   // strict: lowest k wins ties (R19); NaN never wins
            best = phiv; bestk = kset; bestit = status;
#pragma unroll
            for (int j = 0; j < CPL; j++) bd[j] = d[j];
          }
          point_done = (spec == 2) || (kset + 1 >= p.K);
        }
        // ||grad|| of the winner for y (all lanes participate in the reduction)
        float gn = 0.f;
#pragma unroll
        for (int j = 0; j < CPL; j++) gn = fmaf(bd[j], bd[j], gn);
        gn = sqrtf(group_sum<G>(gn));
        const float ign = (gn > 0.f) ? __fdividef(1.f, gn) : 0.f;
        if (point_done) {
          const bool nanpt = (spec == 2) || bestk < 0;
          if (gl == 0) {
            p.phi[pt] = nanpt ? __int_as_float(0x7fc00000) : best;
            p.iters[pt] = nanpt ? INT32_MIN : bestit;
            if (p.kstar) p.kstar[pt] = nanpt ? -1 : bestk;
          }
          float *grow = p.grad + pt * (int64_t)n;
          float *yrow = p.Y ? p.Y + pt * (int64_t)n : nullptr;
#pragma unroll
          for (int j = 0; j < CPL; j++) {
            const int i = gl + G * j;
            if (j < jmax) {
              grow[i] = nanpt ? __int_as_float(0x7fc00000) : bd[j];
              if (yrow) {
                float y;
                if (nanpt) y = __int_as_float(0x7fc00000);
                else if (gn > 0.f) y = xr[j] - tt * (bd[j] * ign);
                else y = __ldg(p.c + (size_t)bestk * n + i);                // reading R18
                yrow[i] = y;
              }
            }
          }
        }
      } else if (done) {
        if (gl == 0) { p.phi[pt] = phiv; p.iters[pt] = status; }
        float *grow = p.grad + pt * (int64_t)n;
#pragma unroll
        for (int j = 0; j < CPL; j++) {
          const int i = gl + G * j;
          if (j < jmax) grow[i] = (spec == 2) ? __int_as_float(0x7fc00000) : d[j];
        }
      }
      // ---- refill: the next point of this group ------------------------------------------
      if (point_done) {
        pt += ngroups;
        have = pt < p.M;
      }
      load_point(point_done && have);   // collective (ballot inside): all lanes call it
      if (done) {
        if (have) {
          // union: the next set of the same point, or set 0 of the next point
          kset = point_done ? 0 : kset + 1;
          if (UNION && point_done) { best = __int_as_float(0x7f800000); bestk = -1; bestit = 0; }
          setup_solve();
        } else {
#pragma unroll
          for (int j = 0; j < CPL; j++) { xh[j] = 0.f; d[j] = 0.f; b[j] = 0.f; vp[j] = 0.f; }
          spec = 0;
        }
      }
    }
  }
}

}  // namespace hopf
