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

// Sum of four per-lane partials over a group of G lanes with log2(G)+1 shuffles (instead of
// 4 log2(G)): the first two butterfly levels exchange halves of the value set, so afterwards
// lane gl of the group holds the group total of value q = gl / (G/4) (v0 | v1 | v2 | v3).
// Requires G >= 4.  Returns the total held by this lane.
template <int G>
__device__ __forceinline__ float group_sum4_transposed(float v0, float v1, float v2, float v3) {
  static_assert(G >= 4, "transposed reduction needs at least 4 lanes");
  const int gl = threadIdx.x & (G - 1);
  const bool hi = gl & (G / 2);
  const float send_a = hi ? v0 : v2, send_b = hi ? v1 : v3;
  const float keep_a = hi ? v2 : v0, keep_b = hi ? v3 : v1;
  const float a = keep_a + __shfl_xor_sync(0xffffffffu, send_a, G / 2);
  const float b = keep_b + __shfl_xor_sync(0xffffffffu, send_b, G / 2);
  const bool mid = gl & (G / 4);
  float c = (mid ? b : a) + __shfl_xor_sync(0xffffffffu, mid ? a : b, G / 4);
#pragma unroll
  for (int o = G / 8; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  return c;
}

// Group totals of four partials, delivered as: tot3 (broadcast to every lane of the group) and
// the three predicates (total_q <= tol) for q = 0, 1, 2.
template <int G>
__device__ __forceinline__ void group_reduce4(float v0, float v1, float v2, float v3, float tol,
                                              float &tot3, bool &ok0, bool &ok1, bool &ok2) {
  const int lane = threadIdx.x & 31;
  const int base = lane & ~(G - 1);
  if constexpr (G >= 4) {
    const float c = group_sum4_transposed<G>(v0, v1, v2, v3);
    const unsigned bal = __ballot_sync(0xffffffffu, c <= tol);
    tot3 = __shfl_sync(0xffffffffu, c, base + 3 * (G / 4));
    ok0 = (bal >> (base)) & 1u;
    ok1 = (bal >> (base + G / 4)) & 1u;
    ok2 = (bal >> (base + 2 * (G / 4))) & 1u;
  } else {
    v0 = group_sum<G>(v0);
    v1 = group_sum<G>(v1);
    v2 = group_sum<G>(v2);
    tot3 = group_sum<G>(v3);
    ok0 = v0 <= tol;
    ok1 = v1 <= tol;
    ok2 = v2 <= tol;
  }
}

// kappa_j of this lane from shared memory (non-union kernels).  ld.volatile keeps the load
// inside the loop (no hoisting back into registers): kappa is the same for every point, so it
// is held once per CTA instead of occupying CPL registers per thread.
__device__ __forceinline__ float lds_volatile(const float *p) {
  float v;
  asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ float4 lds_volatile4(const float *p) {
  float4 v;
  asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

// One kernel template for the diagonal and the union entry points.
//   UNION = false: K1/K2 (kappa for the whole CTA in shared memory, one solve per point)
//   UNION = true : K4 (K solves per point, kappa per set in registers, running arg-min,
//                  optional Y / kstar / phi_k)
// Loop trips alternate between two register sets for d and v_prev (A -> B, B -> A), so the
// loop-carried updates are renamings instead of register moves.
template <int G, int CPL, int HK, bool UNION>
__global__ void __launch_bounds__(256) hopf_diag_kernel(const DiagParams p) {
  constexpr bool KSM = !UNION;            // kappa in shared memory
  constexpr int CPL4 = (CPL % 4 == 0) ? CPL / 4 : 0;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int n = p.n;
  const float lam = p.lambda, tol = p.tol;
  // slots j < jmax of this lane hold real coordinates (i = gl + G*j < n)
  const int jmax = (n - gl + G - 1) / G;

  // Per-slot registers.
  float xh[CPL], dA[CPL], dB[CPL], b[CPL], vA[CPL], vB[CPL];
  float kap[KSM ? 1 : CPL];
  float tau[HK == HK_WL1 ? CPL : 1];
  float xr[UNION ? CPL : 1];   // union: the raw point x (sets translate it by c_k)
  float bd[UNION ? CPL : 1];   // union: grad of the best set so far

  // kappa_i = lambda/(D_i+lambda), layout [j/4][G][4] so a lane reads 4 slots with one LDS.128
  __shared__ __align__(16) float kap_s[KSM ? CPL * G : 1];
  if (KSM) {
    for (int e = threadIdx.x; e < CPL * G; e += blockDim.x) {
      int j, l;
      if (CPL4) { j = (e / (4 * G)) * 4 + (e & 3); l = (e / 4) % G; }
      else { j = e / G; l = e % G; }
      const int i = l + G * j;
      kap_s[e] = (i < n) ? __fdividef(lam, __ldg(p.D + i) + lam) : 0.f;
    }
    __syncthreads();
  }
  auto kappa_ptr = [&](int j) -> const float * {
    if (CPL4) return kap_s + (j / 4) * 4 * G + gl * 4 + (j & 3);
    return kap_s + j * G + gl;
  };

  int64_t pt = gid;
  bool have = pt < p.M;
  int it = 0;         // completed (3.4a) half-steps (l2) / iterations (l1) of the current solve
  int kset = 0;       // union: current set
  float tt = 0.f;     // t of the current point
  float tauS = 0.f;   // scalar threshold t/lambda
  int spec = 0;       // 0 normal, 1 t == 0, 2 invalid
  float s_cur = 1.f;  // l2: shrink factor of the pending (3.4b)
  bool sv_ok = false; // l2: ||v^k - v^{k-1}||^2 <= tol of the pending iteration
  float best = 0.f;
  int bestk = -1, bestit = 0;

  // ---- load the point (x, t) into registers; detect t == 0 / invalid (collective) -----------
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
  // Writes the "current" register set (d, v) that the next trip reads.
  auto setup_solve = [&](float (&d)[CPL], float (&vp)[CPL]) {
    const float *Dp = UNION ? p.D + (size_t)kset * n : p.D;
    const float *cp = UNION ? p.c + (size_t)kset * n : p.c;
    // stage D, c (and w) into registers that are re-initialised below
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
      if (!KSM) kap[j] = (j < jmax) ? lam * dinv : 0.f;
      if (HK == HK_WL1) tau[j] *= tl;
      xh[j] = xt * dinv;
      d[j] = xt;                          // d^0 = x - c
      b[j] = (HK == HK_L2) ? xt : 0.f;    // l2: pending u with s = 1 reproduces d^0, b^0 = 0
      vp[j] = xt;                         // v^0 = x - c
    }
    it = 0;
    s_cur = 1.f;
    sv_ok = false;
  };

  load_point(have);
  if (have) {
    setup_solve(dA, vA);
    if (UNION) { best = __int_as_float(0x7f800000); bestk = -1; bestit = 0; }
  } else {
#pragma unroll
    for (int j = 0; j < CPL; j++) { xh[j] = 0.f; dA[j] = 0.f; b[j] = 0.f; vA[j] = 0.f; if (!KSM) kap[j] = 0.f; }
  }

  // ---- one loop trip: reads (di, vi), writes (dO, vO) ------------------------------------
  // l1/wl1: the full iteration k = it+1, one reduction of (sd, sb, sv).
  // l2: software-pipelined so that one reduction per iteration suffices: the trip finishes
  //     iteration k = it ((3.4b), (3.4c) with the shrink factor s_k reduced in the previous
  //     trip, plus the test sums sd_k, sb_k) and starts iteration k+1 ((3.4a), u_{k+1}, the
  //     test sum sv_{k+1} and ||u_{k+1}||^2); the four sums are reduced together.  Between trips
  //     b[j] holds u_{k+1}; dO = d_k is not touched by the (3.4a) half, so a point that stops at
  //     k outputs d_k.  After setup_solve the first trip's (3.4b) half is the identity (s = 1,
  //     u = x - c) and its test is skipped.
  bool conv = false;
  int kdone = 0;
  auto trip = [&](const float (&di)[CPL], float (&dO)[CPL], const float (&vi)[CPL], float (&vO)[CPL]) {
    float pa0 = 0.f, pa1 = 0.f, pb0 = 0.f, pb1 = 0.f, pc0 = 0.f, pc1 = 0.f, pr0 = 0.f, pr1 = 0.f;
    float kv[4];
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      float kj;
      if (KSM) {
        if (CPL4) {
          if ((j & 3) == 0) { const float4 k4 = lds_volatile4(kappa_ptr(j)); kv[0] = k4.x; kv[1] = k4.y; kv[2] = k4.z; kv[3] = k4.w; }
          kj = kv[j & 3];
        } else {
          kj = lds_volatile(kappa_ptr(j));
        }
      } else {
        kj = kap[j];
      }
      if (HK == HK_L2) {
        const float u = b[j];
        const float dn = s_cur * u;                // (3.4b) shrink_2 of iteration k
        const float dd = dn - di[j];
        const float dmv = dn - vi[j];              // d^k - v^k
        const float bn = u - dn;                   // (3.4c): b + v - d' = u - d'
        if (j & 1) { pa1 = fmaf(dd, dd, pa1); pb1 = fmaf(dmv, dmv, pb1); }
        else       { pa0 = fmaf(dd, dd, pa0); pb0 = fmaf(dmv, dmv, pb0); }
        dO[j] = dn;
        const float a = dn - bn;
        const float v = fmaf(kj, a, xh[j]);        // (3.4a) of iteration k+1
        const float dv = v - vi[j];
        const float un = v + bn;                   // u_{k+1}, argument of the next (3.4b)
        if (j & 1) { pc1 = fmaf(dv, dv, pc1); pr1 = fmaf(un, un, pr1); }
        else       { pc0 = fmaf(dv, dv, pc0); pr0 = fmaf(un, un, pr0); }
        vO[j] = v;
        b[j] = un;
      } else {
        const float a = di[j] - b[j];
        const float v = fmaf(kj, a, xh[j]);        // (3.4a)
        const float dv = v - vi[j];
        vO[j] = v;
        const float u = v + b[j];
        const float tj = (HK == HK_WL1) ? tau[j] : tauS;
        const float bn = fminf(fmaxf(u, -tj), tj); // projection on the box [-tau, tau] (Moreau)
        const float dn = u - bn;                   // (3.4b) shrink_1; (3.4c) b' = u - d' = bn
        const float dd = dn - di[j];
        const float dmv = dn - v;                  // d^k - v^k
        if (j & 1) { pa1 = fmaf(dd, dd, pa1); pb1 = fmaf(dmv, dmv, pb1); pc1 = fmaf(dv, dv, pc1); }
        else       { pa0 = fmaf(dd, dd, pa0); pb0 = fmaf(dmv, dmv, pb0); pc0 = fmaf(dv, dv, pc0); }
        dO[j] = dn;
        b[j] = bn;
      }
    }
    if (HK == HK_L2) {
      float r2;
      bool ok_sd, ok_sb, ok_sv;
      group_reduce4<G>(pa0 + pa1, pb0 + pb1, pc0 + pc1, pr0 + pr1, tol, r2, ok_sd, ok_sb, ok_sv);
      kdone = it;
      conv = (it >= 1) && sv_ok && ok_sd && ok_sb;   // P:1597-1601 for iteration k = it
      sv_ok = ok_sv;                                  // ||v^{k+1} - v^k||^2 <= tol, for the next trip
      const float r = sqrtf(r2);
      s_cur = (r > tauS) ? (r - tauS) / r : 0.f;     // shrink_2 factor of iteration k+1
      it++;
    } else {
      float dummy;
      bool ok_sd, ok_sb, ok_sv;
      group_reduce4<G>(pa0 + pa1, pb0 + pb1, pc0 + pc1, 0.f, tol, dummy, ok_sd, ok_sb, ok_sv);
      it++;
      kdone = it;
      conv = ok_sd && ok_sb && ok_sv;
    }
  };

  // ---- finalize the groups whose solve stopped, refill them (collective) ------------------
  // d = the current d^k, vp = the current v register set (scratch for done groups).
  auto finalize = [&](float (&d)[CPL], float (&vp)[CPL], bool done) {
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
    int status = (spec == 1) ? 0 : (conv ? kdone : -p.max_iter);
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
    // ---- refill: the next set of the point (union) or the next point of this group -------
    if (point_done) {
      pt += ngroups;
      have = pt < p.M;
    }
    load_point(point_done && have);   // collective (ballot inside): all lanes call it
    if (done) {
      if (have) {
        kset = point_done ? 0 : kset + 1;
        if (UNION && point_done) { best = __int_as_float(0x7f800000); bestk = -1; bestit = 0; }
        setup_solve(d, vp);
      } else {
#pragma unroll
        for (int j = 0; j < CPL; j++) { xh[j] = 0.f; d[j] = 0.f; b[j] = 0.f; vp[j] = 0.f; }
        spec = 0;
      }
    }
  };

  auto done_now = [&]() {
    return have && (spec != 0 || (kdone >= 1 && (conv || kdone >= p.max_iter)));
  };

  while (__any_sync(0xffffffffu, have)) {
    trip(dA, dB, vA, vB);
    {
      const bool done = done_now();
      if (__any_sync(0xffffffffu, done)) finalize(dB, vB, done);
    }
    trip(dB, dA, vB, vA);
    {
      const bool done = done_now();
      if (__any_sync(0xffffffffu, done)) finalize(dA, vA, done);
    }
  }
}

}  // namespace hopf
