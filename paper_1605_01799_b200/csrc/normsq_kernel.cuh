// normsq_kernel.cuh — NEXT-3: split Bregman for the non-quadratic initial data
//   J = 1/2 ||.||_1^2  (J* = 1/2 ||.||_inf^2)   or   J = 1/2 ||.||_inf^2  (J* = 1/2 ||.||_1^2),
// plus gamma, with H in {l1, weighted l1, l2, l_inf}.  sm_100a, FP32 SIMT.
//
// Paper: split Bregman (3.4a)-(3.4c) P:832-844; stopping rule P:1597-1601; prox of
// 1/2||.||_1^2 by the multiplier beta = alpha ||shrink_1(z, beta)||_1; prox of
// 1/2||.||_inf^2 by Moreau (reading R29); l_inf H by the l1-ball projection
// (P:1348-1428); Tables 2, 3 and 5.
//
// (3.4a) is no longer elementwise: v = prox_{J*/lambda}(z), z = d - b + x/lambda, and both proxes
// reduce to one scalar multiplier per point found from the active set {i : |z_i| > m}:
//   J = 1/2||.||_1^2 : v = clamp(z, -beta, beta),   beta = lambda sum_i max(|z_i| - beta, 0)
//   J = 1/2||.||_inf^2: v = shrink_1(z, beta),       beta = (1/lambda) sum_i max(|z_i| - beta, 0)
// (the first is z - (1/lambda) shrink_1(lambda z, lambda beta) with the paper's beta for
// alpha = lambda, rescaled; reading R29).  The l_inf d-update is the same kind of
// root: d' = clamp(u, -mu, mu), sum_i max(|u_i| - mu, 0) = t / lambda (as HK_LINF in
// diag_kernel.cuh).  Every such root is F(m) = a S(m) - c m - e = 0 with S(m) =
// sum max(|z_i| - m, 0), F convex, decreasing and piecewise affine; its Newton step from m is
// m' = (a S_A - e) / (a |A| + c) over the active set A = {|z_i| > m}, which lands at or left of
// the root from the right and increases monotonically to it from the left; a step whose active
// set is unchanged at m' is exact (the root of the affine piece).  Warm-started at the previous
// iteration's multiplier, clamped at 0.  The paper sorts the breakpoints and interpolates
// (O(n log n)); both give the same root.
//
// Layout and scheduling as hopf_diag_kernel: a group of G lanes owns one point, lane l holds
// coordinates i = l + G j (j < CPL) in registers; persistent grid; a group whose point stops
// writes its results and loads the next point while the rest of the warp iterates.  H is a
// runtime (warp-uniform) switch; J and the shape are template parameters.
#pragma once
#include "diag_kernel.cuh"

namespace hopf {

enum { JK_L1SQ = 0, JK_LINFSQ = 1 };

struct NormsqParams {
  int64_t M;
  int n;
  const float *X, *t, *w;
  float gamma, lambda, tol;
  int max_iter, h;
  float *phi, *grad;
  int *iters;
  unsigned long long *iter_total;
  unsigned long long *claim;   // the launch's point counter (zeroed before the launch); null: static
};

// Root m >= 0 of a S(m) - c m - e (see above) for the values |z_i| of this lane's CPL slots;
// `act` groups iterate, the others keep m.  Collective over the warp.
template <int G, int CPL>
__device__ __forceinline__ float active_set_root(const float (&z)[CPL], float a, float c, float e,
                                                 float m, bool act) {
  // S(me) = sum max(|z_i| - me, 0) summed as small terms and the active count |A| = #{|z_i| > me}
  // (group totals).  Both on the FMA pipe (this kernel is ALU-bound): max(x, 0) = (x + |x|) / 2
  // (exact), and [x > 0] = sat(x 2^126) (exact: under FTZ a positive x is >= 2^-126)
  auto eval = [&](float me, float &sa, float &na) {
    float s2 = 0.f, cn = 0.f;
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      const float ex = fabsf(z[j]) - me;
      s2 += ex + fabsf(ex);
      cn += __saturatef(ex * 8.50705917e37f);
    }
    sa = 0.5f * group_sum<G>(s2);
    na = group_sum<G>(cn);
  };
  float me = m;   // evaluation point
  float sa, na;
  eval(me, sa, na);
  for (int nit = 0;; nit++) {
    // Newton step in delta form me + F(me) / (a |A| + c): S_A - |A| me would cancel
    // catastrophically when the root sits just below a cluster of |z_i| (tiny t / clamped
    // coordinates)
    float mn = me;
    if (act) {
      const float den = fmaf(a, na, c);
      const float F = fmaf(a, sa, -fmaf(c, me, e));
      mn = den > 0.f ? fmaxf(me + __fdividef(F, den), 0.f) : 0.f;
    }
    // an evaluation point above every |z_i| (empty active set; the warm start can overshoot
    // there when the root sits within a few ulps of max |z_i|, e.g. tiny t): the Newton step
    // would fall to 0 and climb back through every breakpoint.  Step instead to the root of the
    // top piece's extension, m = (a max|z| - e) / (a + c), which is at or left of the root
    // (F is convex and decreasing), so the iteration proceeds monotonically from there
    if (__any_sync(0xffffffffu, act && na == 0.f)) {
      float zm = 0.f;
#pragma unroll
      for (int j = 0; j < CPL; j++) zm = fmaxf(zm, fabsf(z[j]));
      zm = group_max<G>(zm);
      if (act && na == 0.f) mn = fmaxf(__fdividef(fmaf(a, zm, -e), a + c), 0.f);
    }
    // a breakpoint at the root (|z_i| = m: coordinates clamped exactly at the multiplier, the
    // typical state of these l1 / l_inf problems near convergence) makes fp32 steps alternate
    // across it; a step within a few ulps of m is accepted as the root
    const bool tiny = fabsf(mn - me) <= HOPF_TINY_STEP * fmaxf(mn, 1e-30f);
    if (act && (tiny || nit >= 63)) { m = mn; act = false; }
    if (!__any_sync(0xffffffffu, act)) break;
    // the step is exact when no |z_i| lies between me and mn, i.e. when the active count at mn
    // equals the one at me; otherwise the evaluation at mn is the next Newton evaluation
    float sn, nn;
    eval(mn, sn, nn);
    if (act && nn == na) { m = mn; act = false; }
    if (!__any_sync(0xffffffffu, act)) break;
    if (act) { me = mn; sa = sn; na = nn; }
  }
  return m;
}

// H is a template parameter (HKr): the loop body carries only its own prox
template <int G, int CPL, int JK, int HKr>
__global__ void __launch_bounds__(128, CPL <= 8 ? 4 : 3) hopf_normsq_kernel(const NormsqParams p) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int n = p.n;
  const float lam = p.lambda, ilam = 1.f / p.lambda, tol = p.tol;
  const int jmax = (n - gl + G - 1) / G;

  float x[CPL], d[CPL], b[CPL], v[CPL], wr[CPL];
  // points: the first two of a group static (gid, gid + ngroups), later ones claimed by the
  // group from p.claim one point ahead.  Iteration counts vary widely here (Table 5: 30 to
  // max_iter), so a static assignment leaves long tails of nearly idle warps.
  __shared__ unsigned zero_lanes[32];
  zero_lanes_init(zero_lanes);
  __syncthreads();
  int64_t pt = gid, pnext = gid + ngroups;
  unsigned long long gclaim = 0;   // group lane 0: the claim made at the last point start
  bool have = pt < p.M;
  int it = 0, spec = 0;
  float tt = 0.f, tau = 0.f, beta = 0.f, mu = 0.f;
  float dbeta = 0.f, dmu = 0.f;   // last change of each multiplier: the warm start extrapolates
  unsigned my_iters = 0;

  auto load = [&](bool active) {
    bool bad = false;
    const unsigned zoff = lane_zero(zero_lanes, lane);
    if (active) {
      if (gl == 0 && p.claim) gclaim = atomicAdd(p.claim + zoff, 1ull);
      tt = __ldg(p.t + pt);
      bad = !(tt >= 0.f) || !finite_f(tt);
      const float *xrow = p.X + pt * (int64_t)n;
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        x[j] = j < jmax ? __ldg(xrow + gl + G * j) : 0.f;
        bad |= !finite_f(x[j]);
      }
    }
    bad = group_any<G>(bad);
    if (active) {
      spec = bad ? 2 : (tt == 0.f ? 1 : 0);
      tau = tt * ilam;
      // v^0 = d^0 = x, b^0 = 0
#pragma unroll
      for (int j = 0; j < CPL; j++) { v[j] = x[j]; d[j] = x[j]; b[j] = 0.f; }
      it = 0;
      beta = 0.f;
      mu = 0.f;
      dbeta = dmu = 0.f;
    }
  };
#pragma unroll
  for (int j = 0; j < CPL; j++) {
    wr[j] = (p.w && j < jmax) ? __ldg(p.w + gl + G * j) : (j < jmax ? 1.f : 0.f);
    x[j] = d[j] = b[j] = v[j] = 0.f;
  }
  load(have);

  while (__any_sync(0xffffffffu, have)) {
    const bool act = have && spec == 0;
    // ---- (3.4a): v = prox_{J*/lambda}(z), z = d - b + x / lambda ---------------------------
    float z[CPL];
#pragma unroll
    for (int j = 0; j < CPL; j++) z[j] = fmaf(x[j], ilam, d[j] - b[j]);
    // beta = alpha S(beta): a = alpha, c = 1, e = 0; alpha = lambda (J = 1/2||.||_1^2, the
    // rescaled multiplier) or 1/lambda (J = 1/2||.||_inf^2)
    {
      // warm start at the linear extrapolation of the multiplier (the split Bregman iterates
      // converge geometrically): closer starts keep the active set, so more first steps are exact
      const float b0 = fmaxf(beta + dbeta, 0.f);
      const float bn = active_set_root<G, CPL>(z, JK == JK_L1SQ ? lam : ilam, 1.f, 0.f, b0, act);
      if (act) { dbeta = bn - beta; beta = bn; }
    }
    float sv = 0.f, u[CPL];
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      const float cz = fminf(fmaxf(z[j], -beta), beta);
      const float vn = (JK == JK_L1SQ) ? cz : z[j] - cz;   // clamp / shrink_1
      const float dv = vn - v[j];
      sv = fmaf(dv, dv, sv);
      v[j] = vn;
      u[j] = vn + b[j];
    }
    // ---- (3.4b): d' = prox_{(t/lambda) H}(u) ------------------------------------------------
    float s2 = 0.f;
    if constexpr (HKr == HK_L2) {
#pragma unroll
      for (int j = 0; j < CPL; j++) s2 = fmaf(u[j], u[j], s2);
      s2 = group_sum<G>(s2);
    }
    if constexpr (HKr == HK_LINF) {
      const float m0 = fmaxf(mu + dmu, 0.f);
      const float mn = active_set_root<G, CPL>(u, 1.f, 0.f, tau, m0, act);
      if (act) { dmu = mn - mu; mu = mn; }
    }
    const float sh = (s2 > tau * tau) ? fmaf(-tau, rsqrtf(s2), 1.f) : 0.f;
    float sd = 0.f, sb = 0.f;
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      float dn;
      if constexpr (HKr == HK_L2) dn = sh * u[j];
      else if constexpr (HKr == HK_LINF) dn = fminf(fmaxf(u[j], -mu), mu);
      else {
        const float th = (HKr == HK_WL1 ? wr[j] : 1.f) * tau;
        dn = u[j] - fminf(fmaxf(u[j], -th), th);         // shrink_1 (Moreau)
      }
      const float dd = dn - d[j];
      sd = fmaf(dd, dd, sd);
      const float dmv = dn - v[j];
      sb = fmaf(dmv, dmv, sb);
      d[j] = dn;                                         // (inactive groups: values unused)
      b[j] = u[j] - dn;                                  // (3.4c): b + v - d' = u - d'
    }
    float r3;
    bool ok_sd, ok_sb, ok_sv;
    group_reduce4<G>(sd, sb, sv, 0.f, tol, r3, ok_sd, ok_sb, ok_sv);
    (void)r3;
    bool done = false;
    int status = 0;
    if (have) {
      if (spec != 0) {
        done = true;
        status = spec == 2 ? INT32_MIN : 0;
      } else {
        it++;
        const bool conv = ok_sd && ok_sb && ok_sv;
        if (conv || it >= p.max_iter) {
          done = true;
          status = conv ? it : -p.max_iter;
          my_iters += (unsigned)it;
        }
      }
    }
    if (!__any_sync(0xffffffffu, done)) continue;

    // ---- finalize (all lanes; stores by the groups that stopped) ---------------------------
    // phi = <x, d> - J*(d) - t H(d) + gamma ((3.3) at d, reading R2); t == 0: J(x) and the
    // minimal-norm subgradient of J (reading R30)
    float xd = 0.f, l1 = 0.f, mx = 0.f, l2 = 0.f, wl = 0.f;
    const bool t0 = spec == 1;
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      const float q = t0 ? x[j] : d[j];
      xd = fmaf(x[j], q, xd);
      l1 += fabsf(q);
      mx = fmaxf(mx, fabsf(q));
      l2 = fmaf(q, q, l2);
      wl = fmaf(wr[j], fabsf(q), wl);
    }
    xd = group_sum<G>(xd);
    l1 = group_sum<G>(l1);
    mx = group_max<G>(mx);
    l2 = group_sum<G>(l2);
    wl = group_sum<G>(wl);
    float cnt = 0.f;   // t == 0, J = 1/2||.||_inf^2: number of maximal |x_i|
#pragma unroll
    for (int j = 0; j < CPL; j++) cnt += (j < jmax && fabsf(x[j]) == mx) ? 1.f : 0.f;
    cnt = group_sum<G>(cnt);
    const int64_t claimed = p.claim ? (int64_t)__shfl_sync(0xffffffffu, gclaim, lane & ~(G - 1)) + 2 * ngroups
                                    : pnext + ngroups;   // no counter: static stride
    if (done) {
      float phiv, g[CPL];
      if (spec == 2) {
        phiv = __int_as_float(0x7fc00000);
#pragma unroll
        for (int j = 0; j < CPL; j++) g[j] = __int_as_float(0x7fc00000);
      } else if (t0) {
        const float s = (JK == JK_L1SQ) ? l1 : mx;
        phiv = 0.5f * s * s + p.gamma;
#pragma unroll
        for (int j = 0; j < CPL; j++) {
          const float sg = x[j] > 0.f ? 1.f : (x[j] < 0.f ? -1.f : 0.f);
          g[j] = (JK == JK_L1SQ) ? s * sg
                                 : ((mx > 0.f && fabsf(x[j]) == mx) ? s * sg / cnt : 0.f);
        }
      } else {
        const float js = (JK == JK_L1SQ) ? mx : l1;   // J*(d) = 1/2 ||d||_inf^2 or 1/2 ||d||_1^2
        const float hv = HKr == HK_L2 ? sqrtf(l2) : (HKr == HK_LINF ? mx : (HKr == HK_WL1 ? wl : l1));
        phiv = xd - 0.5f * js * js - tt * hv + p.gamma;
#pragma unroll
        for (int j = 0; j < CPL; j++) g[j] = d[j];
      }
      if (gl == 0) { p.phi[pt] = phiv; p.iters[pt] = status; }
      float *grow = p.grad + pt * (int64_t)n;
#pragma unroll
      for (int j = 0; j < CPL; j++)
        if (j < jmax) grow[gl + G * j] = g[j];
      pt = pnext;
      pnext = claimed;
      have = pt < p.M;
    }
    load(done && have);   // collective
    if (done && !have) spec = 0;
  }
  if (p.iter_total && gl == 0 && my_iters) atomicAdd(p.iter_total, (unsigned long long)my_iters);
}

}  // namespace hopf
