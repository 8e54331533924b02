// ella_kernel.cuh — NEXT-2, last column: H(p) = ||p||_A = sqrt(<p, A p>) with a full SPD A,
// diagonal J.  sm_100a, FP32 SIMT, one warp per point.
//
// Paper: ||.||_A and the projection on the ellipsoid E_A = {y : <y, A^-1 y> <= 1}
// (P:1433-1486): pi_{E_A}(w) = Q pi_{E_Lambda}(Q^T w) with A = Q diag(Lambda) Q^T, and the
// diagonal projection by Newton on its multiplier (as HK_ELL, reading R27); (3.4b) =
// prox_{tau ||.||_A}(u) = u - tau pi_{E_A}(u / tau) (Moreau).  The rest of the
// iteration is the diagonal one of diag_kernel.cuh.
//
// Per iteration and point: (3.4a) elementwise, u = v + b, u~ = Q^T u (n^2 FMAs), the diagonal
// prox d~ = mu u~ / (Lambda + mu) in the eigenbasis, d = Q d~ (n^2 FMAs), b = u - d.  The two
// rotations read Q and Q^T from shared memory (row-major, coalesced across lanes) and the
// vector being rotated from a per-warp staging buffer (broadcast reads).  Lane l owns
// coordinates i = l + 32 j (j < CPL) in both bases.
#pragma once
#include "diag_kernel.cuh"

namespace hopf {

struct EllAParams {
  int64_t M;
  int n;
  const float *X, *t, *D, *c, *Q, *Lam;   // Q [n*n] row-major, columns = eigenvectors of A
  float gamma, lambda, tol;
  int max_iter;
  float *phi, *grad;
  int *iters;
  unsigned long long *iter_total;
};

constexpr int ELLA_WARPS = 4;

// dynamic shared memory: Q, Q^T [n*n each], Lambda [n], per-warp staging [ELLA_WARPS * n]
template <int CPL>
__global__ void __launch_bounds__(32 * ELLA_WARPS) hopf_ella_kernel(const EllAParams p) {
  extern __shared__ float sm[];
  const int n = p.n;
  float *Qs = sm, *Qt = sm + n * n, *Ls = sm + 2 * n * n, *stg = Ls + n;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const float q = __ldg(p.Q + e);
    Qs[e] = q;
    Qt[(e % n) * n + e / n] = q;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) Ls[i] = __ldg(p.Lam + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float *buf = stg + wib * n;
  float lmin = __int_as_float(0x7f800000);
  for (int i = 0; i < n; i++) lmin = fminf(lmin, Ls[i]);
  const float lam = p.lambda;

  float xt[CPL], kap[CPL], xh[CPL], Dv[CPL], v[CPL], d[CPL], b[CPL], L[CPL];
#pragma unroll
  for (int j = 0; j < CPL; j++) {
    const int i = lane + 32 * j;
    const bool ok = i < n;
    Dv[j] = ok ? __ldg(p.D + i) : 1.f;
    kap[j] = ok ? lam / (Dv[j] + lam) : 0.f;
    L[j] = ok ? Ls[i] : 1.f;
  }
  // rotate: out_i = sum_k R[k][i] in_k for this lane's i (R = Qs gives Q^T in, R = Qt gives Q in)
  auto rotate = [&](const float *R, const float (&in)[CPL], float (&out)[CPL]) {
    __syncwarp();
#pragma unroll
    for (int j = 0; j < CPL; j++)
      if (lane + 32 * j < n) buf[lane + 32 * j] = in[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < CPL; j++) out[j] = 0.f;
    for (int k = 0; k < n; k++) {
      const float a = buf[k];
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const int i = lane + 32 * j;
        out[j] = fmaf(i < n ? R[k * n + i] : 0.f, a, out[j]);
      }
    }
  };

  const int64_t nwarps = (int64_t)gridDim.x * ELLA_WARPS;
  unsigned my_iters = 0;
  for (int64_t pt = (int64_t)blockIdx.x * ELLA_WARPS + wib; pt < p.M; pt += nwarps) {
    const float tt = __ldg(p.t + pt);
    bool bad = !(tt >= 0.f) || !finite_f(tt);
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      const int i = lane + 32 * j;
      const float xv = i < n ? __ldg(p.X + pt * n + i) : 0.f;
      bad |= !finite_f(xv);
      xt[j] = i < n ? xv - (p.c ? __ldg(p.c + i) : 0.f) : 0.f;
      xh[j] = xt[j] / (Dv[j] + lam);
      v[j] = d[j] = xt[j];   // v^0 = d^0 = x - c, b^0 = 0 (R5)
      b[j] = 0.f;
    }
    bad = __any_sync(0xffffffffu, bad);
    float *grow = p.grad + pt * n;
    if (bad || tt == 0.f) {
      // invalid: NaN; t == 0: J(x), grad J(x) (R6)
      float qs = 0.f;
#pragma unroll
      for (int j = 0; j < CPL; j++) qs = fmaf(0.5f * xt[j], xt[j] / Dv[j], qs);
      qs = group_sum<32>(qs);
#pragma unroll
      for (int j = 0; j < CPL; j++)
        if (lane + 32 * j < n) grow[lane + 32 * j] = bad ? __int_as_float(0x7fc00000) : xt[j] / Dv[j];
      if (lane == 0) {
        p.phi[pt] = bad ? __int_as_float(0x7fc00000) : qs + p.gamma;
        p.iters[pt] = bad ? INT32_MIN : 0;
      }
      continue;
    }
    const float tau = tt / lam, itau = 1.f / tau;
    float mu = 0.f, dr[CPL];
    int status = -p.max_iter;
    for (int k = 1; k <= p.max_iter; k++) {
      float u[CPL], ur[CPL], sv = 0.f;
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const float vn = fmaf(kap[j], d[j] - b[j], xh[j]);   // (3.4a)
        const float dv = vn - v[j];
        sv = fmaf(dv, dv, sv);
        v[j] = vn;
        u[j] = vn + b[j];
      }
      rotate(Qs, u, ur);   // u~ = Q^T u
      // diagonal ellipsoid in the eigenbasis: S1(mu) = sum Lambda u~^2 / (Lambda + mu)^2 =
      // tau^2, Newton on 1/sqrt(S1) - 1/tau from the warm start, clamp at 0 (inside: d = 0)
      for (int nit = 0; nit < 30; nit++) {
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int j = 0; j < CPL; j++) {
          const float r = 1.f / (L[j] + mu);
          const float h = ur[j] * r;
          const float wh2 = L[j] * h * h;
          s1 += wh2;
          s2 = fmaf(wh2, r, s2);
        }
        s1 = group_sum<32>(s1);
        s2 = group_sum<32>(s2);
        const float mun = s2 > 0.f ? fmaxf(fmaf(s1 / s2, fmaf(sqrtf(s1), itau, -1.f), mu), 0.f) : 0.f;
        const bool stop = fabsf(mun - mu) <= 1e-6f * (mun + lmin);
        mu = mun;
        if (stop) break;
      }
#pragma unroll
      for (int j = 0; j < CPL; j++) dr[j] = mu * ur[j] / (L[j] + mu);   // (3.4b) in the eigenbasis
      float dn[CPL];
      rotate(Qt, dr, dn);   // d = Q d~
      float sd = 0.f, sb = 0.f;
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const float dd = dn[j] - d[j];
        sd = fmaf(dd, dd, sd);
        const float dmv = dn[j] - v[j];
        sb = fmaf(dmv, dmv, sb);
        d[j] = dn[j];
        b[j] = u[j] - dn[j];                                  // (3.4c)
      }
      sv = group_sum<32>(sv);
      sd = group_sum<32>(sd);
      sb = group_sum<32>(sb);
      if (sv <= p.tol && sd <= p.tol && sb <= p.tol) { status = k; break; }
    }
    my_iters += (unsigned)(status > 0 ? status : -status);
    // phi = <x - c, d> - 1/2 <d, D d> - t ||d||_A + gamma, ||d||_A^2 = sum Lambda d~^2
    float qs = 0.f, ha = 0.f;
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      qs = fmaf(xt[j], d[j], fmaf(-0.5f * Dv[j] * d[j], d[j], qs));
      ha = fmaf(L[j] * dr[j], dr[j], ha);
    }
    qs = group_sum<32>(qs);
    ha = group_sum<32>(ha);
#pragma unroll
    for (int j = 0; j < CPL; j++)
      if (lane + 32 * j < n) grow[lane + 32 * j] = d[j];
    if (lane == 0) {
      p.phi[pt] = qs - tt * sqrtf(ha) + p.gamma;
      p.iters[pt] = status;
    }
  }
  if (p.iter_total && lane == 0 && my_iters) atomicAdd(p.iter_total, (unsigned long long)my_iters);
}

}  // namespace hopf
