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
  unsigned long long *claim;   // the launch's point counter (zeroed before the launch); null: static
};

constexpr int ELLA_WARPS = 4;

// sum over the G lanes of this lane's group, with only those lanes' mask (the groups of a warp
// may have taken different branches at the end of a point)
template <int G>
__device__ __forceinline__ float group_sum_sub(float v) {
  const int lane = threadIdx.x & 31;
  const unsigned m = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o);
  return v;
}

// dynamic shared memory: Q, Q^T [n*n each], Lambda [n], per-point staging [ELLA_WARPS * 32/G * n].
// G lanes per point (G = 16: two points per warp for n <= 16, the paper's Table 4 sizes); the
// points of a warp iterate in lockstep, a finished one frozen until its partner stops.
template <int G, int CPL>
__global__ void __launch_bounds__(32 * ELLA_WARPS) hopf_ella_kernel(const EllAParams p) {
  constexpr int GPW = 32 / G;
  extern __shared__ float sm[];
  const int n = p.n;
  // rows padded to nr = n rounded up to 16 floats (>= CPL, a multiple of 4): a lane's CPL
  // contiguous coordinates of a row are vector loads (lane l owns coordinates CPL l + j)
  const int nr = (n + 15) & ~15;
  float *Qs = sm, *Qt = sm + n * nr, *Ls = sm + 2 * n * nr, *stg = Ls + n;
  for (int e = threadIdx.x; e < n * nr; e += blockDim.x) {
    const int r = e / nr, col = e % nr;
    Qs[e] = col < n ? __ldg(p.Q + r * n + col) : 0.f;
    Qt[e] = col < n ? __ldg(p.Q + col * n + r) : 0.f;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) Ls[i] = __ldg(p.Lam + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gl = lane & (G - 1), sub = lane / G;
  float *buf = stg + (wib * GPW + sub) * n;
  float lmin = __int_as_float(0x7f800000);
  for (int i = 0; i < n; i++) lmin = fminf(lmin, Ls[i]);
  const float lam = p.lambda;

  float xt[CPL], kap[CPL], xh[CPL], Dv[CPL], v[CPL], d[CPL], b[CPL], L[CPL];
#pragma unroll
  for (int j = 0; j < CPL; j++) {
    const int i = CPL * gl + j;
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
      if (CPL * gl + j < n) buf[CPL * gl + j] = in[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < CPL; j++) out[j] = 0.f;
    if (CPL * gl < nr) {   // lanes past the padded row have only padded slots
      for (int k = 0; k < n; k++) {
        const float a = buf[k];
        const float *row = R + k * nr + CPL * gl;   // padded columns hold 0
        if constexpr (CPL % 4 == 0) {
#pragma unroll
          for (int j4 = 0; j4 < CPL / 4; j4++) {
            const float4 r4 = *reinterpret_cast<const float4 *>(row + 4 * j4);
            out[4 * j4] = fmaf(r4.x, a, out[4 * j4]); out[4 * j4 + 1] = fmaf(r4.y, a, out[4 * j4 + 1]);
            out[4 * j4 + 2] = fmaf(r4.z, a, out[4 * j4 + 2]); out[4 * j4 + 3] = fmaf(r4.w, a, out[4 * j4 + 3]);
          }
        } else if constexpr (CPL == 2) {
          const float2 r2 = *reinterpret_cast<const float2 *>(row);
          out[0] = fmaf(r2.x, a, out[0]); out[1] = fmaf(r2.y, a, out[1]);
        } else {
#pragma unroll
          for (int j = 0; j < CPL; j++) out[j] = fmaf(row[j], a, out[j]);
        }
      }
    }
  };

  const int64_t nslots = (int64_t)gridDim.x * ELLA_WARPS * GPW;
  unsigned my_iters = 0;
  // batches of GPW points: the first two of a warp static, later ones claimed from p.claim one
  // batch ahead (warps that drew cheap batches take more; the launch ends within one batch)
  __shared__ unsigned zero_lanes[32];
  zero_lanes_init(zero_lanes);
  __syncthreads();
  int64_t bnext = ((int64_t)blockIdx.x * ELLA_WARPS + wib) * GPW + nslots;
  unsigned long long wclaim = 0;   // lane 0: the claim made at the current batch's start
  auto next_batch = [&]() {
    const int64_t nb = bnext;
    bnext = p.claim ? (int64_t)__shfl_sync(0xffffffffu, wclaim, 0) + 2 * nslots : bnext + nslots;
    return nb;
  };
  for (int64_t base = ((int64_t)blockIdx.x * ELLA_WARPS + wib) * GPW; base < p.M; base = next_batch()) {
    {
      const unsigned zoff = lane_zero(zero_lanes, lane);
      if (lane == 0 && p.claim) wclaim = atomicAdd(p.claim + zoff, (unsigned long long)GPW);
    }
    const int64_t pt = base + sub;
    const bool have = pt < p.M;
    const float tt = have ? __ldg(p.t + pt) : 1.f;
    bool bad = !(tt >= 0.f) || !finite_f(tt);
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      const int i = CPL * gl + j;
      const float xv = (have && i < n) ? __ldg(p.X + pt * n + i) : 0.f;
      bad |= !finite_f(xv);
      xt[j] = i < n ? xv - (p.c ? __ldg(p.c + i) : 0.f) : 0.f;
      xh[j] = xt[j] / (Dv[j] + lam);
      v[j] = d[j] = xt[j];   // v^0 = d^0 = x - c, b^0 = 0 (R5)
      b[j] = 0.f;
    }
    bad = group_any<G>(bad);
    const bool direct = bad || tt == 0.f;   // invalid: NaN; t == 0: J(x), grad J(x) (R6)
    const float tau = tt / lam, itau = 1.f / tau;
    float mu = 0.f, dr[CPL];
#pragma unroll
    for (int j = 0; j < CPL; j++) dr[j] = 0.f;
    bool live = have && !direct;
    int status = -p.max_iter;
    for (int k = 1; k <= p.max_iter; k++) {
      if (!__any_sync(0xffffffffu, live)) break;
      float u[CPL], ur[CPL], sv = 0.f;
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const float vn = fmaf(kap[j], d[j] - b[j], xh[j]);   // (3.4a)
        const float dv = vn - v[j];
        sv = fmaf(dv, dv, sv);
        u[j] = vn + b[j];
        if (live) v[j] = vn;
      }
      rotate(Qs, u, ur);   // u~ = Q^T u
      // diagonal ellipsoid in the eigenbasis: S1(mu) = sum Lambda u~^2 / (Lambda + mu)^2 =
      // tau^2, Newton on 1/sqrt(S1) - 1/tau from the warm start, clamp at 0 (inside: d = 0)
      bool act = live;
      float mut = mu;
      for (int nit = 0; nit < 30; nit++) {
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int j = 0; j < CPL; j++) {
          const float r = 1.f / (L[j] + mut);
          const float h = ur[j] * r;
          const float wh2 = L[j] * h * h;
          s1 += wh2;
          s2 = fmaf(wh2, r, s2);
        }
        s1 = group_sum<G>(s1);
        s2 = group_sum<G>(s2);
        if (act) {
          const float mun = s2 > 0.f ? fmaxf(fmaf(s1 / s2, fmaf(sqrtf(s1), itau, -1.f), mut), 0.f) : 0.f;
          act = !(fabsf(mun - mut) <= 1e-6f * (mun + lmin));
          mut = mun;
        }
        if (!__any_sync(0xffffffffu, act)) break;
      }
      float drn[CPL];
#pragma unroll
      for (int j = 0; j < CPL; j++) drn[j] = mut * ur[j] / (L[j] + mut);   // (3.4b) in the eigenbasis
      float dn[CPL];
      rotate(Qt, drn, dn);   // d = Q d~
      float sd = 0.f, sb = 0.f;
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const float dd = dn[j] - d[j];
        sd = fmaf(dd, dd, sd);
        const float dmv = dn[j] - v[j];
        sb = fmaf(dmv, dmv, sb);
      }
      sv = group_sum<G>(sv);
      sd = group_sum<G>(sd);
      sb = group_sum<G>(sb);
      if (live) {
        mu = mut;
#pragma unroll
        for (int j = 0; j < CPL; j++) {
          d[j] = dn[j];
          b[j] = u[j] - dn[j];                                // (3.4c)
          dr[j] = drn[j];
        }
        if (sv <= p.tol && sd <= p.tol && sb <= p.tol) { status = k; live = false; }
      }
    }
    if (!have) continue;
    float *grow = p.grad + pt * n;
    if (direct) {
      float qs = 0.f;
#pragma unroll
      for (int j = 0; j < CPL; j++) qs = fmaf(0.5f * xt[j], xt[j] / Dv[j], qs);
      qs = group_sum_sub<G>(qs);
#pragma unroll
      for (int j = 0; j < CPL; j++)
        if (CPL * gl + j < n) grow[CPL * gl + j] = bad ? __int_as_float(0x7fc00000) : xt[j] / Dv[j];
      if (gl == 0) {
        p.phi[pt] = bad ? __int_as_float(0x7fc00000) : qs + p.gamma;
        p.iters[pt] = bad ? INT32_MIN : 0;
      }
      continue;
    }
    my_iters += (unsigned)(status > 0 ? status : -status);
    // phi = <x - c, d> - 1/2 <d, D d> - t ||d||_A + gamma, ||d||_A^2 = sum Lambda d~^2
    float qs = 0.f, ha = 0.f;
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      qs = fmaf(xt[j], d[j], fmaf(-0.5f * Dv[j] * d[j], d[j], qs));
      ha = fmaf(L[j] * dr[j], dr[j], ha);
    }
    qs = group_sum_sub<G>(qs);
    ha = group_sum_sub<G>(ha);
#pragma unroll
    for (int j = 0; j < CPL; j++)
      if (CPL * gl + j < n) grow[CPL * gl + j] = d[j];
    if (gl == 0) {
      p.phi[pt] = qs - tt * sqrtf(ha) + p.gamma;
      p.iters[pt] = status;
    }
  }
  if (p.iter_total && gl == 0 && my_iters) atomicAdd(p.iter_total, (unsigned long long)my_iters);
}

}  // namespace hopf
