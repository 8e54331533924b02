// diag_tmu.cuh — K4g: the union of K diagonal initial data (phi = min_k phi_k) with
// G lanes per point and tensor memory as an extension of the register file (H = l2; C5).
// sm_100a, FP32 SIMT; no MMA.
//
// Paper: min over initial data P:628-667 (phi = min_k phi_k, the lowest k wins ties, R19); each
// phi_k by split Bregman (3.4a)-(3.4c) P:832-844 on the centred problem at x - c_k (R5) with the
// paper's stopping rule P:1595-1601, shrink_2 P:279-287, phi_k = (3.3) at d (R2); the closest
// (Hopf-Lax terminal) point y = x - t grad/||grad||, y = c_k* when
// grad = 0 (R18).  Same arithmetic as hopf_diag_kernel<G, CPL, HK_L2, true> (diag_kernel.cuh);
// the storage and control flow are those of the grouped kernel (diag_tmg.cuh):
//
//   registers : d (as -d), b (the pending u) of the current set — 2 x CPL floats per lane
//   TMEM      : x_hat_k (columns 0-31), v (32-63), -kappa_k (64-95) of the current set
//   shared    : (D_k, c_k) of every set and gamma_k; per group two x rows (the current point and
//               the prefetched next one, bulk copies), and two grad rows (the best set's grad and
//               the candidate of the set that just stopped)
//
// A group's K set solves run one after another; a set that stops parks its d in the candidate
// row and the group waits.  When enough groups of the warp wait, the warp runs one batched event:
// phi_k of every parked set, the running minimum (the candidate row becomes the best row on an
// improvement: a swap, no copy), the point's outputs for groups whose last set finished (phi,
// iters, k*, the grad row and the y row by bulk stores, y formed in place in the x row), and the
// next set's (or next point's) x_hat, v, kappa into TMEM.  x is read once per point from HBM.
#pragma once
#include <cfloat>
#include <cstdint>
#include <cuda_runtime.h>

#include "diag_tmg.cuh"

namespace hopf {
namespace dtu {

using dtg::THREADS;
// TMEM: three regions of 16 columns (x_hat, v, -kappa) fit a 64-column allocation for CPL <= 16,
// so up to 8 blocks fit the SM's 512 columns; registers and shared memory then set residency
template <int CPL> struct Cols {
  static constexpr int R = CPL <= 16 ? 16 : 32;          // region width
  static constexpr int XH = 0, V = R, K = 2 * R, U = 3 * R;   // U: u_k parked by non-final trips
  static constexpr int ALLOC = 3 * R <= 64 ? 64 : 128;   // power of two >= 32
};
#ifndef HOPF_TMU_BLOCKS
#define HOPF_TMU_BLOCKS 4   // resident blocks per SM (C5: 4 -> 11.04 ms at 127 registers, 5 -> 12.07 at 96, 6 -> 15.6)
#endif
constexpr int BLOCKS_PER_SM = HOPF_TMU_BLOCKS;
constexpr int DYN_SMEM = (226 * 1024) / BLOCKS_PER_SM - 1024;

// shared-memory bytes for K sets: (D, c) tables, gamma, 4 rows per group, 2 mbarriers per group
// (UNAL: rows start at offset (r n) mod 4 in their buffers, 3 floats more)
template <int G, int CPL, bool UNAL>
__host__ __device__ constexpr size_t smem_bytes(int K) {
  return (size_t)K * G * CPL * 8 + (((size_t)K * 4 + 15) & ~(size_t)15) +
         (size_t)4 * (THREADS / G) * dtg::row_pitch(G * CPL + (UNAL ? 4 : 0), G) * 4 + (size_t)(THREADS / G) * 16;
}

#ifndef HOPF_TMU_WAIT8
#define HOPF_TMU_WAIT8 8  // run the event when this many eighths of the warp's groups wait
#endif                    // (C5, 8 groups: 2 -> 11.75 ms, 3 -> 12.38, 4 -> 11.04, 5 -> 13.98, 6 -> 12.53, 7 -> 11.39, 8 -> 9.79)

// UNAL: n % 4 != 0 (rows do not all start on a 16-byte boundary; a separate instance keeps the
// aligned case's code as it was: the unaligned bookkeeping cost C5 ~4 % when shared)
template <int G, int CPL, bool UNAL>
__global__ void __launch_bounds__(THREADS, BLOCKS_PER_SM) hopf_union_tmg_kernel(const DiagParams p) {
  constexpr int C_XH = Cols<CPL>::XH, C_V = Cols<CPL>::V, C_K = Cols<CPL>::K, C_U = Cols<CPL>::U,
                TMEM_COLS = Cols<CPL>::ALLOC;
  static_assert(Cols<CPL>::U + Cols<CPL>::R <= Cols<CPL>::ALLOC, "u region inside the allocation");
  static_assert(G >= 2 && G <= 16 && (G & (G - 1)) == 0, "G in {2, 4, 8, 16}");
  static_assert(CPL % 2 == 0 && CPL <= 32 && (CPL % 8 == 0 || CPL % 8 == 2 || CPL % 8 == 4),
                "CPL = 8 a + {0, 2, 4}, at most 32");
  constexpr int NP = CPL / 2;
  constexpr int GPW = 32 / G, GPB = THREADS / G;
  constexpr int PITCH = dtg::row_pitch(G * CPL + (UNAL ? 4 : 0), G);   // UNAL: rows at offset (r n) mod 4
  constexpr int WAIT_THRESHOLD = (GPW * HOPF_TMU_WAIT8 / 8) > 0 ? (GPW * HOPF_TMU_WAIT8 / 8) : 1;
  using dtg::ldn;
  using dtg::stn;
  using dtg::wait_ld;
  using dtg::for_chunks;
  extern __shared__ __align__(16) uint8_t dyn_smem[];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int grp = threadIdx.x / G;
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int n = p.n, K = p.K;
  const int64_t M = p.M;
  const float lam = p.lambda, tol = p.tol;
  const int jmax = (n - gl + G - 1) / G;
  // shared memory layout (see smem_bytes)
  float2 *const DC_s = reinterpret_cast<float2 *>(dyn_smem);            // [K][G * CPL] (D, c)
  float *const gk_s = reinterpret_cast<float *>(DC_s + K * G * CPL);    // [K]
  float *const rows = reinterpret_cast<float *>(dyn_smem + (((size_t)K * G * CPL * 8 + (size_t)K * 4 + 15) & ~(size_t)15));
  float *const xrow0 = rows + (size_t)(4 * grp) * PITCH;   // x rows 0, 1; grad rows 2, 3
  uint64_t *const bars = reinterpret_cast<uint64_t *>(rows + (size_t)4 * GPB * PITCH) + 2 * grp;
  const unsigned gmask = ((1u << G) - 1u) << (lane & ~(G - 1));
  for (int e = threadIdx.x; e < K * G * CPL; e += THREADS) {
    const int k = e / (G * CPL), i = e % (G * CPL);
    const bool real = i < n;
    DC_s[e] = make_float2(real ? __ldg(p.D + (size_t)k * n + i) : 1.f,
                          real ? __ldg(p.c + (size_t)k * n + i) : 0.f);
  }
  for (int k = threadIdx.x; k < K; k += THREADS) gk_s[k] = __ldg(p.gk + k);
  if (gl == 0) {
    dtg::mbar_init(dtg::smem_u32(bars), 1);
    dtg::mbar_init(dtg::smem_u32(bars + 1), 1);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&tmem_slot)), "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tl0 = __shfl_sync(0xffffffffu, tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16), 0);
  auto xrow = [&](int s) { return xrow0 + s * PITCH; };
  auto grow_s = [&](int s) { return xrow0 + (2 + s) * PITCH; };

  float2 d[NP], b[NP];   // -d, pending u (l2 storage of the trip)
  // points: the first three of a group static (gid + r ngroups, r < 3), later ones claimed by
  // the group from p.claim one point ahead (the atomic's latency is hidden by a whole point), so
  // groups that drew cheap points take more of them and the launch ends within about one point
  int64_t pt = gid, p1 = gid + ngroups, p2 = gid + 2 * ngroups;
  unsigned long long gclaim = 0;   // group lane 0: the claim made at the last point start
  bool have = pt < M;
  bool waiting = false;
  int wstatus = 0, it = 0, lim = 0, spec = 0, kset = 0;
  float tt = 0.f, tauS = 0.f, s_cur = 1.f;
  bool sv_ok = false;
  // A non-final trip does not form -d_k = -s_k u_k: it parks u_k in the TMEM region C_U and the
  // warp-uniform dfull goes false; fix_d forms -d from there (per lane s_prev = s_k) when a final
  // trip or a stopping set needs it.  A set start writes u := x - c_k with s_prev = 1, so the
  // rule -d = -s_prev u holds for every group whenever dfull is false.
  bool dfull = true;
  float s_prev = 1.f;
  // distance mode (NEXT-1): non-null p.dist; the point is the query y, evaluated at
  // s_0 = 0 and then at the Newton iterates s_l (p.t is not read)
  const bool DIST = p.dist != nullptr;
  float tpre = (have && !DIST) ? __ldg(p.t + pt) : 0.f;
  int nn = 0;               // Newton evaluations at s > 0 so far
  float s_lo = 0.f, s_hi = 0.f;   // bracket of the root (R25)
  uint32_t xph = 0;        // parity bits of the two x-row mbarriers
  int xs = 0;              // x row of the current point
  int cand = 0;            // grad row that receives the next stopped set's d (the other is the best)
  float best = 0.f, bgn = 0.f;
  int bestk = -1, bestit = 0;
#pragma unroll
  for (int q = 0; q < NP; q++) d[q] = b[q] = splat2(0.f);
  // x row of point r into row buffer sb: the 16-byte aligned part by a bulk copy (leader) at
  // buffer offset (r n) mod 4, the last (r n + n) mod 4 floats by 4-byte cp.async of lanes
  // gl < that count (no registers held; waited for when the point starts) -- as K1g, diag_tmg.cuh
  auto prefetch_x = [&](int64_t r, int sb) {
    const int64_t off = r * (int64_t)n;
    if constexpr (!UNAL) {
      if (gl == 0) dtg::bulk_load(dtg::smem_u32(xrow(sb)), p.X + off, (uint32_t)n * 4u, dtg::smem_u32(bars + sb));
    } else {
      const int64_t a0 = off & ~(int64_t)3, a1 = (off + n) & ~(int64_t)3;
      if (gl == 0)
        dtg::bulk_load(dtg::smem_u32(xrow(sb)), p.X + a0, (uint32_t)(a1 - a0) * 4u, dtg::smem_u32(bars + sb));
      const int tl = (int)((off + n) & 3);
      if (gl < tl)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;"
                     :: "r"(dtg::smem_u32(xrow(sb) + (off & 3) + n - tl + gl)), "l"(p.X + (off + n - tl) + gl) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  if (have) prefetch_x(pt, 0);
  if (have && p1 < M) prefetch_x(p1, 1);
  // (pt n) mod 4: offset of the current point's rows in their buffers (0 unless UNAL)
  auto xo = [&]() { return UNAL ? (int)((pt * (int64_t)n) & 3) : 0; };

  // ---- set k of the current point for the groups with `fresh` (collective): x_hat = (x - c_k) /
  // (D_k + lambda), v^0 = d^0 = x - c_k, b^0 = 0 (R5), -kappa_k = -lambda / (D_k + lambda)
  auto set_setup = [&](bool fresh) {
    const float *xr = xrow(xs) + xo() + gl;
    const float2 *dc = DC_s + kset * (G * CPL) + gl;
    // lanes that keep their set write back what they read; in the lockstep case (every lane
    // starts a set or has no point left) nothing is read
    const bool keep_any = __any_sync(0xffffffffu, have && !fresh);
    for_chunks<CPL>([&](auto ci, auto szc) {
      constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
      float ch[4][8];
#pragma unroll
      for (int e = 0; e < 8; e++) ch[0][e] = ch[1][e] = ch[2][e] = ch[3][e] = 0.f;
      if (keep_any) {
        ldn<SZ, C_XH + 8 * c>(tl0, ch[0]);
        ldn<SZ, C_V + 8 * c>(tl0, ch[1]);
        ldn<SZ, C_K + 8 * c>(tl0, ch[2]);
        ldn<SZ, C_U + 8 * c>(tl0, ch[3]);
        wait_ld(ch);
      }
      if (fresh) {
#pragma unroll
        for (int e = 0; e < SZ; e++) {
          const int j = 8 * c + e;
          const float2 Dc = dc[G * j];
          const float xt = (j < jmax) ? xr[G * j] - Dc.y : 0.f;
          const float di = __fdividef(1.f, Dc.x + lam);
          ch[0][e] = xt * di;
          ch[1][e] = xt;
          ch[2][e] = -__fdividef(lam, Dc.x + lam);
          ch[3][e] = xt;                          // u with s_prev = 1: -d^0 = -(x - c_k)
          float2 &dq = d[4 * c + (e >> 1)];
          float2 &bq = b[4 * c + (e >> 1)];
          if (e & 1) { dq.y = -xt; bq.y = xt; } else { dq.x = -xt; bq.x = xt; }
        }
      }
      stn<SZ, C_XH + 8 * c>(tl0, ch[0]);
      stn<SZ, C_V + 8 * c>(tl0, ch[1]);
      stn<SZ, C_K + 8 * c>(tl0, ch[2]);
      stn<SZ, C_U + 8 * c>(tl0, ch[3]);
    });
    asm volatile("tcgen05.wait::st.sync.aligned;");
    if (fresh) {
      s_prev = 1.f;
      lim = spec ? 0 : p.max_iter;
      it = 0;
      s_cur = 1.f;
      sv_ok = false;
      waiting = false;
    }
  };

  // ---- start the point pt (x already requested into row xs): t, validity, running minimum ----
  auto point_start = [&](bool fresh) {
    bool bad = false;
    if (fresh) {
      tt = DIST ? 0.f : tpre;   // distance mode starts at s_0 = 0 (R24)
      bad = !(tt >= 0.f) || !finite_f(tt);
      tpre = (p1 < M && !DIST) ? __ldg(p.t + p1) : 0.f;
      if (gl == 0 && p.claim) gclaim = atomicAdd(p.claim, 1ull);
      nn = 0;
      dtg::mbar_wait(dtg::smem_u32(bars + xs), (xph >> xs) & 1u);
      xph ^= 1u << xs;
      // the row's tail: this lane's cp.async of it (at most the two rows' groups are pending;
      // waiting for all of them is exact: the other row's tail is in flight at most one point)
      if constexpr (UNAL) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp(gmask);
      }
      float fin = 0.f;   // x * 0 accumulates NaN iff some x is NaN or infinite
      const float *xr = xrow(xs) + xo() + gl;
#pragma unroll
      for (int j = 0; j < CPL; j++)
        if (j < jmax) fin = fmaf(xr[G * j], 0.f, fin);
      bad |= !(fin == 0.f);
      if (gl == 0) dtg::bulk_wait_read();   // this group's previous grad / y rows have left
    }
    __syncwarp();
    bad = group_any<G>(bad);
    if (fresh) {
      spec = bad ? 2 : (tt == 0.f ? 1 : 0);
      tauS = tt / lam;
      kset = 0;
      best = __int_as_float(0x7f800000);
      bestk = -1;
      bestit = 0;
      bgn = 0.f;
    }
  };
  point_start(have);
  set_setup(have);

  // -d = -s_prev u from the parked u_k (collective; every group, see dfull)
  auto fix_d = [&]() {
    const float2 ns = splat2(-s_prev);
    for_chunks<CPL>([&](auto ci, auto szc) {
      constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
      float uk[1][8];
      ldn<SZ, C_U + 8 * c>(tl0, uk[0]);
      wait_ld(uk);
#pragma unroll
      for (int e2 = 0; e2 < SZ / 2; e2++)
        d[4 * c + e2] = __fmul2_rn(ns, make_float2(uk[0][2 * e2], uk[0][2 * e2 + 1]));
    });
    dfull = true;
  };
  // a stopped set parks its d^k (grad := d, R1) in the candidate row; collective
  auto park = [&](bool stop) {
    if (stop) {
      float *gr = grow_s(cand) + xo() + gl;
#pragma unroll
      for (int q = 0; q < NP; q++) {
        gr[G * (2 * q)] = -d[q].x;
        gr[G * (2 * q + 1)] = -d[q].y;
      }
    }
  };

  unsigned my_iters = 0;
  bool any_have = __any_sync(0xffffffffu, have);
  while (any_have) {
    const bool live = have && !waiting;
    float2 a0 = splat2(0.f), b0 = a0, c0 = a0, r0 = a0;
    const float2 sP = splat2(s_cur);
    const float2 omsP = splat2(1.f - s_cur), na_sP = splat2(1.f - 2.f * s_cur);
    const bool full_test = __any_sync(0xffffffffu, live && sv_ok);
    auto trip = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      for_chunks<CPL>([&](auto ci, auto szc) {
        constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
        float ch[3][8];   // -kappa, x_hat, v
        ldn<SZ, C_K + 8 * c>(tl0, ch[0]);
        ldn<SZ, C_XH + 8 * c>(tl0, ch[1]);
        ldn<SZ, C_V + 8 * c>(tl0, ch[2]);
        if constexpr (!FULL) {   // u_k of the chunk -> C_U (-d_k is formed only if needed)
          float uk[8];
#pragma unroll
          for (int e2 = 0; e2 < 4; e2++) {
            uk[2 * e2] = e2 < SZ / 2 ? b[4 * c + e2].x : 0.f;
            uk[2 * e2 + 1] = e2 < SZ / 2 ? b[4 * c + e2].y : 0.f;
          }
          stn<SZ, C_U + 8 * c>(tl0, uk);
        }
        wait_ld(ch);
#pragma unroll
        for (int e2 = 0; e2 < SZ / 2; e2++) {
          const int q = 4 * c + e2;
          const float2 kq = make_float2(ch[0][2 * e2], ch[0][2 * e2 + 1]);
          const float2 xh = make_float2(ch[1][2 * e2], ch[1][2 * e2 + 1]);
          const float2 v = make_float2(ch[2][2 * e2], ch[2][2 * e2 + 1]);
          // d[q] = -d_{k-1}, b[q] = u_k; d_k = s_k u_k, b_k = (1 - s_k) u_k, d_k - b_k = (2 s_k - 1) u_k
          const float2 u = b[q];
          if (FULL) {
            const float2 dd = fma2(sP, u, d[q]);                  // d_k - d_{k-1}
            d[q] = sub2(d[q], dd);                                // -d_k
            const float2 dmv = add2(d[q], v);                     // v^k - d^k
            a0 = fma2(dd, dd, a0); b0 = fma2(dmv, dmv, b0);
          }
          const float2 na = __fmul2_rn(na_sP, u);                 // -(d_k - b_k)
          const float2 vn = fma2(kq, na, xh);                     // (3.4a): v_{k+1}
          const float2 dv = sub2(vn, v);
          b[q] = fma2(omsP, u, vn);                               // u_{k+1} = v_{k+1} + b_k, b_k = (1 - s_k) u_k
          c0 = fma2(dv, dv, c0);
          r0 = fma2(b[q], b[q], r0);
          ch[2][2 * e2] = vn.x;
          ch[2][2 * e2 + 1] = vn.y;
        }
        stn<SZ, C_V + 8 * c>(tl0, ch[2]);
      });
    };
    if (full_test) {
      if (!dfull) fix_d();
      trip(std::true_type{});
    } else {
      trip(std::false_type{});
      dfull = false;
      s_prev = s_cur;
    }
    {
      // group totals by a plain xor butterfly (every lane ends with every total: no broadcast, the
      // dependent chain is log2(G) shuffles deep); the stores of v drain meanwhile
      float sd = 0.f, sb = 0.f, sv, r2;
      if (full_test) {
        float4 t4 = make_float4(a0.x + a0.y, b0.x + b0.y, c0.x + c0.y, r0.x + r0.y);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          t4.x += __shfl_xor_sync(0xffffffffu, t4.x, o);
          t4.y += __shfl_xor_sync(0xffffffffu, t4.y, o);
          t4.z += __shfl_xor_sync(0xffffffffu, t4.z, o);
          t4.w += __shfl_xor_sync(0xffffffffu, t4.w, o);
        }
        sd = t4.x; sb = t4.y; sv = t4.z; r2 = t4.w;
      } else {
        float2 t2 = make_float2(c0.x + c0.y, r0.x + r0.y);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          t2.x += __shfl_xor_sync(0xffffffffu, t2.x, o);
          t2.y += __shfl_xor_sync(0xffffffffu, t2.y, o);
        }
        sv = t2.x; r2 = t2.y;
      }
      const int kdone = it;
      // P:1597-1601 for iteration k = it (sd, sb are only formed in FULL trips, where sv_ok may hold)
      const bool conv = full_test && sv_ok && sd <= tol && sb <= tol;
      sv_ok = sv <= tol;
      s_cur = (r2 > tauS * tauS) ? fmaf(-tauS, rsqrtf(r2), 1.f) : 0.f;   // P:283-285, R20
      it += live ? 1 : 0;
      // t == 0 / invalid points have lim = 0 and stop at their first trip
      const bool stop = live && ((kdone >= 1 && conv) || kdone >= lim);
      asm volatile("tcgen05.wait::st.sync.aligned;");
      if (!__any_sync(0xffffffffu, stop)) continue;
      if (stop) {
        waiting = true;
        wstatus = spec == 2 ? INT32_MIN : (spec == 1 ? 0 : (conv ? kdone : -lim));
        if (spec == 0) my_iters += (unsigned)kdone;
      }
      if (!dfull) fix_d();   // a set that stops at its limit after a non-final trip
      park(stop);
    }
    {
      const unsigned gbit = (gl == 0) ? 1u : 0u;
      const int nwait = __popc(__ballot_sync(0xffffffffu, waiting && gbit));
      const int nhave = __popc(__ballot_sync(0xffffffffu, have && gbit));
      if (nwait < WAIT_THRESHOLD && nwait < nhave) continue;
    }

    // ================= event: the parked sets of the waiting groups ===========================
    const bool done = waiting;
    const float gnan = __int_as_float(0x7fc00000);
    const int xoff = xo();
    const float *xr = xrow(xs) + xoff + gl;
    const float2 *dc = DC_s + kset * (G * CPL) + gl;
    float *const cr = grow_s(cand) + xoff + gl;
    // t == 0 (R6): the set's grad is grad J_k(x) = D_k^{-1}(x - c_k)
    if (done && spec == 1) {
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const float2 Dc = dc[G * j];
        cr[G * j] = (j < jmax) ? __fdividef(xr[G * j] - Dc.y, Dc.x) : 0.f;
      }
    }
    // phi_k = <x - c_k, g> - 1/2 <g, D_k g> - t ||g|| + gamma_k ((3.3) at d, R2)
    float qs0 = 0.f, qs1 = 0.f, hs0 = 0.f, hs1 = 0.f;
#pragma unroll
    for (int j = 0; j < CPL; j++) {
      const float2 Dc = dc[G * j];
      const float g = cr[G * j];
      const float xt = (j < jmax) ? xr[G * j] - Dc.y : 0.f;
      float &qs = (j & 1) ? qs1 : qs0;
      float &hs = (j & 1) ? hs1 : hs0;
      qs = fmaf(xt, g, qs);
      qs = fmaf(-0.5f * Dc.x * g, g, qs);
      hs = fmaf(g, g, hs);
    }
    const float qs = group_sum<G>(qs0 + qs1), hs = group_sum<G>(hs0 + hs1);
    const float gnorm = sqrtf(hs);
    float phik = (spec == 1) ? qs + gk_s[kset] : qs - tt * gnorm + gk_s[kset];
    bool point_done = false;
    if (done) {
      if (spec == 2) phik = gnan;
      if (p.phik && gl == 0) p.phik[pt * K + kset] = phik;
      if (phik < best) {   // strict: the lowest k wins ties (R19); NaN never wins
        best = phik; bestk = kset; bestit = wstatus; bgn = gnorm;
        cand ^= 1;         // the parked row becomes the best row
      }
      point_done = spec == 2 || kset + 1 >= K;
    }
    bool restart = false;   // distance mode: the K sets again at the next Newton iterate
    if (DIST && point_done && spec != 2 && bestk >= 0) {
      // psi(y,s) = best, ||grad psi|| = bgn; Newton in s with d psi/dt = -||grad psi|| (eq.
      // Newton_zero), the same step / stop / safeguard order as the oracle (R24-R26)
      const float s0 = tt;
      bool fin = false;
      if (nn == 0 && s0 == 0.f) {
        if (!(best > 0.f)) fin = true;                  // y in Omega: dist 0, proj y
        else { s_lo = 0.f; s_hi = __int_as_float(0x7f800000); }
      } else if (best > 0.f) {
        s_lo = s0;
      } else {
        s_hi = s0;
      }
      if (!fin && (nn >= p.max_newton || !(bgn > 0.f))) fin = true;
      if (!fin) {
        float sn = s0 + best / bgn;
        if (fabsf(sn - s0) <= p.stol * fmaxf(1.f, s0)) {
          fin = true;                                   // R26: keep the evaluated s
        } else {
          if (!(sn > s_lo && sn < s_hi)) sn = 0.5f * (s_lo + s_hi);   // R25
          point_done = false;
          restart = true;
          nn++;
          tt = sn;
          tauS = sn / lam;
          spec = 0;
        }
      }
    }
    // ---- the point's outputs (groups whose last set finished) ---------------------------------
    if (__any_sync(0xffffffffu, point_done)) {
      const int xoff = xo();
      float *const br = grow_s(cand ^ 1) + xoff + gl;   // best grad row
      float *const yr = xrow(xs) + xoff + gl;           // y formed in place in the x row
      const bool nanpt = spec == 2 || bestk < 0;
      if (point_done) {
        const float ign = bgn > 0.f ? __fdividef(1.f, bgn) : 0.f;
        const float2 *dck = DC_s + (bestk < 0 ? 0 : bestk) * (G * CPL) + gl;
#pragma unroll
        for (int j = 0; j < CPL; j++) {
          const float g = br[G * j];
          // y = x - t grad / ||grad||, c_k* if grad = 0 (R18); distance mode:
          // pi = y - s grad / ||grad|| at the evaluated s, y itself inside
          const float y = DIST ? ((tt > 0.f && bgn > 0.f) ? yr[G * j] - tt * (g * ign) : yr[G * j])
                               : (bgn > 0.f ? yr[G * j] - tt * (g * ign) : dck[G * j].y);
          br[G * j] = nanpt ? gnan : g;
          yr[G * j] = nanpt ? gnan : y;
        }
        if (nanpt && p.phik)   // an invalid point's phi_k are NaN for every k
          for (int k = gl; k < K; k += G) p.phik[pt * K + k] = gnan;
        if (gl == 0) {
          p.phi[pt] = nanpt ? gnan : best;
          p.iters[pt] = nanpt ? INT32_MIN : (DIST ? nn : bestit);
          if (p.kstar) p.kstar[pt] = nanpt ? -1 : bestk;
          if (DIST) p.dist[pt] = nanpt ? gnan : tt;
        }
      }
      if constexpr (!UNAL) {
        dtg::fence_proxy_async();
        __syncwarp();
        if (point_done && gl == 0) {
          const int64_t off = pt * (int64_t)n;
          dtg::bulk_store(p.grad + off, dtg::smem_u32(br - gl), (uint32_t)n * 4u);
          if (p.Y) dtg::bulk_store(p.Y + off, dtg::smem_u32(yr - gl), (uint32_t)n * 4u);
          // the x row is free once y has left it: the point after the next one goes there
          if (p2 < M) {
            dtg::bulk_wait_read();
            prefetch_x(p2, xs);
          }
        }
      } else {
        // rows leave as a bulk store of their 16-byte aligned interior [h, e) plus up to 3 plain
        // stores at each end (element i of the rows at br - gl + i, yr - gl + i)
        const int64_t off = pt * (int64_t)n;
        const int h = (4 - xoff) & 3, e = (int)(((off + n) & ~(int64_t)3) - off);
        dtg::fence_proxy_async();
        __syncwarp();
        if (point_done) {   // (the tail elements were written by other lanes: after the sync)
          if (gl < h) {
            p.grad[off + gl] = br[0];
            if (p.Y) p.Y[off + gl] = yr[0];
          }
          if (gl < n - e) {
            p.grad[off + e + gl] = br[e];
            if (p.Y) p.Y[off + e + gl] = yr[e];
          }
        }
        if (point_done && gl == 0) {
          dtg::bulk_store(p.grad + off + h, dtg::smem_u32(br - gl + h), (uint32_t)(e - h) * 4u);
          if (p.Y) dtg::bulk_store(p.Y + off + h, dtg::smem_u32(yr - gl + h), (uint32_t)(e - h) * 4u);
        }
        // the x row is free once y has left it: the point after the next one goes there
        if (point_done && p2 < M) {
          if (gl == 0) dtg::bulk_wait_read();
          __syncwarp(gmask);
          prefetch_x(p2, xs);
        }
      }
    }
    // ---- next set, or next point --------------------------------------------------------------
    const bool next_set = done && !point_done && !restart;
    if (next_set) kset++;
    if (restart) {
      kset = 0;
      best = __int_as_float(0x7f800000);
      bestk = -1;
      bestit = 0;
      bgn = 0.f;
    }
    const int64_t claimed = p.claim ? (int64_t)__shfl_sync(0xffffffffu, gclaim, lane & ~(G - 1)) + 3 * ngroups
                                    : p2 + ngroups;   // no counter: static stride
    if (point_done) {
      pt = p1;
      p1 = p2;
      p2 = claimed;
      have = pt < M;
      xs ^= 1;
      if (!have) {
        waiting = false;
        spec = 0;
#pragma unroll
        for (int q = 0; q < NP; q++) d[q] = b[q] = splat2(0.f);
      }
    }
    const bool started = point_done && have;
    if (__any_sync(0xffffffffu, started)) point_start(started);
    if (__any_sync(0xffffffffu, next_set || started || restart)) set_setup(next_set || started || restart);
    any_have = __any_sync(0xffffffffu, have);
  }
  if (gl == 0) dtg::bulk_wait_all();
  if (p.iter_total && gl == 0 && my_iters) atomicAdd(p.iter_total, (unsigned long long)my_iters);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_slot), "r"(TMEM_COLS));
}

}  // namespace dtu
}  // namespace hopf
