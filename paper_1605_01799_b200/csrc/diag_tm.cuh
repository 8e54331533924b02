// diag_tm.cuh — K1/K2 for wide points (n in (512, 1024], one warp per point) with tensor memory
// as an extension of the register file.  sm_100a, FP32 SIMT; no MMA is involved.
//
// Same method and arithmetic as hopf_diag_kernel<32, 32, HK, false> (diag_kernel.cuh): split
// Bregman (3.4a)-(3.4c) with the paper's stopping rule, shrink_1
// / shrink_2, phi = (3.3) at d (reading R2).  Only the storage differs:
//
//   registers : d, b (u between l2 trips) — 2 x 32 floats per lane
//   TMEM      : x_hat (columns 0-31), v (32-63), -kappa / kappa (64-95), tau_i (96-127, wl1)
//
// Because v is reloaded every trip, (3.4a) is formed directly as v^{k+1} = x_hat - kappa (d - b)
// (one FFMA; the register kernel updates v in place: v + ((x_hat - v) - kappa (d - b))), so an
// l2 trip far from convergence costs 9 packed FP32 ops per coordinate pair.
//
// The register kernel keeps x_hat, d, b, v resident (128 of its 168 registers), which limits it
// to 3 warps per SM sub-partition; with two vectors moved to TMEM this one runs at <= 128
// registers, i.e. 4 warps per sub-partition (4 CTAs of 128 threads per SM, 128 TMEM columns
// each = the SM's 512).  Warp w of a CTA owns TMEM lanes 32 (w % 4) + lane, so each thread's
// 32 slot values of a vector are one 32x32b row of 32 columns, moved in x8 chunks per trip.
#pragma once
#include <cfloat>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "diag_kernel.cuh"

namespace hopf {
namespace dtm {

constexpr int CPL = 32, NP = 16, THREADS = 128, TMEM_COLS = 128;
constexpr int DYN_SMEM = 48 * 1024;   // caps residency at 4 CTAs per SM (4 x 128 TMEM columns)

__device__ __forceinline__ void ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])),
                  "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])),
                  "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])));
}
// The same with a compile-time column offset folded into the instruction (tmem[UR + imm]): the
// base stays in one uniform register across the loop instead of one R2UR per address per trip
template <int OFF>
__device__ __forceinline__ void ld8o(uint32_t base, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8+%9];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(base), "n"(OFF));
#pragma unroll
  for (int i = 0; i < 8; i++) v[i] = __uint_as_float(r[i]);
}
template <int OFF>
__device__ __forceinline__ void st8o(uint32_t base, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0+%9], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(base), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])),
                  "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])),
                  "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
                  "n"(OFF));
}
template <typename F>
__device__ __forceinline__ void static_for4(F &&f) {
  f(std::integral_constant<int, 0>{});
  f(std::integral_constant<int, 1>{});
  f(std::integral_constant<int, 2>{});
  f(std::integral_constant<int, 3>{});
}

// wait for this thread's outstanding tcgen05.ld, naming the destination registers so the
// compiler does not read them before the wait
template <int N>
__device__ __forceinline__ void wait_ld(float (&a)[N][8]) {
  static_assert(N >= 1 && N <= 4, "1..4 chunks");
  if constexpr (N == 1)
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(a[0][0]), "+f"(a[0][1]), "+f"(a[0][2]), "+f"(a[0][3]), "+f"(a[0][4]), "+f"(a[0][5]), "+f"(a[0][6]), "+f"(a[0][7])
                 :: "memory");
  else if constexpr (N == 2)
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(a[0][0]), "+f"(a[0][1]), "+f"(a[0][2]), "+f"(a[0][3]), "+f"(a[0][4]), "+f"(a[0][5]), "+f"(a[0][6]), "+f"(a[0][7]),
                   "+f"(a[1][0]), "+f"(a[1][1]), "+f"(a[1][2]), "+f"(a[1][3]), "+f"(a[1][4]), "+f"(a[1][5]), "+f"(a[1][6]), "+f"(a[1][7])
                 :: "memory");
  else if constexpr (N == 3)
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(a[0][0]), "+f"(a[0][1]), "+f"(a[0][2]), "+f"(a[0][3]), "+f"(a[0][4]), "+f"(a[0][5]), "+f"(a[0][6]), "+f"(a[0][7]),
                   "+f"(a[1][0]), "+f"(a[1][1]), "+f"(a[1][2]), "+f"(a[1][3]), "+f"(a[1][4]), "+f"(a[1][5]), "+f"(a[1][6]), "+f"(a[1][7]),
                   "+f"(a[2][0]), "+f"(a[2][1]), "+f"(a[2][2]), "+f"(a[2][3]), "+f"(a[2][4]), "+f"(a[2][5]), "+f"(a[2][6]), "+f"(a[2][7])
                 :: "memory");
  else
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+f"(a[0][0]), "+f"(a[0][1]), "+f"(a[0][2]), "+f"(a[0][3]), "+f"(a[0][4]), "+f"(a[0][5]), "+f"(a[0][6]), "+f"(a[0][7]),
                   "+f"(a[1][0]), "+f"(a[1][1]), "+f"(a[1][2]), "+f"(a[1][3]), "+f"(a[1][4]), "+f"(a[1][5]), "+f"(a[1][6]), "+f"(a[1][7]),
                   "+f"(a[2][0]), "+f"(a[2][1]), "+f"(a[2][2]), "+f"(a[2][3]), "+f"(a[2][4]), "+f"(a[2][5]), "+f"(a[2][6]), "+f"(a[2][7]),
                   "+f"(a[3][0]), "+f"(a[3][1]), "+f"(a[3][2]), "+f"(a[3][3]), "+f"(a[3][4]), "+f"(a[3][5]), "+f"(a[3][6]), "+f"(a[3][7])
                 :: "memory");
}

template <int HK>
__global__ void __launch_bounds__(THREADS, 4) hopf_diag_tm_kernel(const DiagParams p) {
  // dynamic shared memory (48 KB, which also caps residency at 4 CTAs per SM): D at [0, 4 KB),
  // w at [4, 8 KB) (wl1): per-coordinate parameters loaded once per CTA
  extern __shared__ __align__(16) uint8_t dyn_smem[];
  __shared__ uint32_t tmem_slot;
  constexpr int G = 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gl = lane;
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int n = p.n;
  const float lam = p.lambda, tol = p.tol;
  // slot j of lane gl is coordinate 128 (j / 4) + 4 gl + j % 4: four contiguous coordinates per
  // lane and block of 128, so x rows load and grad rows store as float4 (vrow) when rows are
  // 16-byte aligned; the valid slots are a prefix j < jmax of every lane's 32
  const int jmax = 4 * (n >> 7) + min(4, max(0, (n & 127) - 4 * gl));
  auto cidx = [&](int j) { return 128 * (j >> 2) + 4 * gl + (j & 3); };
  const bool vrow = (n & 3) == 0 && ((reinterpret_cast<uintptr_t>(p.X) | reinterpret_cast<uintptr_t>(p.grad) |
                                      reinterpret_cast<uintptr_t>(p.c)) & 15) == 0;
  float *const D_s = reinterpret_cast<float *>(dyn_smem);
  float *const w_s = reinterpret_cast<float *>(dyn_smem + 4096);
  float *const di_s = reinterpret_cast<float *>(dyn_smem + 8192);   // 1 / (D_i + lambda)
  for (int i = threadIdx.x; i < 1024; i += THREADS) {
    const float Dv = i < n ? __ldg(p.D + i) : 1.f;
    D_s[i] = Dv;
    di_s[i] = 1.f / (Dv + lam);
    if (HK == HK_WL1) w_s[i] = i < n ? __ldg(p.w + i) : 0.f;
  }
  __syncthreads();

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&tmem_slot)), "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp-uniform TMEM base; read back through a lane-0 shuffle so that the compiler can prove it
  // uniform and keep it in one uniform register (otherwise it re-issues an R2UR before every
  // tcgen05.ld / st: 16 per trip)
  const uint32_t tl0 = __shfl_sync(0xffffffffu, tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16), 0);
  const uint32_t T_XH = tl0, T_V = tl0 + 32, T_K = tl0 + 64, T_TAU = tl0 + 96;   // (the trip
  // uses the same layout as immediate offsets from tl0)

  // kappa (l2: -kappa) of this lane's slots -> TMEM, once
  const float ksign = (HK == HK_L2) ? -1.f : 1.f;
#pragma unroll
  for (int c = 0; c < 4; c++) {
    float kv[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int j = 8 * c + e, i = cidx(j);
      kv[e] = (j < jmax) ? ksign * __fdividef(lam, D_s[i] + lam) : 0.f;
    }
    st8(T_K + 8 * c, kv);
  }

  float2 d[NP], b[NP];
  // points: the first two of a warp static (gid, gid + ngroups), later ones claimed from p.claim
  // one point ahead, so warps that drew cheap points take more and the launch ends within
  // about one point
  int64_t pt = gid, pnext = gid + ngroups;
  unsigned long long wclaim = 0;   // lane 0: the claim made at the last point start
  bool have = pt < p.M;
  int it = 0;
  float tt = 0.f, tauS = 0.f;
  int spec = 0;
  int lim = 0;   // the solve stops at iteration lim at the latest: 0 for t == 0 / invalid input
  float s_cur = 1.f;
  bool sv_ok = false;
  bool dfull = true;    // l2: d holds -d_k (else u_k is parked in T_U and s_prev = s_k)
  float s_prev = 1.f;

  // load the point and set up the solve: x_hat, v -> TMEM; d, b -> registers (reading R5).
  // All global loads are issued first (x into d, D into b: both are dead at this point), so
  // their latency overlaps instead of being paid per TMEM chunk.
  auto start_point = [&](bool active) {
    bool bad = false;
    if (active) {
      tt = p.tscale * __ldg(p.t + pt);
      bad = !(tt >= 0.f) || !finite_f(tt);
      if (lane == 0 && p.claim) wclaim = atomicAdd(p.claim, 1ull);
    }
    const float *xrow = p.X + (active ? pt : 0) * (int64_t)n;
    if (vrow) {   // rows on the 16-byte grid: one float4 per block of 128 (n % 4 == 0: all or none)
#pragma unroll
      for (int m = 0; m < 8; m++) {
        const bool ok = active && 4 * m < jmax;
        const float4 x4 = ok ? __ldg(reinterpret_cast<const float4 *>(xrow + 128 * m + 4 * gl))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
        d[2 * m] = make_float2(x4.x, x4.y);
        d[2 * m + 1] = make_float2(x4.z, x4.w);
      }
    } else {
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const int j0 = 2 * q, j1 = 2 * q + 1;
        const bool ok0 = active && j0 < jmax, ok1 = active && j1 < jmax;
        d[q] = make_float2(ok0 ? __ldg(xrow + cidx(j0)) : 0.f, ok1 ? __ldg(xrow + cidx(j1)) : 0.f);
      }
    }
#pragma unroll
    for (int q = 0; q < NP; q++)   // padded slots: x = 0 anyway
      b[q] = *reinterpret_cast<const float2 *>(di_s + cidx(2 * q));
    if (p.c) {
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const int j0 = 2 * q, j1 = 2 * q + 1;
        const bool ok0 = active && j0 < jmax, ok1 = active && j1 < jmax;
        d[q].x -= ok0 ? __ldg(p.c + cidx(j0)) : 0.f;
        d[q].y -= ok1 ? __ldg(p.c + cidx(j1)) : 0.f;
      }
    }
    const float tl = tt / lam;
    float2 fin = splat2(0.f);   // x * 0 accumulates NaN iff some x is NaN or infinite
#pragma unroll
    for (int q = 0; q < NP; q++) fin = fma2(d[q], splat2(0.f), fin);
    bad |= !(fin.x == 0.f && fin.y == 0.f);
#pragma unroll
    for (int c = 0; c < 4; c++) {
      float xh8[8], v8[8], tau8[8];
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const int j = 8 * c + e;
        const float2 xq = d[4 * c + (e >> 1)], Dq = b[4 * c + (e >> 1)];
        const float xt = (e & 1) ? xq.y : xq.x;        // x - c (0 on padded slots)
        const float di = (e & 1) ? Dq.y : Dq.x;
        xh8[e] = xt * di;
        v8[e] = xt;                                     // v^0 = x - c
        if (HK == HK_WL1) tau8[e] = (active && j < jmax) ? tl * w_s[cidx(j)] : 0.f;
      }
      st8(T_XH + 8 * c, xh8);
      st8(T_V + 8 * c, v8);
      if (HK == HK_WL1) st8(T_TAU + 8 * c, tau8);
    }
#pragma unroll
    for (int q = 0; q < NP; q++) {
      const float2 xt = d[q];
      if (HK == HK_L2) { d[q] = make_float2(-xt.x, -xt.y); b[q] = xt; }   // -d^0, pending u
      else { b[q] = splat2(0.f); }                                        // d^0 = x - c, b^0 = 0
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    bad = __any_sync(0xffffffffu, bad);
    if (active) {
      spec = bad ? 2 : (tt == 0.f ? 1 : 0);
      lim = spec ? 0 : max(p.max_iter, 1);
      tauS = tt / lam;
    }
    it = 0;
    s_cur = 1.f;
    sv_ok = false;
    dfull = true;
  };
  start_point(have);

  unsigned my_iters = 0;   // this warp's share of p.iter_total (lane 0 counts)
  while (have) {   // one point per warp: `have` is warp-uniform
    float2 a0 = splat2(0.f), b0 = a0, c0 = a0, r0 = a0;   // one packed accumulator per sum
    const float2 sP = splat2(s_cur), tP = splat2(tauS);
    const float2 omsP = splat2(1.f - s_cur), na_sP = splat2(1.f - 2.f * s_cur);
    // (warp votes make the per-trip predicates provably uniform: plain branches, no reconvergence)
    const bool full_test = (HK != HK_L2) || __any_sync(0xffffffffu, sv_ok);   // see hopf_diag_kernel: exact
    // l2: -d_k = -s_k u_k from the u_k a non-final trip parked in T_U (when a final trip or the
    // finalize needs it; a non-final trip does not form d: 7 -> 6 packed ops per pair)
    auto fix_d = [&]() {
      const float2 ns = splat2(-s_prev);
      static_for4([&](auto ci) {
        constexpr int c = decltype(ci)::value;
        float uk[1][8];
        ld8o<96 + 8 * c>(tl0, uk[0]);
        wait_ld(uk);
#pragma unroll
        for (int e2 = 0; e2 < 4; e2++)
          d[4 * c + e2] = __fmul2_rn(ns, make_float2(uk[0][2 * e2], uk[0][2 * e2 + 1]));
      });
    };
    auto trip = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      static_for4([&](auto ci) {
        constexpr int c = decltype(ci)::value;
        float ch[(HK == HK_WL1) ? 4 : 3][8];   // kappa, x_hat, v (, tau)
        ld8o<64 + 8 * c>(tl0, ch[0]);          // T_K
        ld8o<0 + 8 * c>(tl0, ch[1]);           // T_XH
        ld8o<32 + 8 * c>(tl0, ch[2]);          // T_V
        if constexpr (HK == HK_WL1) ld8o<96 + 8 * c>(tl0, ch[3]);   // T_TAU
        if constexpr (HK == HK_L2 && !FULL) {   // u_k of the chunk -> T_U (l2 leaves 96-127 free)
          const float uk[8] = {b[4 * c].x, b[4 * c].y, b[4 * c + 1].x, b[4 * c + 1].y,
                               b[4 * c + 2].x, b[4 * c + 2].y, b[4 * c + 3].x, b[4 * c + 3].y};
          st8o<96 + 8 * c>(tl0, uk);
        }
        wait_ld(ch);
#pragma unroll
        for (int e2 = 0; e2 < 4; e2++) {
          const int q = 4 * c + e2;
          const float2 kq = make_float2(ch[0][2 * e2], ch[0][2 * e2 + 1]);
          const float2 xh = make_float2(ch[1][2 * e2], ch[1][2 * e2 + 1]);
          float2 v = make_float2(ch[2][2 * e2], ch[2][2 * e2 + 1]);
          if (HK == HK_L2) {
            // d[q] = -d_{k-1}, kq = -kappa, b[q] = u_k
            // d_k = s_k u_k, b_k = u_k - d_k = (1 - s_k) u_k, d_k - b_k = (2 s_k - 1) u_k:
            // three independent scalings of u_k = b[q] ((3.4b), (3.4c))
            const float2 u = b[q];
            if (FULL) {
              const float2 dd = fma2(sP, u, d[q]);                  // d_k - d_{k-1}
              d[q] = sub2(d[q], dd);                                // -d_k
              const float2 dmv = add2(d[q], v);                     // v^k - d^k
              a0 = fma2(dd, dd, a0); b0 = fma2(dmv, dmv, b0);
            }   // non-final trip: u_k went to TMEM (T_U) at the chunk start instead of forming -d_k
            const float2 na = __fmul2_rn(na_sP, u);                 // -(d_k - b_k)
            const float2 vn = fma2(kq, na, xh);                     // (3.4a): v_{k+1}
            const float2 dv = sub2(vn, v);                          // v_{k+1} - v_k
            v = vn;
            b[q] = fma2(omsP, u, v);                                // u_{k+1} = v_{k+1} + b_k, b_k = (1 - s_k) u_k
            c0 = fma2(dv, dv, c0);          // one packed accumulator per sum: the loop has ample
            r0 = fma2(b[q], b[q], r0);      // independent work, and the serial tail is shorter
          } else {
            const float2 a = sub2(d[q], b[q]);
            const float2 vn = fma2(kq, a, xh);                      // (3.4a): v^k
            const float2 dv = sub2(vn, v);                          // v^k - v^{k-1}
            v = vn;
            const float2 u = add2(v, b[q]);
            const float2 tq = (HK == HK_WL1) ? make_float2(ch[HK == HK_WL1 ? 3 : 0][2 * e2], ch[HK == HK_WL1 ? 3 : 0][2 * e2 + 1]) : tP;
            b[q] = clamp2(u, tq);                                   // projection (Moreau)
            const float2 dn = sub2(u, b[q]);                        // (3.4b) shrink_1
            const float2 dd = sub2(dn, d[q]);
            d[q] = add2(d[q], dd);                                  // d^k (as the register kernel)
            const float2 dmv = sub2(d[q], v);                       // d^k - v^k
            a0 = fma2(dd, dd, a0); b0 = fma2(dmv, dmv, b0); c0 = fma2(dv, dv, c0);
          }
          ch[2][2 * e2] = v.x;
          ch[2][2 * e2 + 1] = v.y;
        }
        st8o<32 + 8 * c>(tl0, ch[2]);          // T_V
      });
    };
    if (HK == HK_L2 && full_test && !dfull) fix_d();
    if (full_test) trip(std::true_type{});
    else trip(std::false_type{});
    if (HK == HK_L2) {
      dfull = full_test;
      if (!full_test) s_prev = s_cur;
    }

    bool conv;
    int kdone;
    if (HK == HK_L2 && !full_test) {
      // non-final l2 trip: only ||v^{k+1} - v^k||^2 and ||u_{k+1}||^2 are needed; transposed
      // 2-value butterfly: lanes 0-15 end with the first total, lanes 16-31 with the second
      const float psv = c0.x + c0.y, pr2 = r0.x + r0.y;
      const bool hi = lane & 16;
      float c = (hi ? pr2 : psv) + __shfl_xor_sync(0xffffffffu, hi ? psv : pr2, 16);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      const bool ok_sv = __shfl_sync(0xffffffffu, c, 0) <= tol;
      const float r2 = __shfl_sync(0xffffffffu, c, 16);
      kdone = it;
      conv = false;            // no group had ||v^k - v^{k-1}||^2 <= tol
      sv_ok = ok_sv;
      s_cur = (r2 > tauS * tauS) ? fmaf(-tauS, rsqrtf(r2), 1.f) : 0.f;   // P:283-285, R20
      it++;
    } else {
      const float psd = a0.x + a0.y, psb = b0.x + b0.y;
      const float psv = c0.x + c0.y, pr2 = r0.x + r0.y;
      float r2;
      bool ok_sd, ok_sb, ok_sv;
      group_reduce4<G>(psd, psb, psv, pr2, tol, r2, ok_sd, ok_sb, ok_sv);
      if (HK == HK_L2) {
        kdone = it;
        conv = (it >= 1) && sv_ok && ok_sd && ok_sb;   // P:1597-1601 for iteration k = it
        sv_ok = ok_sv;
        // shrink_2 factor of k+1, max(||u|| - tau, 0) / ||u|| = 1 - tau / ||u||,
        // with the hardware reciprocal square root (reading R20)
        s_cur = (r2 > tauS * tauS) ? fmaf(-tauS, rsqrtf(r2), 1.f) : 0.f;
        it++;
      } else {
        it++;
        kdone = it;
        conv = ok_sd && ok_sb && ok_sv;
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    // spec != 0 stops at once; otherwise conv (which needs k >= 1) or the iteration limit
    if (!__any_sync(0xffffffffu, conv || kdone >= lim)) continue;
    const int wstatus = spec == 2 ? INT32_MIN : (spec == 1 ? 0 : (conv ? kdone : -p.max_iter));
    if (spec == 0) my_iters += (unsigned)kdone;

    // ---- finalize: phi = <x - c, d> - 1/2 <d, D d> - t H(d) + gamma ((3.3) at d, R2); grad ----
    // t == 0: phi = J(x), grad = D^{-1}(x - c) (reading R6); invalid input: NaN (R6)
    if (HK == HK_L2 && !dfull) fix_d();
    float qs = 0.f, hsum = 0.f;
    float *grow = p.grad + pt * (int64_t)n;
#pragma unroll
    for (int q = 0; q < NP; q++) {   // D of this lane's slots into b (dead), loads in flight together
      const int j0 = 2 * q, j1 = 2 * q + 1;
      b[q] = make_float2(j0 < jmax ? D_s[cidx(j0)] : 1.f, j1 < jmax ? D_s[cidx(j1)] : 1.f);
    }
    // spec is warp-uniform (one point per warp): one branch outside the slot loops, and no
    // per-slot validity test in the sums (padded slots hold x_hat = 0 and d = 0, so they add 0;
    // only the stores are predicated)
    const bool t0 = spec == 1;
    const float gnan = __int_as_float(0x7fc00000);
#pragma unroll
    for (int c = 0; c < 4; c++) {
      float xh8[1][8];
      ld8(T_XH + 8 * c, xh8[0]);
      wait_ld(xh8);
      float g8[8];
#pragma unroll
      for (int e = 0; e < 8; e++) {
        const float2 dqq = d[4 * c + (e >> 1)], Dq = b[4 * c + (e >> 1)];
        float dq = (e & 1) ? dqq.y : dqq.x;
        if (HK == HK_L2) dq = 0.f - dq;
        const float Dv = (e & 1) ? Dq.y : Dq.x;
        const float xt = xh8[0][e] * (Dv + lam);
        // t == 0 (rare; warp-uniform): dq = D^{-1} xt, and the same quadratic form
        // <xt, dq> - 1/2 <dq, D dq> = 1/2 <xt, D^{-1} xt> = J(x) - gamma; the division sits in a
        // real branch (not if-converted into every finalize)
        if (__builtin_expect(t0, 0)) dq = __fdividef(xt, Dv);
        qs = fmaf(xt, dq, qs);
        qs = fmaf(-0.5f * Dv * dq, dq, qs);
        if (HK == HK_L2) hsum = fmaf(dq, dq, hsum);
        else if (HK == HK_WL1) hsum = fmaf(w_s[cidx(8 * c + e)], fabsf(dq), hsum);
        else hsum += fabsf(dq);
        g8[e] = dq;
      }
      if (spec == 2) {
#pragma unroll
        for (int e = 0; e < 8; e++) g8[e] = gnan;
      }
      if (vrow) {
#pragma unroll
        for (int h = 0; h < 2; h++)
          if (8 * c + 4 * h < jmax)
            *reinterpret_cast<float4 *>(grow + 128 * (2 * c + h) + 4 * gl) =
                make_float4(g8[4 * h], g8[4 * h + 1], g8[4 * h + 2], g8[4 * h + 3]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; e++)
          if (8 * c + e < jmax) grow[cidx(8 * c + e)] = g8[e];
      }
    }
    qs = group_sum<G>(qs);
    hsum = group_sum<G>(hsum);
    float phiv = (spec == 1) ? qs + p.gamma : qs - tt * (HK == HK_L2 ? sqrtf(hsum) : hsum) + p.gamma;
    if (spec == 2) phiv = __int_as_float(0x7fc00000);
    if (gl == 0) { p.phi[pt] = phiv; p.iters[pt] = wstatus; }
    const int64_t claimed = p.claim ? (int64_t)__shfl_sync(0xffffffffu, wclaim, 0) + 2 * ngroups
                                    : pnext + ngroups;   // no counter: static stride
    pt = pnext;
    pnext = claimed;
    have = pt < p.M;
    if (have) start_point(true);
  }
  if (p.iter_total && lane == 0 && my_iters) atomicAdd(p.iter_total, (unsigned long long)my_iters);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_slot), "r"(TMEM_COLS));
}

}  // namespace dtm
}  // namespace hopf
