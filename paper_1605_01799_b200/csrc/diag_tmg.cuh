// diag_tmg.cuh — K1g: split Bregman for diagonal J with G lanes per point (G < 32, several
// points per warp) and tensor memory as an extension of the register file.  sm_100a, FP32
// SIMT; no MMA is involved.  Default for narrow/medium points (C2: n = 100, G = 4, 26 slots).
//
// Paper: split Bregman (3.4a)-(3.4c) P:832-844, stopping rule P:1595-1601, shrink_1 P:239-247,
// shrink_2 P:279-287, phi = (3.3) at d (reading R2), t == 0 / invalid input (R6).  Same method
// and arithmetic as hopf_diag_kernel (diag_kernel.cuh) and hopf_diag_tm_kernel (diag_tm.cuh);
// only the storage and the control flow differ:
//
//   registers : l1 / wl1: a = d - b and b; l2: -d and the pending u — 2 x CPL floats per lane
//   TMEM      : x_hat (columns 0-31), v (32-63), kappa / -kappa (64-95), tau_i (96-127, wl1)
//
// A group of G lanes owns a point, lane gl of the group owns coordinates gl + G j (j < CPL).
// Thread (warp w, lane l) owns TMEM lane 32 (w % 4) + l: its slot values of a vector are one
// 32x32b row, moved in x8 / x4 / x2 chunks per trip (chunk sizes of CPL = 8 a + {0, 2, 4}).
//
// Per trip (l1 / wl1) and coordinate pair: 8 packed FP32 ops ((3.4a) as one FFMA2,
// v^k - v^{k-1}, u, d', d' - d, two test sums) + 4 FMNMX (clamp) + 2 SEL (a waiting group keeps
// its d) + the chunked TMEM traffic.  The stopping test is exact and lazy:
//  * every lane's partial sums are non-negative, so a group whose total passes has every lane's
//    partial passing.  One ballot of the lane predicate (plus "t == 0 / invalid / max_iter")
//    and an AND-fold over the G bits of each group decide whether ANY group can stop; in the
//    common trip none can and no shuffle is executed (the survey's exact ballot prefilter);
//  * otherwise the group totals of ||d^k - d^{k-1}||^2 and ||v^k - v^{k-1}||^2 are formed
//    (transposed butterfly), and where both pass ||d^k - v^k||^2 is summed from d (registers)
//    and v^k (TMEM), so the decision is the paper's at every iteration.
// l2 needs ||u||^2 of every point in every trip (shrink_2): the trip is the pipelined one of
// the register kernel (one 2- or 4-value transposed reduction per trip).
// A stopped group waits (d frozen by a select) until half of the warp's groups wait, then the
// warp finalizes and refills them together: phi / grad stores, next point's x_hat, v, tau into
// TMEM (the chunk stores are warp-collective, so other groups write back what they read).
#pragma once
#include <cfloat>
#include <cstdint>
#include <type_traits>
#include <utility>
#include <cuda_runtime.h>

#include "diag_kernel.cuh"

namespace hopf {
namespace dtg {

constexpr int THREADS = 128, TMEM_COLS = 128;
constexpr int DYN_SMEM = 55 * 1024;   // caps residency at 4 CTAs per SM (4 x 128 TMEM columns)
constexpr int C_XH = 0, C_V = 32, C_K = 64, C_TAU = 96;

// tcgen05.ld / st of N in {2, 4, 8} consecutive columns of this thread's lane, column offset OFF
// folded into the instruction (the base stays in one uniform register)
template <int N, int OFF>
__device__ __forceinline__ void ldn(uint32_t base, float (&v)[8]) {
  uint32_t r[8];
  if constexpr (N == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8+%9];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(base), "n"(OFF));
  } else if constexpr (N == 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4+%5];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(base), "n"(OFF));
  } else {
    static_assert(N == 2, "chunk of 2, 4 or 8 columns");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2+%3];"
                 : "=r"(r[0]), "=r"(r[1]) : "r"(base), "n"(OFF));
  }
#pragma unroll
  for (int i = 0; i < N; i++) v[i] = __uint_as_float(r[i]);
}
template <int N, int OFF>
__device__ __forceinline__ void stn(uint32_t base, const float (&v)[8]) {
  if constexpr (N == 8) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0+%9], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(base), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])),
                    "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])),
                    "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
                    "n"(OFF));
  } else if constexpr (N == 4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0+%5], {%1,%2,%3,%4};"
                 :: "r"(base), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])),
                    "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])), "n"(OFF));
  } else {
    static_assert(N == 2, "chunk of 2, 4 or 8 columns");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0+%3], {%1,%2};"
                 :: "r"(base), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "n"(OFF));
  }
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

// compile-time loop over the TMEM chunks of a CPL-slot vector: f(chunk index, chunk size)
template <int CPL, typename F, int... C>
__device__ __forceinline__ void for_chunks_impl(F &&f, std::integer_sequence<int, C...>) {
  (f(std::integral_constant<int, C>{}, std::integral_constant<int, (CPL - 8 * C < 8 ? CPL - 8 * C : 8)>{}), ...);
}
template <int CPL, typename F>
__device__ __forceinline__ void for_chunks(F &&f) {
  for_chunks_impl<CPL>(f, std::make_integer_sequence<int, (CPL + 7) / 8>{});
}

__device__ __forceinline__ float2 sel2(bool c, float2 a, float2 b) {
  return make_float2(c ? a.x : b.x, c ? a.y : b.y);
}

// ---- bulk asynchronous copies (TMA engine, no tensor map): one lane moves a point's row ------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 "selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  }
}
// global row -> shared buffer, completion (bytes) signalled on `bar`
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// shared buffer -> global row (bulk group of the issuing thread)
__device__ __forceinline__ void bulk_store(void *dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst), "r"(src), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// row pitch (floats) of the per-group shared buffers: >= the variant's padded width, a
// multiple of 4 (16-byte bulk copies) and an odd multiple of G (G >= 4), so that the strided
// reads / writes of a warp (lane gl of group g at g * pitch + gl + G j) hit 32 different banks:
// g * pitch mod 32 then runs over the 32 / G distinct multiples of G
__host__ __device__ constexpr int row_pitch(int w, int G) {
  int r = (w + 3) & ~3;
  while (r % G != 0 || (r / G) % 2 == 0) r += 4;
  return r;
}
template <int G, int CPL>
__host__ __device__ constexpr size_t smem_bytes() {
  return (size_t)2 * G * CPL * 16 + (size_t)2 * (THREADS / G) * row_pitch(G * CPL + 4, G) * 4 +
         (size_t)(THREADS / G) * 8;
}

// The bases of X and grad must be 16-byte aligned (the dispatcher in tmg_api.cu checks): x of a
// group's next point is prefetched into shared memory by a bulk copy one point ahead (plus up to
// 3 plain loads for a row end off the 16-byte grid), and grad leaves through a shared buffer by a
// bulk store (plus up to 3 plain stores at each end).
template <int G, int CPL, int HK, bool BULK>
#ifndef HOPF_TMG_MINB
#define HOPF_TMG_MINB 4
#endif
__global__ void __launch_bounds__(THREADS, HOPF_TMG_MINB) hopf_diag_tmg_kernel(const DiagParams p) {
  static_assert(BULK, "instantiated with bulk row copies only (unaligned rows use the register kernel)");
  static_assert(G >= 2 && G <= 16 && (G & (G - 1)) == 0, "G in {2, 4, 8, 16}");
  static_assert(CPL % 2 == 0 && CPL <= 32 && (CPL % 8 == 0 || CPL % 8 == 2 || CPL % 8 == 4),
                "CPL = 8 a + {0, 2, 4}, at most 32");
  static_assert(HK == HK_L1 || HK == HK_WL1 || HK == HK_L2 || HK == HK_ELL || HK == HK_LINF, "l1, wl1, l2, ell, linf");
  static_assert(smem_bytes<G, CPL>() <= (size_t)DYN_SMEM, "shared buffers exceed the budget");
  constexpr int NP = CPL / 2;
  constexpr int GPW = 32 / G, GPB = THREADS / G;
  constexpr int PITCH = row_pitch(G * CPL + 4, G);   // a row starts at offset (r n) mod 4 in its buffer
  constexpr bool L2 = HK == HK_L2, WL1 = HK == HK_WL1, ELL = HK == HK_ELL, LINF = HK == HK_LINF;
  constexpr bool WTAB = WL1 || ELL;   // per-coordinate weights in the tables
  extern __shared__ __align__(16) uint8_t dyn_smem[];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int base = lane & ~(G - 1);
  const int grp = threadIdx.x / G;   // group index in the block
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int n = p.n;
  const int64_t M = p.M;
  const float lam = p.lambda, tol = p.tol;
  const int jmax = (n - gl + G - 1) / G;   // slots j < jmax are real coordinates
  // shared memory: per-coordinate constants (padded coordinates: D = 1, w = c = 0)
  //   A_s[i] = (1/(D_i + lambda), w_i, c_i, 0)   (setup)
  //   B_s[i] = (D_i + lambda, w_i, -D_i/2, 1/D_i) (finalize)
  // then per group the next point's x row, the grad row on its way out, and the x mbarrier
  float4 *const A_s = reinterpret_cast<float4 *>(dyn_smem);
  float4 *const B_s = A_s + G * CPL;
  float *const xbuf = reinterpret_cast<float *>(B_s + G * CPL);
  float *const gbuf = xbuf + GPB * PITCH;
  uint64_t *const xbar = reinterpret_cast<uint64_t *>(gbuf + GPB * PITCH);
  // this lane's slot j of the current point's x / grad row: my_x[G j], my_g[G j].  Element i of
  // row r sits at buffer offset (r n) mod 4 + i, so that the row's 16-byte aligned part maps to
  // 16-byte aligned shared memory (bulk copies need both ends aligned); set at each refill
  float *my_x = xbuf + grp * PITCH + gl;
  float *my_g = gbuf + grp * PITCH + gl;
  const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << (lane & ~(G - 1));
  const float4 *const my_A = A_s + gl;
  const float4 *const my_B = B_s + gl;
  const uint32_t my_bar = smem_u32(xbar + grp);
  for (int i = threadIdx.x; i < G * CPL; i += THREADS) {
    const bool real = i < n;
    const float Dv = real ? __ldg(p.D + i) : 1.f;
    const float wv = (WTAB && real) ? __ldg(p.w + i) : (ELL ? 1.f : 0.f);   // ELL pads with w = 1
    const float cv = (p.c && real) ? __ldg(p.c + i) : 0.f;
    A_s[i] = make_float4(1.f / (Dv + lam), wv, cv, 0.f);
    B_s[i] = make_float4(Dv + lam, wv, -0.5f * Dv, 1.f / Dv);
  }
  if (gl == 0) mbar_init(my_bar, 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&tmem_slot)), "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp-uniform TMEM base (lane-0 shuffle: provably uniform, one uniform register)
  const uint32_t tl0 = __shfl_sync(0xffffffffu, tmem_slot + ((uint32_t)(32 * (warp & 3)) << 16), 0);

  // kappa (l2: -kappa) = lambda / (D + lambda) of this lane's slots -> TMEM, once
  const float ksign = L2 ? -lam : lam;
  for_chunks<CPL>([&](auto ci, auto szc) {
    constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
    float kv[8];
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const int j = 8 * c + e;
      kv[e] = (e < SZ && j < jmax) ? ksign * my_A[G * j].x : 0.f;
    }
    stn<SZ, C_K + 8 * c>(tl0, kv);
    if constexpr (ELL) {   // w_i of this lane's slots (padded slots: w = 1, their u is 0)
      float wv8[8];
#pragma unroll
      for (int e = 0; e < 8; e++) wv8[e] = e < SZ ? my_A[G * (8 * c + e)].y : 1.f;
      stn<SZ, C_TAU + 8 * c>(tl0, wv8);
    }
  });
  // ELL: min_i w_i, the scale of the Newton stopping test on mu
  float wmin = 1.f;
  if constexpr (ELL) {
    wmin = __int_as_float(0x7f800000);
    for (int i = 0; i < n; i++) wmin = fminf(wmin, A_s[i].y);
  }

  float2 d[NP], b[NP];
  // points: generations 0 and 1 static (gid, gid + ngroups), later ones claimed by the warp from
  // p.claim one generation ahead (GPW consecutive points, one per group), so warps that drew
  // cheap points take more of them and the launch ends within about one generation
  int64_t pt = gid;
  int64_t pnext = gid + ngroups;
  unsigned long long wclaim = 0;   // lane 0: the claim made at the last refill
  bool have = pt < M;
  bool waiting = false;   // the solve stopped; d frozen until the warp finalizes
  int wstatus = 0;
  int it = 0;
  int lim = 0;            // iteration at which the solve must stop: max_iter, 0 for t == 0 / invalid
  float tt = 0.f, tauS = 0.f;
  float tpre = have ? __ldg(p.t + pt) : 0.f;   // t of the group's next point (prefetched)
  uint32_t xph = 0;       // parity of the group's x-row mbarrier
  int spec = 0;           // 0 normal, 1 t == 0, 2 invalid
  float s_cur = 1.f;      // l2: shrink factor of the pending (3.4b)
  bool sv_ok = false;     // l2: ||v^k - v^{k-1}||^2 <= tol of the pending iteration
  float mu = 0.f;         // ELL / LINF: multiplier of the last projection (warm start of the next)
#pragma unroll
  for (int q = 0; q < NP; q++) d[q] = b[q] = splat2(0.f);
  // x row of point r: its 16-byte aligned part [a0, a1) by one bulk copy (leader), the last
  // (r n + n) mod 4 floats by plain loads of lanes gl < that count into xtail (stored into the
  // buffer at the refill); with n % 4 == 0 the whole row is one bulk copy
  auto prefetch_x = [&](int64_t r) {
    const int64_t off = r * (int64_t)n, a0 = off & ~(int64_t)3, a1 = (off + n) & ~(int64_t)3;
    if (gl == 0) bulk_load(smem_u32(xbuf + grp * PITCH), p.X + a0, (uint32_t)(a1 - a0) * 4u, my_bar);
    const int64_t e = off + n;
    const int tl = (int)(e & 3);
    return gl < tl ? __ldg(p.X + (e - tl) + gl) : 0.f;
  };
  float xtail = have ? prefetch_x(pt) : 0.f;

  // ---- start the point pt of the groups with `fresh` set (collective: every lane executes the
  // TMEM chunk traffic; other lanes write back what they read).  Setup: x_hat = (x - c)/(D + lambda),
  // v^0 = d^0 = x - c, b^0 = 0 (reading R5); l2 keeps -d and the pending u = x - c.
  auto refill = [&](bool fresh) {
    bool bad = false;
    if (fresh) {
      tt = p.tscale * tpre;
      bad = !(tt >= 0.f) || !finite_f(tt);
      tpre = pnext < M ? __ldg(p.t + pnext) : 0.f;
      mbar_wait(my_bar, xph);
      xph ^= 1u;
      {
        const int64_t off = pt * (int64_t)n;
        const int o = (int)(off & 3), tl = (int)((off + n) & 3);
        float *const xr = xbuf + grp * PITCH + o;   // element i at xr[i]
        if (gl < tl) xr[n - tl + gl] = xtail;
        __syncwarp(gmask);
        my_x = xr + gl;
        my_g = gbuf + grp * PITCH + o + gl;
      }
#pragma unroll
      for (int q = 0; q < NP; q++) {   // x from the prefetched row (padding slots read 0 below)
        const int j0 = 2 * q, j1 = 2 * q + 1;
        d[q] = make_float2(j0 < jmax ? my_x[G * j0] : 0.f, j1 < jmax ? my_x[G * j1] : 0.f);
      }
      float2 fin = splat2(0.f);   // x * 0 accumulates NaN iff some x is NaN or infinite
#pragma unroll
      for (int q = 0; q < NP; q++) fin = fma2(d[q], splat2(0.f), fin);
      bad |= !(fin.x == 0.f && fin.y == 0.f);
    }
    // the group's row has been read (and its tail written): its leader prefetches the following
    // point's x into it (generic-proxy accesses ordered before the async-proxy copy)
    if (fresh) fence_proxy_async();
    __syncwarp();
    if (fresh && pnext < M) xtail = prefetch_x(pnext);
    // the generation after next (consumed at the next finalize: the atomic's latency is hidden)
    const bool any_fresh = __any_sync(0xffffffffu, fresh);
    if (lane == 0 && any_fresh && p.claim) wclaim = atomicAdd(p.claim, (unsigned long long)GPW);
    const float tl = tt / lam;
    // the chunk stores are warp-collective: lanes that keep their point write back what they
    // read; when every lane starts a point or has none left (the lockstep case), nothing is read
#ifndef HOPF_TMG_SKIPLOAD
#define HOPF_TMG_SKIPLOAD 0   // skipping the reads when every lane is new measured slower (C2 1.265 vs 1.231 ms)
#endif
    const bool keep_any = !HOPF_TMG_SKIPLOAD || __any_sync(0xffffffffu, have && !fresh);
    for_chunks<CPL>([&](auto ci, auto szc) {
      constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
      float ch[3][8];
#pragma unroll
      for (int e = 0; e < 8; e++) ch[0][e] = ch[1][e] = ch[2][e] = 0.f;
      if (keep_any) {
        ldn<SZ, C_XH + 8 * c>(tl0, ch[0]);
        ldn<SZ, C_V + 8 * c>(tl0, ch[1]);
        if constexpr (WL1) ldn<SZ, C_TAU + 8 * c>(tl0, ch[2]);
        wait_ld(ch);
      }
      if (fresh) {
#pragma unroll
        for (int e = 0; e < SZ; e++) {
          const int j = 8 * c + e;
          const float4 A = my_A[G * j];
          float &xv = (e & 1) ? d[4 * c + (e >> 1)].y : d[4 * c + (e >> 1)].x;
          xv -= A.z;                       // x - c (padded slots: 0 - 0)
          ch[0][e] = xv * A.x;             // x_hat
          ch[1][e] = xv;                   // v^0 = x - c
          if (WL1) ch[2][e] = tl * A.y;    // tau_i = t w_i / lambda
        }
      }
      stn<SZ, C_XH + 8 * c>(tl0, ch[0]);
      stn<SZ, C_V + 8 * c>(tl0, ch[1]);
      if constexpr (WL1) stn<SZ, C_TAU + 8 * c>(tl0, ch[2]);
    });
    if (fresh) {
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const float2 xt = d[q];
        if (L2) { d[q] = make_float2(-xt.x, -xt.y); b[q] = xt; }   // -d^0, pending u
        else b[q] = splat2(0.f);                                    // a^0 = d^0 = x - c, b^0 = 0
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    bad = group_any<G>(bad);
    if (fresh) {
      spec = bad ? 2 : (tt == 0.f ? 1 : 0);
      lim = spec ? 0 : p.max_iter;
      tauS = tt / lam;
      it = 0;
      mu = 0.f;
      s_cur = 1.f;
      sv_ok = false;
      waiting = false;
    }
  };
  refill(have);

  // A stopped group's result d^k goes to its grad row buffer at once (grad := d, R1; NaN for an
  // invalid point): the group then keeps iterating harmlessly until the warp finalizes, so the
  // trip needs no per-slot select to freeze d.  Collective; `stop` marks the stopping groups.
  auto stash = [&](bool stop) {
    if (stop && gl == 0) bulk_wait_read();   // the group's previous grad row has left the buffer
    __syncwarp();
    if (stop) {
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const float2 g = L2 ? make_float2(-d[q].x, -d[q].y)
                            : ((ELL || LINF) ? d[q] : add2(d[q], b[q]));   // l1 / wl1: d = a + b
        my_g[G * (2 * q)] = g.x;   // (an invalid point's row is set to NaN at finalize)
        my_g[G * (2 * q + 1)] = g.y;
      }
    }
  };

  unsigned my_iters = 0;   // this lane's share of p.iter_total (group lane 0 counts)
  bool any_have = __any_sync(0xffffffffu, have);
  while (any_have) {
    const bool live = have && !waiting;
    float2 a0 = splat2(0.f), b0 = a0, c0 = a0, r0 = a0;   // one packed accumulator per sum
    const float2 sP = splat2(s_cur), tP = splat2(tauS);
    const float2 nsP = splat2(-s_cur), omsP = splat2(1.f - s_cur), na_sP = splat2(1.f - 2.f * s_cur);
    // l2: the ||d^k - d^{k-1}||^2, ||d^k - v^k||^2 sums only matter where ||v^k - v^{k-1}||^2 <= tol
    // (sv_ok, known before the trip); trips where no group of the warp has it skip both (exact)
    const bool full_test = L2 && __any_sync(0xffffffffu, live && sv_ok);
    auto trip = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      for_chunks<CPL>([&](auto ci, auto szc) {
        constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
        float ch[WL1 ? 4 : 3][8];   // kappa, x_hat, v (, tau)
        ldn<SZ, C_K + 8 * c>(tl0, ch[0]);
        ldn<SZ, C_XH + 8 * c>(tl0, ch[1]);
        ldn<SZ, C_V + 8 * c>(tl0, ch[2]);
        if constexpr (WL1) ldn<SZ, C_TAU + 8 * c>(tl0, ch[WL1 ? 3 : 0]);
        wait_ld(ch);
#pragma unroll
        for (int e2 = 0; e2 < SZ / 2; e2++) {
          const int q = 4 * c + e2;
          const float2 kq = make_float2(ch[0][2 * e2], ch[0][2 * e2 + 1]);
          const float2 xh = make_float2(ch[1][2 * e2], ch[1][2 * e2 + 1]);
          const float2 v = make_float2(ch[2][2 * e2], ch[2][2 * e2 + 1]);
          float2 vn;
          if constexpr (L2) {
            // d[q] = -d_{k-1}, kq = -kappa, b[q] = u_k; d_k = s_k u_k, b_k = (1 - s_k) u_k,
            // d_k - b_k = (2 s_k - 1) u_k: scalings of u_k ((3.4b), (3.4c))
            const float2 u = b[q];
            if (FULL) {
              const float2 dd = fma2(sP, u, d[q]);                  // d_k - d_{k-1}
              const float2 nd = sub2(d[q], dd);                     // -d_k
              const float2 dmv = add2(nd, v);                       // v^k - d^k
              d[q] = nd;
              a0 = fma2(dd, dd, a0); b0 = fma2(dmv, dmv, b0);
            } else {
              d[q] = __fmul2_rn(nsP, u);                             // -d_k
            }
            const float2 bk = __fmul2_rn(omsP, u);                  // b_k
            const float2 na = __fmul2_rn(na_sP, u);                 // -(d_k - b_k)
            vn = fma2(kq, na, xh);                                  // (3.4a): v_{k+1}
            const float2 dv = sub2(vn, v);
            b[q] = add2(vn, bk);                                    // u_{k+1} = v_{k+1} + b_k
            c0 = fma2(dv, dv, c0);
            r0 = fma2(b[q], b[q], r0);
          } else {
            // l1 / wl1 state: d[q] holds a = d - b (what (3.4a) consumes), b[q] = b; both are
            // updated in place (no register moves of loop-carried values)
            vn = fma2(kq, d[q], xh);                                // (3.4a): v^k = x_hat + kappa a
            const float2 dv = sub2(vn, v);                          // v^k - v^{k-1}
            const float2 u = add2(vn, b[q]);
            const float2 tq = WL1 ? make_float2(ch[WL1 ? 3 : 0][2 * e2], ch[WL1 ? 3 : 0][2 * e2 + 1]) : tP;
            const float2 t = sub2(vn, d[q]);                        // v^k - a^{k-1}
            b[q] = clamp2(u, tq);                                   // b^k: projection (Moreau)
            d[q] = fma2(b[q], splat2(-2.f), u);                     // a^k = d^k - b^k, d^k = u - b^k
            const float2 dd = sub2(t, b[q]);                        // d^k - d^{k-1} = v^k - b^k - a^{k-1}
            a0 = fma2(dd, dd, a0); c0 = fma2(dv, dv, c0);
          }
          ch[2][2 * e2] = vn.x;
          ch[2][2 * e2 + 1] = vn.y;
        }
        stn<SZ, C_V + 8 * c>(tl0, ch[2]);
      });
    };
    bool conv = false;
    int kdone;
    if constexpr (ELL || LINF) {
      // (3.4a), u = v + b for every coordinate (b holds u until the projection is known), fused
      // with the first evaluation of the projection's sums at the warm-start mu
      float2 s1 = splat2(0.f), s2 = s1;
      {
        const float2 muP = splat2(mu);
        for_chunks<CPL>([&](auto ci, auto szc) {
          constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
          float ch[4][8];   // kappa, x_hat, v, w
          ldn<SZ, C_K + 8 * c>(tl0, ch[0]);
          ldn<SZ, C_XH + 8 * c>(tl0, ch[1]);
          ldn<SZ, C_V + 8 * c>(tl0, ch[2]);
          if constexpr (ELL) ldn<SZ, C_TAU + 8 * c>(tl0, ch[3]);
          else {
#pragma unroll
            for (int e = 0; e < 8; e++) ch[3][e] = 0.f;
          }
          wait_ld(ch);
#pragma unroll
          for (int e2 = 0; e2 < SZ / 2; e2++) {
            const int q = 4 * c + e2;
            const float2 kq = make_float2(ch[0][2 * e2], ch[0][2 * e2 + 1]);
            const float2 xh = make_float2(ch[1][2 * e2], ch[1][2 * e2 + 1]);
            const float2 v = make_float2(ch[2][2 * e2], ch[2][2 * e2 + 1]);
            const float2 a = sub2(d[q], b[q]);
            const float2 vn = fma2(kq, a, xh);                    // (3.4a): v^k
            const float2 dv = sub2(vn, v);
            c0 = fma2(dv, dv, c0);
            const float2 u = add2(vn, b[q]);
            b[q] = u;
            if constexpr (ELL) {   // S1 = sum w u^2/(w + mu)^2, S2 = sum w u^2/(w + mu)^3
              const float2 w = make_float2(ch[3][2 * e2], ch[3][2 * e2 + 1]);
              const float2 ee = add2(w, muP);
              const float2 r = make_float2(rcp_approx(ee.x), rcp_approx(ee.y));
              const float2 hh = __fmul2_rn(u, r);
              const float2 wh2 = __fmul2_rn(__fmul2_rn(w, hh), hh);
              s1 = add2(s1, wh2);
              s2 = fma2(wh2, r, s2);
            } else {               // S1 = sum max(|u| - mu, 0), S2 = #{|u| > mu}
              const float ex = fabsf(u.x) - mu, ey = fabsf(u.y) - mu;
              s1.x += fmaxf(ex, 0.f);
              s1.y += fmaxf(ey, 0.f);
              s2.x += ex > 0.f ? 1.f : 0.f;
              s2.y += ey > 0.f ? 1.f : 0.f;
            }
            ch[2][2 * e2] = vn.x;
            ch[2][2 * e2 + 1] = vn.y;
          }
          stn<SZ, C_V + 8 * c>(tl0, ch[2]);
        });
      }
      float S1, S2;
      bool ok_sv;
      group_reduce3<G>(s1.x + s1.y, s2.x + s2.y, c0.x + c0.y, tol, S1, S2, ok_sv);
      bool act = live && spec == 0;
      int nit = 0;
      if constexpr (ELL) {
        // the dual-ellipsoid projection's multiplier by Newton on 1/sqrt(S1) - 1/tau, warm start,
        // clamp at 0 (the inside case), a step below 1e-3 (mu + min w) accepted (reading R27;
        // the same scheme as the register kernel)
        const float itau = rcp_approx(tauS);
        for (;;) {
          if (act) {
            const float mun = S2 > 0.f ? fmaxf(fmaf(S1 * rcp_approx(S2), fmaf(sqrtf(S1), itau, -1.f), mu), 0.f)
                                       : 0.f;   // u = 0: d' = 0
            act = !(fabsf(mun - mu) <= 1e-3f * (mun + wmin)) && ++nit < 30;
            mu = mun;
          }
          if (!__any_sync(0xffffffffu, act)) break;
          float2 t1 = splat2(0.f), t2 = splat2(0.f);
          const float2 muP = splat2(mu);
          for_chunks<CPL>([&](auto ci, auto szc) {
            constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
            float wv[1][8];
            ldn<SZ, C_TAU + 8 * c>(tl0, wv[0]);
            wait_ld(wv);
#pragma unroll
            for (int e2 = 0; e2 < SZ / 2; e2++) {
              const float2 w = make_float2(wv[0][2 * e2], wv[0][2 * e2 + 1]);
              const float2 ee = add2(w, muP);
              const float2 r = make_float2(rcp_approx(ee.x), rcp_approx(ee.y));
              const float2 hh = __fmul2_rn(b[4 * c + e2], r);
              const float2 wh2 = __fmul2_rn(__fmul2_rn(w, hh), hh);
              t1 = add2(t1, wh2);
              t2 = fma2(wh2, r, t2);
            }
          });
          S1 = group_sum<G>(t1.x + t1.y);
          S2 = group_sum<G>(t2.x + t2.y);
        }
        // (3.4b): d' = mu u / (w + mu); (3.4c): b' = u - d'
        const float2 muP = splat2(mu);
        for_chunks<CPL>([&](auto ci, auto szc) {
          constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
          float wv[1][8];
          ldn<SZ, C_TAU + 8 * c>(tl0, wv[0]);
          wait_ld(wv);
#pragma unroll
          for (int e2 = 0; e2 < SZ / 2; e2++) {
            const int q = 4 * c + e2;
            const float2 w = make_float2(wv[0][2 * e2], wv[0][2 * e2 + 1]);
            const float2 ee = add2(w, muP);
            const float2 r = make_float2(rcp_approx(ee.x), rcp_approx(ee.y));
            const float2 u = b[q];
            const float2 dn = __fmul2_rn(__fmul2_rn(muP, u), r);
            b[q] = sub2(u, dn);
            const float2 dd = sub2(dn, d[q]);
            d[q] = dn;
            a0 = fma2(dd, dd, a0);
          }
        });
      } else {
        // the l1-ball multiplier by active-set Newton, exact acceptance when no |u_i| lies between
        // two iterates (reading R28; the same scheme as the register kernel)
        float mu_e = mu;
        for (;;) {
          float mun = mu_e;
          if (act) mun = S2 > 0.f ? fmaxf(mu_e + __fdividef(S1 - tauS, S2), 0.f) : 0.f;
          // empty active set at mu_e (a warm start above every |u_i|): step to the root of the
          // top piece, max |u| - tau, at or left of the root, instead of falling back to 0
          if (__any_sync(0xffffffffu, act && S2 == 0.f)) {
            float um = 0.f;
#pragma unroll
            for (int q = 0; q < NP; q++) um = fmaxf(um, fmaxf(fabsf(b[q].x), fabsf(b[q].y)));
            um = group_max<G>(um);
            if (act && S2 == 0.f) mun = fmaxf(um - tauS, 0.f);
          }
          bool cross = false;
#pragma unroll
          for (int q = 0; q < NP; q++) {
            const float ax = fabsf(b[q].x), ay = fabsf(b[q].y);
            cross |= ((ax > mu_e) != (ax > mun)) || ((ay > mu_e) != (ay > mun));
          }
          cross = group_any<G>(cross);
          const bool tiny = fabsf(mun - mu_e) <= HOPF_TINY_STEP * fmaxf(mun, 1e-30f);
          if (act && (!cross || tiny || ++nit >= 64)) { mu = mun; act = false; }
          if (!__any_sync(0xffffffffu, act)) break;
          if (act) mu_e = mun;
          float2 ta = splat2(0.f), tn = ta;
#pragma unroll
          for (int q = 0; q < NP; q++) {
            const float ex = fabsf(b[q].x) - mu_e, ey = fabsf(b[q].y) - mu_e;
            ta.x += fmaxf(ex, 0.f);
            ta.y += fmaxf(ey, 0.f);
            tn.x += ex > 0.f ? 1.f : 0.f;
            tn.y += ey > 0.f ? 1.f : 0.f;
          }
          S1 = group_sum<G>(ta.x + ta.y);
          S2 = group_sum<G>(tn.x + tn.y);
        }
        // (3.4b): d' = u - shrink_1(u, mu) = clamp(u, -mu, mu); (3.4c): b' = u - d'
        const float2 muP = splat2(mu);
#pragma unroll
        for (int q = 0; q < NP; q++) {
          const float2 u = b[q];
          const float2 dn = clamp2(u, muP);
          b[q] = sub2(u, dn);
          const float2 dd = sub2(dn, d[q]);
          d[q] = dn;
          a0 = fma2(dd, dd, a0);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;");
      if (live) it++;
      kdone = it;
      // ||v^k - v^{k-1}||^2 came with the projection sums; ||d^k - d^{k-1}||^2 now;
      // ||d^k - v^k||^2 only where both pass (v^k from TMEM)
      const float sd = group_sum<G>(a0.x + a0.y);
      const bool need = live && spec == 0 && ok_sv && sd <= tol;
      if (__any_sync(0xffffffffu, need)) {
        float2 sb2 = splat2(0.f);
        for_chunks<CPL>([&](auto ci, auto szc) {
          constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
          float vv[1][8];
          ldn<SZ, C_V + 8 * c>(tl0, vv[0]);
          wait_ld(vv);
#pragma unroll
          for (int e2 = 0; e2 < SZ / 2; e2++) {
            const float2 dmv = sub2(d[4 * c + e2], make_float2(vv[0][2 * e2], vv[0][2 * e2 + 1]));
            sb2 = fma2(dmv, dmv, sb2);
          }
        });
        const float sb = group_sum<G>(sb2.x + sb2.y);
        conv = need && sb <= tol;
      }
      const bool stop = live && (spec != 0 || conv || kdone >= lim);
      if (!__any_sync(0xffffffffu, stop)) continue;
      if (stop) {
        waiting = true;
        wstatus = spec == 2 ? INT32_MIN : (spec == 1 ? 0 : (conv ? kdone : -lim));
        if (spec == 0) my_iters += (unsigned)kdone;
      }
      stash(stop);
    } else {
    constexpr unsigned LEADERS = G == 2 ? 0x55555555u : G == 4 ? 0x11111111u : G == 8 ? 0x01010101u : 0x00010001u;
    unsigned ev = 0;
    if constexpr (L2) {
      if (full_test) trip(std::true_type{});
      else trip(std::false_type{});
      asm volatile("tcgen05.wait::st.sync.aligned;");
    } else {
      // l1 / wl1: trips until some group may stop.  Exact prefilter: a group total <= tol needs
      // every lane's (non-negative) partial <= tol; t == 0 / invalid points (lim = 0) and
      // max_iter are forced events.  Two trips per pass of the loop.
      auto fast = [&]() -> bool {
        a0 = c0 = splat2(0.f);
        trip(std::false_type{});
        asm volatile("tcgen05.wait::st.sync.aligned;");
        it += live ? 1 : 0;
        const float psd = a0.x + a0.y, psv = c0.x + c0.y;
        const bool lane_ev = live && ((psd <= tol && psv <= tol) || it >= lim);
        ev = __ballot_sync(0xffffffffu, lane_ev);
#pragma unroll
        for (int o = 1; o < G; o <<= 1) ev &= ev >> o;   // bit base of a group: all G lanes set
        return (ev & LEADERS) != 0u;
      };
      while (!fast() && !fast()) {
      }
    }

    if constexpr (L2) {
      const float psd = a0.x + a0.y, psb = b0.x + b0.y, psv = c0.x + c0.y, pr2 = r0.x + r0.y;
      float r2;
      bool ok_sd = false, ok_sb = false, ok_sv;
      if (full_test) group_reduce4<G>(psd, psb, psv, pr2, tol, r2, ok_sd, ok_sb, ok_sv);
      else group_reduce2<G>(psv, pr2, tol, ok_sv, r2);
      kdone = it;
      conv = (it >= 1) && sv_ok && ok_sd && ok_sb;   // P:1597-1601 for iteration k = it
      sv_ok = ok_sv;
      // shrink_2 factor of k+1 with the hardware reciprocal square root (R20)
      s_cur = (r2 > tauS * tauS) ? fmaf(-tauS, rsqrtf(r2), 1.f) : 0.f;
      it += live ? 1 : 0;
      const bool stop = live && (spec != 0 || (kdone >= 1 && (conv || kdone >= lim)));
      if (!__any_sync(0xffffffffu, stop)) continue;
      if (stop) {
        waiting = true;
        wstatus = spec == 2 ? INT32_MIN : (spec == 1 ? 0 : (conv ? kdone : -lim));
        if (spec == 0) my_iters += (unsigned)kdone;
      }
      stash(stop);
    } else {
      kdone = it;
      const float psd = a0.x + a0.y, psv = c0.x + c0.y;
      const bool cand = (ev >> base) & 1u;
      bool ok_sd, ok_sv;
      group_test2<G>(psd, psv, tol, ok_sd, ok_sv);
      // ||d^k - v^k||^2 only where the first two pass (v^k from TMEM)
      const bool need = cand && spec == 0 && ok_sd && ok_sv;
      if (__any_sync(0xffffffffu, need)) {
        float2 sb2 = splat2(0.f), sb3 = sb2;
        for_chunks<CPL>([&](auto ci, auto szc) {
          constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
          float vv[1][8];
          ldn<SZ, C_V + 8 * c>(tl0, vv[0]);
          wait_ld(vv);
#pragma unroll
          for (int e2 = 0; e2 < SZ / 2; e2++) {
            const int q = 4 * c + e2;
            const float2 dk = (L2 || ELL || LINF) ? d[q] : add2(d[q], b[q]);   // l1: d^k = a + b
            const float2 dmv = sub2(dk, make_float2(vv[0][2 * e2], vv[0][2 * e2 + 1]));
            if (e2 & 1) sb3 = fma2(dmv, dmv, sb3);
            else sb2 = fma2(dmv, dmv, sb2);
          }
        });
        const float sb = group_sum<G>((sb2.x + sb2.y) + (sb3.x + sb3.y));
        conv = need && sb <= tol;
      }
      const bool stop = cand && (spec != 0 || conv || kdone >= lim);
      if (!__any_sync(0xffffffffu, stop)) continue;
      if (stop) {
        waiting = true;
        wstatus = spec == 2 ? INT32_MIN : (spec == 1 ? 0 : (conv ? kdone : -lim));
        if (spec == 0) my_iters += (unsigned)kdone;
      }
      stash(stop);
    }
    }   // H in {l1, wl1, l2}
    {
      const unsigned gbit = (gl == 0) ? 1u : 0u;
      const int nwait = __popc(__ballot_sync(0xffffffffu, waiting && gbit));
      if (nwait == 0) continue;
      const int nhave = __popc(__ballot_sync(0xffffffffu, have && gbit));
      if (nwait < nhave) continue;   // lockstep generations: finalize when every group waits
                                     // (C2: half the groups 1.65 ms, three quarters 1.50, all 1.26)
    }

    // ============ finalize the waiting groups (all lanes compute, waiting groups store) ========
    // phi = <x - c, d> - 1/2 <d, D d> - t H(d) + gamma ((3.3) at d, R2), x - c = x_hat (D + lambda);
    // t == 0: d := D^{-1}(x - c), the same expression gives J(x) (R6); invalid: NaN (R6)
    const bool done = waiting;
    const float gnan = __int_as_float(0x7fc00000);
    if (__any_sync(0xffffffffu, done && spec == 1)) {   // rare: t == 0 points, grad = D^{-1}(x - c)
      for_chunks<CPL>([&](auto ci, auto szc) {
        constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
        float xh8[1][8];
        ldn<SZ, C_XH + 8 * c>(tl0, xh8[0]);
        wait_ld(xh8);
        if (done && spec == 1) {
#pragma unroll
          for (int e = 0; e < SZ; e++) {
            const float4 B = my_B[G * (8 * c + e)];
            my_g[G * (8 * c + e)] = xh8[0][e] * B.x * B.w;
          }
        }
      });
    }
    if (__any_sync(0xffffffffu, done && spec == 2)) {   // rare: invalid points, grad = NaN
      if (done && spec == 2) {
#pragma unroll
        for (int j = 0; j < CPL; j++) my_g[G * j] = gnan;
      }
    }
    // the grad rows (stashed at stop) are read back for phi; non-finalized lanes read their own
    // (irrelevant) buffer contents
    float qs0 = 0.f, qs1 = 0.f, hs0 = 0.f, hs1 = 0.f;
    for_chunks<CPL>([&](auto ci, auto szc) {
      constexpr int c = decltype(ci)::value, SZ = decltype(szc)::value;
      float xh8[1][8];
      ldn<SZ, C_XH + 8 * c>(tl0, xh8[0]);
      wait_ld(xh8);
#pragma unroll
      for (int e = 0; e < SZ; e++) {
        const int j = 8 * c + e;
        const float4 B = my_B[G * j];
        const float dq = my_g[G * j];
        const float xt = xh8[0][e] * B.x;
        float &qs = (e & 1) ? qs1 : qs0;
        float &hs = (e & 1) ? hs1 : hs0;
        qs = fmaf(xt, dq, qs);
        qs = fmaf(B.z * dq, dq, qs);
        if (L2) hs = fmaf(dq, dq, hs);
        else if (ELL) hs = fmaf(B.y * dq, dq, hs);
        else if (LINF) hs = fmaxf(hs, fabsf(dq));
        else if (WL1) hs = fmaf(B.y, fabsf(dq), hs);
        else hs += fabsf(dq);
      }
    });
    fence_proxy_async();
    __syncwarp();
    if (done) {   // the row's aligned interior by a bulk store, up to 3 floats at each end by lanes
      const int64_t off = pt * (int64_t)n;
      const int o = (int)(off & 3), h = (4 - o) & 3, e = (int)(((off + n) & ~(int64_t)3) - off);
      const float *const gr = gbuf + grp * PITCH + o;   // element i at gr[i]
      if (gl == 0) bulk_store(p.grad + off + h, smem_u32(gr + h), (uint32_t)(e - h) * 4u);
      if (gl < h) p.grad[off + gl] = gr[gl];
      if (gl < n - e) p.grad[off + e + gl] = gr[e + gl];
    }
    const float qs = group_sum<G>(qs0 + qs1);
    const float hsum = LINF ? group_max<G>(fmaxf(hs0, hs1)) : group_sum<G>(hs0 + hs1);
    if (done && gl == 0) {
      float phiv = (spec == 1) ? qs + p.gamma : qs - tt * ((L2 || ELL) ? sqrtf(hsum) : hsum) + p.gamma;
      if (spec == 2) phiv = gnan;
      p.phi[pt] = phiv;
      p.iters[pt] = wstatus;
    }
    // ---- refill: the next point of each finalized group --------------------------------------
    const int64_t claimed = p.claim ? (int64_t)__shfl_sync(0xffffffffu, wclaim, 0) + 2 * ngroups + (lane / G)
                                    : pnext + ngroups;   // no counter: static stride
    if (done) {
      pt = pnext;
      pnext = claimed;
      have = pt < M;
      if (!have) {
        waiting = false;
        spec = 0;
#pragma unroll
        for (int q = 0; q < NP; q++) d[q] = b[q] = splat2(0.f);
      }
    }
    refill(done && have);
    any_have = __any_sync(0xffffffffu, have);
  }
  if (gl == 0) bulk_wait_all();
  if (p.iter_total && gl == 0 && my_iters) atomicAdd(p.iter_total, (unsigned long long)my_iters);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem_slot), "r"(TMEM_COLS));
}

}  // namespace dtg
}  // namespace hopf
