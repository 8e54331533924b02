// dense_tc2.cu — tensor-core dense v-update (K3, v3): CTA pairs (cta_group::2).
//
// Paper: (3.4a) for J = 1/2<x,Ax> is the quadratic prox v = M_lambda (x + lambda (d - b)),
// M_lambda = (A^{-1} + lambda I)^{-1}; (3.4b) shrink_1
// (P:239-247); (3.4c); stopping rule P:1595-1601.  n = 256, H in {l1, wl1}.
//
// Why pairs: a kind::f16 M=128 MMA reads its 4 KB A operand per K=16 step at ~128 B/clk
// (profiles/r01/tcgen05_mma_rate.txt): below N=128 columns the MMA is operand-bandwidth bound.
// Full rate therefore needs >= 128 x 256 x 16 per instruction, i.e. 128 points per MMA, but a
// point carries 2 KB of iteration state (u, v_prev fp32) + 1 KB x + 1 KB operand — 128 points do
// not fit one SM next to M_lambda.  A cta_group::2 MMA with M = 128 splits the points over the
// two SMs of a TPC (64 each) and N = 256 (the coordinates) over their shared memories:
//   D[128 points x 256 coords] = U[128 x 256] . M_lambda^T, each SM receiving its 64 points'
//   rows in TMEM in the "2x2" layout (lanes 0-63: coordinates 0-127, lanes 64-127: 128-255).
// Measured 64 cycles per 128x256x16 pair-MMA = 4096 MAC/clk/SM (tcgen05_2sm_probe.txt).
//
// Per CTA (16 warps, 64 point slots):
//  * smem: U (A operand, this CTA's 64 points, fp16 hi + lo, K-major) 64 KB; M_lambda rows
//    [128 r, 128 r + 128) (B operand, fp16 hi + lo of 2^s M_lambda, K-major) 128 KB.
//  * thread (warp w, lane l): TMEM lane quarter q = w % 4, column chunk j = w / 4: point
//    p = 32 (q & 1) + l, coordinates c in [128 (q >> 1) + 32 j, +32).  x, u (pre-shrink) and
//    v_prev of those 32 coordinates live in registers; per-point sums are thread-local over 32
//    coordinates, then 8 partials per point are combined through shared memory.
//  * 3 MMAs per K-step (Mh Uh + Mh Ul + Ml Uh) for ~2^-22 relative accuracy (see dense_tc.cu).
//  * The leader CTA (rank 0) issues the 48 MMAs of an iteration once both CTAs have written
//    their U (mbarrier epi_done, count 2, the follower arrives remotely); tcgen05.commit
//    multicasts completion to both CTAs' mma_done barriers.
//  * phi: reading R23 (g = A^{-1} v^k = U^k - lambda v^k); t == 0, invalid points, fp16
//    overflow and max_iter go to the fix-up list re-solved by the FP32 SIMT kernel.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/hopf.h"
#include "common.cuh"
#include "dense_kernel.cuh"
#include "diag_kernel.cuh"  // HK_* constants

namespace hopf {
namespace tc2 {

constexpr int N_DIM = 256;
constexpr int PTS = 64;                      // point slots per CTA (128 per pair)
constexpr int WARPS = 16;
constexpr int THREADS = WARPS * 32;
constexpr int CPT = 32;                      // coordinates per thread
constexpr int OFF_UH = 0;                    // U hi: 64 rows x 256 fp16 (32 KB)
constexpr int OFF_UL = 32768;                // U lo
constexpr int OFF_BH = 65536;                // M_lambda rows hi: 128 x 256 fp16 (64 KB)
constexpr int OFF_BL = 131072;               // M_lambda rows lo
constexpr int OFF_RED = 196608;              // [64 points][8 parts][4 q] floats (8 KB)
constexpr int OFF_CTRL = OFF_RED + PTS * 8 * 4 * 4;
struct Ctrl {
  float t;
  int it;
  int mode;   // 0 empty, 1 loading, 2 active
  int done;   // 1: converged this iteration (write grad)
  long long pt;
};
constexpr int OFF_MISC = OFF_CTRL + PTS * (int)sizeof(Ctrl);
// misc: [0] mma_done (8 B), [8] epi_done (8 B, leader), [16] tmem base, [20] busy[0], [24] busy[1],
//       [28] terminate
constexpr int SMEM_BYTES = OFF_MISC + 64;
static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB dynamic shared memory of a CTA");

// element (row r, k) of a K-major no-swizzle operand with 256 K (core matrix 8 rows x 16 B)
__host__ __device__ inline uint32_t kmaj(int r, int k) {
  return (r >> 3) * 4096 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count));
}
// Poll with CTA-scope acquire (a cluster-scope try_wait makes ptxas emit an L1 invalidation,
// CCTL.IVALL, on every poll), then one cluster-scope acquire fence for the remote stores
// (busy / terminate flags) that were released before the remote arrive.
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 "selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  }
  asm volatile("fence.acq_rel.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mma2_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}"
               :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ float clampf(float u, float t) { return fminf(fmaxf(u, -t), t); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.f, -1.f), a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 clamp2(float2 u, float2 t) {
  return make_float2(clampf(u.x, t.x), clampf(u.y, t.y));
}

template <int HK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    hopf_dense_tc2_kernel(const DenseParams p, const uint4 *__restrict__ mlam_rows,
                          float mscale_inv, int *__restrict__ fix_count,
                          int *__restrict__ fix_list) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Ctrl *ctrl = reinterpret_cast<Ctrl *>(smem + OFF_CTRL);
  float *red = reinterpret_cast<float *>(smem + OFF_RED);
  uint8_t *misc = smem + OFF_MISC;
  volatile uint32_t *tmem_slot = reinterpret_cast<volatile uint32_t *>(misc + 16);
  volatile int *busy = reinterpret_cast<volatile int *>(misc + 20);     // [2], leader's copy used
  volatile int *terminate = reinterpret_cast<volatile int *>(misc + 28);
  const uint32_t mma_done = smem_u32(misc), epi_done = smem_u32(misc + 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const float lam = p.lambda, tol = p.tol, ilam = 1.f / p.lambda;
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int64_t stride = npairs * 2 * PTS;

  // ---- setup: this CTA's half of M_lambda (B operand) -> smem; barriers; TMEM (both CTAs) ---
  for (int e = tid; e < 131072 / 16; e += THREADS)
    reinterpret_cast<uint4 *>(smem + OFF_BH)[e] = __ldg(mlam_rows + (size_t)rank * 8192 + e);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32((const void *)tmem_slot)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(mma_done, 1);
    mbar_init(epi_done, 2);
    busy[0] = busy[1] = 1;
    *terminate = 0;
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sm0 = smem_u32(smem);

  // ---- the 48 MMAs of one iteration (leader CTA, thread 0) --------------------------------
  const uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint64_t a_h0 = make_sdesc(sm0 + OFF_UH, 128, 4096), a_l0 = make_sdesc(sm0 + OFF_UL, 128, 4096);
  const uint64_t b_h0 = make_sdesc(sm0 + OFF_BH, 128, 4096), b_l0 = make_sdesc(sm0 + OFF_BL, 128, 4096);
  auto issue_mmas = [&]() {
    uint64_t ah = a_h0, al = a_l0, bh = b_h0, bl = b_l0;
#pragma unroll
    for (int ks = 0; ks < 16; ks++) {
      mma2_f16(tmem, ah, bh, idesc, ks > 0 ? 1u : 0u);   // Uh Mh
      mma2_f16(tmem, al, bh, idesc, 1u);                 // Ul Mh
      mma2_f16(tmem, ah, bl, idesc, 1u);                 // Uh Ml
      ah += 256 >> 4; al += 256 >> 4; bh += 256 >> 4; bl += 256 >> 4;
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(mma_done), "h"((uint16_t)3));
  };

  // ---- thread geometry ---------------------------------------------------------------------
  const int q = warp & 3, j = warp >> 2;
  const int pl = 32 * (q & 1) + lane;                 // local point slot 0..63
  const int cb = 128 * (q >> 1) + 32 * j;             // first coordinate of this thread
  const int part = (q >> 1) * 4 + j;                  // 0..7: which partial of the point
  const uint32_t t_addr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(32 * j);
  float2 wv[CPT / 2];
#pragma unroll
  for (int i = 0; i < CPT / 2; i++)
    wv[i] = HK == HK_WL1 ? make_float2(__ldg(p.w + cb + 2 * i), __ldg(p.w + cb + 2 * i + 1))
                         : make_float2(1.f, 1.f);
  float2 xs[CPT / 2], us[CPT / 2], vs[CPT / 2];   // x, u (pre-shrink), v_prev of 32 coordinates

  auto store_u8 = [&](int g, const float2 (&U)[4]) {   // coordinates cb + 8g .. +8: hi + lo
    {
      uint32_t hw[4], lw[4];
#pragma unroll
      for (int h = 0; h < 4; h++) {
        const float2 u2 = U[h];
        const __half2 hi = __float22half2_rn(u2);
        const float2 hb = __half22float2(hi);
        const __half2 lo = __floats2half2_rn(u2.x - hb.x, u2.y - hb.y);
        hw[h] = *reinterpret_cast<const uint32_t *>(&hi);
        lw[h] = *reinterpret_cast<const uint32_t *>(&lo);
      }
      const uint32_t off = kmaj(pl, cb + 8 * g);
      *reinterpret_cast<uint4 *>(smem + OFF_UH + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4 *>(smem + OFF_UL + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
  };
  auto store_u_zero = [&]() {
    const float2 z[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
#pragma unroll
    for (int g = 0; g < 4; g++) store_u8(g, z);
  };
  auto load_x = [&]() {   // x of the slot's (new) point: 32 coordinates, 8 x 16-byte loads
    const long long pt = ctrl[pl].pt;
    const float4 *xr = reinterpret_cast<const float4 *>(p.X + pt * (int64_t)N_DIM + cb);
#pragma unroll
    for (int g = 0; g < CPT / 4; g++) {
      const float4 v4 = __ldg(xr + g);
      xs[2 * g] = make_float2(v4.x, v4.y);
      xs[2 * g + 1] = make_float2(v4.z, v4.w);
    }
  };

  // initial admission: pair slot g = 64 rank + s takes point pair * 128 + g (+ stride ...)
  float t_pending = 0.f;   // owner thread (tid < 64) of slot tid: t of the point being loaded
  if (tid < PTS) {
    Ctrl c{};
    c.pt = pair * 2 * PTS + (int64_t)rank * PTS + tid;
    c.mode = c.pt < p.M ? 1 : 0;
    c.it = 0; c.t = 0.f; c.done = 0;
    if (c.mode) t_pending = __ldg(p.t + c.pt);
    ctrl[tid] = c;
  }
  __syncthreads();
  {
#pragma unroll
    for (int i = 0; i < CPT / 2; i++) xs[i] = us[i] = vs[i] = make_float2(0.f, 0.f);
    store_u_zero();
    if (ctrl[pl].mode == 1) load_x();
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  uint32_t epi_phase = 0, mma_phase = 0;
  auto epilogue_done = [&](int my_busy) {   // after __syncthreads: tell the leader
    if (tid == 0) {
      if (rank == 0) {
        busy[0] = my_busy;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(epi_done) : "memory");
      } else {
        st_cluster_u32(mapa(smem_u32((const void *)(busy + 1)), 0), (uint32_t)my_busy);
        mbar_arrive_remote(mapa(epi_done, 0));
      }
    }
  };
  auto leader_step = [&]() {   // leader thread 0: wait for both epilogues, then MMA or stop
    if (rank == 0 && tid == 0) {
      mbar_wait_cluster(epi_done, epi_phase);
      const int any = busy[0] | busy[1];
      if (any) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        issue_mmas();
      } else {   // both CTAs are out of points: wake everybody with the terminate flag
        *terminate = 1;
        st_cluster_u32(mapa(smem_u32((const void *)terminate), 1), 1u);
        asm volatile("mbarrier.arrive.release.cluster.shared::cta.b64 _, [%0];" :: "r"(mma_done) : "memory");
        mbar_arrive_remote(mapa(mma_done, 1));
      }
    }
    epi_phase ^= 1;
  };
  epilogue_done(1);
  leader_step();

  while (true) {
    mbar_wait_cluster(mma_done, mma_phase);
    mma_phase ^= 1;
    if (*terminate) break;
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- elementwise update over this thread's 32 coordinates of point pl --------------------
    const Ctrl cc = ctrl[pl];
    const int mode = cc.mode, first = cc.it == 0;
    const float tt = cc.t;
    float s_sd = 0.f, s_sb = 0.f, s_sv = 0.f, s_ph = 0.f;
#pragma unroll
    for (int h16 = 0; h16 < 2; h16++) {
      float2 Un[8];
      float va[16];
      tmem_ld16(t_addr + (uint32_t)(16 * h16), va);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int i2 = 0; i2 < 8; i2++) {
        const int i = 8 * h16 + i2;   // coordinate pair index 0..15
        const float2 tau = make_float2(tt * wv[i].x * ilam, tt * wv[i].y * ilam);
        const float2 v = make_float2(va[2 * i2] * mscale_inv, va[2 * i2 + 1] * mscale_inv);
        float2 x = xs[i];
        if (mode != 2) {
          if (mode == 0) x = make_float2(0.f, 0.f);
          us[i] = make_float2(0.f, 0.f);
          vs[i] = x;
          Un[i2] = fma2(make_float2(lam, lam), x, x);   // U^1 = (1 + lambda) x
          continue;
        }
        const float2 u = us[i], vp = vs[i];
        const float2 bo = first ? make_float2(0.f, 0.f) : clamp2(u, tau);
        const float2 dprev = first ? x : sub2(u, bo);
        const float2 un = add2(v, bo);                   // argument of (3.4b)
        const float2 bn = clamp2(un, tau);               // b^k
        const float2 dn = sub2(un, bn);                  // d^k = shrink_1
        const float2 ed = sub2(dn, dprev);               // d^k - d^{k-1}
        const float2 fd = sub2(dn, v);                   // d^k - v^k
        const float2 gd = sub2(v, vp);                   // v^k - v^{k-1}
        s_sd = fmaf(ed.x, ed.x, fmaf(ed.y, ed.y, s_sd));
        s_sb = fmaf(fd.x, fd.x, fmaf(fd.y, fd.y, s_sb));
        s_sv = fmaf(gd.x, gd.x, fmaf(gd.y, gd.y, s_sv));
        // phi partial: <x,d> - <A^{-1} v, d - v/2> - t w |d|, A^{-1} v = U^k - lambda v
        const float2 Uk = fma2(make_float2(lam, lam), sub2(dprev, bo), x);
        const float2 gi = fma2(make_float2(-lam, -lam), v, Uk);
        const float2 hv = fma2(make_float2(-0.5f, -0.5f), v, dn);
        const float2 qq = sub2(__fmul2_rn(x, dn), __fmul2_rn(gi, hv));
        s_ph += qq.x + qq.y;
        s_ph = fmaf(-tt, fmaf(wv[i].x, fabsf(dn.x), wv[i].y * fabsf(dn.y)), s_ph);
        us[i] = un;
        vs[i] = v;
        Un[i2] = fma2(make_float2(lam, lam), sub2(dn, bn), x);   // U^{k+1} = x + lambda (d - b)
      }
      const float2 U0[4] = {Un[0], Un[1], Un[2], Un[3]}, U1[4] = {Un[4], Un[5], Un[6], Un[7]};
      store_u8(2 * h16, U0);
      store_u8(2 * h16 + 1, U1);
    }
    *reinterpret_cast<float4 *>(red + (pl * 8 + part) * 4) = make_float4(s_sd, s_sb, s_sv, s_ph);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    // ---- finaliser: one thread per point slot ----------------------------------------------
    if (tid < PTS) {
      Ctrl c = ctrl[tid];
      c.done = 0;
      bool reload = false;
      if (c.mode == 2) {
        float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const float4 r4 = *reinterpret_cast<const float4 *>(red + (tid * 8 + k) * 4);
          s4[0] += r4.x; s4[1] += r4.y; s4[2] += r4.z; s4[3] += r4.w;
        }
        c.it += 1;
        const bool finite = fabsf(s4[0] + s4[1] + s4[2] + s4[3]) <= 3.402823466e38f;
        const bool conv = finite && s4[0] <= tol && s4[1] <= tol && s4[2] <= tol;
        if (conv) {
          p.phi[c.pt] = s4[3] + p.gamma;
          p.iters[c.pt] = c.it;
          c.done = 1;
          reload = true;
        } else if (!finite || c.it >= p.max_iter) {
          fix_list[atomicAdd(fix_count, 1)] = (int)c.pt;
          reload = true;
        }
      } else if (c.mode == 1) {
        if (t_pending > 0.f && t_pending <= 3.402823466e38f) {
          c.t = t_pending; c.it = 0; c.mode = 2;
        } else {
          fix_list[atomicAdd(fix_count, 1)] = (int)c.pt;   // t == 0, t < 0, non-finite t
          reload = true;
        }
      }
      if (reload) {
        c.pt += stride;
        c.mode = c.pt < p.M ? 1 : 0;
        c.it = 0;
        if (c.mode) t_pending = __ldg(p.t + c.pt);
      }
      ctrl[tid] = c;
    }
    __syncthreads();
    // ---- converged: grad := d = u - clamp(u); loading slots: x loads, U row zero -------------
    const Ctrl c2 = ctrl[pl];
    if (c2.done == 1) {
      float4 *g4 = reinterpret_cast<float4 *>(p.grad + (c2.pt - stride) * (int64_t)N_DIM + cb);
#pragma unroll
      for (int g = 0; g < CPT / 4; g++) {
        float4 o;
        const float2 a0 = us[2 * g], a1 = us[2 * g + 1];
        const float2 t0 = make_float2(c2.t * wv[2 * g].x * ilam, c2.t * wv[2 * g].y * ilam);
        const float2 t1 = make_float2(c2.t * wv[2 * g + 1].x * ilam, c2.t * wv[2 * g + 1].y * ilam);
        o.x = a0.x - clampf(a0.x, t0.x); o.y = a0.y - clampf(a0.y, t0.y);
        o.z = a1.x - clampf(a1.x, t1.x); o.w = a1.y - clampf(a1.y, t1.y);
        g4[g] = o;
      }
    }
    if (c2.mode != 2) {
      store_u_zero();
      if (c2.mode == 1) load_x();
    }
    const int my_busy = __syncthreads_or(tid < PTS && ctrl[tid].mode != 0);
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    epilogue_done(my_busy);
    leader_step();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(128));
}

}  // namespace tc2

// M_lambda rows for the pair: rank r holds rows [128 r, 128 r + 128) of 2^s M_lambda as fp16
// hi (64 KB) then lo (64 KB), K-major no-swizzle; layout [rank][hi|lo][kmaj(row, k)].
int dense_tc2_prepare(int n, const double *Ml, void **rows_dev, float *mscale_inv) {
  if (n != tc2::N_DIM) return HOPF_EUNSUPPORTED;
  double mx = 0.0;
  for (int i = 0; i < n * n; i++) mx = fmax(mx, fabs(Ml[i]));
  int s = 0;
  while (mx * ldexp(1.0, s + 1) < 16384.0 && s < 60) s++;
  const double sc = ldexp(1.0, s);
  std::vector<__half> hb(2 * 2 * 128 * 256);
  for (int r = 0; r < 2; r++)
    for (int row = 0; row < 128; row++)
      for (int k = 0; k < 256; k++) {
        const double v = Ml[(size_t)(128 * r + row) * n + k] * sc;
        const __half hi = __float2half_rn((float)v);
        const __half lo = __float2half_rn((float)(v - (double)__half2float(hi)));
        const size_t base = (size_t)r * 2 * 128 * 256;
        hb[base + tc2::kmaj(row, k) / 2] = hi;
        hb[base + 128 * 256 + tc2::kmaj(row, k) / 2] = lo;
      }
  if (cudaMalloc(rows_dev, hb.size() * sizeof(__half)) != cudaSuccess)
    return set_error(HOPF_ECUDA, "cudaMalloc for tensor-core operands failed");
  cudaMemcpy(*rows_dev, hb.data(), hb.size() * sizeof(__half), cudaMemcpyHostToDevice);
  *mscale_inv = (float)ldexp(1.0, -s);
  return HOPF_OK;
}

int dense_tc2_launch(const DenseParams &p, int hk, const void *rows, float mscale_inv,
                     int *fix_count, int *fix_list, cudaStream_t stream) {
  auto fn = hk == HK_WL1 ? tc2::hopf_dense_tc2_kernel<HK_WL1> : tc2::hopf_dense_tc2_kernel<HK_L1>;
  static bool attr_set[2] = {false, false};
  if (!attr_set[hk == HK_WL1]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, tc2::SMEM_BYTES);
    attr_set[hk == HK_WL1] = true;
  }
  int64_t pairs = num_sms() / 2;
  const int64_t need = (p.M + 2 * tc2::PTS - 1) / (2 * tc2::PTS);
  if (pairs > need) pairs = need;
  if (pairs < 1) pairs = 1;
  fn<<<(unsigned)(2 * pairs), tc2::THREADS, tc2::SMEM_BYTES, stream>>>(
      p, reinterpret_cast<const uint4 *>(rows), mscale_inv, fix_count, fix_list);
  g_launches += 1;
  return check_launch("hopf_dense_tc2_kernel");
}

}  // namespace hopf
