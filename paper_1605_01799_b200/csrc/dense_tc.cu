// dense_tc.cu — tensor-core dense v-update (K3, v2): tcgen05.mma (kind::f16, TMEM accumulator)
// for n = 256 and H in {l1, wl1}, fused with the shrink / Bregman / stopping-test epilogue.
//
// Paper: (3.4a) for J = 1/2<x,Ax> is the quadratic prox v = M_lambda (x + lambda (d - b)),
// M_lambda = (A^{-1} + lambda I)^{-1}; (3.4b) shrink_1
// (P:239-247); (3.4c); stopping rule P:1595-1601.
//
// Layout (one CTA per SM, 32 points per CTA, 16 warps; MMA and epilogue alternate, thread 0
// issues the 96 MMAs of an iteration after the epilogue barrier):
//  * D^T = M_lambda U^T: the MMA M dimension is the coordinate (two M = 128 halves), N = the 32
//    points of the CTA, K = 256.  The fp32 accumulators D0 (coordinates 0-127) and D1
//    (128-255) live in TMEM columns [0,32) and [32,64).
//  * M_lambda stays resident in shared memory for the whole kernel: it is symmetric, so only the
//    blocks A11, A12, A22 are stored (A21 = A12^T is the same bytes read through an MN-major
//    descriptor), each as fp16 hi + lo of 2^s M_lambda (s fixed by the plan): 6 x 32 KB.
//  * U^T (32 points x 256) is the B operand, fp16 hi + lo, MN-major (points contiguous), 32 KB,
//    rewritten by the epilogue every iteration.
//  * 3 MMAs per K-step (Mh Uh + Mh Ul + Ml Uh) reproduce the fp32 product to ~2^-22 relative
//    (plain fp16/TF32 products stall the paper's 1e-8 test in a limit cycle).
//  * Epilogue thread (warp w of 16, lane l): coordinates c = 32 (w % 4) + l and c + 128 (a
//    float2), for the 8 points of group w / 4.  x, u (pre-shrink), v_prev of those 8 points stay
//    in registers; per-point sums (three test sums and the phi partial) are reduced with a
//    transposed butterfly per warp and across the 4 warps of the group through shared memory.
//  * phi at convergence uses g = A^{-1} v^k = U^k - lambda v^k (exact consequence of (3.4a)):
//      1/2<d, A^{-1} d> = <g, d - v/2> + 1/2<d - v, A^{-1}(d - v)>,
//    the last term <= lambda_max(A^{-1}) tol / 2 is dropped (reading R23).
//  * Points with t == 0, non-finite sums (invalid input, fp16 overflow) or no convergence within
//    max_iter are appended to a fix-up list that the exact FP32 SIMT kernel re-solves.
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
namespace tc {

constexpr int N_DIM = 256;
constexpr int NT = 32;                       // points per CTA
constexpr int EPI_WARPS = 16;
constexpr int THREADS = EPI_WARPS * 32;
constexpr int GROUPS = EPI_WARPS / 4;        // warp groups; group g owns points [PPG g, PPG g + PPG)
constexpr int PPG = NT / GROUPS;             // points per group (8)
constexpr int NCH = PPG / 8;                 // chunks of 8 points per thread
constexpr int BLK_BYTES = 128 * 128 * 2;     // one fp16 128x128 block
constexpr int SM_MLAM = 6 * BLK_BYTES;       // A11h, A12h, A22h, A11l, A12l, A22l
constexpr int SM_U = NT * N_DIM * 2;         // one of U hi / U lo
constexpr int OFF_UH = SM_MLAM;
constexpr int OFF_UL = SM_MLAM + SM_U;
constexpr int OFF_RED = OFF_UL + SM_U;       // [GROUPS][4 warps][PPG points][4 q] floats
constexpr int RED_BYTES = GROUPS * 4 * PPG * 4 * 4;
constexpr int OFF_CTRL = OFF_RED + RED_BYTES;
struct Ctrl {
  float t;
  int it;         // iterations completed
  int mode;       // 0 empty, 1 loading (x in flight; U column 0), 2 active
  int done;       // set by the finaliser this iteration: 1 converged (write grad)
  long long pt;   // global point index (mode 1, 2)
};
constexpr int OFF_MISC = OFF_CTRL + NT * (int)sizeof(Ctrl);
constexpr int SMEM_BYTES = OFF_MISC + 64;
static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB dynamic shared memory of a CTA");

// element (m, k) of a 128x128 K-major no-swizzle block (core matrix 8 rows x 16 bytes)
__host__ __device__ inline uint32_t a_off(int m, int k) {
  return (m >> 3) * 2048 + (k >> 3) * 128 + (m & 7) * 16 + (k & 7) * 2;
}
// element (point p, coordinate c) of U^T, MN-major no swizzle: 8 points contiguous (16 bytes)
__device__ inline uint32_t u_off(int p, int c) {
  return (c >> 3) * 512 + (p >> 3) * 128 + (c & 7) * 16 + (p & 7) * 2;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
  return d;                 // base offset 0, lbo mode 0, SWIZZLE_NONE
}
__device__ __forceinline__ uint32_t make_idesc(int a_mn_major) {
  uint32_t d = 0;
  d |= 1u << 4;                      // accumulate in F32
  d |= (uint32_t)a_mn_major << 15;   // A major (0 K, 1 MN); A, B formats F16 (0)
  d |= 1u << 16;                     // B (U^T) is MN-major
  d |= (uint32_t)(NT >> 3) << 17;    // N
  d |= (uint32_t)(128 >> 4) << 24;   // M
  return d;
}
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
               :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 "selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(phase));
  }
}
// 8 consecutive TMEM columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ float clampf(float u, float t) { return fminf(fmaxf(u, -t), t); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.f, -1.f), a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 clamp2(float2 u, float2 t) {
  return make_float2(clampf(u.x, t.x), clampf(u.y, t.y));
}

// split x into fp16 hi + lo (x ~ hi + lo to ~2^-22 relative)
__device__ __forceinline__ void split_h(float x, __half &hi, __half &lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn(x - __half2float(hi));
}

template <int HK>
__global__ void __launch_bounds__(THREADS, 1)
    hopf_dense_tc_kernel(const DenseParams p, const uint4 *__restrict__ mlam_blocks,
                         float mscale_inv, int *__restrict__ fix_count,
                         int *__restrict__ fix_list) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Ctrl *ctrl = reinterpret_cast<Ctrl *>(smem + OFF_CTRL);
  float *red = reinterpret_cast<float *>(smem + OFF_RED);
  uint64_t *mma_done = reinterpret_cast<uint64_t *>(smem + OFF_MISC);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(mma_done + 2);
  volatile int *busy_flag = reinterpret_cast<volatile int *>(mma_done + 3);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const float lam = p.lambda, tol = p.tol, ilam = 1.f / p.lambda;
  const int64_t stride = (int64_t)gridDim.x * NT;

  // ---- one-time setup: M_lambda blocks -> smem, barrier, TMEM ------------------------------
  for (int e = tid; e < SM_MLAM / 16; e += THREADS)
    reinterpret_cast<uint4 *>(smem)[e] = __ldg(mlam_blocks + e);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(tmem_slot)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (lane == 0) {
      mbar_init(mma_done, 1);
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sm0 = smem_u32(smem);

  // ---- the 96 MMAs of one iteration (thread 0) -------------------------------------------
  // Descriptors are formed once; consecutive K-steps only advance the start-address field
  // (bits [0,14), 16-byte units), so the issue loop is one add and one UTCHMMA per MMA.
  const uint32_t id_k = make_idesc(0), id_mn = make_idesc(1);
  const uint64_t a_seg[4] = {make_sdesc(sm0 + 0 * BLK_BYTES, 128, 2048),    // A11 (h 0, K 0-127)
                             make_sdesc(sm0 + 1 * BLK_BYTES, 128, 2048),    // A12 (h 0, K 128-255)
                             make_sdesc(sm0 + 1 * BLK_BYTES, 2048, 128),    // A21 = A12^T, MN-major
                             make_sdesc(sm0 + 2 * BLK_BYTES, 128, 2048)};   // A22
  const uint64_t lo_off = (uint64_t)(3 * BLK_BYTES) >> 4;                  // hi -> lo block
  const uint64_t b_h0 = make_sdesc(sm0 + OFF_UH, 512, 128), b_l0 = make_sdesc(sm0 + OFF_UL, 512, 128);
  auto issue_mmas = [&]() {
#pragma unroll
    for (int seg = 0; seg < 4; seg++) {
      const uint32_t dt = tmem + (uint32_t)((seg >> 1) * NT);   // D0 or D1 columns
      const uint32_t idesc = seg == 2 ? id_mn : id_k;
      const uint64_t a_step = seg == 2 ? (2 * 2048) >> 4 : 256 >> 4;
      uint64_t ah = a_seg[seg], al = a_seg[seg] + lo_off;
      uint64_t bh = b_h0 + (uint64_t)(((seg & 1) * 8 * 1024) >> 4), bl = b_l0 + (uint64_t)(((seg & 1) * 8 * 1024) >> 4);
#pragma unroll
      for (int k8 = 0; k8 < 8; k8++) {
        mma_f16(dt, ah, bh, idesc, ((seg & 1) | k8) ? 1u : 0u);   // Mh Uh
        mma_f16(dt, ah, bl, idesc, 1u);                            // Mh Ul
        mma_f16(dt, al, bh, idesc, 1u);                            // Ml Uh
        ah += a_step; al += a_step; bh += 1024 >> 4; bl += 1024 >> 4;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(mma_done)));
  };

  const int half = warp >> 2;                 // group: points [PPG half, PPG half + PPG)
  const int wq = warp & 3;                    // TMEM lane quarter
  const int c0 = 32 * wq + lane, c1 = c0 + 128;   // this thread's two coordinates
  const uint32_t t_lane = tmem + ((uint32_t)(32 * wq) << 16);
  float w0 = 1.f, w1 = 1.f;
  if (HK == HK_WL1) { w0 = __ldg(p.w + c0); w1 = __ldg(p.w + c1); }
  float2 xs[PPG], us[PPG], vs[PPG];   // per point (c0, c1): x, u (pre-shrink), v_prev

  // Slot life cycle (one thread of warp 0 per slot owns the control word):
  //   loading: the finaliser picked the slot's next point; every thread issues its two x loads
  //            into xs[] and the owner loads t, all in the shadow of the next MMA (the slot's U
  //            column is 0 for that MMA); the following epilogue initialises the state, writes
  //            U^1 = (1 + lambda) x and validates t (t <= 0 / non-finite -> fix-up list).
  //   active:  split Bregman iterations; converged -> grad/phi/iters; max_iter or non-finite
  //            sums -> fix-up list; either way the slot goes back to loading (or empty).
  float t_pending = 0.f;   // owner lane: t of the point being loaded
  auto zero_u = [&](int slot) {
    const __half z = __float2half_rn(0.f);
    *reinterpret_cast<__half *>(smem + OFF_UH + u_off(slot, c0)) = z;
    *reinterpret_cast<__half *>(smem + OFF_UL + u_off(slot, c0)) = z;
    *reinterpret_cast<__half *>(smem + OFF_UH + u_off(slot, c1)) = z;
    *reinterpret_cast<__half *>(smem + OFF_UL + u_off(slot, c1)) = z;
  };
  auto issue_loads = [&](int p16) {   // x of the slot's new point into registers (no wait)
    const long long pt = ctrl[PPG * half + p16].pt;
    const float *xr = p.X + pt * (int64_t)N_DIM;
    xs[p16] = make_float2(__ldg(xr + c0), __ldg(xr + c1));
  };

  // initial admission: slot s takes point blockIdx.x * NT + s
  if (tid < NT) {
    Ctrl c{};
    c.pt = (long long)blockIdx.x * NT + tid;
    c.mode = c.pt < p.M ? 1 : 0;
    c.it = 0; c.t = 0.f; c.done = 0;
    if (c.mode) t_pending = __ldg(p.t + c.pt);
    ctrl[tid] = c;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PPG; q++) {
    zero_u(PPG * half + q);
    xs[q] = make_float2(0.f, 0.f);
    us[q] = vs[q] = xs[q];
    if (ctrl[PPG * half + q].mode == 1) issue_loads(q);
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    issue_mmas();
  }

  uint32_t phase = 0;
  while (true) {
    mbar_wait(mma_done, phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- elementwise update, 8 points per chunk, packed FP32x2 over the coordinate pair ---
#pragma unroll
    for (int ch = 0; ch < NCH; ch++) {
      float va[8], vb[8];
      tmem_ld8(t_lane + (uint32_t)(PPG * half + 8 * ch), va);        // D0: coordinate c0
      tmem_ld8(t_lane + (uint32_t)(NT + PPG * half + 8 * ch), vb);   // D1: coordinate c1
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      float qv[32];   // [point j][quantity]: sd, sb, sv, phi partial
      uint32_t ph0[4], pl0[4], ph1[4], pl1[4];   // packed fp16 U^{k+1} for the 8 points
      const float2 msc = make_float2(mscale_inv, mscale_inv);
      const float2 lam2 = make_float2(lam, lam), nlam2 = make_float2(-lam, -lam);
#pragma unroll
      for (int jj = 0; jj < 4; jj++) {
        float2 Unj[2];
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int j = 2 * jj + e;
          const int p16 = 8 * ch + j, slot = PPG * half + p16;
          const float2 tm = *reinterpret_cast<const float2 *>(&ctrl[slot].t);   // t, it
          const int2 md = *reinterpret_cast<const int2 *>(&ctrl[slot].mode);    // mode, done
          const float tt = tm.x;
          const int mode = md.x, first = __float_as_int(tm.y) == 0;
          const float2 tau = make_float2(tt * w0 * ilam, tt * w1 * ilam);
          const float2 v = __fmul2_rn(make_float2(va[j], vb[j]), msc);
          float2 x = xs[p16];
          if (mode != 2) {   // loading (x has landed): v^0 = x; empty: zeros
            if (mode == 0) x = make_float2(0.f, 0.f);
            us[p16] = make_float2(0.f, 0.f);
            vs[p16] = x;
          }
          const float2 u = us[p16], vp = vs[p16];
          if (mode == 2) {
            // previous d, b (from u, or the initial d^0 = x, b^0 = 0)
            const float2 bo = first ? make_float2(0.f, 0.f) : clamp2(u, tau);
            const float2 dprev = first ? x : sub2(u, bo);
            const float2 un = add2(v, bo);                         // argument of (3.4b)
            const float2 bn = clamp2(un, tau);                     // b^k
            const float2 dn = sub2(un, bn);                        // d^k = shrink_1
            const float2 ed = sub2(dn, dprev);                     // d^k - d^{k-1}
            const float2 fd = sub2(dn, v);                         // d^k - v^k
            const float2 gd = sub2(v, vp);                         // v^k - v^{k-1}
            // phi partial: <x,d> - <A^{-1} v, d - v/2> - t w |d|, A^{-1} v = U^k - lambda v
            const float2 Uk = fma2(lam2, sub2(dprev, bo), x);
            const float2 gi = fma2(nlam2, v, Uk);
            const float2 hv = fma2(make_float2(-0.5f, -0.5f), v, dn);
            float2 q = __fmul2_rn(x, dn);
            q = sub2(q, __fmul2_rn(gi, hv));
            float ph = q.x + q.y;
            ph = fmaf(-tt, fmaf(w0, fabsf(dn.x), w1 * fabsf(dn.y)), ph);
            const float2 e2 = __fmul2_rn(ed, ed), f2 = __fmul2_rn(fd, fd), g2 = __fmul2_rn(gd, gd);
            qv[4 * j + 0] = e2.x + e2.y;
            qv[4 * j + 1] = f2.x + f2.y;
            qv[4 * j + 2] = g2.x + g2.y;
            qv[4 * j + 3] = ph;
            us[p16] = un;
            vs[p16] = v;
            Unj[e] = fma2(lam2, sub2(dn, bn), x);   // next operand U^{k+1} = x + lambda (d^k - b^k)
          } else {
            qv[4 * j + 0] = qv[4 * j + 1] = qv[4 * j + 2] = qv[4 * j + 3] = 0.f;
            Unj[e] = fma2(lam2, x, x);              // U^1 = (1 + lambda) x of a loaded point
          }
        }
        // fp16 hi/lo of the pair of points (jj, jj+1) for each coordinate: packed conversions
        const __half2 h0 = __floats2half2_rn(Unj[0].x, Unj[1].x);   // coordinate c0
        const __half2 h1 = __floats2half2_rn(Unj[0].y, Unj[1].y);   // coordinate c1
        const float2 hb0 = __half22float2(h0), hb1 = __half22float2(h1);
        const __half2 l0 = __floats2half2_rn(Unj[0].x - hb0.x, Unj[1].x - hb0.y);
        const __half2 l1 = __floats2half2_rn(Unj[0].y - hb1.x, Unj[1].y - hb1.y);
        ph0[jj] = *reinterpret_cast<const uint32_t *>(&h0);
        pl0[jj] = *reinterpret_cast<const uint32_t *>(&l0);
        ph1[jj] = *reinterpret_cast<const uint32_t *>(&h1);
        pl1[jj] = *reinterpret_cast<const uint32_t *>(&l1);
      }
      // 8 points are contiguous in the MN-major U^T layout: one 16-byte store per (c, hi/lo)
      {
        const int pg = PPG * half + 8 * ch;
        *reinterpret_cast<uint4 *>(smem + OFF_UH + u_off(pg, c0)) = make_uint4(ph0[0], ph0[1], ph0[2], ph0[3]);
        *reinterpret_cast<uint4 *>(smem + OFF_UL + u_off(pg, c0)) = make_uint4(pl0[0], pl0[1], pl0[2], pl0[3]);
        *reinterpret_cast<uint4 *>(smem + OFF_UH + u_off(pg, c1)) = make_uint4(ph1[0], ph1[1], ph1[2], ph1[3]);
        *reinterpret_cast<uint4 *>(smem + OFF_UL + u_off(pg, c1)) = make_uint4(pl1[0], pl1[1], pl1[2], pl1[3]);
      }
      // transposed butterfly: afterwards lane l holds the warp total of qv index l = 4 j + q
#pragma unroll
      for (int lev = 16; lev >= 1; lev >>= 1) {
        const bool up = lane & lev;
#pragma unroll
        for (int i = 0; i < lev; i++) {
          const float send = up ? qv[i] : qv[i + lev];
          const float keep = up ? qv[i + lev] : qv[i];
          qv[i] = keep + __shfl_xor_sync(0xffffffffu, send, lev);
        }
      }
      red[((half * 4 + wq) * PPG + (8 * ch + (lane >> 2))) * 4 + (lane & 3)] = qv[0];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    // ---- finaliser: one thread per point slot (warp 0) ------------------------------------
    if (tid < NT) {
      const int slot = tid, hf = slot / PPG, p16 = slot % PPG;
      Ctrl c = ctrl[slot];
      c.done = 0;
      bool reload = false;
      if (c.mode == 2) {
        float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int w4 = 0; w4 < 4; w4++)
#pragma unroll
          for (int qq = 0; qq < 4; qq++) s4[qq] += red[((hf * 4 + w4) * PPG + p16) * 4 + qq];
        c.it += 1;
        const bool finite = fabsf(s4[0] + s4[1] + s4[2] + s4[3]) <= 3.402823466e38f;
        const bool conv = finite && s4[0] <= tol && s4[1] <= tol && s4[2] <= tol;
        if (conv) {
          p.phi[c.pt] = s4[3] + p.gamma;
          p.iters[c.pt] = c.it;
          c.done = 1;
          reload = true;
        } else if (!finite || c.it >= p.max_iter) {
          fix_list[atomicAdd(fix_count, 1)] = (int)c.pt;   // exact FP32 re-solve
          reload = true;
        }
      } else if (c.mode == 1) {
        // the point's x landed in this epilogue (its state and U^1 are set); validate t
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
        if (c.mode) t_pending = __ldg(p.t + c.pt);   // consumed by the next finaliser
      }
      ctrl[slot] = c;
      const unsigned act = __ballot_sync(0xffffffffu, c.mode != 0);
      if (tid == 0) *busy_flag = act != 0u;
    }
    __syncthreads();
    // ---- converged slots: grad := d^k = u - clamp(u); reloads: x in flight, U column 0 ----
#pragma unroll
    for (int q = 0; q < PPG; q++) {
      const int slot = PPG * half + q;
      const Ctrl c = ctrl[slot];
      if (c.done == 1) {
        const float ta = c.t * w0 * ilam, tb = c.t * w1 * ilam;
        float *g = p.grad + (c.pt - stride) * (int64_t)N_DIM;   // the finaliser advanced pt
        g[c0] = us[q].x - clampf(us[q].x, ta);
        g[c1] = us[q].y - clampf(us[q].y, tb);
      }
    }
#pragma unroll
    for (int q = 0; q < PPG; q++) {
      const int slot = PPG * half + q;
      if (ctrl[slot].mode == 1) { zero_u(slot); issue_loads(q); }
      else if (ctrl[slot].mode == 0) zero_u(slot);
    }
    if (!*busy_flag) break;
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      issue_mmas();
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(64));
}

}  // namespace tc

// host side -----------------------------------------------------------------------------------
// M_lambda blocks in smem order: fp16 hi/lo of 2^s M (A11, A12, A22), K-major no-swizzle.
int dense_tc_prepare(int n, const double *Ml, void **blocks_dev, float *mscale_inv) {
  if (n != tc::N_DIM) return HOPF_EUNSUPPORTED;
  double mx = 0.0;
  for (int i = 0; i < n * n; i++) mx = fmax(mx, fabs(Ml[i]));
  int s = 0;
  while (mx * ldexp(1.0, s + 1) < 16384.0 && s < 60) s++;
  const double sc = ldexp(1.0, s);
  std::vector<__half> hb(6 * 128 * 128);
  const int blk_r[3] = {0, 0, 128}, blk_c[3] = {0, 128, 128};
  for (int b = 0; b < 3; b++)
    for (int m = 0; m < 128; m++)
      for (int k = 0; k < 128; k++) {
        const double v = Ml[(size_t)(blk_r[b] + m) * n + blk_c[b] + k] * sc;
        const __half hi = __float2half_rn((float)v);
        const __half lo = __float2half_rn((float)(v - (double)__half2float(hi)));
        const uint32_t off = tc::a_off(m, k) / 2;
        hb[(size_t)b * 128 * 128 + off] = hi;
        hb[(size_t)(b + 3) * 128 * 128 + off] = lo;
      }
  if (cudaMalloc(blocks_dev, hb.size() * sizeof(__half)) != cudaSuccess)
    return set_error(HOPF_ECUDA, "cudaMalloc for tensor-core operands failed");
  cudaMemcpy(*blocks_dev, hb.data(), hb.size() * sizeof(__half), cudaMemcpyHostToDevice);
  *mscale_inv = (float)ldexp(1.0, -s);
  return HOPF_OK;
}

int dense_tc_launch(const DenseParams &p, int hk, const void *blocks, float mscale_inv,
                    int *fix_count, int *fix_list, cudaStream_t stream) {
  auto fn = hk == HK_WL1 ? tc::hopf_dense_tc_kernel<HK_WL1> : tc::hopf_dense_tc_kernel<HK_L1>;
  static bool attr_set[2] = {false, false};
  if (!attr_set[hk == HK_WL1]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_BYTES);
    attr_set[hk == HK_WL1] = true;
  }
  int64_t blocks_n = num_sms();
  const int64_t need = (p.M + tc::NT - 1) / tc::NT;
  if (blocks_n > need) blocks_n = need;
  if (blocks_n < 1) blocks_n = 1;
  fn<<<(unsigned)blocks_n, tc::THREADS, tc::SMEM_BYTES, stream>>>(
      p, reinterpret_cast<const uint4 *>(blocks), mscale_inv, fix_count, fix_list);
  g_launches += 1;
  return check_launch("hopf_dense_tc_kernel");
}

}  // namespace hopf
