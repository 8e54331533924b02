// dense_tc3.cu — tensor-core dense v-update (K3, v4): CTA pairs with the MMA of round r+1
// pipelined against the epilogue of round r.
//
// Paper: (3.4a) for J = 1/2<x,Ax> is the quadratic prox v = M_lambda (x + lambda (d - b)),
// M_lambda = (A^{-1} + lambda I)^{-1}; (3.4b) shrink_1
// (P:239-247); (3.4c); stopping rule P:1595-1601.  n = 256, H in {l1, wl1}.
//
// What v4 changes against v3 (dense_tc2.cu); every choice below was measured (profiles/r01,
// tools/tcgen05_probe/*):
//  * a pair-MMA sequence of one iteration (48 x cta_group::2 kind::f16, M=128, N=256, K=16) runs
//    at 64 cycles per instruction, i.e. 3072 cycles per round for 128 points; v3 spent ~18000
//    cycles per round because MMA, epilogue, per-slot finalisation and the global reload of
//    finished slots ran one after the other.
//  * D is triple-buffered in TMEM (3 x 128 columns): MMA r+1 accumulates into D[(r+1) % 3] while
//    the epilogue of round r reads v^k from D[r % 3] and v^{k-1} from D[(r-1) % 3] (the previous
//    accumulator doubles as v_prev); x sits in the last 128 TMEM columns; only u stays in
//    registers (b = clamp(u), d = u - b are recomputed).
//  * The contraction index is permuted (K' = pi(c)) so that stage s (0..3) of every epilogue
//    thread completes the K-block [64 s, 64 s + 64): the MMA thread issues the 12 MMAs of that
//    block as soon as all 32 epilogue warps of the pair have written it (mbarrier stage_ready[s]),
//    i.e. MMA r+1 chases the epilogue of round r stage by stage.
//  * A dedicated MMA warp (one thread issues: a tcgen05.mma issue blocks its thread ~200 cycles,
//    and an elect.sync issue by a converged warp ran the round skeleton 2.5-4x slower) in a fifth
//    warpgroup; setmaxnreg gives the epilogue 112 registers and the MMA warpgroup 32.
//  * Per-slot decisions are taken redundantly by the 8 threads that share a point (they read the
//    same 8 partial sums), so the only per-round CTA-level sync is the partial-sum mbarrier; a
//    converged point outputs grad and phi in the following round (using v^{k+1}, reading R23)
//    and its slot's next x is loaded at the end of that round (its t one lifetime earlier).
//  * Remote mbarrier arrives use the default .release.cta semantics (.release.cluster compiled
//    to MEMBAR.ALL.GPU + ERRBAR and waited for the warp's global stores on every stage).
//
// Thread geometry (16 epilogue warps per CTA; warp 16 of the leader CTA issues the MMAs):
//   warp w < 16: TMEM lane quarter q = w & 3, column group j = w >> 2; point slot
//   pl = 32 (q & 1) + lane, coordinates c = 128 (q >> 1) + 32 j + [0, 32) ("2x2" layout of the
//   M = 128 pair MMA, profiles/r01/tcgen05_2sm_probe.txt); stage s handles c0 + 8 s .. + 8.
//   pi(c) = 64 s + 32 h + 8 j + i for c = 128 h + 32 j + 8 s + i.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/hopf.h"
#include "common.cuh"
#include "dense_kernel.cuh"
#include "diag_kernel.cuh"  // HK_* constants

namespace hopf {
namespace tc3 {

#ifdef HOPF_TC3_TRACE
// timing-only build (tools/tc3_trace.py): clock64 stamps of rounds [TR0, TR0 + TRN) in CTA 0
constexpr int TR0 = 200, TRN = 16, TRW = 40;
__device__ long long g_trace[TRN][TRW];
#define TC3_STAMP(r, k) do { if (blockIdx.x == 0 && (r) >= TR0 && (r) < TR0 + TRN) g_trace[(r) - TR0][(k)] = clock64(); } while (0)
#else
#define TC3_STAMP(r, k) do { } while (0)
#endif

constexpr int N_DIM = 256;
constexpr int PTS = 64;                  // point slots per CTA (128 per pair)
constexpr int EPI_WARPS = 16;
constexpr int EPI_THREADS = EPI_WARPS * 32;
// + one warpgroup whose first warp issues the MMAs (a lone 17th warp caps everyone at 96
// registers and measured 8 % slower than setmaxnreg 112/32)
constexpr int THREADS = EPI_THREADS + 128;
// setmaxnreg moves registers inside the CTA's own allocation (640 threads x 96 at launch):
// 16 warps x 112 + 4 warps x 32 = 20 warps x 96 (asking for more never returns)
constexpr int EPI_REGS = 112, MMA_REGS = 32;
static_assert(EPI_WARPS * EPI_REGS + 4 * MMA_REGS <= (EPI_WARPS + 4) * 96, "setmaxnreg budget");
constexpr int OFF_UH = 0;                // U hi: 64 rows x 256 fp16, K-major (32 KB)
constexpr int OFF_UL = 32768;            // U lo
constexpr int OFF_BH = 65536;            // M_lambda rows hi: 128 x 256 fp16 (64 KB)
constexpr int OFF_BL = 131072;           // M_lambda rows lo
constexpr int OFF_RED = 196608;          // [2][8 parts][64 slots] float4 (16 KB)
constexpr int OFF_W = OFF_RED + 2 * PTS * 8 * 16;   // w[256] (wl1)
constexpr int OFF_BAR = OFF_W + N_DIM * 4;
// bars: [0] mma_done, [8] term, [16..48) stage_ready[4], [48] busy[2] (int), [56] tmem base,
//       [64] red_ready (slots 0-31), [72] red_ready (slots 32-63), [80] fin (leader)
constexpr int SMEM_BYTES = OFF_BAR + 88;
static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB dynamic shared memory of a CTA");

// slot states: START = first round of a point whose x is already in ds (loaded at the end of the
// previous FINISH round); START_LD = the same, x loaded now (first point, non-converged refill)
enum { M_EMPTY = 0, M_START = 1, M_ACTIVE = 2, M_FINISH = 3, M_START_LD = 4 };

__host__ __device__ inline uint32_t kmaj(int r, int k) {
  return (r >> 3) * 4096 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}
// coordinate c -> permuted contraction index K'
__host__ __device__ inline int kperm(int c) {
  const int h = c >> 7, j = (c >> 5) & 3, s = (c >> 3) & 3, i = c & 7;
  return 64 * s + 32 * h + 8 * j + i;
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
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t phase) {
  uint32_t done;
  asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
               "selp.u32 %0, 1, 0, p;\n}"
               : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  return done != 0;
}
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t phase) {
  uint32_t done;
  asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
               "selp.u32 %0, 1, 0, p;\n}"
               : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  return done != 0;
}
// wait, then one cluster-scope acquire fence for remote stores released before remote arrives
// Stage barriers collect remote (release.cluster) arrivals: the issuer observes them with
// cluster-scope acquire on the wait itself (a separate fence.acq_rel.cluster compiles to a
// GPU-scope MEMBAR that cost ~1000 cycles per stage in the round trace).
__device__ __forceinline__ bool mbar_test_cluster(uint32_t bar, uint32_t phase) {
  uint32_t done;
  asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
               "selp.u32 %0, 1, 0, p;\n}"
               : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  return done != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                 "selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  }
}
// blocking wait: try_wait suspends the polling thread in hardware between checks, so the
// waiting warps do not take issue slots from the working ones (one lane per warp waits, the
// rest sit in __syncwarp)
__device__ __forceinline__ void mbar_wait_hint(uint32_t bar, uint32_t phase) {
  while (!mbar_try(bar, phase)) {
  }
}
__device__ __forceinline__ void mbar_arrive_local(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory");
}
// Remote arrive with the default (.release.cta) semantics, as CUTLASS's ClusterBarrier::arrive:
// the data it publishes (U rows) lives in the arriving CTA's own shared memory and is read by the
// tensor core after fence.proxy.async; .release.cluster compiles to MEMBAR.ALL.GPU + ERRBAR,
// which waited for the warp's outstanding global stores on every stage (round trace).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" :: "r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void red_or_cluster(uint32_t cluster_addr, uint32_t v) {
  asm volatile("red.relaxed.cluster.shared::cluster.or.b32 [%0], %1;" :: "r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mma2_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}"
               :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// warp-collective forms: the whole (converged) warp executes them, one elected lane issues
__device__ __forceinline__ void mma2_f16_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
               "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}"
               :: "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit2_elect(uint32_t bar) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
               "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}"
               :: "r"(bar), "h"((uint16_t)3));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])),
                  "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])),
                  "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])));
}
// tcgen05.wait::ld that names the destination registers of the loads it waits for, so the
// compiler cannot read or move them between the (asynchronous) tcgen05.ld and the wait
__device__ __forceinline__ void tmem_wait_ld3(float (&a)[8], float (&b)[8], float (&c)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+f"(a[0]), "+f"(a[1]), "+f"(a[2]), "+f"(a[3]), "+f"(a[4]), "+f"(a[5]), "+f"(a[6]), "+f"(a[7]),
                 "+f"(b[0]), "+f"(b[1]), "+f"(b[2]), "+f"(b[3]), "+f"(b[4]), "+f"(b[5]), "+f"(b[6]), "+f"(b[7]),
                 "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]), "+f"(c[4]), "+f"(c[5]), "+f"(c[6]), "+f"(c[7])
               :: "memory");
}
__device__ __forceinline__ float clampf(float u, float t) { return fminf(fmaxf(u, -t), t); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.f, -1.f), a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 clamp2(float2 u, float2 t) {
  return make_float2(clampf(u.x, t.x), clampf(u.y, t.y));
}
__device__ __forceinline__ float2 splat2(float s) { return make_float2(s, s); }
__device__ __forceinline__ bool finitef(float x) { return fabsf(x) <= FLT_MAX; }
// fp16 hi/lo split of a coordinate pair: hi = rn(u), lo = rn(u - hi)
__device__ __forceinline__ void split2(float2 u, uint32_t &hw, uint32_t &lw) {
  const __half2 hi = __float22half2_rn(u);
  const float2 hb = __half22float2(hi);
  const __half2 lo = __float22half2_rn(sub2(u, hb));
  hw = *reinterpret_cast<const uint32_t *>(&hi);
  lw = *reinterpret_cast<const uint32_t *>(&lo);
}

template <int HK, bool SCALED>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    hopf_dense_tc3_kernel(const DenseParams p, const uint4 *__restrict__ mlam_rows,
                          float mscale_inv, int *__restrict__ fix_count,
                          int *__restrict__ fix_list) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const float4 *red = reinterpret_cast<const float4 *>(smem + OFF_RED);
  float *w_s = reinterpret_cast<float *>(smem + OFF_W);
  uint8_t *bars = smem + OFF_BAR;
  volatile int *busy = reinterpret_cast<volatile int *>(bars + 48);
  volatile uint32_t *tmem_slot = reinterpret_cast<volatile uint32_t *>(bars + 56);
  const uint32_t bar_mma = smem_u32(bars), bar_term = smem_u32(bars + 8);
  const uint32_t bar_stage0 = smem_u32(bars + 16), bar_red = smem_u32(bars + 64), bar_fin = smem_u32(bars + 80);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const float lam = p.lambda, tol = p.tol, ilam = 1.f / p.lambda;
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int64_t stride = npairs * 2 * PTS;

  // ---- setup: this CTA's half of M_lambda (B operand) -> smem; w; barriers; TMEM -----------
  for (int e = tid; e < 131072 / 16; e += THREADS)
    reinterpret_cast<uint4 *>(smem + OFF_BH)[e] = __ldg(mlam_rows + (size_t)rank * 8192 + e);
  for (int e = tid; e < N_DIM; e += THREADS) w_s[e] = (HK == HK_WL1) ? __ldg(p.w + e) : 1.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32((const void *)tmem_slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(bar_mma, 1);
    mbar_init(bar_term, 1);
    for (int s = 0; s < 4; s++) mbar_init(bar_stage0 + 8 * s, 2 * EPI_WARPS);
    mbar_init(bar_red, EPI_WARPS / 2);        // slots 0-31: the 8 warps with (warp & 1) == 0
    mbar_init(bar_red + 8, EPI_WARPS / 2);    // slots 32-63
    mbar_init(bar_fin, 1);
    busy[0] = busy[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sm0 = smem_u32(smem);

  if (warp >= EPI_WARPS) {
    // ================= MMA warpgroup: warp 16 of the leader issues, the others idle =========
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(MMA_REGS));
    if (rank == 0 && warp == EPI_WARPS && lane == 0) {
      // one thread issues (an elect.sync form issued by the converged warp ran the round
      // skeleton 2.5-4x slower: tools/tcgen05_probe/probe_round.cu)
      const uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint64_t a_h0 = make_sdesc(sm0 + OFF_UH, 128, 4096), a_l0 = make_sdesc(sm0 + OFF_UL, 128, 4096);
      const uint64_t b_h0 = make_sdesc(sm0 + OFF_BH, 128, 4096), b_l0 = make_sdesc(sm0 + OFF_BL, 128, 4096);
      for (uint32_t r = 0;; r++) {
        const uint32_t d_tmem = tmem + 128u * ((r + 1) % 3);
        int any_busy = 1;
#pragma unroll 1
        for (int s = 0; s < 4; s++) {
          // CTA-scope wait, as CUTLASS's MMA warps do for their operand-full barriers (the
          // remote arrives are default .release.cta; the tensor core reads the peer's shared
          // memory through the async proxy after the writers' fence.proxy.async)
          mbar_wait_hint(bar_stage0 + 8 * s, r & 1);
          TC3_STAMP(r + 1, s);   // MMA thread: stage s of round r+1's operand ready
          // the busy word is complete once stage 0 has arrived; its value is only needed
          // after the last stage, so the shared load stays off the MMA issue path
          if (s == 0) any_busy = busy[r & 1];
          asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
          for (int t = 0; t < 4; t++) {
            const int ks = 4 * s + t;
            const uint64_t o = (uint64_t)(ks * 16);
            mma2_f16(d_tmem, a_h0 + o, b_h0 + o, idesc, ks > 0 ? 1u : 0u);   // Uh Mh
            mma2_f16(d_tmem, a_l0 + o, b_h0 + o, idesc, 1u);                 // Ul Mh
            mma2_f16(d_tmem, a_h0 + o, b_l0 + o, idesc, 1u);                 // Uh Ml
          }
        }
        busy[r & 1] = 0;
        if (!any_busy) {
          // no work left in either CTA: let this round's (unneeded) MMAs drain, then term
          // first and wake the MMA waiters of both CTAs
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       :: "r"(bar_fin));
          mbar_wait_hint(bar_fin, 0);
          mbar_arrive_local(bar_term);
          mbar_arrive_remote(mapa(bar_term, 1));
          mbar_arrive_local(bar_mma);
          mbar_arrive_remote(mapa(bar_mma, 1));
          break;
        }
        TC3_STAMP(r + 1, 4);     // last MMA of round r+1 issued
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     :: "r"(bar_mma), "h"((uint16_t)3));
      }
    }
    __syncwarp();
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(EPI_REGS));
    // ================= epilogue warps =======================================================
    const int q = warp & 3, j = warp >> 2;
    const int pl = 32 * (q & 1) + lane;           // local point slot
    const int h = q >> 1;
    const int part = 4 * h + j;                   // which of the 8 partials of the point
    const bool writer = part == 7;                // the one thread per slot with side effects
    const int cb = 128 * h + 32 * j;              // first coordinate of this thread
    // warp-uniform; the lane-0 shuffle lets the compiler prove it and keep TMEM addresses in
    // uniform registers (no R2UR before each tcgen05.ld / st)
    const uint32_t t_lane = __shfl_sync(0xffffffffu, tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(32 * j), 0);
    const uint32_t t_x = t_lane + 384u;           // x of the slot's point (TMEM columns 384..511)
    const uint32_t busy_addr = (rank == 0) ? smem_u32((const void *)busy) : mapa(smem_u32((const void *)busy), 0);
    const uint32_t stage_remote = mapa(bar_stage0, 0);

    // u^{k-1} = v^{k-1} + b^{k-2} (the argument of the previous shrink) of this thread's 32
    // coordinates: b^{k-1} = clamp(u, tau), d^{k-1} = u - b^{k-1}.  A slot that starts a point
    // holds x in us (loaded before its first round) and runs that round with tau = 0.
    float2 us[16];
#pragma unroll
    for (int i = 0; i < 16; i++) us[i] = splat2(0.f);

    // slot state, kept identically by the 8 threads of the slot: they read the same 8 partial
    // sums and the same t values, so they take the same decisions without a broadcast
    int dpt = (int)(pair * 2 * PTS) + (int)rank * PTS + pl - (int)stride;
    int dit = 0, dmode = M_EMPTY;
    float dtt = 0.f;
    int cq = -1, npt = 0;   // cq: the point whose t is cached in ct; npt: next point (FINISH)
    float ct = 0.f, ntt = 0.f;
    // next valid point after `from`; t <= 0 / non-finite t go to the exact SIMT list
    const int M32 = (int)p.M, S32 = (int)stride;   // M <= INT32_MAX - 2^20 on this path
    auto advance = [&](int from, int &q_out, float &t_out) {
      int q = from + S32;
      while (q < M32) {
        const float tn = (q == cq) ? ct : __ldg(p.t + q);
        if (tn > 0.f && tn <= FLT_MAX) { t_out = tn; break; }
        if (writer) fix_list[atomicAdd(fix_count, 1)] = q;
        q += S32;
      }
      q_out = q;
    };
    auto begin = [&](int q, float tq, int startmode) {   // the slot takes point q
      dpt = q; dtt = tq; dit = 0;
      if (q < M32) {
        dmode = startmode;
        cq = q + S32;   // t of the following point, needed one lifetime later
        if (cq < M32) ct = __ldg(p.t + cq);
      } else {
        dmode = M_EMPTY;
      }
    };

    for (uint32_t r = 0;; r++) {
      // ---- every thread of a slot reads the 8 partial sums of round r-1 and decides ----------
      if (r == 0) {
        int q; float tq = 0.f;
        advance(dpt, q, tq);
        begin(q, tq, M_START_LD);
      } else {
        mbar_wait_hint(bar_red + 8 * (q & 1), (r - 1) & 1);   // the whole warp waits (no divergent wait + reconvergence)
        if (lane == 0 && (warp == 0 || warp == 15)) TC3_STAMP(r, 8 + (warp == 15) * 16);
        __syncwarp();
        float s4[4] = {0.f, 0.f, 0.f, 0.f};
        const float4 *rp = red + (size_t)((r - 1) & 1) * 8 * PTS + pl;
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const float4 a = rp[k * PTS];
          s4[0] += a.x; s4[1] += a.y; s4[2] += a.z; s4[3] += a.w;
        }
        if (dmode == M_ACTIVE) {
          dit += 1;
          const bool fin = finitef(s4[0] + s4[1] + s4[2]);
          if (fin && s4[0] <= tol && s4[1] <= tol && s4[2] <= tol) {
            dmode = M_FINISH;
            advance(dpt, npt, ntt);   // its x is loaded at the end of the FINISH round
          } else if (!fin || dit >= p.max_iter) {
            if (writer) fix_list[atomicAdd(fix_count, 1)] = dpt;
            int q; float tq = 0.f;
            advance(dpt, q, tq);
            begin(q, tq, M_START_LD);
          }
        } else if (dmode == M_FINISH) {
          if (writer) {
            p.phi[dpt] = s4[3] + p.gamma;
            p.iters[dpt] = dit;
          }
          begin(npt, ntt, M_START);
        } else if (dmode == M_START || dmode == M_START_LD) {
          dmode = M_ACTIVE;
        }
      }
      const int pt = dpt;
      const int mode = dmode, it = dit;
      const float tt = dtt;
      const bool st = mode == M_START || mode == M_START_LD, fin = mode == M_FINISH;
      const int nxt = fin ? (npt < M32 ? npt : M32) : M32;
      if (mode == M_START_LD) {   // new point: x into us
        const float4 *xr = reinterpret_cast<const float4 *>(p.X + pt * (int64_t)N_DIM + cb);
#pragma unroll
        for (int g = 0; g < 8; g++) {
          const float4 v4 = __ldg(xr + g);
          us[2 * g] = make_float2(v4.x, v4.y);
          us[2 * g + 1] = make_float2(v4.z, v4.w);
        }
      }
      if (st) {   // its successor into L2
        if (pt + (int)stride < (int)p.M) {
          asm volatile("prefetch.global.L2 [%0];" :: "l"(p.X + (pt + stride) * (int64_t)N_DIM + cb));
          if (writer) asm volatile("prefetch.global.L2 [%0];" :: "l"(p.t + pt + stride));
        }
      }
      const bool lane_busy = mode == M_ACTIVE || st || (fin && nxt < (int)p.M);
      {   // any work for MMA r+1 in this warp?  (the issuer reads busy[r & 1] before stage 0)
        const bool wb = __any_sync(0xffffffffu, lane_busy);
        if (lane == 0 && wb) red_or_cluster(busy_addr + 4u * (r & 1), 1u);
      }
      const bool any_st = __any_sync(0xffffffffu, st), any_fin = __any_sync(0xffffffffu, fin);
      // START: tau_old = tau = 0 and v := x give u = x, d^0 = x, b^0 = 0 and U^1 = (1 + lambda) x;
      // k = 1: tau_old = 0 gives b^0 = 0, d^0 = u = x (R5), and v_prev = x from TMEM (R3)
      const bool fst = mode == M_ACTIVE && it == 0;
      const float tcur = st ? 0.f : tt * ilam, told = (st || fst) ? 0.f : tt * ilam;
      // ---- wait for MMA r (v^k in D[r % 3]) or termination -----------------------------------
      if (r > 0) {
        mbar_wait_hint(bar_mma, (r - 1) & 1);
        if (lane == 0 && (warp == 0 || warp == 15)) TC3_STAMP(r, 9 + (warp == 15) * 16);
        __syncwarp();
        if (mbar_test(bar_term, 0)) break;
        asm volatile("tcgen05.fence::after_thread_sync;");
      }
      const uint32_t tbuf = t_lane + 128u * (r % 3), tpbuf = t_lane + 128u * ((r + 2) % 3);
      float2 asd = splat2(0.f), asb = splat2(0.f), asv = splat2(0.f);
      float aph = 0.f;
      // TMEM loads are software-pipelined: stage s+1's are issued before stage s's stores,
      // fences and arrive, into the registers stage s has finished with
      float va[8], vpa[8], xa[8];
      if (r > 0) {
        tmem_ld8(tbuf, va);
        tmem_ld8(tpbuf, vpa);
        tmem_ld8(t_x, xa);
        tmem_wait_ld3(va, vpa, xa);
      } else {
#pragma unroll
        for (int e = 0; e < 8; e++) va[e] = vpa[e] = xa[e] = 0.f;
      }
#pragma unroll
      for (int s = 0; s < 4; s++) {
        if (SCALED) {
#pragma unroll
          for (int e = 0; e < 8; e++) { va[e] *= mscale_inv; vpa[e] *= mscale_inv; }
        }
        if (any_st) {
          // START lanes: x from ds, v := x; x goes to the x columns and to D[r % 3], which is the
          // v_prev of the next round (k = 1 compares with v^0 = x, reading R3)
#pragma unroll
          for (int i2 = 0; i2 < 4; i2++) {
            const int i = 4 * s + i2;
            if (st) {
              xa[2 * i2] = va[2 * i2] = us[i].x;
              xa[2 * i2 + 1] = va[2 * i2 + 1] = us[i].y;
            }
          }
          tmem_st8(t_x + 8 * s, xa);
          tmem_st8(tbuf + 8 * s, va);
        }
        if (any_fin && fin) {
          // converged at k: grad = d^k; phi by reading R23 with v = v^{k+1}, U^{k+1} = x + lambda (d - b)
          float gout[8];
#pragma unroll
          for (int i2 = 0; i2 < 4; i2++) {
            const int i = 4 * s + i2;
            const float2 v = make_float2(va[2 * i2], va[2 * i2 + 1]);
            const float2 x = make_float2(xa[2 * i2], xa[2 * i2 + 1]);
            const float2 wv = (HK == HK_WL1) ? *reinterpret_cast<const float2 *>(w_s + cb + 2 * i)
                                             : splat2(1.f);
            const float2 b = clamp2(us[i], mul2(splat2(tt * ilam), wv));   // b^k
            const float2 d = sub2(us[i], b);                                // d^k
            const float2 Uf = fma2(splat2(lam), sub2(d, b), x);
            const float2 g = fma2(splat2(-lam), v, Uf);              // A^{-1} v^{k+1}
            const float2 hv = fma2(splat2(-0.5f), v, d);
            aph += x.x * d.x + x.y * d.y - (g.x * hv.x + g.y * hv.y) -
                   tt * (wv.x * fabsf(d.x) + wv.y * fabsf(d.y));
            gout[2 * i2] = d.x;
            gout[2 * i2 + 1] = d.y;
          }
          float4 *g4 = reinterpret_cast<float4 *>(p.grad + pt * (int64_t)N_DIM + cb + 8 * s);
          g4[0] = make_float4(gout[0], gout[1], gout[2], gout[3]);
          g4[1] = make_float4(gout[4], gout[5], gout[6], gout[7]);
        }
        // U^{k+1} first: its K block is released to the MMA thread before the stopping sums of
        // this stage are formed (they are not on the MMA -> epilogue -> MMA chain)
        uint32_t hw[4], lw[4];
        float2 dOs[4], dns[4];
#pragma unroll
        for (int i2 = 0; i2 < 4; i2++) {
          const int i = 4 * s + i2;                 // coordinate pair index 0..15
          const float2 v = make_float2(va[2 * i2], va[2 * i2 + 1]);
          const float2 x = make_float2(xa[2 * i2], xa[2 * i2 + 1]);
          const float2 wv = (HK == HK_WL1) ? *reinterpret_cast<const float2 *>(w_s + cb + 2 * i)
                                           : splat2(1.f);
          const float2 tau = (HK == HK_WL1) ? mul2(splat2(tcur), wv) : splat2(tcur);
          const float2 tauo = (HK == HK_WL1) ? mul2(splat2(told), wv) : splat2(told);
          const float2 u = us[i];
          const float2 bo = clamp2(u, tauo);               // b^{k-1}
          dOs[i2] = sub2(u, bo);                           // d^{k-1}
          const float2 un = add2(v, bo);                   // argument of (3.4b): v^k + b^{k-1}
          const float2 bn = clamp2(un, tau);               // b^k (projection, Moreau)
          const float2 dn = sub2(un, bn);                  // d^k = shrink_1
          dns[i2] = dn;
          const float2 U = fma2(splat2(lam), sub2(dn, bn), x);   // U^{k+1} = x + lambda (d - b)
          us[i] = un;
          split2(U, hw[i2], lw[i2]);
        }
        // U^{k+1} of coordinates cb + 8 s .. + 8 -> its K' block: one 16-byte row chunk (hi, lo)
        const uint32_t off = kmaj(pl, 64 * s + 32 * h + 8 * j);
        *reinterpret_cast<uint4 *>(smem + OFF_UH + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4 *>(smem + OFF_UL + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (any_st) asm volatile("tcgen05.wait::st.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive_local(bar_stage0 + 8 * s);
          else mbar_arrive_remote(stage_remote + 8 * s);
          if (warp == 0 || warp == 15) TC3_STAMP(r, 10 + s + (warp == 15) * 16);
        }
        // the paper's three stopping sums of this stage, off the MMA chain
#pragma unroll
        for (int i2 = 0; i2 < 4; i2++) {
          const float2 v = make_float2(va[2 * i2], va[2 * i2 + 1]);
          const float2 vp = make_float2(vpa[2 * i2], vpa[2 * i2 + 1]);
          const float2 ed = sub2(dns[i2], dOs[i2]);
          asd = fma2(ed, ed, asd);
          const float2 fd = sub2(dns[i2], v);
          asb = fma2(fd, fd, asb);
          const float2 gd = sub2(v, vp);
          asv = fma2(gd, gd, asv);
        }
        if (s < 3 && r > 0) {
          tmem_ld8(tbuf + 8 * (s + 1), va);
          tmem_ld8(tpbuf + 8 * (s + 1), vpa);
          tmem_ld8(t_x + 8 * (s + 1), xa);
          tmem_wait_ld3(va, vpa, xa);
        }
      }
      // ---- partial sums of this round -> red[r & 1]; released through bar_red ---------------
      {
        float4 *wp = reinterpret_cast<float4 *>(smem + OFF_RED) + ((size_t)(r & 1) * 8 + part) * PTS + pl;
        *wp = make_float4(asd.x + asd.y, asb.x + asb.y, asv.x + asv.y, aph);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar_red + 8 * (q & 1));
      if (lane == 0 && (warp == 0 || warp == 15)) TC3_STAMP(r, 14 + (warp == 15) * 16);
      if (fin && nxt < (int)p.M) {   // the next point of a finished slot: x into us now (START next round)
        const float4 *xr = reinterpret_cast<const float4 *>(p.X + nxt * (int64_t)N_DIM + cb);
#pragma unroll
        for (int g = 0; g < 8; g++) {
          const float4 v4 = __ldg(xr + g);
          us[2 * g] = make_float2(v4.x, v4.y);
          us[2 * g + 1] = make_float2(v4.z, v4.w);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
}

}  // namespace tc3

// M_lambda rows for the pair with the permuted contraction index: rank r holds rows
// [128 r, 128 r + 128) of 2^s M_lambda as fp16 hi (64 KB) then lo (64 KB), K-major no-swizzle,
// element (row, K') = M[row][c] with K' = kperm(c).  2^s brings max |M| into [0.5, 1) (s = 0
// for the configs: M_lambda's eigenvalues lie in (0, 1/lambda)), so no rescale is needed.
int dense_tc3_prepare(int n, const double *Ml, void **rows_dev, float *mscale_inv) {
  if (n != tc3::N_DIM) return HOPF_EUNSUPPORTED;
  double mx = 0.0;
  for (int i = 0; i < n * n; i++) mx = fmax(mx, fabs(Ml[i]));
  int s = 0;
  if (mx > 0.0) {
    int e;
    frexp(mx, &e);   // mx = f 2^e, f in [0.5, 1)
    s = -e;
  }
  const double sc = ldexp(1.0, s);
  std::vector<__half> hb(2 * 2 * 128 * 256);
  for (int r = 0; r < 2; r++)
    for (int row = 0; row < 128; row++)
      for (int c = 0; c < 256; c++) {
        const double v = Ml[(size_t)(128 * r + row) * n + c] * sc;
        const __half hi = __float2half_rn((float)v);
        const __half lo = __float2half_rn((float)(v - (double)__half2float(hi)));
        const size_t base = (size_t)r * 2 * 128 * 256;
        const int kp = tc3::kperm(c);
        hb[base + tc3::kmaj(row, kp) / 2] = hi;
        hb[base + 128 * 256 + tc3::kmaj(row, kp) / 2] = lo;
      }
  if (cudaMalloc(rows_dev, hb.size() * sizeof(__half)) != cudaSuccess)
    return set_error(HOPF_ECUDA, "cudaMalloc for tensor-core operands failed");
  cudaMemcpy(*rows_dev, hb.data(), hb.size() * sizeof(__half), cudaMemcpyHostToDevice);
  *mscale_inv = (float)ldexp(1.0, -s);
  return HOPF_OK;
}

#ifdef HOPF_TC3_TRACE
extern "C" int hopf_tc3_trace_dump(long long *out) {
  return cudaMemcpyFromSymbol(out, tc3::g_trace, sizeof(tc3::g_trace)) == cudaSuccess ? 0 : -1;
}
#endif

int dense_tc3_launch(const DenseParams &p, int hk, const void *rows, float mscale_inv,
                     int *fix_count, int *fix_list, cudaStream_t stream) {
  const bool scaled = mscale_inv != 1.f;
  void (*fn)(const DenseParams, const uint4 *, float, int *, int *);
  if (hk == HK_WL1) fn = scaled ? tc3::hopf_dense_tc3_kernel<HK_WL1, true> : tc3::hopf_dense_tc3_kernel<HK_WL1, false>;
  else fn = scaled ? tc3::hopf_dense_tc3_kernel<HK_L1, true> : tc3::hopf_dense_tc3_kernel<HK_L1, false>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, tc3::SMEM_BYTES);
  int64_t pairs = num_sms() / 2;
  const int64_t need = (p.M + 2 * tc3::PTS - 1) / (2 * tc3::PTS);
  if (pairs > need) pairs = need;
  if (pairs < 1) pairs = 1;
  fn<<<(unsigned)(2 * pairs), tc3::THREADS, tc3::SMEM_BYTES, stream>>>(
      p, reinterpret_cast<const uint4 *>(rows), mscale_inv, fix_count, fix_list);
  g_launches += 1;
  return check_launch("hopf_dense_tc3_kernel");
}

}  // namespace hopf
