// Probe: the dense tc3 round skeleton with an empty epilogue.  16 "epilogue" warps per CTA wait
// for the round's MMA completion and arrive on 4 stage barriers in the leader; warp 16 of the
// leader issues 4 x 12 pair-MMAs (M=128, N=256, K=16, 3-term pattern) into D[(r+1) % 3] and
// commits (multicast).  Variants (argv): bit0 = setmaxnreg, bit1 = elect.sync issue (else one
// thread), bit2 = rotate D (else D[0]), bit3 = acquire.cluster waits.  Prints cycles per round
// and the stage-0 issue time.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32; d |= (uint64_t)1 << 46; return d; }
__device__ int g_poll_mode = 0;   // 0: try_wait, 1: test_wait
__device__ __forceinline__ bool test_wait(uint32_t bar, uint32_t ph) {
  uint32_t d;
  if (g_poll_mode) asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(d) : "r"(bar), "r"(ph) : "memory");
  else asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(d) : "r"(bar), "r"(ph) : "memory");
  return d; }
__device__ __forceinline__ bool test_wait_cl(uint32_t bar, uint32_t ph) {
  uint32_t d; asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(d) : "r"(bar), "r"(ph) : "memory"); return d; }
template <int V>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(640, 1) probe(long long* out, int rounds) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bmma, bst[4]; __shared__ uint32_t tbase;
  uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31;
  for (int e = tid; e < 196608 / 16; e += blockDim.x) reinterpret_cast<uint4*>(smem)[e] = make_uint4(0x3c003c00u, 0x1c00u, 0x3c00u, 0x2000);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&bmma)), "r"(1));
    for (int s = 0; s < 4; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&bst[s])), "r"(32));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase, s0 = smem_u32(smem);
  const uint32_t bar_mma = smem_u32(&bmma), bar_st = smem_u32(&bst[0]);
  uint32_t st_remote; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(st_remote) : "r"(bar_st), "r"(0u));
  if (warp >= 16) {
    if (V & 1) asm volatile("setmaxnreg.dec.sync.aligned.u32 32;");
    if (rank == 0 && warp == 16) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint64_t ah = make_desc(s0, 128, 4096), al = make_desc(s0 + 32768, 128, 4096);
      const uint64_t bh = make_desc(s0 + 65536, 128, 4096), bl = make_desc(s0 + 131072, 128, 4096);
      long long tstart = clock64(), s0sum = 0;
      for (int r = 0; r < rounds; r++) {
        const uint32_t d = tm + ((V & 4) ? 128u * ((r + 1) % 3) : 0u);
        long long ta = 0;
        for (int s = 0; s < 4; s++) {
          if (lane == 0) { if (V & 8) { while (!test_wait_cl(bar_st + 8 * s, r & 1)) {} } else { while (!test_wait(bar_st + 8 * s, r & 1)) {} } }
          __syncwarp();
          if (s == 0) ta = clock64();
          if (s == 0 && lane == 0 && r == 101) out[11] = ta;
          asm volatile("tcgen05.fence::after_thread_sync;");
          for (int t = 0; t < 4; t++) {
            const uint64_t o = (uint64_t)((4 * s + t) * 16);
            const uint32_t acc0 = (s + t) > 0;
            if (V & 2) {
              asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(ah + o), "l"(bh + o), "r"(idesc), "r"(acc0));
              asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(al + o), "l"(bh + o), "r"(idesc), "r"(1u));
              asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(ah + o), "l"(bl + o), "r"(idesc), "r"(1u));
            } else if (lane == 0) {
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(ah + o), "l"(bh + o), "r"(idesc), "r"(acc0));
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(al + o), "l"(bh + o), "r"(idesc), "r"(1u));
              asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(ah + o), "l"(bl + o), "r"(idesc), "r"(1u));
            }
          }
          __syncwarp();
          if (s == 0) s0sum += clock64() - ta;
        }
        if (lane == 0 && r == 100) out[10] = clock64();
        if (V & 2) asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}" :: "r"(bar_mma), "h"((uint16_t)3));
        else if (lane == 0) asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" :: "r"(bar_mma), "h"((uint16_t)3));
        __syncwarp();
      }
      if (lane == 0) { out[0] = clock64() - tstart; out[1] = s0sum; }
    }
  } else {
    if (V & 1) asm volatile("setmaxnreg.inc.sync.aligned.u32 112;");
    for (int r = 0; r < rounds; r++) {
      if (r > 0) { if (lane == 0) { while (!test_wait(bar_mma, (r - 1) & 1)) {} } __syncwarp(); asm volatile("tcgen05.fence::after_thread_sync;"); }
      if (r == 101 && rank == 0 && tid == 0) out[12] = clock64();
      for (int s = 0; s < 4; s++) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(bar_st + 8 * s) : "memory");
          else asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" :: "r"(st_remote + 8 * s) : "memory");
        }
        if (r == 101 && s == 0 && rank == 0 && tid == 0) out[13] = clock64();
      }
    }
    if (lane == 0) { while (!test_wait(bar_mma, (rounds - 1) & 1)) {} }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(512));
}
template <int V> void run(long long* d, int rounds) {
  const int smem = 196608;
  cudaFuncSetAttribute(probe<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaMemset(d, 0, 128);
  probe<V><<<2, 640, smem>>>(d, rounds);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("V=%d err %s\n", V, cudaGetErrorString(e)); exit(1); }
  long long h[16]; cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
  printf("V=%2d (setmaxnreg %d elect %d rotate %d acq.cluster %d): %.0f cycles/round, stage-0 issue %.0f | commit->epi seen %lld ->arrive0 %lld ->mma obs0 %lld\n", V, V & 1, (V >> 1) & 1, (V >> 2) & 1, (V >> 3) & 1,
         (double)h[0] / rounds, (double)h[1] / rounds, h[12] - h[10], h[13] - h[12], h[11] - h[13]);
}
int main() {
  long long* d; cudaMalloc(&d, 128);
  const int R = 200;
  for (int pm = 0; pm < 2; pm++) {
    cudaMemcpyToSymbol(g_poll_mode, &pm, sizeof(int));
    printf("poll mode %s\n", pm ? "test_wait" : "try_wait");
    run<0>(d, R); run<1>(d, R); run<2>(d, R); run<3>(d, R); run<4>(d, R); run<8>(d, R); run<15>(d, R);
  }
  return 0;
}
