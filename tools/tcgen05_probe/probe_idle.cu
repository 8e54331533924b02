// Probe (idle variant): does an idle gap before a burst of 12 pair-MMAs slow it?
// (derived from probe_q) Probe: how many pair-MMAs (kind::f16, M=128, N=256, K=16) can one thread issue into an idle
// tensor pipe before the issue blocks?  Prints issue cycles for k = 1..24 back-to-back MMAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32; d |= (uint64_t)1 << 46; return d; }
__global__ void __cluster_dims__(2, 1, 1) probe(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar; __shared__ uint32_t tbase;
  uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 196608 / 16; e += blockDim.x) reinterpret_cast<uint4*>(smem)[e] = make_uint4(0x3c003c00u, 0, 0x3c00u, 0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1)); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase, s0 = smem_u32(smem);
  if (rank == 0 && tid == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t a0 = make_desc(s0, 128, 4096), b0 = make_desc(s0 + 65536, 128, 4096);
    uint32_t phase = 0;
    const int idles[6] = {0, 500, 1000, 2000, 4000, 10000};
    for (int rep = 0; rep < 12; rep++) {
      const int idle = idles[rep % 6];
      long long w0 = clock64();
      while (clock64() - w0 < idle) { }
      long long t0 = clock64();
      for (int i = 0; i < 12; i++) {
        const uint64_t o = (i % 16) * 16;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(tm), "l"(a0 + o), "l"(b0 + o), "r"(idesc), "r"((uint32_t)(i > 0)));
      }
      long long t1 = clock64();
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "h"((uint16_t)3));
      uint32_t done = 0; while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(phase));
      long long t2 = clock64();
      phase ^= 1;
      out[3 * rep] = idle; out[3 * rep + 1] = t1 - t0; out[3 * rep + 2] = t2 - t0;
    }
  } else if (rank == 1 && tid == 0) {
    uint32_t phase = 0;
    for (int k = 0; k < 12; k++) {
      uint32_t done = 0; while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(phase));
      phase ^= 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(512));
}
int main() {
  long long* d; cudaMalloc(&d, 64 * 8); cudaMemset(d, 0, 64 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
  probe<<<2, 128, 196608>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  long long h[64]; cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
  for (int r = 0; r < 12; r++) printf("idle %6lld: 12 MMAs issue %6lld cycles, issue->complete %6lld\n", h[3 * r], h[3 * r + 1], h[3 * r + 2]);
  return 0;
}
