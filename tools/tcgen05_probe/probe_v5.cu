// Probe: does epilogue traffic slow the pair MMA?  Thread 0 of the leader issues R rounds of the
// 48-MMA 3-term sequence (M=128, N=256, K=256) while the other 15 warps of both CTAs run a
// background load: 0 none, 1 tcgen05.ld (columns 384..511), 2 st.shared 16 B (region above the
// operands), 3 FFMA chains, 4 tcgen05.ld + st.shared.  Reports cycles per pair-MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32; d |= (uint64_t)1 << 46; return d; }
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) probe(long long* out, int reps, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar; __shared__ uint32_t tbase; __shared__ volatile int stop;
  uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31;
  for (int e = tid; e < 196608 / 16; e += blockDim.x) reinterpret_cast<uint4*>(smem)[e] = make_uint4(0x3c003c00u, 0, 0x3c00u, 0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) { stop = 0; asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1)); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t s0 = smem_u32(smem);
  float acc = 0.f;
  if (warp == 0) {
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint64_t ah0 = make_desc(s0, 128, 4096), al0 = make_desc(s0 + 32768, 128, 4096);
      const uint64_t bh0 = make_desc(s0 + 65536, 128, 4096), bl0 = make_desc(s0 + 131072, 128, 4096);
      long long t0 = clock64();
      for (int r = 0; r < reps; r++) {
        const uint32_t d = tm + (uint32_t)(128 * (r % 3));
#pragma unroll
        for (int ks = 0; ks < 16; ks++) {
          const uint64_t o = ks * 16;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(ah0 + o), "l"(bh0 + o), "r"(idesc), "r"((uint32_t)(ks > 0)));
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(al0 + o), "l"(bh0 + o), "r"(idesc), "r"(1u));
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(ah0 + o), "l"(bl0 + o), "r"(idesc), "r"(1u));
        }
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "h"((uint16_t)3));
      uint32_t done = 0; while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
      out[0] = clock64() - t0;
    }
    __syncwarp();
  } else {
    // background: until the MMA completes (mbarrier phase 0)
    const uint32_t base = tm + ((uint32_t)(32 * (warp & 3)) << 16) + 384u + (uint32_t)(32 * ((warp >> 2) & 3));
    uint8_t* sbuf = smem + 196608 + (tid % 64) * 256;  // 16 KB region above the operands
    int it = 0;
    while (true) {
      uint32_t done;
      asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
      if (done) break;
      for (int k = 0; k < 8; k++) {
        if (mode == 1 || mode == 4) {
          uint32_t v[8];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(base + 8 * (k & 3)));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          for (int i = 0; i < 8; i++) acc += __uint_as_float(v[i]);
        }
        if (mode == 2 || mode == 4) {
          *reinterpret_cast<uint4*>(sbuf + 16 * (k & 15)) = make_uint4(it, k, it, k);
        }
        if (mode == 3) {
          for (int i = 0; i < 16; i++) acc = fmaf(acc, 1.0001f, 0.5f);
        }
      }
      it++;
    }
  }
  if (acc == 12345.f) out[15] = 1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(512));
}
int main() {
  long long* d; cudaMalloc(&d, 16 * 8);
  const int smem = 196608 + 16384;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"none", "tcgen05.ld", "st.shared", "ffma", "ld+sts"};
  for (int mode = 0; mode < 5; mode++) {
    const int reps = 200;
    cudaMemset(d, 0, 128);
    probe<<<2, 512, smem>>>(d, reps, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    long long h[16]; cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
    printf("background %-11s: %.1f cycles per pair-MMA\n", names[mode], (double)h[0] / (reps * 48.0));
  }
  return 0;
}
