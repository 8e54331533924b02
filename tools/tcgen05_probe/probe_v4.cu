// Probe for the dense v4 design (CTA pair, kind::f16, M=128 x N=256, K=256):
//  (1) the 3-term split sequence (Uh Mh, Ul Mh, Uh Ml per K-step, distinct descriptors), cycles
//      per pair-MMA over many repetitions;
//  (2) TMEM read throughput: 16 warps each reading their lane quarter x 32 columns (x8 / x16 / x32
//      shapes), cycles per KB per SM;
//  (3) TMEM store throughput (32x32b.x8).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32; d |= (uint64_t)1 << 46; return d; }
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) probe(long long* out, int reps) {
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
  const uint32_t tm = tbase;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t s0 = smem_u32(smem);
  long long t0 = clock64();
  if (rank == 0 && tid == 0) {
    const uint64_t ah0 = make_desc(s0, 128, 4096), al0 = make_desc(s0 + 32768, 128, 4096);
    const uint64_t bh0 = make_desc(s0 + 65536, 128, 4096), bl0 = make_desc(s0 + 131072, 128, 4096);
    for (int r = 0; r < reps; r++) {
      uint64_t ah = ah0, al = al0, bh = bh0, bl = bl0;
      const uint32_t d = tm + (uint32_t)(128 * (r % 3));
#pragma unroll
      for (int ks = 0; ks < 16; ks++) {
        const uint32_t acc = ks > 0;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(ah), "l"(bh), "r"(idesc), "r"(acc));
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(al), "l"(bh), "r"(idesc), "r"(1u));
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(d), "l"(ah), "l"(bl), "r"(idesc), "r"(1u));
        ah += 256 >> 4; al += 256 >> 4; bh += 256 >> 4; bl += 256 >> 4;
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "h"((uint16_t)3));
  }
  { uint32_t done = 0; while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0)); }
  if (tid == 0) out[rank * 8 + 0] = clock64() - t0;
  asm volatile("tcgen05.fence::after_thread_sync;");
  __syncthreads();
  // (2) TMEM reads: warp (q = w%4, j = w/4) reads lanes 32q.., columns 32j .. +32 of 3 buffers, x8 shape
  const uint32_t base = tm + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(32 * (warp >> 2));
  float acc = 0.f;
  t0 = clock64();
  for (int r = 0; r < reps; r++) {
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(base + (uint32_t)(128 * (r % 3)) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int i = 0; i < 8; i++) acc += __uint_as_float(v[i]);
    }
  }
  __syncthreads();
  if (tid == 0) out[rank * 8 + 1] = clock64() - t0;
  // (2b) same, x32 shape, one wait per 32 columns
  t0 = clock64();
  for (int r = 0; r < reps; r++) {
    uint32_t v[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]) : "r"(base + (uint32_t)(128 * (r % 3))));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int i = 0; i < 32; i++) acc += __uint_as_float(v[i]);
  }
  __syncthreads();
  if (tid == 0) out[rank * 8 + 2] = clock64() - t0;
  // (3) TMEM stores x8
  t0 = clock64();
  for (int r = 0; r < reps; r++) {
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      const uint32_t a = __float_as_uint(acc + r);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" :: "r"(base + 384u + c), "r"(a));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  __syncthreads();
  if (tid == 0) out[rank * 8 + 3] = clock64() - t0;
  if (acc == 12345.f) out[15] = 1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(512));
}
int main() {
  long long* d; cudaMalloc(&d, 16 * 8);
  const int smem = 196608;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int reps : {3, 300}) {
    cudaMemset(d, 0, 128);
    probe<<<2, 512, smem>>>(d, reps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    long long h[16]; cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
    const double kb = 16.0 * 32 * 32 * 4 / 1024;  // KB per SM per rep (16 warps x 32 lanes x 32 cols)
    printf("reps=%d: 3-term seq %.1f cyc/pair-MMA (ideal 64); TMEM ld x8 %.1f cyc/rep (%.1f B/cyc/SM); "
           "ld x32 %.1f cyc/rep (%.1f B/cyc/SM); st x8 %.1f cyc/rep (%.1f B/cyc/SM)\n",
           reps, (double)h[0] / (reps * 48.0), (double)h[1] / reps, kb * 1024 * reps / h[1],
           (double)h[2] / reps, kb * 1024 * reps / h[2], (double)h[3] / reps, kb * 1024 * reps / h[3]);
  }
  return 0;
}
