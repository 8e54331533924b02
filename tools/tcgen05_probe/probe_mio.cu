// Probe: issue latency of a burst of 12 pair-MMAs (kind::f16 M=128 N=256 K=16) issued by one
// warp while 15 other warps of each CTA generate background traffic:
// 0 none, 1 tcgen05.ld x8 + wait, 2 st.shared.v4, 3 mbarrier try_wait spin, 4 ld.shared.v4,
// 5 tcgen05.ld + st.shared (epilogue-like), 6 st.shared + proxy fence into other K-blocks of the
// A operand, 7 tcgen05.ld from the other accumulator buffers.  Reports issue cycles and issue->complete cycles.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32; d |= (uint64_t)1 << 46; return d; }
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) probe(long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar, never, stopb; __shared__ uint32_t tbase;
  uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31;
  for (int e = tid; e < 196608 / 16; e += blockDim.x) {
    if (mode >= 8) {   // random fp16 operands in [-1, 1)
      uint32_t h = (uint32_t)e * 2654435761u + blockIdx.x * 97u;
      uint32_t w[4];
      for (int q = 0; q < 4; q++) {
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        const __half a = __float2half((float)((h & 0xffff) / 32768.0 - 1.0));
        const __half b = __float2half((float)((h >> 16) / 32768.0 - 1.0));
        w[q] = (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
      }
      reinterpret_cast<uint4*>(smem)[e] = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
      reinterpret_cast<uint4*>(smem)[e] = make_uint4(0x3c003c00u, 0, 0x3c00u, 0);
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&never)), "r"(1000000));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&stopb)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase, s0 = smem_u32(smem);
  float acc = 0.f;
  if (warp == 0) {
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint64_t a0 = make_desc(s0, 128, 4096), b0 = make_desc(s0 + 65536, 128, 4096);
      uint32_t phase = 0;
      long long w0 = clock64(); while (clock64() - w0 < 20000) { }   // let the background start
      for (int rep = 0; rep < 8; rep++) {
        long long t0 = clock64();
        for (int i = 0; i < 12; i++) {
          const uint64_t o = (i % 16) * 16;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(tm), "l"(a0 + o), "l"(b0 + o), "r"(idesc), "r"((uint32_t)(i > 0)));
        }
        long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "h"((uint16_t)3));
        uint32_t done = 0; while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(phase));
        long long t2 = clock64();
        phase ^= 1;
        if (blockIdx.x == 0) { out[2 * rep] = t1 - t0; out[2 * rep + 1] = t2 - t0; }
        w0 = clock64(); while (clock64() - w0 < 3000) { }
      }
      // stop the background in both CTAs
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&stopb)));
      uint32_t remote; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&stopb)), "r"(1));
      asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" :: "r"(remote));
    } else if (rank == 1 && lane == 0) {
      for (int rep = 0; rep < 8; rep++) {
        uint32_t done = 0; while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"((uint32_t)(rep & 1)));
      }
    }
    __syncwarp();
  } else {
    const uint32_t base = tm + ((uint32_t)(32 * (warp & 3)) << 16) + 384u + (uint32_t)(32 * ((warp >> 2) & 3));
    uint8_t* sbuf = smem + 196608 + (tid % 64) * 256;
    int it = 0;
    while (true) {
      uint32_t done;
      asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&stopb)), "r"(0));
      if (done) break;
      for (int k = 0; k < 8; k++) {
        if (mode == 1 || mode == 5) {
          uint32_t v[8];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(base + 8 * (k & 3)));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          for (int i = 0; i < 8; i++) acc += __uint_as_float(v[i]);
        }
        if (mode == 2 || mode == 5) *reinterpret_cast<uint4*>(sbuf + 16 * (k & 15)) = make_uint4(it, k, it, k);
        if (mode == 3 && lane == 0) {
          uint32_t d2;
          asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(d2) : "r"(smem_u32(&never)), "r"(0));
          acc += d2;
        }
        if (mode == 6) {   // st.shared into the A operand region, K-blocks the MMA does not read
          const int row = tid & 63, blk = 8 + (k & 7) + 8 * ((it >> 3) % 3);   // core matrices 8..31
          *reinterpret_cast<uint4*>(smem + (row >> 3) * 4096 + blk * 128 + (row & 7) * 16) = make_uint4(0x3c00u, 0, 0, 0);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        if (mode == 7) {   // tcgen05.ld from the other accumulator buffers (columns 128..383)
          uint32_t v[8];
          const uint32_t b2 = tm + ((uint32_t)(32 * (warp & 3)) << 16) + 128u + (uint32_t)(32 * ((warp >> 2) & 3)) + 128u * (k & 1);
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(b2));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          for (int i = 0; i < 8; i++) acc += __uint_as_float(v[i]);
        }
        if (mode >= 10) {   // epilogue-like: 3 x tcgen05.ld x8 + wait, st.shared, proxy fence, tcgen05 fence, arrive
          uint32_t v[8], v2[8], v3[8];
          const uint32_t b2 = tm + ((uint32_t)(32 * (warp & 3)) << 16) + 128u + (uint32_t)(32 * ((warp >> 2) & 3));
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(b2 + 8 * (k & 3)));
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v2[0]), "=r"(v2[1]), "=r"(v2[2]), "=r"(v2[3]), "=r"(v2[4]), "=r"(v2[5]), "=r"(v2[6]), "=r"(v2[7]) : "r"(b2 + 128 + 8 * (k & 3)));
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v3[0]), "=r"(v3[1]), "=r"(v3[2]), "=r"(v3[3]), "=r"(v3[4]), "=r"(v3[5]), "=r"(v3[6]), "=r"(v3[7]) : "r"(b2 + 256 + 8 * (k & 3)));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          for (int i = 0; i < 8; i++) acc += __uint_as_float(v[i]) + __uint_as_float(v2[i]) + __uint_as_float(v3[i]);
          const int row = tid & 63, blk = 8 + (k & 7) + 8 * ((it >> 3) % 3);
          *reinterpret_cast<uint4*>(smem + (row >> 3) * 4096 + blk * 128 + (row & 7) * 16) = make_uint4(0x3c00u, 0, 0, 0);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (mode >= 11) asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (mode >= 12 && lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&never)));
        }
        if (mode == 4) { uint32_t q; asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(q) : "r"(smem_u32(sbuf + 16 * (k & 15)))); acc += q; }
      }
      __syncwarp();
      it++;
    }
  }
  if (acc == 12345.f) out[31] = 1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(512));
}
int main() {
  long long* d; cudaMalloc(&d, 32 * 8);
  const int smem = 196608 + 16384;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"none", "tcgen05.ld", "st.shared", "try_wait spin", "ld.shared", "ld+sts", "sts A-region", "tcgen05.ld D", "random data", "random, 148 SMs", "epi: ld3+sts+pfence", "epi +tc fence", "epi +arrive"};
  for (int mode = 0; mode < 13; mode++) {
    cudaMemset(d, 0, 256);
    probe<<<mode == 9 ? 148 : 2, 512, smem>>>(d, mode == 9 ? 8 : mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    long long h[32]; cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
    printf("%-14s:", names[mode]);
    for (int r = 0; r < 8; r++) printf(" %lld/%lld", h[2 * r], h[2 * r + 1]);
    printf("   (issue/complete cycles for 12 MMAs)\n");
  }
  return 0;
}
