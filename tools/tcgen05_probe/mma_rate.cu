// Throughput probe: back-to-back tcgen05.mma kind::f16 M=128, K=16, N in {32,64,128,256},
// A/B from shared memory (no swizzle), one CTA per SM, one issuing thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32; d |= (uint64_t)1 << 46; return d; }
template <int N, int AMN, int NACC>
__global__ void rate(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar; __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (128 * 256 + N * 256) / 8; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3c003c00u, 0, 0x3c003c00u, 0);
  constexpr int NA = NACC == 99 ? 1 : NACC;
  constexpr int COLS = (N * NA < 32 ? 32 : (N * NA <= 64 ? 64 : (N * NA <= 128 ? 128 : (N * NA <= 256 ? 256 : 512))));
  if (threadIdx.x < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1)); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;"); asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t sa = smem_u32(smem), sb = sa + 128 * 256 * 2;
  uint32_t idesc = (1u << 4) | ((uint32_t)AMN << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    if (NACC == 99) {   // incremental descriptors, fully unrolled K loop
      const uint64_t a0 = make_desc(sa, 128, 4096), b0 = make_desc(sb, (N / 8) * 128, 128);
      for (int r = 0; r < reps; r++) {
        uint64_t a = a0, b = b0;
#pragma unroll
        for (int ks = 0; ks < 16; ks++) {
          const uint32_t acc = (r | ks) ? 1u : 0u;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(tbase), "l"(a), "l"(b), "r"(idesc), "r"(acc));
          a += 256 >> 4; b += (2 * (N / 8) * 128) >> 4;
        }
      }
    } else
    for (int r = 0; r < reps; r++) {
      for (int ks = 0; ks < 16; ks++) {
        uint64_t a = AMN ? make_desc(sa + ks * 2 * 4096, 4096, 128) : make_desc(sa + ks * 256, 128, 4096);
        uint64_t b = make_desc(sb + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
        uint32_t acc = (r | (ks / NA)) ? 1u : 0u;
        const uint32_t dcol = tbase + (uint32_t)((ks % NA) * N);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(dcol), "l"(a), "l"(b), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
    uint32_t done = 0;
    while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase), "r"(COLS));
}
template <int N, int AMN, int NACC> void run() {
  long long* d; cudaMalloc(&d, 148 * 8);
  int smem = 128 * 256 * 2 + N * 256 * 2;
  cudaFuncSetAttribute(rate<N, AMN, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int reps = 200;
  rate<N, AMN, NACC><<<148, 128, smem>>>(d, reps);
  cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double cyc = (double)h[0] / (reps * 16);
  printf("NACC=%d N=%3d A_MN=%d: %.1f cycles per MMA (128x%dx16) -> %.0f MAC/clk/SM  err=%s\n", NACC, N, AMN, cyc, N, 128.0 * N * 16 / cyc, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() { run<32,0,1>(); run<32,0,99>(); run<64,0,99>(); run<128,0,99>(); run<256,0,99>(); return 0; }
