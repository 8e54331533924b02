// Probe (N sweep): cta_group::2 tcgen05.mma kind::f16, M=128 (64 rows per CTA), N = 64 / 128 / 256 issued
// as 256/N instructions per K step into adjacent D columns (the N-split of the dense kernel), K=256 in 16 steps,
// A and B from shared memory split across the CTA pair, multicast commit, TMEM layout of D.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
constexpr int M = 128, N = 256, K = 256;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32; d |= (uint64_t)1 << 46; return d; }
__host__ __device__ inline uint32_t kmaj(int r, int k) { return (r >> 3) * ((K / 8) * 128) + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2; }
template <int NI>
__global__ void __cluster_dims__(2, 1, 1) probe(const __half* A, const __half* B, float* Dout, long long* cyc, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                    // 64 x 256 fp16 = 32 KB
  uint8_t* sB = smem + 64 * K * 2;       // 128 x 256 fp16 = 64 KB
  __shared__ __align__(8) uint64_t mbar; __shared__ uint32_t tbase;
  uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31;
  for (int e = tid; e < 64 * K; e += blockDim.x) { int r = e / K, k = e % K; *(__half*)(sA + kmaj(r, k)) = A[(rank * 64 + r) * K + k]; }
  for (int e = tid; e < 128 * K; e += blockDim.x) { int r = e / K, k = e % K; *(__half*)(sB + kmaj(r, k)) = B[(rank * 128 + r) * K + k]; }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1)); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(NI >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  long long t0 = clock64();
  if (rank == 0 && tid == 0) {
    const uint64_t a0 = make_desc(smem_u32(sA), 128, (K / 8) * 128), b0 = make_desc(smem_u32(sB), 128, (K / 8) * 128);
    for (int r = 0; r < reps; r++) {
      uint64_t a = a0, b = b0;
#pragma unroll
      for (int ks = 0; ks < 16; ks++) {
        const uint32_t acc = (ks > 0) ? 1u : 0u;   // every rep recomputes the same product
#pragma unroll
        for (int nb = 0; nb < N / NI; nb++) {
          // N block nb: B rows [NI/2 nb, NI/2 (nb+1)) of each CTA's half -> D columns [NI/2 nb, ...)
          const uint64_t bo = (uint64_t)(((NI / 2) * nb / 8) * ((K / 8) * 128)) >> 4;
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" :: "r"(tm + (uint32_t)((NI / 2) * nb)), "l"(a), "l"(b + bo), "r"(idesc), "r"(acc));
        }
        a += 256 >> 4; b += 256 >> 4;
      }
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "h"((uint16_t)3));
  }
  { uint32_t done = 0; while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0)); }
  if (tid == 0) cyc[rank] = clock64() - t0;
  asm volatile("tcgen05.fence::after_thread_sync;");
  // read all 128 lanes x 128 columns of this CTA's TMEM
  for (int c0 = 0; c0 < 128; c0 += 32) {
    uint32_t r[32];
    const uint32_t a = tm + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int c = 0; c < 32; c++) Dout[(rank * 128 + warp * 32 + lane) * 128 + c0 + c] = __uint_as_float(r[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(128));
}
template <int NI> int run();
int main() { return run<256>() | run<128>() | run<64>(); }
template <int NI> int run() {
  std::vector<__half> A(M * K), B(N * K); std::vector<float> Af(M * K), Bf(N * K);
  srand(7);
  for (int i = 0; i < M * K; i++) { float v = (float)(rand() % 64 - 32) / 16.f; A[i] = __float2half(v); Af[i] = v; }
  for (int i = 0; i < N * K; i++) { float v = (float)(rand() % 64 - 32) / 8.f; B[i] = __float2half(v); Bf[i] = v; }
  std::vector<double> ref(M * N);
  for (int m = 0; m < M; m++) for (int n = 0; n < N; n++) { double s = 0; for (int k = 0; k < K; k++) s += (double)Af[m * K + k] * Bf[n * K + k]; ref[m * N + n] = s; }
  __half *dA, *dB; float* dD; long long* dc;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, 2 * 128 * 128 * 4); cudaMalloc(&dc, 16);
  cudaMemcpy(dA, A.data(), M * K * 2, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), N * K * 2, cudaMemcpyHostToDevice);
  const int smem = 64 * K * 2 + 128 * K * 2;
  cudaFuncSetAttribute(probe<NI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int reps : {1, 200}) {
    cudaMemset(dD, 0, 2 * 128 * 128 * 4);
    probe<NI><<<2, 128, smem>>>(dA, dB, dD, dc, reps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("reps=%d err=%s\n", reps, cudaGetErrorString(e)); return 1; }
    std::vector<float> D(2 * 128 * 128); long long cyc[2];
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost); cudaMemcpy(cyc, dc, 16, cudaMemcpyDeviceToHost);
    // hypothesis (CUTLASS 2SM M=128 "2x2" atom): CTA r, lane l < 64: row 64 r + l, cols n = c;
    //   lane l >= 64: row 64 r + (l - 64), cols n = 128 + c
    double maxerr = 0; int bad = 0;
    for (int r = 0; r < 2; r++) for (int l = 0; l < 128; l++) for (int c = 0; c < 128; c++) {
      const int row = 64 * r + (l & 63), col = (l < 64 ? 0 : 128) + c;
      const double e2 = fabs(D[(r * 128 + l) * 128 + c] - ref[row * N + col]);
      if (e2 > maxerr) maxerr = e2; if (e2 > 1e-3) bad++;
    }
    printf("NI=%d reps=%d 2x2-layout maxerr %.3g bad %d ; cycles %lld %lld -> %.1f cycles per K step of N=256 (%d instr)\n", NI, reps, maxerr, bad, cyc[0], cyc[1], (double)cyc[0] / (reps * 16), N / NI);
    if (bad) { // print a few raw values to help locate
      for (int l : {0, 1, 63, 64, 65, 127}) printf("  cta0 lane %d col0 %.4f (ref row %d: %.4f / %.4f)\n", l, D[l * 128], l & 63, ref[(l & 63) * N], ref[(l & 63) * N + 128]);
    }
  }
  return 0;
}
