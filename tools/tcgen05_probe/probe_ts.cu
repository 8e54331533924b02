// Probe: tcgen05.mma kind::f16 with A from TMEM (M=128, K=256 in 16 steps), B from shared
// memory MN-major (N=32), D in TMEM; plus timing of back-to-back TMEM-A MMAs.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
constexpr int M = 128, N = 32, K = 256;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0; d |= (uint64_t)((saddr >> 4) & 0x3FFF); d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32; d |= (uint64_t)1 << 46; return d; }
// B (N x K) MN-major: (p, c) at (c/8)*((N/8)*128) + (p/8)*128 + (c%8)*16 + (p%8)*2
__host__ __device__ inline uint32_t b_off(int p, int c) { return (c >> 3) * ((N / 8) * 128) + (p >> 3) * 128 + (c & 7) * 16 + (p & 7) * 2; }
__global__ void probe(const __half* A, const __half* B, float* D, long long* cyc, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar; __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31;
  for (int e = tid; e < N * K; e += blockDim.x) { int p = e / K, c = e % K; *(__half*)(smem + b_off(p, c)) = B[p * K + c]; }
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1)); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;        // columns [0,32): D; [128, 256): A (128 columns = 256 fp16)
  // A row m = lane 32w + l; column 128 + c holds (A[m][2c], A[m][2c+1]) as a half2
  {
    const int m = warp * 32 + lane;
    for (int c0 = 0; c0 < 128; c0 += 8) {
      uint32_t r[8];
      for (int i = 0; i < 8; i++) { __half2 h = __halves2half2(A[m * K + 2 * (c0 + i)], A[m * K + 2 * (c0 + i) + 1]); r[i] = *(uint32_t*)&h; }
      const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16) + 128 + c0;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (0u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (tid == 0) {
    long long t0 = clock64();
    for (int r = 0; r < reps; r++)
      for (int ks = 0; ks < 16; ks++) {
        const uint32_t a_t = tm + 128 + ks * 8;
        const uint64_t b = make_desc(smem_u32(smem) + ks * 2 * ((N / 8) * 128), (N / 8) * 128, 128);
        const uint32_t acc = ks > 0;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" :: "r"(tm), "r"(a_t), "l"(b), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
    uint32_t done = 0;
    while (!done) asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    cyc[0] = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    uint32_t r[32];
    const uint32_t a = tm + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]) : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int c = 0; c < 32; c++) D[(warp * 32 + lane) * N + c] = __uint_as_float(r[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(256));
}
int main() {
  std::vector<__half> A(M * K), B(N * K); std::vector<float> Af(M * K), Bf(N * K);
  srand(3);
  for (int i = 0; i < M * K; i++) { float v = (float)(rand() % 64 - 32) / 16.f; A[i] = __float2half(v); Af[i] = v; }
  for (int i = 0; i < N * K; i++) { float v = (float)(rand() % 64 - 32) / 8.f; B[i] = __float2half(v); Bf[i] = v; }
  std::vector<double> ref(M * N);
  for (int m = 0; m < M; m++) for (int n = 0; n < N; n++) { double s = 0; for (int k = 0; k < K; k++) s += (double)Af[m * K + k] * Bf[n * K + k]; ref[m * N + n] = s; }
  __half *dA, *dB; float* dD; long long* dc;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), M * K * 2, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), N * K * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, N * K * 2);
  for (int reps : {1, 100}) {
    probe<<<1, 128, N * K * 2>>>(dA, dB, dD, dc, reps);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(M * N); long long cyc; cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost); cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    double maxerr = 0; for (int i = 0; i < M * N; i++) maxerr = fmax(maxerr, fabs(D[i] - ref[i]));
    printf("reps=%d err=%s maxerr(vs 1 pass)=%.3g  %.1f cycles per MMA\n", reps, cudaGetErrorString(e), reps == 1 ? maxerr : -1.0, (double)cyc / (reps * 16));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
