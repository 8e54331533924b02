// Probe of the tcgen05 building blocks the dense kernel uses (sm_100a):
// kind::f16 MMA M=128 N=32 K=16, A/B in shared memory (no swizzle, K-major and MN-major A),
// fp32 accumulator in TMEM, tcgen05.commit -> mbarrier, tcgen05.ld 32x32b.x32.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int M = 128, N = 32, K = 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// no-swizzle K-major canonical layout: core matrix = 8 rows x 16 bytes (8 fp16 along K)
// offset(r, k) = (r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2
__host__ __device__ inline uint32_t kmaj_off(int r, int k, uint32_t lbo, uint32_t sbo) {
  return (r / 8) * sbo + (k / 8) * lbo + (r % 8) * 16 + (k % 8) * 2;
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}

__device__ __forceinline__ uint32_t make_idesc(int m, int n, int a_major, int b_major) {
  uint32_t d = 0;
  d |= 1u << 4;              // c_format F32
  d |= 0u << 7;              // a_format F16
  d |= 0u << 10;             // b_format F16
  d |= (uint32_t)a_major << 15;
  d |= (uint32_t)b_major << 16;
  d |= (uint32_t)(n >> 3) << 17;
  d |= (uint32_t)(m >> 4) << 24;
  return d;
}

__global__ void probe(const __half* A, const __half* B, float* D, int a_mn_major) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                 // 128 x 256 fp16 = 64 KB
  uint8_t* sB = smem + 65536;         // 32 x 256 fp16 = 16 KB
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  // A layout: K-major: rows m, LBO = 128 (next 8-k chunk), SBO = 32*128 = 4096 (next 8-row block)
  // A MN-major test: store A^T in K-major form (rows = k, "K" = m) and describe it as MN-major.
  for (int e = tid; e < M * K; e += blockDim.x) {
    int m = e / K, k = e % K;
    __half val = A[m * K + k];
    uint32_t off = a_mn_major ? kmaj_off(k, m, 128, (M / 8) * 128) : kmaj_off(m, k, 128, (K / 8) * 128);
    *(__half*)(sA + off) = val;
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    int nn = e / K, k = e % K;
    *(__half*)(sB + kmaj_off(nn, k, 128, (K / 8) * 128)) = B[nn * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");   // generic-proxy smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = make_idesc(M, N, a_mn_major ? 1 : 0, 0);
    for (int ks = 0; ks < K / 16; ks++) {
      uint64_t adesc, bdesc;
      if (!a_mn_major) {
        adesc = make_desc(smem_u32(sA) + ks * 2 * 128, 128, (K / 8) * 128);
      } else {
        // MN-major: MN blocks of 8 m at stride 128 B (SBO), K blocks of 8 k at stride (M/8)*128 (LBO)
        adesc = make_desc(smem_u32(sA) + ks * 2 * (M / 8) * 128, (M / 8) * 128, 128);
      }
      bdesc = make_desc(smem_u32(sB) + ks * 2 * 128, 128, (K / 8) * 128);
      const uint32_t acc = ks > 0;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                   :: "r"(taddr), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  // wait for the MMA to complete (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    uint32_t r[32];
    const uint32_t a = taddr + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = warp * 32 + (tid & 31);
    for (int c = 0; c < 32; c++) D[row * N + c] = __uint_as_float(r[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(32));
}

int main() {
  std::vector<__half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K);
  srand(1);
  for (int i = 0; i < M * K; i++) { float v = (float)(rand() % 64 - 32) / 16.f; A[i] = __float2half(v); Af[i] = v; }
  for (int i = 0; i < N * K; i++) { float v = (float)(rand() % 64 - 32) / 8.f; B[i] = __float2half(v); Bf[i] = v; }
  std::vector<double> ref(M * N);
  for (int m = 0; m < M; m++) for (int n = 0; n < N; n++) { double s = 0; for (int k = 0; k < K; k++) s += (double)Af[m * K + k] * Bf[n * K + k]; ref[m * N + n] = s; }
  __half *dA, *dB; float* dD;
  CK(cudaMalloc(&dA, M * K * 2)); CK(cudaMalloc(&dB, N * K * 2)); CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), M * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), N * K * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 16384));
  for (int mn = 0; mn < 2; mn++) {
    CK(cudaMemset(dD, 0, M * N * 4));
    probe<<<1, 128, 65536 + 16384>>>(dA, dB, dD, mn);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> D(M * N);
    CK(cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0; int bad = 0;
    for (int i = 0; i < M * N; i++) { double e = fabs(D[i] - ref[i]); if (e > maxerr) maxerr = e; if (e > 1e-3) bad++; }
    printf("a_mn_major=%d max err %.3g bad %d  D[0]=%f ref %f D[77*32+5]=%f ref %f\n", mn, maxerr, bad, D[0], ref[0], D[77*32+5], ref[77*32+5]);
  }
  return 0;
}
