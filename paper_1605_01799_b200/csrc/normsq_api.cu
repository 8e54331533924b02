// normsq_api.cu — C ABI of NEXT-3 (hopf_eval_normsq, include/hopf.h): argument validation,
// variant selection and launch of hopf_normsq_kernel (normsq_kernel.cuh).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../include/hopf.h"
#include "common.cuh"
#include "normsq_kernel.cuh"

namespace hopf {
extern thread_local int32_t g_last_threads, g_last_blocks;
extern thread_local unsigned long long *g_iter_counter;

using NormsqFn = void (*)(const NormsqParams);
struct NormsqVariant {
  int G, CPL;
  NormsqFn fn[2][5];   // [J kind][H kind] (no ELL)
};
#define HOPF_NSQ_JH(G_, C_, J_)                                                                \
  {hopf_normsq_kernel<G_, C_, J_, HK_L1>, hopf_normsq_kernel<G_, C_, J_, HK_WL1>,              \
   hopf_normsq_kernel<G_, C_, J_, HK_L2>, nullptr, hopf_normsq_kernel<G_, C_, J_, HK_LINF>}
#define HOPF_NSQ_VARIANT(G_, C_) {G_, C_, {HOPF_NSQ_JH(G_, C_, JK_L1SQ), HOPF_NSQ_JH(G_, C_, JK_LINFSQ)}}
// thread per point up to n = 8, pairs of lanes up to 16 (the paper's Tables 2, 3 and 5 use
// n = 4..16; at n = 16 (t5): (2, 8) 24.7 ms, (4, 4) 29.5, (1, 16) 31.6, (8, 2) 40.3, (4, 16) 77.5),
// then groups
static const NormsqVariant kNormsqVariants[] = {
    HOPF_NSQ_VARIANT(1, 4),  HOPF_NSQ_VARIANT(1, 8),   HOPF_NSQ_VARIANT(2, 8),
    HOPF_NSQ_VARIANT(4, 16), HOPF_NSQ_VARIANT(16, 16), HOPF_NSQ_VARIANT(32, 16)};
}  // namespace hopf

using namespace hopf;

extern "C" int hopf_eval_normsq(int64_t M, int32_t n, const float *X, const float *t,
                                hopf_j_kind j, float gamma, hopf_h_kind h, const float *w,
                                float lambda, int32_t max_iter, float tol, float *phi,
                                float *grad, int32_t *iters, hopf_stream_t stream) {
  g_launches = 0;
  if (M < 0 || n < 1) return set_error(HOPF_EINVAL, "M=%lld n=%d", (long long)M, n);
  if ((int)j < 0 || (int)j > 1) return set_error(HOPF_EINVAL, "unknown J kind %d", (int)j);
  if (!(h == HOPF_H_L1 || h == HOPF_H_WL1 || h == HOPF_H_L2 || h == HOPF_H_LINF))
    return set_error(HOPF_EINVAL, "H kind %d is not available with hopf_eval_normsq", (int)h);
  if (!(lambda > 0.f) || !std::isfinite(lambda)) return set_error(HOPF_EINVAL, "lambda must be > 0 and finite");
  if (!(tol >= 0.f) || !std::isfinite(tol)) return set_error(HOPF_EINVAL, "tol must be >= 0");
  if (max_iter < 1) return set_error(HOPF_EINVAL, "max_iter must be >= 1");
  if (h == HOPF_H_WL1 && !w) return set_error(HOPF_EINVAL, "w is required for HOPF_H_WL1");
  const NormsqVariant *v = nullptr;
  static const char *force = getenv("HOPF_NSQ_VARIANT");
  if (force) {
    int fg = 0, fc = 0;
    if (sscanf(force, "%d,%d", &fg, &fc) == 2)
      for (const NormsqVariant &c : kNormsqVariants)
        if (c.G == fg && c.CPL == fc && fg * fc >= n) { v = &c; break; }
  }
  if (!v)
    for (const NormsqVariant &c : kNormsqVariants)
      if (c.G * c.CPL >= n) { v = &c; break; }
  if (!v) return set_error(HOPF_EUNSUPPORTED, "hopf_eval_normsq supports n <= 512 (n=%d)", n);
  if (M == 0) return HOPF_OK;
  if (!X || !t || !phi || !grad || !iters) return set_error(HOPF_EINVAL, "a required pointer is NULL");
  NormsqParams p{};
  p.M = M; p.n = n; p.X = X; p.t = t; p.w = h == HOPF_H_WL1 ? w : nullptr;
  p.gamma = gamma; p.lambda = lambda; p.tol = tol; p.max_iter = max_iter; p.h = (int)h;
  p.phi = phi; p.grad = grad; p.iters = iters; p.iter_total = g_iter_counter;
  NormsqFn fn = v->fn[(int)j][(int)h];
  const int threads = 128;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  int64_t blocks = (int64_t)num_sms() * per_sm;
  const int64_t need = (M * v->G + threads - 1) / threads;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  int rc = claim_counter(M, blocks * threads / v->G, (cudaStream_t)stream, &p.claim);
  if (rc != HOPF_OK) return rc;
  fn<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(p);
  scratch_free(p.claim, (cudaStream_t)stream);
  g_launches = 1;
  g_last_threads = threads;
  g_last_blocks = (int)blocks;
  g_last_kernel = j == HOPF_J_L1SQ ? "hopf_normsq_kernel<l1sq>" : "hopf_normsq_kernel<linfsq>";
  return check_launch("hopf_normsq_kernel");
}

// ---------------------------------------------------------------- NEXT-2: ||.||_A, full SPD A
#include "ella_kernel.cuh"

extern "C" int hopf_eval_diag_A(int64_t M, int32_t n, const float *X, const float *t,
                                const float *Dj, const float *c, float gamma, const float *Q,
                                const float *Lam, float lambda, int32_t max_iter, float tol,
                                float *phi, float *grad, int32_t *iters, hopf_stream_t stream) {
  using namespace hopf;
  g_launches = 0;
  if (M < 0 || n < 1) return set_error(HOPF_EINVAL, "M=%lld n=%d", (long long)M, n);
  if (!(lambda > 0.f) || !std::isfinite(lambda)) return set_error(HOPF_EINVAL, "lambda must be > 0 and finite");
  if (!(tol >= 0.f) || !std::isfinite(tol)) return set_error(HOPF_EINVAL, "tol must be >= 0");
  if (max_iter < 1) return set_error(HOPF_EINVAL, "max_iter must be >= 1");
  if (n > 128) return set_error(HOPF_EUNSUPPORTED, "hopf_eval_diag_A supports n <= 128 (n=%d)", n);
  if (M == 0) return HOPF_OK;
  if (!X || !t || !Dj || !Q || !Lam || !phi || !grad || !iters)
    return set_error(HOPF_EINVAL, "a required pointer is NULL");
  EllAParams p{};
  p.M = M; p.n = n; p.X = X; p.t = t; p.D = Dj; p.c = c; p.Q = Q; p.Lam = Lam;
  p.gamma = gamma; p.lambda = lambda; p.tol = tol; p.max_iter = max_iter;
  p.phi = phi; p.grad = grad; p.iters = iters; p.iter_total = g_iter_counter;
  // two points per warp up to n = 16, then one
  // n <= 16 (the paper's sizes): G lanes per point, 32/G points per warp; HOPF_ELLA_G selects
  // G in {2, 4, 8, 16} (experiments)
  static const char *ev = getenv("HOPF_ELLA_G");
  const int gsel = ev ? atoi(ev) : 2;   // t4a (n = 16): G=2 2.41 ms, 4 2.61, 8 2.75, 16 5.3
  void (*fn)(const EllAParams);
  int gpw = 1;
  if (n <= 16) {
    switch (gsel) {
      case 2: fn = hopf_ella_kernel<2, 8>; gpw = 16; break;
      case 4: fn = hopf_ella_kernel<4, 4>; gpw = 8; break;
      case 16: fn = hopf_ella_kernel<16, 1>; gpw = 2; break;
      case 8: fn = hopf_ella_kernel<8, 2>; gpw = 4; break;
      default: fn = hopf_ella_kernel<2, 8>; gpw = 16; break;
    }
  } else {
    fn = n <= 32 ? hopf_ella_kernel<32, 1> : (n <= 64 ? hopf_ella_kernel<32, 2> : hopf_ella_kernel<32, 4>);
  }
  const size_t nr = (size_t)((n + 15) & ~15);   // as ella_kernel.cuh
  const size_t smem = sizeof(float) * ((size_t)2 * n * nr + n + (size_t)ELLA_WARPS * gpw * n);
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * ELLA_WARPS, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  int64_t blocks = (int64_t)num_sms() * per_sm;
  const int64_t need = (M + ELLA_WARPS * gpw - 1) / (ELLA_WARPS * gpw);
  if (blocks > need) blocks = need;
  int rc = claim_counter(M, blocks * ELLA_WARPS * gpw, (cudaStream_t)stream, &p.claim);
  if (rc != HOPF_OK) return rc;
  fn<<<(unsigned)blocks, 32 * ELLA_WARPS, smem, (cudaStream_t)stream>>>(p);
  scratch_free(p.claim, (cudaStream_t)stream);
  g_launches = 1;
  g_last_threads = 32 * ELLA_WARPS;
  g_last_blocks = (int)blocks;
  g_last_kernel = "hopf_ella_kernel";
  return check_launch("hopf_ella_kernel");
}
