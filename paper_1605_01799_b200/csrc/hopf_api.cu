// hopf_api.cu — the C ABI of libhopf.so (declared in include/hopf.h).
// Argument validation, kernel-variant selection and launch; no arithmetic of the method
// happens on the host except the fp64 dense-plan construction (dense_plan.cu).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hopf.h"
#include "common.cuh"
#include "diag_kernel.cuh"
#include "diag_tm.cuh"
#include "tmg_api.h"

namespace hopf {

thread_local std::string g_last_error;
thread_local int32_t g_launches = 0;
thread_local int32_t g_last_threads = 0, g_last_blocks = 0;
thread_local const char *g_last_kernel = "";
thread_local unsigned long long *g_iter_counter = nullptr;

int set_error(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(HOPF_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return HOPF_OK;
}

int num_sms() {
  static std::atomic<int> sms[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int v = sms[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

int scratch_alloc(void **ptr, size_t bytes, cudaStream_t stream) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  *ptr = nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return set_error(HOPF_EINVAL, "device index %d", dev);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      cudaMemPool_t p = nullptr;
      if (cudaMemPoolCreate(&p, &props) != cudaSuccess)
        return set_error(HOPF_ECUDA, "cudaMemPoolCreate failed");
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
      pools[dev] = p;
    }
    pool = pools[dev];
  }
  if (bytes == 0) return HOPF_OK;
  cudaError_t e = cudaMallocFromPoolAsync(ptr, bytes, pool, stream);
  if (e != cudaSuccess) {
    *ptr = nullptr;
    return set_error(HOPF_ECUDA, "scratch allocation of %zu bytes: %s", bytes, cudaGetErrorString(e));
  }
  return HOPF_OK;
}

void scratch_free(void *ptr, cudaStream_t stream) {
  if (ptr) cudaFreeAsync(ptr, stream);
}

int claim_counter(int64_t M, int64_t resident, cudaStream_t stream, unsigned long long **ctr) {
  *ctr = nullptr;
  // HOPF_CLAIMS=0 / 1: never / always (tests and A/B runs); default: M >= 8 x resident
  const char *env = getenv("HOPF_CLAIMS");   // read per launch: tests switch it
  const int mode = env ? atoi(env) : -1;
  if (mode == 0 || (mode != 1 && M < 8 * resident)) return HOPF_OK;
  const int rc = scratch_alloc((void **)ctr, sizeof(unsigned long long), stream);
  if (rc != HOPF_OK) return rc;
  cudaMemsetAsync(*ctr, 0, sizeof(unsigned long long), stream);
  return HOPF_OK;
}

// ---------------------------------------------------------------- diag / union variants
using KernFn = void (*)(const DiagParams);

struct Variant {
  int G, CPL;
  KernFn fn[3][2];  // [h kind][union]
};

// union kernels: n <= 256 (G * CPL <= 256), CPL <= 32
template <int G, int C, int H>
constexpr KernFn union_fn() {
  if constexpr (C <= 32 && G * C <= 256) return hopf_diag_kernel<G, C, H, true>;
  else return nullptr;
}
#define HOPF_VARIANT(G_, C_)                                                                 \
  {G_, C_,                                                                                   \
   {{hopf_diag_kernel<G_, C_, HK_L1, false>, union_fn<G_, C_, HK_L1>()},                     \
    {hopf_diag_kernel<G_, C_, HK_WL1, false>, union_fn<G_, C_, HK_WL1>()},                   \
    {hopf_diag_kernel<G_, C_, HK_L2, false>, union_fn<G_, C_, HK_L2>()}}}

// Ordered by padded width G*CPL (roughly), then G: the first variant with G*CPL >= n is used.
// (8, 13) precedes (4, 25): for C2 (n = 100) its 127 registers give 4 warps per SMSP instead of 3
// (1.995 vs 2.070 ms) despite 4 % padding.
static const Variant kVariants[] = {
    HOPF_VARIANT(1, 1),  HOPF_VARIANT(1, 2),  HOPF_VARIANT(1, 4),   HOPF_VARIANT(1, 8),
    HOPF_VARIANT(1, 16), HOPF_VARIANT(2, 12), HOPF_VARIANT(2, 16),  HOPF_VARIANT(4, 16),
    HOPF_VARIANT(8, 13), HOPF_VARIANT(4, 25), HOPF_VARIANT(4, 32), HOPF_VARIANT(8, 16),
    HOPF_VARIANT(8, 32),
    HOPF_VARIANT(16, 32), HOPF_VARIANT(32, 32)};

// HOPF_H_ELL (hopf_eval_diag only): its own list.  The projection adds per-point scalar work and
// group reductions (Newton on mu); measured on C2e (n = 100): (8, 13) 5.3 ms, (16, 7) 6.5 ms,
// (32, 4) 8.2 ms, so narrow groups first, as in the main list.
// HOPF_H_LINF (same entry points) uses the same list with its own instantiations.
#define HOPF_X_VARIANT(HK_, G_, C_) {G_, C_, {{hopf_diag_kernel<G_, C_, HK_, false>, nullptr}}}
#define HOPF_X_VARIANTS(HK_)                                                                 \
  {HOPF_X_VARIANT(HK_, 1, 4),  HOPF_X_VARIANT(HK_, 2, 4),   HOPF_X_VARIANT(HK_, 4, 4),       \
   HOPF_X_VARIANT(HK_, 8, 4),  HOPF_X_VARIANT(HK_, 16, 4),  HOPF_X_VARIANT(HK_, 8, 13),      \
   HOPF_X_VARIANT(HK_, 16, 7), HOPF_X_VARIANT(HK_, 32, 4),  HOPF_X_VARIANT(HK_, 32, 8),      \
   HOPF_X_VARIANT(HK_, 32, 16), HOPF_X_VARIANT(HK_, 32, 32)}
static const Variant kEllVariants[] = HOPF_X_VARIANTS(HK_ELL);
static const Variant kLinfVariants[] = HOPF_X_VARIANTS(HK_LINF);

static const Variant *pick_variant(int n, bool is_union, int hx = -1) {
  if (hx == HK_ELL || hx == HK_LINF) {
    const Variant *list = hx == HK_ELL ? kEllVariants : kLinfVariants;
    const int cnt = (int)(sizeof(kEllVariants) / sizeof(kEllVariants[0]));
    static const char *force = getenv("HOPF_DIAG_VARIANT");
    if (force) {
      int fg = 0, fc = 0;
      if (sscanf(force, "%d,%d", &fg, &fc) == 2)
        for (int i = 0; i < cnt; i++)
          if (list[i].G == fg && list[i].CPL == fc && fg * fc >= n) return &list[i];
    }
    for (int i = 0; i < cnt; i++)
      if (list[i].G * list[i].CPL >= n) return &list[i];
    return nullptr;
  }
  // HOPF_DIAG_VARIANT=G,CPL forces a variant (experiments)
  static const char *force = getenv("HOPF_DIAG_VARIANT");
  if (force) {
    int fg = 0, fc = 0;
    if (sscanf(force, "%d,%d", &fg, &fc) == 2)
      for (const Variant &v : kVariants)
        if (v.G == fg && v.CPL == fc && v.G * v.CPL >= n && (!is_union || v.fn[0][1])) return &v;
  }
  for (const Variant &v : kVariants) {
    if (v.G * v.CPL < n) continue;
    if (is_union && v.fn[0][1] == nullptr) continue;
    return &v;
  }
  return nullptr;
}

// Wide points (the (32, 32) variant, n in (512, 1024]), not union: the kernel that keeps x_hat,
// v, kappa (and tau) in tensor memory (diag_tm.cuh).  HOPF_DIAG_TM=0 selects the register kernel.
static int launch_diag_tm(const DiagParams &p, hopf_h_kind h, cudaStream_t stream) {
  using namespace dtm;
  KernFn fn = h == HOPF_H_L2 ? hopf_diag_tm_kernel<HK_L2>
              : (h == HOPF_H_WL1 ? hopf_diag_tm_kernel<HK_WL1> : hopf_diag_tm_kernel<HK_L1>);
  // the attribute is per device: one flag bit per (device, H kind)
  static std::atomic<uint32_t> attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint32_t bit = 1u << (int)h;
  if (dev < 0 || dev >= 64 || !(attr_done[dev].load(std::memory_order_relaxed) & bit)) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, DYN_SMEM);
    if (dev >= 0 && dev < 64) attr_done[dev].fetch_or(bit, std::memory_order_relaxed);
  }
  int64_t blocks = (int64_t)num_sms() * 4;
  const int64_t need = (p.M + 3) / 4;   // 4 points (warps) per block
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  DiagParams q = p;
  int rc = claim_counter(p.M, blocks * (THREADS / 32), stream, &q.claim);
  if (rc != HOPF_OK) return rc;
  fn<<<(unsigned)blocks, THREADS, DYN_SMEM, stream>>>(q);
  scratch_free(q.claim, stream);
  g_launches += 1;
  g_last_threads = THREADS;
  g_last_blocks = (int)blocks;
  g_last_kernel = h == HOPF_H_L2 ? "hopf_diag_tm_kernel<l2>"
                  : (h == HOPF_H_WL1 ? "hopf_diag_tm_kernel<wl1>" : "hopf_diag_tm_kernel<l1>");
  return check_launch("hopf_diag_tm_kernel");
}

// ---------------------------------------------------------------- NEXT-4 helpers
// istar = 0 where the first solve is valid, -1 on invalid points
__global__ void hopf_istar_init_kernel(int64_t M, const int32_t *iters, int32_t *istar) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
    istar[i] = iters[i] == INT32_MIN ? -1 : 0;
}
// one warp per point: keep the larger phi (strict: the lowest i wins ties; NaN never wins)
__global__ void hopf_maxh_combine_kernel(int64_t M, int n, int idx, const float *phi_i,
                                         const float *grad_i, const int32_t *it_i, float *phi,
                                         float *grad, int32_t *iters, int32_t *istar) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = w0; p < M; p += nw) {
    const bool win = phi_i[p] > phi[p];
    if (win) {
      for (int j = lane; j < n; j += 32) grad[p * n + j] = grad_i[p * n + j];
      if (lane == 0) { phi[p] = phi_i[p]; iters[p] = it_i[p]; if (istar) istar[p] = idx; }
    }
  }
}

static int launch_diag_like(const DiagParams &p_in, hopf_h_kind h, bool is_union,
                            cudaStream_t stream) {
  DiagParams p = p_in;
  p.iter_total = g_iter_counter;
  const bool ell = h == HOPF_H_ELL || h == HOPF_H_LINF;
  if (ell && is_union)
    return set_error(HOPF_EUNSUPPORTED, "HOPF_H_ELL / HOPF_H_LINF are supported by hopf_eval_diag only");
  const Variant *v = pick_variant(p.n, is_union, h == HOPF_H_ELL ? HK_ELL : (h == HOPF_H_LINF ? HK_LINF : -1));
  if (!v) return set_error(HOPF_EUNSUPPORTED, "n=%d exceeds the compiled diag kernels", p.n);
  static const char *tm_env = getenv("HOPF_DIAG_TM");
  if (!ell && !is_union && v->G == 32 && v->CPL == 32 && !(tm_env && strcmp(tm_env, "0") == 0))
    return launch_diag_tm(p, h, stream);
  {   // grouped TMEM kernels (tmg_api.cu) where a variant fits
    bool handled = false;
    const int rc = tmg_try_launch(p, (int)h, is_union, stream, &handled);
    if (handled) return rc;
  }
  KernFn fn = ell ? v->fn[0][0] : v->fn[(int)h][is_union ? 1 : 0];
  // Block size: the one that keeps the most warps resident per SM (register-limited kernels
  // lose whole 256-thread blocks to the allocation granularity); ties go to the larger block.
  struct Occ { int threads, per_sm; };
  // per-kernel cache (hopf_eval_maxh alternates kernels every launch: a one-entry cache re-ran
  // the attribute and occupancy queries on the host before each of them)
  // (keyed by device too: the carveout attribute is set per device)
  static thread_local KernFn cache_fn[32] = {};
  static thread_local int cache_dev[32] = {};
  static thread_local Occ cache_occ[32];
  static thread_local int cache_n = 0;
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  // union: the kappa table of all K sets in dynamic shared memory ([K][NP*G + 1] float2)
  const size_t dyn = is_union ? (size_t)p.K * (size_t)(((v->CPL + 1) / 2) * v->G + 1) * 8 : 0;
  if (dyn > 48 * 1024 &&
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) != cudaSuccess)
    return set_error(HOPF_EUNSUPPORTED, "union kappa table of %zu bytes does not fit", dyn);
  int ci = -1;
  for (int i = 0; i < cache_n && dyn == 0; i++)
    if (cache_fn[i] == fn && cache_dev[i] == cur_dev) { ci = i; break; }
  Occ cached{128, 1};
  if (ci >= 0) cached = cache_occ[ci];
  if (ci < 0) {
    // kappa lives in static shared memory: ask for the full carveout so that several small
    // blocks fit per SM (the default carveout only fits one block's 4 KB + reserved 1 KB)
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    Occ bestc{128, 0};
    for (int th : {128, 64, 32}) {   // the kernels are built with __launch_bounds__(128, 3)
      if (th < v->G) continue;
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, th, dyn) != cudaSuccess) continue;
      if (per_sm * th > bestc.per_sm * bestc.threads) bestc = {th, per_sm};
    }
    if (bestc.per_sm < 1) bestc = {128, 1};
    cached = bestc;
    if (cache_n < 32 && dyn == 0) {
      cache_fn[cache_n] = fn;
      cache_dev[cache_n] = cur_dev;
      cache_occ[cache_n] = bestc;
      cache_n++;
    }
  }
  const int threads = cached.threads;
  const int64_t groups_needed = p.M;
  const int64_t blocks_needed = (groups_needed * v->G + threads - 1) / threads;
  int64_t blocks = (int64_t)num_sms() * cached.per_sm;
  if (blocks > blocks_needed) blocks = blocks_needed;
  if (blocks < 1) blocks = 1;
  DiagParams q = p;
  int rc = v->G > 1 ? claim_counter(p.M, blocks * threads / v->G, stream, &q.claim) : HOPF_OK;   // (G = 1: static)
  if (rc != HOPF_OK) return rc;
  fn<<<(unsigned)blocks, threads, dyn, stream>>>(q);
  scratch_free(q.claim, stream);
  g_launches += 1;
  g_last_threads = threads;
  g_last_blocks = (int)blocks;
  g_last_kernel = is_union ? "hopf_diag_kernel<union>"
                           : (h == HOPF_H_ELL ? "hopf_diag_kernel<ell>"
                                              : (h == HOPF_H_LINF ? "hopf_diag_kernel<linf>" : "hopf_diag_kernel"));
  return check_launch("hopf_diag_kernel");
}

static bool finite_pos(float x) { return std::isfinite(x) && x > 0.f; }

}  // namespace hopf

using namespace hopf;

extern "C" {

int hopf_eval_diag(int64_t M, int32_t n, const float *X, const float *t, const float *Dj,
                   const float *c, float gamma, hopf_h_kind h, const float *w, float lambda,
                   int32_t max_iter, float tol, float *phi, float *grad, int32_t *iters,
                   hopf_stream_t stream) {
  g_launches = 0;
  g_last_error.clear();
  if (M < 0 || n < 1) return set_error(HOPF_EINVAL, "M=%lld n=%d", (long long)M, n);
  if ((int)h < 0 || (int)h > 4) return set_error(HOPF_EINVAL, "unknown H kind %d", (int)h);
  if (!finite_pos(lambda)) return set_error(HOPF_EINVAL, "lambda must be > 0 and finite");
  if (!(tol >= 0.f) || !std::isfinite(tol)) return set_error(HOPF_EINVAL, "tol must be >= 0");
  if (max_iter < 1) return set_error(HOPF_EINVAL, "max_iter must be >= 1");
  if ((h == HOPF_H_WL1 || h == HOPF_H_ELL) && !w) return set_error(HOPF_EINVAL, "w is required for HOPF_H_WL1 / HOPF_H_ELL");
  if (M == 0) return HOPF_OK;
  if (!X || !t || !Dj || !phi || !grad || !iters)
    return set_error(HOPF_EINVAL, "a required pointer is NULL");
  DiagParams p{};
  p.M = M; p.n = n; p.X = X; p.t = t; p.D = Dj; p.c = c; p.w = w; p.gk = nullptr;
  p.gamma = gamma; p.lambda = lambda; p.max_iter = max_iter; p.tol = tol; p.K = 0;
  p.phi = phi; p.grad = grad; p.iters = iters; p.Y = nullptr; p.kstar = nullptr; p.phik = nullptr;
  return launch_diag_like(p, h, false, (cudaStream_t)stream);
}

int hopf_eval_union(int64_t M, int32_t n, int32_t K, const float *X, const float *t,
                    const float *Dj, const float *C, const float *gamma, hopf_h_kind h,
                    const float *w, float lambda, int32_t max_iter, float tol, float *phi,
                    float *grad, int32_t *iters, float *Y, int32_t *kstar, float *phi_k,
                    hopf_stream_t stream) {
  g_launches = 0;
  g_last_error.clear();
  if (M < 0 || n < 1 || K < 1) return set_error(HOPF_EINVAL, "M=%lld n=%d K=%d", (long long)M, n, K);
  if ((int)h < 0 || (int)h > 4) return set_error(HOPF_EINVAL, "unknown H kind %d", (int)h);
  if (!finite_pos(lambda)) return set_error(HOPF_EINVAL, "lambda must be > 0 and finite");
  if (!(tol >= 0.f) || !std::isfinite(tol)) return set_error(HOPF_EINVAL, "tol must be >= 0");
  if (max_iter < 1) return set_error(HOPF_EINVAL, "max_iter must be >= 1");
  if ((h == HOPF_H_WL1 || h == HOPF_H_ELL) && !w) return set_error(HOPF_EINVAL, "w is required for HOPF_H_WL1 / HOPF_H_ELL");
  if (Y && h != HOPF_H_L2) return set_error(HOPF_EINVAL, "Y (closest point) requires HOPF_H_L2");
  if (K > 64 || n > 256) return set_error(HOPF_EUNSUPPORTED, "union supports K<=64, n<=256");
  if (M == 0) return HOPF_OK;
  if (!X || !t || !Dj || !C || !gamma || !phi || !grad || !iters)
    return set_error(HOPF_EINVAL, "a required pointer is NULL");
  DiagParams p{};
  p.M = M; p.n = n; p.X = X; p.t = t; p.D = Dj; p.c = C; p.w = w; p.gk = gamma;
  p.gamma = 0.f; p.lambda = lambda; p.max_iter = max_iter; p.tol = tol; p.K = K;
  p.phi = phi; p.grad = grad; p.iters = iters; p.Y = Y; p.kstar = kstar; p.phik = phi_k;
  return launch_diag_like(p, h, true, (cudaStream_t)stream);
}

int hopf_distance_union(int64_t M, int32_t n, int32_t K, const float *Y, const float *Dj,
                        const float *C, const float *gamma, float lambda, int32_t max_iter,
                        float tol, int32_t max_newton, float stol, float *dist, float *proj,
                        float *psi, float *grad, int32_t *kstar, int32_t *newton,
                        hopf_stream_t stream) {
  g_launches = 0;
  g_last_error.clear();
  if (M < 0 || n < 1 || K < 1) return set_error(HOPF_EINVAL, "M=%lld n=%d K=%d", (long long)M, n, K);
  if (!finite_pos(lambda)) return set_error(HOPF_EINVAL, "lambda must be > 0 and finite");
  if (!(tol >= 0.f) || !std::isfinite(tol)) return set_error(HOPF_EINVAL, "tol must be >= 0");
  if (max_iter < 1) return set_error(HOPF_EINVAL, "max_iter must be >= 1");
  if (max_newton < 1) return set_error(HOPF_EINVAL, "max_newton must be >= 1");
  if (!(stol >= 0.f) || !std::isfinite(stol)) return set_error(HOPF_EINVAL, "stol must be >= 0");
  if (K > 64 || n > 256) return set_error(HOPF_EUNSUPPORTED, "union supports K<=64, n<=256");
  if (M == 0) return HOPF_OK;
  if (!Y || !Dj || !C || !gamma || !dist || !proj || !psi || !grad || !kstar || !newton)
    return set_error(HOPF_EINVAL, "a required pointer is NULL");
  DiagParams p{};
  p.M = M; p.n = n; p.X = Y; p.t = nullptr; p.D = Dj; p.c = C; p.w = nullptr; p.gk = gamma;
  p.gamma = 0.f; p.lambda = lambda; p.max_iter = max_iter; p.tol = tol; p.K = K;
  p.phi = psi; p.grad = grad; p.iters = newton; p.Y = proj; p.kstar = kstar; p.phik = nullptr;
  p.dist = dist; p.max_newton = max_newton; p.stol = stol;
  int rc = launch_diag_like(p, HOPF_H_L2, true, (cudaStream_t)stream);
  if (rc == HOPF_OK && strcmp(g_last_kernel, "hopf_diag_kernel<union>") == 0)
    g_last_kernel = "hopf_diag_kernel<union, distance>";
  return rc;
}


int hopf_eval_maxh(int64_t M, int32_t n, const float *X, const float *t, const float *Dj,
                   const float *c, float gamma, int32_t K, const int32_t *h_kinds, const float *a,
                   const float *W, float lambda, int32_t max_iter, float tol, float *phi,
                   float *grad, int32_t *iters, int32_t *istar, hopf_stream_t stream) {
  g_launches = 0;
  g_last_error.clear();
  if (M < 0 || n < 1 || K < 1) return set_error(HOPF_EINVAL, "M=%lld n=%d K=%d", (long long)M, n, K);
  if (!h_kinds || !a) return set_error(HOPF_EINVAL, "h_kinds and a (host arrays) are required");
  for (int i = 0; i < K; i++) {
    if (h_kinds[i] < 0 || h_kinds[i] > 4) return set_error(HOPF_EINVAL, "unknown H kind %d", h_kinds[i]);
    if (!finite_pos(a[i])) return set_error(HOPF_EINVAL, "a[%d] must be > 0 and finite", i);
    if ((h_kinds[i] == HOPF_H_WL1 || h_kinds[i] == HOPF_H_ELL) && !W)
      return set_error(HOPF_EINVAL, "W is required for HOPF_H_WL1 / HOPF_H_ELL");
  }
  if (!finite_pos(lambda)) return set_error(HOPF_EINVAL, "lambda must be > 0 and finite");
  if (!(tol >= 0.f) || !std::isfinite(tol)) return set_error(HOPF_EINVAL, "tol must be >= 0");
  if (max_iter < 1) return set_error(HOPF_EINVAL, "max_iter must be >= 1");
  if (n > 1024) return set_error(HOPF_EUNSUPPORTED, "n=%d exceeds the compiled diag kernels", n);
  if (M == 0) return HOPF_OK;
  if (!X || !t || !Dj || !phi || !grad || !iters) return set_error(HOPF_EINVAL, "a required pointer is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  // scratch for phi_i, grad_i, iters_i (i >= 1): stream-ordered, per call (scratch_alloc), so
  // calls on different streams never share it
  float *phs = nullptr, *gs = nullptr;
  int32_t *its = nullptr;
  char *scratch = nullptr;
  if (K > 1) {
    const size_t a1 = ((size_t)M * 4 + 255) & ~(size_t)255, a2 = ((size_t)M * n * 4 + 255) & ~(size_t)255;
    int rc0 = scratch_alloc((void **)&scratch, 2 * a1 + a2, st);
    if (rc0 != HOPF_OK) return rc0;
    phs = (float *)scratch;
    its = (int32_t *)(scratch + a1);
    gs = (float *)(scratch + 2 * a1);
  }
  const int nb = num_sms() * 8;
  int rc = HOPF_OK;
  for (int i = 0; i < K && rc == HOPF_OK; i++) {
    // phi_i: the diag solve with H_i = a_i H_kind(.; w_i), at time a_i t
    DiagParams p{};
    p.M = M; p.n = n; p.X = X; p.t = t; p.tscale = a[i]; p.D = Dj; p.c = c;
    p.w = (h_kinds[i] == HOPF_H_WL1 || h_kinds[i] == HOPF_H_ELL) ? W + (size_t)i * n : nullptr;
    p.gamma = gamma; p.lambda = lambda; p.max_iter = max_iter; p.tol = tol; p.K = 0;
    p.phi = i == 0 ? phi : phs; p.grad = i == 0 ? grad : gs; p.iters = i == 0 ? iters : its;
    rc = launch_diag_like(p, (hopf_h_kind)h_kinds[i], false, st);
    if (rc != HOPF_OK) break;
    if (i == 0) {
      if (istar) hopf_istar_init_kernel<<<nb, 256, 0, st>>>(M, iters, istar);
    } else {
      hopf_maxh_combine_kernel<<<nb, 256, 0, st>>>(M, n, i, phs, gs, its, phi, grad, iters, istar);
    }
  }
  scratch_free(scratch, st);
  if (rc != HOPF_OK) return rc;
  g_launches = 2 * K - (istar ? 0 : 1);   // K solves, K-1 combines (+ istar init)
  g_last_kernel = "hopf_diag kernels + hopf_maxh_combine_kernel";
  return check_launch("hopf_maxh_combine_kernel");
}

int hopf_set_iteration_counter(unsigned long long *counter) {
  g_iter_counter = counter;
  return HOPF_OK;
}

int32_t hopf_last_launch_count(void) { return g_launches; }

const char *hopf_last_kernel(void) { return g_last_kernel ? g_last_kernel : ""; }

int32_t hopf_last_launch_config(int32_t *threads_per_block, int32_t *blocks) {
  if (threads_per_block) *threads_per_block = g_last_threads;
  if (blocks) *blocks = g_last_blocks;
  return g_launches;
}

const char *hopf_last_error(void) { return g_last_error.c_str(); }

const char *hopf_strerror(int code) {
  switch (code) {
    case HOPF_OK: return "ok";
    case HOPF_EINVAL: return "invalid argument";
    case HOPF_EUNSUPPORTED: return "unsupported shape";
    case HOPF_ECUDA: return "CUDA error";
    default: return "unknown error code";
  }
}

int32_t hopf_version(void) { return 200; }   // 0.2.0: NEXT-1..4 entry points

}  // extern "C"
