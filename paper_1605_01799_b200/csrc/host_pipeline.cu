// host_pipeline.cu — end-to-end entry point on host buffers (hopf_eval_diag_host).
// Points are processed in chunks; chunk c runs on internal stream c % kStreams as
//   H2D(X_c, t_c) -> hopf_diag_kernel -> D2H(grad_c, phi_c, iters_c)
// so the PCIe copies of neighbouring chunks overlap each other (full duplex) and the kernels.
// Streams and device buffers live in pooled per-device contexts (one per concurrent call, buffers
// grown on demand, never shrunk).
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <vector>

#include "../../include/hopf.h"
#include "common.cuh"

namespace hopf {
namespace {
constexpr int kMaxStreams = 8;

// HOPF_HOST_STREAMS (2..8, default 3) and HOPF_HOST_CHUNK_MB (default 32): tuning knobs
int env_int(const char *name, int dflt, int lo, int hi) {
  const char *e = getenv(name);
  int v = e ? atoi(e) : dflt;
  return v < lo ? lo : (v > hi ? hi : v);
}

// One pipeline context = internal streams + device chunk buffers + the entry event.  Contexts
// are pooled per device: a call takes a free one (or creates one) under a per-device mutex that
// is held only for the pop / push, so concurrent calls (threads, devices) never share buffers
// and never wait for each other's copies or kernels.
struct Ctx {
  cudaStream_t s[kMaxStreams];
  cudaEvent_t entry;
  char *buf = nullptr;
  size_t bytes = 0;
};
struct DevPool {
  std::mutex mu;
  std::vector<Ctx *> free;
};
DevPool g_pool[64];

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

Ctx *ctx_take(int dev) {
  {
    std::lock_guard<std::mutex> lock(g_pool[dev].mu);
    if (!g_pool[dev].free.empty()) {
      Ctx *c = g_pool[dev].free.back();
      g_pool[dev].free.pop_back();
      return c;
    }
  }
  Ctx *c = new Ctx();
  for (int i = 0; i < kMaxStreams; i++) cudaStreamCreateWithFlags(&c->s[i], cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&c->entry, cudaEventDisableTiming);
  return c;
}
void ctx_give(int dev, Ctx *c) {
  std::lock_guard<std::mutex> lock(g_pool[dev].mu);
  g_pool[dev].free.push_back(c);
}
}  // namespace
}  // namespace hopf

using namespace hopf;

extern "C" int hopf_eval_diag_host(int64_t M, int32_t n, const float *X_host,
                                   const float *t_host, const float *Dj, const float *c,
                                   float gamma, hopf_h_kind h, const float *w, float lambda,
                                   int32_t max_iter, float tol, float *phi_host,
                                   float *grad_host, int32_t *iters_host) {
  if (M < 0 || n < 1) return set_error(HOPF_EINVAL, "M=%lld n=%d", (long long)M, n);
  if (M == 0) return HOPF_OK;
  if (!X_host || !t_host || !phi_host || !grad_host || !iters_host || !Dj)
    return set_error(HOPF_EINVAL, "a required pointer is NULL");
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return set_error(HOPF_EINVAL, "device index %d", dev);
  static const int kStreams = env_int("HOPF_HOST_STREAMS", 3, 2, kMaxStreams);
  static const int chunk_mb = env_int("HOPF_HOST_CHUNK_MB", 32, 1, 1024);
  // ~32 MB of X per chunk: large enough to amortise launch + copy latency (C3 e2e: 16 MB
  // 9.2e6 evals/s, 32 MB 9.9e6, 64 MB 9.6e6; 2-4 streams alike; ~79 GB/s of PCIe both ways)
  int64_t chunk = (int64_t)(((size_t)chunk_mb << 20) / ((size_t)n * sizeof(float)));
  if (chunk < 1024) chunk = 1024;
  if (chunk > M) chunk = M;
  const size_t xb = align_up((size_t)chunk * n * 4), vb = align_up((size_t)chunk * 4);
  const size_t per = 2 * xb + 3 * vb;  // X, grad, t, phi, iters
  Ctx *ctx = ctx_take(dev);
  Ctx &dc = *ctx;
  if (dc.bytes < per * kStreams) {
    if (dc.buf) cudaFree(dc.buf);
    dc.buf = nullptr;
    dc.bytes = 0;
    if (cudaMalloc(&dc.buf, per * kStreams) != cudaSuccess) {
      ctx_give(dev, ctx);
      return set_error(HOPF_ECUDA, "cudaMalloc of %zu bytes failed", per * kStreams);
    }
    dc.bytes = per * kStreams;
  }
  // ordering contract: the chunks run after all work enqueued earlier on the legacy default
  // stream of this device (which itself waits for every blocking stream), e.g. the caller's
  // writes of Dj / c / w; work on the caller's non-blocking streams must be synchronised first
  cudaEventRecord(dc.entry, cudaStreamLegacy);
  for (int i = 0; i < kStreams; i++) cudaStreamWaitEvent(dc.s[i], dc.entry, 0);
  int32_t launches = 0;
  int rc = HOPF_OK;
  for (int64_t off = 0, ci = 0; off < M; off += chunk, ci++) {
    const int64_t cnt = (M - off < chunk) ? (M - off) : chunk;
    const int slot = (int)(ci % kStreams);
    cudaStream_t s = dc.s[slot];
    char *base = dc.buf + per * slot;
    float *dX = (float *)base, *dG = (float *)(base + xb);
    float *dt = (float *)(base + 2 * xb), *dphi = (float *)(base + 2 * xb + vb);
    int32_t *dit = (int32_t *)(base + 2 * xb + 2 * vb);
    cudaMemcpyAsync(dX, X_host + off * n, (size_t)cnt * n * 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dt, t_host + off, (size_t)cnt * 4, cudaMemcpyHostToDevice, s);
    rc = hopf_eval_diag(cnt, n, dX, dt, Dj, c, gamma, h, w, lambda, max_iter, tol, dphi, dG, dit,
                        (hopf_stream_t)s);
    launches += hopf_last_launch_count();
    if (rc != HOPF_OK) break;
    cudaMemcpyAsync(grad_host + off * n, dG, (size_t)cnt * n * 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(phi_host + off, dphi, (size_t)cnt * 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(iters_host + off, dit, (size_t)cnt * 4, cudaMemcpyDeviceToHost, s);
  }
  for (int i = 0; i < kStreams; i++) {
    cudaError_t e = cudaStreamSynchronize(dc.s[i]);
    if (e != cudaSuccess && rc == HOPF_OK)
      rc = set_error(HOPF_ECUDA, "hopf_eval_diag_host: %s", cudaGetErrorString(e));
  }
  ctx_give(dev, ctx);
  g_launches = launches;
  return rc;
}
