// tmg_api.cu — variant choice and launch of the grouped TMEM kernels (K1g, K4g).
// A variant applies when it holds n (G * CPL >= n) with at most a quarter of padding, the bases of
// X, grad (and Y) are 16-byte aligned (bulk row copies; rows that do not start on a 16-byte
// boundary move their ends by plain loads / stores), and, for the union, the per-set tables fit
// the block's shared memory.  HOPF_DIAG_TMG=0 / HOPF_UNION_TMG=0 select the
// register kernels (A/B experiments).
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/hopf.h"
#include "common.cuh"
#include "diag_tmg.cuh"
#include "diag_tmu.cuh"
#include "tmg_api.h"

namespace hopf {
extern thread_local int32_t g_last_threads, g_last_blocks;
extern const TmgVariant kTmgG4[], kTmgG8[], kTmgG16[];
extern const int kTmgG4Count, kTmgG8Count, kTmgG16Count;
extern const TmuVariant kTmu[];
extern const int kTmuCount;

namespace {
const TmgVariant *pick_tmg(int n, int *index) {
  static const char *env = getenv("HOPF_DIAG_TMG");
  if (env && strcmp(env, "0") == 0) return nullptr;
  const TmgVariant *lists[3] = {kTmgG4, kTmgG8, kTmgG16};
  const int counts[3] = {kTmgG4Count, kTmgG8Count, kTmgG16Count};
  int idx = 0;
  for (int l = 0; l < 3; l++)
    for (int i = 0; i < counts[l]; i++, idx++) {
      const TmgVariant &v = lists[l][i];
      if (v.G * v.CPL >= n) {
        *index = idx;
        return 4 * (v.G * v.CPL - n) <= v.G * v.CPL ? &v : nullptr;
      }
    }
  return nullptr;
}

const TmuVariant *pick_tmu(const DiagParams &p, int *index) {
  static const char *env = getenv("HOPF_UNION_TMG");
  if (env && strcmp(env, "0") == 0) return nullptr;
  for (int i = 0; i < kTmuCount; i++) {
    const TmuVariant &v = kTmu[i];
    if (v.G * v.CPL >= p.n) {
      *index = i;
      return (4 * (v.G * v.CPL - p.n) <= v.G * v.CPL && v.smem[p.n % 4 != 0](p.K) <= (size_t)dtu::DYN_SMEM) ? &v : nullptr;
    }
  }
  return nullptr;
}

// cudaFuncSetAttribute once per (device, kernel)
void ensure_smem_attr(TmgFn fn, int slot, int bytes) {
  static std::atomic<uint64_t> done[64][4] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || slot < 0 || slot >= 256) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    return;
  }
  const uint64_t bit = 1ull << (slot & 63);
  if (!(done[dev][slot >> 6].load(std::memory_order_relaxed) & bit)) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done[dev][slot >> 6].fetch_or(bit, std::memory_order_relaxed);
  }
}
}  // namespace

const TmgVariant *tmg_variants(int *count) {
  *count = kTmgG4Count;
  return kTmgG4;
}
const TmuVariant *tmu_variants(int *count) {
  *count = kTmuCount;
  return kTmu;
}

int tmg_try_launch(const DiagParams &p, int h, bool is_union, cudaStream_t stream, bool *handled) {
  *handled = false;
  // bulk row copies: 16-byte aligned bases; any n (a row's unaligned ends move by plain loads /
  // stores)
  const bool bases = (((uintptr_t)p.X | (uintptr_t)p.grad) & 15) == 0;
  static const char *benv = getenv("HOPF_TMG_BULK");
  if (!bases || (benv && strcmp(benv, "0") == 0)) return HOPF_OK;
  if (!is_union) {
    if (h < HOPF_H_L1 || h > HOPF_H_LINF) return HOPF_OK;
    int idx = 0;
    const TmgVariant *v = pick_tmg(p.n, &idx);
    if (!v || !v->fn[h]) return HOPF_OK;
    TmgFn fn = v->fn[h];
    ensure_smem_attr(fn, 5 * idx + h, dtg::DYN_SMEM);
    const int per_block = dtg::THREADS / v->G;   // points in flight per block
    int64_t blocks = (int64_t)num_sms() * 4;
    const int64_t need = (p.M + per_block - 1) / per_block;
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    DiagParams q = p;
    int rc = claim_counter(p.M, blocks * per_block, stream, &q.claim);
    if (rc != HOPF_OK) return rc;
    fn<<<(unsigned)blocks, dtg::THREADS, dtg::DYN_SMEM, stream>>>(q);
    scratch_free(q.claim, stream);
    *handled = true;
    g_launches += 1;
    g_last_threads = dtg::THREADS;
    g_last_blocks = (int)blocks;
    static const char *names[5] = {"hopf_diag_tmg_kernel<l1>", "hopf_diag_tmg_kernel<wl1>",
                                   "hopf_diag_tmg_kernel<l2>", "hopf_diag_tmg_kernel<ell>",
                                   "hopf_diag_tmg_kernel<linf>"};
    g_last_kernel = names[h];
    return check_launch("hopf_diag_tmg_kernel");
  }
  // union (l2), also in distance mode (NEXT-1: p.dist non-null, p.Y = the projections)
  static const char *denv = getenv("HOPF_DIST_TMG");
  if (p.dist && denv && strcmp(denv, "0") == 0) return HOPF_OK;
  if (h != HOPF_H_L2 || (p.Y && ((uintptr_t)p.Y & 15) != 0)) return HOPF_OK;
  int idx = 0;
  const TmuVariant *v = pick_tmu(p, &idx);
  if (!v) return HOPF_OK;
  const int un = p.n % 4 != 0;
  ensure_smem_attr(v->fn[un], 240 + 2 * idx + un, dtu::DYN_SMEM);
  const int per_block = dtu::THREADS / v->G;
  int64_t blocks = (int64_t)num_sms() * dtu::BLOCKS_PER_SM;
  const int64_t need = (p.M + per_block - 1) / per_block;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  DiagParams q = p;
  int rc = claim_counter(p.M, blocks * per_block, stream, &q.claim);
  if (rc != HOPF_OK) return rc;
  v->fn[un]<<<(unsigned)blocks, dtu::THREADS, dtu::DYN_SMEM, stream>>>(q);
  scratch_free(q.claim, stream);
  *handled = true;
  g_launches += 1;
  g_last_threads = dtu::THREADS;
  g_last_blocks = (int)blocks;
  g_last_kernel = p.dist ? "hopf_union_tmg_kernel<l2, distance>" : "hopf_union_tmg_kernel<l2>";
  return check_launch("hopf_union_tmg_kernel");
}

}  // namespace hopf
