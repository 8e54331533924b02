// tmu.cu — instances of the grouped TMEM union kernel (diag_tmu.cuh), H = l2: rows on 16-byte
// boundaries (n % 4 == 0) and not (UNAL).
#include "diag_tmu.cuh"
#include "tmg_api.h"

namespace hopf {
#define HOPF_TMU(G_, C_)                                                                     \
  {G_, C_, {dtu::hopf_union_tmg_kernel<G_, C_, false>, dtu::hopf_union_tmg_kernel<G_, C_, true>}, \
   {dtu::smem_bytes<G_, C_, false>, dtu::smem_bytes<G_, C_, true>}}
// ordered by width; (4, 20) and (4, 24) cover n = 61..96 (their per-set tables fit for K <= 20
// and K <= 6; larger K falls back to the register union kernel)
extern const TmuVariant kTmu[] = {HOPF_TMU(4, 8),  HOPF_TMU(4, 12), HOPF_TMU(4, 16), HOPF_TMU(4, 20),
                                  HOPF_TMU(4, 24), HOPF_TMU(8, 16), HOPF_TMU(16, 16)};
extern const int kTmuCount = 7;
}  // namespace hopf
