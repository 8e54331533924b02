// tmu.cu — instances of the grouped TMEM union kernel (diag_tmu.cuh), H = l2.
#include "diag_tmu.cuh"
#include "tmg_api.h"

namespace hopf {
extern const TmuVariant kTmu[] = {
    {4, 8, dtu::hopf_union_tmg_kernel<4, 8>, dtu::smem_bytes<4, 8>},
    {4, 12, dtu::hopf_union_tmg_kernel<4, 12>, dtu::smem_bytes<4, 12>},
    {4, 16, dtu::hopf_union_tmg_kernel<4, 16>, dtu::smem_bytes<4, 16>},
    {8, 16, dtu::hopf_union_tmg_kernel<8, 16>, dtu::smem_bytes<8, 16>},
    {16, 16, dtu::hopf_union_tmg_kernel<16, 16>, dtu::smem_bytes<16, 16>}};
extern const int kTmuCount = 5;
}  // namespace hopf
