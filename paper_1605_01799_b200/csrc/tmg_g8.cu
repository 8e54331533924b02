// tmg_g8.cu — instances of the grouped TMEM kernel (diag_tmg.cuh) with 8 lanes per point, every H kind.
#include "diag_tmg.cuh"
#include "tmg_api.h"

namespace hopf {
extern const TmgVariant kTmgG8[] = {
    {8, 20, {dtg::hopf_diag_tmg_kernel<8, 20, HK_L1, true>, dtg::hopf_diag_tmg_kernel<8, 20, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<8, 20, HK_L2, true>, dtg::hopf_diag_tmg_kernel<8, 20, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<8, 20, HK_LINF, true>}},
    {8, 24, {dtg::hopf_diag_tmg_kernel<8, 24, HK_L1, true>, dtg::hopf_diag_tmg_kernel<8, 24, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<8, 24, HK_L2, true>, dtg::hopf_diag_tmg_kernel<8, 24, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<8, 24, HK_LINF, true>}},
    {8, 28, {dtg::hopf_diag_tmg_kernel<8, 28, HK_L1, true>, dtg::hopf_diag_tmg_kernel<8, 28, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<8, 28, HK_L2, true>, dtg::hopf_diag_tmg_kernel<8, 28, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<8, 28, HK_LINF, true>}},
    {8, 32, {dtg::hopf_diag_tmg_kernel<8, 32, HK_L1, true>, dtg::hopf_diag_tmg_kernel<8, 32, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<8, 32, HK_L2, true>, dtg::hopf_diag_tmg_kernel<8, 32, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<8, 32, HK_LINF, true>}}};
extern const int kTmgG8Count = 4;
}  // namespace hopf
