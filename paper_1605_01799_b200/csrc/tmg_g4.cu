// tmg_g4.cu — instances of the grouped TMEM kernel (diag_tmg.cuh) with 4 lanes per point, every H kind.
#include "diag_tmg.cuh"
#include "tmg_api.h"

namespace hopf {
extern const TmgVariant kTmgG4[] = {
    {4, 8, {dtg::hopf_diag_tmg_kernel<4, 8, HK_L1, true>, dtg::hopf_diag_tmg_kernel<4, 8, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<4, 8, HK_L2, true>, dtg::hopf_diag_tmg_kernel<4, 8, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<4, 8, HK_LINF, true>}},
    {4, 10, {dtg::hopf_diag_tmg_kernel<4, 10, HK_L1, true>, dtg::hopf_diag_tmg_kernel<4, 10, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<4, 10, HK_L2, true>, dtg::hopf_diag_tmg_kernel<4, 10, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<4, 10, HK_LINF, true>}},
    {4, 12, {dtg::hopf_diag_tmg_kernel<4, 12, HK_L1, true>, dtg::hopf_diag_tmg_kernel<4, 12, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<4, 12, HK_L2, true>, dtg::hopf_diag_tmg_kernel<4, 12, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<4, 12, HK_LINF, true>}},
    {4, 16, {dtg::hopf_diag_tmg_kernel<4, 16, HK_L1, true>, dtg::hopf_diag_tmg_kernel<4, 16, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<4, 16, HK_L2, true>, dtg::hopf_diag_tmg_kernel<4, 16, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<4, 16, HK_LINF, true>}},
    {4, 20, {dtg::hopf_diag_tmg_kernel<4, 20, HK_L1, true>, dtg::hopf_diag_tmg_kernel<4, 20, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<4, 20, HK_L2, true>, dtg::hopf_diag_tmg_kernel<4, 20, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<4, 20, HK_LINF, true>}},
    {4, 24, {dtg::hopf_diag_tmg_kernel<4, 24, HK_L1, true>, dtg::hopf_diag_tmg_kernel<4, 24, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<4, 24, HK_L2, true>, dtg::hopf_diag_tmg_kernel<4, 24, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<4, 24, HK_LINF, true>}},
    {4, 26, {dtg::hopf_diag_tmg_kernel<4, 26, HK_L1, true>, dtg::hopf_diag_tmg_kernel<4, 26, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<4, 26, HK_L2, true>, dtg::hopf_diag_tmg_kernel<4, 26, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<4, 26, HK_LINF, true>}},
    {4, 28, {dtg::hopf_diag_tmg_kernel<4, 28, HK_L1, true>, dtg::hopf_diag_tmg_kernel<4, 28, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<4, 28, HK_L2, true>, dtg::hopf_diag_tmg_kernel<4, 28, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<4, 28, HK_LINF, true>}},
    {4, 32, {dtg::hopf_diag_tmg_kernel<4, 32, HK_L1, true>, dtg::hopf_diag_tmg_kernel<4, 32, HK_WL1, true>, dtg::hopf_diag_tmg_kernel<4, 32, HK_L2, true>, dtg::hopf_diag_tmg_kernel<4, 32, HK_ELL, true>, dtg::hopf_diag_tmg_kernel<4, 32, HK_LINF, true>}}};
extern const int kTmgG4Count = 9;
}  // namespace hopf
