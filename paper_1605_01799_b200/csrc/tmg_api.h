// tmg_api.h — dispatch to the grouped TMEM kernels (K1g diag_tmg.cuh, K4g diag_tmu.cuh).
// Their template instances live in tmg_g*.cu / tmu.cu (one translation unit per lane-group width,
// compiled in parallel); tmg_api.cu picks the variant and launches it.
#pragma once
#include <cuda_runtime.h>

#include "diag_kernel.cuh"

namespace hopf {

using TmgFn = void (*)(const DiagParams);
struct TmgVariant {
  int G, CPL;
  TmgFn fn[5];   // [h kind]: l1, wl1, l2, ell, linf (bulk row copies; null = not instantiated)
};
struct TmuVariant {
  int G, CPL;
  TmgFn fn[2];              // union, l2: [n % 4 != 0]
  size_t (*smem[2])(int K); // shared-memory bytes for K sets: [n % 4 != 0]
};
// tables, ordered by padded width G * CPL
const TmgVariant *tmg_variants(int *count);
const TmuVariant *tmu_variants(int *count);

// Launches the grouped kernel for p if one applies (non-union l1 / wl1 / l2, or union l2 without
// distance mode; 16-byte aligned rows; padding of n at most a quarter of the variant's width).
// *handled = false leaves the call to the register kernels.
int tmg_try_launch(const DiagParams &p, int h, bool is_union, cudaStream_t stream, bool *handled);

}  // namespace hopf
