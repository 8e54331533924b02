// dense_kernel.cuh — split Bregman for full SPD J (K3): the batched v-update
//     V = U M_lambda,   U = X + lambda (D_it - B_it)         ((3.4a))
// fused with the shrink / Bregman update / stopping-test epilogue ((3.4b)-(3.4c)).
//
// v1: FP32 SIMT tile kernel (correctness baseline for the tensor-core kernel).  A CTA owns a
// tile of TP = 32 point rows; all per-point state (x, d, b, v_prev, U) lives in shared memory;
// M_lambda is streamed from L2 in 32-row K-slices.  Warp w owns rows 4w..4w+3 for both the
// GEMM (lane l holds columns 8l..8l+7) and the epilogue, so no CTA barrier separates them.
// Finished rows are refilled with the next point of the CTA in place (row-level refill).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hopf {

struct DenseParams {
  int64_t M;
  int n;
  const float *X, *t, *w;
  float gamma, lambda;
  int max_iter;
  float tol;
  float *phi, *grad;
  int *iters;
  // optional index list (fix-up pass): process points idx[0 .. *idx_count) only
  const int *idx = nullptr;
  const int *idx_count = nullptr;
};

struct DensePlanDev {
  int n = 0;
  float *Ml = nullptr;    // [n*n] fp32 M_lambda
  float *Ainv = nullptr;  // [n*n] fp32 A^{-1}
  float *A = nullptr;     // [n*n] fp32 A
  // tensor-core operands (n == 256): fp16 hi/lo rows of 2^s M_lambda in smem order for the
  // CTA-pair kernel (dense_tc3.cu)
  void *tc3_rows = nullptr;
  float tc3_scale_inv = 0.f;
};

bool dense_supported_n(int n);
const char *dense_supported_list();
int dense_plan_upload(int n, const double *Ml, const double *Ainv, const double *A,
                      DensePlanDev *out);
void dense_plan_free(DensePlanDev *d);
int dense_launch(const DenseParams &p, int hk, const DensePlanDev &plan, cudaStream_t stream);
int dense_tc3_prepare(int n, const double *Ml, void **rows_dev, float *mscale_inv);
int dense_tc3_launch(const DenseParams &p, int hk, const void *rows, float mscale_inv,
                     int *fix_count, int *fix_list, cudaStream_t stream);

}  // namespace hopf
