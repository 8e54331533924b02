// dense_plan.cu — hopf_dense_plan_create/destroy and hopf_eval_dense.
//
// (3.4a) for J(x) = 1/2<x,Ax> + gamma is the quadratic prox:
//     (A^{-1} + lambda I) v = x + lambda (d - b)  =>  v = M_lambda (x + lambda (d - b)),
//     M_lambda = (A^{-1} + lambda I)^{-1} = Q diag(Lambda / (1 + lambda Lambda)) Q^T.
// The plan builds M_lambda and A^{-1} = Q diag(1/Lambda) Q^T in fp64 on the host, then stores
// the operands the dense kernel consumes (dense_kernel.cuh).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/hopf.h"
#include "common.cuh"
#include "dense_kernel.cuh"

struct hopf_dense_plan {
  int n;
  float lambda;
  int device;
  hopf::DensePlanDev dev;  // device operands (owned)
};

using namespace hopf;

extern "C" int hopf_dense_plan_create(int32_t n, const double *Q_host, const double *Lambda_host,
                                      float lambda, hopf_dense_plan **out) {
  g_last_error.clear();
  if (!out || !Q_host || !Lambda_host) return set_error(HOPF_EINVAL, "NULL argument");
  *out = nullptr;
  if (n < 1) return set_error(HOPF_EINVAL, "n=%d", n);
  if (!(lambda > 0.f) || !std::isfinite(lambda)) return set_error(HOPF_EINVAL, "lambda must be > 0");
  if (!dense_supported_n(n))
    return set_error(HOPF_EUNSUPPORTED, "dense kernel supports n in {%s}, got %d",
                     dense_supported_list(), n);
  for (int i = 0; i < n; i++)
    if (!(Lambda_host[i] > 0.0) || !std::isfinite(Lambda_host[i]))
      return set_error(HOPF_EINVAL, "Lambda[%d] must be > 0 and finite", i);
  const double lam = (double)lambda;
  std::vector<double> Ml((size_t)n * n, 0.0), Ai((size_t)n * n, 0.0), Am((size_t)n * n, 0.0);
  std::vector<double> sM(n), sA(n);
  for (int k = 0; k < n; k++) {
    sM[k] = Lambda_host[k] / (1.0 + lam * Lambda_host[k]);
    sA[k] = 1.0 / Lambda_host[k];
  }
  // Ml = Q diag(sM) Q^T, Ai = Q diag(sA) Q^T, Am = Q diag(Lambda) Q^T (fp64, symmetric)
  for (int i = 0; i < n; i++) {
    for (int j = i; j < n; j++) {
      double a = 0.0, c = 0.0, e = 0.0;
      const double *qi = Q_host + (size_t)i * n, *qj = Q_host + (size_t)j * n;
      for (int k = 0; k < n; k++) {
        const double qq = qi[k] * qj[k];
        a += qq * sM[k];
        c += qq * sA[k];
        e += qq * Lambda_host[k];
      }
      Ml[(size_t)i * n + j] = Ml[(size_t)j * n + i] = a;
      Ai[(size_t)i * n + j] = Ai[(size_t)j * n + i] = c;
      Am[(size_t)i * n + j] = Am[(size_t)j * n + i] = e;
    }
  }
  hopf_dense_plan *p = new hopf_dense_plan();
  p->n = n;
  p->lambda = lambda;
  cudaGetDevice(&p->device);
  int rc = dense_plan_upload(n, Ml.data(), Ai.data(), Am.data(), &p->dev);
  if (rc != HOPF_OK) {
    delete p;
    return rc;
  }
  *out = p;
  return HOPF_OK;
}

extern "C" int hopf_dense_plan_destroy(hopf_dense_plan *plan) {
  if (!plan) return HOPF_OK;
  dense_plan_free(&plan->dev);
  delete plan;
  return HOPF_OK;
}

extern "C" int hopf_eval_dense(int64_t M, int32_t n, const float *X, const float *t,
                               const hopf_dense_plan *plan, float gamma, hopf_h_kind h,
                               const float *w, float lambda, int32_t max_iter, float tol,
                               float *phi, float *grad, int32_t *iters, hopf_stream_t stream) {
  g_launches = 0;
  g_last_error.clear();
  if (!plan) return set_error(HOPF_EINVAL, "plan is NULL");
  if (M < 0 || n != plan->n) return set_error(HOPF_EINVAL, "M=%lld n=%d (plan n=%d)", (long long)M, n, plan->n);
  if ((int)h < 0 || (int)h > 2) return set_error(HOPF_EINVAL, "unknown H kind %d", (int)h);
  if (lambda != plan->lambda) return set_error(HOPF_EINVAL, "lambda differs from the plan's");
  if (!(tol >= 0.f) || !std::isfinite(tol)) return set_error(HOPF_EINVAL, "tol must be >= 0");
  if (max_iter < 1) return set_error(HOPF_EINVAL, "max_iter must be >= 1");
  if (h == HOPF_H_WL1 && !w) return set_error(HOPF_EINVAL, "w is required for HOPF_H_WL1");
  if (M == 0) return HOPF_OK;
  if (!X || !t || !phi || !grad || !iters) return set_error(HOPF_EINVAL, "a required pointer is NULL");
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev != plan->device)
    return set_error(HOPF_EINVAL, "the plan lives on device %d, the current device is %d", plan->device, dev);
  DenseParams p{};
  p.M = M; p.n = n; p.X = X; p.t = t; p.w = w; p.gamma = gamma; p.lambda = lambda;
  p.max_iter = max_iter; p.tol = tol; p.phi = phi; p.grad = grad; p.iters = iters;
  return dense_launch(p, (int)h, plan->dev, (cudaStream_t)stream);
}
