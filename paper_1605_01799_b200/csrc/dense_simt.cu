// dense_simt.cu — v1 dense kernel (FP32 SIMT) and the dense plan's device operands.
// See dense_kernel.cuh for the paper mapping.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/hopf.h"
#include "common.cuh"
#include "dense_kernel.cuh"
#include "diag_kernel.cuh"  // HK_* constants, finite_f

namespace hopf {

bool dense_supported_n(int n) { return n >= 32 && n <= 256 && n % 32 == 0; }
const char *dense_supported_list() { return "32, 64, ..., 256 (multiples of 32)"; }

int dense_plan_upload(int n, const double *Ml, const double *Ainv, const double *Amat,
                      DensePlanDev *out) {
  const size_t nn = (size_t)n * n;
  std::vector<float> f(nn), g(nn), a(nn);
  for (size_t i = 0; i < nn; i++) {
    f[i] = (float)Ml[i];
    g[i] = (float)Ainv[i];
  }
  for (size_t i = 0; i < nn; i++) a[i] = (float)Amat[i];
  out->n = n;
  if (n == 256) {   // tensor-core operands for the tcgen05 kernels
    int rc = dense_tc3_prepare(n, Ml, &out->tc3_rows, &out->tc3_scale_inv);
    if (rc != HOPF_OK) return rc;
  }
  if (cudaMalloc(&out->Ml, nn * 4) != cudaSuccess || cudaMalloc(&out->Ainv, nn * 4) != cudaSuccess ||
      cudaMalloc(&out->A, nn * 4) != cudaSuccess) {
    dense_plan_free(out);
    return set_error(HOPF_ECUDA, "cudaMalloc for the dense plan failed");
  }
  cudaMemcpy(out->Ml, f.data(), nn * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(out->Ainv, g.data(), nn * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(out->A, a.data(), nn * 4, cudaMemcpyHostToDevice);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    dense_plan_free(out);
    return set_error(HOPF_ECUDA, "dense plan upload: %s", cudaGetErrorString(e));
  }
  return HOPF_OK;
}

void dense_plan_free(DensePlanDev *d) {
  if (d->Ml) cudaFree(d->Ml);
  if (d->Ainv) cudaFree(d->Ainv);
  if (d->A) cudaFree(d->A);
  if (d->tc3_rows) cudaFree(d->tc3_rows);
  d->Ml = d->Ainv = d->A = nullptr;
  d->tc3_rows = nullptr;
}

namespace {
constexpr int TP = 32;   // point rows per CTA
constexpr int KC = 32;   // K-slice of M_lambda staged per step
constexpr int NT = 256;  // threads

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// NW = n/32 columns per lane (n <= 256 => NW <= 8)
template <int NW, int HK>
__global__ void __launch_bounds__(NT, 1)
    hopf_dense_simt_kernel(const DenseParams p, const float *__restrict__ Ml,
                           const float *__restrict__ Ainv, const float *__restrict__ A) {
  constexpr int n = NW * 32;
  extern __shared__ float sm[];
  float *xs = sm;                // [TP][n]
  float *ds = xs + TP * n;       // [TP][n]
  float *bs = ds + TP * n;       // [TP][n]
  float *vps = bs + TP * n;      // [TP][n]
  float *Us = vps + TP * n;      // [TP][n]
  float *Mls = Us + TP * n;      // [KC][n]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float lam = p.lambda;
  const int64_t stride = (int64_t)gridDim.x * TP;

  // per-row bookkeeping, owned by the row's warp (lane-replicated)
  int64_t pt[4], pos[4];
  int it[4], spec[4];
  float tt[4];
  bool have[4];

  auto load_row = [&](int r) {
    const int row = warp * 4 + r;
    bool bad = false;
    if (have[r]) {
      tt[r] = __ldg(p.t + pt[r]);
      bad = !(tt[r] >= 0.f) || !finite_f(tt[r]);
      const float *xrow = p.X + pt[r] * (int64_t)n;
#pragma unroll
      for (int c = 0; c < NW; c++) {
        const int j = lane + 32 * c;
        const float xv = __ldg(xrow + j);
        bad |= !finite_f(xv);
        xs[row * n + j] = xv;
        ds[row * n + j] = xv;   // d0 = x
        bs[row * n + j] = 0.f;  // b0 = 0
        vps[row * n + j] = xv;  // v0 = x
        Us[row * n + j] = fmaf(p.lambda, xv, xv);   // U = x + lambda (d0 - b0) = (1 + lambda) x
      }
    } else {
#pragma unroll
      for (int c = 0; c < NW; c++) {
        const int j = lane + 32 * c;
        xs[row * n + j] = 0.f; ds[row * n + j] = 0.f; bs[row * n + j] = 0.f;
        vps[row * n + j] = 0.f; Us[row * n + j] = 0.f;
      }
    }
    bad = __any_sync(0xffffffffu, bad);
    spec[r] = bad ? 2 : (have[r] && tt[r] == 0.f ? 1 : 0);
    it[r] = 0;
  };

  const int64_t nlist = p.idx ? (int64_t)*p.idx_count : 0;
  auto position = [&](int r) {   // global point of list position pos[r]
    if (p.idx) {
      have[r] = pos[r] < nlist;
      pt[r] = have[r] ? (int64_t)p.idx[pos[r]] : 0;
    } else {
      pt[r] = pos[r];
      have[r] = pt[r] < p.M;
    }
  };
#pragma unroll
  for (int r = 0; r < 4; r++) {
    pos[r] = (int64_t)blockIdx.x * TP + warp * 4 + r;
    position(r);
    load_row(r);
  }
  __syncthreads();

  while (__syncthreads_or(have[0] || have[1] || have[2] || have[3])) {
    // ---------------- V = U M_lambda (rows 4w..4w+3, columns 8l..8l+7 of this lane) -------
    float acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int c = 0; c < 8; c++) acc[r][c] = 0.f;
    for (int k0 = 0; k0 < n; k0 += KC) {
      // stage M_lambda[k0:k0+KC, :] (coalesced float4)
      for (int e = threadIdx.x * 4; e < KC * n; e += NT * 4)
        *reinterpret_cast<float4 *>(Mls + e) = __ldg(reinterpret_cast<const float4 *>(Ml + (size_t)k0 * n + e));
      __syncthreads();
      if (lane * 8 < n) {
#pragma unroll 8
        for (int k = 0; k < KC; k++) {
          float a[4];
#pragma unroll
          for (int r = 0; r < 4; r++) a[r] = Us[(warp * 4 + r) * n + k0 + k];
          const float4 b0 = *reinterpret_cast<const float4 *>(Mls + k * n + lane * 8);
          const float4 b1 = *reinterpret_cast<const float4 *>(Mls + k * n + lane * 8 + 4);
          const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int r = 0; r < 4; r++)
#pragma unroll
            for (int c = 0; c < 8; c++) acc[r][c] = fmaf(a[r], bb[c], acc[r][c]);
        }
      }
      __syncthreads();
    }
    // ---------------- epilogue: shrink, Bregman update, test, next U (per row, per warp) --
    // lane l holds V[row][8l + c]; the row's state is in shared memory.
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int row = warp * 4 + r;
      float *xr = xs + row * n, *dr = ds + row * n, *br = bs + row * n, *vr = vps + row * n,
            *ur = Us + row * n;
      const bool live = lane * 8 < n;
      const float tauS = tt[r] / lam;
      float sv = 0.f, sd = 0.f, sb = 0.f, s = 0.f;
      if (HK == HK_L2) {
        float r2 = 0.f;
#pragma unroll
        for (int c = 0; c < 8; c++) {
          const int j = lane * 8 + c;
          if (live) { const float u = acc[r][c] + br[j]; r2 = fmaf(u, u, r2); }
        }
        r2 = warp_sum(r2);
        const float rn = sqrtf(r2);
        s = (rn > tauS) ? (rn - tauS) / rn : 0.f;
      }
#pragma unroll
      for (int c = 0; c < 8; c++) {
        const int j = lane * 8 + c;
        if (!live) break;
        const float v = acc[r][c];
        const float dv = v - vr[j];
        sv = fmaf(dv, dv, sv);
        const float bo = br[j], dold = dr[j];
        const float u = v + bo;
        float dn, bn;
        if (HK == HK_L2) {
          dn = s * u;
          bn = u - dn;
        } else {
          const float tj = (HK == HK_WL1) ? tt[r] * __ldg(p.w + j) / lam : tauS;
          bn = fminf(fmaxf(u, -tj), tj);
          dn = u - bn;
        }
        const float dd = dn - dold;
        sd = fmaf(dd, dd, sd);
        const float db = bo - bn;
        sb = fmaf(db, db, sb);
        vr[j] = v;
        dr[j] = dn;
        br[j] = bn;
        ur[j] = xr[j] + lam * (dn - bn);   // next U (3.4a)
      }
      sv = warp_sum(sv);
      sd = warp_sum(sd);
      sb = warp_sum(sb);
      it[r]++;
      const bool conv = sv <= p.tol && sd <= p.tol && sb <= p.tol;
      const bool done = have[r] && (spec[r] != 0 || conv || it[r] >= p.max_iter);
      if (done) {  // warp-uniform
        __syncwarp();
        // phi = <x,d> - 1/2 <d, A^{-1} d> - t H(d) + gamma; t == 0: J(x) = 1/2<x,Ax> + gamma
        const float *Mq = (spec[r] == 1) ? A : Ainv;
        const float *vec = (spec[r] == 1) ? xr : dr;
        float q = 0.f, hs = 0.f;
        float *grow = p.grad + pt[r] * (int64_t)n;
#pragma unroll
        for (int c = 0; c < NW; c++) {
          const int j = lane + 32 * c;
          float mv = 0.f;
          const float *mrow = Mq + (size_t)j * n;
          for (int k = 0; k < n; k += 4) {
            const float4 m4 = __ldg(reinterpret_cast<const float4 *>(mrow + k));
            mv = fmaf(m4.x, vec[k], mv);
            mv = fmaf(m4.y, vec[k + 1], mv);
            mv = fmaf(m4.z, vec[k + 2], mv);
            mv = fmaf(m4.w, vec[k + 3], mv);
          }
          float gj;
          if (spec[r] == 1) {
            gj = mv;                                  // grad J(x) = A x
            q = fmaf(0.5f * xr[j], mv, q);
          } else {
            gj = dr[j];
            q = fmaf(xr[j], dr[j], q);
            q = fmaf(-0.5f * dr[j], mv, q);
            if (HK == HK_L2) hs = fmaf(dr[j], dr[j], hs);
            else if (HK == HK_WL1) hs = fmaf(__ldg(p.w + j), fabsf(dr[j]), hs);
            else hs += fabsf(dr[j]);
          }
          grow[j] = (spec[r] == 2) ? __int_as_float(0x7fc00000) : gj;
        }
        q = warp_sum(q);
        hs = warp_sum(hs);
        if (lane == 0) {
          float ph;
          int st;
          if (spec[r] == 2) { ph = __int_as_float(0x7fc00000); st = INT32_MIN; }
          else if (spec[r] == 1) { ph = q + p.gamma; st = 0; }
          else { ph = q - tt[r] * (HK == HK_L2 ? sqrtf(hs) : hs) + p.gamma; st = conv ? it[r] : -p.max_iter; }
          p.phi[pt[r]] = ph;
          p.iters[pt[r]] = st;
        }
        __syncwarp();
        pos[r] += stride;
        position(r);
        load_row(r);
      }
    }
    __syncthreads();
  }
}

template <int NW>
int launch_nw(const DenseParams &p, int hk, const DensePlanDev &plan, cudaStream_t stream) {
  // list mode: the count is on the device, so the grid is the resident maximum
  const size_t smem = (size_t)(5 * TP + KC) * NW * 32 * sizeof(float);
  void (*fn)(const DenseParams, const float *, const float *, const float *) =
      hk == HK_L1 ? hopf_dense_simt_kernel<NW, HK_L1>
                  : (hk == HK_WL1 ? hopf_dense_simt_kernel<NW, HK_WL1> : hopf_dense_simt_kernel<NW, HK_L2>);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)num_sms() * per_sm;
  const int64_t need = (p.M + TP - 1) / TP;
  if (!p.idx && blocks > need) blocks = need;
  fn<<<(unsigned)blocks, NT, smem, stream>>>(p, plan.Ml, plan.Ainv, plan.A);
  g_launches += 1;
  g_last_kernel = "hopf_dense_simt_kernel";
  return check_launch("hopf_dense_simt_kernel");
}
}  // namespace

static int launch_simt(const DenseParams &p, int hk, const DensePlanDev &plan, cudaStream_t stream) {
  switch (p.n / 32) {
    case 1: return launch_nw<1>(p, hk, plan, stream);
    case 2: return launch_nw<2>(p, hk, plan, stream);
    case 3: return launch_nw<3>(p, hk, plan, stream);
    case 4: return launch_nw<4>(p, hk, plan, stream);
    case 5: return launch_nw<5>(p, hk, plan, stream);
    case 6: return launch_nw<6>(p, hk, plan, stream);
    case 7: return launch_nw<7>(p, hk, plan, stream);
    case 8: return launch_nw<8>(p, hk, plan, stream);
  }
  return set_error(HOPF_EUNSUPPORTED, "dense n=%d", p.n);
}

// n == 256 and H in {l1, wl1}: tcgen05 kernel, then the exact SIMT kernel on its fix-up list
// (t == 0, invalid points, fp16 overflow, no convergence within max_iter).  Otherwise SIMT.
int dense_launch(const DenseParams &p, int hk, const DensePlanDev &plan, cudaStream_t stream) {
  const bool use_tc = plan.tc3_rows && p.n == 256 && hk != HK_L2 && p.M <= 0x7fffffffLL - (1LL << 20);
  if (!use_tc) return launch_simt(p, hk, plan, stream);
  // the fix-up list [count, idx...] is per call and stream-ordered (scratch_alloc), so calls on
  // different streams never share it, whatever plan they use
  int *fix = nullptr;
  int rc = scratch_alloc((void **)&fix, sizeof(int) * (size_t)(p.M + 1), stream);
  if (rc != HOPF_OK) return rc;
  cudaMemsetAsync(fix, 0, sizeof(int), stream);
  rc = dense_tc3_launch(p, hk, plan.tc3_rows, plan.tc3_scale_inv, fix, fix + 1, stream);
  if (rc == HOPF_OK) {
    DenseParams q = p;
    q.idx = fix + 1;
    q.idx_count = fix;
    rc = launch_simt(q, hk, plan, stream);
  }
  scratch_free(fix, stream);
  g_last_kernel = "hopf_dense_tc3_kernel";
  return rc;
}

}  // namespace hopf
