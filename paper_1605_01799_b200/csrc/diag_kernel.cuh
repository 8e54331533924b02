// diag_kernel.cuh — register-resident split Bregman kernels for diagonal J (K1/K2) and the
// min-over-K-sets union kernel (K4).  sm_100a, FP32 SIMT.
//
// Paper: Hopf formula (3.3) P:815-818; split Bregman (3.4a)-(3.4c) P:832-844; stopping rule
// P:1595-1601; shrink_1 P:239-247; shrink_2 P:279-287; quadratic prox P:901-906, P:1336-1347;
// Moreau / prox = I - projection P:924-992; union (min over initial data) P:628-667;
// closest point y = x - t grad/||grad|| P:1049-1051.
//
// Execution model.  A "group" of G lanes (G in {1,2,4,8,16,32}) owns one point; lane l of the
// group owns coordinates i = l + G*j, j < CPL (CPL = coordinates per lane, compile time), so
// every per-point vector lives in registers (x_hat, kappa, d, b, v_prev: 5*CPL floats) and
// the per-point sums (||u||^2 for shrink_2, the three stopping sums, phi) are xor-shuffle
// reductions inside the group.  Padded coordinates (i >= n) hold zeros, which the iteration
// maps to zeros, so they never contribute.  Grids are persistent (SMs x resident blocks);
// groups take points p = gid, gid + ngroups, ...  When a group's point stops (paper test or
// max_iter) the warp runs the finalize/refill branch: that group writes phi, grad, iters and
// immediately loads its next point while the other groups of the warp keep iterating, so a
// finished point stops costing cycles after one pass of the branch (per-point masking with
// in-place refill instead of lockstep batches).
//
// Per coordinate and iteration (exact rearrangement of (3.4a)-(3.4c)):
//   a = d - b;  v = x_hat + kappa*a          (3.4a), kappa = lambda/(D+lambda), x_hat = (x-c)/(D+lambda)
//   u = v + b;                               argument of (3.4b)
//   l1/wl1:  b' = clamp(u, -tau_i, tau_i);  d' = u - b'          shrink_1 via Moreau
//   l2:      s = max(0, 1 - tau/||u||);     d' = s u;  b' = u - d'   shrink_2
//   (3.4c): b + v - d' = u - d' = b'  (identical in exact arithmetic; the clamp form is also
//   bit-identical to sign(u) max(|u|-tau,0) in IEEE arithmetic)
//   test:  ||v - v_prev||^2, ||d' - d||^2, ||d' - v||^2 = ||b - b'||^2  <= tol
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace hopf {

// HK_ELL (NEXT-2): H(p) = sqrt(<p, W p>), W = diag(w) > 0.  (3.4b) is prox_{tau ||.||_W}(u) =
// u - tau P(u / tau), P the projection on the dual ellipsoid {z : <z, W^-1 z> <= 1}, computed by
// Newton on its multiplier mu; see the ELL branch of the trip below.
// HK_LINF (NEXT-2): H(p) = ||p||_inf.  (3.4b) is u - pi_{tau B1}(u) (Moreau; B1 the unit l1 ball,
// P:1348-1428) = clamp(u, -mu, mu) with mu the l1-ball multiplier; see the LINF branch.
enum { HK_L1 = 0, HK_WL1 = 1, HK_L2 = 2, HK_ELL = 3, HK_LINF = 4 };

// active-set Newton (HK_LINF, normsq_kernel.cuh): a step below this fraction of the multiplier
// is accepted as the root even if the active set changed (fp32 breakpoint noise)
#ifndef HOPF_TINY_STEP
#define HOPF_TINY_STEP 4e-7f
#endif

struct DiagParams {
  int64_t M;
  int n;
  const float *X, *t;
  const float *D, *c, *w;  // diag: D[n], c[n] or null; union: D = Dj[K*n], c = C[K*n]
  const float *gk;         // union: gamma[K]
  float gamma;
  float lambda;
  int max_iter;
  float tol;
  int K;  // 0 = plain diag
  float *phi, *grad;
  int *iters;
  float *Y;
  int *kstar;
  float *phik;
  // optional instrumentation: total split Bregman iterations of all solves (bench roofline)
  unsigned long long *iter_total = nullptr;
  // distance mode (union, H = l2; NEXT-1): non-null dist selects Newton in s on psi(y,s) = 0
  float *dist = nullptr;
  // hopf_eval_maxh: H_i = a_i H_kind is solved as time a_i t (t a_i H = (a_i t) H)
  float tscale = 1.f;
  int max_newton = 0;
  float stol = 0.f;
  // the launch's point counter (zeroed before the launch); null: static point stride
  unsigned long long *claim = nullptr;
};

// Dynamic point claims (one atomic on the launch's counter per claim).  `zero_lanes` is a shared
// array of zeros written at kernel start; reading it at a lane-dependent address outside the
// claiming lane's branch keeps the counter address non-uniform in the compiler's view, so a
// single lane's atomic is not turned into a warp-aggregated one whose result is shuffled at
// once (that would expose the atomic's latency; here the result is consumed one point later).
__device__ __forceinline__ void zero_lanes_init(unsigned *zero_lanes) {
  if (threadIdx.x < 32) {
    unsigned z;
    asm volatile("mov.u32 %0, 0;" : "=r"(z));
    zero_lanes[threadIdx.x] = z;
  }
}
__device__ __forceinline__ unsigned lane_zero(const unsigned *zero_lanes, int lane) {
  unsigned z;
  asm volatile("ld.shared.u32 %0, [%1];"
               : "=r"(z) : "r"((uint32_t)__cvta_generic_to_shared(zero_lanes + lane)));
  return z;
}

template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int G>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int G>
__device__ __forceinline__ bool group_any(bool f) {
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  if constexpr (G == 32) {
    return bal != 0u;
  } else {
    const int lane = threadIdx.x & 31;
    const unsigned gm = ((1u << G) - 1u) << (lane & ~(G - 1));
    return (bal & gm) != 0u;
  }
}

__device__ __forceinline__ bool finite_f(float x) { return fabsf(x) <= 3.402823466e38f; }

// Sum of four per-lane partials over a group of G lanes with log2(G)+1 shuffles (instead of
// 4 log2(G)): the first two butterfly levels exchange halves of the value set, so afterwards
// lane gl of the group holds the group total of value q = gl / (G/4) (v0 | v1 | v2 | v3).
// Requires G >= 4.  Returns the total held by this lane.
template <int G>
__device__ __forceinline__ float group_sum4_transposed(float v0, float v1, float v2, float v3) {
  static_assert(G >= 4, "transposed reduction needs at least 4 lanes");
  const int gl = threadIdx.x & (G - 1);
  const bool hi = gl & (G / 2);
  const float send_a = hi ? v0 : v2, send_b = hi ? v1 : v3;
  const float keep_a = hi ? v2 : v0, keep_b = hi ? v3 : v1;
  const float a = keep_a + __shfl_xor_sync(0xffffffffu, send_a, G / 2);
  const float b = keep_b + __shfl_xor_sync(0xffffffffu, send_b, G / 2);
  const bool mid = gl & (G / 4);
  float c = (mid ? b : a) + __shfl_xor_sync(0xffffffffu, mid ? a : b, G / 4);
#pragma unroll
  for (int o = G / 8; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  return c;
}

// Group totals of four partials, delivered as: tot3 (broadcast to every lane of the group) and
// the three predicates (total_q <= tol) for q = 0, 1, 2.
template <int G>
__device__ __forceinline__ void group_reduce4(float v0, float v1, float v2, float v3, float tol,
                                              float &tot3, bool &ok0, bool &ok1, bool &ok2) {
  const int lane = threadIdx.x & 31;
  const int base = lane & ~(G - 1);
  if constexpr (G >= 4) {
    const float c = group_sum4_transposed<G>(v0, v1, v2, v3);
    const unsigned bal = __ballot_sync(0xffffffffu, c <= tol);
    tot3 = __shfl_sync(0xffffffffu, c, base + 3 * (G / 4));
    ok0 = (bal >> (base)) & 1u;
    ok1 = (bal >> (base + G / 4)) & 1u;
    ok2 = (bal >> (base + 2 * (G / 4))) & 1u;
  } else {
    v0 = group_sum<G>(v0);
    v1 = group_sum<G>(v1);
    v2 = group_sum<G>(v2);
    tot3 = group_sum<G>(v3);
    ok0 = v0 <= tol;
    ok1 = v1 <= tol;
    ok2 = v2 <= tol;
  }
}

// Group totals of (S1, S2, sv): S1 and S2 broadcast to every lane of the group, ok_sv = (sv <= tol).
template <int G>
__device__ __forceinline__ void group_reduce3(float s1, float s2, float sv, float tol, float &S1,
                                              float &S2, bool &ok_sv) {
  const int lane = threadIdx.x & 31;
  const int base = lane & ~(G - 1);
  if constexpr (G >= 4) {
    const float c = group_sum4_transposed<G>(sv, 0.f, s1, s2);
    ok_sv = (__ballot_sync(0xffffffffu, c <= tol) >> base) & 1u;
    S1 = __shfl_sync(0xffffffffu, c, base + 2 * (G / 4));
    S2 = __shfl_sync(0xffffffffu, c, base + 3 * (G / 4));
  } else {
    S1 = group_sum<G>(s1);
    S2 = group_sum<G>(s2);
    ok_sv = group_sum<G>(sv) <= tol;
  }
}

// Group totals of two partials (sv, r2) with log2(G) shuffles (transposed butterfly): ok_sv =
// (sv total <= tol) for the whole group, r2 broadcast.
template <int G>
__device__ __forceinline__ void group_reduce2(float sv, float r2, float tol, bool &ok_sv, float &R2) {
  if constexpr (G >= 2) {
    const int lane = threadIdx.x & 31;
    const int base = lane & ~(G - 1);
    const bool hi = lane & (G / 2);
    float c = (hi ? r2 : sv) + __shfl_xor_sync(0xffffffffu, hi ? sv : r2, G / 2);
#pragma unroll
    for (int o = G / 4; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    ok_sv = (__ballot_sync(0xffffffffu, c <= tol) >> base) & 1u;
    R2 = __shfl_sync(0xffffffffu, c, base + G / 2);
  } else {
    ok_sv = sv <= tol;
    R2 = r2;
  }
}

// Two predicates (total_a <= tol, total_b <= tol) for the group with log2(G) shuffles + a ballot
template <int G>
__device__ __forceinline__ void group_test2(float va, float vb, float tol, bool &ok_a, bool &ok_b) {
  if constexpr (G >= 2) {
    const int lane = threadIdx.x & 31;
    const int base = lane & ~(G - 1);
    const bool hi = lane & (G / 2);
    float c = (hi ? vb : va) + __shfl_xor_sync(0xffffffffu, hi ? va : vb, G / 2);
#pragma unroll
    for (int o = G / 4; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    const unsigned bal = __ballot_sync(0xffffffffu, c <= tol);
    ok_a = (bal >> base) & 1u;
    ok_b = (bal >> (base + G / 2)) & 1u;
  } else {
    ok_a = va <= tol;
    ok_b = vb <= tol;
  }
}

// ---- packed fp32x2 helpers (sm_100 FADD2 / FFMA2: two slots of FP32 work per issue) --------
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
// a - b as one FFMA2 with a broadcast -1 (exact: b * -1 is exact, one rounding of the sum);
// FADD2 has no operand-negate modifier, so a negated pair would cost two scalar FADDs.
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.f, -1.f), a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 splat2(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 clamp2(float2 u, float2 t) {
  return make_float2(fminf(fmaxf(u.x, -t.x), t.x), fminf(fmaxf(u.y, -t.y), t.y));
}

// MUFU reciprocal (rcp.approx.ftz: ~1 ulp; __frcp_rn adds an IEEE fix-up with a slow path)
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

#define HOPF_SLOT(arr, j) (((j) & 1) ? (arr)[(j) >> 1].y : (arr)[(j) >> 1].x)

// kappa pair of this lane from shared memory (non-union kernels).  ld.volatile keeps the load
// inside the loop (no hoisting back into registers): kappa is the same for every point, so it
// is held once per CTA instead of occupying CPL registers per thread.
__device__ __forceinline__ float2 lds_volatile2(const float2 *p) {
  float2 v;
  asm volatile("ld.volatile.shared.v2.f32 {%0,%1}, [%2];"
               : "=f"(v.x), "=f"(v.y)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

// One kernel template for the diagonal and the union entry points.
//   UNION = false: K1/K2 (kappa for the whole CTA in shared memory, one solve per point)
//   UNION = true : K4 (K solves per point, kappa per set in registers, running arg-min,
//                  optional Y / kstar / phi_k)
//
// Slots are processed in pairs (slot j <-> pair j/2, half j&1) with packed FP32x2
// instructions, and every state variable is updated in place (no loop-carried copies):
//   d <- d + (d' - d), v <- v + (v' - v) reproduce d', v' to within one rounding and keep the
//   exact zeros of the shrink (d' = 0 gives d - d = 0).  The l2 path carries nd = -d and the
//   CTA holds -kappa, so that every subtraction it needs is a plain FADD2/FFMA2.
//
// Per-point stop handling: a group whose solve stops (paper test, max_iter, t == 0, invalid)
// freezes its d (the in-place update is multiplied by live = 0) and waits; the warp runs the
// finalize/refill branch once at least half of its groups wait (or all of its remaining ones),
// so that with G < 32 the branch is shared by several groups instead of run once per group.
// __launch_bounds__(128, 3): at most 168 registers, i.e. 3 warps per SM sub-partition (each
// SMSP has a 16K-register file); the widest variants otherwise take ~195 registers and only
// 2 warps per SMSP, which leaves the dependent FP32x2 chains exposed.
template <int G, int CPL, int HK, bool UNION>
__global__ void __launch_bounds__(128, ((HK >= 3 || UNION) && CPL <= 16) ? 4 : 3) hopf_diag_kernel(const DiagParams p) {
  constexpr bool KSM = !UNION;            // -kappa in shared memory
  constexpr int NP = (CPL + 1) / 2;       // slot pairs (an odd CPL gets one padding slot)
  constexpr int GPW = 32 / G;             // groups per warp
#ifndef HOPF_WAIT_NUM
#define HOPF_WAIT_NUM 2
#endif
  constexpr int WAIT_THRESHOLD = GPW > 1 ? (GPW * HOPF_WAIT_NUM / 4 > 0 ? GPW * HOPF_WAIT_NUM / 4 : 1) : 1;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int n = p.n;
  const float lam = p.lambda, tol = p.tol;
  // slots j < jmax of this lane hold real coordinates (i = gl + G*j < n)
  const int jmax = (n - gl + G - 1) / G;

  // Per-slot registers (pairs).  d holds -d on the l2 path.
  float2 xh[NP], d[NP], b[NP], v[NP];
  float2 tau[HK == HK_WL1 ? NP : 1];
  // union: -kappa / kappa of every set in dynamic shared memory ([K][NP*G + 1] float2, the odd
  // row stride spreads groups at different sets over the banks); x is re-read from global (L1 /
  // L2) at each set start, and the best set's grad (and y) go to global memory when a set
  // improves the running minimum: no per-point vectors beyond x_hat, d, b, v in registers
  extern __shared__ float2 kapk_s[];
  constexpr int KROW = NP * G + 1;

  // -kappa_i (l2) or kappa_i (l1) = lambda/(D_i+lambda), layout [pair][G] of float2
  __shared__ __align__(16) float2 kap_s[KSM ? NP * G : 1];
  // non-union: D_i, 1/(D_i + lambda) and w_i by coordinate, staged once per CTA for the
  // per-point setup and finalize (they were re-fetched from global per point)
  constexpr bool WSM = KSM && (HK == HK_WL1 || HK == HK_ELL);
  __shared__ float D_s[KSM ? G * CPL : 1], di_s[KSM ? G * CPL : 1], w_s[WSM ? G * CPL : 1];
  // ELL: (w_i, 1/w_i) pairs in the kappa layout; padded slots hold w = 1 (their u is 0)
  constexpr bool ELL = HK == HK_ELL;
  constexpr bool LINF = HK == HK_LINF;
  static_assert(!((ELL || LINF) && UNION), "ELL / LINF are instantiated for hopf_eval_diag only");
  __shared__ __align__(16) float2 w2_s[ELL ? NP * G : 1];
  const float ksign = (HK == HK_L2) ? -1.f : 1.f;
  if (KSM) {
    for (int e = threadIdx.x; e < NP * G; e += blockDim.x) {
      const int pp = e / G, l = e % G;
      const int i0 = l + G * (2 * pp), i1 = l + G * (2 * pp + 1);
      float2 kv;
      kv.x = (2 * pp < CPL && i0 < n) ? ksign * __fdividef(lam, __ldg(p.D + i0) + lam) : 0.f;
      kv.y = (2 * pp + 1 < CPL && i1 < n) ? ksign * __fdividef(lam, __ldg(p.D + i1) + lam) : 0.f;
      kap_s[e] = kv;
    }
    for (int i = threadIdx.x; i < G * CPL; i += blockDim.x) {
      const float Dv = i < n ? __ldg(p.D + i) : 1.f;
      D_s[i] = Dv;
      di_s[i] = __fdividef(1.f, Dv + lam);
      if (WSM) w_s[i] = i < n ? __ldg(p.w + i) : 0.f;
    }
    if (ELL) {
      for (int e = threadIdx.x; e < NP * G; e += blockDim.x) {
        const int pp = e / G, l = e % G;
        const int i0 = l + G * (2 * pp), i1 = l + G * (2 * pp + 1);
        const float w0 = (2 * pp < CPL && i0 < n) ? __ldg(p.w + i0) : 1.f;
        const float w1 = (2 * pp + 1 < CPL && i1 < n) ? __ldg(p.w + i1) : 1.f;
        w2_s[e] = make_float2(w0, w1);
      }
    }
    __syncthreads();
  }
  if (UNION) {
    for (int e = threadIdx.x; e < p.K * KROW; e += blockDim.x) {
      const int k = e / KROW, r = e % KROW;
      float2 kv = splat2(0.f);
      if (r < NP * G) {
        const int pp = r / G, l = r % G;
        const int i0 = l + G * (2 * pp), i1 = l + G * (2 * pp + 1);
        const float *Dk = p.D + (size_t)k * n;
        kv.x = (2 * pp < CPL && i0 < n) ? ksign * __fdividef(lam, __ldg(Dk + i0) + lam) : 0.f;
        kv.y = (2 * pp + 1 < CPL && i1 < n) ? ksign * __fdividef(lam, __ldg(Dk + i1) + lam) : 0.f;
      }
      kapk_s[e] = kv;
    }
    __syncthreads();
  }
  // ELL: min_i w_i, the scale of the Newton stopping test on mu
  float wmin = 1.f;
  if (ELL) {
    wmin = __int_as_float(0x7f800000);
    for (int i = 0; i < n; i++) wmin = fminf(wmin, w_s[i]);
  }

  // points: the first two of a group static (gid, gid + ngroups); later ones claimed from
  // p.claim, one claim per event for all groups that start a point (lane 0 adds their count; a
  // group's index is base + its rank), resolved at the warp's next event and used at the
  // group's next start, so the atomic's latency is off the critical path.  Not for a thread per
  // point (G = 1: n <= 16, launches of about 3 points per thread, where the claims cost more
  // than they balance: p16_id_l2 0.064 -> 0.076 ms); the host passes no counter there.
  constexpr bool CLAIMS = G > 1;
  __shared__ unsigned zero_lanes[CLAIMS ? 32 : 1];
  if constexpr (CLAIMS) {
    zero_lanes_init(zero_lanes);
    __syncthreads();
  }
  int64_t pt = gid, pn = gid + ngroups, pc = 0;   // current, next, resolved claim
  unsigned long long wclaim = 0;                 // lane 0: base of the last claim
  bool pend = false;                             // this group's claim is not resolved yet
  unsigned rk = 0;                               // its rank in that claim
  const unsigned gbase = (unsigned)(lane & ~(G - 1));
  auto claim = [&](bool start) {   // collective: the groups with `start` set claim one point each
    if constexpr (!CLAIMS) return;
    const unsigned cm = __ballot_sync(0xffffffffu, gl == 0 && start);
    if (start) { pend = true; rk = __popc(cm & ((1u << gbase) - 1u)); }
    const unsigned zoff = lane_zero(zero_lanes, lane);
    if (lane == 0 && cm && p.claim) wclaim = atomicAdd(p.claim + zoff, (unsigned long long)__popc(cm));
  };
  bool have = pt < p.M;
  bool waiting = false; // the current solve stopped; d is frozen until the warp finalizes
  int wstatus = 0;      // its status (iteration, 0, -max_iter or INT32_MIN)
  int it = 0;           // completed (3.4a) half-steps (l2) / iterations (l1) of the solve
  int kset = 0;         // union: current set
  float tt = 0.f;       // t of the current point
  float tauS = 0.f;     // scalar threshold t/lambda
  int spec = 0;         // 0 normal, 1 t == 0, 2 invalid
  float s_cur = 1.f;    // l2: shrink factor of the pending (3.4b)
  float mu = 0.f;       // ELL / LINF: multiplier of the last projection (warm start of the next)
  bool sv_ok = false;   // l2: ||v^k - v^{k-1}||^2 <= tol of the pending iteration
  float best = 0.f, bgn = 0.f;   // union: running minimum and ||grad|| of its set
  int bestk = -1, bestit = 0;
  // distance mode: Newton evaluations at s > 0 so far, bracket (s_lo, s_hi) of the root
  int nn = 0;
  float s_lo = 0.f, s_hi = 0.f;
  const bool DIST = UNION && p.dist != nullptr;
  // thread per point (G = 1, CPL a multiple of 4) with 16-byte aligned rows (n % 4 == 0 and aligned
  // bases; warp-uniform): x loads and grad stores as float4 (padded slots hold zeros)
  const bool VEC1 = (G == 1 && CPL % 4 == 0 && !UNION) && (n & 3) == 0 &&
                    (((uintptr_t)p.X | (uintptr_t)p.grad) & 15) == 0;

  // ---- load the point (x, t) into registers; detect t == 0 / invalid (collective) -----------
  auto load_point = [&](bool active) {
    bool bad = false;
    if (active) {
      tt = DIST ? 0.f : p.tscale * __ldg(p.t + pt);   // distance mode starts at s_0 = 0 (R24)
      bad = !(tt >= 0.f) || !finite_f(tt);
      const float *xrow = p.X + pt * (int64_t)n;
      float2 fin = splat2(0.f);   // x * 0 accumulates NaN iff some x is NaN or infinite
      if (VEC1) {
        // thread per point with 16-byte rows: the row as float4 loads (slots j = coordinates)
#pragma unroll
        for (int q4 = 0; q4 < NP / 2; q4++) {
          const float4 x4 = (4 * q4 < jmax) ? __ldg(reinterpret_cast<const float4 *>(xrow) + q4)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
          fin = fma2(make_float2(x4.x, x4.y), splat2(0.f), fin);
          fin = fma2(make_float2(x4.z, x4.w), splat2(0.f), fin);
          if (!UNION) { xh[2 * q4] = make_float2(x4.x, x4.y); xh[2 * q4 + 1] = make_float2(x4.z, x4.w); }
        }
      } else {
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const int j0 = 2 * q, j1 = 2 * q + 1;
        const float x0 = (j0 < CPL && j0 < jmax) ? __ldg(xrow + gl + G * j0) : 0.f;
        const float x1 = (j1 < CPL && j1 < jmax) ? __ldg(xrow + gl + G * j1) : 0.f;
        fin = fma2(make_float2(x0, x1), splat2(0.f), fin);
        if (!UNION) xh[q] = make_float2(x0, x1);   // union: re-read per set in setup_solve
      }
      }
      bad |= !(fin.x == 0.f && fin.y == 0.f);
    }
    bad = group_any<G>(bad);
    if (active) {
      spec = bad ? 2 : (tt == 0.f ? 1 : 0);
      tauS = tt / lam;
    }
  };

  // ---- set up one solve: centred start v0 = d0 = x - c, b0 = 0 (reading R5) -------
  auto setup_solve = [&]() {
    const float *Dp = UNION ? p.D + (size_t)kset * n : p.D;
    const float *cp = UNION ? p.c + (size_t)kset * n : p.c;
    const float tl = tt / lam;
#pragma unroll
    for (int q = 0; q < NP; q++) {
      const int j0 = 2 * q, j1 = 2 * q + 1;
      const bool ok0 = j0 < CPL && j0 < jmax, ok1 = j1 < CPL && j1 < jmax;
      const int i0 = gl + G * j0, i1 = gl + G * j1;
      const float c0 = (cp && ok0) ? __ldg(cp + i0) : 0.f, c1 = (cp && ok1) ? __ldg(cp + i1) : 0.f;
      float2 xv = xh[q];
      if (UNION) {
        const float *xrow = p.X + pt * (int64_t)n;
        xv = make_float2(ok0 ? __ldg(xrow + i0) : 0.f, ok1 ? __ldg(xrow + i1) : 0.f);
      }
      const float xt0 = xv.x - c0, xt1 = xv.y - c1;   // padded slots: x = c = 0
      float di0, di1;
      if (KSM) {   // shared-memory tables are padded (D = 1, w = 0)
        di0 = j0 < CPL ? di_s[i0] : 1.f;
        di1 = j1 < CPL ? di_s[i1] : 1.f;
      } else {
        const float D0 = ok0 ? __ldg(Dp + i0) : 1.f, D1 = ok1 ? __ldg(Dp + i1) : 1.f;
        di0 = __fdividef(1.f, D0 + lam);
        di1 = __fdividef(1.f, D1 + lam);
      }
      if (HK == HK_WL1)
        tau[q] = KSM ? make_float2(j0 < CPL ? tl * w_s[i0] : 0.f, j1 < CPL ? tl * w_s[i1] : 0.f)
                     : make_float2(ok0 ? tl * __ldg(p.w + i0) : 0.f, ok1 ? tl * __ldg(p.w + i1) : 0.f);
      const float2 xt = make_float2(xt0, xt1);
      xh[q] = make_float2(xt0 * di0, xt1 * di1);
      if (HK == HK_L2) {
        d[q] = make_float2(-xt0, -xt1);   // -d^0 = -(x - c)
        b[q] = xt;                        // pending u with s = 1 reproduces d^0 and b^0 = 0
      } else {
        d[q] = xt;                        // d^0 = x - c
        b[q] = splat2(0.f);               // b^0 = 0
      }
      v[q] = xt;                          // v^0 = x - c
    }
    it = 0;
    s_cur = 1.f;
    mu = 0.f;
    sv_ok = false;
    waiting = false;
  };

  load_point(have);
  claim(have);
  if (have) {
    setup_solve();
    if (UNION) { best = __int_as_float(0x7f800000); bestk = -1; bestit = 0; }
  } else {
#pragma unroll
    for (int q = 0; q < NP; q++) {
      xh[q] = d[q] = b[q] = v[q] = splat2(0.f);
    }
  }

  unsigned my_iters = 0;   // this lane's share of p.iter_total (group lane 0 counts)
  while (__any_sync(0xffffffffu, have)) {
    // ================= one loop trip (all lanes, branch-free) ===============================
    // l1/wl1: the full iteration k = it+1, one reduction of (sd, sb, sv).
    // l2: software-pipelined so that one reduction per iteration suffices: the trip finishes
    //     iteration k = it ((3.4b), (3.4c) with the shrink factor s_k reduced in the previous
    //     trip, plus the test sums sd_k, sb_k) and starts iteration k+1 ((3.4a), u_{k+1}, the
    //     test sum sv_{k+1} and ||u_{k+1}||^2); the four sums are reduced together.  Between trips
    //     b holds u_{k+1}; d = d_k is not touched by the (3.4a) half, so a point that stops at
    //     k outputs d_k.  After setup_solve the first trip's (3.4b) half is the identity
    //     (s = 1, u = x - c) and its test is skipped.
    float2 a0 = splat2(0.f), b0 = a0, c0 = a0, r0 = a0;   // one packed accumulator per sum
    const float2 sP = splat2(s_cur), tP = splat2(tauS);
    const float2 nsP = splat2(-s_cur), omsP = splat2(1.f - s_cur), na_sP = splat2(1.f - 2.f * s_cur);
    const float live = waiting ? 0.f : 1.f;
    // l2: ||d^k - d^{k-1}||^2 and ||d^k - v^k||^2 only matter when ||v^k - v^{k-1}||^2 <= tol
    // (sv_ok, known before the trip): trips in which no group of the warp has sv_ok skip both
    // sums (10 instead of 13 packed ops per coordinate pair); the stopping decisions are the
    // paper's exactly (a group without sv_ok cannot stop at k whatever the other two sums are).
    const bool full_test = (HK != HK_L2) || __any_sync(0xffffffffu, sv_ok);
    auto trip = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const float2 kq = KSM ? lds_volatile2(kap_s + q * G + gl) : lds_volatile2(kapk_s + kset * KROW + q * G + gl);
        if (HK == HK_L2) {
          // d[q] = -d_{k-1}, kq = -kappa, b[q] = u_k.  d_k = s_k u_k, b_k = (1 - s_k) u_k and
          // d_k - b_k = (2 s_k - 1) u_k are scalings of u_k ((3.4b), (3.4c)); a waiting group
          // keeps its d (select)
          const float2 u = b[q];
          if (FULL) {
            const float2 dd = fma2(sP, u, d[q]);         // d_k - d_{k-1}
            d[q] = fma2(dd, splat2(-live), d[q]);        // -d_k (frozen while waiting)
            const float2 dmv = add2(d[q], v[q]);         // v^k - d^k
            a0 = fma2(dd, dd, a0); b0 = fma2(dmv, dmv, b0);
          } else {
            const float2 dn = __fmul2_rn(nsP, u);        // -d_k
            d[q] = waiting ? d[q] : dn;
          }
          const float2 bk = __fmul2_rn(omsP, u);         // b_k
          const float2 na = __fmul2_rn(na_sP, u);        // -(d_k - b_k)
          const float2 t = sub2(xh[q], v[q]);
          const float2 dv = fma2(kq, na, t);             // (3.4a): v_{k+1} - v_k
          v[q] = add2(v[q], dv);                         // v_{k+1}
          b[q] = add2(v[q], bk);                         // u_{k+1} = v_{k+1} + b_k
          c0 = fma2(dv, dv, c0); r0 = fma2(b[q], b[q], r0);
        } else {
          const float2 a = sub2(d[q], b[q]);
          const float2 t = sub2(xh[q], v[q]);
          const float2 dv = fma2(kq, a, t);              // (3.4a): v^k - v^{k-1}
          v[q] = add2(v[q], dv);                         // v^k
          const float2 u = add2(v[q], b[q]);
          b[q] = clamp2(u, HK == HK_WL1 ? tau[q] : tP);  // projection on [-tau, tau] (Moreau)
          const float2 dn = sub2(u, b[q]);               // (3.4b) shrink_1; b^k = u - d^k
          const float2 dd = sub2(dn, d[q]);
          d[q] = fma2(dd, splat2(live), d[q]);           // d^k (exact zeros kept; frozen while waiting)
          // ||d^k - v^k||^2 is formed after the trip only for groups whose other two sums pass
          a0 = fma2(dd, dd, a0); c0 = fma2(dv, dv, c0);
        }
      }
    };
    bool ell_ok_sv = false;
    if constexpr (ELL) {
      // (3.4a) and u = v + b for every coordinate (b holds u until the projection is known),
      // fused with the first Newton evaluation at the warm-start mu (below)
      float2 s1 = splat2(0.f), s2 = s1;
      // 1 / (w + mu_e) at the last evaluated mu_e, reused by (3.4b) below when it fits in
      // registers (CPL <= 16); wider variants recompute it (MUFU)
      constexpr bool RR = NP <= 8;
      float2 rr[RR ? NP : 1];
      float mu_e = mu;
      {
        const float2 muP = splat2(mu);
#pragma unroll
        for (int q = 0; q < NP; q++) {
          const float2 kq = lds_volatile2(kap_s + q * G + gl);
          const float2 a = sub2(d[q], b[q]);
          const float2 t = sub2(xh[q], v[q]);
          const float2 dv = fma2(kq, a, t);
          v[q] = add2(v[q], dv);
          const float2 u = add2(v[q], b[q]);
          b[q] = u;
          c0 = fma2(dv, dv, c0);
          const float2 w = lds_volatile2(w2_s + q * G + gl);
          const float2 e = add2(w, muP);
          const float2 r = make_float2(rcp_approx(e.x), rcp_approx(e.y));
          if (RR) rr[q] = r;
          const float2 h = __fmul2_rn(u, r);             // u / (w + mu)
          const float2 wh2 = __fmul2_rn(__fmul2_rn(w, h), h);
          s1 = add2(s1, wh2);
          s2 = fma2(wh2, r, s2);
        }
      }
      // (3.4b) = prox_{tau ||.||_W}(u) = u - tau P(u / tau), P the projection on the dual
      // ellipsoid {z : <z, W^-1 z> <= 1} (Moreau): P(z) = w z / (w + mu), mu >= 0,
      // mu = 0 iff u / tau is inside (sum u^2 / w <= tau^2), else the root of
      // S1(mu) = sum w u^2 / (w + mu)^2 = tau^2.  Newton on psi(mu) = 1 / sqrt(S1) - 1 / tau
      // (the trust-region secular form: psi is concave and nearly linear, so from either side a
      // step lands at or left of the root, then the iteration is monotone):
      //   mu <- max(0, mu + (S1 / S2) (sqrt(S1) / tau - 1)),   S2 = sum w u^2 / (w + mu)^3,
      // warm-started at the previous iteration's mu.  The clamp at 0 is the inside case: the
      // root is then negative, the iterates stop at 0 and d' = 0 * u / w = 0 exactly.  Newton's
      // error after a step h is O(h^2 / (w + mu)) (psi'' / psi' ~ 1 / (w + mu)), so a step below
      // 1e-3 (mu + min w) leaves ~1e-6 (mu + min w): the iterate after that step is accepted
      // without another evaluation (on C2e 1.7 evaluations per split Bregman iteration).
      // The paper runs Newton on the same root from mu_0 = 0 on sum w u^2/(w+mu) + mu tau^2 and
      // stops at |step| <= 1e-8, after testing inside-ness (the oracle does; reading R27)
      float S1, S2;
      group_reduce3<G>(s1.x + s1.y, s2.x + s2.y, c0.x + c0.y, tol, S1, S2, ell_ok_sv);
      const float itau = rcp_approx(tauS);
      bool act = have && !waiting && spec == 0;
      int nit = 0;
      for (;;) {
        if (act) {
          const float mun = S2 > 0.f ? fmaxf(fmaf(S1 * rcp_approx(S2), fmaf(sqrtf(S1), itau, -1.f), mu), 0.f)
                                     : 0.f;   // u = 0: d' = 0
          act = !(fabsf(mun - mu) <= 1e-3f * (mun + wmin)) && ++nit < 30;
          mu = mun;
        }
        if (!__any_sync(0xffffffffu, act)) break;
        float2 t1 = splat2(0.f), t2 = splat2(0.f);
        const float2 muP = splat2(mu);
        mu_e = mu;
#pragma unroll
        for (int q = 0; q < NP; q++) {
          const float2 w = lds_volatile2(w2_s + q * G + gl);
          const float2 e = add2(w, muP);
          const float2 r = make_float2(rcp_approx(e.x), rcp_approx(e.y));
          if (RR) rr[q] = r;
          const float2 h = __fmul2_rn(b[q], r);
          const float2 wh2 = __fmul2_rn(__fmul2_rn(w, h), h);
          t1 = add2(t1, wh2);
          t2 = fma2(wh2, r, t2);
        }
        S1 = group_sum<G>(t1.x + t1.y);
        S2 = group_sum<G>(t2.x + t2.y);
      }
      // (3.4b): d' = u - w u / (w + mu) = mu u / (w + mu);  (3.4c): b' = u - d'.
      // 1 / (w + mu) from the last evaluation at mu_e: mu - mu_e is the final Newton step
      // (<= 1e-3 (mu + min w) unless the cap stopped it), corrected to first order,
      // r (1 - (mu - mu_e) r), i.e. to ~1e-6 relative
      const float mf = mu;
      const float2 muP = splat2(mf);
      const float2 ndel = splat2(mu_e - mf);
#pragma unroll
      for (int q = 0; q < NP; q++) {
        float2 r;
        if constexpr (RR) {
          r = __fmul2_rn(rr[q], fma2(ndel, rr[q], splat2(1.f)));
        } else {
          const float2 e = add2(lds_volatile2(w2_s + q * G + gl), muP);
          r = make_float2(rcp_approx(e.x), rcp_approx(e.y));
        }
        const float2 u = b[q];
        const float2 dn = __fmul2_rn(__fmul2_rn(muP, u), r);
        b[q] = sub2(u, dn);
        const float2 dd = sub2(dn, d[q]);
        d[q] = fma2(dd, splat2(live), d[q]);
        a0 = fma2(dd, dd, a0);
      }
    } else if constexpr (LINF) {
      // (3.4a) and u = v + b (b holds u until the projection is known), fused with the first
      // evaluation of the l1-ball sums at the warm-start mu: S1 = sum max(|u_i| - mu, 0) (small
      // terms: the Newton step is formed in delta form, mu + (S1 - tau) / S2, because
      // sum_{A} |u_i| - |A| mu cancels catastrophically when the root sits just below a cluster
      // of |u_i|), S2 = #{|u_i| > mu}
      float2 sa = splat2(0.f), na = sa;
      float mu_e = mu;
      {
        const float2 muP = splat2(mu);
#pragma unroll
        for (int q = 0; q < NP; q++) {
          const float2 kq = lds_volatile2(kap_s + q * G + gl);
          const float2 a = sub2(d[q], b[q]);
          const float2 t = sub2(xh[q], v[q]);
          const float2 dv = fma2(kq, a, t);
          v[q] = add2(v[q], dv);
          const float2 u = add2(v[q], b[q]);
          b[q] = u;
          c0 = fma2(dv, dv, c0);
          const float ex = fabsf(u.x) - muP.x, ey = fabsf(u.y) - muP.y;
          sa.x += fmaxf(ex, 0.f);
          sa.y += fmaxf(ey, 0.f);
          na.x += ex > 0.f ? 1.f : 0.f;
          na.y += ey > 0.f ? 1.f : 0.f;
        }
      }
      // pi_{tau B1}(u) = shrink_1(u, mu), mu >= 0 with sum_i max(|u_i| - mu, 0) = tau
      // (eq. condition_mu_linfty); mu = 0 iff ||u||_1 <= tau (inside: d' = 0).
      // F(mu) = sum max(|u_i| - mu, 0) - tau is convex, decreasing and piecewise affine, and its
      // Newton step from mu is mu' = mu + (S1(mu) - tau) / S2(mu) (the active-set average): from the
      // right of the root it lands at or left of it, from the left it increases monotonically
      // and stops at the root as soon as the active set stops changing.  Warm-started at the
      // previous iteration's mu and clamped at 0.  A step whose active set is unchanged at the
      // new mu (no |u_i| between mu and mu', a ballot, no reduction) is exact: accepted with no
      // further evaluation.  The paper (and the oracle) sorts the breakpoints {0} U {|u_i|/tau}
      // and interpolates on the bracketing affine piece; both give the same root (reading R28)
      float S1, S2;
      group_reduce3<G>(sa.x + sa.y, na.x + na.y, c0.x + c0.y, tol, S1, S2, ell_ok_sv);
      bool act = have && !waiting && spec == 0;
      int nit = 0;
      for (;;) {
        float mun = mu_e;
        if (act) mun = S2 > 0.f ? fmaxf(mu_e + __fdividef(S1 - tauS, S2), 0.f) : 0.f;
        // empty active set at mu_e (a warm start above every |u_i|): step to the root of the top
        // piece, max |u| - tau, at or left of the root, instead of falling back to 0
        if (__any_sync(0xffffffffu, act && S2 == 0.f)) {
          float um = 0.f;
#pragma unroll
          for (int q = 0; q < NP; q++) um = fmaxf(um, fmaxf(fabsf(b[q].x), fabsf(b[q].y)));
          um = group_max<G>(um);
          if (act && S2 == 0.f) mun = fmaxf(um - tauS, 0.f);
        }
        bool cross = false;
#pragma unroll
        for (int q = 0; q < NP; q++) {
          const float ax = fabsf(b[q].x), ay = fabsf(b[q].y);
          cross |= ((ax > mu_e) != (ax > mun)) || ((ay > mu_e) != (ay > mun));
        }
        cross = group_any<G>(cross);
        // a breakpoint at the root makes fp32 steps alternate across it: a step within a few
        // ulps of mu is accepted as the root
        const bool tiny = fabsf(mun - mu_e) <= HOPF_TINY_STEP * fmaxf(mun, 1e-30f);
        if (act && (!cross || tiny || ++nit >= 64)) { mu = mun; act = false; }
        if (!__any_sync(0xffffffffu, act)) break;
        if (act) mu_e = mun;
        float2 ta = splat2(0.f), tn = ta;
#pragma unroll
        for (int q = 0; q < NP; q++) {
          const float ex = fabsf(b[q].x) - mu_e, ey = fabsf(b[q].y) - mu_e;
          ta.x += fmaxf(ex, 0.f);
          ta.y += fmaxf(ey, 0.f);
          tn.x += ex > 0.f ? 1.f : 0.f;
          tn.y += ey > 0.f ? 1.f : 0.f;
        }
        S1 = group_sum<G>(ta.x + ta.y);
        S2 = group_sum<G>(tn.x + tn.y);
      }
      // (3.4b): d' = u - shrink_1(u, mu) = clamp(u, -mu, mu);  (3.4c): b' = u - d'
      const float2 muP = splat2(mu);
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const float2 u = b[q];
        const float2 dn = clamp2(u, muP);
        b[q] = sub2(u, dn);
        const float2 dd = sub2(dn, d[q]);
        d[q] = fma2(dd, splat2(live), d[q]);
        a0 = fma2(dd, dd, a0);
      }
    } else if (full_test) {
      trip(std::true_type{});
    } else {
      trip(std::false_type{});
    }
    const float psd = a0.x + a0.y, psb = b0.x + b0.y;
    const float psv = c0.x + c0.y, pr2 = r0.x + r0.y;
    bool conv;
    int kdone;
    {
      float r2;
      bool ok_sd, ok_sb, ok_sv;
      if constexpr (ELL || LINF) {   // sv was reduced with the Newton sums
        ok_sd = group_sum<G>(psd) <= tol;
        ok_sv = ell_ok_sv;
        ok_sb = false;
        r2 = 0.f;
      } else if (HK != HK_L2) {
        // l1 / wl1: the trip accumulated only ||d^k - d^{k-1}||^2 and ||v^k - v^{k-1}||^2
        group_test2<G>(psd, psv, tol, ok_sd, ok_sv);
        ok_sb = false;
        r2 = 0.f;
      } else if (!full_test) {
        // no group of the warp can stop at this iteration (none had ||v^k - v^{k-1}||^2 <=
        // tol): only ||v^{k+1} - v^k||^2 and ||u_{k+1}||^2 are needed, two values per group
        group_reduce2<G>(psv, pr2, tol, ok_sv, r2);
        ok_sd = ok_sb = false;
      } else {
        group_reduce4<G>(psd, psb, psv, pr2, tol, r2, ok_sd, ok_sb, ok_sv);
      }
      if (HK == HK_L2) {
        kdone = it;
        conv = (it >= 1) && sv_ok && ok_sd && ok_sb;   // P:1597-1601 for iteration k = it
        sv_ok = ok_sv;                                  // ||v^{k+1} - v^k||^2 <= tol, next trip
        // shrink_2 factor of k+1, max(||u|| - tau, 0) / ||u|| = 1 - tau / ||u||,
        // with the hardware reciprocal square root (reading R20)
        s_cur = (r2 > tauS * tauS) ? fmaf(-tauS, rsqrtf(r2), 1.f) : 0.f;
        it++;
      } else {
        it++;
        kdone = it;
        // P:1597-1601.  The trip accumulated ||d^k - d^{k-1}||^2 and ||v^k - v^{k-1}||^2 only;
        // where both pass, ||d^k - v^k||^2 is summed now from the registers (d = d^k, v = v^k),
        // so the decision is the paper's at every iteration (the third sum is rarely needed)
        const bool need = ok_sd && ok_sv;
        conv = false;
        if (__any_sync(0xffffffffu, need)) {
          float sb = 0.f;
#pragma unroll
          for (int q = 0; q < NP; q++) {
            const float2 dmv = sub2(d[q], v[q]);
            sb = fmaf(dmv.x, dmv.x, fmaf(dmv.y, dmv.y, sb));
          }
          sb = group_sum<G>(sb);
          conv = need && sb <= tol;
        }
        (void)ok_sb;
      }
    }
    if (have && !waiting && (spec != 0 || (kdone >= 1 && (conv || kdone >= p.max_iter)))) {
      waiting = true;
      wstatus = spec == 2 ? INT32_MIN : (spec == 1 ? 0 : (conv ? kdone : -p.max_iter));
      if (spec == 0) my_iters += (unsigned)kdone;
    }
    {
      const unsigned gbit = (gl == 0) ? 1u : 0u;
      const unsigned wb = __ballot_sync(0xffffffffu, waiting && gbit);
      if (wb == 0u) continue;   // the common case: one vote
      const int nwait = __popc(wb);
      const int nhave = __popc(__ballot_sync(0xffffffffu, have && gbit));
      if (nwait < WAIT_THRESHOLD && nwait < nhave) continue;
    }
    const bool done = waiting;

    // ============ finalize (all lanes compute; waiting groups store and refill) ==============
    // phi = <x - c, d> - 1/2 <d, D d> - t H(d) + gamma   ((3.3) at d, reading R2), with
    //   x - c = x_hat (D + lambda) recovered from registers.
    // t == 0: phi = J(x) = 1/2 <x-c, D^{-1}(x-c)> + gamma, grad = D^{-1}(x-c) (reading R6)
    const float *Dp = UNION ? p.D + (size_t)kset * n : p.D;
    // Padded slots (i >= n) hold x_hat = d = 0 and add nothing, so only global loads are
    // guarded (shared-memory tables are padded: D = 1, w = 0).  t == 0: dq = D^{-1}(x - c) and
    // the same expression <xt, dq> - 1/2 <dq, D dq> is J(x) - gamma = 1/2 <xt, D^{-1} xt>.
    float qs = 0.f, hsum = 0.f;
    // t == 0 groups are rare: one vote keeps their pass (divisions) out of the common path; it
    // replaces d by D^{-1}(x - c) (in the l2 path's negated storage) before the common loop
    if (__any_sync(0xffffffffu, done && spec == 1)) {
      if (done && spec == 1) {
#pragma unroll
        for (int q = 0; q < NP; q++) {
          const int j0 = 2 * q, j1 = 2 * q + 1;
          const bool ok0 = j0 < CPL && j0 < jmax, ok1 = j1 < CPL && j1 < jmax;
          const int i0 = gl + G * j0, i1 = gl + G * j1;
          const float D0 = KSM ? (j0 < CPL ? D_s[i0] : 1.f) : (ok0 ? __ldg(Dp + i0) : 1.f);
          const float D1 = KSM ? (j1 < CPL ? D_s[i1] : 1.f) : (ok1 ? __ldg(Dp + i1) : 1.f);
          const float g0 = __fdividef(xh[q].x * (D0 + lam), D0), g1 = __fdividef(xh[q].y * (D1 + lam), D1);
          d[q] = (HK == HK_L2) ? make_float2(0.f - g0, 0.f - g1) : make_float2(g0, g1);
        }
      }
    }
    if (done && spec != 2) {
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const int j0 = 2 * q, j1 = 2 * q + 1;
        const bool ok0 = j0 < CPL && j0 < jmax, ok1 = j1 < CPL && j1 < jmax;
        const int i0 = gl + G * j0, i1 = gl + G * j1;
        const float D0 = KSM ? (j0 < CPL ? D_s[i0] : 1.f) : (ok0 ? __ldg(Dp + i0) : 1.f);
        const float D1 = KSM ? (j1 < CPL ? D_s[i1] : 1.f) : (ok1 ? __ldg(Dp + i1) : 1.f);
        const float xt0 = xh[q].x * (D0 + lam), xt1 = xh[q].y * (D1 + lam);
        float2 dq = (HK == HK_L2) ? make_float2(0.f - d[q].x, 0.f - d[q].y) : d[q];
        qs = fmaf(xt0, dq.x, qs);
        qs = fmaf(-0.5f * D0 * dq.x, dq.x, qs);
        qs = fmaf(xt1, dq.y, qs);
        qs = fmaf(-0.5f * D1 * dq.y, dq.y, qs);
        if (HK == HK_L2) hsum = fmaf(dq.x, dq.x, fmaf(dq.y, dq.y, hsum));
        else if (ELL)
          hsum = fmaf((j0 < CPL ? w_s[i0] : 0.f) * dq.x, dq.x, fmaf((j1 < CPL ? w_s[i1] : 0.f) * dq.y, dq.y, hsum));
        else if (LINF)
          hsum = fmaxf(hsum, fmaxf(fabsf(dq.x), fabsf(dq.y)));
        else if (HK == HK_WL1)
          hsum = fmaf(KSM ? (j0 < CPL ? w_s[i0] : 0.f) : (ok0 ? __ldg(p.w + i0) : 0.f), fabsf(dq.x),
                      fmaf(KSM ? (j1 < CPL ? w_s[i1] : 0.f) : (ok1 ? __ldg(p.w + i1) : 0.f), fabsf(dq.y), hsum));
        else hsum += fabsf(dq.x) + fabsf(dq.y);
        d[q] = dq;   // from here on d holds the solve's gradient (+d)
      }
    }
    qs = group_sum<G>(qs);
    hsum = LINF ? group_max<G>(hsum) : group_sum<G>(hsum);
    const float gam = UNION ? __ldg(p.gk + kset) : p.gamma;
    float phiv;
    if (spec == 1) phiv = qs + gam;
    else phiv = qs - tt * ((HK == HK_L2 || ELL) ? sqrtf(hsum) : hsum) + gam;
    if (spec == 2) phiv = __int_as_float(0x7fc00000);

    bool point_done = done;
    bool restart = false;   // distance mode: the same point, the K sets again at a new s
    if (UNION) {
      // ||grad|| of this set's solve (all lanes take part in the reduction)
      float gc = 0.f;
#pragma unroll
      for (int q = 0; q < NP; q++) gc = fmaf(d[q].x, d[q].x, fmaf(d[q].y, d[q].y, gc));
      gc = sqrtf(group_sum<G>(gc));
      if (done) {
        if (p.phik && gl == 0) p.phik[pt * p.K + kset] = phiv;
        if (phiv < best) {   // strict: lowest k wins ties (R19); NaN never wins
          best = phiv; bestk = kset; bestit = wstatus; bgn = gc;
          // the new best set's grad and closest point go to memory now (a later, better set
          // overwrites them): y = x - t grad/||grad||, c_k if grad = 0 (R18);
          // distance mode: pi = y - s grad/||grad|| at the evaluated s
          const float ign = (gc > 0.f) ? __fdividef(1.f, gc) : 0.f;
          float *grow = p.grad + pt * (int64_t)n;
          float *yrow = p.Y ? p.Y + pt * (int64_t)n : nullptr;
          const float *xrow = p.X + pt * (int64_t)n;
#pragma unroll
          for (int j = 0; j < CPL; j++) {
            const int i = gl + G * j;
            if (j < jmax) {
              const float gj = HOPF_SLOT(d, j);
              grow[i] = spec == 2 ? __int_as_float(0x7fc00000) : gj;
              if (yrow) {
                const float xj = __ldg(xrow + i);
                float y;
                if (DIST) y = (tt > 0.f && gc > 0.f) ? xj - tt * (gj * ign) : xj;
                else if (gc > 0.f) y = xj - tt * (gj * ign);
                else y = __ldg(p.c + (size_t)kset * n + i);
                yrow[i] = y;
              }
            }
          }
        }
        point_done = (spec == 2) || (kset + 1 >= p.K);
      }
      const float gn = bgn;
      if (DIST && point_done && spec != 2 && bestk >= 0) {
        // distance mode: psi(y,s) = best, ||grad psi|| = gn; Newton in s with
        // d psi/dt = -||grad psi||, same step / stop / safeguard order as the oracle (R24-R26)
        const float s0 = tt;
        bool fin = false;
        if (nn == 0 && s0 == 0.f) {
          if (!(best > 0.f)) fin = true;                  // y in Omega: dist 0, proj y
          else { s_lo = 0.f; s_hi = __int_as_float(0x7f800000); }
        } else if (best > 0.f) {
          s_lo = s0;
        } else {
          s_hi = s0;
        }
        if (!fin && (nn >= p.max_newton || !(gn > 0.f))) fin = true;
        if (!fin) {
          float sn = s0 + best / gn;                        // eq. Newton_zero
          if (fabsf(sn - s0) <= p.stol * fmaxf(1.f, s0)) {
            fin = true;                                     // R26: keep the evaluated s
          } else {
            if (!(sn > s_lo && sn < s_hi)) sn = 0.5f * (s_lo + s_hi);   // R25
            point_done = false;                             // evaluate the K sets at sn
            restart = true;
            nn++;
            tt = sn;
            tauS = sn / lam;
            spec = 0;
          }
        }
      }
      if (point_done) {
        const bool nanpt = (spec == 2) || bestk < 0;
        if (gl == 0) {
          p.phi[pt] = nanpt ? __int_as_float(0x7fc00000) : best;
          p.iters[pt] = nanpt ? INT32_MIN : (DIST ? nn : bestit);
          if (p.kstar) p.kstar[pt] = nanpt ? -1 : bestk;
          if (DIST) p.dist[pt] = nanpt ? __int_as_float(0x7fc00000) : tt;
        }
        if (nanpt && p.phik)   // an invalid point's phi_k are NaN for every k
          for (int k = gl; k < p.K; k += G) p.phik[pt * p.K + k] = __int_as_float(0x7fc00000);
        if (nanpt) {   // grad and y of a valid point were written when its best set finished
          float *grow = p.grad + pt * (int64_t)n;
          float *yrow = p.Y ? p.Y + pt * (int64_t)n : nullptr;
#pragma unroll
          for (int j = 0; j < CPL; j++) {
            const int i = gl + G * j;
            if (j < jmax) {
              grow[i] = __int_as_float(0x7fc00000);
              if (yrow) yrow[i] = __int_as_float(0x7fc00000);
            }
          }
        }
      }
    } else if (done) {
      if (gl == 0) { p.phi[pt] = phiv; p.iters[pt] = wstatus; }
      float *grow = p.grad + pt * (int64_t)n;
      if (VEC1) {   // the row as float4 stores
        const float g = (spec == 2) ? __int_as_float(0x7fc00000) : 1.f;
#pragma unroll
        for (int q4 = 0; q4 < NP / 2; q4++)
          if (4 * q4 < jmax)
            reinterpret_cast<float4 *>(grow)[q4] =
                (spec == 2) ? make_float4(g, g, g, g)
                            : make_float4(d[2 * q4].x, d[2 * q4].y, d[2 * q4 + 1].x, d[2 * q4 + 1].y);
      } else {
#pragma unroll
      for (int j = 0; j < CPL; j++) {
        const int i = gl + G * j;
        if (j < jmax) grow[i] = (spec == 2) ? __int_as_float(0x7fc00000) : HOPF_SLOT(d, j);
      }
      }
    }
    // ---- refill: the next set of the point (union) or the next point of this group ---------
    if constexpr (CLAIMS) {
      const unsigned long long wb = __shfl_sync(0xffffffffu, wclaim, 0);   // the last claim's base
      if (pend) { pc = (int64_t)wb + 2 * ngroups + rk; pend = false; }
    }
    if (point_done) {
      pt = pn;
      pn = (CLAIMS && p.claim) ? pc : pn + ngroups;   // no counter: static stride
      have = pt < p.M;
    }
    load_point(point_done && have);   // collective (ballot inside): all lanes call it
    claim(point_done && have);
    if (done) {
      if (have) {
        kset = (point_done || restart) ? 0 : kset + 1;
        if (UNION && (point_done || restart)) { best = __int_as_float(0x7f800000); bestk = -1; bestit = 0; }
        if (point_done) nn = 0;
        setup_solve();
      } else {
#pragma unroll
        for (int q = 0; q < NP; q++) xh[q] = d[q] = b[q] = v[q] = splat2(0.f);
        spec = 0;
        waiting = false;
      }
    }
  }
  if (p.iter_total && gl == 0 && my_iters) atomicAdd(p.iter_total, (unsigned long long)my_iters);
}

}  // namespace hopf
