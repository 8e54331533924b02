/*
 * hopf.h — C ABI of the B200-native batched Hopf-formula evaluator (libhopf.so).
 *
 * For M independent queries (x, t) in R^n the library evaluates the Hopf formula
 *     phi(x,t) = -min_v { J*(v) + t H(v) - <x,v> }              PAPER.md (1.2)/(3.3)
 * and its gradient grad phi(x,t) = the unique minimiser
 * by split Bregman iterations
 *     v^{k+1} = argmin_v J*(v) - <x,v> + lambda/2 ||d^k - v - b^k||^2     (3.4a) P:834-836
 *     d^{k+1} = argmin_d t H(d) + lambda/2 ||d - v^{k+1} - b^k||^2         (3.4b) P:837-839
 *     b^{k+1} = b^k + v^{k+1} - d^{k+1}                                    (3.4c) P:840
 * started at v^0 = d^0 = x, b^0 = 0 and stopped at the first k with
 *     ||v^k - v^{k-1}||^2 <= tol, ||d^k - d^{k-1}||^2 <= tol, ||d^k - v^k||^2 <= tol.
 * (3.4b) is the prox of a 1-homogeneous H: shrink_1 or shrink_2
 * via Moreau's identity.  (3.4a) is the quadratic prox.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Array pointers are DEVICE pointers (except where a name ends in _host), caller-allocated
 *    and caller-owned, row-major point-major: X[i*n + j] is coordinate j of point i.
 *    fp32 unless stated.  The library never allocates, frees or retains caller memory.
 *  - Calls validate host-side arguments, enqueue their kernels on `stream` and return
 *    (asynchronous).  Outputs are valid once `stream` has been synchronised.
 *  - Return codes: HOPF_OK (0); HOPF_EINVAL (-1) invalid argument (M < 0, n < 1, K < 1,
 *    a required pointer NULL, lambda <= 0 or non-finite, tol < 0 or non-finite,
 *    max_iter < 1, unknown H kind, w NULL for HOPF_H_WL1, lambda different from the
 *    plan's, Y requested with a non-l2 H); HOPF_EUNSUPPORTED (-2) shape outside the
 *    compiled kernels (e.g. n > 1024 for the diagonal kernels, n != 256-multiple for dense);
 *    HOPF_ECUDA (-3) a CUDA launch/runtime error (hopf_last_error() has the text).
 *    M == 0 is a successful no-op.  Device-resident parameter values (D <= 0, NaN) are not
 *    validated on the host.
 *  - Per-point status iters[i]: k >= 1 converged at iteration k (the paper's test);
 *    0: t[i] == 0, answered directly as phi = J(x), grad = grad J(x) (Hopf needs t > 0,
 *    P:106-107); -max_iter: not converged, phi/grad from the last d are still written;
 *    INT32_MIN: invalid point (t < 0 or a non-finite x/t coordinate), phi/grad = NaN.
 *  - Outputs: grad := d at termination (reading R1 of DESIGN.md); phi := the Hopf
 *    objective (3.3) evaluated at d (R2).
 *  - Thread safety and concurrency: every entry point may be called from several host threads
 *    at once and on several streams / devices at once.  Per-call scratch (the maxh member
 *    buffers, the dense fix-up list) is stream-ordered memory from a library-owned pool of the
 *    current device (allocated and freed on the call's `stream`), so calls on different
 *    streams never share it.  hopf_eval_diag_host takes one of a per-device pool of pipeline
 *    contexts (internal streams + buffers) for the duration of the call.  Process-wide state
 *    otherwise consists of write-once caches (SM count, kernel attributes per device) and the
 *    per-thread error string / launch statistics.  All device pointers of a call, and a dense
 *    plan, must belong to the CURRENT device (hopf_eval_dense checks the plan's).
 *  - Point counter: long launches of the persistent kernels hand out points from a 64-bit
 *    counter in the same stream-ordered scratch (zeroed by a memset on `stream`); the
 *    environment variable HOPF_CLAIMS=0 / 1 forces the static point stride / the counter.
 *  - CUDA graphs: every device entry point is purely stream-ordered (scratch allocation and
 *    free, memsets and kernels on `stream`; no host synchronisation), so a call may be captured
 *    into a CUDA graph and replayed (make one uncaptured call first: it sets kernel attributes
 *    and warms the scratch pool).  hopf_eval_diag_host and hopf_dense_plan_create synchronise
 *    and cannot be captured.
 */
#ifndef HOPF_H_
#define HOPF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *hopf_stream_t; /* == cudaStream_t; NULL = legacy default stream */

enum {
  HOPF_OK = 0,
  HOPF_EINVAL = -1,
  HOPF_EUNSUPPORTED = -2,
  HOPF_ECUDA = -3
};

/* Hamiltonians (support functions of a box / a ball / an ellipsoid):
 *   HOPF_H_L1  : H(p) = sum_i |p_i|        (shrink_1, threshold t/lambda)
 *   HOPF_H_WL1 : H(p) = sum_i w_i |p_i|    (shrink_1, threshold t w_i/lambda), w_i > 0
 *   HOPF_H_L2  : H(p) = ||p||_2            (shrink_2, threshold t/lambda)
 *   HOPF_H_ELL : H(p) = sqrt(<p, diag(w) p>), w_i > 0  (NEXT-2: prox by projection on the dual
 *                ellipsoid, Newton on its multiplier)
 *   HOPF_H_LINF: H(p) = max_i |p_i|         (NEXT-2: prox by projection on the l1 ball,
 *                P:1348-1428)
 *   ELL and LINF: hopf_eval_diag and hopf_eval_maxh only (hopf_eval_union: HOPF_EUNSUPPORTED) */
typedef enum { HOPF_H_L1 = 0, HOPF_H_WL1 = 1, HOPF_H_L2 = 2, HOPF_H_ELL = 3, HOPF_H_LINF = 4 } hopf_h_kind;

/* Diagonal (ellipsoidal) initial data:
 *   J(x) = 1/2 <x - c, diag(Dj)^{-1} (x - c)> + gamma,  J*(v) = 1/2 <v, Dj v> + <c, v> - gamma
 * (P:209-263 with Dj_i = a_i^2; Table 4's J = 1/2<., D^{-1}.>).
 *   M, n      number of points, dimension (1 <= n <= 1024)
 *   X [M*n]   query points;  t [M] times (t >= 0)
 *   Dj [n]    diagonal of J's curvature inverse (> 0);  c [n] centre or NULL (= 0)
 *   gamma     additive constant of J
 *   h, w      Hamiltonian kind and weights w [n] (HOPF_H_WL1 / HOPF_H_ELL, else may be NULL)
 *   lambda    split Bregman penalty (> 0; the paper uses 1)
 *   max_iter  iteration cap (>= 1); tol squared-norm stopping threshold (>= 0, paper 1e-8)
 *   phi [M], grad [M*n], iters [M]   outputs                                               */
int hopf_eval_diag(int64_t M, int32_t n, const float *X, const float *t, const float *Dj,
                   const float *c, float gamma, hopf_h_kind h, const float *w, float lambda,
                   int32_t max_iter, float tol, float *phi, float *grad, int32_t *iters,
                   hopf_stream_t stream);

/* Union of K diagonal initial data (min-plus over initial data):
 *   J(x) = min_k [ 1/2 <x - c_k, diag(Dj_k)^{-1} (x - c_k)> + gamma_k ]
 *   phi = min_k phi_k, the lowest k wins ties (R19); grad = grad of the winner;
 *   each phi_k is solved centred at x - c_k with v^0 = d^0 = x - c_k (R5).
 *   Dj [K*n], C [K*n] (row k = set k), gamma [K]  (HOST-side copy not needed: device pointers)
 *   iters[i] = the winning set's status.
 *   Y [M*n] or NULL   closest (Hopf-Lax terminal) point y = x - t grad/||grad||
 *                     (P:1049-1051), y = c_k* if grad == 0 (R18); HOPF_H_L2 only.
 *   kstar [M] or NULL winning set index;  phi_k [M*K] or NULL every phi_k (an invalid point:
 *   NaN for every k, kstar -1).
 *   Constraints: 1 <= K <= 64, n <= 256.                                                   */
int hopf_eval_union(int64_t M, int32_t n, int32_t K, const float *X, const float *t,
                    const float *Dj, const float *C, const float *gamma, hopf_h_kind h,
                    const float *w, float lambda, int32_t max_iter, float tol, float *phi,
                    float *grad, int32_t *iters, float *Y, int32_t *kstar, float *phi_k,
                    hopf_stream_t stream);

/* H(p) = ||p||_A = sqrt(<p, A p>) with a full SPD A (NEXT-2; the ||y||_A column of
 * Tables 1-4) and the diagonal J of hopf_eval_diag.  A is given in spectral form,
 * A = Q diag(Lam) Q^T: Q [n*n] DEVICE row-major with the eigenvectors as columns (orthogonal),
 * Lam [n] DEVICE > 0.  The prox is u - tau Q pi_{E_Lam}(Q^T u / tau) (ellipsoid projection in the
 * eigenbasis, Newton on its multiplier, reading R27).  1 <= n <= 128.  Other arguments, outputs,
 * status codes and errors as hopf_eval_diag. */
int hopf_eval_diag_A(int64_t M, int32_t n, const float *X, const float *t, const float *Dj,
                     const float *c, float gamma, const float *Q, const float *Lam, float lambda,
                     int32_t max_iter, float tol, float *phi, float *grad, int32_t *iters,
                     hopf_stream_t stream);

/* Non-quadratic initial data (NEXT-3; Tables 2, 3 and 5):
 *   HOPF_J_L1SQ  : J(x) = 1/2 ||x||_1^2 + gamma    (J* = 1/2 ||.||_inf^2)
 *   HOPF_J_LINFSQ: J(x) = 1/2 ||x||_inf^2 + gamma  (J* = 1/2 ||.||_1^2)
 * (3.4a) is the prox of J* / lambda, found per iteration through the multiplier of
 * eq. optimality_beta_l1_2 (Moreau for 1/2||.||_inf^2, reading R29).
 *   h in {HOPF_H_L1, HOPF_H_WL1 (w [n] required), HOPF_H_L2, HOPF_H_LINF}; 1 <= n <= 512.
 *   t == 0: phi = J(x), grad = the minimal-norm subgradient of J (reading R30).
 * Other arguments, outputs, status codes and errors as hopf_eval_diag.  The minimiser grad may
 * be non-unique for these J (J* is not strictly convex); phi is unique. */
typedef enum { HOPF_J_L1SQ = 0, HOPF_J_LINFSQ = 1 } hopf_j_kind;
int hopf_eval_normsq(int64_t M, int32_t n, const float *X, const float *t, hopf_j_kind j,
                     float gamma, hopf_h_kind h, const float *w, float lambda, int32_t max_iter,
                     float tol, float *phi, float *grad, int32_t *iters, hopf_stream_t stream);

/* Maximum over a minimum of Hamiltonians (NEXT-4): for H = min_i H_i,
 *   phi(x,t) = max_i phi_i(x,t),  phi_i the solution with H_i and the same diagonal J,
 * the lowest i winning ties; grad = the winner's gradient, iters = its status.
 *   K (>= 1)       number of Hamiltonians
 *   h_kinds [K]    HOST array of hopf_h_kind;  a [K] HOST array of scales a_i > 0
 *   W [K*n]        DEVICE weights (row i used when h_kinds[i] is HOPF_H_WL1 / HOPF_H_ELL), else may be NULL
 *   H_i(p) = a_i H_{kind_i}(p; W_i); evaluated as the kind's solve at time a_i t (t a_i H = (a_i t) H)
 *   istar [M] or NULL   index of the winning Hamiltonian (-1 on invalid points)
 * Other arguments as hopf_eval_diag.  Launches K solves (each at time a_i t inside the kernel)
 * and K-1 combine steps (+ one istar initialisation) on `stream`; scratch for K > 1 (M (n + 2)
 * floats) is stream-ordered per call (see the concurrency convention above); results valid
 * after the stream syncs. */
int hopf_eval_maxh(int64_t M, int32_t n, const float *X, const float *t, const float *Dj,
                   const float *c, float gamma, int32_t K, const int32_t *h_kinds, const float *a,
                   const float *W, float lambda, int32_t max_iter, float tol, float *phi,
                   float *grad, int32_t *iters, int32_t *istar, hopf_stream_t stream);

/* Distance and closest point to a union of ellipsoids (NEXT-1):
 *   Omega = union_k {y : L_k(y) <= 0},  L_k(y) = 1/2 <y - c_k, diag(Dj_k)^{-1}(y - c_k)> + gamma_k
 *   (gamma_k < 0; gamma_k = -1/2 is the ellipsoid with semi-axes sqrt(Dj_k)).
 * psi(y,s) = min_k psi_k(y,s) solves the eikonal problem psi_t + ||grad psi|| = 0, psi(.,0) = L
 * (H = l2); each evaluation runs split Bregman for the K sets (as hopf_eval_union with t = s).
 * Newton in s on psi(y,s) = 0 (eq. Newton_zero): s_0 = 0 (psi(y,0) = L(y), R24),
 *   s_{l+1} = s_l + psi(y,s_l) / ||grad psi(y,s_l)||,
 * stopping when |s_{l+1} - s_l| <= stol max(1, s_l) or after max_newton evaluations (the
 * result is the last evaluated s, R26); a step leaving the bracket of the root is replaced by
 * bisection (R25).
 *   Y [M*n]      query points (device)
 *   Dj, C [K*n], gamma [K]   the sets (device)
 *   lambda, max_iter, tol    the inner split Bregman parameters (as hopf_eval_union)
 *   max_newton (>= 1), stol (>= 0)   the outer Newton parameters
 *   dist [M]     s = dist(y, Omega) (0 for y in Omega)
 *   proj [M*n]   pi_Omega(y) = y - s grad/||grad||; y itself for y in Omega
 *   psi [M]      psi(y, s) at the returned s (residual of the root)
 *   grad [M*n]   grad_x psi(y, s)
 *   kstar [M]    winning set;  newton [M] number of evaluations at s > 0 (0 for y in Omega,
 *                INT32_MIN for a non-finite point: all outputs NaN)
 * Constraints: 1 <= K <= 64, n <= 256.  Asynchronous on `stream`; errors as hopf_eval_union. */
int hopf_distance_union(int64_t M, int32_t n, int32_t K, const float *Y, const float *Dj,
                        const float *C, const float *gamma, float lambda, int32_t max_iter,
                        float tol, int32_t max_newton, float stol, float *dist, float *proj,
                        float *psi, float *grad, int32_t *kstar, int32_t *newton,
                        hopf_stream_t stream);


/* Full SPD initial data J(x) = 1/2 <x, A x> + gamma with A = Q diag(Lambda) Q^T (spectral
 * form as in P:1287-1290).  The plan owns device copies of
 *   M_lambda = (A^{-1} + lambda I)^{-1} = Q diag(Lambda/(1 + lambda Lambda)) Q^T
 * (the quadratic prox of (3.4a)) split into tensor-core operands, and of A^{-1}
 * (for phi).  Built on the host in fp64 from HOST arrays Q_host [n*n] (row-major, orthogonal)
 * and Lambda_host [n] (> 0).  Synchronous.                                                  */
typedef struct hopf_dense_plan hopf_dense_plan;
int hopf_dense_plan_create(int32_t n, const double *Q_host, const double *Lambda_host,
                           float lambda, hopf_dense_plan **out);
int hopf_dense_plan_destroy(hopf_dense_plan *plan);

/* Dense evaluation; arguments as hopf_eval_diag, lambda must equal the plan's.
 * n == 256 with H in {l1, wl1} runs the tensor-core kernel (tcgen05, fp16 hi/lo split of
 * M_lambda and of x + lambda (d - b), fp32 accumulation in TMEM); its points with t == 0,
 * invalid input or no convergence are re-solved by the FP32 kernel from a device-side list.
 * Other n (multiples of 32 up to 256) and H = l2 run the FP32 SIMT kernel.  The list is
 * per-call stream-ordered scratch, so one plan may serve concurrent calls on several streams
 * (the plan itself is read-only after creation).  HOPF_EINVAL if the current device is not the
 * device the plan was created on. */
int hopf_eval_dense(int64_t M, int32_t n, const float *X, const float *t,
                    const hopf_dense_plan *plan, float gamma, hopf_h_kind h, const float *w,
                    float lambda, int32_t max_iter, float tol, float *phi, float *grad,
                    int32_t *iters, hopf_stream_t stream);

/* End-to-end variant of hopf_eval_diag on HOST buffers (X_host, t_host in, phi_host,
 * grad_host, iters_host out; pinned memory strongly recommended).  Dj, c, w are DEVICE
 * pointers as above.  The call splits the points into chunks and pipelines
 * host->device copies, kernels and device->host copies on internal streams of the
 * current device; it returns after all results are in host memory (synchronous).
 * Ordering: the first chunk starts after all work enqueued earlier on the legacy default
 * stream of the current device (an event recorded there at entry; the legacy stream itself
 * waits for all blocking streams), so parameters written there (e.g. by PyTorch's default
 * stream) are visible; writes on the caller's non-blocking streams must be synchronised first.
 * Internal streams and buffers are pooled per device (one context per concurrent call).     */
int hopf_eval_diag_host(int64_t M, int32_t n, const float *X_host, const float *t_host,
                        const float *Dj, const float *c, float gamma, hopf_h_kind h,
                        const float *w, float lambda, int32_t max_iter, float tol,
                        float *phi_host, float *grad_host, int32_t *iters_host);

/* Instrumentation (benchmarks): while `counter` (a DEVICE pointer to one unsigned 64-bit
 * integer, or NULL to switch off) is set on this thread, hopf_eval_diag / hopf_eval_union /
 * hopf_distance_union atomically add the split Bregman iterations of every solve they run
 * (t > 0 solves; the union's K solves per point, every Newton evaluation) to *counter.  The
 * caller zeroes and reads it.  Not used by the dense path.  Returns HOPF_OK. */
int hopf_set_iteration_counter(unsigned long long *counter);

/* Number of kernel launches the most recent successful call made on this thread. */
int32_t hopf_last_launch_count(void);

/* Launch shape of the most recent diag/union kernel launch on this thread (threads per block,
 * blocks); returns hopf_last_launch_count().  Either pointer may be NULL. */
int32_t hopf_last_launch_config(int32_t *threads_per_block, int32_t *blocks);

/* Name of the main kernel the most recent successful call launched on this thread (static
 * string, "" if none), e.g. "hopf_diag_tm_kernel<l2>"; for benchmarks and profiles. */
const char *hopf_last_kernel(void);

/* Text of the most recent error on this thread ("" if none) and a static string for a code. */
const char *hopf_last_error(void);
const char *hopf_strerror(int code);

/* Library version (semantic, e.g. 200 = 0.2.0: adds hopf_distance_union, hopf_eval_maxh,
 * hopf_eval_normsq, hopf_eval_diag_A and the HOPF_H_ELL / HOPF_H_LINF kinds to 0.1.0). */
int32_t hopf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HOPF_H_ */
