// common.cuh — host-side helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <string>

namespace hopf {
extern thread_local std::string g_last_error;
extern thread_local int32_t g_launches;
extern thread_local const char *g_last_kernel;
int set_error(int code, const char *fmt, ...);
int check_launch(const char *what);
int num_sms();
// Stream-ordered scratch (per call): allocated from a library-owned memory pool of the current
// device (release threshold = unlimited, so after warm-up an allocation is a pool hit with no
// host synchronisation) and freed on the same stream.  Calls on different streams therefore
// never share scratch; the pool's event tracking orders reuse across streams.
int scratch_alloc(void **ptr, size_t bytes, cudaStream_t stream);
void scratch_free(void *ptr, cudaStream_t stream);
// Dynamic point claims pay when each resident group (or warp batch) processes many points; for
// short launches (about 3 points per group: the paper-protocol lines at n <= 16) the counter's
// memset and the claims cost more than the balance gains (p4_id_l1 0.026 -> 0.039 ms), and the
// kernels keep the static stride.  *ctr = a zeroed stream-ordered counter (free it with
// scratch_free after the launch) or null; returns HOPF_OK or the allocation error.
// HOPF_CLAIMS=1 / 0 forces the counter on / off (tests, A/B runs).
int claim_counter(int64_t M, int64_t resident, cudaStream_t stream, unsigned long long **ctr);
}  // namespace hopf
