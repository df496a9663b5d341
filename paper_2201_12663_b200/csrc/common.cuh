// common.cuh - shared device/host helpers for librhosvd (sm_100a, FP64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/rhosvd.h"

namespace rhosvd {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);

#define RH_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t e__ = (expr);                                                      \
    if (e__ != cudaSuccess)                                                        \
      return ::rhosvd::fail(RHOSVD_ECUDA, std::string(#expr " -> ") +              \
                                              cudaGetErrorString(e__) + " @" +     \
                                              __FILE__ ":" + std::to_string(__LINE__)); \
  } while (0)

#define RH_CHECK(expr)                        \
  do {                                        \
    int s__ = (expr);                         \
    if (s__ != RHOSVD_OK) return s__;         \
  } while (0)

#define RH_LAUNCH_CHECK() RH_CUDA(cudaGetLastError())

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t cdiv(int64_t x, int64_t m) { return (x + m - 1) / m; }

int num_sms();

// One CUDA device per process: the workspace, the output caches, the cached SM count and
// the per-kernel shared-memory attributes are process-wide.  The first library call pins
// the current device; a later call on another device fails with EINVAL (instead of
// reusing the first device's buffers).
int device_guard();

// Small device -> host readbacks (ranks, Ritz values, flags) go through pinned memory: a
// cudaMemcpyAsync into pageable memory is staged by the driver and can queue behind the
// large pinned copies already in flight (rhosvd_c2t_host's H2D of the side matrices),
// which stalled every host decision of the eigensolvers until the whole input had landed.
// d2h_wait copies `bytes` from device `src` to host `dst` through this thread's pinned
// buffer and waits for stream `st`.
int d2h_wait(void* dst, const void* src, size_t bytes, cudaStream_t st);
// host -> device counterpart (through a pinned staging block; waits for `st`)
int h2d_wait(void* dst, const void* src, size_t bytes, cudaStream_t st);

// count of kernels launched by the library (per-thread; reset by rhosvd_c2t)
extern thread_local int g_launches;
// cap on cooperative grids launched from this thread (0 = none): the three concurrent
// per-mode solves share the GPU, so each caps its grid-synchronised kernels at a third of
// the SMs by default (rhosvd.cu CapGuard; RHOSVD_COOP_MODE_CTAS / RHOSVD_COOP_MODE_CAP).
// History: a full-GPU cooperative grid blocks the other modes' kernels for its whole
// duration (cfg 4 eigensolve: no cap 151 ms, 1 CTA/SM 138-142 ms, a third of the SMs 126).
extern thread_local int g_coop_cap;
inline void count_launch(int k = 1) { g_launches += k; }

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  // D = A(8x4, row) * B(4x8, col) + D ; the only FP64 tensor instruction on sm_100a
  // (lowers to SASS DMMA.8x8x4).  Fragments: a = A[lane/4][lane%4],
  // b = B[lane%4][lane/4], {d0,d1} = D[lane/4][2*(lane%4) + {0,1}].
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy global->shared; src_bytes in {0, 8, 16} (rest zero-filled)
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rhosvd
