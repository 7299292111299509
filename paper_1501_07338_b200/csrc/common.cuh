// common.cuh -- shared helpers for the sm_100a VCNN kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>

#include "vcnn_cuda.h"

namespace vcnn_b200 {

// ---- error plumbing (thread-local message, status codes of vcnn_cuda.h) ----
void set_error(const std::string& msg);
const char* last_error();
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
extern std::atomic<int64_t> g_launches;

#define VCNN_CUDA_TRY(expr)                                          \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) return ::vcnn_b200::cuda_fail(_e, #expr); \
  } while (0)

// after a kernel launch: count it and surface launch errors
#define VCNN_LAUNCHED()                                                   \
  do {                                                                    \
    ::vcnn_b200::g_launches.fetch_add(1, std::memory_order_relaxed);      \
    cudaError_t _e = cudaGetLastError();                                  \
    if (_e != cudaSuccess) return ::vcnn_b200::cuda_fail(_e, "launch");   \
  } while (0)

// ---- programmatic dependent launch (PDL) ------------------------------------
// Every kernel is launched with programmatic stream serialisation: it lets
// its dependents launch at once (launch_dependents at entry) and waits for
// its predecessor's memory (griddepcontrol.wait) only after its own
// data-independent prologue, so launch latency and setup (barrier init, TMEM
// allocation) overlap the previous kernel's tail -- inside CUDA graphs too.
// Without a programmatic predecessor the wait returns at once.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#define PDL_ENTRY()             \
  do {                          \
    pdl_launch_dependents();    \
    pdl_wait();                 \
  } while (0)

// programmatic launch on/off (per host thread): the per-op CUDA-event
// breakdown turns it off so every op is timed alone, not overlapped with
// (or starved by) its early-launched successors
inline bool& pdl_enabled() {
  thread_local bool on = true;
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// fails with VCNN_ECUDA unless an sm_100-class device is current
int require_device();
int sm_count();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- activations (layers.hpp:25-48): forward, and derivative from OUTPUT ----
__device__ __forceinline__ float act_fwd(int act, float x) {
  switch (act) {
    case VCNN_ACT_RELU: return x > 0.f ? x : 0.f;  // NaN -> 0 like x>0?x:0
    case VCNN_ACT_SIGMOID: return 1.f / (1.f + expf(-x));
    case VCNN_ACT_TANH: return tanhf(x);
    default: return x;
  }
}

__device__ __forceinline__ float act_grad_from_out(int act, float y) {
  switch (act) {
    case VCNN_ACT_RELU: return y > 0.f ? 1.f : 0.f;  // relu'(0) = 0
    case VCNN_ACT_SIGMOID: return y * (1.f - y);
    case VCNN_ACT_TANH: return 1.f - y * y;
    default: return 1.f;
  }
}

// ceil-div
__host__ __device__ __forceinline__ int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace vcnn_b200
