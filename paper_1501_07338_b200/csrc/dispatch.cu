// dispatch.cu -- error plumbing, device checks and the precision dispatch of
// the GEMM-shaped launchers (tcgen05 for TF32 / 3xTF32, SIMT for FP32).
#include <mutex>
#include <string>

#include "kernels.cuh"

namespace vcnn_b200 {

namespace {
thread_local std::string t_err;
int g_sm_count = -1;
int g_dev_status = -1;
std::mutex g_dev_mu;
}  // namespace

std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { t_err = msg; }
const char* last_error() { return t_err.c_str(); }

int fail(int status, const std::string& msg) {
  t_err = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  t_err = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return VCNN_ECUDA;
}

int require_device() {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (g_dev_status >= 0) {
    if (g_dev_status != VCNN_OK) t_err = "no usable sm_100 CUDA device";
    return g_dev_status;
  }
  int dev = 0, n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    g_dev_status = VCNN_ECUDA;
    t_err = std::string("no CUDA device: ") + cudaGetErrorString(e);
    return g_dev_status;
  }
  cudaGetDevice(&dev);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.major != 10) {
    g_dev_status = VCNN_ECUDA;
    t_err = "libvcnn_cuda is built for sm_100a (B200); current device is not compute 10.x";
    return g_dev_status;
  }
  g_sm_count = prop.multiProcessorCount;
  g_dev_status = VCNN_OK;
  return g_dev_status;
}

int sm_count() {
  if (g_sm_count < 0) require_device();
  return g_sm_count > 0 ? g_sm_count : 148;
}

size_t conv_workspace(const ConvDesc& d, int prec) {
  return prec == VCNN_PREC_FP32 ? 0 : tc::conv_workspace(d);
}

size_t full_workspace(int B, int in, int out, int prec) {
  return prec == VCNN_PREC_FP32 ? 0 : tc::full_workspace(B, in, out);
}

size_t matmul_workspace(int64_t m, int64_t k, int64_t n, int prec) {
  return prec == VCNN_PREC_FP32 ? 0 : tc::matmul_workspace(m, k, n);
}

int launch_conv_fwd(const ConvDesc& d, const float* x, const float* w, const float* b, int act,
                    float* y, int prec, const Workspace& ws, cudaStream_t st, const float* wf) {
  if (prec == VCNN_PREC_FP32) return simt::conv_fwd(d, x, w, b, act, y, st);
  // TF32 stride-1 convs whose input window fits shared memory: slab kernel
  if (prec == VCNN_PREC_TF32 && wf && tc::slab_fwd_ok(d, 0))
    return tc::slab_conv_fwd(d, x, wf, b, act, y, PoolFuse{}, st);
  return tc::conv_fwd(d, x, w, b, act, y, prec == VCNN_PREC_3XTF32, ws, st);
}

int launch_conv_wgrad(const ConvDesc& d, const float* x, const float* gpre, float* dw,
                      float* db, int prec, const Workspace& ws, cudaStream_t st) {
  if (prec == VCNN_PREC_FP32) return simt::conv_wgrad(d, x, gpre, dw, db, st);
  if (prec == VCNN_PREC_TF32 && tc::slab_wgrad_ok(d)) {
    GradSrc gs;
    gs.g = gpre;
    return tc::slab_conv_wgrad(d, x, gs, dw, db, ws, st);
  }
  return tc::conv_wgrad(d, x, gpre, dw, db, prec == VCNN_PREC_3XTF32, ws, st);
}

int launch_conv_dgrad(const ConvDesc& d, const float* gpre, const float* w, float* dx,
                      const float* yprev, int act_prev, int prec, const Workspace& ws,
                      cudaStream_t st, const float* wt) {
  if (prec == VCNN_PREC_FP32) return simt::conv_dgrad(d, gpre, w, dx, yprev, act_prev, st);
  if (prec == VCNN_PREC_TF32 && wt && tc::slab_dgrad_ok(d)) {
    GradSrc gs;
    gs.g = gpre;
    return tc::slab_conv_dgrad(d, gs, wt, dx, yprev, act_prev, st);
  }
  return tc::conv_dgrad(d, gpre, w, dx, yprev, act_prev, prec == VCNN_PREC_3XTF32, ws, st);
}

// GEMMs below this many MACs run on the SIMT path in every precision mode:
// a 128x10x64 FC layer is ~80K MACs -- far below one tcgen05 tile's worth of
// work, where a tensor-core launch only adds TMEM / barrier setup latency.
constexpr int64_t kTinyGemmMacs = 1 << 20;
inline bool tiny(int64_t m, int64_t n, int64_t k) { return m * n * k < kTinyGemmMacs; }

int launch_full_fwd(int B, int in, int out, const float* x, const float* w, const float* b,
                    int act, float* y, int prec, const Workspace& ws, cudaStream_t st) {
  if (prec == VCNN_PREC_FP32 || tiny(B, out, in)) {
    if (simt::full_fwd_warp_ok(B, in, out, x, w))
      return simt::full_fwd_mid(B, in, out, x, w, b, act, y, st);
    return simt::full_fwd(B, in, out, x, w, b, act, y, st);
  }
  if (simt::full_fwd_warp_ok(B, in, out, x, w))  // exact fp32, no split-K reduce
    return simt::full_fwd_mid(B, in, out, x, w, b, act, y, st);
  return tc::full_fwd(B, in, out, x, w, b, act, y, prec == VCNN_PREC_3XTF32, ws, st);
}

int launch_full_wgrad(int B, int in, int out, const float* x, const float* gpre, float* dw,
                      float* db, int prec, const Workspace& ws, cudaStream_t st) {
  if (prec == VCNN_PREC_FP32 || tiny(out, in, B))
    return simt::full_wgrad(B, in, out, x, gpre, dw, db, st);
  return tc::full_wgrad(B, in, out, x, gpre, dw, db, prec == VCNN_PREC_3XTF32, ws, st);
}

int launch_full_dgrad(int B, int in, int out, const float* gpre, const float* w, float* dx,
                      const float* yprev, int act_prev, int prec, const Workspace& ws,
                      cudaStream_t st) {
  if (prec == VCNN_PREC_FP32 || tiny(B, in, out))
    return simt::full_dgrad(B, in, out, gpre, w, dx, yprev, act_prev, st);
  return tc::full_dgrad(B, in, out, gpre, w, dx, yprev, act_prev, prec == VCNN_PREC_3XTF32, ws,
                        st);
}

int launch_matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c,
                  bool transB, int prec, const Workspace& ws, cudaStream_t st) {
  if (prec == VCNN_PREC_FP32) return simt::matmul(m, k, n, a, b, c, transB, st);
  return tc::matmul(m, k, n, a, b, c, transB, prec == VCNN_PREC_3XTF32, ws, st);
}

}  // namespace vcnn_b200
