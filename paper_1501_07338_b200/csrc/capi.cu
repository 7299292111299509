// capi.cu -- op-level C ABI (include/vcnn_cuda.h).  Host-side validation
// mirrors the reference constructors and checks so the same error classes
// fire before any launch; everything else is a thin call into kernels.cuh.
#include <string>

#include "kernels.cuh"

using namespace vcnn_b200;

namespace {

std::string dims(int a, int b) { return std::to_string(a) + "x" + std::to_string(b); }

int conv_desc(const vcnn_conv_geometry* g, int maps, ConvDesc& d) {
  if (!g) return fail(VCNN_EGEOMETRY, "null conv geometry");
  vcnn_conv_geometry chk;
  int s = vcnn_conv_geometry_init(&chk, g->in_h, g->in_w, g->channels, g->batch, g->kh, g->kw,
                                  g->stride);
  if (s) return s;
  if (maps < 1) return fail(VCNN_ESHAPE, "conv: output map count must be >= 1");
  d.B = g->batch;
  d.C = g->channels;
  d.H = g->in_h;
  d.W = g->in_w;
  d.K = maps;
  d.kh = g->kh;
  d.kw = g->kw;
  d.s = g->stride;
  d.OH = chk.out_h;
  d.OW = chk.out_w;
  return VCNN_OK;
}

int pool_desc(const vcnn_pool_geometry* g, PoolDesc& d) {
  if (!g) return fail(VCNN_EGEOMETRY, "null pool geometry");
  vcnn_pool_geometry chk;
  int s = vcnn_pool_geometry_init(&chk, g->in_h, g->in_w, g->channels, g->batch, g->ph, g->pw,
                                  g->stride, g->mode);
  if (s) return s;
  d.B = g->batch;
  d.C = g->channels;
  d.H = g->in_h;
  d.W = g->in_w;
  d.ph = g->ph;
  d.pw = g->pw;
  d.s = g->stride;
  d.mode = g->mode;
  d.OH = chk.out_h;
  d.OW = chk.out_w;
  return VCNN_OK;
}

int check_prec(int prec) {
  if (prec != VCNN_PREC_TF32 && prec != VCNN_PREC_3XTF32 && prec != VCNN_PREC_FP32)
    return fail(VCNN_ECONFIG, "unknown precision " + std::to_string(prec));
  return VCNN_OK;
}

int check_act(int act) {
  if (act < VCNN_ACT_IDENTITY || act > VCNN_ACT_TANH)
    return fail(VCNN_ECONFIG, "unknown activation " + std::to_string(act));
  return VCNN_OK;
}

// scratch buffer from the stream-ordered allocator, freed on scope exit
struct Scratch {
  void* p = nullptr;
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) {}
  int alloc(size_t bytes) {
    if (bytes == 0) return VCNN_OK;
    VCNN_CUDA_TRY(cudaMallocAsync(&p, bytes, st));
    return VCNN_OK;
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, st);
  }
};

#define TRY(expr)         \
  do {                    \
    int _s = (expr);      \
    if (_s) return _s;    \
  } while (0)

// stream-ordered scratch for the GEMM launchers (split-K partials, dP)
#define WORKSPACE(var, bytes_expr)                                   \
  Scratch var##_s(st);                                               \
  const size_t var##_b = (bytes_expr);                               \
  TRY(var##_s.alloc(var##_b));                                       \
  Workspace var{static_cast<float*>(var##_s.p), var##_b}

}  // namespace

extern "C" {

int vcnn_copy_h2d(void* dev, const void* host, size_t bytes) {
  TRY(require_device());
  VCNN_CUDA_TRY(cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice));
  return VCNN_OK;
}

int vcnn_abi_version(void) { return VCNN_ABI_VERSION; }
const char* vcnn_last_error(void) { return last_error(); }
int64_t vcnn_launch_count(void) { return g_launches.load(); }

int vcnn_device_info(int* sm, int* major, int* minor) {
  int dev = 0, n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(VCNN_ECUDA, "no CUDA device");
  cudaGetDevice(&dev);
  cudaDeviceProp p;
  VCNN_CUDA_TRY(cudaGetDeviceProperties(&p, dev));
  if (sm) *sm = p.multiProcessorCount;
  if (major) *major = p.major;
  if (minor) *minor = p.minor;
  return VCNN_OK;
}

// ConvGeometry (vectorize.hpp:19-29); Shape extents must be >= 1 (tensor.hpp:27-34)
int vcnn_conv_geometry_init(vcnn_conv_geometry* g, int in_h, int in_w, int channels, int batch,
                            int kh, int kw, int stride) {
  if (in_h < 1 || in_w < 1 || channels < 1 || batch < 1)
    return fail(VCNN_ESHAPE, "shape extent must be >= 1");
  if (kh < 1 || kw < 1) return fail(VCNN_EGEOMETRY, "kernel extents must be >= 1");
  if (stride < 1) return fail(VCNN_EGEOMETRY, "stride must be >= 1");
  if (kh > in_h || kw > in_w)
    return fail(VCNN_EGEOMETRY, "kernel " + dims(kh, kw) + " exceeds input " + dims(in_h, in_w));
  if (g) {
    g->in_h = in_h;
    g->in_w = in_w;
    g->channels = channels;
    g->batch = batch;
    g->kh = kh;
    g->kw = kw;
    g->stride = stride;
    g->out_h = (in_h - kh) / stride + 1;
    g->out_w = (in_w - kw) / stride + 1;
  }
  return VCNN_OK;
}

// PoolGeometry (vectorize.hpp:141-151)
int vcnn_pool_geometry_init(vcnn_pool_geometry* g, int in_h, int in_w, int channels, int batch,
                            int ph, int pw, int stride, int mode) {
  if (in_h < 1 || in_w < 1 || channels < 1 || batch < 1)
    return fail(VCNN_ESHAPE, "shape extent must be >= 1");
  if (ph < 1 || pw < 1) return fail(VCNN_EGEOMETRY, "pooling window extents must be >= 1");
  if (stride < 1) return fail(VCNN_EGEOMETRY, "pooling stride must be >= 1");
  if (ph > in_h || pw > in_w)
    return fail(VCNN_EGEOMETRY,
                "pooling window " + dims(ph, pw) + " exceeds input " + dims(in_h, in_w));
  if (mode != VCNN_POOL_MAX && mode != VCNN_POOL_AVG)
    return fail(VCNN_ECONFIG, "unknown pool mode");
  if (g) {
    g->in_h = in_h;
    g->in_w = in_w;
    g->channels = channels;
    g->batch = batch;
    g->ph = ph;
    g->pw = pw;
    g->stride = stride;
    g->mode = mode;
    g->out_h = (in_h - ph) / stride + 1;
    g->out_w = (in_w - pw) / stride + 1;
  }
  return VCNN_OK;
}

// ---------------------------------------------------------------- tensor.hpp
int vcnn_matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c,
                int precision, void* stream) {
  TRY(check_prec(precision));
  if (m < 0 || k < 0 || n < 0) return fail(VCNN_ESHAPE, "matrix extents must be non-negative");
  TRY(require_device());
  if (m == 0 || n == 0) return VCNN_OK;
  if (k == 0) {
    VCNN_CUDA_TRY(cudaMemsetAsync(c, 0, sizeof(float) * m * n, as_stream(stream)));
    return VCNN_OK;
  }
  cudaStream_t st = as_stream(stream);
  WORKSPACE(ws, matmul_workspace(m, k, n, precision));
  return launch_matmul(m, k, n, a, b, c, false, precision, ws, st);
}

int vcnn_matmul_transB(int64_t m, int64_t k, int64_t n, const float* a, const float* b,
                       float* c, int precision, void* stream) {
  TRY(check_prec(precision));
  if (m < 0 || k < 0 || n < 0) return fail(VCNN_ESHAPE, "matrix extents must be non-negative");
  TRY(require_device());
  if (m == 0 || n == 0) return VCNN_OK;
  if (k == 0) {
    VCNN_CUDA_TRY(cudaMemsetAsync(c, 0, sizeof(float) * m * n, as_stream(stream)));
    return VCNN_OK;
  }
  cudaStream_t st = as_stream(stream);
  WORKSPACE(ws, matmul_workspace(m, k, n, precision));
  return launch_matmul(m, k, n, a, b, c, true, precision, ws, st);
}

// the general GEMM of the C ABI: op(A) [m][k], op(B) [k][n],
// C [m][n] with leading dimensions, + bias[n] + activation
int vcnn_gemm(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, const float* a,
              int64_t lda, const float* b, int64_t ldb, float* c, int64_t ldc, const float* bias,
              int act, int precision, void* stream) {
  TRY(check_prec(precision));
  if (m < 0 || k < 0 || n < 0) return fail(VCNN_ESHAPE, "matrix extents must be non-negative");
  if (act < VCNN_ACT_IDENTITY || act > VCNN_ACT_TANH) return fail(VCNN_ECONFIG, "unknown activation");
  if (ldc < n || lda < (trans_a ? m : k) || ldb < (trans_b ? k : n))
    return fail(VCNN_ESHAPE, "gemm: leading dimension smaller than the row length");
  TRY(require_device());
  if (m == 0 || n == 0) return VCNN_OK;
  const int64_t as_m = trans_a ? 1 : lda, as_k = trans_a ? lda : 1;
  const int64_t bs_k = trans_b ? 1 : ldb, bs_n = trans_b ? ldb : 1;
  cudaStream_t st = as_stream(stream);
  if (precision == VCNN_PREC_FP32 || k == 0)
    return simt::gemm(m, n, k, a, as_m, as_k, b, bs_k, bs_n, c, ldc, bias, act, st);
  WORKSPACE(ws, tc::matmul_workspace(m, k, n));
  return tc::gemm(m, n, k, a, as_m, as_k, b, bs_k, bs_n, c, ldc, bias, act,
                  precision == VCNN_PREC_3XTF32, ws, st);
}

int vcnn_accumulate_by_index(const float* values, int64_t source_len, const int64_t* source,
                             const int64_t* target, int64_t pairs, int64_t target_len,
                             int reducer, float* out, void* stream) {
  if (source_len < 0 || target_len < 1 || pairs < 0)
    return fail(VCNN_EBOUNDS, "index map: invalid domain lengths");
  if (reducer < VCNN_REDUCE_SUM || reducer > VCNN_REDUCE_MEAN)
    return fail(VCNN_ECONFIG, "unknown reducer");
  TRY(require_device());
  return launch_accumulate(values, source, target, pairs, target_len, reducer, out, nullptr,
                           as_stream(stream));
}

int vcnn_accumulate_max_arg(const float* values, int64_t source_len, const int64_t* source,
                            const int64_t* target, int64_t pairs, int64_t target_len, float* out,
                            int64_t* arg, void* stream) {
  if (source_len < 0 || target_len < 1 || pairs < 0)
    return fail(VCNN_EBOUNDS, "index map: invalid domain lengths");
  if (!arg) return fail(VCNN_EBOUNDS, "accumulate_max_arg: null arg");
  TRY(require_device());
  return launch_accumulate(values, source, target, pairs, target_len, VCNN_REDUCE_MAX, out, arg,
                           as_stream(stream));
}

// ------------------------------------------------------------- vectorize.hpp
int vcnn_im2col(const vcnn_conv_geometry* g, const float* x, float* patch, void* stream) {
  ConvDesc d;
  TRY(conv_desc(g, 1, d));
  TRY(require_device());
  return launch_im2col(d, x, patch, as_stream(stream));
}

int vcnn_col2im(const vcnn_conv_geometry* g, const float* dpatch, float* dx, void* stream) {
  ConvDesc d;
  TRY(conv_desc(g, 1, d));
  TRY(require_device());
  return launch_col2im(d, dpatch, dx, as_stream(stream));
}

int vcnn_col2im_map(const vcnn_conv_geometry* g, int64_t* source, int64_t* target, void* stream) {
  ConvDesc d;
  TRY(conv_desc(g, 1, d));
  TRY(require_device());
  return launch_col2im_map(d, source, target, as_stream(stream));
}

int vcnn_pool_map(const vcnn_pool_geometry* g, int64_t* source, int64_t* target, void* stream) {
  PoolDesc d;
  TRY(pool_desc(g, d));
  TRY(require_device());
  return launch_pool_map(d, source, target, as_stream(stream));
}

int vcnn_pool_forward(const vcnn_pool_geometry* g, const float* x, float* y, int64_t* arg,
                      void* stream) {
  PoolDesc d;
  TRY(pool_desc(g, d));
  TRY(require_device());
  return launch_pool_fwd<int64_t>(d, x, nullptr, VCNN_ACT_IDENTITY, y, arg, as_stream(stream));
}

int vcnn_pool_backward(const vcnn_pool_geometry* g, int bwd_mode, const float* dy,
                       const int64_t* arg, float* dx, void* stream) {
  PoolDesc d;
  TRY(pool_desc(g, d));
  if (bwd_mode != VCNN_POOLBWD_EXACT && bwd_mode != VCNN_POOLBWD_PAPER_NN)
    return fail(VCNN_ECONFIG, "unknown pool backward mode");
  if (bwd_mode == VCNN_POOLBWD_EXACT && d.mode == VCNN_POOL_MAX && !arg)
    return fail(VCNN_EGEOMETRY, "pool_backward: arg index does not match pooled extents");
  TRY(require_device());
  return launch_pool_bwd<int64_t>(d, bwd_mode, dy, arg, dx, nullptr, VCNN_ACT_IDENTITY,
                                  as_stream(stream));
}

// ---------------------------------------------------------------- layers.hpp
int vcnn_activation_forward(int64_t n, int act, const float* x, float* y, void* stream) {
  TRY(check_act(act));
  if (n < 0) return fail(VCNN_ESHAPE, "negative length");
  TRY(require_device());
  if (n == 0) return VCNN_OK;
  return launch_act_fwd(n, act, x, y, as_stream(stream));
}

int vcnn_activation_backward(int64_t n, int act, const float* y, float* grad, void* stream) {
  TRY(check_act(act));
  if (n < 0) return fail(VCNN_ESHAPE, "negative length");
  TRY(require_device());
  if (n == 0 || act == VCNN_ACT_IDENTITY) return VCNN_OK;
  return launch_act_bwd(n, act, y, grad, grad, as_stream(stream));
}

int vcnn_conv_forward(const vcnn_conv_geometry* g, int maps, const float* x, const float* w,
                      const float* bias, int act, int precision, float* y, void* stream) {
  ConvDesc d;
  TRY(conv_desc(g, maps, d));
  TRY(check_prec(precision));
  TRY(check_act(act));
  TRY(require_device());
  cudaStream_t st = as_stream(stream);
  WORKSPACE(ws, conv_workspace(d, precision));
  // TF32: the direct (shifted-view) kernel with prepacked weights, else the
  // slab kernel with a tf32-rounded weight copy
  Scratch wp(st);
  const float* wf = nullptr;
  if (precision == VCNN_PREC_TF32 && direct::fwd_ok(d, 0)) {
    TRY(wp.alloc(sizeof(float) * direct::pack_floats(d, 0)));
    float* pk = static_cast<float*>(wp.p);
    TRY(direct::pack_weights(d, 0, w, pk, st));
    return direct::conv_fwd(d, x, pk, bias, act, y, PoolFuse{}, st);
  }
  if (precision == VCNN_PREC_TF32 && tc::slab_fwd_ok(d, 0)) {
    TRY(wp.alloc(sizeof(float) * tc::prep_floats_f(d)));
    wf = static_cast<float*>(wp.p);
    TRY(tc::prep_weights(d, w, static_cast<float*>(wp.p), nullptr, st));
  }
  return launch_conv_fwd(d, x, w, bias, act, y, precision, ws, st, wf);
}

int vcnn_conv_backward(const vcnn_conv_geometry* g, int maps, const float* x, const float* w,
                       const float* y, const float* dy, int act, int precision, float* dw,
                       float* db, float* dx, void* stream) {
  ConvDesc d;
  TRY(conv_desc(g, maps, d));
  TRY(check_prec(precision));
  TRY(check_act(act));
  TRY(require_device());
  cudaStream_t st = as_stream(stream);
  // gpre = dy * act'(y)  (conv_backward, layers.hpp:186-187)
  Scratch gp(st);
  const float* gpre = dy;
  if (act != VCNN_ACT_IDENTITY) {
    TRY(gp.alloc(sizeof(float) * d.out_size()));
    TRY(launch_act_bwd(d.out_size(), act, y, dy, static_cast<float*>(gp.p), st));
    gpre = static_cast<float*>(gp.p);
  }
  WORKSPACE(ws, conv_workspace(d, precision));
  TRY(launch_conv_wgrad(d, x, gpre, dw, db, precision, ws, st));
  if (!dx) return VCNN_OK;
  // TF32: tf32-rounded transposed weights for the slab dgrad
  Scratch wp(st);
  const float* wt = nullptr;
  if (precision == VCNN_PREC_TF32 && direct::dgrad_ok(d)) {
    TRY(wp.alloc(sizeof(float) * direct::pack_floats(d, 1)));
    float* pk = static_cast<float*>(wp.p);
    TRY(direct::pack_weights(d, 1, w, pk, st));
    GradSrc gs;
    gs.g = gpre;
    return direct::conv_dgrad(d, gs, pk, dx, nullptr, VCNN_ACT_IDENTITY, st);
  }
  if (precision == VCNN_PREC_TF32 && tc::slab_dgrad_ok(d)) {
    const size_t nf = tc::prep_floats_f(d);
    TRY(wp.alloc(sizeof(float) * (nf + tc::prep_floats_t(d))));
    float* wf = static_cast<float*>(wp.p);
    wt = wf + nf;
    TRY(tc::prep_weights(d, w, wf, wf + nf, st));
  }
  TRY(launch_conv_dgrad(d, gpre, w, dx, nullptr, VCNN_ACT_IDENTITY, precision, ws, st, wt));
  return VCNN_OK;
}

int vcnn_full_forward(int batch, int in_units, int out_units, const float* x, const float* w,
                      const float* bias, int act, int precision, float* y, void* stream) {
  if (batch < 1 || in_units < 1 || out_units < 1)
    return fail(VCNN_ESHAPE, "full layer: extents must be >= 1");
  TRY(check_prec(precision));
  TRY(check_act(act));
  TRY(require_device());
  cudaStream_t st = as_stream(stream);
  WORKSPACE(ws, full_workspace(batch, in_units, out_units, precision));
  return launch_full_fwd(batch, in_units, out_units, x, w, bias, act, y, precision, ws, st);
}

int vcnn_full_backward(int batch, int in_units, int out_units, const float* x, const float* w,
                       const float* y, const float* dy, int act, int precision, float* dw,
                       float* db, float* dx, void* stream) {
  if (batch < 1 || in_units < 1 || out_units < 1)
    return fail(VCNN_ESHAPE, "full layer: extents must be >= 1");
  TRY(check_prec(precision));
  TRY(check_act(act));
  TRY(require_device());
  cudaStream_t st = as_stream(stream);
  Scratch gp(st);
  const float* gpre = dy;
  const int64_t n = (int64_t)batch * out_units;
  if (act != VCNN_ACT_IDENTITY) {
    TRY(gp.alloc(sizeof(float) * n));
    TRY(launch_act_bwd(n, act, y, dy, static_cast<float*>(gp.p), st));
    gpre = static_cast<float*>(gp.p);
  }
  WORKSPACE(ws, full_workspace(batch, in_units, out_units, precision));
  TRY(launch_full_wgrad(batch, in_units, out_units, x, gpre, dw, db, precision, ws, st));
  if (dx)
    TRY(launch_full_dgrad(batch, in_units, out_units, gpre, w, dx, nullptr, VCNN_ACT_IDENTITY,
                          precision, ws, st));
  return VCNN_OK;
}

int vcnn_pool_layer_forward(const vcnn_pool_geometry* g, const float* x, const float* bias,
                            int act, float* y, int64_t* arg, void* stream) {
  PoolDesc d;
  TRY(pool_desc(g, d));
  TRY(check_act(act));
  TRY(require_device());
  return launch_pool_fwd<int64_t>(d, x, bias, act, y, arg, as_stream(stream));
}

int vcnn_pool_layer_backward(const vcnn_pool_geometry* g, int bwd_mode, const float* y, int act,
                             const float* dy, const int64_t* arg, float* dx, float* dbias,
                             void* stream) {
  PoolDesc d;
  TRY(pool_desc(g, d));
  TRY(check_act(act));
  if (bwd_mode != VCNN_POOLBWD_EXACT && bwd_mode != VCNN_POOLBWD_PAPER_NN)
    return fail(VCNN_ECONFIG, "unknown pool backward mode");
  if (bwd_mode == VCNN_POOLBWD_EXACT && d.mode == VCNN_POOL_MAX && !arg)
    return fail(VCNN_EGEOMETRY, "pool_backward: arg index does not match pooled extents");
  TRY(require_device());
  cudaStream_t st = as_stream(stream);
  Scratch gp(st);
  const float* gpre = dy;
  if (act != VCNN_ACT_IDENTITY) {
    TRY(gp.alloc(sizeof(float) * d.out_size()));
    TRY(launch_act_bwd(d.out_size(), act, y, dy, static_cast<float*>(gp.p), st));
    gpre = static_cast<float*>(gp.p);
  }
  if (dbias) TRY(launch_pool_bias_grad(d, gpre, dbias, st));
  return launch_pool_bwd<int64_t>(d, bwd_mode, gpre, arg, dx, nullptr, VCNN_ACT_IDENTITY, st);
}

static int loss_common(int kind, int batch, int units, const float* pred, const int* cls,
                       const float* values, float* loss, float* grad, void* stream) {
  if (kind != VCNN_LOSS_SOFTMAX_CE && kind != VCNN_LOSS_MSE)
    return fail(VCNN_ECONFIG, "unknown loss kind");
  if (batch < 1 || units < 1) return fail(VCNN_ESHAPE, "loss: extents must be >= 1");
  if (kind == VCNN_LOSS_SOFTMAX_CE && !cls)
    return fail(VCNN_ESHAPE, "loss: class targets required for softmax_ce");
  if (kind == VCNN_LOSS_MSE && !values)
    return fail(VCNN_ESHAPE, "loss: value targets required for mse");
  TRY(require_device());
  cudaStream_t st = as_stream(stream);
  int* err = nullptr;
  if (kind == VCNN_LOSS_SOFTMAX_CE) {
    VCNN_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&err), sizeof(int), st));
    VCNN_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int), st));
  }
  int s = launch_loss(kind, batch, units, pred, cls, values, loss, grad, VCNN_ACT_IDENTITY, err,
                      st);
  if (err) {
    int h = 0;
    cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(err, st);
    VCNN_CUDA_TRY(cudaStreamSynchronize(st));
    if (!s && h) s = fail(VCNN_EBOUNDS, "loss: class index out of range [0," +
                                           std::to_string(units) + ")");
  }
  return s;
}

int vcnn_loss_forward(int kind, int batch, int units, const float* pred, const int* cls,
                      const float* values, float* loss, void* stream) {
  return loss_common(kind, batch, units, pred, cls, values, loss, nullptr, stream);
}

int vcnn_loss_backward(int kind, int batch, int units, const float* pred, const int* cls,
                       const float* values, float* grad, void* stream) {
  return loss_common(kind, batch, units, pred, cls, values, nullptr, grad, stream);
}

int vcnn_loss_fused(int kind, int batch, int units, const float* pred, const int* cls,
                    const float* values, float* loss, float* grad, void* stream) {
  return loss_common(kind, batch, units, pred, cls, values, loss, grad, stream);
}

// --------------------------------------------------------------- network.hpp
int vcnn_sgd_step(int64_t n, float* w, float* v, const float* g, float lr, float mom,
                  float grad_scale, void* stream) {
  if (!(lr > 0)) return fail(VCNN_ECONFIG, "learning rate must be positive");
  if (mom < 0 || mom >= 1) return fail(VCNN_ECONFIG, "momentum must be in [0,1)");
  if (n < 0) return fail(VCNN_ESHAPE, "negative length");
  TRY(require_device());
  if (n == 0) return VCNN_OK;
  return launch_sgd(n, w, v, g, lr, mom, grad_scale, as_stream(stream));
}

}  // extern "C"
