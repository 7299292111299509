/*
 * vcnn_oracle.h -- CPU restatement of the reference VCNN Imp-6 training path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 kernels.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  The product path (paper_1501_07338_b200,
 * libvcnn_cuda.so) never links, loads or calls anything under oracle/.
 *
 * Every function restates one reference routine in plain C, double precision,
 * with the same element order and summation order; the comment on each names
 * the reference file:line (paths relative to /root/reference/proj).
 *
 * Pinning: tests/test_oracle_golden.py checks this oracle against the
 * known-answer vectors of the reference's own doctest suites
 * (tests/{tensor,vectorize,layers,network}_test.cpp) and against the
 * reference itself, compiled from its sources into oracle/_ref by
 * oracle/Makefile (fixtures generated from it live in tests/golden/).
 */
#ifndef VCNN_ORACLE_H
#define VCNN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: identical numbering to include/vcnn_cuda.h */
enum { ORC_OK = 0, ORC_ESHAPE = 1, ORC_EGEOMETRY = 2, ORC_EBOUNDS = 3, ORC_ECONFIG = 6 };

/* Activation (layers.hpp:13), PoolMode (vectorize.hpp:127),
 * PoolBackwardMode (vectorize.hpp:217), LossKind (layers.hpp:375) */
enum { ORC_ACT_IDENTITY = 0, ORC_ACT_RELU = 1, ORC_ACT_SIGMOID = 2, ORC_ACT_TANH = 3 };
enum { ORC_POOL_MAX = 0, ORC_POOL_AVG = 1 };
enum { ORC_POOLBWD_EXACT = 0, ORC_POOLBWD_PAPER_NN = 1 };
enum { ORC_LOSS_SOFTMAX_CE = 0, ORC_LOSS_MSE = 1 };
enum { ORC_LAYER_CONV = 0, ORC_LAYER_POOL = 1, ORC_LAYER_FULL = 2 };

/* LayerSpec = variant<ConvSpec,PoolSpec,FullSpec> (network.hpp:12-32).
 * Same memory layout as vcnn_layer_spec in include/vcnn_cuda.h. */
typedef struct {
  int kind;      /* ORC_LAYER_* */
  int units;     /* conv maps / full units (unused for pool) */
  int kh, kw;    /* conv kernel or pool window */
  int stride;
  int pool_mode; /* ORC_POOL_* */
  int pool_bias; /* pool bias flag (PoolSpec::bias) */
  int act;       /* ORC_ACT_* */
} orc_layer;

/* NetworkSpec (network.hpp:37-73) */
typedef struct {
  int in_h, in_w, in_c;
  int nlayers;
  const orc_layer* layers;
  int loss;
  uint64_t seed;
} orc_net;

/* ---- Rng (common.hpp:51-96): mt19937_64 + portable extraction ---------- */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int have_spare;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_uniform_range(orc_rng* r, double lo, double hi);
int orc_rng_uniform_int(orc_rng* r, int n);
void orc_rng_fill_uniform(orc_rng* r, double* out, int64_t n, double lo, double hi);

/* ---- L1 tensor primitives (tensor.hpp) ---------------------------------- */
void orc_matmul(int64_t m, int64_t k, int64_t n, const double* a, const double* b, double* c);
void orc_matmul_transB(int64_t m, int64_t k, int64_t n, const double* a, const double* b,
                       double* c);

/* ---- L2 vectorize ops (vectorize.hpp) ------------------------------------ */
int orc_conv_geometry(int h, int w, int c, int n, int kh, int kw, int stride, int* out_h,
                      int* out_w);
int orc_pool_geometry(int h, int w, int c, int n, int ph, int pw, int stride, int* out_h,
                      int* out_w);
int orc_im2col(int B, int C, int H, int W, int kh, int kw, int s, const double* x, double* P);
int orc_col2im_map(int B, int C, int H, int W, int kh, int kw, int s, int64_t* src,
                   int64_t* tgt);
int orc_col2im(int B, int C, int H, int W, int kh, int kw, int s, const double* dP, double* dX);
int orc_pool_map(int B, int C, int H, int W, int ph, int pw, int s, int64_t* src, int64_t* tgt);
int orc_pool_forward(int B, int C, int H, int W, int ph, int pw, int s, int mode,
                     const double* x, double* y, int64_t* arg);
int orc_pool_backward(int B, int C, int H, int W, int ph, int pw, int s, int mode, int bwd_mode,
                      const double* dy, const int64_t* arg, double* dx);

/* ---- L3 layers (layers.hpp) ---------------------------------------------- */
double orc_activate(int act, double x);
double orc_activation_grad_from_output(int act, double y);
int orc_conv_forward(int B, int C, int H, int W, int K, int kh, int kw, int s, int act,
                     const double* x, const double* w, const double* b, double* y);
int orc_conv_backward(int B, int C, int H, int W, int K, int kh, int kw, int s, int act,
                      const double* x, const double* w, const double* y, const double* dy,
                      double* dw, double* db, double* dx /* nullable */);
int orc_full_forward(int B, int in, int out, int act, const double* x, const double* w,
                     const double* b, double* y);
int orc_full_backward(int B, int in, int out, int act, const double* x, const double* w,
                      const double* y, const double* dy, double* dw, double* db,
                      double* dx /* nullable */);
int orc_loss_forward(int kind, int B, int units, const double* pred, const int* cls,
                     const double* values, double* loss);
int orc_loss_backward(int kind, int B, int units, const double* pred, const int* cls,
                      const double* values, double* grad);

/* ---- L4/L5 network + executor (network.hpp, variants.hpp) ---------------- */
/* per-layer single-sample output shapes, 3 ints (h,w,c) per layer */
int orc_net_chain(const orc_net* net, int* shapes);
/* flat parameter layout: per layer, weights then bias (NetGrads order) */
int64_t orc_net_num_params(const orc_net* net);
int orc_net_param_layout(const orc_net* net, int64_t* w_off, int64_t* w_len, int64_t* b_off,
                         int64_t* b_len);
/* build_network (network.hpp:102-130): Glorot from Rng(seed), zero biases */
int orc_net_init(const orc_net* net, double* params);
/* total elements of all per-layer outputs for batch B (trace size) */
int64_t orc_net_trace_size(const orc_net* net, int B);
/* Executor<T>::run_batch, Imp-6 (variants.hpp:353-376, 484-668).
 * targets: cls (softmax_ce) or values (mse).  With compute_grads=0 it is
 * Executor::forward.  trace (nullable): every layer's post-activation output
 * concatenated; args (nullable): for every pool layer, its output size of
 * int64 argmax entries (-1 for avg pools). */
int orc_net_run_batch(const orc_net* net, int B, const double* params, const double* x,
                      const int* cls, const double* values, int pool_bwd_mode,
                      int compute_grads, double* out, double* loss, double* grads,
                      double* trace, int64_t* args);
/* sgd_step (network.hpp:242-273) over the flat buffers */
void orc_sgd_step(int64_t n, double* w, double* v, const double* g, double lr, double mom);
/* synth_bench_data (bench.cpp:29-45) in fp32 */
int orc_synth_bench_data(const orc_net* net, int B, uint64_t seed, float* x, int* cls,
                         float* values);
/* predict_classes (network.hpp:179-192) */
void orc_predict_classes(int B, int units, const double* out, int* cls);

#ifdef __cplusplus
}
#endif
#endif
