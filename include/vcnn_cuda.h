/*
 * vcnn_cuda.h -- C ABI of libvcnn_cuda.so, the B200 (sm_100a) implementation
 * of the VCNN Imp-6 training path (arXiv 1501.07338).
 *
 * The reference (/root/reference/proj) has no FFI: its operator API is the
 * C++ header-template surface of proj/include/vcnn/(name).hpp.  Every entry point
 * below replaces one function of that surface; the comment cites the
 * reference file:line it stands in for (paths relative to
 * /root/reference/proj/include/vcnn).  Plain pointers and sizes only; no
 * torch or C++ types.  Conventions:
 *   - all tensors fp32 NCHW (linear index ((b*C+c)*H+y)*W+x, tensor.hpp:80-82),
 *     matrices row-major (tensor.hpp:106-127);
 *   - op-level functions take CALLER-OWNED DEVICE pointers and a
 *     cudaStream_t passed as void* (NULL = legacy default stream), are
 *     stream-ordered and do not synchronise unless documented;
 *   - every function returns a vcnn_status; on error, vcnn_last_error()
 *     returns a message (thread-local).  Geometry / shape / bounds errors are
 *     raised on the host before any launch, mirroring the exceptions of the
 *     reference constructors (vectorize.hpp:22-26, :144-148; layers.hpp:77-89).
 *   - precision: VCNN_PREC_TF32 (tcgen05 kind::tf32, fp32 accumulate),
 *     VCNN_PREC_3XTF32 (split hi/lo, three tcgen05 MMAs, fp32-faithful),
 *     VCNN_PREC_FP32 (SIMT fp32 FMA; the on-device exactness reference).
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point returns VCNN_ECUDA.
 */
#ifndef VCNN_CUDA_H
#define VCNN_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VCNN_ABI_VERSION 1

/* status codes; the C++ host layer rethrows them as the reference exception
 * types (common.hpp:26-46) */
typedef enum {
  VCNN_OK = 0,
  VCNN_ESHAPE = 1,     /* ShapeError */
  VCNN_EGEOMETRY = 2,  /* GeometryError */
  VCNN_EBOUNDS = 3,    /* BoundsError */
  VCNN_ECUDA = 4,      /* CUDA runtime / no device */
  VCNN_ENCCL = 5,      /* collective failure */
  VCNN_ECONFIG = 6,    /* ConfigError */
  VCNN_ETRAINING = 7   /* TrainingError */
} vcnn_status;

/* Activation (layers.hpp:13) */
enum { VCNN_ACT_IDENTITY = 0, VCNN_ACT_RELU = 1, VCNN_ACT_SIGMOID = 2, VCNN_ACT_TANH = 3 };
/* PoolMode (vectorize.hpp:127) */
enum { VCNN_POOL_MAX = 0, VCNN_POOL_AVG = 1 };
/* PoolBackwardMode (vectorize.hpp:217) */
enum { VCNN_POOLBWD_EXACT = 0, VCNN_POOLBWD_PAPER_NN = 1 };
/* LossKind (layers.hpp:375) */
enum { VCNN_LOSS_SOFTMAX_CE = 0, VCNN_LOSS_MSE = 1 };
/* LayerSpec alternatives (network.hpp:12-32) */
enum { VCNN_LAYER_CONV = 0, VCNN_LAYER_POOL = 1, VCNN_LAYER_FULL = 2 };
/* arithmetic of the GEMM-shaped kernels */
enum { VCNN_PREC_TF32 = 0, VCNN_PREC_3XTF32 = 1, VCNN_PREC_FP32 = 2 };
/* Reducer (tensor.hpp:185) */
enum { VCNN_REDUCE_SUM = 0, VCNN_REDUCE_MAX = 1, VCNN_REDUCE_MEAN = 2 };

/* ConvGeometry (vectorize.hpp:13-42), valid convolution, no padding */
typedef struct {
  int in_h, in_w, channels, batch;
  int kh, kw, stride;
  int out_h, out_w;
} vcnn_conv_geometry;

/* PoolGeometry (vectorize.hpp:134-162), overlap allowed */
typedef struct {
  int in_h, in_w, channels, batch;
  int ph, pw, stride, mode;
  int out_h, out_w;
} vcnn_pool_geometry;

/* one LayerSpec (network.hpp:12-32): conv uses units=maps,kh,kw,stride,act;
 * pool uses kh,kw (=ph,pw),stride,pool_mode,pool_bias,act; full uses units,act */
typedef struct {
  int kind;
  int units;
  int kh, kw;
  int stride;
  int pool_mode;
  int pool_bias;
  int act;
} vcnn_layer_spec;

/* NetworkSpec (network.hpp:37-73) */
typedef struct {
  int in_h, in_w, in_c;
  int nlayers;
  const vcnn_layer_spec* layers;
  int loss;
  uint64_t seed;
} vcnn_net_spec;

/* ------------------------------------------------------------------------ */
/* library                                                                   */
/* ------------------------------------------------------------------------ */
int vcnn_abi_version(void);
const char* vcnn_last_error(void);
/* SM count / compute capability of the current device; VCNN_ECUDA if none */
int vcnn_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* kernels launched by this library since load (gpu_launches evidence) */
int64_t vcnn_launch_count(void);
/* synchronous host -> device copy (lets C / C++ hosts stage batches without
 * CUDA headers); VCNN_ECUDA without a device */
int vcnn_copy_h2d(void* dev, const void* host, size_t bytes);

/* ------------------------------------------------------------------------ */
/* geometry (host only, no device needed)                                    */
/* ------------------------------------------------------------------------ */
/* ConvGeometry(Shape, kh, kw, stride) (vectorize.hpp:19-29) */
int vcnn_conv_geometry_init(vcnn_conv_geometry* g, int in_h, int in_w, int channels, int batch,
                            int kh, int kw, int stride);
/* PoolGeometry(Shape, ph, pw, stride, mode) (vectorize.hpp:141-151) */
int vcnn_pool_geometry_init(vcnn_pool_geometry* g, int in_h, int in_w, int channels, int batch,
                            int ph, int pw, int stride, int mode);
/* NetworkSpec::chain (network.hpp:45-67): per-layer (h,w,c), 3 ints each */
int vcnn_net_spec_chain(const vcnn_net_spec* spec, int* shapes);

/* the reference bench's synthetic batch (bench.cpp:29-45): Rng(seed), X ~
 * U[0,1) NCHW [batch][C][H][W], then cls[batch] = uniform_int(units) for
 * softmax-CE or values[batch][units] ~ U[0,1) for MSE (host buffers) */
int vcnn_synth_bench_data(const vcnn_net_spec* spec, int batch, uint64_t seed, float* x, int* cls,
                          float* values);

/* ------------------------------------------------------------------------ */
/* L1 tensor primitives (tensor.hpp)                                         */
/* ------------------------------------------------------------------------ */
/* matmul: C[m][n] = A[m][k] * B[k][n] (tensor.hpp:131-150) */
int vcnn_matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c,
                int precision, void* stream);
/* matmul_transB: C[m][n] = A[m][k] * B[n][k]^T (tensor.hpp:154-174) */
int vcnn_matmul_transB(int64_t m, int64_t k, int64_t n, const float* a, const float* b,
                       float* c, int precision, void* stream);
/* general GEMM (matmul / matmul_transB / transpose, tensor.hpp:131-182, with
 * the conv_affine / full-layer epilogue, layers.hpp:99-105, :230-247):
 * C[m][n] = act(sum_k op(A)[m][k] op(B)[k][n] + bias[n]); op(A) = A [m][k]
 * (lda) or, trans_a, A^T of A [k][m]; op(B) = B [k][n] (ldb) or, trans_b,
 * B^T of B [n][k]; C row stride ldc; bias nullable */
int vcnn_gemm(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, const float* a,
              int64_t lda, const float* b, int64_t ldb, float* c, int64_t ldc, const float* bias,
              int act, int precision, void* stream);
/* accumulate_by_index (tensor.hpp:228-266): out[t] = reducer over
 * {values[s] : (s,t) in map}, pairs consumed in map order (deterministic);
 * empty buckets 0. */
int vcnn_accumulate_by_index(const float* values, int64_t source_len, const int64_t* source,
                             const int64_t* target, int64_t pairs, int64_t target_len,
                             int reducer, float* out, void* stream);
/* accumulate_max_arg (tensor.hpp:271-289): ties -> lowest source, empty -> (0,-1) */
int vcnn_accumulate_max_arg(const float* values, int64_t source_len, const int64_t* source,
                            const int64_t* target, int64_t pairs, int64_t target_len,
                            float* out, int64_t* arg, void* stream);

/* ------------------------------------------------------------------------ */
/* L2 vectorize ops (vectorize.hpp)                                          */
/* ------------------------------------------------------------------------ */
/* im2col (vectorize.hpp:54-79): patch[(c*kh+ky)*kw+kx][b*OH*OW+oy*OW+ox] */
int vcnn_im2col(const vcnn_conv_geometry* g, const float* x, float* patch, void* stream);
/* col2im (vectorize.hpp:111-120): exact adjoint of im2col, gather form,
 * each input cell sums its patch cells in (ky,kx) ascending order */
int vcnn_col2im(const vcnn_conv_geometry* g, const float* dpatch, float* dx, void* stream);
/* build_col2im_map (vectorize.hpp:84-106): pairs in (c,ky,kx,b,oy,ox) order;
 * source and target each hold patch_len*cols int64 entries */
int vcnn_col2im_map(const vcnn_conv_geometry* g, int64_t* source, int64_t* target, void* stream);
/* build_pool_map (vectorize.hpp:167-191): pairs in (b,c,oy,ox,py,px) order */
int vcnn_pool_map(const vcnn_pool_geometry* g, int64_t* source, int64_t* target, void* stream);
/* pool_forward (vectorize.hpp:197-215): max (strict >, first element seeds,
 * ties -> lowest index; arg = global input index) or avg (sum / window);
 * arg may be NULL; for avg pools it is filled with -1 when given */
int vcnn_pool_forward(const vcnn_pool_geometry* g, const float* x, float* y, int64_t* arg,
                      void* stream);
/* pool_backward (vectorize.hpp:224-249), gather form (deterministic under
 * overlap): exact max -> argmax routing, exact avg -> dy/window, paper_nn ->
 * unscaled nearest-neighbour upsampling */
int vcnn_pool_backward(const vcnn_pool_geometry* g, int bwd_mode, const float* dy,
                       const int64_t* arg, float* dx, void* stream);

/* ------------------------------------------------------------------------ */
/* L3 layers (layers.hpp)                                                    */
/* ------------------------------------------------------------------------ */
/* apply_activation (layers.hpp:50-54): y = act(x); x may equal y */
int vcnn_activation_forward(int64_t n, int act, const float* x, float* y, void* stream);
/* apply_activation_grad (layers.hpp:57-61): grad *= act'(y) (from output) */
int vcnn_activation_backward(int64_t n, int act, const float* y, float* grad, void* stream);
/* conv_forward (layers.hpp:139-149): y = act(W*col(x) + b), NCHW out
 * [batch][maps][out_h][out_w]; implicit GEMM, no patch matrix */
int vcnn_conv_forward(const vcnn_conv_geometry* g, int maps, const float* x, const float* w,
                      const float* bias, int act, int precision, float* y, void* stream);
/* conv_backward (layers.hpp:183-195): dy is the gradient of the
 * post-activation output; dw [maps][C*kh*kw], db [maps], dx (nullable)
 * [batch][C][H][W]. Implicit wgrad (deterministic split-K) and dgrad. */
int vcnn_conv_backward(const vcnn_conv_geometry* g, int maps, const float* x, const float* w,
                       const float* y, const float* dy, int act, int precision, float* dw,
                       float* db, float* dx, void* stream);
/* full_forward (layers.hpp:230-247): y[b][o] = act(sum_i x[b][i] W[o][i] + b[o]) */
int vcnn_full_forward(int batch, int in_units, int out_units, const float* x, const float* w,
                      const float* bias, int act, int precision, float* y, void* stream);
/* full_backward (layers.hpp:269-278) */
int vcnn_full_backward(int batch, int in_units, int out_units, const float* x, const float* w,
                       const float* y, const float* dy, int act, int precision, float* dw,
                       float* db, float* dx, void* stream);
/* pool_layer_forward (layers.hpp:305-321): pool + optional per-channel bias
 * (NULL = none) + activation; arg may be NULL */
int vcnn_pool_layer_forward(const vcnn_pool_geometry* g, const float* x, const float* bias,
                            int act, float* y, int64_t* arg, void* stream);
/* pool_layer_backward (layers.hpp:356-363): dbias may be NULL */
int vcnn_pool_layer_backward(const vcnn_pool_geometry* g, int bwd_mode, const float* y, int act,
                             const float* dy, const int64_t* arg, float* dx, float* dbias,
                             void* stream);
/* loss_forward (layers.hpp:402-434); *loss is a DEVICE scalar.  Class
 * indices are checked on the device; an out-of-range class makes this call
 * synchronise and return VCNN_EBOUNDS (layers.hpp:413-415). */
int vcnn_loss_forward(int kind, int batch, int units, const float* pred, const int* cls,
                      const float* values, float* loss, void* stream);
/* loss_backward (layers.hpp:436-468) */
int vcnn_loss_backward(int kind, int batch, int units, const float* pred, const int* cls,
                       const float* values, float* grad, void* stream);
/* fused loss_forward + loss_backward in one kernel */
int vcnn_loss_fused(int kind, int batch, int units, const float* pred, const int* cls,
                    const float* values, float* loss, float* grad, void* stream);

/* ------------------------------------------------------------------------ */
/* L4 update (network.hpp)                                                   */
/* ------------------------------------------------------------------------ */
/* sgd_step (network.hpp:242-273) over one flat buffer:
 * v = mom*v + grad_scale*g; w -= lr*v  (grad_scale = 1 is the reference) */
int vcnn_sgd_step(int64_t n, float* w, float* v, const float* g, float lr, float mom,
                  float grad_scale, void* stream);

/* ------------------------------------------------------------------------ */
/* L4-L6 network engine: build_network + Executor<float>(imp6) + sgd_step     */
/* with device-resident parameters, trace and CUDA-graph replay              */
/* ------------------------------------------------------------------------ */
typedef struct vcnn_net vcnn_net;

/* build_network (network.hpp:102-130) + Executor<float>(Variant::imp6)
 * (variants.hpp:336): parameters initialised on the host with the
 * reference's Rng(spec.seed) Glorot stream (layers.hpp:473-501), uploaded
 * once; buffers sized for max_batch. */
int vcnn_net_create(const vcnn_net_spec* spec, int max_batch, int precision, vcnn_net** out);
int vcnn_net_destroy(vcnn_net* net);
int64_t vcnn_net_num_params(const vcnn_net* net);
/* flat parameter layout: per layer, weights then bias (NetGrads order) */
int vcnn_net_param_layout(const vcnn_net* net, int64_t* w_off, int64_t* w_len, int64_t* b_off,
                          int64_t* b_len);
/* per-layer output sizes for one sample */
int vcnn_net_layer_out_size(const vcnn_net* net, int layer, int64_t* per_sample);
int vcnn_net_set_stream(vcnn_net* net, void* stream);
/* Executor::set_pool_backward_mode (variants.hpp:342) */
int vcnn_net_set_pool_backward_mode(vcnn_net* net, int mode);
int vcnn_net_set_precision(vcnn_net* net, int precision);
/* conv -> max-pool fusion (default on, TF32): the
 * pool runs in the conv epilogue and its backward is routed inside the conv's
 * wgrad / dgrad.  Results are bit-identical with it off. */
int vcnn_net_set_fusion(vcnn_net* net, int enable);
/* keep the whole forward trace (every layer output) and every layer's
 * pre-activation gradient in device memory, as the reference's LayerTrace
 * does (variants.hpp:305-323); disables fusion.  Default off. */
int vcnn_net_set_trace(vcnn_net* net, int keep);
/* host <-> device parameter / gradient / velocity transfers (synchronous) */
int vcnn_net_get_params(vcnn_net* net, float* host);
int vcnn_net_set_params(vcnn_net* net, const float* host);
int vcnn_net_get_grads(vcnn_net* net, float* host);
int vcnn_net_get_velocity(vcnn_net* net, float* host);
int vcnn_net_set_velocity(vcnn_net* net, const float* host);
/* device pointers of the flat buffers (for collectives: all-reduce grads).
 * `params` is READ-ONLY for callers unless they call vcnn_net_params_updated
 * afterwards: the conv kernels read tf32 weight images derived from it. */
int vcnn_net_device_buffers(vcnn_net* net, float** params, float** grads, float** velocity);
/* re-derive the conv kernels' weight images after params were written
 * through the device pointer (stream-ordered) */
int vcnn_net_params_updated(vcnn_net* net);
/* device pointers of the input slots (x [max_batch][C][H][W], cls, values) */
int vcnn_net_input_buffers(vcnn_net* net, float** x, int** cls, float** values);
/* stage a batch already in device memory (copied, stream-ordered) */
int vcnn_net_set_batch_device(vcnn_net* net, int batch, const float* x, const int* cls,
                              const float* values);
/* a ring of nbatch device batches (x [nbatch][x_stride floats], targets
 * [nbatch][t_stride 32-bit words]: class ids or target values): every
 * following train step first stages the ring's next batch (a kernel captured
 * in the step's graph; a device cursor walks the ring) -- for dataset epochs
 * and benchmarks whose batches are already resident.  nbatch = 0 detaches. */
int vcnn_net_set_batch_ring(vcnn_net* net, int nbatch, int batch, const float* x,
                            int64_t x_stride, const void* targets, int64_t t_stride);
/* Executor::run_batch with targets (variants.hpp:353-376): forward, fused
 * loss, backward; grads land in the device grads buffer, loss in a device
 * scalar.  Stream-ordered, no host sync. */
int vcnn_net_forward_backward(vcnn_net* net, int batch);
/* Executor::forward (variants.hpp:346-348) */
int vcnn_net_forward(vcnn_net* net, int batch);
/* sgd_step over all parameters; grad_scale multiplies the gradient (1/world
 * for a summed data-parallel all-reduce) */
int vcnn_net_sgd_step(vcnn_net* net, float lr, float mom, float grad_scale);
/* forward_backward + sgd_step; replayed from a CUDA graph when enabled */
int vcnn_net_train_step(vcnn_net* net, int batch, float lr, float mom);
/* nsteps train steps, up to 8 captured in one graph launch (with graphs
 * enabled; a batch ring attached makes every step stage its next batch) */
int vcnn_net_train_steps(vcnn_net* net, int nsteps, int batch, float lr, float mom);
/* end-to-end: HOST batch in (validated: class bounds -> VCNN_EBOUNDS),
 * H2D copy, train step, D2H loss; synchronous */
int vcnn_net_train_step_host(vcnn_net* net, int batch, const float* x, const int* cls,
                             const float* values, float lr, float mom, float* loss_out);
/* end-to-end training over a stream of HOST batches: step i reads
 * x + i*x_stride (batch rows) and cls/values + i*t_stride; its loss lands in
 * losses[i] (host).  The H2D copy of batch i+1 runs on a copy stream while
 * step i computes (two device staging slots), so the copies overlap the
 * steps; results equal nsteps calls of vcnn_net_train_step_host.  Host
 * buffers should be pinned (pageable memory serialises the copies).
 * Synchronous: returns after the last loss is on the host. */
int vcnn_net_train_host_stream(vcnn_net* net, int nsteps, int batch, const float* x,
                               int64_t x_stride, const int* cls, const float* values,
                               int64_t t_stride, float lr, float mom, float* losses);
/* Trainer<T>::fit's inner loop for ONE epoch, device-resident
 * (training.hpp:60-88, gather_batch network.hpp:165-176): the dataset
 * (images [count][in], cls [count] or values [count][out]) lives in device
 * memory, `order` is the epoch's permutation (device, count ints -- the
 * reference's Rng::shuffle of 0..count-1, common.hpp:84-90), batches of
 * `batch` rows with a smaller last batch.  Per batch: index-gather kernel +
 * train step (CUDA-graph replayed when enabled); the batch loss lands in
 * losses[b] (device, ceil(count/batch) floats).  Stream-ordered, no host
 * synchronisation; class bounds are the caller's contract (checked on the
 * host by the C++/Python Trainers when the dataset is uploaded). */
int vcnn_net_train_epoch(vcnn_net* net, const float* images, const int* cls,
                         const float* values, int count, const int* order, int batch, float lr,
                         float mom, float* losses);
/* Trainer::fit's non-finite stop (training.hpp:77-80) on the device: while
 * enabled, a step whose batch loss is non-finite skips its sgd_step, and so
 * does every later step until the guard is re-armed (this call again), so the
 * weights stay those the offending batch ran on.  vcnn_net_train_epoch arms
 * it for its own duration. */
int vcnn_net_set_nonfinite_guard(vcnn_net* net, int enable);
/* end-to-end inference: HOST batch in, HOST output out; synchronous */
int vcnn_net_forward_host(vcnn_net* net, int batch, const float* x, float* out);
/* CUDA-graph capture of train_step (per batch size); 0 disables */
int vcnn_net_enable_graph(vcnn_net* net, int enable);
/* results (synchronous reads) */
int vcnn_net_get_loss(vcnn_net* net, float* loss);
int vcnn_net_get_output(vcnn_net* net, float* host);
int vcnn_net_get_layer_output(vcnn_net* net, int layer, float* host);
/* gradient w.r.t. the PRE-activation of a layer (dY * act'(Y)) from the
 * last backward pass, [max_batch][out_per_sample] */
int vcnn_net_get_layer_grad(vcnn_net* net, int layer, float* host);
/* pool argmax of a max-pool layer as int64 global input indices */
int vcnn_net_get_pool_arg(vcnn_net* net, int layer, int64_t* host);
/* kernels per train step (fwd+bwd+sgd) at the current settings */
int vcnn_net_kernels_per_step(vcnn_net* net, int* count);
/* BreakdownTimer (variants.hpp:249-274) with CUDA events: enable, then read
 * the 8 component seconds {conv,pool,full,other}x{f,b} accumulated since the
 * last reset (synchronises) */
int vcnn_net_enable_breakdown(vcnn_net* net, int enable);
int vcnn_net_read_breakdown(vcnn_net* net, double* seconds8);
/* per-op CUDA-event timing collected in breakdown mode: (nlayers+1)*5 slots,
 * slot (layer+1)*5 + op with op 0 fwd, 1 wgrad, 2 dgrad, 3 loss, 4 sgd
 * (layer -1 = whole-net ops); seconds and launch counts since enable */
int vcnn_net_read_op_timing(vcnn_net* net, double* seconds, int64_t* counts);

/* ------------------------------------------------------------------------ */
/* L7 data parallelism: replicas of one network on the GPUs of   */
/* one box, minibatch sharded, one gradient exchange per step at            */
/* Trainer::fit's run_batch -> sgd_step boundary (training.hpp:76-81)       */
/* ------------------------------------------------------------------------ */
typedef struct vcnn_dp vcnn_dp;
/* exchange: one fused kernel per replica reading every replica's gradient
 * over NVLink peer mappings (rank-ordered sum + SGD + conv weight packs), or
 * NCCL all-reduce + sgd */
enum { VCNN_DP_P2P = 0, VCNN_DP_NCCL = 1 };
#define VCNN_DP_ID_BYTES 128
#define VCNN_DP_HANDLE_BYTES 256
/* ncclGetUniqueId (rank 0; the caller broadcasts the 128 bytes) */
int vcnn_dp_unique_id(void* id);
/* process-per-GPU: NCCL communicator from `id`, exchange of the replicas'
 * gradient / signal buffer IPC handles over it, P2P mappings; attaches the
 * group to `net`: from then on vcnn_net_sgd_step / vcnn_net_train_step do the
 * exchange.  Collective: every rank calls it. */
int vcnn_dp_init(vcnn_net* net, int world, int rank, const void* id, vcnn_dp** out);
/* the same in three steps, for hosts that exchange the handles themselves
 * (any all-gather): create, publish VCNN_DP_HANDLE_BYTES, connect with all
 * ranks' handles in rank order (+ an optional NCCL id for the fallback) */
int vcnn_dp_create(vcnn_net* net, int world, int rank, vcnn_dp** out);
int vcnn_dp_handle(const vcnn_dp* dp, void* handle);
int vcnn_dp_connect(vcnn_dp* dp, const void* handles, const void* id);
/* one process, `world` replicas (same or different devices) linked by
 * direct pointers.  barrier = 1: replicas step independently (each on its
 * own stream) and synchronise inside the exchange kernel, exactly as across
 * processes; barrier = 0: G logical shards stepped together by
 * vcnn_dp_group_train_step (event-ordered, no device barrier). */
int vcnn_dp_group(vcnn_net* const* nets, int world, int barrier, vcnn_dp** out);
int vcnn_dp_group_train_step(vcnn_dp* const* dps, int world, const int* batches, float lr,
                             float mom);
int vcnn_dp_set_mode(vcnn_dp* dp, int mode);
int vcnn_dp_get_mode(const vcnn_dp* dp, int* mode);
/* per-rank sample counts of the current global batch (weights B_p / B);
 * default: equal shards */
int vcnn_dp_set_shards(vcnn_dp* dp, const int* batches);
/* the exchange + sgd_step alone (after vcnn_net_forward_backward) */
int vcnn_dp_allreduce_sgd(vcnn_dp* dp, float lr, float mom);
/* forward_backward + exchange + sgd_step (CUDA-graph replayed when enabled) */
int vcnn_dp_train_step(vcnn_dp* dp, int batch, float lr, float mom);
/* synchronises; VCNN_ENCCL if an exchange barrier timed out */
int vcnn_dp_status(vcnn_dp* dp);
/* detaches from the net and frees the group's resources */
int vcnn_dp_destroy(vcnn_dp* dp);

#ifdef __cplusplus
}
#endif
#endif /* VCNN_CUDA_H */
