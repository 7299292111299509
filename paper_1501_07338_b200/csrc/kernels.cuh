// kernels.cuh -- internal launcher API shared by the C ABI (capi.cu) and the
// network engine (engine.cu).  All launchers are stream-ordered and return a
// vcnn_status.  "gpre" is always a gradient w.r.t. a layer's PRE-activation
// (dY * act'(Y)), which is how the engine fuses every activation derivative
// into the kernel that produces the gradient (no standalone act' pass).
#pragma once

#include <vector>

#include "common.cuh"

namespace vcnn_b200 {

// ConvGeometry + map count (vectorize.hpp:13-42)
struct ConvDesc {
  int B, C, H, W;  // input
  int K;           // output maps
  int kh, kw, s;
  int OH, OW;
  __host__ __device__ int64_t kd() const { return (int64_t)C * kh * kw; }
  __host__ __device__ int64_t ohw() const { return (int64_t)OH * OW; }
  __host__ __device__ int64_t pixels() const { return ohw() * B; }
  __host__ __device__ int64_t in_size() const { return (int64_t)B * C * H * W; }
  __host__ __device__ int64_t out_size() const { return (int64_t)B * K * OH * OW; }
};

// PoolGeometry (vectorize.hpp:134-162)
struct PoolDesc {
  int B, C, H, W;
  int ph, pw, s, mode;
  int OH, OW;
  __host__ __device__ int64_t in_size() const { return (int64_t)B * C * H * W; }
  __host__ __device__ int64_t out_size() const { return (int64_t)B * C * OH * OW; }
};

// Device scratch for split-K partial sums and loss reductions.
struct Workspace {
  float* ptr = nullptr;
  size_t bytes = 0;
};

// ---- memory-bound kernels (simt.cu) ----
int launch_im2col(const ConvDesc& d, const float* x, float* P, cudaStream_t st);
// dX = col2im(dP) [* act_prev'(yprev)]
int launch_col2im(const ConvDesc& d, const float* dP, float* dX, cudaStream_t st,
                  const float* yprev = nullptr, int act_prev = VCNN_ACT_IDENTITY);
int launch_col2im_map(const ConvDesc& d, int64_t* src, int64_t* tgt, cudaStream_t st);
int launch_pool_map(const PoolDesc& d, int64_t* src, int64_t* tgt, cudaStream_t st);
template <class IdxT>
int launch_pool_fwd(const PoolDesc& d, const float* x, const float* bias, int act, float* y,
                    IdxT* arg, cudaStream_t st);
// dx = pool_backward(gpre) * act_prev'(yprev)   (yprev may be null)
template <class IdxT>
int launch_pool_bwd(const PoolDesc& d, int bwd_mode, const float* gpre, const IdxT* arg,
                    float* dx, const float* yprev, int act_prev, cudaStream_t st);
int launch_pool_bias_grad(const PoolDesc& d, const float* gpre, float* dbias, cudaStream_t st);
int launch_act_fwd(int64_t n, int act, const float* x, float* y, cudaStream_t st);
// g = dy * act'(y)  (dy may equal g)
int launch_act_bwd(int64_t n, int act, const float* y, const float* dy, float* g,
                   cudaStream_t st);
// fused loss forward+backward; grad = dL/dpred * act_last'(pred); err set on
// out-of-range class.  Any of loss/grad may be null.  ws (nullable, at least
// kLossWsFloats floats, zero-initialised once) lets MSE spread over the whole
// chip: per-CTA partials + a last-CTA fixed-order reduce (deterministic).
constexpr int kMseMaxCtas = 1024;
constexpr int kLossWsFloats = kMseMaxCtas + 4;
int launch_loss(int kind, int B, int units, const float* pred, const int* cls,
                const float* values, float* loss, float* grad, int act_last, int* err,
                cudaStream_t st, float* ws = nullptr);
int launch_sgd(int64_t n, float* w, float* v, const float* g, float lr, float mom, float scale,
               cudaStream_t st);
// batch row j <- dataset row order[start + j] (+ class / value targets)
int launch_gather_rows(int n, int64_t per, const float* src, const int* order, int start,
                       float* dst, int64_t tper, const int* cls_src, int* cls_dst,
                       const float* val_src, float* val_dst, cudaStream_t st);
int launch_store_scalar(const float* src, float* dst, cudaStream_t st);
int launch_stage_batch(const float* xs, float* xd, int64_t nx, const void* ts, void* td,
                       int64_t nt_words, cudaStream_t st);
int launch_ring_stage(const float* xs, float* xd, int64_t nx, int64_t xstride, const void* ts,
                      void* td, int64_t nt, int64_t tstride, int nbatch, const int* cursor,
                      cudaStream_t st, const float* lsrc = nullptr, float* lhist = nullptr,
                      int lmask = 0);
// the network head fused: last full layer fwd + loss fwd/bwd + its
// dW / db / dX (dX * act_prev'(x)); one cluster, fp32
bool head_fusable(int B, int in, int out);
int launch_head(int B, int in, int out, const float* x, const float* W, const float* bias,
                int act, float* y, int loss_kind, const int* cls, const float* values,
                float* loss, float* gpre, float* dW, float* db, float* dx, int act_prev, int* err,
                cudaStream_t st);
// the two-layer tail fused (head.cu): small full layer H + last full layer O
// fwd, loss fwd/bwd, both layers' dW / db and dX; one 16-CTA cluster per
// batch slice (mlp_head_slices): with ncl > 1 slices the layers' dW / db are
// written per slice to part ([ncl][per], param order W_H | b_H | W_O | b_O,
// mlp_head_part_floats) for the caller to sum in slice order; lpart [ncl]
// and the zero-initialised ticket carry the loss partials
constexpr int kMaxSlices = 8;
bool mlp_head_fusable(int B, int in, int h, int out);
int mlp_head_slices(int B, int in, int h, int out);
size_t mlp_head_part_floats(int B, int in, int h, int out);
int launch_mlp_head(int B, int in, int h, int out, const float* x, const float* WH,
                    const float* bH, int actH, const float* WO, const float* bO, int actO,
                    float* yH, float* yO, int loss_kind, const int* cls, const float* values,
                    float* loss, int* err, float* gH, float* gO, float* dWH, float* dbH,
                    float* dWO, float* dbO, float* dx, int act_prev, cudaStream_t st,
                    int ncl = 1, float* part = nullptr, float* lpart = nullptr,
                    unsigned* ticket = nullptr);
int launch_accumulate(const float* values, const int64_t* source, const int64_t* target,
                      int64_t pairs, int64_t target_len, int reducer, float* out, int64_t* arg,
                      cudaStream_t st);

// ---- GEMM-shaped kernels: SIMT fp32 reference (simt.cu) or tcgen05 (tc.cu) ----
// wf / wt: prepared weights (tc::prep_weights) enabling the TF32 slab
// kernels; nullptr -> generic kernels
int launch_conv_fwd(const ConvDesc& d, const float* x, const float* w, const float* b, int act,
                    float* y, int prec, const Workspace& ws, cudaStream_t st,
                    const float* wf = nullptr);
// dw [K][kd], db [K] from the pre-activation gradient gpre [B][K][OH][OW]
int launch_conv_wgrad(const ConvDesc& d, const float* x, const float* gpre, float* dw,
                      float* db, int prec, const Workspace& ws, cudaStream_t st);
// dx [B][C][H][W] = col2im(W^T gpre) * act_prev'(yprev)
int launch_conv_dgrad(const ConvDesc& d, const float* gpre, const float* w, float* dx,
                      const float* yprev, int act_prev, int prec, const Workspace& ws,
                      cudaStream_t st, const float* wt = nullptr);
int launch_full_fwd(int B, int in, int out, const float* x, const float* w, const float* b,
                    int act, float* y, int prec, const Workspace& ws, cudaStream_t st);
int launch_full_wgrad(int B, int in, int out, const float* x, const float* gpre, float* dw,
                      float* db, int prec, const Workspace& ws, cudaStream_t st);
int launch_full_dgrad(int B, int in, int out, const float* gpre, const float* w, float* dx,
                      const float* yprev, int act_prev, int prec, const Workspace& ws,
                      cudaStream_t st);
// C[m][n] = A[m][k] * (transB ? B[n][k] : B[k][n])
int launch_matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c,
                  bool transB, int prec, const Workspace& ws, cudaStream_t st);

// workspace bytes the GEMM launchers need for a shape (0 if none)
size_t conv_workspace(const ConvDesc& d, int prec);
size_t full_workspace(int B, int in, int out, int prec);
size_t matmul_workspace(int64_t m, int64_t k, int64_t n, int prec);

// ---- SIMT implementations (simt.cu) used for VCNN_PREC_FP32 ----
namespace simt {
int conv_fwd(const ConvDesc& d, const float* x, const float* w, const float* b, int act,
             float* y, cudaStream_t st);
int conv_wgrad(const ConvDesc& d, const float* x, const float* gpre, float* dw, float* db,
               cudaStream_t st);
int conv_dgrad(const ConvDesc& d, const float* gpre, const float* w, float* dx,
               const float* yprev, int act_prev, cudaStream_t st);
bool full_fwd_warp_ok(int B, int in, int out, const float* x, const float* w);
int full_fwd_mid(int B, int in, int out, const float* x, const float* w, const float* b, int act,
                 float* y, cudaStream_t st);
int full_fwd(int B, int in, int out, const float* x, const float* w, const float* b, int act,
             float* y, cudaStream_t st);
int full_wgrad(int B, int in, int out, const float* x, const float* gpre, float* dw, float* db,
               cudaStream_t st);
int full_dgrad(int B, int in, int out, const float* gpre, const float* w, float* dx,
               const float* yprev, int act_prev, cudaStream_t st);
int matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c,
           bool transB, cudaStream_t st);
int gemm(int64_t m, int64_t n, int64_t k, const float* a, int64_t as_m, int64_t as_k,
         const float* b, int64_t bs_k, int64_t bs_n, float* c, int64_t ldc, const float* bias,
         int act, cudaStream_t st);
}  // namespace simt

// Source of a conv layer's pre-activation output gradient G [B][K][OH][OW]:
// materialised (g), or routed on the fly from a fused non-overlapping max
// pool (pool = window == stride): dP = the pool-output gradient ALREADY
// multiplied by the conv activation derivative at the argmax (the producer
// applies it with yprev = pool output, act_prev = conv act), parg = int32
// global argmax into [B][K][OH][OW].  G = dP at the argmax, 0 elsewhere.
struct GradSrc {
  const float* g = nullptr;
  const float* dP = nullptr;
  const int32_t* parg = nullptr;
  int pool = 0;
  int POH = 0, POW = 0;
};

// fused max pool written by the conv-forward epilogue
struct PoolFuse {
  int pool = 0;  // window == stride; 0 = none
  int POH = 0, POW = 0;
  float* y = nullptr;
  int32_t* arg = nullptr;
  float* y_nhwc = nullptr;  // small-Kd forward: also the pooled output as tf32 NHWC
};

// data-parallel exchange + update (dp.cu): the replicas' gradient buffers
// (peers through P2P mappings), their signal buffers [2][world][nslot] u32,
// per-rank weights B_p / B_global; barrier = 0 when the caller orders the
// replicas itself (one stream, G logical shards on one device)
constexpr int kMaxWorld = 8;
constexpr int kMaxDpSlots = 256;
struct DpPeers {
  const float* g[kMaxWorld];
  uint32_t* sig[kMaxWorld];
  float scale[kMaxWorld];
  uint32_t* my_sig;
  uint32_t* epoch;  // [nslot], this replica's
  int* err;
  int64_t timeout_ns;
  int world, rank, nslot, barrier;
};
// a data-parallel group attached to a net (dp.cu): the engine's sgd step
// becomes the group exchange + update
struct DpLink {
  int world = 1;
  int mode = 0;  // VCNN_DP_P2P / VCNN_DP_NCCL
  DpPeers peers{};
  bool equal = true;    // all shards the same size (NCCL path: scale 1/world)
  float local_w = 1.f;  // this rank's B_p / B_global
  int version = 0;      // bumped when shard weights / mode change (graph key)
  // NCCL fallback: in-place sum all-reduce of the flat gradient
  int (*allreduce)(DpLink* l, float* buf, int64_t n, cudaStream_t st) = nullptr;
  void* comm = nullptr;
};
int dp_scale(int64_t n, float* buf, float s, cudaStream_t st);
// engine hooks for dp.cu (engine.cu): attach (or detach with null) a group
// to a net -- its sgd step becomes the exchange; drops cached step graphs
int engine_attach_dp(vcnn_net* n, DpLink* link);
cudaStream_t engine_stream(vcnn_net* n);

// ---- direct (shifted-view) stride-1 conv forward / dgrad (direct.cu, TF32) ----
namespace direct {
bool fwd_ok(const ConvDesc& d, int pool);
// small-Kd forward (C*kh*kw <= 96, K <= 32: first layers), mma.sync TF32,
// optional fused 2x2 max pool; reads the fp32 weights [K][Kd] directly
bool small_fwd_ok(const ConvDesc& d, int pool);
int conv_fwd_small(const ConvDesc& d, const float* x, const float* w, const float* bias, int act,
                   float* y, const PoolFuse& pf, cudaStream_t st, const float* ps = nullptr);
// the small forward's weight image: tf32, [nnt*8][wst], zero padded; one TMA
// bulk copy per CTA when passed as `ps` (kept current by sgd_pack)
size_t small_fwd_pack_floats(const ConvDesc& d);
int small_fwd_wst(const ConvDesc& d);  // row stride of that image (0: not supported)
int small_fwd_pack(const ConvDesc& d, const float* w, float* ps, cudaStream_t st);
bool dgrad_ok(const ConvDesc& d, int pool = 0, int POH = 0, int POW = 0);
// prepacked tf32 weights: mode 0 forward, 1 dgrad (0 floats: not supported)
size_t pack_floats(const ConvDesc& d, int mode);
int pack_weights(const ConvDesc& d, int mode, const float* w, float* pk, cudaStream_t st);
// nhwc_map (nullable, nhwc_map_bytes()): the input as a tf32 NHWC copy
// through a tensor map (make_nhwc_map): the slab is one TMA, no build
int conv_fwd(const ConvDesc& d, const float* x, const float* pk, const float* bias, int act,
             float* y, const PoolFuse& pf, cudaStream_t st, const void* nhwc_map = nullptr);
bool fwd_tma_ok(const ConvDesc& d, int pool);
size_t nhwc_map_bytes();
int make_nhwc_map(const ConvDesc& d, const float* x_nhwc, void* map);
int conv_dgrad(const ConvDesc& d, const GradSrc& gs, const float* pk, float* dx,
               const float* yprev, int act_prev, cudaStream_t st);
// sgd_step fused with the refresh of the conv layers' packs (pf / pd may be
// null); pack padding must already be zero (pack_weights at creation).  At
// most kMaxPackLayers layers per launch (the table is a kernel argument).
constexpr int kMaxPackLayers = 8;
struct PackSpec {
  ConvDesc d;
  int64_t w_off;
  float* pf;
  float* pd;
  float* ps = nullptr;  // small-Kd forward image (small_fwd_pack_floats)
};
// a weight gradient left as per-image partials [nimg][stride] (dW then db
// in NetGrads order, `per` values), summed by the update (sgd_pack)
struct ImageSumFold {
  const float* part = nullptr;
  int nimg = 0;
  int64_t per = 0, stride = 0;
};
// guard (nullable): int[2] {armed, tripped}; while armed, a non-finite *loss
// trips it and the update (and every later one) is skipped
// fold (nullable, fold->part set): params [fold_off, fold_off + per) take
// their gradient from the per-image partials (written to g as well)
// out[i] = the fixed-order sum over nimg partials part[k * stride + i], i < per
int sum_partials(int nimg, int64_t per, int64_t stride, const float* part, float* out,
                 cudaStream_t st);
int sgd_pack(int64_t n, float* w, float* v, float* g, float lr, float mom, float scale,
             const std::vector<PackSpec>& layers, cudaStream_t st, const float* loss = nullptr,
             int* guard = nullptr, const ImageSumFold* fold = nullptr, int64_t fold_off = 0,
             const ImageSumFold* fold2 = nullptr, int64_t fold2_off = 0,
             int* ring_step = nullptr);
int dp_blocks(int64_t n);
int dp_sgd_pack(int64_t n, float* w, float* v, float lr, float mom,
                const std::vector<PackSpec>& layers, const DpPeers& peers, cudaStream_t st,
                int* ring_step = nullptr);
// weight gradient of a 1-D (kh == 1) conv with a long kernel (kw 16..128) on
// tcgen05 (wgrad1d.cu): M = taps, N = maps, K = a row's positions, the row
// staged as 4-element granules; row-group partials + fixed-order reduce
bool wgrad1d_ok(const ConvDesc& d);
size_t wgrad1d_workspace(const ConvDesc& d);
int conv_wgrad1d(const ConvDesc& d, const float* x, const float* gpre, float* dw, float* db,
                 const Workspace& ws, cudaStream_t st);
// weight gradient as shifted-view GEMMs (wgrad.cu): dW [K][C][kh][kw] and db
// [K] (nullable) from x and the (possibly pool-routed) gradient; per-image
// partials in ws, fixed-order reduce
bool wgrad_ok(const ConvDesc& d, const GradSrc& gs);
size_t wgrad_workspace(const ConvDesc& d);
int conv_wgrad(const ConvDesc& d, const float* x, const GradSrc& gs, float* dw, float* db,
               const Workspace& ws, cudaStream_t st);
// small-Kd variant (C*kh*kw + 1 <= 96, K <= 32: first layers), mma.sync TF32,
// one CTA per image, same partial layout and fixed-order reduce
bool wgrad_small_ok(const ConvDesc& d, const GradSrc& gs);
size_t wgrad_small_workspace(const ConvDesc& d);
int conv_wgrad_small(const ConvDesc& d, const float* x, const GradSrc& gs, float* dw, float* db,
                     const Workspace& ws, cudaStream_t st, ImageSumFold* defer = nullptr);
}  // namespace direct

// ---- single-output-map convolutions (k1.cu, K = 1, exact fp32, any precision) ----
namespace k1 {
bool fwd_ok(const ConvDesc& d);
int conv_fwd(const ConvDesc& d, const float* x, const float* w, const float* bias, int act,
             float* y, cudaStream_t st);
bool wgrad_ok(const ConvDesc& d);
size_t wgrad_workspace(const ConvDesc& d);
int conv_wgrad(const ConvDesc& d, const float* x, const float* gpre, float* dw, float* db,
               const Workspace& ws, cudaStream_t st);
}  // namespace k1

// ---- tcgen05 implementations (tc.cu) for VCNN_PREC_TF32 / 3XTF32 ----
namespace tc {
// Slab kernels (TF32, stride 1): the CTA stages its input window in shared
// memory once (cp.async), gathers the implicit-GEMM operands from there.
// *_ok() says whether a geometry fits (else use the generic kernels below).
// They read PREPARED weights (prep_weights: tf32-rounded, wf = [K][kd4]
// zero-padded for the forward, wt = [C][K*kh*kw] transposed for dgrad).
bool slab_fwd_ok(const ConvDesc& d, int pool);
bool slab_wgrad_ok(const ConvDesc& d, int pool = 0, int POH = 0, int POW = 0);
bool slab_dgrad_ok(const ConvDesc& d, int pool = 0, int POW = 0);
size_t slab_wgrad_workspace(const ConvDesc& d);
size_t prep_floats_f(const ConvDesc& d);
size_t prep_floats_t(const ConvDesc& d);
int prep_weights(const ConvDesc& d, const float* w, float* wf, float* wt, cudaStream_t st);
// y (nullable when pf.pool) = act(conv(x) + b); pf: fused max pool
int slab_conv_fwd(const ConvDesc& d, const float* x, const float* wf, const float* b, int act,
                  float* y, const PoolFuse& pf, cudaStream_t st);
int slab_conv_wgrad(const ConvDesc& d, const float* x, const GradSrc& gs, float* dw, float* db,
                    const Workspace& ws, cudaStream_t st);
int slab_conv_dgrad(const ConvDesc& d, const GradSrc& gs, const float* wt, float* dx,
                    const float* yprev, int act_prev, cudaStream_t st);
int conv_fwd(const ConvDesc& d, const float* x, const float* w, const float* b, int act,
             float* y, bool split3, const Workspace& ws, cudaStream_t st);
int conv_wgrad(const ConvDesc& d, const float* x, const float* gpre, float* dw, float* db,
               bool split3, const Workspace& ws, cudaStream_t st);
int conv_dgrad(const ConvDesc& d, const float* gpre, const float* w, float* dx,
               const float* yprev, int act_prev, bool split3, const Workspace& ws,
               cudaStream_t st);
int full_fwd(int B, int in, int out, const float* x, const float* w, const float* b, int act,
             float* y, bool split3, const Workspace& ws, cudaStream_t st);
int full_wgrad(int B, int in, int out, const float* x, const float* gpre, float* dw, float* db,
               bool split3, const Workspace& ws, cudaStream_t st);
int full_dgrad(int B, int in, int out, const float* gpre, const float* w, float* dx,
               const float* yprev, int act_prev, bool split3, const Workspace& ws,
               cudaStream_t st);
int matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c,
           bool transB, bool split3, const Workspace& ws, cudaStream_t st);
int gemm(int64_t m, int64_t n, int64_t k, const float* a, int64_t as_m, int64_t as_k,
         const float* b, int64_t bs_k, int64_t bs_n, float* c, int64_t ldc, const float* bias,
         int act, bool split3, const Workspace& ws, cudaStream_t st);
// scratch the launchers above need (split-K partials, explicit-dgrad dP)
size_t conv_workspace(const ConvDesc& d);
size_t full_workspace(int B, int in, int out);
size_t matmul_workspace(int64_t m, int64_t k, int64_t n);
}  // namespace tc

}  // namespace vcnn_b200
