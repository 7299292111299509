// engine.cu -- the device-resident network engine behind the net-level C ABI:
// build_network + Executor<float>(imp6).run_batch + sgd_step
// (network.hpp:102-130, variants.hpp:353-376 / 484-668, network.hpp:242-273).
//
// Layout in HBM (one net):
//   params | grads | velocity : three flat fp32 buffers in NetGrads order
//                               (per layer: weights row-major, then bias), so
//                               SGD is ONE kernel and a data-parallel
//                               all-reduce is ONE collective over `grads`;
//   per layer: out  [B][C][H][W] post-activation (the forward trace; also the
//                                 activation-derivative source in backward),
//              gpre [B][C][H][W] gradient w.r.t. the PRE-activation,
//              arg  [B][C][OH][OW] int32 global argmax (max pools);
//   input slots x / cls / values sized for max_batch.
// Backward writes gpre of layer i-1 directly from layer i's dgrad / pool
// backward / FC dgrad epilogue (act' fused), so there are no standalone
// activation passes.  A whole train step can be captured once into a CUDA
// graph and replayed.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"

using namespace vcnn_b200;

namespace {

struct LayerRt {
  vcnn_layer_spec spec;
  int in_h, in_w, in_c;
  int out_h, out_w, out_c;
  int64_t w_off = 0, w_len = 0, b_off = 0, b_len = 0;
  int64_t in_per = 0, out_per = 0;
  float* out = nullptr;
  float* gpre = nullptr;
  int32_t* arg = nullptr;
  // conv: tf32-rounded weight copies for the slab kernels (prep_weights),
  // refreshed after every parameter update
  float* wf = nullptr;
  float* wt = nullptr;
  // direct (shifted-view) kernels: prepacked tf32 weights, fwd and dgrad
  float* pf = nullptr;
  float* pd = nullptr;
  float* ps = nullptr;  // small-Kd forward weight image (tf32, padded)
  // tensor-TMA input path: a pool output also kept as tf32 NHWC (written by
  // the producing fused conv+pool kernel; `nhwc_fresh` = written this step),
  // and the consuming conv's tensor map over it
  float* nhwc = nullptr;
  bool nhwc_fresh = false;
  bool has_tmap = false;
  alignas(64) unsigned char tmap[128] = {};
};

// host Rng identical to the reference (common.hpp:51-66): mt19937_64 with
// uniform = (u64 >> 11) * 2^-53
struct HostRng {
  uint64_t mt[312];
  int idx;
  explicit HostRng(uint64_t seed) {
    mt[0] = seed;
    for (int i = 1; i < 312; ++i)
      mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    idx = 312;
  }
  uint64_t next() {
    if (idx >= 312) {
      for (int i = 0; i < 312; ++i) {
        uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
        uint64_t y = x >> 1;
        if (x & 1ULL) y ^= 0xB5026F5AA96619E9ULL;
        mt[i] = mt[(i + 156) % 312] ^ y;
      }
      idx = 0;
    }
    uint64_t x = mt[idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
  // fused like the reference build (gnu++20 contracts lo + (hi-lo)*u to an FMA)
  double uniform(double lo, double hi) { return std::fma(hi - lo, uniform(), lo); }
};

enum Comp { CONV_F = 0, CONV_B, POOL_F, POOL_B, FULL_F, FULL_B, OTHER_F, OTHER_B };

}  // namespace

struct vcnn_net {
  std::vector<vcnn_layer_spec> specs;
  vcnn_net_spec spec{};
  std::vector<LayerRt> L;
  int max_batch = 0;
  int precision = VCNN_PREC_TF32;
  int pool_bwd_mode = VCNN_POOLBWD_EXACT;
  // fast path: slab kernels + conv->max-pool fusion (TF32); keep_trace forces
  // every layer output / pre-activation gradient to be materialised
  bool fuse = true;
  bool keep_trace = false;
  int64_t nparams = 0;
  float* params = nullptr;
  float* grads = nullptr;
  float* vel = nullptr;
  float* x = nullptr;
  int* cls = nullptr;
  float* values = nullptr;
  int64_t in_per = 0, out_units = 0;
  float* loss = nullptr;
  int* err = nullptr;
  Workspace ws;
  // backward runs weight gradients on a side stream, concurrently with the
  // data-gradient chain (separate split-K workspace); per-layer fork events
  // and one join event.  Captured into the graph as parallel branches.
  cudaStream_t side = nullptr;
  Workspace ws2;
  std::vector<cudaEvent_t> fork_ev;
  cudaEvent_t join_ev = nullptr;
  cudaStream_t stream = nullptr;
  // graph replay
  bool use_graph = false;
  // instantiated step graphs, one per (batch, lr, momentum) in use (a
  // training epoch alternates full batches and one smaller last batch)
  struct GraphEntry {
    int batch;
    float lr, mom;
    const DpLink* dp;
    int dpv;
    const void* ring;  // the batch ring the graph stages from (null: none)
    int steps;         // training steps captured back to back in the graph
    cudaGraphExec_t exec;
    int kernels;
  };
  std::vector<GraphEntry> graphs;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap_stream = nullptr;  // capture needs a non-legacy stream
  // host-stream training (vcnn_net_train_host_stream): two device staging
  // slots filled by a copy stream while the previous step computes
  static constexpr int kSlots = 3;  // host-stream staging slots (H2D gets two step times)
  static constexpr int kLossRing = 4096;  // host-stream device loss history (power of 2)
  struct Pipe {
    cudaStream_t cp = nullptr;
    cudaStream_t rd = nullptr;  // loss read-back (its own stream: it waits for each step)
    cudaEvent_t start = nullptr, copied[kSlots] = {}, consumed[kSlots] = {};
    cudaEvent_t stored = nullptr;  // a step's loss is in the device ring
    float* xs[kSlots] = {};
    int* cs[kSlots] = {};
    float* vs[kSlots] = {};
    float* hl = nullptr;  // pinned per-step losses (a pageable D2H would block the host)
    float* dl = nullptr;  // device per-step losses (one store kernel per step, one D2H per call)
    int* cur = nullptr;   // the staging ring's own cursor (the caller's ring keeps its place)
    int hl_cap = 0;
  } pipe;
  int g_batch = -1;
  float g_lr = 0, g_mom = 0;
  const DpLink* g_dp = nullptr;
  int g_dpv = 0;
  const void* g_ring = nullptr;
  int g_steps = 1;
  int cap_steps = 1;  // steps in the graph being captured (1 when eager)
  int kernels_per_step = 0;
  bool guard = false;  // Trainer non-finite stop armed (err[2..3] on the device)
  DpLink* dp = nullptr;  // attached data-parallel group (vcnn_dp_*), or none
  // train steps: layer 0's small-Kd weight gradient stays as per-image
  // partials which the update sums itself (one launch less on the critical
  // path); forward_backward alone reduces as usual
  bool defer_fold = false;
  direct::ImageSumFold fold{};
  // the two-layer tail in batch slices (mlp_head_slices): per-slice dW / db
  // partials [kMaxSlices][per] (folded into the update like layer 0's, or
  // summed by a reduce launch), loss partials + ticket (tail_aux[0..kMaxSlices),
  // [kMaxSlices])
  float* tail_part = nullptr;
  float* tail_aux = nullptr;
  // device batch ring (vcnn_net_set_batch_ring): staged by the step itself
  struct Ring {
    const float* x = nullptr;
    const void* t = nullptr;
    int nbatch = 0, batch = 0;
    int64_t xs = 0, ts = 0;
    int* cursor = nullptr;  // [slot, blocks done, steps]
    float* lhist = nullptr;  // (host stream) per-step loss history, or none
  } ring;
  direct::ImageSumFold fold2{};
  int64_t fold2_off = 0;
  // breakdown timer
  bool breakdown = false;
  struct MarkRec {
    int comp, layer, op;
    cudaEvent_t a, b;
  };
  std::vector<MarkRec> marks;
  // per (layer, op) accumulated seconds and launches; op: 0 fwd, 1 wgrad,
  // 2 dgrad, 3 loss, 4 sgd
  std::vector<double> op_sec;
  std::vector<int64_t> op_cnt;
  std::vector<cudaEvent_t> event_pool;
  size_t event_next = 0;
  double seconds[8] = {0};
};

namespace {

#define TRY(expr)      \
  do {                 \
    int _s = (expr);   \
    if (_s) return _s; \
  } while (0)

ConvDesc conv_of(const LayerRt& l, int B) {
  ConvDesc d;
  d.B = B;
  d.C = l.in_c;
  d.H = l.in_h;
  d.W = l.in_w;
  d.K = l.spec.units;
  d.kh = l.spec.kh;
  d.kw = l.spec.kw;
  d.s = l.spec.stride;
  d.OH = l.out_h;
  d.OW = l.out_w;
  return d;
}

PoolDesc pool_of(const LayerRt& l, int B) {
  PoolDesc d;
  d.B = B;
  d.C = l.in_c;
  d.H = l.in_h;
  d.W = l.in_w;
  d.ph = l.spec.kh;
  d.pw = l.spec.kw;
  d.s = l.spec.stride;
  d.mode = l.spec.pool_mode;
  d.OH = l.out_h;
  d.OW = l.out_w;
  return d;
}

// -------- breakdown marks (eager mode only) --------
cudaEvent_t next_event(vcnn_net* n) {
  if (n->event_next == n->event_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    n->event_pool.push_back(e);
  }
  return n->event_pool[n->event_next++];
}

enum OpKind { OP_FWD = 0, OP_WGRAD = 1, OP_DGRAD = 2, OP_LOSS = 3, OP_SGD = 4, OP_KINDS = 5 };

// CUDA-event bracket around one op on the net's stream (breakdown mode)
struct Mark {
  vcnn_net* n;
  int comp, layer, op;
  cudaEvent_t a = nullptr;
  Mark(vcnn_net* net, int c, int l = -1, int o = OP_FWD) : n(net), comp(c), layer(l), op(o) {
    if (n->breakdown) {
      a = next_event(n);
      cudaEventRecord(a, n->stream);
    }
  }
  ~Mark() {
    if (n->breakdown) {
      cudaEvent_t b = next_event(n);
      cudaEventRecord(b, n->stream);
      n->marks.push_back({comp, layer, op, a, b});
    }
  }
};

// a conv layer whose whole output is one patch (OH = OW = 1, the kernel
// covers the input) is a fully connected layer over the flattened input:
// im2col rows (c,ky,kx) == the (c,y,x) flatten order (layers.hpp:224-228)
bool conv_is_dense(const LayerRt& l) {
  return l.spec.kind == VCNN_LAYER_CONV && l.out_h == 1 && l.out_w == 1 &&
         l.spec.kh == l.in_h && l.spec.kw == l.in_w;
}


// conv layer i followed by a max pool that its forward epilogue can compute
// (non-overlapping windows, no pool bias, identity act, exact backward), with
// a backward that can route the pool gradient on the fly
int fused_pool_of(const vcnn_net* n, size_t i, int B) {
  if (!n->fuse || n->keep_trace || n->precision != VCNN_PREC_TF32 ||
      n->pool_bwd_mode != VCNN_POOLBWD_EXACT)
    return 0;
  if (i + 1 >= n->L.size()) return 0;
  const LayerRt& l = n->L[i];
  const LayerRt& p = n->L[i + 1];
  if (l.spec.kind != VCNN_LAYER_CONV || conv_is_dense(l)) return 0;
  if (p.spec.kind != VCNN_LAYER_POOL || p.spec.pool_mode != VCNN_POOL_MAX || p.b_len ||
      p.spec.act != VCNN_ACT_IDENTITY || p.spec.kh != p.spec.kw || p.spec.kh != p.spec.stride ||
      p.spec.kh < 1)
    return 0;
  if (i + 2 >= n->L.size()) return 0;  // the layer above applies the conv act' for the pool
  const ConvDesc d = conv_of(l, B);
  const int pz = p.spec.kh;
  // the small-Kd kernel serves a layer's trace path and its fused path alike
  // (same accumulation -> bit-identical), or neither
  if (direct::small_fwd_ok(d, 0) != direct::small_fwd_ok(d, pz)) return 0;
  const bool fwd = direct::small_fwd_ok(d, pz) || (l.pf && direct::fwd_ok(d, pz)) ||
                   tc::slab_fwd_ok(d, pz);
  const bool dg = i == 0 || (l.pd && direct::dgrad_ok(d, pz, p.out_h, p.out_w)) ||
                  tc::slab_dgrad_ok(d, pz, p.out_w);
  if (!fwd || !dg || !tc::slab_wgrad_ok(d, pz, p.out_h, p.out_w)) return 0;
  return pz;
}

constexpr int kTmaSlabMinBatch = 256;

int conv_forward(vcnn_net* n, size_t i, int B, const float* in, int fpool) {
  const cudaStream_t st = n->stream;
  LayerRt& l = n->L[i];
  const float* W = n->params + l.w_off;
  const float* b = n->params + l.b_off;
  const ConvDesc d = conv_of(l, B);
  if (conv_is_dense(l))
    return launch_full_fwd(B, (int)l.in_per, l.spec.units, in, W, b, l.spec.act, l.out,
                           n->precision, n->ws, st);
  if (!fpool && k1::fwd_ok(d))  // K = 1: exact fp32 direct conv (N = 1 GEMM)
    return k1::conv_fwd(d, in, W, b, l.spec.act, l.out, st);
  // the input as a tf32 NHWC copy written this step by the producer: the
  // direct kernel stages its slab with one tensor TMA
  const void* map = (i >= 1 && l.has_tmap && n->L[i - 1].nhwc_fresh) ? l.tmap : nullptr;
  if (fpool) {
    LayerRt& p = n->L[i + 1];
    PoolFuse pf;
    pf.pool = fpool;
    pf.POH = p.out_h;
    pf.POW = p.out_w;
    pf.y = p.out;
    pf.arg = p.arg;
    if (direct::small_fwd_ok(d, fpool)) {
      // the extra NHWC write pays for itself (the consumer skips its slab
      // build) from a few hundred images up: measured at CIFAR-3 b128 -4%,
      // b1024 +4% img/s
      if (B >= kTmaSlabMinBatch) {
        pf.y_nhwc = p.nhwc;
        p.nhwc_fresh = p.nhwc != nullptr;
      }
      return direct::conv_fwd_small(d, in, W, b, l.spec.act, nullptr, pf, st, l.ps);
    }
    if (l.pf && direct::fwd_ok(d, fpool))
      return direct::conv_fwd(d, in, l.pf, b, l.spec.act, nullptr, pf, st, map);
    return tc::slab_conv_fwd(d, in, l.wf, b, l.spec.act, nullptr, pf, st);
  }
  if (n->precision == VCNN_PREC_TF32 && direct::small_fwd_ok(d, 0))
    return direct::conv_fwd_small(d, in, W, b, l.spec.act, l.out, PoolFuse{}, st, l.ps);
  if (n->precision == VCNN_PREC_TF32 && l.pf && direct::fwd_ok(d, 0))
    return direct::conv_fwd(d, in, l.pf, b, l.spec.act, l.out, PoolFuse{}, st, map);
  return launch_conv_fwd(d, in, W, b, l.spec.act, l.out, n->precision, n->ws, st, l.wf);
}

// How many top layers run fused with the loss in training steps: 2 when the
// last two are small full layers (or a dense conv under a full layer;
// launch_mlp_head), 1 when the last is a small full layer (launch_head),
// else 0 (separate forward / loss / backward kernels).
int tail_fused(const vcnn_net* n, int B) {
  // profiling (trace + breakdown, e.g. Executor::set_timer): every layer in
  // its own kernels, so the components separate as in the reference
  if (n->keep_trace && n->breakdown) return 0;
  const size_t nl = n->L.size();
  const LayerRt& l = n->L.back();
  if (l.spec.kind != VCNN_LAYER_FULL) return 0;
  if (nl >= 2 && n->precision == VCNN_PREC_TF32) {  // its GEMMs run in TF32
    const LayerRt& hl = n->L[nl - 2];
    if ((hl.spec.kind == VCNN_LAYER_FULL || conv_is_dense(hl)) &&
        mlp_head_fusable(B, (int)hl.in_per, hl.spec.units, l.spec.units))
      return 2;
  }
  return head_fusable(B, (int)l.in_per, l.spec.units) ? 1 : 0;
}

int run_forward(vcnn_net* n, int B, int skip_top = 0) {
  const cudaStream_t st = n->stream;
  for (LayerRt& l : n->L) l.nhwc_fresh = false;
  const size_t nl = n->L.size() - (size_t)skip_top;
  for (size_t i = 0; i < nl; ++i) {
    LayerRt& l = n->L[i];
    const float* in = i == 0 ? n->x : n->L[i - 1].out;
    const float* W = n->params + l.w_off;
    const float* b = n->params + l.b_off;
    if (l.spec.kind == VCNN_LAYER_CONV) {
      const int fpool = fused_pool_of(n, i, B);
      Mark m(n, CONV_F, (int)i, OP_FWD);
      TRY(conv_forward(n, i, B, in, fpool));
      if (fpool) ++i;  // the pool layer ran in the conv epilogue
    } else if (l.spec.kind == VCNN_LAYER_POOL) {
      Mark m(n, POOL_F, (int)i, OP_FWD);
      PoolDesc d = pool_of(l, B);
      TRY(launch_pool_fwd<int32_t>(d, in, l.b_len ? b : nullptr, l.spec.act, l.out,
                                   d.mode == VCNN_POOL_MAX ? l.arg : nullptr, st));
    } else {
      Mark m(n, FULL_F, (int)i, OP_FWD);
      TRY(launch_full_fwd(B, (int)l.in_per, l.spec.units, in, W, b, l.spec.act, l.out,
                          n->precision, n->ws, st));
    }
  }
  return VCNN_OK;
}

int run_backward(vcnn_net* n, int B, int tail = 0) {
  const cudaStream_t st = n->stream;
  LayerRt& last = n->L.back();
  const int nl = (int)n->L.size();
  if (tail == 2) {  // last two layers fwd + loss + their backward, one kernel
    Mark m(n, OTHER_F, nl - 1, OP_LOSS);
    LayerRt& hl = n->L[nl - 2];
    const LayerRt* prev = nl > 2 ? &n->L[nl - 3] : nullptr;
    int act_prev = prev ? prev->spec.act : VCNN_ACT_IDENTITY;
    if (nl > 3 && fused_pool_of(n, (size_t)(nl - 4), B)) act_prev = n->L[nl - 4].spec.act;
    const int hin = (int)hl.in_per, hh = hl.spec.units, ho = last.spec.units;
    const int ncl = n->tail_part ? mlp_head_slices(B, hin, hh, ho) : 1;
    TRY(launch_mlp_head(B, hin, hh, ho, prev ? prev->out : n->x, n->params + hl.w_off,
                        n->params + hl.b_off, hl.spec.act, n->params + last.w_off,
                        n->params + last.b_off, last.spec.act, hl.out, last.out, n->spec.loss,
                        n->cls, n->values, n->loss, n->err, hl.gpre, last.gpre,
                        n->grads + hl.w_off, n->grads + hl.b_off, n->grads + last.w_off,
                        n->grads + last.b_off, prev ? prev->gpre : nullptr, act_prev, st, ncl,
                        n->tail_part, n->tail_aux, reinterpret_cast<unsigned*>(n->tail_aux + kMaxSlices)));
    if (ncl > 1) {  // the slices' dW / db: summed in slice order by the update, or here
      const int64_t per = (int64_t)hh * hin + hh + (int64_t)ho * hh + ho;
      if (n->defer_fold) {
        n->fold2 = direct::ImageSumFold{n->tail_part, ncl, per, per};
        n->fold2_off = hl.w_off;
      } else {
        TRY(direct::sum_partials(ncl, per, per, n->tail_part, n->grads + hl.w_off, st));
      }
    }
  } else if (tail == 1) {  // last full layer fwd + loss + its backward, one kernel
    Mark m(n, OTHER_F, nl - 1, OP_LOSS);
    const LayerRt* prev = nl > 1 ? &n->L[nl - 2] : nullptr;
    int act_prev = prev ? prev->spec.act : VCNN_ACT_IDENTITY;
    // below a pool fused into its conv: hand down dP * conv_act'(pooled)
    if (nl > 2 && fused_pool_of(n, (size_t)(nl - 3), B)) act_prev = n->L[nl - 3].spec.act;
    TRY(launch_head(B, (int)last.in_per, last.spec.units, prev ? prev->out : n->x,
                    n->params + last.w_off, n->params + last.b_off, last.spec.act, last.out,
                    n->spec.loss, n->cls, n->values, n->loss, last.gpre, n->grads + last.w_off,
                    n->grads + last.b_off, prev ? prev->gpre : nullptr, act_prev, n->err,
                    st));
  } else {
    Mark m(n, OTHER_F, nl - 1, OP_LOSS);
    TRY(launch_loss(n->spec.loss, B, (int)n->out_units, last.out, n->cls, n->values, n->loss,
                    last.gpre, last.spec.act, n->err, st, n->loss + 4));
  }
  // weight gradients on the side stream (not in breakdown mode, whose
  // per-op events live on the main stream)
  static const bool no_side = getenv("VCNN_NO_SIDE") != nullptr;  // A/B experiments
  const bool par = n->side && !n->breakdown && !no_side;
  const cudaStream_t sws = par ? n->side : st;
  const Workspace& wss = par ? n->ws2 : n->ws;
  static const bool l0_side = getenv("VCNN_L0_SIDE") != nullptr;  // A/B experiments
  bool forked = false;  // the side stream took work (and must be joined)
  for (int i = nl - 1 - (tail ? tail : 0); i >= 0; --i) {
    LayerRt& l = n->L[i];
    // layer 0 has no data gradient: its weight gradient runs on the main
    // stream right after layer 1's data gradient (and its own workspace),
    // not queued behind the side stream's weight gradients above it.  Only
    // in one-step graphs / eager steps: inside a multi-step graph the
    // side-stream placement measured faster (83.4 vs 85.8 us per CIFAR-3
    // b128 step; one-step graphs 84.9 vs 86.1, scripts/dbg_l0.py)
    const bool l0m = par && i == 0 && !l0_side && n->cap_steps == 1;
    const cudaStream_t sw = l0m ? st : sws;
    const Workspace& wsw = l0m ? n->ws : wss;
    if (par && !l0m) {  // this layer's gradient inputs are ready on the main stream
      forked = true;
      VCNN_CUDA_TRY(cudaEventRecord(n->fork_ev[i], st));
      VCNN_CUDA_TRY(cudaStreamWaitEvent(n->side, n->fork_ev[i], 0));
    }
    const float* in = i == 0 ? n->x : n->L[i - 1].out;
    const float* yprev = i > 0 ? n->L[i - 1].out : nullptr;
    int act_prev = i > 0 ? n->L[i - 1].spec.act : VCNN_ACT_IDENTITY;
    // below is a pool fused into its conv: hand down dP * conv_act'(pooled)
    // (the pooled value is the conv output at the argmax), which the conv's
    // backward routes through the argmax
    if (i > 1 && fused_pool_of(n, (size_t)(i - 2), B)) act_prev = n->L[i - 2].spec.act;
    float* gprev = i > 0 ? n->L[i - 1].gpre : nullptr;
    const float* W = n->params + l.w_off;
    float* gW = n->grads + l.w_off;
    float* gB = n->grads + l.b_off;
    if (l.spec.kind == VCNN_LAYER_CONV) {
      ConvDesc d = conv_of(l, B);
      const int fpool = fused_pool_of(n, (size_t)i, B);
      GradSrc gs;
      if (fpool) {  // route the fused pool's gradient on the fly
        const LayerRt& p = n->L[i + 1];
        gs.dP = p.gpre;
        gs.parg = p.arg;
        gs.pool = fpool;
        gs.POH = p.out_h;
        gs.POW = p.out_w;
      } else {
        gs.g = l.gpre;
      }
      const bool dense = conv_is_dense(l);
      {
        Mark m(n, CONV_B, i, OP_WGRAD);
        if (dense)
          TRY(launch_full_wgrad(B, (int)l.in_per, l.spec.units, in, l.gpre, gW, gB, n->precision,
                                wsw, sw));
        else if (!fpool && k1::wgrad_ok(d) && wsw.bytes >= k1::wgrad_workspace(d))
          TRY(k1::conv_wgrad(d, in, l.gpre, gW, gB, wsw, sw));
        else if (n->precision == VCNN_PREC_TF32 && direct::wgrad_small_ok(d, gs) &&
                 wsw.bytes >= direct::wgrad_small_workspace(d))
          TRY(direct::conv_wgrad_small(d, in, gs, gW, gB, wsw, sw,
                                       i == 0 && n->defer_fold ? &n->fold : nullptr));
        else if (n->precision == VCNN_PREC_TF32 && direct::wgrad_ok(d, gs) &&
                 wsw.bytes >= direct::wgrad_workspace(d))
          TRY(direct::conv_wgrad(d, in, gs, gW, gB, wsw, sw));
        else if (!fpool && n->precision == VCNN_PREC_TF32 && direct::wgrad1d_ok(d) &&
                 wsw.bytes >= direct::wgrad1d_workspace(d))
          TRY(direct::conv_wgrad1d(d, in, l.gpre, gW, gB, wsw, sw));
        else if (fpool)
          TRY(tc::slab_conv_wgrad(d, in, gs, gW, gB, wsw, sw));
        else
          TRY(launch_conv_wgrad(d, in, l.gpre, gW, gB, n->precision, wsw, sw));
      }
      if (gprev) {
        Mark m(n, CONV_B, i, OP_DGRAD);
        if (dense)
          TRY(launch_full_dgrad(B, (int)l.in_per, l.spec.units, l.gpre, W, gprev, yprev, act_prev,
                                n->precision, n->ws, st));
        else if (n->precision == VCNN_PREC_TF32 && l.pd &&
                 direct::dgrad_ok(d, gs.pool, gs.POH, gs.POW))
          TRY(direct::conv_dgrad(d, gs, l.pd, gprev, yprev, act_prev, st));
        else if (fpool)
          TRY(tc::slab_conv_dgrad(d, gs, l.wt, gprev, yprev, act_prev, st));
        else
          TRY(launch_conv_dgrad(d, l.gpre, W, gprev, yprev, act_prev, n->precision, n->ws, st,
                                l.wt));
      }
    } else if (l.spec.kind == VCNN_LAYER_POOL) {
      // a pool fused into the conv below: its gradient is routed by that
      // conv's backward (no pool-backward kernel)
      if (i > 0 && fused_pool_of(n, (size_t)(i - 1), B)) continue;
      PoolDesc d = pool_of(l, B);
      if (l.b_len) {
        Mark m(n, POOL_B, i, OP_WGRAD);
        TRY(launch_pool_bias_grad(d, l.gpre, gB, sw));
      }
      if (gprev) {
        Mark m(n, POOL_B, i, OP_DGRAD);
        TRY(launch_pool_bwd<int32_t>(d, n->pool_bwd_mode, l.gpre, l.arg, gprev, yprev, act_prev,
                                     st));
      }
    } else {
      {
        Mark m(n, FULL_B, i, OP_WGRAD);
        TRY(launch_full_wgrad(B, (int)l.in_per, l.spec.units, in, l.gpre, gW, gB, n->precision,
                              wsw, sw));
      }
      if (gprev) {
        Mark m(n, FULL_B, i, OP_DGRAD);
        TRY(launch_full_dgrad(B, (int)l.in_per, l.spec.units, l.gpre, W, gprev, yprev, act_prev,
                              n->precision, n->ws, st));
      }
    }
  }
  if (forked) {  // join: the update (and any host read) sees every gradient
    VCNN_CUDA_TRY(cudaEventRecord(n->join_ev, n->side));
    VCNN_CUDA_TRY(cudaStreamWaitEvent(st, n->join_ev, 0));
  }
  return VCNN_OK;
}

// refresh the slab kernels' tf32 weight copies from params
int prep_weights(vcnn_net* n) {
  for (LayerRt& l : n->L) {
    const ConvDesc d = conv_of(l, 1);
    const float* w = n->params + l.w_off;
    if (l.wf) TRY(tc::prep_weights(d, w, l.wf, l.wt, n->stream));
    if (l.pf) TRY(direct::pack_weights(d, 0, w, l.pf, n->stream));
    if (l.pd) TRY(direct::pack_weights(d, 1, w, l.pd, n->stream));
    if (l.ps) TRY(direct::small_fwd_pack(d, w, l.ps, n->stream));
  }
  return VCNN_OK;
}

int run_sgd(vcnn_net* n, float lr, float mom, float scale, int* ring_step = nullptr) {
  Mark m(n, OTHER_B, -1, OP_SGD);
  // one launch: the update + the direct kernels' weight packs; only layers
  // on the slab fallback still need their plain tf32 copies refreshed
  // (the fused launch carries at most direct::kMaxPackLayers pack tables;
  // deeper nets repack the remaining layers from the updated params)
  std::vector<direct::PackSpec> packs;
  std::vector<const LayerRt*> repack;
  bool slab_copies = false;
  for (LayerRt& l : n->L) {
    if (l.pf || l.pd || l.ps) {
      if ((int)packs.size() < direct::kMaxPackLayers)
        packs.push_back({conv_of(l, 1), l.w_off, l.pf, l.pd, l.ps});
      else
        repack.push_back(&l);
    }
    slab_copies = slab_copies || l.wf;
  }
  DpLink* dp = n->dp;
  if (!dp || dp->world == 1) {
    TRY(direct::sgd_pack(n->nparams, n->params, n->vel, n->grads, lr, mom, scale, packs,
                         n->stream, n->loss, n->err + 2, n->fold.part ? &n->fold : nullptr,
                         n->L[0].w_off, n->fold2.part ? &n->fold2 : nullptr, n->fold2_off,
                         ring_step));
    n->fold = direct::ImageSumFold{};
    n->fold2 = direct::ImageSumFold{};
  } else if (dp->mode == VCNN_DP_P2P) {
    // one kernel: rank-ordered sum of every replica's gradient (peers over
    // NVLink) + SGD + packs
    TRY(direct::dp_sgd_pack(n->nparams, n->params, n->vel, lr, mom, packs, dp->peers,
                            n->stream, ring_step));
  } else {
    // NCCL fallback: weight, all-reduce (sum) in place, replicated update
    if (!dp->equal) TRY(dp_scale(n->nparams, n->grads, dp->local_w, n->stream));
    TRY(dp->allreduce(dp, n->grads, n->nparams, n->stream));
    TRY(direct::sgd_pack(n->nparams, n->params, n->vel, n->grads, lr, mom,
                         dp->equal ? scale / (float)dp->world : scale, packs, n->stream, nullptr,
                         nullptr, nullptr, 0, nullptr, 0, ring_step));
  }
  for (const LayerRt* l : repack) {
    const ConvDesc d = conv_of(*l, 1);
    const float* w = n->params + l->w_off;
    if (l->pf) TRY(direct::pack_weights(d, 0, w, l->pf, n->stream));
    if (l->pd) TRY(direct::pack_weights(d, 1, w, l->pd, n->stream));
    if (l->ps) TRY(direct::small_fwd_pack(d, w, l->ps, n->stream));
  }
  if (!slab_copies) return VCNN_OK;
  for (LayerRt& l : n->L)
    if (l.wf) TRY(tc::prep_weights(conv_of(l, 1), n->params + l.w_off, l.wf, l.wt, n->stream));
  return VCNN_OK;
}

int check_batch(vcnn_net* n, int batch) {
  if (batch < 1 || batch > n->max_batch)
    return fail(VCNN_ESHAPE, "batch " + std::to_string(batch) + " outside [1," +
                                 std::to_string(n->max_batch) + "]");
  return VCNN_OK;
}

int check_cfg(float lr, float mom) {
  if (!(lr > 0)) return fail(VCNN_ECONFIG, "learning rate must be positive");
  if (mom < 0 || mom >= 1) return fail(VCNN_ECONFIG, "momentum must be in [0,1)");
  return VCNN_OK;
}

void drop_graph(vcnn_net* n) {
  for (auto& e : n->graphs) cudaGraphExecDestroy(e.exec);
  n->graphs.clear();
  n->gexec = nullptr;
  n->g_batch = -1;
}

int eager_step(vcnn_net* n, int batch, float lr, float mom) {
  const int64_t before = g_launches.load();
  struct PdlScope {  // breakdown mode: ops timed one at a time
    bool saved;
    explicit PdlScope(bool off) : saved(pdl_enabled()) {
      if (off) pdl_enabled() = false;
    }
    ~PdlScope() { pdl_enabled() = saved; }
  } pdl_scope(n->breakdown);
  const int tail = tail_fused(n, batch);
  if (n->ring.nbatch) {  // the ring's next batch into the input slots
    const bool ce = n->spec.loss == VCNN_LOSS_SOFTMAX_CE;
    TRY(launch_ring_stage(n->ring.x, n->x, n->in_per * batch, n->ring.xs, n->ring.t,
                          ce ? (void*)n->cls : (void*)n->values,
                          ce ? batch : n->out_units * batch, n->ring.ts, n->ring.nbatch,
                          n->ring.cursor, n->stream, n->loss, n->ring.lhist,
                          vcnn_net::kLossRing - 1));
  }
  TRY(run_forward(n, batch, tail));
  n->defer_fold = !n->dp || n->dp->world == 1;
  n->fold = direct::ImageSumFold{};
  n->fold2 = direct::ImageSumFold{};
  const int sb = run_backward(n, batch, tail);
  n->defer_fold = false;
  if (sb) return sb;
  TRY(run_sgd(n, lr, mom, 1.0f, n->ring.nbatch ? n->ring.cursor + 2 : nullptr));
  n->kernels_per_step = (int)(g_launches.load() - before);
  return VCNN_OK;
}

// k training steps in ONE graph launch (k > 1: captured back to back -- each
// stages its own batch when a ring is attached -- so consecutive steps are
// not separated by a graph launch)
int train_steps_graph(vcnn_net* n, int k, int batch, float lr, float mom);

int train_step(vcnn_net* n, int batch, float lr, float mom) { return train_steps_graph(n, 1, batch, lr, mom); }

int train_steps_graph(vcnn_net* n, int k, int batch, float lr, float mom) {
  TRY(check_batch(n, batch));
  TRY(check_cfg(lr, mom));
  if (!n->use_graph || n->breakdown) {
    for (int i = 0; i < k; ++i) TRY(eager_step(n, batch, lr, mom));
    return VCNN_OK;
  }
  const int dpv = n->dp ? n->dp->version : 0;
  const void* ring = n->ring.nbatch ? (const void*)n->ring.x : nullptr;
  if (!n->gexec || n->g_batch != batch || n->g_lr != lr || n->g_mom != mom ||
      n->g_dp != n->dp || n->g_dpv != dpv || n->g_ring != ring || n->g_steps != k) {
    n->gexec = nullptr;
    for (auto& e : n->graphs)
      if (e.batch == batch && e.lr == lr && e.mom == mom && e.dp == n->dp &&
          e.dpv == (n->dp ? n->dp->version : 0) && e.ring == ring && e.steps == k) {
        n->gexec = e.exec;
        n->kernels_per_step = e.kernels;
      }
  }
  if (n->gexec) {
    n->g_batch = batch;
    n->g_lr = lr;
    n->g_mom = mom;
    n->g_dp = n->dp;
    n->g_dpv = dpv;
    n->g_ring = ring;
    n->g_steps = k;
  } else {
    if (n->graphs.size() >= 4) drop_graph(n);
    if (!n->cap_stream)
      VCNN_CUDA_TRY(cudaStreamCreateWithFlags(&n->cap_stream, cudaStreamNonBlocking));
    // capture on a private stream (the caller's may be the legacy default
    // stream, which cannot be captured); the graph is launched on the caller's
    cudaGraph_t g = nullptr;
    cudaStream_t user = n->stream;
    VCNN_CUDA_TRY(cudaStreamSynchronize(user));
    VCNN_CUDA_TRY(cudaStreamBeginCapture(n->cap_stream, cudaStreamCaptureModeRelaxed));
    n->stream = n->cap_stream;
    int s = VCNN_OK;
    n->cap_steps = k;
    for (int i = 0; i < k && !s; ++i) s = eager_step(n, batch, lr, mom);
    n->cap_steps = 1;
    n->stream = user;
    cudaError_t e = cudaStreamEndCapture(n->cap_stream, &g);
    if (s) {
      if (g) cudaGraphDestroy(g);
      return s;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&n->gexec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    n->graphs.push_back(
        vcnn_net::GraphEntry{batch, lr, mom, n->dp, dpv, ring, k, n->gexec, n->kernels_per_step});
    n->g_batch = batch;
    n->g_lr = lr;
    n->g_mom = mom;
    n->g_dp = n->dp;
    n->g_dpv = dpv;
    n->g_ring = ring;
    n->g_steps = k;
  }
  VCNN_CUDA_TRY(cudaGraphLaunch(n->gexec, n->stream));
  g_launches.fetch_add((int64_t)n->kernels_per_step * k);
  return VCNN_OK;
}

int copy_out(vcnn_net* n, void* host, const void* dev, size_t bytes) {
  VCNN_CUDA_TRY(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, n->stream));
  VCNN_CUDA_TRY(cudaStreamSynchronize(n->stream));
  return VCNN_OK;
}

int copy_in(vcnn_net* n, void* dev, const void* host, size_t bytes) {
  VCNN_CUDA_TRY(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, n->stream));
  VCNN_CUDA_TRY(cudaStreamSynchronize(n->stream));
  return VCNN_OK;
}

// the device guard word pair {armed, tripped} read by sgd_pack (stream-ordered)
int write_guard(vcnn_net* n, int armed) {
  VCNN_CUDA_TRY(cudaMemsetAsync(n->err + 2, 0, 2 * sizeof(int), n->stream));
  if (armed) VCNN_CUDA_TRY(cudaMemsetAsync(n->err + 2, 0x01, 1, n->stream));
  return VCNN_OK;
}

int check_errflag(vcnn_net* n) {
  int h = 0;
  TRY(copy_out(n, &h, n->err, sizeof(int)));
  if (h) {
    cudaMemsetAsync(n->err, 0, sizeof(int), n->stream);
    return fail(VCNN_EBOUNDS, "loss: class index out of range [0," +
                                  std::to_string(n->out_units) + ")");
  }
  return VCNN_OK;
}

}  // namespace

namespace vcnn_b200 {
int engine_attach_dp(vcnn_net* n, DpLink* link) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  drop_graph(n);
  n->dp = link;
  return VCNN_OK;
}
cudaStream_t engine_stream(vcnn_net* n) { return n ? n->stream : nullptr; }
}  // namespace vcnn_b200

extern "C" {

// NetworkSpec::chain (network.hpp:45-67)
int vcnn_net_spec_chain(const vcnn_net_spec* spec, int* shapes) {
  if (!spec) return fail(VCNN_ESHAPE, "null spec");
  int h = spec->in_h, w = spec->in_w, c = spec->in_c;
  if (h < 1 || w < 1 || c < 1) return fail(VCNN_ESHAPE, "shape extent must be >= 1");
  if (spec->loss != VCNN_LOSS_SOFTMAX_CE && spec->loss != VCNN_LOSS_MSE)
    return fail(VCNN_ECONFIG, "unknown loss kind");
  for (int i = 0; i < spec->nlayers; ++i) {
    const vcnn_layer_spec& l = spec->layers[i];
    const std::string pre = "layer " + std::to_string(i) + ": ";
    if (l.act < VCNN_ACT_IDENTITY || l.act > VCNN_ACT_TANH)
      return fail(VCNN_ECONFIG, pre + "unknown activation");
    if (l.kind == VCNN_LAYER_CONV) {
      vcnn_conv_geometry g;
      if (vcnn_conv_geometry_init(&g, h, w, c, 1, l.kh, l.kw, l.stride))
        return fail(VCNN_ESHAPE, pre + last_error());
      if (l.units < 1) return fail(VCNN_ESHAPE, pre + "shape extent must be >= 1");
      h = g.out_h;
      w = g.out_w;
      c = l.units;
    } else if (l.kind == VCNN_LAYER_POOL) {
      vcnn_pool_geometry g;
      if (vcnn_pool_geometry_init(&g, h, w, c, 1, l.kh, l.kw, l.stride, l.pool_mode))
        return fail(VCNN_ESHAPE, pre + last_error());
      h = g.out_h;
      w = g.out_w;
    } else if (l.kind == VCNN_LAYER_FULL) {
      if (l.units < 1) return fail(VCNN_ESHAPE, pre + "full layer needs units >= 1");
      h = 1;
      w = 1;
      c = l.units;
    } else {
      return fail(VCNN_ECONFIG, pre + "unknown layer kind");
    }
    if (shapes) {
      shapes[3 * i] = h;
      shapes[3 * i + 1] = w;
      shapes[3 * i + 2] = c;
    }
  }
  return VCNN_OK;
}

// the reference bench's synthetic batch (bench.cpp:29-45): one Rng(seed)
// stream, X ~ U[0,1) in NCHW linear order, then per-sample labels
// uniform_int(units) (common.hpp:63-66) or MSE targets ~ U[0,1); host only
int vcnn_synth_bench_data(const vcnn_net_spec* spec, int batch, uint64_t seed, float* x, int* cls,
                          float* values) {
  if (!spec || batch < 0 || !x) return fail(VCNN_ESHAPE, "synth_bench_data: bad arguments");
  std::vector<int> shapes(3 * (size_t)std::max(spec->nlayers, 1));
  TRY(vcnn_net_spec_chain(spec, shapes.data()));
  const int L = spec->nlayers;
  const int64_t units = L ? (int64_t)shapes[3 * (L - 1)] * shapes[3 * (L - 1) + 1] *
                                shapes[3 * (L - 1) + 2]
                          : (int64_t)spec->in_h * spec->in_w * spec->in_c;
  const bool ce = spec->loss == VCNN_LOSS_SOFTMAX_CE;
  if (ce ? !cls : !values) return fail(VCNN_ESHAPE, "synth_bench_data: null targets");
  HostRng rng(seed);
  const int64_t n = (int64_t)spec->in_h * spec->in_w * spec->in_c * batch;
  for (int64_t i = 0; i < n; ++i) x[i] = (float)rng.uniform();
  if (ce) {
    for (int b = 0; b < batch; ++b) {
      const int64_t k = (int64_t)(rng.uniform() * (double)units);
      cls[b] = (int)std::min(k, units - 1);
    }
  } else {
    for (int64_t i = 0; i < units * batch; ++i) values[i] = (float)rng.uniform();
  }
  return VCNN_OK;
}

int vcnn_net_create(const vcnn_net_spec* spec, int max_batch, int precision, vcnn_net** out) {
  if (!out) return fail(VCNN_ESHAPE, "null out");
  *out = nullptr;
  if (!spec || spec->nlayers < 1) return fail(VCNN_ESHAPE, "network needs at least one layer");
  if (max_batch < 1) return fail(VCNN_ESHAPE, "max_batch must be >= 1");
  if (precision < VCNN_PREC_TF32 || precision > VCNN_PREC_FP32)
    return fail(VCNN_ECONFIG, "unknown precision");
  std::vector<int> shapes(3 * spec->nlayers);
  TRY(vcnn_net_spec_chain(spec, shapes.data()));
  TRY(require_device());

  vcnn_net* n = new vcnn_net();
  n->specs.assign(spec->layers, spec->layers + spec->nlayers);
  n->spec = *spec;
  n->spec.layers = n->specs.data();
  n->max_batch = max_batch;
  n->precision = precision;
  n->in_per = (int64_t)spec->in_h * spec->in_w * spec->in_c;

  // parameter layout + host init (build_network, network.hpp:102-130)
  int h = spec->in_h, w = spec->in_w, c = spec->in_c;
  int64_t off = 0;
  for (int i = 0; i < spec->nlayers; ++i) {
    LayerRt l;
    l.spec = spec->layers[i];
    l.in_h = h;
    l.in_w = w;
    l.in_c = c;
    l.out_h = shapes[3 * i];
    l.out_w = shapes[3 * i + 1];
    l.out_c = shapes[3 * i + 2];
    l.in_per = (int64_t)h * w * c;
    l.out_per = (int64_t)l.out_h * l.out_w * l.out_c;
    if (l.spec.kind == VCNN_LAYER_CONV) {
      l.w_len = (int64_t)l.spec.units * l.spec.kh * l.spec.kw * c;
      l.b_len = l.spec.units;
    } else if (l.spec.kind == VCNN_LAYER_POOL) {
      l.b_len = l.spec.pool_bias ? c : 0;
    } else {
      l.w_len = (int64_t)l.spec.units * l.in_per;
      l.b_len = l.spec.units;
    }
    l.w_off = off;
    off += l.w_len;
    l.b_off = off;
    off += l.b_len;
    n->L.push_back(l);
    h = l.out_h;
    w = l.out_w;
    c = l.out_c;
  }
  n->nparams = off;
  n->out_units = n->L.back().out_per;

  std::vector<float> hp((size_t)(n->nparams > 0 ? n->nparams : 1), 0.f);
  {
    HostRng rng(spec->seed);  // one stream, layer order (layers.hpp:473-501)
    for (const LayerRt& l : n->L) {
      if (l.spec.kind == VCNN_LAYER_POOL) continue;
      double fan_in, fan_out;
      if (l.spec.kind == VCNN_LAYER_CONV) {
        fan_in = (double)l.spec.kh * l.spec.kw * l.in_c;
        fan_out = (double)l.spec.kh * l.spec.kw * l.spec.units;
      } else {
        fan_in = (double)l.in_per;
        fan_out = (double)l.spec.units;
      }
      const double a = std::sqrt(6.0 / (fan_in + fan_out));
      for (int64_t k = 0; k < l.w_len; ++k) hp[l.w_off + k] = (float)rng.uniform(-a, a);
    }
  }

  auto dalloc = [&](void** p, size_t bytes) -> int {
    VCNN_CUDA_TRY(cudaMalloc(p, bytes < 16 ? 16 : bytes));
    return VCNN_OK;
  };
  int s = VCNN_OK;
  const size_t pbytes = sizeof(float) * (size_t)(n->nparams > 0 ? n->nparams : 1);
  s = s ? s : dalloc((void**)&n->params, pbytes);
  s = s ? s : dalloc((void**)&n->grads, pbytes);
  s = s ? s : dalloc((void**)&n->vel, pbytes);
  s = s ? s : dalloc((void**)&n->x, sizeof(float) * n->in_per * max_batch);
  s = s ? s : dalloc((void**)&n->cls, sizeof(int) * max_batch);
  s = s ? s : dalloc((void**)&n->values, sizeof(float) * n->out_units * max_batch);
  s = s ? s : dalloc((void**)&n->loss, sizeof(float) * (4 + kLossWsFloats));
  s = s ? s : dalloc((void**)&n->err, sizeof(int) * 4);
  size_t wsb = 0;
  for (LayerRt& l : n->L) {
    const size_t ob = sizeof(float) * (size_t)(l.out_per * max_batch);
    s = s ? s : dalloc((void**)&l.out, ob);
    s = s ? s : dalloc((void**)&l.gpre, ob);
    if (l.spec.kind == VCNN_LAYER_POOL && l.spec.pool_mode == VCNN_POOL_MAX)
      s = s ? s : dalloc((void**)&l.arg, sizeof(int32_t) * (size_t)(l.out_per * max_batch));
    if (l.spec.kind == VCNN_LAYER_CONV && !conv_is_dense(l)) {
      // tf32 weight copies: the direct kernels' packs where the geometry
      // allows, else the slab kernels' plain copies
      const ConvDesc d1 = conv_of(l, 1);
      const size_t nf = direct::pack_floats(d1, 0);
      const bool first = &l == &n->L[0];  // layer 0 has no data gradient
      const size_t nd = first ? 0 : direct::pack_floats(d1, 1);
      if (nf) s = s ? s : dalloc((void**)&l.pf, sizeof(float) * nf);
      if (nd) s = s ? s : dalloc((void**)&l.pd, sizeof(float) * nd);
      // (the small-Kd kernels read the fp32 params directly)
      const bool small = direct::small_fwd_ok(d1, 0);
      const size_t ns = small ? direct::small_fwd_pack_floats(d1) : 0;
      if (ns) s = s ? s : dalloc((void**)&l.ps, sizeof(float) * ns);
      if ((!nf && !small) || (!first && !nd)) {
        s = s ? s : dalloc((void**)&l.wf, sizeof(float) * tc::prep_floats_f(d1));
        s = s ? s : dalloc((void**)&l.wt, sizeof(float) * tc::prep_floats_t(d1));
      }
    }
    // scratch (split-K partials, explicit-dgrad dP) for every batch size the
    // net may run -- the split plan depends on the batch
    for (int B = 1; B <= max_batch; ++B) {
      size_t need = 0;
      if (l.spec.kind == VCNN_LAYER_CONV) {
        need = conv_workspace(conv_of(l, B), VCNN_PREC_TF32);
        const size_t dw = direct::wgrad_workspace(conv_of(l, B));
        if (dw > need) need = dw;
        const size_t dws = direct::wgrad_small_workspace(conv_of(l, B));
        if (dws > need) need = dws;
        const size_t dk1 = k1::wgrad_workspace(conv_of(l, B));
        if (dk1 > need) need = dk1;
        const size_t dw1 = direct::wgrad1d_workspace(conv_of(l, B));
        if (dw1 > need) need = dw1;
      }
      else if (l.spec.kind == VCNN_LAYER_FULL)
        need = full_workspace(B, (int)l.in_per, l.spec.units, VCNN_PREC_TF32);
      if (need > wsb) wsb = need;
    }
  }
  // conv i fed by pool i-1 of a small-Kd conv+pool pair (i-2): the pair also
  // writes the pooled output as tf32 NHWC, which conv i stages with one TMA
  const bool tma_off = getenv("VCNN_NO_TMA_SLAB") != nullptr;  // A/B experiments
  for (size_t i = 2; i < n->L.size() && !s && !tma_off; ++i) {
    LayerRt& c = n->L[i];
    LayerRt& p = n->L[i - 1];
    const LayerRt& q = n->L[i - 2];
    if (c.spec.kind != VCNN_LAYER_CONV || !c.pf || p.spec.kind != VCNN_LAYER_POOL ||
        q.spec.kind != VCNN_LAYER_CONV || conv_is_dense(c))
      continue;
    if (!direct::small_fwd_ok(conv_of(q, max_batch), p.spec.kh)) continue;
    const ConvDesc dc = conv_of(c, max_batch);
    if (!direct::fwd_tma_ok(dc, 0) || direct::nhwc_map_bytes() > sizeof(c.tmap)) continue;
    s = dalloc((void**)&p.nhwc, sizeof(float) * (size_t)(p.out_per * max_batch));
    if (!s && direct::make_nhwc_map(dc, p.nhwc, c.tmap) == VCNN_OK) c.has_tmap = true;
  }
  {  // the two-layer tail's batch-slice partials (mlp_head_slices <= 2)
    const size_t nl = n->L.size();
    if (nl >= 2 && n->L[nl - 1].spec.kind == VCNN_LAYER_FULL &&
        (n->L[nl - 2].spec.kind == VCNN_LAYER_FULL || conv_is_dense(n->L[nl - 2]))) {
      const LayerRt& hl = n->L[nl - 2];
      const LayerRt& ll = n->L[nl - 1];
      const size_t per = (size_t)(hl.w_len + hl.b_len + ll.w_len + ll.b_len);
      s = s ? s : dalloc((void**)&n->tail_part, sizeof(float) * kMaxSlices * per);
      s = s ? s : dalloc((void**)&n->tail_aux, sizeof(float) * (kMaxSlices + 4));
      if (!s && cudaMemset(n->tail_aux, 0, sizeof(float) * (kMaxSlices + 4)) != cudaSuccess)
        s = fail(VCNN_ECUDA, "net_create: tail buffers");
    }
  }
  if (wsb) {
    s = s ? s : dalloc((void**)&n->ws.ptr, wsb);
    n->ws.bytes = wsb;
    s = s ? s : dalloc((void**)&n->ws2.ptr, wsb);
    n->ws2.bytes = wsb;
  }
  if (!s) {
    n->fork_ev.assign(n->L.size(), nullptr);
    for (auto& e : n->fork_ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
        s = fail(VCNN_ECUDA, "net_create: event");
    if (!s && (cudaEventCreateWithFlags(&n->join_ev, cudaEventDisableTiming) != cudaSuccess ||
               cudaStreamCreateWithFlags(&n->side, cudaStreamNonBlocking) != cudaSuccess))
      s = fail(VCNN_ECUDA, "net_create: side stream");
  }
  if (!s) {
    if (cudaMemcpy(n->params, hp.data(), sizeof(float) * (size_t)n->nparams,
                   cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemset(n->grads, 0, pbytes) != cudaSuccess ||
        cudaMemset(n->vel, 0, pbytes) != cudaSuccess ||
        cudaMemset(n->values, 0, sizeof(float) * n->out_units * max_batch) != cudaSuccess ||
        cudaMemset(n->cls, 0, sizeof(int) * max_batch) != cudaSuccess ||
        cudaMemset(n->err, 0, sizeof(int) * 4) != cudaSuccess ||
        cudaMemset(n->loss, 0, sizeof(float) * (4 + kLossWsFloats)) != cudaSuccess)
      s = fail(VCNN_ECUDA, "net_create: initial upload failed");
  }
  if (!s) {
    s = prep_weights(n);
    if (!s && cudaStreamSynchronize(n->stream) != cudaSuccess)
      s = fail(VCNN_ECUDA, "net_create: weight preparation failed");
  }
  if (s) {
    vcnn_net_destroy(n);
    return s;
  }
  *out = n;
  return VCNN_OK;
}

int vcnn_net_destroy(vcnn_net* n) {
  if (!n) return VCNN_OK;
  if (n->stream) cudaStreamSynchronize(n->stream);
  else cudaDeviceSynchronize();
  drop_graph(n);
  for (LayerRt& l : n->L) {
    cudaFree(l.out);
    cudaFree(l.gpre);
    cudaFree(l.arg);
    cudaFree(l.wf);
    cudaFree(l.wt);
    cudaFree(l.pf);
    cudaFree(l.pd);
    cudaFree(l.ps);
    cudaFree(l.nhwc);
  }
  cudaFree(n->params);
  cudaFree(n->grads);
  cudaFree(n->vel);
  cudaFree(n->x);
  cudaFree(n->cls);
  cudaFree(n->values);
  cudaFree(n->loss);
  cudaFree(n->err);
  cudaFree(n->ws.ptr);
  cudaFree(n->ws2.ptr);
  cudaFree(n->tail_part);
  cudaFree(n->tail_aux);
  cudaFree(n->ring.cursor);
  for (cudaEvent_t e : n->fork_ev)
    if (e) cudaEventDestroy(e);
  if (n->join_ev) cudaEventDestroy(n->join_ev);
  if (n->side) cudaStreamDestroy(n->side);
  if (n->cap_stream) cudaStreamDestroy(n->cap_stream);
  cudaFree(n->pipe.xs[0]);  // (slot 1 lies inside slot 0's allocation)
  cudaFree(n->pipe.cs[0]);
  cudaFree(n->pipe.vs[0]);
  for (int k = 0; k < vcnn_net::kSlots; ++k) {
    if (n->pipe.copied[k]) cudaEventDestroy(n->pipe.copied[k]);
    if (n->pipe.consumed[k]) cudaEventDestroy(n->pipe.consumed[k]);
  }
  if (n->pipe.start) cudaEventDestroy(n->pipe.start);
  if (n->pipe.stored) cudaEventDestroy(n->pipe.stored);
  if (n->pipe.hl) cudaFreeHost(n->pipe.hl);
  cudaFree(n->pipe.dl);
  cudaFree(n->pipe.cur);
  if (n->pipe.cp) cudaStreamDestroy(n->pipe.cp);
  if (n->pipe.rd) cudaStreamDestroy(n->pipe.rd);
  for (cudaEvent_t e : n->event_pool) cudaEventDestroy(e);
  delete n;
  return VCNN_OK;
}

int64_t vcnn_net_num_params(const vcnn_net* n) { return n ? n->nparams : -1; }

int vcnn_net_param_layout(const vcnn_net* n, int64_t* w_off, int64_t* w_len, int64_t* b_off,
                          int64_t* b_len) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  for (size_t i = 0; i < n->L.size(); ++i) {
    if (w_off) w_off[i] = n->L[i].w_off;
    if (w_len) w_len[i] = n->L[i].w_len;
    if (b_off) b_off[i] = n->L[i].b_off;
    if (b_len) b_len[i] = n->L[i].b_len;
  }
  return VCNN_OK;
}

int vcnn_net_layer_out_size(const vcnn_net* n, int layer, int64_t* per_sample) {
  if (!n || layer < 0 || layer >= (int)n->L.size())
    return fail(VCNN_EBOUNDS, "layer index out of range");
  *per_sample = n->L[layer].out_per;
  return VCNN_OK;
}

int vcnn_net_set_stream(vcnn_net* n, void* stream) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  if (n->stream != as_stream(stream)) drop_graph(n);
  n->stream = as_stream(stream);
  return VCNN_OK;
}

int vcnn_net_set_pool_backward_mode(vcnn_net* n, int mode) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  if (mode != VCNN_POOLBWD_EXACT && mode != VCNN_POOLBWD_PAPER_NN)
    return fail(VCNN_ECONFIG, "unknown pool backward mode");
  if (mode != n->pool_bwd_mode) drop_graph(n);
  n->pool_bwd_mode = mode;
  return VCNN_OK;
}

int vcnn_net_set_precision(vcnn_net* n, int precision) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  if (precision < VCNN_PREC_TF32 || precision > VCNN_PREC_FP32)
    return fail(VCNN_ECONFIG, "unknown precision");
  if (precision != n->precision) drop_graph(n);
  n->precision = precision;
  return VCNN_OK;
}

int vcnn_net_set_fusion(vcnn_net* n, int enable) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  if ((enable != 0) != n->fuse) drop_graph(n);
  n->fuse = enable != 0;
  return VCNN_OK;
}

int vcnn_net_set_trace(vcnn_net* n, int keep) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  if ((keep != 0) != n->keep_trace) drop_graph(n);
  n->keep_trace = keep != 0;
  return VCNN_OK;
}

int vcnn_net_get_params(vcnn_net* n, float* host) {
  return copy_out(n, host, n->params, sizeof(float) * n->nparams);
}
int vcnn_net_set_params(vcnn_net* n, const float* host) {
  TRY(copy_in(n, n->params, host, sizeof(float) * n->nparams));
  TRY(prep_weights(n));
  VCNN_CUDA_TRY(cudaStreamSynchronize(n->stream));
  return VCNN_OK;
}
int vcnn_net_set_nonfinite_guard(vcnn_net* n, int enable) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  n->guard = enable != 0;
  return write_guard(n, n->guard ? 1 : 0);
}
int vcnn_net_params_updated(vcnn_net* n) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  TRY(prep_weights(n));
  return VCNN_OK;
}
int vcnn_net_get_grads(vcnn_net* n, float* host) {
  return copy_out(n, host, n->grads, sizeof(float) * n->nparams);
}
int vcnn_net_get_velocity(vcnn_net* n, float* host) {
  return copy_out(n, host, n->vel, sizeof(float) * n->nparams);
}
int vcnn_net_set_velocity(vcnn_net* n, const float* host) {
  return copy_in(n, n->vel, host, sizeof(float) * n->nparams);
}

int vcnn_net_device_buffers(vcnn_net* n, float** params, float** grads, float** velocity) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  if (params) *params = n->params;
  if (grads) *grads = n->grads;
  if (velocity) *velocity = n->vel;
  return VCNN_OK;
}

int vcnn_net_input_buffers(vcnn_net* n, float** x, int** cls, float** values) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  if (x) *x = n->x;
  if (cls) *cls = n->cls;
  if (values) *values = n->values;
  return VCNN_OK;
}

int vcnn_net_set_batch_device(vcnn_net* n, int batch, const float* x, const int* cls,
                              const float* values) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  TRY(check_batch(n, batch));
  // one staging kernel for the images and the targets
  if (cls && values)
    VCNN_CUDA_TRY(cudaMemcpyAsync(n->values, values, sizeof(float) * n->out_units * batch,
                                  cudaMemcpyDeviceToDevice, n->stream));
  return launch_stage_batch(x, n->x, n->in_per * batch, cls ? (const void*)cls : values,
                            cls ? (void*)n->cls : (void*)n->values,
                            cls ? batch : n->out_units * batch, n->stream);
}

int vcnn_net_set_batch_ring(vcnn_net* n, int nbatch, int batch, const float* x,
                            int64_t x_stride, const void* targets, int64_t t_stride) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  // captured steps bake the ring's buffers, strides and size into their
  // staging kernel: a changed ring is a fresh set of graphs
  VCNN_CUDA_TRY(cudaStreamSynchronize(n->stream));
  drop_graph(n);
  if (nbatch <= 0) {
    n->ring.x = nullptr;
    n->ring.t = nullptr;
    n->ring.nbatch = 0;
    return VCNN_OK;
  }
  TRY(check_batch(n, batch));
  const bool ce = n->spec.loss == VCNN_LOSS_SOFTMAX_CE;
  if (!x || !targets || x_stride < n->in_per * batch ||
      t_stride < (ce ? batch : n->out_units * batch))
    return fail(VCNN_ESHAPE, "batch ring: buffers / strides");
  if (!n->ring.cursor) VCNN_CUDA_TRY(cudaMalloc(&n->ring.cursor, 4 * sizeof(int)));
  VCNN_CUDA_TRY(cudaMemsetAsync(n->ring.cursor, 0, 4 * sizeof(int), n->stream));
  n->ring.lhist = nullptr;
  n->ring.x = x;
  n->ring.t = targets;
  n->ring.nbatch = nbatch;
  n->ring.batch = batch;
  n->ring.xs = x_stride;
  n->ring.ts = t_stride;
  return VCNN_OK;
}

int vcnn_net_forward_backward(vcnn_net* n, int batch) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  TRY(check_batch(n, batch));
  const int tail = tail_fused(n, batch);
  TRY(run_forward(n, batch, tail));
  return run_backward(n, batch, tail);
}

int vcnn_net_forward(vcnn_net* n, int batch) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  TRY(check_batch(n, batch));
  return run_forward(n, batch);
}

int vcnn_net_sgd_step(vcnn_net* n, float lr, float mom, float grad_scale) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  TRY(check_cfg(lr, mom));
  return run_sgd(n, lr, mom, grad_scale);
}

int vcnn_net_train_step(vcnn_net* n, int batch, float lr, float mom) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  return train_step(n, batch, lr, mom);
}

int vcnn_net_train_steps(vcnn_net* n, int nsteps, int batch, float lr, float mom) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  if (nsteps < 0) return fail(VCNN_ESHAPE, "train_steps: negative count");
  constexpr int kChunk = 8;  // steps per graph launch
  for (int done = 0; done < nsteps;) {
    const int k = nsteps - done < kChunk ? nsteps - done : kChunk;
    TRY(train_steps_graph(n, k, batch, lr, mom));
    done += k;
  }
  return VCNN_OK;
}

int vcnn_net_train_step_host(vcnn_net* n, int batch, const float* x, const int* cls,
                             const float* values, float lr, float mom, float* loss_out) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  TRY(check_batch(n, batch));
  if (n->spec.loss == VCNN_LOSS_SOFTMAX_CE) {
    if (!cls) return fail(VCNN_ESHAPE, "loss: class targets required");
    for (int b = 0; b < batch; ++b)
      if (cls[b] < 0 || cls[b] >= n->out_units)
        return fail(VCNN_EBOUNDS, "loss: class index " + std::to_string(cls[b]) +
                                      " out of range [0," + std::to_string(n->out_units) + ")");
  } else if (!values) {
    return fail(VCNN_ESHAPE, "loss: value targets required");
  }
  VCNN_CUDA_TRY(cudaMemcpyAsync(n->x, x, sizeof(float) * n->in_per * batch,
                                cudaMemcpyHostToDevice, n->stream));
  if (n->spec.loss == VCNN_LOSS_SOFTMAX_CE)
    VCNN_CUDA_TRY(cudaMemcpyAsync(n->cls, cls, sizeof(int) * batch, cudaMemcpyHostToDevice,
                                  n->stream));
  else
    VCNN_CUDA_TRY(cudaMemcpyAsync(n->values, values, sizeof(float) * n->out_units * batch,
                                  cudaMemcpyHostToDevice, n->stream));
  TRY(train_step(n, batch, lr, mom));
  float l = 0;
  TRY(copy_out(n, &l, n->loss, sizeof(float)));
  if (loss_out) *loss_out = l;
  return VCNN_OK;
}

int vcnn_net_train_host_stream(vcnn_net* n, int nsteps, int batch, const float* x,
                               int64_t x_stride, const int* cls, const float* values,
                               int64_t t_stride, float lr, float mom, float* losses) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  if (nsteps < 1) return VCNN_OK;
  TRY(check_batch(n, batch));
  TRY(check_cfg(lr, mom));
  const bool ce = n->spec.loss == VCNN_LOSS_SOFTMAX_CE;
  if (!x || (ce ? !cls : !values)) return fail(VCNN_ESHAPE, "loss: targets required");
  if (ce)  // the host step's validation (Targets bounds), every batch
    for (int i = 0; i < nsteps; ++i)
      for (int b = 0; b < batch; ++b) {
        const int c = cls[(int64_t)i * t_stride + b];
        if (c < 0 || c >= n->out_units)
          return fail(VCNN_EBOUNDS, "loss: class index " + std::to_string(c) +
                                        " out of range [0," + std::to_string(n->out_units) + ")");
      }
  // the caller's batch ring (and its cursor) is swapped for the staging slots
  // with their own cursor, restored on exit
  struct RingSwap {
    vcnn_net* n;
    vcnn_net::Ring saved;
    explicit RingSwap(vcnn_net* m) : n(m), saved(m->ring) {}
    ~RingSwap() { n->ring = saved; }
  } ring_swap(n);
  auto& P = n->pipe;
  if (!P.cp) {
    VCNN_CUDA_TRY(cudaStreamCreateWithFlags(&P.cp, cudaStreamNonBlocking));
    VCNN_CUDA_TRY(cudaStreamCreateWithFlags(&P.rd, cudaStreamNonBlocking));
    VCNN_CUDA_TRY(cudaEventCreateWithFlags(&P.start, cudaEventDisableTiming));
    VCNN_CUDA_TRY(cudaEventCreateWithFlags(&P.stored, cudaEventDisableTiming));
    // the slots are contiguous: they form the staging ring
    constexpr int K = vcnn_net::kSlots;
    VCNN_CUDA_TRY(cudaMalloc(&P.xs[0], K * sizeof(float) * n->in_per * n->max_batch));
    VCNN_CUDA_TRY(cudaMalloc(&P.cs[0], K * sizeof(int) * n->max_batch));
    VCNN_CUDA_TRY(cudaMalloc(&P.vs[0], K * sizeof(float) * n->out_units * n->max_batch));
    for (int k = 1; k < K; ++k) {
      P.xs[k] = P.xs[0] + k * n->in_per * n->max_batch;
      P.cs[k] = P.cs[0] + k * n->max_batch;
      P.vs[k] = P.vs[0] + k * n->out_units * n->max_batch;
    }
    for (int k = 0; k < K; ++k) {
      VCNN_CUDA_TRY(cudaEventCreateWithFlags(&P.copied[k], cudaEventDisableTiming));
      VCNN_CUDA_TRY(cudaEventCreateWithFlags(&P.consumed[k], cudaEventDisableTiming));
    }
  }
  if (!P.cur) VCNN_CUDA_TRY(cudaMalloc(&P.cur, 4 * sizeof(int)));
  VCNN_CUDA_TRY(cudaMemsetAsync(P.cur, 0, 4 * sizeof(int), n->stream));
  n->ring.x = P.xs[0];
  n->ring.t = ce ? (const void*)P.cs[0] : (const void*)P.vs[0];
  n->ring.nbatch = vcnn_net::kSlots;
  n->ring.batch = batch;
  n->ring.xs = n->in_per * n->max_batch;
  n->ring.ts = ce ? n->max_batch : n->out_units * n->max_batch;
  n->ring.cursor = P.cur;
  if (P.hl_cap < nsteps) {
    if (P.hl) cudaFreeHost(P.hl);
    P.hl = nullptr;
    P.hl_cap = 0;
    VCNN_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&P.hl), sizeof(float) * nsteps,
                                cudaHostAllocDefault));
    P.hl_cap = nsteps;
  }
  // device loss history: a fixed ring (captured step graphs keep its pointer)
  if (!P.dl) VCNN_CUDA_TRY(cudaMalloc(&P.dl, sizeof(float) * vcnn_net::kLossRing));
  n->ring.lhist = P.dl;  // step i's staging kernel files step i-1's loss
  const size_t xb = sizeof(float) * n->in_per * batch;
  const size_t tb = ce ? sizeof(int) * batch : sizeof(float) * n->out_units * batch;
  // every copy is ordered after the work already queued on the net's stream
  VCNN_CUDA_TRY(cudaEventRecord(P.start, n->stream));
  VCNN_CUDA_TRY(cudaStreamWaitEvent(P.cp, P.start, 0));
  for (int i = 0; i < nsteps; ++i) {
    const int k = i % vcnn_net::kSlots;
    // copy stream: batch i into slot k once step i-kSlots has finished with it
    if (i >= vcnn_net::kSlots) VCNN_CUDA_TRY(cudaStreamWaitEvent(P.cp, P.consumed[k], 0));
    VCNN_CUDA_TRY(cudaMemcpyAsync(P.xs[k], x + (int64_t)i * x_stride, xb,
                                  cudaMemcpyHostToDevice, P.cp));
    if (ce)
      VCNN_CUDA_TRY(cudaMemcpyAsync(P.cs[k], cls + (int64_t)i * t_stride, tb,
                                    cudaMemcpyHostToDevice, P.cp));
    else
      VCNN_CUDA_TRY(cudaMemcpyAsync(P.vs[k], values + (int64_t)i * t_stride, tb,
                                    cudaMemcpyHostToDevice, P.cp));
    VCNN_CUDA_TRY(cudaEventRecord(P.copied[k], P.cp));
    // compute stream: slot k -> the input slots, the step, the loss to host
    VCNN_CUDA_TRY(cudaStreamWaitEvent(n->stream, P.copied[k], 0));
    // the step's graph stages slot k (the ring cursor walks 0, 1, 2, 0, ...)
    // and files the previous step's loss into P.dl[i - 1]
    TRY(train_step(n, batch, lr, mom));
    VCNN_CUDA_TRY(cudaEventRecord(P.consumed[k], n->stream));
    if (i > 0) {  // step i-1's loss back to the host on the read-back stream
      const int j = (i - 1) & (vcnn_net::kLossRing - 1);
      VCNN_CUDA_TRY(cudaStreamWaitEvent(P.rd, P.consumed[k], 0));
      VCNN_CUDA_TRY(cudaMemcpyAsync(P.hl + i - 1, P.dl + j, sizeof(float),
                                    cudaMemcpyDeviceToHost, P.rd));
    }
  }
  // the last step's loss
  const int jl = (nsteps - 1) & (vcnn_net::kLossRing - 1);
  TRY(launch_store_scalar(n->loss, P.dl + jl, n->stream));
  VCNN_CUDA_TRY(cudaEventRecord(P.stored, n->stream));
  VCNN_CUDA_TRY(cudaStreamWaitEvent(P.rd, P.stored, 0));
  VCNN_CUDA_TRY(cudaMemcpyAsync(P.hl + nsteps - 1, P.dl + jl, sizeof(float),
                                cudaMemcpyDeviceToHost, P.rd));
  VCNN_CUDA_TRY(cudaStreamSynchronize(n->stream));
  VCNN_CUDA_TRY(cudaStreamSynchronize(P.rd));
  if (losses) std::memcpy(losses, P.hl, sizeof(float) * nsteps);
  return VCNN_OK;
}

int vcnn_net_train_epoch(vcnn_net* n, const float* images, const int* cls, const float* values,
                         int count, const int* order, int batch, float lr, float mom,
                         float* losses) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  if (count < 1) return fail(VCNN_ETRAINING, "fit: empty dataset");
  if (batch < 1 || batch > n->max_batch)
    return fail(VCNN_ESHAPE, "epoch batch outside [1, max_batch]");
  TRY(check_cfg(lr, mom));
  const bool ce = n->spec.loss == VCNN_LOSS_SOFTMAX_CE;
  if (ce ? !cls : !values) return fail(VCNN_ESHAPE, "train_epoch: targets required");
  struct RingOff {  // the epoch loop gathers its own batches
    vcnn_net* n;
    int saved;
    explicit RingOff(vcnn_net* m) : n(m), saved(m->ring.nbatch) { m->ring.nbatch = 0; }
    ~RingOff() { n->ring.nbatch = saved; }
  } ring_off(n);
  // arm the non-finite guard (err[2] armed, err[3] tripped) for this epoch
  TRY(write_guard(n, 1));
  int bi = 0;
  for (int start = 0; start < count; start += batch, ++bi) {
    const int nb = count - start < batch ? count - start : batch;
    TRY(launch_gather_rows(nb, n->in_per, images, order, start, n->x, n->out_units,
                           ce ? cls : nullptr, n->cls, ce ? nullptr : values, n->values,
                           n->stream));
    TRY(train_step(n, nb, lr, mom));
    TRY(launch_store_scalar(n->loss, losses + bi, n->stream));
  }
  TRY(write_guard(n, n->guard ? 1 : 0));
  return VCNN_OK;
}

int vcnn_net_forward_host(vcnn_net* n, int batch, const float* x, float* out) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  TRY(check_batch(n, batch));
  VCNN_CUDA_TRY(cudaMemcpyAsync(n->x, x, sizeof(float) * n->in_per * batch,
                                cudaMemcpyHostToDevice, n->stream));
  TRY(run_forward(n, batch));
  return copy_out(n, out, n->L.back().out, sizeof(float) * n->out_units * batch);
}

int vcnn_net_enable_graph(vcnn_net* n, int enable) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  n->use_graph = enable != 0;
  if (!n->use_graph) drop_graph(n);
  return VCNN_OK;
}

int vcnn_net_get_loss(vcnn_net* n, float* loss) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  TRY(copy_out(n, loss, n->loss, sizeof(float)));
  return check_errflag(n);
}

int vcnn_net_get_output(vcnn_net* n, float* host) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  return copy_out(n, host, n->L.back().out, sizeof(float) * n->out_units * n->max_batch);
}

int vcnn_net_get_layer_output(vcnn_net* n, int layer, float* host) {
  if (!n || layer < 0 || layer >= (int)n->L.size())
    return fail(VCNN_EBOUNDS, "layer index out of range");
  const LayerRt& l = n->L[layer];
  return copy_out(n, host, l.out, sizeof(float) * l.out_per * n->max_batch);
}

int vcnn_net_get_layer_grad(vcnn_net* n, int layer, float* host) {
  if (!n || layer < 0 || layer >= (int)n->L.size())
    return fail(VCNN_EBOUNDS, "layer index out of range");
  const LayerRt& l = n->L[layer];
  return copy_out(n, host, l.gpre, sizeof(float) * l.out_per * n->max_batch);
}

int vcnn_net_get_pool_arg(vcnn_net* n, int layer, int64_t* host) {
  if (!n || layer < 0 || layer >= (int)n->L.size())
    return fail(VCNN_EBOUNDS, "layer index out of range");
  const LayerRt& l = n->L[layer];
  if (!l.arg) return fail(VCNN_ESHAPE, "layer has no argmax (not a max pool)");
  const size_t cnt = (size_t)(l.out_per * n->max_batch);
  std::vector<int32_t> tmp(cnt);
  TRY(copy_out(n, tmp.data(), l.arg, sizeof(int32_t) * cnt));
  for (size_t i = 0; i < cnt; ++i) host[i] = tmp[i];
  return VCNN_OK;
}

int vcnn_net_kernels_per_step(vcnn_net* n, int* count) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  *count = n->kernels_per_step;
  return VCNN_OK;
}

int vcnn_net_enable_breakdown(vcnn_net* n, int enable) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  n->breakdown = enable != 0;
  n->marks.clear();
  n->event_next = 0;
  for (double& s : n->seconds) s = 0;
  const size_t slots = (n->L.size() + 1) * OP_KINDS;
  n->op_sec.assign(slots, 0.0);
  n->op_cnt.assign(slots, 0);
  return VCNN_OK;
}

static int drain_marks(vcnn_net* n) {
  VCNN_CUDA_TRY(cudaStreamSynchronize(n->stream));
  const size_t slots = (n->L.size() + 1) * OP_KINDS;
  if (n->op_sec.size() != slots) {
    n->op_sec.assign(slots, 0.0);
    n->op_cnt.assign(slots, 0);
  }
  for (auto& m : n->marks) {
    float ms = 0;
    cudaEventElapsedTime(&ms, m.a, m.b);
    n->seconds[m.comp] += ms * 1e-3;
    const size_t slot = (size_t)(m.layer + 1) * OP_KINDS + m.op;
    n->op_sec[slot] += ms * 1e-3;
    n->op_cnt[slot] += 1;
  }
  n->marks.clear();
  n->event_next = 0;
  return VCNN_OK;
}

int vcnn_net_read_breakdown(vcnn_net* n, double* seconds8) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  TRY(drain_marks(n));
  for (int i = 0; i < 8; ++i) seconds8[i] = n->seconds[i];
  return VCNN_OK;
}

int vcnn_net_read_op_timing(vcnn_net* n, double* seconds, int64_t* counts) {
  if (!n) return fail(VCNN_ESHAPE, "null net");
  TRY(drain_marks(n));
  for (size_t i = 0; i < n->op_sec.size(); ++i) {
    seconds[i] = n->op_sec[i];
    counts[i] = n->op_cnt[i];
  }
  return VCNN_OK;
}

}  // extern "C"
