// vcnn_b200.hpp -- C++ host API of the B200 training path, header-only over
// the C ABI of libvcnn_cuda.so (include/vcnn_cuda.h).
//
// It mirrors the reference's C++ surface for the Imp-6 forward / backward /
// update path (proj/include/vcnn/*.hpp) with the same names, field names,
// defaults and exception types:
//   ConvSpec / PoolSpec / FullSpec / LayerSpec / NetworkSpec::chain   network.hpp:12-67
//   TrainConfig (+ validate)                                          network.hpp:75-89
//   build_network                                                     network.hpp:102-130
//   Targets::from_classes / from_values                               layers.hpp:379-398
//   RunResult {output, loss, grads, has_grads}                        variants.hpp:325-331
//   Executor::run_batch / forward / set_pool_backward_mode            variants.hpp:333-359
//   sgd_step                                                          network.hpp:242-273
//   Trainer::fit / evaluate_accuracy                                  training.hpp:50-124
//   ShapeError / GeometryError / BoundsError / ConfigError / TrainingError  common.hpp:26-46
// Differences that follow from the device: the Network lives in HBM
// (parameters, gradients, momentum, trace); samples cross as plain float
// arrays in the reference's NCHW order ((b*C+c)*H+y)*W+x (tensor.hpp:80-82);
// gradients and weights come back to the host only when asked for.  To run
// the reference's own Network<float> / Tensor<float> objects unchanged, see
// reference_adapter.hpp.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "../vcnn_cuda.h"

namespace vcnn_b200 {

// ---- errors (common.hpp:26-46) ----------------------------------------------
struct ShapeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct GeometryError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct BoundsError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TrainingError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// status code -> the reference's exception type
inline void check(int status) {
  if (status == VCNN_OK) return;
  const std::string msg = vcnn_last_error();
  switch (status) {
    case VCNN_ESHAPE: throw ShapeError(msg);
    case VCNN_EGEOMETRY: throw GeometryError(msg);
    case VCNN_EBOUNDS: throw BoundsError(msg);
    case VCNN_ECONFIG: throw ConfigError(msg);
    case VCNN_ETRAINING: throw TrainingError(msg);
    default: throw CudaError(msg);
  }
}

// ---- declarative types (layers.hpp:13, :375; vectorize.hpp:127, :217) --------
enum class Activation { identity = VCNN_ACT_IDENTITY, relu = VCNN_ACT_RELU,
                        sigmoid = VCNN_ACT_SIGMOID, tanh = VCNN_ACT_TANH };
enum class PoolMode { max = VCNN_POOL_MAX, avg = VCNN_POOL_AVG };
enum class PoolBackwardMode { exact = VCNN_POOLBWD_EXACT, paper_nn = VCNN_POOLBWD_PAPER_NN };
enum class LossKind { softmax_ce = VCNN_LOSS_SOFTMAX_CE, mse = VCNN_LOSS_MSE };
// arithmetic of the GEMM-shaped kernels (no reference counterpart: the
// reference is scalar fp; these are the tensor-core modes)
enum class Precision { tf32 = VCNN_PREC_TF32, tf32x3 = VCNN_PREC_3XTF32, fp32 = VCNN_PREC_FP32 };

struct Shape {  // one sample: h, w, c (tensor.hpp:20-56)
  int h = 1, w = 1, c = 1;
  int64_t size() const { return (int64_t)h * w * c; }
};

struct ConvSpec {
  int maps = 1;
  int kh = 3, kw = 3;
  int stride = 1;
  Activation act = Activation::relu;
};
struct PoolSpec {
  int ph = 2, pw = 2;
  int stride = 2;
  PoolMode mode = PoolMode::max;
  bool bias = false;
  Activation act = Activation::identity;
};
struct FullSpec {
  int units = 1;
  Activation act = Activation::relu;
};
using LayerSpec = std::variant<ConvSpec, PoolSpec, FullSpec>;

struct NetworkSpec {
  Shape input{1, 1, 1};
  std::vector<LayerSpec> layers;
  LossKind loss = LossKind::softmax_ce;
  uint64_t seed = 0;

  // C mirror (owns the layer array)
  struct CSpec {
    vcnn_net_spec spec{};
    std::vector<vcnn_layer_spec> layers;
  };
  CSpec to_c() const {
    CSpec c;
    for (const LayerSpec& l : layers) {
      vcnn_layer_spec s{};
      if (const auto* cs = std::get_if<ConvSpec>(&l)) {
        s.kind = VCNN_LAYER_CONV, s.units = cs->maps, s.kh = cs->kh, s.kw = cs->kw;
        s.stride = cs->stride, s.act = (int)cs->act;
      } else if (const auto* ps = std::get_if<PoolSpec>(&l)) {
        s.kind = VCNN_LAYER_POOL, s.kh = ps->ph, s.kw = ps->pw, s.stride = ps->stride;
        s.pool_mode = (int)ps->mode, s.pool_bias = ps->bias ? 1 : 0, s.act = (int)ps->act;
      } else {
        const auto& fs = std::get<FullSpec>(l);
        s.kind = VCNN_LAYER_FULL, s.units = fs.units, s.act = (int)fs.act;
      }
      c.layers.push_back(s);
    }
    c.spec.in_h = input.h, c.spec.in_w = input.w, c.spec.in_c = input.c;
    c.spec.nlayers = (int)c.layers.size();
    c.spec.layers = c.layers.data();
    c.spec.loss = (int)loss;
    c.spec.seed = seed;
    return c;
  }
  // per-layer single-sample output shapes; ShapeError on a broken chain
  std::vector<Shape> chain() const {
    CSpec c = to_c();
    std::vector<int> s(3 * layers.size());
    check(vcnn_net_spec_chain(&c.spec, s.data()));
    std::vector<Shape> out;
    for (size_t i = 0; i < layers.size(); ++i) out.push_back(Shape{s[3 * i], s[3 * i + 1], s[3 * i + 2]});
    return out;
  }
  Shape output_shape() const {
    auto c = chain();
    return c.empty() ? input : c.back();
  }
};

struct TrainConfig {
  double lr = 0.01;
  double momentum = 0.0;
  int batch = 1;
  int epochs = 1;
  uint64_t seed = 0;
  void validate() const {
    if (!(lr > 0)) throw ConfigError("learning rate must be positive");
    if (momentum < 0 || momentum >= 1) throw ConfigError("momentum must be in [0,1)");
    if (batch < 1) throw ConfigError("batch size must be >= 1");
    if (epochs < 1) throw ConfigError("epochs must be >= 1");
  }
};

template <typename T = float>
struct Targets {
  std::vector<int> classes;
  std::vector<T> values;  // [batch][output units], NCHW per sample
  static Targets from_classes(std::vector<int> cls) {
    Targets t;
    t.classes = std::move(cls);
    return t;
  }
  static Targets from_values(std::vector<T> v) {
    Targets t;
    t.values = std::move(v);
    return t;
  }
};

// ---- the device network (build_network + its Executor state) -----------------
class Network {
 public:
  Network() = default;
  Network(const NetworkSpec& spec, int max_batch, Precision p = Precision::tf32)
      : spec_(spec), max_batch_(max_batch) {
    NetworkSpec::CSpec c = spec.to_c();
    check(vcnn_net_create(&c.spec, max_batch, (int)p, &h_));
    const size_t n = spec.layers.size();
    w_off_.resize(n), w_len_.resize(n), b_off_.resize(n), b_len_.resize(n);
    check(vcnn_net_param_layout(h_, w_off_.data(), w_len_.data(), b_off_.data(), b_len_.data()));
    in_per_ = spec.input.size();
    out_units_ = spec.output_shape().size();
  }
  Network(const Network&) = delete;
  Network& operator=(const Network&) = delete;
  Network(Network&& o) noexcept { *this = std::move(o); }
  Network& operator=(Network&& o) noexcept {
    std::swap(h_, o.h_);
    spec_ = o.spec_, max_batch_ = o.max_batch_, in_per_ = o.in_per_, out_units_ = o.out_units_;
    w_off_ = o.w_off_, w_len_ = o.w_len_, b_off_ = o.b_off_, b_len_ = o.b_len_;
    return *this;
  }
  ~Network() {
    if (h_) vcnn_net_destroy(h_);
  }

  const NetworkSpec& spec() const { return spec_; }
  int max_batch() const { return max_batch_; }
  int64_t num_params() const { return vcnn_net_num_params(h_); }
  int64_t input_size() const { return in_per_; }
  int64_t output_units() const { return out_units_; }
  vcnn_net* handle() const { return h_; }
  // flat parameter layout (NetGrads order: per layer weights, then bias)
  int64_t weights_offset(size_t i) const { return w_off_.at(i); }
  int64_t weights_size(size_t i) const { return w_len_.at(i); }
  int64_t bias_offset(size_t i) const { return b_off_.at(i); }
  int64_t bias_size(size_t i) const { return b_len_.at(i); }

  std::vector<float> params() const { return fetch(vcnn_net_get_params); }
  std::vector<float> grads() const { return fetch(vcnn_net_get_grads); }
  std::vector<float> velocity() const { return fetch(vcnn_net_get_velocity); }
  void set_params(const std::vector<float>& p) {
    if ((int64_t)p.size() != num_params()) throw ShapeError("set_params: wrong parameter count");
    check(vcnn_net_set_params(h_, p.data()));
  }
  void set_velocity(const std::vector<float>& v) {
    if ((int64_t)v.size() != num_params()) throw ShapeError("set_velocity: wrong count");
    check(vcnn_net_set_velocity(h_, v.data()));
  }
  void set_precision(Precision p) { check(vcnn_net_set_precision(h_, (int)p)); }
  void enable_graph(bool on) { check(vcnn_net_enable_graph(h_, on ? 1 : 0)); }

 private:
  template <class F>
  std::vector<float> fetch(F f) const {
    std::vector<float> v((size_t)num_params());
    check(f(h_, v.data()));
    return v;
  }
  vcnn_net* h_ = nullptr;
  NetworkSpec spec_;
  int max_batch_ = 0;
  int64_t in_per_ = 0, out_units_ = 0;
  std::vector<int64_t> w_off_, w_len_, b_off_, b_len_;
};

// build_network (network.hpp:102-130): Glorot init from Rng(spec.seed), zero
// bias, bit-identical to the reference's build_network<float>
inline Network build_network(const NetworkSpec& spec, int max_batch,
                             Precision p = Precision::tf32) {
  return Network(spec, max_batch, p);
}

struct RunResult {
  std::vector<float> output;  // [batch][output units]
  float loss = 0.f;
  bool has_grads = false;     // gradients stay on the device: Network::grads()
};

class Executor {
 public:
  explicit Executor(Precision p = Precision::tf32) : prec_(p) {}
  void set_pool_backward_mode(PoolBackwardMode m) { mode_ = m; }
  PoolBackwardMode pool_backward_mode() const { return mode_; }

  // Executor::run_batch (variants.hpp:353-376): batch = HOST samples NCHW
  RunResult run_batch(Network& net, const float* batch, int n, const Targets<float>* targets) {
    prepare(net, n);
    RunResult r;
    if (!targets) {
      r.output.resize((size_t)(n * net.output_units()));
      check(vcnn_net_forward_host(net.handle(), n, batch, r.output.data()));
      return r;
    }
    const bool ce = net.spec().loss == LossKind::softmax_ce;
    validate_targets(net, n, *targets, ce);
    float *dx = nullptr, *dv = nullptr;
    int* dc = nullptr;
    check(vcnn_net_input_buffers(net.handle(), &dx, &dc, &dv));
    stage(dx, batch, sizeof(float) * (size_t)(n * net.input_size()));
    if (ce) stage(dc, targets->classes.data(), sizeof(int) * (size_t)n);
    else stage(dv, targets->values.data(), sizeof(float) * targets->values.size());
    check(vcnn_net_forward_backward(net.handle(), n));
    check(vcnn_net_get_loss(net.handle(), &r.loss));
    std::vector<float> full((size_t)(net.max_batch() * net.output_units()));
    check(vcnn_net_get_output(net.handle(), full.data()));
    full.resize((size_t)(n * net.output_units()));
    r.output = std::move(full);
    r.has_grads = true;
    return r;
  }
  // Executor::forward (variants.hpp:346-348)
  std::vector<float> forward(Network& net, const float* batch, int n) {
    return run_batch(net, batch, n, nullptr).output;
  }

 private:
  void prepare(Network& net, int n) {
    if (n < 1 || n > net.max_batch()) throw ShapeError("batch outside [1, max_batch]");
    net.set_precision(prec_);
    check(vcnn_net_set_pool_backward_mode(net.handle(), (int)mode_));
  }
  static void validate_targets(const Network& net, int n, const Targets<float>& t, bool ce) {
    if (ce) {
      if ((int)t.classes.size() != n) throw ShapeError("loss: one class index per sample");
      for (int c : t.classes)
        if (c < 0 || c >= net.output_units())
          throw BoundsError("loss: class index " + std::to_string(c) + " out of range");
    } else if ((int64_t)t.values.size() != n * net.output_units()) {
      throw ShapeError("loss: value targets do not match the output shape");
    }
  }
  static void stage(void* dev, const void* host, size_t bytes) {
    // synchronous copy of a host batch into the network's input slot
    check(cuda_copy(dev, host, bytes));
  }
  static int cuda_copy(void* dev, const void* host, size_t bytes);
  Precision prec_;
  PoolBackwardMode mode_ = PoolBackwardMode::exact;
};

// host -> device copy through the library (keeps the API free of CUDA headers)
inline int Executor::cuda_copy(void* dev, const void* host, size_t bytes) {
  return vcnn_copy_h2d(dev, host, bytes);
}

// sgd_step (network.hpp:242-273) on the gradients of the last run_batch:
// v = momentum*v + g; w -= lr*v (velocity starts at zero, device-resident)
inline void sgd_step(Network& net, const TrainConfig& cfg) {
  cfg.validate();
  check(vcnn_net_sgd_step(net.handle(), (float)cfg.lr, (float)cfg.momentum, 1.0f));
}

// predict_classes (network.hpp:179-192): argmax per sample, ties -> lowest
inline std::vector<int> predict_classes(const std::vector<float>& out, int n) {
  std::vector<int> cls((size_t)n, 0);
  if (n == 0) return cls;
  const size_t units = out.size() / (size_t)n;
  for (int b = 0; b < n; ++b) {
    const float* o = out.data() + (size_t)b * units;
    size_t best = 0;
    for (size_t u = 1; u < units; ++u)
      if (o[u] > o[best]) best = u;
    cls[(size_t)b] = (int)best;
  }
  return cls;
}

// Data parallelism (vcnn_dp_*): the gradient exchange inserted
// between run_batch and sgd_step (training.hpp:76-81).  Attached to its
// Network: from construction on, the net's sgd step (and train steps) are the
// group exchange -- by default ONE kernel per replica reading every replica's
// gradient over NVLink peer mappings (rank-ordered sum weighted by B_p / B,
// SGD, weight packs), else NCCL all-reduce.  Contiguous shards of each
// global batch (Imp-2 chunking, variants.hpp:442-443).
class DataParallel {
 public:
  using Id = std::array<uint8_t, VCNN_DP_ID_BYTES>;
  // rank 0 creates the NCCL id; the host broadcasts the bytes to every rank
  static Id unique_id() {
    Id id{};
    check(vcnn_dp_unique_id(id.data()));
    return id;
  }
  // process-per-GPU (collective: every rank constructs it)
  DataParallel(Network& net, int world, int rank, const Id& id) : world_(world), rank_(rank) {
    check(vcnn_dp_init(net.handle(), world, rank, id.data(), &h_));
  }
  // `world` replicas in one process (one device or several); barrier = false:
  // step them together with Trainer::fit_group / vcnn_dp_group_train_step
  static std::vector<std::unique_ptr<DataParallel>> group(const std::vector<Network*>& nets,
                                                          bool barrier = false) {
    std::vector<vcnn_net*> hs;
    for (Network* n : nets) hs.push_back(n->handle());
    std::vector<vcnn_dp*> out(nets.size(), nullptr);
    check(vcnn_dp_group(hs.data(), (int)hs.size(), barrier ? 1 : 0, out.data()));
    std::vector<std::unique_ptr<DataParallel>> g;
    for (size_t r = 0; r < out.size(); ++r)
      g.emplace_back(new DataParallel(out[r], (int)out.size(), (int)r));
    return g;
  }
  DataParallel(const DataParallel&) = delete;
  DataParallel& operator=(const DataParallel&) = delete;
  ~DataParallel() {
    if (h_) vcnn_dp_destroy(h_);
  }
  int world() const { return world_; }
  int rank() const { return rank_; }
  vcnn_dp* handle() const { return h_; }
  void set_mode(int mode) { check(vcnn_dp_set_mode(h_, mode)); }
  void set_shards(const std::vector<int>& batches) { check(vcnn_dp_set_shards(h_, batches.data())); }
  void status() { check(vcnn_dp_status(h_)); }
  // [lo, hi) of rank's contiguous shard of a global batch
  static std::pair<int, int> shard(int global_batch, int rank, int world) {
    return {(int)((int64_t)global_batch * rank / world),
            (int)((int64_t)global_batch * (rank + 1) / world)};
  }
  static std::vector<int> shard_sizes(int global_batch, int world) {
    std::vector<int> s((size_t)world);
    for (int r = 0; r < world; ++r) {
      auto [lo, hi] = shard(global_batch, r, world);
      s[(size_t)r] = hi - lo;
    }
    return s;
  }

 private:
  DataParallel(vcnn_dp* h, int world, int rank) : h_(h), world_(world), rank_(rank) {}
  vcnn_dp* h_ = nullptr;
  int world_ = 1, rank_ = 0;
};

// Trainer (training.hpp:50-124): seeded shuffle per epoch (Rng::shuffle,
// common.hpp:84-90), batches of cfg.batch with a smaller last batch, one
// device train step per batch (graph-replayed), NaN -> TrainingError.
class Trainer {
 public:
  explicit Trainer(TrainConfig cfg) : cfg_(cfg) { cfg_.validate(); }

  // dp (optional, process-per-GPU): every rank draws the same permutation and
  // trains on its contiguous slice of each global batch of cfg.batch samples;
  // the update is the group exchange, so the replicas follow the single-GPU
  // trajectory.  The returned losses are then this rank's shard losses
  // weighted by B_p / B (sum them over the ranks for the global epoch loss).
  std::vector<double> fit(Network& net, const std::vector<float>& images,
                          const Targets<float>& targets, DataParallel* dp = nullptr) {
    const int64_t per = net.input_size();
    const int count = (int)(images.size() / (size_t)per);
    if (count < 1) throw TrainingError("fit: empty dataset");
    const bool ce = net.spec().loss == LossKind::softmax_ce;
    const int64_t units = net.output_units();
    std::vector<int> order((size_t)count);
    for (int i = 0; i < count; ++i) order[(size_t)i] = i;
    Mt64 rng(cfg_.seed);
    std::vector<double> epoch_loss;
    std::vector<float> xb, vb;
    std::vector<int> cb;
    // a non-finite loss stops BEFORE that batch's sgd_step (training.hpp:77-80):
    // the one-call device step skips its update while the guard is armed
    check(vcnn_net_set_nonfinite_guard(net.handle(), 1));
    struct Disarm {
      vcnn_net* h;
      ~Disarm() { vcnn_net_set_nonfinite_guard(h, 0); }
    } disarm{net.handle()};
    for (int e = 0; e < cfg_.epochs; ++e) {
      rng.shuffle(order);
      double sum = 0;
      int batches = 0;
      for (int gstart = 0; gstart < count; gstart += cfg_.batch) {
        int start = gstart, n = std::min(cfg_.batch, count - gstart);
        double w = 1.0;
        if (dp && dp->world() > 1) {  // this rank's slice of the global batch
          const int gb = n;
          if (gb < dp->world()) throw ShapeError("fit: a global batch smaller than the world");
          auto [lo, hi] = DataParallel::shard(gb, dp->rank(), dp->world());
          dp->set_shards(DataParallel::shard_sizes(gb, dp->world()));
          start = gstart + lo;
          n = hi - lo;
          w = (double)n / gb;
        }
        xb.resize((size_t)(n * per));
        cb.resize((size_t)n);
        vb.resize((size_t)(n * units));
        for (int j = 0; j < n; ++j) {  // gather_batch (network.hpp:165-176)
          const int id = order[(size_t)(start + j)];
          std::copy(images.begin() + (size_t)id * per, images.begin() + (size_t)(id + 1) * per,
                    xb.begin() + (size_t)j * per);
          if (ce) cb[(size_t)j] = targets.classes[(size_t)id];
          else
            std::copy(targets.values.begin() + (size_t)id * units,
                      targets.values.begin() + (size_t)(id + 1) * units,
                      vb.begin() + (size_t)j * units);
        }
        float loss = 0;
        check(vcnn_net_train_step_host(net.handle(), n, xb.data(), ce ? cb.data() : nullptr,
                                       ce ? nullptr : vb.data(), (float)cfg_.lr,
                                       (float)cfg_.momentum, &loss));
        if (!std::isfinite(loss))
          throw TrainingError("non-finite loss at epoch " + std::to_string(e) + ", batch " +
                              std::to_string(batches));
        sum += w * loss;
        ++batches;
      }
      epoch_loss.push_back(sum / batches);
    }
    return epoch_loss;
  }

  // single process, G replicas (one per device, or G logical shards of one
  // device) created by DataParallel::group(nets, false): per global batch every
  // replica gets its contiguous shard and one vcnn_dp_group_train_step runs
  // them all; the epoch loss is the mean of the global-batch losses
  // (sum_p B_p / B * loss_p), as the single-GPU Trainer reports it
  std::vector<double> fit_group(const std::vector<Network*>& nets,
                                const std::vector<std::unique_ptr<DataParallel>>& dps,
                                const std::vector<float>& images, const Targets<float>& targets) {
    const int G = (int)nets.size();
    if (G < 1 || (int)dps.size() != G) throw ConfigError("fit_group: one DataParallel per net");
    const int64_t per = nets[0]->input_size();
    const int count = (int)(images.size() / (size_t)per);
    if (count < 1) throw TrainingError("fit: empty dataset");
    const bool ce = nets[0]->spec().loss == LossKind::softmax_ce;
    const int64_t units = nets[0]->output_units();
    std::vector<int> order((size_t)count);
    for (int i = 0; i < count; ++i) order[(size_t)i] = i;
    Mt64 rng(cfg_.seed);
    std::vector<double> epoch_loss;
    std::vector<vcnn_dp*> hs;
    for (auto& d : dps) hs.push_back(d->handle());
    std::vector<float> xb, vb;
    std::vector<int> cb;
    for (int e = 0; e < cfg_.epochs; ++e) {
      rng.shuffle(order);
      double sum = 0;
      int batches = 0;
      for (int gstart = 0; gstart < count; gstart += cfg_.batch) {
        const int gb = std::min(cfg_.batch, count - gstart);
        if (gb < G) throw ShapeError("fit_group: a global batch smaller than the group");
        const std::vector<int> sizes = DataParallel::shard_sizes(gb, G);
        for (int r = 0; r < G; ++r) {  // stage each replica's shard
          const int lo = DataParallel::shard(gb, r, G).first, n = sizes[(size_t)r];
          xb.resize((size_t)(n * per));
          cb.resize((size_t)n);
          vb.resize((size_t)(n * units));
          for (int j = 0; j < n; ++j) {
            const int id = order[(size_t)(gstart + lo + j)];
            std::copy(images.begin() + (size_t)id * per, images.begin() + (size_t)(id + 1) * per,
                      xb.begin() + (size_t)j * per);
            if (ce) cb[(size_t)j] = targets.classes[(size_t)id];
            else
              std::copy(targets.values.begin() + (size_t)id * units,
                        targets.values.begin() + (size_t)(id + 1) * units,
                        vb.begin() + (size_t)j * units);
          }
          if (ce)
            for (int c : cb)
              if (c < 0 || c >= units) throw BoundsError("loss: class index out of range");
          float *dx = nullptr, *dv = nullptr;
          int* dc = nullptr;
          check(vcnn_net_input_buffers(nets[(size_t)r]->handle(), &dx, &dc, &dv));
          check(vcnn_copy_h2d(dx, xb.data(), sizeof(float) * xb.size()));
          if (ce) check(vcnn_copy_h2d(dc, cb.data(), sizeof(int) * cb.size()));
          else check(vcnn_copy_h2d(dv, vb.data(), sizeof(float) * vb.size()));
        }
        check(vcnn_dp_group_train_step(hs.data(), G, sizes.data(), (float)cfg_.lr,
                                       (float)cfg_.momentum));
        double loss = 0;
        for (int r = 0; r < G; ++r) {
          float l = 0;
          check(vcnn_net_get_loss(nets[(size_t)r]->handle(), &l));
          loss += (double)sizes[(size_t)r] / gb * l;
        }
        if (!std::isfinite(loss))
          throw TrainingError("non-finite loss at epoch " + std::to_string(e) + ", batch " +
                              std::to_string(batches));
        sum += loss;
        ++batches;
      }
      epoch_loss.push_back(sum / batches);
    }
    return epoch_loss;
  }

  double evaluate_accuracy(Network& net, const std::vector<float>& images,
                           const std::vector<int>& labels) {
    const int64_t per = net.input_size();
    const int count = (int)(images.size() / (size_t)per);
    int correct = 0;
    Executor ex;
    for (int start = 0; start < count; start += net.max_batch()) {
      const int n = std::min(net.max_batch(), count - start);
      auto out = ex.forward(net, images.data() + (size_t)start * per, n);
      auto pred = predict_classes(out, n);
      for (int j = 0; j < n; ++j) correct += pred[(size_t)j] == labels[(size_t)(start + j)];
    }
    return count ? (double)correct / count : 0.0;
  }

 private:
  // Rng (common.hpp:51-96): mt19937_64 stream; shuffle = Fisher-Yates with
  // uniform_int(i+1) = min(floor(u*(i+1)), i), u = (x >> 11) * 2^-53
  struct Mt64 {
    uint64_t mt[312];
    int idx = 312;
    explicit Mt64(uint64_t seed) {
      mt[0] = seed;
      for (int i = 1; i < 312; ++i)
        mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    }
    uint64_t next() {
      if (idx >= 312) {
        for (int i = 0; i < 312; ++i) {
          const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
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
    int uniform_int(int n) {
      const double u = (double)(next() >> 11) * 0x1.0p-53;
      const int v = (int)(u * n);
      return v < n ? v : n - 1;
    }
    void shuffle(std::vector<int>& v) {
      for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[(size_t)uniform_int((int)i)]);
    }
  };
  TrainConfig cfg_;
};

}  // namespace vcnn_b200
