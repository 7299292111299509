// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against the
// reference sources where they lie (/root/reference/proj/include +
// proj/src/common.cpp), with -Dvcnn=vcnn_ref so the reference namespace can
// never collide with anything else.  Output goes to oracle/_ref/ only.  It
// serves two purposes:
//   * pinning: tests compare the C restatement (vcnn_oracle.c) with the
//     reference itself on the same inputs, and tests/golden/make_golden.py
//     records fixtures from it;
//   * the cpu_baseline / `bench.py --impl reference` arm: the reference's own
//     Executor<float>(imp6).run_batch + sgd_step, timed on the host cores.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "vcnn/io.hpp"
#include "vcnn/training.hpp"
#include "../oracle/vcnn_oracle.h"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace vcnn_ref;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ShapeError*>(&e)) return ORC_ESHAPE;
  if (dynamic_cast<const GeometryError*>(&e)) return ORC_EGEOMETRY;
  if (dynamic_cast<const BoundsError*>(&e)) return ORC_EBOUNDS;
  if (dynamic_cast<const ConfigError*>(&e)) return ORC_ECONFIG;
  return 99;
}

Activation act_of(int a) {
  switch (a) {
    case ORC_ACT_RELU: return Activation::relu;
    case ORC_ACT_SIGMOID: return Activation::sigmoid;
    case ORC_ACT_TANH: return Activation::tanh;
    default: return Activation::identity;
  }
}

NetworkSpec spec_of(const orc_net* n) {
  NetworkSpec s;
  s.input = Shape{n->in_h, n->in_w, n->in_c};
  s.loss = n->loss == ORC_LOSS_MSE ? LossKind::mse : LossKind::softmax_ce;
  s.seed = n->seed;
  for (int i = 0; i < n->nlayers; ++i) {
    const orc_layer& L = n->layers[i];
    if (L.kind == ORC_LAYER_CONV) {
      s.layers.push_back(ConvSpec{L.units, L.kh, L.kw, L.stride, act_of(L.act)});
    } else if (L.kind == ORC_LAYER_POOL) {
      s.layers.push_back(PoolSpec{L.kh, L.kw, L.stride,
                                  L.pool_mode == ORC_POOL_AVG ? PoolMode::avg : PoolMode::max,
                                  L.pool_bias != 0, act_of(L.act)});
    } else {
      s.layers.push_back(FullSpec{L.units, act_of(L.act)});
    }
  }
  return s;
}

template <typename T>
void params_to_flat(const Network<T>& net, T* out) {
  int64_t off = 0;
  auto put = [&](const std::vector<T>& v) {
    std::memcpy(out + off, v.data(), sizeof(T) * v.size());
    off += static_cast<int64_t>(v.size());
  };
  for (const auto& l : net.layers) {
    if (const auto* c = std::get_if<ConvLayer<T>>(&l)) {
      put(c->weights.data);
      put(c->bias);
    } else if (const auto* p = std::get_if<PoolLayer<T>>(&l)) {
      put(p->bias);
    } else {
      const auto& f = std::get<FullLayer<T>>(l);
      put(f.weights.data);
      put(f.bias);
    }
  }
}

template <typename T>
void flat_to_params(Network<T>& net, const T* in) {
  int64_t off = 0;
  auto get = [&](std::vector<T>& v) {
    std::memcpy(v.data(), in + off, sizeof(T) * v.size());
    off += static_cast<int64_t>(v.size());
  };
  for (auto& l : net.layers) {
    if (auto* c = std::get_if<ConvLayer<T>>(&l)) {
      get(c->weights.data);
      get(c->bias);
    } else if (auto* p = std::get_if<PoolLayer<T>>(&l)) {
      get(p->bias);
    } else {
      auto& f = std::get<FullLayer<T>>(l);
      get(f.weights.data);
      get(f.bias);
    }
  }
}

template <typename T>
void grads_to_flat(const NetGrads<T>& g, T* out) {
  int64_t off = 0;
  for (const auto& l : g.layers) {
    std::memcpy(out + off, l.weights.data.data(), sizeof(T) * l.weights.data.size());
    off += static_cast<int64_t>(l.weights.data.size());
    std::memcpy(out + off, l.bias.data(), sizeof(T) * l.bias.size());
    off += static_cast<int64_t>(l.bias.size());
  }
}

template <typename T>
Targets<T> targets_of(const NetworkSpec& spec, int B, const int* cls, const T* values) {
  if (spec.loss == LossKind::softmax_ce) return Targets<T>::from_classes(std::vector<int>(cls, cls + B));
  Shape o = spec.output_shape();
  Tensor<T> v(Shape::hwcn(o.h(), o.w(), o.c(), B));
  std::memcpy(v.data.data(), values, sizeof(T) * v.data.size());
  return Targets<T>::from_values(std::move(v));
}

Variant variant_of(int v) {
  switch (v) {
    case 1: return Variant::imp1;
    case 2: return Variant::imp2;
    case 3: return Variant::imp3;
    case 4: return Variant::imp4;
    case 5: return Variant::imp5;
    default: return Variant::imp6;
  }
}

struct BenchState {
  NetworkSpec spec;
  Network<float> net;
  Executor<float> exec{Variant::imp6};
  Tensor<float> batch;
  Targets<float> targets;
  TrainConfig cfg;
  Velocity<float> vel;
  float last_loss = 0;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#endif
}

int ref_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void ref_rng_fill_uniform(uint64_t seed, double* out, int64_t n, double lo, double hi) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
}

void ref_rng_fill_uniform_int(uint64_t seed, int* out, int64_t n, int k) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform_int(k);
}

int ref_net_init(const orc_net* n, double* params) {
  try {
    Network<double> net = build_network<double>(spec_of(n));
    params_to_flat(net, params);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_net_init_f32(const orc_net* n, float* params) {
  try {
    Network<float> net = build_network<float>(spec_of(n));
    params_to_flat(net, params);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// Executor<double>(variant).run_batch on explicit parameters.
int ref_net_run_batch(const orc_net* n, int variant, int B, const double* params,
                      const double* x, const int* cls, const double* values, int pool_bwd_mode,
                      int compute_grads, double* out, double* loss, double* grads) {
  try {
    NetworkSpec spec = spec_of(n);
    Network<double> net = build_network<double>(spec);
    flat_to_params(net, params);
    Tensor<double> xb(Shape::hwcn(n->in_h, n->in_w, n->in_c, B));
    std::memcpy(xb.data.data(), x, sizeof(double) * xb.data.size());
    Executor<double> exec(variant_of(variant));
    exec.set_pool_backward_mode(pool_bwd_mode ? PoolBackwardMode::paper_nn
                                              : PoolBackwardMode::exact);
    if (!compute_grads) {
      Tensor<double> o = exec.forward(net, xb);
      std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
      return 0;
    }
    Targets<double> t = targets_of<double>(spec, B, cls, values);
    RunResult<double> r = exec.run_batch(net, xb, &t);
    std::memcpy(out, r.output.data.data(), sizeof(double) * r.output.data.size());
    *loss = r.loss;
    grads_to_flat(r.grads, grads);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// Trainer-free N-step loop: run_batch + sgd_step, steps times, same batch.
int ref_net_train_steps(const orc_net* n, int B, double* params, const double* x,
                        const int* cls, const double* values, double lr, double mom, int steps,
                        double* losses) {
  try {
    NetworkSpec spec = spec_of(n);
    Network<double> net = build_network<double>(spec);
    flat_to_params(net, params);
    Tensor<double> xb(Shape::hwcn(n->in_h, n->in_w, n->in_c, B));
    std::memcpy(xb.data.data(), x, sizeof(double) * xb.data.size());
    Targets<double> t = targets_of<double>(spec, B, cls, values);
    Executor<double> exec(Variant::imp6);
    TrainConfig cfg;
    cfg.lr = lr;
    cfg.momentum = mom;
    Velocity<double> vel;
    for (int s = 0; s < steps; ++s) {
      RunResult<double> r = exec.run_batch(net, xb, &t);
      losses[s] = r.loss;
      sgd_step(net, r.grads, cfg, vel);
    }
    params_to_flat(net, params);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// the reference's own float path (Executor<float>(imp6) + sgd_step): used to
// measure how far an fp32 trajectory legitimately drifts from the f64 one
// (near-tie argmax / ReLU decisions), which sets the N-step tolerances
int ref_net_train_steps_f32(const orc_net* n, int B, float* params, const float* x,
                            const int* cls, const float* values, double lr, double mom,
                            int steps, double* losses) {
  try {
    NetworkSpec spec = spec_of(n);
    Network<float> net = build_network<float>(spec);
    flat_to_params(net, params);
    Tensor<float> xb(Shape::hwcn(n->in_h, n->in_w, n->in_c, B));
    std::memcpy(xb.data.data(), x, sizeof(float) * xb.data.size());
    Targets<float> t = targets_of<float>(spec, B, cls, values);
    Executor<float> exec(Variant::imp6);
    TrainConfig cfg;
    cfg.lr = lr;
    cfg.momentum = mom;
    Velocity<float> vel;
    for (int s = 0; s < steps; ++s) {
      RunResult<float> r = exec.run_batch(net, xb, &t);
      losses[s] = r.loss;
      sgd_step(net, r.grads, cfg, vel);
    }
    params_to_flat(net, params);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// Trainer<double>(cfg).fit + evaluate_accuracy (training.hpp:50-107) over a
// whole dataset: seeded shuffle carried across epochs, smaller last batch,
// mean epoch loss.  params in/out (flat), epoch_loss[epochs]; accuracy
// (nullable) = evaluate_accuracy on the same images after training (class
// targets only).  f32 = 1 runs Trainer<float> (for drift measurements).
int ref_fit(const orc_net* n, int count, double* params, const double* x, const int* cls,
            const double* values, double lr, double mom, int batch, int epochs, uint64_t seed,
            int f32, double* epoch_loss, double* accuracy) {
  try {
    NetworkSpec spec = spec_of(n);
    TrainConfig cfg;
    cfg.lr = lr;
    cfg.momentum = mom;
    cfg.batch = batch;
    cfg.epochs = epochs;
    cfg.seed = seed;
    auto run = [&](auto zero) {
      using T = decltype(zero);
      Network<T> net = build_network<T>(spec);
      const int64_t np = [&] {
        int64_t c = 0;
        for (const auto& l : net.layers) {
          if (const auto* cv = std::get_if<ConvLayer<T>>(&l)) c += cv->weights.data.size() + cv->bias.size();
          else if (const auto* p = std::get_if<PoolLayer<T>>(&l)) c += p->bias.size();
          else c += std::get<FullLayer<T>>(l).weights.data.size() + std::get<FullLayer<T>>(l).bias.size();
        }
        return c;
      }();
      std::vector<T> pt(params, params + np);
      flat_to_params(net, pt.data());
      Tensor<T> xs(Shape::hwcn(n->in_h, n->in_w, n->in_c, count));
      for (size_t i = 0; i < xs.data.size(); ++i) xs.data[i] = static_cast<T>(x[i]);
      std::vector<T> vt;
      if (values) {
        Shape o = spec.output_shape();
        vt.assign(values, values + (size_t)o.h() * o.w() * o.c() * count);
      }
      Targets<T> t = targets_of<T>(spec, count, cls, values ? vt.data() : nullptr);
      Trainer<T> tr(cfg);
      TrainStats<T> st = tr.fit(net, xs, t);
      for (int e = 0; e < epochs; ++e) epoch_loss[e] = static_cast<double>(st.epoch_loss[e]);
      params_to_flat(net, pt.data());
      for (int64_t i = 0; i < np; ++i) params[i] = static_cast<double>(pt[i]);
      if (accuracy && cls)
        *accuracy = tr.evaluate_accuracy(net, xs, std::vector<int>(cls, cls + count));
    };
    if (f32) run(0.0f); else run(0.0);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// the reference's own ModelFile v1 writer / reader (io.cpp:265-404):
// parameters (flat, NetGrads order) <-> file, f32 or f64 networks
int ref_save_model(const orc_net* n, const double* params, int f32, const char* path) {
  try {
    NetworkSpec spec = spec_of(n);
    if (f32) {
      Network<float> net = build_network<float>(spec);
      size_t count = 0;
      for (auto& layer : net.layers)
        std::visit(
            [&](const auto& l) {
              using L = std::decay_t<decltype(l)>;
              if constexpr (!std::is_same_v<L, PoolLayer<float>>) count += l.weights.data.size();
              count += l.bias.size();
            },
            layer);
      std::vector<float> pf(params, params + count);
      flat_to_params(net, pf.data());
      save_model(path, model_from_network(net));
    } else {
      Network<double> net = build_network<double>(spec);
      flat_to_params(net, params);
      save_model(path, model_from_network(net));
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_load_model_f32(const char* path, float* params, int64_t cap) {
  try {
    ModelFile m = load_model(path);
    Network<float> net = network_from_model<float>(m);
    std::vector<float> flat;
    for (auto& layer : net.layers)
      std::visit(
          [&](const auto& l) {
            using L = std::decay_t<decltype(l)>;
            if constexpr (!std::is_same_v<L, PoolLayer<float>>)
              flat.insert(flat.end(), l.weights.data.begin(), l.weights.data.end());
            flat.insert(flat.end(), l.bias.begin(), l.bias.end());
          },
          layer);
    if ((int64_t)flat.size() > cap) return 99;
    std::memcpy(params, flat.data(), sizeof(float) * flat.size());
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_im2col(int B, int C, int H, int W, int kh, int kw, int s, const double* x, double* P) {
  try {
    Tensor<double> f(Shape::hwcn(H, W, C, B));
    std::memcpy(f.data.data(), x, sizeof(double) * f.data.size());
    PatchMatrix<double> p = im2col(f, kh, kw, s);
    std::memcpy(P, p.mat.data.data(), sizeof(double) * p.mat.data.size());
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_col2im_map(int B, int C, int H, int W, int kh, int kw, int s, int64_t* src,
                   int64_t* tgt) {
  try {
    ConvGeometry g(Shape::hwcn(H, W, C, B), kh, kw, s);
    IndexMap m = build_col2im_map(g);
    std::memcpy(src, m.source.data(), sizeof(int64_t) * m.source.size());
    std::memcpy(tgt, m.target.data(), sizeof(int64_t) * m.target.size());
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_col2im(int B, int C, int H, int W, int kh, int kw, int s, const double* dP, double* dX) {
  try {
    ConvGeometry g(Shape::hwcn(H, W, C, B), kh, kw, s);
    Matrix<double> m(g.patch_len(), g.cols());
    std::memcpy(m.data.data(), dP, sizeof(double) * m.data.size());
    Tensor<double> t = col2im(m, g, build_col2im_map(g));
    std::memcpy(dX, t.data.data(), sizeof(double) * t.data.size());
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_pool_map(int B, int C, int H, int W, int ph, int pw, int s, int64_t* src, int64_t* tgt) {
  try {
    PoolGeometry g(Shape::hwcn(H, W, C, B), ph, pw, s, PoolMode::max);
    IndexMap m = build_pool_map(g);
    std::memcpy(src, m.source.data(), sizeof(int64_t) * m.source.size());
    std::memcpy(tgt, m.target.data(), sizeof(int64_t) * m.target.size());
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_pool_forward(int B, int C, int H, int W, int ph, int pw, int s, int mode,
                     const double* x, double* y, int64_t* arg) {
  try {
    Tensor<double> f(Shape::hwcn(H, W, C, B));
    std::memcpy(f.data.data(), x, sizeof(double) * f.data.size());
    PoolGeometry g(f.shape, ph, pw, s, mode ? PoolMode::avg : PoolMode::max);
    auto [o, a] = pool_forward(f, g);
    std::memcpy(y, o.data.data(), sizeof(double) * o.data.size());
    for (int64_t t = 0; t < g.output_size(); ++t) arg[t] = a.empty() ? -1 : a[t];
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_pool_backward(int B, int C, int H, int W, int ph, int pw, int s, int mode, int bwd_mode,
                      const double* dy, const int64_t* arg, double* dx) {
  try {
    PoolGeometry g(Shape::hwcn(H, W, C, B), ph, pw, s, mode ? PoolMode::avg : PoolMode::max);
    Tensor<double> go(g.output_shape());
    std::memcpy(go.data.data(), dy, sizeof(double) * go.data.size());
    ArgIndex a;
    if (!mode) a.assign(arg, arg + g.output_size());
    Tensor<double> gi = pool_backward(go, g, a, bwd_mode ? PoolBackwardMode::paper_nn
                                                         : PoolBackwardMode::exact);
    std::memcpy(dx, gi.data.data(), sizeof(double) * gi.data.size());
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

int ref_synth_bench_data(const orc_net* n, int B, uint64_t seed, float* x, int* cls,
                         float* values) {
  try {
    NetworkSpec spec = spec_of(n);
    Rng rng(seed);
    const int64_t nx = static_cast<int64_t>(n->in_h) * n->in_w * n->in_c * B;
    for (int64_t i = 0; i < nx; ++i) x[i] = static_cast<float>(rng.uniform());
    const Shape out = spec.output_shape();
    if (spec.loss == LossKind::softmax_ce) {
      const int units = static_cast<int>(out.numel());
      for (int b = 0; b < B; ++b) cls[b] = rng.uniform_int(units);
    } else {
      const int64_t nv = out.numel() * B;
      for (int64_t i = 0; i < nv; ++i) values[i] = static_cast<float>(rng.uniform());
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// ---- CPU baseline: reference Executor<float>(imp6) run_batch + sgd_step ----
void* ref_bench_create(const orc_net* n, int B, uint64_t data_seed, double lr, double mom) {
  try {
    auto* st = new BenchState();
    st->spec = spec_of(n);
    st->net = build_network<float>(st->spec);
    st->batch = Tensor<float>(Shape::hwcn(n->in_h, n->in_w, n->in_c, B));
    std::vector<int> cls(B);
    Shape o = st->spec.output_shape();
    std::vector<float> vals(static_cast<size_t>(o.numel() * B));
    ref_synth_bench_data(n, B, data_seed, st->batch.data.data(), cls.data(), vals.data());
    if (st->spec.loss == LossKind::softmax_ce) {
      st->targets = Targets<float>::from_classes(cls);
    } else {
      Tensor<float> v(Shape::hwcn(o.h(), o.w(), o.c(), B), vals);
      st->targets = Targets<float>::from_values(std::move(v));
    }
    st->cfg.lr = lr;
    st->cfg.momentum = mom;
    return st;
  } catch (const std::exception& e) {
    status_of(e);
    return nullptr;
  }
}

// the reference's vectorization ladder (Variant::imp1..imp6, variants.hpp:71-242)
void ref_bench_set_variant(void* h, int variant) {
  static_cast<BenchState*>(h)->exec = Executor<float>(variant_of(variant));
}

// One training step (forward + backward + update); returns the loss.
float ref_bench_step(void* h, int train) {
  auto* st = static_cast<BenchState*>(h);
  if (!train) {
    Tensor<float> o = st->exec.forward(st->net, st->batch);
    return o.data.empty() ? 0.f : o.data[0];
  }
  RunResult<float> r = st->exec.run_batch(st->net, st->batch, &st->targets);
  sgd_step(st->net, r.grads, st->cfg, st->vel);
  st->last_loss = r.loss;
  return r.loss;
}

void ref_bench_get_params(void* h, float* out) {
  params_to_flat(static_cast<BenchState*>(h)->net, out);
}

void ref_bench_destroy(void* h) { delete static_cast<BenchState*>(h); }

}  // extern "C"
