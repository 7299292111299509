// reference_adapter.hpp -- the drop-in: run the reference's OWN objects
// (vcnn::Network<float>, vcnn::Tensor<float>, vcnn::Targets<float>,
// vcnn::RunResult<float>, vcnn::NetGrads<float>) through the B200 engine.
//
// Include AFTER the reference headers (proj/include/vcnn/variants.hpp).  A
// maintainer replaces
//     vcnn::Executor<float> exec(vcnn::Variant::imp6);
// with
//     vcnn_b200::ref::Executor exec;
// and keeps everything else -- build_network, Trainer, sgd_step, the
// RunResult fields -- unchanged (variants.hpp:333-359).  Each run_batch
// uploads the network's parameters (the caller may have updated them with
// the reference's host sgd_step), runs forward + loss + backward on the
// device, and returns the reference's RunResult with its NetGrads filled.
// For device-resident training use vcnn_b200::Network / Trainer directly.
#pragma once

#include <memory>
#include <variant>

#include "vcnn_b200.hpp"

namespace vcnn_b200 {
namespace ref {

inline Activation act_of(vcnn::Activation a) {
  switch (a) {
    case vcnn::Activation::relu: return Activation::relu;
    case vcnn::Activation::sigmoid: return Activation::sigmoid;
    case vcnn::Activation::tanh: return Activation::tanh;
    default: return Activation::identity;
  }
}

// vcnn::NetworkSpec (network.hpp:37-73) -> vcnn_b200::NetworkSpec
inline NetworkSpec spec_of(const vcnn::NetworkSpec& s) {
  NetworkSpec o;
  o.input = Shape{s.input.h(), s.input.w(), s.input.c()};
  o.loss = s.loss == vcnn::LossKind::mse ? LossKind::mse : LossKind::softmax_ce;
  o.seed = s.seed;
  for (const vcnn::LayerSpec& l : s.layers) {
    if (const auto* c = std::get_if<vcnn::ConvSpec>(&l)) {
      o.layers.push_back(ConvSpec{c->maps, c->kh, c->kw, c->stride, act_of(c->act)});
    } else if (const auto* p = std::get_if<vcnn::PoolSpec>(&l)) {
      o.layers.push_back(PoolSpec{p->ph, p->pw, p->stride,
                                  p->mode == vcnn::PoolMode::avg ? PoolMode::avg : PoolMode::max,
                                  p->bias, act_of(p->act)});
    } else {
      const auto& f = std::get<vcnn::FullSpec>(l);
      o.layers.push_back(FullSpec{f.units, act_of(f.act)});
    }
  }
  return o;
}

// parameters of a reference Network<float> in the engine's flat layout
// (per layer: weights row-major, then bias -- NetGrads order)
inline std::vector<float> flat_params(const vcnn::Network<float>& net) {
  std::vector<float> p;
  for (const auto& layer : net.layers) {
    std::visit(
        [&](const auto& l) {
          using L = std::decay_t<decltype(l)>;
          if constexpr (!std::is_same_v<L, vcnn::PoolLayer<float>>)
            p.insert(p.end(), l.weights.data.begin(), l.weights.data.end());
          p.insert(p.end(), l.bias.begin(), l.bias.end());
        },
        layer);
  }
  return p;
}

// flat gradients -> the reference's NetGrads<float> (network.hpp:203-233)
inline vcnn::NetGrads<float> net_grads(const vcnn::Network<float>& net,
                                       const std::vector<float>& flat) {
  vcnn::NetGrads<float> g = vcnn::NetGrads<float>::zeros_like(net);
  size_t off = 0;
  for (auto& lg : g.layers) {
    std::copy(flat.begin() + off, flat.begin() + off + lg.weights.data.size(),
              lg.weights.data.begin());
    off += lg.weights.data.size();
    std::copy(flat.begin() + off, flat.begin() + off + lg.bias.size(), lg.bias.begin());
    off += lg.bias.size();
  }
  return g;
}

// vcnn::Executor<float> with the same public methods (variants.hpp:333-359)
class Executor {
 public:
  explicit Executor(Precision p = Precision::tf32) : prec_(p), exec_(p) {}

  void set_pool_backward_mode(vcnn::PoolBackwardMode m) {
    mode_ = m;
    exec_.set_pool_backward_mode(m == vcnn::PoolBackwardMode::paper_nn
                                     ? PoolBackwardMode::paper_nn
                                     : PoolBackwardMode::exact);
  }
  vcnn::PoolBackwardMode pool_backward_mode() const { return mode_; }
  vcnn::Variant variant() const { return vcnn::Variant::imp6; }

  // Executor::set_timer (variants.hpp:341): per-component device time (CUDA
  // events around every layer op, conv / pool / full / other x fwd / bwd)
  // added to the reference's BreakdownTimer after each call.  While a timer
  // is set the device runs every layer in its own kernels (no conv+pool /
  // tail fusion), so the components separate as in the reference's Imp-6.
  void set_timer(vcnn::BreakdownTimer* t) {
    timer_ = t;
    if (dev_) configure_timing(*dev_);
  }

  vcnn::Tensor<float> forward(const vcnn::Network<float>& net, const vcnn::Tensor<float>& batch) {
    return run_batch(net, batch, nullptr).output;
  }

  vcnn::RunResult<float> run_batch(const vcnn::Network<float>& net,
                                   const vcnn::Tensor<float>& batch,
                                   const vcnn::Targets<float>* targets) {
    const int n = batch.n();
    Network& dev = device_for(net, n);
    dev.set_params(flat_params(net));
    Targets<float> t;
    const Targets<float>* tp = nullptr;
    if (targets) {
      if (net.spec.loss == vcnn::LossKind::softmax_ce) t.classes = targets->classes;
      else t.values = targets->values.data;
      tp = &t;
    }
    double before[8] = {0};
    if (timer_) check(vcnn_net_read_breakdown(dev.handle(), before));
    RunResult r = exec_.run_batch(dev, batch.data.data(), n, tp);
    if (timer_) {
      double after[8] = {0};
      check(vcnn_net_read_breakdown(dev.handle(), after));
      for (int c = 0; c < 8; ++c)
        timer_->add(static_cast<vcnn::Component>(c), after[c] - before[c]);
    }
    vcnn::RunResult<float> out;
    const vcnn::Shape o = net.spec.output_shape();
    out.output = vcnn::Tensor<float>(vcnn::Shape::hwcn(o.h(), o.w(), o.c(), n));
    std::copy(r.output.begin(), r.output.end(), out.output.data.begin());
    if (targets) {
      out.loss = r.loss;
      out.grads = net_grads(net, dev.grads());
      out.has_grads = true;
    }
    return out;
  }

 private:
  // one device network per (spec, batch capacity); rebuilt when either grows
  Network& device_for(const vcnn::Network<float>& net, int n) {
    if (!dev_ || n > dev_->max_batch() || !same_spec(net.spec)) {
      const int cap = dev_ && same_spec(net.spec) && n <= 2 * dev_->max_batch()
                          ? 2 * dev_->max_batch()
                          : n;
      dev_ = std::make_unique<Network>(spec_of(net.spec), cap, prec_);
      spec_ = net.spec;
      configure_timing(*dev_);
    }
    return *dev_;
  }
  bool same_spec(const vcnn::NetworkSpec& s) const {
    if (!dev_) return false;
    if (s.input.h() != spec_.input.h() || s.input.w() != spec_.input.w() ||
        s.input.c() != spec_.input.c() || s.loss != spec_.loss ||
        s.layers.size() != spec_.layers.size())
      return false;
    for (size_t i = 0; i < s.layers.size(); ++i) {
      if (s.layers[i].index() != spec_.layers[i].index()) return false;
      if (const auto* a = std::get_if<vcnn::ConvSpec>(&s.layers[i])) {
        const auto& b = std::get<vcnn::ConvSpec>(spec_.layers[i]);
        if (a->maps != b.maps || a->kh != b.kh || a->kw != b.kw || a->stride != b.stride ||
            a->act != b.act)
          return false;
      } else if (const auto* a = std::get_if<vcnn::PoolSpec>(&s.layers[i])) {
        const auto& b = std::get<vcnn::PoolSpec>(spec_.layers[i]);
        if (a->ph != b.ph || a->pw != b.pw || a->stride != b.stride || a->mode != b.mode ||
            a->bias != b.bias || a->act != b.act)
          return false;
      } else {
        const auto& fa = std::get<vcnn::FullSpec>(s.layers[i]);
        const auto& fb = std::get<vcnn::FullSpec>(spec_.layers[i]);
        if (fa.units != fb.units || fa.act != fb.act) return false;
      }
    }
    return true;
  }
  void configure_timing(Network& dev) {
    check(vcnn_net_set_trace(dev.handle(), timer_ ? 1 : 0));
    check(vcnn_net_enable_breakdown(dev.handle(), timer_ ? 1 : 0));
  }
  Precision prec_;
  vcnn::BreakdownTimer* timer_ = nullptr;
  vcnn_b200::Executor exec_;
  vcnn::PoolBackwardMode mode_ = vcnn::PoolBackwardMode::exact;
  std::unique_ptr<Network> dev_;
  vcnn::NetworkSpec spec_;
};

}  // namespace ref
}  // namespace vcnn_b200
