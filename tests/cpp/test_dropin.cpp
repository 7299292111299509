// The drop-in, literally: the REFERENCE's own objects (vcnn::build_network,
// vcnn::Tensor, vcnn::Targets, vcnn::RunResult, vcnn::sgd_step) with only
// the Executor swapped -- vcnn::Executor<float>(imp6) on the host vs
// vcnn_b200::ref::Executor on the B200 -- compared on identical inputs.
// Built against /root/reference/proj headers in the build container
// (tests/cpp/Makefile), run on the GPU box by tests/test_cpp_api.py.
#include <cmath>
#include <cstdio>

#include "vcnn/training.hpp"
#include "vcnn_b200/reference_adapter.hpp"

static double normwise(const std::vector<float>& a, const std::vector<float>& b) {
  double m = 0, e = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    m = std::fmax(m, std::fabs((double)b[i]));
    e = std::fmax(e, std::fabs((double)a[i] - (double)b[i]));
  }
  return m > 0 ? e / m : e;
}

template <class T>
static std::vector<float> flat(const vcnn::NetGrads<T>& g) {
  std::vector<float> v;
  for (const auto& l : g.layers) {
    v.insert(v.end(), l.weights.data.begin(), l.weights.data.end());
    v.insert(v.end(), l.bias.begin(), l.bias.end());
  }
  return v;
}

static double normwise64(const std::vector<float>& a, const std::vector<double>& b) {
  double m = 0, e = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    m = std::fmax(m, std::fabs(b[i]));
    e = std::fmax(e, std::fabs((double)a[i] - b[i]));
  }
  return m > 0 ? e / m : e;
}

template <class T>
static std::vector<double> flat64(const vcnn::NetGrads<T>& g) {
  std::vector<double> v;
  for (const auto& l : g.layers) {
    v.insert(v.end(), l.weights.data.begin(), l.weights.data.end());
    v.insert(v.end(), l.bias.begin(), l.bias.end());
  }
  return v;
}

// the same network in f64 (the reference's Executor<double>: the parity oracle)
static vcnn::Network<double> as_f64(const vcnn::Network<float>& net) {
  vcnn::Network<double> d = vcnn::build_network<double>(net.spec);
  const std::vector<float> p = vcnn_b200::ref::flat_params(net);
  size_t off = 0;
  for (auto& layer : d.layers)
    std::visit(
        [&](auto& l) {
          using L = std::decay_t<decltype(l)>;
          if constexpr (!std::is_same_v<L, vcnn::PoolLayer<double>>)
            for (auto& w : l.weights.data) w = p[off++];
          for (auto& b : l.bias) b = p[off++];
        },
        layer);
  return d;
}

int main() {
  int fails = 0;
  vcnn::NetworkSpec spec;  // CIFAR-3 shape (BASELINE configs[1]) at batch 16
  spec.input = vcnn::Shape{32, 32, 3};
  spec.layers = {vcnn::ConvSpec{32, 5, 5, 1, vcnn::Activation::relu}, vcnn::PoolSpec{},
                 vcnn::ConvSpec{32, 5, 5, 1, vcnn::Activation::relu}, vcnn::PoolSpec{},
                 vcnn::ConvSpec{64, 5, 5, 1, vcnn::Activation::relu},
                 vcnn::FullSpec{10, vcnn::Activation::identity}};
  spec.seed = 7;
  const int B = 16;
  vcnn::Network<float> net = vcnn::build_network<float>(spec);
  vcnn::Tensor<float> x(vcnn::Shape::hwcn(32, 32, 3, B));
  vcnn::Rng rng(8);
  for (auto& v : x.data) v = (float)rng.uniform();
  std::vector<int> cls(B);
  for (auto& c : cls) c = rng.uniform_int(10);
  auto t = vcnn::Targets<float>::from_classes(cls);

  vcnn::Executor<float> host(vcnn::Variant::imp6);
  // the reference itself in f64 on the same (fp32) values: the parity bar
  vcnn::Network<double> net64 = as_f64(net);
  vcnn::Tensor<double> x64(x.shape);
  std::copy(x.data.begin(), x.data.end(), x64.data.begin());
  auto t64 = vcnn::Targets<double>::from_classes(cls);
  auto r64 = vcnn::Executor<double>(vcnn::Variant::imp6).run_batch(net64, x64, &t64);
  for (auto prec : {vcnn_b200::Precision::tf32x3, vcnn_b200::Precision::tf32}) {
    vcnn_b200::ref::Executor dev(prec);  // <- the only line that changes
    const double tol = prec == vcnn_b200::Precision::tf32 ? 1e-3 : 1e-5;
    auto rh = host.run_batch(net, x, &t);
    auto rd = dev.run_batch(net, x, &t);
    const double eo = normwise(rd.output.data, rh.output.data);
    const double el = std::fabs(rd.loss - rh.loss) / std::fabs(rh.loss);
    std::printf("%s: output %.2e  loss %.2e", prec == vcnn_b200::Precision::tf32 ? "tf32" : "3xtf32",
                eo, el);
    bool ok = eo <= tol && el <= tol && rd.has_grads;
    if (prec == vcnn_b200::Precision::tf32x3) {  // every NetGrads tensor, fp32-faithful path
      // vs the reference in f64 at 1e-5 (the reference's own float build's
      // distance from its f64 build printed beside it)
      const double eg = normwise64(flat(rd.grads), flat64(r64.grads));
      const double eh = normwise64(flat(rh.grads), flat64(r64.grads));
      std::printf("  grads vs f64 %.2e (reference float: %.2e)", eg, eh);
      ok = ok && eg <= tol;
      // 3 reference sgd_steps on each side, weights after
      vcnn::Network<float> nh = net, nd = net;
      vcnn::Velocity<float> vh, vd;
      vcnn::TrainConfig cfg;
      cfg.lr = 0.01;
      cfg.momentum = 0.9;
      for (int s = 0; s < 3; ++s) {
        vcnn::sgd_step(nh, host.run_batch(nh, x, &t).grads, cfg, vh);
        vcnn::sgd_step(nd, dev.run_batch(nd, x, &t).grads, cfg, vd);
      }
      const double ew = normwise(vcnn_b200::ref::flat_params(nd), vcnn_b200::ref::flat_params(nh));
      std::printf("  weights after 3 steps %.2e", ew);
      ok = ok && ew <= 1e-5;
    }
    std::printf("  -> %s\n", ok ? "ok" : "FAIL");
    fails += !ok;
  }
  // Executor::set_timer (variants.hpp:341): the reference's BreakdownTimer
  // filled per component by the device executor
  {
    vcnn::BreakdownTimer bt;
    vcnn_b200::ref::Executor dev;
    dev.set_timer(&bt);
    dev.run_batch(net, x, &t);
    using C = vcnn::Component;
    const bool tok = bt.seconds[(int)C::conv_f] > 0 && bt.seconds[(int)C::conv_b] > 0 &&
                     bt.seconds[(int)C::pool_f] > 0 && bt.seconds[(int)C::pool_b] > 0 &&
                     bt.seconds[(int)C::full_f] > 0 && bt.seconds[(int)C::full_b] > 0 &&
                     bt.total() < 1.0;
    std::printf("set_timer: conv_f %.1f us pool_f %.1f us full_f %.1f us total %.1f us -> %s\n",
                1e6 * bt.seconds[(int)C::conv_f], 1e6 * bt.seconds[(int)C::pool_f],
                1e6 * bt.seconds[(int)C::full_f], 1e6 * bt.total(), tok ? "ok" : "FAIL");
    fails += !tok;
  }
  auto f = vcnn_b200::ref::Executor().forward(net, x);
  auto fh = host.forward(net, x);
  const double ef = normwise(f.data, fh.data);
  std::printf("forward: %.2e -> %s\n", ef, ef <= 1e-3 ? "ok" : "FAIL");
  fails += ef > 1e-3;
  std::printf("%s\n", fails ? "FAILED" : "ALL OK");
  return fails ? 1 : 0;
}
