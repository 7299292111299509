// C++ host API (include/vcnn_b200/vcnn_b200.hpp) on the device: the
// reference-shaped surface end to end.  Run by tests/test_cpp_api.py.
#include <cmath>
#include <cstdio>
#include <vector>

#include "vcnn_b200/vcnn_b200.hpp"

using namespace vcnn_b200;

static int failures = 0;
#define EXPECT(cond, msg)                          \
  do {                                             \
    if (!(cond)) {                                 \
      std::printf("FAIL: %s (%s)\n", msg, #cond);  \
      ++failures;                                  \
    } else {                                       \
      std::printf("ok: %s\n", msg);                \
    }                                              \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  // NetworkSpec::chain (network.hpp:45-67) and its ShapeError
  NetworkSpec spec;
  spec.input = Shape{12, 12, 2};
  spec.layers = {ConvSpec{4, 3, 3, 1, Activation::relu}, PoolSpec{2, 2, 2},
                 FullSpec{3, Activation::identity}};
  spec.seed = 5;
  auto ch = spec.chain();
  EXPECT(ch.size() == 3 && ch[0].h == 10 && ch[1].h == 5 && ch[2].c == 3, "chain shapes");
  NetworkSpec bad = spec;
  bad.layers = {ConvSpec{2, 15, 15}};
  EXPECT(throws<ShapeError>([&] { bad.chain(); }), "broken chain -> ShapeError");
  EXPECT(throws<ConfigError>([&] { TrainConfig c; c.lr = 0; c.validate(); }), "lr <= 0 -> ConfigError");

  // build_network + Executor::run_batch + sgd_step
  const int B = 8;
  Network net = build_network(spec, B);
  std::vector<float> x((size_t)B * 12 * 12 * 2);
  for (size_t i = 0; i < x.size(); ++i) x[i] = (float)((i * 37 % 101) / 101.0);
  auto t = Targets<float>::from_classes({0, 1, 2, 0, 1, 2, 0, 1});
  Executor ex;
  RunResult r = ex.run_batch(net, x.data(), B, &t);
  EXPECT(r.has_grads && std::isfinite(r.loss) && r.loss > 0, "run_batch loss");
  EXPECT(r.output.size() == (size_t)B * 3, "output shape");
  auto g = net.grads();
  double gn = 0;
  for (float v : g) gn += (double)v * v;
  EXPECT(gn > 0, "gradients on device");
  auto p0 = net.params();
  TrainConfig cfg;
  cfg.lr = 0.1;
  cfg.momentum = 0.9;
  sgd_step(net, cfg);
  auto p1 = net.params();
  double dmax = 0;
  for (size_t i = 0; i < p0.size(); ++i) dmax = std::fmax(dmax, std::fabs(p1[i] - p0[i] + 0.1 * g[i]));
  EXPECT(dmax < 1e-6, "sgd_step: first step is w -= lr*g");
  auto bad_t = Targets<float>::from_classes({0, 1, 2, 0, 1, 2, 0, 7});
  EXPECT(throws<BoundsError>([&] { ex.run_batch(net, x.data(), B, &bad_t); }),
         "class out of range -> BoundsError");
  EXPECT(throws<ShapeError>([&] { ex.run_batch(net, x.data(), B + 1, &t); }),
         "batch > max_batch -> ShapeError");
  auto out = ex.forward(net, x.data(), 2);
  EXPECT(out.size() == 6, "forward");

  // Trainer::fit / evaluate_accuracy on a separable toy set
  NetworkSpec ts;
  ts.input = Shape{6, 6, 1};
  ts.layers = {ConvSpec{4, 3, 3, 1, Activation::relu}, PoolSpec{2, 2, 2},
               FullSpec{2, Activation::identity}};
  ts.seed = 12;
  const int n = 64;
  std::vector<float> imgs((size_t)n * 36);
  std::vector<int> labels((size_t)n);
  for (int i = 0; i < n; ++i) {
    labels[(size_t)i] = i % 2;
    for (int k = 0; k < 36; ++k) {
      float v = (float)(((i * 131 + k * 71) % 97) / 97.0 * 0.2);
      if (labels[(size_t)i] == 1 && k < 18) v += 0.8f;
      imgs[(size_t)i * 36 + (size_t)k] = v;
    }
  }
  Network tn = build_network(ts, n);
  TrainConfig tc;
  tc.lr = 0.05;
  tc.momentum = 0.9;
  tc.batch = n;
  tc.epochs = 20;
  tc.seed = 4;
  Trainer tr(tc);
  auto hist = tr.fit(tn, imgs, Targets<float>::from_classes(labels));
  EXPECT(hist.back() < hist.front(), "fit lowers the loss");
  EXPECT(tr.evaluate_accuracy(tn, imgs, labels) > 0.9, "accuracy > 0.9");

  // data parallelism in one process: 2 replicas (logical shards of one
  // device) trained by Trainer::fit_group follow the single-net Trainer on
  // the same global batches (3xTF32), and stay bit-identical to each other
  {
    const int n2 = 40, gb = 16;  // batches 16, 16, 8
    TrainConfig dc;
    dc.lr = 0.05;
    dc.momentum = 0.9;
    dc.batch = gb;
    dc.epochs = 2;
    dc.seed = 9;
    auto tg = Targets<float>::from_classes(std::vector<int>(labels.begin(), labels.begin() + n2));
    std::vector<float> im(imgs.begin(), imgs.begin() + (size_t)n2 * 36);
    Network single(ts, gb, Precision::tf32x3);
    auto h1 = Trainer(dc).fit(single, im, tg);
    Network r0(ts, gb / 2, Precision::tf32x3), r1(ts, gb / 2, Precision::tf32x3);
    std::vector<Network*> reps{&r0, &r1};
    auto dps = DataParallel::group(reps);
    auto h2 = Trainer(dc).fit_group(reps, dps, im, tg);
    double le = 0;
    for (size_t e = 0; e < h1.size(); ++e) le = std::fmax(le, std::fabs(h1[e] - h2[e]) / h1[e]);
    EXPECT(h2.size() == 2 && le < 1e-5, "fit_group epoch losses == single-net fit");
    auto ps = single.params(), p0 = r0.params(), p1 = r1.params();
    double pe = 0, pm = 0;
    bool same = p0 == p1;
    for (size_t i = 0; i < ps.size(); ++i) {
      pe = std::fmax(pe, std::fabs(p0[i] - ps[i]));
      pm = std::fmax(pm, std::fabs(ps[i]));
    }
    EXPECT(same, "replicas bit-identical");
    EXPECT(pe / pm < 1e-5, "fit_group weights == single-net weights");
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL OK", failures);
  return failures ? 1 : 0;
}
