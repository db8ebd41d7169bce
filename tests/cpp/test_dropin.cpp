// C++ drop-in test: the reference's own test cases (tests/test_model.cpp) written
// against include/hmtl_b200.hpp, i.e. what a reference user's code looks like
// after `using namespace hmtl::b200`.  Built and run by tests/test_gpu_cpp.py.
#include <cmath>
#include <cstdio>
#include <random>

#include "hmtl_b200.hpp"

using namespace hmtl::b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    ++g_checks;                                                    \
    if (!(c)) {                                                    \
      ++g_fail;                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
    }                                                              \
  } while (0)
#define CHECK_THROWS_CODE(expr, want)                               \
  do {                                                              \
    bool thrown = false;                                            \
    try {                                                           \
      (void)(expr);                                                 \
    } catch (const Error& e) {                                      \
      thrown = e.code() == (want);                                  \
    }                                                               \
    CHECK(thrown);                                                  \
  } while (0)

static ModelHyper tiny_hyper(int n_heads, int hidden = 8) {  // tests/test_model.cpp:17-26
  ModelHyper hp;
  hp.layers = 2;
  hp.hidden = hidden;
  hp.head_width = hidden;
  hp.head_depth = 3;
  hp.n_heads = n_heads;
  hp.cutoff = 5.0;
  return hp;
}

static AtomisticSample random_sample(std::mt19937_64& rng, int n, uint8_t ds) {
  std::uniform_real_distribution<double> u(0.0, 3.5);
  AtomisticSample s;
  s.dataset_id = ds;
  for (int i = 0; i < n; ++i) {
    s.species.push_back(uint8_t(rng() % 20));
    for (int k = 0; k < 3; ++k) s.positions.push_back(u(rng));
  }
  s.forces.assign(3 * n, 0.0);
  s.energy_per_atom = 0.25;
  return s;
}

int main() {
  // single node, no edges (tests/test_model.cpp:87-108)
  {
    auto hp = tiny_hyper(1);
    ModelT<float> m(hp, 5, {0});
    AtomisticSample s;
    s.species = {3};
    s.positions = {1.0, 2.0, 3.0};
    s.forces = {0, 0, 0};
    auto batch = build_batch<float>({s}, hp.cutoff);
    CHECK(batch.n_edges() == 0);
    ForwardCacheT<float> cache;
    auto pred = m.forward(batch, &cache);
    CHECK(pred.forces[0] == 0.0f);
    CHECK(std::isfinite(pred.energy_per_atom[0]));
  }
  // empty graph rejected (:110-115)
  CHECK_THROWS_CODE(build_batch<float>({AtomisticSample{}}, 5.0), ErrorCode::contract);
  // unknown dataset id rejected (:117-125)
  {
    auto hp = tiny_hyper(2);
    ModelT<float> m(hp, 5, {0});
    std::mt19937_64 rng(2);
    auto s = random_sample(rng, 3, 1);
    auto batch = build_batch<float>({s}, hp.cutoff);
    ForwardCacheT<float> cache;
    CHECK_THROWS_CODE(m.forward(batch, &cache), ErrorCode::contract);
  }
  // two-atom antisymmetry, bit-exact (:225-239)
  {
    auto hp = tiny_hyper(1);
    ModelT<float> m(hp, 9, {0});
    AtomisticSample s;
    s.species = {2, 4};
    s.positions = {0.3, -0.2, 0.1, 1.4, 0.8, -0.5};
    s.forces.assign(6, 0.0);
    auto batch = build_batch<float>({s}, hp.cutoff);
    CHECK(batch.n_edges() == 2);
    ForwardCacheT<float> cache;
    auto pred = m.forward(batch, &cache);
    for (int k = 0; k < 3; ++k) CHECK(pred.forces[k] == -pred.forces[3 + k]);
  }
  // zero upstream -> zero gradients (:320-332)
  {
    auto hp = tiny_hyper(1);
    ModelT<float> m(hp, 3, {0});
    std::mt19937_64 rng(8);
    auto batch = build_batch<float>({random_sample(rng, 4, 0)}, hp.cutoff);
    ForwardCacheT<float> cache;
    (void)m.forward(batch, &cache);
    auto g = m.backward(batch, cache, std::vector<float>(1, 0.f), std::vector<float>(3 * batch.n_nodes(), 0.f));
    bool all0 = true;
    for (float v : g.shared) all0 &= v == 0.f;
    for (float v : g.heads.at(0)) all0 &= v == 0.f;
    CHECK(all0);
  }
  // momentum conservation per graph (:297-318), FP32 tolerance
  {
    auto hp = tiny_hyper(2);
    ModelT<float> m(hp, 19, {0, 1});
    std::mt19937_64 rng(41);
    std::vector<AtomisticSample> ss;
    for (int g = 0; g < 6; ++g) ss.push_back(random_sample(rng, 2 + int(rng() % 6), uint8_t(g % 2)));
    auto batch = build_batch<float>(ss, hp.cutoff);
    ForwardCacheT<float> cache;
    auto pred = m.forward(batch, &cache);
    for (int g = 0; g < batch.n_graphs; ++g) {
      double sx = 0, sy = 0, sz = 0;
      for (int i = batch.graph_offset[g]; i < batch.graph_offset[g + 1]; ++i) {
        sx += pred.forces[3 * i];
        sy += pred.forces[3 * i + 1];
        sz += pred.forces[3 * i + 2];
      }
      CHECK(std::fabs(sx) < 1e-4 && std::fabs(sy) < 1e-4 && std::fabs(sz) < 1e-4);
    }
  }
  // census (:423-456)
  {
    auto hp = tiny_hyper(3);
    ModelT<float> full(hp, 1, {0, 1, 2}), shard(hp, 1, {1});
    CHECK(full.param_count() == memory_footprint(full.shared_size(), full.head_size(), 3, RunMode::base));
    CHECK(shard.param_count() == memory_footprint(shard.shared_size(), shard.head_size(), 3, RunMode::taskpar));
    auto pp = ModelHyper::paper_preset(5);
    ModelT<float> p(pp, 2, {0});
    CHECK(p.shared_size() == 18033584 && p.head_size() == 3126615);
    CHECK(classify_regime(p.shared_size(), p.head_size(), 5) == ParallelRegime::case3);
  }
  // trainer: the loss goes down on a fixed batch
  {
    auto hp = tiny_hyper(2, 16);
    ModelT<float> m(hp, 7, {0, 1});
    std::mt19937_64 rng(3);
    std::vector<AtomisticSample> ss;
    for (int g = 0; g < 8; ++g) ss.push_back(random_sample(rng, 3 + int(rng() % 5), uint8_t(g % 2)));
    auto batch = build_batch<float>(ss, hp.cutoff);
    Trainer t(m, TrainConfig{});
    float first = t.train_step(batch), last = first;
    for (int i = 0; i < 30; ++i) last = t.train_step(batch);
    CHECK(last < first);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
