// hmtl_b200.hpp -- C++ drop-in for the reference's hot-path API, backed by the
// B200 C ABI (hmtl_b200.h).  Mirrors, name for name, what a caller of
// /root/reference/proj/include/hmtl uses on the training-step path:
//
//   hmtl::ErrorCode / hmtl::Error         hmtl/error.hpp:8-34
//   hmtl::ModelHyper                      hmtl/model.hpp:17-37
//   hmtl::AtomisticSample                 hmtl/graph.hpp:13-21
//   hmtl::GraphBatchT<float>              hmtl/graph.hpp:27-42
//   hmtl::build_batch<float>              hmtl/graph.hpp:46-83   (runs on the GPU)
//   hmtl::PredictionT / GradientBufferT   hmtl/model.hpp:92-115
//   hmtl::ForwardCacheT<float>            hmtl/model.hpp:144-151 (device-resident, opaque)
//   hmtl::ModelT<float>                   hmtl/model.hpp:155-242
//   hmtl::classify_regime / memory_footprint  hmtl/model.hpp:246-263
//   hmtl::Trainer::train_step             SPEC.md:392-409 (no reference code)
//
// Differences a caller sees: parameters live on the
// device, so shared_block()/head_block(k) return host COPIES and writes go
// through set_shared_block()/set_head_block(); only S = float is provided
// (the FP32 path); the forward cache is opaque and lives on the device.
// Switching is `#include "hmtl_b200.hpp"` + `using namespace hmtl::b200;`.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hmtl_b200.h"

namespace hmtl {
namespace b200 {

enum class ErrorCode { contract = 1, io = 2, comm = 3, data = 4, config = 5, internal = 6 };

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& what) : std::runtime_error(what), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

inline void check(int rc) {
  if (rc != HMTL_OK) throw Error(static_cast<ErrorCode>(rc), hmtl_last_error());
}

struct ModelHyper {
  int n_species = 20;
  int layers = 2;
  int hidden = 32;
  int head_width = 32;
  int head_depth = 3;
  int n_heads = 1;
  double cutoff = 5.0;
  static ModelHyper paper_preset(int n_heads) {
    ModelHyper hp;
    hp.layers = 4;
    hp.hidden = 866;
    hp.head_width = 889;
    hp.head_depth = 3;
    hp.n_heads = n_heads;
    return hp;
  }
  hmtl_hyper c() const { return {n_species, layers, hidden, head_width, head_depth, n_heads, cutoff}; }
};

struct AtomisticSample {
  std::vector<uint8_t> species;
  std::vector<double> positions;
  std::vector<double> forces;
  double energy_per_atom = 0.0;
  uint8_t dataset_id = 0;
  size_t n_atoms() const { return species.size(); }
};

// Host view of a batch; the edge list is computed on the device.
template <typename S>
struct GraphBatchT {
  int n_graphs = 0;
  std::vector<int> graph_offset, edge_offset;
  std::vector<S> positions;
  std::vector<uint8_t> species;
  std::vector<int> edge_dst, edge_src;
  std::vector<uint8_t> dataset_id;
  std::vector<S> label_energy, label_force;
  // packed samples (what the device consumes)
  std::vector<int> n_atoms_;
  std::vector<double> pos64_, force64_, energy64_;
  int n_nodes() const { return static_cast<int>(species.size()); }
  int n_edges() const { return static_cast<int>(edge_dst.size()); }
  int graph_nodes(int g) const { return graph_offset[g + 1] - graph_offset[g]; }
  hmtl_samples c() const {
    return {n_graphs, n_nodes(), n_atoms_.data(), species.data(), pos64_.data(), force64_.data(),
            energy64_.data(), dataset_id.data()};
  }
};

template <typename S>
struct PredictionT {
  std::vector<S> energy_per_atom;
  std::vector<S> forces;
};

template <typename S>
struct GradientBufferT {
  std::vector<S> shared;
  std::map<int, std::vector<S>> heads;
  void scale(S f) {
    for (S& v : shared) v *= f;
    for (auto& kv : heads)
      for (S& v : kv.second) v *= f;
  }
  void accumulate(const GradientBufferT& o) {
    for (size_t i = 0; i < shared.size(); ++i) shared[i] += o.shared[i];
    for (auto& kv : heads) {
      const auto& oh = o.heads.at(kv.first);
      for (size_t i = 0; i < kv.second.size(); ++i) kv.second[i] += oh[i];
    }
  }
};

template <typename S>
struct ForwardCacheT {
  const void* owner = nullptr;  // the ModelT whose device cache holds this forward
};

enum class ParallelRegime { case1 = 1, case2 = 2, case3 = 3 };
enum class RunMode { serial = 0, base = 1, taskpar = 2 };
inline ParallelRegime classify_regime(size_t p_s, size_t p_h, int n_h) {
  const int r = hmtl_classify_regime(p_s, p_h, n_h);
  if (r < 0) check(-r);
  return static_cast<ParallelRegime>(r);
}
inline size_t memory_footprint(size_t p_s, size_t p_h, int n_h, RunMode mode) {
  return hmtl_memory_footprint(p_s, p_h, n_h, static_cast<int>(mode));
}

namespace detail {
inline hmtl_caps caps_for(const std::vector<int>& n_atoms) {
  long long bound = 0, N = 0;
  for (int n : n_atoms) {
    bound += (long long)n * (n - 1);
    N += n;
  }
  return {int(n_atoms.size()), int(N > 0 ? N : 1), bound > 0 ? bound : 1};
}
struct Ctx {
  hmtl_ctx* p = nullptr;
  ~Ctx() { hmtl_ctx_destroy(p); }
};
}  // namespace detail

template <typename S>
class ModelT;

// build_batch<float>: concatenates the samples on the host and runs the
// bit-exact FP64 neighbour search on the GPU (device 0).
template <typename S>
GraphBatchT<S> build_batch(const std::vector<AtomisticSample>& samples, double cutoff, int device = 0);

template <>
class ModelT<float> {
 public:
  ModelT(const ModelHyper& hp, uint64_t seed, std::vector<int> owned_heads, int device = 0)
      : hp_(hp), seed_(seed), owned_(std::move(owned_heads)), device_(device) {
    create({64, 4096, 1 << 17});
  }
  const ModelHyper& hyper() const { return hp_; }
  size_t shared_size() const {
    hmtl_hyper h = hp_.c();
    return hmtl_shared_size(&h);
  }
  size_t head_size() const {
    hmtl_hyper h = hp_.c();
    return hmtl_head_size(&h);
  }
  int n_owned_heads() const { return int(owned_.size()); }
  bool owns_head(int k) const {
    for (int o : owned_)
      if (o == k) return true;
    return false;
  }
  size_t param_count() const { return shared_size() + owned_.size() * head_size(); }
  std::vector<float> shared_block() const { return get(-1, shared_size()); }
  std::vector<float> head_block(int k) const { return get(k, head_size()); }
  void set_shared_block(const std::vector<float>& v) { check(hmtl_set_block(ctx_->p, -1, v.data())); }
  void set_head_block(int k, const std::vector<float>& v) { check(hmtl_set_block(ctx_->p, k, v.data())); }
  GradientBufferT<float> zero_grads() const {
    GradientBufferT<float> g;
    g.shared.assign(shared_size(), 0.f);
    for (int k : owned_) g.heads[k].assign(head_size(), 0.f);
    return g;
  }

  PredictionT<float> forward(const GraphBatchT<float>& b, ForwardCacheT<float>* cache) const {
    upload(b);
    check(hmtl_build_batch(ctx_->p, nullptr));
    check(hmtl_forward(ctx_->p, nullptr));
    PredictionT<float> p;
    p.energy_per_atom.resize(b.n_graphs);
    p.forces.resize(3 * size_t(b.n_nodes()));
    check(hmtl_predictions(ctx_->p, p.energy_per_atom.data(), p.forces.data()));
    if (cache) cache->owner = this;
    return p;
  }
  GradientBufferT<float> backward(const GraphBatchT<float>& b, const ForwardCacheT<float>& cache,
                                  const std::vector<float>& d_energy, const std::vector<float>& d_forces) const {
    if (cache.owner != this) throw Error(ErrorCode::contract, "model: missing forward cache");
    if (d_energy.size() != size_t(b.n_graphs) || d_forces.size() != 3 * size_t(b.n_nodes()))
      throw Error(ErrorCode::contract, "model: upstream shape mismatch");
    check(hmtl_backward(ctx_->p, d_energy.data(), d_forces.data(), nullptr));
    GradientBufferT<float> g = zero_grads();
    check(hmtl_get_grad(ctx_->p, -1, g.shared.data()));
    for (auto& kv : g.heads) check(hmtl_get_grad(ctx_->p, kv.first, kv.second.data()));
    return g;
  }
  hmtl_ctx* handle() const { return ctx_->p; }
  void reserve(const hmtl_caps& need) const {
    if (need.max_graphs <= caps_.max_graphs && need.max_nodes <= caps_.max_nodes &&
        need.max_edges <= caps_.max_edges)
      return;
    // in place: parameters, AdamW state, step counter and communicator survive
    const hmtl_caps grown{std::max(need.max_graphs, caps_.max_graphs), std::max(need.max_nodes, caps_.max_nodes),
                          std::max(need.max_edges, caps_.max_edges)};
    check(hmtl_ctx_reserve(ctx_->p, &grown));
    const_cast<ModelT*>(this)->caps_ = grown;
  }
  void upload(const GraphBatchT<float>& b) const {
    reserve(detail::caps_for(b.n_atoms_));
    hmtl_samples s = b.c();
    check(hmtl_batch_upload(ctx_->p, &s, nullptr));
  }

 private:
  void create(hmtl_caps caps) {
    auto c = std::make_shared<detail::Ctx>();
    hmtl_hyper h = hp_.c();
    check(hmtl_ctx_create(device_, &h, seed_, owned_.data(), int(owned_.size()), &caps, &c->p));
    ctx_ = c;
    caps_ = caps;
  }
  std::vector<float> get(int which, size_t n) const {
    std::vector<float> v(n);
    check(hmtl_get_block(ctx_->p, which, v.data()));
    return v;
  }
  ModelHyper hp_;
  uint64_t seed_;
  std::vector<int> owned_;
  int device_;
  hmtl_caps caps_{};
  std::shared_ptr<detail::Ctx> ctx_;
};

template <>
inline GraphBatchT<float> build_batch<float>(const std::vector<AtomisticSample>& samples, double cutoff,
                                             int device) {
  GraphBatchT<float> b;
  b.n_graphs = int(samples.size());
  b.graph_offset.push_back(0);
  for (const auto& s : samples) {
    if (s.n_atoms() < 1) throw Error(ErrorCode::contract, "build_batch: empty graph rejected");
    b.n_atoms_.push_back(int(s.n_atoms()));
    for (size_t i = 0; i < s.n_atoms(); ++i) {
      b.species.push_back(s.species[i]);
      for (int k = 0; k < 3; ++k) {
        b.positions.push_back(float(s.positions[3 * i + k]));
        b.label_force.push_back(float(s.forces[3 * i + k]));
        b.pos64_.push_back(s.positions[3 * i + k]);
        b.force64_.push_back(s.forces[3 * i + k]);
      }
    }
    b.graph_offset.push_back(b.n_nodes());
    b.dataset_id.push_back(s.dataset_id);
    b.label_energy.push_back(float(s.energy_per_atom));
    b.energy64_.push_back(s.energy_per_atom);
  }
  // device neighbour search (hmtl/graph.hpp:65-76 semantics, bit-exact), no model context
  const hmtl_samples cs = b.c();
  int E = 0;
  long long cap = 0;
  for (int n : b.n_atoms_) cap += (long long)n * (n - 1);
  b.edge_dst.resize(size_t(cap));
  b.edge_src.resize(size_t(cap));
  b.edge_offset.resize(b.n_graphs + 1);
  check(hmtl_nbr_build(device, &cs, cutoff, cap, &E, b.edge_dst.data(), b.edge_src.data(), b.edge_offset.data(),
                       nullptr, nullptr));
  b.edge_dst.resize(E);
  b.edge_src.resize(E);
  return b;
}

// SPEC trainer on one GPU; attach_comm() turns it into an
// MTL-par rank (head-group + global NCCL allreduce inside the step).
struct TrainConfig {
  float lr = 1e-3f, beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f, weight_decay = 0.01f;
  float w_energy = 1.f, w_force = 1.f;
  bool use_graph = true;
  hmtl_train_cfg c() const { return {lr, beta1, beta2, eps, weight_decay, w_energy, w_force, use_graph ? 1 : 0}; }
};

class Trainer {
 public:
  Trainer(ModelT<float>& m, TrainConfig cfg) : m_(m), cfg_(cfg) {}
  void attach_comm(const uint8_t id[128], int world, int rank) { check(hmtl_comm_init(m_.handle(), id, world, rank)); }
  // one step on `b` (uploads, builds edges, fwd, loss, bwd, sync, AdamW); returns the loss
  float train_step(const GraphBatchT<float>& b) {
    m_.upload(b);
    hmtl_train_cfg c = cfg_.c();
    check(hmtl_train_step(m_.handle(), &c, nullptr));
    float L = 0.f;
    check(hmtl_read_loss(m_.handle(), &L));
    return L;
  }

 private:
  ModelT<float>& m_;
  TrainConfig cfg_;
};

}  // namespace b200
}  // namespace hmtl
