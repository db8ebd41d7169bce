// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile together with the reference's own sources where
// they lie (/root/reference/proj/src/{dataset,sample_io,model_io}.cpp and the
// header-only model in /root/reference/proj/include/hmtl), with the
// reference's own flags (-O3 -g, no -march: /root/reference/proj/CMakeLists.txt:10),
// into oracle/_ref/libhmtl_ref.so.  Uses:
//   * golden fixtures (tests/golden/make_golden.py) that pin oracle/hmtl_oracle.c;
//   * bench.py --impl reference and the cpu_baseline leg: the reference CPU
//     path (build_batch -> ModelT<float>::forward/backward) plus the SPEC
//     loss/AdamW, which the reference specifies but does not
//     implement.  Thread-parallel over structures (the reference model is
//     const and single-threaded per call; gradients of disjoint sub-batches are
//     summed, which is exact for the mean-over-graphs loss).
// Nothing here is linked into the product (paper_2506_21788_b200/).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "hmtl/datastore.hpp"
#include "hmtl/dataset.hpp"
#include "hmtl/graph.hpp"
#include "hmtl/model.hpp"
#include "hmtl/rng.hpp"
#include "hmtl/sample_io.hpp"

using namespace hmtl;

namespace {
thread_local std::string g_err;

struct RefHyper {
  int n_species, layers, hidden, head_width, head_depth, n_heads;
  double cutoff;
};

ModelHyper to_hp(const RefHyper* h) {
  ModelHyper hp;
  hp.n_species = h->n_species;
  hp.layers = h->layers;
  hp.hidden = h->hidden;
  hp.head_width = h->head_width;
  hp.head_depth = h->head_depth;
  hp.n_heads = h->n_heads;
  hp.cutoff = h->cutoff;
  return hp;
}

struct ModelBox {
  bool dbl;
  ModelT<double>* md = nullptr;
  ModelT<float>* mf = nullptr;
  ForwardCacheT<double> cd;
  ForwardCacheT<float> cf;
  GraphBatchT<double> bd;
  GraphBatchT<float> bf;
  ~ModelBox() {
    delete md;
    delete mf;
  }
};

std::vector<AtomisticSample> make_samples(int G, const int* n_atoms, const uint8_t* species,
                                          const double* pos, const double* forces,
                                          const double* energy, const uint8_t* dsid) {
  std::vector<AtomisticSample> ss(G);
  size_t at = 0;
  for (int g = 0; g < G; ++g) {
    const int n = n_atoms[g];
    AtomisticSample& s = ss[g];
    s.species.assign(species + at, species + at + n);
    s.positions.assign(pos + 3 * at, pos + 3 * (at + n));
    if (forces)
      s.forces.assign(forces + 3 * at, forces + 3 * (at + n));
    else
      s.forces.assign(3 * n, 0.0);
    s.energy_per_atom = energy ? energy[g] : 0.0;
    s.dataset_id = dsid ? dsid[g] : 0;
    at += n;
  }
  return ss;
}

// Per-graph SPEC loss with a global graph count.
template <typename S>
double spec_loss(const GraphBatchT<S>& b, const PredictionT<S>& p, double w_e, double w_f,
                 int G_total, std::vector<S>* dE, std::vector<S>* dF) {
  dE->assign(b.n_graphs, S(0));
  dF->assign(3 * b.n_nodes(), S(0));
  double acc = 0.0;
  for (int g = 0; g < b.n_graphs; ++g) {
    const int lo = b.graph_offset[g], hi = b.graph_offset[g + 1];
    const double n = double(hi - lo);
    const double de = double(p.energy_per_atom[g]) - double(b.label_energy[g]);
    double fe = 0.0;
    for (int i = lo; i < hi; ++i)
      for (int k = 0; k < 3; ++k) {
        const double r = double(p.forces[3 * i + k]) - double(b.label_force[3 * i + k]);
        fe += r * r;
        (*dF)[3 * i + k] = S(2.0 * w_f * r / (n * double(G_total)));
      }
    acc += w_e * de * de + w_f * fe / n;
    (*dE)[g] = S(2.0 * w_e * de / double(G_total));
  }
  return acc;
}

template <typename S>
void adamw(std::vector<S>& p, const std::vector<S>& g, std::vector<S>& m, std::vector<S>& v,
           long step, double lr, double b1, double b2, double eps, double wd) {
  const S bc1 = S(1.0 - std::pow(b1, double(step)));
  const S bc2s = S(std::sqrt(1.0 - std::pow(b2, double(step))));
  const S step_size = S(lr) / bc1;
  for (size_t i = 0; i < p.size(); ++i) {
    p[i] *= S(1.0 - lr * wd);
    m[i] = S(b1) * m[i] + S(1.0 - b1) * g[i];
    v[i] = S(b2) * v[i] + S(1.0 - b2) * g[i] * g[i];
    const S denom = std::sqrt(v[i]) / bc2s + S(eps);
    p[i] -= step_size * m[i] / denom;
  }
}

template <typename S>
void copy_out(const std::vector<S>& v, double* out) {
  if (!out) return;
  for (size_t i = 0; i < v.size(); ++i) out[i] = double(v[i]);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- dataset
// default5_specs(), /root/reference/proj/src/dataset.cpp:213-239
int ref_default5_spec(int id, uint8_t* elements, int* n_elements, int* n_min, int* n_max,
                      double* alpha, double* sigma, double* mu20, uint64_t* count) {
  auto specs = data::default5_specs();
  if (id < 0 || id >= int(specs.size())) return -1;
  const auto& s = specs[id];
  *n_elements = int(s.elements.size());
  for (size_t i = 0; i < s.elements.size(); ++i) elements[i] = s.elements[i];
  *n_min = s.n_min;
  *n_max = s.n_max;
  *alpha = s.alpha;
  *sigma = s.sigma;
  for (int e = 0; e < data::kNumElements; ++e) mu20[e] = s.mu[e];
  *count = s.count;
  return 0;
}

// generate_dataset(spec, seed), /root/reference/proj/src/dataset.cpp:106-161
void* ref_dataset_generate(int dataset_id, const uint8_t* elements, int n_elements, int n_min,
                           int n_max, double alpha, double sigma, const double* mu20,
                           uint64_t count, int64_t structure_seed, uint64_t seed) {
  try {
    data::DatasetSpec s;
    s.dataset_id = uint8_t(dataset_id);
    s.elements.assign(elements, elements + n_elements);
    s.n_min = n_min;
    s.n_max = n_max;
    s.alpha = alpha;
    s.sigma = sigma;
    for (int e = 0; e < data::kNumElements; ++e) s.mu[e] = mu20 ? mu20[e] : 0.0;
    s.count = count;
    s.structure_seed = structure_seed;
    return new std::vector<AtomisticSample>(data::generate_dataset(s, seed));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
uint64_t ref_dataset_count(void* h) { return static_cast<std::vector<AtomisticSample>*>(h)->size(); }
uint64_t ref_dataset_atoms(void* h) {
  uint64_t n = 0;
  for (auto& s : *static_cast<std::vector<AtomisticSample>*>(h)) n += s.n_atoms();
  return n;
}
void ref_dataset_export(void* h, int* n_atoms, uint8_t* species, double* pos, double* forces,
                        double* energy, uint8_t* dsid) {
  size_t at = 0;
  auto& v = *static_cast<std::vector<AtomisticSample>*>(h);
  for (size_t g = 0; g < v.size(); ++g) {
    const auto& s = v[g];
    n_atoms[g] = int(s.n_atoms());
    std::memcpy(species + at, s.species.data(), s.n_atoms());
    std::memcpy(pos + 3 * at, s.positions.data(), 3 * s.n_atoms() * sizeof(double));
    std::memcpy(forces + 3 * at, s.forces.data(), 3 * s.n_atoms() * sizeof(double));
    energy[g] = s.energy_per_atom;
    dsid[g] = s.dataset_id;
    at += s.n_atoms();
  }
}
void ref_dataset_free(void* h) { delete static_cast<std::vector<AtomisticSample>*>(h); }

// ------------------------------------------------------------ graph batch
// build_batch<double>, /root/reference/proj/include/hmtl/graph.hpp:46-83.
// Returns E; fills edges when dst != nullptr.  -1 on error.
long ref_build_batch(int G, const int* n_atoms, const uint8_t* species, const double* pos,
                     double cutoff, int* graph_offset, int* edge_offset, int* dst, int* src) {
  try {
    auto ss = make_samples(G, n_atoms, species, pos, nullptr, nullptr, nullptr);
    auto b = build_batch<double>(ss, cutoff);
    if (dst) {
      std::memcpy(graph_offset, b.graph_offset.data(), (G + 1) * sizeof(int));
      std::memcpy(edge_offset, b.edge_offset.data(), (G + 1) * sizeof(int));
      std::memcpy(dst, b.edge_dst.data(), b.n_edges() * sizeof(int));
      std::memcpy(src, b.edge_src.data(), b.n_edges() * sizeof(int));
    }
    return b.n_edges();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// ------------------------------------------------------------------ model
void* ref_model_new(const RefHyper* h, uint64_t seed, const int* owned, int n_owned, int dbl) {
  try {
    auto* box = new ModelBox;
    box->dbl = dbl != 0;
    std::vector<int> heads(owned, owned + n_owned);
    if (box->dbl)
      box->md = new ModelT<double>(to_hp(h), seed, heads);
    else
      box->mf = new ModelT<float>(to_hp(h), seed, heads);
    return box;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_model_free(void* m) { delete static_cast<ModelBox*>(m); }
uint64_t ref_model_shared_size(void* m) {
  auto* b = static_cast<ModelBox*>(m);
  return b->dbl ? b->md->shared_size() : b->mf->shared_size();
}
uint64_t ref_model_head_size(void* m) {
  auto* b = static_cast<ModelBox*>(m);
  return b->dbl ? b->md->head_size() : b->mf->head_size();
}
// which = -1 shared, k = head k
int ref_model_get_block(void* m, int which, double* out) {
  auto* b = static_cast<ModelBox*>(m);
  try {
    if (b->dbl) copy_out(which < 0 ? b->md->shared_block() : b->md->head_block(which), out);
    else copy_out(which < 0 ? b->mf->shared_block() : b->mf->head_block(which), out);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
int ref_model_set_block(void* m, int which, const double* in) {
  auto* b = static_cast<ModelBox*>(m);
  try {
    if (b->dbl) {
      auto& v = which < 0 ? b->md->shared_block() : b->md->head_block(which);
      for (size_t i = 0; i < v.size(); ++i) v[i] = in[i];
    } else {
      auto& v = which < 0 ? b->mf->shared_block() : b->mf->head_block(which);
      for (size_t i = 0; i < v.size(); ++i) v[i] = float(in[i]);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Output layout mirrors ho_cache (oracle/hmtl_oracle.h).
struct RefCacheOut {
  double *h_in, *z1, *a1, *z2, *m, *agg, *vz1, *vp1, *h_final, *pooled, *ez, *fz, *s;
};

extern "C++" {
namespace {
template <typename S>
void dump_cache(const ModelHyper& hp, const GraphBatchT<S>& b, const ForwardCacheT<S>& c,
                RefCacheOut* o) {
  if (!o) return;
  const size_t H = hp.hidden, N = b.n_nodes(), E = b.n_edges(), G = b.n_graphs;
  const size_t W = hp.head_width;
  for (int l = 0; l < hp.layers; ++l) {
    const auto& lc = c.layers[l];
    auto put = [&](double* base, const std::vector<S>& v, size_t per) {
      if (!base) return;
      for (size_t i = 0; i < v.size(); ++i) base[l * per + i] = double(v[i]);
    };
    put(o->h_in, lc.h_in, N * H);
    put(o->z1, lc.z1, E * H);
    put(o->a1, lc.a1, E * H);
    put(o->z2, lc.z2, E * H);
    put(o->m, lc.m, E * H);
    put(o->vz1, lc.vz1, N * H);
    put(o->vp1, lc.vp1, N * H);
    if (o->agg)  // agg is v[:, H:] (hmtl/model.hpp:412-417)
      for (size_t i = 0; i < N; ++i)
        for (size_t k = 0; k < H; ++k) o->agg[l * N * H + i * H + k] = double(lc.v[i * 2 * H + H + k]);
  }
  copy_out(c.h_final, o->h_final);
  for (const auto& [k, hc] : c.heads) {
    for (size_t gi = 0; gi < hc.graphs.size(); ++gi) {
      const int g = hc.graphs[gi];
      if (o->pooled)
        for (size_t t = 0; t < H; ++t) o->pooled[g * H + t] = double(hc.pooled[gi * H + t]);
      if (o->ez)
        for (int i = 0; i < hp.head_depth; ++i) {
          const size_t od = hc.energy.z[i].size() / hc.graphs.size();
          for (size_t t = 0; t < od; ++t)
            o->ez[(i * G + g) * W + t] = double(hc.energy.z[i][gi * od + t]);
        }
    }
    for (size_t ei = 0; ei < hc.edges.size(); ++ei) {
      const int e = hc.edges[ei];
      if (o->s) o->s[e] = double(hc.s[ei]);
      if (o->fz)
        for (int i = 0; i < hp.head_depth; ++i) {
          const size_t od = hc.force.z[i].size() / hc.edges.size();
          for (size_t t = 0; t < od; ++t)
            o->fz[(i * E + e) * W + t] = double(hc.force.z[i][ei * od + t]);
        }
    }
  }
}

template <typename S>
int fwd_bwd(ModelT<S>& model, ForwardCacheT<S>& cache, GraphBatchT<S>& batch, int G,
            const int* n_atoms, const uint8_t* species, const double* pos, const uint8_t* dsid,
            const double* dE, const double* dF, double* energy, double* forces,
            double* g_shared, double* const* g_heads, RefCacheOut* co) {
  auto ss = make_samples(G, n_atoms, species, pos, nullptr, nullptr, dsid);
  batch = build_batch<S>(ss, model.hyper().cutoff);
  cache = ForwardCacheT<S>{};
  auto pred = model.forward(batch, &cache);
  copy_out(pred.energy_per_atom, energy);
  copy_out(pred.forces, forces);
  dump_cache(model.hyper(), batch, cache, co);
  if (dE && dF) {
    std::vector<S> de(dE, dE + G), df(dF, dF + 3 * batch.n_nodes());
    auto g = model.backward(batch, cache, de, df);
    copy_out(g.shared, g_shared);
    for (auto& [k, v] : g.heads)
      if (g_heads && g_heads[k]) copy_out(v, g_heads[k]);
  }
  return 0;
}
}  // namespace
}  // extern "C++"

// ModelT::forward (+ backward when dE/dF given), hmtl/model.hpp:338-625.
int ref_forward_backward(void* m, int G, const int* n_atoms, const uint8_t* species,
                         const double* pos, const uint8_t* dsid, const double* dE,
                         const double* dF, double* energy, double* forces, double* g_shared,
                         double* const* g_heads, RefCacheOut* cache_out) {
  auto* b = static_cast<ModelBox*>(m);
  try {
    if (b->dbl)
      return fwd_bwd(*b->md, b->cd, b->bd, G, n_atoms, species, pos, dsid, dE, dF, energy,
                     forces, g_shared, g_heads, cache_out);
    return fwd_bwd(*b->mf, b->cf, b->bf, G, n_atoms, species, pos, dsid, dE, dF, energy, forces,
                   g_shared, g_heads, cache_out);
  } catch (const Error& e) {
    g_err = e.what();
    return int(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 6;
  }
}

// ---------------------------------------------------------------- trainer
// SPEC-conformant CPU step over the reference ModelT<float> (the reference
// CPU baseline path).  base-mode semantics on one rank: loss = mean over the
// batch's graphs, one AdamW update of the shared block and every owned head.
struct RefTrainer {
  ModelBox* box;
  double lr, b1, b2, eps, wd, w_e, w_f;
  long step = 0;
  std::vector<float> ms, vs;
  std::vector<std::vector<float>> mh, vh;
  std::vector<int> heads;
};

void* ref_trainer_new(void* m, double lr, double b1, double b2, double eps, double wd,
                      double w_e, double w_f) {
  auto* box = static_cast<ModelBox*>(m);
  if (box->dbl) {
    g_err = "trainer: float model required";
    return nullptr;
  }
  auto* t = new RefTrainer{box, lr, b1, b2, eps, wd, w_e, w_f};
  t->ms.assign(box->mf->shared_size(), 0.f);
  t->vs = t->ms;
  for (auto& [k, blk] : box->mf->head_blocks()) {
    t->heads.push_back(k);
    t->mh.emplace_back(blk.size(), 0.f);
    t->vh.emplace_back(blk.size(), 0.f);
  }
  return t;
}
void ref_trainer_free(void* t) { delete static_cast<RefTrainer*>(t); }

// One training step over G samples using n_threads host threads.  Returns the
// batch loss (mean over graphs) or NaN on error.
double ref_train_step(void* tp, int G, const int* n_atoms, const uint8_t* species,
                      const double* pos, const double* forces, const double* energy,
                      const uint8_t* dsid, int n_threads) {
  auto* t = static_cast<RefTrainer*>(tp);
  ModelT<float>& model = *t->box->mf;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > G) n_threads = G;
  std::vector<size_t> atom_off(G + 1, 0);
  for (int g = 0; g < G; ++g) atom_off[g + 1] = atom_off[g] + n_atoms[g];
  struct Part {
    GradientBufferT<float> g;
    double loss = 0.0;
    std::string err;
  };
  std::vector<Part> parts(n_threads);
  auto work = [&](int ti) {
    try {
      const int g0 = int((long)G * ti / n_threads), g1 = int((long)G * (ti + 1) / n_threads);
      const size_t a0 = atom_off[g0];
      auto ss = make_samples(g1 - g0, n_atoms + g0, species + a0, pos + 3 * a0, forces + 3 * a0,
                             energy + g0, dsid + g0);
      auto batch = build_batch<float>(ss, model.hyper().cutoff);
      ForwardCacheT<float> cache;
      auto pred = model.forward(batch, &cache);
      std::vector<float> dE, dF;
      parts[ti].loss = spec_loss(batch, pred, t->w_e, t->w_f, G, &dE, &dF);
      parts[ti].g = model.backward(batch, cache, dE, dF);
    } catch (const std::exception& e) {
      parts[ti].err = e.what();
    }
  };
  std::vector<std::thread> th;
  for (int i = 1; i < n_threads; ++i) th.emplace_back(work, i);
  work(0);
  for (auto& x : th) x.join();
  double loss = 0.0;
  for (auto& p : parts) {
    if (!p.err.empty()) {
      g_err = p.err;
      return NAN;
    }
    loss += p.loss;
  }
  GradientBufferT<float>& g = parts[0].g;
  for (int i = 1; i < n_threads; ++i) g.accumulate(parts[i].g);
  t->step += 1;
  adamw(model.shared_block(), g.shared, t->ms, t->vs, t->step, t->lr, t->b1, t->b2, t->eps, t->wd);
  for (size_t hi = 0; hi < t->heads.size(); ++hi) {
    const int k = t->heads[hi];
    adamw(model.head_block(k), g.heads.at(k), t->mh[hi], t->vh[hi], t->step, t->lr, t->b1, t->b2,
          t->eps, t->wd);
  }
  return loss / double(G);
}

// shuffle_epoch (src/datastore.cpp:47-97) of the reference on Mesh{n_groups, replicas};
// mode 0 base, 1 taskpar.  Writes rank `rank`'s plan; returns its item count.
long ref_shuffle_epoch(const uint8_t* ids, const uint64_t* counts, int n, int n_groups, int replicas, int mode,
                       uint64_t seed, int b_local, int rank, uint8_t* out_ds, uint64_t* out_idx, int* steps) {
  try {
    std::map<uint8_t, uint64_t> cnt;
    for (int i = 0; i < n; ++i) cnt[ids[i]] = counts[i];
    Mesh mesh;
    mesh.n_groups = n_groups;
    mesh.replicas = replicas;
    EpochPlan p = shuffle_epoch(cnt, mesh, mode == 1 ? RunMode::taskpar : RunMode::base, seed, b_local);
    *steps = p.steps;
    const auto& v = p.per_rank[rank];
    for (size_t i = 0; i < v.size(); ++i) out_ds[i] = v[i].dataset, out_idx[i] = v[i].index;
    return long(v.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// make_partition (src/datastore.cpp:25-45) on Mesh{n_groups, replicas}: per
// dataset (ascending id) its serving ranks and balanced_split ranges, flattened
long ref_make_partition(const uint8_t* ids, const uint64_t* counts, int n, int n_groups, int replicas, int mode,
                        int* serving, uint64_t* begin, uint64_t* end, int* n_serving) {
  try {
    std::map<uint8_t, uint64_t> cnt;
    for (int i = 0; i < n; ++i) cnt[ids[i]] = counts[i];
    Mesh mesh;
    mesh.n_groups = n_groups;
    mesh.replicas = replicas;
    DataPartition p = make_partition(cnt, mesh, mode == 1 ? RunMode::taskpar : RunMode::base);
    long k = 0;
    int i = 0;
    for (const auto& kv : p.datasets) {
      n_serving[i++] = int(kv.second.serving_ranks.size());
      for (size_t j = 0; j < kv.second.serving_ranks.size(); ++j, ++k) {
        serving[k] = kv.second.serving_ranks[j];
        begin[k] = kv.second.ranges[j].begin;
        end[k] = kv.second.ranges[j].end;
      }
    }
    return k;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// write_sample_file (src/sample_io.cpp:104-120) of G samples (flat arrays)
int ref_write_samples(const char* path, int dataset_id, int aligned, int G, const int* n_atoms,
                      const uint8_t* species, const double* pos, const double* energy, const double* forces,
                      const uint8_t* dsid) {
  try {
    std::vector<AtomisticSample> v(G);
    size_t a = 0;
    for (int g = 0; g < G; ++g) {
      const size_t n = size_t(n_atoms[g]);
      v[g].species.assign(species + a, species + a + n);
      v[g].positions.assign(pos + 3 * a, pos + 3 * (a + n));
      v[g].forces.assign(forces + 3 * a, forces + 3 * (a + n));
      v[g].energy_per_atom = energy[g];
      v[g].dataset_id = dsid[g];
      a += n;
    }
    io::FileHeader h;
    h.dataset_id = uint8_t(dataset_id);
    h.aligned = uint8_t(aligned);
    h.count = uint64_t(G);
    io::write_sample_file(path, h, v);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// align_energies (src/dataset.cpp:306-356): offsets per dataset (ascending id, 20 each)
int ref_align_energies(const char* const* files, int n, int ref_id, const char* const* out_files, uint8_t* ids,
                       double* offsets, uint8_t* skipped, int* n_skipped) {
  try {
    std::vector<std::string> in(files, files + n), out(out_files, out_files + n);
    data::AlignResult r = data::align_energies(in, uint8_t(ref_id), out);
    int i = 0;
    for (const auto& kv : r.offsets) {
      ids[i] = kv.first;
      for (int e = 0; e < data::kNumElements; ++e) offsets[i * data::kNumElements + e] = kv.second[e];
      ++i;
    }
    for (size_t j = 0; j < r.skipped_elements.size(); ++j) skipped[j] = r.skipped_elements[j];
    *n_skipped = int(r.skipped_elements.size());
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// save_checkpoint (src/model_io.cpp:62-84) of a reference model's blocks
int ref_save_checkpoint(void* m, const char* path) {
  try {
    auto* b = static_cast<ModelBox*>(m);
    if (!b->md) throw std::runtime_error("ref_save_checkpoint: needs the FP64 model");
    std::vector<std::vector<double>> heads;
    for (int k = 0; k < b->md->hyper().n_heads; ++k) heads.push_back(b->md->head_block(k));
    save_checkpoint(path, b->md->hyper(), b->md->shared_block(), heads);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
