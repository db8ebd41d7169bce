// host.cpp -- host-side pieces of the B200 step (no device code):
//   * flat parameter layouts (shared_layout / head_layout, hmtl/model.hpp:56-90)
//   * parameter init identical to ModelT's ctor (hmtl/model.hpp:158-167, 211-225)
//   * the synthetic multi-source generator used as the INPUT SOURCE
//     (src/dataset.cpp:21-161, 213-239) -- re-stated here so the product never
//     touches oracle/ or the reference; bit-identical by construction
//     (std::mt19937_64 is standard-specified, distributions hand-rolled as in
//     hmtl/rng.hpp) and checked against tests/golden/dataset5.npz
//   * MTL-par head placement for uneven meshes (generalises hmtl/mesh.hpp:21-31)
// Compiled with -ffp-contract=off: the reference is built without -march, so
// it never contracts a*b+c into an FMA.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "hmtl_b200.h"
#include "internal.h"

namespace hmtl_b200 {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// ----------------------------------------------------------------- layouts
Layout make_layout(const hmtl_hyper& hp, bool shared) {
  Layout L;
  auto add = [&](const std::string& n, size_t r, size_t c) {
    L.entries.push_back({n, r, c, L.total});
    L.total += r * c;
  };
  const size_t H = hp.hidden;
  if (shared) {
    add("embed", hp.n_species, H);
    for (int l = 0; l < hp.layers; ++l) {
      const std::string p = "layer" + std::to_string(l) + ".";
      add(p + "edge.W1", 2 * H + 1, H);
      add(p + "edge.b1", 1, H);
      add(p + "edge.W2", H, H);
      add(p + "edge.b2", 1, H);
      add(p + "node.W1", 2 * H, H);
      add(p + "node.b1", 1, H);
      add(p + "node.W2", H, H);
      add(p + "node.b2", 1, H);
    }
  } else {
    auto mlp = [&](const std::string& p, size_t in) {
      for (int i = 0; i < hp.head_depth; ++i) {
        size_t out = (i == hp.head_depth - 1) ? 1 : size_t(hp.head_width);
        add(p + ".W" + std::to_string(i), in, out);
        add(p + ".b" + std::to_string(i), 1, out);
        in = out;
      }
    };
    mlp("energy", H);
    mlp("force", H + 1);
  }
  return L;
}

// ------------------------------------------------------------------- RNG
uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t seed_stream(uint64_t master, uint64_t id) {
  return splitmix64(splitmix64(master) ^ splitmix64(id + 1));
}

namespace {
// Same sequence contract as hmtl::Rng (hmtl/rng.hpp:19-77).
struct Rng {
  std::mt19937_64 eng;
  double spare = 0.0;
  bool have = false;
  explicit Rng(uint64_t s) : eng(s) {}
  uint64_t u64() { return eng(); }
  double uniform() { return double(u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  uint64_t uniform_int(uint64_t n) { return uint64_t((__uint128_t(u64()) * n) >> 64); }
  double normal() {
    if (have) {
      have = false;
      return spare;
    }
    double u1 = uniform(), u2 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    double r = std::sqrt(-2.0 * std::log(u1));
    double a = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(a);
    have = true;
    return r * std::cos(a);
  }
  double normal(double m, double s) { return m + s * normal(); }
};

// ---- synthetic Morse-potential corpus (src/dataset.cpp:16-161)
constexpr double kDmin = 0.8;
constexpr uint64_t kMorseSeed = 0x4d4f525345ull;

struct Morse {
  double depth, width, r0;
};
Morse morse_params(uint8_t a, uint8_t b) {
  if (a > b) std::swap(a, b);
  Rng r(splitmix64(kMorseSeed ^ (uint64_t(a) * 131 + b)));
  Morse p;
  p.depth = r.uniform(0.4, 1.2);
  p.width = r.uniform(0.8, 1.3);
  p.r0 = r.uniform(1.0, 1.4);
  return p;
}

void morse_labels(const std::vector<uint8_t>& sp, const std::vector<double>& x, double* e_out,
                  std::vector<double>* f) {
  const size_t n = sp.size();
  double e = 0.0;
  f->assign(3 * n, 0.0);
  for (size_t i = 0; i < n; ++i)
    for (size_t j = i + 1; j < n; ++j) {
      const double dx = x[3 * i] - x[3 * j], dy = x[3 * i + 1] - x[3 * j + 1],
                   dz = x[3 * i + 2] - x[3 * j + 2];
      const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
      const Morse p = morse_params(sp[i], sp[j]);
      const double ex = std::exp(-p.width * (r - p.r0));
      const double om = 1.0 - ex;
      e += p.depth * (om * om - 1.0);
      const double ex2 = std::exp(-p.width * (r - p.r0));
      const double g = (2.0 * p.width * p.depth * ex2 * (1.0 - ex2)) / r;
      (*f)[3 * i] -= g * dx;
      (*f)[3 * i + 1] -= g * dy;
      (*f)[3 * i + 2] -= g * dz;
      (*f)[3 * j] += g * dx;
      (*f)[3 * j + 1] += g * dy;
      (*f)[3 * j + 2] += g * dz;
    }
  *e_out = e;
}

bool place(Rng& r, size_t n, std::vector<double>* x) {
  const double side = 1.6 * std::cbrt(double(n)) + 0.8;
  x->assign(3 * n, 0.0);
  for (size_t i = 0; i < n; ++i) {
    bool ok = false;
    for (int t = 0; t < 200 && !ok; ++t) {
      const double a = r.uniform(0.0, side), b = r.uniform(0.0, side), c = r.uniform(0.0, side);
      ok = true;
      for (size_t j = 0; j < i; ++j) {
        const double dx = a - (*x)[3 * j], dy = b - (*x)[3 * j + 1], dz = c - (*x)[3 * j + 2];
        if (dx * dx + dy * dy + dz * dz < kDmin * kDmin) {
          ok = false;
          break;
        }
      }
      if (ok) {
        (*x)[3 * i] = a;
        (*x)[3 * i + 1] = b;
        (*x)[3 * i + 2] = c;
      }
    }
    if (!ok) return false;
  }
  return true;
}
}  // namespace

// ---------------------------------------------------------------- init
void init_block(const hmtl_hyper& hp, uint64_t seed, int which, float* out) {
  const bool shared = which < 0;
  Layout L = make_layout(hp, shared);
  Rng r(seed_stream(seed, shared ? 0 : uint64_t(1 + which)));
  std::fill(out, out + L.total, 0.0f);
  for (const auto& e : L.entries) {
    if (e.name.find(".b") != std::string::npos) continue;
    const double s = (shared && e.name == "embed") ? 0.5 : 1.0 / std::sqrt(double(e.rows));
    for (size_t i = 0; i < e.rows * e.cols; ++i) out[e.offset + i] = float(r.uniform(-s, s));
  }
}

}  // namespace hmtl_b200

using namespace hmtl_b200;

extern "C" {

int hmtl_abi_version(void) { return HMTL_ABI_VERSION; }
const char* hmtl_last_error(void) { return g_last_error.c_str(); }

size_t hmtl_shared_size(const hmtl_hyper* hp) { return make_layout(*hp, true).total; }
size_t hmtl_head_size(const hmtl_hyper* hp) { return make_layout(*hp, false).total; }

int hmtl_layout_entry(const hmtl_hyper* hp, int shared, int i, char* name, size_t cap,
                      size_t* rows, size_t* cols, size_t* offset) {
  Layout L = make_layout(*hp, shared != 0);
  const int n = int(L.entries.size());
  if (i >= 0 && i < n) {
    const auto& e = L.entries[i];
    if (name && cap) std::snprintf(name, cap, "%s", e.name.c_str());
    if (rows) *rows = e.rows;
    if (cols) *cols = e.cols;
    if (offset) *offset = e.offset;
  }
  return n;
}

int hmtl_init_block(const hmtl_hyper* hp, uint64_t seed, int which, float* out) {
  if (!hp || !out) return fail(HMTL_ERR_CONTRACT, "init_block: null argument");
  if (which >= hp->n_heads) return fail(HMTL_ERR_CONTRACT, "model: head index out of range");
  init_block(*hp, seed, which, out);
  return HMTL_OK;
}

// classify_regime, hmtl/model.hpp:249-255 (x10 threshold)
int hmtl_classify_regime(size_t p_s, size_t p_h, int n_h) {
  if (!(p_s > 0 && p_h > 0 && n_h > 0)) return -fail(HMTL_ERR_CONTRACT, "classify_regime: positive counts");
  const double nhph = double(n_h) * double(p_h);
  if (double(p_s) >= 10.0 * nhph) return 1;
  if (nhph >= 10.0 * double(p_s)) return 2;
  return 3;
}
// memory_footprint, hmtl/model.hpp:260-263
size_t hmtl_memory_footprint(size_t p_s, size_t p_h, int n_h, int mode) {
  if (mode == 2) return p_s + p_h;
  return p_s + size_t(n_h) * p_h;
}

// default5_specs, src/dataset.cpp:213-239
int hmtl_default5_spec(int id, hmtl_dataset_spec* s) {
  struct Row {
    const char* name;
    std::vector<uint8_t> el;
    int nmin, nmax;
    double alpha, sigma;
  };
  static const Row rows[5] = {
      {"organicA", {0, 1, 2, 3}, 4, 12, 1.00, 0.01},
      {"organicB", {0, 2, 3, 4, 5}, 4, 16, 0.70, 0.02},
      {"organicC", {0, 1, 3, 5, 6, 7}, 4, 14, 1.35, 0.01},
      {"inorganicA", {2, 5, 8, 9, 10, 11, 12, 13, 14, 15}, 8, 40, 0.55, 0.03},
      {"inorganicB", {3, 6, 9, 12, 14, 16, 17, 18, 19}, 8, 64, 1.60, 0.02},
  };
  if (id < 0 || id >= 5 || !s) return fail(HMTL_ERR_DATA, "default5: id out of range");
  std::memset(s, 0, sizeof(*s));
  const Row& r = rows[id];
  s->dataset_id = id;
  s->n_elements = int(r.el.size());
  for (size_t i = 0; i < r.el.size(); ++i) s->elements[i] = r.el[i];
  s->n_min = r.nmin;
  s->n_max = r.nmax;
  s->alpha = r.alpha;
  s->sigma = r.sigma;
  s->count = 10000;
  s->structure_seed = -1;
  Rng m(seed_stream(0x0FF5E75, uint64_t(id)));
  for (uint8_t e : r.el) s->mu[e] = m.uniform(-3.0, 3.0);
  return HMTL_OK;
}

// generate_dataset, src/dataset.cpp:106-161
int hmtl_generate(const hmtl_dataset_spec* spec, uint64_t seed, int* G, int* N, int* n_atoms,
                  uint8_t* species, double* positions, double* forces, double* energy,
                  uint8_t* dataset_id) {
  if (!spec || spec->n_min < 2 || spec->n_max < spec->n_min)
    return fail(HMTL_ERR_DATA, "dataset spec: need n_min >= 2");
  if (!(spec->alpha > 0.0)) return fail(HMTL_ERR_DATA, "dataset spec: alpha must be positive");
  if (spec->n_elements < 1) return fail(HMTL_ERR_DATA, "dataset spec: empty element set");
  for (int i = 0; i < spec->n_elements; ++i)
    if (spec->elements[i] >= 20) return fail(HMTL_ERR_DATA, "dataset spec: element index out of range");
  const uint64_t sseed = spec->structure_seed >= 0
                             ? seed_stream(uint64_t(spec->structure_seed), 0xA)
                             : seed_stream(seed, 0xA00 + uint64_t(spec->dataset_id));
  Rng sr(sseed), nr(seed_stream(seed, 0xB00 + uint64_t(spec->dataset_id)));
  size_t at = 0;
  for (uint64_t k = 0; k < spec->count; ++k) {
    const size_t n = size_t(spec->n_min) + sr.uniform_int(uint64_t(spec->n_max - spec->n_min + 1));
    std::vector<uint8_t> sp(n);
    for (size_t i = 0; i < n; ++i) sp[i] = spec->elements[sr.uniform_int(uint64_t(spec->n_elements))];
    std::vector<double> x;
    bool ok = false;
    for (int t = 0; t < 20 && !ok; ++t) ok = place(sr, n, &x);
    if (!ok) return fail(HMTL_ERR_DATA, "generate_dataset: rejection sampling failed (box too dense)");
    double e_true;
    std::vector<double> f_true;
    morse_labels(sp, x, &e_true, &f_true);
    double off = 0.0;
    for (size_t i = 0; i < n; ++i) off += spec->mu[sp[i]];
    double epa = spec->alpha * e_true / double(n) + off / double(n);
    if (spec->sigma > 0.0) epa += nr.normal(0.0, spec->sigma);
    if (n_atoms) {
      n_atoms[k] = int(n);
      std::memcpy(species + at, sp.data(), n);
      std::memcpy(positions + 3 * at, x.data(), 3 * n * sizeof(double));
      energy[k] = epa;
      dataset_id[k] = uint8_t(spec->dataset_id);
    }
    for (size_t i = 0; i < 3 * n; ++i) {
      double v = spec->alpha * f_true[i];
      if (spec->sigma > 0.0) v += nr.normal(0.0, spec->sigma);
      if (n_atoms) forces[3 * at + i] = v;
    }
    at += n;
  }
  if (G) *G = int(spec->count);
  if (N) *N = int(at);
  return HMTL_OK;
}

// Head placement for MTL-par on uneven meshes.  Head k is split evenly over
// m_k replicas (sub-group of size m_k); the pieces (size w_k/m_k) are packed
// into `world` ranks of equal load, each replica of a head on a distinct rank.
// The search enumerates replica vectors by increasing piece count (fewest
// pieces = most task-parallel, least communication) and packs by backtracking.
int hmtl_head_placement(int world, int n_heads, const double* w, double* share) {
  if (world < 1 || n_heads < 1 || !w || !share) return fail(HMTL_ERR_CONTRACT, "head_placement: bad args");
  double total = 0.0;
  for (int k = 0; k < n_heads; ++k) {
    if (!(w[k] > 0.0)) return fail(HMTL_ERR_CONFIG, "head_placement: weights must be positive");
    total += w[k];
  }
  const double cap = total / world;
  std::fill(share, share + size_t(world) * n_heads, 0.0);
  if (world == 1) {
    for (int k = 0; k < n_heads; ++k) share[k] = 1.0;
    return HMTL_OK;
  }
  std::vector<int> m(n_heads, 1);
  for (int pieces = n_heads; pieces <= world * n_heads; ++pieces) {
    // enumerate m with sum == pieces, each 1..world
    std::function<bool(int, int)> rec_m = [&](int k, int left) -> bool {
      if (k == n_heads) {
        if (left != 0) return false;
        struct Piece {
          int head;
          double size;
        };
        std::vector<Piece> ps;
        for (int h = 0; h < n_heads; ++h)
          for (int r = 0; r < m[h]; ++r) ps.push_back({h, w[h] / m[h]});
        std::sort(ps.begin(), ps.end(), [](const Piece& a, const Piece& b) {
          return a.size > b.size || (a.size == b.size && a.head < b.head);
        });
        std::vector<double> load(world, 0.0);
        std::vector<std::vector<int>> has(world, std::vector<int>(n_heads, 0));
        std::function<bool(size_t)> pack = [&](size_t i) -> bool {
          if (i == ps.size()) {
            for (int r = 0; r < world; ++r)
              if (std::fabs(load[r] - cap) > 1e-9 * total) return false;
            return true;
          }
          double prev = -1.0;
          for (int r = 0; r < world; ++r) {
            if (has[r][ps[i].head]) continue;
            if (load[r] + ps[i].size > cap + 1e-9 * total) continue;
            if (load[r] == prev) continue;  // symmetric bins
            prev = load[r];
            load[r] += ps[i].size;
            has[r][ps[i].head] = 1;
            if (pack(i + 1)) return true;
            load[r] -= ps[i].size;
            has[r][ps[i].head] = 0;
          }
          return false;
        };
        if (!pack(0)) return false;
        for (int r = 0; r < world; ++r)
          for (int h = 0; h < n_heads; ++h)
            if (has[r][h]) share[size_t(r) * n_heads + h] = 1.0 / m[h];
        return true;
      }
      const int rest = n_heads - k - 1;
      for (int v = 1; v <= world && v <= left - rest; ++v) {
        m[k] = v;
        if (rec_m(k + 1, left - v)) return true;
      }
      return false;
    };
    if (rec_m(0, pieces)) return HMTL_OK;
  }
  return fail(HMTL_ERR_CONFIG, "head_placement: no balanced placement of the heads on this mesh");
}

}  // extern "C"

// ---- epoch plan: shuffle_epoch (src/datastore.cpp:47-97) -------------------
// Per-rank ordered sample lists of one epoch.  taskpar: per dataset (ascending
// id, as the reference's std::map), a seeded Fisher-Yates permutation
// (seed_stream(seed, 0x700 + id)) of that dataset only, dealt in steps of
// replicas x b_local over the dataset's serving group; steps = min over the
// datasets of count / (replicas * b_local).  base: one permutation
// (seed_stream(seed, 0x77)) of the mixed (dataset, index) set dealt over all
// ranks.  The reference's Mesh (hmtl/mesh.hpp:21-31) is the special case
// members[g] = {g*M .. g*M+M-1}; any placement's head groups are accepted.
extern "C" int hmtl_epoch_plan(int mode, const uint8_t* ids, const uint64_t* counts, int n_datasets,
                               const int* members, const int* member_off, int world, uint64_t seed, int b_local,
                               int rank, uint8_t* out_ds, uint64_t* out_idx, size_t cap, int* steps_out,
                               size_t* n_items) {
  using namespace hmtl_b200;
  if (b_local < 1) return fail(HMTL_ERR_CONTRACT, "b_local must be >= 1");
  if (!ids || !counts || n_datasets < 1 || world < 1 || rank < 0 || rank >= world || !steps_out || !n_items)
    return fail(HMTL_ERR_CONTRACT, "epoch_plan: bad arguments");
  std::vector<int> order(n_datasets);  // ascending dataset id (std::map order)
  for (int i = 0; i < n_datasets; ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return ids[a] < ids[b]; });
  for (int i = 1; i < n_datasets; ++i)
    if (ids[order[i]] == ids[order[i - 1]]) return fail(HMTL_ERR_CONTRACT, "epoch_plan: duplicate dataset id");
  std::vector<uint8_t> ds;
  std::vector<uint64_t> ix;
  int steps = 0;
  if (mode == 1) {  // taskpar
    if (!members || !member_off) return fail(HMTL_ERR_CONTRACT, "taskpar: dataset id without sub-group");
    steps = -1;
    for (int i : order) {
      const int M = member_off[i + 1] - member_off[i];
      if (M < 1) return fail(HMTL_ERR_CONTRACT, "taskpar: dataset id without sub-group");
      const int g = int(counts[i] / (uint64_t(M) * uint64_t(b_local)));
      steps = steps < 0 ? g : std::min(steps, g);
    }
    steps = std::max(steps, 0);
    for (int i : order) {
      const int M = member_off[i + 1] - member_off[i];
      int slot = -1;
      for (int s = 0; s < M; ++s)
        if (members[member_off[i] + s] == rank) slot = s;
      if (slot < 0) continue;
      std::vector<uint64_t> idx(counts[i]);
      for (uint64_t j = 0; j < counts[i]; ++j) idx[j] = j;
      Rng rng(seed_stream(seed, 0x700 + ids[i]));
      for (size_t j = idx.size(); j > 1; --j) std::swap(idx[j - 1], idx[size_t(rng.uniform_int(j))]);
      for (int s = 0; s < steps; ++s) {
        const uint64_t at = (uint64_t(s) * M + slot) * b_local;
        for (int b = 0; b < b_local; ++b) ds.push_back(ids[i]), ix.push_back(idx[at + b]);
      }
    }
  } else {  // base / serial
    std::vector<std::pair<uint8_t, uint64_t>> all;
    for (int i : order)
      for (uint64_t j = 0; j < counts[i]; ++j) all.push_back({ids[i], j});
    Rng rng(seed_stream(seed, 0x77));
    for (size_t j = all.size(); j > 1; --j) std::swap(all[j - 1], all[size_t(rng.uniform_int(j))]);
    steps = int(all.size() / (uint64_t(world) * uint64_t(b_local)));
    for (int s = 0; s < steps; ++s) {
      const uint64_t at = (uint64_t(s) * world + rank) * b_local;
      for (int b = 0; b < b_local; ++b) ds.push_back(all[at + b].first), ix.push_back(all[at + b].second);
    }
  }
  *steps_out = steps;
  *n_items = ds.size();
  if (out_ds || out_idx) {
    if (cap < ds.size()) return fail(HMTL_ERR_CONTRACT, "epoch_plan: output buffer too small");
    if (out_ds) std::copy(ds.begin(), ds.end(), out_ds);
    if (out_idx) std::copy(ix.begin(), ix.end(), out_idx);
  }
  return HMTL_OK;
}

// ---- HMTD sample files (hmtl/sample_io.hpp:9-15, src/sample_io.cpp) -----------
// Little-endian: "HMTD", version u32 = 1, dataset_id u8, aligned u8, count u64,
// then per record: n u32, species u8[n], positions f64[3n], energy_per_atom f64,
// forces f64[3n], dataset_id u8, crc32 u32 (CRC-32 of the record before it).
namespace hmtl_b200 {
uint32_t crc32_ieee(const uint8_t* p, size_t n) {  // zlib crc32 (reflected 0xEDB88320)
  static uint32_t table[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    init = true;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) c = table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}
}  // namespace hmtl_b200

namespace {
void put_le(std::vector<uint8_t>& v, uint64_t x, int bytes) {
  for (int i = 0; i < bytes; ++i) v.push_back(uint8_t(x >> (8 * i)));
}
}  // namespace

extern "C" int hmtl_hmtd_write(const char* path, uint8_t dataset_id, uint8_t aligned, const hmtl_samples* s) {
  using namespace hmtl_b200;
  if (!path || !s || s->G < 0) return fail(HMTL_ERR_CONTRACT, "hmtd_write: bad arguments");
  std::vector<uint8_t> buf;
  put_le(buf, 0x44544d48u, 4);
  put_le(buf, 1, 4);
  buf.push_back(dataset_id);
  buf.push_back(aligned);
  put_le(buf, uint64_t(s->G), 8);
  size_t a = 0;
  for (int g = 0; g < s->G; ++g) {
    const size_t n = size_t(s->n_atoms[g]), start = buf.size();
    put_le(buf, n, 4);
    buf.insert(buf.end(), s->species + a, s->species + a + n);
    auto f64 = [&](double d) {
      uint64_t x;
      std::memcpy(&x, &d, 8);
      put_le(buf, x, 8);
    };
    for (size_t i = 0; i < 3 * n; ++i) f64(s->positions[3 * a + i]);
    f64(s->energy_per_atom ? s->energy_per_atom[g] : 0.0);
    for (size_t i = 0; i < 3 * n; ++i) f64(s->forces ? s->forces[3 * a + i] : 0.0);
    buf.push_back(s->dataset_id[g]);
    put_le(buf, crc32_ieee(buf.data() + start, buf.size() - start), 4);
    a += n;
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(HMTL_ERR_IO, std::string("cannot open for write: ") + path);
  const size_t w = std::fwrite(buf.data(), 1, buf.size(), f);
  std::fclose(f);
  if (w != buf.size()) return fail(HMTL_ERR_IO, std::string("short write: ") + path);
  return HMTL_OK;
}

extern "C" int hmtl_hmtd_read_header(const char* path, uint8_t* dataset_id, uint8_t* aligned, uint64_t* count) {
  using namespace hmtl_b200;
  FILE* f = path ? std::fopen(path, "rb") : nullptr;
  if (!f) return fail(HMTL_ERR_IO, std::string("cannot open for read: ") + (path ? path : "(null)"));
  uint8_t h[18];
  const size_t got = std::fread(h, 1, sizeof h, f);
  std::fclose(f);
  if (got != sizeof h) return fail(HMTL_ERR_IO, std::string("short read: ") + path);
  auto u32 = [&](int o) { return uint32_t(h[o]) | uint32_t(h[o + 1]) << 8 | uint32_t(h[o + 2]) << 16 | uint32_t(h[o + 3]) << 24; };
  if (u32(0) != 0x44544d48u) return fail(HMTL_ERR_IO, std::string("bad magic: ") + path);
  if (u32(4) != 1) return fail(HMTL_ERR_IO, std::string("bad version: ") + path);
  if (dataset_id) *dataset_id = h[8];
  if (aligned) *aligned = h[9];
  if (count) {
    uint64_t c = 0;
    for (int i = 0; i < 8; ++i) c |= uint64_t(h[10 + i]) << (8 * i);
    *count = c;
  }
  return HMTL_OK;
}

// ---- HMTP checkpoints (src/model_io.cpp:7-13, 62-118) + optimizer section ----
// v1 body exactly as save_checkpoint: "HMTP", version 1, hyper record (6 x u32,
// cutoff f64), activation u8 = 1, then the shared block and every head block in
// head order, each u64 count + f64 elements.  Resume extension (SURVEY.md
// 8(f)3), appended after the v1 body so the reference's load_checkpoint (which
// stops after the last head block) still reads the file: "HMTO", version u32 = 1,
// AdamW step u64, then per block in the same order: u64 count, m f64[count],
// v f64[count].  FP32 values are stored widened to f64 (exact both ways).
namespace hmtl_b200 {
namespace {
struct Wr {
  std::vector<uint8_t> b;
  void raw(const void* p, size_t n) { b.insert(b.end(), (const uint8_t*)p, (const uint8_t*)p + n); }
  void u32(uint32_t x) { raw(&x, 4); }
  void u64(uint64_t x) { raw(&x, 8); }
  void f64(double x) { raw(&x, 8); }
  void block(const float* p, size_t n) {
    u64(n);
    for (size_t i = 0; i < n; ++i) f64(double(p[i]));
  }
};
}  // namespace

int hmtp_write(const char* path, const hmtl_hyper& hp, const float* shared, size_t ps, const float* const* heads,
               size_t ph, int n_heads, const hmtl_ckpt_opt* opt) {
  Wr w;
  w.u32(0x50544d48u);
  w.u32(1);
  for (uint32_t x : {uint32_t(hp.n_species), uint32_t(hp.layers), uint32_t(hp.hidden), uint32_t(hp.head_width),
                     uint32_t(hp.head_depth), uint32_t(hp.n_heads)})
    w.u32(x);
  w.f64(hp.cutoff);
  const uint8_t act = 1;
  w.raw(&act, 1);
  w.block(shared, ps);
  for (int k = 0; k < n_heads; ++k) w.block(heads[k], ph);
  if (opt) {
    w.u32(0x4f544d48u);  // "HMTO"
    w.u32(1);
    w.u64(opt->step);
    w.block(opt->m_shared, ps);
    w.block(opt->v_shared, ps);
    for (int k = 0; k < n_heads; ++k) {
      w.block(opt->m_heads[k], ph);
      w.block(opt->v_heads[k], ph);
    }
  }
  FILE* f = std::fopen(path, "wb");
  if (!f) return fail(HMTL_ERR_IO, std::string("cannot open for write: ") + path);
  const size_t n = std::fwrite(w.b.data(), 1, w.b.size(), f);
  std::fclose(f);
  if (n != w.b.size()) return fail(HMTL_ERR_IO, "checkpoint: short write");
  return HMTL_OK;
}

// parse into host vectors: shared, heads[n_heads], optional optimizer section
int hmtp_read(const char* path, hmtl_hyper* hp, std::vector<double>* shared, std::vector<std::vector<double>>* heads,
              bool* has_opt, uint64_t* step, std::vector<std::vector<double>>* opt_blocks) {
  FILE* f = path ? std::fopen(path, "rb") : nullptr;
  if (!f) return fail(HMTL_ERR_IO, std::string("cannot open for read: ") + (path ? path : "(null)"));
  std::vector<uint8_t> b;
  std::fseek(f, 0, SEEK_END);
  const long len = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  b.resize(len > 0 ? size_t(len) : 0);
  const size_t got = std::fread(b.data(), 1, b.size(), f);
  std::fclose(f);
  size_t o = 0;
  bool short_read = got != b.size();
  auto rd = [&](void* p, size_t n) {
    if (o + n > b.size()) {
      short_read = true;
      std::memset(p, 0, n);
      return;
    }
    std::memcpy(p, b.data() + o, n);
    o += n;
  };
  auto u32 = [&] { uint32_t x; rd(&x, 4); return x; };
  auto u64 = [&] { uint64_t x; rd(&x, 8); return x; };
  auto blk = [&](std::vector<double>& v) -> bool {
    const uint64_t n = u64();
    if (short_read || n > (b.size() - o) / 8) return false;
    v.resize(n);
    rd(v.data(), 8 * n);
    return true;
  };
  if (u32() != 0x50544d48u) return fail(HMTL_ERR_IO, std::string("not a checkpoint: ") + path);
  if (u32() != 1) return fail(HMTL_ERR_IO, std::string("unsupported checkpoint version: ") + path);
  hmtl_hyper h{};
  h.n_species = int(u32());
  h.layers = int(u32());
  h.hidden = int(u32());
  h.head_width = int(u32());
  h.head_depth = int(u32());
  h.n_heads = int(u32());
  rd(&h.cutoff, 8);
  uint8_t act = 0;
  rd(&act, 1);
  if (short_read) return fail(HMTL_ERR_IO, "checkpoint: short read");
  if (act != 1) return fail(HMTL_ERR_IO, "unknown activation id in checkpoint");
  const size_t ps = make_layout(h, true).total, ph = make_layout(h, false).total;
  if (!blk(*shared)) return fail(HMTL_ERR_IO, "checkpoint: short read");
  if (shared->size() != ps) return fail(HMTL_ERR_IO, "checkpoint: shared block size mismatch");
  heads->assign(h.n_heads, {});
  for (int k = 0; k < h.n_heads; ++k) {
    if (!blk((*heads)[k])) return fail(HMTL_ERR_IO, "checkpoint: short read");
    if ((*heads)[k].size() != ph) return fail(HMTL_ERR_IO, "checkpoint: head block size mismatch");
  }
  *hp = h;
  *has_opt = false;
  if (o + 8 <= b.size()) {
    if (u32() != 0x4f544d48u || u32() != 1) return fail(HMTL_ERR_IO, "checkpoint: unknown trailing section");
    *step = u64();
    opt_blocks->assign(2 + 2 * size_t(h.n_heads), {});
    for (size_t i = 0; i < opt_blocks->size(); ++i) {
      if (!blk((*opt_blocks)[i])) return fail(HMTL_ERR_IO, "checkpoint: short read");
      if ((*opt_blocks)[i].size() != (i < 2 ? ps : ph)) return fail(HMTL_ERR_IO, "checkpoint: optimizer block size mismatch");
    }
    *has_opt = true;
  }
  return HMTL_OK;
}
}  // namespace hmtl_b200

extern "C" int hmtl_checkpoint_write(const char* path, const hmtl_hyper* hp, const float* shared,
                                     const float* heads, const hmtl_ckpt_opt* opt) {
  using namespace hmtl_b200;
  if (!path || !hp || !shared || !heads) return fail(HMTL_ERR_CONTRACT, "checkpoint: need all head blocks in head-index order");
  const size_t ps = make_layout(*hp, true).total, ph = make_layout(*hp, false).total;
  std::vector<const float*> hs(hp->n_heads);
  for (int k = 0; k < hp->n_heads; ++k) hs[k] = heads + size_t(k) * ph;
  return hmtp_write(path, *hp, shared, ps, hs.data(), ph, hp->n_heads, opt);
}

extern "C" int hmtl_checkpoint_read_hyper(const char* path, hmtl_hyper* hp, int* has_optimizer) {
  using namespace hmtl_b200;
  std::vector<double> sh;
  std::vector<std::vector<double>> hd, opt;
  bool has = false;
  uint64_t step = 0;
  hmtl_hyper h{};
  if (int rc = hmtp_read(path, &h, &sh, &hd, &has, &step, &opt)) return rc;
  if (hp) *hp = h;
  if (has_optimizer) *has_optimizer = has ? 1 : 0;
  return HMTL_OK;
}
