// store.cu -- device-resident sample store (the DataStore of
// hmtl/datastore.hpp:77-115, src/datastore.cpp:100-250, re-designed for HBM).
//
// The reference keeps each rank's shard as raw record bytes in host memory and
// assembles every step's batch by local slicing plus request/response reads
// from the owners over TCP (fetch_samples, src/datastore.cpp:174-248), then
// build_batch concatenates on the host.  Here the whole pool a rank may be
// dealt (its head group's datasets -- a few GB even at the paper's 24M
// structures, next to 180 GB of HBM) is uploaded once; a step's batch is the
// plan's (dataset, index) list, and the concatenation into the batch arena is
// a gather kernel: per step only the G selected sample ids and the graph
// offsets cross PCIe.  The arena it writes is byte-identical to the one
// hmtl_batch_upload packs on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "ctx.cuh"

using namespace hmtl_b200;

struct hmtl_store {
  int device = 0;
  int G = 0;
  long long N = 0;
  // device pool: atoms back to back in pool order
  long long* d_atom_off = nullptr;  // [G + 1]
  uint8_t *d_ds = nullptr, *d_species = nullptr;
  double *d_energy = nullptr, *d_pos = nullptr, *d_forces = nullptr;
  // host metadata (selection validation and graph offsets need no device round trip)
  std::vector<int> n_atoms;
  std::vector<uint8_t> ds;
  std::map<int, std::vector<int>> by_dataset;  // dataset id -> pool sample per local index
  // per-bind staging: [sel ids | graph_offset]
  int* h_stage = nullptr;  // pinned
  int* d_sel = nullptr;
  int stage_cap = 0;
  cudaEvent_t staged = nullptr;  // last bind's staging copy has been consumed
};

namespace {
__global__ void store_gather_kernel(const int* __restrict__ sel, int G, const long long* __restrict__ atom_off,
                                    const uint8_t* __restrict__ ds, const uint8_t* __restrict__ species,
                                    const double* __restrict__ energy, const double* __restrict__ pos,
                                    const double* __restrict__ forces, uint8_t* __restrict__ arena) {
  pdl_wait();
  const int g = blockIdx.x;
  if (g >= G) return;
  const int* hdr = reinterpret_cast<const int*>(arena);
  const ArenaLayout al = arena_layout(hdr[0], hdr[1]);
  const int* go = reinterpret_cast<const int*>(arena + al.go);
  const int s = sel[g], dst0 = go[g], n = go[g + 1] - go[g];
  const long long src0 = atom_off[s];
  if (threadIdx.x == 0) {
    arena[al.ds + g] = ds[s];
    reinterpret_cast<double*>(arena + al.le)[g] = energy[s];
  }
  uint8_t* sp = arena + al.sp;
  double* p = reinterpret_cast<double*>(arena + al.pos);
  double* f = reinterpret_cast<double*>(arena + al.lf);
  for (int t = threadIdx.x; t < n; t += blockDim.x) sp[dst0 + t] = species[src0 + t];
  for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) {
    p[3LL * dst0 + t] = pos[3 * src0 + t];
    f[3LL * dst0 + t] = forces[3 * src0 + t];
  }
}
}  // namespace

extern "C" {

int hmtl_store_create(int device, const hmtl_samples* s, hmtl_store** out) {
  if (!s || !out || s->G < 1 || s->N < 1 || !s->n_atoms || !s->species || !s->positions || !s->dataset_id)
    return fail(HMTL_ERR_CONTRACT, "store_create: empty or incomplete sample pool");
  if (device < 0 || device >= hmtl_device_count())
    return fail(HMTL_ERR_INTERNAL, "store_create: no CUDA device (the B200 path has no CPU fallback)");
  HMTL_CUDA(cudaSetDevice(device));
  auto* st = new hmtl_store;
  st->device = device;
  st->G = s->G;
  st->N = s->N;
  st->n_atoms.assign(s->n_atoms, s->n_atoms + s->G);
  st->ds.assign(s->dataset_id, s->dataset_id + s->G);
  std::vector<long long> off(size_t(s->G) + 1, 0);
  for (int g = 0; g < s->G; ++g) {
    if (s->n_atoms[g] < 1) {
      delete st;
      return fail(HMTL_ERR_CONTRACT, "build_batch: empty graph rejected");
    }
    off[g + 1] = off[g] + s->n_atoms[g];
    st->by_dataset[s->dataset_id[g]].push_back(g);
  }
  if (off[s->G] != s->N) {
    delete st;
    return fail(HMTL_ERR_CONTRACT, "samples: sum(n_atoms) != N");
  }
  std::vector<double> zeros;
  const double* E = s->energy_per_atom;
  const double* F = s->forces;
  if (!E || !F) zeros.assign(size_t(3) * s->N + s->G, 0.0);
  bool ok = cudaMalloc(&st->d_atom_off, off.size() * sizeof(long long)) == cudaSuccess &&
            cudaMalloc(&st->d_ds, size_t(s->G)) == cudaSuccess &&
            cudaMalloc(&st->d_species, size_t(s->N)) == cudaSuccess &&
            cudaMalloc(&st->d_energy, size_t(s->G) * 8) == cudaSuccess &&
            cudaMalloc(&st->d_pos, size_t(s->N) * 24) == cudaSuccess &&
            cudaMalloc(&st->d_forces, size_t(s->N) * 24) == cudaSuccess &&
            cudaEventCreateWithFlags(&st->staged, cudaEventDisableTiming) == cudaSuccess;
  if (ok)
    ok = cudaMemcpy(st->d_atom_off, off.data(), off.size() * sizeof(long long), cudaMemcpyHostToDevice) ==
             cudaSuccess &&
         cudaMemcpy(st->d_ds, s->dataset_id, size_t(s->G), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(st->d_species, s->species, size_t(s->N), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(st->d_energy, E ? E : zeros.data(), size_t(s->G) * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(st->d_pos, s->positions, size_t(s->N) * 24, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(st->d_forces, F ? F : zeros.data(), size_t(s->N) * 24, cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) {
    hmtl_store_destroy(st);
    return fail(HMTL_ERR_INTERNAL, "store_create: device allocation/upload failed");
  }
  *out = st;
  return HMTL_OK;
}

int hmtl_store_counts(const hmtl_store* st, uint8_t* ids, uint64_t* counts, int cap, int* n) {
  if (!st || !n) return fail(HMTL_ERR_CONTRACT, "store_counts: null argument");
  *n = int(st->by_dataset.size());
  if (!ids && !counts) return HMTL_OK;
  if (cap < *n) return fail(HMTL_ERR_CONTRACT, "store_counts: buffer too small");
  int i = 0;
  for (const auto& kv : st->by_dataset) {
    if (ids) ids[i] = uint8_t(kv.first);
    if (counts) counts[i] = kv.second.size();
    ++i;
  }
  return HMTL_OK;
}

int hmtl_store_bind(hmtl_ctx* h, hmtl_store* st, const uint8_t* ds, const uint64_t* idx, int n, void* stream) {
  if (!h || !st || !ds || !idx || n < 1) return fail(HMTL_ERR_CONTRACT, "model: empty batch rejected");
  Ctx& c = h->c;
  if (st->device != c.device) return fail(HMTL_ERR_CONTRACT, "store_bind: store and context on different devices");
  if (n > c.Gc) return fail(HMTL_ERR_CONTRACT, "batch exceeds context capacity (graphs/nodes)");
  cudaSetDevice(c.device);
  cudaStream_t sm = stream ? static_cast<cudaStream_t>(stream) : c.stream;
  // validate on the host metadata (the checks pack() does for host batches)
  std::vector<int> sel(n);
  long long N = 0, bound = 0;
  for (int g = 0; g < n; ++g) {
    auto it = st->by_dataset.find(ds[g]);
    if (it == st->by_dataset.end() || idx[g] >= it->second.size())
      return fail(HMTL_ERR_CONTRACT, "owner_of: index out of range");
    if (c.slot_of[ds[g]] < 0)
      return fail(HMTL_ERR_CONTRACT, "model: unknown dataset id " + std::to_string(ds[g]) +
                                         " (head not owned by this rank)");
    sel[g] = it->second[idx[g]];
    const long long na = st->n_atoms[sel[g]];
    N += na;
    bound += na * (na - 1);
  }
  if (N > c.Nc) return fail(HMTL_ERR_CONTRACT, "batch exceeds context capacity (graphs/nodes)");
  if (bound > c.Ec) return fail(HMTL_ERR_CONTRACT, "batch may exceed the context's edge capacity");
  const ArenaLayout al = arena_layout(n, int(N));
  // staging: [G, N, 0, 0, graph_offset[G+1] ... | sel[G]]
  const int words = 4 + (n + 1) + n;
  if (words > st->stage_cap) {
    if (st->h_stage) cudaEventSynchronize(st->staged), cudaFreeHost(st->h_stage);
    if (st->d_sel) cudaFree(st->d_sel);
    st->stage_cap = std::max(words, 4096);
    HMTL_CUDA(cudaMallocHost(&st->h_stage, size_t(st->stage_cap) * 4));
    HMTL_CUDA(cudaMalloc(&st->d_sel, size_t(st->stage_cap) * 4));
  } else {
    HMTL_CUDA(cudaEventSynchronize(st->staged));  // the previous bind's copies have been consumed
  }
  int* hs = st->h_stage;
  hs[0] = n;
  hs[1] = int(N);
  hs[2] = hs[3] = 0;
  int* go = hs + 4;
  go[0] = 0;
  for (int g = 0; g < n; ++g) go[g + 1] = go[g] + st->n_atoms[sel[g]];
  std::memcpy(go + n + 1, sel.data(), size_t(n) * 4);
  // header + graph offsets straight into the arena (al.go == 16 == 4 ints), ids to staging
  static_assert(sizeof(int) * 4 == 16, "arena header");
  HMTL_CUDA(cudaMemcpyAsync(c.arena, hs, size_t(4 + n + 1) * 4, cudaMemcpyHostToDevice, sm));
  HMTL_CUDA(cudaMemcpyAsync(st->d_sel, go + n + 1, size_t(n) * 4, cudaMemcpyHostToDevice, sm));
  kl(store_gather_kernel, dim3(n), dim3(128), 0, sm, static_cast<const int*>(st->d_sel), n,
     static_cast<const long long*>(st->d_atom_off), static_cast<const uint8_t*>(st->d_ds),
     static_cast<const uint8_t*>(st->d_species), static_cast<const double*>(st->d_energy),
     static_cast<const double*>(st->d_pos), static_cast<const double*>(st->d_forces), c.arena);
  HMTL_CUDA(cudaEventRecord(st->staged, sm));
  HMTL_CUDA(cudaGetLastError());
  (void)al;
  c.host_G = n;
  c.host_N = int(N);
  return HMTL_OK;
}

int hmtl_store_destroy(hmtl_store* st) {
  if (!st) return HMTL_OK;
  cudaSetDevice(st->device);
  if (st->staged) cudaEventSynchronize(st->staged), cudaEventDestroy(st->staged);
  void* ptrs[] = {st->d_atom_off, st->d_ds, st->d_species, st->d_energy, st->d_pos, st->d_forces, st->d_sel};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (st->h_stage) cudaFreeHost(st->h_stage);
  delete st;
  return HMTL_OK;
}

}  // extern "C"
