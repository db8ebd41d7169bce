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
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <limits>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "ctx.cuh"

using namespace hmtl_b200;

namespace hmtl_b200 {
ncclComm_t comm_world(Ctx& c, int* rank, int* size);  // comm.cu
}

// DataPartition::Dataset (hmtl/datastore.hpp:25-40): serving ranks ascending,
// one balanced contiguous range each
struct StorePart {
  uint64_t count = 0;
  std::vector<int> serving;
  std::vector<uint64_t> lo;  // range i = [lo[i], lo[i+1])
  uint64_t my_begin = 0;     // this rank's range (sharded stores)
  std::vector<int> n_atoms;  // every sample of the dataset (all shards), for batch offsets
  int owner_of(uint64_t index) const {
    for (size_t i = 0; i + 1 < lo.size(); ++i)
      if (index >= lo[i] && index < lo[i + 1]) return serving[i];
    return -1;
  }
};
// one batch item of a sharded fetch: pool sample (kind 0) or byte offset in
// the receive buffer (kind 1); pack items: pool sample -> send-buffer offset
struct FetchItem {
  long long src;
  long long dst;
  int n, kind, ds, pad;
};

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
  // sharded store (hmtl_store_create_sharded): only this rank's shard is in the
  // pool; fetches exchange remote samples with NCCL send/recv
  bool sharded = false;
  int rank = 0, world = 1;
  std::map<int, StorePart> part;
  FetchItem* h_items = nullptr;  // pinned [pack items | assemble items]
  FetchItem* d_items = nullptr;
  int items_cap = 0;
  uint8_t *d_send = nullptr, *d_recv = nullptr;
  size_t send_cap = 0, recv_cap = 0;
  int* d_flag = nullptr;  // fetch plan consensus (allreduce min)
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
// sample wire format of a sharded fetch (8-byte aligned blocks):
// [energy f64 | positions 3n f64 | forces 3n f64 | species n u8, padded to 8]
__host__ __device__ inline long long wire_bytes(int n) { return 8 + 48LL * n + ((n + 7) & ~7); }
__global__ void store_pack_kernel(const FetchItem* __restrict__ it, int n_items, const long long* __restrict__ atom_off,
                                  const uint8_t* __restrict__ species, const double* __restrict__ energy,
                                  const double* __restrict__ pos, const double* __restrict__ forces,
                                  uint8_t* __restrict__ out) {
  for (int k = blockIdx.x; k < n_items; k += gridDim.x) {
    const FetchItem f = it[k];
    const long long a0 = atom_off[f.src];
    double* o = reinterpret_cast<double*>(out + f.dst);
    if (threadIdx.x == 0) o[0] = energy[f.src];
    for (int t = threadIdx.x; t < 3 * f.n; t += blockDim.x) {
      o[1 + t] = pos[3 * a0 + t];
      o[1 + 3 * f.n + t] = forces[3 * a0 + t];
    }
    uint8_t* sp = out + f.dst + 8 + 48LL * f.n;
    for (int t = threadIdx.x; t < f.n; t += blockDim.x) sp[t] = species[a0 + t];
  }
}
// batch item g -> the arena (same bytes as store_gather_kernel / batch_upload)
__global__ void store_assemble_kernel(const FetchItem* __restrict__ it, int G, const long long* __restrict__ atom_off,
                                      const uint8_t* __restrict__ species, const double* __restrict__ energy,
                                      const double* __restrict__ pos, const double* __restrict__ forces,
                                      const uint8_t* __restrict__ recv, uint8_t* __restrict__ arena) {
  pdl_wait();
  const int g = blockIdx.x;
  if (g >= G) return;
  const int* hdr = reinterpret_cast<const int*>(arena);
  const ArenaLayout al = arena_layout(hdr[0], hdr[1]);
  const int* go = reinterpret_cast<const int*>(arena + al.go);
  const FetchItem f = it[g];
  const int dst0 = go[g], n = f.n;
  uint8_t* sp = arena + al.sp;
  double* p = reinterpret_cast<double*>(arena + al.pos);
  double* fo = reinterpret_cast<double*>(arena + al.lf);
  if (f.kind == 0) {
    const long long a0 = atom_off[f.src];
    if (threadIdx.x == 0) {
      arena[al.ds + g] = uint8_t(f.ds);
      reinterpret_cast<double*>(arena + al.le)[g] = energy[f.src];
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x) sp[dst0 + t] = species[a0 + t];
    for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) {
      p[3LL * dst0 + t] = pos[3 * a0 + t];
      fo[3LL * dst0 + t] = forces[3 * a0 + t];
    }
  } else {
    const double* w = reinterpret_cast<const double*>(recv + f.src);
    if (threadIdx.x == 0) {
      arena[al.ds + g] = uint8_t(f.ds);
      reinterpret_cast<double*>(arena + al.le)[g] = w[0];
    }
    const uint8_t* ws = recv + f.src + 8 + 48LL * n;
    for (int t = threadIdx.x; t < n; t += blockDim.x) sp[dst0 + t] = ws[t];
    for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) {
      p[3LL * dst0 + t] = w[1 + t];
      fo[3LL * dst0 + t] = w[1 + 3 * n + t];
    }
  }
}
// CRC-32 (zlib's reflected 0xEDB88320) of each record body against its stored
// value: one thread per record, table in shared memory (load-time check only).
__global__ void hmtd_crc_kernel(const uint8_t* __restrict__ raw, const long long* __restrict__ rec_off, int R,
                                int* __restrict__ bad) {
  __shared__ uint32_t table[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = uint32_t(i);
    for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    table[i] = c;
  }
  __syncthreads();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < R; r += gridDim.x * blockDim.x) {
    const long long a = rec_off[r], b = rec_off[r + 1] - 4;
    uint32_t c = 0xFFFFFFFFu;
    for (long long i = a; i < b; ++i) c = table[(c ^ raw[i]) & 0xFF] ^ (c >> 8);
    c ^= 0xFFFFFFFFu;
    const uint32_t stored = uint32_t(raw[b]) | uint32_t(raw[b + 1]) << 8 | uint32_t(raw[b + 2]) << 16 |
                            uint32_t(raw[b + 3]) << 24;
    if (c != stored) atomicMin(bad, r);
  }
}
__device__ __forceinline__ double le_f64(const uint8_t* p) {  // unaligned little-endian
  unsigned long long x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x |= static_cast<unsigned long long>(p[i]) << (8 * i);
  return __longlong_as_double(static_cast<long long>(x));
}
// record r -> the pool's SoA (species, positions, energy, forces); CTA per record
__global__ void hmtd_parse_kernel(const uint8_t* __restrict__ raw, const long long* __restrict__ rec_off,
                                  const long long* __restrict__ atom_off, int R, uint8_t* __restrict__ species,
                                  double* __restrict__ pos, double* __restrict__ energy,
                                  double* __restrict__ forces) {
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    const uint8_t* rec = raw + rec_off[r];
    const long long a0 = atom_off[r];
    const int n = int(atom_off[r + 1] - a0);
    const uint8_t* sp = rec + 4;
    const uint8_t* ps = sp + n;
    const uint8_t* en = ps + 24 * n;
    const uint8_t* fs = en + 8;
    for (int t = threadIdx.x; t < n; t += blockDim.x) species[a0 + t] = sp[t];
    for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) {
      pos[3 * a0 + t] = le_f64(ps + 8 * t);
      forces[3 * a0 + t] = le_f64(fs + 8 * t);
    }
    if (threadIdx.x == 0) energy[r] = le_f64(en);
  }
}
// ---- energy alignment (align_energies, src/dataset.cpp:263-356) on the device pool ----
constexpr int kElems = 20;  // kNumElements (hmtl/dataset.hpp:14)
// per-sample element fractions over the dataset's present elements (idx[z] = column or -1)
__global__ void align_frac_kernel(const int* __restrict__ sel, int G, const long long* __restrict__ atom_off,
                                  const uint8_t* __restrict__ species, const int* __restrict__ idx, int k,
                                  double* __restrict__ F) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
    const int s = sel[g];
    const long long a0 = atom_off[s], a1 = atom_off[s + 1];
    const double inv = 1.0 / double(a1 - a0);
    double f[kElems];
#pragma unroll
    for (int a = 0; a < kElems; ++a) f[a] = 0.0;
    for (long long i = a0; i < a1; ++i) {
      const int c = idx[species[i]];
#pragma unroll
      for (int a = 0; a < kElems; ++a)
        if (a == c) f[a] += inv;  // frac[a] += 1/n per atom, atom order (as the reference)
    }
    for (int a = 0; a < k; ++a) F[size_t(g) * kElems + a] = f[a];
  }
}
// normal equations X^T X | X^T y over a fixed chunk of samples per block (thread = entry),
// then align_sum_kernel adds the chunk partials in chunk order: deterministic
constexpr int kAlignChunk = 256;
__global__ void align_normal_kernel(const double* __restrict__ F, const int* __restrict__ sel,
                                    const double* __restrict__ energy, int G, int k, double* __restrict__ part) {
  const int t = threadIdx.x, T = k * k + k;
  if (t >= T) return;
  const int g0 = blockIdx.x * kAlignChunk, g1 = min(G, g0 + kAlignChunk);
  double acc = 0.0;
  if (t < k * k) {
    const int a = t / k, b = t % k;
    for (int g = g0; g < g1; ++g) acc += F[size_t(g) * kElems + a] * F[size_t(g) * kElems + b];
  } else {
    const int a = t - k * k;
    for (int g = g0; g < g1; ++g) acc += F[size_t(g) * kElems + a] * energy[sel[g]];
  }
  part[size_t(blockIdx.x) * T + t] = acc;
}
__global__ void align_sum_kernel(const double* __restrict__ part, int nb, int T, double* __restrict__ out) {
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc += part[size_t(b) * T + t];
    out[t] = acc;
  }
}
// energy_per_atom -= sum over atoms (mu_d[z] - mu_ref[z]) / n (NaN offsets count as 0)
__global__ void align_apply_kernel(const int* __restrict__ sel, int G, const long long* __restrict__ atom_off,
                                   const uint8_t* __restrict__ species, const double* __restrict__ mu_d,
                                   const double* __restrict__ mu_ref, double* __restrict__ energy) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
    const int s = sel[g];
    const long long a0 = atom_off[s], a1 = atom_off[s + 1];
    const double n = double(a1 - a0);
    double corr = 0.0;
    for (long long i = a0; i < a1; ++i) {
      const int z = species[i];
      const double d = isnan(mu_d[z]) ? 0.0 : mu_d[z], r = isnan(mu_ref[z]) ? 0.0 : mu_ref[z];
      corr += (d - r) / n;
    }
    energy[s] -= corr;
  }
}
}  // namespace

namespace {
bool store_alloc(hmtl_store* st) {
  return cudaMalloc(&st->d_atom_off, (size_t(st->G) + 1) * sizeof(long long)) == cudaSuccess &&
         cudaMalloc(&st->d_ds, size_t(st->G)) == cudaSuccess &&
         cudaMalloc(&st->d_species, size_t(st->N)) == cudaSuccess &&
         cudaMalloc(&st->d_energy, size_t(st->G) * 8) == cudaSuccess &&
         cudaMalloc(&st->d_pos, size_t(st->N) * 24) == cudaSuccess &&
         cudaMalloc(&st->d_forces, size_t(st->N) * 24) == cudaSuccess &&
         cudaEventCreateWithFlags(&st->staged, cudaEventDisableTiming) == cudaSuccess;
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
  bool ok = store_alloc(st);
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

// HMTD files -> device pool.  The host reads each file once
// and checks its structure as read_sample_file_raw (src/sample_io.cpp:122-160:
// magic, version, `count` records, no trailing bytes); the raw record bytes go
// to HBM as they are, and the per-record CRC check (parse_record,
// src/sample_io.cpp:80-93) and the parse into the pool's SoA run on the GPU.
int hmtl_store_from_hmtd(int device, const char* const* paths, int n_files, hmtl_store** out) {
  if (!paths || n_files < 1 || !out) return fail(HMTL_ERR_CONTRACT, "store_from_hmtd: no files");
  if (device < 0 || device >= hmtl_device_count())
    return fail(HMTL_ERR_INTERNAL, "store_from_hmtd: no CUDA device (the B200 path has no CPU fallback)");
  std::vector<uint8_t> raw;
  std::vector<long long> rec_off{0}, atom_off{0};
  std::vector<int> n_atoms;
  std::vector<uint8_t> ds;
  auto u32 = [](const uint8_t* p) { return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24; };
  for (int fi = 0; fi < n_files; ++fi) {
    const std::string path = paths[fi] ? paths[fi] : "";
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return fail(HMTL_ERR_IO, "cannot open for read: " + path);
    std::fseek(f, 0, SEEK_END);
    const long len = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    std::vector<uint8_t> buf(len > 0 ? size_t(len) : 0);
    const size_t got = std::fread(buf.data(), 1, buf.size(), f);
    std::fclose(f);
    if (len < 18) return fail(HMTL_ERR_IO, "sample file too short: " + path);
    if (got != buf.size()) return fail(HMTL_ERR_IO, "short read: " + path);
    if (u32(buf.data()) != 0x44544d48u) return fail(HMTL_ERR_IO, "bad magic (not a sample file): " + path);
    if (u32(buf.data() + 4) != 1) return fail(HMTL_ERR_IO, "unsupported sample file version: " + path);
    uint64_t count = 0;
    for (int i = 0; i < 8; ++i) count |= uint64_t(buf[10 + i]) << (8 * i);
    size_t off = 18;
    for (uint64_t r = 0; r < count; ++r) {
      if (off + 4 > buf.size()) return fail(HMTL_ERR_IO, "truncated record in " + path);
      const uint32_t n = u32(buf.data() + off);
      const size_t total = 4 + size_t(n) + 24 * size_t(n) + 8 + 24 * size_t(n) + 1 + 4;
      if (off + total > buf.size()) return fail(HMTL_ERR_IO, "truncated record in " + path);
      if (n < 1) return fail(HMTL_ERR_CONTRACT, "build_batch: empty graph rejected");
      n_atoms.push_back(int(n));
      ds.push_back(buf[off + total - 5]);
      atom_off.push_back(atom_off.back() + n);
      off += total;
      rec_off.push_back(rec_off.back() + static_cast<long long>(total));
    }
    if (off != buf.size()) return fail(HMTL_ERR_IO, "trailing bytes in " + path);
    raw.insert(raw.end(), buf.begin() + 18, buf.end());
  }
  const int R = int(n_atoms.size());
  if (R < 1) return fail(HMTL_ERR_CONTRACT, "store_from_hmtd: no records");
  HMTL_CUDA(cudaSetDevice(device));
  auto* st = new hmtl_store;
  st->device = device;
  st->G = R;
  st->N = atom_off.back();
  st->n_atoms = n_atoms;
  st->ds = ds;
  for (int g = 0; g < R; ++g) st->by_dataset[ds[g]].push_back(g);
  uint8_t* d_raw = nullptr;
  long long* d_rec = nullptr;
  int* d_bad = nullptr;
  int bad = R;
  bool ok = store_alloc(st) && cudaMalloc(&d_raw, raw.size()) == cudaSuccess &&
            cudaMalloc(&d_rec, rec_off.size() * sizeof(long long)) == cudaSuccess &&
            cudaMalloc(&d_bad, sizeof(int)) == cudaSuccess;
  if (ok)
    ok = cudaMemcpy(d_raw, raw.data(), raw.size(), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(d_rec, rec_off.data(), rec_off.size() * sizeof(long long), cudaMemcpyHostToDevice) ==
             cudaSuccess &&
         cudaMemcpy(d_bad, &bad, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(st->d_atom_off, atom_off.data(), atom_off.size() * sizeof(long long),
                    cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(st->d_ds, ds.data(), ds.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  if (ok) {
    hmtd_crc_kernel<<<(R + 255) / 256, 256>>>(d_raw, d_rec, R, d_bad);
    hmtd_parse_kernel<<<std::min(R, 148 * 16), 128>>>(d_raw, d_rec, st->d_atom_off, R, st->d_species, st->d_pos,
                                                      st->d_energy, st->d_forces);
    ok = cudaDeviceSynchronize() == cudaSuccess && cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess;
  }
  cudaFree(d_raw), cudaFree(d_rec), cudaFree(d_bad);
  if (!ok) {
    hmtl_store_destroy(st);
    return fail(HMTL_ERR_INTERNAL, "store_from_hmtd: device upload/parse failed");
  }
  if (bad < R) {
    hmtl_store_destroy(st);
    return fail(HMTL_ERR_IO, "record: CRC mismatch (record " + std::to_string(bad) + ")");
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
  c.head_sorted = sorted_by_slot(c, ds, n);
  c.host_N = int(N);
  return HMTL_OK;
}

// ---- sharded store (remote samples over NVLink) ----

// balanced_split (src/datastore.cpp:11-23): the first count % n shards get one extra
int hmtl_shard_range(uint64_t count, int n, int i, uint64_t* begin, uint64_t* end) {
  if (n < 1) return fail(HMTL_ERR_CONTRACT, "balanced_split: need at least one shard");
  if (i < 0 || i >= n || !begin || !end) return fail(HMTL_ERR_CONTRACT, "shard_range: bad shard index");
  const uint64_t base = count / uint64_t(n), extra = count % uint64_t(n);
  *begin = base * uint64_t(i) + std::min<uint64_t>(uint64_t(i), extra);
  *end = *begin + base + (uint64_t(i) < extra ? 1 : 0);
  return HMTL_OK;
}

int hmtl_store_create_sharded(hmtl_ctx* h, const hmtl_samples* s, const uint8_t* ids, const uint64_t* counts,
                              const int* members, const int* member_off, int n_datasets, hmtl_store** out) {
  if (!h || !s || !out || !ids || !counts || !members || !member_off || n_datasets < 1)
    return fail(HMTL_ERR_CONTRACT, "store_create_sharded: null argument");
  Ctx& c = h->c;
  int rank = 0, world = 1;
  ncclComm_t comm = comm_world(c, &rank, &world);
  if (!comm) return fail(HMTL_ERR_CONTRACT, "store_create_sharded: hmtl_comm_init first");
  // the partition (make_partition, src/datastore.cpp:25-45) and this rank's expected shard
  std::map<int, StorePart> part;
  std::map<int, uint64_t> expect;
  for (int d = 0; d < n_datasets; ++d) {
    StorePart sp;
    sp.count = counts[d];
    sp.serving.assign(members + member_off[d], members + member_off[d + 1]);
    if (sp.serving.empty() || !std::is_sorted(sp.serving.begin(), sp.serving.end()))
      return fail(HMTL_ERR_CONTRACT, "store_create_sharded: serving ranks must be non-empty and ascending");
    const int ns = int(sp.serving.size());
    sp.lo.resize(ns + 1);
    for (int i = 0; i < ns; ++i) {
      uint64_t b, e;
      hmtl_shard_range(sp.count, ns, i, &b, &e);
      sp.lo[i] = b, sp.lo[i + 1] = e;
      if (sp.serving[i] < 0 || sp.serving[i] >= world) return fail(HMTL_ERR_CONTRACT, "store_create_sharded: bad rank");
      if (sp.serving[i] == rank) sp.my_begin = b, expect[ids[d]] = e - b;
    }
    if (part.count(ids[d])) return fail(HMTL_ERR_DATA, "duplicate dataset id across files");
    part[ids[d]] = std::move(sp);
  }
  // the shard: per served dataset its range, in order; nothing else
  std::map<int, uint64_t> have;
  for (int g = 0; g < s->G; ++g) ++have[s->dataset_id[g]];
  for (const auto& kv : have)
    if (!expect.count(kv.first) || expect[kv.first] != kv.second)
      return fail(HMTL_ERR_CONTRACT, "store_create_sharded: shard does not match this rank's ranges");
  for (const auto& kv : expect)
    if (kv.second && !have.count(kv.first))
      return fail(HMTL_ERR_CONTRACT, "store_create_sharded: shard does not match this rank's ranges");
  hmtl_store* st = nullptr;
  if (int rc = hmtl_store_create(c.device, s, &st)) return rc;
  st->sharded = true;
  st->rank = rank;
  st->world = world;
  // every sample's atom count, all shards (one grouped broadcast per range
  // owner, 4 B per sample): a fetch then needs no request round trip
  size_t total = 0;
  for (auto& kv : part) total += kv.second.count;
  int* d_n = nullptr;
  if (cudaMalloc(&d_n, std::max<size_t>(total, 1) * 4) != cudaSuccess) {
    hmtl_store_destroy(st);
    return fail(HMTL_ERR_INTERNAL, "store_create_sharded: allocation failed");
  }
  std::vector<int> h_n(total, 0);
  {
    size_t at = 0;
    for (auto& kv : part) {  // my ranges from the shard (datasets appear in pool order)
      const auto it = st->by_dataset.find(kv.first);
      if (it != st->by_dataset.end())
        for (size_t j = 0; j < it->second.size(); ++j) h_n[at + kv.second.my_begin + j] = st->n_atoms[it->second[j]];
      at += kv.second.count;
    }
  }
  cudaStream_t sm = c.stream;
  bool ok = cudaMemcpy(d_n, h_n.data(), total * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  ok = ok && ncclGroupStart() == ncclSuccess;
  {
    size_t at = 0;
    for (auto& kv : part) {
      const StorePart& sp = kv.second;
      for (size_t i = 0; i < sp.serving.size(); ++i) {
        const size_t len = sp.lo[i + 1] - sp.lo[i];
        if (len && ok)
          ok = ncclBroadcast(d_n + at + sp.lo[i], d_n + at + sp.lo[i], len, ncclInt32, sp.serving[i], comm, sm) ==
               ncclSuccess;
      }
      at += sp.count;
    }
  }
  ok = (ncclGroupEnd() == ncclSuccess) && ok;
  ok = ok && cudaStreamSynchronize(sm) == cudaSuccess &&
       cudaMemcpy(h_n.data(), d_n, total * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
  cudaFree(d_n);
  if (!ok) {
    hmtl_store_destroy(st);
    return fail(HMTL_ERR_COMM, "store_create_sharded: sample-size exchange failed");
  }
  size_t at = 0;
  for (auto& kv : part) {
    kv.second.n_atoms.assign(h_n.begin() + at, h_n.begin() + at + kv.second.count);
    at += kv.second.count;
  }
  st->part = std::move(part);
  *out = st;
  return HMTL_OK;
}

// fetch_samples(plan, step) (src/datastore.cpp:192-248), B200 edition: the
// step's plan rows of every rank are known to every rank (shuffle_epoch is
// deterministic), so owners push what their peers need without a request
// message; every pair's samples go in one ncclSend/ncclRecv of a grouped call
// (NVLink/NVSwitch), and one kernel assembles the batch arena from the local
// pool and the receive buffer.
int hmtl_store_fetch(hmtl_ctx* h, hmtl_store* st, const uint8_t* plan_ds, const uint64_t* plan_idx, int b_local,
                     void* stream) {
  if (!h || !st || !plan_ds || !plan_idx || b_local < 1) return fail(HMTL_ERR_CONTRACT, "model: empty batch rejected");
  if (!st->sharded) return fail(HMTL_ERR_CONTRACT, "store_fetch: not a sharded store (use store_bind)");
  Ctx& c = h->c;
  if (st->device != c.device) return fail(HMTL_ERR_CONTRACT, "store_fetch: store and context on different devices");
  int rank = 0, world = 1;
  ncclComm_t comm = comm_world(c, &rank, &world);
  if (!comm || rank != st->rank || world != st->world)
    return fail(HMTL_ERR_CONTRACT, "store_fetch: context communicator differs from the store's");
  const int n = b_local;
  cudaSetDevice(c.device);
  cudaStream_t sm = stream ? static_cast<cudaStream_t>(stream) : c.stream;
  // A rank that rejects its plan must not return while its peers enter the
  // grouped send/recv (they would wait forever): every check below only records
  // the first failure, and all ranks agree on the outcome with one tiny
  // allreduce(min) before any exchange.
  int bad_rc = 0;
  std::string bad_msg;
  auto reject = [&](int rc, const std::string& msg) {
    if (!bad_rc) bad_rc = rc, bad_msg = msg;
  };
  if (n > c.Gc) reject(HMTL_ERR_CONTRACT, "batch exceeds context capacity (graphs/nodes)");
  auto find = [&](uint8_t d, uint64_t i, const StorePart** sp) -> int {
    auto it = st->part.find(d);
    if (it == st->part.end() || i >= it->second.count) return -1;
    *sp = &it->second;
    return it->second.owner_of(i);
  };
  // plan walk: my items (local or from their owner), and what I owe each peer
  std::vector<FetchItem> mine(n), pack;
  std::vector<long long> send_b(world, 0), recv_b(world, 0), send_off(world + 1, 0), recv_off(world + 1, 0);
  // pass 1: byte counts per peer
  for (int r = 0; r < world; ++r)
    for (int b = 0; b < n; ++b) {
      const uint8_t d = plan_ds[size_t(r) * n + b];
      const uint64_t i = plan_idx[size_t(r) * n + b];
      const StorePart* sp = nullptr;
      const int o = find(d, i, &sp);
      if (o < 0) {
        if (r == rank) reject(HMTL_ERR_CONTRACT, "owner_of: index out of range");
        continue;  // (a peer's bad row: that peer rejects it)
      }
      if (r == rank && o != rank) recv_b[o] += wire_bytes(sp->n_atoms[i]);
      if (r != rank && o == rank) send_b[r] += wire_bytes(sp->n_atoms[i]);
    }
  for (int p = 0; p < world; ++p) send_off[p + 1] = send_off[p] + send_b[p], recv_off[p + 1] = recv_off[p] + recv_b[p];
  // pass 2: descriptors (per peer in batch order, the order both sides walk)
  std::vector<long long> sat(send_off.begin(), send_off.end() - 1), rat(recv_off.begin(), recv_off.end() - 1);
  long long N = 0, bound = 0;
  for (int r = 0; r < world; ++r)
    for (int b = 0; b < n; ++b) {
      const uint8_t d = plan_ds[size_t(r) * n + b];
      const uint64_t i = plan_idx[size_t(r) * n + b];
      const StorePart* sp = nullptr;
      const int o = find(d, i, &sp);
      if (o < 0) continue;
      const int na = sp->n_atoms[i];
      if (r == rank) {
        if (c.slot_of[d] < 0)
          reject(HMTL_ERR_CONTRACT, "model: unknown dataset id " + std::to_string(d) + " (head not owned by this rank)");
        if (b >= int(mine.size())) continue;
        FetchItem& f = mine[b];
        f.n = na, f.ds = d, f.dst = 0, f.pad = 0;
        if (o == rank) f.kind = 0, f.src = st->by_dataset[d][i - sp->my_begin];
        else f.kind = 1, f.src = rat[o], rat[o] += wire_bytes(na);
        N += na;
        bound += (long long)na * (na - 1);
      } else if (o == rank) {
        pack.push_back(FetchItem{st->by_dataset[d][i - sp->my_begin], sat[r], na, 0, d, 0});
        sat[r] += wire_bytes(na);
      }
    }
  if (N > c.Nc) reject(HMTL_ERR_CONTRACT, "batch exceeds context capacity (graphs/nodes)");
  if (bound > c.Ec) reject(HMTL_ERR_CONTRACT, "batch may exceed the context's edge capacity");
  if (world > 1) {  // consensus: every rank learns whether any rank rejected its plan
    if (!st->d_flag) HMTL_CUDA(cudaMalloc(&st->d_flag, sizeof(int)));
    const int mine_ok = bad_rc ? 0 : 1;
    int all_ok = 0;
    HMTL_CUDA(cudaMemcpyAsync(st->d_flag, &mine_ok, sizeof(int), cudaMemcpyHostToDevice, sm));
    if (ncclAllReduce(st->d_flag, st->d_flag, 1, ncclInt32, ncclMin, comm, sm) != ncclSuccess)
      return fail(HMTL_ERR_COMM, "store_fetch: plan consensus allreduce failed");
    HMTL_CUDA(cudaMemcpyAsync(&all_ok, st->d_flag, sizeof(int), cudaMemcpyDeviceToHost, sm));
    HMTL_CUDA(cudaStreamSynchronize(sm));
    if (!all_ok && !bad_rc) reject(HMTL_ERR_CONTRACT, "store_fetch: a peer rank rejected its plan rows");
  }
  if (bad_rc) return fail(bad_rc, bad_msg);
  // staging: [G, N, 0, 0, graph_offset[G+1]] -> arena; items -> device
  const int words = 4 + (n + 1);
  const int n_items = int(pack.size()) + n;
  if (words > st->stage_cap || n_items > st->items_cap) {
    if (st->h_stage) cudaEventSynchronize(st->staged);
    if (words > st->stage_cap) {
      if (st->h_stage) cudaFreeHost(st->h_stage);
      if (st->d_sel) cudaFree(st->d_sel);
      st->stage_cap = std::max(words, 4096);
      HMTL_CUDA(cudaMallocHost(&st->h_stage, size_t(st->stage_cap) * 4));
      HMTL_CUDA(cudaMalloc(&st->d_sel, size_t(st->stage_cap) * 4));
    }
    if (n_items > st->items_cap) {
      if (st->h_items) cudaFreeHost(st->h_items);
      if (st->d_items) cudaFree(st->d_items);
      st->items_cap = std::max(n_items, 1024);
      HMTL_CUDA(cudaMallocHost(&st->h_items, size_t(st->items_cap) * sizeof(FetchItem)));
      HMTL_CUDA(cudaMalloc(&st->d_items, size_t(st->items_cap) * sizeof(FetchItem)));
    }
  } else {
    HMTL_CUDA(cudaEventSynchronize(st->staged));
  }
  auto grow = [&](uint8_t** p, size_t* cap, size_t need) -> bool {
    if (need <= *cap) return true;
    cudaStreamSynchronize(sm);
    if (*p) cudaFree(*p);
    *cap = std::max(need, size_t(1) << 20);
    return cudaMalloc(p, *cap) == cudaSuccess;
  };
  if (!grow(&st->d_send, &st->send_cap, size_t(send_off[world])) ||
      !grow(&st->d_recv, &st->recv_cap, size_t(recv_off[world])))
    return fail(HMTL_ERR_INTERNAL, "store_fetch: exchange buffer allocation failed");
  int* hs = st->h_stage;
  hs[0] = n, hs[1] = int(N), hs[2] = hs[3] = 0;
  int* go = hs + 4;
  go[0] = 0;
  for (int g = 0; g < n; ++g) go[g + 1] = go[g] + mine[g].n;
  std::memcpy(st->h_items, pack.data(), pack.size() * sizeof(FetchItem));
  std::memcpy(st->h_items + pack.size(), mine.data(), size_t(n) * sizeof(FetchItem));
  HMTL_CUDA(cudaMemcpyAsync(c.arena, hs, size_t(4 + n + 1) * 4, cudaMemcpyHostToDevice, sm));
  HMTL_CUDA(cudaMemcpyAsync(st->d_items, st->h_items, size_t(n_items) * sizeof(FetchItem), cudaMemcpyHostToDevice, sm));
  if (!pack.empty())
    store_pack_kernel<<<std::min<int>(int(pack.size()), 148 * 8), 128, 0, sm>>>(
        st->d_items, int(pack.size()), st->d_atom_off, st->d_species, st->d_energy, st->d_pos, st->d_forces,
        st->d_send);
  HMTL_CUDA(cudaGetLastError());
  if (world > 1) {
    if (ncclGroupStart() != ncclSuccess) return fail(HMTL_ERR_COMM, "store_fetch: ncclGroupStart");
    ncclResult_t r = ncclSuccess;
    for (int p = 0; p < world && r == ncclSuccess; ++p) {
      if (p == rank) continue;
      if (send_b[p]) r = ncclSend(st->d_send + send_off[p], size_t(send_b[p]), ncclUint8, p, comm, sm);
      if (r == ncclSuccess && recv_b[p]) r = ncclRecv(st->d_recv + recv_off[p], size_t(recv_b[p]), ncclUint8, p, comm, sm);
    }
    const ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
      return fail(HMTL_ERR_COMM, std::string("store_fetch: NCCL send/recv: ") +
                                     ncclGetErrorString(r != ncclSuccess ? r : r2));
  }
  kl(store_assemble_kernel, dim3(n), dim3(128), 0, sm, static_cast<const FetchItem*>(st->d_items + pack.size()), n,
     static_cast<const long long*>(st->d_atom_off), static_cast<const uint8_t*>(st->d_species),
     static_cast<const double*>(st->d_energy), static_cast<const double*>(st->d_pos),
     static_cast<const double*>(st->d_forces), static_cast<const uint8_t*>(st->d_recv), c.arena);
  HMTL_CUDA(cudaEventRecord(st->staged, sm));
  HMTL_CUDA(cudaGetLastError());
  c.host_G = n;
  {
    std::vector<uint8_t> dsm(n);
    for (int g = 0; g < n; ++g) dsm[g] = mine[g].ds;
    c.head_sorted = sorted_by_slot(c, dsm.data(), n);
  }
  c.host_N = int(N);
  return HMTL_OK;
}

}  // extern "C"

namespace {
// num::solve_gepp_dropping (hmtl/linalg.hpp:11-58): Gaussian elimination with partial
// pivoting through a row permutation; a column whose best pivot is below
// drop_tol * max |diag| is dropped (x = 0, index reported)
std::vector<double> gepp_dropping(std::vector<double> A, size_t k, std::vector<double> b, double drop_tol,
                                  std::vector<size_t>* dropped) {
  double scale = 0.0;
  for (size_t i = 0; i < k; ++i) scale = std::max(scale, std::fabs(A[i * k + i]));
  if (scale == 0.0) scale = 1.0;
  const double tol = drop_tol * scale;
  std::vector<size_t> perm(k);
  for (size_t i = 0; i < k; ++i) perm[i] = i;
  std::vector<char> gone(k, 0);
  for (size_t col = 0; col < k; ++col) {
    size_t best = col;
    double best_v = 0.0;
    for (size_t r = col; r < k; ++r) {
      const double v = std::fabs(A[perm[r] * k + col]);
      if (v > best_v) best_v = v, best = r;
    }
    if (best_v < tol) {
      gone[col] = 1;
      dropped->push_back(col);
      continue;
    }
    std::swap(perm[col], perm[best]);
    const size_t pr = perm[col];
    for (size_t r = col + 1; r < k; ++r) {
      const size_t q = perm[r];
      const double f = A[q * k + col] / A[pr * k + col];
      if (f == 0.0) continue;
      for (size_t c = col; c < k; ++c) A[q * k + c] -= f * A[pr * k + c];
      b[q] -= f * b[pr];
    }
  }
  std::vector<double> x(k, 0.0);
  for (size_t ci = k; ci-- > 0;) {
    if (gone[ci]) continue;
    const size_t pr = perm[ci];
    double acc = b[pr];
    for (size_t c = ci + 1; c < k; ++c) acc -= A[pr * k + c] * x[c];
    x[ci] = acc / A[pr * k + ci];
  }
  return x;
}
}  // namespace

extern "C" {

// align_energies (src/dataset.cpp:306-356) on a device store, in place: per dataset,
// per-element offsets mu_hat by least squares of energy_per_atom on the element
// fractions (normal equations accumulated on the GPU in FP64, deterministic chunk
// order; the <= 20-column solve on the host), then energy -= sum_atoms (mu_d - mu_ref)/n.
int hmtl_store_align(hmtl_store* st, uint8_t ref_dataset_id, uint8_t* ids, double* offsets, int cap,
                     uint8_t* skipped, int* n_skipped) {
  if (!st || !n_skipped) return fail(HMTL_ERR_CONTRACT, "store_align: null argument");
  if (st->by_dataset.size() < 2) return fail(HMTL_ERR_DATA, "align: need at least two datasets");
  if (!st->by_dataset.count(ref_dataset_id)) return fail(HMTL_ERR_DATA, "align: reference dataset not among inputs");
  if (ids && cap < int(st->by_dataset.size())) return fail(HMTL_ERR_CONTRACT, "store_align: buffer too small");
  HMTL_CUDA(cudaSetDevice(st->device));
  // present elements per dataset (host copy of the species: counts are integers)
  std::vector<uint8_t> sp(size_t(st->N));
  HMTL_CUDA(cudaMemcpy(sp.data(), st->d_species, sp.size(), cudaMemcpyDeviceToHost));
  std::vector<long long> off(size_t(st->G) + 1, 0);
  for (int g = 0; g < st->G; ++g) off[g + 1] = off[g] + st->n_atoms[g];
  std::map<int, std::array<double, kElems>> mu;
  std::vector<uint8_t> skip;
  int *d_sel = nullptr, *d_idx = nullptr;
  double *d_F = nullptr, *d_part = nullptr, *d_out = nullptr, *d_mu = nullptr;
  size_t maxg = 0;
  for (const auto& kv : st->by_dataset) maxg = std::max(maxg, kv.second.size());
  const int nbmax = int((maxg + kAlignChunk - 1) / kAlignChunk);
  bool ok = cudaMalloc(&d_sel, maxg * 4) == cudaSuccess && cudaMalloc(&d_idx, 256 * 4) == cudaSuccess &&
            cudaMalloc(&d_F, maxg * kElems * 8) == cudaSuccess &&
            cudaMalloc(&d_part, size_t(nbmax) * (kElems * kElems + kElems) * 8) == cudaSuccess &&
            cudaMalloc(&d_out, (kElems * kElems + kElems) * 8) == cudaSuccess &&
            cudaMalloc(&d_mu, 2 * kElems * 8) == cudaSuccess;
  for (const auto& kv : st->by_dataset) {
    if (!ok) break;
    const std::vector<int>& sel = kv.second;
    const int G = int(sel.size());
    std::array<long long, kElems> cnt{};
    for (int s : sel)
      for (long long i = off[s]; i < off[s + 1]; ++i) cnt[sp[i] < kElems ? sp[i] : 0]++;
    std::vector<int> present, idx(256, -1);
    for (int e = 0; e < kElems; ++e)
      if (cnt[e] > 0) idx[e] = int(present.size()), present.push_back(e);
    const int k = int(present.size()), T = k * k + k, nb = (G + kAlignChunk - 1) / kAlignChunk;
    ok = cudaMemcpy(d_sel, sel.data(), size_t(G) * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(d_idx, idx.data(), 256 * 4, cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) break;
    align_frac_kernel<<<std::min((G + 255) / 256, 148 * 8), 256>>>(d_sel, G, st->d_atom_off, st->d_species, d_idx, k,
                                                                     d_F);
    align_normal_kernel<<<nb, 448>>>(d_F, d_sel, st->d_energy, G, k, d_part);
    align_sum_kernel<<<1, 448>>>(d_part, nb, T, d_out);
    std::vector<double> ne(T);
    ok = cudaMemcpy(ne.data(), d_out, size_t(T) * 8, cudaMemcpyDeviceToHost) == cudaSuccess;
    if (!ok) break;
    std::vector<double> xtx(ne.begin(), ne.begin() + size_t(k) * k), xty(ne.begin() + size_t(k) * k, ne.end());
    std::vector<size_t> dropped;
    const std::vector<double> x = gepp_dropping(xtx, size_t(k), xty, 1e-10, &dropped);
    std::array<double, kElems> m;
    m.fill(std::numeric_limits<double>::quiet_NaN());
    for (int a = 0; a < k; ++a) m[present[a]] = x[a];
    for (size_t d : dropped) m[present[d]] = std::numeric_limits<double>::quiet_NaN(), skip.push_back(uint8_t(present[d]));
    mu[kv.first] = m;
  }
  const std::array<double, kElems> ref = ok ? mu[ref_dataset_id] : std::array<double, kElems>{};
  for (const auto& kv : st->by_dataset) {
    if (!ok) break;
    const std::vector<int>& sel = kv.second;
    const int G = int(sel.size());
    double h_mu[2 * kElems];
    std::copy(mu[kv.first].begin(), mu[kv.first].end(), h_mu);
    std::copy(ref.begin(), ref.end(), h_mu + kElems);
    ok = cudaMemcpy(d_sel, sel.data(), size_t(G) * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(d_mu, h_mu, sizeof h_mu, cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) break;
    align_apply_kernel<<<std::min((G + 255) / 256, 148 * 8), 256>>>(d_sel, G, st->d_atom_off, st->d_species, d_mu,
                                                                     d_mu + kElems, st->d_energy);
    ok = cudaDeviceSynchronize() == cudaSuccess;
  }
  cudaFree(d_sel), cudaFree(d_idx), cudaFree(d_F), cudaFree(d_part), cudaFree(d_out), cudaFree(d_mu);
  if (!ok) return fail(HMTL_ERR_INTERNAL, "store_align: device failure");
  int i = 0;
  for (const auto& kv : mu) {
    if (ids) ids[i] = uint8_t(kv.first);
    if (offsets) std::copy(kv.second.begin(), kv.second.end(), offsets + size_t(i) * kElems);
    ++i;
  }
  if (skipped) std::copy(skip.begin(), skip.end(), skipped);
  *n_skipped = int(skip.size());
  return HMTL_OK;
}

// samples of the store back to host arrays (store order), e.g. to write aligned files
int hmtl_store_download(const hmtl_store* st, int* n_atoms, uint8_t* species, double* positions, double* forces,
                        double* energy, uint8_t* dataset_id) {
  if (!st) return fail(HMTL_ERR_CONTRACT, "store_download: null store");
  HMTL_CUDA(cudaSetDevice(st->device));
  if (n_atoms) std::copy(st->n_atoms.begin(), st->n_atoms.end(), n_atoms);
  if (dataset_id) std::copy(st->ds.begin(), st->ds.end(), dataset_id);
  if (species) HMTL_CUDA(cudaMemcpy(species, st->d_species, size_t(st->N), cudaMemcpyDeviceToHost));
  if (positions) HMTL_CUDA(cudaMemcpy(positions, st->d_pos, size_t(st->N) * 24, cudaMemcpyDeviceToHost));
  if (forces) HMTL_CUDA(cudaMemcpy(forces, st->d_forces, size_t(st->N) * 24, cudaMemcpyDeviceToHost));
  if (energy) HMTL_CUDA(cudaMemcpy(energy, st->d_energy, size_t(st->G) * 8, cudaMemcpyDeviceToHost));
  return HMTL_OK;
}

// align_energies(files, ref, out_files) (hmtl/dataset.hpp:62-70): HMTD files -> device
// store (CRC + parse on the GPU) -> hmtl_store_align -> one aligned file per input
// (header aligned = 1, samples in input order).  offsets[i*20..] for dataset ids[i].
int hmtl_align_energies(int device, const char* const* files, int n_files, uint8_t ref_dataset_id,
                        const char* const* out_files, uint8_t* ids, double* offsets, int cap, uint8_t* skipped,
                        int* n_skipped) {
  if (!files || !out_files || !n_skipped) return fail(HMTL_ERR_CONTRACT, "align: null argument");
  if (n_files < 2) return fail(HMTL_ERR_DATA, "align: need at least two datasets");
  std::vector<uint8_t> file_ds(n_files);
  std::vector<uint64_t> file_n(n_files);
  for (int i = 0; i < n_files; ++i) {
    uint8_t al = 0;
    if (int rc = hmtl_hmtd_read_header(files[i], &file_ds[i], &al, &file_n[i])) return rc;
    if (file_n[i] == 0) return fail(HMTL_ERR_DATA, std::string("align: empty dataset ") + files[i]);
  }
  hmtl_store* st = nullptr;
  if (int rc = hmtl_store_from_hmtd(device, files, n_files, &st)) return rc;
  int rc = hmtl_store_align(st, ref_dataset_id, ids, offsets, cap, skipped, n_skipped);
  std::vector<int> na(st->G);
  std::vector<uint8_t> sp(size_t(st->N)), dsv(st->G);
  std::vector<double> pos(size_t(st->N) * 3), frc(size_t(st->N) * 3), en(st->G);
  if (!rc) rc = hmtl_store_download(st, na.data(), sp.data(), pos.data(), frc.data(), en.data(), dsv.data());
  // the pool holds the files back to back, in order
  long long g0 = 0, a0 = 0;
  for (int i = 0; i < n_files && !rc; ++i) {
    const int G = int(file_n[i]);
    long long n = 0;
    for (int g = 0; g < G; ++g) n += na[g0 + g];
    hmtl_samples smp{G, int(n), na.data() + g0, sp.data() + a0, pos.data() + 3 * a0, frc.data() + 3 * a0,
                     en.data() + g0, dsv.data() + g0};
    rc = hmtl_hmtd_write(out_files[i], file_ds[i], 1, &smp);
    g0 += G, a0 += n;
  }
  hmtl_store_destroy(st);
  return rc;
}

int hmtl_store_shape(const hmtl_store* st, int* G, long long* N) {
  if (!st || !G || !N) return fail(HMTL_ERR_CONTRACT, "store_shape: null argument");
  *G = st->G;
  *N = st->N;
  return HMTL_OK;
}

int hmtl_store_destroy(hmtl_store* st) {
  if (!st) return HMTL_OK;
  cudaSetDevice(st->device);
  if (st->staged) cudaEventSynchronize(st->staged), cudaEventDestroy(st->staged);
  void* ptrs[] = {st->d_atom_off, st->d_ds,    st->d_species, st->d_energy, st->d_pos,
                  st->d_forces,   st->d_sel,   st->d_items,   st->d_send,   st->d_recv, st->d_flag};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (st->h_stage) cudaFreeHost(st->h_stage);
  if (st->h_items) cudaFreeHost(st->h_items);
  delete st;
  return HMTL_OK;
}

}  // extern "C"
