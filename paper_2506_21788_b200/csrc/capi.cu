// capi.cu -- the C ABI (include/hmtl_b200.h): device context, batch upload,
// and the stream-ordered training step.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"

using namespace hmtl_b200;

hmtl_b200::LaunchPrio& hmtl_b200::launch_prio() {
  static thread_local LaunchPrio p;
  return p;
}

bool hmtl_b200::pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("HMTL_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

namespace {

template <class T>
int dalloc(T** p, size_t n) {
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
  if (e != cudaSuccess) return fail(HMTL_ERR_INTERNAL, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return 0;
}

cudaStream_t pick(Ctx& c, void* s) { return s ? static_cast<cudaStream_t>(s) : c.stream; }

int check_hdr(Ctx& c) {
  DevHdr h;
  HMTL_CUDA(cudaMemcpy(&h, c.hdr, sizeof(DevHdr), cudaMemcpyDeviceToHost));
  if (h.err & kErrUnowned) return fail(HMTL_ERR_CONTRACT, "model: unknown dataset id (head not owned by this rank)");
  if (h.err & kErrEmptyGraph) return fail(HMTL_ERR_CONTRACT, "build_batch: empty graph rejected");
  if (h.err & kErrEdgeOverflow) return fail(HMTL_ERR_CONTRACT, "build_batch: edge capacity exceeded");
  if (h.err & kErrNonFinite) return fail(HMTL_ERR_CONTRACT, "model: non-finite prediction");
  return 0;
}

}  // namespace
bool hmtl_b200::sorted_by_slot(const Ctx& c, const uint8_t* ds, int G) {
  for (int g = 1; g < G; ++g)
    if (c.slot_of[ds[g]] < c.slot_of[ds[g - 1]]) return false;
  return true;
}
namespace {

// pack AtomisticSamples into the batch arena format (common.cuh: arena_layout)
int pack(Ctx& c, const hmtl_samples* s, uint8_t* dst, size_t cap, size_t* bytes, bool pbc = false) {
  if (!s || s->G <= 0 || s->N <= 0) return fail(HMTL_ERR_CONTRACT, "model: empty batch rejected");
  if (s->G > c.Gc || s->N > c.Nc) return fail(HMTL_ERR_CONTRACT, "batch exceeds context capacity (graphs/nodes)");
  const ArenaLayout al = arena_layout(s->G, s->N);
  if (al.total > cap) return fail(HMTL_ERR_INTERNAL, "arena too small");
  long long bound = 0, n_sum = 0;
  for (int g = 0; g < s->G; ++g) {
    const long long n = s->n_atoms[g];
    if (n < 1) return fail(HMTL_ERR_CONTRACT, "build_batch: empty graph rejected");
    bound += n * (n - 1);
    n_sum += n;
    if (s->dataset_id[g] >= 255 || c.slot_of[s->dataset_id[g]] < 0)
      return fail(HMTL_ERR_CONTRACT, "model: unknown dataset id " + std::to_string(s->dataset_id[g]) +
                                         " (head not owned by this rank)");
  }
  if (n_sum != s->N) return fail(HMTL_ERR_CONTRACT, "samples: sum(n_atoms) != N");
  // (periodic images can exceed n(n-1): that bound is checked on the device, kErrEdgeOverflow)
  if (!pbc && bound > c.Ec) return fail(HMTL_ERR_CONTRACT, "batch may exceed the context's edge capacity");
  int* hdr = reinterpret_cast<int*>(dst);
  hdr[0] = s->G;
  hdr[1] = s->N;
  hdr[2] = hdr[3] = 0;
  int* go = reinterpret_cast<int*>(dst + al.go);
  go[0] = 0;
  for (int g = 0; g < s->G; ++g) go[g + 1] = go[g] + s->n_atoms[g];
  std::memcpy(dst + al.ds, s->dataset_id, s->G);
  std::memcpy(dst + al.sp, s->species, s->N);
  std::memcpy(dst + al.pos, s->positions, 24 * size_t(s->N));
  if (s->energy_per_atom) std::memcpy(dst + al.le, s->energy_per_atom, 8 * size_t(s->G));
  else std::memset(dst + al.le, 0, 8 * size_t(s->G));
  if (s->forces) std::memcpy(dst + al.lf, s->forces, 24 * size_t(s->N));
  else std::memset(dst + al.lf, 0, 24 * size_t(s->N));
  *bytes = al.total;
  c.host_G = s->G;
  c.host_N = s->N;
  c.head_sorted = sorted_by_slot(c, s->dataset_id, s->G);
  return 0;
}

void free_ctx(Ctx& c) {
  void* ptrs[] = {c.params, c.grads, c.adam_m, c.adam_v, c.hdr, c.d_slot_of, c.arena, c.graph_offset, c.node_graph,
                  c.deg, c.row_ptr, c.edge_src, c.edge_dst, c.rev, c.edge_offset, c.pos32, c.geo, c.dist,
                  c.species, c.gslot, c.gperm, c.gnode_base, c.gedge_base, c.node_perm, c.edge_perm, c.node_arena,
                  c.z2, c.pooled, c.ez, c.energy, c.Qf, c.zf, c.s, c.forces, c.dE, c.dF,
                  c.dzAb, c.dzBb, c.Sb, c.fzA, c.fzB, c.ds, c.dpooled, c.edA, c.edB,
                  c.scratch, c.partial, c.partial_w, c.partial_w2, c.partial_w3, c.loss_terms, c.cells, c.eimg, c.pbc_meta, c.pbc_bins,
                  c.pbc_order, c.pbc_acoord, c.pbc_w2, c.bimg, c.a1, c.af0, c.sf0, c.bimg_all, c.d_bjobs, c.tpart, c.s1pb, c.ptab, c.d_ns};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto* p : c.pool) cudaFree(p);
  if (c.h_arena) cudaFreeHost(c.h_arena);
  if (c.h_arena2) cudaFreeHost(c.h_arena2);
  for (auto& e : c.h_arena_ev)
    if (e) cudaEventDestroy(e);
  if (c.h_hdr_ring) cudaFreeHost(c.h_hdr_ring);
  for (auto& e : c.hdr_ev)
    if (e) cudaEventDestroy(e);
  if (c.h_cells) cudaFreeHost(c.h_cells);
  if (c.step_done) cudaEventDestroy(c.step_done);
  if (c.step_exec) cudaGraphExecDestroy(c.step_exec);
  if (c.prof_exec) cudaGraphExecDestroy(c.prof_exec);
  comm_destroy(c.comm);
  c.comm = nullptr;
  for (auto e : c.evs) cudaEventDestroy(e);
  c.evs.clear();
  if (c.s_e) cudaStreamDestroy(c.s_e);
  if (c.s_w) cudaStreamDestroy(c.s_w);
  if (c.s_w2) cudaStreamDestroy(c.s_w2);
  if (c.s_w3) cudaStreamDestroy(c.s_w3);
  if (c.s_c) cudaStreamDestroy(c.s_c);
  if (c.stream) cudaStreamDestroy(c.stream);
}

int count_kernel_nodes(cudaGraph_t g) {
  size_t n = 0;
  if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess) return -1;
  std::vector<cudaGraphNode_t> nodes(n);
  cudaGraphGetNodes(g, nodes.data(), &n);
  int k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

// add the elapsed time of every recorded (start, end) pair to the scope totals
void prof_harvest(Ctx& c) {
  for (auto& r : c.prof)
    for (size_t i = 0; i + 1 < r.used; i += 2) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, r.ev[i], r.ev[i + 1]) == cudaSuccess) r.acc_ms += t, r.calls += 1;
    }
}

int enqueue_step(Ctx& c, const hmtl_train_cfg& cfg, cudaStream_t st) {
  c.ev_i = 0;
  struct PrioScope {  // kernels on `st` high priority, side streams low, while this step is enqueued
    explicit PrioScope(const Ctx& c, cudaStream_t st) {
      LaunchPrio& p = launch_prio();
      p.on = c.launch_prio;
      p.hi_stream = st;
      cudaDeviceGetStreamPriorityRange(&p.lo, &p.hi);
    }
    ~PrioScope() { launch_prio().on = false; }
  } prio(c, st);
  if (!c.bimg_ready && c.use_tc) {  // record this step's B-image jobs (call order is fixed)
    c.bjobs.clear();
    c.bimg_recording = true;
  }
  // the previous step's AdamW left the tensor-core B images stale: rebuild them on a
  // side stream while the batch preparation and neighbour list run (every graph replay
  // does this; the images are needed from the first layer's GEMM on)
  const bool images = c.bimg_ready && c.use_tc && !c.bimg_recording;
  cudaStream_t sb = c.side(c.s_w, st);
  c.ptab_ready = false;
  if (images) {
    c.dep(st, sb);
    launch_bimg_all(c, sb);
    launch_ptab(c, sb);
  }
  launch_prep(c, st);
  launch_nbr(c, st);
  if (images) c.dep(sb, st);
  launch_forward(c, st);
  c.ptab_ready = false;  // (only this step's captured forward reads the table)
  launch_loss(c, cfg.w_energy, cfg.w_force, st);
  launch_backward(c, st, true);  // with a communicator: bucketed allreduces overlap it
  if (c.comm_err) {
    c.comm_err = 0;
    return fail(HMTL_ERR_COMM, "NCCL: bucketed gradient allreduce failed");
  }
  if (c.comm && !comm_overlap(c)) {
    int rc = comm_sync_grads(c, st);
    if (rc) return rc;
  }
  launch_adamw(c, cfg, st, /*defer_images=*/!c.bimg_recording);
  return 0;
}

// standalone API calls after a train step: refresh the deferred B images first
int fresh_images(Ctx& c, cudaStream_t st) {
  if (c.bimg_stale) {
    launch_bimg_all(c, st);
    c.bimg_stale = false;
  }
  return 0;
}

}  // namespace

extern "C" {

int hmtl_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

namespace {
// persisting L2 window over the node tables on every step stream and (graph capture
// keeps it per kernel node) in the captured step: the ~100 MB of edge tensors each
// layer streams through the 126 MB L2 no longer evict the node rows the next
// kernels gather and the node chains read
cudaAccessPolicyWindow l2_window(const Ctx& c) {
  cudaAccessPolicyWindow w{};
  if (c.l2_persist_mb <= 0 || !c.node_arena) return w;
  int dev = 0, max_win = 0, max_persist = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  const size_t persist = std::min(size_t(c.l2_persist_mb) << 20, size_t(max_persist));
  w.base_ptr = c.node_arena;
  w.num_bytes = std::min(c.node_arena_bytes, size_t(max_win));
  w.hitRatio = w.num_bytes ? float(std::min(1.0, double(persist) / double(w.num_bytes))) : 0.f;
  w.hitProp = cudaAccessPropertyPersisting;
  w.missProp = cudaAccessPropertyStreaming;
  return w;
}
void apply_l2_window(Ctx& c) {
  const cudaAccessPolicyWindow w = l2_window(c);
  if (!w.num_bytes) return;
  int dev = 0, max_persist = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(size_t(c.l2_persist_mb) << 20, size_t(max_persist)));
  cudaStreamAttrValue v{};
  v.accessPolicyWindow = w;
  for (cudaStream_t s : {c.stream, c.s_e, c.s_w, c.s_w2, c.s_w3})
    if (s) cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
  if (std::getenv("HMTL_COMM_LOG"))
    std::fprintf(stderr, "hmtl: L2 persisting window %zu B, hit ratio %.2f (device max %d B)\n", w.num_bytes,
                 double(w.hitRatio), max_persist);
}
void graph_l2_window(const Ctx& c, cudaGraph_t g) {
  const cudaAccessPolicyWindow w = l2_window(c);
  if (!w.num_bytes) return;
  size_t n = 0;
  cudaGraphGetNodes(g, nullptr, &n);
  std::vector<cudaGraphNode_t> nodes(n);
  cudaGraphGetNodes(g, nodes.data(), &n);
  cudaKernelNodeAttrValue v{};
  v.accessPolicyWindow = w;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel)
      cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v);
  }
}
}  // namespace

int hmtl_ctx_create(int device, const hmtl_hyper* hp, uint64_t seed, const int* owned, int n_owned,
                    const hmtl_caps* caps, hmtl_ctx** out) {
  if (!hp || !caps || !out) return fail(HMTL_ERR_CONTRACT, "ctx_create: null argument");
  if (hp->hidden < 1 || hp->head_width < 1 || hp->layers < 1 || hp->n_species < 1 || hp->n_heads < 1 ||
      hp->n_heads > 255)
    return fail(HMTL_ERR_CONFIG, "ctx_create: invalid hyperparameters");
  if (hp->head_depth < 2) return fail(HMTL_ERR_CONFIG, "ctx_create: head_depth >= 2 required on the GPU path");
  if (n_owned < 1 || n_owned > kMaxSlots) return fail(HMTL_ERR_CONFIG, "ctx_create: 1..16 owned heads per rank");
  if (caps->max_graphs < 1 || caps->max_nodes < 1 || caps->max_edges < 1)
    return fail(HMTL_ERR_CONFIG, "ctx_create: capacities must be positive");
  int ndev = hmtl_device_count();
  if (device < 0 || device >= ndev)
    return fail(HMTL_ERR_INTERNAL, "ctx_create: no CUDA device " + std::to_string(device) +
                                       " (the B200 path has no CPU fallback)");
  HMTL_CUDA(cudaSetDevice(device));
  auto* h = new hmtl_ctx;
  Ctx& c = h->c;
  c.device = device;
  c.hp = *hp;
  c.H = hp->hidden;
  c.W = hp->head_width;
  c.L = hp->layers;
  c.D = hp->head_depth;
  c.NS = hp->n_species;
  c.rc2 = hp->cutoff * hp->cutoff;
  std::fill(c.slot_of, c.slot_of + 256, -1);
  c.owned.assign(owned, owned + n_owned);
  std::sort(c.owned.begin(), c.owned.end());
  for (size_t s = 0; s < c.owned.size(); ++s) {
    const int k = c.owned[s];
    if (k < 0 || k >= hp->n_heads || (s && c.owned[s - 1] == k)) {
      delete h;
      return fail(HMTL_ERR_CONTRACT, "model: head index out of range");
    }
    c.slot_of[k] = int(s);
  }
  c.S = int(c.owned.size());
  c.shared_lay = make_layout(*hp, true);
  c.head_lay = make_layout(*hp, false);
  c.PS = c.shared_lay.total;
  c.PH = c.head_lay.total;
  c.PT = c.PS + size_t(c.S) * c.PH;
  c.Gc = caps->max_graphs;
  c.Nc = caps->max_nodes;
  c.Ec = caps->max_edges;
  cudaDeviceGetAttribute(&c.sm_count, cudaDevAttrMultiProcessorCount, device);
  int rc = 0;
  auto A = [&](auto** p, size_t n) {
    if (!rc) rc = dalloc(p, n);
  };
  const size_t H = c.H, W = c.W, L = c.L, D = c.D;
  const size_t N = c.Nc, E = c.Ec, G = c.Gc;
  {  // step stream at the highest priority: side-branch CTAs yield SMs to the critical path
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&c.stream, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c.s_e, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c.s_w, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c.s_w2, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c.s_w3, cudaStreamNonBlocking, lo) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c.s_c, cudaStreamNonBlocking, hi) != cudaSuccess)
      rc = HMTL_ERR_INTERNAL;
  }
  if (const char* e = std::getenv("HMTL_SINGLE_STREAM")) c.multi_stream = e[0] == '0';
  if (const char* e = std::getenv("HMTL_NO_CHAIN")) c.fuse_chain = e[0] == '0';
  if (const char* e = std::getenv("HMTL_CHAIN_PAIR")) c.chain_pair = std::atoi(e) != 0;
  if (const char* e = std::getenv("HMTL_L2_PERSIST_MB")) c.l2_persist_mb = std::atoi(e);
  if (const char* e = std::getenv("HMTL_CHAIN_PREFETCH")) c.chain_prefetch = std::atoi(e);
  if (const char* e = std::getenv("HMTL_ROW_PREFETCH")) c.row_prefetch = std::atoi(e);
  if (const char* e = std::getenv("HMTL_FUSE_EDGE")) c.fuse_edge = e[0] == '1';
  if (const char* e = std::getenv("HMTL_ASYNC_FWD")) c.async_fwd = e[0] == '1';
  if (const char* e = std::getenv("HMTL_FUSE_FORCE_OUT")) c.fuse_force_out = e[0] == '1';
  if (const char* e = std::getenv("HMTL_LAUNCH_PRIO")) c.launch_prio = e[0] == '1';
  if (const char* e = std::getenv("HMTL_BIMG_BLOCKS")) c.bimg_blocks = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("HMTL_ASYNC_BWD")) c.async_bwd = std::atoi(e);
  if (const char* e = std::getenv("HMTL_TC_DEBUG")) set_tc_debug(std::atoi(e));
  if (const char* e = std::getenv("HMTL_TC_GRID")) c.tc_grid_mult = std::atoi(e);
  // weight-gradient grids over ~13/16 of the SMs: the side-stream reduce GEMMs then leave SMs to the
  // critical path (measured: 120 of 148 -> step 1.003 -> 0.994 ms; profiles/r01_ab_red_knobs.txt)
  c.red_sms = std::max(1, c.sm_count * 13 / 16);
  if (const char* e = std::getenv("HMTL_CHAIN_M")) c.chain_mr = std::atoi(e) == 64 ? 64 : 128;
  if (const char* e = std::getenv("HMTL_CHAIN_M_FWD")) c.chain_mr_fwd = std::atoi(e) == 64 ? 64 : (std::atoi(e) == 128 ? 128 : 0);
  if (const char* e = std::getenv("HMTL_CHAIN_CS")) c.chain_cs = std::atoi(e) == 4 ? 4 : (std::atoi(e) == 2 ? 2 : 1);
  if (const char* e = std::getenv("HMTL_NO_RED_TMA")) c.red_tma = e[0] == '0';
  if (const char* e = std::getenv("HMTL_RED_SEGX")) c.red_seg_mult = std::max(1, std::min(8, std::atoi(e)));
  if (const char* e = std::getenv("HMTL_RED_MINCH")) c.red_min_chunks = std::max(1, std::atoi(e));
  c.red_min_tail = c.red_min_chunks;
  if (const char* e = std::getenv("HMTL_RED_MINCH_TAIL")) c.red_min_tail = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("HMTL_RED_SMS")) c.red_sms = std::max(1, std::min(c.sm_count, std::atoi(e)));
  c.red_sms_early = c.red_sms_now = c.red_sms;
  if (const char* e = std::getenv("HMTL_RED_CLUSTER")) {
    const int v = std::atoi(e);
    c.red_cluster = v >= 8 ? 8 : (v >= 4 ? 4 : (v >= 2 ? 2 : 1));
  }
  if (const char* e = std::getenv("HMTL_RED_SMS_EARLY")) c.red_sms_early = std::max(1, std::min(c.sm_count, std::atoi(e)));
  c.row_sms = c.sm_count;
  if (const char* e = std::getenv("HMTL_ROW_SMS")) c.row_sms = std::max(1, std::min(c.sm_count, std::atoi(e)));
  if (const char* e = std::getenv("HMTL_NO_PREFETCH")) c.prefetch_l2 = e[0] == '0';
  if (const char* e = std::getenv("HMTL_NO_COMM_OVERLAP")) c.overlap_comm = e[0] == '0';
  if (std::getenv("HMTL_CHAIN_STAMPS")) A(&c.chain_stamps, size_t(4096) * 32);
  if (const char* e = std::getenv("HMTL_CHAIN_DBG")) c.chain_dbg = std::atoi(e);
  if (const char* e = std::getenv("HMTL_DBG_SKIP_WGRAD")) c.dbg_skip_wgrad = e[0] == '1';
  A(&c.params, c.PT);
  A(&c.grads, c.PT);
  A(&c.adam_m, c.PT);
  A(&c.adam_v, c.PT);
  A(&c.hdr, 1);
  A(&c.d_slot_of, 256);
  c.arena_cap = arena_layout(c.Gc, c.Nc).total;
  A(&c.arena, c.arena_cap);
  A(&c.graph_offset, G + 1);
  A(&c.node_graph, N);
  A(&c.deg, N);
  A(&c.row_ptr, N + 1);
  A(&c.edge_src, E);
  A(&c.edge_dst, E);
  A(&c.rev, E);
  A(&c.edge_offset, G + 1);
  A(&c.pos32, N);
  A(&c.geo, E);
  A(&c.dist, E);
  A(&c.cells, G * 9);
  A(&c.eimg, E);
  A(&c.pbc_meta, G);
  A(&c.pbc_bins, G * 65);
  A(&c.pbc_order, N);
  A(&c.pbc_acoord, N);
  A(&c.pbc_w2, N);
  A(&c.species, N);
  A(&c.gslot, G);
  A(&c.gperm, G);
  A(&c.gnode_base, G);
  A(&c.gedge_base, G);
  A(&c.node_perm, N);
  A(&c.edge_perm, E);
  {  // node tables: one allocation (256 B aligned pieces), the L2 persisting window
    const size_t parts[] = {(L + 1) * N * H, L * N * 2 * H, L * N * H, L * N * H, N * H, (L + 1) * N * H, L * N * H};
    float** dst[] = {&c.hs, &c.P, &c.agg, &c.vz1, &c.dagg, &c.dhb, &c.dvz1b};
    size_t tot = 0;
    for (size_t n : parts) tot += (n + 63) & ~size_t(63);
    A(&c.node_arena, tot);
    if (!rc) {
      size_t o = 0;
      for (int i = 0; i < 7; ++i) *dst[i] = c.node_arena + o, o += (parts[i] + 63) & ~size_t(63);
    }
    c.node_arena_bytes = tot * sizeof(float);
  }
  A(&c.z2, L * E * H);
  A(&c.pooled, G * H);
  A(&c.ez, D * G * W);
  A(&c.energy, G);
  A(&c.Qf, N * W);
  A(&c.zf, std::max<size_t>(D - 2, 1) * E * W);
  A(&c.s, E);
  A(&c.forces, 3 * N);
  A(&c.dE, G);
  A(&c.dF, 3 * N);
  A(&c.dzAb, L * E * H);
  A(&c.dzBb, L * E * H);
  A(&c.Sb, (L + 1) * N * 2 * std::max(H, W));
  A(&c.fzA, E * W);
  A(&c.fzB, E * W);
  A(&c.ds, E);
  A(&c.dpooled, G * H);
  A(&c.loss_terms, G);
  A(&c.edA, G * W);
  A(&c.edB, G * W);
  A(&c.scratch, E * std::max(H, W));
  auto clampi = [](long long v, long long lo, long long hi) { return int(std::min(std::max(v, lo), hi)); };
  c.nsplit_node = clampi((c.Nc + 63) / 64, 1, 64);
  c.nsplit_edge = clampi((c.Ec + 127) / 128, 1, 64);
  c.nsplit_graph = clampi((c.Gc + 15) / 16, 1, 16);
  const size_t kn_shared = (2 * H + 1) * H;
  const size_t kn_head = std::max({(H + 1) * W, (W + 1) * W, H * W, 2 * W});
  c.partial_cap = std::max(size_t(64) * kn_shared, size_t(c.S) * 64 * kn_head);
  c.partial_cap = std::max(c.partial_cap, size_t(std::max(c.S, 1)) * 128 * (2 * std::max(H, W) + 1) * std::max(H, W));
  // chunked column sums (colsum2, force output layer): [S][E/128 chunks][2*max(H,W)+1]
  c.partial_cap = std::max(c.partial_cap, size_t(std::max(c.S, 1)) * size_t((E + 127) / 128 + 1) * (2 * std::max(H, W) + 1));
  A(&c.partial, c.partial_cap);
  A(&c.partial_w, c.partial_cap);
  A(&c.partial_w2, c.partial_cap);
  A(&c.partial_w3, c.partial_cap);
  c.bimg_cap = size_t(std::max(c.S, 2)) * 2 * (2 * std::max(H, W)) * (2 * std::max(H, W));
  A(&c.bimg, c.bimg_cap);
  if (const char* e = std::getenv("HMTL_NO_TC")) c.use_tc = e[0] == '0';
  c.store_a1 = c.use_tc && H % 32 == 0;
  c.store_af0 = c.use_tc && W % 32 == 0 && H % 4 == 0;
  c.store_sf0 = c.store_af0;  // (regathering silu'(zf0) from Qf in FDx's epilogue measured slower)
  A(&c.a1, c.store_a1 ? L * E * H : 1);
  if (const char* e = std::getenv("HMTL_Z1_ONLY")) c.z1_only = e[0] == '1';
  c.z1_only = c.z1_only && c.store_a1 && !c.fuse_edge && !c.async_fwd;
  A(&c.s1pb, c.store_a1 && (c.async_fwd || (c.async_bwd == 1 && !c.z1_only)) ? L * E * H : 1);
  A(&c.af0, c.store_af0 ? E * W : 1);
  A(&c.sf0, c.store_sf0 ? E * W : 1);
  c.tcap = int((E + 127) / 128 + 1);
  A(&c.tpart, size_t(2) * c.tcap * H);
  A(&c.ptab, size_t(std::max(c.NS, 1)) * 2 * H);
  A(&c.d_ns, 1);
  if (!rc) cudaMemcpy(c.d_ns, &c.NS, sizeof(int), cudaMemcpyHostToDevice);
  if (const char* e = std::getenv("HMTL_PTAB")) c.ptab_on = e[0] != '0';
  if (const char* e = std::getenv("HMTL_WGRAD3")) c.wgrad3 = std::atoi(e);
  if (const char* e = std::getenv("HMTL_ROW_PAIR")) c.row_pair = e[0] == '1';
  if (rc) {
    free_ctx(c);
    delete h;
    return rc;
  }
  apply_l2_window(c);
  // parameters exactly as ModelT's ctor (hmtl/model.hpp:162-166)
  std::vector<float> host(c.PT);
  init_block(*hp, seed, -1, host.data());
  for (int s = 0; s < c.S; ++s) init_block(*hp, seed, c.owned[s], host.data() + c.PS + size_t(s) * c.PH);
  cudaMemcpy(c.params, host.data(), c.PT * sizeof(float), cudaMemcpyHostToDevice);
  cudaMemset(c.adam_m, 0, c.PT * sizeof(float));
  cudaMemset(c.adam_v, 0, c.PT * sizeof(float));
  cudaMemset(c.grads, 0, c.PT * sizeof(float));
  cudaMemset(c.hdr, 0, sizeof(DevHdr));
  cudaMemcpy(c.d_slot_of, c.slot_of, 256 * sizeof(int), cudaMemcpyHostToDevice);
  c.h_arena_cap = c.arena_cap;
  bool pinned_ok = cudaMallocHost(&c.h_arena2, c.h_arena_cap) == cudaSuccess &&
                   cudaMallocHost(&c.h_hdr_ring, sizeof(DevHdr) * Ctx::kLossRing) == cudaSuccess;
  for (auto& e : c.h_arena_ev) pinned_ok = pinned_ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  for (auto& e : c.hdr_ev) pinned_ok = pinned_ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  if (!pinned_ok || cudaMallocHost(&c.h_arena, c.h_arena_cap) != cudaSuccess) {
    free_ctx(c);
    delete h;
    return fail(HMTL_ERR_INTERNAL, "cudaMallocHost failed");
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    free_ctx(c);
    delete h;
    return fail(HMTL_ERR_INTERNAL, std::string("ctx_create: ") + cudaGetErrorString(e));
  }
  *out = h;
  return 0;
}

void hmtl_ctx_destroy(hmtl_ctx* h) {
  if (!h) return;
  cudaSetDevice(h->c.device);
  cudaDeviceSynchronize();
  free_ctx(h->c);
  delete h;
}

void* hmtl_ctx_stream(hmtl_ctx* h) { return h ? h->c.stream : nullptr; }

// Grow the capacity-padded batch buffers in place.  Everything that outlives a
// batch -- parameters, gradients, AdamW m/v, the device header (step counter),
// streams (callers may hold hmtl_ctx_stream), the NCCL communicators, the
// recorded tensor-core B images and the batch pool -- stays with the handle; only
// the capacity-sized buffers are replaced and the captured step graph dropped.
int hmtl_ctx_reserve(hmtl_ctx* h, const hmtl_caps* need) {
  if (!h || !need) return fail(HMTL_ERR_CONTRACT, "ctx_reserve: null argument");
  Ctx& c = h->c;
  if (need->max_graphs <= c.Gc && need->max_nodes <= c.Nc && need->max_edges <= c.Ec) return 0;
  hmtl_caps caps{std::max(need->max_graphs, c.Gc), std::max(need->max_nodes, c.Nc), std::max(need->max_edges, c.Ec)};
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaDeviceSynchronize());
  hmtl_ctx* fresh = nullptr;
  if (int rc = hmtl_ctx_create(c.device, &c.hp, 0, c.owned.data(), int(c.owned.size()), &caps, &fresh)) return rc;
  Ctx& n = fresh->c;
  std::swap(c, n);  // c: new capacity buffers; n: the old context
  // state that outlives a batch goes back to the handle (n's copies are freed with it)
  std::swap(c.params, n.params);
  std::swap(c.grads, n.grads);
  std::swap(c.adam_m, n.adam_m);
  std::swap(c.adam_v, n.adam_v);
  std::swap(c.hdr, n.hdr);
  std::swap(c.stream, n.stream);
  std::swap(c.s_e, n.s_e);
  std::swap(c.s_w, n.s_w);
  std::swap(c.s_w2, n.s_w2);
  std::swap(c.s_w3, n.s_w3);
  std::swap(c.s_c, n.s_c);
  std::swap(c.comm, n.comm);
  std::swap(c.pool, n.pool);
  std::swap(c.pool_bytes, n.pool_bytes);
  std::swap(c.pool_sorted, n.pool_sorted);
  c.head_sorted = n.head_sorted;
  std::swap(c.bimg_all, n.bimg_all);
  std::swap(c.bimg_all_cap, n.bimg_all_cap);
  std::swap(c.d_bjobs, n.d_bjobs);
  std::swap(c.bjobs, n.bjobs);
  std::swap(c.n_djobs, n.n_djobs);
  std::swap(c.bimg_rows, n.bimg_rows);
  std::swap(c.bimg_ready, n.bimg_ready);
  std::swap(c.bimg_stale, n.bimg_stale);
  std::swap(c.prof_on, n.prof_on);
  std::swap(c.host_G, n.host_G);
  std::swap(c.host_N, n.host_N);
  // tuning knobs set after creation
  c.multi_stream = n.multi_stream;
  c.overlap_comm = n.overlap_comm;
  apply_l2_window(c);  // (the step streams came back from the old context: window over the new arena)
  hmtl_ctx_destroy(fresh);  // frees the old capacity buffers and the old step graph
  return 0;
}

static int block_span(Ctx& c, int which, size_t* off, size_t* n) {
  if (which < 0) {
    *off = 0;
    *n = c.PS;
    return 0;
  }
  if (which >= 256 || c.slot_of[which] < 0) return fail(HMTL_ERR_CONTRACT, "head not owned by this rank");
  *off = c.PS + size_t(c.slot_of[which]) * c.PH;
  *n = c.PH;
  return 0;
}

int hmtl_set_block(hmtl_ctx* h, int which, const float* host) {
  size_t off, n;
  if (int rc = block_span(h->c, which, &off, &n)) return rc;
  cudaSetDevice(h->c.device);
  HMTL_CUDA(cudaMemcpy(h->c.params + off, host, n * sizeof(float), cudaMemcpyHostToDevice));
  if (h->c.bimg_ready) {  // prebuilt B images are stale now
    launch_bimg_all(h->c, h->c.stream);
    HMTL_CUDA(cudaStreamSynchronize(h->c.stream));
  }
  return 0;
}
int hmtl_get_block(hmtl_ctx* h, int which, float* host) {
  size_t off, n;
  if (int rc = block_span(h->c, which, &off, &n)) return rc;
  cudaSetDevice(h->c.device);
  HMTL_CUDA(cudaStreamSynchronize(h->c.stream));
  HMTL_CUDA(cudaMemcpy(host, h->c.params + off, n * sizeof(float), cudaMemcpyDeviceToHost));
  return 0;
}
int hmtl_get_grad(hmtl_ctx* h, int which, float* host) {
  size_t off, n;
  if (int rc = block_span(h->c, which, &off, &n)) return rc;
  cudaSetDevice(h->c.device);
  HMTL_CUDA(cudaStreamSynchronize(h->c.stream));
  HMTL_CUDA(cudaMemcpy(host, h->c.grads + off, n * sizeof(float), cudaMemcpyDeviceToHost));
  return 0;
}

int hmtl_checkpoint_save(hmtl_ctx* h, const char* path, int with_optimizer) {
  Ctx& c = h->c;
  if (!path) return fail(HMTL_ERR_CONTRACT, "checkpoint: null path");
  if (int(c.owned.size()) != c.hp.n_heads)
    return fail(HMTL_ERR_CONTRACT, "checkpoint: need all head blocks in head-index order");
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaDeviceSynchronize());
  std::vector<float> p(c.PT), m, v;
  HMTL_CUDA(cudaMemcpy(p.data(), c.params, c.PT * 4, cudaMemcpyDeviceToHost));
  std::vector<const float*> hp(c.hp.n_heads), hm(c.hp.n_heads), hv(c.hp.n_heads);
  for (int k = 0; k < c.hp.n_heads; ++k) hp[k] = p.data() + c.PS + size_t(c.slot_of[k]) * c.PH;
  hmtl_ckpt_opt opt{};
  if (with_optimizer) {
    m.resize(c.PT), v.resize(c.PT);
    DevHdr hd;
    HMTL_CUDA(cudaMemcpy(m.data(), c.adam_m, c.PT * 4, cudaMemcpyDeviceToHost));
    HMTL_CUDA(cudaMemcpy(v.data(), c.adam_v, c.PT * 4, cudaMemcpyDeviceToHost));
    HMTL_CUDA(cudaMemcpy(&hd, c.hdr, sizeof hd, cudaMemcpyDeviceToHost));
    for (int k = 0; k < c.hp.n_heads; ++k) {
      hm[k] = m.data() + c.PS + size_t(c.slot_of[k]) * c.PH;
      hv[k] = v.data() + c.PS + size_t(c.slot_of[k]) * c.PH;
    }
    opt = hmtl_ckpt_opt{uint64_t(hd.step), m.data(), v.data(), hm.data(), hv.data()};
  }
  return hmtp_write(path, c.hp, p.data(), c.PS, hp.data(), c.PH, c.hp.n_heads, with_optimizer ? &opt : nullptr);
}

int hmtl_checkpoint_load(hmtl_ctx* h, const char* path) {
  Ctx& c = h->c;
  hmtl_hyper fh{};
  std::vector<double> sh;
  std::vector<std::vector<double>> hd, opt;
  bool has_opt = false;
  uint64_t step = 0;
  if (int rc = hmtp_read(path, &fh, &sh, &hd, &has_opt, &step, &opt)) return rc;
  if (fh.n_species != c.hp.n_species || fh.layers != c.hp.layers || fh.hidden != c.hp.hidden ||
      fh.head_width != c.hp.head_width || fh.head_depth != c.hp.head_depth || fh.n_heads != c.hp.n_heads)
    return fail(HMTL_ERR_CONFIG, "checkpoint: hyperparameters differ from the context's");
  std::vector<float> p(c.PT), m(c.PT, 0.f), v(c.PT, 0.f);
  auto put = [&](std::vector<float>& dst, size_t off, const std::vector<double>& src) {
    for (size_t i = 0; i < src.size(); ++i) dst[off + i] = float(src[i]);  // exact: written from FP32
  };
  put(p, 0, sh);
  if (has_opt) put(m, 0, opt[0]), put(v, 0, opt[1]);
  for (size_t s = 0; s < c.owned.size(); ++s) {
    const int k = c.owned[s];
    put(p, c.PS + s * c.PH, hd[k]);
    if (has_opt) put(m, c.PS + s * c.PH, opt[2 + 2 * k]), put(v, c.PS + s * c.PH, opt[3 + 2 * k]);
  }
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaDeviceSynchronize());
  HMTL_CUDA(cudaMemcpy(c.params, p.data(), c.PT * 4, cudaMemcpyHostToDevice));
  HMTL_CUDA(cudaMemcpy(c.adam_m, m.data(), c.PT * 4, cudaMemcpyHostToDevice));
  HMTL_CUDA(cudaMemcpy(c.adam_v, v.data(), c.PT * 4, cudaMemcpyHostToDevice));
  DevHdr hdr;
  HMTL_CUDA(cudaMemcpy(&hdr, c.hdr, sizeof hdr, cudaMemcpyDeviceToHost));
  hdr.step = has_opt ? int(step) : 0;
  HMTL_CUDA(cudaMemcpy(c.hdr, &hdr, sizeof hdr, cudaMemcpyHostToDevice));
  if (c.bimg_ready) {  // weights changed: rebuild the tensor-core B images
    launch_bimg_all(c, c.stream);
    HMTL_CUDA(cudaStreamSynchronize(c.stream));
  }
  return 0;
}

int hmtl_batch_upload(hmtl_ctx* h, const hmtl_samples* s, void* stream) {
  Ctx& c = h->c;
  c.pbc = false;
  cudaSetDevice(c.device);
  cudaStream_t st = pick(c, stream);
  // two pinned staging arenas used alternately: packing this batch waits only for
  // the copy that last read this buffer, so the host packs step i+1 while the
  // device still runs step i (the copy itself is stream-ordered after it)
  const int k = c.h_arena_k;
  uint8_t* buf = k ? c.h_arena2 : c.h_arena;
  HMTL_CUDA(cudaEventSynchronize(c.h_arena_ev[k]));
  size_t bytes = 0;
  if (int rc = pack(c, s, buf, c.h_arena_cap, &bytes)) return rc;
  HMTL_CUDA(cudaMemcpyAsync(c.arena, buf, bytes, cudaMemcpyHostToDevice, st));
  HMTL_CUDA(cudaEventRecord(c.h_arena_ev[k], st));
  c.h_arena_k = k ^ 1;
  return 0;
}

int hmtl_batch_upload_pbc(hmtl_ctx* h, const hmtl_samples* s, const double* cells, void* stream) {
  Ctx& c = h->c;
  if (!cells) return fail(HMTL_ERR_CONTRACT, "pbc: null cell array");
  cudaSetDevice(c.device);
  cudaStream_t st = pick(c, stream);
  HMTL_CUDA(cudaStreamSynchronize(st));  // the pinned staging buffers may still be read
  for (auto& e : c.h_arena_ev) HMTL_CUDA(cudaEventSynchronize(e));
  size_t bytes = 0;
  if (int rc = pack(c, s, c.h_arena, c.h_arena_cap, &bytes, true)) return rc;
  if (!c.h_cells) HMTL_CUDA(cudaMallocHost(&c.h_cells, size_t(c.Gc) * 9 * sizeof(double)));
  std::memcpy(c.h_cells, cells, size_t(s->G) * 9 * sizeof(double));
  HMTL_CUDA(cudaMemcpyAsync(c.arena, c.h_arena, bytes, cudaMemcpyHostToDevice, st));
  HMTL_CUDA(cudaMemcpyAsync(c.cells, c.h_cells, size_t(s->G) * 9 * sizeof(double), cudaMemcpyHostToDevice, st));
  c.pbc = true;
  return 0;
}

int hmtl_batch_edge_images(hmtl_ctx* h, int* img) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaDeviceSynchronize());
  if (int rc = check_hdr(c)) return rc;
  DevHdr hd;
  HMTL_CUDA(cudaMemcpy(&hd, c.hdr, sizeof hd, cudaMemcpyDeviceToHost));
  std::vector<int> key(hd.E > 0 ? hd.E : 1, 2184);  // 2184 = image (0, 0, 0)
  if (c.pbc && hd.E > 0) HMTL_CUDA(cudaMemcpy(key.data(), c.eimg, size_t(hd.E) * 4, cudaMemcpyDeviceToHost));
  for (int e = 0; e < hd.E; ++e) {
    img[3 * e] = (key[e] >> 8) - 8;
    img[3 * e + 1] = ((key[e] >> 4) & 15) - 8;
    img[3 * e + 2] = (key[e] & 15) - 8;
  }
  return 0;
}

int hmtl_pool_add(hmtl_ctx* h, const hmtl_samples* s, int* slot) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  std::vector<uint8_t> tmp(c.arena_cap);
  size_t bytes = 0;
  if (int rc = pack(c, s, tmp.data(), tmp.size(), &bytes)) return rc;
  uint8_t* d = nullptr;
  HMTL_CUDA(cudaMalloc(&d, bytes));
  HMTL_CUDA(cudaMemcpy(d, tmp.data(), bytes, cudaMemcpyHostToDevice));
  c.pool.push_back(d);
  c.pool_bytes.push_back(bytes);
  c.pool_sorted.push_back(c.head_sorted);
  if (slot) *slot = int(c.pool.size()) - 1;
  return 0;
}

int hmtl_pool_bind(hmtl_ctx* h, int slot, void* stream) {
  Ctx& c = h->c;
  if (slot < 0 || slot >= int(c.pool.size())) return fail(HMTL_ERR_CONTRACT, "pool_bind: bad slot");
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaMemcpyAsync(c.arena, c.pool[slot], c.pool_bytes[slot], cudaMemcpyDeviceToDevice, pick(c, stream)));
  c.head_sorted = c.pool_sorted[slot];
  return 0;
}

int hmtl_build_batch(hmtl_ctx* h, void* stream) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  cudaStream_t st = pick(c, stream);
  launch_prep(c, st);
  launch_nbr(c, st);
  HMTL_CUDA(cudaGetLastError());
  return 0;
}

// build_batch's edge construction without a model (hmtl/graph.hpp:46-83): a
// scratch context sized to the batch (every dataset id accepted), the same
// kernels as the training step (bit-exact FP64 cutoff test, dst-major CSR).
int hmtl_nbr_build(int device, const hmtl_samples* s, double cutoff, long long cap, int* E, int* edge_dst,
                   int* edge_src, int* edge_offset, int* row_ptr, int* rev) {
  if (!s || !E) return fail(HMTL_ERR_CONTRACT, "nbr_build: null argument");
  if (s->G <= 0 || s->N <= 0) return fail(HMTL_ERR_CONTRACT, "build_batch: empty batch rejected");
  long long bound = 0;
  for (int g = 0; g < s->G; ++g) {
    const long long n = s->n_atoms[g];
    if (n < 1) return fail(HMTL_ERR_CONTRACT, "build_batch: empty graph rejected");
    bound += n * (n - 1);
  }
  hmtl_hyper hp{1, 1, 1, 1, 2, 1, cutoff};
  const int owned = 0;
  const hmtl_caps caps{s->G, s->N, std::max(bound, 1LL)};
  hmtl_ctx* h = nullptr;
  if (int rc = hmtl_ctx_create(device, &hp, 0, &owned, 1, &caps, &h)) return rc;
  Ctx& c = h->c;
  std::fill(c.slot_of, c.slot_of + 256, 0);  // no heads here: every dataset id maps to slot 0
  int rc = 0;
  if (cudaMemcpy(c.d_slot_of, c.slot_of, 256 * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess)
    rc = fail(HMTL_ERR_INTERNAL, "nbr_build: slot table upload failed");
  if (!rc) rc = hmtl_batch_upload(h, s, nullptr);
  if (!rc) rc = hmtl_build_batch(h, nullptr);
  if (!rc) rc = hmtl_batch_edges(h, E, nullptr, nullptr, nullptr);
  if (!rc && (edge_dst || edge_src || rev) && *E > cap)
    rc = fail(HMTL_ERR_CONTRACT, "nbr_build: " + std::to_string(*E) + " edges exceed the output capacity");
  if (!rc) rc = hmtl_batch_edges(h, E, edge_dst, edge_src, edge_offset);
  const size_t ne = size_t(*E);
  if (!rc && row_ptr && cudaMemcpy(row_ptr, c.row_ptr, (size_t(s->N) + 1) * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(HMTL_ERR_INTERNAL, "nbr_build: row_ptr copy failed");
  if (!rc && rev && ne && cudaMemcpy(rev, c.rev, ne * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(HMTL_ERR_INTERNAL, "nbr_build: rev copy failed");
  hmtl_ctx_destroy(h);
  return rc;
}

int hmtl_batch_edges(hmtl_ctx* h, int* E, int* edge_dst, int* edge_src, int* edge_offset) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaStreamSynchronize(c.stream));
  HMTL_CUDA(cudaDeviceSynchronize());
  if (int rc = check_hdr(c)) return rc;
  DevHdr hd;
  HMTL_CUDA(cudaMemcpy(&hd, c.hdr, sizeof hd, cudaMemcpyDeviceToHost));
  if (E) *E = hd.E;
  if (edge_dst) HMTL_CUDA(cudaMemcpy(edge_dst, c.edge_dst, size_t(hd.E) * 4, cudaMemcpyDeviceToHost));
  if (edge_src) HMTL_CUDA(cudaMemcpy(edge_src, c.edge_src, size_t(hd.E) * 4, cudaMemcpyDeviceToHost));
  if (edge_offset) HMTL_CUDA(cudaMemcpy(edge_offset, c.edge_offset, size_t(hd.G + 1) * 4, cudaMemcpyDeviceToHost));
  return 0;
}

int hmtl_forward(hmtl_ctx* h, void* stream) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  fresh_images(c, pick(c, stream));
  launch_forward(c, pick(c, stream));
  HMTL_CUDA(cudaGetLastError());
  return 0;
}

int hmtl_predictions(hmtl_ctx* h, float* energy, float* forces) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaDeviceSynchronize());
  if (int rc = check_hdr(c)) return rc;
  DevHdr hd;
  HMTL_CUDA(cudaMemcpy(&hd, c.hdr, sizeof hd, cudaMemcpyDeviceToHost));
  if (energy) HMTL_CUDA(cudaMemcpy(energy, c.energy, size_t(hd.G) * 4, cudaMemcpyDeviceToHost));
  if (forces) HMTL_CUDA(cudaMemcpy(forces, c.forces, size_t(hd.N) * 12, cudaMemcpyDeviceToHost));
  return 0;
}

int hmtl_loss(hmtl_ctx* h, float w_e, float w_f, void* stream) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  launch_loss(c, w_e, w_f, pick(c, stream));
  HMTL_CUDA(cudaGetLastError());
  return 0;
}

int hmtl_read_loss(hmtl_ctx* h, float* loss) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  if (c.comm) {  // the step's collectives may be in flight: wait with failure detection
    if (!c.step_done) HMTL_CUDA(cudaEventCreateWithFlags(&c.step_done, cudaEventDisableTiming));
    HMTL_CUDA(cudaEventRecord(c.step_done, c.stream));
    if (int rc = comm_wait_event(c, c.step_done)) return rc;
  }
  HMTL_CUDA(cudaDeviceSynchronize());
  if (int rc = check_hdr(c)) return rc;
  DevHdr hd;
  HMTL_CUDA(cudaMemcpy(&hd, c.hdr, sizeof hd, cudaMemcpyDeviceToHost));
  *loss = float(hd.loss);
  return 0;
}

namespace {
int hdr_errors(const DevHdr& h) {  // the reference's errors for the device error bits (as check_hdr)
  if (h.err & kErrUnowned) return fail(HMTL_ERR_CONTRACT, "model: unknown dataset id (head not owned by this rank)");
  if (h.err & kErrEmptyGraph) return fail(HMTL_ERR_CONTRACT, "build_batch: empty graph rejected");
  if (h.err & kErrEdgeOverflow) return fail(HMTL_ERR_CONTRACT, "build_batch: edge capacity exceeded");
  if (h.err & kErrNonFinite) return fail(HMTL_ERR_CONTRACT, "model: non-finite prediction");
  return 0;
}
}  // namespace

int hmtl_loss_post(hmtl_ctx* h, int slot, void* stream) {
  Ctx& c = h->c;
  if (slot < 0) return fail(HMTL_ERR_CONTRACT, "loss_post: negative slot");
  cudaSetDevice(c.device);
  cudaStream_t st = pick(c, stream);
  const int k = slot % Ctx::kLossRing;
  HMTL_CUDA(cudaEventSynchronize(c.hdr_ev[k]));  // the slot's previous read has landed
  HMTL_CUDA(cudaMemcpyAsync(c.h_hdr_ring + k, c.hdr, sizeof(DevHdr), cudaMemcpyDeviceToHost, st));
  HMTL_CUDA(cudaEventRecord(c.hdr_ev[k], st));
  return 0;
}

int hmtl_loss_wait(hmtl_ctx* h, int slot, float* loss) {
  Ctx& c = h->c;
  if (slot < 0 || !loss) return fail(HMTL_ERR_CONTRACT, "loss_wait: bad argument");
  cudaSetDevice(c.device);
  const int k = slot % Ctx::kLossRing;
  if (int rc = comm_wait_event(c, c.hdr_ev[k])) return rc;
  if (int rc = hdr_errors(c.h_hdr_ring[k])) return rc;
  *loss = float(c.h_hdr_ring[k].loss);
  return 0;
}

int hmtl_backward(hmtl_ctx* h, const float* dE, const float* dF, void* stream) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  cudaStream_t st = pick(c, stream);
  if ((dE == nullptr) != (dF == nullptr)) return fail(HMTL_ERR_CONTRACT, "model: upstream shape mismatch");
  fresh_images(c, st);
  if (dE) {
    HMTL_CUDA(cudaMemcpyAsync(c.dE, dE, size_t(c.host_G) * 4, cudaMemcpyHostToDevice, st));
    HMTL_CUDA(cudaMemcpyAsync(c.dF, dF, size_t(c.host_N) * 12, cudaMemcpyHostToDevice, st));
  }
  launch_backward(c, st);
  HMTL_CUDA(cudaGetLastError());
  if (dE) HMTL_CUDA(cudaStreamSynchronize(st));  // host upstreams must outlive the copy
  return 0;
}

int hmtl_adamw(hmtl_ctx* h, const hmtl_train_cfg* cfg, void* stream) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  launch_adamw(c, *cfg, pick(c, stream));
  HMTL_CUDA(cudaGetLastError());
  return 0;
}

int hmtl_train_step(hmtl_ctx* h, const hmtl_train_cfg* cfg, void* stream) {
  Ctx& c = h->c;
  if (comm_aborted(c)) return fail(HMTL_ERR_COMM, "train_step: communicators were aborted after an earlier failure");
  cudaSetDevice(c.device);
  cudaStream_t st = pick(c, stream);
  if (!cfg->use_graph) {
    if (int rc = enqueue_step(c, *cfg, st)) return rc;
    HMTL_CUDA(cudaGetLastError());
    return 0;
  }
  if (c.step_exec && (std::memcmp(&c.graph_cfg, cfg, sizeof *cfg) != 0 || c.graph_pbc != c.pbc ||
                      c.graph_sorted != c.head_sorted)) {
    cudaGraphExecDestroy(c.step_exec);
    c.step_exec = nullptr;
  }
  if (!c.bimg_ready && c.use_tc) {  // first step: eager, records the batched B-image jobs
    if (int rc = enqueue_step(c, *cfg, st)) return rc;
    HMTL_CUDA(cudaGetLastError());
    return 0;
  }
  if (c.prof_on) {  // profiled replay (outside any timed region)
    if (!c.prof_exec) {
      for (auto& r : c.prof) r.used = 0;
      cudaGraph_t g;
      // serialised copy of the step: every scope's time is its own kernels' time,
      // not stretched by concurrent side-stream kernels competing for SMs
      const bool ms = c.multi_stream;
      c.multi_stream = false;
      HMTL_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      int rc = enqueue_step(c, *cfg, st);
      cudaError_t e = cudaStreamEndCapture(st, &g);
      c.multi_stream = ms;
      if (rc) return rc;
      if (e != cudaSuccess) return fail(HMTL_ERR_INTERNAL, std::string("graph capture: ") + cudaGetErrorString(e));
      HMTL_CUDA(cudaGraphInstantiate(&c.prof_exec, g, 0));
      cudaGraphDestroy(g);
    }
    HMTL_CUDA(cudaGraphLaunch(c.prof_exec, st));
    HMTL_CUDA(cudaStreamSynchronize(st));
    prof_harvest(c);
    return 0;
  }
  if (!c.step_exec) {
    cudaGraph_t g;
    HMTL_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_step(c, *cfg, st);
    cudaError_t e = cudaStreamEndCapture(st, &g);
    if (rc) return rc;
    if (e != cudaSuccess) return fail(HMTL_ERR_INTERNAL, std::string("graph capture: ") + cudaGetErrorString(e));
    c.step_kernels = count_kernel_nodes(g);
    graph_l2_window(c, g);
    c.graph_pbc = c.pbc;
    c.graph_sorted = c.head_sorted;
    // per-node priorities (the capturing streams' / launch attributes'): without this flag a
    // graph runs every node at the priority of the stream it is launched into
    static const unsigned long long inst_flags = [] {
      const char* e = std::getenv("HMTL_NODE_PRIO");
      return (e && e[0] == '0') ? 0ull : (unsigned long long)cudaGraphInstantiateFlagUseNodePriority;
    }();
    HMTL_CUDA(cudaGraphInstantiate(&c.step_exec, g, inst_flags));
    cudaGraphDestroy(g);
    c.graph_cfg = *cfg;
  }
  HMTL_CUDA(cudaGraphLaunch(c.step_exec, st));
  return 0;
}

int hmtl_debug_fetch(hmtl_ctx* h, const char* name, int layer, float* host, size_t cap, size_t* n) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaDeviceSynchronize());
  DevHdr hd;
  HMTL_CUDA(cudaMemcpy(&hd, c.hdr, sizeof hd, cudaMemcpyDeviceToHost));
  const size_t H = c.H, W = c.W, N = hd.N, E = hd.E, G = hd.G;
  const size_t NH = size_t(c.Nc) * H, EH = size_t(c.Ec) * H;
  const std::string nm(name);
  const float* src = nullptr;
  size_t cnt = 0;
  auto lay_ok = [&](int lo, int hi) { return layer >= lo && layer <= hi; };
  if (nm == "h" && lay_ok(0, c.L)) src = c.hs + layer * NH, cnt = N * H;
  else if (nm == "P" && lay_ok(0, c.L - 1)) src = c.P + layer * 2 * NH, cnt = N * 2 * H;
  else if (nm == "z2" && lay_ok(0, c.L - 1)) src = c.z2 + layer * EH, cnt = E * H;
  else if (nm == "agg" && lay_ok(0, c.L - 1)) src = c.agg + layer * NH, cnt = N * H;
  else if (nm == "vz1" && lay_ok(0, c.L - 1)) src = c.vz1 + layer * NH, cnt = N * H;
  else if (nm == "pooled") src = c.pooled, cnt = G * H;
  else if (nm == "ez" && lay_ok(0, c.D - 1)) src = c.ez + layer * size_t(c.Gc) * W, cnt = G * W;
  else if (nm == "Qf") src = c.Qf, cnt = N * W;
  else if (nm == "zf" && lay_ok(1, c.D - 2)) src = c.zf + (layer - 1) * size_t(c.Ec) * W, cnt = E * W;
  else if (nm == "s") src = c.s, cnt = E;
  else if (nm == "grads") src = c.grads, cnt = c.PT;  // [shared | owned head slots] of the last backward
  else if (nm == "dE") src = c.dE, cnt = G;
  else if (nm == "dF") src = c.dF, cnt = 3 * N;
  else if (nm == "z1" && lay_ok(0, c.L - 1)) {
    launch_debug_z1(c, layer, c.scratch, c.stream);
    HMTL_CUDA(cudaStreamSynchronize(c.stream));
    src = c.scratch, cnt = E * H;
  } else {
    return fail(HMTL_ERR_CONTRACT, "debug_fetch: unknown tensor/layer " + nm);
  }
  if (n) *n = cnt;
  if (!host) return 0;
  if (cap < cnt) return fail(HMTL_ERR_CONTRACT, "debug_fetch: buffer too small");
  HMTL_CUDA(cudaMemcpy(host, src, cnt * 4, cudaMemcpyDeviceToHost));
  return 0;
}

int hmtl_debug_chain_stamps(hmtl_ctx* h, long long* out, int n) {
  Ctx& c = h->c;
  if (!c.chain_stamps) return fail(HMTL_ERR_CONTRACT, "chain stamps: set HMTL_CHAIN_STAMPS before ctx_create");
  HMTL_CUDA(cudaDeviceSynchronize());
  HMTL_CUDA(cudaMemcpy(out, c.chain_stamps, size_t(n) * sizeof(long long), cudaMemcpyDeviceToHost));
  return 0;
}

int hmtl_batch_shape(hmtl_ctx* h, int* G, int* N) {
  if (!h || !G || !N) return fail(HMTL_ERR_CONTRACT, "batch_shape: null argument");
  *G = h->c.host_G;
  *N = h->c.host_N;
  return 0;
}

int hmtl_step_kernel_count(hmtl_ctx* h, int* n) {
  if (!n) return fail(HMTL_ERR_CONTRACT, "step_kernel_count: null argument");
  *n = h->c.step_kernels;
  return 0;
}

int hmtl_set_stream_mode(hmtl_ctx* h, int multi) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaDeviceSynchronize());
  if (c.multi_stream != (multi != 0) && c.step_exec) {
    cudaGraphExecDestroy(c.step_exec);
    c.step_exec = nullptr;
  }
  c.multi_stream = multi != 0;
  return 0;
}

int hmtl_profile_enable(hmtl_ctx* h, int on) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaDeviceSynchronize());
  c.prof_on = on != 0;
  if (c.prof_exec) {
    cudaGraphExecDestroy(c.prof_exec);
    c.prof_exec = nullptr;
  }
  for (auto& r : c.prof) r.used = 0, r.acc_ms = 0.0, r.calls = 0;
  return 0;
}

int hmtl_profile_report(hmtl_ctx* h, char* json, size_t cap) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  HMTL_CUDA(cudaDeviceSynchronize());
  if (!c.prof_exec) prof_harvest(c);  // eager steps: events recorded once each
  std::string out = "[";
  for (auto& r : c.prof) {
    if (out.size() > 1) out += ",";
    out += "{\"name\":\"" + r.name + "\",\"calls\":" + std::to_string(r.calls) + ",\"ms\":" +
           std::to_string(r.acc_ms) + "}";
    if (!c.prof_exec) r.used = 0;
    r.acc_ms = 0.0;
    r.calls = 0;
  }
  out += "]";
  if (out.size() + 1 > cap) return fail(HMTL_ERR_CONTRACT, "profile_report: buffer too small");
  std::memcpy(json, out.c_str(), out.size() + 1);
  return 0;
}

}  // extern "C"
