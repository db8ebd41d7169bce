// ctx.cuh -- the per-GPU device context behind hmtl_ctx (one host thread per GPU).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace hmtl_b200 {

struct Comm;  // comm.cu (NCCL)

// Descriptor of a GEMM B operand B(k, n) read from a weight tensor:
// base[seg*seg_stride + k*sk + n*sn], optionally split in two sources along n
// (split 1) or k (split 2) at `at` (the second source sees n-at / k-at).
struct BDesc {
  const float* base0;
  const float* base1;
  int split, at;
  long long sk, sn;
  int K, N, nseg;
  long long seg_stride;
  float* out;  // image destination (filled in when batched)
  int halves = 0;  // 2: CTA-pair chain layout (per column half, per 32-k chunk, [hi | lo] contiguous)
};

// Optional per-launch CUDA-event timing (hmtl_profile); off in timed steps.
struct ProfRec {
  std::string name;
  std::vector<cudaEvent_t> ev;  // pairs (start, end)
  size_t used = 0;
  double acc_ms = 0.0;  // harvested elapsed time
  long calls = 0;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  hmtl_hyper hp{};
  int H = 0, W = 0, L = 0, D = 0, S = 0, NS = 0;
  std::vector<int> owned;  // head id per slot (ascending)
  int slot_of[256];
  Layout shared_lay, head_lay;
  size_t PS = 0, PH = 0, PT = 0;  // shared, head, total owned parameter counts
  int Gc = 0, Nc = 0;
  long long Ec = 0;
  double rc2 = 0.0;  // cutoff^2 in FP64, as build_batch (hmtl/graph.hpp:53)

  // parameters / optimiser state: [shared | slot0 head | slot1 head | ...]
  float *params = nullptr, *grads = nullptr, *adam_m = nullptr, *adam_v = nullptr;
  DevHdr* hdr = nullptr;
  int* d_slot_of = nullptr;

  // batch arena (device) + pinned staging + device pool
  uint8_t* arena = nullptr;
  size_t arena_cap = 0;
  uint8_t* h_arena = nullptr;
  size_t h_arena_cap = 0;
  // second pinned staging arena: batch_upload alternates and waits only for the
  // copy that last read the buffer (two uploads back), not for the stream
  uint8_t* h_arena2 = nullptr;
  cudaEvent_t h_arena_ev[2] = {nullptr, nullptr};
  int h_arena_k = 0;
  // pinned ring of device headers for pipelined loss reads (hmtl_loss_post/wait)
  static constexpr int kLossRing = 8;
  DevHdr* h_hdr_ring = nullptr;
  cudaEvent_t hdr_ev[kLossRing] = {};
  std::vector<uint8_t*> pool;
  std::vector<size_t> pool_bytes;
  int host_G = 0, host_N = 0;  // last bound batch (host view)

  // derived batch structure
  int *graph_offset = nullptr, *node_graph = nullptr, *deg = nullptr, *row_ptr = nullptr;
  int *edge_src = nullptr, *edge_dst = nullptr, *rev = nullptr, *edge_offset = nullptr;
  float4 *pos32 = nullptr, *geo = nullptr;  // geo = (dx, dy, dz, d2) per edge, FP32
  float* dist = nullptr;
  uint8_t* species = nullptr;
  // periodic cells: lattice [G][3][3] of the bound batch, per-edge
  // image key, cell-list scratch; `pbc` selects the periodic neighbour list
  double* cells = nullptr;
  double* h_cells = nullptr;  // pinned staging
  int *eimg = nullptr, *pbc_meta = nullptr, *pbc_bins = nullptr, *pbc_order = nullptr, *pbc_acoord = nullptr,
      *pbc_w2 = nullptr;
  bool pbc = false, graph_pbc = false;
  // graphs of the bound batch grouped by owned head in ascending slot order (as a rank's
  // batch of its heads' sources is): the head-sorted node/edge/graph orders are then the
  // identity, so head-segmented row sets need no permutation (and can use TMA operands)
  bool head_sorted = false, graph_sorted = false;
  std::vector<char> pool_sorted;
  int *gslot = nullptr, *gperm = nullptr, *gnode_base = nullptr, *gedge_base = nullptr;
  int *node_perm = nullptr, *edge_perm = nullptr;

  // forward cache (device)
  float *hs = nullptr, *P = nullptr, *z2 = nullptr, *agg = nullptr, *vz1 = nullptr;
  // node tables (hs, P, agg, vz1, dagg, dhb, dvz1b) in one allocation: the L2 persisting window
  float* node_arena = nullptr;
  size_t node_arena_bytes = 0;
  int l2_persist_mb = 0;  // persisting L2 set-aside for the node tables (HMTL_L2_PERSIST_MB; 0 = off)
  float *pooled = nullptr, *ez = nullptr, *energy = nullptr, *Qf = nullptr, *zf = nullptr;
  float *s = nullptr, *forces = nullptr;
  // backward workspace
  float *dE = nullptr, *dF = nullptr, *dagg = nullptr;
  float *ds = nullptr, *dpooled = nullptr;
  double* loss_terms = nullptr;  // [G] per-graph loss terms
  float *edA = nullptr, *edB = nullptr, *scratch = nullptr;
  float* partial = nullptr;    // split-K partials of kernels on the main stream
  float* partial_w = nullptr;   // ... and of the weight-gradient streams
  float* partial_w3 = nullptr;
  float* partial_w2 = nullptr;
  size_t partial_cap = 0;
  // backward buffers that weight-gradient kernels read: one per layer, so the
  // main stream never overwrites what the side stream has yet to read
  float *dhb = nullptr;    // [L+1][N][H]: dL/dh_l
  float *dvz1b = nullptr;  // [L][N][H]
  float *dzAb = nullptr, *dzBb = nullptr;  // [L][E][H]
  float *Sb = nullptr;     // [L+1][N][2max(H,W)] (slot L: force head)
  float *fzA = nullptr, *fzB = nullptr;    // force head dz ping-pong [E][W]
  // concurrency inside the step: s_e runs the energy head branch, s_w the
  // weight gradients; both fork from / join into the step stream via events
  cudaStream_t s_e = nullptr, s_w = nullptr, s_w2 = nullptr, s_w3 = nullptr;
  cudaStream_t s_c = nullptr;  // gradient allreduces (high priority), overlapped with the backward
  bool overlap_comm = true;
  int comm_err = 0;
  cudaEvent_t step_done = nullptr;  // host waits on the step (read_loss) go through comm_wait_event
  std::vector<cudaEvent_t> evs;
  size_t ev_i = 0;
  bool multi_stream = true;
  bool fuse_chain = true;  // node-row GEMM chains in one launch (chain.cuh)
  bool ptab_on = true;     // layer 0's P from a per-species table (HMTL_PTAB=0: the node-row GEMM)
  bool ptab_ready = false;  // (this step's table was launched)
  float* ptab = nullptr;    // [NS][2H]
  int* d_ns = nullptr;      // device copy of NS (row count of the table GEMM)
  int wgrad3 = 0;          // edge eW2 weight gradient on a third side stream: 0 never, 1 layer 0 (the step's
                           // tail), 2 every layer (HMTL_WGRAD3)
  bool row_pair = false;    // row GEMMs over one segment as CTA pairs (cta_group::2; HMTL_ROW_PAIR=1)
  int row_prefetch = 0;    // row GEMMs prefetch the next tile's forward-written rows into L2 (HMTL_ROW_PREFETCH=1; measured slower)
  int chain_prefetch = 0;  // chains prefetch their operands into L2 at launch (HMTL_CHAIN_PREFETCH=1; measured neutral)
  bool chain_pair = false;  // ... as CTA-pair (cta_group::2) kernels (HMTL_CHAIN_PAIR=1; measured slower)
  int rec_halves = 0;      // B-image layout tag of the jobs being recorded (the pair chain's GEMMs)
  // fused edge passes (gather producer + segmented epilogue, tc.cuh kSeg): correct but slower on this
  // engine (96-register cap of the 17-warp CTA -> producer spills), opt-in HMTL_FUSE_EDGE=1
  bool fuse_edge = false;
  // cp.async two-operand gather producers (tc.cuh kAsync) replacing the separate elementwise
  // passes: forward message GEMM (HMTL_ASYNC_FWD=1), backward dz1 GEMM (HMTL_ASYNC_BWD: 0 off,
  // 1 silu'(z1) stored by the forward's edge pass, 2 regathered from P in the epilogue)
  bool async_fwd = false;
  // force output layer's dz formed in the dx GEMM producer (HMTL_FUSE_FORCE_OUT=1; measured
  // slower: its side-stream column sums contend with the critical path for SMs)
  bool fuse_force_out = false;
  bool launch_prio = false;  // per-launch priority attribute, critical path high (HMTL_LAUNCH_PRIO=1; no gain)
  int async_bwd = 1;
  float* s1pb = nullptr;  // [L][E][H] silu'(z1) stored by the forward for the backward
  // the forward's edge pass stores z1 alone (in the a1 buffer); the message GEMM producer, the
  // eW2 weight gradient and the dz1 epilogue apply silu / silu' to it (HMTL_Z1_ONLY=0: a1 + silu'(z1))
  bool z1_only = false;  // (measured slower: silu' in the dz1 epilogue, silu in the eW2 gradient converter)
  int tc_grid_mult = 1;
  bool prefetch_l2 = true;  // L2 prefetch of re-read activations ahead of the critical path    // row GEMM grid cap in SMs (0: one CTA per tile)
  long long* chain_stamps = nullptr;
  int chain_dbg = 0;
  bool dbg_skip_wgrad = false;  // timing experiments: skip weight gradients (wrong training)  // engine tuning: phase timestamps of the last chain launch
  float* bimg = nullptr;  // tcgen05 B-operand images (hi/lo, K-major)
  size_t bimg_cap = 0;
  bool use_tc = true;     // tcgen05 path for GEMMs whose shapes allow it
  // batched B-image builds: recorded in call order during the first step, rebuilt
  // in one launch after every AdamW (weights only change there) and on set_block
  std::vector<BDesc> bjobs;
  bool bimg_ready = false;
  bool bimg_recording = false;  // set by a train step before the images exist
  bool bimg_stale = false;      // params updated by a train step's AdamW, images not yet rebuilt
  int bimg_idx = 0;
  float* bimg_all = nullptr;
  size_t bimg_all_cap = 0;
  BDesc* d_bjobs = nullptr;
  int n_djobs = 0;
  int bimg_rows = 1;  // max (segments x K) over the recorded images: bimg_all grid.x
  int bimg_blocks = 32;  // CTAs per image of the batched rebuild (HMTL_BIMG_BLOCKS; 16-128 measured equal)
  bool store_a1 = false;  // forward producer materialises a1 = silu(z1) [L][E][H]
  bool store_af0 = false; // ... and silu(zf0) [E][W]
  // silu'(zf0) [E][W] too only when the force output layer's backward needs it
  // (head_depth 2); deeper heads regather it from the L2-resident Qf table
  bool store_sf0 = false;
  int red_sms = 0;          // SMs a weight-gradient (tc_red) launch spreads over (HMTL_RED_SMS; default 13/16 of them)
  int row_sms = 148;        // persistent row-GEMM grid (HMTL_ROW_SMS; default every SM)
  int red_cluster = 1;      // split-K CTAs per cluster reducing partials through DSMEM (HMTL_RED_CLUSTER 1/2/4/8; opt-in, slower)
  int red_sms_early = 0;    // ... for the weight gradients of the heads and layers >= 1 (HMTL_RED_SMS_EARLY)
  int red_sms_now = 0;      // (the value atb() uses while the backward is enqueued)
  int red_seg_mult = 1;     // CTA multiplier for head-segmented weight gradients (HMTL_RED_SEGX)
  int red_min_chunks = 4;   // >= this many 32-row chunks per weight-gradient CTA (HMTL_RED_MINCH)
  int red_min_tail = 4;     // ... for layer 0's weight gradients, the step's tail (HMTL_RED_MINCH_TAIL)
  int red_min_now = 4;      // (the value atb() uses while the backward is enqueued)
  bool red_tma = true;      // TMA operand path for plain row-major weight gradients (HMTL_NO_RED_TMA=1 off)
  int chain_mr_fwd = 64;    // ... for the forward chains (HMTL_CHAIN_M_FWD; 0 = chain_mr)
  int chain_mr = 128;       // node rows per chain CTA: 128 or 64 (HMTL_CHAIN_M; 64 only with the 2-CTA split)
  int chain_cs = 2;         // node-chain cluster size: 2 = column split over a CTA pair (HMTL_CHAIN_CS=1: one CTA)
  float *a1 = nullptr, *af0 = nullptr, *sf0 = nullptr;
  float* tpart = nullptr;  // [2][tcap][H] per-128-edge-tile pieces of straddling destinations (fused edge passes)
  int tcap = 0;
  int nsplit_node = 1, nsplit_edge = 1, nsplit_graph = 1;

  // CUDA graph of a whole training step
  cudaGraphExec_t step_exec = nullptr;
  hmtl_train_cfg graph_cfg{};
  int step_kernels = -1;  // kernel nodes in step_exec (launches per step)

  Comm* comm = nullptr;
  int sm_count = 148;
  bool prof_on = false;
  std::vector<ProfRec> prof;
  // profiled copy of the step graph: every Prof scope is a pair of external
  // event-record nodes, so per-scope times are taken inside a real graph replay
  cudaGraphExec_t prof_exec = nullptr;

  // helpers
  float* shared_param(const char* name) const { return params + shared_lay.at(name).offset; }
  float* shared_grad(const char* name) const { return grads + shared_lay.at(name).offset; }
  size_t shared_off(const std::string& name) const { return shared_lay.at(name).offset; }
  size_t head_off(const std::string& name) const { return head_lay.at(name).offset; }
  float* head_params() const { return params + PS; }
  float* head_grads() const { return grads + PS; }
  float* part(cudaStream_t st) const {
    return st == s_w ? partial_w : (st == s_w2 ? partial_w2 : (st == s_w3 ? partial_w3 : partial));
  }
  // stream for a side branch (the step stream itself while B images are being
  // recorded: that eager step shares one image scratch buffer)
  cudaStream_t side(cudaStream_t which, cudaStream_t st) const {
    return (multi_stream && bimg_ready && which) ? which : st;
  }
  // make `to` wait for everything enqueued so far on `from`
  void dep(cudaStream_t from, cudaStream_t to) {
    if (from == to) return;
    if (ev_i == evs.size()) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      evs.push_back(e);
    }
    cudaEvent_t e = evs[ev_i++];
    cudaEventRecord(e, from);
    cudaStreamWaitEvent(to, e, 0);
  }
};

// launchers (stream-ordered; sizes come from the device header)
bool sorted_by_slot(const Ctx& c, const uint8_t* ds, int G);  // graphs grouped by ascending owned slot
void launch_prep(Ctx& c, cudaStream_t st);      // arena -> node/graph tables, routing
void launch_nbr(Ctx& c, cudaStream_t st);       // neighbour list, CSR, rev, edge offsets
void launch_nbr_pbc(Ctx& c, cudaStream_t st);   // ... with periodic images (cell list)
void launch_route(Ctx& c, cudaStream_t st, bool routed);  // head routing (unless `routed`) + head-sorted permutations
void launch_forward(Ctx& c, cudaStream_t st);   // ModelT::forward
void launch_loss(Ctx& c, float w_e, float w_f, cudaStream_t st);
void launch_backward(Ctx& c, cudaStream_t st, bool comm_sync = false);  // ModelT::backward (upstreams in c.dE/c.dF)
void launch_adamw(Ctx& c, const hmtl_train_cfg& cfg, cudaStream_t st, bool defer_images = false);
void launch_debug_z1(Ctx& c, int layer, float* out, cudaStream_t st);
void launch_bimg_all(Ctx& c, cudaStream_t st);  // rebuild every recorded B image
void launch_ptab(Ctx& c, cudaStream_t st);      // layer 0's per-species P table (after launch_bimg_all)
void set_tc_debug(int bits);                     // HMTL_TC_DEBUG: engine ablation bits (timing only)

int comm_sync_grads(Ctx& c, cudaStream_t st);
int comm_wait_event(Ctx& c, cudaEvent_t ev);  // host wait with NCCL failure detection (comm.cu)
bool comm_aborted(const Ctx& c);               // the communicators were aborted after a failure
bool comm_overlap(const Ctx& c);                                    // bucketed sync inside the backward
void comm_heads_async(Ctx& c, cudaStream_t sc);                     // owned heads, head groups
void comm_shared_async(Ctx& c, size_t off, size_t count, cudaStream_t sc);  // shared range, world

// RAII timing scope: records start/end events on `st` when profiling is on.
struct Prof {
  Ctx& c;
  cudaStream_t st;
  cudaEvent_t end = nullptr;
  Prof(Ctx& c_, const char* name, cudaStream_t s) : c(c_), st(s) {
    if (!c.prof_on) return;
    ProfRec* r = nullptr;
    for (auto& x : c.prof)
      if (x.name == name) r = &x;
    if (!r) {
      c.prof.push_back(ProfRec{name, {}, 0});
      r = &c.prof.back();
    }
    if (r->used + 2 > r->ev.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      r->ev.push_back(a);
      r->ev.push_back(b);
    }
    rec(r->ev[r->used]);
    end = r->ev[r->used + 1];
    r->used += 2;
  }
  void rec(cudaEvent_t e) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else cudaEventRecord(e, st);
  }
  ~Prof() {
    if (end) rec(end);
  }
};
void comm_destroy(Comm* m);

#define HMTL_CUDA(call)                                                                 \
  do {                                                                                  \
    cudaError_t e__ = (call);                                                           \
    if (e__ != cudaSuccess)                                                             \
      return ::hmtl_b200::fail(HMTL_ERR_INTERNAL, std::string("CUDA: ") + #call + ": " + \
                                                      cudaGetErrorString(e__));         \
  } while (0)

}  // namespace hmtl_b200

struct hmtl_ctx {
  hmtl_b200::Ctx c;
};
