// comm.cpp -- MTL-par gradient synchronisation over NCCL (NVLink 5 / NVSwitch).
//
// Replaces collective::allreduce_mean over RankGroup (hmtl/mesh.hpp:276-278,
// 322-334; tree schedule src/mesh.cpp:624-659) with:
//   * one world communicator  -> shared-block gradients, mean over all ranks
//     (global_group, hmtl/mesh.hpp:45-50; category encoder_sync);
//   * one communicator per head, ncclCommSplit(color = head if owned)
//     -> head-block gradients, mean over the ranks that own that head
//     (head_group, hmtl/mesh.hpp:52-58; category head_sync).
// Heads first, then the shared block, all on the step's
// stream so the sync is captured inside the step's CUDA graph.  NCCL's
// reduction order differs from the reference's binomial tree, so parity is
// within tolerance rather than bitwise.
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "ctx.cuh"

namespace hmtl_b200 {

struct Comm {
  ncclComm_t world = nullptr;
  int world_size = 1, rank = 0;
  std::vector<ncclComm_t> head;  // per head id (nullptr if not owned)
  std::vector<int> head_size;
  uint64_t bytes_encoder = 0, bytes_head = 0;
  bool aborted = false;
  std::vector<std::pair<ncclComm_t, void*>> reg;  // user-buffer registrations (HMTL_NCCL_REG=1)
};
void comm_abort(Comm* m);

#define HMTL_NCCL(call)                                                                        \
  do {                                                                                         \
    ncclResult_t r__ = (call);                                                                 \
    if (r__ != ncclSuccess)                                                                    \
      return fail(HMTL_ERR_COMM, std::string("NCCL: ") + #call + ": " + ncclGetErrorString(r__)); \
  } while (0)

int comm_sync_grads(Ctx& c, cudaStream_t st) {
  Comm* m = c.comm;
  if (!m) return 0;
  HMTL_NCCL(ncclGroupStart());
  for (int s = 0; s < c.S; ++s) {
    const int k = c.owned[s];
    if (m->head[k] && m->head_size[k] > 1) {
      HMTL_NCCL(ncclAllReduce(c.grads + c.PS + size_t(s) * c.PH, c.grads + c.PS + size_t(s) * c.PH, c.PH,
                              ncclFloat32, ncclAvg, m->head[k], st));
      m->bytes_head += c.PH * sizeof(float);
    }
  }
  if (m->world_size > 1) {
    HMTL_NCCL(ncclAllReduce(c.grads, c.grads, c.PS, ncclFloat32, ncclAvg, m->world, st));
    m->bytes_encoder += c.PS * sizeof(float);
  }
  HMTL_NCCL(ncclGroupEnd());
  return 0;
}

// ---- overlapped (bucketed) sync, issued from inside launch_backward on the
// comm stream as soon as each bucket's gradients are final: the owned heads'
// blocks (head groups) right after the heads' backward, then each encoder
// layer's contiguous shared block, top layer first, and finally the rest of the
// shared block (the embedding).  ncclAvg is elementwise, so bucketing gives
// the same group means as one allreduce of the whole block.
bool comm_overlap(const Ctx& c) { return c.comm && c.comm->world_size > 1 && c.overlap_comm; }

void comm_heads_async(Ctx& c, cudaStream_t sc) {
  Comm* m = c.comm;
  for (int s = 0; s < c.S; ++s) {
    const int k = c.owned[s];
    if (m->head[k] && m->head_size[k] > 1) {
      float* g = c.grads + c.PS + size_t(s) * c.PH;
      if (ncclAllReduce(g, g, c.PH, ncclFloat32, ncclAvg, m->head[k], sc) != ncclSuccess) c.comm_err = 1;
      m->bytes_head += c.PH * sizeof(float);
    }
  }
}

void comm_shared_async(Ctx& c, size_t off, size_t count, cudaStream_t sc) {
  Comm* m = c.comm;
  if (!count) return;
  if (ncclAllReduce(c.grads + off, c.grads + off, count, ncclFloat32, ncclAvg, m->world, sc) != ncclSuccess)
    c.comm_err = 1;
  m->bytes_encoder += count * sizeof(float);
}

void comm_destroy(Comm* m) {
  if (!m) return;
  if (m->aborted) {  // ncclCommAbort already released the communicators
    delete m;
    return;
  }
  for (auto& r : m->reg) ncclCommDeregister(r.first, r.second);
  for (auto& h : m->head)
    if (h) ncclCommDestroy(h);
  if (m->world) ncclCommDestroy(m->world);
  delete m;
}

// Failure detection for the collectives captured in the step graph (the reference
// bounds every blocking wait with a timeout and closes its endpoints on failure,
// src/mesh.cpp:142-146, 161-171): a host wait on a stream-ordered event polls
// ncclCommGetAsyncError of every communicator; an asynchronous NCCL error or a
// wait longer than HMTL_COMM_TIMEOUT_S (default 600 s) aborts all of this rank's
// communicators (ncclCommAbort: pending collectives return, peers see the
// failure) and reports ErrorCode::comm.  Without a communicator it is
// cudaEventSynchronize.
int comm_wait_event(Ctx& c, cudaEvent_t ev) {
  Comm* m = c.comm;
  if (!m || m->world_size <= 1) {
    HMTL_CUDA(cudaEventSynchronize(ev));
    return 0;
  }
  if (m->aborted) return fail(HMTL_ERR_COMM, "comm: communicators were aborted after an earlier failure");
  static const double timeout_s = [] {
    const char* e = std::getenv("HMTL_COMM_TIMEOUT_S");
    return e ? std::atof(e) : 600.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) return 0;
    if (q != cudaErrorNotReady)
      return fail(HMTL_ERR_INTERNAL, std::string("CUDA: step event: ") + cudaGetErrorString(q));
    std::string why;
    ncclResult_t st = ncclSuccess;
    if (ncclCommGetAsyncError(m->world, &st) != ncclSuccess || (st != ncclSuccess && st != ncclInProgress))
      why = std::string("world communicator: ") + ncclGetErrorString(st);
    for (size_t k = 0; why.empty() && k < m->head.size(); ++k)
      if (m->head[k] && (ncclCommGetAsyncError(m->head[k], &st) != ncclSuccess || (st != ncclSuccess && st != ncclInProgress)))
        why = "head " + std::to_string(k) + " communicator: " + ncclGetErrorString(st);
    if (why.empty() && std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
      why = "collective did not complete within HMTL_COMM_TIMEOUT_S=" + std::to_string(timeout_s) + " s";
    if (!why.empty()) {
      comm_abort(m);
      return fail(HMTL_ERR_COMM, "comm: " + why + " (communicators aborted)");
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

void comm_abort(Comm* m) {
  if (!m || m->aborted) return;
  for (auto& h : m->head)
    if (h) ncclCommAbort(h), h = nullptr;
  if (m->world) ncclCommAbort(m->world), m->world = nullptr;
  m->aborted = true;
}

bool comm_aborted(const Ctx& c) { return c.comm && c.comm->aborted; }

ncclComm_t comm_world(Ctx& c, int* rank, int* size) {
  if (!c.comm) return nullptr;
  *rank = c.comm->rank;
  *size = c.comm->world_size;
  return c.comm->world;
}

}  // namespace hmtl_b200

using namespace hmtl_b200;

extern "C" {

int hmtl_comm_unique_id(uint8_t out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  HMTL_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, &id, 128);
  return 0;
}

int hmtl_comm_init(hmtl_ctx* h, const uint8_t id_bytes[128], int world, int rank) {
  Ctx& c = h->c;
  if (world < 1 || rank < 0 || rank >= world) return fail(HMTL_ERR_CONTRACT, "comm_init: bad rank/world");
  cudaSetDevice(c.device);
  auto* m = new Comm;
  m->world_size = world;
  m->rank = rank;
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, 128);
  ncclResult_t r = ncclCommInitRank(&m->world, world, id, rank);
  if (r != ncclSuccess) {
    delete m;
    return fail(HMTL_ERR_COMM, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  const int n_heads = c.hp.n_heads;
  m->head.assign(n_heads, nullptr);
  m->head_size.assign(n_heads, 0);
  for (int k = 0; k < n_heads; ++k) {
    const int color = c.slot_of[k] >= 0 ? k : NCCL_SPLIT_NOCOLOR;
    r = ncclCommSplit(m->world, color, rank, &m->head[k], nullptr);
    if (r != ncclSuccess) {
      delete m;
      return fail(HMTL_ERR_COMM, std::string("ncclCommSplit: ") + ncclGetErrorString(r));
    }
    if (m->head[k]) ncclCommCount(m->head[k], &m->head_size[k]);
  }
  if (const char* e = std::getenv("HMTL_NCCL_REG"); e && e[0] == '1') {
    // the gradient buffer registered with every communicator that reduces it
    // (zero-copy NVLink transfers / NVLS when the platform offers them)
    int ok = 0, tried = 0;
    auto reg = [&](ncclComm_t cm, void* p, size_t bytes) {
      void* hd = nullptr;
      ++tried;
      if (ncclCommRegister(cm, p, bytes, &hd) == ncclSuccess && hd) m->reg.emplace_back(cm, hd), ++ok;
    };
    reg(m->world, c.grads, c.PS * sizeof(float));
    for (int s = 0; s < c.S; ++s)
      if (m->head[c.owned[s]]) reg(m->head[c.owned[s]], c.grads + c.PS + size_t(s) * c.PH, c.PH * sizeof(float));
    std::fprintf(stderr, "[hmtl comm] rank %d: registered %d of %d gradient buffers with NCCL\n", rank, ok, tried);
  }
  if (const char* e = std::getenv("HMTL_COMM_LOG"); e && e[0] == '1') {
    std::string g;
    for (int k = 0; k < n_heads; ++k) g += (k ? "," : "") + std::to_string(m->head_size[k]);
    std::fprintf(stderr, "[hmtl comm] rank %d/%d device %d: world comm %d ranks; head-group sizes [%s] (0 = not owned)\n",
                 rank, world, c.device, world, g.c_str());
  }
  if (c.step_exec) {
    cudaGraphExecDestroy(c.step_exec);
    c.step_exec = nullptr;
  }
  if (c.prof_exec) {
    cudaGraphExecDestroy(c.prof_exec);
    c.prof_exec = nullptr;
  }
  c.comm = m;
  return 0;
}

int hmtl_comm_sync_grads(hmtl_ctx* h, void* stream) {
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  return comm_sync_grads(c, stream ? static_cast<cudaStream_t>(stream) : c.stream);
}

int hmtl_comm_info(hmtl_ctx* h, int* world, int* rank, int* head_sizes, int n) {
  Comm* m = h ? h->c.comm : nullptr;
  if (!m) return fail(HMTL_ERR_CONTRACT, "comm_info: no communicator attached");
  if (world) ncclCommCount(m->world, world);
  if (rank) ncclCommUserRank(m->world, rank);
  for (int k = 0; head_sizes && k < n && k < int(m->head_size.size()); ++k) head_sizes[k] = m->head_size[k];
  return 0;
}

int hmtl_comm_bytes(hmtl_ctx* h, uint64_t out[2]) {
  Comm* m = h->c.comm;
  out[0] = m ? m->bytes_encoder : 0;
  out[1] = m ? m->bytes_head : 0;
  return 0;
}

}  // extern "C"
