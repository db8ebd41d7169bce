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

#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"

namespace hmtl_b200 {

struct Comm {
  ncclComm_t world = nullptr;
  int world_size = 1, rank = 0;
  std::vector<ncclComm_t> head;  // per head id (nullptr if not owned)
  std::vector<int> head_size;
  uint64_t bytes_encoder = 0, bytes_head = 0;
};

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
  for (auto& h : m->head)
    if (h) ncclCommDestroy(h);
  if (m->world) ncclCommDestroy(m->world);
  delete m;
}

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

int hmtl_comm_bytes(hmtl_ctx* h, uint64_t out[2]) {
  Comm* m = h->c.comm;
  out[0] = m ? m->bytes_encoder : 0;
  out[1] = m ? m->bytes_head : 0;
  return 0;
}

}  // extern "C"
