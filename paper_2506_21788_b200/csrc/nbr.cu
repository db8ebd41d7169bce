// nbr.cu -- batch preparation and the neighbour list (build_batch on the GPU).
//
// build_batch<S> (/root/reference/proj/include/hmtl/graph.hpp:46-83) does an
// O(n^2) FP64 pair test per graph, emitting edges dst-major (i outer, j inner)
// with `(dx*dx + dy*dy) + dz*dz <= rc*rc` evaluated in double WITHOUT FMA
// (reference built without -march).  Here: one warp per destination node,
// lanes test 32 sources at a time with __dmul_rn/__dadd_rn (no contraction),
// a warp ballot + popcount gives each hit its rank, so the CSR rows come out
// in ascending-src order directly -- no sort, bit-exact edge set.  Graphs are
// small (<= a few hundred atoms) so the per-graph all-pairs tile is the
// cheapest exact search; rows of different graphs never interact.
#include "ctx.cuh"

namespace hmtl_b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;

// arena -> node tables.  One thread per node (and per graph).
__global__ void prep_kernel(const uint8_t* __restrict__ arena, DevHdr* hdr, const int* __restrict__ slot_of,
                            int* graph_offset, int* node_graph, uint8_t* species, float4* pos32, int* gslot,
                            int Gc, int Nc) {
  pdl_wait();
  const int G = reinterpret_cast<const int*>(arena)[0];
  const int N = reinterpret_cast<const int*>(arena)[1];
  const ArenaLayout al = arena_layout(G, N);
  const int* go = reinterpret_cast<const int*>(arena + al.go);
  const uint8_t* ds = arena + al.ds;
  const uint8_t* sp = arena + al.sp;
  const double* pos = reinterpret_cast<const double*>(arena + al.pos);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0) {
    hdr->G = G;
    hdr->N = N;
  }
  if (tid <= G) graph_offset[tid] = go[tid];
  if (tid < G) {
    const int s = slot_of[ds[tid]];
    gslot[tid] = s;
    if (s < 0) atomicOr(&hdr->err, kErrUnowned);
    if (go[tid + 1] - go[tid] <= 0) atomicOr(&hdr->err, kErrEmptyGraph);
  }
  if (tid < N) {
    // graph of node tid: last g with go[g] <= tid
    int lo = 0, hi = G - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (go[mid] <= tid) lo = mid;
      else hi = mid - 1;
    }
    node_graph[tid] = lo;
    species[tid] = sp[tid];
    // positions cast to S (hmtl/graph.hpp:61-62)
    pos32[tid] = make_float4(float(pos[3 * tid]), float(pos[3 * tid + 1]), float(pos[3 * tid + 2]), 0.f);
  }
}

__device__ __forceinline__ bool within(const double* __restrict__ pos, int i, int j, double rc2) {
  const double dx = __dsub_rn(pos[3 * i], pos[3 * j]);
  const double dy = __dsub_rn(pos[3 * i + 1], pos[3 * j + 1]);
  const double dz = __dsub_rn(pos[3 * i + 2], pos[3 * j + 2]);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return d2 <= rc2;
}

// pass 1: degree of every destination node (warp per node)
__global__ void nbr_count_kernel(const uint8_t* __restrict__ arena, const DevHdr* hdr,
                                 const int* __restrict__ graph_offset, const int* __restrict__ node_graph,
                                 int* __restrict__ deg, double rc2) {
  pdl_wait();
  const int N = hdr->N, G = hdr->G;
  const double* pos = reinterpret_cast<const double*>(arena + arena_layout(G, N).pos);
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += (gridDim.x * blockDim.x) >> 5) {
    const int g = node_graph[i];
    const int lo = graph_offset[g], hi = graph_offset[g + 1];
    int cnt = 0;
    for (int j0 = lo; j0 < hi; j0 += 32) {
      const int j = j0 + lane;
      const bool hit = j < hi && j != i && within(pos, i, j, rc2);
      cnt += __popc(__ballot_sync(kFull, hit));
    }
    if (lane == 0) deg[i] = cnt;
  }
}

// exclusive scan of deg -> row_ptr (single CTA, 1024 threads), edge offsets, E
__global__ void __launch_bounds__(1024) scan_kernel(DevHdr* hdr, const int* __restrict__ deg, int* row_ptr,
                                                    const int* __restrict__ graph_offset, int* edge_offset,
                                                    long long Ec) {
  pdl_wait();
  __shared__ int warp_sums[32];
  __shared__ int carry;
  const int N = hdr->N, G = hdr->G;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < N; base += 1024) {
    const int i = base + tid;
    const int v = i < N ? deg[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const int incl = x + (wid ? warp_sums[wid - 1] : 0) + carry;
    if (i < N) row_ptr[i] = incl - v;
    __syncthreads();
    if (tid == 1023) carry = incl;
    __syncthreads();
  }
  if (tid == 0) {
    row_ptr[N] = carry;
    hdr->E = carry;
    if (carry > Ec) atomicOr(&hdr->err, kErrEdgeOverflow);
  }
  __syncthreads();
  for (int g = tid; g <= G; g += 1024) edge_offset[g] = row_ptr[graph_offset[g]];
}

// pass 2: write edges (warp per node), ascending src within each dst row,
// plus the FP32 geometry of ModelT<float>::forward (hmtl/model.hpp:357-366).
__global__ void nbr_write_kernel(const uint8_t* __restrict__ arena, const DevHdr* hdr,
                                 const int* __restrict__ graph_offset, const int* __restrict__ node_graph,
                                 const int* __restrict__ row_ptr, const float4* __restrict__ pos32,
                                 int* __restrict__ edge_src, int* __restrict__ edge_dst, float4* __restrict__ geo,
                                 float* __restrict__ dist, double rc2, long long Ec) {
  pdl_wait();
  const int N = hdr->N, G = hdr->G;
  if (hdr->E > Ec) return;
  const double* pos = reinterpret_cast<const double*>(arena + arena_layout(G, N).pos);
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += (gridDim.x * blockDim.x) >> 5) {
    const int g = node_graph[i];
    const int lo = graph_offset[g], hi = graph_offset[g + 1];
    int at = row_ptr[i];
    const float4 pi = pos32[i];
    for (int j0 = lo; j0 < hi; j0 += 32) {
      const int j = j0 + lane;
      const bool hit = j < hi && j != i && within(pos, i, j, rc2);
      const unsigned m = __ballot_sync(kFull, hit);
      if (hit) {
        const int e = at + __popc(m & ((1u << lane) - 1));
        edge_src[e] = j;
        edge_dst[e] = i;
        const float4 pj = pos32[j];
        const float dx = __fsub_rn(pi.x, pj.x), dy = __fsub_rn(pi.y, pj.y), dz = __fsub_rn(pi.z, pj.z);
        const float d2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
        geo[e] = make_float4(dx, dy, dz, d2);
        dist[e] = __fsqrt_rn(d2);
      }
      at += __popc(m);
    }
  }
}

// reverse-edge permutation: rev[(i,j)] = index of (j,i).  The FP64 test is
// symmetric bit-for-bit ((a-b)^2 == (b-a)^2), so (j,i) always exists.
__global__ void rev_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr, const int* __restrict__ edge_src,
                           const int* __restrict__ edge_dst, int* __restrict__ rev, long long Ec) {
  pdl_wait();
  const int E = hdr->E;
  if (E > Ec) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int i = edge_dst[e], j = edge_src[e];
    int lo = row_ptr[j], hi = row_ptr[j + 1];
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (edge_src[mid] < i) lo = mid + 1;
      else hi = mid;
    }
    rev[e] = lo;
  }
}

// Head routing (hmtl/model.hpp:430-433: graphs grouped per head, heads
// ascending, graphs ascending).  One CTA: for each slot, a stable scan over
// graphs gives every graph its position in the head-sorted graph/node/edge
// orders.
__global__ void __launch_bounds__(1024) route_kernel(DevHdr* hdr, const int* __restrict__ gslot,
                                                     const int* __restrict__ graph_offset,
                                                     const int* __restrict__ edge_offset, int* gperm,
                                                     int* gnode_base, int* gedge_base, int S) {
  pdl_wait();
  __shared__ int wsum[3][32];
  __shared__ int carry[3];
  const int G = hdr->G;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    carry[0] = carry[1] = carry[2] = 0;
    hdr->n_slots = S;
    hdr->seg_graph[0] = hdr->seg_node[0] = hdr->seg_edge[0] = 0;
  }
  __syncthreads();
  for (int s = 0; s < S; ++s) {
    for (int base = 0; base < G; base += 1024) {
      const int g = base + tid;
      const bool f = g < G && gslot[g] == s;
      int v[3] = {f ? 1 : 0, f ? graph_offset[g + 1] - graph_offset[g] : 0,
                  f ? edge_offset[g + 1] - edge_offset[g] : 0};
      int x[3] = {v[0], v[1], v[2]};
#pragma unroll
      for (int q = 0; q < 3; ++q) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, x[q], o);
          if (lane >= o) x[q] += y;
        }
        if (lane == 31) wsum[q][wid] = x[q];
      }
      __syncthreads();
      if (wid < 3) {
        int w = wsum[wid][lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(kFull, w, o);
          if (lane >= o) w += y;
        }
        wsum[wid][lane] = w;
      }
      __syncthreads();
      int excl[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) excl[q] = x[q] - v[q] + (wid ? wsum[q][wid - 1] : 0) + carry[q];
      if (f) {
        gperm[excl[0]] = g;
        gnode_base[g] = excl[1];
        gedge_base[g] = excl[2];
      }
      __syncthreads();
      if (tid == 1023) {
#pragma unroll
        for (int q = 0; q < 3; ++q) carry[q] = excl[q] + v[q];
      }
      __syncthreads();
    }
    if (tid == 0) {
      hdr->seg_graph[s + 1] = carry[0];
      hdr->seg_node[s + 1] = carry[1];
      hdr->seg_edge[s + 1] = carry[2];
    }
    __syncthreads();
  }
}

__global__ void perm_kernel(const DevHdr* hdr, const int* __restrict__ node_graph, const int* __restrict__ graph_offset,
                            const int* __restrict__ edge_offset, const int* __restrict__ edge_dst,
                            const int* __restrict__ gnode_base, const int* __restrict__ gedge_base, int* node_perm,
                            int* edge_perm) {
  pdl_wait();
  const int N = hdr->N, E = hdr->E;
  const int M = N > E ? N : E;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < M; t += gridDim.x * blockDim.x) {
    if (t < N) {
      const int g = node_graph[t];
      node_perm[gnode_base[g] + t - graph_offset[g]] = t;
    }
    if (t < E) {
      const int g = node_graph[edge_dst[t]];
      edge_perm[gedge_base[g] + t - edge_offset[g]] = t;
    }
  }
}

int grid_for(long long n, int threads, int cap) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return int(b < cap ? b : cap);
}

}  // namespace

void launch_prep(Ctx& c, cudaStream_t st) {
  cudaMemsetAsync(&c.hdr->err, 0, sizeof(int), st);
  const int n = (c.Nc > c.Gc + 1 ? c.Nc : c.Gc + 1);
  {
    Prof pr(c, "prep", st);
    kl(prep_kernel, grid_for(n, 256, 1 << 20), 256, 0, st, c.arena, c.hdr, c.d_slot_of, c.graph_offset, c.node_graph,
                                                            c.species, c.pos32, c.gslot, c.Gc, c.Nc);
  }
}

void launch_nbr(Ctx& c, cudaStream_t st) {
  const int warps_blocks = grid_for((long long)c.Nc * 32, 256, c.sm_count * 16);
  {
    Prof pr(c, "nbr.count", st);
    kl(nbr_count_kernel, warps_blocks, 256, 0, st, c.arena, c.hdr, c.graph_offset, c.node_graph, c.deg, c.rc2);
  }
  {
    Prof pr(c, "nbr.scan", st);
    kl(scan_kernel, 1, 1024, 0, st, c.hdr, c.deg, c.row_ptr, c.graph_offset, c.edge_offset, c.Ec);
  }
  {
    Prof pr(c, "nbr.write", st);
    kl(nbr_write_kernel, warps_blocks, 256, 0, st, c.arena, c.hdr, c.graph_offset, c.node_graph, c.row_ptr, c.pos32,
                                                   c.edge_src, c.edge_dst, c.geo, c.dist, c.rc2, c.Ec);
  }
  {
    Prof pr(c, "nbr.rev", st);
    kl(rev_kernel, grid_for(c.Ec, 256, c.sm_count * 8), 256, 0, st, c.hdr, c.row_ptr, c.edge_src, c.edge_dst, c.rev,
                                                                     c.Ec);
  }
  {
    Prof pr(c, "route", st);
    kl(route_kernel, 1, 1024, 0, st, c.hdr, c.gslot, c.graph_offset, c.edge_offset, c.gperm, c.gnode_base,
                                     c.gedge_base, c.S);
  }
  const long long m = c.Nc > c.Ec ? c.Nc : c.Ec;
  {
    Prof pr(c, "route.perm", st);
    kl(perm_kernel, grid_for(m, 256, c.sm_count * 8), 256, 0, st, c.hdr, c.node_graph, c.graph_offset, c.edge_offset,
                                                                   c.edge_dst, c.gnode_base, c.gedge_base, c.node_perm,
                                                                   c.edge_perm);
  }
}

}  // namespace hmtl_b200
