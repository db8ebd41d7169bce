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
#include <algorithm>
#include <cmath>

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
  if (N <= 4 * 1024) {  // one pass: 4 consecutive degrees per thread, loads all in flight at once
    int d[4], t = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = 4 * tid + q < N ? deg[4 * tid + q] : 0, t += d[q];
    int x = t;
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
    int run = x - t + (wid ? warp_sums[wid - 1] : 0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (4 * tid + q < N) row_ptr[4 * tid + q] = run;
      run += d[q];
    }
    if (tid == 1023) carry = run;
    __syncthreads();
  }
  for (int base = 0; N > 4 * 1024 && base < N; base += 1024) {
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
// Edge-capacity overflow (open boundaries: E > Ec; periodic: a row past the
// per-row bound) leaves a partial edge set.  The reference throws in build_batch
// (hmtl/graph.hpp:56 contract); the device step instead empties the batch's edge
// structure (E = 0, every CSR row and graph edge range empty) so no later kernel
// of the captured step reads past the Ec-sized buffers, and the error bit makes
// the host raise and AdamW skip the update.  Returns true when it did.
__device__ __forceinline__ bool overflow_guard(DevHdr* hdr, int* row_ptr, int* edge_offset) {
  if (!(hdr->err & kErrEdgeOverflow)) return false;
  const int N = hdr->N, G = hdr->G;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t <= N || t <= G; t += gridDim.x * blockDim.x) {
    if (t <= N) row_ptr[t] = 0;
    if (t <= G) edge_offset[t] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) hdr->E = 0;
  return true;
}

__global__ void rev_kernel(DevHdr* hdr, int* __restrict__ row_ptr, const int* __restrict__ edge_src,
                           const int* __restrict__ edge_dst, int* __restrict__ rev, int* __restrict__ edge_offset) {
  pdl_wait();
  if (overflow_guard(hdr, row_ptr, edge_offset)) return;
  const int E = hdr->E;
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
  // (an edge overflow empties every edge range: the guard in rev_kernel may be rewriting
  // edge_offset concurrently, this kernel running beside the neighbour-list writers)
  const bool ovf = hdr->err & kErrEdgeOverflow;
  if (G <= 1024) {  // one graph per thread: its slot, node and edge counts loaded once for every slot's pass
    const int g = tid;
    const int gs = g < G ? gslot[g] : -1;
    const int nn = g < G ? graph_offset[g + 1] - graph_offset[g] : 0;
    const int ne = g < G && !ovf ? edge_offset[g + 1] - edge_offset[g] : 0;
    for (int s = 0; s < S; ++s) {
      const bool f = gs == s;
      int v[3] = {f ? 1 : 0, f ? nn : 0, f ? ne : 0};
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
      if (tid == 0) {
        hdr->seg_graph[s + 1] = carry[0];
        hdr->seg_node[s + 1] = carry[1];
        hdr->seg_edge[s + 1] = carry[2];
      }
    }
    return;
  }
  for (int s = 0; s < S; ++s) {
    for (int base = 0; base < G; base += 1024) {
      const int g = base + tid;
      const bool f = g < G && gslot[g] == s;
      int v[3] = {f ? 1 : 0, f ? graph_offset[g + 1] - graph_offset[g] : 0,
                  f && !ovf ? edge_offset[g + 1] - edge_offset[g] : 0};
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
  if (c.pbc) return launch_nbr_pbc(c, st), launch_route(c, st, false);
  const int warps_blocks = grid_for((long long)c.Nc * 32, 256, c.sm_count * 16);
  {
    Prof pr(c, "nbr.count", st);
    kl(nbr_count_kernel, warps_blocks, 256, 0, st, c.arena, c.hdr, c.graph_offset, c.node_graph, c.deg, c.rc2);
  }
  {
    Prof pr(c, "nbr.scan", st);
    kl(scan_kernel, 1, 1024, 0, st, c.hdr, c.deg, c.row_ptr, c.graph_offset, c.edge_offset, c.Ec);
  }
  // the head routing (one CTA) needs only the graph and edge offsets: it runs on a side
  // stream beside the edge writers instead of after them
  cudaStream_t sr = c.side(c.s_e, st);
  if (sr != st) {
    c.dep(st, sr);
    Prof pr(c, "route", sr);
    kl(route_kernel, 1, 1024, 0, sr, c.hdr, c.gslot, c.graph_offset, c.edge_offset, c.gperm, c.gnode_base,
       c.gedge_base, c.S);
  }
  {
    Prof pr(c, "nbr.write", st);
    kl(nbr_write_kernel, warps_blocks, 256, 0, st, c.arena, c.hdr, c.graph_offset, c.node_graph, c.row_ptr, c.pos32,
                                                   c.edge_src, c.edge_dst, c.geo, c.dist, c.rc2, c.Ec);
  }
  {
    Prof pr(c, "nbr.rev", st);
    kl(rev_kernel, grid_for(std::max<long long>(c.Ec, c.Nc + 1), 256, c.sm_count * 8), 256, 0, st, c.hdr, c.row_ptr,
       c.edge_src, c.edge_dst, c.rev, c.edge_offset);
  }
  c.dep(sr, st);
  launch_route(c, st, sr != st);
}

#ifdef HMTL_CHECKED
namespace {
// Checked builds (-DHMTL_CHECKED, tests/test_checked_build.py): every index structure the
// gather / scatter / GEMM kernels of the step dereference, validated on the device after
// the neighbour list and routing; a violation traps (sticky CUDA error -> the step fails).
#define HMTL_REQUIRE(cond, what)                                                        \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("HMTL_CHECKED: %s violated (block %d thread %d)\n", what, blockIdx.x, threadIdx.x); \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
__global__ void check_structure_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr,
                                       const int* __restrict__ dst, const int* __restrict__ src,
                                       const int* __restrict__ rev, const int* __restrict__ graph_offset,
                                       const int* __restrict__ edge_offset, const int* __restrict__ node_graph,
                                       const int* __restrict__ node_perm, const int* __restrict__ edge_perm,
                                       const int* __restrict__ gperm, int Gc, int Nc, long long Ec) {
  pdl_wait();
  const int G = hdr->G, N = hdr->N, E = hdr->E;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  if (tid == 0) {
    HMTL_REQUIRE(G >= 1 && G <= Gc && N >= 1 && N <= Nc && E >= 0 && E <= Ec, "batch sizes within capacity");
    HMTL_REQUIRE(row_ptr[0] == 0 && row_ptr[N] == E, "CSR row_ptr[0] = 0, row_ptr[N] = E");
    HMTL_REQUIRE(graph_offset[0] == 0 && graph_offset[G] == N, "graph_offset spans the nodes");
    HMTL_REQUIRE(edge_offset[0] == 0 && edge_offset[G] == E, "edge_offset spans the edges");
    int prev = 0;
    for (int s = 0; s <= hdr->n_slots; ++s) {
      HMTL_REQUIRE(hdr->seg_edge[s] >= prev && hdr->seg_edge[s] <= E, "head edge segments monotone");
      prev = hdr->seg_edge[s];
    }
  }
  for (int i = tid; i < N; i += nth) {
    HMTL_REQUIRE(row_ptr[i] <= row_ptr[i + 1], "CSR rows monotone");
    HMTL_REQUIRE(node_graph[i] >= 0 && node_graph[i] < G, "node_graph in range");
    HMTL_REQUIRE(node_perm[i] >= 0 && node_perm[i] < N, "node_perm in range");
  }
  for (int g = tid; g < G; g += nth) HMTL_REQUIRE(gperm[g] >= 0 && gperm[g] < G, "gperm in range");
  for (int e = tid; e < E; e += nth) {
    const int d = dst[e], s = src[e], r = rev[e];
    HMTL_REQUIRE(d >= 0 && d < N && s >= 0 && s < N, "edge endpoints in range");
    HMTL_REQUIRE(e >= row_ptr[d] && e < row_ptr[d + 1], "edge in its destination's CSR row");
    HMTL_REQUIRE(r >= 0 && r < E && dst[r] == s && src[r] == d && rev[r] == e, "reverse edge");
    HMTL_REQUIRE(node_graph[d] == node_graph[s], "edge within one graph");
    HMTL_REQUIRE(edge_perm[e] >= 0 && edge_perm[e] < E, "edge_perm in range");
  }
}
}  // namespace
#endif

// head routing + head-sorted permutations (shared by both neighbour lists)
void launch_route(Ctx& c, cudaStream_t st, bool routed) {
  if (!routed) {
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
#ifdef HMTL_CHECKED
  kl(check_structure_kernel, grid_for(m, 256, c.sm_count * 8), 256, 0, st, c.hdr, c.row_ptr, c.edge_dst, c.edge_src,
     c.rev, c.graph_offset, c.edge_offset, c.node_graph, c.node_perm, c.edge_perm, c.gperm, c.Gc, c.Nc, c.Ec);
#endif
}

}  // namespace hmtl_b200

// ============================================================================
// Periodic cells (the reference has no PBC -- parity against
// the builder's FP64 brute force, oracle ho_build_edges_pbc).  Cell list per
// structure: fractional coordinates f = x A^-1 (A rows = lattice vectors),
// nb_k = clamp(floor(width_k / rc), 1, 4) bins per axis (width = perpendicular
// cell width), stencil of r_k bins each way (r_k >= ceil(rc / bin width), + a
// rounding margin); a stencil bin b + o maps to wrapped bin b' and cell image
// s.  Every (j, image) is visited once; the FP64 test is the oracle's,
// ((xi - xj) - S)^2 with S = (n1 a1 + n2 a2) + n3 a3 per component.  Rows come
// out sorted by (src, image key) after a per-warp bitonic sort in shared memory.
namespace hmtl_b200 {
namespace {

constexpr int kPbcMaxDeg = 512;  // per-row sort buffer (cfg4-class crystals: <= ~200)
constexpr int kPbcMaxImg = 7;    // |n_k| bound of the packed image key

__device__ __forceinline__ int img_key(int n1, int n2, int n3) { return (n1 + 8) * 256 + (n2 + 8) * 16 + (n3 + 8); }
__device__ __forceinline__ void img_of(int key, int& n1, int& n2, int& n3) {
  n1 = (key >> 8) - 8, n2 = ((key >> 4) & 15) - 8, n3 = (key & 15) - 8;
}
__device__ __forceinline__ void lat_shift(const double* A, int n1, int n2, int n3, double* S) {
#pragma unroll
  for (int k = 0; k < 3; ++k)
    S[k] = __dadd_rn(__dadd_rn(__dmul_rn(double(n1), A[k]), __dmul_rn(double(n2), A[3 + k])), __dmul_rn(double(n3), A[6 + k]));
}
__device__ __forceinline__ bool within_pbc(const double* __restrict__ pos, int i, int j, const double* S, double rc2) {
  const double dx = __dsub_rn(__dsub_rn(pos[3 * i], pos[3 * j]), S[0]);
  const double dy = __dsub_rn(__dsub_rn(pos[3 * i + 1], pos[3 * j + 1]), S[1]);
  const double dz = __dsub_rn(__dsub_rn(pos[3 * i + 2], pos[3 * j + 2]), S[2]);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)) <= rc2;
}

// CTA per structure: geometry of the cell, per-atom wrap + bin, counting sort into bins
// acoord[i] = bin coords (4 bits each) | (w0 + 128) << 12 | (w1 + 128) << 20; w2[i] = wrap 3
__global__ void pbc_bin_kernel(const uint8_t* __restrict__ arena, const DevHdr* hdr, const int* __restrict__ go,
                               const double* __restrict__ cells, double rc, int* __restrict__ meta,
                               int* __restrict__ bin_start, int* __restrict__ order, int* __restrict__ acoord,
                               int* __restrict__ w2) {
  pdl_wait();
  __shared__ double c[3][3];
  __shared__ double invV;
  __shared__ int nb[3], cnt[64], cur[64];
  const int G = hdr->G, N = hdr->N;
  const double* pos = reinterpret_cast<const double*>(arena + arena_layout(G, N).pos);
  for (int g = blockIdx.x; g < G; g += gridDim.x) {
    const double* A = cells + 9 * size_t(g);
    if (threadIdx.x == 0) {
      for (int k = 0; k < 3; ++k) {
        const int u = (k + 1) % 3, v = (k + 2) % 3;
        c[k][0] = A[3 * u + 1] * A[3 * v + 2] - A[3 * u + 2] * A[3 * v + 1];
        c[k][1] = A[3 * u + 2] * A[3 * v + 0] - A[3 * u + 0] * A[3 * v + 2];
        c[k][2] = A[3 * u + 0] * A[3 * v + 1] - A[3 * u + 1] * A[3 * v + 0];
      }
      const double V = A[0] * c[0][0] + A[1] * c[0][1] + A[2] * c[0][2];
      invV = 1.0 / V;
      int packed = 0;
      for (int k = 0; k < 3; ++k) {
        const double width = fabs(V) / sqrt(c[k][0] * c[k][0] + c[k][1] * c[k][1] + c[k][2] * c[k][2]);
        int n = int(width / rc);
        n = n < 1 ? 1 : (n > 4 ? 4 : n);
        int r = int(rc / (width / n) * (1.0 + 1e-9)) + 1;  // >= ceil(rc / bin width), rounding margin
        r = r > 15 ? 15 : r;
        nb[k] = n;
        packed |= (n << (4 * k)) | (r << (12 + 4 * k));
      }
      meta[g] = packed;
    }
    if (threadIdx.x < 64) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int a0 = go[g], a1 = go[g + 1];
    for (int i = a0 + threadIdx.x; i < a1; i += blockDim.x) {
      int b[3], w[3];
      for (int k = 0; k < 3; ++k) {
        const double f = (pos[3 * i] * c[k][0] + pos[3 * i + 1] * c[k][1] + pos[3 * i + 2] * c[k][2]) * invV;
        const double fl = floor(f);
        w[k] = int(fl);
        const int bb = int((f - fl) * nb[k]);
        b[k] = bb < 0 ? 0 : (bb >= nb[k] ? nb[k] - 1 : bb);
      }
      acoord[i] = b[0] | (b[1] << 4) | (b[2] << 8) | ((w[0] + 128) << 12) | ((w[1] + 128) << 20);
      w2[i] = w[2];
      atomicAdd(&cnt[(b[0] * nb[1] + b[1]) * nb[2] + b[2]], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int s = a0;
      const int nbin = nb[0] * nb[1] * nb[2];
      for (int q = 0; q < nbin; ++q) bin_start[65 * g + q] = s, cur[q] = s, s += cnt[q];
      bin_start[65 * g + nbin] = s;
    }
    __syncthreads();
    for (int i = a0 + threadIdx.x; i < a1; i += blockDim.x) {  // order within a bin is irrelevant:
      const int p = acoord[i];                                   // every row is sorted afterwards
      order[atomicAdd(&cur[((p & 15) * nb[1] + ((p >> 4) & 15)) * nb[2] + ((p >> 8) & 15)], 1)] = i;
    }
    __syncthreads();
  }
}

// warp per destination atom: visit the stencil; pass 1 counts, pass 2 collects,
// sorts and writes its row
template <bool kWrite>
__global__ void __launch_bounds__(256) pbc_row_kernel(const uint8_t* __restrict__ arena, DevHdr* hdr,
                                                      const int* __restrict__ node_graph,
                                                      const double* __restrict__ cells, const int* __restrict__ meta,
                                                      const int* __restrict__ bin_start, const int* __restrict__ order,
                                                      const int* __restrict__ acoord, const int* __restrict__ w2,
                                                      const int* __restrict__ row_ptr,
                                                      const float4* __restrict__ pos32, int* __restrict__ deg,
                                                      int* __restrict__ edge_src, int* __restrict__ edge_dst,
                                                      int* __restrict__ eimg, float4* __restrict__ geo,
                                                      float* __restrict__ dist, double rc2, long long Ec) {
  pdl_wait();
  __shared__ long long buf[8][kPbcMaxDeg];
  const int N = hdr->N, G = hdr->G;
  if (kWrite && hdr->E > Ec) return;
  const double* pos = reinterpret_cast<const double*>(arena + arena_layout(G, N).pos);
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  long long* kb = buf[wl];
  auto wrap_of = [&](int a) {
    const int pa = acoord[a];
    return make_int3(((pa >> 12) & 255) - 128, ((pa >> 20) & 255) - 128, w2[a]);
  };
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += (gridDim.x * blockDim.x) >> 5) {
    const int g = node_graph[i];
    const int mt = meta[g];
    const int nb0 = mt & 15, nb1 = (mt >> 4) & 15, nb2 = (mt >> 8) & 15;
    const int r0 = (mt >> 12) & 15, r1 = (mt >> 16) & 15, r2 = (mt >> 20) & 15;
    const double* A = cells + 9 * size_t(g);
    const int pi = acoord[i];
    const int bi0 = pi & 15, bi1 = (pi >> 4) & 15, bi2 = (pi >> 8) & 15;
    const int3 wi = wrap_of(i);
    int cntr = 0;
    bool overflow = false;
    for (int o0 = -r0; o0 <= r0; ++o0)
      for (int o1 = -r1; o1 <= r1; ++o1)
        for (int o2 = -r2; o2 <= r2; ++o2) {
          const int b0 = bi0 + o0, b1 = bi1 + o1, b2 = bi2 + o2;
          const int s0 = b0 >= 0 ? b0 / nb0 : -((nb0 - 1 - b0) / nb0);  // floor division
          const int s1 = b1 >= 0 ? b1 / nb1 : -((nb1 - 1 - b1) / nb1);
          const int s2 = b2 >= 0 ? b2 / nb2 : -((nb2 - 1 - b2) / nb2);
          const int q = ((b0 - s0 * nb0) * nb1 + (b1 - s1 * nb1)) * nb2 + (b2 - s2 * nb2);
          const int t0 = bin_start[65 * g + q], t1 = bin_start[65 * g + q + 1];
          for (int t = t0; t < t1; t += 32) {
            bool hit = false;
            long long key = 0;
            if (t + lane < t1) {
              const int j = order[t + lane];
              const int3 wj = wrap_of(j);
              const int n1 = s0 - wj.x + wi.x, n2 = s1 - wj.y + wi.y, n3 = s2 - wj.z + wi.z;
              if (!(j == i && n1 == 0 && n2 == 0 && n3 == 0)) {
                double S[3];
                lat_shift(A, n1, n2, n3, S);
                hit = within_pbc(pos, i, j, S, rc2);
                if (hit && (abs(n1) > kPbcMaxImg || abs(n2) > kPbcMaxImg || abs(n3) > kPbcMaxImg)) {
                  atomicOr(&hdr->err, kErrEdgeOverflow);
                  hit = false;
                }
                key = (long long)j * 4096 + img_key(n1, n2, n3);
              }
            }
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (kWrite && hit) {
              const int at = cntr + __popc(m & ((1u << lane) - 1));
              if (at < kPbcMaxDeg) kb[at] = key;
              else overflow = true;
            }
            cntr += __popc(m);
          }
        }
    if (!kWrite) {
      if (lane == 0) deg[i] = cntr;
      continue;
    }
    if (__any_sync(0xffffffffu, overflow) || cntr > kPbcMaxDeg) {
      if (lane == 0) atomicOr(&hdr->err, kErrEdgeOverflow);
      continue;
    }
    // bitonic sort of the row's keys (ascending (src, image))
    int P2 = 1;
    while (P2 < cntr) P2 <<= 1;
    for (int t = cntr + lane; t < P2; t += 32) kb[t] = 0x7FFFFFFFFFFFFFFFLL;
    __syncwarp();
    for (int k = 2; k <= P2; k <<= 1)
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        for (int t = lane; t < P2; t += 32) {
          const int u = t ^ jj;
          if (u > t) {
            const long long a = kb[t], b = kb[u];
            if (((t & k) == 0) == (a > b)) kb[t] = b, kb[u] = a;
          }
        }
        __syncwarp();
      }
    const int base = row_ptr[i];
    const float4 p4 = pos32[i];
    for (int t = lane; t < cntr; t += 32) {
      const long long key = kb[t];
      const int j = int(key >> 12), ik = int(key & 4095);
      int n1, n2, n3;
      img_of(ik, n1, n2, n3);
      double S[3];
      lat_shift(A, n1, n2, n3, S);
      const float4 q4 = pos32[j];
      // FP32 geometry as the open-boundary path (pos32 differences), minus the FP32 image shift
      const float dx = __fsub_rn(__fsub_rn(p4.x, q4.x), float(S[0]));
      const float dy = __fsub_rn(__fsub_rn(p4.y, q4.y), float(S[1]));
      const float dz = __fsub_rn(__fsub_rn(p4.z, q4.z), float(S[2]));
      const float d2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
      const int e = base + t;
      edge_src[e] = j;
      edge_dst[e] = i;
      eimg[e] = ik;
      geo[e] = make_float4(dx, dy, dz, d2);
      dist[e] = __fsqrt_rn(d2);
    }
    __syncwarp();
  }
}

// reverse of (i, j, n) is (j, i, -n): binary search of row j on the (src, image) key
__global__ void pbc_rev_kernel(DevHdr* hdr, int* __restrict__ row_ptr, const int* __restrict__ edge_src,
                               const int* __restrict__ edge_dst, const int* __restrict__ eimg, int* __restrict__ rev,
                               int* __restrict__ edge_offset) {
  pdl_wait();
  if (overflow_guard(hdr, row_ptr, edge_offset)) return;
  const int E = hdr->E;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int i = edge_dst[e], j = edge_src[e];
    int n1, n2, n3;
    img_of(eimg[e], n1, n2, n3);
    const long long want = (long long)i * 4096 + img_key(-n1, -n2, -n3);
    int lo = row_ptr[j], hi = row_ptr[j + 1];
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((long long)edge_src[mid] * 4096 + eimg[mid] < want) lo = mid + 1;
      else hi = mid;
    }
    rev[e] = lo;
  }
}

}  // namespace

void launch_nbr_pbc(Ctx& c, cudaStream_t st) {
  const int warps_blocks = grid_for((long long)c.Nc * 32, 256, c.sm_count * 16);
  const double rc = std::sqrt(c.rc2);
  {
    Prof pr(c, "nbr.pbc_bin", st);
    kl(pbc_bin_kernel, grid_for(c.Gc, 1, c.sm_count * 4), 256, 0, st, c.arena, c.hdr, c.graph_offset, c.cells, rc,
       c.pbc_meta, c.pbc_bins, c.pbc_order, c.pbc_acoord, c.pbc_w2);
  }
  {
    Prof pr(c, "nbr.count", st);
    kl(pbc_row_kernel<false>, warps_blocks, 256, 0, st, c.arena, c.hdr, c.node_graph, c.cells, c.pbc_meta,
       c.pbc_bins, c.pbc_order, c.pbc_acoord, c.pbc_w2, c.row_ptr, c.pos32, c.deg, c.edge_src, c.edge_dst, c.eimg, c.geo,
       c.dist, c.rc2, c.Ec);
  }
  {
    Prof pr(c, "nbr.scan", st);
    kl(scan_kernel, 1, 1024, 0, st, c.hdr, c.deg, c.row_ptr, c.graph_offset, c.edge_offset, c.Ec);
  }
  {
    Prof pr(c, "nbr.write", st);
    kl(pbc_row_kernel<true>, warps_blocks, 256, 0, st, c.arena, c.hdr, c.node_graph, c.cells, c.pbc_meta,
       c.pbc_bins, c.pbc_order, c.pbc_acoord, c.pbc_w2, c.row_ptr, c.pos32, c.deg, c.edge_src, c.edge_dst, c.eimg, c.geo,
       c.dist, c.rc2, c.Ec);
  }
  {
    Prof pr(c, "nbr.rev", st);
    kl(pbc_rev_kernel, grid_for(std::max<long long>(c.Ec, c.Nc + 1), 256, c.sm_count * 8), 256, 0, st, c.hdr,
       c.row_ptr, c.edge_src, c.edge_dst, c.eimg, c.rev, c.edge_offset);
  }
}

}  // namespace hmtl_b200
