// common.cuh -- device-side building blocks shared by every kernel file.
#pragma once
#include <cuda_runtime.h>

#include <utility>
#include <stdint.h>

namespace hmtl_b200 {

constexpr int kMaxSlots = 16;  // owned heads per rank

// Device-resident batch header.  Every kernel reads sizes from here so that a
// whole training step can be captured once into a CUDA graph and replayed for
// any batch that fits the context's capacities.
struct DevHdr {
  int G, N, E;
  int err;  // bit0 edge overflow, bit1 unowned dataset id, bit2 non-finite prediction, bit3 empty graph
  int n_slots;
  int seg_graph[kMaxSlots + 1];  // head-sorted graph segments
  int seg_node[kMaxSlots + 1];   // head-sorted node segments
  int seg_edge[kMaxSlots + 1];   // head-sorted edge segments
  int step;                      // AdamW step counter
  int loss_done;  // CTAs of the loss kernel finished (the last one reduces and resets it)
  double loss;
};

enum : int { kErrEdgeOverflow = 1, kErrUnowned = 2, kErrNonFinite = 4, kErrEmptyGraph = 8 };

// Packed host->device batch ("arena"): one contiguous byte buffer so the
// upload is a single cudaMemcpyAsync.  Sections follow the header in order;
// offsets depend only on (G, N).
struct ArenaLayout {
  size_t go, ds, sp, pos, le, lf, total;
};
__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline ArenaLayout arena_layout(int G, int N) {
  ArenaLayout a;
  a.go = 16;
  a.ds = align16(a.go + 4 * size_t(G + 1));
  a.sp = align16(a.ds + size_t(G));
  a.pos = align16(a.sp + size_t(N));
  a.le = a.pos + 24 * size_t(N);
  a.lf = a.le + 8 * size_t(G);
  a.total = align16(a.lf + 24 * size_t(N));
  return a;
}

// ---- activation, hmtl/kernels.hpp:62-82 (two-branch stable sigmoid).
// Hardware exp2 (__expf, ~2 ulp) and fast division: |rel err| ~1e-7, far inside
// the FP32 parity bar, and ~5x fewer instructions than expf + IEEE division.
__device__ __forceinline__ float sigm(float x) {
  const float e = __expf(-fabsf(x));
  const float r = __fdividef(1.f, 1.f + e);
  return x >= 0.f ? r : e * r;
}
// (explicitly rounded products/sums: no FMA contraction with the caller's
// arithmetic, so every kernel that evaluates silu/silu' -- fused or not -- gets
// the same bits)
#ifdef HMTL_SILU_FMA  // (A/B: contraction allowed)
__device__ __forceinline__ float silu(float x) { return x * sigm(x); }
__device__ __forceinline__ float silu_grad(float x) {
  const float s = sigm(x);
  return s * (1.f + x * (1.f - s));
}
#else
__device__ __forceinline__ float silu(float x) { return __fmul_rn(x, sigm(x)); }
__device__ __forceinline__ float silu_grad(float x) {
  const float s = sigm(x);
  return __fmul_rn(s, __fadd_rn(1.f, __fmul_rn(x, __fsub_rn(1.f, s))));
}
#endif

// ---- programmatic dependent launch (PDL).  Every kernel calls pdl_wait()
// before it touches memory an earlier kernel of the step wrote (a no-op when it
// was launched without the attribute); kl() launches with the attribute, so the
// next kernel's CTAs are scheduled as the current kernel's CTAs retire and its
// launch latency / prologue overlap the tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
bool pdl_enabled();
// Launch priority of every kernel: the step's critical-path stream (set by the
// context while it enqueues a step) gets the device's highest priority, side streams
// the lowest, as a per-launch attribute so it survives CUDA-graph capture: when a
// critical kernel and a weight-gradient kernel become ready together, the block
// scheduler dispatches the critical kernel's CTAs first (both kinds need a whole
// SM's shared memory, so whichever starts first holds the SMs).
struct LaunchPrio {
  cudaStream_t hi_stream = nullptr;
  int hi = 0, lo = 0;
  bool on = false;
};
LaunchPrio& launch_prio();
template <typename... KArgs, typename... Args>
inline void kl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n++].val.programmaticStreamSerializationAllowed = 1;
  }
  const LaunchPrio& lp = launch_prio();
  if (lp.on) {
    at[n].id = cudaLaunchAttributePriority;
    at[n++].val.priority = st == lp.hi_stream ? lp.hi : lp.lo;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// kl() with a thread-block cluster shape
template <typename... KArgs, typename... Args>
inline void kl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, dim3 cluster,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[3];
  int n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n++].val.programmaticStreamSerializationAllowed = 1;
  }
  at[n].id = cudaLaunchAttributeClusterDimension;
  at[n].val.clusterDim.x = cluster.x, at[n].val.clusterDim.y = cluster.y, at[n++].val.clusterDim.z = cluster.z;
  const LaunchPrio& lp = launch_prio();
  if (lp.on) {
    at[n].id = cudaLaunchAttributePriority;
    at[n++].val.priority = st == lp.hi_stream ? lp.hi : lp.lo;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Sum of n values src[q*stride], q = 0..n-1, with 8 independent accumulators
// (8 loads in flight) combined in a fixed tree: the association depends only on
// n, so results are bit-reproducible run to run.
__device__ __forceinline__ float sum_strided(const float* __restrict__ src, int n, size_t stride) {
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  int q = 0;
  for (; q + 8 <= n; q += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] += src[size_t(q + j) * stride];
  }
  for (int j = 0; q < n; ++q, ++j) a[j] += src[size_t(q) * stride];
  return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

// Deterministic split-partial reduction: out(seg, t) = sum_{q < f.count(seg)}
// src[seg*seg_stride + q*stride + t] for t < T.  CTA = 32 consecutive t of one
// segment (coalesced 128 B rows); warp w sums q = w, w+8, ... with sum_strided,
// and the 8 warp sums combine in a fixed tree, so the association depends only
// on the count.  8x the memory-level parallelism of one thread per output.
template <class F>
__global__ void __launch_bounds__(256) split_reduce_kernel(const float* __restrict__ src, size_t seg_stride,
                                                           size_t stride, int T, F f) {
  pdl_wait();
  __shared__ float red[8][32];
  const int seg = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 32 + lane;
  const int n = f.count(seg);
  float v = 0.f;
  if (t < T && warp < n)
    v = sum_strided(src + size_t(seg) * seg_stride + size_t(warp) * stride + t, (n - warp + 7) / 8, 8 * stride);
  red[warp][lane] = v;
  __syncthreads();
  if (warp == 0 && t < T)
    f.store(seg, t, ((red[0][lane] + red[1][lane]) + (red[2][lane] + red[3][lane])) +
                        ((red[4][lane] + red[5][lane]) + (red[6][lane] + red[7][lane])));
}

// ---- row sets: identity rows [0, *count) or head-sorted segments via a perm
struct RowSet {
  const int* perm = nullptr;     // virtual -> actual row; nullptr = identity
  const int* seg_off = nullptr;  // [nseg+1] device offsets; nullptr = one segment [0, *count)
  const int* count = nullptr;
  int nseg = 1;
  __device__ __forceinline__ int begin(int s) const { return seg_off ? seg_off[s] : 0; }
  __device__ __forceinline__ int end(int s) const { return seg_off ? seg_off[s + 1] : *count; }
  __device__ __forceinline__ int row(int v) const { return perm ? perm[v] : v; }
};

// ============================================================ C = A * B
// C[row, n] = epi(sum_k a(seg,row,k) * b(seg,k,n)); rows from a RowSet, tiles
// never cross a head segment (each segment has its own B = that head's weights).
// 64x64x16 tiles, 256 threads, 4x4 outputs per thread; persistent over tiles.
template <class P>
__global__ void __launch_bounds__(256) gemm_ab_kernel(P p) {
  pdl_wait();
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  int mt_seg[kMaxSlots + 1];
  int total_m = 0;
  for (int s = 0; s < p.rows.nseg; ++s) {
    mt_seg[s] = total_m;
    const int cnt = p.rows.end(s) - p.rows.begin(s);
    total_m += (cnt + BM - 1) / BM;
  }
  mt_seg[p.rows.nseg] = total_m;
  const int ntn = (p.Ncols + BN - 1) / BN;
  for (int t = blockIdx.x; t < total_m * ntn; t += gridDim.x) {
    const int tm = t / ntn, tn = t % ntn;
    int seg = 0;
    while (tm >= mt_seg[seg + 1]) ++seg;
    const int v0 = p.rows.begin(seg) + (tm - mt_seg[seg]) * BM;
    const int v1 = min(v0 + BM, p.rows.end(seg));
    const int n0 = tn * BN;
    // the rows this thread loads (fixed across k)
    int lrow[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + 256 * i, r = idx / BK, v = v0 + r;
      lrow[i] = v < v1 ? p.rows.row(v) : -1;
    }
    float acc[4][4] = {};
    for (int k0 = 0; k0 < p.K; k0 += BK) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int idx = tid + 256 * i, r = idx / BK, kk = idx % BK;
        As[kk][r] = (lrow[i] >= 0 && k0 + kk < p.K) ? p.a(seg, lrow[i], k0 + kk) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int idx = tid + 256 * i, kk = idx / BN, n = idx % BN;
        Bs[kk][n] = (k0 + kk < p.K && n0 + n < p.Ncols) ? p.b(seg, k0 + kk, n0 + n) : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int v = v0 + ty * 4 + i;
      if (v >= v1) continue;
      const int row = p.rows.row(v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int n = n0 + tx * 4 + j;
        if (n < p.Ncols) p.epi(seg, row, n, acc[i][j]);
      }
    }
  }
}

// ============================================================ C = A^T * B
// Weight gradients: C_seg[k, n] = sum over rows r of segment seg of
// a(seg,r,k) * b(seg,r,n).  Deterministic split over rows: CTA (tile, p, seg)
// owns row chunks p, p+P, p+2P, ... (static assignment) and writes a partial
// tile; gemm_atb_reduce sums the P partials in ascending p and stores.
template <class P>
__global__ void __launch_bounds__(256) gemm_atb_kernel(P p, float* __restrict__ partial, int nsplit) {
  pdl_wait();
  constexpr int BK = 64, BN = 64, RC = 16;
  __shared__ float As[RC][BK + 4];
  __shared__ float Bs[RC][BN + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int ntn = (p.Ncols + BN - 1) / BN;
  const int tk = blockIdx.x / ntn, tn = blockIdx.x % ntn;
  const int k0 = tk * BK, n0 = tn * BN;
  const int split = blockIdx.y, seg = blockIdx.z;
  const int rb = p.rows.begin(seg), re = p.rows.end(seg);
  const int nchunks = (re - rb + RC - 1) / RC;
  float acc[4][4] = {};
  for (int c = split; c < nchunks; c += nsplit) {
    const int v0 = rb + c * RC;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + 256 * i, r = idx / BK, kk = idx % BK, v = v0 + r;
      const bool ok = v < re && k0 + kk < p.K;
      As[r][kk] = ok ? p.a(seg, p.rows.row(v), k0 + kk) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + 256 * i, r = idx / BN, n = idx % BN, v = v0 + r;
      const bool ok = v < re && n0 + n < p.Ncols;
      Bs[r][n] = ok ? p.b(seg, p.rows.row(v), n0 + n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RC; ++r) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[r][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[r][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
    }
    __syncthreads();
  }
  const size_t KN = size_t(p.K) * p.Ncols;
  float* out = partial + (size_t(seg) * nsplit + split) * KN;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + ty * 4 + i;
    if (k >= p.K) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n < p.Ncols) out[size_t(k) * p.Ncols + n] = acc[i][j];
    }
  }
}

template <class P>
__global__ void gemm_atb_reduce(P p, const float* __restrict__ partial, int nsplit) {
  pdl_wait();
  const size_t KN = size_t(p.K) * p.Ncols;
  const size_t total = KN * p.rows.nseg;
  for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
       idx += size_t(gridDim.x) * blockDim.x) {
    const int seg = int(idx / KN);
    const size_t kn = idx % KN;
    p.store(seg, int(kn / p.Ncols), int(kn % p.Ncols), sum_strided(partial + size_t(seg) * nsplit * KN + kn, nsplit, KN));
  }
}

}  // namespace hmtl_b200
