// chain.cuh -- fused node-row GEMM chains on tcgen05 (3xTF32, FP32 accumulate).
//
// The node-level MLP work of a message-passing layer is a chain of row-local
// GEMMs whose output feeds the next GEMM's A operand:
//   forward  (hmtl/model.hpp:412-426 + the next layer's factorised edge input)
//            [h | agg] nW1 + nb1 -> vz1 ; h + (silu(vz1) nW2 + nb2) -> h' ; h' [W1a | W1b] -> P'
//   backward (hmtl/model.hpp:569-587, 607-615 regrouped by row)
//            dh2 + S eW1[:2H]^T -> dh ; (dh nW2^T) * silu'(vz1) -> dvz1 ;
//            dvz1 nW1^T -> [dh + dv_h | dagg]
// One CTA owns 128 node rows for the whole chain: GEMM 1's A streams from
// global through a 4-slot ring, every B operand (pre-split weight images)
// streams by bulk async copy through a 3-slot ring, and each intermediate is
// written by the epilogue straight back into shared memory as the next GEMM's
// K-major SW128 A operand (tf32 hi/lo split), so it never round-trips through
// a separate launch.  Intermediates that later kernels need (vz1, h', dh,
// dvz1, ...) are still stored to global by the same epilogue.
//
// Shared memory: X = 4 x 32 KB (GEMM 1: A ring; later: the chained operand,
// K <= 128), B ring = 3 x 32 KB.  TMEM: one accumulator region per GEMM
// (sum of widths <= 512 columns).
#pragma once
#include <type_traits>

#include "tc.cuh"

namespace hmtl_b200 {
namespace chain {

enum Role : int {
  kFwdNode1 = 0,  // A = [h | agg] (K = 2H); y0 = vz1 = acc + bias; next = silu(vz1)
  kFwdNode2 = 1,  // y0 = h' = x0 + (acc + bias); next = h'
  kFwdP = 2,      // A = x0 (first GEMM only, K = H); y0 = P = acc (N = 2H)
  kBwdL11 = 3,    // A = x1 = S (K = 2H); y0 = dh = y0 + acc (in place); next = dh
  kBwdL1 = 4,     // A = x1 (first GEMM only, K = H); y0 = dvz1 = acc * silu'(x0); next = dvz1
  kBwdL4 = 5,     // y0[:, :H] = x0 + acc[:, :H] ; y1 = acc[:, H:]   (N = 2H)
};

struct Gemm {
  int role, K, N;
  const float* img;  // B image: per 32-k chunk [hi | lo], N rows x 128 B each (SW128)
  const float* x0;   // role operand (see Role)
  const float* x1;
  const float* bias;
  float* y0;
  float* y1;
};
struct Chain {
  const int* count;  // node rows (device header)
  int G, H;
  Gemm g[3];
  long long* stamps;  // optional phase timestamps [CTA][32] (engine tuning; null on the training path)
  int dbg;            // engine ablation bits (0 on the training path): 1 no stores, 2 no X writes, 4 no aux loads
  int rows_cap;       // allocated node rows of every operand table
  int prefetch;       // L2 prefetch of the CTA's operands at launch
};
#define CHAIN_STAMP(i)                                                   \
  do {                                                                   \
    if (p.stamps) p.stamps[blockIdx.x * 32 + (i)] = clock64() - t_start; \
  } while (0)

constexpr int kProdWarps = 8, kEpiWarps = 8;
constexpr int kMmaWarp = kProdWarps, kBWarp = kProdWarps + 1, kEpiWarp0 = kProdWarps + 2;
constexpr int kThreads = (kProdWarps + 2 + kEpiWarps) * 32;  // 576
constexpr int kXSlots = 4, kBSlots = 2;
constexpr uint32_t kSlot = 32768;  // hi 16 KB | lo 16 KB (128 rows x 32 k)
constexpr size_t kSlabBytes = size_t(kEpiWarps) * 32 * 32 * 4;  // per-warp 32x32 transpose tiles
constexpr size_t kSmem = size_t(kXSlots + kBSlots) * kSlot + kSlabBytes + 256 + 1024;

__device__ __forceinline__ float4 ld4c(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4c(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
// the same activation code as the unfused kernels (common.cuh), so a fused
// chain is bit-identical to the separate launches it replaces
__device__ __forceinline__ float silu1(float x) { return silu(x); }
__device__ __forceinline__ float sgrad1(float x) { return silu_grad(x); }

// GEMM 1's A operand, 4 consecutive k of row r
template <int R>
__device__ __forceinline__ float4 a1_load(const Gemm& g, int H, int r, int k) {
  if constexpr (R == kFwdNode1) return k < H ? ld4c(g.x0 + size_t(r) * H + k) : ld4c(g.x1 + size_t(r) * H + k - H);
  else if constexpr (R == kFwdP) return ld4c(g.x0 + size_t(r) * H + k);
  else if constexpr (R == kBwdL11) return ld4c(g.x1 + size_t(r) * 2 * H + k);
  else return ld4c(g.x1 + size_t(r) * H + k);  // kBwdL1
}

// epilogue operands that do not depend on the accumulator, for row r, columns n..n+3
template <int R>
__device__ __forceinline__ float4 aux_load(const Gemm& g, int H, int r, int n) {
  if constexpr (R == kFwdNode2) return ld4c(g.x0 + size_t(r) * H + n);  // residual h
  else if constexpr (R == kBwdL11) return ld4c(g.y0 + size_t(r) * H + n);  // dh2 (accumulated in place)
  else if constexpr (R == kBwdL1) return ld4c(g.x0 + size_t(r) * H + n);  // vz1
  else if constexpr (R == kBwdL4) return n < H ? ld4c(g.x0 + size_t(r) * H + n) : make_float4(0.f, 0.f, 0.f, 0.f);
  else return make_float4(0.f, 0.f, 0.f, 0.f);
}
template <int V>
using IC = std::integral_constant<int, V>;

// L2 prefetch (bulk, fire and forget) of the row-major operands this CTA's rows
// [r0, r0 + nr) will read -- GEMM 1's A and every epilogue operand -- plus slice
// `part` of `parts` of the chain's B images.  The step streams ~100 MB of edge
// tensors per layer through the 126 MB L2, so these node tables mostly come from
// DRAM: issued before pdl_wait, the prefetches overlap the previous kernel's tail
// and turn the chain's dependent loads into L2 hits.  (L2 is the coherence
// point: a prefetch racing the previous kernel's writes is harmless.)
using tc::prefetch_l2;
template <int R0, int R1, int R2>
__device__ __forceinline__ void chain_prefetch(const Chain& p, int r0, int nr, int part, int parts) {
  const int H = p.H;
  if (r0 >= p.rows_cap) return;
  if (nr > p.rows_cap - r0) nr = p.rows_cap - r0;
  const size_t row = size_t(H) * 4, rows = size_t(nr) * row;
  const Gemm& g0 = p.g[0];
  if constexpr (R0 == kFwdNode1) {
    prefetch_l2(g0.x0 + size_t(r0) * H, rows), prefetch_l2(g0.x1 + size_t(r0) * H, rows);
  } else if constexpr (R0 == kFwdP) {
    prefetch_l2(g0.x0 + size_t(r0) * H, rows);
  } else if constexpr (R0 == kBwdL11) {
    prefetch_l2(g0.x1 + size_t(r0) * 2 * H, 2 * rows), prefetch_l2(g0.y0 + size_t(r0) * H, rows);
  } else if constexpr (R0 == kBwdL1) {
    prefetch_l2(g0.x1 + size_t(r0) * H, rows), prefetch_l2(g0.x0 + size_t(r0) * H, rows);
  }
  auto aux = [&](auto rc, const Gemm& g) {
    constexpr int R = decltype(rc)::value;
    if constexpr (R == kFwdNode2 || R == kBwdL1 || R == kBwdL4) prefetch_l2(g.x0 + size_t(r0) * H, rows);
  };
  if constexpr (R1 >= 0) aux(IC<R1>{}, p.g[1]);
  if constexpr (R2 >= 0) aux(IC<R2>{}, p.g[2]);
  constexpr int G = R2 >= 0 ? 3 : (R1 >= 0 ? 2 : 1);
  for (int i = 0; i < G; ++i) {  // this CTA's share of every B image (each image is read by all CTAs)
    const size_t bytes = size_t(2) * p.g[i].K * p.g[i].N * 4, sl = (bytes / parts + 255) & ~size_t(255);
    const size_t o = sl * size_t(part);
    if (o < bytes) prefetch_l2(reinterpret_cast<const char*>(p.g[i].img) + o, bytes - o < sl ? bytes - o : sl);
  }
}

// epilogue of one GEMM for row r, columns n..n+3 (acc a, operands x); stores the
// outputs when `store` and returns the next GEMM's A values
template <int R>
__device__ __forceinline__ float4 epi_apply(const Gemm& g, int H, int r, int n, float4 a, float4 x, bool store) {
  if constexpr (R == kFwdNode1) {
    const float4 b = ld4c(g.bias + n);
    const float4 v = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    if (store) st4c(g.y0 + size_t(r) * H + n, v);
    return make_float4(silu1(v.x), silu1(v.y), silu1(v.z), silu1(v.w));
  } else if constexpr (R == kFwdNode2) {
    const float4 b = ld4c(g.bias + n);
    const float4 v = make_float4(x.x + (a.x + b.x), x.y + (a.y + b.y), x.z + (a.z + b.z), x.w + (a.w + b.w));
    if (store) st4c(g.y0 + size_t(r) * H + n, v);
    return v;
  } else if constexpr (R == kFwdP) {
    if (store) st4c(g.y0 + size_t(r) * 2 * H + n, a);
    return a;
  } else if constexpr (R == kBwdL11) {
    const float4 v = make_float4(x.x + a.x, x.y + a.y, x.z + a.z, x.w + a.w);
    if (store) st4c(g.y0 + size_t(r) * H + n, v);
    return v;
  } else if constexpr (R == kBwdL1) {
    const float4 v = make_float4(a.x * sgrad1(x.x), a.y * sgrad1(x.y), a.z * sgrad1(x.z), a.w * sgrad1(x.w));
    if (store) st4c(g.y0 + size_t(r) * H + n, v);
    return v;
  } else {  // kBwdL4
    if (store) {
      if (n < H) st4c(g.y0 + size_t(r) * H + n, make_float4(x.x + a.x, x.y + a.y, x.z + a.z, x.w + a.w));
      else st4c(g.y1 + size_t(r) * H + n - H, a);
    }
    return a;
  }
}


// ---- CS-CTA cluster column split (CS = 2 or 4): rank r of a cluster computes
// columns [r N/CS, (r+1) N/CS) of every GEMM of the same 128 rows and writes its
// slice of the chained A operand into every CTA's shared memory (DSMEM),
// arriving on every CTA's per-chunk barriers with cluster-scope release
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster4(uint32_t addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void arrive_cluster(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(tc::smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// The role sequence is a compile-time parameter: a switch over roles in the
// unrolled epilogue made every iteration distinct code (instruction-fetch bound).
// MR = node rows per CTA: 128 (M=128 MMAs, accumulator row r in TMEM lane r) or 64
// (M=64 MMAs: twice the CTAs for the same rows; accumulator row r in TMEM lane
// (r % 16) + 32 (r / 16), so each epilogue warp owns 16 rows of its lane quadrant).
template <int R0, int R1, int R2, int CS = 1, int MR = 128>
__global__ void __launch_bounds__(kThreads, 1) chain_kernel(Chain p) {
  constexpr int G = R2 >= 0 ? 3 : (R1 >= 0 ? 2 : 1);
  constexpr int QR = MR / 4;  // rows per TMEM lane quadrant (epilogue warp)
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  const long long t_start = clock64();
  const int M = *p.count;
  const int row0 = (blockIdx.x / CS) * MR;
  const uint32_t crank = CS > 1 ? cluster_rank() : 0;
  if (row0 >= M) return;  // whole CTA (and its cluster peer), before any barrier or TMEM use
  uint8_t* sm = align1k(smem_dyn);
  uint8_t* X = sm;                          // kXSlots x kSlot
  uint8_t* Bq = sm + kXSlots * kSlot;       // kBSlots x kSlot
  float* slabs = reinterpret_cast<float*>(sm + (kXSlots + kBSlots) * kSlot);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (kXSlots + kBSlots) * kSlot + kSlabBytes);
  uint64_t* afull = bars;                   // [4] producer threads
  uint64_t* aempty = bars + 4;              // [4] MMA commit
  uint64_t* bfull = bars + 8;               // [3] tx
  uint64_t* bempty = bars + 11;             // [3] MMA commit
  uint64_t* accd = bars + 14;               // [3] MMA commit: GEMM g complete
  uint64_t* xrdy = bars + 17;               // [2][4] the 4 warps of a slab: X chunk c of GEMM g+1's A
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 25);
  uint64_t* pd = bars + 26;                 // [3] cluster peer's GEMM g complete (CS > 1)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = p.H;
  uint32_t acc_off[3];
  int nb_[3], ne_[3];  // this CTA's column range of GEMM i
  {
    uint32_t o = 0;
    for (int i = 0; i < G; ++i) {
      nb_[i] = int(crank) * (p.g[i].N / CS), ne_[i] = nb_[i] + p.g[i].N / CS;
      acc_off[i] = o, o += uint32_t(p.g[i].N / CS);
    }
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
  if (tid == 0) {
    for (int s = 0; s < kXSlots; ++s) mbar_init(&afull[s], kProdWarps * 32), mbar_init(&aempty[s], 1);
    for (int s = 0; s < kBSlots; ++s) mbar_init(&bfull[s], 1), mbar_init(&bempty[s], 1);
    for (int i = 0; i < 3; ++i) mbar_init(&accd[i], 1);
    for (int i = 0; i < 8; ++i) mbar_init(&xrdy[i], 4 * 32);
    for (int i = 0; i < 3; ++i) mbar_init(&pd[i], CS > 1 ? CS - 1 : 1);
    fence_mbar_init();
  }
  tc_fence_before();
  if constexpr (CS > 1) cluster_sync();  // the peer's barriers exist before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // setup above overlaps the previous kernel's tail
  if (tid == 0) CHAIN_STAMP(0);

  if (warp < kProdWarps) {  // ---------------------------- GEMM 1's A operand
    const int kq = lane & 3, rsub = lane >> 2;
    const int nch = p.g[0].K / KC;
    constexpr int kIt = MR / 64;  // 8-row groups per producer warp
    int rows[2];
    for (int it = 0; it < 2; ++it) {
      const int v = row0 + warp * 8 * kIt + it * 8 + rsub;
      rows[it] = (it < kIt && v < M) ? v : -1;
    }
    // three chunk buffers: the one being stored and the next two in flight
    float4 x0[2][2], x1[2][2], x2[2][2];
    auto load = [&](int c, float4 (&d)[2][2]) {
      if (c >= nch) return;
#pragma unroll
      for (int it = 0; it < 2; ++it)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          d[it][h] = rows[it] >= 0 ? a1_load<R0>(p.g[0], H, rows[it], c * KC + 8 * kq + 4 * h) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    auto store = [&](int c, const float4 (&d)[2][2]) {
      const int s = c % kXSlots;
      mbar_wait(&aempty[s], ((c / kXSlots) & 1) ^ 1);
      float* hi = reinterpret_cast<float*>(X + s * kSlot);
      float* lo = hi + 128 * KC;
#pragma unroll
      for (int it = 0; it < kIt; ++it)
#pragma unroll
        for (int h = 0; h < 2; ++h) put4(hi, lo, 2 * kq + h, warp * 8 * kIt + it * 8 + rsub, d[it][h]);
      fence_proxy_async();
      mbar_arrive(&afull[s]);
    };
    load(0, x0);
    load(1, x1);
    for (int c = 0; c < nch; c += 3) {
      load(c + 2, x2);
      store(c, x0);
      if (c + 1 >= nch) break;
      load(c + 3, x0);
      store(c + 1, x1);
      if (c + 2 >= nch) break;
      load(c + 4, x1);
      store(c + 2, x2);
    }
    if (tid == 0) CHAIN_STAMP(1);
  } else if (warp == kBWarp) {  // ------------------------------- B images
    if (lane == 0) {
      int q = 0;
      for (int gi = 0; gi < G; ++gi) {
        const Gemm& g = p.g[gi];
        for (int n0 = nb_[gi]; n0 < ne_[gi]; n0 += 128) {
          const int nr = ne_[gi] - n0 < 128 ? ne_[gi] - n0 : 128;
          const uint32_t bytes = uint32_t(nr) * 128;
          for (int c = 0; c < g.K / KC; ++c, ++q) {
            const int s = q % kBSlots;
            mbar_wait(&bempty[s], ((q / kBSlots) & 1) ^ 1);
            mbar_expect_tx(&bfull[s], 2 * bytes);
            uint8_t* dst = Bq + s * kSlot;
            const float* src = g.img + size_t(c) * 2 * g.N * KC + size_t(n0) * KC;
            bulk_g2s(dst, src, bytes, &bfull[s]);
            bulk_g2s(dst + 16384, src + size_t(g.N) * KC, bytes, &bfull[s]);
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {  // ---------------------------- MMA issuer
    int q = 0;
    for (int gi = 0; gi < G; ++gi) {
      const Gemm& g = p.g[gi];
      const int nch = g.K / KC;
      if (lane == 0) CHAIN_STAMP(2 + 2 * gi);
      for (int n0 = nb_[gi]; n0 < ne_[gi]; n0 += 128) {
        const int nr = ne_[gi] - n0 < 128 ? ne_[gi] - n0 : 128;
        const uint32_t idesc = (idesc_tf32(nr) & ~(31u << 24)) | (uint32_t(MR >> 4) << 24);
        for (int c = 0; c < nch; ++c, ++q) {
          const int s = q % kBSlots;
          int xs = c;
          if (gi == 0) {  // A ring slot c % 4 (chunks of GEMM 1 stream through X)
            xs = c % kXSlots;
            if (n0 == nb_[gi]) {
              mbar_wait(&afull[xs], (c / kXSlots) & 1);
              tc_fence_after();
            }
          } else if (n0 == nb_[gi]) {  // chunk c of the chained operand, written slab by slab by
            // the previous epilogue (of either CTA of the cluster): MMAs start early
            if constexpr (CS > 1) wait_cluster(&xrdy[(gi - 1) * 4 + c], 0);
            else mbar_wait(&xrdy[(gi - 1) * 4 + c], 0);
            tc_fence_after();
          }
          mbar_wait(&bfull[s], (q / kBSlots) & 1);
          tc_fence_after();
          const uint32_t ah = smem_u32(X + xs * kSlot), bh = smem_u32(Bq + s * kSlot);
          issue_chunk_warp(tmem + acc_off[gi] + uint32_t(n0 - nb_[gi]), ah, ah + 16384, bh, bh + 16384, idesc,
                           c != 0);
          commit_warp(&bempty[s]);
          if (gi == 0 && n0 + 128 >= ne_[gi]) commit_warp(&aempty[xs]);
          __syncwarp();
        }
      }
      commit_warp(&accd[gi]);
      if (lane == 0) CHAIN_STAMP(3 + 2 * gi);
      __syncwarp();
    }
  } else {  // ----------------------------------------------------- epilogue
    const int ew = warp - kEpiWarp0, qd = warp & 3, half = ew >> 2;
    float* slab = slabs + ew * 32 * 32;
    auto phase = [&](auto role_c, auto gi_c) {
      constexpr int R = decltype(role_c)::value, gi = decltype(gi_c)::value;
      constexpr bool last = gi == G - 1;
      const Gemm& g = p.g[gi];
      mbar_wait(&accd[gi], 0);
      tc_fence_after();
      if constexpr (CS > 1) {
        if (!last) {  // the peers write into our X (and we into theirs) only once every CTA's
          // MMAs of GEMM gi -- which read X -- are complete
          if (ew == 0 && lane == 0)
            for (uint32_t pr = 1; pr < uint32_t(CS); ++pr) arrive_cluster(mapa(smem_u32(&pd[gi]), (crank + pr) % CS));
          wait_cluster(&pd[gi], 0);
        }
      }
      if (ew == 0 && lane == 0) CHAIN_STAMP(8 + 2 * gi);
      // per 32-column slab: TMEM (thread = row) -> XOR-swizzled smem tile -> read back
      // transposed (8 lanes x 16 B per row, 4 rows per instruction) so the operand
      // loads, output stores and next-operand writes are row-coalesced
      const int cc = lane & 7;
      for (int sl = half; nb_[gi] + sl * 32 < ne_[gi]; sl += 2) {
        const int j = nb_[gi] + sl * 32;
        constexpr int kRit = QR / 4;  // rows of this warp's quadrant, 4 per read-back pass
        float4 x[kRit];  // the slab's operand loads are in flight before the TMEM read
#pragma unroll
        for (int it = 0; it < kRit; ++it) {
          const int rr = row0 + qd * QR + it * 4 + (lane >> 3);
          x[it] = (rr < M && !(p.dbg & 4)) ? aux_load<R>(g, H, rr, j + 4 * cc) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float acc[32];
        tmem_ld32(tmem + acc_off[gi] + (uint32_t(qd * 32) << 16) + uint32_t(j - nb_[gi]), acc);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4*>(slab + lane * 32 + ((i ^ (lane & 7)) << 2)) =
              make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
        __syncwarp();
#pragma unroll
        for (int it = 0; it < kRit; ++it) {  // (M=64: lanes 16-31 of the slab are not rows)
          const int rl = it * 4 + (lane >> 3), rr = row0 + qd * QR + rl;
          const float4 a = *reinterpret_cast<const float4*>(slab + rl * 32 + ((cc ^ (rl & 7)) << 2));
          const float4 v = epi_apply<R>(g, H, rr < M ? rr : 0, j + 4 * cc, a, x[it], rr < M && !(p.dbg & 1));
          if (!last && !(p.dbg & 2)) {  // next GEMM's A: k = j + 4cc -> chunk j / 32, piece cc of row rl
            float* hi = reinterpret_cast<float*>(X + (j / KC) * kSlot);
            put4(hi, hi + 128 * KC, cc, qd * QR + rl, v);
            if constexpr (CS > 1) {  // the same 16 B pieces into every peer's X (DSMEM)
              const float4 h4 = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
              const float4 l4 = make_float4(v.x - h4.x, v.y - h4.y, v.z - h4.z, v.w - h4.w);
              const uint32_t o = smem_u32(hi) + sw128(qd * QR + rl, cc);
#pragma unroll
              for (int pr = 1; pr < CS; ++pr) {
                const uint32_t peer = (crank + uint32_t(pr)) % CS;
                st_cluster4(mapa(o, peer), h4);
                st_cluster4(mapa(o + 128 * KC * 4, peer), l4);
              }
            }
          }
        }
        __syncwarp();
        if (!last) {  // this warp's 32 rows of X chunk j / 32 are written
          if constexpr (CS > 1) {
            asm volatile("fence.proxy.async;" ::: "memory");
            tc_fence_before();
            mbar_arrive(&xrdy[gi * 4 + j / KC]);
#pragma unroll
            for (int pr = 1; pr < CS; ++pr)
              arrive_cluster(mapa(smem_u32(&xrdy[gi * 4 + j / KC]), (crank + uint32_t(pr)) % CS));
          } else {
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(&xrdy[gi * 4 + sl]);
          }
        }
      }
      if (ew == 0 && lane == 0) CHAIN_STAMP(9 + 2 * gi);
    };
    phase(IC<R0>{}, IC<0>{});
    if constexpr (G > 1) phase(IC<R1>{}, IC<1>{});
    if constexpr (G > 2) phase(IC<R2>{}, IC<2>{});
  }
  tc_fence_before();
  if constexpr (CS > 1) cluster_sync();  // no CTA leaves while its peer may still write into it
  else __syncthreads();
  if (tid == 0) CHAIN_STAMP(31);
  if (warp == kMmaWarp) tmem_dealloc(tmem, 512);
}

// GEMM 1's A operand: address of 4 consecutive k of row r (the cp.async producer)
template <int R>
__device__ __forceinline__ const float* a1_src(const Gemm& g, int H, int r, int k) {
  if constexpr (R == kFwdNode1) return k < H ? g.x0 + size_t(r) * H + k : g.x1 + size_t(r) * H + k - H;
  else if constexpr (R == kFwdP) return g.x0 + size_t(r) * H + k;
  else if constexpr (R == kBwdL11) return g.x1 + size_t(r) * 2 * H + k;
  else return g.x1 + size_t(r) * H + k;  // kBwdL1
}

__device__ __forceinline__ float2 ld2c(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void st2c(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }
// aux_load / epi_apply for 2 consecutive columns n, n+1 (the pair kernel's .16x256b fragments)
template <int R>
__device__ __forceinline__ float2 aux_load2(const Gemm& g, int H, int r, int n) {
  if constexpr (R == kFwdNode2) return ld2c(g.x0 + size_t(r) * H + n);
  else if constexpr (R == kBwdL11) return ld2c(g.y0 + size_t(r) * H + n);
  else if constexpr (R == kBwdL1) return ld2c(g.x0 + size_t(r) * H + n);
  else if constexpr (R == kBwdL4) return n < H ? ld2c(g.x0 + size_t(r) * H + n) : make_float2(0.f, 0.f);
  else return make_float2(0.f, 0.f);
}
template <int R>
__device__ __forceinline__ float2 epi_apply2(const Gemm& g, int H, int r, int n, float2 a, float2 x, bool store) {
  if constexpr (R == kFwdNode1) {
    const float2 b = ld2c(g.bias + n);
    const float2 v = make_float2(a.x + b.x, a.y + b.y);
    if (store) st2c(g.y0 + size_t(r) * H + n, v);
    return make_float2(silu1(v.x), silu1(v.y));
  } else if constexpr (R == kFwdNode2) {
    const float2 b = ld2c(g.bias + n);
    const float2 v = make_float2(x.x + (a.x + b.x), x.y + (a.y + b.y));
    if (store) st2c(g.y0 + size_t(r) * H + n, v);
    return v;
  } else if constexpr (R == kFwdP) {
    if (store) st2c(g.y0 + size_t(r) * 2 * H + n, a);
    return a;
  } else if constexpr (R == kBwdL11) {
    const float2 v = make_float2(x.x + a.x, x.y + a.y);
    if (store) st2c(g.y0 + size_t(r) * H + n, v);
    return v;
  } else if constexpr (R == kBwdL1) {
    const float2 v = make_float2(a.x * sgrad1(x.x), a.y * sgrad1(x.y));
    if (store) st2c(g.y0 + size_t(r) * H + n, v);
    return v;
  } else {  // kBwdL4
    if (store) {
      if (n < H) st2c(g.y0 + size_t(r) * H + n, make_float2(x.x + a.x, x.y + a.y));
      else st2c(g.y1 + size_t(r) * H + n - H, a);
    }
    return a;
  }
}
// 2 consecutive k-values (k even, k < 32) of row r into the hi/lo operand tiles
__device__ __forceinline__ void put2(uint8_t* hi, int r, int k, float2 v) {
  const float2 h = make_float2(tc::tf32_hi(v.x), tc::tf32_hi(v.y));
  const uint32_t o = tc::sw128(r, k >> 2) + uint32_t(k & 3) * 4;
  *reinterpret_cast<float2*>(hi + o) = h;
  *reinterpret_cast<float2*>(hi + 128 * tc::KC * 4 + o) = make_float2(v.x - h.x, v.y - h.y);
}

// ---- CTA-pair chain (cta_group::2).  A cluster of two CTAs runs every GEMM of
// the chain as M = 256 MMAs issued by the leader (rank 0): CTA r owns node rows
// [pair + 128 r, +128) -- its A operand and its accumulator rows (TMEM lanes 0-127,
// all N columns) -- and holds columns [r N/2, (r+1) N/2) of every B operand, so
// each weight byte crosses into the pair once and no activation crosses between
// the two SMs (the column-split chain above pushed the chained operand through
// DSMEM, ~21 B/clk).  B images use the pair layout (per half, per 32-k chunk,
// [hi | lo] contiguous: one 32 KB bulk copy per ring slot).  Readiness of the
// peer's operands reaches the leader by remote mbarrier arrivals; MMA completion
// reaches both CTAs by multicast commits.
namespace pairk {
constexpr int kAWarp = kEpiWarp0 + kEpiWarps;               // GEMM 1's A tiles (TMA issue)
constexpr int kThreads = (kProdWarps + 3 + kEpiWarps) * 32;  // 608 (still 5 warps per SMSP: 96 registers)
constexpr uint32_t kBSlot = 32768;                           // one bulk copy: 1-4 chunks of one GEMM
constexpr int kBRing = 3;
constexpr size_t kSmem = size_t(kXSlots) * kSlot + size_t(kBRing) * kBSlot + 512 + 1024;
}  // namespace pairk

template <int R0, int R1, int R2>
__global__ void __launch_bounds__(pairk::kThreads, 1)
    pair_kernel(Chain p, const __grid_constant__ CUtensorMap ma0, const __grid_constant__ CUtensorMap ma1) {
  constexpr int G = R2 >= 0 ? 3 : (R1 >= 0 ? 2 : 1);
  using namespace tc;
  using pairk::kBRing;
  using pairk::kBSlot;
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  const long long t_start = clock64();
  const int M = *p.count;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int prow0 = (blockIdx.x / 2) * 256, row0 = prow0 + int(crank) * 128;
  if (prow0 >= M) return;  // the whole pair, before any barrier or TMEM use
  uint8_t* sm = align1k(smem_dyn);
  uint8_t* X = sm;                            // kXSlots x kSlot
  uint8_t* Bq = sm + kXSlots * kSlot;         // kBRing x kBSlot
  uint64_t* bars = reinterpret_cast<uint64_t*>(Bq + kBRing * kBSlot);
  uint64_t* afull = bars;       // [4] leader: 8 producer warps of each CTA
  uint64_t* aempty = bars + 4;  // [4] multicast commit
  uint64_t* bfull = bars + 8;   // [3] tx (+ the peer's forwarded arrival on the leader)
  uint64_t* bempty = bars + 11; // [3] multicast commit
  uint64_t* accd = bars + 14;   // [3] multicast commit: GEMM g complete
  uint64_t* xrdy = bars + 17;   // [2][4] leader: chunk c of GEMM g+1's A, 4 epilogue warps of each CTA
  uint64_t* tfull = bars + 25;  // [4] tx: GEMM 1's A tile landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 29);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = p.H;
  uint32_t acc_off[3];
  {
    uint32_t o = 0;
    for (int i = 0; i < G; ++i) acc_off[i] = o, o += uint32_t(p.g[i].N);
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kXSlots; ++s) mbar_init(&afull[s], 2 * kProdWarps), mbar_init(&aempty[s], 1);
    for (int s = 0; s < kBRing; ++s) mbar_init(&bfull[s], leader ? 2 : 1), mbar_init(&bempty[s], 1);
    for (int i = 0; i < 3; ++i) mbar_init(&accd[i], 1);
    for (int i = 0; i < 8; ++i) mbar_init(&xrdy[i], 2 * 4);
    for (int s = 0; s < kXSlots; ++s) mbar_init(&tfull[s], 1);
    fence_mbar_init();
  }
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs exist before any remote arrive; TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tid == pairk::kThreads - 1) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&ma0) : "memory");
    if (R0 == kFwdNode1) asm volatile("prefetch.tensormap [%0];" ::"l"(&ma1) : "memory");
  }
  if (p.prefetch && tid == pairk::kThreads - 1) chain_prefetch<R0, R1, R2>(p, row0, 128, blockIdx.x, gridDim.x);
  pdl_wait();
  if (tid == 0) CHAIN_STAMP(0);
  // this CTA's arrival on the leader's barrier (local when we are the leader)
  auto arrive_leader = [&](uint64_t* bar) {
    if (leader) mbar_arrive(bar);
    else arrive_cluster(mapa(smem_u32(bar), 0));
  };

  if (warp == pairk::kAWarp) {  // ------------- GEMM 1's A: 32 k x 128 row TMA tiles (SW128) into the X ring
    if (lane == 0) {
      const int nch = p.g[0].K / KC;
      for (int c = 0; c < nch; ++c) {
        const int s = c % kXSlots;
        mbar_wait(&aempty[s], ((c / kXSlots) & 1) ^ 1);
        mbar_expect_tx(&tfull[s], 128u * 128u);
        int col = c * KC;
        const CUtensorMap* m = &ma0;
        if (R0 == kFwdNode1 && col >= H) m = &ma1, col -= H;
        tma_2d(X + s * kSlot, m, col, row0, &tfull[s]);
      }
    }
  } else if (warp < kProdWarps) {  // ------------- split the landed fp32 tiles into tf32 hi | lo in place
    const int nch = p.g[0].K / KC;
    for (int c = 0; c < nch; ++c) {
      const int s = c % kXSlots;
      mbar_wait(&tfull[s], (c / kXSlots) & 1);
      float4* hi = reinterpret_cast<float4*>(X + s * kSlot);
      float4* lo = hi + 128 * KC / 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // (the same swizzled offset in both tiles)
        const int o = tid + i * kProdWarps * 32;
        const float4 v = hi[o];
        const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        hi[o] = h;
        lo[o] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) arrive_leader(&afull[s]);
      if (tid == 0 && (c == 0 || c == 3)) CHAIN_STAMP(26 + (c == 3));
    }
    if (tid == 0) CHAIN_STAMP(1);
  } else if (warp == kBWarp) {  // ------------- B: this CTA's column half, 32 KB bulk copies
    if (lane == 0) {
      int q = 0;
      for (int gi = 0; gi < G; ++gi) {
        const Gemm& g = p.g[gi];
        const int nch = g.K / KC;
        const uint32_t cb = uint32_t(g.N) * 128;  // one chunk of this half: [hi | lo], N/2 rows x 128 B each
        const int per = int(kBSlot / cb);
        for (int c0 = 0; c0 < nch; c0 += per, ++q) {
          const int s = q % kBRing;
          mbar_wait(&bempty[s], ((q / kBRing) & 1) ^ 1);
          const int n = nch - c0 < per ? nch - c0 : per;
          mbar_expect_tx(&bfull[s], uint32_t(n) * cb);
          bulk_g2s(Bq + s * kBSlot, g.img + (size_t(crank) * nch + c0) * KC * g.N, uint32_t(n) * cb, &bfull[s]);
        }
      }
    }
  } else if (warp == kMmaWarp) {  // ------------- MMA issuer (leader) / B-copy completion forwarder (peer)
    if (!leader) {
      if (lane == 0) {
        int q = 0;
        for (int gi = 0; gi < G; ++gi) {
          const int nch = p.g[gi].K / KC, per = int(kBSlot / (uint32_t(p.g[gi].N) * 128));
          for (int c0 = 0; c0 < nch; c0 += per, ++q) {
            mbar_wait(&bfull[q % kBRing], (q / kBRing) & 1);
            arrive_cluster(mapa(smem_u32(&bfull[q % kBRing]), 0));
          }
        }
      }
    } else {
      int q = 0;
      for (int gi = 0; gi < G; ++gi) {
        const Gemm& g = p.g[gi];
        const int nch = g.K / KC;
        const uint32_t cb = uint32_t(g.N) * 128;
        const int per = int(kBSlot / cb);
        const uint32_t idesc = (idesc_tf32(g.N) & ~(31u << 24)) | (uint32_t(256 >> 4) << 24);
        if (lane == 0) CHAIN_STAMP(2 + 2 * gi);
        for (int c = 0; c < nch; ++c) {
          const int s = q % kBRing;
          if (c % per == 0) {
            wait_cluster(&bfull[s], (q / kBRing) & 1);
            tc_fence_after();
          }
          int xs = c;
          if (gi == 0) {
            xs = c % kXSlots;
            wait_cluster(&afull[xs], (c / kXSlots) & 1);
            if (lane == 0 && (c == 0 || c == 7)) CHAIN_STAMP(28 + (c == 7));
          } else {
            wait_cluster(&xrdy[(gi - 1) * 4 + c], 0);
          }
          tc_fence_after();
          const uint32_t ah = smem_u32(X + xs * kSlot);
          const uint32_t bh = smem_u32(Bq + s * kBSlot) + uint32_t(c % per) * cb;
          issue_chunk_pair(tmem + acc_off[gi], ah, ah + 16384, bh, bh + cb / 2, idesc, c != 0);
          if (gi == 0) commit_pair(&aempty[xs]);
          if (c % per == per - 1 || c == nch - 1) {
            commit_pair(&bempty[s]);
            ++q;
          }
          __syncwarp();
        }
        commit_pair(&accd[gi]);
        if (lane == 0) CHAIN_STAMP(3 + 2 * gi);
        __syncwarp();
      }
    }
  }
  if (warp < kProdWarps || (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps)) {  // ---- epilogue: 16 warps,
    // (the producer warps join once GEMM 1's A is staged).  .16x256b fragments: a warp
    // owns slab sl (32 columns) of its quadrant's 32 rows; lane t holds rows t/4 and
    // t/4 + 8 of each 16-lane half, 2 adjacent columns of each 8-column group, so the
    // output stores and operand loads are full 32 B sectors and no shared-memory
    // transpose is needed
    const int qd = warp & 3, wq = warp < kProdWarps ? warp >> 2 : 2 + ((warp - kEpiWarp0) >> 2);
    const int tr = lane >> 2, tc2 = 2 * (lane & 3);
    auto phase = [&](auto role_c, auto gi_c) {
      constexpr int R = decltype(role_c)::value, gi = decltype(gi_c)::value;
      constexpr bool last = gi == G - 1;
      const Gemm& g = p.g[gi];
      mbar_wait(&accd[gi], 0);
      tc_fence_after();
      if (warp == kEpiWarp0 + 2 && lane == 0) CHAIN_STAMP(8 + 2 * gi);  // (quadrant 0)
      for (int sl = wq; sl * 32 < g.N; sl += 4) {
        const int j = sl * 32;
        const bool stamp = warp == kEpiWarp0 + 2 && lane == 0 && sl == wq;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int rl0 = qd * 32 + 16 * h + tr;  // rows rl0 and rl0 + 8 of this CTA
          float2 x[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {  // e = 2 jj + (second row)
            const int rr = row0 + rl0 + 8 * (e & 1);
            x[e] = (rr < M && !(p.dbg & 4)) ? aux_load2<R>(g, H, rr, j + 8 * (e >> 1) + tc2) : make_float2(0.f, 0.f);
          }
          float v[16];
          tmem_ld16x32(tmem + acc_off[gi] + (uint32_t(qd * 32 + 16 * h) << 16) + uint32_t(j), v);
          tmem_wait_ld();
          if (stamp && h == 0) CHAIN_STAMP(14 + 4 * gi);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int jj = e >> 1, second = e & 1, rl = rl0 + 8 * second, rr = row0 + rl, col = j + 8 * jj + tc2;
            const float2 a = make_float2(v[4 * jj + 2 * second], v[4 * jj + 2 * second + 1]);
            const float2 y = epi_apply2<R>(g, H, rr < M ? rr : 0, col, a, x[e], rr < M && !(p.dbg & 1));
            if (!last && !(p.dbg & 2)) put2(X + (j / KC) * kSlot, rl, 8 * jj + tc2, y);
          }
        }
        if (stamp) CHAIN_STAMP(15 + 4 * gi);
        if (!last) {  // this warp's 32 rows of X chunk j / 32 are written
          fence_proxy_async();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&xrdy[gi * 4 + j / KC]);
        }
        if (stamp) CHAIN_STAMP(16 + 4 * gi);
      }
      if (warp == kEpiWarp0 + 2 && lane == 0) CHAIN_STAMP(9 + 2 * gi);
    };
    phase(IC<R0>{}, IC<0>{});
    if constexpr (G > 1) phase(IC<R1>{}, IC<1>{});
    if constexpr (G > 2) phase(IC<R2>{}, IC<2>{});
  }
  tc_fence_before();
  cluster_sync();  // the leader's MMAs read both CTAs' shared memory: nobody leaves early
  if (tid == 0) CHAIN_STAMP(31);
  if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

}  // namespace chain
}  // namespace hmtl_b200
