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

template <int V>
using IC = std::integral_constant<int, V>;

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

}  // namespace chain
}  // namespace hmtl_b200
