// tc.cuh -- tcgen05 (5th-gen tensor core) GEMM engine for the FP32 path.
//
// Precision: kind::tf32 with the 3xTF32 split (x = hi + lo, hi = x with the
// low 13 mantissa bits cleared; D += A_lo*B_hi + A_hi*B_lo + A_hi*B_hi,
// FP32 accumulation in TMEM) -> ~FP32 accuracy (error ~2^-22 |a||b|), which
// keeps the rel 1e-4 parity bar of the FP32 path.
//
// Operands live in shared memory in the canonical K-major SWIZZLE_128B UMMA
// layout: a K-chunk of 32 fp32 is one 128 B line per row (row r at r*128 B,
// 1 KB atoms of 8 rows), its 16 B chunk c stored at chunk position c ^ (r % 8).
// One MMA (K = 8 -> 32 B) advances the descriptor start by 32 B inside the
// atom; SBO = 1024 B (8-row atom stride).  (The SWIZZLE_NONE "interleaved"
// layout ran the MMAs at ~40% of the tensor floor -- measured with
// hmtl_selftest_time.)  B comes from a pre-split global image with the same
// byte layout (contiguous rows: plain coalesced 16 B copies, L2-resident).
//
// Two engines, both templated on a problem functor:
//   tc_row_kernel : C[row, n] = epi(sum_k A(row,k) B(k,n)), 128-row tiles of a
//                   RowSet (tiles never straddle head segments), N <= 256.
//   tc_red_kernel : C_seg[m, n] = sum_rows A(row,m) B(row,n) for weight
//                   gradients: M-tile 128 features, the ROWS are the reduction
//                   dim (K), statically split over CTAs; fixed-order reduce after.
#pragma once
#include <cuda.h>  // CUtensorMap (the TMA reduce GEMM's operand maps)
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "common.cuh"

namespace hmtl_b200 {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {  // warp-wide
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // warp-wide
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 consecutive TMEM columns of this warp's 32 lanes -> 32 registers / thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 TMEM lanes x 32 consecutive columns (.16x256b, 4 repetitions): thread t holds
// v[4j + {0, 1}] = lane t/4, columns 8j + 2(t%4) + {0, 1} and v[4j + {2, 3}] = lane
// t/4 + 8, same columns (the m16n8 accumulator fragment, repeated along N)
__device__ __forceinline__ void tmem_ld16x32(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// K-major, SWIZZLE_128B shared-memory matrix descriptor (sm100 "version 1",
// layout type 2): LBO unused for swizzled K-major (set to 16 B), SBO = 1024 B.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// instruction descriptor: kind::tf32, D f32, A/B tf32 K-major, M = 128, N
__host__ __device__ constexpr uint32_t idesc_tf32(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// byte offset of 16 B chunk c (k = 4c..4c+3 of the 32-k chunk) of row r
__host__ __device__ __forceinline__ uint32_t sw128(int r, int c) { return uint32_t(r * 128 + ((c ^ (r & 7)) << 4)); }
// write 4 consecutive k-values (chunk c) of row r into the hi/lo operand tiles
__device__ __forceinline__ void put4(float* hi, float* lo, int c, int r, float4 v) {
  float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
  float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
  const uint32_t o = sw128(r, c);
  *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(hi) + o) = h;
  *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(lo) + o) = l;
}

constexpr int KC = 32;  // k values per chunk (4 MMAs of K=8)

// issue the 3xTF32 MMAs of one chunk (single thread); operand tiles are SW128
__device__ __forceinline__ void issue_chunk(uint32_t tmem, const float* a_hi, const float* a_lo, const float* b_hi,
                                            const float* b_lo, uint32_t idesc, bool first) {
  const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
  for (int j = 0; j < KC / 8; ++j) {
    const uint32_t o = 32 * j;  // K = 8 fp32 = 32 B inside the 128 B swizzle atom row
    const uint64_t dah = sdesc_sw128(ah + o), dal = sdesc_sw128(al + o);
    const uint64_t dbh = sdesc_sw128(bh + o), dbl = sdesc_sw128(bl + o);
    mma_tf32(tmem, dal, dbh, idesc, (first && j == 0) ? 0u : 1u);
    mma_tf32(tmem, dah, dbl, idesc, 1u);
    mma_tf32(tmem, dah, dbh, idesc, 1u);
  }
}

// Warp-wide variant: called by all 32 lanes with warp-uniform arguments (the
// descriptors stay in uniform registers); one elected lane issues the chunk's
// 12 MMAs from a single asm block (K step = +32 B = +2 in the descriptor's
// address field) and, when `commit_bar` is set, commits them to that mbarrier.
__device__ __forceinline__ void issue_chunk_warp(uint32_t tmem, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi,
                                                 uint32_t b_lo, uint32_t idesc, uint32_t accumulate) {
  const uint64_t dah = sdesc_sw128(a_hi), dal = sdesc_sw128(a_lo);
  const uint64_t dbh = sdesc_sw128(b_hi), dbl = sdesc_sw128(b_lo);
  asm volatile(
      "{\n\t.reg .pred e, p0, pt;\n\t.reg .b64 ah, al, bh, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p0, %5, 0;\n\t"
      "setp.ne.b32 pt, %6, 0;\n\t"
      "mov.b64 ah, %1;\n\tmov.b64 al, %2;\n\tmov.b64 bh, %3;\n\tmov.b64 bl, %4;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], al, bh, %7, p0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bl, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bh, %7, pt;\n\t"
      "add.s64 ah, ah, 2;\n\tadd.s64 al, al, 2;\n\tadd.s64 bh, bh, 2;\n\tadd.s64 bl, bl, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], al, bh, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bl, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bh, %7, pt;\n\t"
      "add.s64 ah, ah, 2;\n\tadd.s64 al, al, 2;\n\tadd.s64 bh, bh, 2;\n\tadd.s64 bl, bl, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], al, bh, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bl, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bh, %7, pt;\n\t"
      "add.s64 ah, ah, 2;\n\tadd.s64 al, al, 2;\n\tadd.s64 bh, bh, 2;\n\tadd.s64 bl, bl, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], al, bh, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bl, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bh, %7, pt;\n\t"
      "}" ::"r"(tmem),
      "l"(dah), "l"(dal), "l"(dbh), "l"(dbl), "r"(accumulate), "r"(1u), "r"(idesc));
}
// CTA-pair variant (cta_group::2, issued by the pair's leader CTA): M = 256, A rows
// split over the two CTAs, B columns split over them; same shared-memory offsets in both
__device__ __forceinline__ void issue_chunk_pair(uint32_t tmem, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi,
                                                 uint32_t b_lo, uint32_t idesc, uint32_t accumulate) {
  const uint64_t dah = sdesc_sw128(a_hi), dal = sdesc_sw128(a_lo);
  const uint64_t dbh = sdesc_sw128(b_hi), dbl = sdesc_sw128(b_lo);
  asm volatile(
      "{\n\t.reg .pred e, p0, pt;\n\t.reg .b64 ah, al, bh, bl;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p0, %5, 0;\n\t"
      "setp.ne.b32 pt, %6, 0;\n\t"
      "mov.b64 ah, %1;\n\tmov.b64 al, %2;\n\tmov.b64 bh, %3;\n\tmov.b64 bl, %4;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], al, bh, %7, p0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, pt;\n\t"
      "add.s64 ah, ah, 2;\n\tadd.s64 al, al, 2;\n\tadd.s64 bh, bh, 2;\n\tadd.s64 bl, bl, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], al, bh, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, pt;\n\t"
      "add.s64 ah, ah, 2;\n\tadd.s64 al, al, 2;\n\tadd.s64 bh, bh, 2;\n\tadd.s64 bl, bl, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], al, bh, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, pt;\n\t"
      "add.s64 ah, ah, 2;\n\tadd.s64 al, al, 2;\n\tadd.s64 bh, bh, 2;\n\tadd.s64 bl, bl, 2;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], al, bh, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bl, %7, pt;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ah, bh, %7, pt;\n\t"
      "}" ::"r"(tmem),
      "l"(dah), "l"(dal), "l"(dbh), "l"(dbl), "r"(accumulate), "r"(1u), "r"(idesc));
}
// warp-wide: the elected lane (the one that issued the MMAs) commits them to `bar`
// warp-wide, CTA pair: the elected lane's MMAs arrive on `bar` in both CTAs of the pair
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(uint16_t(3))
      : "memory");
}
__device__ __forceinline__ void commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// B images (weights) are built per problem by bimg_prob_kernel (model.cu):
// per 32-k chunk c, [hi | lo], each N rows x 128 B in the SW128 layout above.

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ================================================================ row GEMM
// Warp-specialised, persistent.  Warps 0-7 produce A: 4 lanes per row (32
// contiguous bytes each -> coalesced 128 B row segments), 16 rows per warp;
// the chunk sequence runs across tile boundaries with the next chunk's loads
// in flight while the current one is split into tf32 hi/lo and stored (the
// per-row gather context is computed once per tile).  Warp 8 issues the
// 3xTF32 MMAs (one lane) and owns B: when the whole B image slice (hi+lo,
// K x Nt) fits next to two A stages it is made resident by bulk async copies
// (cp.async.bulk -> mbarrier tx count) and reloaded only when the tile's
// (segment, n0) changes, after the MMAs that read it have completed;
// otherwise an elected producer lane bulk-copies each stage's B slice.
// Warps 9-16 drain a double-buffered TMEM accumulator (two warps per TMEM
// lane quadrant, alternate 32-column slabs), transposing each 32x32 slab
// through an XOR-swizzled 4 KB smem tile so global stores are row-coalesced,
// overlapping tile t's epilogue with tile t+1's MMAs.
// P must provide: RowSet rows; int K, Ncols; const float* bimg; size_t bimg_seg;
//   typename P::RC rctx(int seg, int row) const;                    // per-row gather context
//   typename P::Raw raw4(int seg, int row, const RC&, int k) const; // loads of A(row, k..k+3)
//   float4 fin4(int seg, int row, const RC&, int k, const Raw&) const;  // -> A(row, k..k+3)
//   typename P::Aux epi_aux(int seg, int row, const RC&, int n) const;  // prefetched epilogue inputs
//   void epi4(int seg, int row, const RC&, int n, float4 acc, const Aux&) const;  // C(row, n..n+3)
// Segmented-sum epilogue (P::kSeg; identity RowSet of one segment whose rows are
// sorted by key, e.g. edges by destination): epi4r stores C like epi4 and returns
// the value to reduce; out(key, n) = sum over the rows of that key, in ascending
// row order, is stored (seg_store) for every key whose rows lie inside one
// 128-row tile.  A key that straddles tiles leaves one piece per tile instead:
// tile_store(0, t, n, v) = its rows in tile t when they start the tile (a "head"
// piece, the whole tile if the key covers it), tile_store(1, t, n, v) = its rows
// in tile t when it starts there and continues (a "tail" piece); a fix-up pass
// adds a straddling key's pieces in tile order.
//   int seg_key(int row) const;  float4 epi4r(...same as epi4...) const;
//   void seg_store(int key, int n, float v) const;  void tile_store(int which, int t, int n, float v) const;
constexpr int kMaxStages = 4;
// engine ablation switches for hmtl_selftest_time and HMTL_TC_DEBUG (bit0: producers
// skip A loads/stores, bit1: epilogue skips global stores, bit2: no segmented sums);
// always 0 on the training path.
static __device__ int g_tc_debug = 0;
constexpr int kProdWarps = 8;                                  // 16 rows each
constexpr int kRowIt = 128 / (kProdWarps * 8);                 // row groups of 8 per producer warp
// epilogue warps: kEpiHalves per TMEM lane quadrant, each taking every kEpiHalves-th
// 32-column slab.  (17 warps -- 2 per quadrant -- cap a thread at 96 registers: 5 warps
// share one SM sub-partition's 16K registers; 13 warps allow 128.)
#ifndef HMTL_EPI_HALVES
#define HMTL_EPI_HALVES 2
#endif
constexpr int kEpiHalves = HMTL_EPI_HALVES;
constexpr int kEpiWarps = 4 * kEpiHalves;
constexpr int kMmaWarp = kProdWarps, kEpiWarp0 = kProdWarps + 1;
constexpr int kRowThreads = (kProdWarps + 1 + kEpiWarps) * 32;  // 544 (416 with one epilogue warp per quadrant)
constexpr size_t kSmemLimit = 227 * 1024;
constexpr size_t kEpiBytes = size_t(kEpiWarps) * 32 * 32 * 4;  // one 4 KB slab per epilogue warp
constexpr size_t kRowBars = 256;

// segmented-sum epilogues (P::kSegSum): the tile's row keys, one array per
// epilogue column half (the 4 quadrant warps of a half exchange through it)
constexpr size_t kSegKeyBytes = size_t(2) * 128 * 4;
template <class P, class = void>
struct RowPf : std::false_type {};
template <class P>
struct RowPf<P, std::void_t<decltype(P::kPrefetch)>> : std::bool_constant<P::kPrefetch> {};
template <class P, class = void>
struct RowAsync : std::false_type {};
template <class P>
struct RowAsync<P, std::void_t<decltype(P::kAsync)>> : std::bool_constant<P::kAsync> {};

// cp.async (Ampere-style, no register staging): 16 B global -> shared; src_bytes
// 0 zero-fills (rows past the segment end)
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <class P, class = void>
struct RowSeg : std::false_type {};
template <class P>
struct RowSeg<P, std::void_t<decltype(P::kSeg)>> : std::bool_constant<P::kSeg> {};
// epilogue through shared-memory transpose slabs: segmented sums, and problems whose
// store-only epilogue measured faster with row-coalesced 128 B stores (P::kSlabEpi)
template <class P, class = void>
struct RowSlab : std::bool_constant<RowSeg<P>::value> {};
template <class P>
struct RowSlab<P, std::void_t<decltype(P::kSlabEpi)>> : std::bool_constant<P::kSlabEpi || RowSeg<P>::value> {};

// L2 prefetch (bulk, fire and forget) of a contiguous byte range
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  for (size_t o = 0; o < bytes; o += 65536) {
    const uint32_t n = uint32_t(bytes - o < 65536 ? bytes - o : 65536) & ~15u;
    if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const char*>(p) + o), "r"(n)
                        : "memory");
  }
}
struct RowPlan {
  int Nt, stages, resident, prefetch = 0;
  size_t a_stage, b_stage, b_res, smem;
  size_t epi_bytes;  // transpose slabs of the epilogue (0: register-fragment epilogue, no shared memory)
};
// slabs: the epilogue transposes through per-warp shared-memory slabs (segmented-sum
// problems need them; every other problem reads .16x256b fragments and pairs lanes
// with shuffles, leaving the 32 KB to one more A stage)
inline RowPlan row_plan(int K, int Nt, size_t extra = 0, bool slabs = false, bool pair = false) {
  RowPlan r;
  r.Nt = Nt;
  r.epi_bytes = slabs ? kEpiBytes : 0;
  r.a_stage = size_t(2 * 128 * KC) * 4;  // hi + lo
  const size_t b_chunk = size_t(2 * (pair ? Nt / 2 : Nt) * KC) * 4;  // (pair: this CTA's column half)
  const size_t b_all = b_chunk * (K / KC);
  const size_t fixed = r.epi_bytes + kRowBars + extra + 1024;  // +1 KB: manual 1 KB alignment
  r.resident = (b_all + 2 * r.a_stage + fixed <= kSmemLimit) ? 1 : 0;
  r.b_res = r.resident ? b_all : 0;
  r.b_stage = r.resident ? 0 : b_chunk;
  const size_t per = r.a_stage + r.b_stage;
  int st = int((kSmemLimit - fixed - r.b_res) / per);
  r.stages = st < 2 ? 2 : (st > kMaxStages ? kMaxStages : st);
  r.smem = r.b_res + r.stages * per + fixed;
  return r;
}
// thread-block cluster helpers (split-K partial reduction through DSMEM)
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// wait with cluster-scope acquire (arrivals may come from the cluster peer)
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// arrive on the same-offset barrier of cluster CTA `rank` (release at cluster scope)
__device__ __forceinline__ void mbar_arrive_rank(uint64_t* bar, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ float ld_dsmem(uint32_t saddr, uint32_t rank) {
  uint32_t a;
  float v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(saddr), "r"(rank));
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
// Weight-gradient GEMMs launched as clusters of CL CTAs along the split dimension:
// every CTA stages its accumulator tile T[n][m] (+ the column-sum column) in shared
// memory, then CTA rank r sums rows [r N/CL, (r+1) N/CL) of all CL tiles in rank order
// (DSMEM) and writes them as ONE partial: CL x fewer partials for split_reduce_kernel to
// read, same fixed association for every run.
constexpr int kRedTS = 129;  // T row stride: 128 m-tile features + the column-sum slot
__device__ __forceinline__ void red_cluster_reduce(const float* T, float* partial, int seg, int split, int nsplit,
                                                   int N, int Mo, int m0, int Mt, int M, bool do_colsum, int tid,
                                                   int nthreads) {
  const uint32_t CL = cl_size(), r = cl_rank();
  float* out = partial + (size_t(seg) * (nsplit / CL) + split / CL) * size_t(Mo) * N;
  const int nb = int(r) * N / int(CL), ne = int(r + 1) * N / int(CL);
  const uint32_t tbase = smem_u32(T);
  for (int idx = tid; idx < (ne - nb) * kRedTS; idx += nthreads) {
    const int n = nb + idx / kRedTS, m = idx % kRedTS;
    if (!(m < Mt || (m == kRedTS - 1 && do_colsum))) continue;
    float sum = 0.f;
    for (uint32_t q = 0; q < CL; ++q) sum += ld_dsmem(tbase + uint32_t(n * kRedTS + m) * 4, q);
    out[size_t(n) * Mo + (m < kRedTS - 1 ? m0 + m : M)] = sum;
  }
}

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ uint8_t* align1k(uint8_t* p) {
  return p + ((1024 - (smem_u32(p) & 1023)) & 1023);
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// bulk async copy global -> shared (16 B aligned, bytes % 16 == 0), completes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// kPair: CTA pairs (cta_group::2, 2-CTA clusters) -- M = 256 MMAs issued by the leader,
// CTA r owning m-tile 2t + r of pair-tile t and columns [r Nt/2, (r+1) Nt/2) of the resident
// B (half the shared memory for B: more A stages); one head segment, one column block
template <class P, bool kPair = false>
__global__ void __launch_bounds__(kRowThreads, 1) tc_row_kernel(P p, RowPlan plan) {
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  uint8_t* smem_raw = align1k(smem_dyn);  // SW128 atoms need 1 KB alignment
  const int Nt = plan.Nt, kStages = plan.stages;
  const size_t SB = plan.a_stage + plan.b_stage;
  float* bres = reinterpret_cast<float*>(smem_raw);  // resident B (hi/lo per chunk)
  uint8_t* stages = smem_raw + plan.b_res;
  float* epi_smem = reinterpret_cast<float*>(stages + kStages * SB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kStages * SB + plan.epi_bytes);
  uint64_t* full = bars;                        // [kStages], count = producer threads (+ tx)
  uint64_t* empty = bars + kStages;             // [kStages], count 1 (MMA commit)
  uint64_t* accfull = bars + 2 * kStages;       // [2], count 1
  uint64_t* accempty = bars + 2 * kStages + 2;  // [2], count = epilogue threads
  uint64_t* bfull = bars + 2 * kStages + 4;     // resident B landed (tx)
  uint64_t* bdone = bars + 2 * kStages + 5;     // MMAs reading the resident B completed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 6);
  int* tkeys = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(bars) + kRowBars);  // [2][128] (P::kSeg)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t acc_cols = Nt <= 32 ? 32 : (Nt <= 64 ? 64 : (Nt <= 128 ? 128 : 256));
  constexpr int kProdThreads = kProdWarps * 32;
  const uint32_t crank = kPair ? cl_rank() : 0;
  const bool leader = crank == 0;
  if (warp == kMmaWarp) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(2 * acc_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      tmem_alloc(tmem_slot, 2 * acc_cols);
    }
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kPair ? 2 * kProdWarps : kProdThreads);  // (pair: one arrival per warp of each CTA)
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accfull[b], 1);
      mbar_init(&accempty[b], kPair ? 2 * kEpiWarps : kEpiWarps * 32);
    }
    mbar_init(bfull, kPair && leader ? 2 : 1);  // (pair leader: + the peer's forwarded completion)
    mbar_init(bdone, 1);
    fence_mbar_init();
  }
  const uint32_t b_slice = uint32_t(kPair ? Nt / 2 : Nt) * 128;  // bytes of one (chunk, hi|lo) B slice
  const int nchunks = p.K / KC;
  tc_fence_before();
  if constexpr (kPair) cl_sync();  // both CTAs' barriers exist before any remote arrival
  else __syncthreads();
  tc_fence_after();
  // this CTA's arrival on a barrier the pair leader waits on (pair: one elected lane per warp)
  auto arrive_lead = [&](uint64_t* bar) {
    if constexpr (kPair) {
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(bar);
        else mbar_arrive_rank(bar, 0);
      }
    } else {
      mbar_arrive(bar);
    }
  };
  const uint32_t tmem = *tmem_slot;
  // ablation bits read once: a global load per chunk sat on the producer's critical path
  const int dbg = g_tc_debug;
  if constexpr (RowPf<P>::value && !kPair) {  // the first tile's rows of a plain row range, streamed into L2
    // while the previous kernel drains (inputs written long before it: safe before pdl_wait);
    // the producer prefetches each next tile as it starts one (below)
    if (plan.prefetch && tid == kRowThreads - 1 && !p.rows.perm && !p.rows.seg_off) {
      const int cnt = *p.rows.count, ntn = p.Ncols / Nt;
      const int tot = (cnt + 127) / 128 * ntn;
      const int tb = int((long long)blockIdx.x * tot / gridDim.x), te = int((long long)(blockIdx.x + 1) * tot / gridDim.x);
      const int r0 = (tb / ntn) * 128;
      if (te > tb && r0 < cnt) p.prefetch_rows(r0, r0 + 128 < cnt ? r0 + 128 : cnt);
    }
  }
  pdl_wait();  // setup above overlaps the previous kernel's tail
  // first m-tile of every head segment, in shared memory: a dynamically indexed
  // per-thread array lands in local memory, whose misses go to L2 (the L1 left
  // next to ~227 KB of shared memory is tiny)
  int* mt_seg = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(bars) + 128);  // [kMaxSlots + 1]
  if (tid == 0) {
    int acc = 0;
    for (int s = 0; s < p.rows.nseg; ++s) {
      mt_seg[s] = acc;
      acc += (p.rows.end(s) - p.rows.begin(s) + 127) / 128;
    }
    mt_seg[p.rows.nseg] = acc;
  }
  __syncthreads();
  const int total_m = mt_seg[p.rows.nseg];
  const int ntn = p.Ncols / Nt;
  const int total = kPair ? (total_m + 1) / 2 : total_m * ntn;  // (pair: pair-tiles)
  // contiguous tile range per CTA: consecutive tiles share a head segment / column block,
  // so the resident B image is reloaded only at segment boundaries
  const int units = kPair ? int(gridDim.x) / 2 : int(gridDim.x), unit = kPair ? int(blockIdx.x) / 2 : int(blockIdx.x);
  const int t_beg = int((long long)unit * total / units);
  const int t_end = int((long long)(unit + 1) * total / units);
  // this CTA's m-tile of tile t (pair: m-tile 2t + rank of the single segment)
  auto m_of = [&](int t) { return kPair ? 2 * t + int(crank) : t / ntn; };
  auto seg_of = [&](int tm) {
    int seg = 0;
    if constexpr (!kPair)
      while (tm >= mt_seg[seg + 1]) ++seg;
    return seg;
  };

  if (warp < kProdWarps) {  // ------------------------------------- producers
    // 4 lanes per row, each lane two k-groups (32 contiguous bytes of the row):
    // 8 consecutive rows per store instruction -> all 8 16B bank groups, no conflicts
    const int kq = lane & 3, rsub = lane >> 2;
    struct Cur {
      int t, c, seg, n0;
      int rows[kRowIt];
      typename P::RC rc[kRowIt];
    };
    auto set_tile = [&](Cur& u) {
      if (u.t >= t_end) return;
      const int tm = m_of(u.t);
      u.n0 = kPair ? 0 : (u.t % ntn) * Nt;
      const int seg = seg_of(tm);
      u.seg = seg;
      if constexpr (RowPf<P>::value && !kPair) {  // the next tile's row streams into L2, one tile ahead
        if (plan.prefetch && tid == 0 && !p.rows.perm && !p.rows.seg_off && u.t + 1 < t_end && (u.t + 1) / ntn != tm) {
          const int r0 = (tm + 1) * 128, cnt = p.rows.end(0);
          if (r0 < cnt) p.prefetch_rows(r0, r0 + 128 < cnt ? r0 + 128 : cnt);
        }
      }
#pragma unroll
      for (int it = 0; it < kRowIt; ++it) {  // rows warp*8*kRowIt + it*8 + rsub
        const int v = p.rows.begin(seg) + (tm - mt_seg[seg]) * 128 + warp * 8 * kRowIt + it * 8 + rsub;
        u.rows[it] = v < p.rows.end(seg) ? p.rows.row(v) : -1;
        if (u.rows[it] >= 0) u.rc[it] = p.rctx(seg, u.rows[it]);
      }
    };
    auto succ = [&](Cur& u) {
      if (u.t >= t_end) return;
      if (++u.c == nchunks) {
        u.c = 0;
        u.t += 1;
        set_tile(u);
      }
    };
    if constexpr (RowAsync<P>::value) {
      // Two-operand gather producer without register staging (P::kAsync): every
      // thread cp.asyncs the two 16 B source pieces of each of its (row, k4) slots of
      // a chunk straight into the stage's hi / lo tiles at the slot's SW128 position;
      // one chunk later (the next chunk's copies in flight) it converts its own slots
      // in place: v = p.combine(a, b) (+ the problem's side stores), tf32 hi -> hi
      // tile, lo -> lo tile.  No registers hold loads in flight, so the 17-warp CTA's
      // 96-register cap no longer forces spills on gathered operands.
      auto slot_off = [&](int it, int h) { return sw128(warp * 8 * kRowIt + it * 8 + rsub, 2 * kq + h); };
      auto issue = [&](const Cur& u, int st) {
        const uint32_t hi = smem_u32(stages + st * SB), lo = hi + 128 * KC * 4;
#pragma unroll
        for (int it = 0; it < kRowIt; ++it)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = u.c * KC + 8 * kq + 4 * h;
            const bool ok = u.rows[it] >= 0;
            const uint32_t o = slot_off(it, h);
            cp_async16(hi + o, ok ? p.src_a(u.seg, u.rows[it], u.rc[it], k) : p.bimg, ok ? 16u : 0u);
            cp_async16(lo + o, ok ? p.src_b(u.seg, u.rows[it], u.rc[it], k) : p.bimg, ok ? 16u : 0u);
          }
        cp_async_commit();
      };
      auto convert = [&](const Cur& u, int st) {
        uint8_t* hi = stages + st * SB;
        uint8_t* lo = hi + 128 * KC * 4;
#pragma unroll
        for (int it = 0; it < kRowIt; ++it)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t o = slot_off(it, h);
            float4* ph = reinterpret_cast<float4*>(hi + o);
            float4* pl = reinterpret_cast<float4*>(lo + o);
            const float4 v = u.rows[it] >= 0 ? p.combine(u.seg, u.rows[it], u.rc[it], u.c * KC + 8 * kq + 4 * h, *ph, *pl)
                                             : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 vh = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
            *ph = vh;
            *pl = make_float4(v.x - vh.x, v.y - vh.y, v.z - vh.z, v.w - vh.w);
          }
        fence_proxy_async();
        if (!plan.resident && tid == 0) {  // this stage's B slice rides on the same barrier
          mbar_expect_tx(&full[st], 2 * b_slice);
          const float* bsrc = p.bimg + u.seg * p.bimg_seg;
          for (int part = 0; part < 2; ++part)
            bulk_g2s(lo + 128 * KC * 4 + part * b_slice,
                     bsrc + (size_t(u.c) * 2 + part) * p.Ncols * KC + size_t(u.n0) * KC, b_slice, &full[st]);
        } else {
          arrive_lead(&full[st]);
        }
      };
      Cur prev;
      prev.t = t_beg;
      prev.c = 0;
      set_tile(prev);
      if (prev.t < t_end) {
        mbar_wait(&empty[0], 1);
        issue(prev, 0);
      }
      for (int i = 1; prev.t < t_end; ++i) {  // chunk i issued, chunk i - 1 converted
        Cur nxt = prev;
        succ(nxt);
        if (nxt.t < t_end) {
          mbar_wait(&empty[i % kStages], ((i / kStages) & 1) ^ 1);
          issue(nxt, i % kStages);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        convert(prev, (i - 1) % kStages);
        prev = nxt;
      }
    } else {
    using Raw = typename P::Raw;  // raw A loads of a chunk; P::fin4 turns them into A values
    auto load = [&](const Cur& u, Raw (&x)[kRowIt][2]) {
      const bool skip = dbg & 1;
#pragma unroll
      for (int it = 0; it < kRowIt; ++it)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (u.rows[it] >= 0 && !skip) x[it][h] = p.raw4(u.seg, u.rows[it], u.rc[it], u.c * KC + 8 * kq + 4 * h);
    };
    int stage = 0;
    uint32_t phase = 0;
    auto fill = [&](const Cur& u, const Raw (&x)[kRowIt][2]) {
      float4 v[kRowIt][2];
#pragma unroll
      for (int it = 0; it < kRowIt; ++it)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          v[it][h] = (u.rows[it] >= 0 && !(dbg & 1))
                         ? p.fin4(u.seg, u.rows[it], u.rc[it], u.c * KC + 8 * kq + 4 * h, x[it][h])
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      mbar_wait(&empty[stage], phase ^ 1);
      float* a_hi = reinterpret_cast<float*>(stages + stage * SB);
      float* a_lo = a_hi + 128 * KC;
      if (!(dbg & 1))
#pragma unroll
        for (int it = 0; it < kRowIt; ++it)
#pragma unroll
          for (int h = 0; h < 2; ++h) put4(a_hi, a_lo, 2 * kq + h, warp * 8 * kRowIt + it * 8 + rsub, v[it][h]);
      fence_proxy_async();
      if (!plan.resident && tid == 0) {  // this stage's B slice rides on the same barrier
        mbar_expect_tx(&full[stage], 2 * b_slice);
        const float* bsrc = p.bimg + u.seg * p.bimg_seg;
        for (int part = 0; part < 2; ++part)
          bulk_g2s(reinterpret_cast<uint8_t*>(a_lo + 128 * KC) + part * b_slice,
                   bsrc + (size_t(u.c) * 2 + part) * p.Ncols * KC + size_t(u.n0) * KC, b_slice, &full[stage]);
      } else {
        arrive_lead(&full[stage]);
      }
      if (++stage == kStages) stage = 0, phase ^= 1;
    };
    Cur A, B;
    A.t = t_beg;
    A.c = 0;
    set_tile(A);
    B = A;
    succ(B);
    Raw xa[kRowIt][2], xb[kRowIt][2];
    if (A.t < t_end) load(A, xa);
    if (B.t < t_end) load(B, xb);
    while (A.t < t_end) {  // two chunks in registers: one being stored, the next in flight
      fill(A, xa);
      A = B;
      succ(A);
      if (A.t < t_end) load(A, xa);
      if (B.t >= t_end) break;
      fill(B, xb);
      B = A;
      succ(B);
      if (B.t < t_end) load(B, xb);
    }
    }
  } else if (kPair && warp == kMmaWarp) {  // ------------------- pair: resident B half + MMA issue (leader)
    // this CTA's column half of the single resident B image, once
    if (t_beg < t_end) {
      if (lane == 0) {
        mbar_expect_tx(bfull, uint32_t(nchunks) * 2 * b_slice);
        for (int c = 0; c < nchunks; ++c)
          for (int part = 0; part < 2; ++part)
            bulk_g2s(reinterpret_cast<uint8_t*>(bres) + (size_t(c) * 2 + part) * b_slice,
                     p.bimg + (size_t(c) * 2 + part) * p.Ncols * KC + size_t(crank) * (Nt / 2) * KC, b_slice, bfull);
      }
      __syncwarp();
      if (!leader) {  // the leader's MMAs read our half: forward its arrival
        mbar_wait(bfull, 0);
        if (lane == 0) mbar_arrive_rank(bfull, 0);
      } else {
        mbar_wait_cl(bfull, 0);
        tc_fence_after();
        int stage = 0;
        uint32_t phase = 0;
        int ab = 0;
        uint32_t aphase = 0;
        const uint32_t idesc = (idesc_tf32(Nt) & ~(31u << 24)) | (uint32_t(256 >> 4) << 24);
        for (int t = t_beg; t < t_end; ++t) {
          mbar_wait_cl(&accempty[ab], aphase ^ 1);
          tc_fence_after();
          for (int c = 0; c < nchunks; ++c) {
            mbar_wait_cl(&full[stage], phase);
            tc_fence_after();
            const uint32_t a_hi = smem_u32(stages + stage * SB), a_lo = a_hi + 128 * KC * 4;
            const uint32_t b_hi = smem_u32(bres) + uint32_t(c) * 2 * b_slice, b_lo = b_hi + b_slice;
            issue_chunk_pair(tmem + ab * acc_cols, a_hi, a_lo, b_hi, b_lo, idesc, c != 0);
            commit_pair(&empty[stage]);
            if (c == nchunks - 1) commit_pair(&accfull[ab]);
            __syncwarp();
            if (++stage == kStages) stage = 0, phase ^= 1;
          }
          if (++ab == 2) ab = 0, aphase ^= 1;
        }
      }
    }
  } else if (warp == kMmaWarp) {  // --------------------------------- MMA issuer + resident B
    int stage = 0;
    uint32_t phase = 0, bphase = 0, dphase = 0;
    int ab = 0;
    uint32_t aphase = 0;
    int res_key = -1;
    const uint32_t idesc = idesc_tf32(Nt);
    for (int t = t_beg; t < t_end; ++t) {
      if (plan.resident) {
        const int tm = t / ntn, n0 = (t % ntn) * Nt;
        int seg = 0;
        while (tm >= mt_seg[seg + 1]) ++seg;
        const int key = seg * 4096 + n0;
        if (key != res_key) {
          if (res_key >= 0) {  // every MMA that reads the old image must have completed
            commit_warp(bdone);
            __syncwarp();
            mbar_wait(bdone, dphase);
            dphase ^= 1;
          }
          if (lane == 0) {
            mbar_expect_tx(bfull, uint32_t(nchunks) * 2 * b_slice);
            const float* bsrc = p.bimg + seg * p.bimg_seg;
            for (int c = 0; c < nchunks; ++c)
              for (int part = 0; part < 2; ++part)
                bulk_g2s(reinterpret_cast<uint8_t*>(bres) + (size_t(c) * 2 + part) * b_slice,
                         bsrc + (size_t(c) * 2 + part) * p.Ncols * KC + size_t(n0) * KC, b_slice, bfull);
          }
          __syncwarp();
          mbar_wait(bfull, bphase);
          bphase ^= 1;
          res_key = key;
        }
      }
      mbar_wait(&accempty[ab], aphase ^ 1);
      tc_fence_after();
      for (int c = 0; c < nchunks; ++c) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        {
          const uint32_t a_hi = smem_u32(stages + stage * SB), a_lo = a_hi + 128 * KC * 4;
          const uint32_t b_hi = plan.resident ? smem_u32(bres) + uint32_t(c) * 2 * KC * Nt * 4 : a_lo + 128 * KC * 4;
          const uint32_t b_lo = b_hi + Nt * KC * 4;
          issue_chunk_warp(tmem + ab * acc_cols, a_hi, a_lo, b_hi, b_lo, idesc, c != 0);
          commit_warp(&empty[stage]);
          if (c == nchunks - 1) commit_warp(&accfull[ab]);
        }
        __syncwarp();
        if (++stage == kStages) stage = 0, phase ^= 1;
      }
      if (++ab == 2) ab = 0, aphase ^= 1;
    }
  } else {  // ------------------------------------------------------- epilogue
    const int q = warp & 3;                 // TMEM lane quadrant this warp may access
    const int half = (warp - kEpiWarp0) >> 2;  // which alternate 32-column slabs
    int ab = 0;
    uint32_t aphase = 0;
    float* slab = epi_smem + (warp - kEpiWarp0) * 32 * 32;  // 32 rows x 32 cols, 16 B chunks XOR-swizzled
    const int nslab = (Nt + 31) / 32;
    for (int t = t_beg; t < t_end; ++t) {
      const int tm = m_of(t), n0 = kPair ? 0 : (t % ntn) * Nt;
      const int seg = seg_of(tm);
      if constexpr (!RowSlab<P>::value) {
        {  // ---- register-fragment epilogue (no shared memory; plan.epi_bytes == 0)
          // .16x256b reads of this quadrant's two 16-lane halves; lane pairs (l, l^1) swap
          // halves of their 8-column groups so lane l owns row 16h + l/4 + 8(l&1) of the
          // quadrant, columns 8jj + 4((l>>1)&1) .. +3: the same float4 epi4 calls as the
          // slab path (bit-identical), full 32 B sectors per store instruction
          const int fr = (lane >> 2) + 8 * (lane & 1), fc = 4 * ((lane >> 1) & 1);
          const bool odd = lane & 1;
          int frow[2];
          typename P::RC frc[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int v = p.rows.begin(seg) + (tm - mt_seg[seg]) * 128 + q * 32 + 16 * h + fr;
            frow[h] = v < p.rows.end(seg) ? p.rows.row(v) : -1;
            if (frow[h] >= 0) frc[h] = p.rctx(seg, frow[h]);
          }
          typename P::Aux fa[2][4];
          auto load_aux = [&](int j) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int jj = 0; jj < 4; ++jj)
                if (frow[h] >= 0) fa[h][jj] = p.epi_aux(seg, frow[h], frc[h], n0 + j + 8 * jj + fc);
          };
          if (half < nslab) load_aux(half * 32);
          mbar_wait(&accfull[ab], aphase);
          tc_fence_after();
          for (int sl = half; sl < nslab; sl += kEpiHalves) {
            const int j = sl * 32;
            if (sl != half) load_aux(j);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              float v[16];
              tmem_ld16x32(tmem + ab * acc_cols + (uint32_t(q * 32 + 16 * h) << 16) + j, v);
              tmem_wait_ld();
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const float s0 = odd ? v[4 * jj] : v[4 * jj + 2], s1 = odd ? v[4 * jj + 1] : v[4 * jj + 3];
                const float r0 = __shfl_xor_sync(0xffffffffu, s0, 1), r1 = __shfl_xor_sync(0xffffffffu, s1, 1);
                const float4 a = odd ? make_float4(r0, r1, v[4 * jj + 2], v[4 * jj + 3])
                                     : make_float4(v[4 * jj], v[4 * jj + 1], r0, r1);
                if (frow[h] >= 0 && !(dbg & 2)) p.epi4(seg, frow[h], frc[h], n0 + j + 8 * jj + fc, a, fa[h][jj]);
              }
            }
          }
          tc_fence_before();
          arrive_lead(&accempty[ab]);
          if (++ab == 2) ab = 0, aphase ^= 1;
          continue;
        }
      }
      if constexpr (RowSlab<P>::value) {  // ---- slab epilogue
      int rows_it[8];
      typename P::RC rc[8];
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int v = p.rows.begin(seg) + (tm - mt_seg[seg]) * 128 + q * 32 + it * 4 + (lane >> 3);
        rows_it[it] = v < p.rows.end(seg) ? p.rows.row(v) : -1;
        if (rows_it[it] >= 0) rc[it] = p.rctx(seg, rows_it[it]);
      }
      // segmented sums: this quadrant's row keys and the tile's neighbours
      int tprev = -1, tnext = -1;
      if constexpr (RowSeg<P>::value) {
        const int base = p.rows.begin(seg) + (tm - mt_seg[seg]) * 128, endv = p.rows.end(seg);
        const int v = base + q * 32 + lane;
        tkeys[half * 128 + q * 32 + lane] = v < endv ? p.seg_key(p.rows.row(v)) : -1;
        tprev = base > p.rows.begin(seg) ? p.seg_key(p.rows.row(base - 1)) : -1;
        tnext = base + 128 < endv ? p.seg_key(p.rows.row(base + 128)) : -1;
      }
      // epilogue operands that do not depend on the accumulator (residuals, saved
      // activations): the first slab's are loaded before waiting for the MMAs, later
      // slabs' are issued ahead of their TMEM load and transpose
      typename P::Aux aux[8];
      const int cc = lane & 7, c4 = cc * 4;
      if (half < nslab) {
#pragma unroll
        for (int it = 0; it < 8; ++it)
          if (rows_it[it] >= 0) aux[it] = p.epi_aux(seg, rows_it[it], rc[it], n0 + half * 32 + c4);
      }
      mbar_wait(&accfull[ab], aphase);
      tc_fence_after();
      for (int sl = half; sl < nslab; sl += kEpiHalves) {
        const int j = sl * 32;
        if (sl != half) {
#pragma unroll
          for (int it = 0; it < 8; ++it)
            if (rows_it[it] >= 0) aux[it] = p.epi_aux(seg, rows_it[it], rc[it], n0 + j + c4);
        }
        float acc[32];
        tmem_ld32(tmem + ab * acc_cols + (uint32_t(q * 32) << 16) + j, acc);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4*>(slab + lane * 32 + ((i ^ (lane & 7)) << 2)) =
              make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int rl = it * 4 + (lane >> 3);
          float4* sp = reinterpret_cast<float4*>(slab + rl * 32 + ((cc ^ (rl & 7)) << 2));
          const float4 a = *sp;
          if constexpr (RowSeg<P>::value) {  // store C; the reduced value replaces the accumulator in the slab
            *sp = rows_it[it] >= 0 ? p.epi4r(seg, rows_it[it], rc[it], n0 + j + c4, a, aux[it])
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            if (rows_it[it] >= 0 && !(dbg & 2)) p.epi4(seg, rows_it[it], rc[it], n0 + j + c4, a, aux[it]);
          }
        }
        if constexpr (RowSeg<P>::value) {
          if (dbg & 4) continue;  // (ablation: no segmented sums)
          // the 4 quadrant slabs of these 32 columns (this half's warps) now hold the
          // reduced values of all 128 rows: lane = column, rows summed in ascending order;
          // a key whose rows continue past the quadrant is finished by the quadrant where
          // it starts (reading the following quadrants' slabs)
          __syncwarp();
          named_bar(1 + half, 128);
          const int* tk = tkeys + half * 128;
          auto colv = [&](int qq, int r) {
            const float* sb = epi_smem + (half * 4 + ((qq + 3) & 3)) * 32 * 32;
            return sb[r * 32 + ((((lane >> 2) ^ (r & 7))) << 2) + (lane & 3)];
          };
          const int col = n0 + j + lane, tile = tm - mt_seg[seg];
          int cur = tk[q * 32];
          bool head = q == 0 && tprev == cur;  // the key started in an earlier tile: this tile's head piece
          bool owned = head || (q == 0 ? tprev : tk[q * 32 - 1]) != cur;
          float sum = 0.f;
          for (int r = 0; r < 32; ++r) {
            const int k = tk[q * 32 + r];
            if (k != cur) {
              if (owned && cur >= 0) {
                if (head) p.tile_store(0, tile, col, sum);
                else p.seg_store(cur, col, sum);
              }
              sum = 0.f, cur = k, owned = true, head = false;
            }
            sum += colv(q, r);
          }
          if (owned && cur >= 0) {
            bool done = false;
            for (int qq = q + 1; qq < 4 && !done; ++qq)
              for (int r = 0; r < 32; ++r) {
                if (tk[qq * 32 + r] != cur) {
                  done = true;
                  break;
                }
                sum += colv(qq, r);
              }
            if (!done) done = tnext != cur;  // reached the tile end: complete unless the key continues
            if (head) p.tile_store(0, tile, col, sum);
            else if (done) p.seg_store(cur, col, sum);
            else p.tile_store(1, tile, col, sum);
          }
          named_bar(1 + half, 128);  // every quadrant's slab read: free for the next 32 columns
        }
      }
      tc_fence_before();
      arrive_lead(&accempty[ab]);
      if (++ab == 2) ab = 0, aphase ^= 1;
      }
    }
  }
  tc_fence_before();
  if constexpr (kPair) {  // the leader's MMAs read both CTAs' shared memory: nobody leaves early
    cl_sync();
    if (warp == kMmaWarp)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * acc_cols));
  } else {
    __syncthreads();
    if (warp == kMmaWarp) tmem_dealloc(tmem, 2 * acc_cols);
  }
}

// ================================================================ reduce GEMM
// Weight gradients C_seg[m, n] = sum over rows r of segment seg of X(r, m) Y(r, n)
// with X, Y ROW-MAJOR per row (features contiguous).  K-chunk = 32 rows.  A
// producer lane loads a 4-row x 4-feature block (4 coalesced float4 row
// segments), transposes it in registers, and stores 4 k-values per feature
// into the K-major SWIZZLE_NONE layout (lane-rotated store order ->
// conflict-free).  CTA (mtile, split, seg) owns chunks split, split+nsplit, ...
// (static -> the fixed-order reduce is deterministic).  Warps 0-3 produce
// (warp w = rows 8w..8w+7 of the chunk), warp 4 issues MMAs; the producers run
// the epilogue.  If p.colsum, m-tile 0 also accumulates sum_rows Y(r, n).
// P must provide: RowSet rows; int M, Ncols, colsum;
//   float4 x4(int seg, int row, int m) const;  float4 y4(int seg, int row, int n) const;
// Output partial: [seg][split][Ncols][M + colsum] (transposed: coalesced stores).
constexpr int kRedProd = 8;                      // producer warps (warp w = k-group w of a chunk)
constexpr int kRedThreads = (kRedProd + 1) * 32;  // + 1 MMA warp
__host__ __device__ inline size_t red_stage_bytes(int N) { return size_t(2 * 128 * KC + 2 * N * KC) * 4; }
constexpr size_t kRedCsum = size_t(kRedProd) * 256 * 4;
inline int red_stages(int N) {
  int s = int((kSmemLimit - 2048 - 1024 - kRedCsum) / red_stage_bytes(N));
  return s < 2 ? 2 : (s > kMaxStages ? kMaxStages : s);
}
inline size_t tc_red_smem(int N) { return red_stages(N) * red_stage_bytes(N) + kRedCsum + 2048 + 1024; }

__device__ __forceinline__ float4 col4(const float4* v, int j) {  // column j of a 4x4 block
  return j == 0 ? make_float4(v[0].x, v[1].x, v[2].x, v[3].x)
       : j == 1 ? make_float4(v[0].y, v[1].y, v[2].y, v[3].y)
       : j == 2 ? make_float4(v[0].z, v[1].z, v[2].z, v[3].z)
                : make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
}

template <class P>
__global__ void __launch_bounds__(kRedThreads, 1) tc_red_kernel(P p, float* __restrict__ partial, int nsplit,
                                                                int kStages) {
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  uint8_t* smem_raw = align1k(smem_dyn);
  const int N = p.Ncols;
  const size_t SB = red_stage_bytes(N);
  float* csum_smem = reinterpret_cast<float*>(smem_raw + kStages * SB);  // [kRedProd][N]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + kStages * SB + kRedCsum);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* accfull = bars + 2 * kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mtile = blockIdx.x, split = blockIdx.y, seg = blockIdx.z;
  const uint32_t acc_cols = N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : 256));
  constexpr int kProdThreads = kRedProd * 32;
  if (warp == kRedProd) tmem_alloc(tmem_slot, acc_cols);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kProdThreads);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&accfull[0], 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // setup above overlaps the previous kernel's tail
  const int rb = p.rows.begin(seg), re = p.rows.end(seg);
  const int nchunks = (re - rb + KC - 1) / KC;
  int my_chunks = 0;
  for (int c = split; c < nchunks; c += nsplit) ++my_chunks;
  const int Mo = p.M + (p.colsum ? 1 : 0);
  float* out = partial + (size_t(seg) * nsplit + split) * size_t(Mo) * N;
  const bool clustered = cl_size() > 1;  // (launched as split clusters: partials reduced in the cluster)
  float* T = reinterpret_cast<float*>(smem_raw);  // [N][kRedTS] accumulator staging (stage memory, free by then)
  const int m0 = mtile * 128;
  const int Mt = p.M - m0 < 128 ? p.M - m0 : 128;  // features of this m-tile (mult of 4)
  const bool do_colsum = p.colsum && mtile == 0;

  if (warp < kRedProd) {
    float4 cs[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
    int stage = 0;
    uint32_t phase = 0;
    const int f = lane * 4;
    // register double buffer: chunk c+nsplit's loads are in flight while chunk c
    // is transposed into shared memory
    auto load = [&](int c, float4 (&xa)[4], float4 (&yb)[2][4]) {
      const int vj = rb + c * KC + warp * 4 + (lane & 3);  // this warp's 4 rows (k-group `warp`)
      const int rj = (c < nchunks && vj < re) ? p.rows.row(vj) : -1;
      int rows[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) rows[j] = __shfl_sync(0xffffffffu, rj, j);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        xa[j] = (rows[j] >= 0 && f < Mt) ? p.x4(seg, rows[j], m0 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int n = f + 128 * u;
          yb[u][j] = (rows[j] >= 0 && n < N) ? p.y4(seg, rows[j], n) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    };
    float4 xa[4], yb[2][4], xn[4], yn[2][4];
    if (split < nchunks) load(split, xa, yb);
    for (int c = split; c < nchunks; c += nsplit) {
      if (c + nsplit < nchunks) load(c + nsplit, xn, yn);
      if (do_colsum)
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            cs[u] = make_float4(cs[u].x + yb[u][j].x, cs[u].y + yb[u][j].y, cs[u].z + yb[u][j].z,
                                cs[u].w + yb[u][j].w);
      mbar_wait(&empty[stage], phase ^ 1);
      float* a_hi = reinterpret_cast<float*>(smem_raw + stage * SB);
      float* a_lo = a_hi + 128 * KC;
      float* b_hi = a_lo + 128 * KC;
      float* b_lo = b_hi + N * KC;
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // feature rows f+jj, k-chunk `warp` (rows 4w..4w+3 of the chunk)
        const int jj = (i + lane) & 3;
        put4(a_hi, a_lo, warp, f + jj, col4(xa, jj));
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (f + 128 * u < N) put4(b_hi, b_lo, warp, f + 128 * u + jj, col4(yb[u], jj));
      }
      fence_proxy_async();
      mbar_arrive(&full[stage]);
      if (++stage == kStages) stage = 0, phase ^= 1;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        xa[j] = xn[j];
        yb[0][j] = yn[0][j];
        yb[1][j] = yn[1][j];
      }
    }
    if (do_colsum) {  // per-warp partial column sums -> fixed-order combine below
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (f + 128 * u < N) *reinterpret_cast<float4*>(csum_smem + warp * N + f + 128 * u) = cs[u];
    }
    // epilogue: warp w reads TMEM lanes 32*(w%4) (features), column half w/4;
    // the partial is stored transposed ([n][m]) so stores are coalesced
    if (my_chunks > 0) {
      mbar_wait(&accfull[0], 0);
      tc_fence_after();
    }
    const int q = warp & 3, half = warp >> 2;
    const int nh = ((N / 32) + 1) / 2 * 32;  // columns of half 0
    const int nb = half ? nh : 0, ne = half ? N : nh;
    const int mloc = q * 32 + lane;
    for (int n0 = nb; n0 < ne; n0 += 32) {
      float acc[32];
      __syncwarp();
      tmem_ld32(tmem + (uint32_t(q * 32) << 16) + n0, acc);
      if (mloc < Mt) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (n0 + i < N) {
            const float v = my_chunks ? acc[i] : 0.f;
            if (clustered) T[(n0 + i) * kRedTS + mloc] = v;
            else out[size_t(n0 + i) * Mo + m0 + mloc] = v;
          }
      }
    }
    if (do_colsum) {
      asm volatile("bar.sync 1, %0;" ::"r"(kProdThreads) : "memory");
      for (int n = tid; n < N; n += kProdThreads) {
        float v = 0.f;
        for (int w = 0; w < kRedProd; ++w) v += csum_smem[w * N + n];
        if (clustered) T[n * kRedTS + kRedTS - 1] = v;
        else out[size_t(n) * Mo + p.M] = v;
      }
    }
  } else {  // MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t idesc = idesc_tf32(N);
    int i = 0;
    for (int c = split; c < nchunks; c += nsplit, ++i) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      if (lane == 0) {
        float* a_hi = reinterpret_cast<float*>(smem_raw + stage * SB);
        float* a_lo = a_hi + 128 * KC;
        float* b_hi = a_lo + 128 * KC;
        float* b_lo = b_hi + N * KC;
        issue_chunk(tmem, a_hi, a_lo, b_hi, b_lo, idesc, i == 0);
        mma_commit(&empty[stage]);
        if (i == my_chunks - 1) mma_commit(&accfull[0]);
      }
      __syncwarp();
      if (++stage == kStages) stage = 0, phase ^= 1;
    }
  }
  tc_fence_before();
  if (clustered) {
    cl_sync();  // every CTA's accumulator tile staged
    red_cluster_reduce(T, partial, seg, split, nsplit, N, Mo, m0, Mt, p.M, do_colsum, tid, blockDim.x);
    cl_sync();  // peers done reading this CTA's tile
  } else {
    __syncthreads();
  }
  if (warp == kRedProd) tmem_dealloc(tmem, acc_cols);
}

// partial is [seg][split][n][Mo] (transposed); store C[m][n]
template <class P>
struct RedStore {
  P p;
  int nsplit, Mo;
  __device__ int count(int) const { return nsplit; }
  __device__ void store(int seg, int t, float v) const { p.store(seg, t % Mo, t / Mo, v); }
};
template <class P>
inline void tc_red_reduce(const P& p, const float* partial, int nsplit, cudaStream_t st) {
  const int Mo = p.M + (p.colsum ? 1 : 0);
  const size_t KN = size_t(Mo) * p.Ncols;
  dim3 grid(unsigned((KN + 31) / 32), p.rows.nseg);
  kl(split_reduce_kernel<RedStore<P>>, grid, 256, 0, st, partial, nsplit * KN, KN, int(KN), RedStore<P>{p, nsplit, Mo});
}

// ================================================================ reduce GEMM, TMA operands
// Same contract as tc_red_kernel for problems whose X and Y are plain row-major
// matrices over contiguous rows (identity RowSet): TMA brings each 32-row chunk
// in as 32-feature x 32-row boxes swizzled in 32 B atoms -- exactly the
// MN-major 128B_BASE32B canonical layout tcgen05 takes for tf32 (LBO = 4 KB
// between 32-feature atoms, SBO = 512 B between 4-row groups), so neither
// operand is transposed in registers.
// Converter warps 0-7 then split each 16 B in place (raw -> tf32 hi, lo to the
// lo tile at the same offset; rows past the segment end are zeroed; P::xfin /
// P::yfin apply an elementwise transform such as silu), warp 8 issues the
// 3xTF32 MMAs with A and B MN-major, warp 9 lane 0 keeps kStages chunks of TMA
// loads in flight.  Deterministic: same chunk order and colsum order always.
constexpr int kRedTmaThreads = (kRedProd + 2) * 32;
// MN-major tf32 operands take the 128B_BASE32B layout (32 B granules of each
// 128 B row XOR-swizzled by row % 4; atom = 4 rows x 128 B): LBO = 4 KB between
// 32-feature boxes, SBO = 512 B between 4-row groups, layout type 1
__device__ __forceinline__ uint64_t sdesc_sw128_mn(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(4096 >> 4) << 16) | (uint64_t(512 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(1) << 61);
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// 2-D tensor map over a row-major [rows x ld] fp32 matrix: 32 x 32 boxes, 128 B span
// swizzled in 32 B atoms (the MN-major tf32 operand layout)
inline bool tmap_2d(CUtensorMap* m, const float* base, long long rows, int ld,
                    CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, int box_rows = 32) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 4) % 16) return false;
  cuuint64_t dims[2] = {cuuint64_t(ld), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
  cuuint32_t box[2] = {32, cuuint32_t(box_rows)}, es[2] = {1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
inline size_t tc_red_tma_smem(int N, int stages) {
  return size_t(stages) * red_stage_bytes(N) + size_t(32) * N * 4 + 2048 + 1024;
}

template <class P>
__global__ void __launch_bounds__(kRedTmaThreads, 1)
    tc_red_tma_kernel(P p, const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap tx1,
                      const __grid_constant__ CUtensorMap ty, int xsplit, float* __restrict__ partial, int nsplit,
                      int kStages) {
  extern __shared__ __align__(1024) uint8_t smem_dyn[];
  uint8_t* smem_raw = align1k(smem_dyn);
  const int N = p.Ncols;
  const size_t SB = red_stage_bytes(N);
  float* csum_smem = reinterpret_cast<float*>(smem_raw + kStages * SB);  // [32 rows][N]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + kStages * SB + size_t(32) * N * 4);
  uint64_t* tfull = bars;                // TMA bytes landed
  uint64_t* cfull = bars + kStages;      // converted (hi/lo) -> MMA
  uint64_t* empty = bars + 2 * kStages;  // MMAs done -> TMA may refill
  uint64_t* accfull = bars + 3 * kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kStages + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mtile = blockIdx.x, split = blockIdx.y, seg = blockIdx.z;
  const uint32_t acc_cols = N <= 32 ? 32 : (N <= 64 ? 64 : (N <= 128 ? 128 : 256));
  constexpr int kProdThreads = kRedProd * 32;
  if (warp == kRedProd) tmem_alloc(tmem_slot, acc_cols);
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&cfull[s], kProdThreads);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&accfull[0], 1);
    fence_mbar_init();
  }
  if (warp == kRedProd + 1 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tx) : "memory");
    if (xsplit) asm volatile("prefetch.tensormap [%0];" ::"l"(&tx1) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&ty) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  const int rb = p.rows.begin(seg), re = p.rows.end(seg);
  const int nchunks = (re - rb + KC - 1) / KC;
  int my_chunks = 0;
  for (int c = split; c < nchunks; c += nsplit) ++my_chunks;
  const int Mo = p.M + (p.colsum ? 1 : 0);
  float* out = partial + (size_t(seg) * nsplit + split) * size_t(Mo) * N;
  const bool clustered = cl_size() > 1;  // (launched as split clusters: partials reduced in the cluster)
  float* T = reinterpret_cast<float*>(smem_raw);  // [N][kRedTS] accumulator staging (stage memory, free by then)
  const int m0 = mtile * 128;
  const int Mt = p.M - m0 < 128 ? p.M - m0 : 128;
  const int nxb = (Mt + 31) / 32, nyb = N / 32;  // 32-feature boxes per chunk
  const bool do_colsum = p.colsum && mtile == 0;

  if (warp == kRedProd + 1) {  // ------------------------------------ TMA
    if (lane == 0) {
      // X features >= xsplit (a multiple of 128) come from the second matrix
      const bool second = xsplit && m0 >= xsplit;
      const CUtensorMap* xm = second ? &tx1 : &tx;
      const int xc = second ? m0 - xsplit : m0;
      int stage = 0;
      uint32_t phase = 0;
      for (int c = split; c < nchunks; c += nsplit) {
        mbar_wait(&empty[stage], phase ^ 1);
        float* x_hi = reinterpret_cast<float*>(smem_raw + stage * SB);
        float* y_hi = x_hi + 2 * 128 * KC;
        mbar_expect_tx(&tfull[stage], uint32_t(nxb + nyb) * 32 * KC * 4);
        const int r0 = rb + c * KC;
        for (int b = 0; b < nxb; ++b) tma_2d(x_hi + b * 32 * KC, xm, xc + 32 * b, r0, &tfull[stage]);
        for (int b = 0; b < nyb; ++b) tma_2d(y_hi + b * 32 * KC, &ty, 32 * b, r0, &tfull[stage]);
        if (++stage == kStages) stage = 0, phase ^= 1;
      }
    }
  } else if (warp < kRedProd) {  // ------------------------------- convert
    // thread t owns 16 B slot t of every 4 KB box: row t/8 of the chunk; its 32 B
    // granule (t%8)/2 holds logical granule ((t%8)/2) ^ (row%4) (128B_BASE32B)
    const int row = tid >> 3, fq = (((((tid & 7) >> 1) ^ (row & 3)) << 1) | (tid & 1)) * 4;
    float4 cs[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) cs[b] = make_float4(0.f, 0.f, 0.f, 0.f);
    int stage = 0;
    uint32_t phase = 0;
    for (int c = split; c < nchunks; c += nsplit) {
      mbar_wait(&tfull[stage], phase);
      float* x_hi = reinterpret_cast<float*>(smem_raw + stage * SB);
      float* x_lo = x_hi + 128 * KC;
      float* y_hi = x_lo + 128 * KC;
      float* y_lo = y_hi + N * KC;
      const bool live = rb + c * KC + row < re;
      for (int b = 0; b < nxb; ++b) {
        float4* h = reinterpret_cast<float4*>(x_hi + b * 32 * KC) + tid;
        float4 v = live ? p.xfin(*h) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (m0 + 32 * b + fq >= p.M) v = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 hv = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        *h = hv;
        reinterpret_cast<float4*>(x_lo + b * 32 * KC)[tid] = make_float4(v.x - hv.x, v.y - hv.y, v.z - hv.z, v.w - hv.w);
      }
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        if (b < nyb) {
          float4* h = reinterpret_cast<float4*>(y_hi + b * 32 * KC) + tid;
          const float4 v = live ? p.yfin(*h) : make_float4(0.f, 0.f, 0.f, 0.f);
          if (do_colsum) cs[b] = make_float4(cs[b].x + v.x, cs[b].y + v.y, cs[b].z + v.z, cs[b].w + v.w);
          const float4 hv = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
          *h = hv;
          reinterpret_cast<float4*>(y_lo + b * 32 * KC)[tid] =
              make_float4(v.x - hv.x, v.y - hv.y, v.z - hv.z, v.w - hv.w);
        }
      }
      fence_proxy_async();
      mbar_arrive(&cfull[stage]);
      if (++stage == kStages) stage = 0, phase ^= 1;
    }
    if (do_colsum)
#pragma unroll
      for (int b = 0; b < 8; ++b)
        if (b < nyb) *reinterpret_cast<float4*>(csum_smem + row * N + 32 * b + fq) = cs[b];
    // epilogue (as tc_red_kernel): warp w reads TMEM lanes 32*(w%4), column half w/4
    if (my_chunks > 0) {
      mbar_wait(&accfull[0], 0);
      tc_fence_after();
    }
    const int q = warp & 3, half = warp >> 2;
    const int nh = ((N / 32) + 1) / 2 * 32;
    const int nb = half ? nh : 0, ne = half ? N : nh;
    const int mloc = q * 32 + lane;
    for (int n0 = nb; n0 < ne; n0 += 32) {
      float acc[32];
      __syncwarp();
      tmem_ld32(tmem + (uint32_t(q * 32) << 16) + n0, acc);
      if (mloc < Mt) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (n0 + i < N) {
            const float v = my_chunks ? acc[i] : 0.f;
            if (clustered) T[(n0 + i) * kRedTS + mloc] = v;
            else out[size_t(n0 + i) * Mo + m0 + mloc] = v;
          }
      }
    }
    if (do_colsum) {
      asm volatile("bar.sync 1, %0;" ::"r"(kProdThreads) : "memory");
      for (int n = tid; n < N; n += kProdThreads) {
        float v = 0.f;
        for (int r = 0; r < 32; ++r) v += csum_smem[r * N + n];
        if (clustered) T[n * kRedTS + kRedTS - 1] = v;
        else out[size_t(n) * Mo + p.M] = v;
      }
    }
  } else {  // -------------------------------------------------------- MMA
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t idesc = idesc_tf32(N) | (1u << 15) | (1u << 16);  // A and B MN-major
    int i = 0;
    for (int c = split; c < nchunks; c += nsplit, ++i) {
      mbar_wait(&cfull[stage], phase);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t ah = smem_u32(smem_raw + stage * SB), al = ah + 128 * KC * 4;
        const uint32_t bh = al + 128 * KC * 4, bl = bh + uint32_t(N) * KC * 4;
#pragma unroll
        for (int j = 0; j < KC / 8; ++j) {
          const uint32_t o = 1024 * j;  // rows 8j..8j+7 (two 4-row groups) of every box
          mma_tf32(tmem, sdesc_sw128_mn(al + o), sdesc_sw128_mn(bh + o), idesc, (i == 0 && j == 0) ? 0u : 1u);
          mma_tf32(tmem, sdesc_sw128_mn(ah + o), sdesc_sw128_mn(bl + o), idesc, 1u);
          mma_tf32(tmem, sdesc_sw128_mn(ah + o), sdesc_sw128_mn(bh + o), idesc, 1u);
        }
        mma_commit(&empty[stage]);
        if (i == my_chunks - 1) mma_commit(&accfull[0]);
      }
      __syncwarp();
      if (++stage == kStages) stage = 0, phase ^= 1;
    }
  }
  tc_fence_before();
  if (clustered) {
    cl_sync();  // every CTA's accumulator tile staged
    red_cluster_reduce(T, partial, seg, split, nsplit, N, Mo, m0, Mt, p.M, do_colsum, tid, blockDim.x);
    cl_sync();  // peers done reading this CTA's tile
  } else {
    __syncthreads();
  }
  if (warp == kRedProd) tmem_dealloc(tmem, acc_cols);
}

}  // namespace tc
}  // namespace hmtl_b200
