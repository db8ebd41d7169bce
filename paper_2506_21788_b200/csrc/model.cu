// model.cu -- ModelT<float>::forward/backward on the GPU (FP32 parity path).
//
// Math: /root/reference/proj/include/hmtl/model.hpp:338-625 (restated in
// SURVEY.md Appendix A).  Dataflow changes (exact in real arithmetic):
//   * first edge layer factorised: z1_e = (h W1a)[dst] + (h W1b)[src] + d2_e w + b1
//     -- a node GEMM (N x H x 2H) plus an L2-resident gather instead of an
//     E x (2H+1) x H GEMM; its backward uses two CSR segment sums
//     (S_dst, S_src via the reverse-edge permutation) and node GEMMs;
//   * force-MLP layer 0 factorised the same way over h_i + h_j;
//   * a1 / z1 / zf0 are recomputed from node tables instead of stored
//     (saved per layer: z2 [E x H] only);
//   * every scatter-add is a destination-sorted CSR segment reduction in
//     ascending edge order (no float atomics, bit-reproducible), and every
//     weight gradient is a split-row A^T B with a fixed-order reduction.
// Head-specific weights: rows are grouped per owned head (head-sorted
// permutations built by route_kernel); GEMM tiles never straddle heads.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>

#include "chain.cuh"
#include "ctx.cuh"
#include "tc.cuh"

namespace hmtl_b200 {

namespace {

int gridn(long long n, int threads, int cap) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return int(b < cap ? b : cap);
}

// first edge layer pre-activation z1(e, k), factorised (see header)
__device__ __forceinline__ float z1_of(const float* __restrict__ P, int H, int d, int s, float d2,
                                       const float* __restrict__ wd, const float* __restrict__ b1, int k) {
  return __fadd_rn(__fadd_rn(__fadd_rn(P[size_t(d) * 2 * H + k], P[size_t(s) * 2 * H + H + k]), __fmul_rn(d2, wd[k])),
                   b1[k]);
}

// force-MLP layer 0 pre-activation: psi_in = [h_i + h_j, d_ij] (hmtl/model.hpp:466-473)
__device__ __forceinline__ float zf0_of(const float* __restrict__ Qf, int W, int d, int s, float dist,
                                        const float* __restrict__ wdist, const float* __restrict__ b0, int k) {
  return __fadd_rn(__fadd_rn(__fadd_rn(Qf[size_t(d) * W + k], Qf[size_t(s) * W + k]), __fmul_rn(dist, wdist[k])),
                   b0[k]);
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 f4z() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 add4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ float4 silu4(float4 a) { return make_float4(silu(a.x), silu(a.y), silu(a.z), silu(a.w)); }
__device__ __forceinline__ float4 mul4(float4 a, float4 b) { return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w); }
__device__ __forceinline__ float4 sgrad4(float4 a) {
  return make_float4(silu_grad(a.x), silu_grad(a.y), silu_grad(a.z), silu_grad(a.w));
}
// factorised pre-activation for 4 consecutive columns (same op order as z1_of/zf0_of)
__device__ __forceinline__ float4 pre4(float4 a, float4 b, float s, float4 w, float4 bias) {
  return make_float4(__fadd_rn(__fadd_rn(__fadd_rn(a.x, b.x), __fmul_rn(s, w.x)), bias.x),
                     __fadd_rn(__fadd_rn(__fadd_rn(a.y, b.y), __fmul_rn(s, w.y)), bias.y),
                     __fadd_rn(__fadd_rn(__fadd_rn(a.z, b.z), __fmul_rn(s, w.z)), bias.z),
                     __fadd_rn(__fadd_rn(__fadd_rn(a.w, b.w), __fmul_rn(s, w.w)), bias.w));
}

// head-block vectors are not 16 B aligned (reference layout: energy.b2 is one float)
__device__ __forceinline__ float4 ldu4(const float* p) { return make_float4(p[0], p[1], p[2], p[3]); }

struct NoAux {};
struct NoRC {};

struct HeadW {  // a head-block tensor of slot `seg`: base + seg*PH + off
  const float* base;
  size_t PH, off;
  __device__ __forceinline__ const float* at(int seg) const { return base + size_t(seg) * PH + off; }
};
struct HeadG {
  float* base;
  size_t PH, off;
  __device__ __forceinline__ float* at(int seg) const { return base + size_t(seg) * PH + off; }
};

// ================================================================ forward
// P = h [W1a | W1b]
struct PProb {
  BDesc bd() const { return BDesc{W1, W1 + size_t(H) * H, 1, H, H, 1, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "fwd.node_P";
  __device__ float4 a4(int, int r, int k) const { return ld4(h + size_t(r) * H + k); }
  __device__ void epi4(int, int r, int n, float4 acc) const { st4(P + size_t(r) * 2 * H + n, acc); }
  RowSet rows;
  int K, Ncols, H;
  const float *h, *W1;
  float* P;
  __device__ float a(int, int r, int k) const { return h[size_t(r) * H + k]; }
  __device__ float b(int, int k, int n) const { return n < H ? W1[size_t(k) * H + n] : W1[size_t(H + k) * H + n - H]; }
  __device__ void epi(int, int r, int n, float acc) const { P[size_t(r) * 2 * H + n] = acc; }
};

// z2 = silu(z1) W2 + b2   (hmtl/model.hpp:398-404)
struct MsgProb {
  static constexpr bool kSlabEpi = true;  // store-only epilogue: row-coalesced slab stores measured faster
  BDesc bd() const { return BDesc{W2, nullptr, 0, 0, H, 1, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "fwd.edge_msg_gemm";
  struct RC {
    int d, s;
    float w;
  };
  __device__ RC rctx(int, int e) const { return a1out ? RC{0, 0, 0.f} : RC{dst[e], src[e], geo[e].w}; }
  __device__ float4 a4c(int, int e, const RC& r, int k) const {
    if (a1out) return ld4(a1out + size_t(e) * H + k);  // a1 materialised by edge_a1_kernel
    return silu4(pre4(ld4(P + size_t(r.d) * 2 * H + k), ld4(P + size_t(r.s) * 2 * H + H + k), r.w, ld4(wd + k),
                      ld4(b1 + k)));
  }
  __device__ void epi4c(int, int e, const RC&, int n, float4 acc) const {
    st4(z2 + size_t(e) * H + n, add4(acc, ld4(b2 + n)));
  }
  __device__ float4 a4(int, int e, int k) const {
    const int d = dst[e], s = src[e];
    return silu4(pre4(ld4(P + size_t(d) * 2 * H + k), ld4(P + size_t(s) * 2 * H + H + k), geo[e].w, ld4(wd + k),
                      ld4(b1 + k)));
  }
  __device__ void epi4(int, int e, int n, float4 acc) const { st4(z2 + size_t(e) * H + n, add4(acc, ld4(b2 + n))); }
  RowSet rows;
  int K, Ncols, H;
  const float *P, *wd, *b1, *W2, *b2;
  const int *dst, *src;
  const float4* geo;
  float* z2;
  float* a1out;
  __device__ float a(int, int e, int k) const { return silu(z1_of(P, H, dst[e], src[e], geo[e].w, wd, b1, k)); }
  __device__ float b(int, int k, int n) const { return W2[size_t(k) * H + n]; }
  __device__ void epi(int, int e, int n, float acc) const { z2[size_t(e) * H + n] = acc + b2[n]; }
};

// z2 = silu(z1) W2 + b2 with the A operand gathered by cp.async (tc.cuh kAsync):
// the two node-table rows P_a[dst], P_b[src] of every edge land in shared memory
// and are combined in place into a1 = silu(z1); a1 (eW2 weight gradient) and
// silu'(z1) (the backward's dz1 epilogue) are stored on the way.  Replaces
// edge_a1 -> MsgProb (same operations: bit-identical a1, z2).
struct MsgAsyncProb {
  BDesc bd() const { return BDesc{W2, nullptr, 0, 0, H, 1, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "fwd.edge_msg_gather";
  static constexpr bool kAsync = true;
  struct RC {
    int d, s;
    float w;
  };
  __device__ RC rctx(int, int e) const { return RC{dst[e], src[e], geo[e].w}; }
  __device__ const float* src_a(int, int, const RC& r, int k) const { return P + size_t(r.d) * 2 * H + k; }
  __device__ const float* src_b(int, int, const RC& r, int k) const { return P + size_t(r.s) * 2 * H + H + k; }
  __device__ float4 combine(int, int e, const RC& r, int k, float4 a, float4 b) const {
    const float4 z = pre4(a, b, r.w, ld4(wd + k), ld4(b1 + k));
    const float4 v = silu4(z);
    st4(a1out + size_t(e) * H + k, v);
    st4(s1p + size_t(e) * H + k, sgrad4(z));
    return v;
  }
  __device__ void epi4c(int, int e, const RC&, int n, float4 acc) const {
    st4(z2 + size_t(e) * H + n, add4(acc, ld4(b2 + n)));
  }
  RowSet rows;
  int K, Ncols, H;
  const float *P, *wd, *b1, *W2, *b2;
  const int *dst, *src;
  const float4* geo;
  float *z2, *a1out, *s1p;
  __device__ float b(int, int k, int n) const { return W2[size_t(k) * H + n]; }
};

// z2 = silu(z1) W2 + b2 from the stored pre-activation z1 (z1_only: the forward's edge
// pass stores z1 alone; this producer, the eW2 weight gradient and the backward's dz1
// epilogue apply silu / silu' themselves -- the same values as storing a1 and silu'(z1))
struct MsgZ1Prob {
  BDesc bd() const { return BDesc{W2, nullptr, 0, 0, H, 1, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "fwd.edge_msg_gemm";
  static constexpr bool kTcOnly = true;
  using Raw = float4;
  __device__ Raw raw4(int, int e, const NoRC&, int k) const { return ld4(z1 + size_t(e) * H + k); }
  __device__ float4 fin4(int, int, const NoRC&, int, const Raw& z) const { return silu4(z); }
  __device__ float4 a4(int, int e, int k) const { return silu4(ld4(z1 + size_t(e) * H + k)); }
  __device__ void epi4(int, int e, int n, float4 acc) const { st4(z2 + size_t(e) * H + n, add4(acc, ld4(b2 + n))); }
  RowSet rows;
  int K, Ncols, H;
  const float *z1, *W2, *b2;
  float* z2;
  __device__ float b(int, int k, int n) const { return W2[size_t(k) * H + n]; }
};

// Fused message passing of one layer (hmtl/model.hpp:388-411) in one tensor-core
// pass over the edges: the producer gathers a1 = silu(P_a[dst] + P_b[src] + d2 w
// + b1) straight into the A operand (and stores a1 for the eW2 weight gradient),
// the epilogue stores z2 = a1 W2 + b2 and sums m = silu(z2) per destination
// (segmented epilogue, ascending edge order) into agg; destinations whose edge
// rows straddle a 128-edge tile are finished by agg_fix_kernel.  Bit-identical
// to edge_a1 -> MsgProb -> agg4 (same operations in the same order).
struct MsgSegProb {
  BDesc bd() const { return BDesc{W2, nullptr, 0, 0, H, 1, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "fwd.edge_msg_fused";
  static constexpr bool kSegSum = true;
  struct RC {
    int d, s;
    float w;
  };
  struct Raw {
    float4 a, b;
  };
  __device__ RC rctx(int, int e) const { return RC{dst[e], src[e], geo[e].w}; }
  __device__ Raw raw4(int, int, const RC& r, int k) const {
    return Raw{ld4(P + size_t(r.d) * 2 * H + k), ld4(P + size_t(r.s) * 2 * H + H + k)};
  }
  __device__ float4 fin4(int, int e, const RC& r, int k, const Raw& x) const {
    const float4 v = silu4(pre4(x.a, x.b, r.w, ld4(wd + k), ld4(b1 + k)));
    st4(a1out + size_t(e) * H + k, v);
    return v;
  }
  __device__ float4 epi4r(int, int e, const RC&, int n, float4 acc, const NoAux&) const {
    const float4 z = add4(acc, ld4(b2 + n));
    st4(z2 + size_t(e) * H + n, z);
    return silu4(z);
  }
  __device__ int seg_key(int e) const { return dst[e]; }
  __device__ void seg_store(int i, int n, float v) const { agg[size_t(i) * H + n] = v; }
  RowSet rows;
  int K, Ncols, H;
  const float *P, *wd, *b1, *W2, *b2;
  const int *dst, *src;
  const float4* geo;
  float *z2, *a1out, *agg;
  float* tpart;  // [2][tcap][H] straddling destinations' per-tile pieces (agg_fix_kernel adds them)
  int tcap;
  __device__ float a(int, int e, int k) const { return silu(z1_of(P, H, dst[e], src[e], geo[e].w, wd, b1, k)); }
  __device__ float b(int, int k, int n) const { return W2[size_t(k) * H + n]; }
};

// vz1 = [h, agg] nW1 + nb1   (hmtl/model.hpp:412-420)
struct Node1Prob {
  BDesc bd() const { return BDesc{W, nullptr, 0, 0, H, 1, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "fwd.node_mlp1";
  __device__ float4 a4(int, int r, int k) const {
    return k < H ? ld4(h + size_t(r) * H + k) : ld4(agg + size_t(r) * H + k - H);
  }
  __device__ void epi4(int, int r, int n, float4 acc) const { st4(vz1 + size_t(r) * H + n, add4(acc, ld4(bias + n))); }
  RowSet rows;
  int K, Ncols, H;
  const float *h, *agg, *W, *bias;
  float* vz1;
  __device__ float a(int, int r, int k) const { return k < H ? h[size_t(r) * H + k] : agg[size_t(r) * H + k - H]; }
  __device__ float b(int, int k, int n) const { return W[size_t(k) * H + n]; }
  __device__ void epi(int, int r, int n, float acc) const { vz1[size_t(r) * H + n] = acc + bias[n]; }
};

// h' = h + (silu(vz1) nW2 + nb2)   (hmtl/model.hpp:421-426, residual)
struct Node2Prob {
  struct Aux {
    float4 h;
  };
  __device__ Aux epi_aux(int, int r, int n) const { return Aux{ld4(h + size_t(r) * H + n)}; }
  __device__ void epi4a(int, int r, int n, float4 acc, const Aux& a) const {
    st4(hn + size_t(r) * H + n, add4(a.h, add4(acc, ld4(bias + n))));  // h + (acc + b), as the SIMT path
  }
  BDesc bd() const { return BDesc{W, nullptr, 0, 0, H, 1, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "fwd.node_mlp2";
  __device__ float4 a4(int, int r, int k) const { return silu4(ld4(vz1 + size_t(r) * H + k)); }
  __device__ void epi4(int, int r, int n, float4 acc) const {
    st4(hn + size_t(r) * H + n, add4(ld4(h + size_t(r) * H + n), add4(acc, ld4(bias + n))));
  }
  RowSet rows;
  int K, Ncols, H;
  const float *vz1, *W, *bias, *h;
  float* hn;
  __device__ float a(int, int r, int k) const { return silu(vz1[size_t(r) * H + k]); }
  __device__ float b(int, int k, int n) const { return W[size_t(k) * H + n]; }
  __device__ void epi(int, int r, int n, float acc) const {
    hn[size_t(r) * H + n] = h[size_t(r) * H + n] + (acc + bias[n]);
  }
};

// energy MLP layer i over graph rows of each head (mlp_forward_, :282-306)
struct EnergyProb {
  BDesc bd() const { return BDesc{Wt.base + Wt.off, nullptr, 0, 0, Ncols, 1, K, Ncols, rows.nseg, (long long)Wt.PH, nullptr}; }
  static constexpr const char* kName = "fwd.energy_mlp";
  RowSet rows;
  int K, Ncols, H, W, layer, last;
  const float *pooled, *ezp;  // ezp = ez of layer-1
  HeadW Wt, Bt;
  float *ez, *energy;
  __device__ float a(int, int g, int k) const {
    return layer == 0 ? pooled[size_t(g) * H + k] : silu(ezp[size_t(g) * W + k]);
  }
  __device__ float b(int seg, int k, int n) const { return Wt.at(seg)[size_t(k) * Ncols + n]; }
  __device__ void epi(int seg, int g, int n, float acc) const {
    const float z = acc + Bt.at(seg)[n];
    ez[size_t(g) * W + n] = z;
    if (last) energy[g] = z;
  }
};

// Qf = h_L Wf0[:H]  (node rows per head)
struct QfProb {
  BDesc bd() const { return BDesc{Wt.base + Wt.off, nullptr, 0, 0, W, 1, K, Ncols, rows.nseg, (long long)Wt.PH, nullptr}; }
  static constexpr const char* kName = "fwd.force_Qf";
  __device__ float4 a4(int, int r, int k) const { return ld4(h + size_t(r) * H + k); }
  __device__ void epi4(int, int r, int n, float4 acc) const { st4(Qf + size_t(r) * W + n, acc); }
  RowSet rows;
  int K, Ncols, H, W;
  const float* h;
  HeadW Wt;
  float* Qf;
  __device__ float a(int, int r, int k) const { return h[size_t(r) * H + k]; }
  __device__ float b(int seg, int k, int n) const { return Wt.at(seg)[size_t(k) * W + n]; }
  __device__ void epi(int, int r, int n, float acc) const { Qf[size_t(r) * W + n] = acc; }
};

// force MLP layer i >= 1 over edge rows per head; last layer writes s_e
struct ForceProb {
  static constexpr bool kSlabEpi = true;  // store-only epilogue: row-coalesced slab stores measured faster
  BDesc bd() const { return BDesc{Wt.base + Wt.off, nullptr, 0, 0, Ncols, 1, K, Ncols, rows.nseg, (long long)Wt.PH, nullptr}; }
  static constexpr const char* kName = "fwd.force_edge_gemm";
  struct RC {
    int d, s;
    float dist;
  };
  __device__ RC rctx(int, int e) const {
    return (af0out || layer != 1) ? RC{0, 0, 0.f} : RC{dst[e], src[e], dist[e]};
  }
  __device__ float4 a4c(int seg, int e, const RC& r, int k) const {
    if (layer == 1) {
      if (af0out) return ld4(af0out + size_t(e) * W + k);  // silu(zf0) materialised by edge_af0_kernel
      return silu4(pre4(ld4(Qf + size_t(r.d) * W + k), ld4(Qf + size_t(r.s) * W + k), r.dist,
                        ldu4(Wd.at(seg) + k), ldu4(B0.at(seg) + k)));
    }
    return silu4(ld4(zf + size_t(layer - 2) * Ec * W + size_t(e) * W + k));
  }
  __device__ void epi4c(int seg, int e, const RC&, int n, float4 acc) const { epi4(seg, e, n, acc); }
  __device__ float4 a4(int seg, int e, int k) const {
    if (layer == 1)
      return silu4(pre4(ld4(Qf + size_t(dst[e]) * W + k), ld4(Qf + size_t(src[e]) * W + k), dist[e],
                        ldu4(Wd.at(seg) + k), ldu4(B0.at(seg) + k)));
    return silu4(ld4(zf + size_t(layer - 2) * Ec * W + size_t(e) * W + k));
  }
  __device__ void epi4(int seg, int e, int n, float4 acc) const {
    const float4 z = add4(acc, ldu4(Bt.at(seg) + n));
    if (last) {
      s[e] = z.x;  // Ncols == 1 never reaches the tensor-core path
    } else {
      st4(zf_out + size_t(layer - 1) * Ec * W + size_t(e) * W + n, z);
    }
  }
  RowSet rows;
  int K, Ncols, H, W, layer, last;
  long long Ec;
  const float *Qf, *zf, *dist;
  const int *dst, *src;
  HeadW Wd, B0, Wt, Bt;  // Wd = row H of Wf0 (distance weight), B0 = bf0
  float *zf_out, *s;
  float* af0out;
  __device__ float a(int seg, int e, int k) const {
    if (layer == 1) return silu(zf0_of(Qf, W, dst[e], src[e], dist[e], Wd.at(seg), B0.at(seg), k));
    return silu(zf[size_t(layer - 2) * Ec * W + size_t(e) * W + k]);
  }
  __device__ float b(int seg, int k, int n) const { return Wt.at(seg)[size_t(k) * Ncols + n]; }
  __device__ void epi(int seg, int e, int n, float acc) const {
    const float z = acc + Bt.at(seg)[n];
    if (last) s[e] = z;
    else zf_out[size_t(layer - 1) * Ec * W + size_t(e) * W + n] = z;
  }
};

__global__ void embed_kernel(const DevHdr* hdr, const uint8_t* __restrict__ species, const float* __restrict__ embed,
                             float* __restrict__ h, int H, const float* __restrict__ ptab, float* __restrict__ P0) {
  pdl_wait();
  const long long total = (long long)hdr->N * H;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int i = int(t / H), k = int(t % H), sp = species[i];
    h[t] = embed[size_t(sp) * H + k];
    if (ptab) {  // layer 0's P = h0 [W1a | W1b] is a per-species table (h0 = embed[species])
      P0[size_t(i) * 2 * H + k] = ptab[size_t(sp) * 2 * H + k];
      P0[size_t(i) * 2 * H + H + k] = ptab[size_t(sp) * 2 * H + H + k];
    }
  }
}

// agg_i = sum_{e: dst(e)=i, ascending e} silu(z2_e)   (segment_sum, hmtl/kernels.hpp:97-108)
__global__ void agg_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr, const float* __restrict__ z2,
                           float* __restrict__ agg, int H) {
  pdl_wait();
  const int N = hdr->N;
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += (gridDim.x * blockDim.x) >> 5) {
    const int e0 = row_ptr[i], e1 = row_ptr[i + 1];
    for (int c = lane; c < H; c += 32) {
      float acc = 0.f;
      for (int e = e0; e < e1; ++e) acc += silu(z2[size_t(e) * H + c]);
      agg[size_t(i) * H + c] = acc;
    }
  }
}

// mean pool: (sum_i h_i) * (S(1)/S(n))   (hmtl/model.hpp:444-453)
__global__ void pool_kernel(const DevHdr* hdr, const int* __restrict__ graph_offset, const float* __restrict__ h,
                            float* __restrict__ pooled, int H) {
  pdl_wait();
  const int G = hdr->G;
  const int lane = threadIdx.x & 31;
  for (int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < G; g += (gridDim.x * blockDim.x) >> 5) {
    const int lo = graph_offset[g], hi = graph_offset[g + 1];
    const float inv = 1.f / float(hi - lo);
    for (int c = lane; c < H; c += 32) {
      float acc = 0.f;
      for (int i = lo; i < hi; ++i) acc += h[size_t(i) * H + c];
      pooled[size_t(g) * H + c] = acc * inv;
    }
  }
}

// Energy head, whole (hmtl/model.hpp:440-452): pooled_g = mean_{i in g} h_L[i],
// z_0 = pooled W0 + b0, z_i = silu(z_{i-1}) W_i + b_i, E_g = z_{D-1} (width 1).
// One launch replaces pool + D GEMM launches of a few hundred rows each: CTA =
// kEhRows graphs of one head segment; warp r pools graph r (float4 columns, 8
// atom rows in flight, ascending atom order); each layer stages its weights in
// shared memory in 64-row K chunks (one round of loads) and a thread
// computes 4 rows x 1 column in exact FP32 (ascending k); the width-1 layer is a
// warp dot product per graph.  Writes pooled and every z_i (the backward's inputs).
constexpr int kEhRows = 8, kEhMaxD = 8, kEhKC = 64;
struct EHeadArgs {
  const float* hp;  // head block of slot 0; slot s at + s*PH
  size_t PH;
  size_t w[kEhMaxD], b[kEhMaxD];
  int D, H, W;
};
__global__ void __launch_bounds__(256) energy_head_kernel(const DevHdr* hdr, RowSet rows, const int* __restrict__ go,
                                                          const float* __restrict__ h, EHeadArgs a,
                                                          float* __restrict__ pooled, float* __restrict__ ez, int Gc,
                                                          float* __restrict__ energy) {
  pdl_wait();
  extern __shared__ float4 ehs4[];
  float* smf = reinterpret_cast<float*>(ehs4);
  const int KM = max(a.H, a.W);
  float* X = smf;                    // [kEhRows][KM] layer input
  float* Y = X + kEhRows * KM;       // [kEhRows][KM] next layer input
  float* Ws = Y + kEhRows * KM;      // [kEhKC][W] weight chunk
  const int seg = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rb = rows.begin(seg), re = rows.end(seg);
  const float* hp = a.hp + size_t(seg) * a.PH;
  for (int v0 = rb + blockIdx.x * kEhRows; v0 < re; v0 += gridDim.x * kEhRows) {
    const int nr = min(kEhRows, re - v0);
    if (warp < nr) {
      const int g = rows.row(v0 + warp), lo = go[g], hi = go[g + 1];
      const float inv = 1.f / float(hi - lo);
      for (int c = lane * 4; c < a.H; c += 128) {
        float4 acc = f4z();
        for (int i = lo; i < hi; i += 8) {
          float4 x[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) x[u] = i + u < hi ? ld4(h + size_t(i + u) * a.H + c) : f4z();
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (i + u < hi) acc = add4(acc, x[u]);
        }
        const float4 m = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
        st4(pooled + size_t(g) * a.H + c, m);
        *reinterpret_cast<float4*>(X + warp * KM + c) = m;
      }
    }
    for (int l = 0; l < a.D; ++l) {
      const int K = l ? a.W : a.H;
      const float* Wt = hp + a.w[l];
      const float* bt = hp + a.b[l];
      float* ezl = ez + size_t(l) * Gc * a.W;
      if (l == a.D - 1) {  // width-1 output: warp dot product per graph
        __syncthreads();
        if (warp < nr) {
          const int g = rows.row(v0 + warp);
          float acc = 0.f;
          for (int k = lane; k < K; k += 32) acc = fmaf(X[warp * KM + k], Wt[k], acc);
#pragma unroll
          for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (lane == 0) {
            const float z = acc + bt[0];
            ezl[size_t(g) * a.W] = z;
            energy[g] = z;
          }
        }
        __syncthreads();
        break;
      }
      const int n0 = tid & 127, r0 = (tid >> 7) * 4;  // 4 rows x 1 column per thread per 128-column block
      float acc[4][2] = {};
      for (int k0 = 0; k0 < K; k0 += kEhKC) {
        const int kc = min(kEhKC, K - k0);
        __syncthreads();  // X complete / previous chunk consumed
        // (scalar: head tensors follow the reference's BlockLayout, not 16-byte aligned)
#pragma unroll 8
        for (int t = tid; t < kc * a.W; t += 256) Ws[t] = __ldg(Wt + size_t(k0) * a.W + t);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int n = n0 + 128 * j;
          if (n < a.W) {
            for (int k = 0; k < kc; ++k) {
              const float w = Ws[k * a.W + n];
#pragma unroll
              for (int u = 0; u < 4; ++u) acc[u][j] = fmaf(X[(r0 + u) * KM + k0 + k], w, acc[u][j]);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = n0 + 128 * j;
        if (n >= a.W) continue;
        const float bn = bt[n];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (r0 + u >= nr) continue;
          const float z = acc[u][j] + bn;
          ezl[size_t(rows.row(v0 + r0 + u)) * a.W + n] = z;
          Y[(r0 + u) * KM + n] = silu(z);
        }
      }
      __syncthreads();
      float* t = X;
      X = Y;
      Y = t;
    }
    __syncthreads();
  }
}

// F_i = sum_{e in row i} dvec_e * s_e   (hmtl/model.hpp:475-480)
__global__ void forces_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr, const float4* __restrict__ geo,
                              const float* __restrict__ s, float* __restrict__ F) {
  pdl_wait();
  // warp per node: lane l sums edges l, l+32, ... of the row, then a fixed xor tree
  // (the association depends only on the degree: deterministic)
  const int N = hdr->N, lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += (gridDim.x * blockDim.x) >> 5) {
    const int e0 = row_ptr[i], e1 = row_ptr[i + 1];
    float fx = 0.f, fy = 0.f, fz = 0.f;
    for (int e = e0 + lane; e < e1; e += 32) {
      const float4 g = geo[e];
      const float se = s[e];
      fx += g.x * se;
      fy += g.y * se;
      fz += g.z * se;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      fx += __shfl_xor_sync(0xffffffffu, fx, o);
      fy += __shfl_xor_sync(0xffffffffu, fy, o);
      fz += __shfl_xor_sync(0xffffffffu, fz, o);
    }
    if (lane == 0) F[3 * i] = fx, F[3 * i + 1] = fy, F[3 * i + 2] = fz;
  }
}

__global__ void finite_kernel(DevHdr* hdr, const float* __restrict__ energy, const float* __restrict__ F) {
  pdl_wait();
  const int G = hdr->G, N = hdr->N;
  bool bad = false;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < G + 3 * N; t += gridDim.x * blockDim.x) {
    const float v = t < G ? energy[t] : F[t - G];
    if (!isfinite(v)) bad = true;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&hdr->err, kErrNonFinite);
}

// ---- tcgen05 adapters over the SIMT problem functors (same math, same epilogues)
template <class P, class = void>
struct HasA4 : std::false_type {};
template <class P>
struct HasA4<P, std::void_t<decltype(std::declval<const P&>().a4(0, 0, 0))>> : std::true_type {};
template <class P, class = void>
struct HasEpi4 : std::false_type {};
template <class P>
struct HasEpi4<P, std::void_t<decltype(std::declval<const P&>().epi4(0, 0, 0, float4{}))>> : std::true_type {};

template <class P, class = void>
struct RCOf {
  using type = NoRC;
  static constexpr bool has = false;
};
template <class P>
struct RCOf<P, std::void_t<typename P::RC>> {
  using type = typename P::RC;
  static constexpr bool has = true;
};

template <class P, class = void>
struct AuxOf {
  using type = NoAux;
  static constexpr bool has = false;
};
template <class P>
struct AuxOf<P, std::void_t<typename P::Aux>> {
  using type = typename P::Aux;
  static constexpr bool has = true;
};

// optional two-phase A producer: raw4 issues the loads (kept in the producer's
// prefetch registers), fin4 does the math (and any side store) when the chunk is
// written to shared memory -- so gathered/elementwise A operands keep their loads
// in flight across the previous chunk's stores
template <class P, class = void>
struct RawOf {
  using type = float4;
  static constexpr bool has = false;
};
template <class P>
struct RawOf<P, std::void_t<typename P::Raw>> {
  using type = typename P::Raw;
  static constexpr bool has = true;
};
template <class P, class = void>
struct HasAuxC : std::false_type {};
template <class P>
struct HasAuxC<P, std::void_t<decltype(&P::epi_auxc)>> : std::true_type {};

template <class P, class = void>
struct TcOnly : std::false_type {};  // problems without a SIMT fallback (P::kTcOnly)
template <class P>
struct TcOnly<P, std::void_t<decltype(P::kTcOnly)>> : std::bool_constant<P::kTcOnly> {};
template <class P, class = void>
struct AsyncOf : std::false_type {};
template <class P>
struct AsyncOf<P, std::void_t<decltype(P::kAsync)>> : std::bool_constant<P::kAsync> {};
template <class P, class = void>
struct SegOf : std::false_type {};
template <class P>
struct SegOf<P, std::void_t<decltype(P::kSegSum)>> : std::bool_constant<P::kSegSum> {};

template <class P, class = void>
struct HasRowPrefetch : std::false_type {};
template <class P>
struct HasRowPrefetch<P, std::void_t<decltype(std::declval<const P&>().prefetch_rows(0, 0))>> : std::true_type {};
template <class P>
struct TcRow {
  using RC = typename RCOf<P>::type;
  static constexpr bool kPrefetch = HasRowPrefetch<P>::value;
  static constexpr bool kSlabEpi = SegOf<P>::value || tc::RowSlab<P>::value;  // (tc.cuh: slab vs fragment epilogue)
  // L2 prefetch of the row-contiguous streams of rows [r0, r1) (tc.cuh: issued at launch)
  __device__ __forceinline__ void prefetch_rows(int r0, int r1) const {
    if constexpr (kPrefetch) p.prefetch_rows(r0, r1);
  }
  using Aux = typename AuxOf<P>::type;
  using Raw = typename RawOf<P>::type;
  static constexpr bool kSeg = SegOf<P>::value;  // segmented-sum epilogue (tc.cuh)
  static constexpr bool kAsync = AsyncOf<P>::value;  // cp.async two-operand producer (tc.cuh)
  __device__ __forceinline__ const float* src_a(int seg, int row, const RC& rc, int k) const {
    if constexpr (kAsync) return p.src_a(seg, row, rc, k);
    else return nullptr;
  }
  __device__ __forceinline__ const float* src_b(int seg, int row, const RC& rc, int k) const {
    if constexpr (kAsync) return p.src_b(seg, row, rc, k);
    else return nullptr;
  }
  __device__ __forceinline__ float4 combine(int seg, int row, const RC& rc, int k, float4 a, float4 b) const {
    if constexpr (kAsync) return p.combine(seg, row, rc, k, a, b);
    else return a;
  }
  RowSet rows;
  int K, Ncols;
  const float* bimg;
  size_t bimg_seg;
  P p;
  __device__ __forceinline__ RC rctx(int seg, int row) const {
    if constexpr (RCOf<P>::has) return p.rctx(seg, row);
    else return RC{};
  }
  __device__ __forceinline__ float4 a4(int seg, int row, const RC& rc, int k) const {
    if constexpr (RCOf<P>::has) return p.a4c(seg, row, rc, k);
    else if constexpr (HasA4<P>::value) return p.a4(seg, row, k);
    else return make_float4(p.a(seg, row, k), p.a(seg, row, k + 1), p.a(seg, row, k + 2), p.a(seg, row, k + 3));
  }
  __device__ __forceinline__ Raw raw4(int seg, int row, const RC& rc, int k) const {
    if constexpr (RawOf<P>::has) return p.raw4(seg, row, rc, k);
    else return a4(seg, row, rc, k);
  }
  __device__ __forceinline__ float4 fin4(int seg, int row, const RC& rc, int k, const Raw& r) const {
    if constexpr (RawOf<P>::has) return p.fin4(seg, row, rc, k, r);
    else return r;
  }
  __device__ __forceinline__ Aux epi_aux(int seg, int row, const RC& rc, int n) const {
    if constexpr (HasAuxC<P>::value) return p.epi_auxc(seg, row, rc, n);
    else if constexpr (AuxOf<P>::has) return p.epi_aux(seg, row, n);
    else return Aux{};
  }
  __device__ __forceinline__ int seg_key(int row) const {
    if constexpr (kSeg) return p.seg_key(row);
    else return -1;
  }
  __device__ __forceinline__ float4 epi4r(int seg, int row, const RC& rc, int n, float4 acc, const Aux& ax) const {
    if constexpr (kSeg) return p.epi4r(seg, row, rc, n, acc, ax);
    else return acc;
  }
  __device__ __forceinline__ void seg_store(int key, int n, float v) const {
    if constexpr (kSeg) p.seg_store(key, n, v);
  }
  __device__ __forceinline__ void tile_store(int which, int t, int n, float v) const {
    if constexpr (kSeg) p.tpart[(size_t(which) * p.tcap + t) * p.Ncols + n] = v;
  }
  __device__ __forceinline__ void epi4(int seg, int row, const RC& rc, int n, float4 acc, const Aux& ax) const {
    if constexpr (HasAuxC<P>::value) {
      p.epi4ac(seg, row, rc, n, acc, ax);
    } else if constexpr (AuxOf<P>::has) {
      p.epi4a(seg, row, n, acc, ax);
    } else if constexpr (RCOf<P>::has) {
      p.epi4c(seg, row, rc, n, acc);
    } else if constexpr (HasEpi4<P>::value) {
      p.epi4(seg, row, n, acc);
    } else {
      p.epi(seg, row, n, acc.x);
      p.epi(seg, row, n + 1, acc.y);
      p.epi(seg, row, n + 2, acc.z);
      p.epi(seg, row, n + 3, acc.w);
    }
  }
};
template <class P, class = void>
struct HasX4 : std::false_type {};
template <class P>
struct HasX4<P, std::void_t<decltype(std::declval<const P&>().x4(0, 0, 0))>> : std::true_type {};
template <class P, class = void>
struct HasY4 : std::false_type {};
template <class P>
struct HasY4<P, std::void_t<decltype(std::declval<const P&>().y4(0, 0, 0))>> : std::true_type {};
// B image of problem P: B(n, k) = p.b(seg, k, n), layout of tc::bimg_kernel
template <class P>
__global__ void bimg_prob_kernel(P p, float* __restrict__ out, int nseg) {
  pdl_wait();
  const int K = p.K, N = p.Ncols;
  const size_t total = size_t(nseg) * K * N;
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; t < total; t += size_t(gridDim.x) * blockDim.x) {
    const int seg = int(t / (size_t(K) * N));
    const int rem = int(t % (size_t(K) * N));
    const int n = rem % N, k = rem / N;
    const float x = p.b(seg, k, n);
    const float h = tc::tf32_hi(x);
    const int ch = k / tc::KC, c16 = (k % tc::KC) / 4, q = k % 4;
    float* o = out + size_t(seg) * 2 * K * N + size_t(ch) * 2 * tc::KC * N;
    const uint32_t off = tc::sw128(n, c16) / 4 + q;
    o[off] = h;
    o[size_t(tc::KC) * N + off] = x - h;
  }
}
template <class P, class = void>
struct HasTmaFin : std::false_type {};
template <class P>
struct HasTmaFin<P, std::void_t<decltype(std::declval<const P&>().xfin(float4{}))>> : std::true_type {};
// TMA reduce path operands (P::tma fills it; nullptr = computed on the fly):
// X = x (or [x | x1], x1 from feature xsplit on), Y = y; row-major, ld floats
struct TmaOps {
  const float* x = nullptr;
  int ldx = 0;
  const float* x1 = nullptr;
  int xsplit = 0;
  const float* y = nullptr;
  int ldy = 0;
};
template <class P, class = void>
struct HasTma : std::false_type {};
template <class P>
struct HasTma<P, std::void_t<decltype(&P::tma)>> : std::true_type {};

template <class P>
struct TcRed {
  RowSet rows;
  int M, Ncols, colsum;
  P p;
  int n_off = 0;  // first output column of this launch (outputs wider than 256 go in slices)
  __device__ __forceinline__ float4 x4(int seg, int row, int m) const {
    if constexpr (HasX4<P>::value) return p.x4(seg, row, m);
    else return make_float4(p.a(seg, row, m), p.a(seg, row, m + 1), p.a(seg, row, m + 2), p.a(seg, row, m + 3));
  }
  __device__ __forceinline__ float4 y4(int seg, int row, int n) const {
    n += n_off;
    if constexpr (HasY4<P>::value) return p.y4(seg, row, n);
    else return make_float4(p.b(seg, row, n), p.b(seg, row, n + 1), p.b(seg, row, n + 2), p.b(seg, row, n + 3));
  }
  __device__ __forceinline__ void store(int seg, int k, int n, float v) const { p.store(seg, k, n + n_off, v); }
  // TMA operand path (tc_red_tma_kernel): elementwise transforms of the raw rows
  __device__ __forceinline__ float4 xfin(float4 v) const {
    if constexpr (HasTmaFin<P>::value) return p.xfin(v);
    else return v;
  }
  __device__ __forceinline__ float4 yfin(float4 v) const { return v; }
};

// one launch builds every B image of the step: blockIdx.y = job
// grid (blocks, jobs); elements walk the contiguous source dimension (coalesced
// reads), 32-bit index math
__global__ void __launch_bounds__(256) bimg_all_kernel(const BDesc* __restrict__ jobs) {
  // one thread per 16 B piece of the image (4 consecutive k of one column n: one
  // float4 store each for hi and lo); a few CTAs per job, grid-stride
  pdl_wait();
  const BDesc J = jobs[blockIdx.y];
  const int K = J.K, N = J.N, K4 = K / 4, KN4 = K4 * N;
  const int total = J.nseg * KN4;
  const bool kfast = J.sk == 1;  // walk the contiguous source dimension
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int seg = t / KN4;
    const int rem = t - seg * KN4;
    const int k4 = kfast ? rem % K4 : rem / N, n = kfast ? rem / K4 : rem % N;
    const int k0 = 4 * k4;
    float x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int kk = k0 + q, nn = n;
      const float* b = J.base0;
      if (J.split == 1 && n >= J.at) b = J.base1, nn = n - J.at;
      if (J.split == 2 && kk >= J.at) b = J.base1, kk -= J.at;
      x[q] = b[size_t(seg) * J.seg_stride + size_t(kk) * J.sk + size_t(nn) * J.sn];
    }
    const float4 h = make_float4(tc::tf32_hi(x[0]), tc::tf32_hi(x[1]), tc::tf32_hi(x[2]), tc::tf32_hi(x[3]));
    const float4 l = make_float4(x[0] - h.x, x[1] - h.y, x[2] - h.z, x[3] - h.w);
    const int ch = k0 / tc::KC, c16 = (k0 % tc::KC) / 4;
    float* o;
    uint32_t off;
    size_t lo;
    if (J.halves) {  // pair layout: block (half, chunk) = [hi | lo] of N/2 rows
      const int Nh = N / 2, hf = n / Nh, nl = n - hf * Nh;
      o = J.out + size_t(seg) * 8 * KN4 + (size_t(hf) * (K / tc::KC) + ch) * 2 * tc::KC * Nh;
      off = tc::sw128(nl, c16) / 4;
      lo = size_t(tc::KC) * Nh;
    } else {
      o = J.out + size_t(seg) * 8 * KN4 + size_t(ch) * 2 * tc::KC * N;
      off = tc::sw128(n, c16) / 4;
      lo = size_t(tc::KC) * N;
    }
    *reinterpret_cast<float4*>(o + off) = h;
    *reinterpret_cast<float4*>(o + lo + off) = l;
  }
}

template <class Kern>
void set_smem(Kern k, size_t bytes) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

template <class P>
void ab(const P& p, long long rows_cap, int nseg, cudaStream_t st, int sm, Ctx& c, const float* img_fixed = nullptr) {
  Prof pr(c, P::kName, st);
  const bool use_tc = c.use_tc && p.K % tc::KC == 0 && p.Ncols % 32 == 0 &&
                      (p.Ncols <= 256 || p.Ncols % 256 == 0) && size_t(nseg) * 2 * p.K * p.Ncols <= c.bimg_cap;
  if (use_tc) {
    const float* img = c.bimg;
    const int idx = img_fixed ? -1 : c.bimg_idx++;  // (img_fixed: a prebuilt image, outside the call order)
    if (img_fixed) {
      img = img_fixed;
    } else if (c.bimg_ready && idx < int(c.bjobs.size()) && !c.bjobs[idx].halves) {
      img = c.bjobs[idx].out;  // prebuilt by the batched builder after the last weight update
    } else {  // (a pair-layout image -- recorded for a chain that did not run -- is rebuilt here)
      kl(bimg_prob_kernel<P>, gridn((long long)nseg * p.K * p.Ncols, 256, sm * 4), 256, 0, st, p, c.bimg, nseg);
      if (c.bimg_recording) {
        BDesc d = p.bd();
        d.nseg = nseg;
        d.halves = c.rec_halves;
        c.bjobs.push_back(d);
      }
    }
    TcRow<P> q{p.rows, p.K, p.Ncols, img, size_t(2) * p.K * p.Ncols, p};
    const long long mtiles = (rows_cap + 127) / 128 + nseg;
    // split N when there are too few row tiles to fill the GPU (node-row GEMMs)
    int Nt = p.Ncols <= 256 ? p.Ncols : 256;  // column block per tile (<= one 256-col accumulator)
    // (one wave: the largest split whose tile count still fits the SMs)
    while (Nt > 32 && mtiles * (p.Ncols / Nt) * 2 <= sm && (Nt / 2) % 32 == 0) Nt /= 2;
    const int cap_ctas = c.tc_grid_mult > 0 ? c.row_sms * c.tc_grid_mult : (1 << 30);  // persistent when capped
    if constexpr (!TcRow<P>::kSeg) {  // CTA pairs (cta_group::2): half of B per SM, more A stages
      if (c.row_pair && nseg == 1 && !p.rows.perm && !p.rows.seg_off && Nt == p.Ncols && Nt % 32 == 0) {
        tc::RowPlan pp = tc::row_plan(p.K, Nt, 0, TcRow<P>::kSlabEpi, true);
        if (pp.resident) {
          set_smem(tc::tc_row_kernel<TcRow<P>, true>, pp.smem);
          const long long pairs = std::min<long long>((mtiles + 1) / 2, std::max(1, cap_ctas / 2));
          kl_cluster(tc::tc_row_kernel<TcRow<P>, true>, dim3(unsigned(2 * pairs)), dim3(tc::kRowThreads), pp.smem, st,
                     dim3(2, 1, 1), q, pp);
          return;
        }
      }
    }
    tc::RowPlan plan = tc::row_plan(p.K, Nt, TcRow<P>::kSeg ? tc::kSegKeyBytes : 0, TcRow<P>::kSlabEpi);
    plan.prefetch = c.row_prefetch;
    set_smem(tc::tc_row_kernel<TcRow<P>>, plan.smem);
    kl(tc::tc_row_kernel<TcRow<P>>, gridn(mtiles * (p.Ncols / Nt), 1, cap_ctas), tc::kRowThreads, plan.smem, st, q,
       plan);
    return;
  }
  if constexpr (TcRow<P>::kSeg || TcRow<P>::kAsync || TcOnly<P>::value) {  // tensor-core engine only
    fail(HMTL_ERR_INTERNAL, std::string(P::kName) + ": shape outside the tensor-core engine");
  } else {
    const long long tiles = ((rows_cap + 63) / 64 + nseg) * ((p.Ncols + 63) / 64);
    kl(gemm_ab_kernel<P>, gridn(tiles, 1, sm * 8), 256, 0, st, p);
  }
}

template <class P>
void atb(const P& p, Ctx& c, int nsplit, cudaStream_t st, long long rows_cap = 0) {
  if (c.dbg_skip_wgrad) return;  // timing experiments only (HMTL_DBG_SKIP_WGRAD)
  Prof pr(c, P::kName, st);
  const int M = p.K - P::kBias;
  const int NW = p.Ncols <= 256 ? p.Ncols : 256;  // accumulator width; wider outputs in slices
  if (c.use_tc && P::kTc && NW % 32 == 0 && p.Ncols % NW == 0 && M % 4 == 0) {
    const int mtiles = (M + 127) / 128;
    const long long chunks = (rows_cap > 0 ? rows_cap : (long long)c.Ec) / tc::KC + 1;
    // enough CTAs to fill the GPU, >= 4 chunks each (bounded partial traffic)
    // one wave over red_sms SMs (side-stream weight gradients leave the rest to the critical path)
    // head-segmented rows: segments differ in size (edge shares 1:1:1:2:3), so each gets up to
    // red_seg_mult x its even share of CTAs; CTAs past a short segment's chunks store zeros
    const long long segx = p.rows.nseg > 1 ? c.red_seg_mult : 1;
    long long want = std::max<long long>(1, (long long)c.red_sms_now * segx / (mtiles * p.rows.nseg));
    int ns = int(std::max<long long>(1, std::min<long long>(want, chunks / c.red_min_now)));
    float* partial = c.part(st);
    while (ns > 1 && size_t(p.rows.nseg) * ns * size_t(M + P::kBias) * NW > c.partial_cap) ns /= 2;
    // split clusters of `cl` CTAs reduce their partials through DSMEM first (tc.cuh)
    int cl = c.red_cluster;
    while (cl > 1 && ns < 2 * cl) cl /= 2;
    ns = ns / cl * cl;
    const dim3 cdim(1, unsigned(cl), 1);
    if constexpr (HasTma<P>::value) {  // plain row-major operands over contiguous rows: TMA path
      TmaOps o;
      p.tma(o);
      const int NT = p.Ncols <= 128 ? p.Ncols : 128;  // column slices of <= 128 (stage fits 3 in smem)
      const long long cap_rows = rows_cap > 0 ? rows_cap : (long long)c.Ec;
      CUtensorMap mx, mx1, my;
      const bool split_ok = !o.x1 || (o.xsplit % 128 == 0 && o.xsplit > 0);
      if (c.red_tma && o.x && o.y && split_ok && !p.rows.perm && p.Ncols % NT == 0 && NT % 32 == 0 &&
          size_t(p.rows.nseg) * ns * size_t(M + P::kBias) * NT <= c.partial_cap &&
          tc::tmap_2d(&mx, o.x, cap_rows, o.ldx) && (!o.x1 || tc::tmap_2d(&mx1, o.x1, cap_rows, o.ldx))) {
        const size_t SB = tc::red_stage_bytes(NT);
        const int stages = int(std::min<size_t>(4, (tc::kSmemLimit - size_t(32) * NT * 4 - 4096) / SB));
        const size_t smem = tc::tc_red_tma_smem(NT, stages);
        set_smem(tc::tc_red_tma_kernel<TcRed<P>>, smem);
        bool ok = true;
        for (int n0 = 0; n0 < p.Ncols && ok; n0 += NT) {
          ok = tc::tmap_2d(&my, o.y + n0, cap_rows, o.ldy);
          if (!ok) break;
          TcRed<P> q{p.rows, M, NT, P::kBias, p, n0};  // each slice sums its own bias columns
          if (cl > 1)
            kl_cluster(tc::tc_red_tma_kernel<TcRed<P>>, dim3(mtiles, ns, p.rows.nseg), tc::kRedTmaThreads, smem, st,
                       cdim, q, mx, o.x1 ? mx1 : mx, my, o.x1 ? o.xsplit : 0, partial, ns, stages);
          else
            kl(tc::tc_red_tma_kernel<TcRed<P>>, dim3(mtiles, ns, p.rows.nseg), tc::kRedTmaThreads, smem, st, q, mx,
               o.x1 ? mx1 : mx, my, o.x1 ? o.xsplit : 0, partial, ns, stages);
          tc::tc_red_reduce(q, partial, ns / cl, st);
        }
        if (ok) return;
      }
    }
    if (size_t(p.rows.nseg) * ns * size_t(M + P::kBias) * NW <= c.partial_cap) {
      const size_t smem = tc::tc_red_smem(NW);
      set_smem(tc::tc_red_kernel<TcRed<P>>, smem);
      for (int n0 = 0; n0 < p.Ncols; n0 += NW) {
        TcRed<P> q{p.rows, M, NW, P::kBias, p, n0};
        dim3 grid(mtiles, ns, p.rows.nseg);
        if (cl > 1)
          kl_cluster(tc::tc_red_kernel<TcRed<P>>, grid, tc::kRedThreads, smem, st, cdim, q, partial, ns,
                     tc::red_stages(NW));
        else
          kl(tc::tc_red_kernel<TcRed<P>>, grid, tc::kRedThreads, smem, st, q, partial, ns, tc::red_stages(NW));
        tc::tc_red_reduce(q, partial, ns / cl, st);
      }
      return;
    }
  }
  const int tiles = ((p.K + 63) / 64) * ((p.Ncols + 63) / 64);
  dim3 grid(tiles, nsplit, p.rows.nseg);
  kl(gemm_atb_kernel<P>, grid, 256, 0, st, p, c.part(st), nsplit);
  const long long total = (long long)p.K * p.Ncols * p.rows.nseg;
  kl(gemm_atb_reduce<P>, gridn(total, 256, c.sm_count * 8), 256, 0, st, p, c.part(st), nsplit);
}

// fused node-row GEMM chain (chain.cuh) over the prebuilt B images of the next
// `G` tensor-core GEMMs in recorded call order; false = use the unfused path
bool chain_ok(const Ctx& c) {
  return c.use_tc && c.bimg_ready && c.fuse_chain && c.H % 32 == 0 && c.H <= 128;
}
// the recording step's GEMMs that later steps run inside CTA-pair chains get the pair image layout
int chain_rec_halves(const Ctx& c) {
  return c.use_tc && c.fuse_chain && c.chain_pair && c.H % 32 == 0 && c.H <= 128 ? 2 : 0;
}
struct RecHalves {  // scope: jobs recorded inside carry the pair layout tag
  Ctx& c;
  RecHalves(Ctx& c_, bool on) : c(c_) { c.rec_halves = on ? chain_rec_halves(c) : 0; }
  ~RecHalves() { c.rec_halves = 0; }
};
void launch_chain(Ctx& c, const char* name, int G, const chain::Gemm* gs, cudaStream_t st) {
  Prof pr(c, name, st);
  chain::Chain q{};
  q.count = &c.hdr->N;
  q.G = G;
  q.H = c.H;
  for (int i = 0; i < G; ++i) {
    q.g[i] = gs[i];
    q.g[i].img = c.bjobs[c.bimg_idx++].out;
  }
  {  // stamps of the chains named HMTL_CHAIN_STAMP_NAME (any chain when unset; the last launch wins)
    static const char* sel = std::getenv("HMTL_CHAIN_STAMP_NAME");
    q.stamps = (!sel || !std::strcmp(sel, name)) ? c.chain_stamps : nullptr;
  }
  q.dbg = c.chain_dbg;
  q.rows_cap = int(c.Nc);
  q.prefetch = c.chain_prefetch;
  // node rows per CTA (128 or 64): the forward chains run alone on the GPU, so 64-row CTAs
  // (twice the CTAs) pay off there; the backward's share the SMs with weight gradients
  const bool fwd = name[0] == 'f';
  const int mr = fwd && c.chain_mr_fwd ? c.chain_mr_fwd : c.chain_mr;
  const int grid = int((c.Nc + mr - 1) / mr);
  // CS-CTA clusters split every GEMM's columns (chained operand exchanged through DSMEM)
  int cs = c.chain_cs;
  for (int i = 0; i < G; ++i)
    while (cs > 1 && (gs[i].N / cs) % 32 != 0) cs /= 2;
  const bool split = cs == 2, quad = cs == 4;
  auto go = [&](auto kern, int cs) {
    set_smem(kern, chain::kSmem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid * cs);
    cfg.blockDim = dim3(chain::kThreads);
    cfg.dynamicSmemBytes = chain::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[3];
    int n = 0;
    if (pdl_enabled()) {
      at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[n++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (launch_prio().on) {  // (as kl: critical-path kernels dispatch first)
      at[n].id = cudaLaunchAttributePriority;
      at[n++].val.priority = st == launch_prio().hi_stream ? launch_prio().hi : launch_prio().lo;
    }
    if (cs > 1) {
      at[n].id = cudaLaunchAttributeClusterDimension;
      at[n].val.clusterDim.x = cs, at[n].val.clusterDim.y = 1, at[n++].val.clusterDim.z = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    cudaLaunchKernelEx(&cfg, kern, q);
  };
  using namespace chain;
  const int r0 = gs[0].role, r1 = G > 1 ? gs[1].role : -1, r2 = G > 2 ? gs[2].role : -1;
  if (c.chain_pair) {  // CTA-pair kernels over pair-layout B images
    // GEMM 1's A operand as TMA tiles (32 k x 128 rows, 128 B swizzle = the K-major SW128 operand layout)
    CUtensorMap ma0{}, ma1{};
    {
      const chain::Gemm& g = gs[0];
      const float* a0 = g.role == kFwdNode1 || g.role == kFwdP ? g.x0 : g.x1;
      const int ld0 = g.role == kBwdL11 ? 2 * c.H : c.H;
      bool ok = tc::tmap_2d(&ma0, a0, c.Nc, ld0, CU_TENSOR_MAP_SWIZZLE_128B, 128);
      if (g.role == kFwdNode1) ok = ok && tc::tmap_2d(&ma1, g.x1, c.Nc, c.H, CU_TENSOR_MAP_SWIZZLE_128B, 128);
      else ma1 = ma0;
      if (!ok) {
        std::fprintf(stderr, "hmtl: chain A tensor map\n");
        std::abort();
      }
    }
    for (int i = 0; i < G; ++i)
      if (!c.bjobs[c.bimg_idx - G + i].halves) {
        std::fprintf(stderr, "hmtl: chain B image %d not in the pair layout\n", c.bimg_idx - G + i);
        std::abort();
      }
    auto gop = [&](auto kern) {
      set_smem(kern, pairk::kSmem);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(unsigned((c.Nc + 255) / 256 * 2));
      cfg.blockDim = dim3(pairk::kThreads);
      cfg.dynamicSmemBytes = pairk::kSmem;
      cfg.stream = st;
      cudaLaunchAttribute at[2];
      int n = 0;
      if (pdl_enabled()) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n++].val.programmaticStreamSerializationAllowed = 1;
      }
      at[n].id = cudaLaunchAttributeClusterDimension;
      at[n].val.clusterDim.x = 2, at[n].val.clusterDim.y = 1, at[n++].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = n;
      cudaLaunchKernelEx(&cfg, kern, q, ma0, ma1);
    };
    if (r0 == kFwdNode1 && r1 == kFwdNode2 && r2 == kFwdP) gop(pair_kernel<kFwdNode1, kFwdNode2, kFwdP>);
    else if (r0 == kFwdNode1 && r1 == kFwdNode2 && r2 < 0) gop(pair_kernel<kFwdNode1, kFwdNode2, -1>);
    else if (r0 == kBwdL11 && r1 == kBwdL1 && r2 == kBwdL4) gop(pair_kernel<kBwdL11, kBwdL1, kBwdL4>);
    else if (r0 == kBwdL1 && r1 == kBwdL4 && r2 < 0) gop(pair_kernel<kBwdL1, kBwdL4, -1>);
    return;
  }
  auto pick = [&](auto k128_1, auto k128_2, auto k128_4, auto k64_2) {
    if (mr == 64 && split) go(k64_2, 2);
    else if (quad) go(k128_4, 4);
    else if (split) go(k128_2, 2);
    else go(k128_1, 1);
  };
  if (r0 == kFwdNode1 && r1 == kFwdNode2 && r2 == kFwdP)
    pick(chain_kernel<kFwdNode1, kFwdNode2, kFwdP>, chain_kernel<kFwdNode1, kFwdNode2, kFwdP, 2>,
         chain_kernel<kFwdNode1, kFwdNode2, kFwdP, 4>, chain_kernel<kFwdNode1, kFwdNode2, kFwdP, 2, 64>);
  else if (r0 == kFwdNode1 && r1 == kFwdNode2 && r2 < 0)
    pick(chain_kernel<kFwdNode1, kFwdNode2, -1>, chain_kernel<kFwdNode1, kFwdNode2, -1, 2>,
         chain_kernel<kFwdNode1, kFwdNode2, -1, 4>, chain_kernel<kFwdNode1, kFwdNode2, -1, 2, 64>);
  else if (r0 == kBwdL11 && r1 == kBwdL1 && r2 == kBwdL4)
    pick(chain_kernel<kBwdL11, kBwdL1, kBwdL4>, chain_kernel<kBwdL11, kBwdL1, kBwdL4, 2>,
         chain_kernel<kBwdL11, kBwdL1, kBwdL4, 4>, chain_kernel<kBwdL11, kBwdL1, kBwdL4, 2, 64>);
  else if (r0 == kBwdL1 && r1 == kBwdL4 && r2 < 0)
    pick(chain_kernel<kBwdL1, kBwdL4, -1>, chain_kernel<kBwdL1, kBwdL4, -1, 2>, chain_kernel<kBwdL1, kBwdL4, -1, 4>,
         chain_kernel<kBwdL1, kBwdL4, -1, 2, 64>);
}

RowSet node_rows(Ctx& c) {
  RowSet r;
  r.count = &c.hdr->N;
  return r;
}
RowSet edge_rows(Ctx& c) {
  RowSet r;
  r.count = &c.hdr->E;
  return r;
}
// (head-sorted batches: the head-sorted orders are the identity -- no permutation)
RowSet node_rows_by_head(Ctx& c) {
  RowSet r;
  r.perm = c.head_sorted ? nullptr : c.node_perm;
  r.seg_off = c.hdr->seg_node;
  r.nseg = c.S;
  return r;
}
RowSet edge_rows_by_head(Ctx& c) {
  RowSet r;
  r.perm = c.head_sorted ? nullptr : c.edge_perm;
  r.seg_off = c.hdr->seg_edge;
  r.nseg = c.S;
  return r;
}
RowSet graph_rows_by_head(Ctx& c) {
  RowSet r;
  r.perm = c.head_sorted ? nullptr : c.gperm;
  r.seg_off = c.hdr->seg_graph;
  r.nseg = c.S;
  return r;
}

}  // namespace

namespace {
__global__ void agg4_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr, const float* __restrict__ z2,
                            float* __restrict__ agg, int H);
__global__ void agg_fix_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr, const float* __restrict__ tp,
                               int tcap, float* __restrict__ agg, int H);


// ---- elementwise producers of the tensor-core A operands.  Warp per group of
// kEwU edges, lane = float4 column group: the per-edge indices are warp-uniform
// loads and every row load of the group is issued before the math.
constexpr int kEwU = 4;
// a1 = silu(z1), z1 = (P_a[dst] + P_b[src]) + d2 w + b1
__global__ void __launch_bounds__(256) edge_a1_kernel(const DevHdr* hdr, const float* __restrict__ P,
                                                      const int* __restrict__ dst, const int* __restrict__ src,
                                                      const float4* __restrict__ geo, const float* __restrict__ wd,
                                                      const float* __restrict__ b1, float* __restrict__ a1,
                                                      float* __restrict__ s1p, int H, int pre) {
  pdl_wait();
  const int E = hdr->E, lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int eb = gw * kEwU; eb < E; eb += nw * kEwU) {
    for (int c = lane * 4; c < H; c += 128) {
      const float4 w = ld4(wd + c), bb = ld4(b1 + c);
      float4 pa[kEwU], pb[kEwU];
      float d2[kEwU];
#pragma unroll
      for (int u = 0; u < kEwU; ++u) {
        const int e = min(eb + u, E - 1);
        pa[u] = ld4(P + size_t(dst[e]) * 2 * H + c);
        pb[u] = ld4(P + size_t(src[e]) * 2 * H + H + c);
        d2[u] = geo[e].w;
      }
#pragma unroll
      for (int u = 0; u < kEwU; ++u)
        if (eb + u < E) {
          const float4 z = pre4(pa[u], pb[u], d2[u], w, bb);
          st4(a1 + size_t(eb + u) * H + c, pre ? z : silu4(z));  // (pre: z1 itself; consumers apply silu/silu')
          if (s1p) st4(s1p + size_t(eb + u) * H + c, sgrad4(z));  // silu'(z1) for the backward's dz1 epilogue
        }
    }
  }
}
// backward: dz2 = dagg[dst] * silu'(z2) and s1p = silu'(z1)
__global__ void __launch_bounds__(256) edge_bwd_prep_kernel(const DevHdr* hdr, const float* __restrict__ P,
                                                            const int* __restrict__ dst, const int* __restrict__ src,
                                                            const float4* __restrict__ geo,
                                                            const float* __restrict__ wd, const float* __restrict__ b1,
                                                            const float* __restrict__ dagg,
                                                            const float* __restrict__ z2, float* __restrict__ dz2,
                                                            float* __restrict__ s1p, int H) {
  pdl_wait();
  const int E = hdr->E, lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int eb = gw * kEwU; eb < E; eb += nw * kEwU) {
    for (int c = lane * 4; c < H; c += 128) {
      const float4 w = ld4(wd + c), bb = ld4(b1 + c);
      float4 pa[kEwU], pb[kEwU], ga[kEwU], zz[kEwU];
      float d2[kEwU];
#pragma unroll
      for (int u = 0; u < kEwU; ++u) {
        const int e = min(eb + u, E - 1), d = dst[e];
        pa[u] = ld4(P + size_t(d) * 2 * H + c);
        pb[u] = ld4(P + size_t(src[e]) * 2 * H + H + c);
        ga[u] = ld4(dagg + size_t(d) * H + c);
        zz[u] = ld4(z2 + size_t(e) * H + c);
        d2[u] = geo[e].w;
      }
#pragma unroll
      for (int u = 0; u < kEwU; ++u)
        if (eb + u < E) {
          const size_t o = size_t(eb + u) * H + c;
          st4(dz2 + o, mul4(ga[u], sgrad4(zz[u])));
          st4(s1p + o, sgrad4(pre4(pa[u], pb[u], d2[u], w, bb)));
        }
    }
  }
}
// force head layer 0: af0 = silu(zf0), sf0 = silu'(zf0) with the edge's head weights
// (warp per group of kEwU edges, lane = float4 column group, as edge_a1_kernel)
__global__ void __launch_bounds__(256) edge_af0_kernel(const DevHdr* hdr, const float* __restrict__ Qf,
                                                       const int* __restrict__ dst, const int* __restrict__ src,
                                                       const float* __restrict__ dist,
                                                       const int* __restrict__ node_graph,
                                                       const int* __restrict__ gslot, const float* __restrict__ heads,
                                                       size_t PH, size_t off_wd, size_t off_b0,
                                                       float* __restrict__ af0, float* __restrict__ sf0, int W) {
  pdl_wait();
  const int E = hdr->E, lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int eb = gw * kEwU; eb < E; eb += nw * kEwU) {
    int d[kEwU], sl[kEwU];
#pragma unroll
    for (int u = 0; u < kEwU; ++u) {
      const int e = min(eb + u, E - 1);
      d[u] = dst[e];
      sl[u] = gslot[node_graph[d[u]]];
    }
    bool uni = true;  // (head-sorted batches: the group's edges nearly always share one head)
#pragma unroll
    for (int u = 1; u < kEwU; ++u) uni = uni && sl[u] == sl[0];
    for (int c = lane * 4; c < W; c += 128) {
      float4 qa[kEwU], qb[kEwU], w[kEwU], b[kEwU];
      float r[kEwU];
      if (uni) {
        const float* hb = heads + size_t(sl[0]) * PH;
        w[0] = ldu4(hb + off_wd + c);
        b[0] = ldu4(hb + off_b0 + c);
#pragma unroll
        for (int u = 1; u < kEwU; ++u) w[u] = w[0], b[u] = b[0];
      }
#pragma unroll
      for (int u = 0; u < kEwU; ++u) {
        const int e = min(eb + u, E - 1);
        qa[u] = ld4(Qf + size_t(d[u]) * W + c);
        qb[u] = ld4(Qf + size_t(src[e]) * W + c);
        if (!uni) {
          const float* hb = heads + size_t(sl[u]) * PH;
          w[u] = ldu4(hb + off_wd + c);
          b[u] = ldu4(hb + off_b0 + c);
        }
        r[u] = dist[e];
      }
#pragma unroll
      for (int u = 0; u < kEwU; ++u)
        if (eb + u < E) {
          const float4 z = pre4(qa[u], qb[u], r[u], w[u], b[u]);
          const size_t o = size_t(eb + u) * W + c;
          st4(af0 + o, silu4(z));
          if (sf0) st4(sf0 + o, sgrad4(z));
        }
    }
  }
}
}  // namespace

namespace {
// force MLP output layer (width 1; mlp_forward_'s last layer, hmtl/model.hpp:282-306):
// s_e = x_e . w_slot + b_slot, x_e = silu(zf_{i-1}[e]) (act) or the materialised
// silu(zf0).  8 lanes per edge, fixed lane split + xor tree: deterministic.
__global__ void force_out_fwd_kernel(const DevHdr* hdr, const float* __restrict__ x, int act,
                                     const int* __restrict__ dst, const int* __restrict__ node_graph,
                                     const int* __restrict__ gslot, const float* __restrict__ heads, size_t PH,
                                     size_t off_w, size_t off_b, float* __restrict__ s, int W) {
  pdl_wait();
  const int l8 = threadIdx.x & 7;
  const unsigned gm = 0xffu << (threadIdx.x & 24);
  const long long E = hdr->E;
  const long long step = ((long long)gridDim.x * blockDim.x) >> 3;
  for (long long e = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 3; e < E; e += step) {
    const float* hb = heads + size_t(gslot[node_graph[dst[e]]]) * PH;
    const float* xr = x + size_t(e) * W;
    float acc = 0.f;
    for (int k = l8 * 4; k < W; k += 32) {
      float4 v = ld4(xr + k);
      if (act) v = silu4(v);
      const float4 w = ldu4(hb + off_w + k);
      acc += v.x * w.x + v.y * w.y + v.z * w.z + v.w * w.w;
    }
    acc += __shfl_xor_sync(gm, acc, 4);
    acc += __shfl_xor_sync(gm, acc, 2);
    acc += __shfl_xor_sync(gm, acc, 1);
    if (l8 == 0) s[e] = acc + hb[off_b];
  }
}
}  // namespace

namespace {
// width-1 force output layer through the dedicated kernels (x row = W floats, 16 B aligned)
bool force_out_fast(const Ctx& c, int i) { return c.W % 4 == 0 && c.W <= 256 && (i >= 2 || c.store_af0); }
}  // namespace

// engine ablation bits of this translation unit's tc kernels (timing experiments only)
void set_tc_debug(int bits) { cudaMemcpyToSymbol(tc::g_tc_debug, &bits, sizeof(int)); }

void launch_bimg_all(Ctx& c, cudaStream_t st) {
  if (c.bjobs.empty()) return;
  if (!c.d_bjobs || c.n_djobs < int(c.bjobs.size())) {  // lay out the image buffer once
    size_t total = 0;
    for (auto& j : c.bjobs) total += size_t(2) * j.K * j.N * j.nseg;
    if (c.bimg_all) cudaFree(c.bimg_all);
    if (c.d_bjobs) cudaFree(c.d_bjobs);
    cudaMalloc(&c.bimg_all, total * 4);
    c.bimg_all_cap = total;
    size_t off = 0;
    for (auto& j : c.bjobs) {
      j.out = c.bimg_all + off;
      off += size_t(2) * j.K * j.N * j.nseg;
    }
    cudaMalloc(&c.d_bjobs, c.bjobs.size() * sizeof(BDesc));
    cudaMemcpy(c.d_bjobs, c.bjobs.data(), c.bjobs.size() * sizeof(BDesc), cudaMemcpyHostToDevice);
    c.n_djobs = int(c.bjobs.size());
    c.bimg_rows = 1;
    for (auto& j : c.bjobs) c.bimg_rows = std::max(c.bimg_rows, j.K * j.N * j.nseg);  // elements
  }
  Prof pr(c, "bimg_all", st);
  // a few CTAs per image (grid-stride): the rebuild overlaps the batch preparation and
  // neighbour list without taking every SM from those small critical-path kernels
  kl(bimg_all_kernel, dim3(std::min({(c.bimg_rows / 4 + 255) / 256, c.bimg_blocks}), c.n_djobs), 256, 0, st,
     c.d_bjobs);
  c.bimg_ready = true;
  c.bimg_recording = false;
}

// layer 0's P table per species: T = embed [W1a | W1b] (NS rows), from the weights alone,
// on the B-image side stream at the step start; the embed kernel then gathers P0 = T[species]
// (the same tensor-core GEMM per row as the node-row P GEMM it replaces)
bool ptab_ok(const Ctx& c) {
  return c.ptab_on && c.use_tc && c.bimg_ready && !c.bimg_recording && !c.bjobs.empty() && !c.bjobs[0].halves &&
         c.H % 32 == 0 && c.ptab;
}
void launch_ptab(Ctx& c, cudaStream_t st) {
  c.ptab_ready = ptab_ok(c);
  if (!c.ptab_ready) return;
  const int H = c.H;
  RowSet rows{nullptr, nullptr, c.d_ns, 1};
  PProb q{rows, H, 2 * H, H, c.shared_param("embed"), c.params + c.shared_off("layer0.edge.W1"), c.ptab};
  ab(q, c.NS, 1, st, c.sm_count, c, c.bjobs[0].out);
}

void launch_forward(Ctx& c, cudaStream_t st) {
  c.bimg_idx = 0;
  const int H = c.H, W = c.W, L = c.L, D = c.D, sm = c.sm_count;
  const size_t NH = size_t(c.Nc) * H, EH = size_t(c.Ec) * H;
  {
    Prof pr(c, "fwd.embed", st);
    kl(embed_kernel, gridn(NH, 256, sm * 16), 256, 0, st, c.hdr, c.species, c.shared_param("embed"), c.hs, H,
       c.ptab_ready ? c.ptab : nullptr, c.P);
  }
  bool p_done = c.ptab_ready;  // P of this layer already produced (by the previous node chain / the species table)
  if (c.ptab_ready) ++c.bimg_idx;  // (layer 0's P GEMM image, used by launch_ptab)
  for (int l = 0; l < L; ++l) {
    const std::string p = "layer" + std::to_string(l) + ".";
    const float* h = c.hs + size_t(l) * NH;
    float* hn = c.hs + size_t(l + 1) * NH;
    float* P = c.P + size_t(l) * 2 * NH;
    float* z2 = c.z2 + size_t(l) * EH;
    float* agg = c.agg + size_t(l) * NH;
    float* vz1 = c.vz1 + size_t(l) * NH;
    const float* W1 = c.params + c.shared_off(p + "edge.W1");
    if (!p_done) {
      RecHalves rh(c, l > 0);  // (layer 0's P is never inside a chain)
      PProb q{node_rows(c), H, 2 * H, H, h, W1, P};
      ab(q, c.Nc, 1, st, sm, c);
    }
    p_done = false;
    if (c.store_a1 && c.async_fwd && !c.fuse_edge) {  // cp.async gather producer -> GEMM (a1, s1p, z2)
      MsgAsyncProb q{edge_rows(c), H, H, H, P, W1 + size_t(2) * H * H, c.params + c.shared_off(p + "edge.b1"),
                     c.params + c.shared_off(p + "edge.W2"), c.params + c.shared_off(p + "edge.b2"), c.edge_dst,
                     c.edge_src, c.geo, z2, c.a1 + size_t(l) * EH, c.s1pb + size_t(l) * EH};
      ab(q, c.Ec, 1, st, sm, c);
      Prof pr(c, "fwd.agg_segsum", st);
      kl(agg4_kernel, gridn((long long)c.Nc * 32, 256, sm * 16), 256, 0, st, c.hdr, c.row_ptr, z2, agg, H);
    } else if (c.store_a1 && c.fuse_edge) {  // gather -> GEMM -> z2 + per-destination sum, one pass
      MsgSegProb q{edge_rows(c), H, H, H, P, W1 + size_t(2) * H * H, c.params + c.shared_off(p + "edge.b1"),
                   c.params + c.shared_off(p + "edge.W2"), c.params + c.shared_off(p + "edge.b2"), c.edge_dst,
                   c.edge_src, c.geo, z2, c.a1 + size_t(l) * EH, agg, c.tpart, c.tcap};
      ab(q, c.Ec, 1, st, sm, c);
      Prof pr(c, "fwd.agg_fix", st);
      kl(agg_fix_kernel, gridn((long long)c.Nc * (H / 4), 256, sm * 4), 256, 0, st, c.hdr, c.row_ptr, c.tpart, c.tcap,
         agg, H);
    } else {
    if (c.store_a1) {
      Prof pr(c, "fwd.edge_act", st);
      kl(edge_a1_kernel, gridn((c.Ec + kEwU - 1) / kEwU * 32, 256, sm * 16), 256, 0, st,
          c.hdr, P, c.edge_dst, c.edge_src, c.geo, W1 + size_t(2) * H * H, c.params + c.shared_off(p + "edge.b1"),
          c.a1 + size_t(l) * EH, c.async_bwd == 1 && !c.z1_only ? c.s1pb + size_t(l) * EH : nullptr, H,
          c.z1_only ? 1 : 0);
    }
    if (c.store_a1 && c.z1_only) {
      MsgZ1Prob q{edge_rows(c), H, H, H, c.a1 + size_t(l) * EH, c.params + c.shared_off(p + "edge.W2"),
                  c.params + c.shared_off(p + "edge.b2"), z2};
      ab(q, c.Ec, 1, st, sm, c);
    } else {
      MsgProb q{edge_rows(c), H, H, H, P, W1 + size_t(2) * H * H, c.params + c.shared_off(p + "edge.b1"),
                c.params + c.shared_off(p + "edge.W2"), c.params + c.shared_off(p + "edge.b2"), c.edge_dst,
                c.edge_src, c.geo, z2, c.store_a1 ? c.a1 + size_t(l) * EH : nullptr};
      ab(q, c.Ec, 1, st, sm, c);
    }
    {
      Prof pr(c, "fwd.agg_segsum", st);
      if (H % 4 == 0) kl(agg4_kernel, gridn((long long)c.Nc * 32, 256, sm * 16), 256, 0, st, c.hdr, c.row_ptr, z2, agg, H);
      else kl(agg_kernel, gridn((long long)c.Nc * 32, 256, sm * 16), 256, 0, st, c.hdr, c.row_ptr, z2, agg, H);
    }
    }
    if (chain_ok(c)) {  // node MLP + residual (+ the next layer's P) in one launch
      const int G = l + 1 < L ? 3 : 2;
      chain::Gemm gs[3] = {
          {chain::kFwdNode1, 2 * H, H, nullptr, h, agg, c.params + c.shared_off(p + "node.b1"), vz1, nullptr},
          {chain::kFwdNode2, H, H, nullptr, h, nullptr, c.params + c.shared_off(p + "node.b2"), hn, nullptr},
          {chain::kFwdP, H, 2 * H, nullptr, nullptr, nullptr, nullptr, c.P + size_t(l + 1) * 2 * NH, nullptr}};
      launch_chain(c, "fwd.node_chain", G, gs, st);
      p_done = l + 1 < L;
      continue;
    }
    {
      RecHalves rh(c, true);
      Node1Prob q{node_rows(c), 2 * H, H, H, h, agg, c.params + c.shared_off(p + "node.W1"),
                  c.params + c.shared_off(p + "node.b1"), vz1};
      ab(q, c.Nc, 1, st, sm, c);
    }
    {
      RecHalves rh(c, true);
      Node2Prob q{node_rows(c), H, H, H, vz1, c.params + c.shared_off(p + "node.W2"),
                  c.params + c.shared_off(p + "node.b2"), h, hn};
      ab(q, c.Nc, 1, st, sm, c);
    }
  }
  const float* hL = c.hs + size_t(L) * NH;
  // energy branch (side stream; independent of the force branch until the loss)
  cudaStream_t se = c.side(c.s_e, st);
  c.dep(st, se);
  if (D >= 2 && D <= kEhMaxD && H % 4 == 0 && W % 4 == 0 && W <= 256 && H <= 512) {
    Prof pr(c, "fwd.energy_head", se);
    EHeadArgs a{c.head_params(), c.PH, {}, {}, D, H, W};
    for (int i = 0; i < D; ++i) {
      a.w[i] = c.head_off("energy.W" + std::to_string(i));
      a.b[i] = c.head_off("energy.b" + std::to_string(i));
    }
    const size_t smem = (size_t(2) * kEhRows * std::max(H, W) + size_t(kEhKC) * W) * sizeof(float);
    set_smem(energy_head_kernel, smem);
    const dim3 grid(std::min((c.Gc + kEhRows - 1) / kEhRows, 32), c.S);
    kl(energy_head_kernel, grid, 256, smem, se, c.hdr, graph_rows_by_head(c), c.graph_offset, hL, a, c.pooled, c.ez,
       c.Gc, c.energy);
  } else {
    {
      Prof pr(c, "fwd.pool", se);
      kl(pool_kernel, gridn((long long)c.Gc * 32, 256, sm * 8), 256, 0, se, c.hdr, c.graph_offset, hL, c.pooled, H);
    }
    for (int i = 0; i < D; ++i) {
      const int last = i == D - 1;
      EnergyProb q{graph_rows_by_head(c), i == 0 ? H : W, last ? 1 : W, H, W, i, last, c.pooled,
                   i ? c.ez + size_t(i - 1) * c.Gc * W : nullptr,
                   HeadW{c.head_params(), c.PH, c.head_off("energy.W" + std::to_string(i))},
                   HeadW{c.head_params(), c.PH, c.head_off("energy.b" + std::to_string(i))},
                   c.ez + size_t(i) * c.Gc * W, c.energy};
      ab(q, c.Gc, c.S, se, sm, c);
    }
  }
  // force branch
  {
    QfProb q{node_rows_by_head(c), H, W, H, W, hL, HeadW{c.head_params(), c.PH, c.head_off("force.W0")}, c.Qf};
    ab(q, c.Nc, c.S, st, sm, c);
  }
  const size_t wf0 = c.head_off("force.W0");
  if (c.store_af0) {
    Prof pr(c, "fwd.force_act", st);
    kl(edge_af0_kernel, gridn((c.Ec + kEwU - 1) / kEwU * 32, 256, sm * 16), 256, 0, st,
        c.hdr, c.Qf, c.edge_dst, c.edge_src, c.dist, c.node_graph, c.gslot, c.head_params(), c.PH,
        wf0 + size_t(H) * W, c.head_off("force.b0"), c.af0, c.store_sf0 ? c.sf0 : nullptr, W);
  }
  for (int i = 1; i < D; ++i) {
    const int last = i == D - 1;
    if (last && force_out_fast(c, i)) {
      Prof pr(c, "fwd.force_out", st);
      kl(force_out_fwd_kernel, gridn((long long)c.Ec * 8, 256, sm * 16), 256, 0, st,
          c.hdr, i >= 2 ? c.zf + size_t(i - 2) * c.Ec * W : c.af0, i >= 2, c.edge_dst, c.node_graph, c.gslot,
          c.head_params(), c.PH, c.head_off("force.W" + std::to_string(i)),
          c.head_off("force.b" + std::to_string(i)), c.s, W);
      continue;
    }
    ForceProb q{edge_rows_by_head(c), W, last ? 1 : W, H, W, i, last, c.Ec, c.Qf, c.zf, c.dist, c.edge_dst,
                c.edge_src, HeadW{c.head_params(), c.PH, wf0 + size_t(H) * W},
                HeadW{c.head_params(), c.PH, c.head_off("force.b0")},
                HeadW{c.head_params(), c.PH, c.head_off("force.W" + std::to_string(i))},
                HeadW{c.head_params(), c.PH, c.head_off("force.b" + std::to_string(i))}, c.zf, c.s,
                c.store_af0 ? c.af0 : nullptr};
    ab(q, c.Ec, c.S, st, sm, c);
  }
  {
    Prof pr(c, "fwd.forces_segsum", st);
    kl(forces_kernel, gridn((long long)c.Nc * 32, 256, sm * 16), 256, 0, st, c.hdr, c.row_ptr, c.geo, c.s, c.forces);
  }
  c.dep(se, st);
  {
    Prof pr(c, "fwd.finite", st);
    kl(finite_kernel, gridn(c.Gc + 3LL * c.Nc, 256, sm * 4), 256, 0, st, c.hdr, c.energy, c.forces);
  }
}

// ----------------------------------------------------------------- loss
// SPEC.md:383-391; one CTA, warp per graph, fixed-order reductions.
namespace {
__global__ void __launch_bounds__(256) loss_kernel(DevHdr* hdr, const uint8_t* __restrict__ arena,
                                                   const int* __restrict__ graph_offset,
                                                   const float* __restrict__ energy, const float* __restrict__ F,
                                                   float* __restrict__ dE, float* __restrict__ dF, double* terms,
                                                   float w_e, float w_f) {
  pdl_wait();
  __shared__ bool last;
  const int G = hdr->G, N = hdr->N;
  const ArenaLayout al = arena_layout(G, N);
  const double* le = reinterpret_cast<const double*>(arena + al.le);
  const double* lf = reinterpret_cast<const double*>(arena + al.lf);
  const int lane = threadIdx.x & 31;
  // warp per graph: w_E (E^ - E)^2 + w_F mean_i |F^_i - F_i|^2 and the upstreams
  for (int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < G; g += (gridDim.x * blockDim.x) >> 5) {
    const int lo = graph_offset[g], hi = graph_offset[g + 1];
    const double n = double(hi - lo);
    double fe = 0.0;
    for (int t = 3 * lo + lane; t < 3 * hi; t += 32) {
      const double r = double(F[t]) - lf[t];
      fe += r * r;
      dF[t] = float(2.0 * double(w_f) * r / (n * double(G)));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) fe += __shfl_xor_sync(0xffffffffu, fe, o);
    const double de = double(energy[g]) - le[g];
    if (lane == 0) {
      terms[g] = double(w_e) * de * de + double(w_f) * fe / n;
      dE[g] = float(2.0 * double(w_e) * de / double(G));
    }
  }
  // the last CTA to finish sums the per-graph terms in graph order (deterministic)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&hdr->loss_done, 1) == int(gridDim.x) - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double part[256];
  double a = 0.0;
  for (int g = threadIdx.x; g < G; g += blockDim.x) a += terms[g];
  part[threadIdx.x] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < int(blockDim.x); ++i) t += part[i];
    hdr->loss = t / double(G);
    hdr->loss_done = 0;
  }
}
}  // namespace

void launch_loss(Ctx& c, float w_e, float w_f, cudaStream_t st) {
  {
    Prof pr(c, "loss", st);
    kl(loss_kernel, gridn((long long)c.Gc * 32, 256, c.sm_count * 2), 256, 0, st, c.hdr, c.arena, c.graph_offset, c.energy, c.forces,
       c.dE, c.dF, c.loss_terms, w_e, w_f);
  }
}

// ================================================================ backward
namespace {

// A^T B problems: store(seg, k, n, v) writes the gradient element
struct EGradProb {  // energy MLP layer i weight+bias
  static constexpr const char* kName = "bwd.energy_wgrad";
  static constexpr int kBias = 1;
  static constexpr bool kTc = true;
  __device__ float4 x4(int, int g, int m) const {
    return layer == 0 ? ld4(pooled + size_t(g) * H + m) : silu4(ld4(ezp + size_t(g) * W + m));
  }
  __device__ float4 y4(int, int g, int n) const { return ld4(dz + size_t(g) * ldz + n); }
  RowSet rows;
  int K, Ncols, H, W, layer;  // K = in + 1
  const float *pooled, *ezp, *dz;
  int ldz;
  HeadG G;
  __device__ float a(int, int g, int k) const {
    if (k == K - 1) return 1.f;
    return layer == 0 ? pooled[size_t(g) * H + k] : silu(ezp[size_t(g) * W + k]);
  }
  __device__ float b(int, int g, int n) const { return dz[size_t(g) * ldz + n]; }
  __device__ void store(int seg, int k, int n, float v) const { G.at(seg)[size_t(k) * Ncols + n] = v; }
};
// dx = dz W^T, epilogue dz_prev = dx * silu'(z_prev) (or plain dpooled)
struct EDxProb {
  BDesc bd() const { return BDesc{Wt.base + Wt.off, nullptr, 0, 0, 1, K, K, Ncols, rows.nseg, (long long)Wt.PH, nullptr}; }
  static constexpr const char* kName = "bwd.energy_dx";
  RowSet rows;
  int K, Ncols, W, H;  // K = out_i, Ncols = in_i
  const float *dz, *zprev;
  int ldz;
  HeadW Wt;
  float* out;
  int ldo, act;
  __device__ float a(int, int g, int k) const { return dz[size_t(g) * ldz + k]; }
  __device__ float b(int seg, int k, int n) const { return Wt.at(seg)[size_t(n) * K + k]; }
  __device__ void epi(int, int g, int n, float acc) const {
    out[size_t(g) * ldo + n] = act ? acc * silu_grad(zprev[size_t(g) * W + n]) : acc;
  }
};

struct FGradProb {  // force MLP layer i >= 1 weight+bias (edge rows per head)
  static constexpr const char* kName = "bwd.force_edge_wgrad";
  static constexpr int kBias = 1;
  static constexpr bool kTc = true;
  __device__ float4 x4(int seg, int e, int m) const {
    if (layer == 1) {
      if (af0s) return ld4(af0s + size_t(e) * W + m);
      return silu4(pre4(ld4(Qf + size_t(dst[e]) * W + m), ld4(Qf + size_t(src[e]) * W + m), dist[e],
                        ldu4(Wd.at(seg) + m), ldu4(B0.at(seg) + m)));
    }
    return silu4(ld4(zf + size_t(layer - 2) * Ec * W + size_t(e) * W + m));
  }
  __device__ float4 y4(int, int e, int n) const { return ld4(dz + size_t(e) * ldz + n); }
  RowSet rows;
  int K, Ncols, H, W, layer;
  long long Ec;
  const float *Qf, *zf, *dist, *dz;
  int ldz;
  const int *dst, *src;
  HeadW Wd, B0;
  HeadG G;
  const float* af0s;  // silu(zf0) materialised by the forward producer (nullable)
  // TMA operands when the head-segmented rows are contiguous (head-sorted batch): X = silu(zf0)
  void tma(TmaOps& o) const {
    if (layer == 1 && af0s) o.x = af0s, o.ldx = W, o.y = dz, o.ldy = ldz;
  }
  __device__ float a(int seg, int e, int k) const {
    if (k == K - 1) return 1.f;
    if (layer == 1) return silu(zf0_of(Qf, W, dst[e], src[e], dist[e], Wd.at(seg), B0.at(seg), k));
    return silu(zf[size_t(layer - 2) * Ec * W + size_t(e) * W + k]);
  }
  __device__ float b(int, int e, int n) const { return dz[size_t(e) * ldz + n]; }
  __device__ void store(int seg, int k, int n, float v) const { G.at(seg)[size_t(k) * Ncols + n] = v; }
};
// FDxProb's layer-1 case with silu'(zf0) materialised by edge_af0 (the TC
// configuration): no row context, no gather branch -> no spills in the engine
struct FDxSfProb {  // dz_0 = (dz_1 W_1^T) * sf0
  BDesc bd() const { return BDesc{Wt.base + Wt.off, nullptr, 0, 0, 1, K, K, Ncols, rows.nseg, (long long)Wt.PH, nullptr}; }
  static constexpr const char* kName = "bwd.force_edge_dx";
  struct Aux {
    float4 v;
  };
  __device__ float4 a4(int, int e, int k) const { return ld4(dz + size_t(e) * ldz + k); }
  __device__ Aux epi_aux(int, int e, int n) const { return Aux{ld4(sf0 + size_t(e) * W + n)}; }
  __device__ void epi4a(int, int e, int n, float4 acc, const Aux& a) const {
    st4(out + size_t(e) * W + n, mul4(acc, a.v));
  }
  RowSet rows;
  int K, Ncols, W;
  const float* dz;
  int ldz;
  HeadW Wt;
  float* out;
  const float* sf0;
  __device__ float a(int, int e, int k) const { return dz[size_t(e) * ldz + k]; }
  __device__ float b(int seg, int k, int n) const { return Wt.at(seg)[size_t(n) * K + k]; }
  __device__ void epi(int, int e, int n, float acc) const { out[size_t(e) * W + n] = acc * sf0[size_t(e) * W + n]; }
};
// FDxSfProb with its A operand dz_1 = ds_e w_2 * silu'(zf1_e) -- the width-1 output
// layer's backward (mlp_backward_, hmtl/model.hpp:308-336) -- formed by the producer
// (and stored on the way for the W_1 weight gradient): the output layer's elementwise
// pass leaves the critical path (its W_2/b_2 column sums run on a side stream).
struct FDxDsProb {
  BDesc bd() const { return BDesc{Wt.base + Wt.off, nullptr, 0, 0, 1, K, K, Ncols, rows.nseg, (long long)Wt.PH, nullptr}; }
  static constexpr const char* kName = "bwd.force_edge_dx";
  static constexpr bool kTcOnly = true;
  struct RC {
    float g;
  };
  using Raw = float4;
  struct Aux {
    float4 v;
  };
  __device__ RC rctx(int, int e) const { return RC{ds[e]}; }
  __device__ Raw raw4(int, int e, const RC&, int k) const { return ld4(zf1 + size_t(e) * W + k); }
  __device__ float4 fin4(int seg, int e, const RC& r, int k, const Raw& z) const {
    const float4 w = ldu4(W2.at(seg) + k);
    const float4 gw = make_float4(r.g * w.x, r.g * w.y, r.g * w.z, r.g * w.w);
    const float4 v = mul4(gw, sgrad4(z));  // force_out_bwd_kernel's dz, same operations
    st4(dz1out + size_t(e) * W + k, v);
    return v;
  }
  __device__ Aux epi_aux(int, int e, int n) const { return Aux{ld4(sf0 + size_t(e) * W + n)}; }
  __device__ void epi4a(int, int e, int n, float4 acc, const Aux& a) const {
    st4(out + size_t(e) * W + n, mul4(acc, a.v));
  }
  RowSet rows;
  int K, Ncols, W;
  const float *zf1, *ds;
  HeadW W2, Wt;
  float *dz1out, *out;
  const float* sf0;
  __device__ float b(int seg, int k, int n) const { return Wt.at(seg)[size_t(n) * K + k]; }
};
struct FDxProb {  // dz_{i-1} = (dz_i W_i^T) * silu'(z_{i-1})
  BDesc bd() const { return BDesc{Wt.base + Wt.off, nullptr, 0, 0, 1, K, K, Ncols, rows.nseg, (long long)Wt.PH, nullptr}; }
  static constexpr const char* kName = "bwd.force_edge_dx";
  struct RC {
    int d, s;
    float dist;
  };
  __device__ RC rctx(int, int e) const {
    return (sf0 || layer != 1) ? RC{0, 0, 0.f} : RC{dst[e], src[e], dist[e]};
  }
  __device__ float4 a4c(int, int e, const RC&, int k) const { return ld4(dz + size_t(e) * ldz + k); }
  // silu'(z_{i-1}) does not depend on the accumulator: prefetched by the epilogue (Aux)
  struct Aux {
    float4 v;
  };
  __device__ Aux epi_auxc(int seg, int e, const RC& r, int n) const {
    if (layer == 1 && sf0) return Aux{ld4(sf0 + size_t(e) * W + n)};
    const float4 zp = layer == 1 ? pre4(ld4(Qf + size_t(r.d) * W + n), ld4(Qf + size_t(r.s) * W + n), r.dist,
                                        ldu4(Wd.at(seg) + n), ldu4(B0.at(seg) + n))
                                 : ld4(zf + size_t(layer - 2) * Ec * W + size_t(e) * W + n);
    return Aux{sgrad4(zp)};
  }
  __device__ void epi4ac(int, int e, const RC&, int n, float4 acc, const Aux& a) const {
    st4(out + size_t(e) * W + n, mul4(acc, a.v));
  }
  __device__ void epi4c(int seg, int e, const RC& r, int n, float4 acc) const {
    epi4ac(seg, e, r, n, acc, epi_auxc(seg, e, r, n));
  }
  __device__ float4 a4(int, int e, int k) const { return ld4(dz + size_t(e) * ldz + k); }
  __device__ void epi4(int seg, int e, int n, float4 acc) const {
    const float4 zp = layer == 1 ? pre4(ld4(Qf + size_t(dst[e]) * W + n), ld4(Qf + size_t(src[e]) * W + n), dist[e],
                                        ldu4(Wd.at(seg) + n), ldu4(B0.at(seg) + n))
                                 : ld4(zf + size_t(layer - 2) * Ec * W + size_t(e) * W + n);
    st4(out + size_t(e) * W + n, mul4(acc, sgrad4(zp)));
  }
  RowSet rows;
  int K, Ncols, H, W, layer;  // layer = i
  long long Ec;
  const float *Qf, *zf, *dist, *dz;
  int ldz;
  const int *dst, *src;
  HeadW Wd, B0, Wt;
  float* out;
  const float* sf0;  // non-null: silu'(zf0) materialised
  __device__ float a(int, int e, int k) const { return dz[size_t(e) * ldz + k]; }
  __device__ float b(int seg, int k, int n) const { return Wt.at(seg)[size_t(n) * K + k]; }
  __device__ void epi(int seg, int e, int n, float acc) const {
    const float zp = layer == 1 ? zf0_of(Qf, W, dst[e], src[e], dist[e], Wd.at(seg), B0.at(seg), n)
                                : zf[size_t(layer - 2) * Ec * W + size_t(e) * W + n];
    out[size_t(e) * W + n] = acc * silu_grad(zp);
  }
};
struct F0NodeGrad {  // g_Wf0[:H] = h^T T  (node rows per head)
  static constexpr const char* kName = "bwd.force0_node_wgrad";
  static constexpr int kBias = 0;
  static constexpr bool kTc = true;
  __device__ float4 x4(int, int r, int m) const { return ld4(h + size_t(r) * H + m); }
  __device__ float4 y4(int, int r, int n) const { return ld4(T + size_t(r) * W + n); }
  RowSet rows;
  int K, Ncols, H, W;
  const float *h, *T;
  HeadG G;
  __device__ float a(int, int r, int k) const { return h[size_t(r) * H + k]; }
  __device__ float b(int, int r, int n) const { return T[size_t(r) * W + n]; }
  __device__ void store(int seg, int k, int n, float v) const { G.at(seg)[size_t(k) * W + n] = v; }
};
struct F0EdgeGrad {  // g_Wf0[H] (distance row) and g_bf0 (edge rows per head)
  static constexpr const char* kName = "bwd.force0_edge_wgrad";
  static constexpr int kBias = 0;
  static constexpr bool kTc = false;
  RowSet rows;
  int K, Ncols, H, W;
  const float *dist, *dz;
  HeadG G;  // points at row H of Wf0
  __device__ float a(int, int e, int k) const { return k == 0 ? dist[e] : 1.f; }
  __device__ float b(int, int e, int n) const { return dz[size_t(e) * W + n]; }
  __device__ void store(int seg, int k, int n, float v) const { G.at(seg)[size_t(k) * W + n] = v; }
};
struct F0Dh {  // dh += T Wf0[:H]^T  (node rows per head)
  struct Aux {
    float4 v;
  };
  __device__ Aux epi_aux(int, int r, int n) const { return Aux{ld4(dh + size_t(r) * H + n)}; }
  __device__ void epi4a(int, int r, int n, float4 acc, const Aux& a) const { st4(dh + size_t(r) * H + n, add4(a.v, acc)); }
  BDesc bd() const { return BDesc{Wt.base + Wt.off, nullptr, 0, 0, 1, W, K, Ncols, rows.nseg, (long long)Wt.PH, nullptr}; }
  static constexpr const char* kName = "bwd.force0_dh";
  __device__ float4 a4(int, int r, int k) const { return ld4(T + size_t(r) * W + k); }
  __device__ void epi4(int, int r, int n, float4 acc) const {
    float* o = dh + size_t(r) * H + n;
    st4(o, add4(ld4(o), acc));
  }
  RowSet rows;
  int K, Ncols, H, W;
  const float* T;
  HeadW Wt;
  float* dh;
  __device__ float a(int, int r, int k) const { return T[size_t(r) * W + k]; }
  __device__ float b(int seg, int k, int n) const { return Wt.at(seg)[size_t(n) * W + k]; }
  __device__ void epi(int, int r, int n, float acc) const { dh[size_t(r) * H + n] += acc; }
};

// ---- encoder layer backward problems (shared weights, identity rows)
struct L1Prob {  // dvz1 = (dh nW2^T) * silu'(vz1)
  struct Aux {
    float4 v;
  };
  __device__ Aux epi_aux(int, int r, int n) const { return Aux{sgrad4(ld4(vz1 + size_t(r) * H + n))}; }
  __device__ void epi4a(int, int r, int n, float4 acc, const Aux& a) const { st4(dvz1 + size_t(r) * H + n, mul4(acc, a.v)); }
  BDesc bd() const { return BDesc{W, nullptr, 0, 0, 1, H, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "bwd.node_dvz1";
  __device__ float4 a4(int, int r, int k) const { return ld4(dh + size_t(r) * H + k); }
  __device__ void epi4(int, int r, int n, float4 acc) const {
    st4(dvz1 + size_t(r) * H + n, mul4(acc, sgrad4(ld4(vz1 + size_t(r) * H + n))));
  }
  RowSet rows;
  int K, Ncols, H;
  const float *dh, *W, *vz1;
  float* dvz1;
  __device__ float a(int, int r, int k) const { return dh[size_t(r) * H + k]; }
  __device__ float b(int, int k, int n) const { return W[size_t(n) * H + k]; }
  __device__ void epi(int, int r, int n, float acc) const {
    dvz1[size_t(r) * H + n] = acc * silu_grad(vz1[size_t(r) * H + n]);
  }
};
struct L2Prob {  // [g_nW2; g_nb2] = [silu(vz1), 1]^T dh
  static constexpr const char* kName = "bwd.node_w2grad";
  static constexpr int kBias = 1;
  static constexpr bool kTc = true;
  __device__ float4 x4(int, int r, int m) const { return silu4(ld4(vz1 + size_t(r) * H + m)); }
  __device__ float4 y4(int, int r, int n) const { return ld4(dh + size_t(r) * H + n); }
  RowSet rows;
  int K, Ncols, H;
  const float *vz1, *dh;
  float* G;
  void tma(TmaOps& o) const { o.x = vz1, o.ldx = H, o.y = dh, o.ldy = H; }
  __device__ float4 xfin(float4 v) const { return silu4(v); }
  __device__ float a(int, int r, int k) const { return k < H ? silu(vz1[size_t(r) * H + k]) : 1.f; }
  __device__ float b(int, int r, int n) const { return dh[size_t(r) * H + n]; }
  __device__ void store(int, int k, int n, float v) const { G[size_t(k) * H + n] = v; }
};
struct L3Prob {  // [g_nW1; g_nb1] = [h, agg, 1]^T dvz1
  static constexpr const char* kName = "bwd.node_w1grad";
  static constexpr int kBias = 1;
  static constexpr bool kTc = true;
  __device__ float4 x4(int, int r, int m) const {
    return m < H ? ld4(h + size_t(r) * H + m) : ld4(agg + size_t(r) * H + m - H);
  }
  __device__ float4 y4(int, int r, int n) const { return ld4(dvz1 + size_t(r) * H + n); }
  RowSet rows;
  int K, Ncols, H;
  const float *h, *agg, *dvz1;
  float* G;
  // (TMA path measured slower here in the overlapped step: the row-walking producer stays)
  __device__ float a(int, int r, int k) const {
    return k < H ? h[size_t(r) * H + k] : (k < 2 * H ? agg[size_t(r) * H + k - H] : 1.f);
  }
  __device__ float b(int, int r, int n) const { return dvz1[size_t(r) * H + n]; }
  __device__ void store(int, int k, int n, float v) const { G[size_t(k) * H + n] = v; }
};
struct L4Prob {  // dv = dvz1 nW1^T ; dh2 = dh + dv[:, :H] ; dagg = dv[:, H:]
  struct Aux {
    float4 v;
  };
  __device__ Aux epi_aux(int, int r, int n) const {
    return Aux{n < H ? ld4(dh + size_t(r) * H + n) : make_float4(0.f, 0.f, 0.f, 0.f)};
  }
  __device__ void epi4a(int, int r, int n, float4 acc, const Aux& a) const {
    if (n < H) st4(dh2 + size_t(r) * H + n, add4(a.v, acc));
    else st4(dagg + size_t(r) * H + n - H, acc);
  }
  BDesc bd() const { return BDesc{W, nullptr, 0, 0, 1, H, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "bwd.node_dv";
  __device__ float4 a4(int, int r, int k) const { return ld4(dvz1 + size_t(r) * H + k); }
  __device__ void epi4(int, int r, int n, float4 acc) const {
    if (n < H) st4(dh2 + size_t(r) * H + n, add4(ld4(dh + size_t(r) * H + n), acc));
    else st4(dagg + size_t(r) * H + n - H, acc);
  }
  RowSet rows;
  int K, Ncols, H;
  const float *dvz1, *W, *dh;
  float *dh2, *dagg;
  __device__ float a(int, int r, int k) const { return dvz1[size_t(r) * H + k]; }
  __device__ float b(int, int k, int n) const { return W[size_t(n) * H + k]; }
  __device__ void epi(int, int r, int n, float acc) const {
    if (n < H) dh2[size_t(r) * H + n] = dh[size_t(r) * H + n] + acc;
    else dagg[size_t(r) * H + n - H] = acc;
  }
};
struct L6Prob {  // [g_eW2; g_eb2] = [silu(z1), 1]^T dz2   (E rows)
  static constexpr const char* kName = "bwd.edge_w2grad";
  static constexpr int kBias = 1;
  static constexpr bool kTc = true;
  __device__ float4 x4(int, int e, int m) const {
    if (a1s) return a1_is_z1 ? silu4(ld4(a1s + size_t(e) * H + m)) : ld4(a1s + size_t(e) * H + m);
    return silu4(pre4(ld4(P + size_t(dst[e]) * 2 * H + m), ld4(P + size_t(src[e]) * 2 * H + H + m), geo[e].w,
                      ld4(wd + m), ld4(b1 + m)));
  }
  __device__ float4 y4(int, int e, int n) const {
    if (dagg) return mul4(ld4(dagg + size_t(dst[e]) * H + n), sgrad4(ld4(z2s + size_t(e) * H + n)));
    return ld4(dz2 + size_t(e) * H + n);
  }
  RowSet rows;
  int K, Ncols, H;
  const float *P, *wd, *b1, *dz2;
  const int *dst, *src;
  const float4* geo;
  float* G;
  const float* a1s;  // a1 materialised by the forward producer (nullable)
  const float *dagg, *z2s;  // non-null: dz2 = dagg[dst] * silu'(z2) computed on the fly
  int a1_is_z1 = 0;         // a1s holds z1 (the forward stored the pre-activation): X = silu(z1)
  void tma(TmaOps& o) const { o.x = a1s, o.ldx = H, o.y = dagg ? nullptr : dz2, o.ldy = H; }
  __device__ float4 xfin(float4 v) const { return a1_is_z1 ? silu4(v) : v; }
  __device__ float a(int, int e, int k) const {
    return k < H ? silu(z1_of(P, H, dst[e], src[e], geo[e].w, wd, b1, k)) : 1.f;
  }
  __device__ float b(int, int e, int n) const { return dz2[size_t(e) * H + n]; }
  __device__ void store(int, int k, int n, float v) const { G[size_t(k) * H + n] = v; }
};
struct L7Prob {  // dz1 = (dz2 eW2^T) * silu'(z1)
  struct Aux {
    float4 v;
  };
  __device__ Aux epi_aux(int, int e, int n) const { return Aux{ld4(s1p + size_t(e) * H + n)}; }
  __device__ void epi4a(int, int e, int n, float4 acc, const Aux& a) const { st4(dz1 + size_t(e) * H + n, mul4(acc, a.v)); }
  BDesc bd() const { return BDesc{W, nullptr, 0, 0, 1, H, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "bwd.edge_dz1_gemm";
  struct RC {
    int d, s;
    float w;
  };
  __device__ RC rctx(int, int e) const { return s1p ? RC{0, 0, 0.f} : RC{dst[e], src[e], geo[e].w}; }
  __device__ float4 a4c(int, int e, const RC& r, int k) const {
    if (dagg) return mul4(ld4(dagg + size_t(r.d) * H + k), sgrad4(ld4(z2s + size_t(e) * H + k)));
    return ld4(dz2 + size_t(e) * H + k);
  }
  __device__ void epi4c(int, int e, const RC& r, int n, float4 acc) const {
    if (s1p) {  // silu'(z1) materialised by edge_bwd_prep_kernel
      st4(dz1 + size_t(e) * H + n, mul4(acc, ld4(s1p + size_t(e) * H + n)));
      return;
    }
    const float4 z = pre4(ld4(P + size_t(r.d) * 2 * H + n), ld4(P + size_t(r.s) * 2 * H + H + n), r.w, ld4(wd + n),
                          ld4(b1 + n));
    st4(dz1 + size_t(e) * H + n, mul4(acc, sgrad4(z)));
  }
  __device__ float4 a4(int, int e, int k) const { return ld4(dz2 + size_t(e) * H + k); }
  __device__ void epi4(int, int e, int n, float4 acc) const {
    const float4 z = pre4(ld4(P + size_t(dst[e]) * 2 * H + n), ld4(P + size_t(src[e]) * 2 * H + H + n), geo[e].w,
                          ld4(wd + n), ld4(b1 + n));
    st4(dz1 + size_t(e) * H + n, mul4(acc, sgrad4(z)));
  }
  RowSet rows;
  int K, Ncols, H;
  const float *dz2, *W, *P, *wd, *b1;
  const int *dst, *src;
  const float4* geo;
  float* dz1;
  const float *dagg, *z2s;  // non-null: dz2 computed on the fly (tensor-core path)
  const float* s1p;         // non-null: silu'(z1) materialised
  __device__ float a(int, int e, int k) const { return dz2[size_t(e) * H + k]; }
  __device__ float b(int, int k, int n) const { return W[size_t(n) * H + k]; }
  __device__ void epi(int, int e, int n, float acc) const {
    dz1[size_t(e) * H + n] = acc * silu_grad(z1_of(P, H, dst[e], src[e], geo[e].w, wd, b1, n));
  }
};
// Fused edge backward of one layer (hmtl/model.hpp:589-615) in one tensor-core
// pass: the producer forms dz2 = dagg[dst] * silu'(z2) as the A operand (and
// stores it for the eW2 weight gradient), the epilogue stores dz1 = (dz2 eW2^T) *
// silu'(z1) -- z1 regathered from the L2-resident node table P -- and sums dz1 per
// destination into S[:, :H] (segmented epilogue); seg_src_kernel adds S[:, H:]
// (the source-side sums through the reverse-edge permutation) and finishes the
// destinations that straddle a tile.  Bit-identical to edge_bwd_prep -> L7Prob
// -> seg2v.
struct L7SegProb {
  BDesc bd() const { return BDesc{W, nullptr, 0, 0, 1, H, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "bwd.edge_dz1_fused";
  static constexpr bool kSegSum = true;
  struct RC {
    int d, s;
    float w;
  };
  struct Raw {
    float4 g, z;
  };
  struct Aux {
    float4 v;
  };
  __device__ RC rctx(int, int e) const { return RC{dst[e], src[e], geo[e].w}; }
  __device__ Raw raw4(int, int e, const RC& r, int k) const {
    return Raw{ld4(dagg + size_t(r.d) * H + k), ld4(z2s + size_t(e) * H + k)};
  }
  __device__ float4 fin4(int, int e, const RC&, int k, const Raw& x) const {
    const float4 v = mul4(x.g, sgrad4(x.z));
    st4(dz2out + size_t(e) * H + k, v);
    return v;
  }
  // silu'(z1) does not depend on the accumulator: prefetched ahead of the MMAs
  __device__ Aux epi_auxc(int, int, const RC& r, int n) const {
    return Aux{sgrad4(pre4(ld4(P + size_t(r.d) * 2 * H + n), ld4(P + size_t(r.s) * 2 * H + H + n), r.w, ld4(wd + n),
                           ld4(b1 + n)))};
  }
  __device__ float4 epi4r(int, int e, const RC&, int n, float4 acc, const Aux& a) const {
    const float4 v = mul4(acc, a.v);
    st4(dz1 + size_t(e) * H + n, v);
    return v;
  }
  __device__ int seg_key(int e) const { return dst[e]; }
  __device__ void seg_store(int i, int n, float v) const { S[size_t(i) * 2 * H + n] = v; }
  RowSet rows;
  int K, Ncols, H;
  const float *W, *P, *wd, *b1, *dagg, *z2s;
  const int *dst, *src;
  const float4* geo;
  float *dz2out, *dz1, *S;
  float* tpart;  // [2][tcap][H] (seg_src_kernel adds a straddling destination's pieces)
  int tcap;
  __device__ float a(int, int e, int k) const { return dagg[size_t(dst[e]) * H + k] * silu_grad(z2s[size_t(e) * H + k]); }
  __device__ float b(int, int k, int n) const { return W[size_t(n) * H + k]; }
};

// dz1 = (dz2 eW2^T) * silu'(z1) with the A operand dz2 = dagg[dst] * silu'(z2)
// gathered by cp.async (tc.cuh kAsync) and stored on the way (eW2 weight
// gradient); silu'(z1) was stored by the forward (MsgAsyncProb).  Replaces
// edge_bwd_prep -> L7Prob (same operations: bit-identical dz2, dz1).
struct L7AsyncProb {
  BDesc bd() const { return BDesc{W, nullptr, 0, 0, 1, H, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "bwd.edge_dz1_gather";
  static constexpr bool kAsync = true;
  struct RC {
    int d;
  };
  struct Aux {
    float4 v;
  };
  __device__ RC rctx(int, int e) const { return RC{dst[e]}; }
  __device__ const float* src_a(int, int, const RC& r, int k) const { return dagg + size_t(r.d) * H + k; }
  __device__ const float* src_b(int, int e, const RC&, int k) const { return z2s + size_t(e) * H + k; }
  __device__ float4 combine(int, int e, const RC&, int k, float4 a, float4 b) const {
    const float4 v = mul4(a, sgrad4(b));
    st4(dz2out + size_t(e) * H + k, v);
    return v;
  }
  __device__ Aux epi_aux(int, int e, int n) const {
    const float4 v = ld4(s1p + size_t(e) * H + n);
    return Aux{z1_only ? sgrad4(v) : v};  // (z1_only: the forward stored z1, silu'(z1) here)
  }
  __device__ void epi4a(int, int e, int n, float4 acc, const Aux& a) const { st4(dz1 + size_t(e) * H + n, mul4(acc, a.v)); }
  // z2 and silu'(z1) were written by the forward (long evicted from L2): stream this
  // CTA's rows into L2 ahead of the pipeline (HMTL_ROW_PREFETCH)
  __device__ void prefetch_rows(int e0, int e1) const {
    tc::prefetch_l2(z2s + size_t(e0) * H, size_t(e1 - e0) * H * 4);
    tc::prefetch_l2(s1p + size_t(e0) * H, size_t(e1 - e0) * H * 4);
  }
  RowSet rows;
  int K, Ncols, H;
  const float *W, *dagg, *z2s, *s1p;  // s1p: silu'(z1), or z1 itself when z1_only
  const int* dst;
  float *dz2out, *dz1;
  int z1_only;
  __device__ float b(int, int k, int n) const { return W[size_t(n) * H + k]; }
};

// L7AsyncProb with silu'(z1) regathered in the epilogue from the L2-resident node
// table (z1 = P_a[dst] + P_b[src] + d2 w + b1): nothing stored by the forward.
struct L7AsyncPProb {
  BDesc bd() const { return BDesc{W, nullptr, 0, 0, 1, H, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "bwd.edge_dz1_gather";
  static constexpr bool kAsync = true;
  struct RC {
    int d, s;
    float w;
  };
  struct Aux {
    float4 v;
  };
  __device__ RC rctx(int, int e) const { return RC{dst[e], src[e], geo[e].w}; }
  __device__ const float* src_a(int, int, const RC& r, int k) const { return dagg + size_t(r.d) * H + k; }
  __device__ const float* src_b(int, int e, const RC&, int k) const { return z2s + size_t(e) * H + k; }
  __device__ float4 combine(int, int e, const RC&, int k, float4 a, float4 b) const {
    const float4 v = mul4(a, sgrad4(b));
    st4(dz2out + size_t(e) * H + k, v);
    return v;
  }
  __device__ Aux epi_auxc(int, int, const RC& r, int n) const {
    return Aux{sgrad4(pre4(ld4(P + size_t(r.d) * 2 * H + n), ld4(P + size_t(r.s) * 2 * H + H + n), r.w, ld4(wd + n),
                           ld4(b1 + n)))};
  }
  __device__ void epi4ac(int, int e, const RC&, int n, float4 acc, const Aux& a) const {
    st4(dz1 + size_t(e) * H + n, mul4(acc, a.v));
  }
  RowSet rows;
  int K, Ncols, H;
  const float *W, *dagg, *z2s, *P, *wd, *b1;
  const int *dst, *src;
  const float4* geo;
  float *dz2out, *dz1;
  __device__ float b(int, int k, int n) const { return W[size_t(n) * H + k]; }
};

struct L9Prob {  // [g_W1[2H]; g_b1] = [d2, 1]^T dz1   (E rows)
  static constexpr const char* kName = "bwd.edge_w1tail_grad";
  static constexpr int kBias = 0;
  static constexpr bool kTc = false;
  RowSet rows;
  int K, Ncols, H;
  const float4* geo;
  const float* dz1;
  float* G;  // row 2H of g_eW1
  __device__ float a(int, int e, int k) const { return k == 0 ? geo[e].w : 1.f; }
  __device__ float b(int, int e, int n) const { return dz1[size_t(e) * H + n]; }
  __device__ void store(int, int k, int n, float v) const { G[size_t(k) * H + n] = v; }
};
struct L10Prob {  // g_W1a = h^T S_dst, g_W1b = h^T S_src
  static constexpr const char* kName = "bwd.edge_w1ab_grad";
  static constexpr int kBias = 0;
  static constexpr bool kTc = true;
  __device__ float4 x4(int, int r, int m) const { return ld4(h + size_t(r) * H + m); }
  __device__ float4 y4(int, int r, int n) const { return ld4(S + size_t(r) * 2 * H + n); }
  RowSet rows;
  int K, Ncols, H;
  const float *h, *S;
  float* G;  // g_eW1
  __device__ float a(int, int r, int k) const { return h[size_t(r) * H + k]; }
  __device__ float b(int, int r, int n) const { return S[size_t(r) * 2 * H + n]; }
  __device__ void store(int, int k, int n, float v) const {
    if (n < H) G[size_t(k) * H + n] = v;
    else G[size_t(H + k) * H + n - H] = v;
  }
};
struct L11Prob {  // dh2 += S_dst W1a^T + S_src W1b^T
  struct Aux {
    float4 v;
  };
  __device__ Aux epi_aux(int, int r, int n) const { return Aux{ld4(dh2 + size_t(r) * H + n)}; }
  __device__ void epi4a(int, int r, int n, float4 acc, const Aux& a) const { st4(dh2 + size_t(r) * H + n, add4(a.v, acc)); }
  BDesc bd() const { return BDesc{W1, W1 + size_t(H) * H, 2, H, 1, H, K, Ncols, 1, 0, nullptr}; }
  static constexpr const char* kName = "bwd.edge_dh_gemm";
  __device__ float4 a4(int, int r, int k) const { return ld4(S + size_t(r) * 2 * H + k); }
  __device__ void epi4(int, int r, int n, float4 acc) const {
    float* o = dh2 + size_t(r) * H + n;
    st4(o, add4(ld4(o), acc));
  }
  RowSet rows;
  int K, Ncols, H;
  const float *S, *W1;
  float* dh2;
  __device__ float a(int, int r, int k) const { return S[size_t(r) * 2 * H + k]; }
  __device__ float b(int, int k, int n) const {
    return k < H ? W1[size_t(n) * H + k] : W1[size_t(H + n) * H + k - H];
  }
  __device__ void epi(int, int r, int n, float acc) const { dh2[size_t(r) * H + n] += acc; }
};

// dh_i = dpooled_g * (1/n)  (first contribution; hmtl/model.hpp:517-524)
// L2 prefetch of a tensor the critical path will read soon (it was written long
// enough ago to have left L2): prefetch.global.L2 per 128 B line, no registers
__global__ void l2_prefetch_kernel(const DevHdr* hdr, const float* __restrict__ x, int per_edge) {
  pdl_wait();
  const size_t bytes = size_t(hdr->E) * per_edge * sizeof(float);
  const char* p = reinterpret_cast<const char*>(x);
  for (size_t o = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) * 128; o < bytes; o += size_t(gridDim.x) * blockDim.x * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + o));
}
__global__ void dh_pool_kernel(const DevHdr* hdr, const int* __restrict__ node_graph,
                               const int* __restrict__ graph_offset, const float* __restrict__ dpooled,
                               float* __restrict__ dh, int H) {
  pdl_wait();
  const long long total = (long long)hdr->N * H;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int i = int(t / H), k = int(t % H);
    const int g = node_graph[i];
    const float inv = 1.f / float(graph_offset[g + 1] - graph_offset[g]);
    dh[t] = dpooled[size_t(g) * H + k] * inv;
  }
}

// ds_e = sum_c dF[dst,c] * dvec[e,c]  (hmtl/model.hpp:528-536)
__global__ void ds_kernel(const DevHdr* hdr, const int* __restrict__ dst, const float4* __restrict__ geo,
                          const float* __restrict__ dF, float* __restrict__ ds) {
  pdl_wait();
  const int E = hdr->E;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    const int i = dst[e];
    const float4 g = geo[e];
    float acc = 0.f;
    acc += dF[3 * i] * g.x;
    acc += dF[3 * i + 1] * g.y;
    acc += dF[3 * i + 2] * g.z;
    ds[e] = acc;
  }
}

// dz2 = dagg[dst] * silu'(z2)  (hmtl/model.hpp:590-597)
__global__ void dz2_kernel(const DevHdr* hdr, const int* __restrict__ dst, const float* __restrict__ dagg,
                           const float* __restrict__ z2, float* __restrict__ dz2, int H) {
  pdl_wait();
  const long long total = (long long)hdr->E * H;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int e = int(t / H), k = int(t % H);
    dz2[t] = dagg[size_t(dst[e]) * H + k] * silu_grad(z2[t]);
  }
}

// S[i] = [ sum_{e in row i} x_e | sum_{e in row i} x_{rev(e)} ]; x is [E x C].
// The second half is the src-segment sum: edges with src == i are exactly the
// reverses of row i.  If `fold`, the two halves are added (force head: T).
__global__ void seg2_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr, const int* __restrict__ rev,
                            const float* __restrict__ x, float* __restrict__ S, int C, int fold) {
  pdl_wait();
  const int N = hdr->N;
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < N; i += (gridDim.x * blockDim.x) >> 5) {
    const int e0 = row_ptr[i], e1 = row_ptr[i + 1];
    for (int c = lane; c < C; c += 32) {
      float a = 0.f, b = 0.f;
      for (int e = e0; e < e1; ++e) {
        a += x[size_t(e) * C + c];
        b += x[size_t(rev[e]) * C + c];
      }
      if (fold) S[size_t(i) * C + c] = a + b;
      else {
        S[size_t(i) * 2 * C + c] = a;
        S[size_t(i) * 2 * C + C + c] = b;
      }
    }
  }
}

// ---- vectorised CSR segment sums: warp per node, lane = float4 column group,
// 4 independent edge loads in flight; ascending-edge accumulation per column.

// agg_i = sum_{e in row i} silu(z2_e).  Warp per node, lane = float4 column
// group; edges in batches of 8 with all 8 row loads issued before the
// ascending-edge accumulation (high-degree inorganic nodes set the kernel time).
constexpr int kAggU = 8;
__global__ void __launch_bounds__(256) agg4_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr,
                                                   const float* __restrict__ z2, float* __restrict__ agg, int H) {
  pdl_wait();
  const int N = hdr->N, lane = threadIdx.x & 31, R = (N + 7) >> 3;
  // node v of the grid-stride walk -> node (v % 8) * R + v / 8: a CTA's 8 warps take
  // nodes from 8 regions of the batch, spreading the heavy (inorganic) degree tail
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < 8 * R; v += (gridDim.x * blockDim.x) >> 5) {
    const int i = (v & 7) * R + (v >> 3);
    if (i >= N) continue;
    const int e0 = row_ptr[i], e1 = row_ptr[i + 1];
    for (int c = lane * 4; c < H; c += 128) {
      float4 acc = f4z();
      for (int e = e0; e < e1; e += kAggU) {
        float4 v[kAggU];
#pragma unroll
        for (int u = 0; u < kAggU; ++u) v[u] = e + u < e1 ? ld4(z2 + size_t(e + u) * H + c) : f4z();
#pragma unroll
        for (int u = 0; u < kAggU; ++u)
          if (e + u < e1) acc = add4(acc, silu4(v[u]));
      }
      st4(agg + size_t(i) * H + c, acc);
    }
  }
}

// S[i] = [sum_{e in row i} x_e | sum_{e in row i} x_{rev(e)}] (or folded a + b).
// The row's rev indices are read once per 32-edge window (one per lane) and
// broadcast by shuffle; 4 edges per batch -> 8 row loads in flight per lane.
constexpr int kSegU = 8;
__global__ void __launch_bounds__(256) seg2v_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr,
                                                    const int* __restrict__ rev, const float* __restrict__ x,
                                                    float* __restrict__ S, int C, int fold) {
  pdl_wait();
  const int N = hdr->N, lane = threadIdx.x & 31, R = (N + 7) >> 3;
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < 8 * R; v += (gridDim.x * blockDim.x) >> 5) {
    const int i = (v & 7) * R + (v >> 3);  // spread over the batch, as agg4_kernel
    if (i >= N) continue;
    const int e0 = row_ptr[i], e1 = row_ptr[i + 1];
    for (int c0 = 0; c0 < C; c0 += 128) {  // warp-uniform bound: the shuffles need every lane
      const int c = c0 + lane * 4;
      const bool col = c < C;
      float4 a = f4z(), b = f4z();
      for (int w0 = e0; w0 < e1; w0 += 32) {
        const int myrev = w0 + lane < e1 ? rev[w0 + lane] : 0;
        const int cnt = min(32, e1 - w0);
        for (int j = 0; j < cnt; j += kSegU) {
          float4 va[kSegU], vb[kSegU];
#pragma unroll
          for (int u = 0; u < kSegU; ++u) {
            const int r = __shfl_sync(0xffffffffu, myrev, (j + u) & 31);
            const bool ok = col && j + u < cnt;
            va[u] = ok ? ld4(x + size_t(w0 + j + u) * C + c) : f4z();
            vb[u] = ok ? ld4(x + size_t(r) * C + c) : f4z();
          }
#pragma unroll
          for (int u = 0; u < kSegU; ++u)
            if (j + u < cnt) a = add4(a, va[u]), b = add4(b, vb[u]);
        }
      }
      if (!col) continue;
      if (fold) {
        st4(S + size_t(i) * C + c, add4(a, b));
      } else {
        st4(S + size_t(i) * 2 * C + c, a);
        st4(S + size_t(i) * 2 * C + C + c, b);
      }
    }
  }
}

// A destination's edge rows straddle a 128-edge tile of the fused (segmented-
// epilogue) edge kernels, or it has none: its sum is not written there.
__device__ __forceinline__ bool tile_straddle(int e0, int e1) { return e1 == e0 || (e0 >> 7) != ((e1 - 1) >> 7); }

// sum of a straddling destination's per-tile pieces (tc.cuh segmented epilogue):
// its tail piece in its first tile, then the head pieces of the following tiles
__device__ __forceinline__ float4 tile_pieces(const float* __restrict__ tp, int tcap, int C, int e0, int e1, int c) {
  const int t0 = e0 >> 7, t1 = (e1 - 1) >> 7;
  float4 acc = ld4(tp + (size_t(tcap) + t0) * C + c);
  for (int t = t0 + 1; t <= t1; ++t) acc = add4(acc, ld4(tp + size_t(t) * C + c));
  return acc;
}

// agg_i for the destinations the fused forward left: pieces of straddling
// destinations summed in tile order, zeros for nodes without edges
__global__ void __launch_bounds__(256) agg_fix_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr,
                                                      const float* __restrict__ tp, int tcap, float* __restrict__ agg,
                                                      int H) {
  pdl_wait();
  const int N = hdr->N;
  const int per = H >> 2;  // float4 columns per node
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < N * per; t += gridDim.x * blockDim.x) {
    const int i = t / per, c = (t - i * per) * 4;
    const int e0 = row_ptr[i], e1 = row_ptr[i + 1];
    if (!tile_straddle(e0, e1)) continue;
    st4(agg + size_t(i) * H + c, e1 == e0 ? f4z() : tile_pieces(tp, tcap, H, e0, e1, c));
  }
}

// S[i][C:2C] = sum_{e in row i} x_{rev(e)} for every node (the source-side sums,
// ascending-edge accumulation as seg2v_kernel), and S[i][0:C] for the
// destinations the fused backward left (straddling pieces / zeros)
constexpr int kSrcU = 8;
__global__ void __launch_bounds__(256) seg_src_kernel(const DevHdr* hdr, const int* __restrict__ row_ptr,
                                                      const int* __restrict__ rev, const float* __restrict__ x,
                                                      const float* __restrict__ tp, int tcap, float* __restrict__ S,
                                                      int C) {
  pdl_wait();
  const int N = hdr->N, lane = threadIdx.x & 31, R = (N + 7) >> 3;
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < 8 * R; v += (gridDim.x * blockDim.x) >> 5) {
    const int i = (v & 7) * R + (v >> 3);  // spread over the batch, as agg4_kernel
    if (i >= N) continue;
    const int e0 = row_ptr[i], e1 = row_ptr[i + 1];
    for (int c0 = 0; c0 < C; c0 += 128) {
      const int c = c0 + lane * 4;
      const bool col = c < C;
      float4 b = f4z();
      for (int w0 = e0; w0 < e1; w0 += 32) {
        const int myrev = w0 + lane < e1 ? rev[w0 + lane] : 0;
        const int cnt = min(32, e1 - w0);
        for (int j = 0; j < cnt; j += kSrcU) {
          float4 vb[kSrcU];
#pragma unroll
          for (int u = 0; u < kSrcU; ++u) {
            const int r = __shfl_sync(0xffffffffu, myrev, (j + u) & 31);
            vb[u] = (col && j + u < cnt) ? ld4(x + size_t(r) * C + c) : f4z();
          }
#pragma unroll
          for (int u = 0; u < kSrcU; ++u)
            if (j + u < cnt) b = add4(b, vb[u]);
        }
      }
      if (!col) continue;
      if (tile_straddle(e0, e1)) st4(S + size_t(i) * 2 * C + c, e1 == e0 ? f4z() : tile_pieces(tp, tcap, C, e0, e1, c));
      st4(S + size_t(i) * 2 * C + C + c, b);
    }
  }
}

// Column sums over the rows of each head segment: out[seg] = [sum_r w(r) x_r ; sum_r x_r]
// (the [distance-or-d2 ; bias] rows of a factorised first layer's gradient).
// Deterministic: CTA (chunk, seg) owns a fixed row range, 8 warps split it in
// fixed sub-ranges, smem combine in warp order; colsum2_reduce sums chunks in order.
constexpr int kCs2Rows = 128;
__global__ void __launch_bounds__(256) colsum2_kernel(RowSet rows, const float* __restrict__ wvec, int wstride,
                                                      const float* __restrict__ x, int C,
                                                      float* __restrict__ partial, int nchunk_cap) {
  pdl_wait();
  __shared__ float4 red[8][2][64];
  const int seg = blockIdx.y, chunk = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = rows.begin(seg), re = rows.end(seg);
  const int r0 = rb + chunk * kCs2Rows;
  if (r0 >= re) return;  // beyond this segment: not counted by the reduce
  const int sub = kCs2Rows / 8;
  const int w0 = r0 + warp * sub, w1 = min(w0 + sub, re);
  for (int c = lane * 4, u = 0; c < C; c += 128, ++u) {
    float4 sw = f4z(), sx = f4z();
    int v = w0;
    for (; v + 4 <= w1; v += 4) {
      int r[4];
      float4 xv[4];
      float w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) r[q] = rows.row(v + q);
#pragma unroll
      for (int q = 0; q < 4; ++q) xv[q] = ld4(x + size_t(r[q]) * C + c), w[q] = wvec[size_t(r[q]) * wstride];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        sw = make_float4(sw.x + w[q] * xv[q].x, sw.y + w[q] * xv[q].y, sw.z + w[q] * xv[q].z, sw.w + w[q] * xv[q].w);
        sx = add4(sx, xv[q]);
      }
    }
    for (; v < w1; ++v) {
      const int r = rows.row(v);
      const float4 xv = ld4(x + size_t(r) * C + c);
      const float w = wvec[size_t(r) * wstride];
      sw = make_float4(sw.x + w * xv.x, sw.y + w * xv.y, sw.z + w * xv.z, sw.w + w * xv.w);
      sx = add4(sx, xv);
    }
    red[warp][0][lane + 32 * u] = sw;
    red[warp][1][lane + 32 * u] = sx;
  }
  __syncthreads();
  float* out = partial + (size_t(seg) * nchunk_cap + chunk) * 2 * C;
  for (int t = threadIdx.x; t < 2 * (C / 4); t += blockDim.x) {
    const int which = t / (C / 4), cg = t % (C / 4);
    float4 acc = f4z();
    for (int w = 0; w < 8; ++w) acc = add4(acc, red[w][which][cg]);
    st4(out + which * C + cg * 4, acc);
  }
}
// force MLP output layer backward (width 1), for the edge rows of head segment seg:
//   dz_{i-1}[e] = (ds_e w_seg) * silu'(z_{i-1}[e])                   (elementwise)
//   partial[seg][chunk] = [sum_e ds_e silu(z_{i-1}[e]) ; sum_e ds_e]   (W and b grads)
// Same fixed chunk / warp split as colsum2_kernel; split_reduce sums chunks in order.
constexpr int kFoRows = 128;
__global__ void __launch_bounds__(256) force_out_bwd_kernel(RowSet rows, const float* __restrict__ x,
                                                            const float* __restrict__ xd, int act,
                                                            const float* __restrict__ ds,
                                                            const float* __restrict__ heads, size_t PH, size_t off_w,
                                                            float* __restrict__ dzp, float* __restrict__ partial,
                                                            int nchunk_cap, int W) {
  pdl_wait();
  __shared__ float red[8][257];
  const int seg = blockIdx.y, chunk = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rb = rows.begin(seg), re = rows.end(seg);
  const int r0 = rb + chunk * kFoRows;
  if (r0 >= re) return;  // beyond this segment: not counted by the reduce
  const int w0 = r0 + warp * (kFoRows / 8), w1 = min(w0 + kFoRows / 8, re);
  const float* wv = heads + size_t(seg) * PH + off_w;
  float4 wr[2], acc[2];
  float accb = 0.f;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int c = lane * 4 + 128 * u;
    wr[u] = c < W ? ldu4(wv + c) : f4z();
    acc[u] = f4z();
  }
  for (int v = w0; v < w1; v += 2) {  // two rows per iteration, all loads issued before the math
    int e[2];
    float g[2];
    float4 z[2][2], zd[2][2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      e[j] = v + j < w1 ? rows.row(v + j) : -1;
      g[j] = e[j] >= 0 ? ds[e[j]] : 0.f;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = lane * 4 + 128 * u;
        const bool ok = e[j] >= 0 && c < W;
        z[j][u] = ok ? ld4(x + size_t(e[j]) * W + c) : f4z();
        zd[j][u] = (ok && !act) ? ld4(xd + size_t(e[j]) * W + c) : f4z();
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = lane * 4 + 128 * u;
        if (e[j] < 0 || c >= W) continue;
        const float4 sg = act ? silu4(z[j][u]) : z[j][u];
        const float4 sd = act ? sgrad4(z[j][u]) : zd[j][u];
        const float4 gw = make_float4(g[j] * wr[u].x, g[j] * wr[u].y, g[j] * wr[u].z, g[j] * wr[u].w);
        if (dzp) st4(dzp + size_t(e[j]) * W + c, mul4(gw, sd));  // (null: the next GEMM's producer forms it)
        acc[u] = make_float4(acc[u].x + g[j] * sg.x, acc[u].y + g[j] * sg.y, acc[u].z + g[j] * sg.z,
                             acc[u].w + g[j] * sg.w);
      }
      accb += g[j];
    }
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int c = lane * 4 + 128 * u;
    if (c < W) {
      red[warp][c] = acc[u].x;
      red[warp][c + 1] = acc[u].y;
      red[warp][c + 2] = acc[u].z;
      red[warp][c + 3] = acc[u].w;
    }
  }
  if (lane == 0) red[warp][W] = accb;
  __syncthreads();
  float* out = partial + (size_t(seg) * nchunk_cap + chunk) * (W + 1);
  for (int t = threadIdx.x; t <= W; t += blockDim.x) {
    float a = 0.f;
    for (int w = 0; w < 8; ++w) a += red[w][t];
    out[t] = a;
  }
}

// split_reduce functor: chunk partials of a head-segmented row set -> G + seg*seg_stride
struct ChunkStore {
  RowSet rows;
  int rows_per_chunk;
  float* G;
  size_t seg_stride;
  __device__ int count(int seg) const { return (rows.end(seg) - rows.begin(seg) + rows_per_chunk - 1) / rows_per_chunk; }
  __device__ void store(int seg, int t, float v) const { G[seg * seg_stride + t] = v; }
};

// g_embed[s] = sum_{i: species_i = s} dh_i: CTA = 128-node chunk, thread = column,
// smem accumulator [species][H] updated in ascending node order; chunks summed in order.
constexpr int kEmbChunk = 64;
__global__ void embed_grad_part(const DevHdr* hdr, const uint8_t* __restrict__ species, const float* __restrict__ dh,
                                float* __restrict__ partial, int H, int NS) {
  pdl_wait();
  extern __shared__ float acc[];  // [NS][H]
  const int N = hdr->N, chunk = blockIdx.x;
  const int i0 = chunk * kEmbChunk;
  if (i0 >= N) return;
  for (int t = threadIdx.x; t < NS * H; t += blockDim.x) acc[t] = 0.f;
  __syncthreads();
  const int i1 = min(i0 + kEmbChunk, N);
  for (int c = threadIdx.x; c < H; c += blockDim.x) {
    int i = i0;
    for (; i + 8 <= i1; i += 8) {  // 8 loads in flight, updates in ascending node order
      float v[8];
      int sp[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = dh[size_t(i + j) * H + c], sp[j] = species[i + j];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[sp[j] * H + c] += v[j];
    }
    for (; i < i1; ++i) acc[species[i] * H + c] += dh[size_t(i) * H + c];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < NS * H; t += blockDim.x) partial[size_t(chunk) * NS * H + t] = acc[t];
}
struct EmbedStore {
  const DevHdr* hdr;
  float* G;
  __device__ int count(int) const { return (hdr->N + kEmbChunk - 1) / kEmbChunk; }
  __device__ void store(int, int t, float v) const { G[t] = v; }
};

// g_embed[s] = sum_{i: species_i = s} dh_i (ascending i; hmtl/model.hpp:619-622)
__global__ void embed_grad_kernel(const DevHdr* hdr, const uint8_t* __restrict__ species, const float* __restrict__ dh,
                                  float* __restrict__ G, int H, int NS) {
  pdl_wait();
  const int N = hdr->N;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < NS * H; t += gridDim.x * blockDim.x) {
    const int s = t / H, k = t % H;
    float acc = 0.f;
    for (int i = 0; i < N; ++i)
      if (species[i] == s) acc += dh[size_t(i) * H + k];
    G[t] = acc;
  }
}

}  // namespace

namespace {
void segsum2(Ctx& c, const float* x, int C, int fold, float* out, cudaStream_t st) {
  Prof pr(c, "bwd.segsum_dst_src", st);
  const int blocks = gridn((long long)c.Nc * 32, 256, c.sm_count * 16);
  if (C % 4 == 0) kl(seg2v_kernel, blocks, 256, 0, st, c.hdr, c.row_ptr, c.rev, x, out, C, fold);
  else kl(seg2_kernel, blocks, 256, 0, st, c.hdr, c.row_ptr, c.rev, x, out, C, fold);
}
// [sum w*x ; sum x] per head segment into G + seg*seg_stride (rows are contiguous)
void colsum2(Ctx& c, RowSet rows, const float* w, int wstride, const float* x, int C, float* G, size_t seg_stride,
             cudaStream_t st) {
  if (c.dbg_skip_wgrad) return;
  Prof pr(c, "bwd.colsum_tail", st);
  const int chunk_cap = int((c.Ec + kCs2Rows - 1) / kCs2Rows);
  dim3 grid(chunk_cap, rows.nseg);
  kl(colsum2_kernel, grid, 256, 0, st, rows, w, wstride, x, C, c.part(st), chunk_cap);
  kl(split_reduce_kernel<ChunkStore>, dim3((2 * C + 31) / 32, rows.nseg), 256, 0, st,
      c.part(st), size_t(chunk_cap) * 2 * C, size_t(2) * C, 2 * C, ChunkStore{rows, kCs2Rows, G, seg_stride});
}
}  // namespace

void launch_backward(Ctx& c, cudaStream_t st, bool comm_sync) {
  const int H = c.H, W = c.W, L = c.L, D = c.D, sm = c.sm_count;
  const size_t NH = size_t(c.Nc) * H, EH = size_t(c.Ec) * H;
  const size_t SBS = size_t(c.Nc) * 2 * std::max(H, W);  // one Sb slot
  const float* hL = c.hs + size_t(L) * NH;
  const size_t GW = size_t(c.Gc) * W;
  // streams: st = critical path (dx chain), se = energy head branch, sw = weight
  // gradients (consumed only by the gradient sync / AdamW after the final join)
  cudaStream_t se = c.side(c.s_e, st), sw = c.side(c.s_w, st), sw2 = c.side(c.s_w2, st), sw3 = c.side(c.s_w3, st);
  bool own3 = false, used3 = false;  // the eW2 gradient of this layer / of any layer on sw3
  // gradient sync buckets (MTL-par), issued on the comm stream as they become final
  const bool cs = comm_sync && comm_overlap(c);
  cudaStream_t sc = c.side(c.s_c, st);
  float* dhL = c.dhb + size_t(L) * NH;  // dL/dh_L, written by the heads

  // silu'(zf0), written by the forward's force head long before, is re-read by the
  // force-head dx GEMM on the critical path: pull it back into L2 from a side stream
  if (c.store_sf0 && c.prefetch_l2) {
    c.dep(st, sw2);
    Prof pr(c, "bwd.l2_prefetch", sw2);
    kl(l2_prefetch_kernel, sm * 4, 256, 0, sw2, static_cast<const DevHdr*>(c.hdr), static_cast<const float*>(c.sf0), W);
  }
  // weight gradients that have most of the backward left to finish in (heads, layers >= 1)
  // spread over fewer SMs: they hold fewer SMs the critical path needs; layer 0's, which
  // the optimizer waits on, spread over red_sms
  c.red_sms_now = c.red_sms_early;
  c.red_min_now = c.red_min_chunks;
  // ---------------- energy heads (hmtl/model.hpp:512-524)
  c.dep(st, se);
  {
    const float* dz = c.dE;
    int ldz = 1;
    float* bufs[2] = {c.edA, c.edB};
    for (int i = D - 1; i >= 0; --i) {
      const int in = i == 0 ? H : W, out = i == D - 1 ? 1 : W;
      c.dep(se, sw);
      EGradProb gq{graph_rows_by_head(c), in + 1, out, H, W, i, c.pooled,
                   i ? c.ez + size_t(i - 1) * GW : nullptr, dz, ldz,
                   HeadG{c.head_grads(), c.PH, c.head_off("energy.W" + std::to_string(i))}};
      atb(gq, c, c.nsplit_graph, sw, c.Gc);
      float* nxt = i ? bufs[i & 1] : c.dpooled;
      EDxProb dq{graph_rows_by_head(c), out, in, W, H, dz, i ? c.ez + size_t(i - 1) * GW : nullptr, ldz,
                 HeadW{c.head_params(), c.PH, c.head_off("energy.W" + std::to_string(i))}, nxt, i ? W : H,
                 i ? 1 : 0};
      ab(dq, c.Gc, c.S, se, sm, c);
      dz = nxt;
      ldz = W;
    }
    {
      Prof pr(c, "bwd.pool", se);
      kl(dh_pool_kernel, gridn(NH, 256, sm * 16), 256, 0, se, c.hdr, c.node_graph, c.graph_offset, c.dpooled, dhL, H);
    }
  }
  // ---------------- force heads (hmtl/model.hpp:526-549)
  {
    {
      Prof pr(c, "bwd.force_ds", st);
      kl(ds_kernel, gridn(c.Ec, 256, sm * 8), 256, 0, st, c.hdr, c.edge_dst, c.geo, c.dF, c.ds);
    }
    const size_t wf0 = c.head_off("force.W0");
    const HeadW Wd{c.head_params(), c.PH, wf0 + size_t(H) * W};
    const HeadW B0{c.head_params(), c.PH, c.head_off("force.b0")};
    const float* dz = c.ds;
    int ldz = 1;
    float* bufs[2] = {c.fzA, c.fzB};
    // (head_depth 3: the output layer's dz is formed inside the next dx GEMM's producer)
    const bool fuse_out = D == 3 && force_out_fast(c, 2) && c.store_sf0 && c.use_tc && c.fuse_force_out;
    for (int i = D - 1; i >= 1; --i) {
      const int out = i == D - 1 ? 1 : W;
      float* nxt = bufs[i & 1];
      if (i == D - 1 && fuse_out) {  // W_2 / b_2 gradients only, off the critical path
        c.dep(st, sw2);
        Prof pr(c, "bwd.force_out", sw2);
        const int cap = int((c.Ec + kFoRows - 1) / kFoRows);
        const RowSet rows = edge_rows_by_head(c);
        kl(force_out_bwd_kernel, dim3(cap, rows.nseg), 256, 0, sw2, rows, c.zf, c.sf0, 1, c.ds, c.head_params(), c.PH,
           c.head_off("force.W2"), static_cast<float*>(nullptr), c.part(sw2), cap, W);
        kl(split_reduce_kernel<ChunkStore>, dim3((W + 1 + 31) / 32, rows.nseg), 256, 0, sw2, c.part(sw2),
           size_t(cap) * (W + 1), size_t(W + 1), W + 1,
           ChunkStore{rows, kFoRows, c.head_grads() + c.head_off("force.W2"), c.PH});
        continue;
      }
      if (i == 1 && fuse_out) {  // dz_1 (stored) and dz_0 in one GEMM, then W_1's gradient
        const HeadW Wi{c.head_params(), c.PH, c.head_off("force.W1")};
        FDxDsProb dq{edge_rows_by_head(c), W, W, W, c.zf, c.ds, HeadW{c.head_params(), c.PH, c.head_off("force.W2")},
                     Wi, bufs[0], nxt, c.sf0};
        ab(dq, c.Ec, c.S, st, sm, c);
        c.dep(st, sw);
        FGradProb gq{edge_rows_by_head(c), W + 1, W, H, W, 1, c.Ec, c.Qf, c.zf, c.dist, bufs[0], W, c.edge_dst,
                     c.edge_src, Wd, B0, HeadG{c.head_grads(), c.PH, c.head_off("force.W1")},
                     c.store_af0 ? c.af0 : nullptr};
        atb(gq, c, c.nsplit_edge, sw, c.Ec);
        dz = nxt;
        ldz = W;
        continue;
      }
      if (i == D - 1 && force_out_fast(c, i)) {
        Prof pr(c, "bwd.force_out", st);
        const int cap = int((c.Ec + kFoRows - 1) / kFoRows);
        const RowSet rows = edge_rows_by_head(c);
        kl(force_out_bwd_kernel, dim3(cap, rows.nseg), 256, 0, st,
            rows, i >= 2 ? c.zf + size_t(i - 2) * c.Ec * W : c.af0, c.sf0, i >= 2, c.ds, c.head_params(), c.PH,
            c.head_off("force.W" + std::to_string(i)), nxt, c.partial, cap, W);
        kl(split_reduce_kernel<ChunkStore>, dim3((W + 1 + 31) / 32, rows.nseg), 256, 0, st,
            c.partial, size_t(cap) * (W + 1), size_t(W + 1), W + 1,
            ChunkStore{rows, kFoRows, c.head_grads() + c.head_off("force.W" + std::to_string(i)), c.PH});
        dz = nxt;
        ldz = W;
        continue;
      }
      c.dep(st, sw);
      FGradProb gq{edge_rows_by_head(c), W + 1, out, H, W, i, c.Ec, c.Qf, c.zf, c.dist, dz, ldz, c.edge_dst,
                   c.edge_src, Wd, B0, HeadG{c.head_grads(), c.PH, c.head_off("force.W" + std::to_string(i))},
                   c.store_af0 ? c.af0 : nullptr};
      atb(gq, c, c.nsplit_edge, sw, c.Ec);
      const HeadW Wi{c.head_params(), c.PH, c.head_off("force.W" + std::to_string(i))};
      if (i == 1 && c.store_sf0) {
        FDxSfProb dq{edge_rows_by_head(c), out, W, W, dz, ldz, Wi, nxt, c.sf0};
        ab(dq, c.Ec, c.S, st, sm, c);
      } else {
        FDxProb dq{edge_rows_by_head(c), out, W, H, W, i, c.Ec, c.Qf, c.zf, c.dist, dz, ldz, c.edge_dst, c.edge_src,
                   Wd, B0, Wi, nxt, c.store_sf0 ? c.sf0 : nullptr};
        ab(dq, c.Ec, c.S, st, sm, c);
      }
      dz = nxt;
      ldz = W;
    }
    // layer 0 (factorised): T = S_dst(dz0) + S_src(dz0)
    float* Sf = c.Sb + size_t(L) * SBS;
    segsum2(c, dz, W, 1, Sf, st);
    c.dep(st, sw2);
    F0NodeGrad ng{node_rows_by_head(c), H, W, H, W, hL, Sf, HeadG{c.head_grads(), c.PH, wf0}};
    atb(ng, c, c.nsplit_node, sw2, c.Nc);
    if (W % 4 == 0) {
      colsum2(c, edge_rows_by_head(c), c.dist, 1, dz, W, c.head_grads() + wf0 + size_t(H) * W, c.PH, sw2);
    } else {
      F0EdgeGrad eg{edge_rows_by_head(c), 2, W, H, W, c.dist, dz, HeadG{c.head_grads(), c.PH, wf0 + size_t(H) * W}};
      atb(eg, c, c.nsplit_edge, sw2, c.Ec);
    }
    c.dep(se, st);  // dL/dh_L = energy part (written) + force part (accumulated next)
    F0Dh dhq{node_rows_by_head(c), W, H, H, W, Sf, HeadW{c.head_params(), c.PH, wf0}, dhL};
    ab(dhq, c.Nc, c.S, st, sm, c);
  }
  if (cs) {  // every owned head's gradient block is final: head-group means
    c.dep(st, sc);
    c.dep(sw, sc);
    c.dep(sw2, sc);
    comm_heads_async(c, sc);
  }
  // ---------------- encoder layers in reverse (hmtl/model.hpp:552-617)
  const bool fused = chain_ok(c);
  bool node_done = false;
  for (int l = L - 1; l >= 0; --l) {
    const std::string p = "layer" + std::to_string(l) + ".";
    const float* h = c.hs + size_t(l) * NH;
    const float* P = c.P + size_t(l) * 2 * NH;
    const float* z2 = c.z2 + size_t(l) * EH;
    const float* agg = c.agg + size_t(l) * NH;
    const float* vz1 = c.vz1 + size_t(l) * NH;
    const float* eW1 = c.params + c.shared_off(p + "edge.W1");
    const float* wd = eW1 + size_t(2) * H * H;
    const float* b1 = c.params + c.shared_off(p + "edge.b1");
    float* geW1 = c.grads + c.shared_off(p + "edge.W1");
    const float* dh = c.dhb + size_t(l + 1) * NH;  // dL/dh_{l+1}
    float* dh2 = c.dhb + size_t(l) * NH;           // dL/dh_l
    float* dvz1 = c.dvz1b + size_t(l) * NH;
    float* dzA = c.dzAb + size_t(l) * EH;
    float* dzB = c.dzBb + size_t(l) * EH;
    float* Sl = c.Sb + size_t(l) * SBS;
    if (l == 0) c.red_sms_now = c.red_sms, c.red_min_now = c.red_min_tail;
    if (!node_done) {  // (else: the previous layer's chain produced dvz1, dh2, dagg)
      if (fused && l == L - 1) {  // [L1, L4] of the top layer as one chain
        chain::Gemm gs[2] = {
            {chain::kBwdL1, H, H, nullptr, vz1, dh, nullptr, dvz1, nullptr},
            {chain::kBwdL4, H, 2 * H, nullptr, dh, nullptr, nullptr, dh2, c.dagg}};
        launch_chain(c, "bwd.node_chain", 2, gs, st);
      } else {
        RecHalves rh(c, true);
        L1Prob q1{node_rows(c), H, H, H, dh, c.params + c.shared_off(p + "node.W2"), vz1, dvz1};
        ab(q1, c.Nc, 1, st, sm, c);
        L4Prob q4{node_rows(c), H, 2 * H, H, dvz1, c.params + c.shared_off(p + "node.W1"), dh, dh2, c.dagg};
        ab(q4, c.Nc, 1, st, sm, c);
      }
    }
    node_done = false;
    const bool mat = c.store_a1;  // tensor-core shapes: gathered operands materialised elementwise
    const bool fz = mat && c.fuse_edge;
    const bool az = mat && c.async_bwd && !fz;
    if (az && c.async_bwd == 1) {  // cp.async dz2 gather producer -> GEMM (dz2, dz1; silu'(z1) from the forward)
      L7AsyncProb q{edge_rows(c), H, H, H, c.params + c.shared_off(p + "edge.W2"), c.dagg, z2,
                    (c.z1_only ? c.a1 : c.s1pb) + size_t(l) * EH, c.edge_dst, dzA, dzB, c.z1_only ? 1 : 0};
      ab(q, c.Ec, 1, st, sm, c);
    } else if (az) {  // ... with silu'(z1) regathered from the node table P in the epilogue
      L7AsyncPProb q{edge_rows(c), H, H, H, c.params + c.shared_off(p + "edge.W2"), c.dagg, z2, P, wd, b1,
                     c.edge_dst, c.edge_src, c.geo, dzA, dzB};
      ab(q, c.Ec, 1, st, sm, c);
    } else if (fz) {  // dz2 producer -> GEMM -> dz1 + per-destination sum, one pass
      L7SegProb q{edge_rows(c), H, H, H, c.params + c.shared_off(p + "edge.W2"), P, wd, b1, c.dagg, z2,
                  c.edge_dst, c.edge_src, c.geo, dzA, dzB, Sl, c.tpart, c.tcap};
      ab(q, c.Ec, 1, st, sm, c);
    } else if (mat) {  // (unfused: elementwise dz2, silu'(z1) materialised, then the dz1 GEMM)
      Prof pr(c, "bwd.edge_act", st);
      kl(edge_bwd_prep_kernel, gridn((c.Ec + kEwU - 1) / kEwU * 32, 256, sm * 16), 256, 0, st,
          c.hdr, P, c.edge_dst, c.edge_src, c.geo, wd, b1, c.dagg, z2, dzA, c.scratch, H);
    } else {
      Prof pr(c, "bwd.edge_dz2_gather", st);
      kl(dz2_kernel, gridn(EH, 256, sm * 16), 256, 0, st, c.hdr, c.edge_dst, c.dagg, z2, dzA, H);
    }
    if (!fz && !az) {
      L7Prob q{edge_rows(c), H, H, H, dzA, c.params + c.shared_off(p + "edge.W2"), P, wd, b1, c.edge_dst,
               c.edge_src, c.geo, dzB, nullptr, z2, mat ? c.scratch : nullptr};
      ab(q, c.Ec, 1, st, sm, c);
    }
    // this layer's node and eW2 weight gradients fork only now: they then overlap the
    // segment sums and the 28-CTA node chain instead of competing with the persistent
    // edge GEMM for SMs
    c.dep(st, sw);
    {
      L2Prob q{node_rows(c), H + 1, H, H, vz1, dh, c.grads + c.shared_off(p + "node.W2")};
      atb(q, c, c.nsplit_node, sw, c.Nc);
    }
    {
      L3Prob q{node_rows(c), 2 * H + 1, H, H, h, agg, dvz1, c.grads + c.shared_off(p + "node.W1")};
      atb(q, c, c.nsplit_node, sw, c.Nc);
    }
    {
      // (on its own stream for layer 0: the step's tail runs the last layer's weight
      // gradients side by side instead of one after another on sw)
      own3 = sw3 != st && (c.wgrad3 >= 2 || (c.wgrad3 == 1 && l == 0));
      used3 = used3 || own3;
      cudaStream_t s6 = own3 ? sw3 : sw;
      if (own3) c.dep(st, s6);
      L6Prob q{edge_rows(c), H + 1, H, H, P, wd, b1, dzA, c.edge_dst, c.edge_src, c.geo,
               c.grads + c.shared_off(p + "edge.W2"), mat ? c.a1 + size_t(l) * EH : nullptr, nullptr, z2,
               c.z1_only ? 1 : 0};
      atb(q, c, c.nsplit_edge, s6, c.Ec);
    }
    if (fz) {
      Prof pr(c, "bwd.segsum_src", st);
      kl(seg_src_kernel, gridn((long long)c.Nc * 32, 256, c.sm_count * 16), 256, 0, st, c.hdr, c.row_ptr, c.rev, dzB,
         c.tpart, c.tcap, Sl, H);
    } else {
      segsum2(c, dzB, H, 0, Sl, st);
    }
    c.dep(st, sw2);  // dz1 and its segment sums ready (second weight-gradient stream)
    colsum2(c, edge_rows(c), &c.geo[0].w, 4, dzB, H, geW1 + size_t(2) * H * H, 0, sw2);
    {
      L10Prob q{node_rows(c), H, 2 * H, H, h, Sl, geW1};
      atb(q, c, c.nsplit_node, sw2, c.Nc);
    }
    if (cs) {  // layer l's shared block is final once its weight-gradient kernels finish
      c.dep(sw, sc);
      c.dep(sw2, sc);
      if (own3) c.dep(sw3, sc);  // (a stream joins the captured graph only once work was put on it)
      const size_t o0 = c.shared_off(p + "edge.W1"), o1 = c.shared_off(p + "node.b2") + size_t(H);
      comm_shared_async(c, o0, o1 - o0, sc);
    }
    if (fused && l > 0) {  // L11 of this layer + [L1, L4] of the layer below
      const std::string pb = "layer" + std::to_string(l - 1) + ".";
      const float* vz1b = c.vz1 + size_t(l - 1) * NH;
      float* dhb2 = c.dhb + size_t(l - 1) * NH;
      chain::Gemm gs[3] = {
          {chain::kBwdL11, 2 * H, H, nullptr, nullptr, Sl, nullptr, dh2, nullptr},
          {chain::kBwdL1, H, H, nullptr, vz1b, nullptr, nullptr, c.dvz1b + size_t(l - 1) * NH, nullptr},
          {chain::kBwdL4, H, 2 * H, nullptr, dh2, nullptr, nullptr, dhb2, c.dagg}};
      launch_chain(c, "bwd.node_chain", 3, gs, st);
      node_done = true;
      continue;
    }
    {
      RecHalves rh(c, l > 0);  // (layer 0's L11 is never inside a chain)
      L11Prob q{node_rows(c), 2 * H, H, H, Sl, eW1, dh2};
      ab(q, c.Nc, 1, st, sm, c);
    }
  }
  {
    const float* dh0 = c.dhb;
    Prof pr(c, "bwd.embed_grad", st);
    const size_t shm = size_t(c.NS) * H * 4;
    if (shm <= 48 * 1024 && size_t(c.Nc + kEmbChunk - 1) / kEmbChunk * c.NS * H <= c.partial_cap) {
      kl(embed_grad_part, (c.Nc + kEmbChunk - 1) / kEmbChunk, 128, shm, st, c.hdr, c.species, dh0, c.partial, H, c.NS);
      kl(split_reduce_kernel<EmbedStore>, dim3((c.NS * H + 31) / 32, 1), 256, 0, st,
          c.partial, 0, size_t(c.NS) * H, c.NS * H, EmbedStore{c.hdr, c.grads + c.shared_off("embed")});
    } else {
      kl(embed_grad_kernel, gridn((long long)c.NS * H, 128, sm * 8), 128, 0, st,
          c.hdr, c.species, dh0, c.grads + c.shared_off("embed"), H, c.NS);
    }
  }
  if (cs) {  // the rest of the shared block (the embedding)
    c.dep(st, sc);
    comm_shared_async(c, 0, c.shared_off("layer0.edge.W1"), sc);
  }
  c.dep(sw, st);  // every weight gradient is final (and, with MTL-par, averaged)
  c.dep(sw2, st);
  if (used3) c.dep(sw3, st);
  if (cs) c.dep(sc, st);
}

// debug probe: z1 of layer l (the factorised pre-activation), [E x H]
namespace {
__global__ void z1_kernel(const DevHdr* hdr, const float* __restrict__ P, const int* __restrict__ dst,
                          const int* __restrict__ src, const float4* __restrict__ geo, const float* __restrict__ wd,
                          const float* __restrict__ b1, float* __restrict__ out, int H) {
  pdl_wait();
  const long long total = (long long)hdr->E * H;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int e = int(t / H), k = int(t % H);
    out[t] = z1_of(P, H, dst[e], src[e], geo[e].w, wd, b1, k);
  }
}
}  // namespace

void launch_debug_z1(Ctx& c, int l, float* out, cudaStream_t st) {
  const std::string p = "layer" + std::to_string(l) + ".";
  const float* W1 = c.params + c.shared_off(p + "edge.W1");
  kl(z1_kernel, gridn((long long)c.Ec * c.H, 256, c.sm_count * 16), 256, 0, st,
      c.hdr, c.P + size_t(l) * 2 * c.Nc * c.H, c.edge_dst, c.edge_src, c.geo, W1 + size_t(2) * c.H * c.H,
      c.params + c.shared_off(p + "edge.b1"), out, c.H);
}

// ---------------------------------------------------------------- AdamW
namespace {
// A step whose batch raised a device error (edge overflow, unowned head, empty
// graph, non-finite prediction) leaves the parameters, m/v and the step counter
// untouched: the reference throws before any update (hmtl/model.hpp:341-347,
// 483-486) and the host raises the same error when it reads the step's result.
__global__ void adam_tick(DevHdr* hdr) {
  pdl_wait();
  if (hdr->err == 0) hdr->step += 1;
}
// torch.optim.AdamW ordering (decision recorded in DESIGN.md)
__global__ void adamw_kernel(const DevHdr* hdr, float* __restrict__ p, const float* __restrict__ g,
                             float* __restrict__ m, float* __restrict__ v, size_t n, float lr, float b1, float b2,
                             float eps, float wd) {
  pdl_wait();
  if (hdr->err != 0) return;  // see adam_tick
  const int t = hdr->step;
  const float bc1 = float(1.0 - pow(double(b1), double(t)));
  const float bc2s = float(sqrt(1.0 - pow(double(b2), double(t))));
  const float step_size = lr / bc1;
  const float decay = float(1.0 - double(lr) * double(wd));
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    float pi = p[i] * decay;
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float denom = sqrtf(vi) / bc2s + eps;
    p[i] = pi - step_size * mi / denom;
  }
}
}  // namespace

void launch_adamw(Ctx& c, const hmtl_train_cfg& cfg, cudaStream_t st, bool defer_images) {
  struct Rebuild {
    Ctx& c;
    cudaStream_t st;
    bool defer;
    ~Rebuild() {  // weights changed: refresh the B images (after the update) -- or, inside a
      if (defer && c.bimg_ready) c.bimg_stale = true;  // train step, at the start of the next
      else launch_bimg_all(c, st);                     // step, overlapped with its batch prep
    }
  } rebuild{c, st, defer_images};
  kl(adam_tick, 1, 1, 0, st, c.hdr);
  {
    Prof pr(c, "adamw", st);
    kl(adamw_kernel, gridn(c.PT, 256, c.sm_count * 8), 256, 0, st, c.hdr, c.params, c.grads, c.adam_m, c.adam_v, c.PT,
                                                                   cfg.lr, cfg.beta1, cfg.beta2, cfg.eps,
                                                                   cfg.weight_decay);
  }
}

}  // namespace hmtl_b200
