// selftest.cu -- direct checks of the tcgen05 engines on plain matrices
// (hmtl_selftest_gemm, used by tests/test_gpu_tc.py; not on the training path).
#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "tc.cuh"

namespace hmtl_b200 {
namespace {

// row GEMM: C[r][n] = sum_k X[r][k] * B[k][n]
struct StRow {
  RowSet rows;
  int K, Ncols;
  const float* bimg;
  size_t bimg_seg;
  const float* X;
  float* C;
  struct RC {};
  struct Aux {};
  __device__ RC rctx(int, int) const { return RC{}; }
  __device__ Aux epi_aux(int, int, const RC&, int) const { return Aux{}; }
  __device__ float4 a4(int, int r, const RC&, int k) const {
    return *reinterpret_cast<const float4*>(X + size_t(r) * K + k);
  }
  using Raw = float4;
  __device__ float4 raw4(int s, int r, const RC& rc, int k) const { return a4(s, r, rc, k); }
  __device__ float4 fin4(int, int, const RC&, int, const float4& x) const { return x; }
  __device__ void epi4(int, int r, const RC&, int n, float4 acc, const Aux&) const {
    *reinterpret_cast<float4*>(C + size_t(r) * Ncols + n) = acc;
  }
};
// reduce GEMM: C[m][n] = sum_r X[r][m] * Y[r][n]
struct StRed {
  RowSet rows;
  int M, Ncols, colsum;
  const float *X, *Y;
  float* C;
  __device__ float4 x4(int, int r, int m) const { return *reinterpret_cast<const float4*>(X + size_t(r) * M + m); }
  __device__ float4 y4(int, int r, int n) const {
    return *reinterpret_cast<const float4*>(Y + size_t(r) * Ncols + n);
  }
  __device__ void store(int, int m, int n, float v) const { C[size_t(m) * Ncols + n] = v; }
  __device__ float4 xfin(float4 v) const { return v; }
  __device__ float4 yfin(float4 v) const { return v; }
};

__global__ void st_bimg(const float* B, int K, int N, float* out) {  // B is [K][N]
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < K * N; t += gridDim.x * blockDim.x) {
    const int n = t % N, k = t / N;
    const float x = B[size_t(k) * N + n], h = tc::tf32_hi(x);
    const int ch = k / tc::KC, c16 = (k % tc::KC) / 4, q = k % 4;
    float* o = out + size_t(ch) * 2 * tc::KC * N;
    const uint32_t off = tc::sw128(n, c16) / 4 + q;
    o[off] = h;
    o[size_t(tc::KC) * N + off] = x - h;
  }
}

}  // namespace
}  // namespace hmtl_b200

using namespace hmtl_b200;

namespace hmtl_b200 {
namespace {
__global__ void set_dbg(int v) { tc::g_tc_debug = v; }
}  // namespace
}  // namespace hmtl_b200

extern "C" int hmtl_selftest_gemm(int mode, int variant, int rows, int K, int N, const float* X, const float* Y,
                                  float* C) {
  cudaSetDevice(0);
  float *dX, *dY, *dC, *img, *part;
  int* dcnt;
  const size_t nx = size_t(rows) * K, ny = mode == 0 ? size_t(K) * N : size_t(rows) * N;
  const size_t nc = mode == 0 ? size_t(rows) * N : size_t(K + 1) * N;
  HMTL_CUDA(cudaMalloc(&dX, nx * 4));
  HMTL_CUDA(cudaMalloc(&dY, ny * 4));
  HMTL_CUDA(cudaMalloc(&dC, nc * 4));
  HMTL_CUDA(cudaMalloc(&img, 2 * size_t(K) * N * 4));
  HMTL_CUDA(cudaMalloc(&part, size_t(64) * (K + 1) * N * 4));
  HMTL_CUDA(cudaMalloc(&dcnt, 4));
  cudaMemcpy(dX, X, nx * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Y, ny * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dcnt, &rows, 4, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, nc * 4);
  (void)variant;
  RowSet rs;
  rs.count = dcnt;
  if (mode == 0) {
    st_bimg<<<64, 256>>>(dY, K, N, img);
    StRow p{rs, K, N, img, 0, dX, dC};
    const tc::RowPlan plan = tc::row_plan(K, N);
    cudaFuncSetAttribute(tc::tc_row_kernel<StRow>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(plan.smem));
    tc::tc_row_kernel<StRow><<<(rows + 127) / 128, tc::kRowThreads, plan.smem>>>(p, plan);
  } else {
    StRed p{rs, K, N, 0, dX, dY, dC};
    const int ns = 4;
    dim3 grid((K + 127) / 128, ns, 1);
    if (variant & 1) {  // TMA operand path (tc_red_tma_kernel)
      CUtensorMap mx, my;
      if (!tc::tmap_2d(&mx, dX, rows, K) || !tc::tmap_2d(&my, dY, rows, N)) return fail(HMTL_ERR_INTERNAL, "tmap");
      const size_t SB = tc::red_stage_bytes(N);
      const int stages = int(std::min<size_t>(4, (tc::kSmemLimit - size_t(32) * N * 4 - 4096) / SB));
      const size_t smem = tc::tc_red_tma_smem(N, stages);
      cudaFuncSetAttribute(tc::tc_red_tma_kernel<StRed>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      tc::tc_red_tma_kernel<StRed><<<grid, tc::kRedTmaThreads, smem>>>(p, mx, mx, my, 0, part, ns, stages);
      const cudaError_t le = cudaGetLastError();
      if (le != cudaSuccess) return fail(HMTL_ERR_INTERNAL, std::string("tma launch: ") + cudaGetErrorString(le));
    } else {
      const size_t smem = tc::tc_red_smem(N);
      cudaFuncSetAttribute(tc::tc_red_kernel<StRed>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      tc::tc_red_kernel<StRed><<<grid, tc::kRedThreads, smem>>>(p, part, ns, tc::red_stages(N));
    }
    tc::tc_red_reduce(p, part, ns, 0);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) cudaMemcpy(C, dC, (mode == 0 ? nc : size_t(K) * N) * 4, cudaMemcpyDeviceToHost);
  cudaFree(dX), cudaFree(dY), cudaFree(dC), cudaFree(img), cudaFree(part), cudaFree(dcnt);
  if (e != cudaSuccess) return fail(HMTL_ERR_INTERNAL, std::string("selftest: ") + cudaGetErrorString(e));
  return 0;
}

// Timed engine run on device-resident random matrices: returns the mean kernel
// time (ms) of `iters` launches (CUDA events), for roofline work on the engine.
namespace hmtl_b200 {
namespace {
}  // namespace
}  // namespace hmtl_b200

extern "C" int hmtl_selftest_time(int mode, int rows, int K, int N, int iters, float* ms) {
  cudaSetDevice(0);
  const int dbg = mode >> 4;
  mode &= 15;
  set_dbg<<<1, 1>>>(dbg);
  float *dX, *dY, *dC, *img, *part;
  int* dcnt;
  const size_t nx = size_t(rows) * K, ny = mode == 0 ? size_t(K) * N : size_t(rows) * N;
  const size_t nc = mode == 0 ? size_t(rows) * N : size_t(K + 1) * N;
  const int ns = mode == 0 ? 1 : 148 / ((K + 127) / 128);
  HMTL_CUDA(cudaMalloc(&dX, nx * 4));
  HMTL_CUDA(cudaMalloc(&dY, ny * 4));
  HMTL_CUDA(cudaMalloc(&dC, nc * 4));
  HMTL_CUDA(cudaMalloc(&img, 2 * size_t(K) * N * 4));
  HMTL_CUDA(cudaMalloc(&part, size_t(ns) * (K + 1) * N * 4));
  HMTL_CUDA(cudaMalloc(&dcnt, 4));
  cudaMemset(dX, 0, nx * 4);
  cudaMemset(dY, 0, ny * 4);
  cudaMemcpy(dcnt, &rows, 4, cudaMemcpyHostToDevice);
  RowSet rs;
  rs.count = dcnt;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto launch = [&]() {
    if (mode == 0) {
      StRow p{rs, K, N, img, 0, dX, dC};
      const tc::RowPlan plan = tc::row_plan(K, N);
      cudaFuncSetAttribute(tc::tc_row_kernel<StRow>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(plan.smem));
      const int tiles = (rows + 127) / 128;
      tc::tc_row_kernel<StRow><<<tiles < 148 ? tiles : 148, tc::kRowThreads, plan.smem>>>(p, plan);
    } else {
      StRed p{rs, K, N, 0, dX, dY, dC};
      const size_t smem = tc::tc_red_smem(N);
      cudaFuncSetAttribute(tc::tc_red_kernel<StRed>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      dim3 grid((K + 127) / 128, ns, 1);
      tc::tc_red_kernel<StRed><<<grid, tc::kRedThreads, smem>>>(p, part, ns, tc::red_stages(N));
    }
  };
  launch();
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) launch();
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  *ms = t / iters;
  cudaEventDestroy(a), cudaEventDestroy(b);
  set_dbg<<<1, 1>>>(0);
  cudaDeviceSynchronize();
  cudaFree(dX), cudaFree(dY), cudaFree(dC), cudaFree(img), cudaFree(part), cudaFree(dcnt);
  if (e != cudaSuccess) return fail(HMTL_ERR_INTERNAL, std::string("selftest_time: ") + cudaGetErrorString(e));
  return 0;
}

// Tensor-pipe issue-rate probe (engine design, not the training path): one CTA
// per SM, lane 0 issues n back-to-back MMAs (M = 128, N, one K step each) into
// one accumulator and reports SM clocks per MMA.  variant: 0 tf32 A,B in smem;
// 1 tf32 A in TMEM; 2 bf16 (kind::f16) A,B in smem; 3 bf16 A in TMEM.
namespace hmtl_b200 {
namespace {
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int variant, int N, int n, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = tc::align1k(sm_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < (16384 + 32768) / 16; i += blockDim.x) reinterpret_cast<float4*>(sm)[i] = make_float4(0, 0, 0, 0);
  if (tid < 32) tc::tmem_alloc(&slot, 512);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_proxy_async();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  if (variant == 4) {  // warp-uniform 12-MMA blocks (the engine's issue path)
    if (tid < 32) {
      const uint32_t a_s = tc::smem_u32(sm), b_s = tc::smem_u32(sm + 16384);
      const long long t0 = clock64();
      for (int i = 0; i < n; i += 12) tc::issue_chunk_warp(tmem, a_s, a_s + 4096, b_s, b_s + 4096, tc::idesc_tf32(N), i ? 1u : 0u);
      tc::commit_warp(&bar);
      tc::mbar_wait(&bar, 0);
      const long long t1 = clock64();
      if (tid == 0) out[blockIdx.x] = t1 - t0;
    }
  } else if (tid == 0) {
    const bool f16 = variant >= 2, ts = variant & 1;
    const uint32_t idesc = f16 ? ((1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24))
                               : tc::idesc_tf32(N);
    const uint32_t a_s = tc::smem_u32(sm), b_s = tc::smem_u32(sm + 16384);
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      const uint32_t o = 32 * (i & 3);
      const uint64_t bd = tc::sdesc_sw128(b_s + o);
      const uint32_t acc = i ? 1u : 0u;
      if (!f16 && !ts) {
        tc::mma_tf32(tmem, tc::sdesc_sw128(a_s + o), bd, idesc, acc);
      } else if (!f16) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                     "r"(tmem + 256 + 8 * (i & 3)), "l"(bd), "r"(idesc), "r"(acc));
      } else if (!ts) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(tc::sdesc_sw128(a_s + o)), "l"(bd), "r"(idesc), "r"(acc));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                     "r"(tmem + 256 + 8 * (i & 3)), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (tid < 32) tc::tmem_dealloc(tmem, 512);
}
}  // namespace
}  // namespace hmtl_b200

extern "C" int hmtl_selftest_mma_rate(int variant, int N, int n, float* clk_per_mma) {
  cudaSetDevice(0);
  long long* d;
  HMTL_CUDA(cudaMalloc(&d, 148 * sizeof(long long)));
  const int smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate_kernel<<<148, 128, smem>>>(variant, N, n, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148] = {0};
  if (e == cudaSuccess) cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(HMTL_ERR_INTERNAL, std::string("mma_rate: ") + cudaGetErrorString(e));
  double s = 0;
  for (long long v : h) s += double(v);
  *clk_per_mma = float(s / 148 / n);
  return 0;
}

// Shared-memory ingress probe (engine design, not the training path): every CTA
// (one per SM) moves `total` bytes into its shared memory in `chunk`-byte bulk
// copies with `depth` in flight and reports SM clocks.  mode 0: from global
// (src + blockIdx * stride: stride 0 = every CTA reads the same bytes, as the
// weight images); mode 1: from the 2-CTA cluster peer's shared memory (both CTAs
// push to each other at once, as the chain's operand exchange).
namespace hmtl_b200 {
namespace {
__global__ void __launch_bounds__(256, 1)
    ingress_kernel(int mode, const uint8_t* src, long long stride, int total, int chunk, int depth, long long* out,
                   const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = tc::align1k(sm_raw);
  __shared__ uint64_t bar[16];
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int i = 0; i < 16; ++i) tc::mbar_init(&bar[i], 1);
    tc::fence_mbar_init();
  }
  uint32_t crank = 0;
  if (mode == 1) {
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncwarp();
  }
  const int n = total / chunk;
  if (mode >= 100) {  // prefetch this CTA's source bytes into L2, then give DRAM 4 us
    mode -= 100;
    if (threadIdx.x == 0) {
      const uint8_t* s = src + size_t(blockIdx.x) * size_t(mode == 3 ? total : stride);
      for (int o = 0; o < total; o += 65536)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s + o), "r"(total - o < 65536 ? total - o : 65536)
                     : "memory");
      const long long t = clock64();
      while (clock64() - t < 8000) {
      }
    }
  }
  __syncthreads();
  long long t0 = clock64();
  if (mode == 2) {  // every thread: cp.async 16 B pieces of the whole range at once
    const uint8_t* s = src + size_t(blockIdx.x) * size_t(stride);
    for (int o = threadIdx.x * 16; o < total; o += blockDim.x * 16) tc::cp_async16(tc::smem_u32(sm + o), s + o, 16u);
    tc::cp_async_commit();
    tc::cp_async_wait<0>();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    return;
  }
  if (threadIdx.x >= 32) return;
  if (mode == 3) {  // tensor TMA: 32 x 128 fp32 boxes (16 KB, 128 B swizzle) through a ring of `depth`
    if (lane == 0) {
      const int rows0 = int(blockIdx.x) * (total / 128);  // (stride ignored: distinct rows per CTA)
      for (int i = 0; i < n; ++i) {
        const int b = i % depth;
        if (i >= depth) tc::mbar_wait(&bar[b], uint32_t((i / depth - 1) & 1));
        tc::mbar_expect_tx(&bar[b], 16384u);
        tc::tma_2d(sm + size_t(b) * 16384, &tm, 0, rows0 + i * 128, &bar[b]);
      }
      for (int i = n > depth ? n - depth : 0; i < n; ++i) tc::mbar_wait(&bar[i % depth], uint32_t((i / depth) & 1));
      out[blockIdx.x] = clock64() - t0;
    }
    return;
  }
  if (lane == 0) {
    if (mode == 0) {
      const uint8_t* s = src + size_t(blockIdx.x) * size_t(stride);
      for (int i = 0; i < n; ++i) {
        const int b = i % depth;
        if (i >= depth) tc::mbar_wait(&bar[b], uint32_t((i / depth - 1) & 1));
        tc::mbar_expect_tx(&bar[b], uint32_t(chunk));
        tc::bulk_g2s(sm + size_t(b) * chunk, s + size_t(i) * chunk, uint32_t(chunk), &bar[b]);
      }
      for (int i = n > depth ? n - depth : 0; i < n; ++i) tc::mbar_wait(&bar[i % depth], uint32_t((i / depth) & 1));
    } else {  // push every chunk into the peer's slot i at once (receiver-side barriers), wait for ours
      const uint32_t peer = crank ^ 1u;
      const uint32_t lsrc = tc::smem_u32(sm + size_t(n) * chunk);  // send area after the receive slots
      for (int i = 0; i < n; ++i) {
        uint32_t rb, rd;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(tc::smem_u32(&bar[i])), "r"(peer));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rd) : "r"(tc::smem_u32(sm + size_t(i) * chunk)), "r"(peer));
        asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(rb), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rd),
                     "r"(lsrc), "r"(chunk), "r"(rb)
                     : "memory");
      }
      for (int i = 0; i < n; ++i) tc::mbar_wait(&bar[i], 0);
    }
    out[blockIdx.x] = clock64() - t0;
  }
  __syncwarp();
  if (mode == 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
}  // namespace
}  // namespace hmtl_b200

extern "C" int hmtl_selftest_ingress(int mode, int grid, long long stride, int total, int chunk, int depth,
                                     float* bytes_per_clk) {
  cudaSetDevice(0);
  const bool pf = mode >= 40, cold = mode >= 20;  // + 20: L2 flushed before the timed pass; + 40: and the
  mode %= 20;                                       // kernel prefetches its source into L2 first (4 us head start)
  const int cl = mode >= 10 ? 2 : 1;  // mode + 10: the same, CTAs in 2-CTA clusters (both SMs of a TPC)
  mode %= 10;
  if (depth < 1 || depth > 16 || chunk % 16 || total % chunk || grid < 1 || grid > 148 ||
      (mode == 1 && (grid % 2 || total / chunk > 16)) || grid % cl)
    return fail(HMTL_ERR_CONTRACT, "ingress: bad arguments");
  if (mode == 3) chunk = 16384;
  const size_t smem = (mode == 1 ? size_t(total + chunk) : mode == 2 ? size_t(total) : size_t(depth) * chunk) + 1024;
  if (smem > 232448) return fail(HMTL_ERR_CONTRACT, "ingress: ring exceeds shared memory");
  uint8_t* src = nullptr;
  long long* d;
  const size_t src_bytes = mode == 0 || mode == 2 ? size_t(stride) * (grid - 1) + size_t(total)
                          : mode == 3 ? size_t(total) * grid : 16;
  HMTL_CUDA(cudaMalloc(&src, src_bytes));
  HMTL_CUDA(cudaMemset(src, 1, src_bytes));
  HMTL_CUDA(cudaMalloc(&d, 148 * sizeof(long long)));
  cudaFuncSetAttribute(ingress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  CUtensorMap tm{};
  if (mode == 3 && !tc::tmap_2d(&tm, reinterpret_cast<const float*>(src), (long long)(src_bytes / 128), 32,
                                CU_TENSOR_MAP_SWIZZLE_128B, 128))
    return fail(HMTL_ERR_INTERNAL, "ingress: tensor map");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(mode == 2 ? 256 : 32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = mode == 1 ? 2 : cl, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  void* flush = nullptr;
  if (cold) HMTL_CUDA(cudaMalloc(&flush, size_t(256) << 20));
  for (int rep = 0; rep < 3 && e == cudaSuccess; ++rep) {  // (the first pass warms L2)
    if (cold) cudaMemset(flush, rep, size_t(256) << 20);
    cudaLaunchKernelEx(&cfg, ingress_kernel, mode + (pf ? 100 : 0), static_cast<const uint8_t*>(src), stride, total, chunk,
                       depth, d, tm);
    e = cudaDeviceSynchronize();
  }
  if (flush) cudaFree(flush);
  std::vector<long long> h(grid, 0);
  if (e == cudaSuccess) cudaMemcpy(h.data(), d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
  cudaFree(d);
  cudaFree(src);
  if (e != cudaSuccess) return fail(HMTL_ERR_INTERNAL, std::string("ingress: ") + cudaGetErrorString(e));
  double s = 0;
  for (long long v : h) s += double(v);
  *bytes_per_clk = float(double(total) / (s / grid));
  return 0;
}

// CTA-pair (cta_group::2) accumulator layout probe (engine design): one MMA of
// M = 128 or 256 (MR = M / 2 rows per CTA) and N columns with A[r][0] = r + 1,
// A[r][1] = 1024, B[n][0] = 1, B[n][1] = n + 1, so D[r][n] = r + 1 + 1024 (n + 1);
// out[cta][lane][col] = TMEM lane `lane`, column col (< 32) of each CTA.
namespace hmtl_b200 {
namespace {
__global__ void __launch_bounds__(128, 1) pair_probe_kernel(int M, int N, float* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = tc::align1k(sm_raw);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint32_t crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, MR = M / 2;
  float* A = reinterpret_cast<float*>(sm);
  float* B = reinterpret_cast<float*>(sm + 16384);
  for (int i = tid; i < (16384 + 16384) / 4; i += 128) A[i] = 0.f;
  __syncthreads();
  if (tid < MR) {
    A[tc::sw128(tid, 0) / 4] = float(int(crank) * MR + tid + 1);
    A[tc::sw128(tid, 0) / 4 + 1] = 1024.f;
  }
  if (tid < N / 2) {
    B[tc::sw128(tid, 0) / 4] = 1.f;
    B[tc::sw128(tid, 0) / 4 + 1] = float(int(crank) * (N / 2) + tid + 1);
  }
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_proxy_async();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc::tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  if (crank == 0 && tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(tc::sdesc_sw128(tc::smem_u32(A))), "l"(tc::sdesc_sw128(tc::smem_u32(B))), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     tc::smem_u32(&bar)),
                 "h"(uint16_t(3))
                 : "memory");
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  float v[32];
  tc::tmem_ld32(tmem + (uint32_t(warp * 32) << 16), v);
  for (int c = 0; c < 32; ++c) out[(size_t(crank) * 128 + warp * 32 + lane) * 32 + c] = v[c];
  float w[16];  // the .16x256b shape of the same accumulator (lanes 32 warp + 16 h, columns 0-31)
  for (int h = 0; h < 2; ++h) {
    tc::tmem_ld16x32(tmem + (uint32_t(warp * 32 + 16 * h) << 16), w);
    tc::tmem_wait_ld();
    for (int i = 0; i < 16; ++i) out[2 * 128 * 32 + ((size_t(crank) * 4 + warp) * 2 + h) * 512 + lane * 16 + i] = w[i];
  }
  tc::tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
}  // namespace
}  // namespace hmtl_b200

extern "C" int hmtl_selftest_pair_layout(int M, int N, float* out) {
  cudaSetDevice(0);
  if ((M != 128 && M != 256) || N < 32 || N > 256 || N % 32) return fail(HMTL_ERR_CONTRACT, "pair_layout: bad shape");
  float* d;
  HMTL_CUDA(cudaMalloc(&d, 4 * 128 * 32 * sizeof(float)));
  HMTL_CUDA(cudaMemset(d, 0, 4 * 128 * 32 * sizeof(float)));
  const int smem = 32768 + 1024;
  cudaFuncSetAttribute(hmtl_b200::pair_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, hmtl_b200::pair_probe_kernel, M, N, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) cudaMemcpy(out, d, 4 * 128 * 32 * sizeof(float), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(HMTL_ERR_INTERNAL, std::string("pair_layout: ") + cudaGetErrorString(e));
  return 0;
}
