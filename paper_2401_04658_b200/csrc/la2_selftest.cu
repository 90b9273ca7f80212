// Self-test of the tcgen05 operand layouts used by la2_tc_kernel.
// D[M][N] = A[M][K] * B[K][N] with A staged K-major or MN-major and B staged
// K-major or MN-major in SW128 regions, exactly as the F kernel stages Q/K/V/P/KV.
// Used by tests/test_gpu_selftest.py and tools/; not on the product path: it is built
// into its own development library, libla2_dev.so (include/la2_dev.h), so the shipping
// libla2.so exports only the reference-replacing ABI of include/la2.h.
#include <cstdio>

#include "../../include/la2_dev.h"
#include "la2_kernels.h"
#include "la2_ptx.cuh"

namespace {
thread_local char g_dev_err[256] = "";
int dev_error(const char* msg) {
  std::snprintf(g_dev_err, sizeof(g_dev_err), "%s", msg);
  return LA2_ERR_VALUE;
}
int dev_cuda_error(const char* where, cudaError_t e) {
  std::snprintf(g_dev_err, sizeof(g_dev_err), "%s: %s", where, cudaGetErrorString(e));
  return LA2_ERR_CUDA;
}
}  // namespace

extern "C" LA2_API const char* la2_dev_last_error(void) { return g_dev_err; }

namespace la2 {

__global__ void __launch_bounds__(128, 1)
    la2_umma_selftest_kernel(const float* __restrict__ A, const float* __restrict__ Bm,
                             float* __restrict__ D, int M, int N, int K, int a_mn, int b_mn) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  // A: up to 128x128 bf16 = 32 KB, B: up to 128x128 = 32 KB
  uint8_t* sA = smem;
  uint8_t* sB = smem + 32768;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 65536 + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // Stage A. K-major: region by K/64 holding [M][64]; MN-major: region by M/64 holding [K][64].
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int m = e / K, kx = e % K;
    const __nv_bfloat16 x = __float2bfloat16_rn(A[e]);
    int row, col, region_rows;
    uint8_t* base;
    if (!a_mn) { row = m; col = kx; region_rows = M; base = sA + (col / 64) * region_rows * 128; }
    else { row = kx; col = m; region_rows = K; base = sA + (col / 64) * region_rows * 128; }
    const int c = col % 64;
    const int chunk = (c / 8) ^ (row & 7);
    *reinterpret_cast<__nv_bfloat16*>(base + row * 128 + chunk * 16 + (c % 8) * 2) = x;
  }
  // Stage B (K x N). K-major: region by K/64 holding [N][64]; MN-major: region by N/64 holding [K][64].
  for (int e = tid; e < K * N; e += blockDim.x) {
    const int kx = e / N, n = e % N;
    const __nv_bfloat16 x = __float2bfloat16_rn(Bm[e]);
    int row, col, region_rows;
    if (!b_mn) { row = n; col = kx; region_rows = N; }
    else { row = kx; col = n; region_rows = K; }
    uint8_t* base = sB + (col / 64) * region_rows * 128;
    const int c = col % 64;
    const int chunk = (c / 8) ^ (row & 7);
    *reinterpret_cast<__nv_bfloat16*>(base + row * 128 + chunk * 16 + (c % 8) * 2) = x;
  }
  fence_proxy_async_smem();
  if (tid == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *slot;
  const bool a_tmem = (a_mn == 2);
  if (a_tmem) {
    // A row m -> TMEM lane m (M = 128) or lane 32*(m/16) + m%16 (M = 64, the D layout
    // of an M = 64 MMA), columns 128.. as packed bf16 pairs (K-major)
    const int m = (M == 128) ? (warp & 3) * 32 + lane : (warp & 3) * 16 + (lane & 15);
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t r[16];
      for (int j = 0; j < 16; ++j)
        r[j] = pack_bf16x2(A[m * K + 2 * (c0 + j)], A[m * K + 2 * (c0 + j) + 1]);
      tmem_st16(tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 128 + c0, r);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (tid == 0) {
    const uint32_t id = idesc_bf16(M, N, a_tmem ? 0 : a_mn, b_mn);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int kk = 0; kk < K / 16; ++kk) {
      uint64_t ad, bd;
      if (!a_mn) ad = sdesc_sw128(a0 + (kk >> 2) * M * 128 + (kk & 3) * 32, 16, 1024);
      else ad = sdesc_sw128(a0 + kk * 2048, K * 128, 1024);
      if (!b_mn) bd = sdesc_sw128(b0 + (kk >> 2) * N * 128 + (kk & 3) * 32, 16, 1024);
      else bd = sdesc_sw128(b0 + kk * 2048, K * 128, 1024);
      if (a_tmem) umma_bf16_ts(tbase, tbase + 128 + kk * 8, bd, id, kk > 0);
      else umma_bf16_ss(tbase, ad, bd, id, kk > 0);
    }
    umma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  const int q4 = warp & 3;
  const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
  int m;
  bool valid;
  if (M == 128) { m = q4 * 32 + lane; valid = true; }
  else { m = q4 * 16 + lane; valid = lane < 16; }
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tbase + lane_off + c0, v);
    tmem_ld_wait();
    if (valid)
      for (int j = 0; j < 16; ++j) D[m * N + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

}  // namespace la2

extern "C" LA2_API int la2_selftest_umma(const float* A, const float* B, float* D, int M, int N, int K,
                                 int a_mn, int b_mn, void* stream) {
  using namespace la2;
  if (!((M == 64 || M == 128) && (N == 64 || N == 128) && (K == 64 || K == 128)))
    return dev_error("selftest: M,N in {64,128}, K in {64,128}");
  const int smem = 65536 + 128 + 1024;
  cudaError_t e = cudaFuncSetAttribute(la2_umma_selftest_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return dev_cuda_error("selftest attr", e);
  la2_umma_selftest_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(A, B, D, M, N, K,
                                                                                a_mn, b_mn);
  e = cudaGetLastError();
  if (e != cudaSuccess) return dev_cuda_error("selftest launch", e);
  return 0;
}

// ---------------------------------------------------------------------------
// Microbenchmark: cycles per tcgen05.mma for one (M, N, A-mode, B-major) shape.
// a_mode: 0 = A K-major smem, 1 = A MN-major smem, 2 = A from TMEM. One CTA per
// SM issues `iters` MMAs back to back (K = 16 each) and reports clock cycles.
namespace la2 {
__global__ void __launch_bounds__(128, 1)
    la2_umma_bench_kernel(int M, int N, int a_mode, int b_mn, int iters, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 65536 + 64);
  for (int e = threadIdx.x; e < 65536 / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(smem)[e] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *slot;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_bf16(M, N, a_mode == 1 ? 1 : 0, b_mn & 1);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 32768);
    const uint64_t ad = a_mode == 1 ? sdesc_sw128(a0, 16384, 1024) : sdesc_sw128(a0, 16, 1024);
    const uint64_t bd = (b_mn & 1) ? sdesc_sw128(b0, 16384, 1024) : sdesc_sw128(b0, 16, 1024);
    const int chains = (b_mn >> 1) < 1 ? 1 : (b_mn >> 1);
    // precomputed descriptors; 16 MMAs per unrolled group, D rotates over `chains`
    const uint32_t d1 = tbase + (chains > 1 ? N : 0), d2 = tbase + (chains > 2 ? 2 * N : 0),
                   d3 = tbase + (chains > 3 ? 3 * N : (chains > 1 ? N : 0));
    const uint32_t dd[4] = {tbase, d1, chains == 3 ? d2 : (chains > 1 ? d2 : tbase), d3};
    const uint32_t at = tbase + 256;
    long long t0 = clock64();
    if (a_mode == 2) {
      for (int i = 0; i < iters; i += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u) umma_bf16_ts(dd[u & 3], at, bd, id, 1);
      }
    } else {
      for (int i = 0; i < iters; i += 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u) umma_bf16_ss(dd[u & 3], ad, bd, id, 1);
      }
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tbase, 512);
}
}  // namespace la2

extern "C" LA2_API int la2_bench_umma(int M, int N, int a_mode, int b_mn, int iters, int ctas,
                                      long long* out, void* stream) {
  using namespace la2;
  const int smem = 65536 + 128 + 1024;
  cudaError_t e = cudaFuncSetAttribute(la2_umma_bench_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return dev_cuda_error("bench attr", e);
  la2_umma_bench_kernel<<<ctas, 128, smem, static_cast<cudaStream_t>(stream)>>>(M, N, a_mode, b_mn,
                                                                               iters, out);
  e = cudaGetLastError();
  if (e != cudaSuccess) return dev_cuda_error("bench launch", e);
  return 0;
}

// ---------------------------------------------------------------------------
// Microbenchmark: TMEM -> register load throughput (tcgen05.ld 32x32b.x16) with
// `warps` warps (multiple of 4); returns cycles for `iters` loads of 16 columns
// per warp (64 B per lane -> 2 KB per warp per load).
namespace la2 {
__global__ void la2_tmem_bench_kernel(int iters, int batch, long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  float acc = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < iters; i += 4) {
    float v[4][16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      tmem_ld16(tbase + ((i + u + warp) & 31) * 16, v[u]);
      if (batch == 1) tmem_ld_wait();
    }
    tmem_ld_wait();
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int e = 0; e < 16; ++e) acc += v[u][e];
  }
  long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(slot, 512);
}
}  // namespace la2

extern "C" LA2_API int la2_bench_tmem(int warps, int iters, int batch, int ctas, long long* out,
                                      float* sink, void* stream) {
  using namespace la2;
  la2_tmem_bench_kernel<<<ctas, warps * 32, 0, static_cast<cudaStream_t>(stream)>>>(iters, batch,
                                                                                    out, sink);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return dev_cuda_error("tmem bench launch", e);
  return 0;
}
