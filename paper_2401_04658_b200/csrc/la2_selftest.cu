// Self-test of the tcgen05 operand layouts used by la2_tc_kernel.
// D[M][N] = A[M][K] * B[K][N] with A staged K-major or MN-major and B staged
// K-major or MN-major in SW128 regions, exactly as the F kernel stages Q/K/V/P/KV.
// Used by tests/test_gpu_selftest.py; not on the product path.
#include "la2_kernels.h"
#include "la2_ptx.cuh"

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
  if (tid == 0) {
    const uint32_t id = idesc_bf16(M, N, a_mn, b_mn);
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    for (int kk = 0; kk < K / 16; ++kk) {
      uint64_t ad, bd;
      if (!a_mn) ad = sdesc_sw128(a0 + (kk >> 2) * M * 128 + (kk & 3) * 32, 16, 1024);
      else ad = sdesc_sw128(a0 + kk * 2048, K * 128, 1024);
      if (!b_mn) bd = sdesc_sw128(b0 + (kk >> 2) * N * 128 + (kk & 3) * 32, 16, 1024);
      else bd = sdesc_sw128(b0 + kk * 2048, K * 128, 1024);
      umma_bf16_ss(tbase, ad, bd, id, kk > 0);
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
    return set_error(LA2_ERR_VALUE, "selftest: M,N in {64,128}, K in {64,128}");
  const int smem = 65536 + 128 + 1024;
  cudaError_t e = cudaFuncSetAttribute(la2_umma_selftest_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_cuda_error("selftest attr", e);
  la2_umma_selftest_kernel<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(A, B, D, M, N, K,
                                                                                a_mn, b_mn);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("selftest launch", e);
  return 0;
}
