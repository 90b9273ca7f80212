// Norm(.) of NormAttention, O = Norm(Q (K^T V)) (the reference leaves it
// out, SPEC.md:167 -- this is an extension for TransNormer-style layers): simple RMS
// normalisation of attention-output rows, y = x / sqrt(mean(x^2) + eps), over the dv
// features of one head (group = 1) or over all H heads' features of a token (group = H,
// TransNormerLLM's SRMSNorm over the concatenated heads). rstd = 1 / sqrt(mean + eps) is
// kept per row for the backward  dx = (dy - y * mean(dy * y)) * rstd.
// These are the standalone kernels; for bf16 dv = 64 the per-head forward is fused into
// the tensor-core epilogue instead (la2_tc.cu).
#include <cuda_bf16.h>

#include "la2_kernels.h"

namespace la2 {

namespace {
template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
}  // namespace

// One warp per normalisation row: (b, h, t) for group = 1, (b, t) over all heads for group = H.
// x, y: [B, H, N, dv] (y may alias x); rstd: [B, H, N] or [B, N].
template <typename T>
__global__ void __launch_bounds__(256)
    la2_rmsnorm_fwd_kernel(const T* x, T* y, float* __restrict__ rstd, int B, int H, int N, int dv, int group,
                           float eps) {
  const long long rows = static_cast<long long>(B) * (H / group) * N;
  const long long row = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int t = static_cast<int>(row % N);
  const long long bg = row / N;                   // (b, head group)
  const int hg = static_cast<int>(bg % (H / group)), b = static_cast<int>(bg / (H / group));
  float ss = 0.f;
  for (int hh = 0; hh < group; ++hh) {
    const size_t base = ((static_cast<size_t>(b) * H + hg * group + hh) * N + t) * dv;
    for (int j = lane; j < dv; j += 32) {
      const float v = to_f<T>(x[base + j]);
      ss = fmaf(v, v, ss);
    }
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / static_cast<float>(group * dv) + eps);
  for (int hh = 0; hh < group; ++hh) {
    const size_t base = ((static_cast<size_t>(b) * H + hg * group + hh) * N + t) * dv;
    for (int j = lane; j < dv; j += 32) y[base + j] = from_f<T>(to_f<T>(x[base + j]) * r);
  }
  if (lane == 0) rstd[row] = r;
}

template <typename T>
__global__ void __launch_bounds__(256)
    la2_rmsnorm_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ y, const float* __restrict__ rstd,
                           T* __restrict__ dx, int B, int H, int N, int dv, int group) {
  const long long rows = static_cast<long long>(B) * (H / group) * N;
  const long long row = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int t = static_cast<int>(row % N);
  const long long bg = row / N;
  const int hg = static_cast<int>(bg % (H / group)), b = static_cast<int>(bg / (H / group));
  float dot = 0.f;
  for (int hh = 0; hh < group; ++hh) {
    const size_t base = ((static_cast<size_t>(b) * H + hg * group + hh) * N + t) * dv;
    for (int j = lane; j < dv; j += 32) dot = fmaf(to_f<T>(dy[base + j]), to_f<T>(y[base + j]), dot);
  }
  dot = warp_sum(dot) / static_cast<float>(group * dv);
  const float r = rstd[row];
  for (int hh = 0; hh < group; ++hh) {
    const size_t base = ((static_cast<size_t>(b) * H + hg * group + hh) * N + t) * dv;
    for (int j = lane; j < dv; j += 32)
      dx[base + j] = from_f<T>((to_f<T>(dy[base + j]) - to_f<T>(y[base + j]) * dot) * r);
  }
}

// Vectorised variant for dv % 8 == 0: a team of TPR threads per normalisation row, each
// thread moving 8 elements (16 B of bf16 / 32 B of fp32) per chunk; the row's chunks are
// its `group` segments of dv contiguous elements (stride N * dv between heads).
template <typename T>
struct Vec8 {
  float v[8];
  __device__ __forceinline__ void load(const T* p);
  __device__ __forceinline__ void store(T* p) const;
};
template <>
__device__ __forceinline__ void Vec8<__nv_bfloat16>::load(const __nv_bfloat16* p) {
  const uint4 w = *reinterpret_cast<const uint4*>(p);
  const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&u[i]);
    const float2 f = __bfloat1622float2(h);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
template <>
__device__ __forceinline__ void Vec8<__nv_bfloat16>::store(__nv_bfloat16* p) const {
  uint32_t u[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    u[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(p) = make_uint4(u[0], u[1], u[2], u[3]);
}
template <>
__device__ __forceinline__ void Vec8<float>::load(const float* p) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <>
__device__ __forceinline__ void Vec8<float>::store(float* p) const {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}

template <int TPR>
__device__ __forceinline__ float team_sum(float v) {
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// BWD = false: y = x * rstd (rstd written); BWD = true: dx = (dy - y mean(dy y)) * rstd
template <typename T, int TPR, bool BWD>
__global__ void __launch_bounds__(256)
    la2_rmsnorm_vec_kernel(const T* a, const T* b, T* out, float* rstd, int B, int H, int N, int dv, int group,
                           float eps) {
  constexpr int MAXC = 4;  // chunks per thread held in registers (rows of <= 4 * TPR * 8 elements)
  // grid: x = blocks of 256 / TPR tokens, y = (b, head group) -- no 64-bit divisions
  const int team = threadIdx.x / TPR, tl = threadIdx.x % TPR;
  const int t = blockIdx.x * (256 / TPR) + team;
  const bool live = t < N;
  const int bg = blockIdx.y;
  const int hg = bg % (H / group), bb = bg / (H / group);
  const long long rr = static_cast<long long>(bg) * N + (live ? t : 0);
  const int cps = dv / 8, nch = group * cps;  // chunks per segment / per row
  Vec8<T> va[MAXC], vb[MAXC];
  float acc = 0.f;
#pragma unroll
  for (int m = 0; m < MAXC; ++m) {
    const int c = tl + m * TPR;
    if (live && c < nch) {
      const int h = c / cps, off = (c % cps) * 8;
      const size_t base = ((static_cast<size_t>(bb) * H + hg * group + h) * N + t) * dv + off;
      va[m].load(a + base);
      if (BWD) {
        vb[m].load(b + base);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(va[m].v[e], vb[m].v[e], acc);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = fmaf(va[m].v[e], va[m].v[e], acc);
      }
    }
  }
  acc = team_sum<TPR>(acc) / static_cast<float>(group * dv);
  const float r = BWD ? (live ? rstd[rr] : 0.f) : rsqrtf(acc + eps);
#pragma unroll
  for (int m = 0; m < MAXC; ++m) {
    const int c = tl + m * TPR;
    if (live && c < nch) {
      const int h = c / cps, off = (c % cps) * 8;
      const size_t base = ((static_cast<size_t>(bb) * H + hg * group + h) * N + t) * dv + off;
      Vec8<T> o;
#pragma unroll
      for (int e = 0; e < 8; ++e) o.v[e] = BWD ? (va[m].v[e] - vb[m].v[e] * acc) * r : va[m].v[e] * r;
      o.store(out + base);
    }
  }
  if (!BWD && live && tl == 0) rstd[rr] = r;
}

template <typename T, bool BWD>
static bool launch_rmsnorm_vec(const void* a, const void* b, void* out, float* rstd, int B, int H, int N, int dv,
                               int group, float eps, cudaStream_t st) {
  if (dv % 8) return false;
  const int nch = group * dv / 8;
  int tpr = 1;
  while (tpr < 32 && tpr * 2 < nch) tpr *= 2;  // ~2 chunks (16 elements) per thread
  if (nch > 4 * tpr) return false;             // rows longer than 4 * 32 * 8 elements
  if (static_cast<long long>(B) * (H / group) > 65535) return false;
  const dim3 blocks((N + 256 / tpr - 1) / (256 / tpr), B * (H / group));
  const T* ta = static_cast<const T*>(a);
  const T* tb = static_cast<const T*>(b);
  T* to = static_cast<T*>(out);
  switch (tpr) {
#define LA2_NV(P) \
  case P: la2_rmsnorm_vec_kernel<T, P, BWD><<<blocks, 256, 0, st>>>(ta, tb, to, rstd, B, H, N, dv, group, eps); break;
    LA2_NV(1) LA2_NV(2) LA2_NV(4) LA2_NV(8) LA2_NV(16) LA2_NV(32)
#undef LA2_NV
  }
  return true;
}

int launch_rmsnorm_fwd(const void* x, void* y, float* rstd, int B, int H, int N, int dv, int group, float eps,
                       int dtype, cudaStream_t st) {
  {
    LaunchScope log_scope(st, "la2_rmsnorm_vec_kernel<fwd>", 0, 1);
    const bool vec = (dtype == LA2_FP32)
                         ? launch_rmsnorm_vec<float, false>(x, nullptr, y, rstd, B, H, N, dv, group, eps, st)
                         : launch_rmsnorm_vec<__nv_bfloat16, false>(x, nullptr, y, rstd, B, H, N, dv, group, eps, st);
    if (vec) {
      cudaError_t e = cudaGetLastError();
      return e == cudaSuccess ? 0 : set_cuda_error("la2_rmsnorm_vec_kernel launch", e);
    }
  }
  const long long rows = static_cast<long long>(B) * (H / group) * N;
  const unsigned blocks = static_cast<unsigned>((rows + 7) / 8);
  LaunchScope log_scope(st, "la2_rmsnorm_fwd_kernel", static_cast<int>(blocks), 1);
  if (dtype == LA2_FP32)
    la2_rmsnorm_fwd_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(x), static_cast<float*>(y),
                                                          rstd, B, H, N, dv, group, eps);
  else
    la2_rmsnorm_fwd_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), rstd, B, H, N, dv, group, eps);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error("la2_rmsnorm_fwd_kernel launch", e);
}

int launch_rmsnorm_bwd(const void* dy, const void* y, const float* rstd, void* dx, int B, int H, int N, int dv,
                       int group, int dtype, cudaStream_t st) {
  {
    LaunchScope log_scope(st, "la2_rmsnorm_vec_kernel<bwd>", 0, 1);
    float* rs = const_cast<float*>(rstd);  // read only in the backward
    const bool vec = (dtype == LA2_FP32)
                         ? launch_rmsnorm_vec<float, true>(dy, y, dx, rs, B, H, N, dv, group, 0.f, st)
                         : launch_rmsnorm_vec<__nv_bfloat16, true>(dy, y, dx, rs, B, H, N, dv, group, 0.f, st);
    if (vec) {
      cudaError_t e = cudaGetLastError();
      return e == cudaSuccess ? 0 : set_cuda_error("la2_rmsnorm_vec_kernel launch", e);
    }
  }
  const long long rows = static_cast<long long>(B) * (H / group) * N;
  const unsigned blocks = static_cast<unsigned>((rows + 7) / 8);
  LaunchScope log_scope(st, "la2_rmsnorm_bwd_kernel", static_cast<int>(blocks), 1);
  if (dtype == LA2_FP32)
    la2_rmsnorm_bwd_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(dy),
                                                          static_cast<const float*>(y), rstd,
                                                          static_cast<float*>(dx), B, H, N, dv, group);
  else
    la2_rmsnorm_bwd_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(y), rstd,
        static_cast<__nv_bfloat16*>(dx), B, H, N, dv, group);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error("la2_rmsnorm_bwd_kernel launch", e);
}

}  // namespace la2
