// SIMT (CUDA-core, fp32 arithmetic) kernels:
//   * la2_simt_kernel  -- the "F" block recurrence for fp32 inputs and for shapes
//     outside the tensor-core envelope (any d, dv <= 128). Decay powers come from
//     an iterated-product table exactly like tila.power_table
//     (pkg/src/tila/reference.py:77-100), so the fp32 path tracks the reference's
//     own fp32 arithmetic.
//   * la2_decode_kernel -- tila.inference_step (pkg/src/tila/reference.py:162-181).
//   * la2_scan_kernel   -- prefix/suffix combine of chunk states (sequence parallel).
#include <cuda_bf16.h>

#include "la2_kernels.h"

namespace la2 {

constexpr int SB = 32;          // tokens per block
constexpr int SIMT_THREADS = 256;

template <typename T>
__device__ __forceinline__ float ld_el(const T* p);
template <>
__device__ __forceinline__ float ld_el<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_el<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ void st_el(T* p, float x);
template <>
__device__ __forceinline__ void st_el<float>(float* p, float x) { *p = x; }
template <>
__device__ __forceinline__ void st_el<__nv_bfloat16>(__nv_bfloat16* p, float x) {
  *p = __float2bfloat16_rn(x);
}

// Same recurrence and conventions as la2_tc_kernel (see la2_tc.cu), block size 32.
// One CTA per (b, h, value slice of width <= 64): the state slice is dk x dvs.
template <typename T, bool REV>
__global__ void __launch_bounds__(SIMT_THREADS)
    la2_simt_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                    T* __restrict__ o, FParams p, int dk, int dvs_max) {
  extern __shared__ float sm[];
  const int dvt = p.dv_total;
  const int c0 = blockIdx.x * dvs_max;              // first value column of this slice
  const int dv = min(dvs_max, dvt - c0);            // slice width
  const int h = blockIdx.y;
  const int bh = blockIdx.z * p.H + h;
  const int N = p.N;
  const int ldq = dk + 1, ldv = dv + 1;
  float* KV = sm;                       // [dk][dv]
  float* Qs = KV + dk * dv;             // [SB][dk+1]
  float* Ks = Qs + SB * ldq;            // [SB][dk+1]
  float* Vs = Ks + SB * ldq;            // [SB][dv+1]
  float* S = Vs + SB * ldv;             // [SB][SB+1]
  float* pw = S + SB * (SB + 1);        // lam^0 .. lam^SB
  const bool so = (o == nullptr);

  const int tid = threadIdx.x;
  if (tid == 0) {
    // iterated products with underflow flush, as tila.power_table
    const float lam = checked_decay(p.decay[h]);
    float acc = 1.f;
    bool flushed = false;
    for (int j = 0; j <= SB; ++j) {
      pw[j] = flushed ? 0.f : acc;
      acc = acc * lam;
      if (acc < 1.17549435e-38f) flushed = true;
    }
  }
  const size_t sbase = static_cast<size_t>(bh) * dk * dvt;
  for (int e = tid; e < dk * dv; e += SIMT_THREADS) {
    float x = 0.f;
    if (p.kv_in != nullptr) {
      const int c = e / dv, j = e % dv;
      x = p.kv_in_T ? p.kv_in[sbase + static_cast<size_t>(c0 + j) * dk + c]
                    : p.kv_in[sbase + static_cast<size_t>(c) * dvt + c0 + j];
    }
    KV[e] = x;
  }
  const size_t qbase = static_cast<size_t>(bh) * N * dk;
  const size_t vbase = static_cast<size_t>(bh) * N * dvt + c0;
  const int nblk = (N + SB - 1) / SB;
  __syncthreads();

  for (int i = 0; i < nblk; ++i) {
    const int blk = REV ? (nblk - 1 - i) : i;
    const int t0 = blk * SB;
    const int r = min(SB, N - t0);
    for (int e = tid; e < SB * dk; e += SIMT_THREADS) {
      const int t = e / dk, c = e % dk;
      const bool ok = t < r;
      if (!so) Qs[t * ldq + c] = ok ? ld_el<T>(q + qbase + static_cast<size_t>(t0 + t) * dk + c) : 0.f;
      Ks[t * ldq + c] = ok ? ld_el<T>(k + qbase + static_cast<size_t>(t0 + t) * dk + c) : 0.f;
    }
    for (int e = tid; e < SB * dv; e += SIMT_THREADS) {
      const int t = e / dv, j = e % dv;
      Vs[t * ldv + j] = (t < r) ? ld_el<T>(v + vbase + static_cast<size_t>(t0 + t) * dvt + j) : 0.f;
    }
    __syncthreads();
    if (!so) {
      // intra-block scores with the decay mask (lower for forward, upper for reverse)
      for (int e = tid; e < SB * SB; e += SIMT_THREADS) {
        const int t = e / SB, u = e % SB;
        float m = 0.f;
        if (!REV && u <= t) m = pw[t - u];
        if (REV && u >= t) m = pw[u - t];
        float acc = 0.f;
        if (m != 0.f)
          for (int c = 0; c < dk; ++c) acc = fmaf(Qs[t * ldq + c], Ks[u * ldq + c], acc);
        S[t * (SB + 1) + u] = acc * m;
      }
      __syncthreads();
      for (int e = tid; e < SB * dv; e += SIMT_THREADS) {
        const int t = e / dv, j = e % dv;
        if (t >= r) continue;
        float intra = 0.f;
        for (int u = 0; u < SB; ++u) intra = fmaf(S[t * (SB + 1) + u], Vs[u * ldv + j], intra);
        float inter = 0.f;
        for (int c = 0; c < dk; ++c) inter = fmaf(Qs[t * ldq + c], KV[c * dv + j], inter);
        const float a = REV ? pw[r - 1 - t] : pw[t + 1];
        st_el<T>(o + vbase + static_cast<size_t>(t0 + t) * dvt + j, intra + a * inter);
      }
      __syncthreads();
    }
    // state fold: KV <- lam^r KV + sum_u w_u k_u^T v_u
    const float fr = pw[r];
    for (int e = tid; e < dk * dv; e += SIMT_THREADS) {
      const int c = e / dv, j = e % dv;
      float acc = 0.f;
      for (int u = 0; u < r; ++u) {
        const float w = REV ? pw[u + 1] : pw[r - 1 - u];
        acc = fmaf(w * Ks[u * ldq + c], Vs[u * ldv + j], acc);
      }
      KV[e] = fmaf(fr, KV[e], acc);
    }
    __syncthreads();
  }
  if (p.kv_out != nullptr)
    for (int e = tid; e < dk * dv; e += SIMT_THREADS)
      p.kv_out[sbase + static_cast<size_t>(e / dv) * dvt + c0 + e % dv] = KV[e];
}

int launch_simt(const FArgs& a, cudaStream_t st) {
  if (a.dk > 256 || a.dv > 256)
    return set_error(LA2_ERR_UNSUPPORTED, "SIMT path supports d <= 256 and dv <= 256");
  // value slices of <= 64 columns keep the dk x dvs fp32 state in shared memory
  const int dvs = a.dv <= 64 ? a.dv : 64;
  const int nslices = (a.dv + dvs - 1) / dvs;
  FParams p;
  p.N = a.N;
  p.H = a.H;
  p.decay = a.decay;
  p.kv_in = a.kv_in;
  p.kv_in_T = a.kv_in_T;
  p.kv_out = a.kv_out;
  p.dv_total = a.dv;
  const size_t smem = sizeof(float) * (static_cast<size_t>(a.dk) * dvs + 2 * SB * (a.dk + 1) +
                                       SB * (dvs + 1) + SB * (SB + 1) + SB + 1);
  dim3 grid(nslices, a.H, a.B);
  cudaError_t e;
#define LA2_SIMT_LAUNCH(TY, RV)                                                                   \
  do {                                                                                            \
    auto kern = la2_simt_kernel<TY, RV>;                                                          \
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,                   \
                             static_cast<int>(smem));                                             \
    if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(simt)", e);                 \
    LaunchScope log_scope(st, "la2_simt_kernel<" #TY "," #RV ">", nslices * a.H * a.B, 1);      \
    kern<<<grid, SIMT_THREADS, smem, st>>>(static_cast<const TY*>(a.q), static_cast<const TY*>(a.k), \
                                           static_cast<const TY*>(a.v), static_cast<TY*>(a.o), p, \
                                           a.dk, dvs);                                            \
  } while (0)
  if (a.dtype == LA2_FP32) {
    if (a.reverse) LA2_SIMT_LAUNCH(float, true);
    else LA2_SIMT_LAUNCH(float, false);
  } else {
    if (a.reverse) LA2_SIMT_LAUNCH(__nv_bfloat16, true);
    else LA2_SIMT_LAUNCH(__nv_bfloat16, false);
  }
#undef LA2_SIMT_LAUNCH
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("la2_simt_kernel launch", e);
  return 0;
}

// ------------------------------------------------------------------- decode
// One CTA per (b, h); thread (g, j) owns value column j of rows g, g+RG, ...
// Operation order follows _decay_step (pkg/src/tila/reference.py:135-139):
//   new_kv = lam * kv + outer(k, v);  o = q @ new_kv
template <typename T>
__global__ void __launch_bounds__(256)
    la2_decode_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                      const float* __restrict__ decay, float* __restrict__ state,
                      T* __restrict__ o, int H, int d, int dv) {
  extern __shared__ float dsm[];
  float* qs = dsm;
  float* ks = qs + d;
  float* vs = ks + d;
  float* red = vs + dv;  // [256]
  const int bh = blockIdx.x;
  const int h = bh % H;
  const float lam = checked_decay(decay[h]);
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    qs[e] = ld_el<T>(q + static_cast<size_t>(bh) * d + e);
    ks[e] = ld_el<T>(k + static_cast<size_t>(bh) * d + e);
  }
  for (int e = threadIdx.x; e < dv; e += blockDim.x) vs[e] = ld_el<T>(v + static_cast<size_t>(bh) * dv + e);
  __syncthreads();
  const int RG = blockDim.x / dv;  // dv <= 256 guaranteed by the launcher
  const int g = threadIdx.x / dv, j = threadIdx.x % dv;
  float acc = 0.f;
  if (g < RG) {
    float* S = state + static_cast<size_t>(bh) * d * dv;
    const float vj = vs[j];
    for (int i = g; i < d; i += RG) {
      const float x = fmaf(lam, S[static_cast<size_t>(i) * dv + j], ks[i] * vj);
      S[static_cast<size_t>(i) * dv + j] = x;
      acc = fmaf(qs[i], x, acc);
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < dv) {
    float s = 0.f;
    for (int gg = 0; gg < RG; ++gg) s += red[gg * dv + threadIdx.x];
    st_el<T>(o + static_cast<size_t>(bh) * dv + threadIdx.x, s);
  }
}

// Bandwidth-shaped decode for d * dv a multiple of 1024 and dv / 4 dividing 256: each of
// the 256 threads owns PER float4 of the fp32 state (fixed 4 value columns, rows strided
// by 256 / (dv / 4)), issues all its state loads before any arithmetic (PER x 16 bytes
// in flight per thread), writes the updated state back and reduces o over rows in smem.
template <typename T, int PER>
__global__ void __launch_bounds__(256)
    la2_decode_vec_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                          const float* __restrict__ decay, float* __restrict__ state,
                          T* __restrict__ o, int H, int d, int dv) {
  __shared__ float qs[256], ks[256];
  __shared__ float4 red[256];
  const int bh = blockIdx.x, t = threadIdx.x;
  const float lam = checked_decay(decay[bh % H]);
  if (t < d) {
    qs[t] = ld_el<T>(q + static_cast<size_t>(bh) * d + t);
    ks[t] = ld_el<T>(k + static_cast<size_t>(bh) * d + t);
  }
  const int C4 = dv >> 2, R = 256 / C4;
  const int c4 = t % C4, r0 = t / C4;
  float4* S = reinterpret_cast<float4*>(state + static_cast<size_t>(bh) * d * dv);
  float4 x[PER];
#pragma unroll
  for (int m = 0; m < PER; ++m) x[m] = S[(r0 + m * R) * C4 + c4];
  float4 vv;
  vv.x = ld_el<T>(v + static_cast<size_t>(bh) * dv + 4 * c4);
  vv.y = ld_el<T>(v + static_cast<size_t>(bh) * dv + 4 * c4 + 1);
  vv.z = ld_el<T>(v + static_cast<size_t>(bh) * dv + 4 * c4 + 2);
  vv.w = ld_el<T>(v + static_cast<size_t>(bh) * dv + 4 * c4 + 3);
  __syncthreads();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    const int i = r0 + m * R;
    const float ki = ks[i], qi = qs[i];
    float4 y;
    y.x = fmaf(lam, x[m].x, ki * vv.x);
    y.y = fmaf(lam, x[m].y, ki * vv.y);
    y.z = fmaf(lam, x[m].z, ki * vv.z);
    y.w = fmaf(lam, x[m].w, ki * vv.w);
    S[i * C4 + c4] = y;
    acc.x = fmaf(qi, y.x, acc.x);
    acc.y = fmaf(qi, y.y, acc.y);
    acc.z = fmaf(qi, y.z, acc.z);
    acc.w = fmaf(qi, y.w, acc.w);
  }
  red[t] = acc;
  __syncthreads();
  if (t < C4) {
    float4 s = red[t];
    for (int r = 1; r < R; ++r) {
      const float4 w = red[r * C4 + t];
      s.x += w.x; s.y += w.y; s.z += w.z; s.w += w.w;
    }
    T* op = o + static_cast<size_t>(bh) * dv + 4 * t;
    st_el<T>(op, s.x);
    st_el<T>(op + 1, s.y);
    st_el<T>(op + 2, s.z);
    st_el<T>(op + 3, s.w);
  }
}

template <typename T>
static bool launch_decode_vec(const void* q, const void* k, const void* v, const float* decay,
                              float* state, void* o, int B, int H, int d, int dv, cudaStream_t st) {
  if (dv % 4 || 256 % (dv / 4) || (d * dv) % 1024 || d > 256) return false;
  const int per = d * dv / 1024;
  const T* tq = static_cast<const T*>(q);
  const T* tk = static_cast<const T*>(k);
  const T* tv = static_cast<const T*>(v);
  T* to = static_cast<T*>(o);
  switch (per) {
#define LA2_DEC(P) \
  case P: la2_decode_vec_kernel<T, P><<<B * H, 256, 0, st>>>(tq, tk, tv, decay, state, to, H, d, dv); return true;
    LA2_DEC(1) LA2_DEC(2) LA2_DEC(4) LA2_DEC(8) LA2_DEC(16) LA2_DEC(32)
#undef LA2_DEC
    default: return false;
  }
}

int launch_decode(const void* q, const void* k, const void* v, const float* decay, float* state,
                  void* o, int B, int H, int d, int dv, int dtype, cudaStream_t st) {
  if (dv > 256) return set_error(LA2_ERR_UNSUPPORTED, "decode supports dv <= 256");
  LaunchScope log_scope(st, "la2_decode_kernel", B * H, 1);
  const bool vec = (dtype == LA2_FP32)
                       ? launch_decode_vec<float>(q, k, v, decay, state, o, B, H, d, dv, st)
                       : launch_decode_vec<__nv_bfloat16>(q, k, v, decay, state, o, B, H, d, dv, st);
  if (vec) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error("la2_decode_vec_kernel launch", e);
    return 0;
  }
  const size_t smem = sizeof(float) * (2 * d + dv + 256);
  const int threads = (256 / dv) * dv;
  if (dtype == LA2_FP32)
    la2_decode_kernel<float><<<B * H, threads, smem, st>>>(
        static_cast<const float*>(q), static_cast<const float*>(k), static_cast<const float*>(v),
        decay, state, static_cast<float*>(o), H, d, dv);
  else
    la2_decode_kernel<__nv_bfloat16><<<B * H, threads, smem, st>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
        static_cast<const __nv_bfloat16*>(v), decay, state, static_cast<__nv_bfloat16*>(o), H, d,
        dv);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("la2_decode_kernel launch", e);
  return 0;
}

// --------------------------------------------------------------- state scan
struct ScanLens {
  int len[64];
};

__global__ void la2_scan_kernel(const float* __restrict__ states, const float* __restrict__ decay,
                                const float* __restrict__ init, float* __restrict__ out, int G,
                                int BH, int H, int per, ScanLens lens, int reverse) {
  const size_t total = static_cast<size_t>(BH) * per;
  const size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int bh = static_cast<int>(e / per);
  const double l2 = log2(static_cast<double>(checked_decay(decay[bh % H])));
  float acc = init ? init[e] : 0.f;
  if (!reverse) {
    for (int g = 0; g < G; ++g) {
      out[static_cast<size_t>(g) * total + e] = acc;
      float f = static_cast<float>(exp2(l2 * lens.len[g]));
      if (f < 1.17549435e-38f) f = 0.f;
      acc = fmaf(f, acc, states[static_cast<size_t>(g) * total + e]);
    }
  } else {
    for (int g = G - 1; g >= 0; --g) {
      out[static_cast<size_t>(g) * total + e] = acc;
      float f = static_cast<float>(exp2(l2 * lens.len[g]));
      if (f < 1.17549435e-38f) f = 0.f;
      acc = fmaf(f, acc, states[static_cast<size_t>(g) * total + e]);
    }
  }
}

int launch_state_scan(const float* states, const float* decay, const float* init, float* out,
                      int G, int BH, int H, int dk, int dv, const int* lens, int reverse,
                      cudaStream_t st) {
  if (G < 1 || G > 64) return set_error(LA2_ERR_VALUE, "state_scan: G must be in [1, 64]");
  ScanLens L;
  for (int g = 0; g < G; ++g) {
    if (lens[g] < 1) return set_error(LA2_ERR_VALUE, "state_scan: chunk lengths must be >= 1");
    L.len[g] = lens[g];
  }
  const int per = dk * dv;
  const size_t total = static_cast<size_t>(BH) * per;
  const int threads = 256;
  const unsigned blocks = static_cast<unsigned>((total + threads - 1) / threads);
  LaunchScope log_scope(st, "la2_scan_kernel", static_cast<int>(blocks), 1);
  la2_scan_kernel<<<blocks, threads, 0, st>>>(states, decay, init, out, G, BH, H, per, L, reverse);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("la2_scan_kernel launch", e);
  return 0;
}

}  // namespace la2
