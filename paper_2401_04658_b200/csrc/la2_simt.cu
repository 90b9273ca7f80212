// SIMT (CUDA-core, fp32 arithmetic) kernels:
//   * la2_simt_kernel  -- the "F" block recurrence for fp32 inputs and for shapes
//     outside the tensor-core envelope (any d, dv <= 128). Decay powers come from
//     an iterated-product table exactly like tila.power_table
//     (pkg/src/tila/reference.py:77-100), so the fp32 path tracks the reference's
//     own fp32 arithmetic.
//   * la2_decode_kernel -- tila.inference_step (pkg/src/tila/reference.py:162-181).
//   * la2_scan_kernel   -- prefix/suffix combine of chunk states (sequence parallel).
#include <cuda_bf16.h>

#include <type_traits>

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

// Global -> shared staging with U loads in flight per thread before any store (the
// element-wise loop otherwise waits out one global latency per element): element e of
// [0, total) is ld(e) -> st(e, value).
template <int U, typename LD, typename ST>
__device__ __forceinline__ void stage_batched(int total, int tid, LD ld, ST st) {
  for (int base = 0; base < total; base += U * SIMT_THREADS) {
    float r[U];
#pragma unroll
    for (int w = 0; w < U; ++w) {
      const int e = base + w * SIMT_THREADS + tid;
      r[w] = (e < total) ? ld(e) : 0.f;
    }
#pragma unroll
    for (int w = 0; w < U; ++w) {
      const int e = base + w * SIMT_THREADS + tid;
      if (e < total) st(e, r[w]);
    }
  }
}

// Same recurrence and conventions as la2_tc_kernel (see la2_tc.cu), block size 32.
// One CTA per (b, h, value slice of width <= 64): the state slice is dk x dvs.
// Register-tiled: 256 threads = 16 x 16; the scores are 2 x 2 tiles, the outputs 2 rows x 4
// columns, the state fold 4 rows x 4 columns per thread (operands read once per tile from
// shared memory, rows of V and of the state padded to float4).
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
  const int ldq = dk + 1;                           // odd: conflict-free column walks
  const int ldv = (dv + 3) & ~3;                    // float4 rows
  float* KV = sm;                       // [dk][ldv]
  float* Qs = KV + dk * ldv;            // [SB][dk+1]
  float* Ks = Qs + SB * ldq;            // [SB][dk+1]
  float* Vs = Ks + SB * ldq;            // [SB][ldv]
  float* S = Vs + SB * ldv;             // [SB][SB+1]
  float* pw = S + SB * (SB + 1);        // lam^0 .. lam^SB
  const bool so = (o == nullptr);

  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;  // 16 x 16 thread grid
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
  if (p.kv_in != nullptr) {
    stage_batched<8>(dk * dv, tid, [&](int e) {
      const int c = e / dv, j = e % dv;
      return p.kv_in_T ? p.kv_in[sbase + static_cast<size_t>(c0 + j) * dk + c]
                       : p.kv_in[sbase + static_cast<size_t>(c) * dvt + c0 + j];
    }, [&](int e, float x) { KV[(e / dv) * ldv + e % dv] = x; });
  } else {
    for (int e = tid; e < dk * ldv; e += SIMT_THREADS) KV[e] = 0.f;
  }
  // padding columns of V stay zero (the fold reads whole float4 rows)
  for (int e = tid; e < SB * ldv; e += SIMT_THREADS) Vs[e] = 0.f;
  const size_t qbase = static_cast<size_t>(bh) * N * dk;
  const size_t vbase = static_cast<size_t>(bh) * N * dvt + c0;
  const int nblk = (N + SB - 1) / SB;
  const int j0 = 4 * tx;                 // output / fold columns j0 .. j0+3
  const bool jact = j0 < dv;
  __syncthreads();

  for (int i = 0; i < nblk; ++i) {
    const int blk = REV ? (nblk - 1 - i) : i;
    const int t0 = blk * SB;
    const int r = min(SB, N - t0);
    // the block's rows (zero past the sequence end); q, k rows are contiguous spans
    const size_t rbase = qbase + static_cast<size_t>(t0) * dk;
    if (!so)
      stage_batched<8>(SB * dk, tid, [&](int e) { return e < r * dk ? ld_el<T>(q + rbase + e) : 0.f; },
                       [&](int e, float x) { Qs[(e / dk) * ldq + e % dk] = x; });
    stage_batched<8>(SB * dk, tid, [&](int e) { return e < r * dk ? ld_el<T>(k + rbase + e) : 0.f; },
                     [&](int e, float x) { Ks[(e / dk) * ldq + e % dk] = x; });
    stage_batched<8>(SB * dv, tid, [&](int e) {
      const int t = e / dv, j = e % dv;
      return (t < r) ? ld_el<T>(v + vbase + static_cast<size_t>(t0 + t) * dvt + j) : 0.f;
    }, [&](int e, float x) { Vs[(e / dv) * ldv + e % dv] = x; });
    __syncthreads();
    if (!so) {
      // intra-block scores with the decay mask (lower for forward, upper for reverse):
      // rows 2 ty, 2 ty + 1 x columns 2 tx, 2 tx + 1
      {
        const int ta = 2 * ty, ua = 2 * tx;
        const float* qa = Qs + ta * ldq;
        const float* ka = Ks + ua * ldq;
        float s00 = 0.f, s01 = 0.f, s10 = 0.f, s11 = 0.f;
        const bool live = REV ? (ua + 1 >= ta) : (ua <= ta + 1);  // any unmasked entry
        if (live) {
          for (int c = 0; c < dk; ++c) {
            const float x0 = qa[c], x1 = qa[ldq + c], y0 = ka[c], y1 = ka[ldq + c];
            s00 = fmaf(x0, y0, s00);
            s01 = fmaf(x0, y1, s01);
            s10 = fmaf(x1, y0, s10);
            s11 = fmaf(x1, y1, s11);
          }
        }
        auto msk = [&](int t, int u) {
          if (!REV) return (u <= t) ? pw[t - u] : 0.f;
          return (u >= t) ? pw[u - t] : 0.f;
        };
        S[ta * (SB + 1) + ua] = s00 * msk(ta, ua);
        S[ta * (SB + 1) + ua + 1] = s01 * msk(ta, ua + 1);
        S[(ta + 1) * (SB + 1) + ua] = s10 * msk(ta + 1, ua);
        S[(ta + 1) * (SB + 1) + ua + 1] = s11 * msk(ta + 1, ua + 1);
      }
      __syncthreads();
      // outputs: rows 2 ty, 2 ty + 1 x columns j0 .. j0+3
      if (jact) {
        const int ta = 2 * ty;
        float4 in0 = make_float4(0.f, 0.f, 0.f, 0.f), in1 = in0, it0 = in0, it1 = in0;
        const float* sa = S + ta * (SB + 1);
        for (int u = 0; u < SB; ++u) {
          const float a0 = sa[u], a1 = sa[SB + 1 + u];
          const float4 b = *reinterpret_cast<const float4*>(Vs + u * ldv + j0);
          in0.x = fmaf(a0, b.x, in0.x); in0.y = fmaf(a0, b.y, in0.y);
          in0.z = fmaf(a0, b.z, in0.z); in0.w = fmaf(a0, b.w, in0.w);
          in1.x = fmaf(a1, b.x, in1.x); in1.y = fmaf(a1, b.y, in1.y);
          in1.z = fmaf(a1, b.z, in1.z); in1.w = fmaf(a1, b.w, in1.w);
        }
        const float* qa = Qs + ta * ldq;
        for (int c = 0; c < dk; ++c) {
          const float a0 = qa[c], a1 = qa[ldq + c];
          const float4 b = *reinterpret_cast<const float4*>(KV + c * ldv + j0);
          it0.x = fmaf(a0, b.x, it0.x); it0.y = fmaf(a0, b.y, it0.y);
          it0.z = fmaf(a0, b.z, it0.z); it0.w = fmaf(a0, b.w, it0.w);
          it1.x = fmaf(a1, b.x, it1.x); it1.y = fmaf(a1, b.y, it1.y);
          it1.z = fmaf(a1, b.z, it1.z); it1.w = fmaf(a1, b.w, it1.w);
        }
        const float in_[2][4] = {{in0.x, in0.y, in0.z, in0.w}, {in1.x, in1.y, in1.z, in1.w}};
        const float it_[2][4] = {{it0.x, it0.y, it0.z, it0.w}, {it1.x, it1.y, it1.z, it1.w}};
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int t = ta + rr;
          if (t >= r) continue;
          const float a = REV ? pw[r - 1 - t] : pw[t + 1];
          T* op = o + vbase + static_cast<size_t>(t0 + t) * dvt + j0;
#pragma unroll
          for (int z = 0; z < 4; ++z)
            if (j0 + z < dv) st_el<T>(op + z, in_[rr][z] + a * it_[rr][z]);
        }
      }
      __syncthreads();
    }
    // state fold: KV <- lam^r KV + sum_u w_u k_u^T v_u; thread tile: rows 4 g .. 4 g + 3
    // (g = ty, ty + 16, ...) x columns j0 .. j0 + 3
    if (jact) {
      const float fr = pw[r];
      for (int g = ty; 4 * g < dk; g += 16) {
        const int cr = 4 * g;
        float4 acc[4];
#pragma unroll
        for (int z = 0; z < 4; ++z) acc[z] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int u = 0; u < r; ++u) {
          const float w = REV ? pw[u + 1] : pw[r - 1 - u];
          const float4 b = *reinterpret_cast<const float4*>(Vs + u * ldv + j0);
          const float* ku = Ks + u * ldq + cr;
#pragma unroll
          for (int z = 0; z < 4; ++z) {
            const float a = (cr + z < dk) ? w * ku[z] : 0.f;
            acc[z].x = fmaf(a, b.x, acc[z].x); acc[z].y = fmaf(a, b.y, acc[z].y);
            acc[z].z = fmaf(a, b.z, acc[z].z); acc[z].w = fmaf(a, b.w, acc[z].w);
          }
        }
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          if (cr + z >= dk) break;
          float4* kvp = reinterpret_cast<float4*>(KV + (cr + z) * ldv + j0);
          float4 x = *kvp;
          x.x = fmaf(fr, x.x, acc[z].x); x.y = fmaf(fr, x.y, acc[z].y);
          x.z = fmaf(fr, x.z, acc[z].z); x.w = fmaf(fr, x.w, acc[z].w);
          *kvp = x;
        }
      }
    }
    __syncthreads();
  }
  if (p.kv_out != nullptr)
    for (int e = tid; e < dk * dv; e += SIMT_THREADS)
      p.kv_out[sbase + static_cast<size_t>(e / dv) * dvt + c0 + e % dv] = KV[(e / dv) * ldv + e % dv];
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
  const size_t ldv = (dvs + 3) & ~3;
  const size_t smem = sizeof(float) * (static_cast<size_t>(a.dk) * ldv + 2 * SB * (a.dk + 1) +
                                       SB * ldv + SB * (SB + 1) + SB + 1);
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
// ntok successive decode steps per (b, h): tila.inference_step folded over ntok tokens
// (pkg/src/tila/reference.py:162-181), i.e. tila.recurrent_forward (:142-159) continued
// from the given state. Every token runs the arithmetic of a single step in the same
// order, so one call over ntok tokens equals ntok single-token calls bit for bit.
// Operation order follows _decay_step (reference.py:135-139):
//   new_kv = lam * kv + outer(k, v);  o = q @ new_kv
// q, k: [B*H][ntok][d]; v, o: [B*H][ntok][dv]; state: [B*H][d][dv] fp32, in place.
//
// General shapes: one CTA per (b, h); thread (g, j) owns value column j of rows g, g+RG, ...
template <typename T>
__global__ void __launch_bounds__(256)
    la2_decode_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                      const float* __restrict__ decay, float* __restrict__ state,
                      T* __restrict__ o, int H, int d, int dv, int ntok) {
  extern __shared__ float dsm[];
  float* qs = dsm;
  float* ks = qs + d;
  float* vs = ks + d;
  float* red = vs + dv;  // [256]
  const int bh = blockIdx.x;
  const int h = bh % H;
  const float lam = checked_decay(decay[h]);
  const int RG = blockDim.x / dv;  // dv <= 256 guaranteed by the launcher
  const int g = threadIdx.x / dv, j = threadIdx.x % dv;
  float* S = state + static_cast<size_t>(bh) * d * dv;
  for (int t = 0; t < ntok; ++t) {
    const size_t row = static_cast<size_t>(bh) * ntok + t;
    if (t) __syncthreads();  // the previous token's reduction has read red / vs
    for (int e = threadIdx.x; e < d; e += blockDim.x) {
      qs[e] = ld_el<T>(q + row * d + e);
      ks[e] = ld_el<T>(k + row * d + e);
    }
    for (int e = threadIdx.x; e < dv; e += blockDim.x) vs[e] = ld_el<T>(v + row * dv + e);
    __syncthreads();
    float acc = 0.f;
    if (g < RG) {
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
      st_el<T>(o + row * dv + threadIdx.x, s);
    }
  }
}

// 4 consecutive elements <-> float4 (one 8-byte bf16 / 16-byte fp32 access; conversions
// as ld_el / st_el, so the values are the same bits as element-wise accesses)
template <typename T> struct Quad;
template <> struct Quad<float> {
  __device__ static float4 ld(const float* p) { return *reinterpret_cast<const float4*>(p); }
  __device__ static void st(float* p, float4 x) { *reinterpret_cast<float4*>(p) = x; }
};
template <> struct Quad<__nv_bfloat16> {
  __device__ static float4 ld(const __nv_bfloat16* p) {
    const uint2 r = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&r.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
  __device__ static void st(__nv_bfloat16* p, float4 x) {
    uint2 r;
    *reinterpret_cast<__nv_bfloat162*>(&r.x) = __floats2bfloat162_rn(x.x, x.y);
    *reinterpret_cast<__nv_bfloat162*>(&r.y) = __floats2bfloat162_rn(x.z, x.w);
    *reinterpret_cast<uint2*>(p) = r;
  }
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

#ifndef LA2_DEC1_THREADS
#define LA2_DEC1_THREADS 128  // CTA size cap of the single-token decode (A/B: tools/ab_decode_cta.sh)
#endif
#ifndef LA2_DECT_THREADS
#define LA2_DECT_THREADS 128  // ... and of the multi-token decode
#endif

// Bandwidth-shaped decode. Thread layout: a CTA covers dvc value columns of one head
// (gridDim.y = dv / dvc slices) with (dvc / 4) x R threads; thread (r0, c4) owns the
// float4 of columns [4 c4, 4 c4 + 4) in the PER consecutive rows r0 PER ... r0 PER + PER - 1
// (R = d / PER). It loads them once, runs the call's tokens on them in registers and
// writes them back once: the state crosses HBM once per call, not once per token. o is
// reduced over rows in smem per token (the thread's PER-row fma chain, then the R row
// groups in order). (PER, R) depend only on (d, dv) -- the slice width only changes how
// many CTAs share a head -- so every bit of the result is the same whatever the number
// of tokens per call: T tokens in one call == T one-token calls.
// Tokens go in chunks of TC: the chunk's q, k rows (one contiguous span each) and v
// slices arrive by cp.async into smem, double-buffered (the next chunk's copies are in
// flight during the current chunk's packed-fp32x2 arithmetic); bf16 q, k are widened to
// fp32 once per chunk, so a thread reads its rows' values as float4.
template <typename T, int PER, int TC>
__global__ void __launch_bounds__(TC == 1 ? LA2_DEC1_THREADS : LA2_DECT_THREADS,
                                  512 / (TC == 1 ? LA2_DEC1_THREADS : LA2_DECT_THREADS))
    la2_decode_vec_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                          const float* __restrict__ decay, float* __restrict__ state,
                          T* __restrict__ o, int H, int d, int dv, int dvc, int ntok) {
  constexpr int NB = TC == 1 ? 1 : 2;         // staging buffers
  constexpr int EPC = 16 / sizeof(T);         // elements per 16-byte copy (q, k)
  constexpr int EP8 = 8 / sizeof(T);          // elements per 8-byte copy (v)
  // bf16 rows widened to fp32 in smem once per chunk (several tokens); a single token
  // reads its rows' bf16 values directly (no extra pass and barrier on the HBM-bound step)
  constexpr bool WIDEN = !std::is_same<T, float>::value && TC > 1;
  extern __shared__ __align__(16) unsigned char dsm_dec[];
  const int nt = blockDim.x, t = threadIdx.x, bh = blockIdx.x;
  float4* red = reinterpret_cast<float4*>(dsm_dec);          // [TC][nt]
  float* qw = reinterpret_cast<float*>(red + TC * nt);       // [TC][d] fp32 (bf16 inputs)
  float* kw = qw + (WIDEN ? TC * d : 0);                     // [TC][d]
  T* qr = reinterpret_cast<T*>(kw + (WIDEN ? TC * d : 0));   // [NB][TC][d] as loaded
  T* kr = qr + NB * TC * d;                                  // [NB][TC][d]
  T* vr = kr + NB * TC * d;                                  // [NB][TC][dvc]
  const int cb = blockIdx.y * dvc;  // first value column of this CTA's slice
  const float lam = checked_decay(decay[bh % H]);
  const int C4 = dvc >> 2, R = d / PER, DV4 = dv >> 2;
  const int c4 = t % C4, r0 = t / C4;
  float4* S = reinterpret_cast<float4*>(state + static_cast<size_t>(bh) * d * dv + cb) +
              static_cast<size_t>(r0) * PER * DV4 + c4;  // this thread's first row
  float4 x[PER];
#pragma unroll
  for (int m = 0; m < PER; ++m) x[m] = S[m * DV4];
  const size_t row0 = static_cast<size_t>(bh) * ntok;
  auto issue = [&](int c0, int buf) {  // chunk at token c0 -> staging buffer buf
    const int tc = min(TC, ntok - c0);
    const int n16 = tc * d / EPC;
    const T* qs = q + (row0 + c0) * d;
    const T* ks = k + (row0 + c0) * d;
    T* qd = qr + buf * TC * d;
    T* kd = kr + buf * TC * d;
    for (int j = t; j < n16; j += nt) {
      cp_async16(qd + j * EPC, qs + j * EPC);
      cp_async16(kd + j * EPC, ks + j * EPC);
    }
    const int per_row = dvc / EP8, n8 = tc * per_row;
    T* vd = vr + buf * TC * dvc;
    for (int j = t; j < n8; j += nt) {
      const int u = j / per_row, w = j % per_row;
      cp_async8(vd + u * dvc + w * EP8, v + (row0 + c0 + u) * dv + cb + w * EP8);
    }
    cp_async_commit();
  };
  issue(0, 0);
  // TC == 1 is launched for single tokens only: one trip, the state stored as computed
  for (int c0 = 0, it = 0; TC == 1 ? it < 1 : c0 < ntok; c0 += TC, ++it) {
    const int tc = min(TC, ntok - c0);
    const int buf = (NB == 2) ? (it & 1) : 0;
    if (it) __syncthreads();  // chunk it-1 is done with red, the fp32 rows and its buffer
    if (NB == 2 && c0 + TC < ntok) {
      issue(c0 + TC, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* qb = nullptr;
    const float* kb = nullptr;
    if constexpr (WIDEN) {  // bf16 -> fp32 once per chunk (exact), 8 elements per step
      const T* qs = qr + buf * TC * d;
      const T* ks = kr + buf * TC * d;
      for (int j = t; j < tc * d / 8; j += nt) {
        const uint4 a = *reinterpret_cast<const uint4*>(qs + 8 * j);
        const uint4 b = *reinterpret_cast<const uint4*>(ks + 8 * j);
        const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
        float2* qd = reinterpret_cast<float2*>(qw + 8 * j);
        float2* kd = reinterpret_cast<float2*>(kw + 8 * j);
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          qd[z] = __bfloat1622float2(a2[z]);
          kd[z] = __bfloat1622float2(b2[z]);
        }
      }
      __syncthreads();
      qb = qw;
      kb = kw;
    } else if constexpr (std::is_same<T, float>::value) {
      qb = reinterpret_cast<const float*>(qr + buf * TC * d);
      kb = reinterpret_cast<const float*>(kr + buf * TC * d);
    }
    const T* vb = vr + buf * TC * dvc;
#pragma unroll
    for (int u = 0; u < TC; ++u) {
      if (u < tc) {
        // this thread's PER rows of k and q for token u (float4 loads when PER % 4 == 0)
        float kf[PER], qf[PER];
        if constexpr (!WIDEN && !std::is_same<T, float>::value) {  // single bf16 token
          const T* kq = kr + buf * TC * d + u * d + r0 * PER;
          const T* qq = qr + buf * TC * d + u * d + r0 * PER;
#pragma unroll
          for (int m = 0; m < PER; ++m) {
            kf[m] = static_cast<float>(kq[m]);
            qf[m] = static_cast<float>(qq[m]);
          }
        } else if constexpr (PER % 4 == 0) {
          const float* kq = kb + u * d + r0 * PER;
          const float* qq = qb + u * d + r0 * PER;
#pragma unroll
          for (int j = 0; j < PER / 4; ++j) {
            const float4 a = reinterpret_cast<const float4*>(kq)[j];
            const float4 b = reinterpret_cast<const float4*>(qq)[j];
            kf[4 * j] = a.x; kf[4 * j + 1] = a.y; kf[4 * j + 2] = a.z; kf[4 * j + 3] = a.w;
            qf[4 * j] = b.x; qf[4 * j + 1] = b.y; qf[4 * j + 2] = b.z; qf[4 * j + 3] = b.w;
          }
        } else {
          const float* kq = kb + u * d + r0 * PER;
          const float* qq = qb + u * d + r0 * PER;
#pragma unroll
          for (int m = 0; m < PER; ++m) {
            kf[m] = kq[m];
            qf[m] = qq[m];
          }
        }
        // packed fp32x2 (FFMA2 / FMUL2): each lane is the scalar step's rounding,
        // y = fma(lam, x, k * v), acc = fma(q, y, acc)
        const float4 vv = Quad<T>::ld(vb + u * dvc + 4 * c4);
        float2 a01 = make_float2(0.f, 0.f), a23 = make_float2(0.f, 0.f);
        const float2 l2 = make_float2(lam, lam);
        const float2 v01 = make_float2(vv.x, vv.y), v23 = make_float2(vv.z, vv.w);
#pragma unroll
        for (int m = 0; m < PER; ++m) {
          const float2 k2 = make_float2(kf[m], kf[m]), q2 = make_float2(qf[m], qf[m]);
          const float2 y01 = __ffma2_rn(l2, make_float2(x[m].x, x[m].y), __fmul2_rn(k2, v01));
          const float2 y23 = __ffma2_rn(l2, make_float2(x[m].z, x[m].w), __fmul2_rn(k2, v23));
          x[m] = make_float4(y01.x, y01.y, y23.x, y23.y);
          if (TC == 1) S[m * DV4] = x[m];
          a01 = __ffma2_rn(q2, y01, a01);
          a23 = __ffma2_rn(q2, y23, a23);
        }
        red[u * nt + t] = make_float4(a01.x, a01.y, a23.x, a23.y);
      }
    }
    __syncthreads();
    for (int e = t; e < tc * C4; e += nt) {
      const int u = e / C4, c = e % C4;
      float4 s = red[u * nt + c];
      for (int r = 1; r < R; ++r) {
        const float4 w = red[u * nt + r * C4 + c];
        s.x += w.x; s.y += w.y; s.z += w.z; s.w += w.w;
      }
      Quad<T>::st(o + (row0 + c0 + u) * dv + cb + 4 * c, s);
    }
  }
  if (TC != 1) {
#pragma unroll
    for (int m = 0; m < PER; ++m) S[m * DV4] = x[m];
  }
}

// Row split of the vector decode for (d, dv): PER rows per thread (a power of two <= 16
// dividing d, ~d*dv/1024), or 0 when the shape does not fit it.
static int decode_vec_per(int d, int dv) {
  if (d > 256 || dv % 4) return 0;
  int per = 1;
  while (2 * per <= 16 && 2 * per * 1024 <= d * dv && d % (2 * per) == 0) per *= 2;
  return per;
}

template <typename T>
static bool launch_decode_vec(const void* q, const void* k, const void* v, const float* decay,
                              float* state, void* o, int B, int H, int d, int dv, int ntok, cudaStream_t st) {
  const int per = decode_vec_per(d, dv);
  // 16-byte q / k copies within a row; 8-byte v copies and 4-element o stores aligned
  const uintptr_t al = reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k);
  const uintptr_t al4 = reinterpret_cast<uintptr_t>(v) | reinterpret_cast<uintptr_t>(o);
  if (per == 0 || (d * sizeof(T)) % 16 || al % 16 || al4 % (4 * sizeof(T))) return false;
  // value-column slice: the widest with at most 256 threads (one token) / 128 threads
  // (several: more, smaller CTAs to overlap the per-chunk barriers)
  const int R = d / per, cap = (ntok == 1) ? LA2_DEC1_THREADS : LA2_DECT_THREADS;
  int dvc = dv;
  while ((dvc / 4) * R > cap && dvc % 8 == 0) dvc /= 2;
  if ((dvc / 4) * R > cap) return false;
  const int nt = (dvc / 4) * R;
  const dim3 grid(B * H, dv / dvc);
  const int tc = (ntok == 1) ? 1 : 8, nb = (ntok == 1) ? 1 : 2;
  const size_t widen = (sizeof(T) == 4 || tc == 1) ? 0 : static_cast<size_t>(2) * tc * d * sizeof(float);
  const size_t smem = static_cast<size_t>(tc) * nt * 16 + widen +
                      static_cast<size_t>(nb) * tc * (2 * d + dvc) * sizeof(T);
  const T* tq = static_cast<const T*>(q);
  const T* tk = static_cast<const T*>(k);
  const T* tv = static_cast<const T*>(v);
  T* to = static_cast<T*>(o);
  auto go = [&](auto kern) {
    // > 48 KB of dynamic smem (fp32 with d > 128, several tokens) needs the opt-in
    if (smem > 48 * 1024) {
      const cudaError_t e =
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (e != cudaSuccess) return false;
    }
    kern<<<grid, nt, smem, st>>>(tq, tk, tv, decay, state, to, H, d, dv, dvc, ntok);
    return true;
  };
  switch (per) {
#define LA2_DEC(P) \
  case P: return ntok == 1 ? go(la2_decode_vec_kernel<T, P, 1>) : go(la2_decode_vec_kernel<T, P, 8>);
    LA2_DEC(1) LA2_DEC(2) LA2_DEC(4) LA2_DEC(8) LA2_DEC(16)
#undef LA2_DEC
    default: return false;
  }
}

int launch_decode(const void* q, const void* k, const void* v, const float* decay, float* state,
                  void* o, int B, int H, int d, int dv, int ntok, int dtype, cudaStream_t st) {
  if (dv > 256) return set_error(LA2_ERR_UNSUPPORTED, "decode supports dv <= 256");
  LaunchScope log_scope(st, "la2_decode_kernel", B * H, 1);
  const bool vec = (dtype == LA2_FP32)
                       ? launch_decode_vec<float>(q, k, v, decay, state, o, B, H, d, dv, ntok, st)
                       : launch_decode_vec<__nv_bfloat16>(q, k, v, decay, state, o, B, H, d, dv, ntok, st);
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
        decay, state, static_cast<float*>(o), H, d, dv, ntok);
  else
    la2_decode_kernel<__nv_bfloat16><<<B * H, threads, smem, st>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
        static_cast<const __nv_bfloat16*>(v), decay, state, static_cast<__nv_bfloat16*>(o), H, d,
        dv, ntok);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("la2_decode_kernel launch", e);
  return 0;
}

// --------------------------------------------------------------- state scan
struct ScanLens {
  int len[64];
};

// The chunk factors lam^len_g depend only on (head, g): they are computed once per CTA
// into shared memory (double-precision exp2, as before, so the values are unchanged) for
// the head of the CTA's first element; an element of another head (a CTA straddling two
// heads) computes its own. Loads run 8 chunks ahead of the serial combine.
__global__ void la2_scan_kernel(const float* __restrict__ states, const float* __restrict__ decay,
                                const float* __restrict__ init, float* __restrict__ out, int G,
                                int BH, int H, int per, ScanLens lens, int reverse) {
  __shared__ float fac[64];
  const size_t total = static_cast<size_t>(BH) * per;
  const size_t first = static_cast<size_t>(blockIdx.x) * blockDim.x;
  const int bh0 = static_cast<int>(first / per);
  auto factor = [&](int bh, int g) {
    const double l2 = log2(static_cast<double>(checked_decay(decay[bh % H])));
    float f = static_cast<float>(exp2(l2 * lens.len[g]));
    return (f < 1.17549435e-38f) ? 0.f : f;
  };
  if (threadIdx.x < G) fac[threadIdx.x] = factor(bh0, threadIdx.x);
  __syncthreads();
  const size_t e = first + threadIdx.x;
  if (e >= total) return;
  const int bh = static_cast<int>(e / per);
  const bool own = (bh == bh0);
  float acc = init ? init[e] : 0.f;
  constexpr int U = 8;
  for (int g0 = 0; g0 < G; g0 += U) {
    float x[U];
#pragma unroll
    for (int w = 0; w < U; ++w) {
      const int gi = g0 + w;
      const int g = reverse ? G - 1 - gi : gi;
      x[w] = (gi < G) ? states[static_cast<size_t>(g) * total + e] : 0.f;
    }
#pragma unroll
    for (int w = 0; w < U; ++w) {
      const int gi = g0 + w;
      if (gi >= G) break;
      const int g = reverse ? G - 1 - gi : gi;
      out[static_cast<size_t>(g) * total + e] = acc;
      const float f = own ? fac[g] : factor(bh, g);
      acc = fmaf(f, acc, x[w]);
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
