// Double-precision (fp64 storage and arithmetic) kernels -- the reference's default
// precision ("double", pkg/src/tila/matrix.py; every tila routine computes in the input
// dtype, np.result_type). They let the tila adapter (paper_2401_04658_b200/tila_api.py)
// run the reference's own fp64 gates (1e-10 .. 1e-12) on the GPU instead of narrowing
// fp64 inputs to fp32. CUDA cores (DFMA); a correctness path, not a throughput path.
//
//   la2_f64_kernel<REV>   the "F" block recurrence (same conventions as la2_simt_kernel /
//                         la2_tc_kernel; F_rev for the backward's reverse sweeps), with the
//                         decay powers from an iterated-product table flushed to zero below
//                         the smallest normal double -- tila.power_table
//                         (pkg/src/tila/reference.py:75-100) entry for entry.
//   la2_decode_f64_kernel tila.inference_step / _decay_step (reference.py:135-139, 162-181).
#include <cfloat>

#include "la2_kernels.h"

namespace la2 {

constexpr int FB = 16;            // tokens per block (maximum; the caller's block when it fits)
constexpr int FDV = 32;           // value columns per CTA
constexpr int F64_THREADS = 256;

// lam in (0, 1] (reference.py:42-44); anything else (or NaN) becomes NaN, as in the
// single-precision kernels
__device__ __forceinline__ double checked_decay64(double lam) {
  return (lam > 0.0 && lam <= 1.0) ? lam : __longlong_as_double(0x7ff8000000000000ll);
}

// One CTA per (b, h, value slice of <= FDV columns); the dk x dvs state lives in smem.
// kv_in: [B,H,dk,dv] (kv_in_T: stored [B,H,dv,dk]); kv_out: [B,H,dk,dv].
// 256 threads as 16 x 16, register-tiled: a score per thread, 1 x 2 outputs, 4 x 2 state
// entries (per group of 64 state rows) -- every output keeps the sequential fma order of
// the element-wise formulation, so the results are unchanged bit for bit.
template <bool REV>
__global__ void __launch_bounds__(F64_THREADS)
    la2_f64_kernel(const double* __restrict__ q, const double* __restrict__ k, const double* __restrict__ v,
                   double* __restrict__ o, const double* __restrict__ decay, const double* __restrict__ kv_in,
                   int kv_in_T, double* __restrict__ kv_out, int N, int H, int dk, int dvt, int fb) {
  extern __shared__ double smd[];
  const int c0 = blockIdx.x * FDV;
  const int dv = min(FDV, dvt - c0);
  const int h = blockIdx.y;
  const int bh = blockIdx.z * H + h;
  const int ldq = dk + 1;
  constexpr int LDV = FDV;             // V and state rows padded to the slice width
  double* KV = smd;                    // [dk][LDV]
  double* Qs = KV + dk * LDV;          // [FB][dk+1]
  double* Ks = Qs + FB * ldq;          // [FB][dk+1]
  double* Vs = Ks + FB * ldq;          // [FB][LDV]
  double* S = Vs + FB * LDV;           // [FB][FB+1]
  double* pw = S + FB * (FB + 1);      // lam^0 .. lam^FB
  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;
  if (tid == 0) {
    const double lam = checked_decay64(decay[h]);
    double acc = 1.0;
    bool flushed = false;
    for (int j = 0; j <= fb; ++j) {  // power_table: out[j] = acc; acc *= lam; flush < tiny
      pw[j] = flushed ? 0.0 : acc;
      acc = acc * lam;
      if (acc < DBL_MIN) flushed = true;
    }
  }
  const size_t sbase = static_cast<size_t>(bh) * dk * dvt;
  for (int e = tid; e < dk * LDV; e += F64_THREADS) {
    const int c = e / LDV, j = e % LDV;
    double x = 0.0;
    if (kv_in != nullptr && j < dv)
      x = kv_in_T ? kv_in[sbase + static_cast<size_t>(c0 + j) * dk + c]
                  : kv_in[sbase + static_cast<size_t>(c) * dvt + c0 + j];
    KV[e] = x;
  }
  for (int e = tid; e < FB * LDV; e += F64_THREADS) Vs[e] = 0.0;
  const size_t qbase = static_cast<size_t>(bh) * N * dk;
  const size_t vbase = static_cast<size_t>(bh) * N * dvt + c0;
  const int nblk = (N + fb - 1) / fb;
  const int j0 = 2 * tx;  // output / state columns j0, j0 + 1
  __syncthreads();
  for (int i = 0; i < nblk; ++i) {
    const int blk = REV ? (nblk - 1 - i) : i;
    const int t0 = blk * fb;
    const int r = min(fb, N - t0);
    for (int e = tid; e < fb * dk; e += F64_THREADS) {
      const int t = e / dk, c = e % dk;
      const bool ok = t < r;
      Qs[t * ldq + c] = ok ? q[qbase + static_cast<size_t>(t0 + t) * dk + c] : 0.0;
      Ks[t * ldq + c] = ok ? k[qbase + static_cast<size_t>(t0 + t) * dk + c] : 0.0;
    }
    for (int e = tid; e < fb * dv; e += F64_THREADS) {
      const int t = e / dv, j = e % dv;
      Vs[t * LDV + j] = (t < r) ? v[vbase + static_cast<size_t>(t0 + t) * dvt + j] : 0.0;
    }
    __syncthreads();
    // intra-block scores with the decay mask (lower for the forward scan, upper reversed)
    if (ty < fb && tx < fb) {
      const int t = ty, u = tx;
      double m = 0.0;
      if (!REV && u <= t) m = pw[t - u];
      if (REV && u >= t) m = pw[u - t];
      double acc = 0.0;
      if (m != 0.0)
        for (int c = 0; c < dk; ++c) acc = fma(Qs[t * ldq + c], Ks[u * ldq + c], acc);
      S[t * (FB + 1) + u] = acc * m;
    }
    __syncthreads();
    if (ty < r && j0 < dv) {
      const int t = ty;
      double in0 = 0.0, in1 = 0.0, it0 = 0.0, it1 = 0.0;
      for (int u = 0; u < fb; ++u) {
        const double a = S[t * (FB + 1) + u];
        const double2 b = *reinterpret_cast<const double2*>(Vs + u * LDV + j0);
        in0 = fma(a, b.x, in0);
        in1 = fma(a, b.y, in1);
      }
      for (int c = 0; c < dk; ++c) {
        const double a = Qs[t * ldq + c];
        const double2 b = *reinterpret_cast<const double2*>(KV + c * LDV + j0);
        it0 = fma(a, b.x, it0);
        it1 = fma(a, b.y, it1);
      }
      const double a = REV ? pw[r - 1 - t] : pw[t + 1];
      double* op = o + vbase + static_cast<size_t>(t0 + t) * dvt + j0;
      op[0] = in0 + a * it0;
      if (j0 + 1 < dv) op[1] = in1 + a * it1;
    }
    __syncthreads();
    // state fold: KV <- lam^r KV + sum_u w_u k_u^T v_u (rows 4 g .. 4 g + 3, g = ty, ty+16, ...)
    if (j0 < dv) {
      const double fr = pw[r];
      for (int g = ty; 4 * g < dk; g += 16) {
        const int cr = 4 * g;
        double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
        for (int u = 0; u < r; ++u) {
          const double w = REV ? pw[u + 1] : pw[r - 1 - u];
          const double2 b = *reinterpret_cast<const double2*>(Vs + u * LDV + j0);
#pragma unroll
          for (int z = 0; z < 4; ++z) {
            if (cr + z < dk) {
              const double a = w * Ks[u * ldq + cr + z];
              acc[z][0] = fma(a, b.x, acc[z][0]);
              acc[z][1] = fma(a, b.y, acc[z][1]);
            }
          }
        }
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          if (cr + z < dk) {
            double* kv = KV + (cr + z) * LDV + j0;
            kv[0] = fma(fr, kv[0], acc[z][0]);
            kv[1] = fma(fr, kv[1], acc[z][1]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (kv_out != nullptr)
    for (int e = tid; e < dk * dv; e += F64_THREADS)
      kv_out[sbase + static_cast<size_t>(e / dv) * dvt + c0 + e % dv] = KV[(e / dv) * LDV + e % dv];
}

int launch_f64(const double* q, const double* k, const double* v, double* o, const double* decay,
               const double* kv_in, int kv_in_T, double* kv_out, int B, int H, int N, int dk, int dv,
               int reverse, int block, cudaStream_t st) {
  if (dk > 256 || dv > 256) return set_error(LA2_ERR_UNSUPPORTED, "fp64 path supports d <= 256 and dv <= 256");
  // tile = the caller's block when it fits, else its largest divisor <= FB: chunk boundaries
  // aligned to the caller's block stay tile-aligned, so the reference's "aligned chunks are
  // bitwise equal to one call" property (pkg/tests/test_kernel.py:190-199) holds here too
  // (a block covering the whole sequence stays one tile when the sequence fits in one)
  int fb = FB;
  if (block > 0 && !(block >= N && N <= FB)) {
    fb = 1;
    for (int c = (block < FB ? block : FB); c >= 1; --c)
      if (block % c == 0) { fb = c; break; }
  }
  const int dvs = dv < FDV ? dv : FDV;
  const int nslices = (dv + FDV - 1) / FDV;
  (void)dvs;
  const size_t smem = sizeof(double) * (static_cast<size_t>(dk) * FDV + 2 * FB * (dk + 1) +
                                        FB * FDV + FB * (FB + 1) + FB + 1);
  const dim3 grid(nslices, H, B);
  auto kern = reverse ? la2_f64_kernel<true> : la2_f64_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(f64)", e);
  LaunchScope log_scope(st, reverse ? "la2_f64_kernel<1>" : "la2_f64_kernel<0>", nslices * H * B, 1);
  kern<<<grid, F64_THREADS, smem, st>>>(q, k, v, o, decay, kv_in, kv_in_T, kv_out, N, H, dk, dv, fb);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("la2_f64_kernel launch", e);
  return 0;
}

// One CTA per (b, h); thread (g, j) owns value column j of rows g, g+RG, ... ntok tokens
// per call (q, k: [B*H][ntok][d]; v, o: [B*H][ntok][dv]), each one single step's arithmetic:
//   new_kv = lam * kv + outer(k, v);  o = q @ new_kv        (_decay_step, reference.py:135-139)
// so a call over ntok tokens equals ntok one-token calls bit for bit (tila.recurrent_forward
// continued from the state, reference.py:142-159).
__global__ void __launch_bounds__(256)
    la2_decode_f64_kernel(const double* __restrict__ q, const double* __restrict__ k,
                          const double* __restrict__ v, const double* __restrict__ decay,
                          double* __restrict__ state, double* __restrict__ o, int H, int d, int dv,
                          int ntok) {
  extern __shared__ double dsm64[];
  double* qs = dsm64;
  double* ks = qs + d;
  double* vs = ks + d;
  double* red = vs + dv;  // [256]
  const int bh = blockIdx.x;
  const double lam = checked_decay64(decay[bh % H]);
  const int RG = blockDim.x / dv;
  const int g = threadIdx.x / dv, j = threadIdx.x % dv;
  double* Sst = state + static_cast<size_t>(bh) * d * dv;
  for (int t = 0; t < ntok; ++t) {
    const size_t row = static_cast<size_t>(bh) * ntok + t;
    if (t) __syncthreads();  // the previous token's reduction has read red / vs
    for (int e = threadIdx.x; e < d; e += blockDim.x) {
      qs[e] = q[row * d + e];
      ks[e] = k[row * d + e];
    }
    for (int e = threadIdx.x; e < dv; e += blockDim.x) vs[e] = v[row * dv + e];
    __syncthreads();
    double acc = 0.0;
    if (g < RG) {
      const double vj = vs[j];
      for (int i = g; i < d; i += RG) {
        // lam * kv, then += outer(k, v): two roundings, as _decay_step does them
        const double x = __dadd_rn(__dmul_rn(lam, Sst[static_cast<size_t>(i) * dv + j]), __dmul_rn(ks[i], vj));
        Sst[static_cast<size_t>(i) * dv + j] = x;
        acc = fma(qs[i], x, acc);
      }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < dv) {
      double s = 0.0;
      for (int gg = 0; gg < RG; ++gg) s += red[gg * dv + threadIdx.x];
      o[row * dv + threadIdx.x] = s;
    }
  }
}

int launch_decode_f64(const double* q, const double* k, const double* v, const double* decay,
                      double* state, double* o, int B, int H, int d, int dv, int ntok, cudaStream_t st) {
  if (dv > 256 || d > 256) return set_error(LA2_ERR_UNSUPPORTED, "fp64 decode supports d, dv <= 256");
  const size_t smem = sizeof(double) * (2 * d + dv + 256);
  const int threads = (256 / dv) * dv;
  LaunchScope log_scope(st, "la2_decode_f64_kernel", B * H, 1);
  la2_decode_f64_kernel<<<B * H, threads, smem, st>>>(q, k, v, decay, state, o, H, d, dv, ntok);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("la2_decode_f64_kernel launch", e);
  return 0;
}

}  // namespace la2
