// Shared device-side pieces of the tcgen05 Lightning-2 kernels (F: la2_tc.cu,
// G: la2_bwd.cu): tile constants, trace hooks, row copy/store helpers.
#pragma once
#include "la2_kernels.h"
#include "la2_ptx.cuh"

namespace la2 {

// Optional phase trace (build with -DLA2_TRACE): CTA (0,0,0) records clock64()
// stamps per role / block / event into g_trace[role][block][event].
#ifdef LA2_TRACE
static __device__ long long* g_trace = nullptr;  // per translation unit
constexpr int TR_MAXB = 64, TR_EV = 8;  // roles 0..4
#define TR(role, blk, ev)                                                                        \
  do {                                                                                           \
    if (g_trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (blk) < TR_MAXB &&  \
        (threadIdx.x & 31) == 0)                                                                 \
      g_trace[((role) * TR_MAXB + (blk)) * TR_EV + (ev)] = clock64();                            \
  } while (0)
#else
#define TR(role, blk, ev) \
  do {                    \
  } while (0)
#endif

constexpr int BT = 128;        // tokens per block
constexpr int DVS = 64;        // value columns per CTA (dv slice)
constexpr int REGION = BT * 64 * 2;  // one [128][64] bf16 SW128 region = 16 KB

// Copy one token row of a K-major SW128 tile, scaled by f, into the same row of dst.
template <int DK>
__device__ __forceinline__ void scale_row_copy(const uint8_t* src, uint8_t* dst, int row, float f) {
#pragma unroll
  for (int reg = 0; reg < DK / 64; ++reg) {
    const uint8_t* sp = src + reg * REGION + row * 128;
    uint8_t* dp = dst + reg * REGION + row * 128;
    uint4 w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = *reinterpret_cast<const uint4*>(sp + ((k + row) & 7) * 16);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t* u = reinterpret_cast<uint32_t*>(&w[k]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 x = unpack_bf16x2(u[e]);
        u[e] = pack_bf16x2(x.x * f, x.y * f);
      }
      // chunks are rotated by row to spread banks across the warp
      *reinterpret_cast<uint4*>(dp + ((k + row) & 7) * 16) = w[k];
    }
  }
}

// Write 16 fp32 values as bf16 into logical chunks 2q, 2q+1 of one SW128 row.
__device__ __forceinline__ void store_chunk16_bf16(uint8_t* region, int row, int q, const float* x) {
  uint8_t* rp = region + row * 128;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = 2 * q + h;
    uint4 w;
    w.x = pack_bf16x2(x[8 * h + 0], x[8 * h + 1]);
    w.y = pack_bf16x2(x[8 * h + 2], x[8 * h + 3]);
    w.z = pack_bf16x2(x[8 * h + 4], x[8 * h + 5]);
    w.w = pack_bf16x2(x[8 * h + 6], x[8 * h + 7]);
    *reinterpret_cast<uint4*>(rp + ((c ^ (row & 7)) * 16)) = w;
  }
}

template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

}  // namespace la2
