// Shared device-side pieces of the tcgen05 Lightning-2 kernels (la2_tc.cu):
// tile constants, trace hooks, row copy/store helpers.
#pragma once
#include "la2_kernels.h"
#include "la2_ptx.cuh"

namespace la2 {

// Optional phase trace (build with -DLA2_TRACE): CTA (0,0,0) records clock64()
// stamps per role / block / event into g_trace[role][block][event].
#ifndef LA2_TRW
#define LA2_TRW 2  // the row warp whose phases are traced
#endif
#ifdef LA2_TRACE
static __device__ long long* g_trace = nullptr;  // per translation unit
constexpr int TR_MAXB = 64, TR_EV = 8;  // roles 0..4
// TR_INIT caches the buffer pointer (and the "is CTA 0" test) in registers at kernel
// start: re-reading the __device__ pointer per event put an L2 round trip on every stamp.
#ifndef LA2_TRB
#define LA2_TRB 0  // the CTA whose phases are traced
#endif
#define TR_INIT                                                                                  \
  long long* const tr_buf =                                                                      \
      (blockIdx.x == LA2_TRB && blockIdx.y == 0 && blockIdx.z == 0) ? g_trace : nullptr
#define TR(role, blk, ev)                                                                        \
  do {                                                                                           \
    if (tr_buf && (blk) < TR_MAXB && (threadIdx.x & 31) == 0)                                    \
      tr_buf[((role) * TR_MAXB + (blk)) * TR_EV + (ev)] = clock64();                             \
  } while (0)
#else
#define TR_INIT \
  do {          \
  } while (0)
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
        const float2 x = __fmul2_rn(unpack_bf16x2(u[e]), make_float2(f, f));
        u[e] = pack_bf16x2(x.x, x.y);
      }
      // chunks are rotated by row to spread banks across the warp
      *reinterpret_cast<uint4*>(dp + ((k + row) & 7) * 16) = w[k];
    }
  }
}

// Half of scale_row_copy<64>: logical 16-byte chunks [4h, 4h+4) of one row (columns
// 32h..32h+31), scaled by f, into the same chunks of dst.
__device__ __forceinline__ void scale_row_copy_half(const uint8_t* src, uint8_t* dst, int row, int h,
                                                    float f) {
  const uint8_t* sp = src + row * 128;
  uint8_t* dp = dst + row * 128;
  uint4 w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) w[k] = *reinterpret_cast<const uint4*>(sp + (((4 * h + k) ^ (row & 7)) * 16));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t* u = reinterpret_cast<uint32_t*>(&w[k]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = __fmul2_rn(unpack_bf16x2(u[e]), make_float2(f, f));
      u[e] = pack_bf16x2(x.x, x.y);
    }
    *reinterpret_cast<uint4*>(dp + (((4 * h + k) ^ (row & 7)) * 16)) = w[k];
  }
}
// scale_row_copy_half into a compact [rows][32] SW64 tile (64-byte rows, chunk' = chunk ^
// ((row >> 1) & 3)): the N = 32 B operand of the shared-recurrence fold.
__device__ __forceinline__ void scale_row_copy_half_sw64(const uint8_t* src, uint8_t* dst, int row, int h,
                                                         float f) {
  const uint8_t* sp = src + row * 128;
  uint8_t* dp = dst + row * 64;
  uint4 w[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) w[k] = *reinterpret_cast<const uint4*>(sp + (((4 * h + k) ^ (row & 7)) * 16));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t* u = reinterpret_cast<uint32_t*>(&w[k]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = __fmul2_rn(unpack_bf16x2(u[e]), make_float2(f, f));
      u[e] = pack_bf16x2(x.x, x.y);
    }
    *reinterpret_cast<uint4*>(dp + ((k ^ ((row >> 1) & 3)) * 16)) = w[k];
  }
}
// store_chunk16_bf16 into this CTA's region and the same-offset region of a cluster peer
// (remote = mapa_shared of the region's base).
__device__ __forceinline__ void store_chunk16_bf16_dup(uint8_t* region, uint32_t remote, int row, int q,
                                                       const float* x) {
  const uint32_t off = row * 128;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = 2 * q + h;
    uint4 w;
    w.x = pack_bf16x2(x[8 * h + 0], x[8 * h + 1]);
    w.y = pack_bf16x2(x[8 * h + 2], x[8 * h + 3]);
    w.z = pack_bf16x2(x[8 * h + 4], x[8 * h + 5]);
    w.w = pack_bf16x2(x[8 * h + 6], x[8 * h + 7]);
    const uint32_t o = off + ((c ^ (row & 7)) * 16);
    *reinterpret_cast<uint4*>(region + o) = w;
    st_cluster_v4(remote + o, w);
  }
}
// Write 16 fp32 values as bf16 into logical chunks 2q, 2q+1 of one 64-byte SW64 row
// (chunk' = chunk ^ ((row >> 1) & 3)).
__device__ __forceinline__ void store_chunk16_bf16_sw64(uint8_t* region, int row, int q, const float* x) {
  uint8_t* rp = region + row * 64;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = 2 * q + h;
    uint4 w;
    w.x = pack_bf16x2(x[8 * h + 0], x[8 * h + 1]);
    w.y = pack_bf16x2(x[8 * h + 2], x[8 * h + 3]);
    w.z = pack_bf16x2(x[8 * h + 4], x[8 * h + 5]);
    w.w = pack_bf16x2(x[8 * h + 6], x[8 * h + 7]);
    *reinterpret_cast<uint4*>(rp + ((c ^ ((row >> 1) & 3)) * 16)) = w;
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

// ------------------------------------------------------- persistent schedule
// The flattened work space is units x nblk blocks (a unit = one (b, h, value slice)
// recurrence, or a cluster's pair of them). P persistent CTAs (or clusters) each take
// the contiguous range [c*W/P, (c+1)*W/P). When W/P >= nblk a range holds at most one
// partial unit at each end, processed in this order:
//   prefix  unit ub, blocks [0, ib)        first: from kv_in, publishes its end state
//   full    units ufull0 .. ufull0+nfull-1 from kv_in to kv_out
//   suffix  unit ua, blocks [ia, nblk)     last: starts from the state the previous
//                                          range's prefix published
// so a suffix only ever waits for work its neighbour did first (stream-K for the
// sequential scan; no extra HBM traffic, only a d x 64 fp32 handoff per split unit).
struct Sched {
  int nblk, npre, upre, nfull, ufull0, usuf, isuf, T;
  __device__ __forceinline__ void init(int c, int P, int units, int nblk_) {
    nblk = nblk_;
    const long long W = static_cast<long long>(units) * nblk;
    const long long a = W * c / P, b = W * (c + 1) / P;
    const int ua = static_cast<int>(a / nblk), ia = static_cast<int>(a % nblk);
    const int ub = static_cast<int>(b / nblk), ib = static_cast<int>(b % nblk);
    npre = ib;
    upre = ub;
    usuf = ua;
    isuf = ia;
    ufull0 = ia > 0 ? ua + 1 : ua;
    nfull = ub - ufull0;
    T = static_cast<int>(b - a);
  }
  // g-th block in processing order -> (unit, position i in the unit's scan order)
  __device__ __forceinline__ void map(int g, int& u, int& i) const {
    if (g < npre) {
      u = upre;
      i = g;
      return;
    }
    g -= npre;
    if (g < nfull * nblk) {
      u = ufull0 + g / nblk;
      i = g - (u - ufull0) * nblk;
      return;
    }
    u = usuf;
    i = isuf + (g - nfull * nblk);
  }
};

// Sequential walk over a Sched range without per-block integer division (a division
// chain costs ~100s of cycles and the walk sits on the critical path of the state and
// row warps). Unit -> (b*H+h, value slice) is recomputed only when the unit changes.
//   CM 0: unit = (bh, slice)   CM 1: unit = (bh, slice pair), slice = 2*pair + crank
//   CM 2: unit = bh      CM 3: as CM 1 (each pass's pair walks the same units)
template <int CM>
struct Walk {
  int g, u, pos, bh, slice, h;
  __device__ __forceinline__ void set_unit(int uu, int nsl, int H, int crank) {
    u = uu;
    if (CM == 0) {
      bh = u / nsl;
      slice = u - bh * nsl;
    } else if (CM == 1 || CM == 3) {
      const int np = nsl >> 1;
      bh = u / np;
      slice = 2 * (u - bh * np) + crank;
    } else {
      bh = u;
      slice = 0;
    }
    h = bh % H;
  }
  __device__ __forceinline__ void start(const Sched& s, int g0, int nsl, int H, int crank) {
    g = g0;
    int uu, pp;
    s.map(g0 < s.T ? g0 : s.T - 1, uu, pp);
    pos = pp;
    set_unit(uu, nsl, H, crank);
  }
  __device__ __forceinline__ void next(const Sched& s, int nsl, int H, int crank) {
    ++g;
    ++pos;
    if (g == s.npre) {  // prefix done -> first full unit, or the suffix
      if (s.nfull > 0) {
        pos = 0;
        set_unit(s.ufull0, nsl, H, crank);
      } else {
        pos = s.isuf;
        set_unit(s.usuf, nsl, H, crank);
      }
    } else if (pos == s.nblk && g < s.T) {  // a full unit done -> next full unit or suffix
      if (u + 1 < s.ufull0 + s.nfull) {
        pos = 0;
        set_unit(u + 1, nsl, H, crank);
      } else {
        pos = s.isuf;
        set_unit(s.usuf, nsl, H, crank);
      }
    }
  }
};

// Per-block schedule record: written by the TMA producer (which walks the Sched range)
// before the stage's FULL arrive, read by the row and state warps after their FULL wait,
// so those warps carry no schedule state of their own.
constexpr int REC_SEG_START = 1;  // first block of a segment: load kv_in / handoff
constexpr int REC_SEG_END = 2;    // last block of a segment: store kv_out / handoff
struct __align__(16) BlkRec {
  int bh, slice, pos, blk;
  float l2;  // log2(decay) of the head
  int h, flags, pad;
};

__device__ __forceinline__ void flag_release(int* f, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ int flag_acquire(const int* f) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}
// Wait for a handoff flag, then consume it (each flag has exactly one reader).
// Bounded: a missing producer traps instead of hanging the GPU.
__device__ __forceinline__ void flag_wait_consume(int* f) {
  long long spins = 0;
  while (flag_acquire(f) == 0) {
    __nanosleep(64);
    if (++spins > (1ll << 27)) __trap();
  }
  *reinterpret_cast<volatile int*>(f) = 0;
}

}  // namespace la2
