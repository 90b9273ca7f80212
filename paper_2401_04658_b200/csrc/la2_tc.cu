// Lightning-2 block recurrence on sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// One kernel, "F", covers the whole hot path:
//   forward   O  = F(Q, K, V)          dQ = F(dO, V, K)        (forward scan)
//   backward  dK = F_rev(V, dO, Q)     dV = F_rev(K, Q, dO)    (reverse scan)
// F follows the reference block loop pkg/src/tila/kernel.py:95-119
// (_forward_blocks); F_rev is the reverse sweep of tiled_backward
// (pkg/src/tila/kernel.py:207-231) written as a forward pass over reversed time.
//
// Per 128-token block i (rows t, u in [0,128), r = rows present):
//   S      = Q_i K_i^T                                   (tcgen05, TMEM fp32)
//   P      = bf16(S * M)   M[t][u] = lam^(t-u), u<=t     (fwd; transposed for rev)
//   Q~     = bf16(a_t * Q_i)    a_t = lam^(t+1)  | rev: lam^(r-1-t)    (in place)
//   K~     = bf16(c_t * K_i)    c_t = lam^(r-1-t)| rev: lam^(t+1)      (in place)
//   O_i    = P V_i + Q~ KV_{i-1}                          (one TMEM accumulator)
//   dKV    = K~^T V_i                                     (tcgen05)
//   KV_i   = lam^r KV_{i-1} + dKV                         (fp32, registers)
// The fp32 KV state never leaves the SM; its bf16 copy is the B operand of the
// next block's Q~ KV product.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer + TMEM
// owner, warps 2-5 "row" warps (thread <-> TMEM lane <-> token row).
#include <cudaTypedefs.h>

#include <cstdio>

#include "la2_kernels.h"
#include "la2_ptx.cuh"

namespace la2 {

constexpr int BT = 128;        // tokens per block
constexpr int DVS = 64;        // value columns per CTA (dv slice)
constexpr int TC_THREADS = 192;
constexpr int REGION = BT * 64 * 2;  // one [128][64] bf16 SW128 region = 16 KB

template <int DK, bool SO>
struct TcLayout {
  static constexpr int NS = 2;  // Q/K/V stages
  static constexpr int Q_BYTES = SO ? 0 : BT * DK * 2;
  static constexpr int K_BYTES = BT * DK * 2;
  static constexpr int V_BYTES = BT * DVS * 2;
  static constexpr int P_BYTES = SO ? 0 : BT * BT * 2;
  static constexpr int KV_BYTES = SO ? 0 : DK * DVS * 2;
  static constexpr int O_BYTES = SO ? 0 : BT * DVS * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NS * Q_BYTES;
  static constexpr int OFF_V = OFF_K + NS * K_BYTES;
  static constexpr int OFF_P = OFF_V + NS * V_BYTES;
  static constexpr int OFF_KV = OFF_P + P_BYTES;
  static constexpr int OFF_O = OFF_KV + KV_BYTES;
  static constexpr int OFF_BAR = OFF_O + O_BYTES;
  static constexpr int BAR_BYTES = 256;
  static constexpr int TOTAL = OFF_BAR + BAR_BYTES + 1024;  // + alignment slack
  static constexpr uint32_t STAGE_TX = Q_BYTES + K_BYTES + V_BYTES;
  // S[2] + O[2] + dKV[2]; the state-only pass needs dKV[2] only
  static constexpr uint32_t TMEM_COLS = SO ? 128 : 512;
};

// Barrier slots inside the barrier area.
enum : int {
  B_FULL = 0,      // [2] TMA -> MMA / row warps
  B_EMPTY = 2,     // [2] MMA commit -> TMA
  B_SFULL = 4,     // [2] S ready
  B_SEMPTY = 6,    // [2] S consumed
  B_OFULL = 8,     // [2] O + dKV ready
  B_OEMPTY = 10,   // [2] O + dKV consumed
  B_PREADY = 12,   // P, Q~, K~ written
  B_PFREE = 13,    // P consumed by the P.V product
  B_KVREADY = 14,  // bf16 KV state written
  B_COUNT = 15
};

// Scale one token row (all DK columns) of a K-major SW128 tile in place.
template <int DK>
__device__ __forceinline__ void scale_row_inplace(uint8_t* tile, int row, float f) {
#pragma unroll
  for (int reg = 0; reg < DK / 64; ++reg) {
    uint8_t* rp = tile + reg * REGION + row * 128;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = (k + row) & 7;  // rotate to spread banks across the warp
      uint4 w = *reinterpret_cast<uint4*>(rp + c * 16);
      uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 x = unpack_bf16x2(u[e]);
        u[e] = pack_bf16x2(x.x * f, x.y * f);
      }
      *reinterpret_cast<uint4*>(rp + c * 16) = w;
    }
  }
}

// Write 64 fp32 values as one bf16 SW128 row (128 bytes) of a [rows][64] region.
__device__ __forceinline__ void store_row64_bf16(uint8_t* region, int row, const float* x) {
  uint8_t* rp = region + row * 128;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint4 w;
    w.x = pack_bf16x2(x[8 * c + 0], x[8 * c + 1]);
    w.y = pack_bf16x2(x[8 * c + 2], x[8 * c + 3]);
    w.z = pack_bf16x2(x[8 * c + 4], x[8 * c + 5]);
    w.w = pack_bf16x2(x[8 * c + 6], x[8 * c + 7]);
    *reinterpret_cast<uint4*>(rp + ((c ^ (row & 7)) * 16)) = w;
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

template <int DK, bool REV, bool SO>
__global__ void __launch_bounds__(TC_THREADS, 1)
    la2_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                  const FParams p) {
  using L = TcLayout<DK, SO>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + B_COUNT);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int slice = blockIdx.x;
  const int h = blockIdx.y;
  const int bh = blockIdx.z * p.H + h;
  const int N = p.N;
  const int nblk = (N + BT - 1) / BT;

  if (threadIdx.x == 0) {
    mbar_init(&bars[B_FULL + 0], 1);
    mbar_init(&bars[B_FULL + 1], 1);
    mbar_init(&bars[B_EMPTY + 0], 1);
    mbar_init(&bars[B_EMPTY + 1], 1);
    mbar_init(&bars[B_SFULL + 0], 1);
    mbar_init(&bars[B_SFULL + 1], 1);
    mbar_init(&bars[B_SEMPTY + 0], 4);
    mbar_init(&bars[B_SEMPTY + 1], 4);
    mbar_init(&bars[B_OFULL + 0], 1);
    mbar_init(&bars[B_OFULL + 1], 1);
    mbar_init(&bars[B_OEMPTY + 0], 4);
    mbar_init(&bars[B_OEMPTY + 1], 4);
    mbar_init(&bars[B_PREADY], 4);
    mbar_init(&bars[B_PFREE], 1);
    mbar_init(&bars[B_KVREADY], 4);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    if (!SO) tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    if (!SO) tma_prefetch_desc(&tm_o);
  }
  if (warp == 1) tmem_alloc(tmem_slot, L::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // TMEM column map: S[2] @0,128  O[2] @256,320  dKV[2] @384,448 (state-only: dKV @0,64)
  auto tS = [&](int b) { return tbase + b * 128; };
  auto tO = [&](int b) { return tbase + 256 + b * 64; };
  auto tKV = [&](int b) { return tbase + (SO ? 0 : 384) + b * 64; };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int i = 0; i < nblk; ++i) {
        const int blk = REV ? (nblk - 1 - i) : i;
        const int s = i & 1;
        if (i >= 2) mbar_wait(&bars[B_EMPTY + s], ((i >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&bars[B_FULL + s], L::STAGE_TX);
        const int row = blk * BT;
#pragma unroll
        for (int c = 0; c < DK / 64; ++c) {
          if (!SO)
            tma_load_3d(smem + L::OFF_Q + s * L::Q_BYTES + c * REGION, &tm_q, &bars[B_FULL + s],
                        c * 64, row, bh);
          tma_load_3d(smem + L::OFF_K + s * L::K_BYTES + c * REGION, &tm_k, &bars[B_FULL + s],
                      c * 64, row, bh);
        }
        tma_load_3d(smem + L::OFF_V + s * L::V_BYTES, &tm_v, &bars[B_FULL + s], slice * DVS, row,
                    bh);
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t ID_S = idesc_bf16(128, 128, 0, 0);   // Q (K-major) x K (K-major)
      constexpr uint32_t ID_O = idesc_bf16(128, DVS, 0, 1);   // P/Q~ (K-major) x V/KV (MN-major)
      constexpr uint32_t ID_KV = idesc_bf16(DK, DVS, 1, 1);   // K~^T (MN-major) x V (MN-major)
      const uint32_t sQ = smem_u32(smem + L::OFF_Q), sK = smem_u32(smem + L::OFF_K);
      const uint32_t sV = smem_u32(smem + L::OFF_V), sP = smem_u32(smem + L::OFF_P);
      const uint32_t sKV = smem_u32(smem + L::OFF_KV);

      auto issue_S = [&](int j) {
        const int s = j & 1;
        mbar_wait(&bars[B_FULL + s], (j >> 1) & 1);
        if (j >= 2) mbar_wait(&bars[B_SEMPTY + s], ((j >> 1) - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DK / 16; ++kk) {
          const uint32_t off = (kk >> 2) * REGION + (kk & 3) * 32;
          umma_bf16_ss(tS(s), sdesc_sw128(sQ + s * L::Q_BYTES + off, 16, 1024),
                       sdesc_sw128(sK + s * L::K_BYTES + off, 16, 1024), ID_S, kk > 0);
        }
        umma_commit(&bars[B_SFULL + s]);
      };

      if (!SO) issue_S(0);
      for (int i = 0; i < nblk; ++i) {
        const int s = i & 1;
        if (!SO) {
          if (i + 1 < nblk) issue_S(i + 1);
        } else {
          mbar_wait(&bars[B_FULL + s], (i >> 1) & 1);
        }
        mbar_wait(&bars[B_PREADY], i & 1);
        if (i >= 2) mbar_wait(&bars[B_OEMPTY + s], ((i >> 1) - 1) & 1);
        tc_fence_after();
        if (!SO) {
          // O = P V   (K = 128 tokens)
#pragma unroll
          for (int kk = 0; kk < BT / 16; ++kk) {
            umma_bf16_ss(tO(s),
                         sdesc_sw128(sP + (kk >> 2) * REGION + (kk & 3) * 32, 16, 1024),
                         sdesc_sw128(sV + s * L::V_BYTES + kk * 2048, REGION, 1024), ID_O,
                         kk > 0);
          }
          umma_commit(&bars[B_PFREE]);
        }
        // dKV = K~^T V   (M = DK, K = 128 tokens)
#pragma unroll
        for (int kk = 0; kk < BT / 16; ++kk) {
          umma_bf16_ss(tKV(s), sdesc_sw128(sK + s * L::K_BYTES + kk * 2048, REGION, 1024),
                       sdesc_sw128(sV + s * L::V_BYTES + kk * 2048, REGION, 1024), ID_KV,
                       kk > 0);
        }
        if (!SO) {
          // O += Q~ KV_{i-1}   (K = DK)
          mbar_wait(&bars[B_KVREADY], i & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < DK / 16; ++kk) {
            const uint32_t off = (kk >> 2) * REGION + (kk & 3) * 32;
            umma_bf16_ss(tO(s), sdesc_sw128(sQ + s * L::Q_BYTES + off, 16, 1024),
                         sdesc_sw128(sKV + kk * 2048, DK * 128, 1024), ID_O, 1);
          }
        }
        umma_commit(&bars[B_OFULL + s]);
        umma_commit(&bars[B_EMPTY + s]);
      }
    }
  } else {
    // --------------------------------------------------------------- row warps
    const int q4 = warp & 3;                 // TMEM lane quarter owned by this warp
    const int row = q4 * 32 + lane;          // token row within the block
    const int ct = threadIdx.x - 64;         // 0..127
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const float lam = p.decay[h];
    // exact log2 (fast-math log2f is off by ~2^-22 absolute, which compounds over
    // 64K tokens when lam is close to 1)
    const float l2 = (lam >= 1.f) ? 0.f : static_cast<float>(log2(static_cast<double>(lam)));
    // KV rows: M=128 -> lane == d row; M=64 -> lanes 0-15 of each quarter hold 16 rows.
    const bool has_kv = (DK == 128) || (lane < 16);
    const int kvrow = (DK == 128) ? row : (q4 * 16 + lane);
    const int dvt = p.dv_total;
    const size_t sbase = static_cast<size_t>(bh) * DK * dvt;

    // Mask factors for this row (block-invariant): M[row][16ch + j] =
    //   ch == dch ? Dg[j] : F[ch] * G[j]   (F = 0 for the zero side).
    float G[16], Dg[16], F[8];
    const int dch = row >> 4, tt = row & 15;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (!REV) {
        G[j] = lam_pow(l2, 15 - j);
        Dg[j] = (j <= tt) ? lam_pow(l2, tt - j) : 0.f;
      } else {
        G[j] = lam_pow(l2, j);
        Dg[j] = (j >= tt) ? lam_pow(l2, j - tt) : 0.f;
      }
    }
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) {
      if (!REV) F[ch] = (ch < dch) ? lam_pow(l2, row - 16 * ch - 15) : 0.f;
      else F[ch] = (ch > dch) ? lam_pow(l2, 16 * ch - row) : 0.f;
    }

    float kv[DVS];
#pragma unroll
    for (int j = 0; j < DVS; ++j) kv[j] = 0.f;
    if (p.kv_in != nullptr && has_kv) {
      const int c0 = slice * DVS;
      if (!p.kv_in_T) {
        const float* src = p.kv_in + sbase + static_cast<size_t>(kvrow) * dvt + c0;
#pragma unroll
        for (int j = 0; j < DVS; j += 4) {
          float4 w = *reinterpret_cast<const float4*>(src + j);
          kv[j] = w.x; kv[j + 1] = w.y; kv[j + 2] = w.z; kv[j + 3] = w.w;
        }
      } else {
        // state stored transposed: [dv_total][DK]
#pragma unroll
        for (int j = 0; j < DVS; ++j) kv[j] = p.kv_in[sbase + static_cast<size_t>(c0 + j) * DK + kvrow];
      }
    }
    uint8_t* sKVb = smem + L::OFF_KV;
    uint8_t* sO = smem + L::OFF_O;
    if (!SO) {
      if (has_kv) store_row64_bf16(sKVb, kvrow, kv);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[B_KVREADY]);
    }

    for (int j = 0; j <= nblk; ++j) {
      // ---------------- phase A(j): S -> P, scale Q and K rows in place
      if (j < nblk) {
        const int i = j, s = i & 1;
        const int blk = REV ? (nblk - 1 - i) : i;
        const int r = min(BT, N - blk * BT);
        const float a = REV ? (row < r ? lam_pow(l2, r - 1 - row) : 0.f) : lam_pow(l2, row + 1);
        const float c = REV ? lam_pow(l2, row + 1) : (row < r ? lam_pow(l2, r - 1 - row) : 0.f);
        if (!SO) {
          mbar_wait(&bars[B_SFULL + s], (i >> 1) & 1);
          tc_fence_after();
          scale_row_inplace<DK>(smem + L::OFF_Q + s * L::Q_BYTES, row, a);
          scale_row_inplace<DK>(smem + L::OFF_K + s * L::K_BYTES, row, c);
          if (i >= 1) mbar_wait(&bars[B_PFREE], (i - 1) & 1);
          uint8_t* sP = smem + L::OFF_P;
#pragma unroll
          for (int cp = 0; cp < 4; ++cp) {  // pairs of 16-column chunks
            float v0[16], v1[16];
            tmem_ld16(tS(s) + lane_off + cp * 32, v0);
            tmem_ld16(tS(s) + lane_off + cp * 32 + 16, v1);
            tmem_ld_wait();
            float x[32];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int ch0 = 2 * cp, ch1 = 2 * cp + 1;
              const float m0 = (ch0 == dch) ? Dg[e] : F[ch0] * G[e];
              const float m1 = (ch1 == dch) ? Dg[e] : F[ch1] * G[e];
              x[e] = v0[e] * m0;
              x[16 + e] = v1[e] * m1;
            }
            // columns 32cp .. 32cp+31 -> region cp/2, logical chunks 4*(cp&1) .. +3
            uint8_t* rp = sP + (cp >> 1) * REGION + row * 128;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int lc = 4 * (cp & 1) + q;
              uint4 w;
              w.x = pack_bf16x2(x[8 * q + 0], x[8 * q + 1]);
              w.y = pack_bf16x2(x[8 * q + 2], x[8 * q + 3]);
              w.z = pack_bf16x2(x[8 * q + 4], x[8 * q + 5]);
              w.w = pack_bf16x2(x[8 * q + 6], x[8 * q + 7]);
              *reinterpret_cast<uint4*>(rp + ((lc ^ (row & 7)) * 16)) = w;
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[B_SEMPTY + s]);
        } else {
          mbar_wait(&bars[B_FULL + s], (i >> 1) & 1);
          scale_row_inplace<DK>(smem + L::OFF_K + s * L::K_BYTES, row, c);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_PREADY]);
      }
      // ---------------- phase B(j-1): O epilogue and KV state update
      if (j >= 1) {
        const int i = j - 1, s = i & 1;
        const int blk = REV ? (nblk - 1 - i) : i;
        const int r = min(BT, N - blk * BT);
        mbar_wait(&bars[B_OFULL + s], (i >> 1) & 1);
        tc_fence_after();
        const float fr = lam_pow(l2, static_cast<float>(r));
        if (!SO) {
          // previous O tile must have been read out of the staging buffer
          if (ct == 0) tma_store_wait_read0();
          named_bar_sync(1, 128);
        }
#pragma unroll
        for (int q = 0; q < DVS / 16; ++q) {
          float d16[16], o16[16];
          tmem_ld16(tKV(s) + lane_off + q * 16, d16);
          if (!SO) tmem_ld16(tO(s) + lane_off + q * 16, o16);
          tmem_ld_wait();
          if (has_kv) {
#pragma unroll
            for (int e = 0; e < 16; ++e) kv[16 * q + e] = fmaf(fr, kv[16 * q + e], d16[e]);
          }
          if (!SO) {
            if (has_kv) store_chunk16_bf16(sKVb, kvrow, q, kv + 16 * q);
            store_chunk16_bf16(sO, row, q, o16);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_OEMPTY + s]);
        if (!SO) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[B_KVREADY]);
          // O tile -> TMA store (rows >= r are clipped by the tensor map)
          named_bar_sync(1, 128);
          if (ct == 0) {
            tma_store_3d(&tm_o, sO, slice * DVS, blk * BT, bh);
            tma_store_commit();
          }
        }
      }
    }
    if (!SO && ct == 0) tma_store_wait_all0();
    if (p.kv_out != nullptr && has_kv) {
      float* dst = p.kv_out + sbase + static_cast<size_t>(kvrow) * dvt + slice * DVS;
#pragma unroll
      for (int j = 0; j < DVS; j += 4)
        *reinterpret_cast<float4*>(dst + j) = make_float4(kv[j], kv[j + 1], kv[j + 2], kv[j + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tbase, L::TMEM_COLS);
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encode() {
  if (g_encode) return 0;
  cudaDriverEntryPointQueryResult qres;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres);
  if (e != cudaSuccess || qres != cudaDriverEntryPointSuccess || fn == nullptr) return -1;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return 0;
}

// [BH][N][cols] bf16, box (64 cols, 128 rows, 1 head), 128B swizzle.
static int make_tmap(CUtensorMap* m, const void* ptr, int cols, int N, int BH) {
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(N),
                        static_cast<cuuint64_t>(BH)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 2,
                           static_cast<cuuint64_t>(cols) * 2 * static_cast<cuuint64_t>(N)};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(BT), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -static_cast<int>(r) - 1000;
}

template <int DK, bool REV, bool SO>
static int launch_tc_t(const FArgs& a, cudaStream_t st) {
  using L = TcLayout<DK, SO>;
  auto kern = la2_tc_kernel<DK, REV, SO>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
  if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(tc)", e);
  CUtensorMap mq, mk, mv, mo;
  const int BH = a.B * a.H;
  const void* ptrs[4] = {a.q, a.k, a.v, a.o};
  CUtensorMap* maps[4] = {&mq, &mk, &mv, &mo};
  const int cols[4] = {DK, DK, a.dv, a.dv};
  for (int t = 0; t < 4; ++t) {
    if (SO && (t == 0 || t == 3)) continue;
    const int rc = make_tmap(maps[t], ptrs[t], cols[t], a.N, BH);
    if (rc != 0) {
      char buf[256];
      std::snprintf(buf, sizeof(buf),
                    "cuTensorMapEncodeTiled failed for %c: CUresult %d (ptr=%p cols=%d N=%d BH=%d)",
                    "qkvo"[t], -(rc + 1000), ptrs[t], cols[t], a.N, BH);
      return set_error(LA2_ERR_CUDA, buf);
    }
  }
  if (SO) { mq = mk; mo = mv; }
  FParams p;
  p.N = a.N;
  p.H = a.H;
  p.decay = a.decay;
  p.kv_in = a.kv_in;
  p.kv_in_T = a.kv_in_T;
  p.kv_out = a.kv_out;
  p.dv_total = a.dv;
  dim3 grid(a.dv / DVS, a.H, a.B);
  kern<<<grid, TC_THREADS, L::TOTAL, st>>>(mq, mk, mv, mo, p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("la2_tc_kernel launch", e);
  return 0;
}

int launch_tc(const FArgs& a, cudaStream_t st) {
  if (get_encode() != 0) return set_error(LA2_ERR_CUDA, "cannot resolve cuTensorMapEncodeTiled");
  const bool so = (a.o == nullptr);
  if (a.dk == 64) {
    if (a.reverse) return so ? launch_tc_t<64, true, true>(a, st) : launch_tc_t<64, true, false>(a, st);
    return so ? launch_tc_t<64, false, true>(a, st) : launch_tc_t<64, false, false>(a, st);
  }
  if (a.dk == 128) {
    if (a.reverse) return so ? launch_tc_t<128, true, true>(a, st) : launch_tc_t<128, true, false>(a, st);
    return so ? launch_tc_t<128, false, true>(a, st) : launch_tc_t<128, false, false>(a, st);
  }
  return set_error(LA2_ERR_UNSUPPORTED, "tensor-core path supports head dim 64 or 128");
}

}  // namespace la2
