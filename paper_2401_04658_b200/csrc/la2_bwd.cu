// Fused reverse scan of the Lightning-2 backward pass ("G"): dK and dV in one pass
// over reversed time, sharing the mirrored state dKV. This is the reverse sweep of
// tila.tiled_backward (pkg/src/tila/kernel.py:207-231) for d = dv = 64, bf16.
//
// Per 128-token block i (processed last to first; r rows present; t, u local rows):
//   Sa   = K_i Q_i^T        Pa = bf16(Sa * Mrev)   Mrev[t][u] = lam^(u-t), u >= t
//   Sc   = V_i dO_i^T       Pc = bf16(Sc * Mrev)
//   dV_i = Pa dO_i  + (a . K_i) dKV          a_t = lam^(r-1-t)
//   dK_i = Pc Q_i   + (a . V_i) dKV^T
//   dKV  <- lam^r dKV + Q_i^T (c . dO_i)     c_t = lam^(t+1)   (after the block is emitted)
// dKV holds the contributions of blocks strictly after i (kernel.py:254 ordering).
// P is written back into TMEM over its scores (TS-MMA operand). The inter terms use
// row-scaled operand copies (a . K, a . V, c . dO), so each output needs one
// accumulator and dKV is double-buffered in TMEM.
//
// Warps (480 threads): 0 TMA producer | 1 MMA issuer X (scores) | 2-5 row warps
// path a (Pa, a.K, dV epilogue) | 6-9 row warps path c (Pc, a.V, dK epilogue) |
// 10-13 state warps (c.dO, dKV fp32 state) | 14 MMA issuer Y (fold, dV, dK).
#include <cudaTypedefs.h>

#include <cstdio>

#include "la2_tc_common.cuh"

namespace la2 {

namespace g {

constexpr int THREADS = 480;
constexpr int W0 = 10;  // first state warp
constexpr int WY = 14;  // issuer Y
constexpr int NS = 2;
constexpr int T = REGION;            // one [128][64] bf16 tile (16 KB)
constexpr int STAGE = 4 * T;         // K | Q | dO | V
constexpr int S_K = 0, S_Q = T, S_DO = 2 * T, S_V = 3 * T;
constexpr int OFF_DOT = NS * STAGE;  // c.dO (fold operand)
constexpr int OFF_KT = OFF_DOT + T;  // a.K [2]
constexpr int OFF_VT = OFF_KT + 2 * T;  // a.V [2]
constexpr int OFF_KV = OFF_VT + 2 * T;  // dKV bf16 [64][64]
constexpr int KV_BYTES = 64 * 64 * 2;
constexpr int OFF_MASK = OFF_KV + KV_BYTES;  // Dg[128][16] + G[16] fp32 (mask tables)
constexpr int OFF_BAR = OFF_MASK + 128 * 16 * 4 + 16 * 4;
constexpr int TOTAL = OFF_BAR + 256 + 1024;
static_assert(TOTAL <= 232448, "shared memory budget");
// TMEM columns: Sa (Pa) | Sc (Pc) | dV | dK | dKV[2]
constexpr uint32_t T_SA = 0, T_SC = 128, T_DV = 256, T_DK = 320, T_KV = 384;
// barriers
constexpr int B_FULL = 0, B_EMPTY = 2, B_SFULLA = 4, B_SFULLC = 5, B_SFREE = 6, B_PREADY = 7,
              B_OFULL = 9, B_OEMPTY = 10, B_DTREADY = 11, B_DTFREE = 12, B_DKVFULL = 13,
              B_DKVEMPTY = 15, B_KVREADY = 17, B_COUNT = 18;

}  // namespace g

__global__ void __launch_bounds__(g::THREADS, 1)
    la2_bwd_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_q,
                   const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_v,
                   __nv_bfloat16* __restrict__ gdk, __nv_bfloat16* __restrict__ gdv, const FParams p) {
  using namespace g;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + B_COUNT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TR_INIT;
  const int h = blockIdx.y;
  const int bh = blockIdx.z * p.H + h;
  const int N = p.N;
  const int nblk = (N + BT - 1) / BT;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars[B_FULL + s], 1);
      mbar_init(&bars[B_EMPTY + s], 2);  // X after the scores, Y after dV/dK
    }
    mbar_init(&bars[B_SFULLA], 1);
    mbar_init(&bars[B_SFULLC], 1);
    mbar_init(&bars[B_SFREE], 1);
    for (int b = 0; b < 2; ++b) mbar_init(&bars[B_PREADY + b], 8);
    mbar_init(&bars[B_OFULL], 1);
    mbar_init(&bars[B_OEMPTY], 8);
    mbar_init(&bars[B_DTREADY], 4);
    mbar_init(&bars[B_DTFREE], 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[B_DKVFULL + b], 1);
      mbar_init(&bars[B_DKVEMPTY + b], 4);
    }
    mbar_init(&bars[B_KVREADY], 4);
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const float lam = p.decay[h];
  const float l2 = (lam >= 1.f) ? 0.f : static_cast<float>(log2(static_cast<double>(lam)));

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      constexpr int PF = 3;  // L2 prefetch beyond the 2-stage ring
      auto prefetch = [&](int i) {
        const int row = (nblk - 1 - i) * BT;
        tma_prefetch_l2_3d(&tm_k, 0, row, bh);
        tma_prefetch_l2_3d(&tm_q, 0, row, bh);
        tma_prefetch_l2_3d(&tm_do, 0, row, bh);
        tma_prefetch_l2_3d(&tm_v, 0, row, bh);
      };
      for (int i = NS; i < NS + PF && i < nblk; ++i) prefetch(i);
      for (int i = 0; i < nblk; ++i) {
        if (i + NS + PF < nblk) prefetch(i + NS + PF);
        const int s = i % NS;
        TR(0, i, 0);
        if (i >= NS) mbar_wait(&bars[B_EMPTY + s], ((i / NS) - 1) & 1);
        TR(0, i, 1);
        mbar_arrive_expect_tx(&bars[B_FULL + s], STAGE);
        const int row = (nblk - 1 - i) * BT;
        uint8_t* st = smem + s * STAGE;
        tma_load_3d(st + S_K, &tm_k, &bars[B_FULL + s], 0, row, bh);
        tma_load_3d(st + S_Q, &tm_q, &bars[B_FULL + s], 0, row, bh);
        tma_load_3d(st + S_DO, &tm_do, &bars[B_FULL + s], 0, row, bh);
        tma_load_3d(st + S_V, &tm_v, &bars[B_FULL + s], 0, row, bh);
      }
    }
  } else if (warp == 1 || warp == WY) {
    // ------------------------------------------------------------- MMA issuers
    constexpr uint32_t ID_S = idesc_bf16(128, 128, 0, 0);   // K-major x K-major, N = 128 tokens
    constexpr uint32_t ID_PV = idesc_bf16(128, 64, 0, 1);   // P (TMEM) x MN-major, N = 64
    constexpr uint32_t ID_E = idesc_bf16(128, 64, 0, 1);    // (a.K) x dKV   (MN-major B)
    constexpr uint32_t ID_ET = idesc_bf16(128, 64, 0, 0);   // (a.V) x dKV^T (K-major B)
    constexpr uint32_t ID_KV = idesc_bf16(64, 64, 1, 1);    // Q^T (MN-major) x c.dO (MN-major)
    const bool leader = (lane == 0);
    auto adv = [](uint64_t d, uint32_t bytes) { return d + static_cast<uint64_t>(bytes >> 4); };
    const uint64_t dK0 = sdesc_sw128(smem_u32(smem), 16, 1024);          // K-major view base
    const uint64_t dM0 = sdesc_sw128(smem_u32(smem), REGION, 1024);      // MN-major view base
    const uint64_t dKVk = sdesc_sw128(smem_u32(smem + OFF_KV), 16, 1024);          // K-major
    const uint64_t dKVm = sdesc_sw128(smem_u32(smem + OFF_KV), 64 * 128, 1024);    // MN-major
    if (warp == 1) {
      // ---- X: scores Sa = K Q^T, Sc = V dO^T
      for (int i = 0; i < nblk; ++i) {
        const int s = i % NS;
        const uint32_t so = s * STAGE;
        TR(1, i, 0);
        mbar_wait(&bars[B_FULL + s], (i / NS) & 1);
        if (i >= 1) mbar_wait(&bars[B_SFREE], (i - 1) & 1);
        TR(1, i, 1);
        tc_fence_after();
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_ss(tbase + T_SA, adv(dK0, so + S_K + kk * 32), adv(dK0, so + S_Q + kk * 32), ID_S,
                         kk > 0);
          umma_commit(&bars[B_SFULLA]);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_ss(tbase + T_SC, adv(dK0, so + S_V + kk * 32), adv(dK0, so + S_DO + kk * 32),
                         ID_S, kk > 0);
          umma_commit(&bars[B_SFULLC]);
          umma_commit(&bars[B_EMPTY + s]);
        }
        __syncwarp();
      }
    } else {
      // ---- Y: fold dKV_i = Q^T (c.dO) (early), then dV_i, dK_i (intra + inter)
      for (int i = 0; i < nblk; ++i) {
        const int s = i % NS, db = i & 1, pb = i & 1;
        const uint32_t so = s * STAGE;
        TR(4, i, 0);
        mbar_wait(&bars[B_DTREADY], i & 1);
        if (i >= 2) mbar_wait(&bars[B_DKVEMPTY + db], ((i >> 1) - 1) & 1);
        mbar_wait(&bars[B_FULL + s], (i / NS) & 1);
        TR(4, i, 1);
        tc_fence_after();
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ss(tbase + T_KV + db * 64, adv(dM0, so + S_Q + kk * 2048),
                         adv(dM0, OFF_DOT + kk * 2048), ID_KV, kk > 0);
          umma_commit(&bars[B_DKVFULL + db]);
          umma_commit(&bars[B_DTFREE]);
        }
        __syncwarp();
        mbar_wait(&bars[B_PREADY + pb], (i >> 1) & 1);
        TR(4, i, 2);
        mbar_wait(&bars[B_KVREADY], i & 1);
        if (i >= 1) mbar_wait(&bars[B_OEMPTY], (i - 1) & 1);
        TR(4, i, 3);
        tc_fence_after();
        if (leader) {
          // dV = Pa dO + (a.K) dKV
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts(tbase + T_DV, tbase + T_SA + kk * 8, adv(dM0, so + S_DO + kk * 2048), ID_PV,
                         kk > 0);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_ss(tbase + T_DV, adv(dK0, OFF_KT + pb * T + kk * 32), adv(dKVm, kk * 2048), ID_E, 1);
          // dK = Pc Q + (a.V) dKV^T
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts(tbase + T_DK, tbase + T_SC + kk * 8, adv(dM0, so + S_Q + kk * 2048), ID_PV,
                         kk > 0);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_ss(tbase + T_DK, adv(dK0, OFF_VT + pb * T + kk * 32), adv(dKVk, kk * 32), ID_ET, 1);
          umma_commit(&bars[B_OFULL]);
          umma_commit(&bars[B_SFREE]);
          umma_commit(&bars[B_EMPTY + s]);
        }
        __syncwarp();
        TR(4, i, 4);
      }
    }
  } else if (warp < W0) {
    // --------------------------------------------------------------- row warps
    const int path = (warp - 2) >> 2;  // 0: Sa -> Pa, a.K, dV   1: Sc -> Pc, a.V, dK
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t tS = tbase + (path ? T_SC : T_SA) + lane_off;
    const uint32_t tO = tbase + (path ? T_DK : T_DV) + lane_off;
    __nv_bfloat16* gout = path ? gdk : gdv;
    // reverse mask row factors: M[row][16ch + j] = (ch == dch) ? Dg[row][j] : F[ch] * G[j]
    float* Gs = reinterpret_cast<float*>(smem + OFF_MASK + 128 * 16 * 4);
    float* Dgs = reinterpret_cast<float*>(smem + OFF_MASK) + row * 16;
    const int dch = row >> 4, tt = row & 15;
    if (path == 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j) Dgs[j] = (j >= tt) ? lam_pow(l2, j - tt) : 0.f;
      if (row < 16) Gs[row] = lam_pow(l2, row);
    }
    named_bar_sync(1, 256);  // tables visible to both paths
    float F[8];
#pragma unroll
    for (int ch = 0; ch < 8; ++ch) F[ch] = (ch > dch) ? lam_pow(l2, 16 * ch - row) : 0.f;
    for (int j = 0; j <= nblk; ++j) {
      if (j < nblk) {
        // ---- A(j): scores -> P (bf16 pairs, in place); row-scaled copy a.K or a.V
        const int i = j, s = i % NS, pb = i & 1;
        const int blk = nblk - 1 - i;
        const int r = min(BT, N - blk * BT);
        const float a = row < r ? lam_pow(l2, r - 1 - row) : 0.f;
        if (warp == 2) TR(2, i, 0);
        mbar_wait(&bars[B_FULL + s], (i / NS) & 1);
        scale_row_copy<64>(smem + s * STAGE + (path ? S_V : S_K), smem + (path ? OFF_VT : OFF_KT) + pb * T,
                           row, a);
        fence_proxy_async_smem();
        mbar_wait(&bars[path ? B_SFULLC : B_SFULLA], i & 1);
        if (warp == 2) TR(2, i, 1);
        tc_fence_after();
#pragma unroll
        for (int cp = 0; cp < 4; ++cp) {
          uint32_t raw[32];
          tmem_ld32_raw(tS + cp * 32, raw);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int hc = 0; hc < 2; ++hc) {  // two 16-column chunks
            const int ch = 2 * cp + hc;
            const float* mt = (ch == dch) ? Dgs : Gs;
            const float fc = (ch == dch) ? 1.f : F[ch];
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) {
              const float4 m = *reinterpret_cast<const float4*>(mt + 4 * e4);
              const int b0 = 16 * hc + 4 * e4;
              pk[8 * hc + 2 * e4] = pack_bf16x2(__uint_as_float(raw[b0]) * (fc * m.x),
                                                __uint_as_float(raw[b0 + 1]) * (fc * m.y));
              pk[8 * hc + 2 * e4 + 1] = pack_bf16x2(__uint_as_float(raw[b0 + 2]) * (fc * m.z),
                                                    __uint_as_float(raw[b0 + 3]) * (fc * m.w));
            }
          }
          tmem_st16(tS + cp * 16, pk);  // packed columns 16cp.. were read already
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_PREADY + pb]);
        if (warp == 2) TR(2, i, 2);
      }
      if (j >= 1) {
        // ---- B(j-1): accumulator -> bf16 -> global (each thread one 128-byte row)
        const int i = j - 1;
        const int blk = nblk - 1 - i;
        const int t = blk * BT + row;
        if (warp == 2) TR(2, i, 3);
        mbar_wait(&bars[B_OFULL], i & 1);
        if (warp == 2) TR(2, i, 4);
        tc_fence_after();
        uint4 w[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float x16[16];
          tmem_ld16(tO + q * 16, x16);
          tmem_ld_wait();
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            w[2 * q + hh].x = pack_bf16x2(x16[8 * hh + 0], x16[8 * hh + 1]);
            w[2 * q + hh].y = pack_bf16x2(x16[8 * hh + 2], x16[8 * hh + 3]);
            w[2 * q + hh].z = pack_bf16x2(x16[8 * hh + 4], x16[8 * hh + 5]);
            w[2 * q + hh].w = pack_bf16x2(x16[8 * hh + 6], x16[8 * hh + 7]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_OEMPTY]);
        if (t < N) {
          uint4* dst = reinterpret_cast<uint4*>(gout + (static_cast<size_t>(bh) * N + t) * 64);
#pragma unroll
          for (int c = 0; c < 8; ++c) dst[c] = w[c];
        }
        if (warp == 2) TR(2, i, 5);
      }
    }
  } else if (warp < WY) {
    // ------------------------------------------------------------- state warps
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;  // token row for c.dO
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    const bool has_kv = lane < 16;   // M = 64 fold: rows 16*q4 + lane
    const int kvrow = q4 * 16 + lane;
    const size_t sbase = static_cast<size_t>(bh) * 64 * 64;
    float kv[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) kv[j] = 0.f;
    if (p.kv_in != nullptr && has_kv) {
#pragma unroll
      for (int j = 0; j < 64; j += 4) {
        float4 w = *reinterpret_cast<const float4*>(p.kv_in + sbase + kvrow * 64 + j);
        kv[j] = w.x; kv[j + 1] = w.y; kv[j + 2] = w.z; kv[j + 3] = w.w;
      }
    }
    uint8_t* sKVb = smem + OFF_KV;
    if (has_kv) {
#pragma unroll
      for (int q = 0; q < 4; ++q) store_chunk16_bf16(sKVb, kvrow, q, kv + 16 * q);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[B_KVREADY]);
    const float cfold = lam_pow(l2, row + 1);
    for (int j = 0; j <= nblk; ++j) {
      if (j < nblk) {
        // ---- c.dO(j), c_t = lam^(t+1)
        const int s = j % NS;
        if (warp == W0) TR(3, j, 0);
        mbar_wait(&bars[B_FULL + s], (j / NS) & 1);
        if (j >= 1) mbar_wait(&bars[B_DTFREE], (j - 1) & 1);
        scale_row_copy<64>(smem + s * STAGE + S_DO, smem + OFF_DOT, row, cfold);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_DTREADY]);
        if (warp == W0) TR(3, j, 1);
      }
      if (j >= 1) {
        // ---- dKV <- lam^r dKV + fold(j-1)
        const int i = j - 1, db = i & 1;
        const int blk = nblk - 1 - i;
        const int r = min(BT, N - blk * BT);
        const float fr = lam_pow(l2, static_cast<float>(r));
        if (warp == W0) TR(3, i, 2);
        mbar_wait(&bars[B_DKVFULL + db], (i >> 1) & 1);
        if (warp == W0) TR(3, i, 3);
        tc_fence_after();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float d16[16];
          tmem_ld16(tbase + T_KV + db * 64 + lane_off + q * 16, d16);
          tmem_ld_wait();
          if (has_kv) {
#pragma unroll
            for (int e = 0; e < 16; ++e) kv[16 * q + e] = fmaf(fr, kv[16 * q + e], d16[e]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_DKVEMPTY + db]);
        // the bf16 dKV is the operand of block i's inter products: wait until consumed
        mbar_wait(&bars[B_OFULL], i & 1);
        if (warp == W0) TR(3, i, 4);
        if (has_kv) {
#pragma unroll
          for (int q = 0; q < 4; ++q) store_chunk16_bf16(sKVb, kvrow, q, kv + 16 * q);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_KVREADY]);
        if (warp == W0) TR(3, i, 5);
      }
    }
    if (p.kv_out != nullptr && has_kv) {
      float* dst = p.kv_out + sbase + kvrow * 64;
#pragma unroll
      for (int j = 0; j < 64; j += 4)
        *reinterpret_cast<float4*>(dst + j) = make_float4(kv[j], kv[j + 1], kv[j + 2], kv[j + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

#ifdef LA2_TRACE
int set_trace_bwd(long long* buf) {
  cudaError_t e = cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf));
  return e == cudaSuccess ? 0 : set_cuda_error("set_trace_bwd", e);
}
#endif

int launch_g(const void* q, const void* k, const void* v, const void* dout, void* dk, void* dv,
             const float* decay, const float* dkv_in, float* dkv_out, int B, int H, int N,
             cudaStream_t st) {
  if (tma_encoder_ready() != 0) return set_error(LA2_ERR_CUDA, "cannot resolve cuTensorMapEncodeTiled");
  cudaError_t e = cudaFuncSetAttribute(la2_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       g::TOTAL);
  if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(bwd)", e);
  const int BH = B * H;
  CUtensorMap mk, mq, mdo, mv;
  const void* ptrs[4] = {k, q, dout, v};
  CUtensorMap* maps[4] = {&mk, &mq, &mdo, &mv};
  for (int t = 0; t < 4; ++t) {
    if (make_tmap_bf16(maps[t], ptrs[t], 64, N, BH, BT) != 0)
      return set_error(LA2_ERR_CUDA, "cuTensorMapEncodeTiled failed (bwd)");
  }
  FParams p;
  p.N = N;
  p.H = H;
  p.decay = decay;
  p.kv_in = dkv_in;
  p.kv_in_T = 0;
  p.kv_out = dkv_out;
  p.dv_total = 64;
  dim3 grid(1, H, B);
  la2_bwd_kernel<<<grid, g::THREADS, g::TOTAL, st>>>(mk, mq, mdo, mv, static_cast<__nv_bfloat16*>(dk),
                                                      static_cast<__nv_bfloat16*>(dv), p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("la2_bwd_kernel launch", e);
  return 0;
}

}  // namespace la2
