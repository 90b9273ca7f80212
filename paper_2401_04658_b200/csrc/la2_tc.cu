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
//   S      = Q_i K_i^T                              SS-MMA  -> TMEM S[b] (fp32)
//   P      = bf16(S * M)  M[t][u] = lam^(t-u), u<=t (rev: lam^(u-t), u>=t), written back
//            into TMEM over S[b] (packed bf16 pairs) by the row warps
//   O_i    = P V_i                                  TS-MMA  (A = P from TMEM)
//   Oe_i   = Q_i KV_{i-1}                           SS-MMA  (KV as bf16 B operand)
//   o_t    = O_i[t] + a_t Oe_i[t]    a_t = lam^(t+1) | rev: lam^(r-1-t)   (registers)
//   V~     = bf16(c_t V_i)           c_t = lam^(r-1-t)| rev: lam^(t+1)    (state warps)
//   dKV    = K_i^T V~                               SS-MMA  -> TMEM
//   KV_i   = lam^r KV_{i-1} + dKV                   fp32 registers of the state warps
// The fp32 KV state never leaves the SM.
//
// Warp roles (512 threads = 16 warps, one CTA per SM):
//   warp 0     TMA producer (Q/K/V ring of NS stages)
//   warp 1     MMA issuer X (S = QK^T, O = PV) + TMEM owner
//   warp 14    MMA issuer Y (dKV = K~^T V, Oe = Q KV): the state chain never waits
//              behind the score chain, so a late load cannot stall the recurrence
//   warps 2-9  row warps:   thread <-> token row, two warps per TMEM lane quarter
//              splitting the columns; S -> P, O epilogue + TMA store
//   warps 10-13 state warps: V~ rows, dKV -> fp32 KV state -> bf16 KV operand
//   warp 15    V~ copy warp (d = 128 full passes; idle otherwise)
//
// Scheduling: a persistent stream-K split of the (recurrence, block) space over the
// co-resident CTAs/clusters (Sched, la2_tc_common.cuh) when there are more recurrences
// than SMs; the producer walks the range and publishes a per-block record (head, block,
// segment start/end) in smem so the other roles carry no schedule state.
// d = 128: O lives in the upper half of its S buffer (OIS), so O is double-buffered.
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "la2_tc_common.cuh"

namespace la2 {

constexpr int TC_THREADS = 512;  // 16 warps: 4 per SM sub-partition, 128 registers each
constexpr int NROW = 8;         // row warps (2 per TMEM lane quarter)
constexpr int W0 = 2 + NROW;    // first state warp (4 state warps)
constexpr int WY = W0 + 4;      // second MMA issuer (state chain)
constexpr int WC = WY + 1;      // V~ copy warp
#ifndef LA2_GROUP_WAIT
#define LA2_GROUP_WAIT 0
#endif
// Group waits: one warp of a group polls an mbarrier, its partners sleep in a named
// barrier (fewer spinning warps: less issue pressure and power, one more bar.sync).
constexpr bool GW = (LA2_GROUP_WAIT != 0);
// Backward pair / triple (d = dv = 64): the dV pass's state dKV and the dK pass's state
// dKV^T are the same matrix, so ranks 0 and 1 share ONE recurrence -- each computes the
// fold and the fp32 update for 32 of its 64 columns and writes its half of the bf16
// operand into both CTAs' shared memory (the dK pass reads it K-major, i.e. transposed).
#ifndef LA2_SPLIT_STATE
#define LA2_SPLIT_STATE 1
#endif
// how the peer gets its half of the operand: st.async per 16 bytes (0) or one bulk copy
// per warp through the TMA unit (1)
#ifndef LA2_PEER_BULK
#define LA2_PEER_BULK 0
#endif

#ifndef LA2_SO_NS
#define LA2_SO_NS 4
#endif
// Output epilogue: each row warp stages and TMA-stores its own [32 rows][32 cols] tile
// (SW64, box 32 x 32) instead of the quarter's two warps meeting at two named barriers
// around one [32][64] store
#ifndef LA2_WARP_STORE
#define LA2_WARP_STORE 1
#endif

template <int DK, bool SO, bool TRI = false>
struct TcLayout {
  // Q/K/V stages; state-only passes stage only K and V (32 / 48 KB), so they get a deeper ring
  static constexpr int NS = SO ? LA2_SO_NS : ((DK == 64) ? 3 : 2);
  static constexpr int KTS = 2;                   // V~ buffers (scaled values)
  // O staging buffers (the backward triple spends the second one on its state tiles)
  static constexpr int OS = (DK == 64 && !SO && !TRI) ? 2 : 1;
  static constexpr int Q_BYTES = SO ? 0 : BT * DK * 2;
  static constexpr int K_BYTES = BT * DK * 2;
  static constexpr int V_BYTES = BT * DVS * 2;
  static constexpr int S_BYTES = TRI ? DK * DVS * 2 : 0;  // triple: stored bf16 state per stage
  static constexpr int KV_BYTES = SO ? 0 : DK * DVS * 2;
  static constexpr int O_BYTES = SO ? 0 : BT * DVS * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NS * Q_BYTES;
  static constexpr int OFF_V = OFF_K + NS * K_BYTES;
  static constexpr int OFF_S = OFF_V + NS * V_BYTES;
  static constexpr int OFF_KT = OFF_S + NS * S_BYTES;
  static constexpr int OFF_KV = OFF_KT + KTS * V_BYTES;
  // second bf16 state-operand buffer of the backward pair / triple's shared recurrence
  // (LA2_SPLIT_STATE): the triple's ranks 0-1 use their (otherwise idle) state-tile ring
  static constexpr bool KV2 = (DK == 64) && !SO && !TRI;
  static constexpr int OFF_O = OFF_KV + (KV2 ? 2 : 1) * KV_BYTES;
  static constexpr int OFF_KV2 = TRI ? OFF_S : OFF_KV + KV_BYTES;
  // fused per-head RMS norm (d = dv = 64 forward): each quarter's two row warps exchange
  // their half-row sums of squares through [2][128] floats
  static constexpr int NORM_BYTES = (DK == 64 && !SO && !TRI) ? 1024 : 0;
  static constexpr int OFF_NORM = OFF_O + OS * O_BYTES;
  static constexpr int OFF_BAR = OFF_NORM + NORM_BYTES;
  static constexpr int BAR_BYTES = 512;
  static constexpr int OFF_REC = OFF_BAR + BAR_BYTES;  // per-block schedule records (ring of 8)
  static constexpr int TOTAL = OFF_REC + 8 * 32 + 1024;  // + alignment slack
  static constexpr uint32_t STAGE_TX = Q_BYTES + K_BYTES + V_BYTES;
  // TMEM columns. OIS ("O in S", d = 128): S[b] @128b holds the scores, then P (packed
  // bf16, cols +0..63) and O_i = P_i V_i (fp32, cols +64..127), so O is double-buffered
  // with S and PV_i does not wait for the epilogue of block i-1 | Oe[2] @256,320 |
  // dKV[2] @384,448. Otherwise (d = 64): S[2] @0,128 (P in cols +0..31, +64..95) | O @256
  // | Oe @320 | dKV[2] @384,448 -- S_{i+2} then only waits for PV_i, not for the epilogue.
  // State-only: dKV[2] @0,64.
  static constexpr bool OIS = (DK == 128);
  // d = 128 (full passes): the V~ copy runs on its own warp, overlapping the state update
  // (-10 % at C3). d = 64 keeps it in the state warps: there the kernel is close to
  // issue-bound and a 16th busy warp slows its sub-partition (+8 %). State-only passes
  // must keep it in the state warps: their FULL waits would otherwise let the producer
  // run a full ring ahead of them.
  static constexpr bool CW = (DK == 128) && !SO;
  static constexpr uint32_t TMEM_COLS = SO ? 128 : 512;
  static constexpr uint32_t T_O = 256, T_OE = OIS ? 256 : 320, T_KV = SO ? 0 : 384;
  // barrier slots
  static constexpr int B_FULL = 0, B_EMPTY = NS, B_SFULL = 2 * NS, B_SFREE = B_SFULL + 2,
                       B_PREADY = B_SFREE + 2, B_OFULL = B_PREADY + 2, B_OEFULL = B_OFULL + 2,
                       B_OEMPTY = B_OEFULL + 2, B_KTREADY = B_OEMPTY + 2, B_KTFREE = B_KTREADY + KTS,
                       B_DKVFULL = B_KTFREE + KTS, B_DKVEMPTY = B_DKVFULL + 2,
                       B_KVREADY = B_DKVEMPTY + 2, B_KVFREE = B_KVREADY + 2, B_COUNT = B_KVFREE + 2;
  static_assert(B_COUNT * 8 + 16 <= BAR_BYTES, "barrier area");
  static_assert(TOTAL <= 232448, "shared memory budget");
};

// Cluster modes (2-CTA clusters along blockIdx.x; shared tiles are loaded once and
// multicast, stage release collects both CTAs' MMA commits):
//   CM = 0  no cluster
//   CM = 1  value-slice pair: both CTAs use the same Q and K tiles (rank 0 loads Q,
//           rank 1 loads K), each loads its own 64-column V slice
//   CM = 2  backward pair: rank 0 runs F_rev(K, Q, dO) -> dV, rank 1 runs
//           F_rev(V, dO, Q) -> dK; the Q and dO tiles are shared (rank 0 loads Q,
//           rank 1 loads dO) and play swapped k/v roles in the two CTAs
//   CM = 4  backward triple (d = dv = 64, with the per-block states the forward stored):
//           ranks 0-1 as CM 2, rank 2 computes dQ = F(dO, V, K) block by block from the
//           stored state KV_{i-1} (no recurrence), walking the same blocks in lockstep: dO
//           is multicast to all three, K from rank 0 to ranks 0 and 2, rank 2 loads V
//           itself (an L2 hit: rank 1 loads the same tile at the same time) and the state
//           tile. The backward then reads K, Q, dO, V once instead of also re-reading dO,
//           V, K for a separate dQ scan.
template <int DK, bool REV, bool SO, int CM>
__global__ void __launch_bounds__(TC_THREADS, 1)
    la2_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                  const __grid_constant__ CUtensorMap tm_q1, const __grid_constant__ CUtensorMap tm_k1,
                  const __grid_constant__ CUtensorMap tm_v1, const __grid_constant__ CUtensorMap tm_o1,
                  const FParams p) {
  using L = TcLayout<DK, SO, CM == 4>;
  constexpr bool CL = (CM != 0);
  constexpr int CS = (CM == 3) ? 4 : ((CM == 4) ? 3 : (CL ? 2 : 1));  // CTAs per cluster
  static_assert(CM != 2 || (DK == 64 && REV && !SO), "backward pair needs d = dv = 64");
  static_assert(CM != 4 || (DK == 64 && REV && !SO), "backward triple needs d = dv = 64");
  static_assert(CM != 3 || (DK == 128 && REV && !SO), "backward quad needs d = dv = 128");
  static_assert(!(SO && CM >= 2), "state-only passes run alone or as value-slice pairs");
  constexpr int NS = L::NS, KTS = L::KTS, OS = L::OS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + L::B_COUNT);
  BlkRec* recs = reinterpret_cast<BlkRec*>(smem + L::OFF_REC);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  TR_INIT;
  const uint32_t crank = CL ? cluster_ctarank() : 0;
  // CM 3: ranks 0-1 run one pass (value-slice pair), ranks 2-3 the sibling pass
  const int pair = (CM == 3) ? static_cast<int>(crank >> 1) : 0;
  const uint32_t prank = (CM == 3) ? (crank & 1) : crank;    // rank inside the pair
  // this pair's CTAs (the triple: all three)
  const uint16_t mcmask = (CM == 4) ? uint16_t(0x7) : static_cast<uint16_t>(0x3u << (2 * pair));
  const bool dqr = (CM == 4) && (crank == 2);  // the triple's stateless dQ CTA
  const bool rrev = REV && !dqr;               // scan direction of this CTA's masks / factors
  const bool sib = ((CM == 2 || CM == 4) && (crank == 1)) || ((CM == 3) && pair == 1);  // sibling pass
  // shared recurrence of the backward pair / triple (LA2_SPLIT_STATE): ranks 0-1 fold
  // Q^T (c . dO) (Q at OFF_K, dO at OFF_V in both), columns [32 crank, 32 crank + 32)
  constexpr bool SPLIT = (CM == 2 || CM == 4) && (LA2_SPLIT_STATE != 0);
  constexpr bool NORM_OK = (DK == 64) && !REV && !SO && (CM == 0);  // fused Norm(.) epilogue
  constexpr int KVC = SPLIT ? 32 : DVS;               // state columns held by this CTA
  const int kc0 = SPLIT ? 32 * static_cast<int>(crank) : 0;
  const CUtensorMap* mq = (sib || dqr) ? &tm_q1 : &tm_q;  // dqr: its own copy of V (tm_q1)
  const CUtensorMap* mo = dqr ? &tm_k1 : (sib ? &tm_o1 : &tm_o);  // dqr: dQ through tm_k1
  const CUtensorMap* mk = (CM == 3 && sib) ? &tm_k1 : &tm_k;
  const CUtensorMap* mv = (CM == 3 && sib) ? &tm_v1 : &tm_v;
  // smem regions of this CTA's q / k / v roles. Pair and triple: Q at OFF_K, dO at OFF_V,
  // the CTA's own q (K | V) at OFF_Q; the dQ CTA: q = dO (OFF_V), k = V (own load, OFF_K),
  // v = K (multicast by rank 0, OFF_Q), plus the stored state tile at OFF_S
  const int offq = dqr ? L::OFF_V : L::OFF_Q;
  const int offk = dqr ? L::OFF_K : (((CM == 2 || CM == 4) && sib) ? L::OFF_V : L::OFF_K);
  const int offv = dqr ? L::OFF_Q : (((CM == 2 || CM == 4) && sib) ? L::OFF_K : L::OFF_V);
  const int kv_in_T = SPLIT ? 0 : (sib ? 1 : p.kv_in_T);  // the dK pass carries dKV^T
  float* const kv_out = (SPLIT ? dqr : (sib || dqr)) ? nullptr : p.kv_out;
  const int offsk = SPLIT ? L::OFF_K : offk;  // the state chain's k / v tiles
  const int offsv = SPLIT ? L::OFF_V : offv;
  const int N = p.N;
  const int nblk = (N + BT - 1) / BT;
  const int cid = blockIdx.x / CS;                  // this CTA's (cluster's) work range
  Sched sch;
  sch.init(cid, p.P, p.units, nblk);
  const int T = sch.T;
  const int nsl = p.nsl, H = p.H, cr = static_cast<int>(prank);
  auto blk_of = [&](int pos) { return REV ? (nblk - 1 - pos) : pos; };
  // exact log2 of the head's decay (fast-math log2f is off by ~2^-22 absolute, which
  // compounds over 64K tokens when lam is close to 1); an invalid lam gives NaN
  auto log2_decay = [&](int h) {
    const float lam = checked_decay(p.decay[h]);
    return (lam == 1.f) ? 0.f : static_cast<float>(log2(static_cast<double>(lam)));
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&bars[L::B_FULL + s], 1);
      // X after PV, Y after Oe (x2 in a cluster: the stage is shared)
      mbar_init(&bars[L::B_EMPTY + s], (SO ? 1 : 2) * (CM == 4 ? 3 : (CL ? 2 : 1)));
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[L::B_SFULL + b], 1);
      mbar_init(&bars[L::B_SFREE + b], L::OIS ? NROW : 1);  // OIS: B(i) read O_i out of S[b]
      mbar_init(&bars[L::B_PREADY + b], NROW);
      mbar_init(&bars[L::B_OFULL + b], 1);
      mbar_init(&bars[L::B_OEFULL + b], 1);
      mbar_init(&bars[L::B_OEMPTY + b], NROW);
    }
    for (int b = 0; b < KTS; ++b) {
      mbar_init(&bars[L::B_KTREADY + b], L::CW ? 1 : 4);  // copy warp / state warps
      mbar_init(&bars[L::B_KTFREE + b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[L::B_DKVFULL + b], 1);
      mbar_init(&bars[L::B_DKVEMPTY + b], 4);
    }
    // SPLIT: per operand buffer, both CTAs' state warps / both CTAs' Oe commits
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars[L::B_KVREADY + b], 4);  // SPLIT: + the peer's half by bulk copy (tx bytes)
      mbar_init(&bars[L::B_KVFREE + b], 2);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    if (!SO) tma_prefetch_desc(mq);
    tma_prefetch_desc(mk);
    tma_prefetch_desc(mv);
    if (!SO) tma_prefetch_desc(mo);
    if (dqr) tma_prefetch_desc(&tm_v1);
  }
  if (warp == 1) tmem_alloc(tmem_slot, L::TMEM_COLS);
  if (threadIdx.x == 0) {
    // Programmatic dependent launch: the prologue above overlapped the previous kernel's
    // tail; nothing below touches global memory before that kernel has completed. Our
    // own dependents may start their prologue now (they wait for us the same way).
    griddep_wait();
    griddep_launch_dependents();
  }
  tc_fence_before();
  if (CL) cluster_sync();  // barriers initialised in both CTAs before any remote traffic
  else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      // With a 2-stage ring (d = 128: 80 KB stages) a stage is refilled only one block
      // ahead, which exposes HBM latency; pull the next PF blocks into L2 so the ring's
      // TMA loads hit L2.
      const int PF = (NS == 2) ? p.pf : 0;
      const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
      auto tma_prefetch_l2_3d = [&](const CUtensorMap* m, int c0, int c1, int c2) {
        if (p.hint & 2) la2::tma_prefetch_l2_3d_hint(m, c0, c1, c2, pol_last);
        else la2::tma_prefetch_l2_3d(m, c0, c1, c2);
      };
      auto tma_load_3d = [&](void* d, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2) {
        if (p.hint & 1) la2::tma_load_3d_hint(d, m, b, c0, c1, c2, pol_first);
        else la2::tma_load_3d(d, m, b, c0, c1, c2);
      };
      auto tma_load_3d_mc = [&](void* d, const CUtensorMap* m, uint64_t* b, int c0, int c1, int c2,
                                uint16_t mask) {
        if (p.hint & 1) la2::tma_load_3d_mc_hint(d, m, b, c0, c1, c2, mask, pol_first);
        else la2::tma_load_3d_mc(d, m, b, c0, c1, c2, mask);
      };
      Walk<CM> pw;  // the block PF ahead of the ring
      pw.start(sch, NS, nsl, H, cr);
      auto prefetch = [&]() {  // the tiles this CTA itself fetches for block pw.g
        const int bh = pw.bh, slice = pw.slice, b2 = blk_of(pw.pos);
        pw.next(sch, nsl, H, cr);
        if (CM == 0) {
#pragma unroll
          for (int c = 0; c < DK / 64; ++c) {
            if (!SO) tma_prefetch_l2_3d(mq, c * 64, b2 * BT, bh);
            tma_prefetch_l2_3d(&tm_k, c * 64, b2 * BT, bh);
          }
          tma_prefetch_l2_3d(&tm_v, slice * DVS, b2 * BT, bh);
        } else if (CM == 1 || CM == 3) {
#pragma unroll
          for (int c = 0; c < DK / 64; ++c)
            if (!SO || prank) tma_prefetch_l2_3d(prank ? mk : mq, c * 64, b2 * BT, bh);
          tma_prefetch_l2_3d(mv, slice * DVS, b2 * BT, bh);
        } else {
          tma_prefetch_l2_3d(mq, 0, b2 * BT, bh);
          tma_prefetch_l2_3d(crank ? &tm_v : &tm_k, 0, b2 * BT, bh);
        }
      };
      for (int g = NS; g < NS + PF && g < T; ++g) prefetch();
      Walk<CM> w;
      w.start(sch, 0, nsl, H, cr);
      const int suffix_start = sch.npre + sch.nfull * nblk;
      int rec_h = -1;
      float rec_l2 = 0.f;
      for (int g = 0; g < T; ++g, w.next(sch, nsl, H, cr)) {
        if (PF > 0 && g + NS + PF < T) prefetch();
        const int bh = w.bh, slice = w.slice, blk = blk_of(w.pos);
        const int s = g % NS;
        TR(0, g, 0);
        if (g >= NS) mbar_wait(&bars[L::B_EMPTY + s], ((g / NS) - 1) & 1);
        TR(0, g, 1);
        // Schedule record of block g for the row and state warps, published by the
        // FULL arrive below (ring of 8 > the deepest lag any consumer can have).
        if (w.h != rec_h) {
          rec_h = w.h;
          rec_l2 = log2_decay(w.h);
        }
        {
          BlkRec rc;
          rc.bh = bh;
          rc.slice = slice;
          rc.pos = w.pos;
          rc.blk = blk;
          rc.l2 = rec_l2;
          rc.h = w.h;
          rc.flags = ((w.pos == 0 || g == suffix_start) ? REC_SEG_START : 0) |
                     ((w.pos == nblk - 1 || g == sch.npre - 1) ? REC_SEG_END : 0);
          recs[g & 7] = rc;
        }
        mbar_arrive_expect_tx(&bars[L::B_FULL + s], dqr ? L::STAGE_TX + L::S_BYTES : L::STAGE_TX);
        const int row = blk * BT;
        uint64_t* fb = &bars[L::B_FULL + s];
        uint8_t* dq = smem + L::OFF_Q + s * L::Q_BYTES;
        uint8_t* dk = smem + L::OFF_K + s * L::K_BYTES;   // stage region "K" (tile of tm_k)
        uint8_t* dv = smem + L::OFF_V + s * L::V_BYTES;   // stage region "V" (tile of tm_v)
        if (CM == 0) {
#pragma unroll
          for (int c = 0; c < DK / 64; ++c) {
            if (!SO) tma_load_3d(dq + c * REGION, mq, fb, c * 64, row, bh);
            tma_load_3d(dk + c * REGION, &tm_k, fb, c * 64, row, bh);
          }
          tma_load_3d(dv, &tm_v, fb, slice * DVS, row, bh);
        } else if (CM == 1 || CM == 3) {
#pragma unroll
          for (int c = 0; c < DK / 64; ++c) {
            if (prank == 0) {
              if (!SO) tma_load_3d_mc(dq + c * REGION, mq, fb, c * 64, row, bh, mcmask);
            } else {
              tma_load_3d_mc(dk + c * REGION, mk, fb, c * 64, row, bh, mcmask);
            }
          }
          tma_load_3d(dv, mv, fb, slice * DVS, row, bh);
        } else if (CM == 2) {
          tma_load_3d(dq, mq, fb, 0, row, bh);  // own q: K (rank 0) or V (rank 1)
          if (crank == 0) tma_load_3d_mc(dk, &tm_k, fb, 0, row, bh, 0x3);  // Q -> region K
          else tma_load_3d_mc(dv, &tm_v, fb, 0, row, bh, 0x3);             // dO -> region V
        } else {  // CM 4
          if (crank == 0) {
            tma_load_3d_mc(dq, mq, fb, 0, row, bh, 0x5);    // K -> OFF_Q of ranks 0 and 2
            tma_load_3d_mc(dk, &tm_k, fb, 0, row, bh, 0x3);  // Q -> region K of ranks 0, 1
          } else if (crank == 1) {
            tma_load_3d(dq, mq, fb, 0, row, bh);             // V (own q of the dK pass)
            tma_load_3d_mc(dv, &tm_v, fb, 0, row, bh, 0x7);  // dO -> region V of all three
          } else {
            tma_load_3d(dk, mq, fb, 0, row, bh);             // V (the dQ pass's k)
            tma_load_3d(smem + L::OFF_S + s * L::S_BYTES, &tm_v1, fb, 0, blk * DK, bh);  // KV_{blk-1}
          }
        }
      }
      if (CL) {
        // every MMA of both CTAs that read this CTA's stages has committed
        for (int g = (T > NS ? T - NS : 0); g < T; ++g)
          mbar_wait(&bars[L::B_EMPTY + (g % NS)], (g / NS) & 1);
      }
    }
  } else if (warp == 1 || warp == WY) {
    // ------------------------------------------------------------- MMA issuers
    // The whole warp walks the schedule (converged barrier waits); one lane issues.
    constexpr uint32_t ID_S = idesc_bf16(128, 128, 0, 0);  // Q (K-major) x K (K-major)
    constexpr uint32_t ID_O = idesc_bf16(128, DVS, 0, 1);  // P/Q (K-major) x V/KV (MN-major)
    constexpr uint32_t ID_KV = idesc_bf16(DK, DVS, 1, 1);  // K~^T (MN-major) x V (MN-major)
    // SPLIT: this CTA's 32 state columns; V~ is a compact [128][32] SW64 tile
    constexpr uint32_t ID_KV32 = idesc_bf16(DK, 32, 1, 1);
    const bool leader = (lane == 0);
    const uint32_t tOE = tbase + L::T_OE, tKV = tbase + L::T_KV;
    // descriptor bases (start address is in 16-byte units in the low bits)
    constexpr uint32_t ID_OS = idesc_bf16(128, DVS, 0, 0);  // dO (K-major) x stored KV (K-major)
    const uint64_t dQ0 = sdesc_sw128(smem_u32(smem + offq), 16, 1024);
    const uint64_t dS0 = sdesc_sw128(smem_u32(smem + L::OFF_S), 16, 1024);
    const uint64_t dK0 = sdesc_sw128(smem_u32(smem + offk), 16, 1024);
    const uint64_t dV0 = sdesc_sw128(smem_u32(smem + offv), REGION, 1024);
    auto commit_empty = [&](int s) {
      if (CL) umma_commit_mc(&bars[L::B_EMPTY + s], mcmask);
      else umma_commit(&bars[L::B_EMPTY + s]);
    };
    const uint64_t dKT0 = sdesc_sw128(smem_u32(smem + L::OFF_KT), REGION, 1024);
    const uint64_t dKV0 = sdesc_sw128(smem_u32(smem + L::OFF_KV), DK * 128, 1024);
    auto adv = [](uint64_t d, uint32_t bytes) { return d + static_cast<uint64_t>(bytes >> 4); };

    if (warp == 1) {
      // ---- X: score chain  S_j = Q K^T ; O_i = P_i V_i
      // Event loop: S_j (needs stage j loaded and S buffer j&1 free) and PV_i (needs P_i
      // and the O accumulator free) are issued as soon as each is ready, so PV_i never
      // waits behind the arrival of block i+1 -- that coupling would keep only one stage
      // load in flight with a 2-stage ring. S runs at most one block ahead of PV.
      if (!SO && NS >= 3) {
        // deep ring (d = 64): block i+1 has normally landed before PV_i is due, so the
        // plain order S_{i+1}, PV_i keeps the tensor pipe fed with the least polling
        auto issue_S = [&](int j) {
          const int s = j % NS, b = j & 1;
          mbar_wait(&bars[L::B_FULL + s], (j / NS) & 1);
          if (j >= 2) mbar_wait(&bars[L::B_SFREE + b], ((j >> 1) - 1) & 1);
          tc_fence_after();
          if (leader) {
            const uint64_t q = adv(dQ0, s * L::Q_BYTES), k = adv(dK0, s * L::K_BYTES);
#pragma unroll
            for (int kk = 0; kk < DK / 16; ++kk) {
              const uint32_t off = (kk >> 2) * REGION + (kk & 3) * 32;
              umma_bf16_ss(tbase + b * 128, adv(q, off), adv(k, off), ID_S, kk > 0);
            }
            umma_commit(&bars[L::B_SFULL + b]);
          }
          __syncwarp();
        };
        if (T > 0) issue_S(0);
        for (int i = 0; i < T; ++i) {
          const int s = i % NS, b = i & 1;
          const uint64_t v = adv(dV0, s * L::V_BYTES);
          TR(1, i, 0);
          if (i + 1 < T) issue_S(i + 1);
          TR(1, i, 1);
          mbar_wait(&bars[L::B_PREADY + b], (i >> 1) & 1);
          TR(1, i, 2);
          if (!L::OIS && i >= 1) mbar_wait(&bars[L::B_OEMPTY + ((i - 1) & 1)], ((i - 1) >> 1) & 1);
          TR(1, i, 3);
          tc_fence_after();
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < BT / 16; ++kk) {
              const uint32_t pcol = L::OIS ? kk * 8 : (kk >> 2) * 64 + (kk & 3) * 8;
              umma_bf16_ts(L::OIS ? tbase + b * 128 + 64 : tbase + L::T_O, tbase + b * 128 + pcol,
                           adv(v, kk * 2048), ID_O, kk > 0);
            }
            if (!L::OIS) umma_commit(&bars[L::B_SFREE + b]);
            umma_commit(&bars[L::B_OFULL + b]);
            commit_empty(s);
          }
          __syncwarp();
        }
      } else if (!SO) {
        int nS = 0, nP = 0;
        while (nP < T) {
          bool s_ok = false, p_ok = false;
          if (lane == 0) {
            if (nS < T && nS <= nP + 1)
              s_ok = mbar_test(&bars[L::B_FULL + nS % NS], (nS / NS) & 1) &&
                     (nS < 2 || mbar_test(&bars[L::B_SFREE + (nS & 1)], ((nS >> 1) - 1) & 1));
            if (nP < nS)
              p_ok = mbar_test(&bars[L::B_PREADY + (nP & 1)], (nP >> 1) & 1) &&
                     (L::OIS || nP == 0 || mbar_test(&bars[L::B_OEMPTY + ((nP - 1) & 1)], ((nP - 1) >> 1) & 1));
          }
          s_ok = __shfl_sync(0xffffffffu, s_ok, 0);
          p_ok = __shfl_sync(0xffffffffu, p_ok, 0);
          if (!s_ok && !p_ok) {
            __nanosleep(32);
            continue;
          }
          tc_fence_after();
          if (s_ok) {
            const int s = nS % NS, b = nS & 1;
            TR(1, nS, 1);
            if (leader) {
              const uint64_t q = adv(dQ0, s * L::Q_BYTES), k = adv(dK0, s * L::K_BYTES);
#pragma unroll
              for (int kk = 0; kk < DK / 16; ++kk) {
                const uint32_t off = (kk >> 2) * REGION + (kk & 3) * 32;
                umma_bf16_ss(tbase + b * 128, adv(q, off), adv(k, off), ID_S, kk > 0);
              }
              umma_commit(&bars[L::B_SFULL + b]);
            }
            ++nS;
          }
          if (p_ok) {
            const int s = nP % NS, b = nP & 1;
            const uint64_t v = adv(dV0, s * L::V_BYTES);
            TR(1, nP, 3);
            if (leader) {
#pragma unroll
              for (int kk = 0; kk < BT / 16; ++kk) {
                const uint32_t pcol = L::OIS ? kk * 8 : (kk >> 2) * 64 + (kk & 3) * 8;
                umma_bf16_ts(L::OIS ? tbase + b * 128 + 64 : tbase + L::T_O, tbase + b * 128 + pcol,
                             adv(v, kk * 2048), ID_O, kk > 0);
              }
              if (!L::OIS) umma_commit(&bars[L::B_SFREE + b]);
              umma_commit(&bars[L::B_OFULL + b]);
              commit_empty(s);
            }
            ++nP;
          }
          __syncwarp();
        }
      }
    } else {
      // ---- Y: state chain  dKV_i = K~_i^T V_i (early) ; Oe_i = Q_i KV_{i-1}
      auto issue_fold = [&](int i) {
        const int s = i % NS, kt = i % KTS, db = i & 1;
        tc_fence_after();
        if (leader) {
          // dKV = K^T (c . V): A = K^T (MN-major view of the K stage), B = V~ (MN-major)
          const uint64_t vt_d = SPLIT ? sdesc_sw64(smem_u32(smem + L::OFF_KT + kt * L::V_BYTES), 4096, 512)
                                      : adv(dKT0, kt * L::V_BYTES);
          const uint64_t kA = sdesc_sw128(smem_u32(smem + offsk + s * L::K_BYTES), REGION, 1024);
#pragma unroll
          for (int kk = 0; kk < BT / 16; ++kk)
            umma_bf16_ss(tKV + db * 64, adv(kA, kk * 2048), adv(vt_d, kk * (SPLIT ? 1024 : 2048)),
                         SPLIT ? ID_KV32 : ID_KV, kk > 0);
          umma_commit(&bars[L::B_DKVFULL + db]);
          umma_commit(&bars[L::B_KTFREE + kt]);
          if (SO) commit_empty(s);
        }
        __syncwarp();
      };
      auto issue_oe = [&](int i) {
        const int s = i % NS, db = i & 1;
          tc_fence_after();
          if (leader) {
            const uint64_t q = adv(dQ0, s * L::Q_BYTES);
            if (SPLIT) {
              // the shared operand: two [64 d rows][32 dv cols] SW64 halves (one per CTA,
              // 4 KB apart). dV pass (rank 0): Oe = K dKV, B MN-major (K = d rows, 16 per
              // step = 1024 B; the halves are the two N atoms, LBO 4096). dK pass (rank 1):
              // Oe = V dKV^T, the same bytes K-major (N = d rows; K = dv: 32 B steps inside
              // a half, then the other half).
              const uint32_t kvb = smem_u32(smem + ((i & 1) ? L::OFF_KV2 : L::OFF_KV));
              if (crank == 0) {
                const uint64_t dm = sdesc_sw64(kvb, 4096, 512);
#pragma unroll
                for (int kk = 0; kk < DK / 16; ++kk)
                  umma_bf16_ss(tOE + (L::OIS ? db * 64 : 0), adv(q, (kk >> 2) * REGION + (kk & 3) * 32),
                               adv(dm, kk * 1024), ID_O, kk > 0);
              } else {
                const uint64_t dk = sdesc_sw64(kvb, 16, 512);
#pragma unroll
                for (int kk = 0; kk < DK / 16; ++kk)
                  umma_bf16_ss(tOE + (L::OIS ? db * 64 : 0), adv(q, (kk >> 2) * REGION + (kk & 3) * 32),
                               adv(dk, (kk >> 1) * 4096 + (kk & 1) * 32), ID_OS, kk > 0);
              }
            } else {
              const uint64_t kvd = dKV0;
#pragma unroll
              for (int kk = 0; kk < DK / 16; ++kk)
                umma_bf16_ss(tOE + (L::OIS ? db * 64 : 0), adv(q, (kk >> 2) * REGION + (kk & 3) * 32),
                             adv(kvd, kk * 2048), ID_O, kk > 0);
            }
            umma_commit(&bars[L::B_OEFULL + db]);
            if (SPLIT) umma_commit_mc(&bars[L::B_KVFREE + (i & 1)], 0x3);  // both CTAs' copies read
            commit_empty(s);
          }
          __syncwarp();
      };
      for (int i = 0; i < T; ++i) {
        const int s = i % NS, kt = i % KTS, db = i & 1;
        if (dqr) {
          // the triple's dQ CTA: no recurrence; Oe_i = dO_i (KV_{i-1})^T from the stored state
          mbar_wait(&bars[L::B_FULL + s], (i / NS) & 1);
          if (L::OIS && i >= 2) mbar_wait(&bars[L::B_OEMPTY + db], ((i >> 1) - 1) & 1);
          if (!L::OIS && i >= 1) mbar_wait(&bars[L::B_OEMPTY + ((i - 1) & 1)], ((i - 1) >> 1) & 1);
          tc_fence_after();
          if (leader) {
            const uint64_t q = adv(dQ0, s * L::Q_BYTES), st = adv(dS0, s * L::S_BYTES);
#pragma unroll
            for (int kk = 0; kk < DVS / 16; ++kk)
              umma_bf16_ss(tOE + (L::OIS ? db * 64 : 0), adv(q, (kk & 3) * 32), adv(st, (kk & 3) * 32), ID_OS,
                           kk > 0);
            umma_commit(&bars[L::B_OEFULL + db]);
            commit_empty(s);
          }
          __syncwarp();
          continue;
        }
        mbar_wait(&bars[L::B_KTREADY + kt], (i / KTS) & 1);
        if (i >= 2) mbar_wait(&bars[L::B_DKVEMPTY + db], ((i >> 1) - 1) & 1);
        mbar_wait(&bars[L::B_FULL + s], (i / NS) & 1);  // V visibility for this thread
        TR(1, i, 5);
        issue_fold(i);
        if (!SO) {
          // SPLIT: KV_{i-1} sits in operand buffer i & 1, half of it written by the peer
          if (SPLIT) mbar_wait(&bars[L::B_KVREADY + (i & 1)], (i >> 1) & 1);
          else mbar_wait(&bars[L::B_KVREADY], i & 1);
          if (L::OIS && i >= 2) mbar_wait(&bars[L::B_OEMPTY + db], ((i >> 1) - 1) & 1);
          if (!L::OIS && i >= 1) mbar_wait(&bars[L::B_OEMPTY + ((i - 1) & 1)], ((i - 1) >> 1) & 1);
          TR(1, i, 4);
          issue_oe(i);
        }
        TR(1, i, 6);
      }
      // SPLIT: the last Oe's commits (ours and the peer's) have landed in this CTA's
      // KVFREE barrier before teardown (no tcgen05 arrive may target an exited CTA)
      if (SPLIT && !dqr && T > 0) mbar_wait(&bars[L::B_KVFREE + ((T - 1) & 1)], ((T - 1) >> 1) & 1);
    }
  } else if (warp < W0) {
    // --------------------------------------------------------------- row warps
    if (!SO) {
      const int q4 = warp & 3;             // TMEM lane quarter
      const int half = (warp - 2) >> 2;    // column half handled by this warp
      const int row = q4 * 32 + lane;
      const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
      // Mask factors for this row and this warp's 4 chunks of 16 score columns:
      //   M[row][16ch + j] = (ch == dch) ? Dg[j] : F[ch] * G[j]   (F = 0 on the zero side)
      // recomputed whenever the schedule moves to another head. Each 32-column half hh of
      // the warp's columns is, for all 32 rows of the warp, either entirely masked out
      // (kind 0: no TMEM load, zeros), entirely decayed (kind 1: F[c] * G[j]), or it
      // straddles the diagonal (kind 2, only when 2*half + hh == q4: per-lane factors MX
      // precomputed with the head). Warp-uniform, so no divergence and no per-element
      // selects on the hot path.
      float G[16], F[4], MX[2][16];
      const int dch = row >> 4, tt = row & 15;
      const int hm = q4 - 2 * half;  // the straddling half (0/1) or none
      const int kind0 = (2 * half == q4) ? 2 : ((rrev ? 2 * half > q4 : 2 * half < q4) ? 1 : 0);
      const int kind1 = (2 * half + 1 == q4) ? 2 : ((rrev ? 2 * half + 1 > q4 : 2 * half + 1 < q4) ? 1 : 0);
      int mask_h = -1;
      for (int j = 0; j <= T; ++j) {
        if (j < T) {
          // ---- A(j): S -> P (bf16). This warp reads score columns [64h, 64h+64) and
          // writes the packed P pairs into columns [64h, 64h+32) of the same buffer.
          if (GW) {  // record j published and S_j complete: polled by half 0 only
            if (half == 0) {
              mbar_wait(&bars[L::B_FULL + j % NS], (j / NS) & 1);
              mbar_wait(&bars[L::B_SFULL + (j & 1)], (j >> 1) & 1);
            }
            named_bar_sync(1 + q4, 64);
          } else {
            mbar_wait(&bars[L::B_FULL + j % NS], (j / NS) & 1);  // record j is published
          }
          const BlkRec rc = recs[j & 7];
          if (rc.h != mask_h) {
            mask_h = rc.h;
            const float l2 = rc.l2;
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) G[jj] = rrev ? lam_pow(l2, jj) : lam_pow(l2, 15 - jj);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int ch = 4 * half + c;
              if (!rrev) F[c] = (ch < dch) ? lam_pow(l2, row - 16 * ch - 15) : 0.f;
              else F[c] = (ch > dch) ? lam_pow(l2, 16 * ch - row) : 0.f;
            }
            if (hm == 0 || hm == 1) {
#pragma unroll
              for (int cc = 0; cc < 2; ++cc) {
                const int ch = 4 * half + 2 * hm + cc;
                const float fv = !rrev ? ((ch < dch) ? lam_pow(l2, row - 16 * ch - 15) : 0.f)
                                      : ((ch > dch) ? lam_pow(l2, 16 * ch - row) : 0.f);
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                  const float dg = !rrev ? ((jj <= tt) ? lam_pow(l2, tt - jj) : 0.f)
                                        : ((jj >= tt) ? lam_pow(l2, jj - tt) : 0.f);
                  MX[cc][jj] = (ch == dch) ? dg : fv * G[jj];
                }
              }
            }
          }
          const int b = j & 1;
          const uint32_t tS = tbase + b * 128 + half * 64 + lane_off;
          if (warp == LA2_TRW) TR(2, j, 0);
          if (!GW) mbar_wait(&bars[L::B_SFULL + b], (j >> 1) & 1);
          if (warp == LA2_TRW) TR(2, j, 1);
          tc_fence_after();
          // 64 score columns -> 32 packed P columns at [32h, 32h+32): P ends up contiguous
          // in columns 0..63 of S[b] and columns 64..127 are free for O_i = P_i V_i. The
          // quarter's two warps sync between reading and writing (half 1 writes over
          // score columns half 0 reads).
          uint32_t pk[2][16];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int kd = hh ? kind1 : kind0;
            if (kd == 0) {
#pragma unroll
              for (int e = 0; e < 16; ++e) pk[hh][e] = 0u;
            } else {
              uint32_t raw[32];
              tmem_ld32_raw(tS + hh * 32, raw);
              tmem_ld_wait();
              if (kd == 1) {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  const int c = 2 * hh + (e >> 3), jj = (2 * e) & 15;
                  const float2 m = __fmul2_rn(make_float2(G[jj], G[jj + 1]), make_float2(F[c], F[c]));
                  const float2 x = __fmul2_rn(make_float2(__uint_as_float(raw[2 * e]),
                                                          __uint_as_float(raw[2 * e + 1])), m);
                  pk[hh][e] = pack_bf16x2(x.x, x.y);
                }
              } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  const int cc = e >> 3, jj = (2 * e) & 15;
                  const float2 x = __fmul2_rn(make_float2(__uint_as_float(raw[2 * e]),
                                                          __uint_as_float(raw[2 * e + 1])),
                                              make_float2(MX[cc][jj], MX[cc][jj + 1]));
                  pk[hh][e] = pack_bf16x2(x.x, x.y);
                }
              }
            }
            if (!L::OIS) tmem_st16(tS + hh * 16, pk[hh]);  // in place: no cross-warp hazard
          }
          if (L::OIS) {
            named_bar_sync(1 + q4, 64);
            const uint32_t tP = tbase + b * 128 + half * 32 + lane_off;
            tmem_st16(tP, pk[0]);
            tmem_st16(tP + 16, pk[1]);
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[L::B_PREADY + b]);
          if (warp == LA2_TRW) TR(2, j, 2);
        }
        if (j >= 1) {
          // ---- B(j-1): o = O + a_t Oe for value columns [32h, 32h+32) -> smem -> TMA store
          const int i = j - 1;
          // record i was acquired in A(i); the ring slot is not rewritten before B(i) ends
          const BlkRec rb = recs[i & 7];
          const int bh = rb.bh, slice = rb.slice, blk = rb.blk;
          const float out_l2 = rb.l2;
          const int r = min(BT, N - blk * BT);
          const float a = rrev ? (row < r ? lam_pow(out_l2, r - 1 - row) : 0.f) : lam_pow(out_l2, row + 1);
          uint8_t* sO = smem + L::OFF_O + (i % OS) * L::O_BYTES;
          const bool storer = (half == 0 && lane == 0);
          if (warp == LA2_TRW) TR(2, i, 3);
          const int ob = i & 1;
          if (LA2_WARP_STORE) {
            if (lane == 0) tma_store_wait_read<OS - 1>();  // this warp's previous store read sW
            __syncwarp();
            mbar_wait(&bars[L::B_OFULL + ob], (i >> 1) & 1);
            mbar_wait(&bars[L::B_OEFULL + ob], (i >> 1) & 1);
          } else if (GW) {
            if (half == 0) {
              if (storer) tma_store_wait_read<OS - 1>();
              mbar_wait(&bars[L::B_OFULL + ob], (i >> 1) & 1);
              mbar_wait(&bars[L::B_OEFULL + ob], (i >> 1) & 1);
            }
            named_bar_sync(1 + q4, 64);
          } else {
            if (storer) tma_store_wait_read<OS - 1>();
            named_bar_sync(1 + q4, 64);  // the two warps of this quarter
            if (warp == LA2_TRW) TR(2, i, 4);
            mbar_wait(&bars[L::B_OFULL + ob], (i >> 1) & 1);
            mbar_wait(&bars[L::B_OEFULL + ob], (i >> 1) & 1);
          }
          if (warp == LA2_TRW) TR(2, i, 5);
          tc_fence_after();
          float o16[2][16], e16[2][16];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            tmem_ld16((L::OIS ? tbase + ob * 128 + 64 : tbase + L::T_O) + lane_off + half * 32 + q * 16,
                      o16[q]);
            tmem_ld16(tbase + L::T_OE + (L::OIS ? ob * 64 : 0) + lane_off + half * 32 + q * 16, e16[q]);
          }
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (L::OIS) mbar_arrive(&bars[L::B_SFREE + ob]);
            mbar_arrive(&bars[L::B_OEMPTY + ob]);
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
#pragma unroll
            for (int e = 0; e < 16; e += 2) {
              const float2 y = __ffma2_rn(make_float2(e16[q][e], e16[q][e + 1]), make_float2(a, a),
                                          make_float2(o16[q][e], o16[q][e + 1]));
              o16[q][e] = y.x;
              o16[q][e + 1] = y.y;
            }
          }
          if (NORM_OK && p.norm_eps > 0.f) {
            // Norm(.): y = o / sqrt(mean(o^2) + eps) over the row's 64 values, split over this
            // quarter's two warps (32 each): exchange the half sums through smem
            float ss = 0.f;
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
              for (int e = 0; e < 16; ++e) ss = fmaf(o16[q][e], o16[q][e], ss);
            float* sn = reinterpret_cast<float*>(smem + L::OFF_NORM);
            sn[half * 128 + row] = ss;
            named_bar_sync(1 + q4, 64);
            const float rs = rsqrtf((ss + sn[(1 - half) * 128 + row]) * (1.f / 64.f) + p.norm_eps);
            named_bar_sync(1 + q4, 64);  // both read before the next block overwrites
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
              for (int e = 0; e < 16; ++e) o16[q][e] *= rs;
            if (half == 0 && blk * BT + row < N) p.rstd[static_cast<size_t>(bh) * N + blk * BT + row] = rs;
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (LA2_WARP_STORE) store_chunk16_bf16_sw64(sO + (q4 * 2 + half) * 2048, lane, q, o16[q]);
            else store_chunk16_bf16(sO, row, 2 * half + q, o16[q]);
          }
          fence_proxy_async_smem();
          if (LA2_WARP_STORE) {
            __syncwarp();
            if (lane == 0) {
              uint8_t* sW = sO + (q4 * 2 + half) * 2048;
              const int c0 = slice * DVS + half * 32, r0 = blk * BT + q4 * 32;
              if (p.accum) tma_reduce_add_3d(mo, sW, c0, r0, bh);
              else tma_store_3d(mo, sW, c0, r0, bh);
              tma_store_commit();
            }
          } else {
          named_bar_sync(1 + q4, 64);
          if (storer) {
            if (p.accum)
              tma_reduce_add_3d(mo, sO + q4 * 32 * 128, slice * DVS, blk * BT + q4 * 32, bh);
            else if (p.hint & 4)
              tma_store_3d_hint(mo, sO + q4 * 32 * 128, slice * DVS, blk * BT + q4 * 32, bh,
                                l2_policy_evict_first());
            else
              tma_store_3d(mo, sO + q4 * 32 * 128, slice * DVS, blk * BT + q4 * 32, bh);
            tma_store_commit();
          }
          }
          if (warp == LA2_TRW) TR(2, i, 6);
        }
      }
      if ((LA2_WARP_STORE || half == 0) && lane == 0) tma_store_wait_all0();
    }
  } else if (warp < WY && !dqr) {
    // ------------------------------------------------------------- state warps
    const int q4 = warp & 3;  // warps 10-13 -> quarters 2,3,0,1
    const int row = q4 * 32 + lane;  // token row for K~
    const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
    // dKV rows: M=128 -> lane == d row; M=64 -> lanes 0-15 of each quarter hold 16 rows
    const bool has_kv = (DK == 128) || (lane < 16);
    const int kvrow = (DK == 128) ? row : (q4 * 16 + lane);
    float kv[KVC];
    // SPLIT: the peer's operand buffer and KVREADY barrier (this CTA writes half of both)
    const uint32_t peer = static_cast<uint32_t>(crank) ^ 1u;
    // (operand buffer b at OFF_KV / OFF_KV2 with its KVREADY barrier; KV_m goes to (m + 1) & 1)
    const uint32_t r_base = SPLIT ? mapa_shared(smem_u32(smem), peer) : 0u;
    const uint32_t r_kvready0 = SPLIT ? mapa_shared(smem_u32(&bars[L::B_KVREADY]), peer) : 0u;
    // Segment start: the caller's initial state (or zero) at scan position 0, else the
    // state the previous work range published for this unit.
    auto load_state = [&](int bh, int slice, int pos) {
#pragma unroll
      for (int j = 0; j < KVC; ++j) kv[j] = 0.f;
      if (pos == 0) {
        // (rows >= the real head dim / columns >= the real value width are padding: 0)
        if (p.kv_in != nullptr && has_kv && kvrow < p.dkr) {
          const size_t sbase = static_cast<size_t>(bh) * p.kv_in_bhs;
          const int c0 = slice * DVS + kc0;
          if (!kv_in_T) {
            const float* src = p.kv_in + sbase + static_cast<size_t>(kvrow) * p.kv_in_rs + c0;
#pragma unroll
            for (int j = 0; j < KVC; j += 4) {
              if (c0 + j < p.dv_total) {
                float4 w = *reinterpret_cast<const float4*>(src + j);
                kv[j] = w.x; kv[j + 1] = w.y; kv[j + 2] = w.z; kv[j + 3] = w.w;
              }
            }
          } else {
            // state stored transposed: element (r, c) at c * rs + r
            // the row stride is DK (a [dv][dk] state) or 256 (split-d column halves of a
            // [dv][256] state; the launcher rejects anything else): compile-time strides
            // keep this cold path to one load per element (a runtime stride costs ~4
            // instructions each, enough extra code to slow the d = 128 passes by ~2 %)
            const float* src = p.kv_in + sbase + static_cast<size_t>(c0) * p.kv_in_rs + kvrow;
            if (p.kv_in_rs == DK) {
#pragma unroll
              for (int j = 0; j < KVC; ++j) kv[j] = src[j * DK];
            } else {
#pragma unroll
              for (int j = 0; j < KVC; ++j) kv[j] = src[j * 256];
            }
          }
        }
      } else {
        const int slot = (cid - 1) * CS + static_cast<int>(crank);
        if (warp == W0 && lane == 0) flag_wait_consume(p.flags + slot);
        named_bar_sync(5, 128);
        if (has_kv) {
          const float4* src = reinterpret_cast<const float4*>(
              p.ws + (static_cast<size_t>(slot) * DK + kvrow) * DVS);
#pragma unroll
          for (int j = 0; j < KVC; j += 4) {
            float4 w = __ldcg(src + j / 4);
            kv[j] = w.x; kv[j + 1] = w.y; kv[j + 2] = w.z; kv[j + 3] = w.w;
          }
        }
      }
    };
    // Segment end: the caller's final state at the last scan position, else publish the
    // state for the next work range (which continues this unit).
    auto store_state = [&](int bh, int slice, int pos) {
      if (pos == nblk - 1) {
        if (kv_out != nullptr && has_kv && kvrow < p.dkr) {
          float* dst = kv_out + static_cast<size_t>(bh) * p.kv_out_bhs +
                       static_cast<size_t>(kvrow) * p.kv_out_rs + slice * DVS + kc0;
#pragma unroll
          for (int j = 0; j < KVC; j += 4)
            if (slice * DVS + kc0 + j < p.dv_total)
              *reinterpret_cast<float4*>(dst + j) = make_float4(kv[j], kv[j + 1], kv[j + 2], kv[j + 3]);
        }
      } else {
        const int slot = cid * CS + static_cast<int>(crank);
        if (has_kv) {
          float4* dst = reinterpret_cast<float4*>(p.ws + (static_cast<size_t>(slot) * DK + kvrow) * DVS);
#pragma unroll
          for (int j = 0; j < KVC; j += 4) __stcg(dst + j / 4, make_float4(kv[j], kv[j + 1], kv[j + 2], kv[j + 3]));
        }
        __threadfence();
        named_bar_sync(5, 128);
        if (warp == W0 && lane == 0) flag_release(p.flags + slot, 1);
      }
    };
    uint8_t* sKVb = smem + L::OFF_KV;
    if (T > 0) {
      mbar_wait(&bars[L::B_FULL + 0], 0);
      const BlkRec rc = recs[0];
      load_state(rc.bh, rc.slice, rc.pos);
    }
    // Forward with stored states (p.store_states, d = 64 F passes): the bf16 operand copy
    // of KV_{blk-1} that Oe_blk reads is also written to kv_blocks[bh][blk] by TMA (the
    // backward triple's dQ CTA reads it back instead of replaying the recurrence).
    const bool st_states = !SO && !REV && DK == 64 && p.store_states;
    auto store_block_state = [&](int j) {
      named_bar_sync(5, 128);  // all four warps' rows of the operand are written
      if (warp == W0 && lane == 0) {
        const BlkRec rn = recs[j & 7];
        tma_store_3d(&tm_v1, sKVb, 0, rn.blk * DK, rn.bh);
        tma_store_commit();
      }
    };
    // the bf16 operand copy of the state (SPLIT: this CTA's half, into both CTAs)
    auto write_operand = [&](int b) {
      if constexpr (SPLIT) {
        // this CTA's 32 columns of row kvrow are one contiguous 64-byte half of the
        // swizzled 128-byte row; written here, then bulk-copied into the peer's buffer
        // (completing 64 tx bytes of the peer's KVREADY; its W0 expects all 64 rows)
        // this CTA's half: [64 d rows][32 cols] SW64 at +4096 * crank; a warp's 16 rows
        // are one contiguous KB, bulk-copied into the peer's buffer (completing tx bytes
        // of the peer's KVREADY, whose W0 expects all 4 KB)
        uint8_t* hb = smem + (b ? L::OFF_KV2 : L::OFF_KV) + 4096 * static_cast<int>(crank);
        if (has_kv) {
          const uint32_t ro = static_cast<uint32_t>(hb - smem) + kvrow * 64;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 w;
            w.x = pack_bf16x2(kv[8 * c + 0], kv[8 * c + 1]);
            w.y = pack_bf16x2(kv[8 * c + 2], kv[8 * c + 3]);
            w.z = pack_bf16x2(kv[8 * c + 4], kv[8 * c + 5]);
            w.w = pack_bf16x2(kv[8 * c + 6], kv[8 * c + 7]);
            const uint32_t o = ro + ((c ^ ((kvrow >> 1) & 3)) * 16);
            *reinterpret_cast<uint4*>(smem + o) = w;
#if LA2_PEER_BULK
          }
          fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) {
          const uint32_t off = static_cast<uint32_t>(hb - smem) + q4 * 16 * 64;
          bulk_copy_to_peer(r_base + off, smem + off, 16 * 64, r_kvready0 + 8u * b);
#else
            st_async_peer(r_base + o, w, r_kvready0 + 8u * b);  // the peer's copy, async
          }
          fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) {
#endif
          if (warp == W0) mbar_arrive_expect_tx(&bars[L::B_KVREADY + b], DK * 64);
          else mbar_arrive(&bars[L::B_KVREADY + b]);
        }
      } else {
        uint8_t* dst = sKVb;
        if (has_kv) {
#pragma unroll
          for (int q = 0; q < DVS / 16; ++q) store_chunk16_bf16(dst, kvrow, q, kv + 16 * q);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[L::B_KVREADY]);
      }
    };
    if (!SO) {
      write_operand(0);
      if (st_states && T > 0) store_block_state(0);
    }
    for (int j = 0; j <= T; ++j) {
      if (j < T) {
        // record j (and stage j) is published; FULL cannot run a phase ahead of block j
        // before U(j-1) below (or, state-only, this warp's V~ copy of block j) completes
        const int s = j % NS, kt = j % KTS;
        if (warp == W0) TR(3, j, 0);
        mbar_wait(&bars[L::B_FULL + s], (j / NS) & 1);
        if (!L::CW) {
          // ---- K~(j): scaled copy of the V rows (the fold operand)
          const BlkRec rc = recs[j & 7];
          const int r = min(BT, N - rc.blk * BT);
          const float c = REV ? lam_pow(rc.l2, row + 1) : (row < r ? lam_pow(rc.l2, r - 1 - row) : 0.f);
          if (j >= KTS) mbar_wait(&bars[L::B_KTFREE + kt], ((j / KTS) - 1) & 1);
          if (warp == W0) TR(3, j, 1);
          if (SPLIT)
            scale_row_copy_half_sw64(smem + offsv + s * L::V_BYTES, smem + L::OFF_KT + kt * L::V_BYTES, row,
                                static_cast<int>(crank), c);
          else
            scale_row_copy<64>(smem + offsv + s * L::V_BYTES, smem + L::OFF_KT + kt * L::V_BYTES,
                               row, c);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[L::B_KTREADY + kt]);
          if (warp == W0) TR(3, j, 2);
        }
      }
      if (j >= 1) {
        // ---- U(j-1): KV <- lam^r KV + dKV
        const int i = j - 1;
        // record i was acquired in K~(i); its ring slot outlives U(i) (see the producer)
        const BlkRec ru = recs[i & 7];
        const int bh = ru.bh, slice = ru.slice, pos = ru.pos, blk = ru.blk, flags = ru.flags;
        const float up_l2 = ru.l2;
        const int r = min(BT, N - blk * BT);
        const float fr = lam_pow(up_l2, static_cast<float>(r));
        if (warp == W0) TR(3, i, 3);
        const int db = i & 1;
        if (!GW || warp == W0) mbar_wait(&bars[L::B_DKVFULL + db], (i >> 1) & 1);
        if (GW) named_bar_sync(5, 128);
        if (warp == W0) TR(3, i, 4);
        tc_fence_after();
#pragma unroll
        for (int q = 0; q < KVC / 32; ++q) {  // 32-column loads: half the round trips
          uint32_t d32[32];
          tmem_ld32_raw(tbase + L::T_KV + db * 64 + lane_off + q * 32, d32);
          tmem_ld_wait();
          if (has_kv) {
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const float2 y = __ffma2_rn(make_float2(kv[32 * q + e], kv[32 * q + e + 1]), make_float2(fr, fr),
                                          make_float2(__uint_as_float(d32[e]), __uint_as_float(d32[e + 1])));
              kv[32 * q + e] = y.x;
              kv[32 * q + e + 1] = y.y;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[L::B_DKVEMPTY + db]);
        if (warp == W0) TR(3, i, 6);
        if (flags & REC_SEG_END) store_state(bh, slice, pos);
        if (j < T) {
          const BlkRec rn = recs[j & 7];  // acquired in K~(j) above
          if (rn.flags & REC_SEG_START) load_state(rn.bh, rn.slice, rn.pos);
        }
        if (!SO) {
          // the bf16 copy of KV_{i-1} is the B operand of Oe_i: wait until it is consumed
          // (SPLIT: by both CTAs, whose copies this CTA writes)
          // (SPLIT: KV_i goes to buffer (i + 1) & 1, last read by Oe_{i-1} in both CTAs)
          if (SPLIT) {
            if (i >= 1) mbar_wait(&bars[L::B_KVFREE + ((i - 1) & 1)], ((i - 1) >> 1) & 1);
          }
          else if (!GW || warp == W0) mbar_wait(&bars[L::B_OEFULL + (i & 1)], (i >> 1) & 1);
          if (GW) named_bar_sync(5, 128);
          if (st_states) {  // the previous block's state store has read the operand buffer
            if (warp == W0 && lane == 0) tma_store_wait_read<0>();
            named_bar_sync(5, 128);
          }
          if (warp == W0) TR(3, i, 7);
          // (SPLIT: no copy after the last block -- nothing reads it, and a bulk copy must
          // not land in a peer that has already exited)
          if (!SPLIT || j < T) write_operand((i + 1) & 1);
          if (st_states && j < T) store_block_state(j);
        }
        if (warp == W0) TR(3, i, 5);
      }
    }
    if (st_states && warp == W0 && lane == 0) tma_store_wait_all0();
  } else if (warp == WC && L::CW) {
    // ------------------------------------------------------------- V~ copy warp
    // V~_j = c . V_j (c_t = lam^(r-1-t), rev: lam^(t+1)), the fold operand of dKV_j. Off
    // the state warps, whose state update of block j-1 then overlaps this copy.
    for (int j = 0; j < T; ++j) {
      const int s = j % NS, kt = j % KTS;
      mbar_wait(&bars[L::B_FULL + s], (j / NS) & 1);
      const BlkRec rc = recs[j & 7];
      const int r = min(BT, N - rc.blk * BT);
      if (j >= KTS) mbar_wait(&bars[L::B_KTFREE + kt], ((j / KTS) - 1) & 1);
#pragma unroll 1
      for (int m = 0; m < BT / 32; ++m) {
        const int row = m * 32 + lane;
        const float c = REV ? lam_pow(rc.l2, row + 1) : (row < r ? lam_pow(rc.l2, r - 1 - row) : 0.f);
        scale_row_copy<64>(smem + offv + s * L::V_BYTES, smem + L::OFF_KT + kt * L::V_BYTES, row, c);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[L::B_KTREADY + kt]);
    }
  }
  tc_fence_before();
  if (CL) cluster_sync();  // no remote arrivals / multicasts may target an exited CTA
  else __syncthreads();
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
// (make_tmap_bf16 is declared in la2_kernels.h)
int tma_encoder_ready() { return get_encode(); }
// Tensor maps depend only on (address, shape, box), so they are cached per host thread
// (a map for the same address and shape is valid whatever tensor now lives there).
static int make_tmap(CUtensorMap* m, const void* ptr, int cols, int N, int BH, int box_rows = BT,
                     long long head_stride = 0, long long row_pitch = 0, int box_cols = 64) {
  struct Entry {
    const void* ptr;
    int cols, N, BH, box, boxc;
    long long ld, rp;
    CUtensorMap map;
  };
  static thread_local Entry cache[32];
  static thread_local int next = 0;
  for (const Entry& e : cache) {
    if (e.ptr == ptr && e.cols == cols && e.N == N && e.BH == BH && e.box == box_rows &&
        e.boxc == box_cols && e.ld == head_stride && e.rp == row_pitch && ptr) {
      *m = e.map;
      return 0;
    }
  }
  const int rc = make_tmap_bf16(m, ptr, cols, N, BH, box_rows, head_stride, row_pitch, box_cols);
  if (rc == 0) {
    Entry& e = cache[next];
    next = (next + 1) & 31;
    e.ptr = ptr; e.cols = cols; e.N = N; e.BH = BH; e.box = box_rows; e.boxc = box_cols; e.ld = head_stride;
    e.rp = row_pitch;
    e.map = *m;
  }
  return rc;
}
// L2 sector promotion of the TMA loads (development knob LA2_L2PROMO: 0 none, 1 64 B,
// 2 128 B, 3 256 B = default)
static CUtensorMapL2promotion l2_promotion() {
  static const int v = [] {
    const char* e = std::getenv("LA2_L2PROMO");
    return e ? std::atoi(e) : 3;
  }();
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}
int make_tmap_bf16(CUtensorMap* m, const void* ptr, int cols, int N, int BH, int box_rows,
                   long long head_stride, long long row_pitch, int box_cols) {
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(N),
                        static_cast<cuuint64_t>(BH)};
  const cuuint64_t rp = row_pitch > 0 ? static_cast<cuuint64_t>(row_pitch) : static_cast<cuuint64_t>(cols);
  const cuuint64_t ld = head_stride > 0 ? static_cast<cuuint64_t>(head_stride)
                                        : rp * static_cast<cuuint64_t>(N);
  cuuint64_t strides[2] = {rp * 2, ld * 2};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -static_cast<int>(r) - 1000;
}

// Tuning knobs (la2_set_tuning; defaults overridable by env for development).
static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
static int g_persistent = env_int("LA2_NO_PERSIST", 0) ? 0 : 1;
static int g_prefetch = env_int("LA2_PF", 0);
static int g_l2hint = env_int("LA2_HINT", 0);
static int g_quad = env_int("LA2_NO_QUAD", 0) ? 0 : 1;
static int g_pdl = env_int("LA2_PDL", 4096);
static bool persistent_enabled() { return g_persistent != 0; }
// PDL pays only for short launches (fill/drain dominated): +2-6 % up to N = 4K, but
// -3-7 % for long ones (measured, tools/pdl_ab.py)
static bool pdl_enabled(int N) { return N <= g_pdl; }
static bool quad_enabled() { return g_quad != 0; }
static int prefetch_blocks() { return g_prefetch; }
static int l2_hints() { return g_l2hint; }
static int g_concurrent_bwd = env_int("LA2_CONC_BWD", 16384);
static int g_partition_bwd = env_int("LA2_PARTITION_BWD", 8192);
int tuning_value(int key) {
  switch (key) {
    case LA2_TUNE_PERSISTENT: return g_persistent;
    case LA2_TUNE_PREFETCH: return g_prefetch;
    case LA2_TUNE_L2HINT: return g_l2hint;
    case LA2_TUNE_FUSED_BWD: return g_quad;
    case LA2_TUNE_CONCURRENT_BWD: return g_concurrent_bwd;
    case LA2_TUNE_PARTITION_BWD: return g_partition_bwd;
    case LA2_TUNE_PDL: return g_pdl;
    default: return 0;
  }
}
int set_tuning(int key, int value) {
  switch (key) {
    case LA2_TUNE_CONCURRENT_BWD: g_concurrent_bwd = value; return 0;
    case LA2_TUNE_PARTITION_BWD: g_partition_bwd = value; return 0;
    case LA2_TUNE_PDL: g_pdl = value; return 0;
    case LA2_TUNE_PERSISTENT: g_persistent = value; return 0;
    case LA2_TUNE_PREFETCH: g_prefetch = value; return 0;
    case LA2_TUNE_L2HINT: g_l2hint = value; return 0;
    case LA2_TUNE_FUSED_BWD: g_quad = value; return 0;
    default: return set_error(LA2_ERR_VALUE, "unknown tuning key");
  }
}

template <int DK, bool REV, bool SO, int CM>
static int launch_tc_t(const FArgs& a, cudaStream_t st, const FArgs* a1 = nullptr,
                       const FArgs* a2 = nullptr) {
  using L = TcLayout<DK, SO, CM == 4>;
  auto kern = la2_tc_kernel<DK, REV, SO, CM>;
  cudaError_t e = cudaSuccess;
  static int attr_dev = -1;  // attributes are per device; set once (they cost a driver call)
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  if (attr_dev != cur_dev) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (e != cudaSuccess) return set_cuda_error("cudaFuncSetAttribute(tc)", e);
    attr_dev = cur_dev;
  }
  // maps: q k v o of the pass, and of the sibling pass (CM 2: q1/o1 only; CM 3: all four)
  CUtensorMap mq, mk, mv, mo, mq1, mk1, mv1, mo1;
  const int BH = a.B * a.H;
  const void* ptrs[8] = {a.q, a.k, a.v, a.o, a1 ? a1->q : a.q, a1 ? a1->k : a.k,
                         a1 ? a1->v : a.v, a1 ? a1->o : a.o};
  CUtensorMap* maps[8] = {&mq, &mk, &mv, &mo, &mq1, &mk1, &mv1, &mo1};
  // real operand widths: a q / k narrower than the kernel's DK (or a v / o whose last 64-wide
  // slice is partial) reads as zero beyond its width (TMA out-of-bounds fill) and stores
  // clip there, so any width that is a multiple of 8 runs padded on the tensor cores
  const int cols[8] = {a.dk, a.dk, a.dv, a.dv, a1 ? a1->dk : a.dk, a1 ? a1->dk : a.dk, a1 ? a1->dv : a.dv,
                       a1 ? a1->dv : a.dv};
  for (int t = 0; t < 8; ++t) {
    if (SO && t != 1 && t != 2) continue;
    if (CM != 3 && (t == 5 || t == 6)) continue;
    const long long ld = (t < 4) ? a.ld[t] : (a1 ? a1->ld[t - 4] : a.ld[t - 4]);
    const long long rp = (t < 4) ? a.rp[t] : (a1 ? a1->rp[t - 4] : a.rp[t - 4]);
    const bool omap = (t == 3 || t == 7);  // output: 32-row boxes (32 columns with LA2_WARP_STORE)
    const int rc = make_tmap(maps[t], ptrs[t], cols[t], a.N, BH, omap ? 32 : BT, ld, rp,
                             (omap && LA2_WARP_STORE) ? 32 : 64);
    if (rc != 0) {
      char buf[256];
      std::snprintf(buf, sizeof(buf),
                    "cuTensorMapEncodeTiled failed for operand %d: CUresult %d (ptr=%p cols=%d N=%d BH=%d)",
                    t, -(rc + 1000), ptrs[t], cols[t], a.N, BH);
      return set_error(LA2_ERR_CUDA, buf);
    }
  }
  if (SO) { mq = mk; mo = mv; mq1 = mk; mo1 = mv; }
  if (CM != 3) { mk1 = mk; mv1 = mv; }
  // per-block states (forward store / triple load): tm_v1; the triple's dQ output: tm_k1
  const void* kvb = (CM == 4) ? (a2 ? a2->kv_blocks : nullptr) : a.kv_blocks;
  const bool store_states = (CM == 0 && !REV && !SO && DK == 64 && kvb != nullptr);
  if (CM == 4 || store_states) {
    if (kvb == nullptr) return set_error(LA2_ERR_VALUE, "per-block state buffer is null");
    const int nblk = (a.N + BT - 1) / BT;
    int rc = make_tmap(&mv1, kvb, DK, nblk * DK, BH, DK);
    if (rc == 0 && CM == 4) rc = make_tmap(&mk1, a2->o, DK, a.N, BH, 32, 0, 0, LA2_WARP_STORE ? 32 : 64);
    if (rc != 0) return set_error(LA2_ERR_CUDA, "cuTensorMapEncodeTiled failed for the state blocks / dQ");
  }
  FParams p;
  p.N = a.N;
  p.H = a.H;
  p.decay = a.decay;
  p.kv_in = a.kv_in;
  p.kv_in_T = a.kv_in_T;
  p.kv_out = a.kv_out;
  p.dv_total = a.dv;
  p.kv_in_bhs = a.kv_in_bhs ? a.kv_in_bhs : static_cast<long long>(a.dk) * a.dv;
  p.kv_in_rs = a.kv_in_rs ? a.kv_in_rs : (a.kv_in_T ? a.dk : a.dv);
  if (a.kv_in != nullptr && a.kv_in_T && p.kv_in_rs != DK && p.kv_in_rs != 256)
    return set_error(LA2_ERR_UNSUPPORTED, "transposed state row stride must be the head dim or 256");
  p.kv_out_bhs = a.kv_out_bhs ? a.kv_out_bhs : static_cast<long long>(a.dk) * a.dv;
  p.kv_out_rs = a.kv_out_rs ? a.kv_out_rs : a.dv;
  p.accum = a.accum_o;
  p.store_states = store_states ? 1 : 0;
  p.pf = prefetch_blocks();
  p.hint = l2_hints();
  // persistent schedule: units = independent recurrences (a cluster's pair counts once)
  constexpr int CS = (CM == 3) ? 4 : ((CM == 4) ? 3 : (CM ? 2 : 1));
  p.nsl = (a.dv + DVS - 1) / DVS;
  p.dkr = a.dk;
  p.norm_eps = 0.f;
  p.rstd = nullptr;
  if (a.norm_eps > 0.f) {
    if (!(DK == 64 && !REV && !SO && CM == 0 && a.dv == DVS && a.rstd != nullptr))
      return set_error(LA2_ERR_UNSUPPORTED, "the fused norm epilogue needs a d <= 64, dv = 64 forward");
    p.norm_eps = a.norm_eps;
    p.rstd = a.rstd;
  }
  p.units = (CM == 2 || CM == 4) ? BH : ((CM == 1 || CM == 3) ? BH * p.nsl / 2 : BH * p.nsl);
  p.P = p.units;
  p.ws = nullptr;
  p.flags = nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = L::TOTAL;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int nattr = 0;
  if (CM) {
    attr[nattr].id = cudaLaunchAttributeClusterDimension;
    attr[nattr].val.clusterDim.x = CS;
    attr[nattr].val.clusterDim.y = 1;
    attr[nattr].val.clusterDim.z = 1;
    ++nattr;
  }
  if (pdl_enabled(a.N)) {
    attr[nattr].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[nattr].val.programmaticStreamSerializationAllowed = 1;
    ++nattr;
  }
  cfg.attrs = attr;
  cfg.numAttrs = CM ? 1 : 0;  // cluster only, for the occupancy query below
  if (persistent_enabled()) {
    // co-resident work ranges (one CTA per SM: smem and TMEM are sized for it)
    static int max_ranges = -1;
    if (max_ranges < 0) {
      int n = 0;
      if (CM) {
        cfg.gridDim = dim3(CS);
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
      } else {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TC_THREADS, L::TOTAL) != cudaSuccess)
          per_sm = 0;
        n = sms * per_sm;
      }
      cudaGetLastError();
      max_ranges = n;
    }
    const int cap = (a.max_ranges > 0 && a.max_ranges < max_ranges) ? a.max_ranges : max_ranges;
    if (cap > 0 && p.units > cap) {
      const Workspace w = get_workspace(st);
      if (w.ws != nullptr && w.slots >= cap * CS) {
        p.P = cap;
        p.ws = w.ws;
        p.flags = w.flags;
      }
    }
  }
  cfg.gridDim = dim3(p.P * CS);
  cfg.numAttrs = nattr;
  char kname[48];
  std::snprintf(kname, sizeof(kname), "la2_tc_kernel<%d,%d,%d,%d>", DK, REV ? 1 : 0, SO ? 1 : 0, CM);
  LaunchScope log_scope(st, kname, static_cast<int>(cfg.gridDim.x), CS);
  e = cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, mo, mq1, mk1, mv1, mo1, p);
  if (e != cudaSuccess) return set_cuda_error("la2_tc_kernel launch", e);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error("la2_tc_kernel launch", e);
  return 0;
}

#ifdef LA2_TRACE
extern "C" LA2_API int la2_set_trace(long long* buf) {
  cudaError_t e = cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf));
  if (e != cudaSuccess) return set_cuda_error("la2_set_trace", e);
  return 0;
}
#endif

static bool clusters_enabled() {
  static const bool off = std::getenv("LA2_NO_CLUSTER") != nullptr;
  return !off;
}

int launch_tc(const FArgs& a, cudaStream_t st) {
  if (get_encode() != 0) return set_error(LA2_ERR_CUDA, "cannot resolve cuTensorMapEncodeTiled");
  const bool so = (a.o == nullptr);
  // value-slice pairs share their Q/K tiles through a 2-CTA cluster
  const bool pair = clusters_enabled() && ((a.dv + DVS - 1) / DVS) % 2 == 0;
#define LA2_TC_DISPATCH(DKV)                                                                   \
  if ((a.dk <= 64 ? 64 : 128) == DKV) {                                                      \
    if (so && pair) return a.reverse ? launch_tc_t<DKV, true, true, 1>(a, st)                  \
                                     : launch_tc_t<DKV, false, true, 1>(a, st);                \
    if (so) return a.reverse ? launch_tc_t<DKV, true, true, 0>(a, st)                          \
                             : launch_tc_t<DKV, false, true, 0>(a, st);                        \
    if (pair) return a.reverse ? launch_tc_t<DKV, true, false, 1>(a, st)                       \
                               : launch_tc_t<DKV, false, false, 1>(a, st);                     \
    return a.reverse ? launch_tc_t<DKV, true, false, 0>(a, st)                                 \
                     : launch_tc_t<DKV, false, false, 0>(a, st);                               \
  }
  LA2_TC_DISPATCH(64)
  LA2_TC_DISPATCH(128)
#undef LA2_TC_DISPATCH
  return set_error(LA2_ERR_UNSUPPORTED, "tensor-core path supports head dims up to 128 per pass");
}

// The two reverse scans of the backward pass (dV = F_rev(K, Q, dO), dK = F_rev(V, dO, Q))
// as one 2-CTA cluster per head sharing the Q and dO tiles. d = dv = 64, bf16.
int launch_tc_pair(const FArgs& adv, const FArgs& adk, cudaStream_t st) {
  if (get_encode() != 0) return set_error(LA2_ERR_CUDA, "cannot resolve cuTensorMapEncodeTiled");
  if (!clusters_enabled()) {
    if (int rc = launch_tc_t<64, true, false, 0>(adk, st)) return rc;
    return launch_tc_t<64, true, false, 0>(adv, st);
  }
  return launch_tc_t<64, true, false, 2>(adv, st, &adk);
}

// d = dv = 64 with the forward's per-block states: dV, dK and dQ as one 3-CTA cluster per
// head walking the blocks in reverse (ranks 0-1 the dV / dK scans, rank 2 the stateless dQ).
int launch_tc_triple(const FArgs& adv, const FArgs& adk, const FArgs& adq, cudaStream_t st) {
  if (get_encode() != 0) return set_error(LA2_ERR_CUDA, "cannot resolve cuTensorMapEncodeTiled");
  return launch_tc_t<64, true, false, 4>(adv, st, &adk, &adq);
}

// d = dv = 128: the dV and dK reverse scans as one 4-CTA cluster per unit -- each pass
// a value-slice pair (Q/K multicast inside the pair) -- so the Q and dO tiles both
// passes read are fetched from HBM once and hit L2 for the second pass.
int launch_tc_quad(const FArgs& adv, const FArgs& adk, cudaStream_t st) {
  if (get_encode() != 0) return set_error(LA2_ERR_CUDA, "cannot resolve cuTensorMapEncodeTiled");
  // The quad only pays when each pass alone leaves SMs idle (few heads, e.g. a long
  // single sequence): with >= 148 / 4 pair units per pass two separate persistent
  // launches keep every SM busy and the kernels are not DRAM-bound enough for the
  // saved Q/dO reads to matter (ncu: 1117 us quad vs 2 x 520 us at B=8 H=16 N=16K).
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int pair_units = adv.B * adv.H * (adv.dv / DVS) / 2;
  if (!clusters_enabled() || !quad_enabled() || pair_units * 4 > sms) {
    if (int rc = launch_tc(adk, st)) return rc;
    return launch_tc(adv, st);
  }
  return launch_tc_t<128, true, false, 3>(adv, st, &adk);
}

}  // namespace la2
