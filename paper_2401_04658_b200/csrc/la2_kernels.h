// Internal launcher interface shared by the kernel translation units and the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/la2.h"

namespace la2 {

#ifdef __CUDACC__
// Decay as the kernels use it: lam in (0, 1] (reference.py:42-44), anything else
// (including NaN) becomes NaN so that every output of the launch is NaN -- an invalid
// decay can never produce plausible numbers. The C ABI rejects it up front with
// la2_check_decay (include/la2.h).
__device__ __forceinline__ float checked_decay(float lam) {
  return (lam > 0.f && lam <= 1.f) ? lam : __int_as_float(0x7fc00000);
}
#endif

// Arguments of one "F" pass (see la2_tc.cu header comment).
//   q,k: [B,H,N,dk]   v,o: [B,H,N,dv]   (contiguous; o == nullptr -> state-only pass)
//   kv_in / kv_out: fp32 [B,H,dk,dv] (kv_in_T: kv_in stored [B,H,dv,dk])
struct FArgs {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  const float* decay;
  const float* kv_in;
  int kv_in_T;
  float* kv_out;
  int B, H, N, dk, dv;
  int dtype;
  int reverse;
  int max_ranges = 0;  // persistent schedule: cap on co-resident work ranges (0 = all SMs)
  // elements between consecutive (b, h) rows of q, k, v, o (0 = contiguous N * cols);
  // tensor-core path only (the TMA maps carry the stride)
  long long ld[4] = {0, 0, 0, 0};
  // elements between consecutive tokens of q, k, v, o (0 = the operand's width): column
  // slices of a wider tensor (split-d). Tensor-core path only.
  long long rp[4] = {0, 0, 0, 0};
  // state addressing (0 = contiguous [B,H,dk,dv]): element (r, c) of the pass's state for
  // head bh is at bh * bhs + r * rs + c (kv_in_T: bh * bhs + c * rs + r)
  long long kv_in_bhs = 0, kv_out_bhs = 0;
  int kv_in_rs = 0, kv_out_rs = 0;
  int accum_o = 0;  // add the output into o (TMA reduce-add) instead of storing it
  // per-block bf16 states [B*H][ceil(N/128)][dk][dv] (d = dv = 64): written by a forward
  // (store), read by the backward triple's dQ CTA
  void* kv_blocks = nullptr;
  // per-head RMS norm of the output rows fused into the epilogue (la2_forward_norm)
  float norm_eps = 0.f;
  float* rstd = nullptr;
};

// Kernel-side parameter block (passed by value).
struct FParams {
  int N;
  int H;
  const float* decay;
  const float* kv_in;
  int kv_in_T;
  float* kv_out;
  int dv_total;
  int pf;    // L2 prefetch distance in blocks (2-stage rings)
  int hint;  // L2 cache-policy bits: 1 loads evict_first, 2 prefetch evict_last, 4 stores evict_first
  // persistent schedule (tensor-core kernels): `units` recurrences over P work ranges
  int units, P, nsl;
  float* ws;   // [P * cluster][dk][64] fp32 state handoff between neighbouring ranges
  int* flags;  // [P * cluster] handoff flags (0 = empty), reset by their reader
  // state addressing (see FArgs); resolved to the contiguous defaults by the launcher
  long long kv_in_bhs, kv_out_bhs;
  int kv_in_rs, kv_out_rs;
  int accum;  // output epilogue: TMA reduce-add into o
  int store_states;  // forward (d = 64): write the per-block bf16 states through tm_v1
  int dkr;           // real head dim of the pass (<= the kernel's DK; rows beyond it are padding)
  float norm_eps;    // > 0: per-head RMS norm fused into the output epilogue (d = dv = 64 forward)
  float* rstd;       //   its per-row 1 / rms, [B*H][N]
};

int launch_tc(const FArgs& a, cudaStream_t st);
// dV and dK reverse scans as one 2-CTA cluster per head (shared Q / dO tiles).
int launch_tc_pair(const FArgs& adv, const FArgs& adk, cudaStream_t st);
// d = dv = 64 with stored per-block states (adq.kv_blocks): dV, dK and a stateless dQ pass
// as one 3-CTA cluster per head.
int launch_tc_triple(const FArgs& adv, const FArgs& adk, const FArgs& adq, cudaStream_t st);
// d = dv = 128: dV and dK reverse scans as one 4-CTA cluster per unit (two value-slice pairs).
int launch_tc_quad(const FArgs& adv, const FArgs& adk, cudaStream_t st);
// TMA tensor map of a [BH][N][cols] bf16 tensor, box (64 cols, box_rows, 1), 128B swizzle;
// head_stride = elements between (b, h) rows (0: N * cols).
int tma_encoder_ready();
int make_tmap_bf16(CUtensorMap* m, const void* ptr, int cols, int N, int BH, int box_rows, long long head_stride = 0,
                   long long row_pitch = 0, int box_cols = 64);
int launch_simt(const FArgs& a, cudaStream_t st);
// fp64 F pass (la2_f64.cu): one launch of the block recurrence (reverse = F_rev) and
// the fp64 decode (ntok tokens per call)
int launch_f64(const double* q, const double* k, const double* v, double* o, const double* decay,
               const double* kv_in, int kv_in_T, double* kv_out, int B, int H, int N, int dk, int dv,
               int reverse, int block, cudaStream_t st);
int launch_decode_f64(const double* q, const double* k, const double* v, const double* decay,
                      double* state, double* o, int B, int H, int d, int dv, int ntok, cudaStream_t st);
// Norm(.) of NormAttention (la2_norm.cu): rows of [B,H,N,dv] normalised per head
// (group = 1) or over all heads of a token (group = H); rstd [B*H/group*N]
int launch_rmsnorm_fwd(const void* x, void* y, float* rstd, int B, int H, int N, int dv, int group, float eps,
                       int dtype, cudaStream_t st);
int launch_rmsnorm_bwd(const void* dy, const void* y, const float* rstd, void* dx, int B, int H, int N, int dv,
                       int group, int dtype, cudaStream_t st);
int launch_decode(const void* q, const void* k, const void* v, const float* decay, float* state,
                  void* o, int B, int H, int d, int dv, int ntok, int dtype, cudaStream_t st);
int launch_state_scan(const float* chunk_states, const float* decay, const float* init,
                      float* prefix, int G, int BH, int H, int dk, int dv, const int* lens,
                      int reverse, cudaStream_t st);

// Per-(device, stream) handoff workspace for the persistent schedule; nullptr when it
// cannot be allocated (e.g. first use inside a CUDA graph capture).
struct Workspace {
  float* ws;
  int* flags;
  int slots;
};
Workspace get_workspace(cudaStream_t st);

// Launch log (la2_launch_log, include/la2.h): when enabled, every kernel launch of the
// library is bracketed by CUDA events recorded on the stream it is launched on. A scope
// object around the launch; free when the log is off (one relaxed load).
struct LaunchScope {
  int slot = -1;
  cudaStream_t st = nullptr;
  LaunchScope(cudaStream_t s, const char* kernel, int grid, int cluster);
  ~LaunchScope();
};

int set_tuning(int key, int value);
int tuning_value(int key);
int set_error(int code, const char* msg);
int set_cuda_error(const char* where, cudaError_t e);

}  // namespace la2
