// Internal launcher interface shared by the kernel translation units and the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/la2.h"

namespace la2 {

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
};

int launch_tc(const FArgs& a, cudaStream_t st);
// dV and dK reverse scans as one 2-CTA cluster per head (shared Q / dO tiles).
int launch_tc_pair(const FArgs& adv, const FArgs& adk, cudaStream_t st);
// d = dv = 128: dV and dK reverse scans as one 4-CTA cluster per unit (two value-slice pairs).
int launch_tc_quad(const FArgs& adv, const FArgs& adk, cudaStream_t st);
// Fused reverse scan of the backward pass (dK and dV together), d = dv = 64, bf16.
int launch_g(const void* q, const void* k, const void* v, const void* dout, void* dk, void* dv,
             const float* decay, const float* dkv_in, float* dkv_out, int B, int H, int N,
             cudaStream_t st);
// TMA tensor map of a [BH][N][cols] bf16 tensor, box (64 cols, box_rows, 1), 128B swizzle;
// head_stride = elements between (b, h) rows (0: N * cols).
int tma_encoder_ready();
int make_tmap_bf16(CUtensorMap* m, const void* ptr, int cols, int N, int BH, int box_rows, long long head_stride = 0);
int launch_simt(const FArgs& a, cudaStream_t st);
int launch_decode(const void* q, const void* k, const void* v, const float* decay, float* state,
                  void* o, int B, int H, int d, int dv, int dtype, cudaStream_t st);
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

int set_tuning(int key, int value);
int tuning_value(int key);
int set_error(int code, const char* msg);
int set_cuda_error(const char* where, cudaError_t e);

}  // namespace la2
