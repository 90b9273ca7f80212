// C ABI entry points (include/la2.h): argument validation with the reference's
// error semantics (pkg/src/tila/reference.py:42-74, kernel.py:68-70), kernel
// selection, and the backward pass expressed as three F passes.
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <mutex>
#include <vector>

#include "la2_kernels.h"

namespace la2 {

static thread_local char g_err[512] = "";

int set_error(int code, const char* msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}
int set_cuda_error(const char* where, cudaError_t e) {
  std::snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
  return LA2_ERR_CUDA;
}

// Handoff workspace of the persistent schedule, one per (device, stream) so that
// kernels on different streams never share flags. Allocated once, zeroed, never freed;
// the flags return to zero at the end of every launch (each is consumed by its reader).
static size_t workspace_state_bytes(int slots) {  // d x 64 fp32 state per slot, d <= 128
  return static_cast<size_t>(slots) * 128 * 64 * sizeof(float);
}

Workspace get_workspace(cudaStream_t st) {
  struct Entry {
    int dev;
    cudaStream_t st;
    Workspace w;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return Workspace{nullptr, nullptr, 0};
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& e : cache)
    if (e.dev == dev && e.st == st) return e.w;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess) {
    cudaGetLastError();
    return Workspace{nullptr, nullptr, 0};
  }
  const bool capturing = (cap != cudaStreamCaptureStatusNone);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int slots = sms;  // at most one CTA per SM
  const size_t state_bytes = workspace_state_bytes(slots);
  void* buf = nullptr;
  // First use of a stream inside CUDA-graph capture: allocate and zero the workspace
  // outside the capture (relaxed capture mode for this thread, a private stream for the
  // zeroing), so captured launches keep the persistent schedule -- without it they run
  // one CTA per recurrence, up to 1.7x slower (tools/graphed_step.py).
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  if (capturing) cudaThreadExchangeStreamCaptureMode(&mode);
  cudaStream_t zs = st;
  bool ok = cudaMalloc(&buf, state_bytes + slots * sizeof(int)) == cudaSuccess;
  int* flags = ok ? reinterpret_cast<int*>(static_cast<char*>(buf) + state_bytes) : nullptr;
  if (ok && capturing) ok = cudaStreamCreateWithFlags(&zs, cudaStreamNonBlocking) == cudaSuccess;
  // zeroed on the stream that will use it (a legacy-stream memset would not be ordered
  // before kernels on non-blocking streams), or on the private stream, waited for
  if (ok) ok = cudaMemsetAsync(flags, 0, slots * sizeof(int), zs) == cudaSuccess;
  if (ok && capturing) {
    ok = cudaStreamSynchronize(zs) == cudaSuccess;
    cudaStreamDestroy(zs);
  }
  if (capturing) cudaThreadExchangeStreamCaptureMode(&mode);
  if (!ok) {
    cudaGetLastError();
    if (buf) cudaFree(buf);
    return Workspace{nullptr, nullptr, 0};
  }
  Workspace w{static_cast<float*>(buf), flags, slots};
  cache.push_back(Entry{dev, st, w});
  return w;
}

// ------------------------------------------------------------------ launch log
struct LogRec {
  char kernel[48];
  int grid, cluster;
  cudaEvent_t t0, t1;
};
static std::atomic<int> g_log_on{0};
static std::mutex g_log_mu;
static std::vector<LogRec> g_log;  // events preallocated by la2_launch_log
static int g_log_used = 0, g_log_dropped = 0;

LaunchScope::LaunchScope(cudaStream_t s, const char* kernel, int grid, int cluster) {
  if (!g_log_on.load(std::memory_order_relaxed)) return;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return;  // events inside a captured graph would time the capture, not the replay
  }
  std::lock_guard<std::mutex> lock(g_log_mu);
  if (g_log_used >= static_cast<int>(g_log.size())) {
    ++g_log_dropped;
    return;
  }
  LogRec& r = g_log[g_log_used];
  std::snprintf(r.kernel, sizeof(r.kernel), "%s", kernel);
  r.grid = grid;
  r.cluster = cluster;
  if (cudaEventRecord(r.t0, s) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  slot = g_log_used++;
  st = s;
}

LaunchScope::~LaunchScope() {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lock(g_log_mu);
  if (slot < static_cast<int>(g_log.size()) && cudaEventRecord(g_log[slot].t1, st) != cudaSuccess)
    cudaGetLastError();
}

// Per-device side stream (non-blocking) + fork/join events for the concurrent dQ pass.
// Fork/join through events is also valid inside CUDA graph capture.
// The record/wait pair of each fork and join runs under the side stream's mutex, so two
// host threads cannot interleave their records on the shared events (thread B's fork
// record landing between thread A's record and wait would make A's side work wait on B's
// stream instead of its own).
struct SideStream {
  cudaStream_t s;
  cudaEvent_t fork, join;
  std::mutex mu;
};
static SideStream* side_stream(cudaStream_t caller) {
  static std::mutex mu;
  static SideStream per_dev[16];
  static bool made[16] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 16) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!made[dev]) {
    // never create inside a graph capture (it would invalidate the capture): the first
    // captured backward simply runs serially
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(caller, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return nullptr;
    }
    SideStream& x = per_dev[dev];
    if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    made[dev] = true;
  }
  return &per_dev[dev];
}
static bool fork_side(SideStream* side, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(side->mu);
  if (cudaEventRecord(side->fork, st) == cudaSuccess &&
      cudaStreamWaitEvent(side->s, side->fork, 0) == cudaSuccess)
    return true;
  cudaGetLastError();
  return false;
}
static int join_side(SideStream* side, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(side->mu);
  cudaError_t e = cudaEventRecord(side->join, side->s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, side->join, 0);
  if (e != cudaSuccess) return set_cuda_error("side-stream join", e);
  return 0;
}

// bf16 widths that are multiples of 8 (16-byte TMA row pitch) up to 256 run on the tensor
// cores: d <= 64 / <= 128 on the DK = 64 / 128 kernel (narrower operands zero-padded by the
// TMA unit), d in (128, 256] as split-d; dv in 64-wide value slices, the last one partial.
static bool tc_eligible(int dtype, int dk, int dv) {
  return dtype == LA2_BF16 && dk >= 8 && dk <= 256 && dk % 8 == 0 && dv >= 8 && dv <= 256 && dv % 8 == 0;
}

// Split-d: an F pass with a 256-wide q/k is the sum of two 128-wide passes over the column
// halves of q and k, because the scores and the state are linear in the shared dimension:
//   q_t . k_s = q_t[:128] . k_s[:128] + q_t[128:] . k_s[128:]   (mask and decay are
//   elementwise, so ((Q K^T) * M) V splits the same way), and the state
//   sum_s lam^(..) k_s^T v_s splits by rows: rows [0,128) come from the first half only.
// The first pass stores o, the second adds into it (TMA reduce-add); each pass reads and
// writes its own 128 rows of kv_in / kv_out. Column halves are read in place (the TMA maps
// take the row pitch), so no operand is copied.
static int run_f_split_d(const FArgs& a, cudaStream_t st) {
  const long long dk = a.dk, dv = a.dv;
  for (int h = 0; h < 2; ++h) {
    FArgs b = a;
    b.dk = h == 0 ? 128 : static_cast<int>(dk) - 128;  // the second half may be narrower (padded)
    b.q = static_cast<const uint16_t*>(a.q) + 128 * h;
    b.k = static_cast<const uint16_t*>(a.k) + 128 * h;
    for (int t = 0; t < 2; ++t) b.rp[t] = a.rp[t] ? a.rp[t] : dk;
    if (a.kv_in != nullptr) {
      b.kv_in_bhs = a.kv_in_bhs ? a.kv_in_bhs : dk * dv;
      if (!a.kv_in_T) {
        b.kv_in_rs = a.kv_in_rs ? a.kv_in_rs : static_cast<int>(dv);
        b.kv_in = a.kv_in + static_cast<long long>(128) * h * b.kv_in_rs;
      } else {  // stored [dv][dk]: the pass's rows are the stored columns
        b.kv_in_rs = a.kv_in_rs ? a.kv_in_rs : static_cast<int>(dk);
        b.kv_in = a.kv_in + 128 * h;
      }
    }
    if (a.kv_out != nullptr) {
      b.kv_out_bhs = a.kv_out_bhs ? a.kv_out_bhs : dk * dv;
      b.kv_out_rs = a.kv_out_rs ? a.kv_out_rs : static_cast<int>(dv);
      b.kv_out = a.kv_out + static_cast<long long>(128) * h * b.kv_out_rs;
    }
    b.accum_o = (h == 1 && a.o != nullptr) ? 1 : a.accum_o;
    if (int rc = launch_tc(b, st)) return rc;
  }
  return 0;
}

static int run_f(const FArgs& a, cudaStream_t st) {
  // a transposed carried state is read with compile-time row strides (the kernel's DK or
  // 256); a padded head dim with one runs that pass on the SIMT kernel
  const bool padded_T = a.kv_in != nullptr && a.kv_in_T && a.dk != 64 && a.dk != 128 && a.dk != 256;
  if (tc_eligible(a.dtype, a.dk, a.dv) && !padded_T) return a.dk > 128 ? run_f_split_d(a, st) : launch_tc(a, st);
  return launch_simt(a, st);
}

static int check_common(int B, int H, int N, int d, int dv, int dtype, const float* decay) {
  if (B < 1 || H < 1) return set_error(LA2_ERR_VALUE, "B and H must be >= 1");
  if (N < 1) return set_error(LA2_ERR_VALUE, "sequence length N must be >= 1");
  if (d < 1 || dv < 1) return set_error(LA2_ERR_VALUE, "d and dv must be >= 1");
  if (dtype != LA2_BF16 && dtype != LA2_FP32)
    return set_error(LA2_ERR_UNSUPPORTED, "dtype must be LA2_BF16 or LA2_FP32");
  if (decay == nullptr) return set_error(LA2_ERR_VALUE, "decay pointer is null");
  if (!tc_eligible(dtype, d, dv) && (d > 256 || dv > 256)) {
    char buf[160];
    std::snprintf(buf, sizeof(buf),
                  "unsupported shape d=%d dv=%d for dtype %s (bf16 tensor-core path: d, dv "
                  "multiples of 8 up to 256; otherwise d, dv <= 256)",
                  d, dv, dtype == LA2_BF16 ? "bf16" : "fp32");
    return set_error(LA2_ERR_UNSUPPORTED, buf);
  }
  return 0;
}

// Make this library's runtime current on the device that owns the caller's data.
// The library links its own static cudart, so torch's current device does not carry
// over. (The device comes from the pointer rather than the stream: stream queries
// are not permitted while the caller captures a CUDA graph.)
static int bind_device(void* stream, const void* ptr) {
  (void)stream;
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) return set_cuda_error("cudaPointerGetAttributes", e);
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return set_error(LA2_ERR_VALUE, "tensor pointer is not device memory");
  // Always (re)bind: besides selecting the device this makes the primary context
  // current on the calling thread, which the driver-API tensor-map encoder needs (the
  // autograd engine runs the backward on its own thread).
  e = cudaSetDevice(at.device);
  if (e != cudaSuccess) return set_cuda_error("cudaSetDevice", e);
  return 0;
}

}  // namespace la2

using namespace la2;

extern "C" {

int la2_version(void) { return 100; }

const char* la2_last_error(void) { return g_err; }

int la2_set_tuning(int key, int value) {
  g_err[0] = 0;
  return set_tuning(key, value);
}

long long la2_workspace_bytes(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return static_cast<long long>(la2::workspace_state_bytes(sms) + sms * sizeof(int));
}

int la2_forward(const void* q, const void* k, const void* v, const float* decay, void* o,
                const float* kv_in, float* kv_out, int B, int H, int N, int d, int dv, int dtype,
                void* stream) {
  g_err[0] = 0;
  if (int rc = check_common(B, H, N, d, dv, dtype, decay)) return rc;
  if (!q || !k || !v || !o) return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (int rc = bind_device(stream, q)) return rc;
  FArgs a{q, k, v, o, decay, kv_in, 0, kv_out, B, H, N, d, dv, dtype, 0};
  return run_f(a, static_cast<cudaStream_t>(stream));
}

int la2_forward_strided(const void* q, const void* k, const void* v, const float* decay, void* o,
                        const float* kv_in, float* kv_out, int B, int H, int N, int d, int dv,
                        int dtype, long long ldq, long long ldk, long long ldv, void* stream) {
  g_err[0] = 0;
  if (int rc = check_common(B, H, N, d, dv, dtype, decay)) return rc;
  if (!q || !k || !v || !o) return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (!tc_eligible(dtype, d, dv))
    return set_error(LA2_ERR_UNSUPPORTED,
                     "strided inputs need the tensor-core path (bf16, d and dv multiples of 8 up to 256)");
  const long long need[3] = {1LL * N * d, 1LL * N * d, 1LL * N * dv};
  const long long ld[3] = {ldq, ldk, ldv};
  for (int t = 0; t < 3; ++t)
    if (ld[t] < need[t] || (ld[t] * 2) % 16 != 0)
      return set_error(LA2_ERR_VALUE,
                       "head stride must be >= N * cols elements and a multiple of 8 (16 bytes)");
  if (int rc = bind_device(stream, q)) return rc;
  FArgs a{q, k, v, o, decay, kv_in, 0, kv_out, B, H, N, d, dv, dtype, 0};
  a.ld[0] = ldq;
  a.ld[1] = ldk;
  a.ld[2] = ldv;
  return run_f(a, static_cast<cudaStream_t>(stream));
}

static int backward_reverse(const void* q, const void* k, const void* v, const void* dout,
                            const float* decay, void* dk, void* dv, const float* dkv_in,
                            float* dkv_out, int B, int H, int N, int d, int dvd, int dtype,
                            cudaStream_t st, int max_ranges = 0, const long long* ld = nullptr);

// (b, h) row strides of the operands of one F pass, by role, from the caller's
// q / k / v / dout strides (nullptr: all contiguous)
static void set_ld(FArgs& a, const long long* ld, int iq, int ik, int iv) {
  if (ld == nullptr) return;
  a.ld[0] = ld[iq];
  a.ld[1] = ld[ik];
  a.ld[2] = ld[iv];
}

static int backward_impl(const void* q, const void* k, const void* v, const void* dout,
                         const float* decay, void* dq, void* dk, void* dv, const float* kv_in,
                         const float* dkv_in, float* dkv_out, int B, int H, int N, int d, int dvd,
                         int dtype, void* stream, const long long* ld);

int la2_backward(const void* q, const void* k, const void* v, const void* dout, const float* decay,
                 void* dq, void* dk, void* dv, const float* kv_in, const float* dkv_in,
                 float* dkv_out, int B, int H, int N, int d, int dvd, int dtype, void* stream) {
  return backward_impl(q, k, v, dout, decay, dq, dk, dv, kv_in, dkv_in, dkv_out, B, H, N, d, dvd,
                       dtype, stream, nullptr);
}

int la2_backward_strided(const void* q, const void* k, const void* v, const void* dout,
                         const float* decay, void* dq, void* dk, void* dv, const float* kv_in,
                         const float* dkv_in, float* dkv_out, int B, int H, int N, int d, int dvd,
                         int dtype, long long ldq, long long ldk, long long ldv, long long lddo,
                         void* stream) {
  g_err[0] = 0;
  if (!tc_eligible(dtype, d, dvd))
    return set_error(LA2_ERR_UNSUPPORTED,
                     "strided inputs need the tensor-core path (bf16, d and dv multiples of 8 up to 256)");
  const long long ld[4] = {ldq, ldk, ldv, lddo};
  const long long need[4] = {1LL * N * d, 1LL * N * d, 1LL * N * dvd, 1LL * N * dvd};
  for (int t = 0; t < 4; ++t)
    if (ld[t] < need[t] || (ld[t] * 2) % 16 != 0)
      return set_error(LA2_ERR_VALUE,
                       "head stride must be >= N * cols elements and a multiple of 8 (16 bytes)");
  return backward_impl(q, k, v, dout, decay, dq, dk, dv, kv_in, dkv_in, dkv_out, B, H, N, d, dvd,
                       dtype, stream, ld);
}

static int backward_impl(const void* q, const void* k, const void* v, const void* dout,
                         const float* decay, void* dq, void* dk, void* dv, const float* kv_in,
                         const float* dkv_in, float* dkv_out, int B, int H, int N, int d, int dvd,
                         int dtype, void* stream, const long long* ld) {
  g_err[0] = 0;
  if (int rc = check_common(B, H, N, d, dvd, dtype, decay)) return rc;
  if (int rc = check_common(B, H, N, dvd, d, dtype, decay)) return rc;
  if (!q || !k || !v || !dout || !dq || !dk || !dv)
    return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (int rc = bind_device(stream, q)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // dQ = F(dO, V, K): forward scan, state KV^T  (tiled_backward sweep 1, kernel.py:184-204)
  // It shares no output with the dK/dV scans, so for short sequences (where each launch
  // is dominated by its fill / drain) it runs on a forked side stream concurrently.
  FArgs aq{dout, v, k, dq, decay, kv_in, 1, nullptr, B, H, N, dvd, d, dtype, 0};
  set_ld(aq, ld, 3, 2, 1);  // dO, V, K
  // d = 64 with enough heads: the dQ scan (128 of 148 SMs at B*H = 128) and the dK/dV pair
  // are both bound by the per-SM block rate and dominated by fill/drain for short
  // sequences, so they run concurrently on disjoint SM partitions sized to the work
  // (dQ = 1 scan, the pair = 2 scans): the pair gets 2/3 of the SMs as clusters and is
  // launched first, the dQ scan takes the rest; both keep the persistent schedule inside
  // their partition. Measured (B=8 H=16): -11 % at N=1K, -2.5 % at 16K, +3 % at 64K, so
  // it is used up to N = LA2_TUNE_PARTITION_BWD (default 8192).
  if (dtype == LA2_BF16 && d == 64 && dvd == 64 && N <= tuning_value(LA2_TUNE_PARTITION_BWD)) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int pair_cap = (2 * sms / 3) / 2, dq_cap = sms - 2 * pair_cap;
    SideStream* ps = (B * H > pair_cap && B * H > dq_cap) ? side_stream(st) : nullptr;
    if (ps != nullptr && fork_side(ps, st)) {
      const int rc = backward_reverse(q, k, v, dout, decay, dk, dv, dkv_in, dkv_out, B, H, N, d,
                                      dvd, dtype, st, pair_cap, ld);
      aq.max_ranges = dq_cap;
      const int rq = rc ? 0 : run_f(aq, ps->s);
      const int jr = join_side(ps, st);
      return rc ? rc : (rq ? rq : jr);
    }
    cudaGetLastError();
  }
  SideStream* side = (tuning_value(LA2_TUNE_CONCURRENT_BWD) > 0 &&
                      N <= tuning_value(LA2_TUNE_CONCURRENT_BWD)) ? side_stream(st) : nullptr;
  if (side != nullptr && !fork_side(side, st)) side = nullptr;
  if (int rc = run_f(aq, side ? side->s : st)) {
    if (side) join_side(side, st);
    return rc;
  }
  const int rc = backward_reverse(q, k, v, dout, decay, dk, dv, dkv_in, dkv_out, B, H, N, d, dvd, dtype, st,
                                  0, ld);
  if (side) {
    if (int jr = join_side(side, st)) return rc ? rc : jr;
  }
  return rc;
}

// dK and dV: the reverse sweep of tiled_backward (kernel.py:207-231).
static int backward_reverse(const void* q, const void* k, const void* v, const void* dout,
                            const float* decay, void* dk, void* dv, const float* dkv_in,
                            float* dkv_out, int B, int H, int N, int d, int dvd, int dtype,
                            cudaStream_t st, int max_ranges, const long long* ld) {
  if (dtype == LA2_BF16 && d == 64 && dvd == 64) {
    // dV and dK scans as one cluster pair sharing the Q and dO tiles (sweep 2, kernel.py:207-231)
    FArgs av{k, q, dout, dv, decay, dkv_in, 0, dkv_out, B, H, N, d, dvd, dtype, 1, max_ranges};
    FArgs ak{v, dout, q, dk, decay, dkv_in, 1, nullptr, B, H, N, dvd, d, dtype, 1, max_ranges};
    set_ld(av, ld, 1, 0, 3);  // K, Q, dO
    set_ld(ak, ld, 2, 3, 0);  // V, dO, Q
    return launch_tc_pair(av, ak, st);
  }
  if (dtype == LA2_BF16 && d == 128 && dvd == 128) {
    // dV and dK scans as one 4-CTA cluster per unit (sweep 2, kernel.py:207-231)
    FArgs av{k, q, dout, dv, decay, dkv_in, 0, dkv_out, B, H, N, d, dvd, dtype, 1};
    FArgs ak{v, dout, q, dk, decay, dkv_in, 1, nullptr, B, H, N, dvd, d, dtype, 1};
    set_ld(av, ld, 1, 0, 3);
    set_ld(ak, ld, 2, 3, 0);
    return launch_tc_quad(av, ak, st);
  }
  // dK = F_rev(V, dO, Q): reverse scan, state dKV^T  (sweep 2, kernel.py:207-216)
  FArgs ak{v, dout, q, dk, decay, dkv_in, 1, nullptr, B, H, N, dvd, d, dtype, 1};
  set_ld(ak, ld, 2, 3, 0);
  if (int rc = run_f(ak, st)) return rc;
  // dV = F_rev(K, Q, dO): reverse scan, state dKV   (sweep 2, kernel.py:217-231)
  FArgs av{k, q, dout, dv, decay, dkv_in, 0, dkv_out, B, H, N, d, dvd, dtype, 1};
  set_ld(av, ld, 1, 0, 3);
  return run_f(av, st);
}

long long la2_state_blocks_bytes(int B, int H, int N, int d, int dv) {
  if (B < 1 || H < 1 || N < 1 || d < 1 || dv < 1) return 0;
  return 2LL * B * H * ((N + 127) / 128) * d * dv;
}

static bool states_eligible(int dtype, int d, int dv) { return dtype == LA2_BF16 && d == 64 && dv == 64; }

int la2_forward_states(const void* q, const void* k, const void* v, const float* decay, void* o,
                       const float* kv_in, float* kv_out, void* kv_blocks, int B, int H, int N,
                       int d, int dv, int dtype, void* stream) {
  g_err[0] = 0;
  if (int rc = check_common(B, H, N, d, dv, dtype, decay)) return rc;
  if (!states_eligible(dtype, d, dv))
    return set_error(LA2_ERR_UNSUPPORTED, "stored per-block states need bf16 with d = dv = 64");
  if (!q || !k || !v || !o || !kv_blocks) return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (int rc = bind_device(stream, q)) return rc;
  FArgs a{q, k, v, o, decay, kv_in, 0, kv_out, B, H, N, d, dv, dtype, 0};
  a.kv_blocks = kv_blocks;
  return launch_tc(a, static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- Norm(.) (la2_norm.cu)
static int check_norm(int B, int H, int N, int dv, int group, int dtype) {
  if (B < 1 || H < 1 || N < 1 || dv < 1) return set_error(LA2_ERR_VALUE, "bad shape");
  if (dv > 1024) return set_error(LA2_ERR_UNSUPPORTED, "norm rows must have dv <= 1024");
  if (group != 1 && group != H) return set_error(LA2_ERR_VALUE, "norm group must be 1 (per head) or H (all heads)");
  if (dtype != LA2_BF16 && dtype != LA2_FP32) return set_error(LA2_ERR_UNSUPPORTED, "dtype must be LA2_BF16 or LA2_FP32");
  return 0;
}

int la2_rmsnorm_forward(const void* x, void* y, float* rstd, int B, int H, int N, int dv, int group, float eps,
                        int dtype, void* stream) {
  g_err[0] = 0;
  if (int rc = check_norm(B, H, N, dv, group, dtype)) return rc;
  if (!x || !y || !rstd) return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (!(eps > 0.f)) return set_error(LA2_ERR_VALUE, "eps must be > 0");
  if (int rc = bind_device(stream, x)) return rc;
  return launch_rmsnorm_fwd(x, y, rstd, B, H, N, dv, group, eps, dtype, static_cast<cudaStream_t>(stream));
}

int la2_rmsnorm_backward(const void* dy, const void* y, const float* rstd, void* dx, int B, int H, int N, int dv,
                         int group, int dtype, void* stream) {
  g_err[0] = 0;
  if (int rc = check_norm(B, H, N, dv, group, dtype)) return rc;
  if (!dy || !y || !rstd || !dx) return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (int rc = bind_device(stream, dy)) return rc;
  return launch_rmsnorm_bwd(dy, y, rstd, dx, B, H, N, dv, group, dtype, static_cast<cudaStream_t>(stream));
}

int la2_forward_norm(const void* q, const void* k, const void* v, const float* decay, void* o,
                     const float* kv_in, float* kv_out, void* kv_blocks, float* rstd, float eps, int group,
                     int B, int H, int N, int d, int dv, int dtype, void* stream) {
  g_err[0] = 0;
  if (int rc = check_common(B, H, N, d, dv, dtype, decay)) return rc;
  if (int rc = check_norm(B, H, N, dv, group, dtype)) return rc;
  if (!q || !k || !v || !o || !rstd) return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (!(eps > 0.f)) return set_error(LA2_ERR_VALUE, "eps must be > 0");
  if (kv_blocks != nullptr && !states_eligible(dtype, d, dv))
    return set_error(LA2_ERR_UNSUPPORTED, "stored per-block states need bf16 with d = dv = 64");
  if (int rc = bind_device(stream, q)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  FArgs a{q, k, v, o, decay, kv_in, 0, kv_out, B, H, N, d, dv, dtype, 0};
  a.kv_blocks = kv_blocks;
  // per-head norm of a d <= 64, dv = 64 bf16 forward: fused into the tensor-core epilogue
  if (group == 1 && tc_eligible(dtype, d, dv) && d <= 64 && dv == 64) {
    a.norm_eps = eps;
    a.rstd = rstd;
    return launch_tc(a, st);
  }
  if (int rc = (kv_blocks != nullptr) ? launch_tc(a, st) : run_f(a, st)) return rc;
  return launch_rmsnorm_fwd(o, o, rstd, B, H, N, dv, group, eps, dtype, st);
}

int la2_backward_states(const void* q, const void* k, const void* v, const void* dout,
                        const float* decay, const void* kv_blocks, void* dq, void* dk, void* dv,
                        const float* dkv_in, float* dkv_out, int B, int H, int N, int d, int dvd,
                        int dtype, void* stream) {
  g_err[0] = 0;
  if (int rc = check_common(B, H, N, d, dvd, dtype, decay)) return rc;
  if (!states_eligible(dtype, d, dvd))
    return set_error(LA2_ERR_UNSUPPORTED, "stored per-block states need bf16 with d = dv = 64");
  if (!q || !k || !v || !dout || !dq || !dk || !dv || !kv_blocks)
    return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (int rc = bind_device(stream, q)) return rc;
  // dV = F_rev(K, Q, dO) (state dKV), dK = F_rev(V, dO, Q) (state dKV^T): the reverse
  // sweep of kernel.py:207-231; dQ = F(dO, V, K) from the stored KV_{i-1}: sweep 1
  // (kernel.py:184-204) without replaying the recurrence.
  FArgs av{k, q, dout, dv, decay, dkv_in, 0, dkv_out, B, H, N, d, dvd, dtype, 1};
  FArgs ak{v, dout, q, dk, decay, dkv_in, 1, nullptr, B, H, N, dvd, d, dtype, 1};
  FArgs aq{dout, v, k, dq, decay, nullptr, 0, nullptr, B, H, N, dvd, d, dtype, 0};
  aq.kv_blocks = const_cast<void*>(kv_blocks);
  return launch_tc_triple(av, ak, aq, static_cast<cudaStream_t>(stream));
}

int la2_chunk_state(const void* k, const void* v, const float* decay, float* s_out, int B, int H,
                    int N, int d, int dv, int dtype, void* stream) {
  g_err[0] = 0;
  if (int rc = check_common(B, H, N, d, dv, dtype, decay)) return rc;
  if (!k || !v || !s_out) return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (int rc = bind_device(stream, k)) return rc;
  FArgs a{k, k, v, nullptr, decay, nullptr, 0, s_out, B, H, N, d, dv, dtype, 0};
  return run_f(a, static_cast<cudaStream_t>(stream));
}

int la2_chunk_dstate(const void* q, const void* dout, const float* decay, float* t_out, int B,
                     int H, int N, int d, int dv, int dtype, void* stream) {
  g_err[0] = 0;
  if (int rc = check_common(B, H, N, d, dv, dtype, decay)) return rc;
  if (!q || !dout || !t_out) return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (int rc = bind_device(stream, q)) return rc;
  FArgs a{q, q, dout, nullptr, decay, nullptr, 0, t_out, B, H, N, d, dv, dtype, 1};
  return run_f(a, static_cast<cudaStream_t>(stream));
}

int la2_state_scan(const float* states, const float* decay, const float* init, float* out, int G,
                   int B, int H, int d, int dv, const int* lens, int reverse, void* stream) {
  g_err[0] = 0;
  if (!states || !decay || !out || !lens) return set_error(LA2_ERR_VALUE, "null pointer");
  if (B < 1 || H < 1 || d < 1 || dv < 1) return set_error(LA2_ERR_VALUE, "bad state shape");
  if (int rc = bind_device(stream, states)) return rc;
  return launch_state_scan(states, decay, init, out, G, B * H, H, d, dv, lens, reverse,
                           static_cast<cudaStream_t>(stream));
}

int la2_launch_log(int capacity) {
  g_err[0] = 0;
  if (capacity < 0) return set_error(LA2_ERR_VALUE, "capacity must be >= 0");
  std::lock_guard<std::mutex> lock(g_log_mu);
  g_log_on.store(0);
  for (LogRec& r : g_log) {
    cudaEventDestroy(r.t0);
    cudaEventDestroy(r.t1);
  }
  g_log.clear();
  g_log_used = g_log_dropped = 0;
  if (capacity == 0) return 0;
  g_log.resize(static_cast<size_t>(capacity));
  for (LogRec& r : g_log) {
    cudaError_t e = cudaEventCreate(&r.t0);
    if (e == cudaSuccess) e = cudaEventCreate(&r.t1);
    if (e != cudaSuccess) {
      g_log.clear();
      return set_cuda_error("la2_launch_log: cudaEventCreate", e);
    }
  }
  g_log_on.store(1);
  return 0;
}

int la2_launch_log_read(la2_launch_record* out, int max_records) {
  g_err[0] = 0;
  std::lock_guard<std::mutex> lock(g_log_mu);
  const int n = g_log_used < max_records ? g_log_used : max_records;
  for (int i = 0; i < n; ++i) {
    LogRec& r = g_log[i];
    cudaError_t e = cudaEventSynchronize(r.t1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.t0, r.t1);
    if (e != cudaSuccess) return set_cuda_error("la2_launch_log_read", e);
    std::snprintf(out[i].kernel, sizeof(out[i].kernel), "%s", r.kernel);
    out[i].grid = r.grid;
    out[i].cluster = r.cluster;
    out[i].ms = ms;
  }
  const int dropped = g_log_dropped + (g_log_used - n);
  g_log_used = 0;
  g_log_dropped = 0;
  (void)dropped;
  return n;
}

int la2_check_decay(const float* decay, int H, void* stream) {
  g_err[0] = 0;
  if (decay == nullptr) return set_error(LA2_ERR_VALUE, "decay pointer is null");
  if (H < 1) return set_error(LA2_ERR_VALUE, "H must be >= 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<float> h(static_cast<size_t>(H));
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, decay) != cudaSuccess) cudaGetLastError();
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
    if (int rc = bind_device(stream, decay)) return rc;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return set_error(LA2_ERR_UNSUPPORTED,
                       "la2_check_decay synchronizes the stream: call it before graph capture");
    }
    cudaError_t e = cudaMemcpyAsync(h.data(), decay, H * sizeof(float), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_cuda_error("la2_check_decay", e);
  } else {
    std::memcpy(h.data(), decay, H * sizeof(float));
  }
  for (int i = 0; i < H; ++i) {
    if (!(h[i] > 0.f && h[i] <= 1.f)) {
      char buf[128];
      std::snprintf(buf, sizeof(buf), "decay rate must be in (0, 1], got %g (head %d)",
                    static_cast<double>(h[i]), i);
      return set_error(LA2_ERR_VALUE, buf);
    }
  }
  return 0;
}

// ---------------------------------------------------------------- fp64 (la2_f64.cu)
static int check_f64(int B, int H, int N, int d, int dv, const double* decay) {
  if (B < 1 || H < 1) return set_error(LA2_ERR_VALUE, "B and H must be >= 1");
  if (N < 1) return set_error(LA2_ERR_VALUE, "sequence length N must be >= 1");
  if (d < 1 || dv < 1) return set_error(LA2_ERR_VALUE, "d and dv must be >= 1");
  if (d > 256 || dv > 256) return set_error(LA2_ERR_UNSUPPORTED, "fp64 path supports d, dv <= 256");
  if (decay == nullptr) return set_error(LA2_ERR_VALUE, "decay pointer is null");
  return 0;
}

int la2_forward_f64(const double* q, const double* k, const double* v, const double* decay, double* o,
                    const double* kv_in, double* kv_out, int B, int H, int N, int d, int dv, int block,
                    void* stream) {
  g_err[0] = 0;
  if (int rc = check_f64(B, H, N, d, dv, decay)) return rc;
  if (!q || !k || !v || !o) return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (int rc = bind_device(stream, q)) return rc;
  return launch_f64(q, k, v, o, decay, kv_in, 0, kv_out, B, H, N, d, dv, 0, block,
                    static_cast<cudaStream_t>(stream));
}

// The backward as three F passes, exactly like la2_backward's SIMT path:
// dQ = F(dO, V, K) (state KV^T), dK = F_rev(V, dO, Q) (state dKV^T), dV = F_rev(K, Q, dO).
int la2_backward_f64(const double* q, const double* k, const double* v, const double* dout,
                     const double* decay, double* dq, double* dk, double* dv, const double* kv_in,
                     const double* dkv_in, double* dkv_out, int B, int H, int N, int d, int dvd, int block,
                     void* stream) {
  g_err[0] = 0;
  if (int rc = check_f64(B, H, N, d, dvd, decay)) return rc;
  if (!q || !k || !v || !dout || !dq || !dk || !dv) return set_error(LA2_ERR_VALUE, "null tensor pointer");
  if (int rc = bind_device(stream, q)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = launch_f64(dout, v, k, dq, decay, kv_in, 1, nullptr, B, H, N, dvd, d, 0, block, st)) return rc;
  if (int rc = launch_f64(v, dout, q, dk, decay, dkv_in, 1, nullptr, B, H, N, dvd, d, 1, block, st)) return rc;
  return launch_f64(k, q, dout, dv, decay, dkv_in, 0, dkv_out, B, H, N, d, dvd, 1, block, st);
}

int la2_decode_tokens_f64(const double* q, const double* k, const double* v, const double* decay,
                          double* state, double* o, int B, int H, int T, int d, int dv, void* stream) {
  g_err[0] = 0;
  if (B < 1 || H < 1 || d < 1 || dv < 1 || T < 0) return set_error(LA2_ERR_VALUE, "bad decode shape");
  if (T == 0) return 0;
  if (!q || !k || !v || !decay || !state || !o) return set_error(LA2_ERR_VALUE, "null pointer");
  if (int rc = bind_device(stream, state)) return rc;
  return launch_decode_f64(q, k, v, decay, state, o, B, H, d, dv, T, static_cast<cudaStream_t>(stream));
}

int la2_decode_step_f64(const double* q, const double* k, const double* v, const double* decay,
                        double* state, double* o, int B, int H, int d, int dv, void* stream) {
  return la2_decode_tokens_f64(q, k, v, decay, state, o, B, H, 1, d, dv, stream);
}

int la2_check_decay_f64(const double* decay, int H, void* stream) {
  g_err[0] = 0;
  if (decay == nullptr) return set_error(LA2_ERR_VALUE, "decay pointer is null");
  if (H < 1) return set_error(LA2_ERR_VALUE, "H must be >= 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<double> h(static_cast<size_t>(H));
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, decay) != cudaSuccess) cudaGetLastError();
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
    if (int rc = bind_device(stream, decay)) return rc;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return set_error(LA2_ERR_UNSUPPORTED,
                       "la2_check_decay_f64 synchronizes the stream: call it before graph capture");
    }
    cudaError_t e = cudaMemcpyAsync(h.data(), decay, H * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_cuda_error("la2_check_decay_f64", e);
  } else {
    std::memcpy(h.data(), decay, H * sizeof(double));
  }
  for (int i = 0; i < H; ++i) {
    if (!(h[i] > 0.0 && h[i] <= 1.0)) {
      char buf[128];
      std::snprintf(buf, sizeof(buf), "decay rate must be in (0, 1], got %g (head %d)", h[i], i);
      return set_error(LA2_ERR_VALUE, buf);
    }
  }
  return 0;
}

int la2_decode_tokens(const void* q, const void* k, const void* v, const float* decay, float* state,
                      void* o, int B, int H, int T, int d, int dv, int dtype, void* stream) {
  g_err[0] = 0;
  if (B < 1 || H < 1 || d < 1 || dv < 1 || T < 0) return set_error(LA2_ERR_VALUE, "bad decode shape");
  if (dtype != LA2_BF16 && dtype != LA2_FP32)
    return set_error(LA2_ERR_UNSUPPORTED, "dtype must be LA2_BF16 or LA2_FP32");
  if (T == 0) return 0;
  if (!q || !k || !v || !decay || !state || !o) return set_error(LA2_ERR_VALUE, "null pointer");
  if (int rc = bind_device(stream, state)) return rc;
  return launch_decode(q, k, v, decay, state, o, B, H, d, dv, T, dtype,
                       static_cast<cudaStream_t>(stream));
}

int la2_decode_step(const void* q, const void* k, const void* v, const float* decay, float* state,
                    void* o, int B, int H, int d, int dv, int dtype, void* stream) {
  return la2_decode_tokens(q, k, v, decay, state, o, B, H, 1, d, dv, dtype, stream);
}

}  // extern "C"
