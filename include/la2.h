/*
 * la2.h -- C ABI of the B200-native Lightning Attention-2 hot path.
 *
 * Drop-in boundary for the reference `tila` package (Python/NumPy,
 * /root/reference/pkg/src/tila). Every entry point below replaces one
 * reference function; the citation is given per function. The ABI takes
 * plain device pointers, sizes and a cudaStream_t passed as void*; it has no
 * torch types. All launches are asynchronous on the caller's stream; the
 * library never allocates, frees or retains caller memory. Its only own device
 * memory is one fixed workspace per (device, stream) -- the stream-K state
 * hand-off slots, la2_workspace_bytes() bytes (~4.7 MB on B200), allocated on the
 * first launch on that stream (outside the capture when that launch is being captured
 * into a CUDA graph) and kept for the process lifetime; it does not grow with B, H or N. A CUDA graph captured on a stream bakes
 * in that stream's workspace: replays of graphs captured on the same stream must not
 * run concurrently with each other (capture concurrent graphs on distinct streams).
 *
 * Layouts (all contiguous, row-major):
 *   q, k, dq, dk          [B, H, N, d]
 *   v, o, dout, dv        [B, H, N, dv]
 *   decay                 [H] float32, lambda_h in (0, 1]   (per-head decay)
 *   states (kv, dkv)      [B, H, d, dv] float32
 * Element type of q/k/v/o/... is selected by `dtype` (LA2_BF16 or LA2_FP32); float64
 * (the reference's default dtype) has its own entry points, la2_*_f64, below.
 *
 * Kernel selection is a pure function of (dtype, d, dv):
 *   bf16, d and dv multiples of 8 up to 256 -> tcgen05/TMA tensor-core kernel: d <= 64 /
 *                                           <= 128 on the 64- / 128-wide kernel, narrower
 *                                           operands zero-filled by the TMA unit; d > 128
 *                                           split-d (two passes over the column halves, the
 *                                           second adding into o by TMA reduce-add); dv in
 *                                           64-wide value slices, the last one partial
 *   otherwise, d <= 256 and dv <= 256   -> SIMT fp32-accumulate kernel
 *   anything else                       -> LA2_ERR_UNSUPPORTED (no fallback)
 *
 * Decay: the compute entry points read `decay` on the device, asynchronously, so they
 * cannot return an error for its values. They never clamp: a lambda outside (0, 1]
 * (or NaN) makes every output of the affected heads NaN. la2_check_decay() is the
 * validating entry point (the reference's ValueError, reference.py:42-44); the Python
 * layer calls it once per decay tensor version before the first launch.
 *
 * Return value: 0 on success, a negative LA2_ERR_* code otherwise; the
 * message of the last failure on the calling thread is la2_last_error().
 */
#ifndef LA2_H_
#define LA2_H_

#if defined(__GNUC__)
#define LA2_API __attribute__((visibility("default")))
#else
#define LA2_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum la2_dtype { LA2_BF16 = 0, LA2_FP32 = 1 };

enum la2_status {
  LA2_OK = 0,
  LA2_ERR_VALUE = -1,       /* bad shape / decay / pointer: Python raises ValueError   */
  LA2_ERR_UNSUPPORTED = -2, /* shape/dtype outside the kernels' envelope: ValueError    */
  LA2_ERR_CUDA = -3         /* launch or driver failure: Python raises RuntimeError     */
};

/* ABI version (major*100 + minor). */
LA2_API int la2_version(void);

/* Message for the most recent non-zero return on this thread ("" if none). */
LA2_API const char* la2_last_error(void);

/*
 * Block-tiled forward pass, O = causal decayed linear attention of (q, k, v).
 * Replaces tila.tiled_forward      (pkg/src/tila/kernel.py:122-139),
 *          tila.chunked_forward    (pkg/src/tila/kernel.py:142-162; kv_in = caller state,
 *                                   kv_out = returned KvState.kv),
 *          tila.batched_forward    (pkg/src/tila/kernel.py:252-260; B*H heads, per-head decay).
 * kv_in  (nullable): state carried in, referenced just before token 0.
 * kv_out (nullable): final state sum_s lam^(N-1-s) k_s^T v_s + lam^N kv_in.
 */
LA2_API int la2_forward(const void* q, const void* k, const void* v, const float* decay, void* o,
                const float* kv_in, float* kv_out, int B, int H, int N, int d, int dv, int dtype,
                void* stream);

/*
 * la2_forward on views: q, k, v may have any element stride between consecutive (b, h)
 * rows (ldq, ldk, ldv >= N * d / N * dv, multiples of 8), e.g. a [B, H, N, d] slice of
 * a longer sequence, so streaming over chunks of a resident sequence reads the chunks in
 * place (chunked_forward on slices, kernel.py:142-162). o, kv_in, kv_out contiguous.
 * Tensor-core shapes only (bf16, d in {64,128,256}, dv % 64 == 0); otherwise
 * LA2_ERR_UNSUPPORTED.
 */
LA2_API int la2_forward_strided(const void* q, const void* k, const void* v, const float* decay,
                                void* o, const float* kv_in, float* kv_out, int B, int H, int N,
                                int d, int dv, int dtype, long long ldq, long long ldk,
                                long long ldv, void* stream);

/*
 * Backward pass: gradients of sum(dout * O) with respect to q, k, v.
 * Replaces tila.tiled_backward     (pkg/src/tila/kernel.py:165-233) and
 *          tila.batched_backward   (pkg/src/tila/kernel.py:263-266).
 * kv_in  (nullable): the forward kv_in (state before token 0).
 * dkv_in (nullable): mirrored state from tokens after N-1
 *                    (sum_{s>=N} lam^(s-N+1) q_s^T dout_s), for sequence parallelism.
 * dkv_out(nullable): dkv folded over the whole chunk (referenced before token 0).
 */
LA2_API int la2_backward(const void* q, const void* k, const void* v, const void* dout,
                 const float* decay, void* dq, void* dk, void* dv, const float* kv_in,
                 const float* dkv_in, float* dkv_out, int B, int H, int N, int d, int dv_dim,
                 int dtype, void* stream);

/*
 * la2_backward on views: q, k, v, dout with (b, h) row strides ldq, ldk, ldv, lddo
 * (>= N * d / N * dv elements, multiples of 8), e.g. chunks of a resident sequence
 * (training on sequence chunks with the carried kv_in / dkv_in); dq, dk, dv contiguous.
 * Tensor-core shapes only; otherwise LA2_ERR_UNSUPPORTED.
 */
LA2_API int la2_backward_strided(const void* q, const void* k, const void* v, const void* dout,
                                 const float* decay, void* dq, void* dk, void* dv,
                                 const float* kv_in, const float* dkv_in, float* dkv_out, int B,
                                 int H, int N, int d, int dvd, int dtype, long long ldq,
                                 long long ldk, long long ldv, long long lddo, void* stream);

/*
 * Forward that also stores the per-block states, and the backward that uses them
 * (bf16, d = dv = 64; otherwise LA2_ERR_UNSUPPORTED).
 * kv_blocks: [B, H, ceil(N/128), d, dv] bf16, la2_state_blocks_bytes() bytes: entry
 * [b, h, i] is the bf16 state KV_{i-1} the forward's block i read (128-token blocks;
 * i = 0: kv_in or 0) -- the KV the reference's sweep 1 replays (kernel.py:184-204).
 * la2_backward_states then computes dQ block by block from the stored states instead
 * of replaying the recurrence, inside the same 3-CTA cluster as the dK / dV reverse
 * scans (kernel.py:207-231), so K, Q, dO and V are read once. Results equal
 * la2_backward's up to the rounding of the replayed state (both bf16).
 * dkv_in / dkv_out as in la2_backward; the forward's kv_in is in kv_blocks already.
 */
LA2_API long long la2_state_blocks_bytes(int B, int H, int N, int d, int dv);
LA2_API int la2_forward_states(const void* q, const void* k, const void* v, const float* decay,
                               void* o, const float* kv_in, float* kv_out, void* kv_blocks, int B,
                               int H, int N, int d, int dv, int dtype, void* stream);
LA2_API int la2_backward_states(const void* q, const void* k, const void* v, const void* dout,
                                const float* decay, const void* kv_blocks, void* dq, void* dk,
                                void* dv, const float* dkv_in, float* dkv_out, int B, int H, int N,
                                int d, int dv_dim, int dtype, void* stream);

/*
 * Chunk-local forward state only (no output): S = sum_s lam^(N-1-s) k_s^T v_s.
 * Equals the KvState.kv returned by tila.chunked_forward from a fresh state
 * (pkg/src/tila/kernel.py:142-162). Sequence-parallel pass A.
 */
LA2_API int la2_chunk_state(const void* k, const void* v, const float* decay, float* s_out, int B, int H,
                    int N, int d, int dv, int dtype, void* stream);

/*
 * Chunk-local reverse state only: T = sum_s lam^(s+1) q_s^T dout_s, the dkv of the
 * reverse sweep of tila.tiled_backward folded over the chunk from zero
 * (pkg/src/tila/kernel.py:207-231). Sequence-parallel backward pass A.
 */
LA2_API int la2_chunk_dstate(const void* q, const void* dout, const float* decay, float* t_out, int B,
                     int H, int N, int d, int dv, int dtype, void* stream);

/*
 * Exclusive prefix (reverse=0) or suffix (reverse=1) combine of G chunk states
 * with per-chunk decay lam^len[g]:
 *   reverse=0: out[0] = init (or 0), out[g+1] = lam^len[g] * out[g] + states[g]
 *   reverse=1: out[G-1] = init (or 0), out[g-1] = lam^len[g] * out[g] + states[g]
 * states/out: [G, B*H, d, dv] fp32; lens: host array of G chunk lengths (G <= 64).
 * The fold rule is the state update of pkg/src/tila/kernel.py:111-115 applied per chunk.
 */
LA2_API int la2_state_scan(const float* states, const float* decay, const float* init, float* out, int G,
                   int B, int H, int d, int dv, const int* lens, int reverse, void* stream);

/*
 * Validate a per-head decay vector: every lambda_h must lie in (0, 1]
 * (tila._check_decay, pkg/src/tila/reference.py:42-44). `decay` may be device memory
 * (copied to the host on `stream`, which is synchronized: not usable inside graph
 * capture -> LA2_ERR_UNSUPPORTED) or host memory. Returns LA2_ERR_VALUE with the
 * offending value and head otherwise.
 */
LA2_API int la2_check_decay(const float* decay, int H, void* stream);

/*
 * One decode step per (b, h), in place on `state`:
 *   state <- lam * state + k_t^T v_t ;  o_t = q_t state
 * Replaces tila.inference_step (pkg/src/tila/reference.py:162-181, _decay_step :135-139).
 * q,k: [B,H,d]  v,o: [B,H,dv]  state: [B,H,d,dv] fp32.
 */
LA2_API int la2_decode_step(const void* q, const void* k, const void* v, const float* decay,
                    float* state, void* o, int B, int H, int d, int dv, int dtype, void* stream);

/*
 * T decode steps per (b, h) in one launch, in place on `state`: tila.inference_step folded
 * over T tokens (reference.py:162-181), i.e. tila.recurrent_forward (reference.py:142-159)
 * continued from `state` (a zeroed state gives recurrent_forward itself). Each token
 * runs the single step's arithmetic in the same order, so the result equals T calls of
 * la2_decode_step bit for bit (given the same kernel choice: the vector kernel needs
 * 16-byte aligned q, k, 4-element aligned v, o and d * sizeof(elem) % 16 == 0, else the
 * general kernel runs); the state crosses HBM once per call instead of once per token
 * (multi-token decode: speculative / chunked continuation of a stream).
 * q,k: [B,H,T,d]  v,o: [B,H,T,dv]  state: [B,H,d,dv] fp32. T = 0 is a no-op.
 */
LA2_API int la2_decode_tokens(const void* q, const void* k, const void* v, const float* decay,
                              float* state, void* o, int B, int H, int T, int d, int dv, int dtype,
                              void* stream);

/*
 * Double precision: the reference's default dtype (every tila routine computes in the
 * input dtype, np.result_type; pkg/src/tila/reference.py:54-74). fp64 storage and
 * arithmetic on the CUDA cores (DFMA), decay powers by iterated products flushed below
 * the smallest normal double (tila.power_table, reference.py:75-100). All tensors,
 * decay and states are double; shapes and semantics as the single-precision calls:
 *   la2_forward_f64      tila.tiled_forward / chunked_forward  (kernel.py:122-162)
 *   la2_backward_f64     tila.tiled_backward                  (kernel.py:165-233)
 *   la2_decode_step_f64  tila.inference_step                  (reference.py:162-181)
 *   la2_decode_tokens_f64 tila.recurrent_forward / folded inference_step (reference.py:142-181)
 *   la2_check_decay_f64  the decay validation of reference.py:42-44
 * d, dv <= 256; no sequence split, no tensor cores: a correctness path for the tila
 * adapter (the reference's 1e-10 gates), not a throughput path. `block` is the
 * reference's block argument: the kernels tile by it when it is <= 16 (or when it covers
 * a sequence of <= 16 tokens: one tile), else by its largest divisor <= 16 (0: 16), so
 * results are deterministic per block and chunk boundaries aligned to it give bitwise the
 * one-call result, as in the reference.
 */
LA2_API int la2_forward_f64(const double* q, const double* k, const double* v, const double* decay,
                            double* o, const double* kv_in, double* kv_out, int B, int H, int N,
                            int d, int dv, int block, void* stream);
LA2_API int la2_backward_f64(const double* q, const double* k, const double* v, const double* dout,
                             const double* decay, double* dq, double* dk, double* dv,
                             const double* kv_in, const double* dkv_in, double* dkv_out, int B, int H,
                             int N, int d, int dv_dim, int block, void* stream);
LA2_API int la2_decode_step_f64(const double* q, const double* k, const double* v, const double* decay,
                                double* state, double* o, int B, int H, int d, int dv, void* stream);
LA2_API int la2_decode_tokens_f64(const double* q, const double* k, const double* v, const double* decay,
                                  double* state, double* o, int B, int H, int T, int d, int dv,
                                  void* stream);
LA2_API int la2_check_decay_f64(const double* decay, int H, void* stream);

/*
 * Norm(.) of NormAttention, O = Norm(Q (K^T V)) -- an extension: the
 * reference leaves the normalisation out. Simple RMS normalisation of the
 * attention-output rows, y = x / sqrt(mean(x^2) + eps), over the dv features of each head
 * (group = 1) or over all H heads' features of a token (group = H: TransNormerLLM's SRMSNorm
 * over the concatenated heads). rstd (fp32, [B,H,N] for group 1, [B,N] for group H) keeps
 * 1 / sqrt(mean + eps) for the backward dx = (dy - y mean(dy y)) rstd.
 *   la2_forward_norm      la2_forward (or la2_forward_states when kv_blocks != NULL) with the
 *                         norm applied to o; fused into the tensor-core epilogue for bf16
 *                         per-head norms with d <= 64, dv = 64, else a separate pass in place
 *   la2_rmsnorm_forward   the norm alone (y may alias x)
 *   la2_rmsnorm_backward  its backward from y and rstd
 */
LA2_API int la2_forward_norm(const void* q, const void* k, const void* v, const float* decay, void* o,
                             const float* kv_in, float* kv_out, void* kv_blocks, float* rstd, float eps,
                             int group, int B, int H, int N, int d, int dv, int dtype, void* stream);
LA2_API int la2_rmsnorm_forward(const void* x, void* y, float* rstd, int B, int H, int N, int dv, int group,
                                float eps, int dtype, void* stream);
LA2_API int la2_rmsnorm_backward(const void* dy, const void* y, const float* rstd, void* dx, int B, int H,
                                 int N, int dv, int group, int dtype, void* stream);

/*
 * Scheduling knobs of the tensor-core kernels (process-wide; not a reference
 * interface). Results do not depend on them: the persistent schedule hands the fp32
 * state between work ranges exactly, so outputs are bitwise identical either way.
 *   LA2_TUNE_PERSISTENT  1 (default): when there are more recurrences than co-resident
 *                        CTAs, run one persistent CTA per SM over an even split of the
 *                        (recurrence, block) space; 0: one CTA per recurrence.
 *   LA2_TUNE_PREFETCH    L2 prefetch distance in blocks for 2-stage rings (default 0).
 *   LA2_TUNE_L2HINT      L2 policy bits: 1 loads evict_first, 2 prefetches evict_last,
 *                        4 output stores evict_first (default 0).
 *   LA2_TUNE_FUSED_BWD   1 (default): at d = dv = 128 with few heads (each pass alone
 *                        would leave SMs idle) the dV and dK scans of the backward run as
 *                        one 4-CTA cluster per unit sharing Q / dO through L2;
 *                        0: always two separate launches.
 *   LA2_TUNE_CONCURRENT_BWD  sequences with N <= value (default 16384) run the dQ scan of
 *                        la2_backward on a forked side stream, concurrent with the dK/dV
 *                        scans (joined back before return); 0 disables.
 *   LA2_TUNE_PARTITION_BWD   d = 64 sequences with N <= value (default 8192) run the dQ
 *                        scan and the dK/dV pair concurrently on disjoint SM partitions
 *                        (1/3 : 2/3, both persistent); 0 disables (then the
 *                        LA2_TUNE_CONCURRENT_BWD rule applies).
 *   LA2_TUNE_PDL         sequences with N <= value (default 4096) launch the tensor-core
 *                        kernels with programmatic dependent launch (the prologue overlaps
 *                        the previous kernel's tail; all global accesses wait for it);
 *                        0: plain stream order.
 */
#define LA2_TUNE_PERSISTENT 1
#define LA2_TUNE_PREFETCH 2
#define LA2_TUNE_L2HINT 3
#define LA2_TUNE_FUSED_BWD 4
#define LA2_TUNE_CONCURRENT_BWD 5
#define LA2_TUNE_PARTITION_BWD 6
#define LA2_TUNE_PDL 7
LA2_API int la2_set_tuning(int key, int value);

/*
 * Launch log (instrumentation; not a reference interface). la2_launch_log(capacity)
 * preallocates `capacity` event pairs and starts recording: every kernel launch of the
 * library is then bracketed by two CUDA events recorded on the stream it is launched
 * on (launches inside graph capture are not logged). la2_launch_log_read() waits for
 * the logged launches, copies up to max_records of them (in launch order) and resets
 * the log; it returns the number copied or a negative status. capacity 0 stops
 * logging and frees the events. Used by bench.py for the per-kernel roofline.
 */
typedef struct la2_launch_record {
  char kernel[48]; /* e.g. "la2_tc_kernel<64,1,0,2>" (the ncu kernel name) */
  int grid;        /* CTAs launched */
  int cluster;     /* CTAs per cluster */
  float ms;        /* event-timed duration on the launching stream */
} la2_launch_record;
LA2_API int la2_launch_log(int capacity);
LA2_API int la2_launch_log_read(la2_launch_record* out, int max_records);

/* Bytes of the per-(device, stream) workspace on the current device (0 without a
 * device). Constant in B, H, N: the working set of a pass is independent of the
 * sequence length (the reference's constant-scratch property, scratch.py /
 * test_acceptance.py criterion 6). */
LA2_API long long la2_workspace_bytes(void);

#ifdef __cplusplus
}
#endif

#endif /* LA2_H_ */
