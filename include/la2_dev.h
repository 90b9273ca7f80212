/*
 * la2_dev.h -- development library libla2_dev.so (NOT the shipping ABI).
 *
 * Self-test and micro-benchmarks of the tcgen05 building blocks the kernels in
 * libla2.so use. None of these replaces a reference function; they live in their own
 * library so that libla2.so exports only include/la2.h. Same status codes as la2.h;
 * the message of the last failure on the calling thread is la2_dev_last_error().
 */
#ifndef LA2_DEV_H_
#define LA2_DEV_H_

#include "la2.h"

#ifdef __cplusplus
extern "C" {
#endif

LA2_API const char* la2_dev_last_error(void);

/*
 * Self-test of the tensor-core operand layouts: D[M][N] = A[M][K] B[K][N] through the
 * same SW128 descriptors the tcgen05 kernel uses; a_mn / b_mn select MN-major staging
 * (a_mn = 2: A read from TMEM). fp32 device buffers.
 */
LA2_API int la2_selftest_umma(const float* A, const float* B, float* D, int M, int N, int K,
                              int a_mn, int b_mn, void* stream);

/* Clock cycles per CTA for `iters` back-to-back K=16 tcgen05.mma of one shape;
 * a_mode 0/1/2 = A K-major smem / MN-major smem / TMEM. */
LA2_API int la2_bench_umma(int M, int N, int a_mode, int b_mn, int iters, int ctas, long long* out,
                           void* stream);

/* TMEM -> register load throughput. */
LA2_API int la2_bench_tmem(int warps, int iters, int batch, int ctas, long long* out, float* sink,
                           void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LA2_DEV_H_ */
