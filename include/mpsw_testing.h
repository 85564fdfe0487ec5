/*
 * mpsw_testing.h — verification hooks of libmpsw.so (not part of the serving API).
 *
 * mpsw_test_gemm runs ONE forward GEMM of the library in isolation so the kernels can be checked
 * element by element against a plain CPU reference:
 *   out[m, n] = epi( sum_k X[m, k] * W[n, k] + bias[n] )       (W row-major [N, K], X [M, K])
 * dtype MPSW_BF16: W, X, bias are bf16 bit patterns (uint16); MPSW_FP32: float.
 * impl: 1 = SIMT weight-streaming kernel, 2 = tcgen05/TMA kernel (bf16 only, M <= 256).
 * epi: 0 = fp32 out = (acc + bias) * scale; 1 = out = relu(acc + bias) rounded to the dtype.
 * out is host memory of M*N floats (bf16 results are widened to float). All pointers are host
 * pointers; device buffers are allocated and freed inside. Runs on CUDA device `device`.
 * Errors: EINVAL (shape / impl), ECUDA.
 */
#ifndef MPSW_TESTING_H
#define MPSW_TESTING_H

#include "mpsw.h"

#ifdef __cplusplus
extern "C" {
#endif

mpsw_status mpsw_test_gemm(int device, int dtype, int impl, const void* W, const void* X, const void* bias,
                           int M, int N, int K, int epi, float scale, float* out);

/* Microbenchmark: average device time (us) of `reps` back-to-back launches of one library GEMM
 * (impl 1 SIMT, 2 tcgen05) with N x K bf16 weights, M tokens, fp32 output. Device buffers are
 * allocated, filled with a constant and freed inside. */
mpsw_status mpsw_bench_gemm(int device, int impl, int M, int N, int K, int reps, float* us);

#ifdef __cplusplus
}
#endif
#endif /* MPSW_TESTING_H */
