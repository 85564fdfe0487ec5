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

/* Launch plan of one tcgen05 GEMM (host-side arithmetic only: no device, no CUDA call beyond the
 * SM-count query, which falls back to 148 without a GPU). For N output rows (the sum of the
 * segments' tile-rounded rows), K, M tokens (1..256) it returns in plan[12]:
 *   [0] workers G of the stream-K split   [1] tiles per work unit (1 / 2)   [2] unit tiles
 *   [3] k-blocks per tile                 [4] CTAs launched                 [5] 1 = CTA pairs
 *   [6] ring stages                       [7] dynamic smem bytes per CTA    [8] TMEM columns per CTA
 *   [9] split-tile reducer (0 in-kernel, 1 fix-up grid)                    [10] CTAs per SM (budget)
 *   [11] padded tokens Mp
 * The split ([0]-[3]) must not depend on M (batch invariance); tests/test_capi_cpu.py checks this
 * and the resource bounds. Errors: EINVAL. */
mpsw_status mpsw_tc_plan(int N, int K, int M, int64_t* plan);

/* Intermediate-value tap of the TP forward (a6), for element-by-element parity with the oracle's
 * per-layer values (oracle/forward.py `taps`). Arms a ONE-SHOT tap on `ctx`: the next batch the
 * engine dispatches runs the same kernels as a normal batch (per-op path: the fused layers kernel
 * is bypassed) but stops early, and global rank `rank`'s worker copies one workspace buffer into
 * `dst` before the batch completes. The batch's logits are undefined (lm_head does not run).
 *   what = MPSW_TAP_X   : fp32 residual stream [M, h] after `n_layers` complete decoder layers
 *                         (n_layers = 0: the embedding sum E_tok[x] + E_pos[pos], C5 step 1);
 *          MPSW_TAP_A   : LN output [M, h] (the next GEMM's A operand: LN1 of layer n_layers, or
 *                         the final LN when n_layers = L_m), in the ctx dtype (bf16 bits / fp32);
 *          MPSW_TAP_QKV : fp32 [M, 3*h/t] = [q | k | v] of layer n_layers on that rank (q scaled
 *                         by hd^-0.5 after its bias, HF:opt.py:151);
 *          MPSW_TAP_O   : attention output [M, h/t] of layer n_layers (ctx dtype);
 *          MPSW_TAP_R   : ReLU(fc1) output [M, ff/t] of layer n_layers (ctx dtype);
 *          MPSW_TAP_XM  : fp32 residual stream [M, h] of layer n_layers after its attention block
 *                         (x + all-reduced out_proj + bias);
 *          MPSW_TAP_F   : LN2 output [M, h] of layer n_layers (fc1's A operand, ctx dtype).
 * Rows are the batch's packed token rows (requests in batch order). At most `bytes` bytes are
 * written; dst is host memory that must stay valid until the batch completes.
 * Single-process ctx with pp = 1 only. Errors: EINVAL (bad argument, mp mode, pp > 1). */
enum { MPSW_TAP_X = 0, MPSW_TAP_A = 1, MPSW_TAP_QKV = 2, MPSW_TAP_O = 3, MPSW_TAP_R = 4, MPSW_TAP_XM = 5, MPSW_TAP_F = 6 };
mpsw_status mpsw_test_tap(mpsw_ctx* ctx, int n_layers, int what, int rank, void* dst, uint64_t bytes);

/* Fault injection (runtime robustness tests): global rank `rank`'s worker throws at its next
 * all-reduce point, as a CUDA failure inside a batch would. The ctx is poisoned: the other ranks
 * leave their TP barrier (no hang), pending requests fail with ECUDA and mpsw_shutdown returns.
 * Single-process ctx only. Errors: EINVAL. */
mpsw_status mpsw_test_inject_fault(mpsw_ctx* ctx, int rank);

/* Debug-check self test (mpsw_config.debug_checks = 1): overwrite every local rank's residency
 * stamp of `model_id` with a value no load ever writes, so the model's next forward must trip the
 * check (ctx poisoned, EINVARIANT in the poison message). Errors: EINVAL (checks off / model). */
mpsw_status mpsw_test_corrupt_stamp(mpsw_ctx* ctx, int model_id);

#ifdef __cplusplus
}
#endif
#endif /* MPSW_TESTING_H */
