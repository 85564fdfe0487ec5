// Internal declarations of the mpsw library (not part of the C-ABI).
#pragma once

#include "../../include/mpsw.h"

#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace mpsw {

// ---------------------------------------------------------------- errors
std::string& tls_error();
mpsw_status set_error(mpsw_status s, const std::string& msg);

struct Error : std::runtime_error {
    mpsw_status status;
    Error(mpsw_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define MPSW_CU(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            throw ::mpsw::Error(MPSW_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + \
                                " (" __FILE__ ":" + std::to_string(__LINE__) + ")");         \
    } while (0)

// ---------------------------------------------------------------- layout (C2, product side)
struct Layout {
    std::vector<mpsw_tensor_desc> t;
    uint64_t bytes = 0;
};
mpsw_status compute_layout(const mpsw_opt_dims& d, int tp, int pp, int stage, int rank, int dtype, Layout& out);

// ---------------------------------------------------------------- synthetic fill (C0, product side)
void synth_fill_arena(const mpsw_opt_dims& d, int tp, int pp, int stage, int rank, int dtype, uint64_t seed,
                      uint8_t* dst, int threads);
uint64_t host_checksum(const uint8_t* p, uint64_t bytes, int threads);

// ---------------------------------------------------------------- swap / checksum kernels
// Zero-copy copy: 128-bit loads from `src` (mapped pinned host OR device) and 128-bit stores
// to `dst` (device OR mapped pinned host). bytes % 16 == 0, pointers 16-B aligned.
void launch_zero_copy(void* dst, const void* src, uint64_t bytes, int ctas, cudaStream_t s);
// Order-independent checksum (C4) of a device buffer; result accumulated into *d_out.
void launch_checksum(const void* buf, uint64_t bytes, unsigned long long* d_out, cudaStream_t s);
// Residency stamps of the debug checks (mpsw_config.debug_checks).
constexpr unsigned long long kStampEvicted = ~0ull;
void launch_stamp(unsigned long long* slot, unsigned long long value, cudaStream_t s);
void launch_check_stamp(const unsigned long long* slot, unsigned long long expect, unsigned int* err, cudaStream_t s);

// ---------------------------------------------------------------- forward (per rank)
struct TensorPtrs {          // device pointers of one rank's shard inside a slot
    const void* embed_tok;   // [V/t, h]
    const void* embed_pos;   // [P, h]
    const void* lnf_w;
    const void* lnf_b;
    struct Layer {
        const void *k_w, *k_b, *v_w, *v_b, *q_w, *q_b, *o_w, *o_b;
        const void *ln1_w, *ln1_b, *fc1_w, *fc1_b, *fc2_w, *fc2_b, *ln2_w, *ln2_b;
    };
    std::vector<Layer> layers;
};

struct FwdShape {
    int n_layers, hidden, heads_local, head_dim, ffn_local, vocab_local, vocab, tp, rank;
    int dtype;               // MPSW_BF16 / MPSW_FP32
    int gemm_impl;           // 0 auto (tcgen05 per op for bf16), 1 SIMT, 2 tcgen05 per op
    int max_rows;            // rows of the activation buffers (max_batch * max_tokens)
};

struct FwdWorkspace {        // device buffers of one rank (sized for max_batch*max_tokens rows)
    float* x = nullptr;            // residual stream [M, h] fp32
    void* a = nullptr;             // LN output (GEMM A operand) [M, h]
    float* qkv = nullptr;          // [M, 3*h/t] fp32 (q pre-scaled)
    void* o = nullptr;             // attention output [M, h/t]
    void* r = nullptr;             // relu output [M, ff/t]
    float* partial[2] = {nullptr, nullptr};   // row-parallel partials [M, h] fp32 (peers read)
    float* logits = nullptr;       // [B, V/t] fp32
    int32_t* tokens = nullptr;     // [M]
    int32_t* meta = nullptr;       // seq_start[B+1], last_row[B], pos[M], row_of_m[M]
    float* tc_partial = nullptr;   // tcgen05 split-K partial sums
    int* tc_counters = nullptr;    // per-tile arrival counters (self-resetting)
    size_t tc_partial_cap = 0;     // floats of tc_partial
    int tc_counters_cap = 0;       // entries of tc_counters
    void* base = nullptr;
    size_t bytes = 0;
};
size_t workspace_bytes(const FwdShape& s, int max_rows, int max_batch);
void workspace_carve(FwdWorkspace& w, const FwdShape& s, int max_rows, int max_batch, void* base);

// tcgen05/TMA weight-streaming GEMM (gemm_tc.cu)
size_t tc_partial_floats(int n_total, int K, int Mp);
void tc_set_trace(unsigned long long* p);
int tc_grid_for(int n_total, int K);
int tc_grid_tiles(int tiles, int K);     // stream-K CTAs of a GEMM with `tiles` 128-row tiles
bool tc_supported(int M, int K);
int tc_pair();                           // 1: A/B mode: pair split, always on CTA pairs (cta_group::2)
int tc_split_kt();                       // tiles per stream-K work unit (1 or 2), process-wide
void tc_gemm(const void* const* W, const void* const* bias, const int* N, const float* scale, const int* out_col0,
             int nseg, const void* X, int x_rows, int M, int K, int epi, void* out, int ldo, const int32_t* row_of_m,
             float* partial, int* counters, cudaStream_t st);

// Kernel launchers (forward.cu). Each returns the number of kernels launched.
int fwd_embed(const FwdShape& s, const TensorPtrs& W, const FwdWorkspace& ws, int M, float* partial,
              cudaStream_t st);
int fwd_reduce_ln(const FwdShape& s, int M, const float* const* peer_partials, int n_peers,
                  const float* residual, const void* bias, const void* pos_table, const int32_t* pos,
                  const void* gamma, const void* beta, float* x_out, void* ln_out, cudaStream_t st);
// Reduce-scatter variant: rows [row0, row0 + rows) only, the LN output written to every buffer of
// ln_outs (all TP ranks' A operands: the all-gather of the bf16 LN output).
int fwd_reduce_ln_rows(const FwdShape& s, int row0, int rows, const float* const* peer_partials, int n_peers,
                       const float* residual, const void* bias, const void* pos_table, const int32_t* pos,
                       const void* gamma, const void* beta, float* x_out, void* const* ln_outs, int n_out,
                       cudaStream_t st);
int fwd_qkv(const FwdShape& s, const TensorPtrs::Layer& L, const FwdWorkspace& ws, int M, cudaStream_t st);
int fwd_attention(const FwdShape& s, const FwdWorkspace& ws, int B, cudaStream_t st);
int fwd_out_proj(const FwdShape& s, const TensorPtrs::Layer& L, const FwdWorkspace& ws, int M,
                 float* partial, cudaStream_t st);
int fwd_fc1(const FwdShape& s, const TensorPtrs::Layer& L, const FwdWorkspace& ws, int M, cudaStream_t st);
int fwd_fc2(const FwdShape& s, const TensorPtrs::Layer& L, const FwdWorkspace& ws, int M, float* partial,
            cudaStream_t st);
int fwd_lm_head(const FwdShape& s, const TensorPtrs& W, const FwdWorkspace& ws, int B, int M, cudaStream_t st);

// Programmatic dependent launch (sm_90+): the kernel may be scheduled while the previous kernel
// on the stream is still running; it must execute pdl_wait() before touching anything the
// previous kernels produce (and before any global write). Weights may be read before the wait.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MPSW_CU(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

inline double now_s(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace mpsw
