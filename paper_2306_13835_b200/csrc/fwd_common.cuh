// Device arithmetic of the non-GEMM forward steps (forward.cu). Every rounding step is spelled out
// with _rn intrinsics (no compiler-chosen FMA contraction), so the arithmetic is fixed by the
// source: a request's logits do not depend on how its batch was launched (eager or graph).
// Numerics: DESIGN.md reading #20 (fp32 residual / LN statistics / softmax, bf16 GEMM operands).
#pragma once

#include "internal.h"

#include <cuda_bf16.h>

namespace mpsw {
namespace fc {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ float to_f(bf16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float to_f(float v) { return v; }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }

template <typename T> __device__ __forceinline__ float4 ld4(const T* p);
template <> __device__ __forceinline__ float4 ld4<float>(const float* p) { return *reinterpret_cast<const float4*>(p); }
template <> __device__ __forceinline__ float4 ld4<bf16>(const bf16* p) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
}

// Four consecutive values rounded to T (RNE for bf16) and written with one vector store.
template <typename T> __device__ __forceinline__ void store4(T* p, float a, float b, float c, float d);
template <> __device__ __forceinline__ void store4<float>(float* p, float a, float b, float c, float d) {
    *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
template <> __device__ __forceinline__ void store4<bf16>(bf16* p, float a, float b, float c, float d) {
    const __nv_bfloat162 lo = __halves2bfloat162(__float2bfloat16_rn(a), __float2bfloat16_rn(b));
    const __nv_bfloat162 hi = __halves2bfloat162(__float2bfloat16_rn(c), __float2bfloat16_rn(d));
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&lo);
    u.y = *reinterpret_cast<const uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(p) = u;
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// LayerNorm (HF OPT: biased variance, eps 1e-5) pieces. A row of h columns is handled as h/4
// float4 groups; "virtual thread" v of a 512-thread row owns groups v, v + 512, v + 1024, ...
constexpr int kLnThreads = 512;

__device__ __forceinline__ float ln_sum4(float4 s) { return __fadd_rn(__fadd_rn(s.x, s.y), __fadd_rn(s.z, s.w)); }

__device__ __forceinline__ float ln_var4(float4 x, float mean) {
    const float a = __fsub_rn(x.x, mean), b = __fsub_rn(x.y, mean), c = __fsub_rn(x.z, mean), d = __fsub_rn(x.w, mean);
    return __fadd_rn(__fadd_rn(__fmul_rn(a, a), __fmul_rn(b, b)), __fadd_rn(__fmul_rn(c, c), __fmul_rn(d, d)));
}

__device__ __forceinline__ float ln_norm(float x, float mean, float den, float g, float b) {
    return __fadd_rn(__fmul_rn(__fdiv_rn(__fsub_rn(x, mean), den), g), b);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Sum of the 16 per-warp partials of a 512-thread row in warp order.
__device__ __forceinline__ float ln_red16(const float* red) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kLnThreads / 32; ++i) s = __fadd_rn(s, red[i]);
    return s;
}

// x = residual + (sum_r partial_r + bias + pos), the pre-LN residual stream value of one float4
// group (TP all-reduce in rank order).
template <typename T>
__device__ __forceinline__ float4 ln_input4(const float* const* peers, int n_peers, size_t off, bool has_bias, float4 bias4,
                                            const T* prow, const float* residual, int j) {
    float4 s = *reinterpret_cast<const float4*>(peers[0] + off);
#pragma unroll
    for (int r = 1; r < 8; ++r)
        if (r < n_peers) s = add4(s, *reinterpret_cast<const float4*>(peers[r] + off));
    if (has_bias) s = add4(s, bias4);
    if (prow) s = add4(s, ld4<T>(prow + j));
    if (residual) s = add4(*reinterpret_cast<const float4*>(residual + off), s);
    return s;
}

// Causal attention of one (request b, head) pair: the rows of request b are
// [seq_start[b], seq_start[b+1]); `warp` of `nwarps` takes query rows warp, warp + nwarps, ...;
// sc = this warp's 128-float score row (L <= 128). qkv is [M, 3*hl] fp32 with q pre-scaled.
template <typename T>
__device__ __forceinline__ void attention_item(const float* __restrict__ qkv, const int32_t* __restrict__ seq_start,
                                               T* __restrict__ o, int hl, int hd, int b, int head, float* sc, int warp,
                                               int nwarps, int lane) {
    const int s0 = seq_start[b], L = seq_start[b + 1] - s0;
    const int ld = 3 * hl;
    // lane owns head dims d = lane + 32u (u < 4, d < hd): any hd <= 128
    for (int i = warp; i < L; i += nwarps) {
        const float* q = qkv + (size_t)(s0 + i) * ld + head * hd;
        float qv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) qv[u] = lane + 32 * u < hd ? q[lane + 32 * u] : 0.f;
        float mx = -INFINITY;
        for (int j = 0; j <= i; ++j) {
            const float* k = qkv + (size_t)(s0 + j) * ld + hl + head * hd;
            float d = 0.f;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (lane + 32 * u < hd) d = __fmaf_rn(qv[u], k[lane + 32 * u], d);
            d = warp_sum(d);
            if (lane == 0) sc[j] = d;
            mx = fmaxf(mx, d);
        }
        __syncwarp();
        float sum = 0.f;
        for (int j = lane; j <= i; j += 32) {
            const float e = expf(__fsub_rn(sc[j], mx));
            sc[j] = e;
            sum = __fadd_rn(sum, e);
        }
        sum = warp_sum(sum);
        __syncwarp();
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int j = 0; j <= i; ++j) {
            const float p = __fdiv_rn(sc[j], sum);
            const float* v = qkv + (size_t)(s0 + j) * ld + 2 * hl + head * hd;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (lane + 32 * u < hd) acc[u] = __fmaf_rn(p, v[lane + 32 * u], acc[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (lane + 32 * u < hd) o[(size_t)(s0 + i) * hl + head * hd + lane + 32 * u] = from_f<T>(acc[u]);
        __syncwarp();
    }
}

}  // namespace fc
}  // namespace mpsw
