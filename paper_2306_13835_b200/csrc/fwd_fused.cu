// Fused persistent layers kernel (sm_100a): all decoder layers of one rank's forward in ONE launch
// for small token counts (M = B*L <= 48; the paper's request shapes, P:138 / P:166, are L = 2 or 8).
//
// Why: at small M the forward is a pure HBM weight stream, and with one kernel per
// op the weight stream stalls at every kernel boundary (7 per layer: the next GEMM can only start
// its activation loads after the previous kernel fully completes). Here the weight
// stream of the whole forward is one continuous TMA sequence per CTA, and only the activation
// operand waits for the data dependency, through device-wide phase counters instead of kernel
// boundaries.
//
// Structure: the grid is the per-op GEMM's persistent grid (2 CTAs per SM, all co-resident; the
// host checks occupancy). Per layer l there are 7 phases P = 7l + k:
//   k = 0 QKV GEMM, 1 attention, 2 out_proj GEMM, 3 residual + bias + LN2, 4 fc1 GEMM (+ReLU),
//   5 fc2 GEMM, 6 residual + bias + next LN (LN1 of layer l+1, or the final LN).
// Every CTA arrives on counter[P] once its writes of phase P are done; phase P's consumers wait
// for counter[P-1] to reach G (per-forward epoch). Warp roles per CTA:
//   * warp 0 lane 0: TMA producer. Weight tiles W[l] (3D tensor maps over the equal-stride layers
//     of the arena) are issued as soon as a ring slot is free, across phases and layers; the
//     activation tile of a unit is issued once its phase's input is complete;
//   * warp 1 lane 0: tcgen05.mma issuer (fp32 accumulators in TMEM, double-buffered);
//   * warps 4..7: GEMM epilogues, stream-K fix-ups, attention and LayerNorm phases.
// The GEMM work split (stream-K over (tile, k-block) units), the fix-up order, the epilogue
// arithmetic, attention and LayerNorm (fwd_common.cuh; the 512-thread LN reduction order is
// reproduced with 128 threads) are exactly those of the per-op kernels, so the fused forward is
// bitwise identical to the per-op forward (tested) and keeps the batch invariance of the logits.
#include "fwd_common.cuh"
#include "tc_common.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace mpsw {

namespace {

using namespace tc;
using namespace fc;

constexpr int kPhases = 7;              // per layer
constexpr int kMaxFusedRows = 48;       // in-kernel fix-up (the per-op kernel switches at Mp >= 64)
constexpr int kMaxFusedLayers = 128;

struct FGemm {
    int nseg, tiles, kb, K, G;
    uint64_t units;
    int N[3], tile0[3], col0[3];
    const bf16* bias[3];                // layer 0; + l * lstride_el per layer (null = none)
    float scale[3];
    int epi;                            // 0 fp32 (acc + bias) * scale, 1 bf16 relu(acc + bias)
    void* out;
    int ldo;
};

struct FusedArgs {
    FGemm gm[4];                        // qkv, out_proj, fc1, fc2
    int n_layers, M, Mp, B, stages, Gmax, nacc, nbuf, hidden, hl, hd, heads;
    int64_t lstride_el;                 // bf16 elements between consecutive layers' tensors
    float* x;                           // residual stream [M, h] fp32
    bf16* a;                            // LN output [M, h]
    float* qkv;                         // [M, 3 hl] fp32
    bf16* o;                            // attention output [M, hl]
    float* partial;                     // row-parallel GEMM output [M, h] fp32 (t = 1: the sum)
    float* tcp;                         // stream-K partial runs [Gmax][2][Mp][128]
    int* counters;                      // per-tile arrival counters (self-resetting)
    const int32_t* seq_start;           // [B + 1]
    const bf16 *o_b, *fc2_b, *ln1_w, *ln1_b, *ln2_w, *ln2_b;   // layer 0
    const bf16 *last_w, *last_b;        // LN after the last layer (final LN, or LN2 of a non-last stage)
    unsigned long long* bar;            // [kPhases * n_layers] phase arrival counters (+1: exit counter)
    unsigned long long target;          // arrivals that complete a phase (= Gmax; counters reset at exit)
    unsigned long long* lnflag;         // [kMaxFusedRows][2][4] LayerNorm exchange stamps
    float* lnx;                         // [kMaxFusedRows][2][16] LayerNorm warp partial sums
    unsigned long long stamp0;          // LN exchange stamps of this launch: stamp0 + instance + 1
    int pf;                             // weight units prefetched into L2 ahead of the smem ring
    unsigned long long* trace;          // dev: [Gmax][phases][2] %globaltimer (phase start, arrival) or null
};

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    return t;
}

// Blocking wait for phase P's counter (bounded: traps after 10 s instead of hanging the GPU).
__device__ __forceinline__ void phase_wait(const FusedArgs& g, int P) {
    const unsigned long long* p = g.bar + P;
    if (ld_acquire(p) >= g.target) return;
    const unsigned long long t0 = globaltimer();
    while (ld_acquire(p) < g.target) {
        __nanosleep(64);
        if (globaltimer() - t0 > 10000000000ull) __trap();
    }
}

__device__ __forceinline__ uint64_t ubeg(const FGemm& m, int c) {
    return c >= m.G ? m.units : (uint64_t)c * m.units / (uint64_t)m.G;
}

__device__ __forceinline__ int cta_of(const FGemm& m, uint64_t u) {
    int c = (int)(u * (uint64_t)m.G / m.units);
    while (c + 1 < m.G && ubeg(m, c + 1) <= u) ++c;
    while (c > 0 && ubeg(m, c) > u) --c;
    return c;
}

__device__ __forceinline__ int seg_of(const FGemm& m, int tile) {
    int si = 0;
    while (si + 1 < m.nseg && tile >= m.tile0[si + 1]) ++si;
    return si;
}

// Position in this CTA's unit stream: layer l, GEMM gi, unit u of [u, ue), ring index i, and
// the unit's (tile, k-block, segment) kept incrementally (no 64-bit divisions per unit in the
// producer / MMA loops); rb = first unit of the current GEMM range.
struct Cursor {
    int l, gi;
    uint32_t u, ue, rb;
    int i, tile, kbi, si;
    int slot;                   // = i % stages
    uint32_t ph;                // = (i / stages) & 1
};

__device__ __forceinline__ void cur_enter(const FusedArgs& g, int c, Cursor& k) {
    const FGemm& m = g.gm[k.gi];
    k.u = (uint32_t)ubeg(m, c);
    k.ue = (uint32_t)ubeg(m, c + 1);
    k.rb = k.u;
    k.tile = (int)(k.u / (uint32_t)m.kb);
    k.kbi = (int)(k.u % (uint32_t)m.kb);
    k.si = seg_of(m, k.tile);
}

__device__ __forceinline__ void cur_fix(const FusedArgs& g, int c, Cursor& k) {
    while (k.l < g.n_layers && k.u >= k.ue) {
        if (++k.gi == 4) { k.gi = 0; ++k.l; }
        if (k.l < g.n_layers) cur_enter(g, c, k);
    }
}

__device__ __forceinline__ Cursor cur_begin(const FusedArgs& g, int c) {
    Cursor k{};
    cur_enter(g, c, k);
    cur_fix(g, c, k);
    return k;
}

__device__ __forceinline__ void cur_next(const FusedArgs& g, int c, Cursor& k) {
    ++k.u;
    ++k.i;
    if (++k.slot == g.stages) {
        k.slot = 0;
        k.ph ^= 1u;
    }
    if (k.u < k.ue) {
        const FGemm& m = g.gm[k.gi];
        if (++k.kbi == m.kb) {
            k.kbi = 0;
            ++k.tile;
            if (k.si + 1 < m.nseg && k.tile >= m.tile0[k.si + 1]) ++k.si;
        }
    } else {
        cur_fix(g, c, k);
    }
}

// compute warps (128 threads) named barrier
__device__ __forceinline__ void cw_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__device__ __forceinline__ void phase_arrive(const FusedArgs& g, int P, int ct) {
    asm volatile("fence.proxy.async.global;" ::: "memory");   // generic writes -> later TMA reads
    cw_sync();
    if (ct == 0) {
        if (g.trace) g.trace[((size_t)blockIdx.x * kPhases * g.n_layers + P) * 2 + 1] = globaltimer();
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(g.bar + P) : "memory");
    }
}

__device__ __forceinline__ void cw_phase_wait(const FusedArgs& g, int P, int ct) {
    if (P >= 0 && ct == 0) phase_wait(g, P);
    if (ct == 0 && g.trace) g.trace[((size_t)blockIdx.x * kPhases * g.n_layers + P + 1) * 2] = globaltimer();
    cw_sync();
}

// residual + bias + LayerNorm of row m, split over 4 CTAs: CTA part q plays the virtual threads
// q*128 + ct of the per-op kernel's 512-thread row (virtual warps 4q .. 4q+3, same lanes), so
// every per-thread and per-warp sum is the per-op kernel's; the 16 warp partials of the mean and
// of the variance are exchanged through global memory (stamped flags) and summed in warp order.
// Parameters (bias, gamma, beta) are loaded before the phase wait (they do not depend on it).
template <int VPT>
struct LnPart {                 // raw bf16 x4 (8 bytes) per column group: 2 registers each
    uint2 bi[VPT], ga[VPT], be[VPT];
};

__device__ __forceinline__ float4 bf4(uint2 u) {
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
}

template <int VPT>
__device__ __forceinline__ void ln_load_params(LnPart<VPT>& P, int h4, int v, const bf16* bias, const bf16* gamma,
                                               const bf16* beta) {
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int j4 = v + i * kLnThreads;
        if (j4 < h4) {
            P.bi[i] = *reinterpret_cast<const uint2*>(bias + 4 * j4);
            P.ga[i] = *reinterpret_cast<const uint2*>(gamma + 4 * j4);
            P.be[i] = *reinterpret_cast<const uint2*>(beta + 4 * j4);
        }
    }
}

// Publish this CTA's 4 warp partials of (row m, pass), then wait for the other 3 parts and return
// the sum of all 16 in warp order.
__device__ __forceinline__ float ln_exchange(const FusedArgs& g, int m, int pass, int q, int ct, float v,
                                             unsigned long long stamp) {
    const int w = ct >> 5, lane = ct & 31;
    float* x = g.lnx + ((size_t)m * 2 + pass) * 16;
    unsigned long long* f = g.lnflag + ((size_t)m * 2 + pass) * 4;
    if (lane == 0) __stcg(x + 4 * q + w, v);
    cw_sync();
    if (ct == 0) asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(f + q), "l"(stamp) : "memory");
    if (ct < 4) {
        const unsigned long long t0 = globaltimer();
        while (ld_acquire(f + ct) != stamp)
            if (globaltimer() - t0 > 10000000000ull) __trap();
    }
    cw_sync();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kLnThreads / 32; ++i) s = __fadd_rn(s, __ldcg(x + i));
    return s;
}

template <int VPT>
__device__ __forceinline__ void ln_part(const FusedArgs& g, int m, int q, const LnPart<VPT>& P, int ct, unsigned long long stamp) {
    const int h = g.hidden, h4 = h / 4, v = q * 128 + ct;
    const size_t row = (size_t)m * h;
    float4 xs[VPT], pv[VPT], rv[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int j4 = v + i * kLnThreads;
        if (j4 < h4) {
            pv[i] = __ldcg(reinterpret_cast<const float4*>(g.partial + row) + j4);
            rv[i] = __ldcg(reinterpret_cast<const float4*>(g.x + row) + j4);
        }
    }
    float ls = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int j4 = v + i * kLnThreads;
        if (j4 < h4) {
            // = ln_input4 with one peer: (partial + bias), then residual + that
            const float4 sv = add4(rv[i], add4(pv[i], bf4(P.bi[i])));
            xs[i] = sv;
            reinterpret_cast<float4*>(g.x + row)[j4] = sv;
            ls = __fadd_rn(ls, ln_sum4(sv));
        }
    }
    const float mean = __fdiv_rn(ln_exchange(g, m, 0, q, ct, warp_sum(ls), stamp), (float)h);
    float lv = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i)
        if (v + i * kLnThreads < h4) lv = __fadd_rn(lv, ln_var4(xs[i], mean));
    const float var = __fdiv_rn(ln_exchange(g, m, 1, q, ct, warp_sum(lv), stamp), (float)h);
    const float den = __fsqrt_rn(__fadd_rn(var, 1e-5f));
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int j4 = v + i * kLnThreads;
        if (j4 < h4) {
            const float4 ga = bf4(P.ga[i]), be = bf4(P.be[i]);
            bf16* o = g.a + row + 4 * j4;
            o[0] = __float2bfloat16_rn(ln_norm(xs[i].x, mean, den, ga.x, be.x));
            o[1] = __float2bfloat16_rn(ln_norm(xs[i].y, mean, den, ga.y, be.y));
            o[2] = __float2bfloat16_rn(ln_norm(xs[i].z, mean, den, ga.z, be.z));
            o[3] = __float2bfloat16_rn(ln_norm(xs[i].w, mean, den, ga.w, be.w));
        }
    }
}

// LayerNorm phase P of layer l (k = 3: + out_proj bias, LN2; k = 6: + fc2 bias, next LN1 / last).
template <int VPT>
__device__ __forceinline__ void ln_phase(const FusedArgs& g, int l, int k, int P, int c, int ct) {
    const int64_t lo = (int64_t)l * g.lstride_el;
    const bool lastl = l + 1 == g.n_layers;
    const bf16* bias = (k == 3 ? g.o_b : g.fc2_b) + lo;
    const bf16* gam = k == 3 ? g.ln2_w + lo : (lastl ? g.last_w : g.ln1_w + lo + g.lstride_el);
    const bf16* bet = k == 3 ? g.ln2_b + lo : (lastl ? g.last_b : g.ln1_b + lo + g.lstride_el);
    const unsigned long long stamp = g.stamp0 + (unsigned long long)(2 * l + (k == 6 ? 1 : 0)) + 1;
    if (c < 4 * g.M) {
        const int m = c >> 2, q = c & 3;
        LnPart<VPT> prm;
        ln_load_params<VPT>(prm, g.hidden / 4, q * 128 + ct, bias, gam, bet);
        cw_phase_wait(g, P - 1, ct);
        ln_part<VPT>(g, m, q, prm, ct, stamp);
    } else {
        cw_phase_wait(g, P - 1, ct);
    }
}

// <= 128 registers: two 256-thread CTAs per SM (64K registers)
__global__ void __maxnreg__(128)
fused_layers_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk,
                    const __grid_constant__ CUtensorMap mv, const __grid_constant__ CUtensorMap mo,
                    const __grid_constant__ CUtensorMap m1, const __grid_constant__ CUtensorMap m2,
                    const __grid_constant__ CUtensorMap xa, const __grid_constant__ CUtensorMap xo,
                    const __grid_constant__ CUtensorMap xr, const __grid_constant__ FusedArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t tile_b_bytes = (uint32_t)g.Mp * kBK * 2;
    const int S = g.stages;
    uint8_t* sa = smem;
    uint8_t* sb = smem + S * kTileABytes;
    uint64_t* full = (uint64_t*)(sb + S * tile_b_bytes);
    uint64_t* empty = full + kMaxStages;
    uint64_t* tmem_full = empty + kMaxStages;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_slot = (uint32_t*)(tmem_empty + 2);
    __shared__ float sc[4][128];
    __shared__ int s_last;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int nacc = g.nacc;
    const uint32_t nbuf = (uint32_t)g.nbuf, ncols = (uint32_t)nacc * nbuf;
    pdl_trigger();

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mq) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mk) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mv) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mo) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&m1) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&m2) : "memory");
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tmem_full[b], 1);
            mbar_init(&tmem_empty[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {                                   // ---- TMA producer
            auto wmap = [&](int gi, int si) -> const CUtensorMap* {
                if (gi == 0) return si == 0 ? &mq : (si == 1 ? &mk : &mv);
                return gi == 1 ? &mo : (gi == 2 ? &m1 : &m2);
            };
            auto xmap = [&](int gi) -> const CUtensorMap* { return gi == 0 || gi == 2 ? &xa : (gi == 1 ? &xo : &xr); };
            auto issue_w = [&](const Cursor& k) {
                const FGemm& m = g.gm[k.gi];
                const int s = k.slot;
                mbar_expect_tx(&full[s], kTileABytes + tile_b_bytes);
                tma_load_3d(sa + s * kTileABytes, wmap(k.gi, k.si), &full[s], k.kbi * kBK, (k.tile - m.tile0[k.si]) * kBN,
                            k.l);
            };
            Cursor w = cur_begin(g, c), x = w;
            // weights do not depend on the previous kernel: fill the ring before griddepcontrol.wait
            while (w.l < g.n_layers && w.i < S) {
                issue_w(w);
                cur_next(g, c, w);
            }
            pdl_wait();
            int ready = 0;                                 // phases < ready are known complete
            // L2 prefetch cursor: weight tiles up to g.pf units beyond the ring are requested into
            // L2, so HBM keeps streaming while the ring waits on a phase (LN / attention / tails)
            Cursor pfc = w;
            while (x.l < g.n_layers) {
                bool prog = false;
                if (pfc.l < g.n_layers && pfc.i < w.i + g.pf) {
                    if (pfc.i >= w.i) {
                        const FGemm& m = g.gm[pfc.gi];
                        tma_prefetch_l2_3d(wmap(pfc.gi, pfc.si), pfc.kbi * kBK, (pfc.tile - m.tile0[pfc.si]) * kBN, pfc.l);
                    }
                    cur_next(g, c, pfc);
                }
                if (x.i < w.i) {                           // activation tile of unit x
                    const int P = kPhases * x.l + (x.gi == 0 ? 0 : (x.gi == 1 ? 2 : (x.gi == 2 ? 4 : 5)));
                    bool ok = P <= ready;
                    if (!ok && ld_acquire(g.bar + (P - 1)) >= g.target) {
                        ready = P;
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        ok = true;
                    }
                    if (ok) {
                        tma_load_2d(sb + x.slot * tile_b_bytes, xmap(x.gi), &full[x.slot], x.kbi * kBK, 0);
                        cur_next(g, c, x);
                        prog = true;
                    }
                }
                if (w.l < g.n_layers && mbar_test(&empty[w.slot], w.ph ^ 1u)) {
                    issue_w(w);
                    cur_next(g, c, w);
                    prog = true;
                }
                if (!prog) __nanosleep(20);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {                                   // ---- MMA issuer
            const uint32_t idesc = umma_idesc(g.Mp);
            int run = 0;
            uint32_t tmem_d = tmem_base;
            Cursor k = cur_begin(g, c);
            while (k.l < g.n_layers) {
                const FGemm& m = g.gm[k.gi];
                const int s = k.slot;
                const uint32_t ph = k.ph;
                const bool first = k.u == k.rb || k.kbi == 0;
                const bool last = k.u + 1 == k.ue || k.kbi == m.kb - 1;
                if (first) {
                    const int b = nacc == 2 ? (run & 1) : 0;
                    const int use = nacc == 2 ? (run >> 1) : run;
                    mbar_wait(&tmem_empty[b], ((uint32_t)use & 1u) ^ 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    tmem_d = tmem_base + (uint32_t)b * nbuf;
                }
                mbar_wait(&full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t a0 = smem_u32(sa + s * kTileABytes), b0 = smem_u32(sb + s * tile_b_bytes);
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk)
                    umma_bf16(tmem_d, umma_desc(a0 + kk * 32), umma_desc(b0 + kk * 32), idesc, (!first || kk) ? 1u : 0u);
                umma_commit(&empty[s]);
                if (last) {
                    umma_commit(&tmem_full[nacc == 2 ? (run & 1) : 0]);
                    ++run;
                }
                cur_next(g, c, k);
            }
        }
    } else if (warp >= 4) {                                // ---- epilogue / attention / LayerNorm
        pdl_wait();
        const int ct = threadIdx.x - 128;
        const int q = warp - 4;
        const int row = q * 32 + lane;                     // weight row within the 128-row tile
        int run = 0;
        for (int l = 0; l < g.n_layers; ++l) {
            const int64_t lo = (int64_t)l * g.lstride_el;
            for (int k = 0; k < kPhases; ++k) {
                const int P = kPhases * l + k;
                const int gi = k == 0 ? 0 : (k == 2 ? 1 : (k == 4 ? 2 : (k == 5 ? 3 : -1)));
                if (k != 3 && k != 6) cw_phase_wait(g, P - 1, ct);
                if (gi >= 0) {
                    const FGemm& m = g.gm[gi];
                    const uint64_t u0 = ubeg(m, c), u1 = ubeg(m, c + 1);
                    const int cfirst_run_tile = (int)(u0 / m.kb);
                    for (uint64_t u = u0; u < u1;) {
                        const int tile = (int)(u / m.kb);
                        const uint64_t tend = (uint64_t)(tile + 1) * m.kb;
                        const uint64_t rend = u1 < tend ? u1 : tend;
                        const int si = seg_of(m, tile);
                        const int n = (tile - m.tile0[si]) * kBN + row;
                        const bool nvalid = n < m.N[si];
                        const bf16* bias = m.bias[si] ? m.bias[si] + lo : nullptr;
                        const float bias_n = (bias && nvalid) ? __bfloat162float(bias[n]) : 0.f;
                        const int c_first = cta_of(m, (uint64_t)tile * m.kb), c_last = cta_of(m, tend - 1);
                        const bool whole = c_first == c_last;
                        const int which = tile == cfirst_run_tile ? 0 : 1;
                        float* prow = g.tcp + ((size_t)c * 2 + which) * (size_t)g.Mp * kBN + row;
                        const int b = nacc == 2 ? (run & 1) : 0;
                        const int use = nacc == 2 ? (run >> 1) : run;
                        mbar_wait(&tmem_full[b], (uint32_t)use & 1u);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        float v[16];
                        for (int col = 0; col < g.Mp; col += 16) {
                            tmem_ld16(tmem_base + (uint32_t)b * nbuf + ((uint32_t)(q * 32) << 16) + (uint32_t)col, v);
                            if (!whole) {
#pragma unroll
                                for (int j = 0; j < 16; ++j) prow[(size_t)(col + j) * kBN] = v[j];
                            } else if (nvalid) {
#pragma unroll
                                for (int j = 0; j < 16; ++j)
                                    if (col + j < g.M)
                                        epi_value_store(m.epi, m.out, (size_t)(col + j) * m.ldo + m.col0[si] + n, v[j],
                                                        bias != nullptr, bias_n, m.scale[si]);
                            }
                        }
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0)
                            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[b])) : "memory");
                        ++run;
                        if (!whole) {                      // fix-up: last arriving CTA sums the runs in k order
                            cw_sync();
                            if (ct == 0) {
                                int old;
                                asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                                             : "=r"(old)
                                             : "l"(&g.counters[tile])
                                             : "memory");
                                s_last = old == c_last - c_first;
                            }
                            cw_sync();
                            if (s_last) {
                                if (nvalid) {
                                    const int wh0 = (int)(ubeg(m, c_first) / m.kb) != tile ? 1 : 0;
                                    for (int m0 = 0; m0 < g.M; m0 += 8) {
                                        float acc[8];
#pragma unroll
                                        for (int j = 0; j < 8; ++j) acc[j] = 0.f;
                                        for (int cc = c_first; cc <= c_last; ++cc) {
                                            const int wh = cc == c_first ? wh0 : 0;
                                            const float* p = g.tcp + ((size_t)cc * 2 + wh) * (size_t)g.Mp * kBN + row +
                                                             (size_t)m0 * kBN;
                                            float t[8];
#pragma unroll
                                            for (int j = 0; j < 8; ++j) t[j] = __ldcg(p + j * kBN);
#pragma unroll
                                            for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], t[j]);
                                        }
#pragma unroll
                                        for (int j = 0; j < 8; ++j)
                                            if (m0 + j < g.M)
                                                epi_value_store(m.epi, m.out, (size_t)(m0 + j) * m.ldo + m.col0[si] + n,
                                                                acc[j], bias != nullptr, bias_n, m.scale[si]);
                                    }
                                }
                                if (ct == 0) g.counters[tile] = 0;
                            }
                            cw_sync();
                        }
                        u = rend;
                    }
                } else if (k == 1) {                       // attention: (request, head) items over CTAs
                    for (int it = c; it < g.B * g.heads; it += g.Gmax)
                        attention_item<bf16>(g.qkv, g.seq_start, g.o, g.hl, g.hd, it % g.B, it / g.B, sc[q], q, 4, lane);
                } else {                                   // residual + bias + LayerNorm: 4 CTAs per row
                    const int vpt = (g.hidden / 4 + kLnThreads - 1) / kLnThreads;
                    if (vpt <= 1) ln_phase<1>(g, l, k, P, c, ct);
                    else if (vpt == 2) ln_phase<2>(g, l, k, P, c, ct);
                    else ln_phase<3>(g, l, k, P, c, ct);
                }
                phase_arrive(g, P, ct);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols));
    // The last CTA to exit resets the phase counters for the next launch: every other CTA has
    // passed all its waits by then, and the next launch touches them only after griddepcontrol.wait.
    if (threadIdx.x == 0) {
        unsigned long long* ex = g.bar + kPhases * kMaxFusedLayers;
        unsigned long long old;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(ex) : "memory");
        if (old == (unsigned long long)g.Gmax - 1) {
            for (int P = 0; P < kPhases * g.n_layers; ++P) g.bar[P] = 0;
            *ex = 0;
        }
    }
}

struct Map3Key {
    const void* p;
    uint64_t rows, K, layers, stride;
    uint32_t box;
    bool operator==(const Map3Key& o) const {
        return p == o.p && rows == o.rows && K == o.K && layers == o.layers && stride == o.stride && box == o.box;
    }
};
struct Map3KeyHash {
    size_t operator()(const Map3Key& k) const {
        return std::hash<const void*>()(k.p) ^ (k.rows * 0x9E3779B97F4A7C15ull) ^ (k.K << 20) ^ (k.layers << 40) ^
               (k.stride * 31) ^ k.box;
    }
};

const CUtensorMap& map3(const void* p, uint64_t rows, uint64_t K, uint64_t layers, uint64_t stride, uint32_t box) {
    thread_local std::unordered_map<Map3Key, CUtensorMap, Map3KeyHash> cache;
    const Map3Key k{p, rows, K, layers, stride, box};
    auto it = cache.find(k);
    if (it != cache.end()) return it->second;
    return cache.emplace(k, tc_make_map_3d(p, rows, K, layers, stride, box)).first->second;
}

// CTAs of the fused kernel that fit on one SM at once. cudaOccupancyMaxActiveBlocksPerMultiprocessor
// reports 1 for any kernel that allocates TMEM, but the hardware co-schedules two such 256-thread
// CTAs per SM when registers, shared memory and TMEM columns allow it (measured on B200 with
// tools/occ_probe.cu: 2 x 148 spinning CTAs finish in one period). The grid spins on device-wide
// counters, so this is checked from the resource counts, conservatively.
int fused_occupancy(int dev) {
    static int occ[64];
    static bool done[64];
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) return 0;
    if (!done[dev]) {
        done[dev] = true;
        size_t smem = 0;                               // ring depth differs per Mp: take the largest
        for (int mp = 16; mp <= kMaxFusedRows; mp += 16) smem = std::max(smem, tc_smem_bytes(mp));
        cudaFuncAttributes fa{};
        int regs_sm = 0, smem_sm = 0, reserved = 0;
        if (cudaFuncSetAttribute(fused_layers_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
            cudaFuncSetAttribute(fused_layers_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100) != cudaSuccess ||
            cudaFuncGetAttributes(&fa, fused_layers_kernel) != cudaSuccess ||
            cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess) {
            occ[dev] = 0;
        } else {
            const size_t per_smem = smem + fa.sharedSizeBytes + (size_t)reserved;
            const int per_regs = ((fa.numRegs + 7) / 8 * 8) * kThreads;
            const int by_smem = (int)((size_t)smem_sm / per_smem), by_regs = regs_sm / per_regs;
            const int by_tmem = 512 / (2 * 64);        // <= 2 accumulators of <= 64 columns each
            occ[dev] = std::min(std::min(by_smem, by_regs), by_tmem);
            if (fa.maxThreadsPerBlock < kThreads) occ[dev] = 0;
        }
        if (getenv("MPSW_FUSED_DEBUG"))
            fprintf(stderr, "[mpsw] fused CTAs per SM %d (regs %d, smem %zu + %zu)\n", occ[dev], fa.numRegs, smem,
                    fa.sharedSizeBytes);
        cudaGetLastError();
    }
    return occ[dev];
}

// The grid spins on device-wide phase counters, so two fused launches must never share a GPU
// at the same time (each could hold half the SMs). Every launch records a per-device event; a
// launch from a different stream than the previous one on that device waits for it first (the
// common single-stream case keeps its programmatic-dependent-launch overlap).
struct FusedChain {
    cudaEvent_t ev = nullptr;
    cudaStream_t last = nullptr;
};

std::mutex& fused_mu() {
    static std::mutex mu;
    return mu;
}

FusedChain& fused_chain(int dev) {
    static std::unordered_map<int, FusedChain> m;
    FusedChain& f = m[dev];
    if (!f.ev) MPSW_CU(cudaEventCreateWithFlags(&f.ev, cudaEventDisableTiming));
    return f;
}

}  // namespace

// workspace words (u64): phase counters, exit counter, LN stamps, LN partial sums (floats)
constexpr size_t kLnFlagOff = kPhases * kMaxFusedLayers + 8;
constexpr size_t kLnxOff = kLnFlagOff + kMaxFusedRows * 2 * 4;
size_t fused_bar_count() { return kLnxOff + kMaxFusedRows * 2 * 16 / 2; }

// Launch the fused layers kernel for layers [0, W.layers.size()) of this rank's stage, or return
// 0 (nothing launched) when the shape is not eligible; the caller then runs the per-op kernels.
// Preconditions (as for the per-op path): ws.x holds the residual stream and ws.a the LN1 output
// of the first layer. On return (stream order) ws.x / ws.a hold the residual stream and the LN
// output after the last layer (final LN `last_w/last_b`).
int fwd_layers_fused(const FwdShape& s, const TensorPtrs& W, FwdWorkspace& ws, int B, int M, const void* last_w,
                     const void* last_b, cudaStream_t st) {
    const int L = (int)W.layers.size();
    static const bool dbg = getenv("MPSW_FUSED_DEBUG") != nullptr;
    auto no = [&](const char* why) {
        if (dbg) fprintf(stderr, "[mpsw] fused layers kernel not used: %s\n", why);
        return 0;
    };
    if (tc_pair()) return no("CTA-pair GEMM mode (the fused kernel reproduces the single-CTA split only)");
    if (s.dtype != MPSW_BF16 || s.gemm_impl != 3) return no("dtype / gemm_impl (opt-in: 3)");
    if (s.tp != 1) return no("tp > 1");
    if (M < 1 || M > kMaxFusedRows) return no("M out of range");
    if (L < 1 || L > kMaxFusedLayers || s.head_dim > 128 || s.hidden % 8 || s.hidden > 3 * 4 * kLnThreads ||
        s.ffn_local % 8)
        return no("shape");
    if (!ws.fused_bar) return no("no counters");
    const int hl = s.heads_local * s.head_dim;
    if (hl % 8) return no("hl % 8");
    const int Gmax = tc_ctas_per_sm() * sm_count();
    int dev = 0;
    MPSW_CU(cudaGetDevice(&dev));
    if (tc_ctas_per_sm() != 2) return no("ctas per SM != 2");
    if (fused_occupancy(dev) < 2) return no("occupancy < 2 CTAs per SM");
    // every per-layer tensor must sit at the same stride (canonical arena layout, reading #12)
    int64_t stride = 0;
    if (L > 1) stride = (const char*)W.layers[1].q_w - (const char*)W.layers[0].q_w;
    for (int l = 0; l < L; ++l) {
        const auto& a = W.layers[l];
        const auto& z = W.layers[0];
        const void* pa[16] = {a.k_w, a.k_b, a.v_w, a.v_b, a.q_w, a.q_b, a.o_w, a.o_b,
                              a.ln1_w, a.ln1_b, a.fc1_w, a.fc1_b, a.fc2_w, a.fc2_b, a.ln2_w, a.ln2_b};
        const void* pz[16] = {z.k_w, z.k_b, z.v_w, z.v_b, z.q_w, z.q_b, z.o_w, z.o_b,
                              z.ln1_w, z.ln1_b, z.fc1_w, z.fc1_b, z.fc2_w, z.fc2_b, z.ln2_w, z.ln2_b};
        for (int i = 0; i < 16; ++i)
            if (!pa[i] || (const char*)pa[i] - (const char*)pz[i] != (int64_t)l * stride) return no("layer stride");
    }
    if (stride % 16 || (L > 1 && stride <= 0)) return no("stride alignment");
    const uint64_t lstride = L > 1 ? (uint64_t)stride : 16;
    const int Mp = std::max(16, (M + 15) / 16 * 16);
    const int h = s.hidden, ff = s.ffn_local;

    FusedArgs g{};
    auto gemm = [&](FGemm& m, int nseg, const int* N, const void* const* bias, const float* scale, const int* col0, int K,
                    int epi, void* out, int ldo) {
        m.nseg = nseg;
        int tiles = 0;
        for (int i = 0; i < nseg; ++i) {
            m.N[i] = N[i];
            m.tile0[i] = tiles;
            m.col0[i] = col0[i];
            m.bias[i] = (const bf16*)bias[i];
            m.scale[i] = scale[i];
            tiles += (N[i] + kBN - 1) / kBN;
        }
        m.tiles = tiles;
        m.K = K;
        m.kb = (K + kBK - 1) / kBK;
        m.units = (uint64_t)tiles * m.kb;
        m.G = tc_grid_tiles(tiles, K);                           // = the per-op kernel's grid
        m.epi = epi;
        m.out = out;
        m.ldo = ldo;
    };
    const auto& L0 = W.layers[0];
    {
        const int N[3] = {hl, hl, hl}, col0[3] = {0, hl, 2 * hl};
        const void* b[3] = {L0.q_b, L0.k_b, L0.v_b};
        const float sc[3] = {(float)(1.0 / sqrt((double)s.head_dim)), 1.0f, 1.0f};
        gemm(g.gm[0], 3, N, b, sc, col0, h, 0, ws.qkv, 3 * hl);
    }
    {
        const int N[1] = {h}, col0[1] = {0};
        const void* b[1] = {nullptr};
        const float sc[1] = {1.0f};
        gemm(g.gm[1], 1, N, b, sc, col0, hl, 0, ws.partial[0], h);
        gemm(g.gm[3], 1, N, b, sc, col0, ff, 0, ws.partial[0], h);
    }
    {
        const int N[1] = {ff}, col0[1] = {0};
        const void* b[1] = {L0.fc1_b};
        const float sc[1] = {1.0f};
        gemm(g.gm[2], 1, N, b, sc, col0, h, 1, ws.r, ff);
    }
    for (const FGemm& m : g.gm)                    // split-K partials / counters of the workspace
        if (tc_partial_floats(m.tiles * kBN, m.K, Mp) > ws.tc_partial_cap || m.tiles > ws.tc_counters_cap)
            return no("tcgen05 workspace too small");
    // Launch only the CTAs that have work: the largest GEMM grid, and 4 per row for the LayerNorm
    // phases. Every CTA takes part in every phase barrier, so small models (OPT-125M: GEMM grids
    // of <= 36 CTAs) would otherwise pay 296-way barriers for nothing.
    int Gl = 4 * M;
    for (const FGemm& m : g.gm) Gl = std::max(Gl, m.G);
    Gl = std::min(Gl, Gmax);
    g.n_layers = L;
    g.M = M;
    g.Mp = Mp;
    g.B = B;
    g.stages = tc_stages(Mp);
    g.Gmax = Gl;
    int nbuf = 32;
    while (nbuf < Mp) nbuf <<= 1;
    g.nbuf = nbuf;
    g.nacc = 2 * nbuf * 2 <= 512 ? 2 : 1;
    g.hidden = h;
    g.hl = hl;
    g.hd = s.head_dim;
    g.heads = s.heads_local;
    g.lstride_el = (int64_t)(L > 1 ? stride / 2 : 0);
    g.x = ws.x;
    g.a = (bf16*)ws.a;
    g.qkv = ws.qkv;
    g.o = (bf16*)ws.o;
    g.partial = ws.partial[0];
    g.tcp = ws.tc_partial;
    g.counters = ws.tc_counters;
    g.seq_start = ws.meta;
    g.o_b = (const bf16*)L0.o_b;
    g.fc2_b = (const bf16*)L0.fc2_b;
    g.ln1_w = (const bf16*)L0.ln1_w;
    g.ln1_b = (const bf16*)L0.ln1_b;
    g.ln2_w = (const bf16*)L0.ln2_w;
    g.ln2_b = (const bf16*)L0.ln2_b;
    g.last_w = (const bf16*)last_w;
    g.last_b = (const bf16*)last_b;
    g.bar = ws.fused_bar;
    // dev instrumentation: MPSW_FUSED_TRACE=path appends the per-CTA phase stamps of one launch
    static const char* trace_path = getenv("MPSW_FUSED_TRACE");
    unsigned long long* dT = nullptr;
    const size_t nT = (size_t)Gl * kPhases * L * 2;
    if (trace_path) {
        MPSW_CU(cudaMalloc(&dT, nT * 8));
        MPSW_CU(cudaMemsetAsync(dT, 0, nT * 8, st));
    }
    g.trace = dT;
    ws.fused_epoch += 1;
    g.target = (unsigned long long)Gl;
    g.lnflag = ws.fused_bar + kLnFlagOff;
    g.lnx = reinterpret_cast<float*>(ws.fused_bar + kLnxOff);
    g.stamp0 = (unsigned long long)ws.fused_epoch * (2 * kMaxFusedLayers + 2);
    static const int pf = getenv("MPSW_FUSED_PF") ? atoi(getenv("MPSW_FUSED_PF")) : 0;
    g.pf = pf;

    const CUtensorMap& mq = map3(L0.q_w, hl, h, L, lstride, kBN);
    const CUtensorMap& mk = map3(L0.k_w, hl, h, L, lstride, kBN);
    const CUtensorMap& mv = map3(L0.v_w, hl, h, L, lstride, kBN);
    const CUtensorMap& mo = map3(L0.o_w, h, hl, L, lstride, kBN);
    const CUtensorMap& m1 = map3(L0.fc1_w, ff, h, L, lstride, kBN);
    const CUtensorMap& m2 = map3(L0.fc2_w, h, ff, L, lstride, kBN);
    const CUtensorMap xa = tc_make_map(ws.a, (uint64_t)s.max_rows, h, (uint32_t)Mp);
    const CUtensorMap xo = tc_make_map(ws.o, (uint64_t)s.max_rows, hl, (uint32_t)Mp);
    const CUtensorMap xr = tc_make_map(ws.r, (uint64_t)s.max_rows, ff, (uint32_t)Mp);
    const size_t smem = tc_smem_bytes(Mp);
    std::lock_guard<std::mutex> lk(fused_mu());
    FusedChain& ch = fused_chain(dev);
    if (ch.last && ch.last != st) MPSW_CU(cudaStreamWaitEvent(st, ch.ev, 0));
    try {
        launch_pdl(fused_layers_kernel, Gl, kThreads, smem, st, mq, mk, mv, mo, m1, m2, xa, xo, xr, g);
    } catch (const Error& e) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, fused_layers_kernel);
        throw Error(e.status, std::string("fused layers kernel launch (grid ") + std::to_string(Gl) + ", smem " +
                                  std::to_string(smem) + ", params " + std::to_string(sizeof(FusedArgs) + 9 * sizeof(CUtensorMap)) +
                                  ", max threads " + std::to_string(fa.maxThreadsPerBlock) + ", max dyn smem " +
                                  std::to_string(fa.maxDynamicSharedSizeBytes) + "): " + e.what());
    }
    MPSW_CU(cudaGetLastError());
    MPSW_CU(cudaEventRecord(ch.ev, st));
    ch.last = st;
    if (dT) {
        std::vector<unsigned long long> hv(nT);
        MPSW_CU(cudaStreamSynchronize(st));
        MPSW_CU(cudaMemcpy(hv.data(), dT, nT * 8, cudaMemcpyDeviceToHost));
        cudaFree(dT);
        if (FILE* f = fopen(trace_path, "a")) {
            fprintf(f, "{\"M\":%d,\"L\":%d,\"G\":%d,\"h\":%d,\"t\":[", M, L, Gl, h);
            for (size_t i = 0; i < nT; ++i) fprintf(f, "%s%llu", i ? "," : "", hv[i]);
            fprintf(f, "]}\n");
            fclose(f);
        }
    }
    return 1;
}

}  // namespace mpsw
