// tcgen05 + TMA weight-streaming GEMM for sm_100a (bf16 in, fp32 accumulate in TMEM).
//
// out[m, n] = epilogue( sum_k X[m, k] * W[n, k] ),  W = [N, K] row-major weight (K contiguous),
// X = [M, K] row-major activations, M = B*L tokens (<= 256).
//
// Swap-AB: the weight tile is the MMA's A operand (128 weight rows fill the 128-lane MMA M),
// the few tokens are the B operand (MMA N = M rounded up to 16), so the tensor core is fed at
// any batch size and the kernel is a pure HBM weight stream (arithmetic intensity ~M flop/B):
//   * warp 0 (one elected thread): TMA producer, cp.async.bulk.tensor 2D loads of the W tile
//     [128 x 64] and X tile [Mp x 64] (128B swizzle) into a kStages-deep smem ring;
//   * warp 1 (one elected thread): tcgen05.mma.cta_group::1.kind::f16, 4 x (K=16) per stage,
//     accumulator D[128 x Mp] fp32 in TMEM; tcgen05.commit frees the smem stage;
//   * warp 2: TMEM allocator; warps 4..7: epilogue (tcgen05.ld 32x32b, lane = weight row).
// Split-K over CTAs (stream-K over (tile pair, k-block) units) is chosen from (N, K) only —
// never from M — and the partial sums of a split tile are reduced in fixed split order (by its
// last-arriving CTA below 64 padded tokens, by tc_fixup_kernel from 64), so results are
// deterministic and bitwise batch-invariant. The two tiles of a pair run on two independent CTAs,
// or from 192 padded tokens on a CTA pair (cta_group::2): same bits. Weights are streamed with an
// L2 evict_first policy, the token tile and the partials with evict_last.
#include "tc_common.cuh"

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

namespace mpsw {

namespace {

using namespace tc;

struct TcSeg {
    int N;              // rows of this segment's weight
    int tile0;          // first tile index of the segment
    const __nv_bfloat16* bias;
    float scale;
    int out_col0;
};

struct TcArgs {
    TcSeg seg[3];
    int nseg, tiles, kb, K, M, Mp, stages, G;
    uint64_t units;              // work units: unit tiles (tiles, or tile pairs) * kb
    int vw;                      // workers per CTA (or CTA pair): consecutive ranges, one weight stream
    int epi;                     // 0: fp32 out (bias, scale); 1: bf16 out relu(acc + bias)
    void* out;
    int ldo;
    const int32_t* row_of_m;     // optional: output row for token m (-1 = drop); lm_head
    float* partial;              // [G][kT][2][Mp][128]: a worker's first / last partial run per tile (row fastest)
    int* counters;               // [tiles], self-resetting
    int ext_fixup;               // 1: split tiles are reduced by tc_fixup_kernel, not in-kernel
    int nacc;                    // TMEM accumulator buffers (2 = epilogue overlaps the next run)
    unsigned long long* trace;   // dev: [CTAs][8] %globaltimer stamps per CTA phase, or null
    int l2_prefetch;             // weight units per CTA prefetched into L2 before griddepcontrol.wait
    int l2hint;                  // 1: weights evict_first, token tile and partials evict_last in L2
};

__device__ __forceinline__ void stamp(const TcArgs& g, int c, int i) {
    if (g.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
        g.trace[c * 8 + i] = t;
    }
}

// Stream-K work split: worker w owns units [ubeg(w), ubeg(w+1)) of the linearised (unit tile,
// k-block) space. Depends only on (units, G) — never on M — so it is batch-invariant.
// 32-bit arithmetic: units * G < 2^32 (checked on the host); 64-bit divisions cost ~100
// instructions each and sat in front of every fix-up load.
__device__ __forceinline__ uint64_t ubeg(const TcArgs& g, int c) { return (uint32_t)c * (uint32_t)g.units / (uint32_t)g.G; }

__device__ __forceinline__ int cta_of(const TcArgs& g, uint64_t u) {
    int c = (int)((uint32_t)u * (uint32_t)g.G / (uint32_t)g.units);
    while (c + 1 < g.G && ubeg(g, c + 1) <= u) ++c;
    while (c > 0 && ubeg(g, c) > u) --c;
    return c;
}

// Tiles per work unit: kT = 1 (unit = (tile, k-block)) or 2 (unit = (tile pair, k-block); tile
// 2p + r of pair p is the pair's tile r).
template <int kT> struct TileMap {
    __device__ static int tile(uint64_t u, int kb, int r) { return (int)(u / kb) * kT + r; }
    __device__ static int slot(int w, int r) { return w * kT + r; }   // partial slots of worker w, tile r of a unit
};

// Partial run of worker cc on a split tile: slot 0 if the tile is cc's first unit tile, else 1
// (a worker touches at most two split unit tiles: where its range starts and where it ends).
// first_wh: the slot of c_first's run (first_slot below), computed once per tile.
template <int kT>
__device__ __forceinline__ const float* partial_run(const TcArgs& g, int cc, int c_first, int first_wh, int r, int row) {
    const int wh = cc == c_first ? first_wh : 0;
    return g.partial + ((size_t)TileMap<kT>::slot(cc, r) * 2 + wh) * (size_t)g.Mp * kBN + row;
}
__device__ __forceinline__ int first_slot(const TcArgs& g, int c_first, int unit_tile) {
    return (int)((uint32_t)ubeg(g, c_first) / (uint32_t)g.kb) != unit_tile ? 1 : 0;
}

__device__ __forceinline__ void epi_store(const TcArgs& g, const TcSeg& seg, int n, int m, float x, float bias_n) {
    const int orow = g.row_of_m ? g.row_of_m[m] : m;
    if (orow < 0) return;
    epi_value_store(g.epi, g.out, (size_t)orow * g.ldo + seg.out_col0 + n, x, seg.bias != nullptr, bias_n, seg.scale);
}

__device__ __forceinline__ int seg_of(const TcArgs& g, int tile) {
    int si = 0;
    while (si + 1 < g.nseg && tile >= g.seg[si + 1].tile0) ++si;
    return si;
}

// ---- CTA-pair (cta_group::2) primitives
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem variable in the pair's leader (CTA rank 0)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(a) : "r"(smem_u32(p)));
    return a;
}
// TMA load into this CTA's smem whose completion bytes count on the LEADER's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_leader, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(bar_leader), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair_hint(void* dst, const CUtensorMap* map, uint32_t bar_leader, int c0, int c1,
                                                      uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(bar_leader), "r"(c0), "r"(c1), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// MMA completion arrives on the mbarrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "h"((uint16_t)3)
                 : "memory");
}

// One kernel, three executions of two splits:
//  * kT = 1: unit = (tile, k-block); one CTA per worker, tcgen05.mma.cta_group::1 with M = 128
//    reads its W tile [128 x 64] and the whole token tile [Mp x 64] from its own smem;
//  * kT = 2, kCl = false: unit = (tile pair, k-block); each of the pair's tiles on its own CTA
//    (CTA 2c + r streams tile r of worker c's units), cta_group::1 as above;
//  * kT = 2, kCl = true: the same units on a CTA pair (cluster of 2, cta_group::2): each CTA loads
//    its own W tile and HALF of the token tile (Mp/2 rows), the leader issues one M = 256 MMA that
//    reads A from both CTAs and B split by N across them, D = each CTA's 128 rows x Mp in its own
//    TMEM. Per SM and unit: 16 KB + Mp x 64 B through smem instead of 16 KB + Mp x 128 B.
// Both executions of the pair split accumulate the same k-blocks of a tile in the same TMEM run
// and sum the runs in the same worker order, so they give the same bits (tested); the choice may
// follow M. A CTA (or pair) runs g.vw consecutive workers as one continuous weight stream; a run
// ends at every worker boundary, so the bits do not depend on vw either.
template <int kT, bool kCl>
__global__ void __launch_bounds__(kThreads, 2)   // two resident CTAs per SM (stream-K grid of 2 x #SMs)
tc_gemm_kernel(const __grid_constant__ CUtensorMap map_w0, const __grid_constant__ CUtensorMap map_w1,
               const __grid_constant__ CUtensorMap map_w2, const __grid_constant__ CUtensorMap map_x, TcArgs g) {
    static_assert(kT == 1 || kT == 2, "1 or 2 tiles per unit");
    static_assert(!kCl || kT == 2, "CTA pairs run the pair split");
    using TM = TileMap<kT>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the 128B swizzle atoms (same offset in both CTAs of a pair)
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int xrows = kCl ? g.Mp / 2 : g.Mp;       // token rows of the B tile this CTA holds
    const uint32_t tile_b_bytes = (uint32_t)xrows * kBK * 2;
    const int kStages = g.stages;
    uint8_t* sa = smem;
    uint8_t* sb = smem + kStages * kTileABytes;
    uint64_t* full = (uint64_t*)(sb + kStages * tile_b_bytes);
    uint64_t* empty = full + kMaxStages;
    uint64_t* tmem_full = empty + kMaxStages;      // [2] accumulator ready
    uint64_t* tmem_empty = tmem_full + 2;          // [2] accumulator drained
    uint32_t* tmem_slot = (uint32_t*)(tmem_empty + 2);
    __shared__ int s_last;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = kCl ? (int)cluster_rank() : (kT == 2 ? (int)(blockIdx.x & 1) : 0);   // tile of the unit
    const bool leader = !kCl || r == 0;            // issues the MMAs (the pair's rank 0)
    const int c = kT == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;   // CTA (pair) index
    const int cta = (int)blockIdx.x;
    const int w0 = c * g.vw, w1 = min(w0 + g.vw, g.G);   // workers of this CTA (pair)
    pdl_trigger();                                 // let the next kernel's CTAs get scheduled
    if (w0 >= w1) return;                          // uniform for the whole CTA (and pair)
    const uint64_t u0 = ubeg(g, w0), u1 = ubeg(g, w1);
    if (threadIdx.x == 0) stamp(g, cta, 0);        // phase 0: CTA start
    uint32_t nbuf = 32;                            // TMEM columns per accumulator: pow2 >= max(32, Mp)
    while ((int)nbuf < g.Mp) nbuf <<= 1;
    // double-buffered accumulator while every resident CTA's buffers fit in the 512 TMEM columns
    const int nacc = g.nacc;
    const uint32_t ncols = (uint32_t)nacc * nbuf;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w0) : "memory");
        if (g.nseg > 1) asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w1) : "memory");
        if (g.nseg > 2) asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w2) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tmem_full[b], 1);
            mbar_init(&tmem_empty[b], kCl ? 8 : 4);   // one arrive per epilogue warp (of both CTAs)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        if (kCl) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(ncols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(ncols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (kCl) cluster_sync_all();                   // the peer's barriers exist before any remote arrive
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = *tmem_slot;
    // leader's stage barriers: TMA bytes of both CTAs land there (pair mode)
    const uint32_t stage_bytes = kCl ? 2 * (kTileABytes + tile_b_bytes) : kTileABytes + tile_b_bytes;

    if (warp == 0) {
        if (lane == 0) {                           // ---- TMA producer: continuous across tiles and workers
            const uint64_t pol_w = l2_policy_evict_first(), pol_x = l2_policy_evict_last();
            auto load_w = [&](int s, uint64_t u, int kbi) {
                const int tile = TM::tile(u, g.kb, r);
                const int si = seg_of(g, tile);
                const CUtensorMap* mw = si == 0 ? &map_w0 : (si == 1 ? &map_w1 : &map_w2);
                const int c0 = kbi * kBK, c1 = (tile - g.seg[si].tile0) * kBN;
                // rows past the last tile (odd tile count, pair split) are zero-filled by TMA
                if (kCl) {
                    if (g.l2hint) tma_load_2d_pair_hint(sa + s * kTileABytes, mw, leader_addr(&full[s]), c0, c1, pol_w);
                    else tma_load_2d_pair(sa + s * kTileABytes, mw, leader_addr(&full[s]), c0, c1);
                } else {
                    if (g.l2hint) tma_load_2d_hint(sa + s * kTileABytes, mw, &full[s], c0, c1, pol_w);
                    else tma_load_2d(sa + s * kTileABytes, mw, &full[s], c0, c1);
                }
            };
            auto load_x = [&](int s, int kbi) {
                if (kCl) {
                    if (g.l2hint) tma_load_2d_pair_hint(sb + s * tile_b_bytes, &map_x, leader_addr(&full[s]), kbi * kBK, r * xrows, pol_x);
                    else tma_load_2d_pair(sb + s * tile_b_bytes, &map_x, leader_addr(&full[s]), kbi * kBK, r * xrows);
                } else {
                    if (g.l2hint) tma_load_2d_hint(sb + s * tile_b_bytes, &map_x, &full[s], kbi * kBK, 0, pol_x);
                    else tma_load_2d(sb + s * tile_b_bytes, &map_x, &full[s], kbi * kBK, 0);
                }
            };
            // Weights do not depend on the previous kernel: the first kStages weight tiles are in
            // flight before griddepcontrol.wait, overlapping the previous kernel's tail (PDL).
            stamp(g, cta, 1);                      // phase 1: prologue done (barriers, TMEM)
            const int pre = (int)(u1 - u0 < (uint64_t)kStages ? u1 - u0 : (uint64_t)kStages);
            for (int i = 0; i < pre; ++i) {
                if (leader) mbar_expect_tx(&full[i], stage_bytes);
                load_w(i, u0 + i, (int)((u0 + i) % g.kb));
            }
            // ...and the next l2_prefetch units go to L2, so the weight stream keeps HBM busy
            // across the kernel boundary (the smem ring alone holds only `stages` units)
            {
                const uint64_t pe = u0 + pre + (uint64_t)g.l2_prefetch < u1 ? u0 + pre + g.l2_prefetch : u1;
                for (uint64_t u = u0 + pre; u < pe; ++u) {
                    const int tile = TM::tile(u, g.kb, r), kbi = (int)(u % g.kb);
                    const int si = seg_of(g, tile);
                    const CUtensorMap* mw = si == 0 ? &map_w0 : (si == 1 ? &map_w1 : &map_w2);
                    tma_prefetch_l2(mw, kbi * kBK, (tile - g.seg[si].tile0) * kBN);
                }
            }
            pdl_wait();
            stamp(g, cta, 2);                      // phase 2: previous kernel complete
            for (int i = 0; i < pre; ++i) load_x(i, (int)((u0 + i) % g.kb));
            uint64_t u = u0 + pre;
            int s = pre % kStages;
            uint32_t ph = (uint32_t)(pre / kStages) & 1u;
            int kbi = (int)(u % g.kb);
            for (; u < u1; ++u) {
                mbar_wait(&empty[s], ph ^ 1u);
                if (leader) mbar_expect_tx(&full[s], stage_bytes);
                load_w(s, u, kbi);
                load_x(s, kbi);
                if (++s == kStages) { s = 0; ph ^= 1u; }
                if (++kbi == g.kb) kbi = 0;
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {                 // ---- MMA issuer (the pair's leader)
            // kind::f16: D fp32 (c_format 1), A = B = bf16 (format 1), both K-major,
            // N = Mp (n_dim = N >> 3), M = 128 / 256 (m_dim = M >> 4)
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(g.Mp >> 3) << 17) |
                                   ((uint32_t)((kBN * (kCl ? 2 : 1)) >> 4) << 24);
            int run = 0;
            uint32_t tmem_d = tmem_base;
            int s = 0, kbi = (int)(u0 % g.kb);
            uint32_t ph = 0;
            int w = w0;
            uint64_t wend = ubeg(g, w0 + 1);       // end of the current worker's range
            for (uint64_t u = u0; u < u1; ++u) {
                bool wstart = false;
                while (u >= wend) { ++w; wend = ubeg(g, w + 1); wstart = true; }
                const bool first = u == u0 || kbi == 0 || wstart;
                const bool last = u + 1 == u1 || kbi == g.kb - 1 || u + 1 == wend;
                if (first) {
                    const int b = nacc == 2 ? (run & 1) : 0;
                    const int use = nacc == 2 ? (run >> 1) : run;       // previous uses of buffer b
                    mbar_wait(&tmem_empty[b], ((uint32_t)use & 1u) ^ 1u);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    tmem_d = tmem_base + (uint32_t)b * nbuf;
                }
                mbar_wait(&full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (u == u0) stamp(g, cta, 3);     // phase 3: first stage landed
                const uint32_t a0 = smem_u32(sa + s * kTileABytes), b0 = smem_u32(sb + s * tile_b_bytes);
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                    if (kCl) umma_bf16_pair(tmem_d, umma_desc(a0 + kk * 32), umma_desc(b0 + kk * 32), idesc, (!first || kk) ? 1u : 0u);
                    else umma_bf16(tmem_d, umma_desc(a0 + kk * 32), umma_desc(b0 + kk * 32), idesc, (!first || kk) ? 1u : 0u);
                }
                if (kCl) umma_commit_pair(&empty[s]);   // both CTAs' stage s free once read
                else umma_commit(&empty[s]);
                if (last) {                        // accumulator of this run complete (both CTAs)
                    if (kCl) umma_commit_pair(&tmem_full[nacc == 2 ? (run & 1) : 0]);
                    else umma_commit(&tmem_full[nacc == 2 ? (run & 1) : 0]);
                    ++run;
                }
                if (++s == kStages) { s = 0; ph ^= 1u; }
                if (++kbi == g.kb) kbi = 0;
            }
            stamp(g, cta, 4);                      // phase 4: last MMA issued
        }
    } else if (warp >= 4) {                        // ---- epilogue: TMEM lane = weight row
        pdl_wait();                                // outputs / partials written only after it
        const int q = warp - 4;                    // TMEM lane quarter of this warp
        const int row = q * 32 + lane;             // row within the 128-row tile
        const uint32_t tmem_empty_leader = kCl ? leader_addr(&tmem_empty[0]) : 0;
        const uint64_t pol_p = l2_policy_evict_last();
        int run = 0;
        int w = w0;
        uint64_t wend = ubeg(g, w0 + 1);
        for (uint64_t u = u0; u < u1; ++run) {
            while (u >= wend) { ++w; wend = ubeg(g, w + 1); }
            const int ut = (int)(u / g.kb);        // unit tile (tile, or tile pair)
            const int tile = ut * kT + r;
            const bool phantom = tile >= g.tiles;  // pair split, odd tile count: zero rows
            const uint64_t tend = (uint64_t)(ut + 1) * g.kb;
            const uint64_t rend = wend < tend ? wend : tend;   // a run ends at a tile or worker boundary
            const int si = seg_of(g, phantom ? g.tiles - 1 : tile);
            const TcSeg& seg = g.seg[si];
            const int n = (tile - seg.tile0) * kBN + row;
            const bool nvalid = !phantom && n < seg.N;
            const float bias_n = (seg.bias && nvalid) ? __bfloat162float(seg.bias[n]) : 0.f;
            const int c_first = cta_of(g, (uint64_t)ut * g.kb), c_last = cta_of(g, tend - 1);
            const bool whole = c_first == c_last;
            const int fwh = whole ? 0 : first_slot(g, c_first, ut);
            const int which = ut == (int)((uint32_t)ubeg(g, w) / (uint32_t)g.kb) ? 0 : 1;
            float* prow = g.partial + ((size_t)TM::slot(w, r) * 2 + which) * (size_t)g.Mp * kBN + row;
            const int b = nacc == 2 ? (run & 1) : 0;
            const int use = nacc == 2 ? (run >> 1) : run;
            mbar_wait(&tmem_full[b], (uint32_t)use & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (row == 0 && rend == u1) stamp(g, cta, 5);   // phase 5: last accumulator ready
            float v[16];
            for (int col = 0; col < g.Mp; col += 16) {
                tmem_ld16(tmem_base + (uint32_t)b * nbuf + ((uint32_t)(q * 32) << 16) + (uint32_t)col, v);
                if (phantom) continue;
                if (!whole) {              // token-major partial: one 128-B store per warp per token
                    if (g.l2hint) {        // kept in L2 for the fix-up (the weight stream goes first)
#pragma unroll
                        for (int j = 0; j < 16; ++j) st_hint(prow + (size_t)(col + j) * kBN, v[j], pol_p);
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) prow[(size_t)(col + j) * kBN] = v[j];
                    }
                } else if (nvalid) {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (col + j < g.M) epi_store(g, seg, n, col + j, v[j], bias_n);
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                if (kCl)
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(tmem_empty_leader + (uint32_t)b * 8)
                                 : "memory");
                else
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[b])) : "memory");
            }
            if (row == 0 && rend == u1) stamp(g, cta, 6);   // phase 6: last run drained
            if (!whole && !g.ext_fixup && !phantom) {
                // fix-up: the last worker to finish a run of this tile sums all runs in k order.
                // bar.sync orders the 128 threads' partial stores before thread 0's gpu-scope
                // acq_rel atomic (release is cumulative); the acquire + bar.sync orders the
                // reads of the other CTAs' partials after it. No full fences needed.
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (row == 0) {
                    int old;
                    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(&g.counters[tile]) : "memory");
                    s_last = old == c_last - c_first;
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (s_last) {
                    if (nvalid) {
                        // 8 tokens per step, four runs per iteration: 32 coalesced loads in
                        // flight per thread; the sums stay in fixed run (k) order
                        for (int m0 = 0; m0 < g.M; m0 += 8) {
                            float acc[8];
#pragma unroll
                            for (int j = 0; j < 8; ++j) acc[j] = 0.f;
                            for (int cc = c_first; cc <= c_last; cc += 4) {
                                float t[4][8];
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    if (cc + k <= c_last) {
                                        const float* p = partial_run<kT>(g, cc + k, c_first, fwh, r, row) + (size_t)m0 * kBN;
#pragma unroll
                                        for (int j = 0; j < 8; ++j) t[k][j] = __ldcg(p + j * kBN);
                                    }
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    if (cc + k <= c_last) {
#pragma unroll
                                        for (int j = 0; j < 8; ++j) acc[j] += t[k][j];
                                    }
                            }
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                if (m0 + j < g.M) epi_store(g, seg, n, m0 + j, acc[j], bias_n);
                        }
                    }
                    if (row == 0) g.counters[tile] = 0;   // ready for the next launch
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
            }
            u = rend;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (kCl) cluster_sync_all();                   // no CTA leaves while its peer may still signal it
    else __syncthreads();
    if (threadIdx.x == 0) stamp(g, cta, 7);        // phase 7: CTA done
    if (warp == 2) {
        if (kCl) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols));
    }
}

// Split-tile reduction as its own grid (ext_fixup, large M): CTA (tile, kTok-token group), thread =
// weight row. Same fixed run order as the in-kernel fix-up, so the bits do not depend on which
// of the two reduces (the choice may follow M; the split itself never does).
template <int kT, int kTok>
__global__ void __launch_bounds__(kBN) tc_fixup_kernel(TcArgs g) {
    pdl_wait();                                    // every partial of the GEMM is written
    pdl_trigger();
    const int tile = blockIdx.x, row = threadIdx.x, m0 = blockIdx.y * kTok;
    const int ut = tile / kT, r = tile % kT;
    const uint64_t tend = (uint64_t)(ut + 1) * g.kb;
    const int c_first = cta_of(g, (uint64_t)ut * g.kb), c_last = cta_of(g, tend - 1);
    if (c_first == c_last || m0 >= g.M) return;   // whole tile: stored by the GEMM itself
    const int fwh = first_slot(g, c_first, ut);
    const TcSeg& seg = g.seg[seg_of(g, tile)];
    const int n = (tile - seg.tile0) * kBN + row;
    if (n >= seg.N) return;
    const float bias_n = seg.bias ? __bfloat162float(seg.bias[n]) : 0.f;
    // 4 runs x kTok tokens of coalesced loads in flight per thread, then the adds in fixed run
    // (k) order: one L2 round trip per 4 runs instead of one per run
    float acc[kTok];
#pragma unroll
    for (int j = 0; j < kTok; ++j) acc[j] = 0.f;
    for (int cc = c_first; cc <= c_last; cc += 4) {
        float t[4][kTok];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (cc + k <= c_last) {
                const float* p = partial_run<kT>(g, cc + k, c_first, fwh, r, row) + (size_t)m0 * kBN;
#pragma unroll
                for (int j = 0; j < kTok; ++j) t[k][j] = __ldcg(p + j * kBN);
            }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (cc + k <= c_last) {
#pragma unroll
                for (int j = 0; j < kTok; ++j) acc[j] += t[k][j];
            }
    }
#pragma unroll
    for (int j = 0; j < kTok; ++j)
        if (m0 + j < g.M) epi_store(g, seg, n, m0 + j, acc[j], bias_n);
}

// ----------------------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    });
    if (!fn) throw Error(MPSW_ECUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

struct MapKey {
    const void* p;
    uint64_t rows, K;
    uint32_t box;
    bool operator==(const MapKey& o) const { return p == o.p && rows == o.rows && K == o.K && box == o.box; }
};
struct MapKeyHash {
    size_t operator()(const MapKey& k) const {
        return std::hash<const void*>()(k.p) ^ (k.rows * 0x9E3779B97F4A7C15ull) ^ (k.K << 20) ^ k.box;
    }
};

// per-thread cache: every rank's worker thread encodes its own maps once
const CUtensorMap& cached_map(const void* p, uint64_t rows, uint64_t K, uint32_t box) {
    thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    const MapKey k{p, rows, K, box};
    auto it = cache.find(k);
    if (it != cache.end()) return it->second;
    return cache.emplace(k, tc_make_map(p, rows, K, box)).first->second;
}

}  // namespace

CUtensorMap tc_make_map(const void* ptr, uint64_t rows, uint64_t K, uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {K, rows};
    const cuuint64_t strides[1] = {K * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(MPSW_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

CUtensorMap tc_make_map_3d(const void* ptr, uint64_t rows, uint64_t K, uint64_t layers, uint64_t layer_stride,
                           uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {K, rows, layers};
    const cuuint64_t strides[2] = {K * 2, layer_stride};
    const cuuint32_t box[3] = {(cuuint32_t)kBK, box_rows, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(MPSW_ECUDA, "cuTensorMapEncodeTiled (3d) failed: " + std::to_string((int)r));
    return m;
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Persistent grid: two CTAs per SM (fixed, so the stream-K split never depends on M).
// tuning knobs (development: MPSW_TC_CPS = CTAs per SM, MPSW_TC_SMEM_KB = smem budget per CTA)
static int env_int(const char* n, int dflt) {
    const char* e = getenv(n);
    return e ? atoi(e) : dflt;
}

// tokens (padded) from which split tiles are reduced by a separate wide grid: a single CTA
// summing ~8 runs of 128 x Mp fp32 partials serialises the tail of the GEMM at large M
static int tc_ext_fixup_min() {
    static int v = env_int("MPSW_TC_EXT_MIN", 64);
    return v;
}

static int tc_l2_prefetch() {
    static int v = env_int("MPSW_TC_L2PF", 0);   // measured: any prefetch depth slows the stream
    return v;
}

int tc_ctas_per_sm() {
    static int v = env_int("MPSW_TC_CPS", 2);
    return v;
}

// Persistent grid: a fixed number of CTAs per SM (never a function of M, so the stream-K split
// and the reduction order are batch-invariant).
// At least this many (tile, k-block) units (16 KB of weights each) per CTA. Small GEMMs (OPT-125M /
// 1.3B layers) otherwise run one unit per CTA and split every tile 12-32 ways, so the fix-up
// chain and per-CTA fixed latency dominate. 8 was the best of 1..32 on B200:
// OPT-125M M=2 0.59 -> 0.55 ms, M=32 1.40 -> 0.81 ms; OPT-1.3B M=2 1.36 -> 1.14 ms, M=32 2.54 -> 1.98 ms;
// OPT-13B unchanged (>= 10.8 units per CTA already). Depends on (N, K) only: batch-invariant.
// MPSW_TC_MINU overrides it (dev).
static int tc_min_units() {
    static int v = env_int("MPSW_TC_MINU", 8);
    return v < 1 ? 1 : v;
}

// Tile-aligned split: G = tiles x s with s | kb, the largest s with G <= 2 x #SMs and
// kb / s >= tc_min_units(). Every CTA then covers kb / s k-blocks of ONE tile (no CTA straddles
// two tiles; each tile is reduced from s equal runs). Used only when it keeps >= 80 % of the
// stream-K grid: with fewer CTAs the large-M GEMMs lose tensor throughput (per shape, M = 2 / 256,
// profiles/r01_gemm_align.ndjson: OPT-13B QKV, 240 vs 296 CTAs, 31.3 -> 28.4 / 62.6 -> 59.7 us;
// fc1, 160 vs 296, 38.2 -> 38.4 / 73.6 -> 102.1 us; OPT-125M QKV, 18 vs 27, 16.6 -> 35.6 us at
// M = 256). Depends on (N, K) only. MPSW_TC_ALIGN=0 restores plain stream-K (dev).
static int tc_align() {
    static int v = env_int("MPSW_TC_ALIGN", 1);   // see tc_grid
    return v;
}

// Split (process-wide, never a function of M, so the split and the reduction order are
// batch-invariant): tiles per work unit, 1 = (tile, k-block) units, 2 = (tile pair, k-block)
// units. The pair split can run on independent CTAs or on CTA pairs with the same bits, so the
// execution may follow M (tc_exec). MPSW_TC_SPLIT overrides the default; MPSW_TC_PAIR=1 is the
// round-2 A/B mode (pair split, always CTA pairs, one worker per pair).
int tc_pair() {
    static int v = env_int("MPSW_TC_PAIR", 0);
    return v;
}
int tc_split_kt() {
    static int v = [] {
        if (tc_pair()) return 2;
        const int e = env_int("MPSW_TC_SPLIT", 2);
        return e == 1 ? 1 : 2;
    }();
    return v;
}

// Execution of one launch: CTA pairs (cta_group::2) or independent CTAs, workers per CTA (pair),
// resident CTAs per SM (smem budget, TMEM accumulator buffers).
struct TcExec {
    bool cl;
    int vw;
    int cps;
};
// Padded token rows from which the pair split runs on CTA pairs: at large M the token tile
// dominates the L2 -> smem traffic, and a CTA pair halves it (OPT-13B layer at M = 256: 234 ->
// 217 us; slower below 192 tokens). MPSW_TC_VW=2 runs two workers per pair at one CTA per SM
// (double-buffered 256-column accumulator, 6-deep ring): measured slower, 229 us (dev knob).
static int tc_cl_min_mp() {
    static int v = env_int("MPSW_TC_CL_MIN", 192);
    return v;
}
static TcExec tc_exec(int Mp) {
    const int cps = tc_ctas_per_sm();
    if (tc_split_kt() == 1) return {false, 1, cps};
    if (tc_pair()) return {true, 1, cps};
    if (Mp >= tc_cl_min_mp()) {
        static const int vw = std::max(1, env_int("MPSW_TC_VW", 1));
        return {true, vw, std::max(1, cps / vw)};
    }
    return {false, 1, cps};
}

// Workers of a GEMM with `tiles` 128-row tiles: stream-K over the (unit tile, k-block) units with
// at least tc_min_units() units per worker and at most tc_ctas_per_sm() x #SMs CTAs (a worker of
// the pair split is two CTAs), or the tile-aligned split when it keeps >= 80 % of that grid.
static int tc_grid(int tiles, int K) {
    const int kt = tc_split_kt();
    const int ut = (tiles + kt - 1) / kt;          // unit tiles (tiles or pairs)
    const int kb = (K + kBK - 1) / kBK;
    const uint64_t units = (uint64_t)ut * kb;
    const uint64_t mu = (uint64_t)tc_min_units();
    const uint64_t gmax = (uint64_t)tc_ctas_per_sm() * sm_count() / kt;
    const uint64_t g_sk = std::min<uint64_t>((units + mu - 1) / mu, gmax);
    if (tc_align() && (uint64_t)ut < gmax) {
        int best = 0;
        for (int sp = 1; sp <= kb; ++sp)
            if (kb % sp == 0 && (uint64_t)ut * sp <= gmax && (uint64_t)(kb / sp) >= mu) best = sp;
        if (best && (uint64_t)ut * best * 5 >= g_sk * 4) return ut * best;
        // small per-CTA shares (< 16 units under stream-K): straddling a tile boundary costs more
        // than the lost CTAs, so take the aligned split down to 60 % of the slots (OPT-13B
        // out_proj: 200 aligned CTAs of 16 units instead of 296 of 10.8; forward 5.31 -> 5.22 ms
        // at M = 2 in the MPSW_TC_MINU = 16 sweep, profiles/r02_tc_knobs.ndjson)
        static const int align60 = env_int("MPSW_TC_ALIGN60", 1);
        if (align60 && best && units < 16 * g_sk && (uint64_t)ut * best * 5 >= gmax * 3) return ut * best;
    }
    return (int)g_sk;
}

size_t tc_partial_floats(int n_total, int K, int Mp) {
    const int tiles = (n_total + kBN - 1) / kBN;
    return (size_t)tc_grid(tiles, K) * tc_split_kt() * 2 * kBN * Mp;
}

// Token rows of the B tile one CTA holds: Mp, or Mp / 2 on a CTA pair (N split across the pair).
static int tc_xrows(const TcExec& e, int Mp) { return e.cl ? Mp / 2 : Mp; }

// Ring stages within the per-CTA smem budget (MPSW_TC_SMEM_KB per CTA at 2 CTAs per SM, twice that
// at one CTA per SM).
static int tc_stages(const TcExec& e, int Mp) {
    static int budget_kb = env_int("MPSW_TC_SMEM_KB", 104);
    const size_t budget = (size_t)budget_kb * 1024 * (e.cps == 1 ? 2 : 1);
    const size_t per = kTileABytes + (size_t)tc_xrows(e, Mp) * kBK * 2;
    return (int)std::max<size_t>(2, std::min<size_t>(kMaxStages, budget / per));
}

static size_t tc_smem_bytes(const TcExec& e, int Mp) {
    return 1024 + tc_stages(e, Mp) * (kTileABytes + (size_t)tc_xrows(e, Mp) * kBK * 2) + (2 * kMaxStages + 4) * 8 + 16;
}

static unsigned long long* g_tc_trace = nullptr;   // dev instrumentation (mpsw_bench_gemm only)
void tc_set_trace(unsigned long long* p) { g_tc_trace = p; }
// CTAs a GEMM launches at most (any M): G workers x tiles per unit
int tc_grid_for(int n_total, int K) { return tc_grid((n_total + kBN - 1) / kBN, K) * tc_split_kt(); }
int tc_grid_tiles(int tiles, int K) { return tc_grid(tiles, K); }

bool tc_supported(int M, int K) { return M >= 1 && M <= 256 && K % 8 == 0; }

template <int kT, bool kCl>
static void launch_tc(const TcArgs& g, size_t smem, cudaStream_t st, const CUtensorMap& m0, const CUtensorMap& m1,
                      const CUtensorMap& m2, const CUtensorMap& mx) {
    static thread_local size_t attr_set = 0;
    if (attr_set < smem) {
        MPSW_CU(cudaFuncSetAttribute(tc_gemm_kernel<kT, kCl>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        MPSW_CU(cudaFuncSetAttribute(tc_gemm_kernel<kT, kCl>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attr_set = smem;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kCl ? 2 * ((g.G + g.vw - 1) / g.vw) : g.G * kT);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = kCl ? 2 : 1;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = kCl ? 2 : 1;
    MPSW_CU(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<kT, kCl>, m0, m1, m2, mx, g));
    // MPSW_DEV_NOOP_FIXUP: timing instrumentation only (split tiles are left unreduced)
    static const bool noop_fixup = env_int("MPSW_DEV_NOOP_FIXUP", 0) != 0;
    // 8 tokens per fix-up CTA: 56 registers, twice the CTAs of 16 tokens (88 registers) and more of
    // them resident: OPT-1.3B forward at M = 256 2.67 -> 2.51 ms, OPT-30B TP8 layer 101 -> 94 us
    // (profiles/r02s3_fixup_grid_shape.ndjson). MPSW_TC_FIX_TOK=16 restores the wider CTA (dev).
    static const int fix_tok = env_int("MPSW_TC_FIX_TOK", 8) == 16 ? 16 : 8;
    if (g.ext_fixup && !noop_fixup) {
        if (fix_tok == 8) launch_pdl(tc_fixup_kernel<kT, 8>, dim3(g.tiles, g.Mp / 8), kBN, 0, st, g);
        else launch_pdl(tc_fixup_kernel<kT, 16>, dim3(g.tiles, g.Mp / 16), kBN, 0, st, g);
    }
}

// Launch: W segments (up to 3, each [N_i, K] bf16) times X [M, K] bf16 (rows of a buffer with
// x_rows rows). epi 0: fp32 out = (acc + bias) * scale at out[(row) * ldo + out_col0 + n];
// epi 1: bf16 out = relu(acc + bias).
void tc_gemm(const void* const* W, const void* const* bias, const int* N, const float* scale, const int* out_col0,
             int nseg, const void* X, int x_rows, int M, int K, int epi, void* out, int ldo, const int32_t* row_of_m,
             float* partial, int* counters, cudaStream_t st) {
    const int Mp = std::max(16, (M + 15) / 16 * 16);
    const int kt = tc_split_kt();
    const TcExec ex = tc_exec(Mp);
    TcArgs g{};
    int tiles = 0;
    for (int i = 0; i < nseg; ++i) {
        g.seg[i].N = N[i];
        g.seg[i].tile0 = tiles;
        g.seg[i].bias = (const __nv_bfloat16*)bias[i];
        g.seg[i].scale = scale[i];
        g.seg[i].out_col0 = out_col0[i];
        tiles += (N[i] + kBN - 1) / kBN;
    }
    g.nseg = nseg;
    g.tiles = tiles;
    g.kb = (K + kBK - 1) / kBK;
    g.units = (uint64_t)((tiles + kt - 1) / kt) * g.kb;
    g.G = tc_grid(tiles, K);
    if (g.units * (uint64_t)g.G >= (1ull << 32)) throw Error(MPSW_EINVAL, "tcgen05 GEMM too large for the 32-bit split");
    g.vw = ex.vw;
    g.K = K;
    g.M = M;
    g.Mp = Mp;
    g.stages = tc_stages(ex, Mp);
    g.epi = epi;
    g.out = out;
    g.ldo = ldo;
    g.row_of_m = row_of_m;
    g.partial = partial;
    g.counters = counters;
    const CUtensorMap& m0 = cached_map(W[0], N[0], K, kBN);
    const CUtensorMap& m1 = cached_map(W[nseg > 1 ? 1 : 0], N[nseg > 1 ? 1 : 0], K, kBN);
    const CUtensorMap& m2 = cached_map(W[nseg > 2 ? 2 : 0], N[nseg > 2 ? 2 : 0], K, kBN);
    const CUtensorMap& mx = cached_map(X, (uint64_t)x_rows, K, (uint32_t)tc_xrows(ex, Mp));
    const size_t smem = tc_smem_bytes(ex, Mp);
    g.ext_fixup = Mp >= tc_ext_fixup_min() ? 1 : 0;
    g.trace = g_tc_trace;
    g.l2_prefetch = tc_l2_prefetch();
    static const int l2hint = env_int("MPSW_TC_L2HINT", 1);
    g.l2hint = l2hint;
    int nbuf = 32;
    while (nbuf < Mp) nbuf <<= 1;
    g.nacc = 2 * nbuf * ex.cps <= 512 ? 2 : 1;
    if (kt == 1)
        launch_tc<1, false>(g, smem, st, m0, m1, m2, mx);
    else if (ex.cl)
        launch_tc<2, true>(g, smem, st, m0, m1, m2, mx);
    else
        launch_tc<2, false>(g, smem, st, m0, m1, m2, mx);
    MPSW_CU(cudaGetLastError());
}

}  // namespace mpsw

#include "../../include/mpsw_testing.h"

extern "C" mpsw_status mpsw_tc_plan(int N, int K, int M, int64_t* plan) {
    using namespace mpsw;
    if (N < 1 || K < 8 || K % 8 || M < 1 || M > 256 || !plan) return set_error(MPSW_EINVAL, "bad shape");
    const int Mp = std::max(16, (M + 15) / 16 * 16);
    const int kt = tc_split_kt();
    const TcExec ex = tc_exec(Mp);
    const int tiles = (N + kBN - 1) / kBN;
    const int G = tc_grid(tiles, K);
    int nbuf = 32;
    while (nbuf < Mp) nbuf <<= 1;
    const int nacc = 2 * nbuf * ex.cps <= 512 ? 2 : 1;
    plan[0] = G;
    plan[1] = kt;
    plan[2] = (tiles + kt - 1) / kt;
    plan[3] = (K + kBK - 1) / kBK;
    plan[4] = kt == 1 ? G : (ex.cl ? 2 * ((G + ex.vw - 1) / ex.vw) : 2 * G);
    plan[5] = ex.cl ? 1 : 0;
    plan[6] = tc_stages(ex, Mp);
    plan[7] = (int64_t)tc_smem_bytes(ex, Mp);
    plan[8] = (int64_t)nacc * nbuf;
    plan[9] = Mp >= tc_ext_fixup_min() ? 1 : 0;
    plan[10] = ex.cps;
    plan[11] = Mp;
    return MPSW_OK;
}
