// Swap engine (a2 / a3): load and offload entries of one rank on its copy streams ("two
// additional streams to run loading and offloading operations concurrently"), chunk-paired with
// per-chunk gate events (reading #5), copy engine / zero-copy kernel / NVLink fan-in.
#include "runtime.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace mpsw {

double hybrid_frac() {
    static double f = [] {
        const char* e = getenv("MPSW_HYBRID_FRAC");
        return e ? atof(e) : 0.15;
    }();
    return f;
}

// AUTO: the measured winner per shard-size bucket (tools/auto_table.py). With the
// arenas clean in DRAM (store.cpp flush_to_memory) the copy engine wins every bucket from 1 MiB to
// 1 GiB, idle and under a concurrent forward (profiles/r02_auto_table_clean.ndjson): 1 MiB 25 vs
// 36 us, 4 MiB 82 vs 94 us, 16 MiB 0.31 vs 0.34 ms, >= 64 MiB at the link rate vs 0.93 of it.
// The round-1 zero-copy bucket (<= 8 MiB) only reflected copies from cache-dirty arenas.
struct AutoBucket {
    uint64_t max_bytes;
    bool zero_copy;
};
static const AutoBucket kAutoTable[] = {{~0ull, false}};

bool use_zero_copy(mpsw_ctx* c, uint64_t bytes) {
    if (c->cfg.swap_mode == MPSW_SWAP_ZERO_COPY) return true;
    if (c->cfg.swap_mode == MPSW_SWAP_COPY_ENGINE) return false;
    for (const auto& b : kAutoTable)
        if (bytes <= b.max_bytes) return b.zero_copy;
    return false;
}

int zc_ctas(mpsw_ctx* c) { return c->cfg.zc_ctas > 0 ? c->cfg.zc_ctas : 32; }

uint8_t* arena_of(mpsw_ctx* c, int model, const Rank& R) { return c->models[model]->arena[R.local].p; }

// ----------------------------------------------------------------------------- worker issue
bool event_done(cudaEvent_t ev) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) return true;
    if (q == cudaErrorNotReady) return false;
    MPSW_CU(q);
    return false;
}

// ----------------------------------------------------------------------------- range gates
// Events of gates overlapping [lo, hi) that have not completed (duplicates removed).
static void pending_gates(Rank& R, uint64_t lo, uint64_t hi, std::vector<cudaEvent_t>& out, bool* chunked) {
    out.clear();
    if (chunked) *chunked = false;
    for (const Gate& g : R.gates) {
        if (g.hi <= lo || hi <= g.lo) continue;
        if (std::find(out.begin(), out.end(), g.ev) != out.end() || event_done(g.ev)) continue;
        out.push_back(g.ev);
        if (chunked && g.chunk) *chunked = true;
    }
}

// After a load into [lo, hi) has been ordered after every gate overlapping it, gates lying inside
// the range are superseded (any later writer of those bytes is ordered after this model's
// forwards, hence after this load); completed gates are dropped too.
static void retire_gates(Rank& R, uint64_t lo, uint64_t hi) {
    size_t w = 0;
    for (size_t i = 0; i < R.gates.size(); ++i) {
        Gate& g = R.gates[i];
        if ((lo <= g.lo && g.hi <= hi) || event_done(g.ev)) {
            cudaEventDestroy(g.ev);
        } else {
            R.gates[w++] = g;
        }
    }
    R.gates.resize(w);
}

static void add_gate(Rank& R, uint64_t lo, uint64_t hi, bool chunk, cudaStream_t st) {
    cudaEvent_t ev;
    MPSW_CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    MPSW_CU(cudaEventRecord(ev, st));
    R.gates.push_back({lo, hi, ev, chunk});
}

void issue_load(mpsw_ctx* c, Rank& R, Entry& e) {
    const Model& md = *c->models[e.model];
    const uint64_t S = md.rank_S[R.index], lo = e.off, hi = e.off + S;
    const int n_chunks = (int)((S + c->chunk - 1) / c->chunk);
    uint8_t* base = R.region + e.off;
    const uint8_t* src = arena_of(c, e.model, R);
    const bool zc = use_zero_copy(c, S);
    const int r = R.index;
    if (md.arena_dirty[R.local]) {                 // caller-filled in place: write back from the CPU caches
        flush_to_memory(arena_of(c, e.model, R), S);
        c->models[e.model]->arena_dirty[R.local] = 0;
    }
    {
        const FwdShape& f = md.fs[R.local];
        R.wptr[e.model] = make_ptrs(md.layout[R.local], base, R.stage * f.n_layers, f.n_layers);
    }
    MPSW_CU(cudaEventCreate(&e.ev_start[r]));
    MPSW_CU(cudaEventCreate(&e.ev_done[r]));
    static const bool dbg = getenv("MPSW_SWAP_DEBUG") != nullptr;
    const auto h0 = std::chrono::steady_clock::now();
    MPSW_CU(cudaEventRecord(e.ev_start[r], R.h2d));
    // gates that already completed are skipped (a stream wait on another stream's event costs
    // tens of microseconds, which dominates small-shard swaps: DESIGN.md §8 cfg5)
    std::vector<cudaEvent_t> evs;
    bool chunked = false;
    pending_gates(R, lo, hi, evs, &chunked);
    if (!chunked)   // only whole-range gates (clean eviction): one wait up front
        for (auto ev : evs) MPSW_CU(cudaStreamWaitEvent(R.h2d, ev, 0));
    if (c->cfg.swap_mode == 3 && !chunked && S >= (64ull << 20)) {
        // HYBRID: the copy engine moves the head of the shard while the zero-copy kernel pulls
        // the tail over the same link from the SMs (two independent PCIe read requesters)
        const double f = hybrid_frac();
        const uint64_t zc_bytes = ((uint64_t)(S * f) + 4095) / 4096 * 4096;
        const uint64_t ce_bytes = S - zc_bytes;
        MPSW_CU(cudaEventRecord(R.ev_zc, R.h2d));
        MPSW_CU(cudaStreamWaitEvent(R.h2d_zc, R.ev_zc, 0));
        launch_zero_copy(base + ce_bytes, src + ce_bytes, zc_bytes, zc_ctas(c), R.h2d_zc);
        c->launches++;
        for (uint64_t off = 0; off < ce_bytes; off += c->chunk)
            MPSW_CU(cudaMemcpyAsync(base + off, src + off, std::min<uint64_t>(c->chunk, ce_bytes - off),
                                    cudaMemcpyHostToDevice, R.h2d));
        MPSW_CU(cudaEventRecord(R.ev_zc, R.h2d_zc));
        MPSW_CU(cudaStreamWaitEvent(R.h2d, R.ev_zc, 0));
    } else if (!chunked && zc) {
        launch_zero_copy(base, src, S, zc_ctas(c), R.h2d);
        c->launches++;
    } else if (!c->helpers.empty() && !zc && n_chunks > 1) {
        // fan-in: chunk i goes over link (i mod (1 + helpers)); lane 0 is the owner's own link
        const int lanes = 1 + (int)c->helpers.size();
        std::vector<cudaEvent_t> whole = chunked ? std::vector<cudaEvent_t>() : evs;
        for (int i = 0; i < n_chunks; ++i) {
            const uint64_t off = (uint64_t)i * c->chunk, n = std::min<uint64_t>(c->chunk, S - off);
            std::vector<cudaEvent_t> gate;
            if (chunked) pending_gates(R, lo + off, lo + off + n, gate, nullptr);
            const int lane = i % lanes;
            if (lane == 0) {
                for (auto ev : gate) MPSW_CU(cudaStreamWaitEvent(R.h2d, ev, 0));
                MPSW_CU(cudaMemcpyAsync(base + off, src + off, n, cudaMemcpyHostToDevice, R.h2d));
                continue;
            }
            Helper& H = *c->helpers[lane - 1];
            std::lock_guard<std::mutex> lk(H.mu);
            MPSW_CU(cudaSetDevice(H.device));
            if (i == lane) {                   // first chunk of this load on this helper
                MPSW_CU(cudaStreamWaitEvent(H.stream, e.ev_start[r], 0));
                for (auto ev : whole) MPSW_CU(cudaStreamWaitEvent(H.stream, ev, 0));
            }
            for (auto ev : gate) MPSW_CU(cudaStreamWaitEvent(H.stream, ev, 0));
            const int j = H.next;
            H.next ^= 1;
            if (H.free_valid[j]) MPSW_CU(cudaStreamWaitEvent(H.stream, H.free_ev[j], 0));
            uint8_t* stg = H.staging + (uint64_t)j * c->chunk;
            MPSW_CU(cudaMemcpyAsync(stg, src + off, n, cudaMemcpyHostToDevice, H.stream));
            MPSW_CU(cudaMemcpyPeerAsync(base + off, R.device, stg, H.device, n, H.stream));
            MPSW_CU(cudaEventRecord(H.free_ev[j], H.stream));
            H.free_valid[j] = true;
            if (!e.ev_helper[r][lane - 1]) MPSW_CU(cudaEventCreateWithFlags(&e.ev_helper[r][lane - 1], cudaEventDisableTiming));
            MPSW_CU(cudaEventRecord(e.ev_helper[r][lane - 1], H.stream));
            MPSW_CU(cudaSetDevice(R.device));
        }
        for (int h = 0; h < (int)c->helpers.size(); ++h)
            if (e.ev_helper[r][h]) MPSW_CU(cudaStreamWaitEvent(R.h2d, e.ev_helper[r][h], 0));
    } else {
        // chunk i of the new model waits only for the D2H of the bytes it overwrites (chunk-paired
        // in-place swap, reading #5; for equal-size models: the victim's chunk i)
        std::vector<cudaEvent_t> gate;
        for (int i = 0; i < n_chunks; ++i) {
            const uint64_t off = (uint64_t)i * c->chunk, n = std::min<uint64_t>(c->chunk, S - off);
            if (chunked) {
                pending_gates(R, lo + off, lo + off + n, gate, nullptr);
                for (auto ev : gate) MPSW_CU(cudaStreamWaitEvent(R.h2d, ev, 0));
            }
            if (zc) {
                launch_zero_copy(base + off, src + off, n, zc_ctas(c), R.h2d);
                c->launches++;
            } else {
                MPSW_CU(cudaMemcpyAsync(base + off, src + off, n, cudaMemcpyHostToDevice, R.h2d));
            }
        }
    }
    if (R.d_stamp) {                               // debug checks: this load made the model resident
        launch_stamp(R.d_stamp + e.model, e.id, R.h2d);
        c->launches++;
    }
    // completion marker right behind the last copy; the gate bookkeeping (event destroys) comes
    // after it, so host work never sits between the copy and its completion on the stream
    MPSW_CU(cudaEventRecord(e.ev_done[r], R.h2d));
    if (dbg)
        fprintf(stderr, "[mpsw] load m%d rank %d: %llu B issued in %.1f us (gates %zu, zc %d, chunks %d)\n", e.model, r,
                (unsigned long long)S, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count(),
                evs.size(), (int)zc, n_chunks);
    retire_gates(R, lo, hi);
}

void issue_offload(mpsw_ctx* c, Rank& R, Entry& e) {
    const uint64_t S = c->models[e.model]->rank_S[R.index], lo = e.off;
    const int n_chunks = (int)((S + c->chunk - 1) / c->chunk);
    const uint8_t* base = R.region + e.off;
    uint8_t* dst = arena_of(c, e.model, R);
    const bool zc = use_zero_copy(c, S);
    const int r = R.index;
    MPSW_CU(cudaEventCreate(&e.ev_start[r]));
    MPSW_CU(cudaEventCreate(&e.ev_done[r]));
    // eviction never races an in-flight request: the D2H stream waits for the last forward
    // that read the victim (the engine also only evicts models with no in-flight batch)
    const bool fwd_pending = R.last_compute_valid[e.model] && !event_done(R.last_compute[e.model]);
    if (fwd_pending) MPSW_CU(cudaStreamWaitEvent(R.d2h, R.last_compute[e.model], 0));
    MPSW_CU(cudaEventRecord(e.ev_start[r], R.d2h));
    if (e.writeback) {
        for (int i = 0; i < n_chunks; ++i) {
            const uint64_t off = (uint64_t)i * c->chunk, n = std::min<uint64_t>(c->chunk, S - off);
            if (zc) {
                launch_zero_copy(dst + off, base + off, n, zc_ctas(c), R.d2h);
                c->launches++;
            } else {
                MPSW_CU(cudaMemcpyAsync(dst + off, base + off, n, cudaMemcpyDeviceToHost, R.d2h));
            }
            add_gate(R, lo + off, lo + off + n, true, R.d2h);   // these bytes may now be overwritten
        }
    } else if (fwd_pending) {
        add_gate(R, lo, lo + S, false, R.d2h);                  // after the victim's last forward
    }
    if (R.d_stamp) {                               // debug checks: no longer resident
        launch_stamp(R.d_stamp + e.model, kStampEvicted, R.d2h);
        c->launches++;
    }
    // (clean eviction of a victim whose forwards have all completed needs no gate: the load that
    // reuses its bytes would otherwise pay a cross-stream event wait, ~40 us per swap at small
    // sizes, for an event that orders nothing — DESIGN.md §8 cfg5)
    MPSW_CU(cudaEventRecord(e.ev_done[r], R.d2h));
}

// Device span of a finished swap entry on every local rank; then its events are released (a
// long run would otherwise keep 2 events per rank per swap).
void finish_swap_events(mpsw_ctx* c, Entry& e) {
    record_spans(c, e);
    for (int r = 0; r < c->nr; ++r) {
        if (e.ev_start[r] && e.ev_done[r] && cudaEventElapsedTime(&e.gpu_ms[r], e.ev_start[r], e.ev_done[r]) != cudaSuccess)
            e.gpu_ms[r] = 0;
        cudaGetLastError();
        if (e.ev_start[r]) cudaEventDestroy(e.ev_start[r]), e.ev_start[r] = nullptr;
        if (e.ev_done[r]) cudaEventDestroy(e.ev_done[r]), e.ev_done[r] = nullptr;
        for (auto& ev : e.ev_helper[r])
            if (ev) cudaEventDestroy(ev), ev = nullptr;
    }
}

}  // namespace mpsw
