// Swap engine (a2 / a3): load and offload entries of one rank on its copy streams ("two
// additional streams to run loading and offloading operations concurrently"), chunk-paired with
// per-chunk gate events (reading #5), copy engine / zero-copy kernel / NVLink fan-in.
#include "runtime.h"

#include <algorithm>
#include <cstdlib>

namespace mpsw {

double hybrid_frac() {
    static double f = [] {
        const char* e = getenv("MPSW_HYBRID_FRAC");
        return e ? atof(e) : 0.15;
    }();
    return f;
}

bool use_zero_copy(mpsw_ctx* c, uint64_t bytes) {
    if (c->cfg.swap_mode == MPSW_SWAP_ZERO_COPY) return true;
    if (c->cfg.swap_mode == MPSW_SWAP_COPY_ENGINE) return false;
    return bytes <= (8ull << 20);   // AUTO: zero-copy for shards <= 8 MiB (cfg5 sweep crossover)
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

void issue_load(mpsw_ctx* c, Rank& R, Entry& e) {
    Slot& sl = R.slots[e.slot];
    const uint8_t* src = arena_of(c, e.model, R);
    const bool zc = use_zero_copy(c, R.S);
    const int r = R.index;
    MPSW_CU(cudaEventCreate(&e.ev_start[r]));
    MPSW_CU(cudaEventCreate(&e.ev_done[r]));
    MPSW_CU(cudaEventRecord(e.ev_start[r], R.h2d));
    // gates that already completed are skipped (a stream wait on another stream's event costs
    // tens of microseconds, which dominates small-shard swaps: DESIGN.md §8 cfg5)
    if (sl.whole_gate_valid && !event_done(sl.whole_gate)) MPSW_CU(cudaStreamWaitEvent(R.h2d, sl.whole_gate, 0));
    if (c->cfg.swap_mode == 3 && !sl.chunk_gate_valid && R.S >= (64ull << 20)) {
        // HYBRID: the copy engine moves the head of the shard while the zero-copy kernel pulls
        // the tail over the same link from the SMs (two independent PCIe read requesters)
        const double f = hybrid_frac();
        const uint64_t zc_bytes = ((uint64_t)(R.S * f) + 4095) / 4096 * 4096;
        const uint64_t ce_bytes = R.S - zc_bytes;
        MPSW_CU(cudaEventRecord(R.ev_zc, R.h2d));
        MPSW_CU(cudaStreamWaitEvent(R.h2d_zc, R.ev_zc, 0));
        launch_zero_copy(sl.base + ce_bytes, src + ce_bytes, zc_bytes, zc_ctas(c), R.h2d_zc);
        c->launches++;
        for (uint64_t off = 0; off < ce_bytes; off += c->chunk)
            MPSW_CU(cudaMemcpyAsync(sl.base + off, src + off, std::min<uint64_t>(c->chunk, ce_bytes - off),
                                    cudaMemcpyHostToDevice, R.h2d));
        MPSW_CU(cudaEventRecord(R.ev_zc, R.h2d_zc));
        MPSW_CU(cudaStreamWaitEvent(R.h2d, R.ev_zc, 0));
    } else if (!sl.chunk_gate_valid && zc) {
        launch_zero_copy(sl.base, src, R.S, zc_ctas(c), R.h2d);
        c->launches++;
    } else if (!c->helpers.empty() && !zc && R.n_chunks > 1) {
        // fan-in: chunk i goes over link (i mod (1 + helpers)); lane 0 is the owner's own link
        const int lanes = 1 + (int)c->helpers.size();
        for (int i = 0; i < R.n_chunks; ++i) {
            const uint64_t off = (uint64_t)i * c->chunk, n = std::min<uint64_t>(c->chunk, R.S - off);
            const int lane = i % lanes;
            cudaEvent_t gate = sl.chunk_gate_valid && !event_done(sl.chunk_gate[i]) ? sl.chunk_gate[i] : nullptr;
            if (lane == 0) {
                if (gate) MPSW_CU(cudaStreamWaitEvent(R.h2d, gate, 0));
                MPSW_CU(cudaMemcpyAsync(sl.base + off, src + off, n, cudaMemcpyHostToDevice, R.h2d));
                continue;
            }
            Helper& H = *c->helpers[lane - 1];
            std::lock_guard<std::mutex> lk(H.mu);
            MPSW_CU(cudaSetDevice(H.device));
            if (i == lane) {                   // first chunk of this load on this helper
                MPSW_CU(cudaStreamWaitEvent(H.stream, e.ev_start[r], 0));
                if (sl.whole_gate_valid && !event_done(sl.whole_gate))
                    MPSW_CU(cudaStreamWaitEvent(H.stream, sl.whole_gate, 0));
            }
            if (gate) MPSW_CU(cudaStreamWaitEvent(H.stream, gate, 0));
            const int j = H.next;
            H.next ^= 1;
            if (H.free_valid[j]) MPSW_CU(cudaStreamWaitEvent(H.stream, H.free_ev[j], 0));
            uint8_t* stg = H.staging + (uint64_t)j * c->chunk;
            MPSW_CU(cudaMemcpyAsync(stg, src + off, n, cudaMemcpyHostToDevice, H.stream));
            MPSW_CU(cudaMemcpyPeerAsync(sl.base + off, R.device, stg, H.device, n, H.stream));
            MPSW_CU(cudaEventRecord(H.free_ev[j], H.stream));
            H.free_valid[j] = true;
            if (!e.ev_helper[r][lane - 1]) MPSW_CU(cudaEventCreateWithFlags(&e.ev_helper[r][lane - 1], cudaEventDisableTiming));
            MPSW_CU(cudaEventRecord(e.ev_helper[r][lane - 1], H.stream));
            MPSW_CU(cudaSetDevice(R.device));
        }
        for (int h = 0; h < (int)c->helpers.size(); ++h)
            if (e.ev_helper[r][h]) MPSW_CU(cudaStreamWaitEvent(R.h2d, e.ev_helper[r][h], 0));
    } else {
        for (int i = 0; i < R.n_chunks; ++i) {
            const uint64_t off = (uint64_t)i * c->chunk, n = std::min<uint64_t>(c->chunk, R.S - off);
            if (sl.chunk_gate_valid && !event_done(sl.chunk_gate[i]))
                MPSW_CU(cudaStreamWaitEvent(R.h2d, sl.chunk_gate[i], 0));
            if (zc) {
                launch_zero_copy(sl.base + off, src + off, n, zc_ctas(c), R.h2d);
                c->launches++;
            } else {
                MPSW_CU(cudaMemcpyAsync(sl.base + off, src + off, n, cudaMemcpyHostToDevice, R.h2d));
            }
        }
    }
    sl.chunk_gate_valid = false;
    sl.whole_gate_valid = false;
    MPSW_CU(cudaEventRecord(e.ev_done[r], R.h2d));
}

void issue_offload(mpsw_ctx* c, Rank& R, Entry& e) {
    Slot& sl = R.slots[e.slot];
    uint8_t* dst = arena_of(c, e.model, R);
    const bool zc = use_zero_copy(c, R.S);
    const int r = R.index;
    MPSW_CU(cudaEventCreate(&e.ev_start[r]));
    MPSW_CU(cudaEventCreate(&e.ev_done[r]));
    // eviction never races an in-flight request: the D2H stream waits for the last forward
    // that read the victim (the engine also only evicts models with no in-flight batch)
    if (R.last_compute_valid[e.model] && !event_done(R.last_compute[e.model]))
        MPSW_CU(cudaStreamWaitEvent(R.d2h, R.last_compute[e.model], 0));
    MPSW_CU(cudaEventRecord(e.ev_start[r], R.d2h));
    if (c->cfg.writeback) {
        for (int i = 0; i < R.n_chunks; ++i) {
            const uint64_t off = (uint64_t)i * c->chunk, n = std::min<uint64_t>(c->chunk, R.S - off);
            if (zc) {
                launch_zero_copy(dst + off, sl.base + off, n, zc_ctas(c), R.d2h);
                c->launches++;
            } else {
                MPSW_CU(cudaMemcpyAsync(dst + off, sl.base + off, n, cudaMemcpyDeviceToHost, R.d2h));
            }
            MPSW_CU(cudaEventRecord(sl.chunk_gate[i], R.d2h));   // chunk i may now be overwritten
        }
        sl.chunk_gate_valid = true;
    } else {
        MPSW_CU(cudaEventRecord(sl.whole_gate, R.d2h));
        sl.whole_gate_valid = true;
    }
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
