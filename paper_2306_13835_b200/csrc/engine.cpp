// mpsw runtime: pinned shard store, device slots, per-rank workers, the engine (scheduler)
// thread and the C-ABI entry points.
//
// Architecture (§3.1 Fig. 1, §3.2, §4):
//   * one engine thread = the paper's centralised engine: per-model FIFO request queues with
//     arrival timestamps, oldest-head batch scheduling, LRU replacement via
//     load/offload entries, ack-based completion;
//   * one worker thread per rank = the paper's per-GPU worker: it receives every entry in the
//     same global order ("evaluate batch entries in submitted order") and issues it on
//     its own streams: compute, load (H2D) and offload (D2H). A worker never waits
//     for a copy before moving on to the next entry (P:105 asynchronous load entries);
//   * the engine polls per-rank completion events; an entry is complete when every rank has
//     acked. Batches for a model are submitted only after its load completed on all
//     ranks (load dependency).
// Scheduling semantics are those of DESIGN.md §Scheduler (readings #1-#7, #21, #24, #26);
// the independent numpy oracle (oracle/scheduler.py) replays this engine's trace.
#include "internal.h"

#include <immintrin.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <future>
#include <map>
#include <sstream>
#include <unordered_map>

namespace mpsw {

std::string& tls_error() {
    thread_local std::string e;
    return e;
}
mpsw_status set_error(mpsw_status s, const std::string& msg) {
    tls_error() = msg;
    return s;
}

namespace {

constexpr uint64_t kNoopTicket = ~0ull;
constexpr uint64_t kSlotAlign = 4096;
constexpr int kMaxRanks = 8;
constexpr size_t kMaxModels = 4096;

// ----------------------------------------------------------------------------- pinned store
int gpu_numa_node(int dev) {
    char bus[64] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) != cudaSuccess) return -1;
    for (char* c = bus; *c; ++c) *c = (char)tolower(*c);
    std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
    std::ifstream f(path);
    int node = -1;
    if (f) f >> node;
    return node;
}

struct PinnedBuf {
    uint8_t* p = nullptr;
    uint64_t bytes = 0;
    uint64_t map_bytes = 0;
};

// NUMA-affine page-locked arena: anonymous mmap, transparent huge pages, bound to the
// GPU's NUMA node when the platform reports one, then registered (portable + mapped so the
// zero-copy kernel can read it through UVA).
PinnedBuf pin_alloc(uint64_t bytes, int numa_node) {
    PinnedBuf b;
    b.bytes = bytes;
    b.map_bytes = (std::max<uint64_t>(bytes, 1) + kSlotAlign - 1) / kSlotAlign * kSlotAlign;
    void* p = mmap(nullptr, b.map_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p == MAP_FAILED) throw Error(MPSW_ENOMEM, "mmap of pinned arena failed");
    madvise(p, b.map_bytes, MADV_HUGEPAGE);
    if (numa_node >= 0 && numa_node < 64) {
        unsigned long mask = 1ul << numa_node;
        syscall(SYS_mbind, p, b.map_bytes, 2 /*MPOL_BIND*/, &mask, 64, 0);
    }
    cudaError_t e = cudaHostRegister(p, b.map_bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
    if (e != cudaSuccess) {
        munmap(p, b.map_bytes);
        throw Error(MPSW_ENOMEM, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
    }
    b.p = (uint8_t*)p;
    return b;
}

void pin_free(PinnedBuf& b) {
    if (!b.p) return;
    cudaHostUnregister(b.p);
    munmap(b.p, b.map_bytes);
    b.p = nullptr;
}

void parallel_memcpy(uint8_t* dst, const uint8_t* src, uint64_t n) {
    const int T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (n < (64ull << 20)) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([=] {
            const uint64_t b = n * t / T, e = n * (t + 1) / T;
            std::memcpy(dst + b, src + b, e - b);
        });
    for (auto& x : th) x.join();
}

struct SpinBarrier {
    std::atomic<int> count{0};
    std::atomic<int> gen{0};
    int n = 1;
    void wait() {
        if (n <= 1) return;
        const int g = gen.load(std::memory_order_acquire);
        if (count.fetch_add(1, std::memory_order_acq_rel) + 1 == n) {
            count.store(0, std::memory_order_relaxed);
            gen.fetch_add(1, std::memory_order_acq_rel);
        } else {
            int spins = 0;
            while (gen.load(std::memory_order_acquire) == g) {
                if (++spins < 4096) _mm_pause();
                else std::this_thread::yield();
            }
        }
    }
};

// ----------------------------------------------------------------------------- engine state
enum { E_LOAD = 0, E_OFFLOAD = 1, E_BATCH = 2 };
enum { ST_EVICTED = 0, ST_LOADING = 1, ST_RESIDENT = 2, ST_OFFLOADING = 3 };

struct ReqRec {
    int64_t rid;
    int model;
    std::vector<int32_t> tokens;
    float* out;
    double t_arr = 0, t_done = 0;
    std::atomic<int> done{0};
};

struct Entry {
    uint64_t id = 0;
    int kind = 0, model = -1, slot = -1;
    std::vector<std::shared_ptr<ReqRec>> reqs;
    int ring = 0, M = 0;
    double t_submit = 0;
    // per rank
    cudaEvent_t ev_start[kMaxRanks] = {};
    cudaEvent_t ev_done[kMaxRanks] = {};
    std::atomic<int> issued[kMaxRanks];
    int acked[kMaxRanks] = {};
    double t_ack[kMaxRanks] = {};
    int n_acked = 0;
    std::atomic<int> complete{0};
    Entry() {
        for (auto& a : issued) a.store(0);
    }
};
using EntryP = std::shared_ptr<Entry>;

// Decision of the state machine (mirrors oracle/scheduler.py's dicts).
struct Decision {
    int kind;  // 0 load, 1 offload, 2 batch, 3 complete, 4 noop, 5 reject
    uint64_t id = 0;
    int model = -1, slot = -1;
    std::vector<int64_t> rids;
    const char* status = "";
};

// Deterministic engine state machine.
struct StateMachine {
    int n_models = 0, k = 0, tp = 1, max_batch = 1, D = 1;
    std::vector<std::deque<std::pair<int64_t, double>>> queue;
    std::vector<int> state, outstanding, slot_of;
    std::vector<double> last_use;
    std::vector<int> owner;  // slot -> model or -1
    struct Pend { int kind, model, left; uint32_t mask; };
    std::map<uint64_t, Pend> pending;
    std::map<uint64_t, std::pair<int, std::vector<int64_t>>> batches;
    int inflight = 0;
    uint64_t next_id = 0;

    void add_model() {
        queue.emplace_back();
        state.push_back(ST_EVICTED);
        outstanding.push_back(0);
        slot_of.push_back(-1);
        last_use.push_back(-INFINITY);
        ++n_models;
    }
    bool head_less(int a, int b) const {  // (head t_arr, reg order)
        const double ta = queue[a].front().second, tb = queue[b].front().second;
        return ta < tb || (ta == tb && a < b);
    }
    int free_slot() const {
        for (int s = 0; s < k; ++s)
            if (owner[s] < 0) return s;
        return -1;
    }
    void load(int m, int s, std::vector<Decision>& out) {
        Decision d{0, next_id++, m, s};
        owner[s] = m;
        slot_of[m] = s;
        state[m] = ST_LOADING;
        pending[d.id] = {E_LOAD, m, tp, 0u};
        out.push_back(d);
    }
    int offload(int v, std::vector<Decision>& out) {
        const int s = slot_of[v];
        Decision d{1, next_id++, v, s};
        owner[s] = -1;
        slot_of[v] = -1;
        state[v] = ST_OFFLOADING;
        pending[d.id] = {E_OFFLOAD, v, tp, 0u};
        out.push_back(d);
        return s;
    }
    void schedule(double now, std::vector<Decision>& out) {
        std::vector<char> blocked(n_models, 0);
        for (;;) {
            int m = -1;
            for (int i = 0; i < n_models; ++i)
                if (!queue[i].empty() && !blocked[i] && (m < 0 || head_less(i, m))) m = i;
            if (m < 0) return;
            const int st = state[m];
            if (st == ST_RESIDENT) {
                if (inflight < D) {
                    const int n = std::min<int>(max_batch, (int)queue[m].size());
                    Decision d{2, next_id++, m};
                    for (int i = 0; i < n; ++i) {
                        d.rids.push_back(queue[m].front().first);
                        queue[m].pop_front();
                    }
                    batches[d.id] = {m, d.rids};
                    last_use[m] = now;
                    ++outstanding[m];
                    ++inflight;
                    out.push_back(std::move(d));
                } else {
                    blocked[m] = 1;
                }
            } else if (st == ST_LOADING || st == ST_OFFLOADING) {
                blocked[m] = 1;
            } else {
                const int s = free_slot();
                if (s >= 0) {
                    load(m, s, out);
                } else {
                    int best = -1;
                    auto key_less = [&](int a, int b) {  // prefer empty queue, then LRU, then reg order
                        const int qa = queue[a].empty() ? 0 : 1, qb = queue[b].empty() ? 0 : 1;
                        if (qa != qb) return qa < qb;
                        if (last_use[a] != last_use[b]) return last_use[a] < last_use[b];
                        return a < b;
                    };
                    for (int v = 0; v < n_models; ++v) {
                        if (state[v] != ST_RESIDENT || outstanding[v] != 0) continue;
                        if (!queue[v].empty() && !head_less(m, v)) continue;   // older head: not a victim
                        if (best < 0 || key_less(v, best)) best = v;
                    }
                    if (best >= 0) {
                        const int sv = offload(best, out);
                        load(m, sv, out);
                    }
                }
                blocked[m] = 1;
            }
        }
    }
    // events ------------------------------------------------------------------------------
    void arrival(int64_t rid, int m, double t, std::vector<Decision>& out) {
        queue[m].push_back({rid, t});
        schedule(t, out);
    }
    void ack(uint64_t e, int rank, double t, std::vector<Decision>& out) {
        auto it = pending.find(e);
        if (it == pending.end()) throw Error(MPSW_EINVARIANT, "ack for unknown entry");
        if (it->second.mask & (1u << rank)) throw Error(MPSW_EINVARIANT, "duplicate ack");
        it->second.mask |= 1u << rank;
        if (--it->second.left == 0) {
            state[it->second.model] = it->second.kind == E_LOAD ? ST_RESIDENT : ST_EVICTED;
            pending.erase(it);
        }
        schedule(t, out);
    }
    void batch_done(uint64_t b, double t, std::vector<Decision>& out) {
        auto it = batches.find(b);
        if (it == batches.end()) throw Error(MPSW_EINVARIANT, "unknown batch");
        Decision d{3, b, it->second.first};
        d.rids = it->second.second;
        --outstanding[it->second.first];
        --inflight;
        batches.erase(it);
        out.push_back(std::move(d));
        schedule(t, out);
    }
    void cmd_swap_in(int m, double t, std::vector<Decision>& out) {
        const int st = state[m];
        if (st == ST_RESIDENT || st == ST_LOADING) {
            out.push_back(Decision{4, 0, m});
        } else if (st == ST_OFFLOADING) {
            Decision d{5, 0, m};
            d.status = "EBUSY";
            out.push_back(d);
        } else {
            const int s = free_slot();
            if (s < 0) {
                Decision d{5, 0, m};
                d.status = "ENOMEM";
                out.push_back(d);
            } else {
                load(m, s, out);
            }
        }
        schedule(t, out);
    }
    void cmd_swap_out(int m, double t, std::vector<Decision>& out) {
        const int st = state[m];
        if (st == ST_EVICTED || st == ST_OFFLOADING) {
            out.push_back(Decision{4, 0, m});
        } else if (st == ST_LOADING || outstanding[m] > 0) {
            Decision d{5, 0, m};
            d.status = "EBUSY";
            out.push_back(d);
        } else {
            offload(m, out);
        }
        schedule(t, out);
    }
    void check() const {
        int owned = 0;
        for (int s = 0; s < k; ++s)
            if (owner[s] >= 0) ++owned;
        if (owned > k) throw Error(MPSW_EINVARIANT, "more owned slots than k");
        for (int m = 0; m < n_models; ++m) {
            if (outstanding[m] > 0 && state[m] != ST_RESIDENT)
                throw Error(MPSW_EINVARIANT, "in-flight batch on a non-resident model");
            if ((state[m] == ST_LOADING || state[m] == ST_RESIDENT) && owner[slot_of[m]] != m)
                throw Error(MPSW_EINVARIANT, "slot ownership");
        }
        if (inflight > D) throw Error(MPSW_EINVARIANT, "D exceeded");
    }
};

// ----------------------------------------------------------------------------- per-rank state
struct Slot {
    uint8_t* base = nullptr;
    std::vector<cudaEvent_t> chunk_gate;   // recorded by the last writeback offload, per chunk
    bool chunk_gate_valid = false;
    cudaEvent_t whole_gate = nullptr;      // clean eviction: last forward that read the slot
    bool whole_gate_valid = false;
};

struct Rank {
    int index = 0, device = 0, numa = -1;
    cudaStream_t compute = nullptr, h2d = nullptr, d2h = nullptr, aux = nullptr;
    uint8_t* region = nullptr;             // param budget (one cudaMalloc)
    std::vector<Slot> slots;
    uint8_t* ws_base = nullptr;
    FwdWorkspace ws;
    std::vector<TensorPtrs> wptr;          // per slot
    cudaEvent_t ev_point[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> last_compute; // per model
    std::vector<char> last_compute_valid;
    unsigned long long* d_sum = nullptr;
    // worker
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<EntryP> fifo;
};

struct Model {
    mpsw_opt_dims dims;
    std::vector<PinnedBuf> arena;  // per rank
};

struct Cmd {
    int kind;  // 0 arrival, 1 swap_in, 2 swap_out
    int model;
    std::shared_ptr<ReqRec> req;
    std::promise<std::pair<mpsw_status, uint64_t>>* reply = nullptr;
};

}  // namespace
}  // namespace mpsw

struct mpsw_ctx {
    mpsw_config cfg{};
    std::vector<int> device_ids;
    std::chrono::steady_clock::time_point t0;
    int tp = 1, D = 1;
    uint64_t chunk = 64ull << 20;
    std::vector<std::unique_ptr<mpsw::Rank>> ranks;
    std::vector<std::unique_ptr<mpsw::Model>> models;
    // geometry (fixed by the first registered model; homogeneous slots)
    bool geom = false;
    mpsw_opt_dims dims{};
    mpsw::Layout layout;
    uint64_t S = 0, slot_stride = 0;
    int k = 0, n_chunks = 0;
    mpsw::FwdShape fshape{};
    int max_rows = 0;
    // logits / tokens staging ring (pinned), D + 1 entries
    int ring_n = 2;
    mpsw::PinnedBuf staging;
    size_t ring_stride = 0, ring_tok_off = 0;
    // engine
    mpsw::StateMachine sm;
    std::mutex cmd_mu;
    std::condition_variable cmd_cv;
    std::deque<mpsw::Cmd> cmds;
    std::thread engine;
    std::atomic<bool> stop{false};
    std::atomic<int> poisoned{0};
    std::string poison_msg;
    std::vector<mpsw::EntryP> inflight;
    std::mutex done_mu;
    std::condition_variable done_cv;
    std::unordered_map<uint64_t, mpsw::EntryP> entries;        // swap entries by ticket
    std::unordered_map<int64_t, std::shared_ptr<mpsw::ReqRec>> reqs;
    std::atomic<int64_t> next_rid{0};
    int ring_next = 0;
    mpsw::SpinBarrier barrier;
    std::mutex api_mu;  // serialises register / swap / request submission
    // trace + stats
    bool trace = false;
    std::mutex trace_mu;
    std::vector<std::string> trace_lines;
    std::mutex sm_mu;   // guards sm against readers (residency/checksum) and registration
    std::unordered_map<int64_t, std::shared_ptr<mpsw::ReqRec>> eng_reqs;   // engine-private
    std::atomic<uint64_t> launches{0}, h2d_bytes{0}, d2h_bytes{0}, swaps_in{0}, swaps_out{0}, n_batches{0},
        n_requests{0}, rejected{0};
};

namespace mpsw {
namespace {

std::string fmt_d(double v) {
    char b[64];
    std::snprintf(b, sizeof(b), "%.17g", v);
    return b;
}

void poison(mpsw_ctx* c, const std::string& msg) {
    if (!c->poisoned.exchange(1)) c->poison_msg = msg;
    std::fprintf(stderr, "[mpsw] ctx poisoned: %s\n", msg.c_str());
    c->done_cv.notify_all();
}

bool use_zero_copy(mpsw_ctx* c, uint64_t bytes) {
    if (c->cfg.swap_mode == MPSW_SWAP_ZERO_COPY) return true;
    if (c->cfg.swap_mode == MPSW_SWAP_COPY_ENGINE) return false;
    return bytes <= (4ull << 20);   // AUTO: small shards skip DMA setup (measured crossover: bench cfg5)
}

int zc_ctas(mpsw_ctx* c) { return c->cfg.zc_ctas > 0 ? c->cfg.zc_ctas : 32; }

// ----------------------------------------------------------------------------- worker issue
void issue_load(mpsw_ctx* c, Rank& R, Entry& e) {
    Slot& sl = R.slots[e.slot];
    const uint8_t* src = c->models[e.model]->arena[R.index].p;
    const bool zc = use_zero_copy(c, c->S);
    MPSW_CU(cudaEventCreate(&e.ev_start[R.index]));
    MPSW_CU(cudaEventCreate(&e.ev_done[R.index]));
    MPSW_CU(cudaEventRecord(e.ev_start[R.index], R.h2d));
    if (sl.whole_gate_valid) MPSW_CU(cudaStreamWaitEvent(R.h2d, sl.whole_gate, 0));
    if (!sl.chunk_gate_valid && zc) {
        launch_zero_copy(sl.base, src, c->S, zc_ctas(c), R.h2d);
        c->launches++;
    } else {
        for (int i = 0; i < c->n_chunks; ++i) {
            const uint64_t off = (uint64_t)i * c->chunk, n = std::min<uint64_t>(c->chunk, c->S - off);
            if (sl.chunk_gate_valid) MPSW_CU(cudaStreamWaitEvent(R.h2d, sl.chunk_gate[i], 0));
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
    MPSW_CU(cudaEventRecord(e.ev_done[R.index], R.h2d));
}

void issue_offload(mpsw_ctx* c, Rank& R, Entry& e) {
    Slot& sl = R.slots[e.slot];
    uint8_t* dst = c->models[e.model]->arena[R.index].p;
    const bool zc = use_zero_copy(c, c->S);
    MPSW_CU(cudaEventCreate(&e.ev_start[R.index]));
    MPSW_CU(cudaEventCreate(&e.ev_done[R.index]));
    // eviction never races an in-flight request: the D2H stream waits for the last forward
    // that read the victim (the engine also only evicts models with no in-flight batch)
    if (R.last_compute_valid[e.model]) MPSW_CU(cudaStreamWaitEvent(R.d2h, R.last_compute[e.model], 0));
    MPSW_CU(cudaEventRecord(e.ev_start[R.index], R.d2h));
    if (c->cfg.writeback) {
        for (int i = 0; i < c->n_chunks; ++i) {
            const uint64_t off = (uint64_t)i * c->chunk, n = std::min<uint64_t>(c->chunk, c->S - off);
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
    MPSW_CU(cudaEventRecord(e.ev_done[R.index], R.d2h));
}

void issue_batch(mpsw_ctx* c, Rank& R, Entry& e) {
    const FwdShape& s = c->fshape;
    FwdShape sr = s;
    sr.rank = R.index;
    const int B = (int)e.reqs.size(), M = e.M;
    const TensorPtrs& Wt = R.wptr[e.slot];
    cudaStream_t cs = R.compute;
    const int r = R.index, t = c->tp;
    MPSW_CU(cudaEventCreateWithFlags(&e.ev_done[r], cudaEventDisableTiming));
    // tokens + meta (packed by the engine into the pinned ring entry)
    uint8_t* ring = c->staging.p + (size_t)e.ring * c->ring_stride;
    const size_t meta_n = (size_t)(3 * B + 1 + M);
    MPSW_CU(cudaMemcpyAsync(R.ws.tokens, ring + c->ring_tok_off, (size_t)M * 4, cudaMemcpyHostToDevice, cs));
    MPSW_CU(cudaMemcpyAsync(R.ws.meta, ring + c->ring_tok_off + (size_t)c->max_rows * 4, meta_n * 4,
                            cudaMemcpyHostToDevice, cs));
    const int32_t* pos = R.ws.meta + 2 * B + 1;
    int nl = 0, point = 0;
    // all-reduce point: record my partial, barrier with the other rank threads, then wait for
    // every peer's partial on my stream and run the fused reduce+residual+bias+LN kernel.
    auto allreduce_ln = [&](float* mine, const float* residual, const void* bias, const void* pos_table,
                            const void* g, const void* b) {
        const int pb = point & 1;
        const float* peers[kMaxRanks];
        if (t > 1) {
            MPSW_CU(cudaEventRecord(R.ev_point[pb], cs));
            c->barrier.wait();
            for (int p = 0; p < t; ++p)
                if (p != r) MPSW_CU(cudaStreamWaitEvent(cs, c->ranks[p]->ev_point[pb], 0));
        }
        for (int p = 0; p < t; ++p) peers[p] = c->ranks[p]->ws.partial[pb];
        (void)mine;
        nl += fwd_reduce_ln(sr, M, peers, t, residual, bias, pos_table, pos, g, b, R.ws.x, R.ws.a, cs);
        ++point;
    };
    nl += fwd_embed(sr, Wt, R.ws, M, R.ws.partial[point & 1], cs);
    allreduce_ln(R.ws.partial[point & 1], nullptr, nullptr, Wt.embed_pos, Wt.layers[0].ln1_w, Wt.layers[0].ln1_b);
    for (int l = 0; l < s.n_layers; ++l) {
        const auto& L = Wt.layers[l];
        nl += fwd_qkv(sr, L, R.ws, M, cs);
        nl += fwd_attention(sr, R.ws, B, cs);
        nl += fwd_out_proj(sr, L, R.ws, M, R.ws.partial[point & 1], cs);
        allreduce_ln(R.ws.partial[point & 1], R.ws.x, L.o_b, nullptr, L.ln2_w, L.ln2_b);
        nl += fwd_fc1(sr, L, R.ws, M, cs);
        nl += fwd_fc2(sr, L, R.ws, M, R.ws.partial[point & 1], cs);
        const bool last = l + 1 == s.n_layers;
        allreduce_ln(R.ws.partial[point & 1], R.ws.x, L.fc2_b, nullptr, last ? Wt.lnf_w : Wt.layers[l + 1].ln1_w,
                     last ? Wt.lnf_b : Wt.layers[l + 1].ln1_b);
    }
    nl += fwd_lm_head(sr, Wt, R.ws, B, cs);
    float* logits_host = (float*)(ring) + (size_t)r * s.vocab_local;
    MPSW_CU(cudaMemcpy2DAsync(logits_host, (size_t)s.vocab * 4, R.ws.logits, (size_t)s.vocab_local * 4,
                              (size_t)s.vocab_local * 4, B, cudaMemcpyDeviceToHost, cs));
    MPSW_CU(cudaEventRecord(e.ev_done[r], cs));
    MPSW_CU(cudaEventRecord(R.last_compute[e.model], cs));
    R.last_compute_valid[e.model] = 1;
    c->launches += nl;
}

void worker_main(mpsw_ctx* c, Rank* R) {
    cudaSetDevice(R->device);
    for (;;) {
        EntryP e;
        {
            std::unique_lock<std::mutex> lk(R->mu);
            R->cv.wait(lk, [&] { return !R->fifo.empty() || c->stop.load(); });
            if (R->fifo.empty()) return;
            e = R->fifo.front();
            R->fifo.pop_front();
        }
        try {
            if (!c->poisoned.load()) {
                if (e->kind == E_LOAD) issue_load(c, *R, *e);
                else if (e->kind == E_OFFLOAD) issue_offload(c, *R, *e);
                else issue_batch(c, *R, *e);
            }
        } catch (const Error& err) {
            poison(c, err.what());
        } catch (const std::exception& err) {
            poison(c, err.what());
        }
        e->issued[R->index].store(1, std::memory_order_release);
        c->cmd_cv.notify_all();
    }
}

// ----------------------------------------------------------------------------- engine thread
void log_event(mpsw_ctx* c, const std::string& s) {
    if (!c->trace) return;
    std::lock_guard<std::mutex> lk(c->trace_mu);
    c->trace_lines.push_back(s);
}

void log_decisions(mpsw_ctx* c, const std::vector<Decision>& ds) {
    if (!c->trace) return;
    for (const auto& d : ds) {
        std::ostringstream o;
        switch (d.kind) {
            case 0: o << "{\"dec\":\"load\",\"id\":" << d.id << ",\"model\":" << d.model << ",\"slot\":" << d.slot << "}"; break;
            case 1: o << "{\"dec\":\"offload\",\"id\":" << d.id << ",\"model\":" << d.model << ",\"slot\":" << d.slot << "}"; break;
            case 2:
            case 3: {
                o << "{\"dec\":\"" << (d.kind == 2 ? "batch" : "complete") << "\",\"id\":" << d.id;
                if (d.kind == 2) o << ",\"model\":" << d.model;
                o << ",\"rids\":[";
                for (size_t i = 0; i < d.rids.size(); ++i) o << (i ? "," : "") << d.rids[i];
                o << "]}";
                break;
            }
            case 4: o << "{\"dec\":\"noop\",\"model\":" << d.model << "}"; break;
            default: o << "{\"dec\":\"reject\",\"model\":" << d.model << ",\"status\":\"" << d.status << "\"}"; break;
        }
        std::lock_guard<std::mutex> lk(c->trace_mu);
        c->trace_lines.push_back(o.str());
    }
}

void dispatch(mpsw_ctx* c, const std::vector<Decision>& ds, double now) {
    for (const auto& d : ds) {
        if (d.kind > 2) continue;
        auto e = std::make_shared<Entry>();
        e->id = d.id;
        e->kind = d.kind;
        e->model = d.model;
        e->slot = d.slot;
        e->t_submit = now;
        if (d.kind == E_BATCH) {
            e->slot = c->sm.slot_of[d.model];
            // pack tokens + meta into the pinned ring entry
            e->ring = c->ring_next;
            c->ring_next = (c->ring_next + 1) % c->ring_n;
            uint8_t* ring = c->staging.p + (size_t)e->ring * c->ring_stride;
            int32_t* tok = (int32_t*)(ring + c->ring_tok_off);
            int32_t* meta = tok + c->max_rows;
            const int B = (int)d.rids.size();
            int M = 0;
            for (int b = 0; b < B; ++b) {
                auto rq = c->eng_reqs.at(d.rids[b]);
                e->reqs.push_back(rq);
                meta[b] = M;
                for (size_t i = 0; i < rq->tokens.size(); ++i) {
                    tok[M] = rq->tokens[i];
                    meta[2 * B + 1 + M] = (int32_t)i + 2;   // position id + 2 offset (HF:opt.py:53)
                    ++M;
                }
                meta[B + 1 + b] = M - 1;                    // last row of request b (lm_head)
            }
            meta[B] = M;
            e->M = M;
        } else {
            std::lock_guard<std::mutex> lk(c->done_mu);
            c->entries[e->id] = e;
        }
        c->inflight.push_back(e);
        for (auto& R : c->ranks) {
            std::lock_guard<std::mutex> lk(R->mu);
            R->fifo.push_back(e);
            R->cv.notify_one();
        }
    }
}

void step_and_dispatch(mpsw_ctx* c, const std::function<void(std::vector<Decision>&)>& fn, double now) {
    std::vector<Decision> ds;
    std::lock_guard<std::mutex> lk(c->sm_mu);
    fn(ds);
    c->sm.check();
    log_decisions(c, ds);
    dispatch(c, ds, now);
}

void complete_batch(mpsw_ctx* c, Entry& e, double now) {
    const uint8_t* ring = c->staging.p + (size_t)e.ring * c->ring_stride;
    const int V = c->fshape.vocab;
    for (size_t b = 0; b < e.reqs.size(); ++b) {
        auto& rq = e.reqs[b];
        std::memcpy(rq->out, (const float*)ring + b * (size_t)V, (size_t)V * 4);
        rq->t_done = now;
        c->eng_reqs.erase(rq->rid);
    }
    {
        std::lock_guard<std::mutex> lk(c->done_mu);
        for (auto& rq : e.reqs) rq->done.store(1, std::memory_order_release);
    }
    c->n_batches++;
    c->n_requests += e.reqs.size();
    c->done_cv.notify_all();
}

bool poll_inflight(mpsw_ctx* c) {
    bool progressed = false;
    for (size_t i = 0; i < c->inflight.size();) {
        Entry& e = *c->inflight[i];
        bool finished = false;
        for (int r = 0; r < c->tp; ++r) {
            if (e.acked[r] || !e.issued[r].load(std::memory_order_acquire)) continue;
            cudaError_t q = e.ev_done[r] ? cudaEventQuery(e.ev_done[r]) : cudaSuccess;
            if (q == cudaErrorNotReady) continue;
            if (q != cudaSuccess) throw Error(MPSW_ECUDA, std::string("copy/forward failed: ") + cudaGetErrorString(q));
            const double now = now_s(c->t0);
            e.acked[r] = 1;
            e.t_ack[r] = now;
            ++e.n_acked;
            progressed = true;
            if (e.kind != E_BATCH) {
                // per-rank ack event ("sends a response back to the engine")
                log_event(c, "{\"ev\":\"ack\",\"t\":" + fmt_d(now) + ",\"entry\":" + std::to_string(e.id) +
                                 ",\"rank\":" + std::to_string(r) + "}");
                step_and_dispatch(c, [&](std::vector<Decision>& ds) { c->sm.ack(e.id, r, now, ds); }, now);
                if (e.kind == E_LOAD) c->h2d_bytes += c->S;
                else if (c->cfg.writeback) c->d2h_bytes += c->S;
            }
        }
        if (e.n_acked == c->tp) {
            const double now = now_s(c->t0);
            if (e.kind == E_BATCH) {
                complete_batch(c, e, now);
                log_event(c, "{\"ev\":\"batch_done\",\"t\":" + fmt_d(now) + ",\"batch\":" + std::to_string(e.id) + "}");
                step_and_dispatch(c, [&](std::vector<Decision>& ds) { c->sm.batch_done(e.id, now, ds); }, now);
                for (int r = 0; r < c->tp; ++r)
                    if (e.ev_done[r]) cudaEventDestroy(e.ev_done[r]), e.ev_done[r] = nullptr;
            } else {
                (e.kind == E_LOAD ? c->swaps_in : c->swaps_out)++;
                std::lock_guard<std::mutex> lk(c->done_mu);
                e.complete.store(1, std::memory_order_release);
            }
            c->done_cv.notify_all();
            finished = true;
        }
        if (finished) c->inflight.erase(c->inflight.begin() + i);
        else ++i;
    }
    return progressed;
}

void engine_main(mpsw_ctx* c) {
    cudaSetDevice(c->ranks[0]->device);
    int idle_spins = 0;
    while (true) {
        std::deque<Cmd> batch;
        {
            std::unique_lock<std::mutex> lk(c->cmd_mu);
            if (c->cmds.empty() && c->inflight.empty()) {
                if (c->stop.load()) break;
                c->cmd_cv.wait_for(lk, std::chrono::milliseconds(2));
            }
            batch.swap(c->cmds);
        }
        try {
            for (auto& cmd : batch) {
                if (c->poisoned.load()) {
                    if (cmd.reply) cmd.reply->set_value({MPSW_ECUDA, 0});
                    continue;
                }
                if (cmd.kind == 0) {
                    auto& rq = cmd.req;
                    c->eng_reqs[rq->rid] = rq;
                    log_event(c, "{\"ev\":\"arrival\",\"t\":" + fmt_d(rq->t_arr) + ",\"rid\":" + std::to_string(rq->rid) +
                                     ",\"model\":" + std::to_string(rq->model) + "}");
                    const double now = rq->t_arr;
                    step_and_dispatch(c, [&](std::vector<Decision>& ds) { c->sm.arrival(rq->rid, rq->model, now, ds); },
                                      now_s(c->t0));
                } else {
                    const double now = now_s(c->t0);
                    log_event(c, std::string("{\"ev\":\"") + (cmd.kind == 1 ? "cmd_swap_in" : "cmd_swap_out") +
                                     "\",\"t\":" + fmt_d(now) + ",\"model\":" + std::to_string(cmd.model) + "}");
                    std::vector<Decision> ds;
                    std::unique_lock<std::mutex> smlk(c->sm_mu);
                    if (cmd.kind == 1) c->sm.cmd_swap_in(cmd.model, now, ds);
                    else c->sm.cmd_swap_out(cmd.model, now, ds);
                    c->sm.check();
                    log_decisions(c, ds);
                    mpsw_status st = MPSW_OK;
                    uint64_t ticket = kNoopTicket;
                    const Decision& first = ds.front();
                    if (first.kind == 5) st = std::strcmp(first.status, "EBUSY") == 0 ? MPSW_EBUSY : MPSW_ENOMEM;
                    else if (first.kind <= 1) ticket = first.id;
                    dispatch(c, ds, now);
                    smlk.unlock();
                    cmd.reply->set_value({st, ticket});
                }
            }
            const bool prog = poll_inflight(c);
            if (!c->inflight.empty()) {
                if (prog) idle_spins = 0;
                else if (++idle_spins > 64) std::this_thread::yield();
                else _mm_pause();
            }
        } catch (const std::exception& err) {
            poison(c, err.what());
            for (auto& cmd : batch)
                if (cmd.reply) try { cmd.reply->set_value({MPSW_EINVARIANT, 0}); } catch (...) {}
            c->inflight.clear();
        }
    }
}

TensorPtrs make_ptrs(const Layout& L, const uint8_t* base, int n_layers) {
    TensorPtrs w;
    auto p = [&](int i) { return (const void*)(base + L.t[i].offset); };
    w.embed_tok = p(0);
    w.embed_pos = p(1);
    w.lnf_w = p(2);
    w.lnf_b = p(3);
    for (int l = 0; l < n_layers; ++l) {
        const int b = 4 + 16 * l;
        TensorPtrs::Layer x;
        x.k_w = p(b + 0); x.k_b = p(b + 1); x.v_w = p(b + 2); x.v_b = p(b + 3);
        x.q_w = p(b + 4); x.q_b = p(b + 5); x.o_w = p(b + 6); x.o_b = p(b + 7);
        x.ln1_w = p(b + 8); x.ln1_b = p(b + 9); x.fc1_w = p(b + 10); x.fc1_b = p(b + 11);
        x.fc2_w = p(b + 12); x.fc2_b = p(b + 13); x.ln2_w = p(b + 14); x.ln2_b = p(b + 15);
        w.layers.push_back(x);
    }
    return w;
}

// Fix the slot geometry at the first registration: k = floor(budget / S_r) slots per rank
// carved from the region allocated at init; workspaces sized for max_batch * max_tokens rows.
void setup_geometry(mpsw_ctx* c, const mpsw_opt_dims& d) {
    Layout L;
    if (compute_layout(d, c->tp, 0, c->cfg.dtype, L) != MPSW_OK) throw Error(MPSW_EINVAL, tls_error());
    const int hd = d.hidden / d.heads;
    if (hd % 8 || hd > 128) throw Error(MPSW_EINVAL, "head_dim must be a multiple of 8 and <= 128");
    if ((d.hidden / c->tp) % 8 || (d.ffn / c->tp) % 8 || d.hidden % 8)
        throw Error(MPSW_EINVAL, "hidden/tp, ffn/tp and hidden must be multiples of 8");
    if (d.hidden > 12288) throw Error(MPSW_EINVAL, "hidden too large for the LN kernel");
    const uint64_t S = L.bytes;
    const uint64_t stride = (S + kSlotAlign - 1) / kSlotAlign * kSlotAlign;
    const int k = (int)std::min<uint64_t>(c->cfg.param_budget_bytes_per_gpu / stride, 1024);
    if (k < 1) throw Error(MPSW_ENOMEM, "param budget cannot hold one shard (S_r = " + std::to_string(S) + ")");
    c->dims = d;
    c->layout = L;
    c->S = S;
    c->slot_stride = stride;
    c->k = k;
    c->n_chunks = (int)((S + c->chunk - 1) / c->chunk);
    FwdShape& f = c->fshape;
    f.n_layers = d.n_layers; f.hidden = d.hidden; f.heads_local = d.heads / c->tp; f.head_dim = hd;
    f.ffn_local = d.ffn / c->tp; f.vocab_local = d.vocab / c->tp; f.vocab = d.vocab; f.tp = c->tp; f.rank = 0;
    f.dtype = c->cfg.dtype;
    c->max_rows = c->cfg.max_batch * c->cfg.max_tokens;
    const size_t wsb = workspace_bytes(f, c->max_rows, c->cfg.max_batch);
    for (auto& Rp : c->ranks) {
        Rank& R = *Rp;
        MPSW_CU(cudaSetDevice(R.device));
        R.slots.resize(k);
        for (int s = 0; s < k; ++s) {
            Slot& sl = R.slots[s];
            sl.base = R.region + (uint64_t)s * stride;
            sl.chunk_gate.resize(c->n_chunks);
            for (auto& ev : sl.chunk_gate) MPSW_CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            MPSW_CU(cudaEventCreateWithFlags(&sl.whole_gate, cudaEventDisableTiming));
            R.wptr.push_back(make_ptrs(L, sl.base, d.n_layers));
        }
        MPSW_CU(cudaMalloc(&R.ws_base, wsb));
        MPSW_CU(cudaMemset(R.ws_base, 0, wsb));
        workspace_carve(R.ws, f, c->max_rows, c->cfg.max_batch, R.ws_base);
        for (auto& ev : R.ev_point) MPSW_CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    // staging ring: per entry [max_batch * V] fp32 logits, then tokens [max_rows] + meta
    c->ring_n = c->D + 1;
    const size_t logits_b = ((size_t)c->cfg.max_batch * d.vocab * 4 + 255) & ~size_t(255);
    c->ring_tok_off = logits_b;
    c->ring_stride = (logits_b + (size_t)(c->max_rows * 2 + 3 * c->cfg.max_batch + 8) * 4 + 4095) & ~size_t(4095);
    c->staging = pin_alloc(c->ring_stride * c->ring_n, c->ranks[0]->numa);
    {
        std::lock_guard<std::mutex> lk(c->sm_mu);
        c->sm.k = k;
        c->sm.owner.assign(k, -1);
    }
    c->geom = true;
}

}  // namespace
}  // namespace mpsw

using namespace mpsw;

#define API_BEGIN try {
#define API_END                                                               \
    }                                                                         \
    catch (const Error& e) { return set_error(e.status, e.what()); }         \
    catch (const std::exception& e) { return set_error(MPSW_EINVAL, e.what()); }

extern "C" {

const char* mpsw_last_error(void) { return tls_error().c_str(); }

mpsw_status mpsw_shard_layout(const mpsw_opt_dims* dims, int tp, int rank, int dtype, mpsw_tensor_desc* out,
                              int cap, int* n, uint64_t* shard_bytes) {
    API_BEGIN
    if (!dims) return set_error(MPSW_EINVAL, "dims is NULL");
    Layout L;
    mpsw_status s = compute_layout(*dims, tp, rank, dtype, L);
    if (s != MPSW_OK) return s;
    if (n) *n = (int)L.t.size();
    if (shard_bytes) *shard_bytes = L.bytes;
    if (out)
        for (int i = 0; i < cap && i < (int)L.t.size(); ++i) out[i] = L.t[i];
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_init(const mpsw_config* cfg, mpsw_ctx** out) {
    API_BEGIN
    if (!cfg || !out) return set_error(MPSW_EINVAL, "NULL argument");
    if (cfg->n_gpus < 1 || cfg->n_gpus > kMaxRanks || !cfg->device_ids)
        return set_error(MPSW_EINVAL, "n_gpus must be 1..8 with device_ids");
    if (cfg->tp != cfg->n_gpus) return set_error(MPSW_EINVAL, "tp must equal n_gpus (one TP group per ctx)");
    if (cfg->max_batch < 1 || cfg->max_batch > 256) return set_error(MPSW_EINVAL, "max_batch must be 1..256");
    if (cfg->max_tokens < 1 || cfg->max_tokens > 128) return set_error(MPSW_EINVAL, "max_tokens must be 1..128");
    if (cfg->dtype != MPSW_BF16 && cfg->dtype != MPSW_FP32) return set_error(MPSW_EINVAL, "bad dtype");
    if (cfg->chunk_bytes % 4096) return set_error(MPSW_EINVAL, "chunk_bytes must be a multiple of 4096");
    if (cfg->swap_mode < 0 || cfg->swap_mode > 2) return set_error(MPSW_EINVAL, "bad swap_mode");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) return set_error(MPSW_ECUDA, "no CUDA device");
    auto c = std::make_unique<mpsw_ctx>();
    c->cfg = *cfg;
    c->t0 = std::chrono::steady_clock::now();
    c->tp = cfg->tp;
    c->D = cfg->max_inflight_batches > 0 ? cfg->max_inflight_batches : 1;
    c->chunk = cfg->chunk_bytes ? cfg->chunk_bytes : (64ull << 20);
    c->trace = cfg->trace != 0;
    c->device_ids.assign(cfg->device_ids, cfg->device_ids + cfg->n_gpus);
    c->sm.tp = c->tp;
    c->sm.max_batch = cfg->max_batch;
    c->sm.D = c->D;
    c->barrier.n = c->tp;
    c->models.reserve(kMaxModels);
    for (int r = 0; r < c->tp; ++r) {
        const int dev = c->device_ids[r];
        if (dev < 0 || dev >= ndev) return set_error(MPSW_EINVAL, "device id out of range");
        auto R = std::make_unique<Rank>();
        R->index = r;
        R->device = dev;
        R->numa = gpu_numa_node(dev);
        R->last_compute.reserve(kMaxModels);
        R->last_compute_valid.reserve(kMaxModels);
        MPSW_CU(cudaSetDevice(dev));
        int hp = 0, lp = 0;
        MPSW_CU(cudaDeviceGetStreamPriorityRange(&lp, &hp));
        MPSW_CU(cudaStreamCreateWithPriority(&R->compute, cudaStreamNonBlocking, hp));
        MPSW_CU(cudaStreamCreateWithFlags(&R->h2d, cudaStreamNonBlocking));
        MPSW_CU(cudaStreamCreateWithFlags(&R->d2h, cudaStreamNonBlocking));
        MPSW_CU(cudaStreamCreateWithFlags(&R->aux, cudaStreamNonBlocking));
        if (cfg->param_budget_bytes_per_gpu == 0) return set_error(MPSW_EINVAL, "param budget is 0");
        cudaError_t e = cudaMalloc(&R->region, cfg->param_budget_bytes_per_gpu);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return set_error(MPSW_ENOMEM, std::string("cudaMalloc(param budget): ") + cudaGetErrorString(e));
        }
        MPSW_CU(cudaMalloc(&R->d_sum, sizeof(unsigned long long)));
        c->ranks.push_back(std::move(R));
    }
    // peer access between distinct devices of the group (TP all-reduce reads peer partials)
    for (int a = 0; a < c->tp; ++a)
        for (int b = 0; b < c->tp; ++b) {
            const int da = c->device_ids[a], db = c->device_ids[b];
            if (da == db) continue;
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, da, db);
            if (!ok) return set_error(MPSW_EINVAL, "GPUs of the TP group lack peer access");
            cudaSetDevice(da);
            cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) MPSW_CU(e);
            cudaGetLastError();
        }
    mpsw_ctx* raw = c.release();
    for (auto& R : raw->ranks) R->th = std::thread(worker_main, raw, R.get());
    raw->engine = std::thread(engine_main, raw);
    *out = raw;
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_shutdown(mpsw_ctx* c) {
    if (!c) return MPSW_OK;
    {
        std::lock_guard<std::mutex> lk(c->cmd_mu);
        c->stop.store(true);
    }
    c->cmd_cv.notify_all();
    if (c->engine.joinable()) c->engine.join();
    for (auto& R : c->ranks) {
        {
            std::lock_guard<std::mutex> lk(R->mu);
        }
        R->cv.notify_all();
        if (R->th.joinable()) R->th.join();
    }
    for (auto& R : c->ranks) {
        cudaSetDevice(R->device);
        cudaDeviceSynchronize();
        for (auto& sl : R->slots) {
            for (auto ev : sl.chunk_gate) cudaEventDestroy(ev);
            if (sl.whole_gate) cudaEventDestroy(sl.whole_gate);
        }
        for (auto ev : R->ev_point)
            if (ev) cudaEventDestroy(ev);
        for (auto ev : R->last_compute)
            if (ev) cudaEventDestroy(ev);
        cudaFree(R->region);
        cudaFree(R->ws_base);
        cudaFree(R->d_sum);
        cudaStreamDestroy(R->compute);
        cudaStreamDestroy(R->h2d);
        cudaStreamDestroy(R->d2h);
        cudaStreamDestroy(R->aux);
    }
    for (auto& kv : c->entries)
        for (int r = 0; r < c->tp; ++r) {
            if (kv.second->ev_start[r]) cudaEventDestroy(kv.second->ev_start[r]);
            if (kv.second->ev_done[r]) cudaEventDestroy(kv.second->ev_done[r]);
        }
    for (auto& m : c->models)
        for (auto& a : m->arena) pin_free(a);
    pin_free(c->staging);
    delete c;
    return MPSW_OK;
}

mpsw_status mpsw_register_model(mpsw_ctx* c, const mpsw_opt_dims* dims, int tp, const void* const* shards,
                                const uint64_t* shard_bytes, int* model_id) {
    API_BEGIN
    if (!c || !dims || !model_id) return set_error(MPSW_EINVAL, "NULL argument");
    if (c->poisoned.load()) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
    if (tp != c->tp) return set_error(MPSW_EINVAL, "model tp must equal the ctx tp");
    std::lock_guard<std::mutex> api(c->api_mu);
    Layout L;
    mpsw_status s = compute_layout(*dims, tp, 0, c->cfg.dtype, L);
    if (s != MPSW_OK) return s;
    {
        // the engine thread reads geometry; registration happens while it may be running
        std::lock_guard<std::mutex> lk(c->cmd_mu);
        if (!c->geom) setup_geometry(c, *dims);
        else if (std::memcmp(&c->dims, dims, sizeof(*dims)) != 0)
            return set_error(MPSW_EINVAL, "all models of a ctx must share dims (homogeneous slots, P:229)");
    }
    if (shards && shard_bytes)
        for (int r = 0; r < tp; ++r)
            if (shard_bytes[r] != c->S) return set_error(MPSW_EINVAL, "shard_bytes != S_r of the layout");
    auto m = std::make_unique<Model>();
    m->dims = *dims;
    try {
        for (int r = 0; r < tp; ++r) {
            m->arena.push_back(pin_alloc(c->S, c->ranks[r]->numa));
            if (shards && shards[r]) parallel_memcpy(m->arena[r].p, (const uint8_t*)shards[r], c->S);
        }
    } catch (...) {
        for (auto& a : m->arena) pin_free(a);
        throw;
    }
    for (auto& R : c->ranks) {
        cudaSetDevice(R->device);
        cudaEvent_t ev;
        MPSW_CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        // worker threads read last_compute[model] only for registered models; resize under the
        // cmd lock so the engine never dispatches for a model whose vectors are not ready
        std::lock_guard<std::mutex> lk(R->mu);
        R->last_compute.push_back(ev);
        R->last_compute_valid.push_back(0);
    }
    {
        std::lock_guard<std::mutex> lk(c->cmd_mu);
        std::lock_guard<std::mutex> lk2(c->sm_mu);
        if (c->models.size() >= kMaxModels) return set_error(MPSW_ENOMEM, "too many models");
        c->models.push_back(std::move(m));   // capacity reserved at init: no reallocation
        c->sm.add_model();
        *model_id = (int)c->models.size() - 1;
    }
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_model_arena(mpsw_ctx* c, int model_id, int rank, void** host, uint64_t* bytes) {
    API_BEGIN
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    if (model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_ENOENT, "unknown model");
    if (rank < 0 || rank >= c->tp) return set_error(MPSW_EINVAL, "rank out of range");
    if (host) *host = c->models[model_id]->arena[rank].p;
    if (bytes) *bytes = c->S;
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_synth_fill(mpsw_ctx* c, int model_id, int rank, uint64_t seed, int threads) {
    API_BEGIN
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    if (model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_ENOENT, "unknown model");
    if (rank < -1 || rank >= c->tp) return set_error(MPSW_EINVAL, "rank out of range");
    for (int r = 0; r < c->tp; ++r)
        if (rank < 0 || rank == r)
            synth_fill_arena(c->dims, c->tp, r, c->cfg.dtype, seed, c->models[model_id]->arena[r].p, threads);
    return MPSW_OK;
    API_END
}

static mpsw_status submit_cmd(mpsw_ctx* c, int kind, int model_id, uint64_t* ticket) {
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    if (c->poisoned.load()) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
    if (model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_ENOENT, "unknown model");
    std::promise<std::pair<mpsw_status, uint64_t>> pr;
    auto fut = pr.get_future();
    {
        std::lock_guard<std::mutex> lk(c->cmd_mu);
        c->cmds.push_back(Cmd{kind, model_id, nullptr, &pr});
    }
    c->cmd_cv.notify_all();
    auto res = fut.get();
    if (ticket) *ticket = res.second;
    if (res.first != MPSW_OK)
        return set_error(res.first, res.first == MPSW_EBUSY ? "model busy (in-flight batch, loading or offloading)"
                                                            : res.first == MPSW_ENOMEM ? "no free slot (explicit swaps never evict)"
                                                                                       : "engine failure: " + c->poison_msg);
    return MPSW_OK;
}

mpsw_status mpsw_swap_in(mpsw_ctx* c, int model_id, uint64_t* ticket) {
    API_BEGIN
    return submit_cmd(c, 1, model_id, ticket);
    API_END
}

mpsw_status mpsw_swap_out(mpsw_ctx* c, int model_id, uint64_t* ticket) {
    API_BEGIN
    return submit_cmd(c, 2, model_id, ticket);
    API_END
}

mpsw_status mpsw_wait(mpsw_ctx* c, uint64_t ticket, double timeout_s, double* t_submit, double* t_done_per_rank) {
    API_BEGIN
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    if (ticket == kNoopTicket) {
        if (t_submit) *t_submit = 0;
        return MPSW_OK;
    }
    EntryP e;
    {
        std::lock_guard<std::mutex> lk(c->done_mu);
        auto it = c->entries.find(ticket);
        if (it == c->entries.end()) return set_error(MPSW_ENOENT, "unknown ticket");
        e = it->second;
    }
    std::unique_lock<std::mutex> lk(c->done_mu);
    auto pred = [&] { return e->complete.load() || c->poisoned.load(); };
    if (timeout_s < 0) c->done_cv.wait(lk, pred);
    else if (!c->done_cv.wait_for(lk, std::chrono::duration<double>(timeout_s), pred))
        return set_error(MPSW_ETIMEDOUT, "swap not complete");
    if (!e->complete.load()) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
    if (t_submit) *t_submit = e->t_submit;
    if (t_done_per_rank)
        for (int r = 0; r < c->tp; ++r) t_done_per_rank[r] = e->t_ack[r];
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_entry_gpu_ms(mpsw_ctx* c, uint64_t ticket, int* kind, int* model_id, float* gpu_ms) {
    API_BEGIN
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    EntryP e;
    {
        std::lock_guard<std::mutex> lk(c->done_mu);
        auto it = c->entries.find(ticket);
        if (it == c->entries.end()) return set_error(MPSW_ENOENT, "unknown ticket");
        e = it->second;
    }
    if (!e->complete.load()) return set_error(MPSW_EAGAIN, "not complete");
    if (kind) *kind = e->kind;
    if (model_id) *model_id = e->model;
    if (gpu_ms)
        for (int r = 0; r < c->tp; ++r) {
            float ms = 0;
            MPSW_CU(cudaEventElapsedTime(&ms, e->ev_start[r], e->ev_done[r]));
            gpu_ms[r] = ms;
        }
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_request(mpsw_ctx* c, int model_id, const int32_t* tokens, int n_tokens, float* logits_out,
                         int64_t* request_id) {
    API_BEGIN
    if (!c || !logits_out || !request_id || !tokens) return set_error(MPSW_EINVAL, "NULL argument");
    if (c->poisoned.load()) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
    if (model_id < 0 || model_id >= (int)c->models.size()) {
        c->rejected++;
        return set_error(MPSW_ENOENT, "unknown model");
    }
    if (n_tokens < 1 || n_tokens > c->cfg.max_tokens || n_tokens > c->dims.max_pos)
        return set_error(MPSW_EINVAL, "n_tokens out of range");
    for (int i = 0; i < n_tokens; ++i)
        if (tokens[i] < 0 || tokens[i] >= c->dims.vocab) return set_error(MPSW_EINVAL, "token id out of range");
    auto rq = std::make_shared<ReqRec>();
    rq->model = model_id;
    rq->tokens.assign(tokens, tokens + n_tokens);
    rq->out = logits_out;
    {
        std::lock_guard<std::mutex> lk(c->cmd_mu);
        rq->rid = c->next_rid++;
        rq->t_arr = now_s(c->t0);   // P:74 "pushes the request object along with a timestamp"
        c->reqs[rq->rid] = rq;
        c->cmds.push_back(Cmd{0, model_id, rq, nullptr});
    }
    c->cmd_cv.notify_all();
    *request_id = rq->rid;
    return MPSW_OK;
    API_END
}

static std::shared_ptr<ReqRec> find_req(mpsw_ctx* c, int64_t rid) {
    std::lock_guard<std::mutex> lk(c->cmd_mu);
    auto it = c->reqs.find(rid);
    return it == c->reqs.end() ? nullptr : it->second;
}

mpsw_status mpsw_poll(mpsw_ctx* c, int64_t rid, double* t_arrival, double* t_done) {
    API_BEGIN
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    auto rq = find_req(c, rid);
    if (!rq) return set_error(MPSW_ENOENT, "unknown request");
    if (!rq->done.load(std::memory_order_acquire)) {
        if (c->poisoned.load()) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
        return set_error(MPSW_EAGAIN, "pending");
    }
    if (t_arrival) *t_arrival = rq->t_arr;
    if (t_done) *t_done = rq->t_done;
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_wait_request(mpsw_ctx* c, int64_t rid, double timeout_s, double* t_arrival, double* t_done) {
    API_BEGIN
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    auto rq = find_req(c, rid);
    if (!rq) return set_error(MPSW_ENOENT, "unknown request");
    std::unique_lock<std::mutex> lk(c->done_mu);
    auto pred = [&] { return rq->done.load() || c->poisoned.load(); };
    if (timeout_s < 0) c->done_cv.wait(lk, pred);
    else if (!c->done_cv.wait_for(lk, std::chrono::duration<double>(timeout_s), pred))
        return set_error(MPSW_ETIMEDOUT, "request not complete");
    if (!rq->done.load()) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
    if (t_arrival) *t_arrival = rq->t_arr;
    if (t_done) *t_done = rq->t_done;
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_residency(mpsw_ctx* c, int model_id, int* state) {
    API_BEGIN
    if (!c || !state) return set_error(MPSW_EINVAL, "NULL argument");
    std::lock_guard<std::mutex> lk(c->sm_mu);
    if (model_id < 0 || model_id >= c->sm.n_models) return set_error(MPSW_ENOENT, "unknown model");
    *state = c->sm.state[model_id];
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_checksum(mpsw_ctx* c, int model_id, int rank, int on_device, uint64_t* out) {
    API_BEGIN
    if (!c || !out) return set_error(MPSW_EINVAL, "NULL argument");
    if (model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_ENOENT, "unknown model");
    if (rank < 0 || rank >= c->tp) return set_error(MPSW_EINVAL, "rank out of range");
    if (!on_device) {
        *out = host_checksum(c->models[model_id]->arena[rank].p, c->S, 0);
        return MPSW_OK;
    }
    int slot = -1;
    {
        std::lock_guard<std::mutex> lk(c->sm_mu);
        if (c->sm.state[model_id] != ST_RESIDENT) return set_error(MPSW_EINVAL, "model not RESIDENT");
        slot = c->sm.slot_of[model_id];
    }
    Rank& R = *c->ranks[rank];
    MPSW_CU(cudaSetDevice(R.device));
    MPSW_CU(cudaMemsetAsync(R.d_sum, 0, 8, R.aux));
    launch_checksum(R.slots[slot].base, c->S, R.d_sum, R.aux);
    c->launches += 2;
    unsigned long long h = 0;
    MPSW_CU(cudaMemcpyAsync(&h, R.d_sum, 8, cudaMemcpyDeviceToHost, R.aux));
    MPSW_CU(cudaStreamSynchronize(R.aux));
    *out = h;
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_peek(mpsw_ctx* c, int model_id, int rank, uint64_t offset, uint64_t bytes, void* dst) {
    API_BEGIN
    if (!c || !dst) return set_error(MPSW_EINVAL, "NULL argument");
    if (model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_ENOENT, "unknown model");
    if (rank < 0 || rank >= c->tp || offset + bytes > c->S) return set_error(MPSW_EINVAL, "range");
    int slot = -1;
    {
        std::lock_guard<std::mutex> lk(c->sm_mu);
        if (c->sm.state[model_id] != ST_RESIDENT) return set_error(MPSW_EINVAL, "model not RESIDENT");
        slot = c->sm.slot_of[model_id];
    }
    Rank& R = *c->ranks[rank];
    MPSW_CU(cudaSetDevice(R.device));
    MPSW_CU(cudaMemcpyAsync(dst, R.slots[slot].base + offset, bytes, cudaMemcpyDeviceToHost, R.aux));
    MPSW_CU(cudaStreamSynchronize(R.aux));
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_trace_dump(mpsw_ctx* c, const char* path) {
    API_BEGIN
    if (!c || !path) return set_error(MPSW_EINVAL, "NULL argument");
    if (!c->trace) return set_error(MPSW_EINVAL, "trace disabled (cfg.trace = 0)");
    std::lock_guard<std::mutex> lk(c->trace_mu);
    std::ofstream f(path);
    if (!f) return set_error(MPSW_EINVAL, "cannot open trace path");
    for (const auto& l : c->trace_lines) f << l << "\n";
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_get_stats(mpsw_ctx* c, mpsw_stats* o) {
    API_BEGIN
    if (!c || !o) return set_error(MPSW_EINVAL, "NULL argument");
    o->kernel_launches = c->launches.load();
    o->h2d_bytes = c->h2d_bytes.load();
    o->d2h_bytes = c->d2h_bytes.load();
    o->swaps_in = c->swaps_in.load();
    o->swaps_out = c->swaps_out.load();
    o->batches = c->n_batches.load();
    o->requests = c->n_requests.load();
    o->rejected = c->rejected.load();
    o->k_slots = c->k;
    o->shard_bytes = c->S;
    return MPSW_OK;
    API_END
}

}  // extern "C"
