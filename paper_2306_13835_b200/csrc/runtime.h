// Runtime types shared by the library's translation units (not part of the C-ABI): pinned
// store, shm control plane, entries, per-rank state, the ctx, and cross-file function decls.
#pragma once

#include "internal.h"
#include "statemachine.h"

#include <immintrin.h>

#include <functional>
#include <tuple>
#include <future>
#include <map>
#include <string>
#include <unordered_map>

namespace mpsw {

constexpr uint64_t kNoopTicket = ~0ull;
constexpr uint64_t kSlotAlign = 4096;
constexpr int kMaxRanks = 8;
constexpr int kMaxHelpers = 8;
constexpr size_t kMaxModels = 4096;

struct PinnedBuf {
    uint8_t* p = nullptr;
    uint64_t bytes = 0;
    uint64_t map_bytes = 0;
    int numa = -1;            // node the arena was bound to (-1: none)
    bool numa_ok = false;     // sampled pages verified resident on that node
};

inline void spin_pause(int& spins) {
    if (++spins < 2048) _mm_pause();
    else std::this_thread::yield();
}

// Barrier of the rank threads of one process. `dead()` is polled while spinning (every 4096
// spins): a peer thread that failed (ctx poisoned) or a wait beyond the bound ends the wait with
// false instead of hanging the process (the caller throws, the worker poisons the ctx).
struct SpinBarrier {
    std::atomic<int> count{0};
    std::atomic<int> gen{0};
    int n = 1;
    template <typename Dead>
    bool wait(Dead dead, double timeout_s = 600.0) {
        if (n <= 1) return true;
        const int g = gen.load(std::memory_order_acquire);
        if (count.fetch_add(1, std::memory_order_acq_rel) + 1 == n) {
            count.store(0, std::memory_order_relaxed);
            gen.fetch_add(1, std::memory_order_acq_rel);
            return true;
        }
        int spins = 0;
        const auto t0 = std::chrono::steady_clock::now();
        while (gen.load(std::memory_order_acquire) == g) {
            spin_pause(spins);
            if ((spins & 4095) == 0 &&
                (dead() || std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s))
                return false;
        }
        return true;
    }
};

// ----------------------------------------------------------------------------- shm control plane
constexpr uint64_t kShmMagic = 0x314d485357534d50ull;  // "PMSWSHM1"
constexpr uint64_t kLogCap = 1 << 16;
constexpr uint64_t kAckCap = 1 << 16;

struct ShmRec {            // one decision published by the leader
    uint64_t id;
    uint64_t off;          // load / offload: byte offset of the model's range
    int32_t kind, model, ring, B, M;
    int32_t writeback;     // offload: copy the range back to the arena (else clean eviction)
    uint64_t stamp;        // batch (debug checks): id of the load it is gated on
};

struct ShmCtl {
    std::atomic<uint64_t> magic;
    int32_t world;
    std::atomic<int32_t> joined;
    std::atomic<int32_t> stop;            // leader has shut down
    std::atomic<int32_t> poisoned;
    char poison_msg[256];
    std::atomic<int32_t> bar_count, bar_gen;
    std::atomic<int32_t> stg_ready;       // leader created the staging segment
    uint64_t stg_bytes;
    std::atomic<uint64_t> log_tail;       // records published
    std::atomic<uint64_t> consumed[kMaxRanks];   // records taken by each follower
    cudaIpcMemHandle_t ws_handle[kMaxRanks];
    uint64_t partial_off[kMaxRanks][2];
    cudaIpcEventHandle_t ev_handle[kMaxRanks][2];
    uint64_t a_off[kMaxRanks];                       // A-operand buffer (reduce-scatter all-gather)
    cudaIpcEventHandle_t ev_ag_handle[kMaxRanks][2];
    ShmRec log[kLogCap];
    std::atomic<uint64_t> ack[kAckCap][kMaxRanks];
};

// ----------------------------------------------------------------------------- entries
struct ReqRec {
    int64_t rid;
    int model;
    std::vector<int32_t> tokens;
    float* out;
    double t_arr = 0, t_done = 0;
    std::atomic<int> done{0};
};

// One-shot forward tap (include/mpsw_testing.h, mpsw_test_tap): copied into the next batch entry.
struct Tap {
    int n_layers = -1, what = 0, rank = 0;
    void* dst = nullptr;
    uint64_t bytes = 0;
};

struct Entry {
    Tap tap;                                     // batch: verification tap (dst == nullptr: none)
    uint64_t expect_stamp = 0;                   // batch (debug checks): id of the load it is gated on
    uint64_t id = 0;
    int kind = 0, model = -1;
    uint64_t off = 0;                            // load / offload: byte offset in the region
    int writeback = 0;                           // offload: D2H writeback (else clean eviction)
    std::vector<std::shared_ptr<ReqRec>> reqs;   // leader only
    int ring = 0, B = 0, M = 0;
    double t_submit = 0;
    cudaEvent_t ev_start[kMaxRanks] = {};        // indexed by GLOBAL rank; only local ranks set
    cudaEvent_t ev_done[kMaxRanks] = {};
    std::atomic<int> issued[kMaxRanks];
    int acked[kMaxRanks] = {};
    double t_ack[kMaxRanks] = {};
    float gpu_ms[kMaxRanks] = {};                // device span per local rank, kept after events die
    cudaEvent_t ev_helper[kMaxRanks][kMaxHelpers] = {};   // fan-in: helper h done with rank r's chunks
    int n_acked = 0;
    std::atomic<int> complete{0};
    Entry() {
        for (auto& a : issued) a.store(0);
    }
};
using EntryP = std::shared_ptr<Entry>;

// ----------------------------------------------------------------------------- per-rank state
// A byte range of the region that a load must not overwrite before `ev` completes: one per D2H
// chunk of a writeback offload (the chunk pairing of reading #5), or one per clean-evicted model
// (its last forward). Kept until a load covers the range or the event is found complete.
struct Gate {
    uint64_t lo, hi;
    cudaEvent_t ev;
    bool chunk;        // a writeback D2H chunk (else: a clean-evicted model's last forward)
};

// NVLink-assisted fan-in (NEXT-2): a helper GPU's own PCIe link pulls chunks of another rank's
// shard into a 2-chunk staging ring in its HBM, then forwards each chunk to the owner's slot with
// a peer copy over NVLink. Helpers are shared by all rank worker threads (mutex).
struct Helper {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint8_t* staging = nullptr;            // 2 * chunk bytes
    cudaEvent_t free_ev[2] = {nullptr, nullptr};
    bool free_valid[2] = {false, false};
    int next = 0;
    std::mutex mu;
};

// CUDA graph of one batch's compute (TP = 1, PP = 1): keyed by the model, its range offset (so the
// weight pointers are the captured ones), the token rows M and the batch size B.
struct GraphKey {
    int model;
    uint64_t off;
    int M, B;
    bool operator<(const GraphKey& o) const {
        return std::tie(model, off, M, B) < std::tie(o.model, o.off, o.M, o.B);
    }
};
struct GraphRec {
    cudaGraphExec_t exec = nullptr;
    bool seen = false;       // the first batch of a key runs eagerly, the second is captured
    int kernels = 0;         // kernels in the graph (launch accounting)
    uint64_t points = 0;     // all-reduce points it advances
};

struct Rank {
    int index = 0, local = 0, device = 0, numa = -1;   // index = global rank = stage * tp + trank
    int stage = 0, trank = 0;              // pipeline stage, TP rank inside the stage
    FwdShape fs_max{};                     // workspace shape: elementwise max over the ctx's models
    cudaEvent_t ev_base = nullptr;         // timeline origin of this rank's device (trace = 1)
    // PP (stage < pp - 1): the residual stream of batch e leaves through hop slot e.ring (the
    // staging-ring index: reused only after batch e completed on every rank, so no WAR fence) and
    // ev_hop[slot] marks it written; the next stage reads it in place (peer memory)
    std::vector<float*> hop;
    std::vector<cudaEvent_t> ev_hop;
    float* hop_base = nullptr;
    // broadcast ablation (cfg.pp_broadcast): host handshake on the batch id instead of forwarding
    cudaEvent_t ev_stage = nullptr;
    std::atomic<uint64_t> stage_out{0};
    cudaStream_t compute = nullptr, h2d = nullptr, d2h = nullptr, aux = nullptr;
    cudaStream_t h2d_zc = nullptr;         // hybrid swap: the zero-copy share of a swap-in
    cudaEvent_t ev_zc = nullptr;
    uint8_t* region = nullptr;             // param budget: cap bytes (one cudaMalloc)
    std::vector<Gate> gates;               // worker-thread private
    uint8_t* ws_base = nullptr;
    FwdWorkspace ws;
    std::vector<TensorPtrs> wptr;          // per model: pointers into its current range
    cudaEvent_t ev_point[2] = {nullptr, nullptr};   // partial-ready events (interprocess in mp mode)
    cudaEvent_t ev_ag[2] = {nullptr, nullptr};      // reduce-scatter: my LN rows written to every rank
    // All-reduce points issued so far by this rank, across batches. Point k uses partial buffer
    // k & 1; the parity must alternate across batch boundaries too (a batch has an odd number of
    // points), or with D > 1 a fast peer's next batch overwrites a partial this rank still reads.
    uint64_t ar_point = 0;
    std::map<GraphKey, GraphRec> graphs;  // worker-thread private
    std::vector<cudaEvent_t> last_compute; // per model
    std::vector<char> last_compute_valid;
    unsigned long long* d_sum = nullptr;
    unsigned long long* d_stamp = nullptr;   // debug checks: per model, id of the load that made it resident
    unsigned int* h_err = nullptr;           // debug checks: mapped pinned error word (set by the device)
    unsigned int* d_err = nullptr;           // its device alias
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<EntryP> fifo;
};

struct Model {
    mpsw_opt_dims dims;
    uint64_t size = 0;             // placement bytes: max over global ranks of round_up(S_r, 4 KiB)
    std::vector<PinnedBuf> arena;  // per LOCAL rank
    std::vector<char> arena_dirty; // per LOCAL rank: handed out for in-place writes, not yet flushed
    std::vector<Layout> layout;    // per LOCAL rank (stage-dependent)
    std::vector<FwdShape> fs;      // per LOCAL rank
    uint64_t rank_S[kMaxRanks] = {};   // arena bytes per GLOBAL rank
};

struct Cmd {
    int kind;  // 0 arrival, 1 swap_in, 2 swap_out
    int model;
    std::shared_ptr<ReqRec> req;
    std::promise<std::pair<mpsw_status, uint64_t>>* reply = nullptr;
};

}  // namespace mpsw

struct mpsw_ctx {
    mpsw_config cfg{};
    std::vector<int> device_ids;
    std::chrono::steady_clock::time_point t0;
    int tp = 1, D = 1;
    int pp = 1, nr = 1;        // pipeline stages; ranks = tp * pp (workers, acks per entry)
    mpsw::SpinBarrier stage_barrier[mpsw::kMaxRanks];   // TP barrier of each stage (single process)
    bool mp = false;           // multi-process mode
    bool leader = true;        // runs the engine (single-process mode: always)
    int world_rank = 0;
    uint64_t chunk = 64ull << 20;
    std::vector<std::unique_ptr<mpsw::Rank>> ranks;     // LOCAL ranks
    std::vector<std::unique_ptr<mpsw::Helper>> helpers; // fan-in helper GPUs (single process)
    int local_of[mpsw::kMaxRanks];                        // global rank -> local index or -1
    std::vector<std::unique_ptr<mpsw::Model>> models;
    // geometry: region of cap bytes per rank; forward workspace sized for dims_max (cfg.max_dims,
    // else the first registered model), fixed at the first registration
    bool geom = false;
    mpsw_opt_dims dims_max{};
    uint64_t cap = 0;
    int max_rows = 0;
    // TP peers (global rank -> partial buffers / partial-ready events)
    float* peer_partial[mpsw::kMaxRanks][2] = {};
    cudaEvent_t peer_ev[mpsw::kMaxRanks][2] = {};
    void* peer_a[mpsw::kMaxRanks] = {};              // every rank's A-operand (LN output) buffer
    cudaEvent_t peer_ev_ag[mpsw::kMaxRanks][2] = {};
    std::vector<void*> ipc_mem_opened;
    std::vector<cudaEvent_t> ipc_ev_opened;
    // logits / tokens staging ring (pinned; shm in mp mode), D + 1 entries
    int ring_n = 2;
    uint8_t* stg = nullptr;
    mpsw::PinnedBuf stg_local;
    size_t stg_map_bytes = 0;
    size_t ring_stride = 0, ring_tok_off = 0;
    // multi-process control plane
    std::string shm_name;
    mpsw::ShmCtl* ctl = nullptr;
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
    std::deque<uint64_t> done_tickets;   // completed swap tickets, oldest first (bounded history)
    std::atomic<int> writeback_now{0};   // writeback of the next offload decisions (mpsw_set_writeback)
    std::atomic<uint64_t> swap_gen{0};   // swap entries dispatched so far (checksum / peek consistency)
    std::unordered_map<int64_t, std::shared_ptr<mpsw::ReqRec>> reqs;
    std::atomic<int64_t> next_rid{0};
    int ring_next = 0;
    std::mutex api_mu;
    // result return (a7) off the engine thread: a completer thread copies each finished batch's
    // logits from the staging ring into the callers' buffers; the ring slot stays busy until then
    std::thread completer;
    std::mutex comp_mu;
    std::condition_variable comp_cv;
    std::deque<mpsw::EntryP> comp_q;
    bool comp_stop = false;
    std::unique_ptr<std::atomic<int>[]> slot_busy;
    std::mutex tap_mu;
    mpsw::Tap tap_next;        // armed by mpsw_test_tap, taken by the next dispatched batch
    std::atomic<int> fault_rank{-1};   // mpsw_test_inject_fault: this rank throws at its next all-reduce point
    std::vector<uint64_t> load_id_of;  // engine: id of the load entry that made each model resident
    // follower-local view of residency (mp followers)
    std::vector<int64_t> f_off_of;
    std::vector<int> f_state;
    std::mutex f_mu;
    // trace + stats
    bool trace = false;
    bool timeline_on = false;   // record device spans (cfg.trace), on every rank / process
    std::mutex trace_mu;
    std::vector<std::string> trace_lines;
    std::vector<std::string> timeline;     // device spans of entries (trace = 1), NDJSON
    std::mutex sm_mu;
    std::unordered_map<int64_t, std::shared_ptr<mpsw::ReqRec>> eng_reqs;   // engine-private
    std::atomic<uint64_t> launches{0}, h2d_bytes{0}, d2h_bytes{0}, swaps_in{0}, swaps_out{0}, n_batches{0},
        n_requests{0}, rejected{0}, fwd_us_sum{0}, fwd_n{0}, prefetches{0};
};

namespace mpsw {

// store.cpp
int gpu_numa_node(int dev);
uint64_t host_mem_available();
PinnedBuf pin_alloc(uint64_t bytes, int numa_node);
void pin_free(PinnedBuf& b);
void parallel_memcpy(uint8_t* dst, const uint8_t* src, uint64_t n);
void flush_to_memory(uint8_t* p, uint64_t n);
void* shm_map(const std::string& name, size_t bytes, bool create);

// engine.cpp
std::string fmt_d(double v);
void poison(mpsw_ctx* c, const std::string& msg);
bool group_poisoned(mpsw_ctx* c);
void group_barrier(mpsw_ctx* c, int stage = 0);
void worker_main(mpsw_ctx* c, Rank* R);
void push_to_rank(Rank& R, const EntryP& e);
void engine_main(mpsw_ctx* c);
void completer_main(mpsw_ctx* c);
void follower_main(mpsw_ctx* c);
void setup_geometry(mpsw_ctx* c, const mpsw_opt_dims& dmax);
void check_dims(mpsw_ctx* c, const mpsw_opt_dims& d);   // kernel limits + fits dims_max (after geometry)
FwdShape fwd_shape(mpsw_ctx* c, const mpsw_opt_dims& d, const Rank& R);

// engine.cpp: device timeline (trace = 1): [t0, t1] of an entry on each local rank, relative to
// the rank's device origin event; called before the entry's events are destroyed
void record_spans(mpsw_ctx* c, Entry& e);

// swap.cpp
bool event_done(cudaEvent_t ev);
bool use_zero_copy(mpsw_ctx* c, uint64_t bytes);
void issue_load(mpsw_ctx* c, Rank& R, Entry& e);
void issue_offload(mpsw_ctx* c, Rank& R, Entry& e);
void finish_swap_events(mpsw_ctx* c, Entry& e);

// batch.cpp
void issue_batch(mpsw_ctx* c, Rank& R, Entry& e);
TensorPtrs make_ptrs(const Layout& L, const uint8_t* base, int layer0, int n_layers);

}  // namespace mpsw
