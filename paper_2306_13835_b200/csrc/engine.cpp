// mpsw runtime: pinned shard store, device slots, per-rank workers, the engine (scheduler)
// thread, the multi-process control plane and the C-ABI entry points.
//
// Architecture (§3.1 Fig. 1, §3.2, §4):
//   * one engine thread = the paper's centralised engine (statemachine.h): per-model FIFO
//     queues, oldest-head batching, LRU replacement via load/offload entries, ack completion;
//   * one worker thread per rank = the paper's per-GPU worker: it receives every entry in the
//     same global order ("evaluate batch entries in submitted order") and issues it on its
//     own streams: compute, load (H2D) and offload (D2H). A worker never waits for a
//     copy before moving on to the next entry (P:105 asynchronous load entries);
//   * an entry completes when every rank has acked; batches for a model are
//     submitted only after its load completed on all ranks (load dependency).
// Deployment modes:
//   * single process: one ctx drives all t ranks (threads), peers' partials read directly;
//   * multi-process (one process per GPU): rank 0 = leader runs the engine and publishes
//     decisions into a POSIX shm ring; followers execute them and post acks into the same
//     segment; the fused TP all-reduce reads peer partials through CUDA IPC mappings.
#include "internal.h"
#include "statemachine.h"

#include <fcntl.h>
#include <immintrin.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
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
constexpr int kMaxHelpers = 8;
constexpr size_t kMaxModels = 4096;

// ----------------------------------------------------------------------------- pinned store
int gpu_numa_node(int dev) {
    char bus[64] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof(bus), dev) != cudaSuccess) return -1;
    for (char* c = bus; *c; ++c) *c = (char)tolower(*c);
    std::ifstream f(std::string("/sys/bus/pci/devices/") + bus + "/numa_node");
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
    b.map_bytes = (std::max<uint64_t>(bytes, 1) + (2ull << 20) - 1) / (2ull << 20) * (2ull << 20);
    void* p = mmap(nullptr, b.map_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p == MAP_FAILED) throw Error(MPSW_ENOMEM, "mmap of pinned arena failed");
    madvise(p, b.map_bytes, MADV_HUGEPAGE);
    if (numa_node >= 0 && numa_node < 64) {
        unsigned long mask = 1ul << numa_node;
        syscall(SYS_mbind, p, b.map_bytes, 2 /*MPOL_BIND*/, &mask, 64, 0);
    }
    cudaError_t e = cudaHostRegister(p, b.map_bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
    if (e != cudaSuccess) {
        cudaGetLastError();
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

inline void spin_pause(int& spins) {
    if (++spins < 2048) _mm_pause();
    else std::this_thread::yield();
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
            while (gen.load(std::memory_order_acquire) == g) spin_pause(spins);
        }
    }
};

// ----------------------------------------------------------------------------- shm control plane
constexpr uint64_t kShmMagic = 0x314d485357534d50ull;  // "PMSWSHM1"
constexpr uint64_t kLogCap = 1 << 16;
constexpr uint64_t kAckCap = 1 << 16;

struct ShmRec {            // one decision published by the leader
    uint64_t id;
    int32_t kind, model, slot, ring, B, M;
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
    ShmRec log[kLogCap];
    std::atomic<uint64_t> ack[kAckCap][kMaxRanks];
};

void* shm_map(const std::string& name, size_t bytes, bool create) {
    int fd = create ? shm_open(name.c_str(), O_CREAT | O_RDWR | O_TRUNC, 0600) : shm_open(name.c_str(), O_RDWR, 0600);
    if (fd < 0) return nullptr;
    if (create && ftruncate(fd, (off_t)bytes) != 0) {
        close(fd);
        throw Error(MPSW_ENOMEM, "ftruncate of shm segment failed");
    }
    if (!create) {
        struct stat st;
        if (fstat(fd, &st) != 0 || (size_t)st.st_size < bytes) {
            close(fd);
            return nullptr;
        }
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw Error(MPSW_ENOMEM, "mmap of shm segment failed");
    return p;
}

// ----------------------------------------------------------------------------- entries
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
struct Slot {
    uint8_t* base = nullptr;
    std::vector<cudaEvent_t> chunk_gate;   // recorded by the last writeback offload, per chunk
    bool chunk_gate_valid = false;
    cudaEvent_t whole_gate = nullptr;      // clean eviction: last forward that read the slot
    bool whole_gate_valid = false;
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

struct Rank {
    int index = 0, local = 0, device = 0, numa = -1;   // index = global rank = stage * tp + trank
    int stage = 0, trank = 0;              // pipeline stage, TP rank inside the stage
    Layout layout;                         // this rank's arena layout (stage-dependent)
    uint64_t S = 0, stride = 0;            // arena bytes, slot stride
    int n_chunks = 0;
    FwdShape fs{};                         // forward shape of this rank (its stage's layers)
    cudaEvent_t ev_stage = nullptr;        // PP: residual stream of this stage is ready
    std::atomic<uint64_t> stage_out{0};    // PP: id+1 of the last batch whose ev_stage is recorded
    cudaStream_t compute = nullptr, h2d = nullptr, d2h = nullptr, aux = nullptr;
    cudaStream_t h2d_zc = nullptr;         // hybrid swap: the zero-copy share of a swap-in
    cudaEvent_t ev_zc = nullptr;
    uint8_t* region = nullptr;             // param budget (one cudaMalloc)
    std::vector<Slot> slots;
    uint8_t* ws_base = nullptr;
    FwdWorkspace ws;
    std::vector<TensorPtrs> wptr;          // per slot
    cudaEvent_t ev_point[2] = {nullptr, nullptr};   // partial-ready events (interprocess in mp mode)
    std::vector<cudaEvent_t> last_compute; // per model
    std::vector<char> last_compute_valid;
    unsigned long long* d_sum = nullptr;
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<EntryP> fifo;
};

struct Model {
    mpsw_opt_dims dims;
    std::vector<PinnedBuf> arena;  // per LOCAL rank
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
    // geometry (fixed by the first registered model; homogeneous slots)
    bool geom = false;
    mpsw_opt_dims dims{};
    int k = 0;
    uint64_t rank_S[mpsw::kMaxRanks] = {};   // arena bytes per global rank
    int vocab = 0;
    int max_rows = 0;
    // TP peers (global rank -> partial buffers / partial-ready events)
    float* peer_partial[mpsw::kMaxRanks][2] = {};
    cudaEvent_t peer_ev[mpsw::kMaxRanks][2] = {};
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
    std::unordered_map<int64_t, std::shared_ptr<mpsw::ReqRec>> reqs;
    std::atomic<int64_t> next_rid{0};
    int ring_next = 0;
    std::mutex api_mu;
    // follower-local view of residency (mp followers)
    std::vector<int> f_slot_of;
    std::vector<int> f_state;
    std::mutex f_mu;
    // trace + stats
    bool trace = false;
    std::mutex trace_mu;
    std::vector<std::string> trace_lines;
    std::mutex sm_mu;
    std::unordered_map<int64_t, std::shared_ptr<mpsw::ReqRec>> eng_reqs;   // engine-private
    std::atomic<uint64_t> launches{0}, h2d_bytes{0}, d2h_bytes{0}, swaps_in{0}, swaps_out{0}, n_batches{0},
        n_requests{0}, rejected{0}, fwd_us_sum{0}, fwd_n{0};
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
    std::fprintf(stderr, "[mpsw] ctx poisoned (rank %d): %s\n", c->world_rank, msg.c_str());
    if (c->ctl && !c->ctl->poisoned.exchange(1))
        std::snprintf(c->ctl->poison_msg, sizeof(c->ctl->poison_msg), "rank %d: %s", c->world_rank, msg.c_str());
    c->done_cv.notify_all();
}

bool group_poisoned(mpsw_ctx* c) { return c->poisoned.load() || (c->ctl && c->ctl->poisoned.load()); }

// Barrier of the t rank threads of a TP group (threads of one process, or one thread in each of
// t processes through the shm segment). Bounded so a dead peer cannot hang the process forever.
void group_barrier(mpsw_ctx* c, int stage = 0) {
    if (!c->mp) {
        c->stage_barrier[stage].wait();
        return;
    }
    ShmCtl* s = c->ctl;
    const int g = s->bar_gen.load(std::memory_order_acquire);
    if (s->bar_count.fetch_add(1, std::memory_order_acq_rel) + 1 == c->tp) {
        s->bar_count.store(0, std::memory_order_relaxed);
        s->bar_gen.fetch_add(1, std::memory_order_acq_rel);
        return;
    }
    int spins = 0;
    const auto t0 = std::chrono::steady_clock::now();
    while (s->bar_gen.load(std::memory_order_acquire) == g) {
        spin_pause(spins);
        if ((spins & 4095) == 0) {
            if (s->poisoned.load()) throw Error(MPSW_ECUDA, std::string("peer poisoned: ") + s->poison_msg);
            if (now_s(t0) > 600) throw Error(MPSW_ETIMEDOUT, "group barrier timed out (peer process gone?)");
        }
    }
}

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

void issue_batch(mpsw_ctx* c, Rank& R, Entry& e) {
    const FwdShape& s = R.fs;
    const int B = e.B, M = e.M;
    const TensorPtrs& Wt = R.wptr[e.slot];
    cudaStream_t cs = R.compute;
    const int r = R.index, t = c->tp;
    const int g0 = R.stage * t;                    // first global rank of my stage
    const bool first = R.stage == 0, last = R.stage == c->pp - 1;
    MPSW_CU(cudaEventCreate(&e.ev_start[r]));
    MPSW_CU(cudaEventCreate(&e.ev_done[r]));
    MPSW_CU(cudaEventRecord(e.ev_start[r], cs));
    // tokens + meta (packed by the engine into the pinned ring entry)
    uint8_t* ring = c->stg + (size_t)e.ring * c->ring_stride;
    const size_t meta_n = (size_t)(3 * B + 1 + 2 * M);
    MPSW_CU(cudaMemcpyAsync(R.ws.tokens, ring + c->ring_tok_off, (size_t)M * 4, cudaMemcpyHostToDevice, cs));
    MPSW_CU(cudaMemcpyAsync(R.ws.meta, ring + c->ring_tok_off + (size_t)c->max_rows * 4, meta_n * 4,
                            cudaMemcpyHostToDevice, cs));
    const int32_t* pos = R.ws.meta + 2 * B + 1;
    int nl = 0, point = 0;
    // all-reduce point: record my partial, barrier with the other TP ranks of my stage, wait for
    // every peer's partial on my stream, then the fused reduce + bias + residual + LN kernel
    // reads all t partials directly (peer / IPC mappings over NVLink).
    auto allreduce_ln = [&](const float* residual, const void* bias, const void* pos_table, const void* g,
                            const void* b) {
        const int pb = point & 1;
        const float* peers[kMaxRanks];
        if (t > 1) {
            MPSW_CU(cudaEventRecord(R.ev_point[pb], cs));
            group_barrier(c, R.stage);
            for (int p = 0; p < t; ++p)
                if (g0 + p != r) MPSW_CU(cudaStreamWaitEvent(cs, c->peer_ev[g0 + p][pb], 0));
        }
        for (int p = 0; p < t; ++p) peers[p] = c->peer_partial[g0 + p][pb];
        nl += fwd_reduce_ln(s, M, peers, t, residual, bias, pos_table, pos, g, b, R.ws.x, R.ws.a, cs);
        ++point;
    };
    if (first) {
        nl += fwd_embed(s, Wt, R.ws, M, R.ws.partial[point & 1], cs);
        allreduce_ln(nullptr, nullptr, Wt.embed_pos, Wt.layers[0].ln1_w, Wt.layers[0].ln1_b);
    } else {
        // PP hop ("PP communication occurs through FIFO pipes"): take the residual stream
        // of the same TP rank of the previous stage (peer copy over NVLink), then LN1 of my
        // first layer. D = 1 for pp > 1, so batches never overlap on a stage boundary.
        Rank& P = *c->ranks[c->local_of[r - t]];
        int spins = 0;
        while (P.stage_out.load(std::memory_order_acquire) < e.id + 1) {
            if (group_poisoned(c)) throw Error(MPSW_ECUDA, "peer failed");
            spin_pause(spins);
        }
        MPSW_CU(cudaStreamWaitEvent(cs, P.ev_stage, 0));
        MPSW_CU(cudaMemcpyAsync(R.ws.partial[0], P.ws.x, (size_t)M * s.hidden * 4, cudaMemcpyDeviceToDevice, cs));
        const float* self[1] = {R.ws.partial[0]};
        nl += fwd_reduce_ln(s, M, self, 1, nullptr, nullptr, nullptr, pos, Wt.layers[0].ln1_w, Wt.layers[0].ln1_b,
                            R.ws.x, R.ws.a, cs);
        point = 1;
    }
    for (int l = 0; l < s.n_layers; ++l) {
        const auto& L = Wt.layers[l];
        nl += fwd_qkv(s, L, R.ws, M, cs);
        nl += fwd_attention(s, R.ws, B, cs);
        nl += fwd_out_proj(s, L, R.ws, M, R.ws.partial[point & 1], cs);
        allreduce_ln(R.ws.x, L.o_b, nullptr, L.ln2_w, L.ln2_b);
        nl += fwd_fc1(s, L, R.ws, M, cs);
        nl += fwd_fc2(s, L, R.ws, M, R.ws.partial[point & 1], cs);
        const bool lastl = l + 1 == s.n_layers;
        // after a non-final stage's last layer only the residual stream matters; the LN output
        // (computed with this layer's LN2 parameters) is unused
        const void* ng = lastl ? (last ? Wt.lnf_w : L.ln2_w) : Wt.layers[l + 1].ln1_w;
        const void* nb = lastl ? (last ? Wt.lnf_b : L.ln2_b) : Wt.layers[l + 1].ln1_b;
        allreduce_ln(R.ws.x, L.fc2_b, nullptr, ng, nb);
    }
    if (last) {
        nl += fwd_lm_head(s, Wt, R.ws, B, M, cs);
        float* logits_host = (float*)(ring) + (size_t)R.trank * s.vocab_local;
        MPSW_CU(cudaMemcpy2DAsync(logits_host, (size_t)s.vocab * 4, R.ws.logits, (size_t)s.vocab_local * 4,
                                  (size_t)s.vocab_local * 4, B, cudaMemcpyDeviceToHost, cs));
    } else {
        MPSW_CU(cudaEventRecord(R.ev_stage, cs));
        R.stage_out.store(e.id + 1, std::memory_order_release);
    }
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
            if (!group_poisoned(c)) {
                if (e->kind == E_LOAD) issue_load(c, *R, *e);
                else if (e->kind == E_OFFLOAD) issue_offload(c, *R, *e);
                else issue_batch(c, *R, *e);
            }
        } catch (const std::exception& err) {
            poison(c, err.what());
        }
        e->issued[R->index].store(1, std::memory_order_release);
        c->cmd_cv.notify_all();
    }
}

void push_to_workers(mpsw_ctx* c, const EntryP& e) {
    for (auto& R : c->ranks) {
        std::lock_guard<std::mutex> lk(R->mu);
        R->fifo.push_back(e);
        R->cv.notify_one();
    }
}

// ----------------------------------------------------------------------------- engine (leader)
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

void publish(mpsw_ctx* c, const Entry& e) {
    ShmCtl* s = c->ctl;
    const uint64_t tail = s->log_tail.load(std::memory_order_relaxed);
    // never overwrite a record a follower has not taken yet
    int spins = 0;
    for (int p = 1; p < c->nr; ++p)
        while (tail - s->consumed[p].load(std::memory_order_acquire) >= kLogCap) spin_pause(spins);
    ShmRec& rec = s->log[tail % kLogCap];
    rec.id = e.id;
    rec.kind = e.kind;
    rec.model = e.model;
    rec.slot = e.slot;
    rec.ring = e.ring;
    rec.B = e.B;
    rec.M = e.M;
    s->log_tail.store(tail + 1, std::memory_order_release);
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
            // pack tokens + meta into the pinned ring entry (shm in mp mode: every rank reads it)
            e->ring = c->ring_next;
            c->ring_next = (c->ring_next + 1) % c->ring_n;
            uint8_t* ring = c->stg + (size_t)e->ring * c->ring_stride;
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
            int32_t* row_of_m = meta + 2 * B + 1 + M;      // lm_head: token row -> request (or -1)
            for (int m = 0; m < M; ++m) row_of_m[m] = -1;
            for (int b = 0; b < B; ++b) row_of_m[meta[B + 1 + b]] = b;
            e->B = B;
            e->M = M;
        } else {
            std::lock_guard<std::mutex> lk(c->done_mu);
            c->entries[e->id] = e;
        }
        if (c->mp) publish(c, *e);
        c->inflight.push_back(e);
        push_to_workers(c, e);
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
    const uint8_t* ring = c->stg + (size_t)e.ring * c->ring_stride;
    const int V = c->vocab;
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

// Device span of a finished swap entry on every local rank; then its events are released (a
// long run would otherwise keep 2 events per rank per swap).
void finish_swap_events(mpsw_ctx* c, Entry& e) {
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

// Device time of a finished batch's forward on the first local rank (stats), then free its events.
void record_fwd_time(mpsw_ctx* c, Entry& e) {
    const int r0 = c->ranks[0]->index;
    float ms = 0;
    if (e.ev_start[r0] && e.ev_done[r0] && cudaEventElapsedTime(&ms, e.ev_start[r0], e.ev_done[r0]) == cudaSuccess) {
        c->fwd_us_sum += (uint64_t)(ms * 1000.0f);
        c->fwd_n++;
    }
    cudaGetLastError();
    for (int r = 0; r < c->nr; ++r) {
        if (e.ev_start[r]) cudaEventDestroy(e.ev_start[r]), e.ev_start[r] = nullptr;
        if (e.ev_done[r]) cudaEventDestroy(e.ev_done[r]), e.ev_done[r] = nullptr;
    }
}

// 1 = rank r finished entry e, 0 = not yet. Local ranks: their CUDA event; remote ranks (mp):
// the ack slot the follower wrote into the shm segment.
int rank_done(mpsw_ctx* c, Entry& e, int r) {
    if (c->local_of[r] >= 0) {
        if (!e.issued[r].load(std::memory_order_acquire)) return 0;
        if (!e.ev_done[r]) return 1;   // poisoned before issue
        const cudaError_t q = cudaEventQuery(e.ev_done[r]);
        if (q == cudaErrorNotReady) return 0;
        if (q != cudaSuccess) throw Error(MPSW_ECUDA, std::string("copy/forward failed: ") + cudaGetErrorString(q));
        return 1;
    }
    return c->ctl->ack[e.id % kAckCap][r].load(std::memory_order_acquire) == e.id + 1 ? 1 : 0;
}

bool poll_inflight(mpsw_ctx* c) {
    bool progressed = false;
    for (size_t i = 0; i < c->inflight.size();) {
        Entry& e = *c->inflight[i];
        bool finished = false;
        for (int r = 0; r < c->nr; ++r) {
            if (e.acked[r] || !rank_done(c, e, r)) continue;
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
                if (e.kind == E_LOAD) c->h2d_bytes += c->rank_S[r];
                else if (c->cfg.writeback) c->d2h_bytes += c->rank_S[r];
            }
        }
        if (e.n_acked == c->nr) {
            const double now = now_s(c->t0);
            if (e.kind == E_BATCH) {
                complete_batch(c, e, now);
                log_event(c, "{\"ev\":\"batch_done\",\"t\":" + fmt_d(now) + ",\"batch\":" + std::to_string(e.id) + "}");
                step_and_dispatch(c, [&](std::vector<Decision>& ds) { c->sm.batch_done(e.id, now, ds); }, now);
                record_fwd_time(c, e);
            } else {
                (e.kind == E_LOAD ? c->swaps_in : c->swaps_out)++;
                finish_swap_events(c, e);
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
                if (group_poisoned(c)) {
                    if (cmd.reply) cmd.reply->set_value({MPSW_ECUDA, 0});
                    continue;
                }
                if (cmd.kind == 0) {
                    auto& rq = cmd.req;
                    c->eng_reqs[rq->rid] = rq;
                    log_event(c, "{\"ev\":\"arrival\",\"t\":" + fmt_d(rq->t_arr) + ",\"rid\":" + std::to_string(rq->rid) +
                                     ",\"model\":" + std::to_string(rq->model) + "}");
                    const double t = rq->t_arr;
                    step_and_dispatch(c, [&](std::vector<Decision>& ds) { c->sm.arrival(rq->rid, rq->model, t, ds); },
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
                if (c->ctl && c->ctl->poisoned.load() && !c->poisoned.load())
                    poison(c, std::string("peer: ") + c->ctl->poison_msg);
            }
        } catch (const std::exception& err) {
            poison(c, err.what());
            for (auto& cmd : batch)
                if (cmd.reply) try { cmd.reply->set_value({MPSW_EINVARIANT, 0}); } catch (...) {}
            c->inflight.clear();
        }
    }
}

// ----------------------------------------------------------------------------- follower (mp)
// Takes the leader's published entries in order, hands them to the local worker, and posts
// this rank's acks (swap copy or batch forward finished on this GPU) into the shm segment.
void follower_main(mpsw_ctx* c) {
    Rank& R = *c->ranks[0];
    cudaSetDevice(R.device);
    ShmCtl* s = c->ctl;
    uint64_t cur = 0;
    int spins = 0;
    while (true) {
        bool progressed = false;
        const uint64_t tail = s->log_tail.load(std::memory_order_acquire);
        while (cur < tail) {
            const ShmRec rec = s->log[cur % kLogCap];
            ++cur;
            s->consumed[c->world_rank].store(cur, std::memory_order_release);
            auto e = std::make_shared<Entry>();
            e->id = rec.id;
            e->kind = rec.kind;
            e->model = rec.model;
            e->slot = rec.slot;
            e->ring = rec.ring;
            e->B = rec.B;
            e->M = rec.M;
            e->t_submit = now_s(c->t0);
            if (e->kind != E_BATCH) {
                std::lock_guard<std::mutex> lk(c->done_mu);
                c->entries[e->id] = e;
            }
            {
                std::lock_guard<std::mutex> lk(c->f_mu);
                if (e->kind == E_LOAD) { c->f_slot_of[e->model] = e->slot; c->f_state[e->model] = ST_LOADING; }
                if (e->kind == E_OFFLOAD) { c->f_slot_of[e->model] = -1; c->f_state[e->model] = ST_OFFLOADING; }
            }
            c->inflight.push_back(e);
            push_to_workers(c, e);
            progressed = true;
        }
        try {
            const int r = R.index;
            for (size_t i = 0; i < c->inflight.size();) {
                Entry& e = *c->inflight[i];
                if (!rank_done(c, e, r)) { ++i; continue; }
                e.acked[r] = 1;
                e.t_ack[r] = now_s(c->t0);
                e.n_acked = 1;
                s->ack[e.id % kAckCap][r].store(e.id + 1, std::memory_order_release);
                {
                    std::lock_guard<std::mutex> lk(c->f_mu);
                    if (e.kind == E_LOAD && c->f_slot_of[e.model] == e.slot) c->f_state[e.model] = ST_RESIDENT;
                    if (e.kind == E_OFFLOAD && c->f_state[e.model] == ST_OFFLOADING) c->f_state[e.model] = ST_EVICTED;
                }
                if (e.kind == E_BATCH) {
                    record_fwd_time(c, e);
                    c->n_batches++;
                } else {
                    (e.kind == E_LOAD ? c->swaps_in : c->swaps_out)++;
                    if (e.kind == E_LOAD) c->h2d_bytes += R.S;
                    else if (c->cfg.writeback) c->d2h_bytes += R.S;
                    finish_swap_events(c, e);
                    std::lock_guard<std::mutex> lk(c->done_mu);
                    e.complete.store(1, std::memory_order_release);
                }
                c->done_cv.notify_all();
                c->inflight.erase(c->inflight.begin() + i);
                progressed = true;
            }
        } catch (const std::exception& err) {
            poison(c, err.what());
            c->inflight.clear();
        }
        if (c->inflight.empty() && cur == s->log_tail.load(std::memory_order_acquire) &&
            (s->stop.load(std::memory_order_acquire) || (c->stop.load() && group_poisoned(c))))
            break;
        if (progressed) spins = 0;
        else if (c->inflight.empty()) {
            if (++spins > 4096) std::this_thread::sleep_for(std::chrono::microseconds(50));
        } else {
            spin_pause(spins);
        }
    }
}

// Weight pointers of one rank's slot, looked up by HF name in that rank's layout (stage-local
// layers only; embeddings / final LN only where the stage holds them).
TensorPtrs make_ptrs(const Layout& L, const uint8_t* base, int layer0, int n_layers) {
    std::unordered_map<std::string, const void*> by;
    for (const auto& t : L.t) by[t.name] = base + t.offset;
    auto p = [&](const std::string& n) -> const void* {
        auto it = by.find(n);
        return it == by.end() ? nullptr : it->second;
    };
    TensorPtrs w;
    w.embed_tok = p("decoder.embed_tokens.weight");
    w.embed_pos = p("decoder.embed_positions.weight");
    w.lnf_w = p("decoder.final_layer_norm.weight");
    w.lnf_b = p("decoder.final_layer_norm.bias");
    for (int l = layer0; l < layer0 + n_layers; ++l) {
        const std::string q = "decoder.layers." + std::to_string(l) + ".";
        TensorPtrs::Layer x;
        x.k_w = p(q + "self_attn.k_proj.weight"); x.k_b = p(q + "self_attn.k_proj.bias");
        x.v_w = p(q + "self_attn.v_proj.weight"); x.v_b = p(q + "self_attn.v_proj.bias");
        x.q_w = p(q + "self_attn.q_proj.weight"); x.q_b = p(q + "self_attn.q_proj.bias");
        x.o_w = p(q + "self_attn.out_proj.weight"); x.o_b = p(q + "self_attn.out_proj.bias");
        x.ln1_w = p(q + "self_attn_layer_norm.weight"); x.ln1_b = p(q + "self_attn_layer_norm.bias");
        x.fc1_w = p(q + "fc1.weight"); x.fc1_b = p(q + "fc1.bias");
        x.fc2_w = p(q + "fc2.weight"); x.fc2_b = p(q + "fc2.bias");
        x.ln2_w = p(q + "final_layer_norm.weight"); x.ln2_b = p(q + "final_layer_norm.bias");
        w.layers.push_back(x);
    }
    return w;
}

// Fix the slot geometry at the first registration: k = floor(budget / S_r) slots per rank
// carved from the region allocated at init; workspaces sized for max_batch * max_tokens rows;
// TP peers wired (collective in multi-process mode: IPC handles exchanged through shm).
void setup_geometry(mpsw_ctx* c, const mpsw_opt_dims& d) {
    const int hd = d.hidden / d.heads;
    if (hd % 8 || hd > 128) throw Error(MPSW_EINVAL, "head_dim must be a multiple of 8 and <= 128");
    if ((d.hidden / c->tp) % 8 || (d.ffn / c->tp) % 8 || d.hidden % 8)
        throw Error(MPSW_EINVAL, "hidden/tp, ffn/tp and hidden must be multiples of 8");
    if (d.hidden > 12288) throw Error(MPSW_EINVAL, "hidden too large for the LN kernel");
    // every global rank's arena size (stage-dependent) and the slot count k, the same on all
    // ranks (a model occupies one slot on every worker): k = min_r floor(budget / stride_r)
    int k = 1024;
    for (int g = 0; g < c->nr; ++g) {
        Layout L;
        if (compute_layout(d, c->tp, c->pp, g / c->tp, g % c->tp, c->cfg.dtype, L) != MPSW_OK)
            throw Error(MPSW_EINVAL, tls_error());
        c->rank_S[g] = L.bytes;
        const uint64_t stride = (L.bytes + kSlotAlign - 1) / kSlotAlign * kSlotAlign;
        k = (int)std::min<uint64_t>((uint64_t)k, c->cfg.param_budget_bytes_per_gpu / stride);
    }
    if (k < 1)
        throw Error(MPSW_ENOMEM, "param budget cannot hold one shard (S_r = " + std::to_string(c->rank_S[0]) + ")");
    c->dims = d;
    c->vocab = d.vocab;
    c->k = k;
    c->max_rows = c->cfg.max_batch * c->cfg.max_tokens;
    const unsigned ev_flags = c->mp ? (cudaEventInterprocess | cudaEventDisableTiming) : cudaEventDisableTiming;
    for (auto& Rp : c->ranks) {
        Rank& R = *Rp;
        MPSW_CU(cudaSetDevice(R.device));
        if (compute_layout(d, c->tp, c->pp, R.stage, R.trank, c->cfg.dtype, R.layout) != MPSW_OK)
            throw Error(MPSW_EINVAL, tls_error());
        R.S = R.layout.bytes;
        R.stride = (R.S + kSlotAlign - 1) / kSlotAlign * kSlotAlign;
        R.n_chunks = (int)((R.S + c->chunk - 1) / c->chunk);
        FwdShape& f = R.fs;
        f.n_layers = d.n_layers / c->pp; f.hidden = d.hidden; f.heads_local = d.heads / c->tp; f.head_dim = hd;
        f.ffn_local = d.ffn / c->tp; f.vocab_local = d.vocab / c->tp; f.vocab = d.vocab; f.tp = c->tp;
        f.rank = R.trank;
        f.dtype = c->cfg.dtype;
        f.gemm_impl = c->cfg.gemm_impl;
        f.max_rows = c->max_rows;
        const size_t wsb = workspace_bytes(f, c->max_rows, c->cfg.max_batch);
        R.slots.resize(k);
        for (int s = 0; s < k; ++s) {
            Slot& sl = R.slots[s];
            sl.base = R.region + (uint64_t)s * R.stride;
            sl.chunk_gate.resize(R.n_chunks);
            for (auto& ev : sl.chunk_gate) MPSW_CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            MPSW_CU(cudaEventCreateWithFlags(&sl.whole_gate, cudaEventDisableTiming));
            R.wptr.push_back(make_ptrs(R.layout, sl.base, R.stage * f.n_layers, f.n_layers));
        }
        MPSW_CU(cudaMalloc(&R.ws_base, wsb));
        MPSW_CU(cudaMemset(R.ws_base, 0, wsb));
        workspace_carve(R.ws, f, c->max_rows, c->cfg.max_batch, R.ws_base);
        for (auto& ev : R.ev_point) MPSW_CU(cudaEventCreateWithFlags(&ev, ev_flags));
        MPSW_CU(cudaEventCreateWithFlags(&R.ev_stage, cudaEventDisableTiming));
        for (int pb = 0; pb < 2; ++pb) {
            c->peer_partial[R.index][pb] = R.ws.partial[pb];
            c->peer_ev[R.index][pb] = R.ev_point[pb];
        }
    }
    // staging ring: per entry [max_batch * V] fp32 logits, then tokens [max_rows] + meta
    c->ring_n = c->D + 1;
    const size_t logits_b = ((size_t)c->cfg.max_batch * d.vocab * 4 + 255) & ~size_t(255);
    c->ring_tok_off = logits_b;
    c->ring_stride = (logits_b + (size_t)(c->max_rows * 3 + 3 * c->cfg.max_batch + 8) * 4 + 4095) & ~size_t(4095);
    const size_t stg_bytes = c->ring_stride * c->ring_n;
    if (!c->mp) {
        c->stg_local = pin_alloc(stg_bytes, c->ranks[0]->numa);
        c->stg = c->stg_local.p;
    } else {
        ShmCtl* s = c->ctl;
        Rank& R = *c->ranks[0];
        MPSW_CU(cudaSetDevice(R.device));
        MPSW_CU(cudaIpcGetMemHandle(&s->ws_handle[R.index], R.ws_base));
        for (int pb = 0; pb < 2; ++pb) {
            s->partial_off[R.index][pb] = (uint64_t)((uint8_t*)R.ws.partial[pb] - R.ws_base);
            MPSW_CU(cudaIpcGetEventHandle(&s->ev_handle[R.index][pb], R.ev_point[pb]));
        }
        const std::string stg_name = c->shm_name + "_stg";
        if (c->leader) {
            c->stg = (uint8_t*)shm_map(stg_name, stg_bytes, true);
            s->stg_bytes = stg_bytes;
            s->stg_ready.store(1, std::memory_order_release);
        }
        group_barrier(c);   // every rank published its handles; staging segment exists
        if (!c->leader) {
            if (s->stg_bytes != stg_bytes) throw Error(MPSW_EINVAL, "ranks disagree on the staging geometry");
            c->stg = (uint8_t*)shm_map(stg_name, stg_bytes, false);
            if (!c->stg) throw Error(MPSW_EINVAL, "cannot open the staging segment");
        }
        c->stg_map_bytes = stg_bytes;
        MPSW_CU(cudaHostRegister(c->stg, stg_bytes, cudaHostRegisterPortable));
        for (int p = 0; p < c->tp; ++p) {
            if (p == R.index) continue;
            void* base = nullptr;
            MPSW_CU(cudaIpcOpenMemHandle(&base, s->ws_handle[p], cudaIpcMemLazyEnablePeerAccess));
            c->ipc_mem_opened.push_back(base);
            for (int pb = 0; pb < 2; ++pb) {
                c->peer_partial[p][pb] = (float*)((uint8_t*)base + s->partial_off[p][pb]);
                cudaEvent_t ev;
                MPSW_CU(cudaIpcOpenEventHandle(&ev, s->ev_handle[p][pb]));
                c->ipc_ev_opened.push_back(ev);
                c->peer_ev[p][pb] = ev;
            }
        }
        group_barrier(c);
        if (c->leader) shm_unlink(stg_name.c_str());   // mapped everywhere; name no longer needed
    }
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

static mpsw_status need_leader(mpsw_ctx* c) {
    if (!c->leader) return set_error(MPSW_EINVAL, "multi-process mode: submit on rank 0 (the engine)");
    return MPSW_OK;
}

static int local_index(mpsw_ctx* c, int rank) {
    if (rank < 0 || rank >= c->nr) return -1;
    return c->local_of[rank];
}

extern "C" {

const char* mpsw_last_error(void) { return tls_error().c_str(); }

mpsw_status mpsw_shard_layout(const mpsw_opt_dims* dims, int tp, int pp, int stage, int rank, int dtype,
                              mpsw_tensor_desc* out, int cap, int* n, uint64_t* shard_bytes) {
    API_BEGIN
    if (!dims) return set_error(MPSW_EINVAL, "dims is NULL");
    Layout L;
    mpsw_status s = compute_layout(*dims, tp, pp, stage, rank, dtype, L);
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
    const bool mp = cfg->world_size > 1;
    const int pp = cfg->pp > 0 ? cfg->pp : 1;
    if (cfg->n_gpus < 1 || cfg->n_gpus > kMaxRanks || !cfg->device_ids)
        return set_error(MPSW_EINVAL, "n_gpus must be 1..8 with device_ids");
    if (mp) {
        if (cfg->world_size > kMaxRanks) return set_error(MPSW_EINVAL, "world_size must be <= 8");
        if (cfg->n_gpus != 1 || cfg->tp != cfg->world_size)
            return set_error(MPSW_EINVAL, "multi-process mode: n_gpus = 1 and tp = world_size");
        if (pp != 1) return set_error(MPSW_EINVAL, "pipeline parallelism is single-process only");
        if (cfg->world_rank < 0 || cfg->world_rank >= cfg->world_size) return set_error(MPSW_EINVAL, "bad world_rank");
        if (!cfg->shm_name || cfg->shm_name[0] != '/') return set_error(MPSW_EINVAL, "shm_name must start with '/'");
    } else if (cfg->tp < 1 || cfg->tp * pp != cfg->n_gpus) {
        return set_error(MPSW_EINVAL, "tp * pp must equal n_gpus (one TP x PP group per ctx)");
    }
    if (pp > 1 && cfg->max_inflight_batches > 1)
        return set_error(MPSW_EINVAL, "pp > 1 requires max_inflight_batches = 1");
    if (cfg->max_batch < 1 || cfg->max_batch > 256) return set_error(MPSW_EINVAL, "max_batch must be 1..256");
    if (cfg->max_tokens < 1 || cfg->max_tokens > 128) return set_error(MPSW_EINVAL, "max_tokens must be 1..128");
    if (cfg->dtype != MPSW_BF16 && cfg->dtype != MPSW_FP32) return set_error(MPSW_EINVAL, "bad dtype");
    if (cfg->chunk_bytes % 4096) return set_error(MPSW_EINVAL, "chunk_bytes must be a multiple of 4096");
    if (cfg->swap_mode < 0 || cfg->swap_mode > 3) return set_error(MPSW_EINVAL, "bad swap_mode");
    if (cfg->param_budget_bytes_per_gpu == 0) return set_error(MPSW_EINVAL, "param budget is 0");
    if (cfg->gemm_impl < 0 || cfg->gemm_impl > 2) return set_error(MPSW_EINVAL, "bad gemm_impl");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        return set_error(MPSW_ECUDA, "no CUDA device");
    }
    auto c = std::make_unique<mpsw_ctx>();
    c->cfg = *cfg;
    c->cfg.shm_name = nullptr;
    c->t0 = std::chrono::steady_clock::now();
    c->mp = mp;
    c->world_rank = mp ? cfg->world_rank : 0;
    c->leader = !mp || cfg->world_rank == 0;
    c->tp = cfg->tp;
    c->pp = pp;
    c->nr = mp ? cfg->world_size : cfg->n_gpus;
    c->D = cfg->max_inflight_batches > 0 ? cfg->max_inflight_batches : 1;
    c->chunk = cfg->chunk_bytes ? cfg->chunk_bytes : (64ull << 20);
    c->trace = cfg->trace != 0 && c->leader;
    c->device_ids.assign(cfg->device_ids, cfg->device_ids + cfg->n_gpus);
    c->sm.tp = c->nr;              // acks per entry: one per worker
    c->sm.max_batch = cfg->max_batch;
    c->sm.D = c->D;
    for (auto& b : c->stage_barrier) b.n = mp ? 1 : c->tp;
    c->models.reserve(kMaxModels);
    for (auto& x : c->local_of) x = -1;
    for (int l = 0; l < cfg->n_gpus; ++l) {
        const int dev = c->device_ids[l];
        if (dev < 0 || dev >= ndev) return set_error(MPSW_EINVAL, "device id out of range");
        auto R = std::make_unique<Rank>();
        R->index = mp ? cfg->world_rank : l;
        R->stage = R->index / cfg->tp;
        R->trank = R->index % cfg->tp;
        R->local = l;
        R->device = dev;
        R->numa = gpu_numa_node(dev);
        R->last_compute.reserve(kMaxModels);
        R->last_compute_valid.reserve(kMaxModels);
        c->local_of[R->index] = l;
        MPSW_CU(cudaSetDevice(dev));
        int hp = 0, lp = 0;
        MPSW_CU(cudaDeviceGetStreamPriorityRange(&lp, &hp));
        MPSW_CU(cudaStreamCreateWithPriority(&R->compute, cudaStreamNonBlocking, hp));
        MPSW_CU(cudaStreamCreateWithFlags(&R->h2d, cudaStreamNonBlocking));
        MPSW_CU(cudaStreamCreateWithFlags(&R->d2h, cudaStreamNonBlocking));
        MPSW_CU(cudaStreamCreateWithFlags(&R->aux, cudaStreamNonBlocking));
        MPSW_CU(cudaStreamCreateWithFlags(&R->h2d_zc, cudaStreamNonBlocking));
        MPSW_CU(cudaEventCreateWithFlags(&R->ev_zc, cudaEventDisableTiming));
        cudaError_t e = cudaMalloc(&R->region, cfg->param_budget_bytes_per_gpu);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return set_error(MPSW_ENOMEM, std::string("cudaMalloc(param budget): ") + cudaGetErrorString(e));
        }
        MPSW_CU(cudaMalloc(&R->d_sum, sizeof(unsigned long long)));
        c->ranks.push_back(std::move(R));
    }
    if (cfg->n_helpers < 0 || cfg->n_helpers > kMaxHelpers || (cfg->n_helpers && !cfg->helper_device_ids))
        return set_error(MPSW_EINVAL, "n_helpers must be 0..8 with helper_device_ids");
    if (mp && cfg->n_helpers) return set_error(MPSW_EINVAL, "fan-in helpers are single-process only");
    for (int h = 0; h < cfg->n_helpers; ++h) {
        const int dev = cfg->helper_device_ids[h];
        if (dev < 0 || dev >= ndev) return set_error(MPSW_EINVAL, "helper device id out of range");
        auto H = std::make_unique<Helper>();
        H->device = dev;
        MPSW_CU(cudaSetDevice(dev));
        MPSW_CU(cudaStreamCreateWithFlags(&H->stream, cudaStreamNonBlocking));
        cudaError_t e = cudaMalloc(&H->staging, 2 * c->chunk);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return set_error(MPSW_ENOMEM, "cudaMalloc(fan-in staging)");
        }
        for (auto& ev : H->free_ev) MPSW_CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        for (int r = 0; r < c->nr; ++r) {      // helper <-> owner peer access (NVLink)
            const int od = c->device_ids[r];
            if (od == dev) continue;
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, dev, od);
            if (!ok) return set_error(MPSW_EINVAL, "helper GPU lacks peer access to a rank's GPU");
            cudaError_t pe = cudaDeviceEnablePeerAccess(od, 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) MPSW_CU(pe);
            cudaGetLastError();
        }
        c->helpers.push_back(std::move(H));
    }
    if (!mp) {
        // peer access between distinct devices of the group (TP all-reduce reads peer partials)
        for (int a = 0; a < c->nr; ++a)
            for (int b = 0; b < c->nr; ++b) {
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
    } else {
        // shm control plane: the leader creates and initialises it; followers attach.
        c->shm_name = cfg->shm_name;
        ShmCtl* s = nullptr;
        if (c->leader) {
            s = (ShmCtl*)shm_map(c->shm_name, sizeof(ShmCtl), true);
            if (!s) return set_error(MPSW_EINVAL, "cannot create shm segment " + c->shm_name);
            std::memset((void*)s, 0, sizeof(ShmCtl));
            s->world = c->tp;
            s->magic.store(kShmMagic, std::memory_order_release);
        } else {
            const auto t0 = std::chrono::steady_clock::now();
            while (true) {
                s = (ShmCtl*)shm_map(c->shm_name, sizeof(ShmCtl), false);
                if (s && s->magic.load(std::memory_order_acquire) == kShmMagic) break;
                if (s) munmap((void*)s, sizeof(ShmCtl)), s = nullptr;
                if (now_s(t0) > 120) return set_error(MPSW_ETIMEDOUT, "leader never created " + c->shm_name);
                std::this_thread::sleep_for(std::chrono::milliseconds(20));
            }
            if (s->world != c->tp) return set_error(MPSW_EINVAL, "world_size differs from the leader's");
        }
        c->ctl = s;
        s->joined.fetch_add(1);
        const auto t0 = std::chrono::steady_clock::now();
        while (s->joined.load() < c->tp) {
            if (now_s(t0) > 120) return set_error(MPSW_ETIMEDOUT, "peers did not join the control plane");
            std::this_thread::sleep_for(std::chrono::milliseconds(5));
        }
    }
    mpsw_ctx* raw = c.release();
    for (auto& R : raw->ranks) R->th = std::thread(worker_main, raw, R.get());
    raw->engine = std::thread(raw->leader ? engine_main : follower_main, raw);
    *out = raw;
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_shutdown(mpsw_ctx* c) {
    if (!c) return MPSW_OK;
    if (c->mp && !c->leader) {
        // a follower serves the leader's entries until the leader shuts down
        const auto t0 = std::chrono::steady_clock::now();
        while (!c->ctl->stop.load() && !group_poisoned(c) && now_s(t0) < 3600)
            std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
    {
        std::lock_guard<std::mutex> lk(c->cmd_mu);
        c->stop.store(true);
    }
    c->cmd_cv.notify_all();
    if (c->engine.joinable()) c->engine.join();
    if (c->mp && c->leader) c->ctl->stop.store(1, std::memory_order_release);
    for (auto& R : c->ranks) {
        { std::lock_guard<std::mutex> lk(R->mu); }
        R->cv.notify_all();
        if (R->th.joinable()) R->th.join();
    }
    for (auto& R : c->ranks) {
        cudaSetDevice(R->device);
        cudaDeviceSynchronize();
    }
    for (auto& H : c->helpers) {
        cudaSetDevice(H->device);
        cudaStreamSynchronize(H->stream);
        cudaStreamDestroy(H->stream);
        cudaFree(H->staging);
        for (auto ev : H->free_ev) cudaEventDestroy(ev);
    }
    for (auto p : c->ipc_mem_opened) cudaIpcCloseMemHandle(p);
    for (auto ev : c->ipc_ev_opened) cudaEventDestroy(ev);
    for (auto& R : c->ranks) {
        cudaSetDevice(R->device);
        for (auto& sl : R->slots) {
            for (auto ev : sl.chunk_gate) cudaEventDestroy(ev);
            if (sl.whole_gate) cudaEventDestroy(sl.whole_gate);
        }
        for (auto ev : R->ev_point)
            if (ev) cudaEventDestroy(ev);
        if (R->ev_stage) cudaEventDestroy(R->ev_stage);
        for (auto ev : R->last_compute)
            if (ev) cudaEventDestroy(ev);
        cudaFree(R->region);
        cudaFree(R->ws_base);
        cudaFree(R->d_sum);
        cudaStreamDestroy(R->compute);
        cudaStreamDestroy(R->h2d);
        cudaStreamDestroy(R->d2h);
        cudaStreamDestroy(R->aux);
        cudaStreamDestroy(R->h2d_zc);
        cudaEventDestroy(R->ev_zc);
    }
    for (auto& kv : c->entries)
        for (int r = 0; r < c->nr; ++r) {
            if (kv.second->ev_start[r]) cudaEventDestroy(kv.second->ev_start[r]);
            if (kv.second->ev_done[r]) cudaEventDestroy(kv.second->ev_done[r]);
        }
    for (auto& m : c->models)
        for (auto& a : m->arena) pin_free(a);
    pin_free(c->stg_local);
    if (c->mp) {
        if (c->stg) {
            cudaHostUnregister(c->stg);
            munmap(c->stg, c->stg_map_bytes);
        }
        if (c->ctl) {
            munmap((void*)c->ctl, sizeof(ShmCtl));
            if (c->leader) shm_unlink(c->shm_name.c_str());
        }
    }
    delete c;
    return MPSW_OK;
}

mpsw_status mpsw_register_model(mpsw_ctx* c, const mpsw_opt_dims* dims, int tp, const void* const* shards,
                                const uint64_t* shard_bytes, int* model_id) {
    API_BEGIN
    if (!c || !dims || !model_id) return set_error(MPSW_EINVAL, "NULL argument");
    if (group_poisoned(c)) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
    if (tp != c->tp) return set_error(MPSW_EINVAL, "model tp must equal the ctx tp");
    std::lock_guard<std::mutex> api(c->api_mu);
    Layout L;
    mpsw_status s = compute_layout(*dims, tp, c->pp, 0, 0, c->cfg.dtype, L);
    if (s != MPSW_OK) return s;
    {
        std::lock_guard<std::mutex> lk(c->cmd_mu);
        if (!c->geom) setup_geometry(c, *dims);
        else if (std::memcmp(&c->dims, dims, sizeof(*dims)) != 0)
            return set_error(MPSW_EINVAL, "all models of a ctx must share dims (homogeneous slots, P:229)");
    }
    if (shards && shard_bytes)
        for (auto& R : c->ranks)
            if (shards[R->index] && shard_bytes[R->index] != R->S)
                return set_error(MPSW_EINVAL, "shard_bytes != S_r of the layout");
    auto m = std::make_unique<Model>();
    m->dims = *dims;
    try {
        for (auto& R : c->ranks) {
            m->arena.push_back(pin_alloc(R->S, R->numa));
            if (shards && shards[R->index]) parallel_memcpy(m->arena.back().p, (const uint8_t*)shards[R->index], R->S);
        }
    } catch (...) {
        for (auto& a : m->arena) pin_free(a);
        throw;
    }
    for (auto& R : c->ranks) {
        cudaSetDevice(R->device);
        cudaEvent_t ev;
        MPSW_CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        std::lock_guard<std::mutex> lk(R->mu);
        R->last_compute.push_back(ev);     // capacity reserved at init: no reallocation
        R->last_compute_valid.push_back(0);
    }
    {
        std::lock_guard<std::mutex> lk(c->cmd_mu);
        std::lock_guard<std::mutex> lk2(c->sm_mu);
        std::lock_guard<std::mutex> lk3(c->f_mu);
        if (c->models.size() >= kMaxModels) return set_error(MPSW_ENOMEM, "too many models");
        c->models.push_back(std::move(m));   // capacity reserved at init: no reallocation
        c->sm.add_model();
        c->f_slot_of.push_back(-1);
        c->f_state.push_back(ST_EVICTED);
        *model_id = (int)c->models.size() - 1;
    }
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_model_arena(mpsw_ctx* c, int model_id, int rank, void** host, uint64_t* bytes) {
    API_BEGIN
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    if (model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_ENOENT, "unknown model");
    const int li = local_index(c, rank);
    if (li < 0) return set_error(MPSW_EINVAL, "rank out of range or not driven by this process");
    if (host) *host = c->models[model_id]->arena[li].p;
    if (bytes) *bytes = c->ranks[li]->S;
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_synth_fill(mpsw_ctx* c, int model_id, int rank, uint64_t seed, int threads) {
    API_BEGIN
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    if (model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_ENOENT, "unknown model");
    if (rank != -1 && local_index(c, rank) < 0) return set_error(MPSW_EINVAL, "rank out of range or not local");
    for (auto& R : c->ranks)
        if (rank < 0 || rank == R->index)
            synth_fill_arena(c->dims, c->tp, c->pp, R->stage, R->trank, c->cfg.dtype, seed,
                             c->models[model_id]->arena[R->local].p, threads);
    return MPSW_OK;
    API_END
}

static mpsw_status submit_cmd(mpsw_ctx* c, int kind, int model_id, uint64_t* ticket) {
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    if (need_leader(c) != MPSW_OK) return MPSW_EINVAL;
    if (group_poisoned(c)) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
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
    const auto t0 = std::chrono::steady_clock::now();
    while (true) {   // a follower may see the ticket shortly after the leader published it
        {
            std::lock_guard<std::mutex> lk(c->done_mu);
            auto it = c->entries.find(ticket);
            if (it != c->entries.end()) e = it->second;
        }
        if (e || c->leader) break;
        if (timeout_s >= 0 && now_s(t0) > timeout_s) return set_error(MPSW_ETIMEDOUT, "ticket not seen yet");
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    if (!e) return set_error(MPSW_ENOENT, "unknown ticket");
    std::unique_lock<std::mutex> lk(c->done_mu);
    auto pred = [&] { return e->complete.load() || group_poisoned(c); };
    if (timeout_s < 0) c->done_cv.wait(lk, pred);
    else if (!c->done_cv.wait_for(lk, std::chrono::duration<double>(timeout_s), pred))
        return set_error(MPSW_ETIMEDOUT, "swap not complete");
    if (!e->complete.load()) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
    if (t_submit) *t_submit = e->t_submit;
    if (t_done_per_rank)
        for (int r = 0; r < c->nr; ++r) t_done_per_rank[r] = e->t_ack[r];
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
        for (int r = 0; r < c->nr; ++r) gpu_ms[r] = e->gpu_ms[r];   // 0 for ranks of other processes
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_request(mpsw_ctx* c, int model_id, const int32_t* tokens, int n_tokens, float* logits_out,
                         int64_t* request_id) {
    API_BEGIN
    if (!c || !logits_out || !request_id || !tokens) return set_error(MPSW_EINVAL, "NULL argument");
    if (need_leader(c) != MPSW_OK) return MPSW_EINVAL;
    if (group_poisoned(c)) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
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

// A completed request is released once the caller has observed it (poll/wait returned OK).
static void forget_req(mpsw_ctx* c, int64_t rid) {
    std::lock_guard<std::mutex> lk(c->cmd_mu);
    c->reqs.erase(rid);
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
        if (group_poisoned(c)) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
        return set_error(MPSW_EAGAIN, "pending");
    }
    if (t_arrival) *t_arrival = rq->t_arr;
    if (t_done) *t_done = rq->t_done;
    forget_req(c, rid);
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_wait_request(mpsw_ctx* c, int64_t rid, double timeout_s, double* t_arrival, double* t_done) {
    API_BEGIN
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    auto rq = find_req(c, rid);
    if (!rq) return set_error(MPSW_ENOENT, "unknown request");
    std::unique_lock<std::mutex> lk(c->done_mu);
    auto pred = [&] { return rq->done.load() || group_poisoned(c); };
    if (timeout_s < 0) c->done_cv.wait(lk, pred);
    else if (!c->done_cv.wait_for(lk, std::chrono::duration<double>(timeout_s), pred))
        return set_error(MPSW_ETIMEDOUT, "request not complete");
    if (!rq->done.load()) return set_error(MPSW_ECUDA, "ctx poisoned: " + c->poison_msg);
    if (t_arrival) *t_arrival = rq->t_arr;
    if (t_done) *t_done = rq->t_done;
    lk.unlock();
    forget_req(c, rid);
    return MPSW_OK;
    API_END
}

// Slot of a model that is resident as seen by this process (-1 otherwise).
static int resident_slot(mpsw_ctx* c, int model_id) {
    if (c->leader) {
        std::lock_guard<std::mutex> lk(c->sm_mu);
        return c->sm.state[model_id] == ST_RESIDENT ? c->sm.slot_of[model_id] : -1;
    }
    std::lock_guard<std::mutex> lk(c->f_mu);
    return c->f_state[model_id] == ST_RESIDENT ? c->f_slot_of[model_id] : -1;
}

mpsw_status mpsw_residency(mpsw_ctx* c, int model_id, int* state) {
    API_BEGIN
    if (!c || !state) return set_error(MPSW_EINVAL, "NULL argument");
    if (model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_ENOENT, "unknown model");
    if (c->leader) {
        std::lock_guard<std::mutex> lk(c->sm_mu);
        *state = c->sm.state[model_id];
    } else {
        std::lock_guard<std::mutex> lk(c->f_mu);
        *state = c->f_state[model_id];
    }
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_checksum(mpsw_ctx* c, int model_id, int rank, int on_device, uint64_t* out) {
    API_BEGIN
    if (!c || !out) return set_error(MPSW_EINVAL, "NULL argument");
    if (model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_ENOENT, "unknown model");
    const int li = local_index(c, rank);
    if (li < 0) return set_error(MPSW_EINVAL, "rank out of range or not driven by this process");
    if (!on_device) {
        *out = host_checksum(c->models[model_id]->arena[li].p, c->ranks[li]->S, 0);
        return MPSW_OK;
    }
    const int slot = resident_slot(c, model_id);
    if (slot < 0) return set_error(MPSW_EINVAL, "model not RESIDENT");
    Rank& R = *c->ranks[li];
    MPSW_CU(cudaSetDevice(R.device));
    MPSW_CU(cudaMemsetAsync(R.d_sum, 0, 8, R.aux));
    launch_checksum(R.slots[slot].base, R.S, R.d_sum, R.aux);
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
    const int li = local_index(c, rank);
    if (li < 0 || offset + bytes > c->ranks[li]->S) return set_error(MPSW_EINVAL, "rank or range");
    const int slot = resident_slot(c, model_id);
    if (slot < 0) return set_error(MPSW_EINVAL, "model not RESIDENT");
    Rank& R = *c->ranks[li];
    MPSW_CU(cudaSetDevice(R.device));
    MPSW_CU(cudaMemcpyAsync(dst, R.slots[slot].base + offset, bytes, cudaMemcpyDeviceToHost, R.aux));
    MPSW_CU(cudaStreamSynchronize(R.aux));
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_trace_dump(mpsw_ctx* c, const char* path) {
    API_BEGIN
    if (!c || !path) return set_error(MPSW_EINVAL, "NULL argument");
    if (need_leader(c) != MPSW_OK) return MPSW_EINVAL;
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
    o->shard_bytes = c->rank_S[0];
    o->fwd_gpu_us_sum = c->fwd_us_sum.load();
    o->fwd_gpu_n = c->fwd_n.load();
    return MPSW_OK;
    API_END
}

}  // extern "C"
