// Product-side synthetic weight generator (input generation, NOT the hot path) and a host
// checksum. Implements the counter-based spec of DESIGN.md §Inputs (C0) independently of the
// numpy oracle:  x = splitmix64(seed ^ (tensor_id << 40) ^ flat_index); u = x >> 40;
// w = (u - 2^23) * 2^-28; LN gammas store 1 + w; fp32 RNE, then bf16 RNE in bf16 mode.
// flat_index addresses the FULL tensor, so each rank fills exactly its slice.
#include "internal.h"

namespace mpsw {
void flush_to_memory(uint8_t* p, uint64_t n);   // store.cpp
}

#include <cmath>
#include <cstring>
#include <thread>

namespace mpsw {

static inline uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint16_t f32_to_bf16_rne(float f) {
    uint32_t b;
    std::memcpy(&b, &f, 4);
    b += 0x7FFFu + ((b >> 16) & 1u);
    return (uint16_t)(b >> 16);
}

static inline float value_f32(uint64_t key, uint64_t flat, bool gamma) {
    const uint64_t x = sm64(key ^ flat);
    const int64_t u = (int64_t)(x >> 40);
    const double w = (double)(u - (1 << 23)) * (1.0 / 268435456.0);  // 2^-28, exact
    return (float)(gamma ? 1.0 + w : w);
}

namespace {
struct Job {
    uint64_t key;
    bool gamma;
    int split, rows, cols;  // shard shape
    int full_cols;          // columns of the full tensor
    uint64_t row0, col0;    // shard origin in the full tensor
    uint8_t* dst;
};
}  // namespace

static void run_rows(const Job& j, int es, int r0, int r1) {
    for (int r = r0; r < r1; ++r) {
        const uint64_t base = (j.row0 + r) * (uint64_t)j.full_cols + j.col0;
        for (int c = 0; c < j.cols; ++c) {
            const float v = value_f32(j.key, base + c, j.gamma);
            const uint64_t o = ((uint64_t)r * j.cols + c) * es;
            if (es == 2) {
                const uint16_t b = f32_to_bf16_rne(v);
                std::memcpy(j.dst + o, &b, 2);
            } else {
                std::memcpy(j.dst + o, &v, 4);
            }
        }
    }
}

void synth_fill_arena(const mpsw_opt_dims& d, int tp, int pp, int stage, int rank, int dtype, uint64_t seed,
                      uint8_t* dst, int threads) {
    Layout L;
    if (compute_layout(d, tp, pp, stage, rank, dtype, L) != MPSW_OK) throw Error(MPSW_EINVAL, tls_error());
    const int es = dtype == MPSW_BF16 ? 2 : 4;
    std::memset(dst, 0, L.bytes);  // padding is zero (C2)
    // Split every tensor into row blocks; hand blocks to threads round-robin.
    struct Task { Job j; int r0, r1; };
    std::vector<Task> tasks;
    for (size_t tid = 0; tid < L.t.size(); ++tid) {
        const auto& t = L.t[tid];
        Job j{};
        j.key = seed ^ ((uint64_t)t.tensor_id << 40);   // C0 key: id in the full canonical list
        const std::string name(t.name);
        j.gamma = name.find("layer_norm.weight") != std::string::npos;
        j.split = t.split;
        // vectors are stored as [n, 1]: treat as rows of one column in a [n, 1] full tensor
        j.rows = t.rows;
        j.cols = t.cols;
        if (t.split == 0) {
            j.full_cols = t.cols; j.row0 = 0; j.col0 = 0;
        } else if (t.split == 1) {
            j.full_cols = t.cols; j.row0 = (uint64_t)rank * t.rows; j.col0 = 0;
        } else {
            j.full_cols = t.cols * tp; j.row0 = 0; j.col0 = (uint64_t)rank * t.cols;
        }
        j.dst = dst + t.offset;
        const int step = std::max(1, (int)(4096 / std::max(1, t.cols)) * 16);
        for (int r = 0; r < t.rows; r += step) tasks.push_back({j, r, std::min(t.rows, r + step)});
    }
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    threads = std::max(1, std::min<int>(threads, (int)tasks.size()));
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i)
        pool.emplace_back([&] {
            for (size_t k; (k = next.fetch_add(1)) < tasks.size();) run_rows(tasks[k].j, es, tasks[k].r0, tasks[k].r1);
        });
    for (auto& th : pool) th.join();
    flush_to_memory(dst, L.bytes);      // leave the arena clean in DRAM for the swap DMA (store.cpp)
}

uint64_t host_checksum(const uint8_t* p, uint64_t bytes, int threads) {
    // C4: sum_j splitmix64(word_j ^ (j * 0x9E3779B97F4A7C15)) mod 2^64
    const uint64_t n = bytes / 8;
    if (threads <= 0) threads = (int)std::thread::hardware_concurrency();
    threads = std::max<int>(1, std::min<uint64_t>(threads, n / 65536 + 1));
    std::vector<uint64_t> part(threads, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            const uint64_t b = n * t / threads, e = n * (t + 1) / threads;
            uint64_t h = 0;
            for (uint64_t j = b; j < e; ++j) {
                uint64_t w;
                std::memcpy(&w, p + 8 * j, 8);
                h += sm64(w ^ (j * 0x9E3779B97F4A7C15ull));
            }
            part[t] = h;
        });
    for (auto& th : pool) th.join();
    uint64_t h = 0;
    for (auto v : part) h += v;
    return h;
}

}  // namespace mpsw
