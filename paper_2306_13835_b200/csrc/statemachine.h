// Deterministic engine state machine (DESIGN.md §2 readings #1-#7, #21, #24, #26): per-model FIFO
// queues with arrival timestamps, oldest-head batch scheduling, LRU victim with
// load/offload entries, ack-based completion. The numpy oracle
// (oracle/scheduler.py) replays this engine's recorded event log and must emit identical
// decisions; the two are written independently from the same spec.
#pragma once

#include "internal.h"

#include <algorithm>
#include <cmath>
#include <deque>
#include <map>
#include <vector>

namespace mpsw {

enum { E_LOAD = 0, E_OFFLOAD = 1, E_BATCH = 2 };
enum { ST_EVICTED = 0, ST_LOADING = 1, ST_RESIDENT = 2, ST_OFFLOADING = 3 };

// Decision of the state machine (mirrors oracle/scheduler.py's dicts).
struct Decision {
    int kind;  // 0 load, 1 offload, 2 batch, 3 complete, 4 noop, 5 reject
    uint64_t id = 0;
    int model = -1;
    uint64_t off = 0;  // load / offload: byte offset of the model's range in every rank's region
    std::vector<int64_t> rids;
    const char* status = "";
    bool prefetch = false;  // load issued by the prefetch policy (reading #29), not by a request
};

// Deterministic engine state machine. Placement (reading #28, NEXT-4):
// each rank's parameter region is `cap` bytes; model m occupies [off[m], off[m] + size[m]) on
// every rank (size = its largest per-rank shard, 4 KiB-aligned). A load takes the lowest-address
// free range that fits (first fit). With no fit, eligible victims are taken in victim-key order
// until a first fit appears, and only the victims overlapping that range are evicted. For
// equal-size models this is exactly the k = floor(cap / size) slot scheme (off = slot * size).
struct StateMachine {
    int n_models = 0, tp = 1, max_batch = 1, D = 1;
    uint64_t cap = 0;
    std::vector<uint64_t> size;
    std::vector<std::deque<std::pair<int64_t, double>>> queue;
    std::vector<int> state, outstanding;
    std::vector<int64_t> off_of;   // -1 = owns no range (EVICTED / OFFLOADING)
    std::vector<double> last_use;
    struct Pend { int kind, model, left; uint32_t mask; };
    std::map<uint64_t, Pend> pending;
    std::map<uint64_t, std::pair<int, std::vector<int64_t>>> batches;
    int inflight = 0;
    uint64_t next_id = 0;
    // prefetch (NEXT-3, reading #29): the last kHist arrivals, last arrival time per model
    static constexpr int kHist = 32;
    bool prefetch = false;
    int victim_policy = 0;   // 0: LRU prefix + first fit (reading #28); 1: min-cost window (reading #30)
    std::deque<int> recent;
    std::vector<double> last_arr;

    void add_model(uint64_t bytes) {
        queue.emplace_back();
        state.push_back(ST_EVICTED);
        outstanding.push_back(0);
        off_of.push_back(-1);
        last_use.push_back(-INFINITY);
        size.push_back(bytes);
        last_arr.push_back(-INFINITY);
        ++n_models;
    }
    bool head_less(int a, int b) const {  // (head t_arr, reg order)
        const double ta = queue[a].front().second, tb = queue[b].front().second;
        return ta < tb || (ta == tb && a < b);
    }
    // lowest offset o with [o, o + need) free of every range owned by a model not in `skip`
    int64_t first_fit(uint64_t need, const std::vector<char>& skip) const {
        std::vector<std::pair<uint64_t, uint64_t>> iv;
        for (int m = 0; m < n_models; ++m)
            if (off_of[m] >= 0 && !skip[m]) iv.push_back({(uint64_t)off_of[m], (uint64_t)off_of[m] + size[m]});
        std::sort(iv.begin(), iv.end());
        uint64_t cur = 0;
        for (const auto& r : iv) {
            if (r.first >= cur + need) return (int64_t)cur;
            cur = std::max(cur, r.second);
        }
        return cap >= cur + need ? (int64_t)cur : -1;
    }
    int64_t free_range(int m) const { return first_fit(size[m], std::vector<char>(n_models, 0)); }

    // Reading #30 (victim_policy 1, NEXT-4 knapsack): among windows [o, o + need) inside the region
    // whose every overlapping model is an eligible victim, take the one minimising (bytes evicted,
    // number of victims, the newest victim key, o) — a victim key is (queue non-empty, last_use,
    // model). Windows starting at 0 or at the end of an owned range suffice (sliding a feasible
    // window left to the nearest such start only drops overlapped ranges). The overlapped victims
    // are offloaded in victim-key order (vics is sorted by it), then m is loaded. No feasible
    // window: nothing is emitted (the requester defers).
    void min_cost_window(int m, const std::vector<int>& vics, std::vector<Decision>& out) {
        const uint64_t need = size[m];
        std::vector<char> elig(n_models, 0);
        for (int v : vics) elig[v] = 1;
        std::vector<uint64_t> starts{0};
        for (int v = 0; v < n_models; ++v)
            if (off_of[v] >= 0) starts.push_back((uint64_t)off_of[v] + size[v]);
        std::sort(starts.begin(), starts.end());
        starts.erase(std::unique(starts.begin(), starts.end()), starts.end());
        bool found = false;
        uint64_t best_bytes = 0, best_o = 0;
        int best_n = 0;
        int best_key_m = -1;      // model whose key is the window's newest victim key
        std::vector<char> best_set;
        auto key_less = [&](int a, int b) {
            const int qa = queue[a].empty() ? 0 : 1, qb = queue[b].empty() ? 0 : 1;
            if (qa != qb) return qa < qb;
            if (last_use[a] != last_use[b]) return last_use[a] < last_use[b];
            return a < b;
        };
        for (uint64_t o : starts) {
            if (o + need > cap) continue;
            std::vector<char> set(n_models, 0);
            uint64_t bytes = 0;
            int n = 0, newest = -1;
            bool ok = true;
            for (int v = 0; v < n_models && ok; ++v) {
                if (off_of[v] < 0) continue;
                const uint64_t lo = (uint64_t)off_of[v], hi = lo + size[v];
                if (!(lo < o + need && o < hi)) continue;
                if (!elig[v]) ok = false;
                set[v] = 1;
                bytes += size[v];
                ++n;
                if (newest < 0 || key_less(newest, v)) newest = v;
            }
            if (!ok) continue;
            bool better = !found;
            if (found) {
                if (bytes != best_bytes) better = bytes < best_bytes;
                else if (n != best_n) better = n < best_n;
                else if (newest != best_key_m) better = key_less(newest, best_key_m);
                else better = o < best_o;
            }
            if (better) {
                found = true;
                best_bytes = bytes, best_n = n, best_key_m = newest, best_o = o;
                best_set = set;
            }
        }
        if (!found) return;
        for (int v : vics)
            if (best_set[v]) offload(v, out);
        load(m, best_o, out);
    }
    void load(int m, uint64_t o, std::vector<Decision>& out) {
        Decision d{0, next_id++, m, o};
        off_of[m] = (int64_t)o;
        state[m] = ST_LOADING;
        pending[d.id] = {E_LOAD, m, tp, 0u};
        out.push_back(d);
    }
    void offload(int v, std::vector<Decision>& out) {
        Decision d{1, next_id++, v, (uint64_t)off_of[v]};
        off_of[v] = -1;
        state[v] = ST_OFFLOADING;
        pending[d.id] = {E_OFFLOAD, v, tp, 0u};
        out.push_back(d);
    }
    void schedule(double now, std::vector<Decision>& out) {
        std::vector<char> blocked(n_models, 0);
        for (;;) {
            int m = -1;
            for (int i = 0; i < n_models; ++i)
                if (!queue[i].empty() && !blocked[i] && (m < 0 || head_less(i, m))) m = i;
            if (m < 0) break;
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
                const int64_t o = free_range(m);
                if (o >= 0) {
                    load(m, (uint64_t)o, out);
                } else {
                    auto key_less = [&](int a, int b) {  // prefer empty queue, then LRU, then reg order
                        const int qa = queue[a].empty() ? 0 : 1, qb = queue[b].empty() ? 0 : 1;
                        if (qa != qb) return qa < qb;
                        if (last_use[a] != last_use[b]) return last_use[a] < last_use[b];
                        return a < b;
                    };
                    std::vector<int> vics;
                    for (int v = 0; v < n_models; ++v) {
                        if (state[v] != ST_RESIDENT || outstanding[v] != 0) continue;
                        if (!queue[v].empty() && !head_less(m, v)) continue;   // older head: not a victim
                        vics.push_back(v);
                    }
                    std::sort(vics.begin(), vics.end(), key_less);
                    if (victim_policy == 1) {
                        min_cost_window(m, vics, out);
                        blocked[m] = 1;
                        continue;
                    }
                    std::vector<char> skip(n_models, 0);
                    for (int v : vics) {
                        skip[v] = 1;
                        const int64_t f = first_fit(size[m], skip);
                        if (f < 0) continue;
                        const uint64_t lo = (uint64_t)f, hi = lo + size[m];
                        for (int w : vics) {                       // evict only what overlaps the fit
                            if (!skip[w]) break;
                            const uint64_t wl = (uint64_t)off_of[w], wh = wl + size[w];
                            if (wl < hi && lo < wh) offload(w, out);
                        }
                        load(m, lo, out);
                        break;
                    }
                }
                blocked[m] = 1;
            }
        }
        prefetch_step(out);
    }

    // events ------------------------------------------------------------------------------
    // Prefetch into free space while no load / offload is in flight: among EVICTED models with
    // an empty queue and at least one of the last kHist arrivals, by (count desc, last arrival
    // desc, registration order), the first whose size fits a free range is loaded. Never evicts.
    void prefetch_step(std::vector<Decision>& out) {
        if (!prefetch || !pending.empty()) return;
        std::vector<int> cnt(n_models, 0), cand;
        for (int m : recent) ++cnt[m];
        for (int m = 0; m < n_models; ++m)
            if (state[m] == ST_EVICTED && queue[m].empty() && cnt[m] > 0) cand.push_back(m);
        std::sort(cand.begin(), cand.end(), [&](int a, int b) {
            if (cnt[a] != cnt[b]) return cnt[a] > cnt[b];
            if (last_arr[a] != last_arr[b]) return last_arr[a] > last_arr[b];
            return a < b;
        });
        for (int m : cand) {
            const int64_t o = free_range(m);
            if (o < 0) continue;
            load(m, (uint64_t)o, out);
            out.back().prefetch = true;
            return;
        }
    }
    void arrival(int64_t rid, int m, double t, std::vector<Decision>& out) {
        recent.push_back(m);
        if ((int)recent.size() > kHist) recent.pop_front();
        last_arr[m] = t;
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
            const int64_t o = free_range(m);
            if (o < 0) {
                Decision d{5, 0, m};
                d.status = "ENOMEM";
                out.push_back(d);
            } else {
                load(m, (uint64_t)o, out);
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
        std::vector<std::pair<uint64_t, uint64_t>> iv;
        for (int m = 0; m < n_models; ++m) {
            if (outstanding[m] > 0 && state[m] != ST_RESIDENT)
                throw Error(MPSW_EINVARIANT, "in-flight batch on a non-resident model");
            const bool owns = state[m] == ST_LOADING || state[m] == ST_RESIDENT;
            if (owns != (off_of[m] >= 0)) throw Error(MPSW_EINVARIANT, "range ownership");
            if (owns) iv.push_back({(uint64_t)off_of[m], (uint64_t)off_of[m] + size[m]});
        }
        std::sort(iv.begin(), iv.end());
        for (size_t i = 0; i < iv.size(); ++i) {
            if (iv[i].second > cap) throw Error(MPSW_EINVARIANT, "range beyond the budget");
            if (i && iv[i].first < iv[i - 1].second) throw Error(MPSW_EINVARIANT, "overlapping ranges");
        }
        if (inflight > D) throw Error(MPSW_EINVARIANT, "D exceeded");
    }
};


}  // namespace mpsw
