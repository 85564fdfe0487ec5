// Deterministic engine state machine (DESIGN.md §2 readings #1-#7, #21, #24, #26): per-model FIFO
// queues with arrival timestamps, oldest-head batch scheduling, LRU victim with
// load/offload entries, ack-based completion. The numpy oracle
// (oracle/scheduler.py) replays this engine's recorded event log and must emit identical
// decisions; the two are written independently from the same spec.
#pragma once

#include "internal.h"

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


}  // namespace mpsw
