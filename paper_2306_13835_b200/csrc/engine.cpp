// mpsw runtime core: per-rank workers, the engine (scheduler) thread, the multi-process follower
// and control plane, and the region / workspace geometry. (Store: store.cpp; swap entries: swap.cpp; batch
// entries: batch.cpp; C-ABI: capi.cpp; types and the ctx: runtime.h.)
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
#include "runtime.h"

#include <sys/mman.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>

namespace mpsw {


std::string& tls_error() {
    thread_local std::string e;
    return e;
}
mpsw_status set_error(mpsw_status s, const std::string& msg) {
    tls_error() = msg;
    return s;
}

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
void group_barrier(mpsw_ctx* c, int stage) {
    if (!c->mp) {
        if (!c->stage_barrier[stage].wait([c] { return c->poisoned.load() != 0; }))
            throw Error(group_poisoned(c) ? MPSW_ECUDA : MPSW_ETIMEDOUT,
                        group_poisoned(c) ? "peer rank failed (ctx poisoned)" : "group barrier timed out");
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
        // pipelined entries (NEXT-1): hand the entry to the same TP rank of the next stage
        // as soon as it is issued here — a load without waiting for its copy, a batch once its
        // kernels (and the hop event of its residual stream) are on this rank's stream
        if (c->pp > 1 && !c->cfg.pp_broadcast && R->stage + 1 < c->pp) {
            const int nxt = c->local_of[R->index + c->tp];
            if (nxt >= 0) push_to_rank(*c->ranks[nxt], e);
        }
        c->cmd_cv.notify_all();
    }
}

void push_to_rank(Rank& R, const EntryP& e) {
    std::lock_guard<std::mutex> lk(R.mu);
    R.fifo.push_back(e);
    R.cv.notify_one();
}

// The engine hands every entry, in its one global order, to every worker — or, with pipeline
// stages (default), to the stage-0 workers only: later stages receive it from their predecessor.
void push_to_workers(mpsw_ctx* c, const EntryP& e) {
    for (auto& R : c->ranks)
        if (c->pp == 1 || c->cfg.pp_broadcast || R->stage == 0) push_to_rank(*R, e);
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
            case 0:
                o << "{\"dec\":\"load\",\"id\":" << d.id << ",\"model\":" << d.model << ",\"off\":" << d.off
                  << (d.prefetch ? ",\"prefetch\":true}" : "}");
                break;
            case 1: o << "{\"dec\":\"offload\",\"id\":" << d.id << ",\"model\":" << d.model << ",\"off\":" << d.off << "}"; break;
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
    rec.off = e.off;
    rec.ring = e.ring;
    rec.B = e.B;
    rec.M = e.M;
    rec.writeback = e.writeback;
    rec.stamp = e.expect_stamp;
    s->log_tail.store(tail + 1, std::memory_order_release);
}

void dispatch(mpsw_ctx* c, const std::vector<Decision>& ds, double now) {
    for (const auto& d : ds) {
        if (d.kind > 2) continue;
        if (d.prefetch) c->prefetches++;
        auto e = std::make_shared<Entry>();
        e->id = d.id;
        e->kind = d.kind;
        e->model = d.model;
        e->off = d.off;
        e->t_submit = now;
        if (d.kind == E_LOAD) c->load_id_of[d.model] = e->id;
        if (d.kind == E_BATCH) {
            e->expect_stamp = c->load_id_of[d.model];
            e->off = (uint64_t)c->sm.off_of[d.model];
            // pack tokens + meta into the pinned ring entry (shm in mp mode: every rank reads it)
            e->ring = c->ring_next;
            c->ring_next = (c->ring_next + 1) % c->ring_n;
            // the slot's previous batch may still be copying out on the completer thread
            for (int spins = 0; c->slot_busy[e->ring].load(std::memory_order_acquire);) spin_pause(spins);
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
            std::lock_guard<std::mutex> lk(c->tap_mu);
            if (c->tap_next.dst) {
                e->tap = c->tap_next;
                c->tap_next = Tap{};
            }
        } else {
            e->writeback = d.kind == E_OFFLOAD ? c->writeback_now.load() : 0;
            c->swap_gen.fetch_add(1);
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

// Batch completion on the engine thread: stamp t_done (the last rank's slice has landed, reading
// #15) and hand the logits copy-out to the completer thread, so [B, V] fp32 memcpys (6.4 MB at
// cfg4) never stall scheduling or ack processing.
void complete_batch(mpsw_ctx* c, const EntryP& e, double now) {
    for (auto& rq : e->reqs) {
        rq->t_done = now;
        c->eng_reqs.erase(rq->rid);
    }
    c->n_batches++;
    c->n_requests += e->reqs.size();
    c->slot_busy[e->ring].store(1, std::memory_order_release);
    {
        std::lock_guard<std::mutex> lk(c->comp_mu);
        c->comp_q.push_back(e);
    }
    c->comp_cv.notify_one();
}

void completer_main(mpsw_ctx* c) {
    for (;;) {
        EntryP e;
        {
            std::unique_lock<std::mutex> lk(c->comp_mu);
            c->comp_cv.wait(lk, [&] { return !c->comp_q.empty() || c->comp_stop; });
            if (c->comp_q.empty()) return;
            e = c->comp_q.front();
            c->comp_q.pop_front();
        }
        const uint8_t* ring = c->stg + (size_t)e->ring * c->ring_stride;
        const int V = c->models[e->model]->dims.vocab;
        for (size_t b = 0; b < e->reqs.size(); ++b)
            std::memcpy(e->reqs[b]->out, (const float*)ring + b * (size_t)V, (size_t)V * 4);
        c->slot_busy[e->ring].store(0, std::memory_order_release);
        {
            std::lock_guard<std::mutex> lk(c->done_mu);
            for (auto& rq : e->reqs) rq->done.store(1, std::memory_order_release);
        }
        c->done_cv.notify_all();
    }
}

// Device time of a finished batch's forward on the first local rank (stats), then free its events.
void record_spans(mpsw_ctx* c, Entry& e) {
    if (!c->trace && !c->timeline_on) return;
    static const char* kinds[] = {"load", "offload", "batch"};
    for (auto& Rp : c->ranks) {
        const int r = Rp->index;
        float t0 = 0, t1 = 0;
        if (!Rp->ev_base || !e.ev_start[r] || !e.ev_done[r]) continue;
        if (cudaEventElapsedTime(&t0, Rp->ev_base, e.ev_start[r]) != cudaSuccess ||
            cudaEventElapsedTime(&t1, Rp->ev_base, e.ev_done[r]) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        std::ostringstream o;
        o << "{\"kind\":\"" << kinds[e.kind] << "\",\"id\":" << e.id << ",\"model\":" << e.model << ",\"rank\":" << r
          << ",\"device\":" << Rp->device << ",\"t0_ms\":" << fmt_d(t0) << ",\"t1_ms\":" << fmt_d(t1) << "}";
        std::lock_guard<std::mutex> lk(c->trace_mu);
        c->timeline.push_back(o.str());
    }
}

void record_fwd_time(mpsw_ctx* c, Entry& e) {
    record_spans(c, e);
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

// A completed swap entry stays queryable (mpsw_wait / mpsw_entry_gpu_ms) until kKeepTickets
// newer swaps have completed; then it is dropped (ENOENT), so a long-running server's entry map
// stays bounded. Called with done_mu held.
constexpr size_t kKeepTickets = 4096;
void retire_ticket(mpsw_ctx* c, uint64_t id) {
    c->done_tickets.push_back(id);
    while (c->done_tickets.size() > kKeepTickets) {
        c->entries.erase(c->done_tickets.front());
        c->done_tickets.pop_front();
    }
}

// Debug checks (mpsw_config.debug_checks): after a batch completed, a non-zero error word on
// any local rank means its forward found the model's residency stamp different from the load the
// engine gated the batch on — the batch read parameters that were not (or no longer) resident.
void check_stamps(mpsw_ctx* c, const Entry& e) {
    if (!c->cfg.debug_checks) return;
    for (auto& R : c->ranks)
        if (R->h_err && *(volatile unsigned int*)R->h_err)
            throw Error(MPSW_EINVARIANT, "batch " + std::to_string(e.id) + " of model " + std::to_string(e.model) +
                                             " ran on a range whose residency stamp is not load " +
                                             std::to_string(e.expect_stamp) + " (rank " + std::to_string(R->index) + ")");
}

bool poll_inflight(mpsw_ctx* c) {
    bool progressed = false;
    for (size_t i = 0; i < c->inflight.size();) {
        Entry& e = *c->inflight[i];
        const EntryP ep = c->inflight[i];
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
                if (e.kind == E_LOAD) c->h2d_bytes += c->models[e.model]->rank_S[r];
                else if (e.writeback) c->d2h_bytes += c->models[e.model]->rank_S[r];
            }
        }
        if (e.n_acked == c->nr) {
            const double now = now_s(c->t0);
            if (e.kind == E_BATCH) {
                check_stamps(c, e);
                complete_batch(c, ep, now);
                log_event(c, "{\"ev\":\"batch_done\",\"t\":" + fmt_d(now) + ",\"batch\":" + std::to_string(e.id) + "}");
                step_and_dispatch(c, [&](std::vector<Decision>& ds) { c->sm.batch_done(e.id, now, ds); }, now);
                record_fwd_time(c, e);
            } else {
                (e.kind == E_LOAD ? c->swaps_in : c->swaps_out)++;
                finish_swap_events(c, e);
                std::lock_guard<std::mutex> lk(c->done_mu);
                e.complete.store(1, std::memory_order_release);
                retire_ticket(c, e.id);
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
            e->off = rec.off;
            e->ring = rec.ring;
            e->B = rec.B;
            e->M = rec.M;
            e->writeback = rec.writeback;
            e->expect_stamp = rec.stamp;
            e->t_submit = now_s(c->t0);
            if (e->kind != E_BATCH) {
                c->swap_gen.fetch_add(1);
                std::lock_guard<std::mutex> lk(c->done_mu);
                c->entries[e->id] = e;
            }
            {
                std::lock_guard<std::mutex> lk(c->f_mu);
                if (e->kind == E_LOAD) { c->f_off_of[e->model] = (int64_t)e->off; c->f_state[e->model] = ST_LOADING; }
                if (e->kind == E_OFFLOAD) { c->f_off_of[e->model] = -1; c->f_state[e->model] = ST_OFFLOADING; }
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
                    if (e.kind == E_LOAD && c->f_off_of[e.model] == (int64_t)e.off) c->f_state[e.model] = ST_RESIDENT;
                    if (e.kind == E_OFFLOAD && c->f_state[e.model] == ST_OFFLOADING) c->f_state[e.model] = ST_EVICTED;
                }
                if (e.kind == E_BATCH) {
                    check_stamps(c, e);
                    record_fwd_time(c, e);
                    c->n_batches++;
                } else {
                    (e.kind == E_LOAD ? c->swaps_in : c->swaps_out)++;
                    if (e.kind == E_LOAD) c->h2d_bytes += c->models[e.model]->rank_S[R.index];
                    else if (e.writeback) c->d2h_bytes += c->models[e.model]->rank_S[R.index];
                    finish_swap_events(c, e);
                    std::lock_guard<std::mutex> lk(c->done_mu);
                    e.complete.store(1, std::memory_order_release);
                    retire_ticket(c, e.id);
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

// Kernel limits of a model and, once the geometry is fixed, that it fits the workspace.
void check_dims(mpsw_ctx* c, const mpsw_opt_dims& d) {
    const int hd = d.hidden / d.heads;
    if (hd % 8 || hd > 128) throw Error(MPSW_EINVAL, "head_dim must be a multiple of 8 and <= 128");
    if ((d.hidden / c->tp) % 8 || (d.ffn / c->tp) % 8 || d.hidden % 8)
        throw Error(MPSW_EINVAL, "hidden/tp, ffn/tp and hidden must be multiples of 8");
    if (d.hidden > 12288) throw Error(MPSW_EINVAL, "hidden too large for the LN kernel");
    if (c->geom) {
        const mpsw_opt_dims& x = c->dims_max;
        if (d.hidden > x.hidden || d.ffn > x.ffn || d.vocab > x.vocab)
            throw Error(MPSW_EINVAL, "model exceeds the ctx's workspace dims (set mpsw_config.max_dims, or register "
                                     "the largest model first)");
    }
}

// Forward shape of model d on rank R (its stage's layers).
FwdShape fwd_shape(mpsw_ctx* c, const mpsw_opt_dims& d, const Rank& R) {
    FwdShape f{};
    f.n_layers = d.n_layers / c->pp; f.hidden = d.hidden; f.heads_local = d.heads / c->tp;
    f.head_dim = d.hidden / d.heads;
    f.ffn_local = d.ffn / c->tp; f.vocab_local = d.vocab / c->tp; f.vocab = d.vocab; f.tp = c->tp;
    f.rank = R.trank;
    f.dtype = c->cfg.dtype;
    f.gemm_impl = c->cfg.gemm_impl;
    f.max_rows = c->max_rows;
    return f;
}

// Fix the geometry at the first registration: the region of every rank is `cap` bytes (budget
// rounded down to 4 KiB; models are placed in it by the state machine); the forward workspace is
// sized for dims_max (elementwise max shape) and max_batch * max_tokens rows; TP peers wired
// (collective in multi-process mode: IPC handles exchanged through shm).
void setup_geometry(mpsw_ctx* c, const mpsw_opt_dims& dmax) {
    check_dims(c, dmax);
    c->dims_max = dmax;
    c->cap = c->cfg.param_budget_bytes_per_gpu / kSlotAlign * kSlotAlign;
    c->max_rows = c->cfg.max_batch * c->cfg.max_tokens;
    const unsigned ev_flags = c->mp ? (cudaEventInterprocess | cudaEventDisableTiming) : cudaEventDisableTiming;
    for (auto& Rp : c->ranks) {
        Rank& R = *Rp;
        MPSW_CU(cudaSetDevice(R.device));
        FwdShape f = fwd_shape(c, dmax, R);
        f.n_layers = 1;                                  // the workspace does not depend on depth
        R.fs_max = f;
        const size_t wsb = workspace_bytes(f, c->max_rows, c->cfg.max_batch);
        MPSW_CU(cudaMalloc(&R.ws_base, wsb));
        MPSW_CU(cudaMemset(R.ws_base, 0, wsb));
        workspace_carve(R.ws, f, c->max_rows, c->cfg.max_batch, R.ws_base);
        for (auto& ev : R.ev_point) MPSW_CU(cudaEventCreateWithFlags(&ev, ev_flags));
        for (auto& ev : R.ev_ag) MPSW_CU(cudaEventCreateWithFlags(&ev, ev_flags));
        c->peer_a[R.index] = R.ws.a;
        MPSW_CU(cudaEventCreateWithFlags(&R.ev_stage, cudaEventDisableTiming));
        if (c->pp > 1 && R.stage + 1 < c->pp) {      // hop ring: one [max_rows, h] fp32 slot per ring entry
            const size_t slot = ((size_t)c->max_rows * dmax.hidden * 4 + 255) & ~size_t(255);
            MPSW_CU(cudaMalloc(&R.hop_base, slot * (size_t)(c->D + 1)));
            for (int j = 0; j <= c->D; ++j) {
                R.hop.push_back((float*)((uint8_t*)R.hop_base + slot * j));
                cudaEvent_t ev;
                MPSW_CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                R.ev_hop.push_back(ev);
            }
        }
        for (int pb = 0; pb < 2; ++pb) {
            c->peer_partial[R.index][pb] = R.ws.partial[pb];
            c->peer_ev[R.index][pb] = R.ev_point[pb];
            c->peer_ev_ag[R.index][pb] = R.ev_ag[pb];
        }
    }
    const mpsw_opt_dims& d = dmax;
    // staging ring: per entry [max_batch * V] fp32 logits, then tokens [max_rows] + meta
    c->ring_n = c->D + 1;
    c->slot_busy.reset(new std::atomic<int>[c->ring_n]);
    for (int j = 0; j < c->ring_n; ++j) c->slot_busy[j].store(0);
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
            MPSW_CU(cudaIpcGetEventHandle(&s->ev_ag_handle[R.index][pb], R.ev_ag[pb]));
        }
        s->a_off[R.index] = (uint64_t)((uint8_t*)R.ws.a - R.ws_base);
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
                MPSW_CU(cudaIpcOpenEventHandle(&ev, s->ev_ag_handle[p][pb]));
                c->ipc_ev_opened.push_back(ev);
                c->peer_ev_ag[p][pb] = ev;
            }
            c->peer_a[p] = (uint8_t*)base + s->a_off[p];
        }
        group_barrier(c);
        if (c->leader) shm_unlink(stg_name.c_str());   // mapped everywhere; name no longer needed
    }
    {
        std::lock_guard<std::mutex> lk(c->sm_mu);
        c->sm.cap = c->cap;
    }
    c->geom = true;
}

}  // namespace mpsw
