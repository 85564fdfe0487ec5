// Batch entries (a6 / a7): the TP (x PP) forward of one rank, with the all-reduce fused into the
// LayerNorm kernel over peer memory, and the logits slice returned to the pinned staging ring.
#include "runtime.h"
#include "../../include/mpsw_testing.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace mpsw {

// Reduce-scatter all-reduce from this many bytes of peer partials per rank and point
// ((t-1)·M·h·4); MPSW_RS_MIN_BYTES overrides (0 = always, huge = never).
static uint64_t rs_min_bytes() {
    static uint64_t v = [] {
        const char* e = getenv("MPSW_RS_MIN_BYTES");
        return e ? (uint64_t)atoll(e) : (uint64_t)(2u << 20);
    }();
    return v;
}

static bool graphs_enabled() {
    static const bool v = [] {
        const char* e = getenv("MPSW_GRAPHS");
        return !e || atoi(e) != 0;
    }();
    return v;
}

// Graphs pay where a forward is launch-bound: small shards (OPT-1.3B and below: 7-8 % faster).
// For a 25 GB shard the gain is 2 % while each (model, offset, M, B) costs a capture + instantiate
// of ~280 kernels on the host, so large models stay eager. MPSW_GRAPH_MAX_GB overrides (dev).
static uint64_t graph_max_bytes() {
    static const uint64_t v = [] {
        const char* e = getenv("MPSW_GRAPH_MAX_GB");
        return (uint64_t)((e ? atof(e) : 4.0) * (1ull << 30));
    }();
    return v;
}

void issue_batch(mpsw_ctx* c, Rank& R, Entry& e) {
    const FwdShape& s = c->models[e.model]->fs[R.local];
    const int B = e.B, M = e.M;
    const TensorPtrs& Wt = R.wptr[e.model];      // set by this worker when it issued the load
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
    int nl = 0;
    if (R.d_stamp) {                               // debug checks: the model is resident from that load
        launch_check_stamp(R.d_stamp + e.model, e.expect_stamp, R.d_err, cs);
        ++nl;
    }
    uint64_t& point = R.ar_point;                  // persistent: parity alternates across batches
    // Reduce-scatter all-reduce (large M·h·(t-1)): each rank reduces, adds bias + residual and
    // normalises only its own slice of the M rows, then writes that slice's bf16 LN output into
    // every rank's A operand (the all-gather); the fp32 residual stream stays sharded by rows.
    // Per point and rank that moves (t-1)/t·M·h·(4 + 2) bytes instead of (t-1)·M·h·4. Same adds in
    // the same order per element, same LN code: bitwise identical to the direct mode (tested), so
    // the choice may follow M. Not with pipeline stages (the hop needs every row) or taps.
    const bool rs = t > 1 && c->pp == 1 && e.tap.dst == nullptr &&
                    (uint64_t)(t - 1) * M * s.hidden * 4 >= rs_min_bytes();
    const int rs_row0 = (int)((int64_t)M * R.trank / t), rs_rows = (int)((int64_t)M * (R.trank + 1) / t) - rs_row0;
    // all-reduce point: record my partial, barrier with the other TP ranks of my stage, wait for
    // every peer's partial on my stream, then the fused reduce + bias + residual + LN kernel
    // reads all t partials directly (peer / IPC mappings over NVLink).
    auto allreduce_ln = [&](const float* residual, const void* bias, const void* pos_table, const void* g,
                            const void* b) {
        const int pb = point & 1;
        const float* peers[kMaxRanks];
        int fr = r;
        if (c->fault_rank.load() == r && c->fault_rank.compare_exchange_strong(fr, -1))
            throw Error(MPSW_ECUDA, "injected fault (mpsw_test_inject_fault) at an all-reduce point");
        if (t > 1) {
            MPSW_CU(cudaEventRecord(R.ev_point[pb], cs));
            group_barrier(c, R.stage);
            for (int p = 0; p < t; ++p)
                if (g0 + p != r) MPSW_CU(cudaStreamWaitEvent(cs, c->peer_ev[g0 + p][pb], 0));
        }
        for (int p = 0; p < t; ++p) peers[p] = c->peer_partial[g0 + p][pb];
        if (!rs) {
            nl += fwd_reduce_ln(s, M, peers, t, residual, bias, pos_table, pos, g, b, R.ws.x, R.ws.a, cs);
        } else {
            void* outs[kMaxRanks];
            for (int p = 0; p < t; ++p) outs[p] = c->peer_a[g0 + p];
            nl += fwd_reduce_ln_rows(s, rs_row0, rs_rows, peers, t, residual, bias, pos_table, pos, g, b, R.ws.x, outs, t,
                                     cs);
            // every rank's slice must have landed in my A operand before my next GEMM reads it
            MPSW_CU(cudaEventRecord(R.ev_ag[pb], cs));
            group_barrier(c, R.stage);
            for (int p = 0; p < t; ++p)
                if (g0 + p != r) MPSW_CU(cudaStreamWaitEvent(cs, c->peer_ev_ag[g0 + p][pb], 0));
        }
        ++point;
    };
    // verification tap (mpsw_test_tap): stop after e.tap.n_layers layers (X / A) or inside layer
    // n_layers (QKV / O / R); every rank stops at the same point, so the all-reduce points match
    const Tap& tap = e.tap;
    const bool tapping = tap.dst != nullptr;
    bool tapped = false;
    auto tap_copy = [&](const void* src, size_t bytes) {
        if (R.index == tap.rank)
            MPSW_CU(cudaMemcpyAsync(tap.dst, src, std::min<size_t>(bytes, tap.bytes), cudaMemcpyDeviceToHost, cs));
        tapped = true;
    };
    const size_t esz = s.dtype == MPSW_BF16 ? 2 : 4;
    const int hl = s.heads_local * s.head_dim;
    // The compute of this batch (embedding or hop, layers, lm_head kernel). At TP = 1 / PP = 1 it is
    // captured once per (model, range offset, M, B) into a CUDA graph and replayed: one launch
    // instead of ~7 per layer, so small models are not bound by the worker's launch rate. The
    // graph holds device pointers only (weights at the model's range offset, the rank's workspace,
    // tokens / meta already copied in), so a replay computes exactly the captured kernels.
    auto compute = [&]() {
        if (first) {
            nl += fwd_embed(s, Wt, R.ws, M, R.ws.partial[point & 1], cs);
            allreduce_ln(nullptr, nullptr, Wt.embed_pos, Wt.layers[0].ln1_w, Wt.layers[0].ln1_b);
        } else if (!c->cfg.pp_broadcast) {
            // PP hop ("PP communication occurs through FIFO pipes"): this entry came from the
            // same TP rank of the previous stage after it issued the batch, so its hop event for this
            // ring slot is already recorded: wait on it and read that rank's residual stream in place
            // (peer memory over NVLink) into LN1 of my first layer. Slots are reused only after the
            // batch completed everywhere, so batches of different slots overlap across stages (D > 1).
            Rank& P = *c->ranks[c->local_of[r - t]];
            MPSW_CU(cudaStreamWaitEvent(cs, P.ev_hop[e.ring], 0));
            const float* self[1] = {P.hop[e.ring]};
            nl += fwd_reduce_ln(s, M, self, 1, nullptr, nullptr, nullptr, pos, Wt.layers[0].ln1_w, Wt.layers[0].ln1_b,
                                R.ws.x, R.ws.a, cs);
            ++point;
        } else {
            // broadcast ablation (P:96's ruled-out design, D = 1): the entry reached every stage at
            // once, so wait on the host until the previous stage has issued this batch
            Rank& P = *c->ranks[c->local_of[r - t]];
            int spins = 0;
            while (P.stage_out.load(std::memory_order_acquire) < e.id + 1) {
                if (group_poisoned(c)) throw Error(MPSW_ECUDA, "peer failed");
                spin_pause(spins);
            }
            MPSW_CU(cudaStreamWaitEvent(cs, P.ev_stage, 0));
            float* hop = R.ws.partial[point & 1];
            MPSW_CU(cudaMemcpyAsync(hop, P.ws.x, (size_t)M * s.hidden * 4, cudaMemcpyDeviceToDevice, cs));
            const float* self[1] = {hop};
            nl += fwd_reduce_ln(s, M, self, 1, nullptr, nullptr, nullptr, pos, Wt.layers[0].ln1_w, Wt.layers[0].ln1_b,
                                R.ws.x, R.ws.a, cs);
            ++point;
        }
        for (int l = 0; l < s.n_layers; ++l) {
            if (tapping && l == tap.n_layers && tap.what <= MPSW_TAP_A) break;
            const bool tap_here = tapping && l == tap.n_layers;
            const auto& L = Wt.layers[l];
            nl += fwd_qkv(s, L, R.ws, M, cs);
            if (tap_here && tap.what == MPSW_TAP_QKV) { tap_copy(R.ws.qkv, (size_t)M * 3 * hl * 4); break; }
            nl += fwd_attention(s, R.ws, B, cs);
            if (tap_here && tap.what == MPSW_TAP_O) { tap_copy(R.ws.o, (size_t)M * hl * esz); break; }
            nl += fwd_out_proj(s, L, R.ws, M, R.ws.partial[point & 1], cs);
            allreduce_ln(R.ws.x, L.o_b, nullptr, L.ln2_w, L.ln2_b);
            if (tap_here && tap.what == MPSW_TAP_XM) { tap_copy(R.ws.x, (size_t)M * s.hidden * 4); break; }
            if (tap_here && tap.what == MPSW_TAP_F) { tap_copy(R.ws.a, (size_t)M * s.hidden * esz); break; }
            nl += fwd_fc1(s, L, R.ws, M, cs);
            if (tap_here && tap.what == MPSW_TAP_R) { tap_copy(R.ws.r, (size_t)M * s.ffn_local * esz); break; }
            nl += fwd_fc2(s, L, R.ws, M, R.ws.partial[point & 1], cs);
            const bool lastl = l + 1 == s.n_layers;
            // after a non-final stage's last layer only the residual stream matters; the LN output
            // (computed with this layer's LN2 parameters) is unused
            const void* ng = lastl ? (last ? Wt.lnf_w : L.ln2_w) : Wt.layers[l + 1].ln1_w;
            const void* nb = lastl ? (last ? Wt.lnf_b : L.ln2_b) : Wt.layers[l + 1].ln1_b;
            allreduce_ln(R.ws.x, L.fc2_b, nullptr, ng, nb);
        }
        if (last && !tapping) nl += fwd_lm_head(s, Wt, R.ws, B, M, cs);
    };
    const bool graphable = t == 1 && c->pp == 1 && !tapping && graphs_enabled() && c->fault_rank.load() < 0 &&
                           c->models[e.model]->rank_S[R.index] <= graph_max_bytes();
    if (!graphable) {
        compute();
    } else {
        if (R.graphs.size() > 512) {              // bound the cache (shapes x models x offsets)
            for (auto& kv : R.graphs)
                if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
            R.graphs.clear();
        }
        GraphRec& g = R.graphs[GraphKey{e.model, e.off, M, B}];
        if (g.exec) {
            MPSW_CU(cudaGraphLaunch(g.exec, cs));
            nl += g.kernels;
            point += g.points;
        } else if (!g.seen) {                      // first batch of this shape: eager (sets kernel attributes)
            g.seen = true;
            compute();
        } else {
            const int nl0 = nl;
            const uint64_t p0 = point;
            cudaGraph_t graph = nullptr;
            MPSW_CU(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            try {
                compute();
            } catch (...) {
                cudaStreamEndCapture(cs, &graph);
                if (graph) cudaGraphDestroy(graph);
                throw;
            }
            MPSW_CU(cudaStreamEndCapture(cs, &graph));
            MPSW_CU(cudaGraphInstantiate(&g.exec, graph, 0));
            MPSW_CU(cudaGraphDestroy(graph));
            g.kernels = nl - nl0;
            g.points = point - p0;
            // the batch's device span starts at the graph launch, not before the host-side
            // capture and instantiation (which the idle stream would otherwise count)
            MPSW_CU(cudaEventRecord(e.ev_start[r], cs));
            MPSW_CU(cudaGraphLaunch(g.exec, cs));
        }
    }
    if (tapping && !tapped) {
        if (tap.what == MPSW_TAP_X) tap_copy(R.ws.x, (size_t)M * s.hidden * 4);
        else if (tap.what == MPSW_TAP_A) tap_copy(R.ws.a, (size_t)M * s.hidden * esz);
    }
    if (last && !tapping) {
        float* logits_host = (float*)(ring) + (size_t)R.trank * s.vocab_local;
        MPSW_CU(cudaMemcpy2DAsync(logits_host, (size_t)s.vocab * 4, R.ws.logits, (size_t)s.vocab_local * 4,
                                  (size_t)s.vocab_local * 4, B, cudaMemcpyDeviceToHost, cs));
    } else if (!last && !c->cfg.pp_broadcast) {
        // residual stream out through hop slot e.ring (read in place by the next stage)
        MPSW_CU(cudaMemcpyAsync(R.hop[e.ring], R.ws.x, (size_t)M * s.hidden * 4, cudaMemcpyDeviceToDevice, cs));
        MPSW_CU(cudaEventRecord(R.ev_hop[e.ring], cs));
    } else if (!last) {
        MPSW_CU(cudaEventRecord(R.ev_stage, cs));
        R.stage_out.store(e.id + 1, std::memory_order_release);
    }
    MPSW_CU(cudaEventRecord(e.ev_done[r], cs));
    MPSW_CU(cudaEventRecord(R.last_compute[e.model], cs));
    R.last_compute_valid[e.model] = 1;
    c->launches += nl;
}

// Weight pointers of one model's range on one rank, looked up by HF name in that rank's layout (stage-local
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

}  // namespace mpsw
