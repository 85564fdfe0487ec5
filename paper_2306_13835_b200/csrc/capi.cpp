// The C-ABI entry points of include/mpsw.h (argument checking, ctx construction / teardown, and
// the thin request / swap / query calls into the engine).
#include "runtime.h"
#include "../../include/mpsw_testing.h"

#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <fstream>

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

// Frees what a partially constructed ctx holds (mpsw_init error paths, before any thread runs):
// per-rank streams, events and device allocations, fan-in helpers, the shm control segment.
static void release_init_resources(mpsw_ctx* c) {
    for (auto& R : c->ranks) {
        cudaSetDevice(R->device);
        for (cudaStream_t s : {R->compute, R->h2d, R->d2h, R->aux, R->h2d_zc})
            if (s) cudaStreamDestroy(s);
        if (R->ev_zc) cudaEventDestroy(R->ev_zc);
        if (R->ev_base) {
            for (auto& Q : c->ranks)
                if (Q.get() != R.get() && Q->ev_base == R->ev_base) Q->ev_base = nullptr;
            cudaEventDestroy(R->ev_base);
        }
        if (R->region) cudaFree(R->region);
        if (R->d_sum) cudaFree(R->d_sum);
        if (R->d_stamp) cudaFree(R->d_stamp);
        if (R->h_err) cudaFreeHost(R->h_err);
    }
    for (auto& H : c->helpers) {
        cudaSetDevice(H->device);
        if (H->stream) cudaStreamDestroy(H->stream);
        if (H->staging) cudaFree(H->staging);
        for (auto ev : H->free_ev)
            if (ev) cudaEventDestroy(ev);
    }
    if (c->ctl) {
        munmap((void*)c->ctl, sizeof(ShmCtl));
        if (c->leader) shm_unlink(c->shm_name.c_str());
    }
    cudaGetLastError();
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
    if (pp > 1 && cfg->pp_broadcast && cfg->max_inflight_batches > 1)
        return set_error(MPSW_EINVAL, "pp_broadcast (ablation) requires max_inflight_batches = 1");
    if (cfg->max_batch < 1 || cfg->max_batch > 256) return set_error(MPSW_EINVAL, "max_batch must be 1..256");
    if (cfg->max_tokens < 1 || cfg->max_tokens > 128) return set_error(MPSW_EINVAL, "max_tokens must be 1..128");
    if (cfg->dtype != MPSW_BF16 && cfg->dtype != MPSW_FP32) return set_error(MPSW_EINVAL, "bad dtype");
    if (cfg->chunk_bytes % 4096) return set_error(MPSW_EINVAL, "chunk_bytes must be a multiple of 4096");
    if (cfg->swap_mode < 0 || cfg->swap_mode > 3) return set_error(MPSW_EINVAL, "bad swap_mode");
    if (cfg->param_budget_bytes_per_gpu == 0) return set_error(MPSW_EINVAL, "param budget is 0");
    if (cfg->victim_policy < 0 || cfg->victim_policy > 1) return set_error(MPSW_EINVAL, "victim_policy must be 0 or 1");
    if (cfg->gemm_impl < 0 || cfg->gemm_impl > 2)
        return set_error(MPSW_EINVAL, "bad gemm_impl (0 auto, 1 SIMT, 2 tcgen05; the fused layers kernel was removed)");
    if (cfg->n_helpers < 0 || cfg->n_helpers > kMaxHelpers || (cfg->n_helpers && !cfg->helper_device_ids))
        return set_error(MPSW_EINVAL, "n_helpers must be 0..8 with helper_device_ids");
    if (mp && cfg->n_helpers) return set_error(MPSW_EINVAL, "fan-in helpers are single-process only");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        return set_error(MPSW_ECUDA, "no CUDA device");
    }
    // every argument that can be checked without allocating is checked above / here; past this
    // point an error return frees what was allocated (guard), so a failed init leaks nothing
    for (int l = 0; l < cfg->n_gpus; ++l)
        if (cfg->device_ids[l] < 0 || cfg->device_ids[l] >= ndev) return set_error(MPSW_EINVAL, "device id out of range");
    for (int h = 0; h < cfg->n_helpers; ++h)
        if (cfg->helper_device_ids[h] < 0 || cfg->helper_device_ids[h] >= ndev)
            return set_error(MPSW_EINVAL, "helper device id out of range");
    mpsw_config cfg_eff = *cfg;
    if (getenv("MPSW_DEBUG_CHECKS")) cfg_eff.debug_checks = 1;   // enable the race detector in any process
    cfg = &cfg_eff;
    auto c = std::make_unique<mpsw_ctx>();
    struct Guard {
        mpsw_ctx* c;
        bool armed = true;
        ~Guard() {
            if (armed) release_init_resources(c);
        }
    } guard{c.get()};
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
    c->writeback_now.store(cfg->writeback != 0);
    c->chunk = cfg->chunk_bytes ? cfg->chunk_bytes : (64ull << 20);
    c->trace = cfg->trace != 0 && c->leader;
    c->timeline_on = cfg->trace != 0;
    c->device_ids.assign(cfg->device_ids, cfg->device_ids + cfg->n_gpus);
    c->sm.tp = c->nr;              // acks per entry: one per worker
    c->sm.max_batch = cfg->max_batch;
    c->sm.D = c->D;
    c->sm.prefetch = cfg->prefetch != 0;
    c->sm.victim_policy = cfg->victim_policy;
    for (auto& b : c->stage_barrier) b.n = mp ? 1 : c->tp;
    c->models.reserve(kMaxModels);
    for (auto& x : c->local_of) x = -1;
    for (int l = 0; l < cfg->n_gpus; ++l) {
        const int dev = c->device_ids[l];
        if (dev < 0 || dev >= ndev) return set_error(MPSW_EINVAL, "device id out of range");
        c->ranks.push_back(std::make_unique<Rank>());
        Rank* R = c->ranks.back().get();
        R->index = mp ? cfg->world_rank : l;
        R->stage = R->index / cfg->tp;
        R->trank = R->index % cfg->tp;
        R->local = l;
        R->device = dev;
        R->numa = gpu_numa_node(dev);
        R->last_compute.reserve(kMaxModels);
        R->last_compute_valid.reserve(kMaxModels);
        R->wptr.reserve(kMaxModels);
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
        if (cfg->debug_checks) {
            MPSW_CU(cudaMalloc(&R->d_stamp, kMaxModels * sizeof(unsigned long long)));
            MPSW_CU(cudaMemset(R->d_stamp, 0xFF, kMaxModels * sizeof(unsigned long long)));   // kStampEvicted
            MPSW_CU(cudaHostAlloc(&R->h_err, sizeof(unsigned int), cudaHostAllocMapped | cudaHostAllocPortable));
            *R->h_err = 0;
            MPSW_CU(cudaHostGetDevicePointer(&R->d_err, R->h_err, 0));
        }
        if (cfg->trace) {
            // one timeline origin per device, shared by the ranks that live on it
            for (auto& Q : c->ranks)
                if (Q->device == dev) R->ev_base = Q->ev_base;
            if (!R->ev_base) {
                MPSW_CU(cudaEventCreate(&R->ev_base));
                MPSW_CU(cudaEventRecord(R->ev_base, R->compute));
                MPSW_CU(cudaEventSynchronize(R->ev_base));
            }
        }
    }
    for (int h = 0; h < cfg->n_helpers; ++h) {
        const int dev = cfg->helper_device_ids[h];
        if (dev < 0 || dev >= ndev) return set_error(MPSW_EINVAL, "helper device id out of range");
        c->helpers.push_back(std::make_unique<Helper>());
        Helper* H = c->helpers.back().get();
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
    guard.armed = false;
    mpsw_ctx* raw = c.release();
    for (auto& R : raw->ranks) R->th = std::thread(worker_main, raw, R.get());
    raw->engine = std::thread(raw->leader ? engine_main : follower_main, raw);
    if (raw->leader) raw->completer = std::thread(completer_main, raw);
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
    {
        std::lock_guard<std::mutex> lk(c->comp_mu);
        c->comp_stop = true;
    }
    c->comp_cv.notify_all();
    if (c->completer.joinable()) c->completer.join();
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
        for (auto& g : R->gates) cudaEventDestroy(g.ev);
        R->gates.clear();
        for (auto ev : R->ev_point)
            if (ev) cudaEventDestroy(ev);
        for (auto ev : R->ev_ag)
            if (ev) cudaEventDestroy(ev);
        for (auto& kv : R->graphs)
            if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        R->graphs.clear();
        if (R->ev_stage) cudaEventDestroy(R->ev_stage);
        for (auto ev : R->ev_hop) cudaEventDestroy(ev);
        if (R->hop_base) cudaFree(R->hop_base);
        if (R->ev_base) {
            for (auto& Q : c->ranks)
                if (Q.get() != R.get() && Q->ev_base == R->ev_base) Q->ev_base = nullptr;
            cudaEventDestroy(R->ev_base);
            R->ev_base = nullptr;
        }
        for (auto ev : R->last_compute)
            if (ev) cudaEventDestroy(ev);
        cudaFree(R->region);
        cudaFree(R->ws_base);
        cudaFree(R->d_sum);
        if (R->d_stamp) cudaFree(R->d_stamp);
        if (R->h_err) cudaFreeHost(R->h_err);
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
    auto m = std::make_unique<Model>();
    m->dims = *dims;
    for (int g = 0; g < c->nr; ++g) {       // every global rank's shard (stage-dependent)
        Layout L;
        mpsw_status s = compute_layout(*dims, tp, c->pp, g / tp, g % tp, c->cfg.dtype, L);
        if (s != MPSW_OK) return s;
        m->rank_S[g] = L.bytes;
        m->size = std::max(m->size, (L.bytes + kSlotAlign - 1) / kSlotAlign * kSlotAlign);
    }
    {
        std::lock_guard<std::mutex> lk(c->cmd_mu);
        if (!c->geom) {
            const mpsw_opt_dims& x = c->cfg.max_dims;
            const bool given = x.hidden > 0 && x.ffn > 0 && x.vocab > 0 && x.heads > 0;
            check_dims(c, *dims);
            setup_geometry(c, given ? x : *dims);
        }
    }
    check_dims(c, *dims);                   // kernel limits + fits the workspace
    if (m->size > c->cap)
        return set_error(MPSW_ENOMEM, "param budget cannot hold the model (size " + std::to_string(m->size) + " B)");
    if (shards && shard_bytes)
        for (auto& R : c->ranks)
            if (shards[R->index] && shard_bytes[R->index] != m->rank_S[R->index])
                return set_error(MPSW_EINVAL, "shard_bytes != S_r of the layout");
    {   // host-memory preflight: pinning more than the host has would fail late (or swap-thrash)
        uint64_t need = 0;
        for (auto& R : c->ranks) need += m->rank_S[R->index];
        const uint64_t avail = host_mem_available();
        if (avail && need > avail)
            return set_error(MPSW_ENOMEM, "pinned arenas need " + std::to_string(need) + " B of host memory, " +
                                              std::to_string(avail) + " B available (MemAvailable)");
    }
    try {
        for (auto& R : c->ranks) {
            Layout L;
            if (compute_layout(*dims, tp, c->pp, R->stage, R->trank, c->cfg.dtype, L) != MPSW_OK)
                throw Error(MPSW_EINVAL, tls_error());
            m->layout.push_back(L);
            m->fs.push_back(fwd_shape(c, *dims, *R));
            const uint64_t S = m->rank_S[R->index];
            m->arena.push_back(pin_alloc(S, R->numa));
            m->arena_dirty.push_back(0);
            if (shards && shards[R->index]) {
                parallel_memcpy(m->arena.back().p, (const uint8_t*)shards[R->index], S);
                flush_to_memory(m->arena.back().p, S);
            }
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
        R->wptr.emplace_back();
    }
    {
        std::lock_guard<std::mutex> lk(c->cmd_mu);
        std::lock_guard<std::mutex> lk2(c->sm_mu);
        std::lock_guard<std::mutex> lk3(c->f_mu);
        if (c->models.size() >= kMaxModels) return set_error(MPSW_ENOMEM, "too many models");
        const uint64_t size = m->size;
        c->models.push_back(std::move(m));   // capacity reserved at init: no reallocation
        c->sm.add_model(size);
        c->f_off_of.push_back(-1);
        c->load_id_of.push_back(~0ull);
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
    if (host) {
        *host = c->models[model_id]->arena[li].p;
        c->models[model_id]->arena_dirty[li] = 1;   // flushed from the CPU caches before its first load
    }
    if (bytes) *bytes = c->models[model_id]->rank_S[c->ranks[li]->index];
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
            synth_fill_arena(c->models[model_id]->dims, c->tp, c->pp, R->stage, R->trank, c->cfg.dtype, seed,
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
    const mpsw_opt_dims& md = c->models[model_id]->dims;
    if (n_tokens < 1 || n_tokens > c->cfg.max_tokens || n_tokens > md.max_pos)
        return set_error(MPSW_EINVAL, "n_tokens out of range");
    for (int i = 0; i < n_tokens; ++i)
        if (tokens[i] < 0 || tokens[i] >= md.vocab) return set_error(MPSW_EINVAL, "token id out of range");
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

// Region offset of a model that is resident as seen by this process (-1 otherwise).
static int64_t resident_off(mpsw_ctx* c, int model_id) {
    if (c->leader) {
        std::lock_guard<std::mutex> lk(c->sm_mu);
        return c->sm.state[model_id] == ST_RESIDENT ? c->sm.off_of[model_id] : -1;
    }
    std::lock_guard<std::mutex> lk(c->f_mu);
    return c->f_state[model_id] == ST_RESIDENT ? c->f_off_of[model_id] : -1;
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
    const uint64_t S = c->models[model_id]->rank_S[c->ranks[li]->index];
    if (!on_device) {
        *out = host_checksum(c->models[model_id]->arena[li].p, S, 0);
        return MPSW_OK;
    }
    const uint64_t gen0 = c->swap_gen.load();
    const int64_t off = resident_off(c, model_id);
    if (off < 0) return set_error(MPSW_EINVAL, "model not RESIDENT");
    Rank& R = *c->ranks[li];
    MPSW_CU(cudaSetDevice(R.device));
    MPSW_CU(cudaMemsetAsync(R.d_sum, 0, 8, R.aux));
    launch_checksum(R.region + off, S, R.d_sum, R.aux);
    c->launches += 2;
    unsigned long long h = 0;
    MPSW_CU(cudaMemcpyAsync(&h, R.d_sum, 8, cudaMemcpyDeviceToHost, R.aux));
    MPSW_CU(cudaStreamSynchronize(R.aux));
    // a swap dispatched while the kernel read the range may have overwritten it: retry
    if (c->swap_gen.load() != gen0) return set_error(MPSW_EAGAIN, "swap activity during the read; retry");
    *out = h;
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_peek(mpsw_ctx* c, int model_id, int rank, uint64_t offset, uint64_t bytes, void* dst) {
    API_BEGIN
    if (!c || !dst) return set_error(MPSW_EINVAL, "NULL argument");
    if (model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_ENOENT, "unknown model");
    const int li = local_index(c, rank);
    if (li < 0 || offset + bytes > c->models[model_id]->rank_S[c->ranks[li]->index])
        return set_error(MPSW_EINVAL, "rank or range");
    const uint64_t gen0 = c->swap_gen.load();
    const int64_t off = resident_off(c, model_id);
    if (off < 0) return set_error(MPSW_EINVAL, "model not RESIDENT");
    Rank& R = *c->ranks[li];
    MPSW_CU(cudaSetDevice(R.device));
    MPSW_CU(cudaMemcpyAsync(dst, R.region + off + offset, bytes, cudaMemcpyDeviceToHost, R.aux));
    MPSW_CU(cudaStreamSynchronize(R.aux));
    if (c->swap_gen.load() != gen0) return set_error(MPSW_EAGAIN, "swap activity during the read; retry");
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_set_writeback(mpsw_ctx* c, int writeback) {
    API_BEGIN
    if (!c) return set_error(MPSW_EINVAL, "NULL ctx");
    if (need_leader(c) != MPSW_OK) return MPSW_EINVAL;
    c->writeback_now.store(writeback != 0);
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_test_inject_fault(mpsw_ctx* c, int rank) {
    API_BEGIN
    if (!c || c->mp || rank < 0 || rank >= c->nr) return set_error(MPSW_EINVAL, "bad ctx / rank (single-process only)");
    c->fault_rank.store(rank);
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_test_corrupt_stamp(mpsw_ctx* c, int model_id) {
    API_BEGIN
    if (!c || model_id < 0 || model_id >= (int)c->models.size()) return set_error(MPSW_EINVAL, "bad ctx / model");
    if (!c->cfg.debug_checks) return set_error(MPSW_EINVAL, "debug_checks is off");
    for (auto& R : c->ranks) {
        MPSW_CU(cudaSetDevice(R->device));
        const unsigned long long bogus = 0x5EEDull;
        MPSW_CU(cudaMemcpy(R->d_stamp + model_id, &bogus, sizeof(bogus), cudaMemcpyHostToDevice));
    }
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_test_tap(mpsw_ctx* c, int n_layers, int what, int rank, void* dst, uint64_t bytes) {
    API_BEGIN
    if (!c || !dst || !bytes) return set_error(MPSW_EINVAL, "NULL argument");
    if (c->mp || c->pp != 1) return set_error(MPSW_EINVAL, "tap: single-process ctx with pp = 1 only");
    if (what < MPSW_TAP_X || what > MPSW_TAP_F || n_layers < 0 || rank < 0 || rank >= c->nr)
        return set_error(MPSW_EINVAL, "tap: bad what / n_layers / rank");
    std::lock_guard<std::mutex> lk(c->tap_mu);
    c->tap_next = Tap{n_layers, what, rank, dst, bytes};
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
    {
        std::lock_guard<std::mutex> sl(c->sm_mu);
        f << "{\"cfg\":{\"cap\":" << c->sm.cap << ",\"sizes\":[";
        for (int m = 0; m < c->sm.n_models; ++m) f << (m ? "," : "") << c->sm.size[m];
        f << "],\"acks\":" << c->sm.tp << ",\"max_batch\":" << c->sm.max_batch << ",\"D\":" << c->sm.D
          << ",\"prefetch\":" << (c->sm.prefetch ? "true" : "false") << ",\"victim_policy\":" << c->sm.victim_policy
          << "}}\n";
    }
    for (const auto& l : c->trace_lines) f << l << "\n";
    return MPSW_OK;
    API_END
}

mpsw_status mpsw_timeline_dump(mpsw_ctx* c, const char* path) {
    API_BEGIN
    if (!c || !path) return set_error(MPSW_EINVAL, "NULL argument");
    if (!c->timeline_on) return set_error(MPSW_EINVAL, "timeline disabled (cfg.trace = 0)");
    std::lock_guard<std::mutex> lk(c->trace_mu);
    std::ofstream f(path);
    if (!f) return set_error(MPSW_EINVAL, "cannot open timeline path");
    for (const auto& l : c->timeline) f << l << "\n";
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
    o->k_slots = c->models.empty() ? 0 : (int)(c->cap / c->models[0]->size);
    o->shard_bytes = c->models.empty() ? 0 : c->models[0]->rank_S[0];
    o->region_bytes = c->cap;
    o->prefetches = c->prefetches.load();
    o->fwd_gpu_us_sum = c->fwd_us_sum.load();
    o->fwd_gpu_n = c->fwd_n.load();
    o->numa_requested = o->numa_verified = 0;
    for (auto& m : c->models)
        for (auto& a : m->arena) {
            o->numa_requested += a.numa >= 0;
            o->numa_verified += a.numa_ok;
        }
    return MPSW_OK;
    API_END
}

}  // extern "C"
