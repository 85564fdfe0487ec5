/*
 * mpsw.h — model-parallel swapping (Computron, arXiv 2306.13835) on B200: the C-ABI boundary.
 *
 * One mpsw_ctx is one single-process deployment of ONE tensor-parallel group of t ranks
 * (§3.1 P:72 "Workers are launched per GPU"; every model instance uses the same
 * parallel configuration). Inside the library there is one engine thread (the paper's
 * centralised engine) and one worker thread per rank. Each rank owns:
 *   - a parameter region of `param_budget_bytes_per_gpu` bytes in HBM, allocated ONCE at
 *     mpsw_init; models are placed in it first-fit (readings #8, #28; equal-size
 *     models: k = floor(budget / S_r) slots);
 *   - a compute stream plus two copy streams, load (H2D) and offload (D2H) ("two
 *     additional streams to run loading and offloading operations concurrently");
 *   - page-locked host arenas, one contiguous blob per (model, rank) ("the parameters
 *     are kept pinned in CPU memory").
 * Ranks map to CUDA devices through `device_ids`; repeated ids are allowed and give
 * "virtual ranks" that share one GPU (used to test TP > 1 semantics on a single B200).
 *
 * Multi-process mode (one process per GPU, e.g. under torchrun): set world_size = t > 1,
 * world_rank, shm_name and n_gpus = tp = 1 (this process's rank). Rank 0 is the LEADER: it runs
 * the engine (the only place requests / explicit swaps are accepted) and publishes every
 * decision to a POSIX shared-memory control plane (`shm_name`); ranks 1..t-1 are FOLLOWERS that
 * execute the published entries on their GPU and post per-rank acks back through the same
 * segment ("sends a response back to the engine"). The TP all-reduce of the forward reads
 * peer partials through CUDA IPC mappings (NVLink). mpsw_init, the FIRST mpsw_register_model,
 * every mpsw_register_model (same order on every rank) and mpsw_shutdown are collective.
 *
 * Every call returns mpsw_status (0 = OK, < 0 = error) and never throws across the ABI.
 * On error, mpsw_last_error() returns a thread-local message describing the failure.
 * Pointers are plain host pointers unless stated otherwise; sizes are bytes.
 * Thread safety: all calls may be made from any host thread; calls on one ctx are
 * serialised internally except mpsw_wait / mpsw_poll which only read completion state.
 */
#ifndef MPSW_H
#define MPSW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MPSW_OK = 0,
    MPSW_EINVAL = -1,      /* bad argument / unsupported configuration               */
    MPSW_ENOMEM = -2,      /* budget cannot hold one shard; pinning or cudaMalloc failed      */
    MPSW_EBUSY = -3,       /* swap_out of a model with in-flight batches or a pending load    */
    MPSW_ENOENT = -4,      /* unknown model / ticket / request id              */
    MPSW_EAGAIN = -5,      /* not finished yet (poll/wait with timeout)                       */
    MPSW_ECUDA = -6,       /* a CUDA runtime call failed; ctx is poisoned                     */
    MPSW_ENCCL = -7,       /* reserved: collective backend failure                            */
    MPSW_EINVARIANT = -8,  /* engine invariant violated; ctx poisoned   */
    MPSW_ETIMEDOUT = -9    /* mpsw_wait timed out                                             */
} mpsw_status;

enum { MPSW_BF16 = 0, MPSW_FP32 = 1 };                                 /* parameter/compute dtype */
enum { MPSW_SWAP_AUTO = 0, MPSW_SWAP_COPY_ENGINE = 1, MPSW_SWAP_ZERO_COPY = 2,
       MPSW_SWAP_HYBRID = 3 /* ablation: CE head + zero-copy tail of one shard concurrently */ };
enum { MPSW_EVICTED = 0, MPSW_LOADING = 1, MPSW_RESIDENT = 2, MPSW_OFFLOADING = 3 };

typedef struct mpsw_ctx mpsw_ctx;   /* opaque; owns arenas, the region, streams, threads */

/* OPT shape (HF OPTConfig: num_hidden_layers, hidden_size, num_attention_heads, ffn_dim,
 * vocab_size, max_position_embeddings) */
typedef struct { int n_layers, hidden, heads, ffn, vocab, max_pos; } mpsw_opt_dims;

typedef struct {
    int n_gpus;                   /* ranks driven by THIS process (tp*pp, or 1 in multi-process) */
    const int* device_ids;        /* n_gpus CUDA ordinals (caller-owned, read during init)     */
    int tp;                       /* TP degree t: tp * pp == n_gpus, or tp == world_size       */
    uint64_t param_budget_bytes_per_gpu;  /* parameter region per rank (the swapping budget)   */
    uint64_t workspace_bytes_per_gpu;     /* 0 = auto (activations, partials, logits staging)  */
    int max_batch;                /* requests per batch entry, 1..256 (P:168 uses 8, P:196 32) */
    int max_tokens;               /* tokens per request, 1..128 (P:138 uses 2, P:166 uses 8)   */
    int dtype;                    /* MPSW_BF16 (1e-2 parity) or MPSW_FP32 (1e-5 parity)        */
    int max_inflight_batches;     /* D per TP group (reading #26); 0 => 1            */
    int swap_mode;                /* MPSW_SWAP_*: copy engine, zero-copy kernel, hybrid, or    */
                                  /* auto = the measured winner per shard-size bucket (the copy */
                                  /* engine at every size once arenas are clean) */
    uint64_t chunk_bytes;         /* swap chunk c (multiple of 4096); 0 => 64 MiB              */
    int writeback;                /* 1 = offload copies the slot back to the arena      */
    int trace;                    /* 1 = record the NDJSON event/decision trace                */
    int zc_ctas;                  /* CTAs of the zero-copy kernel; 0 => auto                   */
    int world_size;               /* processes in the TP group; 0/1 = single-process mode      */
    int world_rank;               /* this process's TP rank (0 = leader)                       */
    const char* shm_name;         /* POSIX shm name for the control plane, e.g. "/mpsw_1234"   */
    int gemm_impl;                /* 0 auto (tcgen05/TMA kernels for bf16, M > 256 in 256-row
                                     chunks), 1 SIMT (fp32 FMA), 2 tcgen05; 0 and 2 are identical.
                                     (3, the round-1 fused layers kernel, was removed: EINVAL) */
    int pp;                       /* pipeline stages (0/1 = none); ranks = tp * pp, global rank  */
                                  /* g = stage * tp + tp_rank; single-process only. Entries are */
                                  /* pipelined stage to stage (NEXT-1): the engine feeds */
                                  /* stage 0; each worker forwards an entry to the next stage   */
                                  /* right after issuing it (loads without waiting for the copy)*/
                                  /* and batches overlap across stages for D > 1                 */
    const int* helper_device_ids; /* NVLink fan-in (NEXT-2; single process): GPUs whose PCIe    */
    int n_helpers;                /* links also pull chunks of every swap-in and forward them   */
                                  /* to the owner over NVLink; 0 = off (copy-engine mode only)  */
    mpsw_opt_dims max_dims;
                                  /* heterogeneous models (NEXT-4): the forward workspace is     */
                                  /* sized for hidden/ffn/vocab up to these; all zero = the dims */
                                  /* of the first registered model (later ones must not exceed)  */
    int prefetch;                 /* 1 = prefetch predicted models into free space while no swap  */
                                  /* is in flight (NEXT-3, reading #29); never evicts  */
    int pp_broadcast;             /* pp > 1 ablation: 1 = the engine hands every entry to every  */
                                  /* worker at once (the design P:96 rules out); needs D = 1     */
    int victim_policy;            /* no free range for a load: 0 = evict LRU victims until a     */
                                  /* first fit appears (reading #28); 1 = the window that evicts */
                                  /* the fewest bytes (knapsack, reading #30, NEXT-4)            */
    int debug_checks;             /* 1 = device-side residency check (race detection): each load */
                                  /* stamps its entry id into a per-rank device word of the     */
                                  /* model after its copies, each offload stamps "evicted", and */
                                  /* every forward first checks that the stamp is the load the  */
                                  /* engine gated it on; a mismatch poisons the ctx (EINVARIANT)*/
                                  /* (env MPSW_DEBUG_CHECKS=1 turns it on for any ctx)          */
} mpsw_config;

typedef struct {
    char name[64];                /* HF parameter name, e.g. "decoder.layers.3.fc1.weight"    */
    uint64_t offset, bytes;       /* byte range inside the rank's arena (offset % 256 == 0)    */
    int rows, cols;               /* shard shape (cols == 1 for vectors)                      */
    int split;                    /* 0 replicated, 1 row-block (column-parallel / vocab),     */
                                  /* 2 column-block (row-parallel), reading #12 */
    int tensor_id;                /* index in the full model's canonical tensor list (C0 key) */
} mpsw_tensor_desc;

/* Create a ctx. Allocates each rank's parameter region (one cudaMalloc of the budget) and
 * workspace, creates streams and starts the engine and worker threads.
 * Errors: EINVAL (tp inconsistent with n_gpus/world_size, bad sizes), ENOMEM (cudaMalloc),
 * ECUDA, ETIMEDOUT (multi-process: peers did not join the shm control plane within 120 s). */
mpsw_status mpsw_init(const mpsw_config* cfg, mpsw_ctx** out);

/* Wait for all in-flight work, stop threads, free every arena, slot, stream. NULL is OK. */
mpsw_status mpsw_shutdown(mpsw_ctx* ctx);

/* Pure function (no ctx, no GPU): the arena layout of TP rank `rank` of pipeline stage `stage`
 * of an OPT model at TP degree `tp` and PP degree `pp` (P:138 every TP shard
 * keeps all tensors of its stage; stage s holds layers [s*L/pp, (s+1)*L/pp), stage 0 the
 * embeddings, the last stage the final LayerNorm and a copy of embed_tokens for the tied
 * lm_head). Writes up to `cap` descriptors to `out` (may be NULL), the tensor count to *n and
 * the arena size to *shard_bytes. `dtype` MPSW_BF16 (2-byte elements) or MPSW_FP32.
 * EINVAL if tp does not divide heads, vocab, ffn and hidden, or pp does not divide n_layers. */
mpsw_status mpsw_shard_layout(const mpsw_opt_dims* dims, int tp, int pp, int stage, int rank, int dtype,
                              mpsw_tensor_desc* out, int cap, int* n, uint64_t* shard_bytes);

/* Register a model (P:72 co-located instances). `tp` must equal the ctx's. `shards` is an
 * array of tp caller-owned host blobs in the mpsw_shard_layout format, each of
 * shard_bytes[r] == S_r bytes; they are COPIED into library-owned pinned arenas before
 * return. shards == NULL allocates the arenas and leaves them for in-place filling via
 * mpsw_model_arena / mpsw_synth_fill. Models may differ in size (NEXT-4, §6): every rank's
 * region of budget bytes holds each resident model in one range of size(m) = max_r S_r(m)
 * rounded up to 4 KiB, at the same offset on every rank, placed first-fit (DESIGN.md reading
 * #28); equal-size models reduce to k = floor(budget / size) slots. hidden, ffn and vocab must
 * not exceed mpsw_config.max_dims (or the first registered model's). The model starts EVICTED.
 * Errors: EINVAL (dims/tp/sizes, or beyond the workspace dims), ENOMEM (budget < size(m), or
 * pinning failed). */
mpsw_status mpsw_register_model(mpsw_ctx* ctx, const mpsw_opt_dims* dims, int tp,
                                const void* const* shards, const uint64_t* shard_bytes,
                                int* model_id);

/* Host pointer and size of (model, rank)'s pinned arena, for in-place filling before the
 * first swap-in. Writing it while the model is LOADING/OFFLOADING is undefined. The arena is
 * written back from the CPU caches (clflushopt) before its next load: a copy-engine read of
 * lines still dirty in the CPU's L3 runs at 1/3 - 1/5 of the link rate. */
mpsw_status mpsw_model_arena(mpsw_ctx* ctx, int model_id, int rank, void** host, uint64_t* bytes);

/* Input-generation helper (not the hot path): fill (model, rank)'s arena with the
 * counter-based synthetic weights of DESIGN.md §Inputs (C0) for `model_seed`, using
 * `threads` host threads (0 = all). rank = -1 fills every rank. */
mpsw_status mpsw_synth_fill(mpsw_ctx* ctx, int model_id, int rank, uint64_t model_seed, int threads);

/* Multi-process mode: mpsw_request / mpsw_swap_in / mpsw_swap_out / mpsw_trace_dump are
 * accepted on the leader only (EINVAL on followers); mpsw_checksum / mpsw_peek / mpsw_wait /
 * mpsw_entry_gpu_ms / mpsw_residency act on the calling process's rank. */

/* Explicit load entry: asynchronously copy every rank's shard into the lowest free
 * range of the region that fits it. Goes through the engine queue, ordered with requests.
 * *ticket identifies the entry. OK with an already-complete ticket if RESIDENT or LOADING
 * (no-op). ENOMEM if no free range fits (explicit swaps never evict), EBUSY if OFFLOADING. */
mpsw_status mpsw_swap_in(mpsw_ctx* ctx, int model_id, uint64_t* ticket);

/* Explicit offload entry: write the model's range back to the arena (writeback=1), free it.
 * EBUSY if the model has in-flight batches or is LOADING (eviction never races a request).
 * OK no-op if EVICTED/OFFLOADING. */
mpsw_status mpsw_swap_out(mpsw_ctx* ctx, int model_id, uint64_t* ticket);

/* Offload semantics of the offload decisions the engine makes from now on (explicit and LRU):
 * 1 = writeback (D2H copy of the range into the arena, chunk-paired with the next load, reading
 * #5/#6), 0 = clean eviction (no copy; weights are immutable, NEXT-3). Initial
 * value: mpsw_config.writeback. Entries already dispatched keep theirs; the flag travels with
 * each offload entry to every rank (shm record in multi-process mode). Leader only (EINVAL). */
mpsw_status mpsw_set_writeback(mpsw_ctx* ctx, int writeback);

/* Block until every rank acked `ticket` ("completed when every worker finishes").
 * t_submit: engine time of the decision; t_done_per_rank: array of tp ack times (may be
 * NULL). Times are seconds since mpsw_init (steady clock). timeout_s < 0 waits forever.
 * A completed ticket stays queryable (here and in mpsw_entry_gpu_ms) until 4096 newer swap
 * entries have completed; older tickets are released (ENOENT), bounding the entry history.
 * Errors: ENOENT unknown ticket, ETIMEDOUT. */
mpsw_status mpsw_wait(mpsw_ctx* ctx, uint64_t ticket, double timeout_s, double* t_submit,
                      double* t_done_per_rank);

/* Per-rank device time of a swap entry's copies, from CUDA events on the copy stream
 * (ms, array of tp), plus entry kind (0 load, 1 offload) and model. EAGAIN if not done. */
mpsw_status mpsw_entry_gpu_ms(mpsw_ctx* ctx, uint64_t ticket, int* kind, int* model_id,
                              float* gpu_ms_per_rank);

/* Submit a request (pushed with a timestamp into the model's queue). The engine
 * batches it with other queued requests of the model (oldest first, <= max_batch), swaps
 * the model in via LRU if needed, runs the TP forward and writes the fp32 logits
 * of the LAST token ([vocab] floats) to logits_out, which must stay valid until mpsw_poll
 * returns OK. tokens are copied before return.
 * Errors: ENOENT unknown model (counted), EINVAL n_tokens not in [1, max_tokens] or a
 * token outside [0, vocab). */
mpsw_status mpsw_request(mpsw_ctx* ctx, int model_id, const int32_t* tokens, int n_tokens,
                         float* logits_out, int64_t* request_id);

/* OK once the request's logits are in logits_out (t_arrival, t_done in engine seconds);
 * EAGAIN while pending; ENOENT unknown id. The id is released after the first OK (a later
 * poll/wait of the same id returns ENOENT). */
mpsw_status mpsw_poll(mpsw_ctx* ctx, int64_t request_id, double* t_arrival, double* t_done);

/* Blocking variant of mpsw_poll (timeout_s < 0 = forever). */
mpsw_status mpsw_wait_request(mpsw_ctx* ctx, int64_t request_id, double timeout_s,
                              double* t_arrival, double* t_done);

/* 64-bit order-independent checksum (C4) of (model, rank)'s bytes:
 * on_device = 1 hashes the resident range with the sm_100a checksum kernel (EINVAL unless
 * RESIDENT); on_device = 0 hashes the pinned host arena on the host. EAGAIN (retry) if a swap
 * entry was dispatched while the device range was being read: the bytes may have been changing,
 * so no hash is returned. (mpsw_peek: same rule.) */
mpsw_status mpsw_checksum(mpsw_ctx* ctx, int model_id, int rank, int on_device, uint64_t* out);

/* Copy `bytes` at `offset` of a RESIDENT model's device range (rank) into host `dst`
 * (verification: sampled parity against the oracle). */
mpsw_status mpsw_peek(mpsw_ctx* ctx, int model_id, int rank, uint64_t offset, uint64_t bytes,
                      void* dst);

/* MPSW_EVICTED / LOADING / RESIDENT / OFFLOADING as seen by the engine. */
mpsw_status mpsw_residency(mpsw_ctx* ctx, int model_id, int* state);

/* Write the recorded events and decisions, in engine order, as NDJSON (trace = 1). The first
 * line is {"cfg": {"cap", "sizes", "acks", "max_batch", "D", "prefetch"}}: the state machine's
 * configuration (region bytes, placement bytes per model, acks per entry), enough to replay
 * the log through the oracle scheduler. Decisions: {"dec": "load"|"offload", "id", "model",
 * "off"} (byte offset in every rank's region; prefetch loads add "prefetch": true),
 * {"dec": "batch"|"complete", "id", "rids"}, ... */
mpsw_status mpsw_trace_dump(mpsw_ctx* ctx, const char* ndjson_path);

/* Write this process's device timeline as NDJSON (trace = 1): one line per finished entry per
 * local rank, {"kind": "load"|"offload"|"batch", "id", "model", "rank", "device", "t0_ms",
 * "t1_ms"}, times from CUDA events relative to one origin event per device (so spans of the
 * ranks that share a GPU are comparable: evidence of swap / forward overlap). */
mpsw_status mpsw_timeline_dump(mpsw_ctx* ctx, const char* ndjson_path);

typedef struct {
    uint64_t kernel_launches;     /* kernels this library launched (all ranks)              */
    uint64_t h2d_bytes, d2h_bytes;/* bytes moved by swaps                                   */
    uint64_t swaps_in, swaps_out; /* load / offload entries completed                       */
    uint64_t batches, requests;   /* batch entries / requests completed                     */
    uint64_t rejected;            /* requests rejected with ENOENT                          */
    int k_slots;                  /* floor(region / size(model 0)): the slot count for      */
                                  /* equal-size models (0 before the first registration)    */
    uint64_t shard_bytes;         /* S_r of model 0 on rank 0                               */
    uint64_t fwd_gpu_us_sum;      /* sum of per-batch forward device time (first local rank) */
    uint64_t fwd_gpu_n;           /* batches in that sum                                    */
    uint64_t region_bytes;        /* parameter region per rank (budget rounded down to 4 KiB) */
    uint64_t prefetches;          /* load entries issued by the prefetch policy               */
    uint64_t numa_requested;      /* pinned arenas bound (mbind) to their GPU's NUMA node      */
    uint64_t numa_verified;       /* ...of which sampled pages are resident on that node      */
                                  /* (move_pages); MPSW_NUMA_NODE=n forces node n (tests)      */
} mpsw_stats;

mpsw_status mpsw_get_stats(mpsw_ctx* ctx, mpsw_stats* out);

/* Thread-local description of the last error on this thread ("" if none). */
const char* mpsw_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MPSW_H */
