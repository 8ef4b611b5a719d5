/* psattn_b200.h — device-batched extensions of the PSA C ABI (B200, sm_100a).
 *
 * psattn.h keeps the reference's one-query-at-a-time entry points. A serving
 * loop (reference serving.cpp:161-202 drives psa_attention_batched /
 * topk_attention once per layer per decode step) needs instead ONE stream-ordered
 * launch covering every (request, layer, q-head) of a step with no host
 * round-trip per microbatch. That is what this header adds (SURVEY §8b
 * "What the replacement adds"):
 *
 *   - psattn_pool_*   a unified paged KV block pool in HBM shared by all
 *                     layers (reference TieredBlockStore's Unified policy,
 *                     store.cpp:11-22) with per-slot metadata built on device
 *                     (reference build_metadata, metadata.cpp:8-34);
 *   - psattn_run_batch  scoring (criticality_score, metadata.cpp:41-72),
 *                     ordering (rank_by_scores, metadata.cpp:87-96) and the
 *                     progressive early-terminating loop (engine.cpp:92-171,
 *                     211-231, 240-260) for a whole batch, launched on the
 *                     caller's cudaStream_t.
 * The synthetic workload generator of the benchmark and the tests is a separate
 * fixture library (workload/psattn_synth.h), not part of this one.
 *
 * All pointers in psattn_batch are DEVICE pointers unless stated. Streams are
 * passed as void* (a cudaStream_t), NULL = legacy default stream.
 */
#ifndef PSATTN_B200_H
#define PSATTN_B200_H

#include <stddef.h>
#include <stdint.h>

#include "psattn.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { PSATTN_KV_F32 = 0, PSATTN_KV_BF16 = 1 };

typedef struct psattn_pool psattn_pool;

typedef struct {
    int32_t dim;          /* head dimension d (1..256) */
    int32_t block_tokens; /* tokens per slot B (1..32) */
    int32_t kv_dtype;     /* PSATTN_KV_* */
    int32_t reserved;
    int64_t n_slots;      /* slot capacity */
} psattn_pool_desc;

/* Raw device layout, for callers that write K/V themselves (e.g. a decode
 * step's KV append) and then call psattn_pool_build_metadata. Rows past a
 * slot's ntok must hold finite values (the pool is zero-initialised and every
 * put writes zero padding): the progressive kernel loads all rows of a slot
 * and masks by ntok. */
typedef struct {
    void* kv;            /* [n_slots][2][block_tokens][dim] kv_dtype: K rows then V rows */
    void* meta;          /* [n_slots] records of {mean[dim] f32, lo[dim] kv, hi[dim] kv} */
    int32_t* ntok;       /* [n_slots] valid tokens per slot */
    int64_t slot_bytes;  /* bytes per KV slot */
    int64_t meta_bytes;  /* bytes per metadata record */
} psattn_pool_layout;

int psattn_pool_create(const psattn_pool_desc* desc, psattn_pool** out_pool);
void psattn_pool_destroy(psattn_pool* pool);
int psattn_pool_get_desc(const psattn_pool* pool, psattn_pool_desc* out);
int psattn_pool_get_layout(const psattn_pool* pool, psattn_pool_layout* out);

/* Host fp32 K/V ([n][block_tokens][dim] each, rows past ntok[i] ignored) into
 * slots[i] (host array), then builds their metadata. Synchronous. */
int psattn_pool_put_blocks(psattn_pool* pool, int64_t n, const int32_t* slots, const int32_t* ntok,
                           const float* keys, const float* values);

/* Rebuilds metadata (lo/hi/mean) for slots [slot_begin, slot_end) on device. */
int psattn_pool_build_metadata(psattn_pool* pool, int64_t slot_begin, int64_t slot_end, void* stream);

/* Decode-step KV append + metadata maintenance (the step right before the path
 * every decode step): for i < n, writes one token's K and V (device fp32 [n][dim]
 * each) at row ntok of slot tail_slots[i] (device int32 [n]), increments ntok and
 * rebuilds that slot's metadata on `stream` (reference put_block/build_metadata,
 * store.cpp:59-78, metadata.cpp:8-34). A slot already holding block_tokens rows is
 * left untouched and *status (device int32, caller-zeroed) is set to 1: the caller
 * opens a new slot for that sequence. */
int psattn_pool_append_tokens(psattn_pool* pool, int32_t n, const int32_t* tail_slots, const float* keys,
                              const float* values, int32_t* status, void* stream);

/* Copies back metadata of one slot as fp32 (mean, lo, hi: dim floats each). */
int psattn_pool_read_metadata(psattn_pool* pool, int64_t slot, float* mean, float* lo, float* hi);

/* ---- Multi-head (GQA) progressive attention through the store (C form of the reference's
 * psattn::psa_attention_multi_head, include/psattn/engine.hpp:160-170, engine.cpp:240-260) ----
 * q: [n_q_heads][dim] host floats; q-head h reads kv-head list h / (n_q_heads / n_kv_heads);
 * list k = block_ids[list_off[k] .. list_off[k+1]) (host arrays, n_kv_heads + 1 offsets).
 * out: [n_q_heads][dim]; out_stats: NULL or n_q_heads entries; out_union: NULL or the number of
 * distinct blocks fetched by any head (MultiHeadResult::fetched_union). One device launch for
 * all heads; store accounting and miss latency as the reference's per-head calls. */
int psattn_run_multi_head(psattn_store* store, const float* q, int32_t n_q_heads, int32_t dim,
                          const int64_t* block_ids, const int64_t* list_off, int32_t n_kv_heads,
                          const psattn_config* cfg, float* out, psattn_run_stats* out_stats, int64_t* out_union);

/* ---- Batched progressive attention ---- */

typedef struct {
    /* shape */
    int32_t n_units;       /* independent (request, layer, kv-head) block lists */
    int32_t group;         /* q-heads per kv-head (GQA group g), 1..8 */
    int32_t dim;           /* must equal the pool's dim */
    int32_t max_blocks;    /* max list length over units (host-known) */
    int64_t total_blocks;  /* list_off[n_units] (host-known) */
    /* inputs (device) */
    const float* q;            /* [n_units][group][dim] */
    const int32_t* slots;      /* page table: unit u's list = slots[list_off[u] .. list_off[u+1]) */
    const int64_t* list_off;   /* [n_units + 1] */
    /* Lists are in ascending block-id order (a page table's natural order), so
       the reference's tie rule "score desc, block_id asc" is list position asc. */
    /* config (reference psattn_config semantics) */
    double epsilon;
    int32_t microbatch_size;
    int32_t estimator;         /* PSATTN_EST_* */
    int32_t ranking_mode;      /* PSATTN_RANK_* */
    int32_t audit_coverage;
    double scale_override;
    int64_t topk;              /* 0: PSA threshold stop; >0: top-k budget (epsilon forced to 1) */
    /* outputs (device) */
    float* out;                /* [n_units][group][dim] */
    int64_t* blocks_processed; /* [n_units*group] */
    double* est_coverage;      /* [n_units*group] */
    double* true_coverage;     /* optional [n_units*group]; -1 without audit */
    int32_t* terminated;       /* [n_units*group] */
    /* optional output: rank-ordered list positions per head, at
       ranked_pos[list_off[u]*group + h*n_u + r], defined for r < blocks_processed
       (psattn_rank_batch fills every rank). NULL = kept in workspace. */
    int32_t* ranked_pos;
    /* optional output [total_blocks*group], same indexing: at every microbatch
       boundary rank r that was evaluated, the coverage estimate after rank r. */
    double* iter_est;
} psattn_batch;

/* Full ranking of every head of the batch (plan_blocks' ranked_ids, reference engine.cpp:57-90;
 * rank_by_scores order, metadata.cpp:87-96): every n_u rank of every head into ranked_pos (or the
 * workspace's rank array when NULL), descending score with ties by ascending block id (list
 * position), exactly; fp64 oracle masses computed into the workspace for Oracle ranking / audit.
 * No attention outputs are written. psattn_run_batch instead orders only the ranks it consumes:
 * its ranked_pos / iter_est entries are defined for ranks < blocks_processed. Same workspace size. */
int psattn_rank_batch(psattn_pool* pool, const psattn_batch* b, void* workspace, void* stream);

/* Workspace bytes psattn_run_batch needs for this batch shape. */
size_t psattn_batch_workspace_bytes(const psattn_batch* b);

/* One stream-ordered launch sequence (score -> order -> progressive), no host
 * synchronisation. workspace: device memory of psattn_batch_workspace_bytes. */
int psattn_run_batch(psattn_pool* pool, const psattn_batch* b, void* workspace, void* stream);

/* CUDA-graph capture of one decode step: psattn_run_batch on (pool, b, workspace) recorded once
 * (relaxed stream capture on `stream`, or an internal stream when NULL) and replayed by
 * psattn_graph_launch on any stream, re-reading the same device buffers (queries, page tables)
 * at every replay: the serving loop refreshes q / slots in place and replays. */
typedef struct psattn_graph psattn_graph;
int psattn_graph_create(psattn_pool* pool, const psattn_batch* b, void* workspace, void* stream, psattn_graph** out);
int psattn_graph_launch(psattn_graph* g, void* stream);
void psattn_graph_destroy(psattn_graph* g);

/* Per-unit count of distinct blocks processed by any head of the group (the
 * GQA union the algorithmic byte count uses), after psattn_run_batch on the
 * same stream and workspace. out_union: device int64 [n_units]. */
int psattn_batch_union_blocks(const psattn_batch* b, void* workspace, int64_t* out_union, void* stream);

/* Number of kernels the last psattn_run_batch launched on this process. */
int psattn_batch_last_launches(int32_t* out_count);

/* Progressive-kernel selection (tuning/testing knob): 0 = auto (the warp-specialised
 * stream kernel on the production shape — bf16 HBM pool, dim 128, 16-token blocks,
 * 2 <= group <= 4, dense hand-over on; else the GQA round kernel — one CTA per kv-head
 * list, K/V of the group's union read once — when 2 <= group <= 4, dim in {64,128} and
 * blocks <= 16 tokens; else one CTA per q-head), 1 = always per q-head, 2 = GQA round
 * kernel whenever supported, 3 = stream kernel whenever supported. */
int psattn_set_progressive_kernel(int32_t mode);
/* Benchmark instrumentation of the stream kernel: K tiles fetched, V tiles fetched,
 * rounds decided and units run since the last call (device counters; reading zeroes
 * them). Returns 0, or -1 on a CUDA error. */
int psattn_debug_stream_stats(unsigned long long* out4);
/* Development builds (make EXTRA=-DPSA_STREAM_PROF) only: per role of the stream kernel (producer,
 * decider, scorers, V; summed over warps) total cycles, cycles in wait sites 1-5, producer idle /
 * productive iterations; reading zeroes them. All zero in normal builds. */
int psattn_debug_stream_prof(unsigned long long* out32);
/* Development builds (make PROF=1) only: SM cycles per phase of the GQA round kernel
 * (init, order, union, K pass, decide, V pass, advance, finalize, rounds, 3 warp-0
 * counters); reading zeroes them. -1 in normal builds. */
int psattn_debug_gqa_phases(unsigned long long* out12);
/* Development builds (make STREAM_DEBUG=1) only: attaches a mapped host buffer that collects
 * stuck-wait records of the stream kernel (int[16 + 16*256]: count, then 16-int records) and
 * returns it; nullptr in normal builds. */
int* psattn_debug_stream_attach(void);
/* Score/progressive overlap: psattn_run_batch splits a batch of >= 512 units into
 * sub-batches and runs score(i+1) on the caller's stream while progressive(i) runs on
 * an internal stream joined back by events (stream-ordered, no host sync).
 * 0 = auto (currently off: measured no gain, both stages are SM-bound), 1 = off,
 * k = k sub-batches (<= 16). */
int psattn_set_pipeline(int32_t sub_batches);
/* Dense hand-over of the GQA kernel (kernels_dense.cu): 0 = auto (a unit whose head exhausts
 * 384 ranks without stopping is redone by one K pass + per-head stop rule + one V pass),
 * 1 = off (the round kernel runs every unit to the end). Same results either way. */
int psattn_set_dense(int32_t mode);
/* Early dense hand-over (stream kernel): a unit whose head has criticality scores at ranks 0 and
 * 383 within `nats` of each other (a flat head, e.g. isotropic keys, that would consume the
 * hand-over budget without stopping) goes to the dense kernels after its first round. Default 2.0;
 * 0 = off. Performance only: results are the same either way. */
int psattn_set_dense_early(float nats);
/* Partial dense mode: a handed-over unit first computes the block masses of each head's top
 * ~`ranks` ranks only (a key-space threshold between ranks/2 and 2*ranks keys) and decides on
 * them; a head that does not stop inside that prefix sends its unit to a second round over the
 * rest of the list. Default 1024; 0 = off (every handed-over unit reads its whole list). Flat
 * units (see psattn_set_dense_early) always take the whole list. Results are the same either way. */
int psattn_set_dense_partial(int32_t ranks);
/* Score-kernel selection: 0 = auto (TMA-staged for dim 128), 1 = register-staged, 2 = TMA whenever supported. */
int psattn_set_score_kernel(int32_t mode);

/* Stage timing (benchmark instrumentation). While enabled, psattn_run_batch
 * records CUDA events around each kernel on its own stream (no host sync).
 * psattn_profile_read waits for the recorded events and returns accumulated
 * milliseconds and launch counts per stage [oracle-mass, score, order,
 * progressive]; reset != 0 clears the accumulators. */
int psattn_profile_enable(int32_t enable);
int psattn_profile_read(double* ms, int64_t* count, int32_t reset);

/* ---- Two-tier KV block store: pinned host backing tier + HBM fast tier ----
 * The paper's KV-cache manager with the reference TieredBlockStore's observable semantics
 * (store.hpp:16-120, store.cpp:11-205): every block's K/V lives in pinned, device-mapped
 * host memory; `fast_slots` HBM slots form one Unified LRU/FIFO domain shared by all
 * layers or LayerPartitioned floor(fast_slots / n_layers) slots per layer; metadata of
 * every block stays resident in HBM. Blocks are named by their index in [0, n_blocks). */
typedef struct psattn_tier psattn_tier;
typedef struct {
    int32_t dim;
    int32_t block_tokens;
    int32_t kv_dtype;        /* PSATTN_KV_* */
    int32_t n_layers;
    int64_t n_blocks;        /* backing-tier capacity (logical blocks) */
    int64_t fast_slots;      /* HBM fast-tier capacity (reference fast_capacity_slots) */
    int32_t pool_policy;     /* PSATTN_POOL_* */
    int32_t eviction_policy; /* PSATTN_EVICT_* */
} psattn_tier_desc;

int psattn_tier_create(const psattn_tier_desc* desc, psattn_tier** out);
void psattn_tier_destroy(psattn_tier* t);
/* put_block (reference store.cpp:59-78) for n blocks: host fp32 K/V [n][block_tokens][dim]
 * (rows past ntok ignored) into the host tier, metadata built in HBM, then write-allocated
 * into the fast tier (evictions counted, installed into HBM). owners may be NULL (owner 0).
 * Duplicate index / bad layer / empty block -> PSATTN_ERR_RUNTIME. Synchronous. */
int psattn_tier_put_blocks(psattn_tier* t, int64_t n, const int64_t* blocks, const int32_t* layers,
                           const int32_t* ntok, const int64_t* owners, const float* keys, const float* values);
/* release_request (reference store.cpp:152-170): drops the owner's blocks from both tiers. */
int psattn_tier_release_request(psattn_tier* t, int64_t owner);
/* psattn_run_batch over block indices (b->slots): fast-tier blocks are read from HBM, the others
 * zero-copy from the host tier; then the loads are accounted in psa_attention_batched's order
 * (reference engine.cpp:173-209: lockstep rounds over the batch's queries, one microbatch of
 * ranks each) through the LRU/FIFO domains, and blocks that entered the fast tier are installed
 * into HBM on `stream`. Synchronous (the accounting needs the processed ranks). */
int psattn_tier_run_batch(psattn_tier* t, const psattn_batch* b, void* workspace, void* stream);
/* Reference CacheStats semantics (bytes = fp32 payload 2*n*d*4 per miss); layer -1 = totals. */
int psattn_tier_stats(psattn_tier* t, int32_t layer, psattn_cache_stats* out);
/* HBM slot of a block (-1: host tier only). */
int psattn_tier_resident(psattn_tier* t, int64_t block, int32_t* out_slot);
/* Bytes actually installed host -> HBM so far (pool dtype, whole slots). */
int psattn_tier_h2d_bytes(psattn_tier* t, uint64_t* out);
/* The tier's device pool (metadata, ntok and layout; for psattn_batch_workspace_bytes users). */
psattn_pool* psattn_tier_pool(psattn_tier* t);

/* ---- Batched serving loop on the GPU path (reference run_serving,
 * serving.cpp:100-229). FCFS head-only admission while one microbatch per live (request,
 * layer) fits the fast tier; every decode step runs ONE device batch per layer over the live
 * requests through a fresh two-tier store (psattn_tier); finished requests are released.
 * The reference's simulated TBT cost model (ServingConfig, serving.hpp:26-34; simulate_pipeline,
 * pipeline.cpp:153-175) is evaluated on the device run's hit/miss series, so the report rows
 * (scenario.cpp:303-341) compare with the reference's exactly; gpu_ms is measured device time. */
typedef struct psattn_serving psattn_serving;
typedef struct {
    double miss_cost_ms;
    double hit_cost_ms;
    double compute_cost_ms;
    int32_t overlap;
    int32_t reserved;
} psattn_serving_cost;
typedef struct {
    /* reference ReportRow (scenario.cpp:303-341) */
    double mean_blocks, p99_blocks, kv_fraction, mean_coverage, min_coverage, hit_ratio;
    double tbt_p50_ms, tbt_p99_ms, overlap_eff;
    psattn_cache_stats store_stats;
    int64_t n_calls, n_steps, completed_requests, device_batches;
    double sim_time_ms;
    double gpu_ms; /* device time of the per-layer batches (CUDA events) */
} psattn_serving_report;
enum { PSATTN_METHOD_PSA = 0, PSATTN_METHOD_TOPK = 1, PSATTN_METHOD_EXACT = 2 };
/* store: the fast tier (dim, block_tokens, kv_dtype, n_layers, fast_slots, policies; n_blocks
 * is derived from the requests); engine: reference psattn_config. */
int psattn_serving_create(const psattn_tier_desc* store, const psattn_config* engine, const psattn_serving_cost* cost,
                          psattn_serving** out);
void psattn_serving_destroy(psattn_serving* s);
/* One request (reference workload Request, workload.hpp:36-50): layer_blocks [n_layers][blocks_per_layer]
 * ids in sequence order; blocks (ids, layers, ntok, fp32 K/V [n_blocks][block_tokens][dim]);
 * queries [decode_steps][n_layers][dim]. Copied. */
int psattn_serving_add_request(psattn_serving* s, int64_t request_id, double arrival_s, int32_t decode_steps,
                               int32_t n_layers, int64_t blocks_per_layer, const int64_t* layer_blocks,
                               int64_t n_blocks, const int64_t* block_ids, const int32_t* block_layers,
                               const int32_t* ntok, const float* keys, const float* values, const float* queries);
/* Runs every added request to completion with method PSATTN_METHOD_* (epsilon for PSA, k for top-k). */
int psattn_serving_run(psattn_serving* s, int32_t method, double epsilon, int64_t k, psattn_serving_report* out);

/* ---- Per-call scoring and ranking over host metadata records (metadata_api.cu) ----
 * The reference's criticality_score / rank_by_scores (include/psattn/metadata.hpp:27-36,
 * src/metadata.cpp:41-96) for callers holding BlockMetadata in host memory; computed on the
 * device. The progressive path scores and orders pool metadata inside its own kernels. */
/* scores[i] = criticality_score(q, record i, estimator, scale), bit-identical to the
 * reference's double. mean/lo/hi: host fp32 [n][d]; estimator 0 Mean, 1 CuboidUpperBound,
 * 2 CuboidMean. Synchronous. */
int psattn_criticality_scores(const float* q, int32_t d, const float* mean, const float* lo, const float* hi,
                              int64_t n, int32_t estimator, double scale, double* scores);
/* order[r] = index of the r-th block by descending score, ties by ascending block id
 * (rank_by_scores). Host arrays of n entries. Synchronous. */
int psattn_rank_by_scores(const double* scores, const int64_t* block_ids, int64_t n, int64_t* order);

/* ---- Oracle / audit tooling (test and report mode; reads every block of every list) ---- */

/* fp64 exact attention over every block of each list, in list order
 * (exact_attention_blocks, reference attention.cpp:36-63): out = device double
 * [n_units][group][dim]. Uses the batch's shape, q, slots, list_off, dim <= 256, scale. */
int psattn_exact_attention(psattn_pool* pool, const psattn_batch* b, double* out, void* stream);

/* run_tradeoff (reference scenario.cpp:451-545, TradeoffReport scenario.hpp) for the
 * batch's queries: fp64 block masses and coverage curves in mass order, the smallest
 * uniform top-k whose coverage meets `target` for every query (bisection), and PSA at
 * epsilon = target with the coverage audit (the batch's estimator, ranking mode and
 * microbatch; its epsilon/topk/audit fields are ignored). Synchronous on `stream`. */
typedef struct {
    double target_coverage;
    int64_t n_queries;
    int64_t max_blocks;
    int64_t k_min;
    double worst_coverage_at_kmin;
    double worst_coverage_below_kmin;
    double psa_mean_blocks;
    double psa_p99_blocks;
    double psa_mean_coverage;
    double block_access_ratio;
} psattn_tradeoff_report;
int psattn_tradeoff(psattn_pool* pool, const psattn_batch* b, double target, psattn_tradeoff_report* out,
                    void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PSATTN_B200_H */
