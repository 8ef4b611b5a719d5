/* psa_oracle.h — TEST INFRASTRUCTURE: plain-C restatement of the reference's
 * PSA path (/root/reference/proj/src/{metadata,attention,engine,store}.cpp).
 *
 * Only tests/, bench.py's cpu_baseline leg and __graft_entry__.smoke() may
 * load this library, and only as the checker. It is never part of the product.
 *
 * Parity pin: tests/test_oracle.py checks every function here against the
 * reference's own golden vectors (test_engine.cpp Fig. 4 walkthrough,
 * test_core.cpp hand-computed softmax/tie/cuboid cases) and bit-for-bit
 * against the compiled reference (oracle/_ref) on seeded inputs, with the
 * outputs of that comparison also frozen in tests/golden/.
 */
#ifndef PSA_ORACLE_H
#define PSA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as psattn_config (reference include/psattn.h:75-83). */
typedef struct {
    double epsilon;
    int32_t microbatch_size;
    int32_t block_size;
    int32_t estimator;    /* 0 Mean, 1 CuboidUpperBound, 2 CuboidMean */
    int32_t ranking_mode; /* 0 Estimated, 1 Oracle */
    int32_t audit_coverage;
    double scale_override;
} orc_config;

typedef struct {
    uint64_t blocks_processed;
    uint64_t total_blocks;
    uint64_t n_iterations;
    double estimated_coverage;
    double true_coverage; /* -1 without audit */
    int32_t terminated_early;
    int32_t status;       /* 0 ok, 1 invalid config, 3 runtime error */
} orc_result;

/* Blocks of one query: block i has ntok[i] rows starting at row row_off[i]
 * of the flat row-major K and V arrays (d floats per row). */
typedef struct {
    const float* keys;
    const float* values;
    const int64_t* row_off;
    const int32_t* ntok;
    const int64_t* ids;
    size_t n;
    int32_t d;
} orc_blocks;

int orc_build_metadata(int32_t ntok, int32_t d, const float* keys, float* mean, float* lo, float* hi);
double orc_criticality(const float* q, int32_t d, const float* mean, const float* lo, const float* hi,
                       int32_t estimator, double scale);
void orc_rank_by_scores(const double* scores, const int64_t* ids, size_t n, int64_t* order_out);
/* Partial attention over one block: returns log_as, fills max/exp_sum/out_unnorm[d]. */
float orc_block_partial(const float* q, int32_t d, int32_t ntok, const float* k, const float* v,
                        float scale, float* max_score, float* exp_sum, float* out_unnorm);
double orc_block_log_as_oracle(const float* q, int32_t d, int32_t ntok, const float* k, double scale);
void orc_exact_attention_blocks(const float* q, const orc_blocks* blk, const int64_t* sel, size_t n_sel,
                                double scale, double* out);
double orc_estimate_coverage(double log_as_acc, double log_as_min, uint64_t n_left);

/* psa_attention (topk == 0) or topk_attention (topk > 0) for one query.
 * processed_ids / iter_est may be NULL (capacity n each). */
int orc_psa(const float* q, const orc_blocks* blk, const orc_config* cfg, uint64_t topk,
            float* out, orc_result* res, int64_t* processed_ids, double* iter_est);

/* Fills the ranking the engine would use (plan_blocks' ranked ids) and the
 * criticality scores in input order. */
int orc_plan(const float* q, const orc_blocks* blk, const orc_config* cfg, int64_t* ranked_ids,
             double* scores_in_input_order);

/* ---- Fast-tier cache model (store.cpp:11-124): hit/miss/eviction/bytes ---- */
typedef struct orc_cache orc_cache;
orc_cache* orc_cache_create(int64_t capacity, int32_t n_layers, int32_t partitioned, int32_t fifo);
void orc_cache_destroy(orc_cache* c);
/* put: write-allocate (store.cpp:59-78). load: hit/miss (store.cpp:80-124).
 * Returns 1 on hit for loads, 0 on miss; *evicted_id = victim or -1. */
int orc_cache_put(orc_cache* c, int64_t id, int32_t layer, int64_t* evicted_id);
int orc_cache_load(orc_cache* c, int64_t id, int32_t layer, uint64_t payload_bytes, int64_t* evicted_id);
void orc_cache_release(orc_cache* c, int64_t id, int32_t layer);
int orc_cache_resident(orc_cache* c, int64_t id, int32_t layer);
/* [hits, misses, evictions, bytes] */
void orc_cache_stats(orc_cache* c, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
