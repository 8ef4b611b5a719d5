/* psa_oracle.c — TEST INFRASTRUCTURE ONLY (see psa_oracle.h).
 *
 * A line-by-line *restatement in C* of the reference algorithm, written from the
 * reference's behaviour, each function citing the file:line it follows
 * (paths relative to /root/reference/proj). Compiled with -ffp-contract=off so
 * every float/double operation rounds exactly where the reference's x86-64
 * build rounds; the tests pin it bit-for-bit against oracle/_ref.
 *
 * This library is the parity checker for the CUDA path. It is never called by
 * the product (paper_2503_00392_b200), which fails loudly without its CUDA
 * extension.
 */
#include "psa_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Metadata: build_metadata (src/metadata.cpp:8-34)                          */
/* ------------------------------------------------------------------------ */
int orc_build_metadata(int32_t ntok, int32_t d, const float* keys, float* mean, float* lo, float* hi) {
    if (ntok <= 0 || d <= 0) return 3; /* metadata.cpp:9 "empty block" */
    double* sum = (double*)malloc(sizeof(double) * (size_t)d);
    for (int32_t i = 0; i < d; ++i) {
        lo[i] = keys[i];
        hi[i] = keys[i];
        sum[i] = lo[i];
    }
    for (int32_t t = 1; t < ntok; ++t) {
        const float* k = keys + (size_t)t * d;
        for (int32_t i = 0; i < d; ++i) {
            /* std::min(a,b) = (b < a) ? b : a ; std::max(a,b) = (a < b) ? b : a */
            lo[i] = (k[i] < lo[i]) ? k[i] : lo[i];
            hi[i] = (hi[i] < k[i]) ? k[i] : hi[i];
            sum[i] += k[i];
        }
    }
    for (int32_t i = 0; i < d; ++i) mean[i] = (float)(sum[i] / ntok);
    free(sum);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Criticality: mean_score / cuboid_upper_score / criticality_score          */
/* (src/metadata.cpp:36-72). fp64, sequential in index order.                */
/* ------------------------------------------------------------------------ */
static double mean_score(const float* q, int32_t d, const float* mean, double scale) {
    double acc = 0.0;
    for (int32_t i = 0; i < d; ++i) acc += (double)q[i] * (double)mean[i];
    return acc * scale;
}

static double cuboid_upper_score(const float* q, int32_t d, const float* lo, const float* hi,
                                 double scale) {
    double acc = 0.0;
    for (int32_t i = 0; i < d; ++i) {
        const double qd = q[i];
        const double a = qd * (double)lo[i];
        const double b = qd * (double)hi[i];
        acc += (a < b) ? b : a; /* std::max(a, b) */
    }
    return acc * scale;
}

double orc_criticality(const float* q, int32_t d, const float* mean, const float* lo, const float* hi,
                       int32_t estimator, double scale) {
    switch (estimator) {
        case 0: return mean_score(q, d, mean, scale);
        case 1: return cuboid_upper_score(q, d, lo, hi, scale);
        case 2: return 0.5 * (mean_score(q, d, mean, scale) + cuboid_upper_score(q, d, lo, hi, scale));
    }
    return NAN;
}

/* ------------------------------------------------------------------------ */
/* Ranking: rank_by_scores (src/metadata.cpp:87-96): score desc, id asc.     */
/* ------------------------------------------------------------------------ */
static const double* g_sort_scores;
static const int64_t* g_sort_ids;

static int rank_cmp(const void* pa, const void* pb) {
    const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    const double sa = g_sort_scores[a], sb = g_sort_scores[b];
    if (sa != sb) return sa > sb ? -1 : 1;
    if (g_sort_ids[a] != g_sort_ids[b]) return g_sort_ids[a] < g_sort_ids[b] ? -1 : 1;
    return (a < b) ? -1 : (a > b); /* duplicate ids: identical blocks, any order */
}

void orc_rank_by_scores(const double* scores, const int64_t* ids, size_t n, int64_t* order_out) {
    for (size_t i = 0; i < n; ++i) order_out[i] = (int64_t)i;
    g_sort_scores = scores;
    g_sort_ids = ids;
    qsort(order_out, n, sizeof(int64_t), rank_cmp);
}

/* ------------------------------------------------------------------------ */
/* Block partial attention (include/psattn/attention.hpp:41-79), fp32.       */
/* ------------------------------------------------------------------------ */
static float dot_scaled_f(const float* q, const float* k, int32_t d, float scale) {
    float acc = 0.0f; /* attention.hpp:41-46 */
    for (int32_t i = 0; i < d; ++i) acc += q[i] * k[i];
    return acc * scale;
}

float orc_block_partial(const float* q, int32_t d, int32_t ntok, const float* k, const float* v,
                        float scale, float* max_score, float* exp_sum, float* out_unnorm) {
    float* scores = (float*)malloc(sizeof(float) * (size_t)ntok);
    float mx = -INFINITY;
    for (int32_t t = 0; t < ntok; ++t) {
        const float s = dot_scaled_f(q, k + (size_t)t * d, d, scale);
        scores[t] = s;
        if (s > mx) mx = s;
    }
    float es = 0.0f;
    for (int32_t i = 0; i < d; ++i) out_unnorm[i] = 0.0f;
    for (int32_t t = 0; t < ntok; ++t) {
        const float w = expf(scores[t] - mx);
        es += w;
        const float* vr = v + (size_t)t * d;
        for (int32_t i = 0; i < d; ++i) out_unnorm[i] += w * vr[i];
    }
    free(scores);
    *max_score = mx;
    *exp_sum = es;
    return mx + logf(es); /* attention.hpp:73 */
}

/* SoftmaxAccumulator + merge_partial + finalize (attention.hpp:28-36, 83-110). */
typedef struct {
    float* out;
    float max_score;
    float exp_sum;
    float log_as_acc;
} acc_t;

static void merge_partial(acc_t* acc, const float* p_out, float p_max, float p_sum, float p_log_as,
                          int32_t d) {
    if (acc->exp_sum == 0.0f) { /* empty() absorbs the partial */
        memcpy(acc->out, p_out, sizeof(float) * (size_t)d);
        acc->max_score = p_max;
        acc->exp_sum = p_sum;
        acc->log_as_acc = p_log_as;
        return;
    }
    const float m = acc->max_score > p_max ? acc->max_score : p_max;
    const float sa = expf(acc->max_score - m);
    const float sp = expf(p_max - m);
    for (int32_t i = 0; i < d; ++i) acc->out[i] = acc->out[i] * sa + p_out[i] * sp;
    acc->exp_sum = acc->exp_sum * sa + p_sum * sp;
    acc->max_score = m;
    acc->log_as_acc = m + logf(acc->exp_sum);
}

/* ------------------------------------------------------------------------ */
/* fp64 oracles (src/attention.cpp:36-79).                                   */
/* ------------------------------------------------------------------------ */
static double dot_scaled_d(const float* q, const float* k, int32_t d, double scale) {
    double acc = 0.0;
    for (int32_t i = 0; i < d; ++i) acc += (double)q[i] * (double)k[i];
    return acc * scale;
}

double orc_block_log_as_oracle(const float* q, int32_t d, int32_t ntok, const float* k, double scale) {
    double mx = -INFINITY;
    double* s = (double*)malloc(sizeof(double) * (size_t)ntok);
    for (int32_t t = 0; t < ntok; ++t) {
        s[t] = dot_scaled_d(q, k + (size_t)t * d, d, scale);
        if (s[t] > mx) mx = s[t];
    }
    double es = 0.0;
    for (int32_t t = 0; t < ntok; ++t) es += exp(s[t] - mx);
    free(s);
    return mx + log(es);
}

void orc_exact_attention_blocks(const float* q, const orc_blocks* blk, const int64_t* sel, size_t n_sel,
                                double scale, double* out) {
    const int32_t d = blk->d;
    double mx = -INFINITY;
    for (size_t j = 0; j < n_sel; ++j) {
        const size_t b = (size_t)sel[j];
        const float* k = blk->keys + (size_t)blk->row_off[b] * d;
        for (int32_t t = 0; t < blk->ntok[b]; ++t) {
            const double s = dot_scaled_d(q, k + (size_t)t * d, d, scale);
            if (s > mx) mx = s;
        }
    }
    for (int32_t i = 0; i < d; ++i) out[i] = 0.0;
    double es = 0.0;
    for (size_t j = 0; j < n_sel; ++j) {
        const size_t b = (size_t)sel[j];
        const float* k = blk->keys + (size_t)blk->row_off[b] * d;
        const float* v = blk->values + (size_t)blk->row_off[b] * d;
        for (int32_t t = 0; t < blk->ntok[b]; ++t) {
            const double w = exp(dot_scaled_d(q, k + (size_t)t * d, d, scale) - mx);
            es += w;
            for (int32_t i = 0; i < d; ++i) out[i] += w * (double)v[(size_t)t * d + i];
        }
    }
    for (int32_t i = 0; i < d; ++i) out[i] /= es;
}

/* ------------------------------------------------------------------------ */
/* Coverage estimator (src/engine.cpp:12-24, 38-55).                         */
/* ------------------------------------------------------------------------ */
static double log_add_exp(double a, double b) {
    if (a == -INFINITY) return b;
    if (b == -INFINITY) return a;
    const double hi = (a < b) ? b : a; /* std::max */
    const double lo = (b < a) ? b : a; /* std::min */
    return hi + log1p(exp(lo - hi));
}

double orc_estimate_coverage(double log_as_acc, double log_as_min, uint64_t n_left) {
    if (log_as_acc == -INFINITY) return NAN; /* engine.cpp:47 throws */
    if (n_left == 0) return 1.0;
    const double ratio = (double)n_left * exp(log_as_min - log_as_acc);
    return 1.0 / (1.0 + ratio);
}

/* ------------------------------------------------------------------------ */
/* plan_blocks (src/engine.cpp:57-90).                                       */
/* ------------------------------------------------------------------------ */
static int validate(const orc_config* c) { /* engine.cpp:28-36 */
    if (!(c->epsilon > 0.0) || c->epsilon > 1.0) return 1;
    if (c->microbatch_size < 1) return 1;
    if (c->block_size < 1) return 1;
    if (c->estimator < 0 || c->estimator > 2) return 1;
    if (c->ranking_mode < 0 || c->ranking_mode > 1) return 1;
    return 0;
}

static double scale_for(const orc_config* c, int32_t d) { /* engine.hpp:36-38, attention.hpp:128 */
    return c->scale_override > 0.0 ? c->scale_override : 1.0 / sqrt((double)d);
}

/* Returns status; fills ranked (block indices into blk, rank order) and, when the
 * plan carries oracle masses, oracle_ranked[n] and *total_log_as. */
static int plan(const float* q, const orc_blocks* blk, const orc_config* cfg, int64_t* ranked,
                double* oracle_ranked, double* total_log_as, double* scores_out) {
    int st = validate(cfg);
    if (st) return st;
    if (blk->n == 0) return 3;
    const int32_t d = blk->d;
    const double scale = scale_for(cfg, d);
    const int want_oracle = cfg->ranking_mode == 1 || cfg->audit_coverage;
    const size_t n = blk->n;
    double* oracle_in = want_oracle ? (double*)malloc(sizeof(double) * n) : NULL;
    if (want_oracle)
        for (size_t i = 0; i < n; ++i)
            oracle_in[i] = orc_block_log_as_oracle(q, d, blk->ntok[i], blk->keys + (size_t)blk->row_off[i] * d,
                                                   scale);
    double* scores = (double*)malloc(sizeof(double) * n);
    if (cfg->ranking_mode == 1) {
        memcpy(scores, oracle_in, sizeof(double) * n);
    } else {
        float* mean = (float*)malloc(sizeof(float) * (size_t)d * 3);
        for (size_t i = 0; i < n; ++i) {
            orc_build_metadata(blk->ntok[i], d, blk->keys + (size_t)blk->row_off[i] * d, mean, mean + d,
                               mean + 2 * d);
            scores[i] = orc_criticality(q, d, mean, mean + d, mean + 2 * d, cfg->estimator, scale);
        }
        free(mean);
    }
    if (scores_out) memcpy(scores_out, scores, sizeof(double) * n);
    orc_rank_by_scores(scores, blk->ids, n, ranked);
    if (want_oracle) {
        double tot = -INFINITY;
        for (size_t r = 0; r < n; ++r) {
            oracle_ranked[r] = oracle_in[ranked[r]];
            tot = log_add_exp(tot, oracle_ranked[r]);
        }
        *total_log_as = tot;
    }
    free(scores);
    free(oracle_in);
    return 0;
}

int orc_plan(const float* q, const orc_blocks* blk, const orc_config* cfg, int64_t* ranked_ids,
             double* scores_in_input_order) {
    const size_t n = blk->n;
    int64_t* ranked = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    double* orc = (double*)malloc(sizeof(double) * (n ? n : 1));
    double tot;
    const int st = plan(q, blk, cfg, ranked, orc, &tot, scores_in_input_order);
    if (!st)
        for (size_t r = 0; r < n; ++r) ranked_ids[r] = blk->ids[ranked[r]];
    free(ranked);
    free(orc);
    return st;
}

/* ------------------------------------------------------------------------ */
/* ProgressiveRun + psa_attention / topk_attention (src/engine.cpp:92-238). */
/* ------------------------------------------------------------------------ */
int orc_psa(const float* q, const orc_blocks* blk, const orc_config* cfg_in, uint64_t topk, float* out,
            orc_result* res, int64_t* processed_ids, double* iter_est) {
    memset(res, 0, sizeof(*res));
    res->true_coverage = -1.0;
    const size_t n = blk->n;
    const int32_t d = blk->d;
    int64_t* ranked = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    double* orc = (double*)malloc(sizeof(double) * (n ? n : 1));
    double total_log_as = -INFINITY;
    int st = plan(q, blk, cfg_in, ranked, orc, &total_log_as, NULL);
    if (st) {
        res->status = st;
        free(ranked);
        free(orc);
        return st;
    }
    const int has_oracle = cfg_in->ranking_mode == 1 || cfg_in->audit_coverage;
    const double epsilon = topk ? 1.0 : cfg_in->epsilon; /* engine.cpp:219-220 */
    const size_t take = topk ? (topk < n ? topk : n) : n;
    const size_t mb = (size_t)cfg_in->microbatch_size;
    const float fscale = (float)scale_for(cfg_in, d); /* engine.cpp:113 */

    acc_t acc;
    acc.out = (float*)calloc((size_t)d, sizeof(float));
    acc.max_score = -INFINITY;
    acc.exp_sum = 0.0f;
    acc.log_as_acc = -INFINITY;
    float* p_out = (float*)malloc(sizeof(float) * (size_t)d);

    double ce_acc = -INFINITY, ce_min = INFINITY; /* CoverageEstimator, engine.hpp:44-51 */
    uint64_t n_left = n;
    size_t cursor = 0;
    int stop = 0;
    double last = 0.0;
    uint64_t n_iter = 0;
    while (!stop && cursor < take) {
        size_t count = n - cursor < mb ? n - cursor : mb; /* next_microbatch_size, engine.cpp:98-102 */
        if (topk && take - cursor < count) count = take - cursor; /* engine.cpp:223-224 */
        for (size_t j = 0; j < count; ++j) { /* consume, engine.cpp:104-127 */
            const size_t b = (size_t)ranked[cursor];
            float pm, ps;
            const float pl = orc_block_partial(q, d, blk->ntok[b], blk->keys + (size_t)blk->row_off[b] * d,
                                               blk->values + (size_t)blk->row_off[b] * d, fscale, &pm, &ps,
                                               p_out);
            merge_partial(&acc, p_out, pm, ps, pl, d);
            const double log_as = has_oracle ? orc[cursor] : (double)pl;
            ce_acc = log_add_exp(ce_acc, log_as);
            ce_min = (log_as < ce_min) ? log_as : ce_min;
            --n_left;
            ++cursor;
        }
        last = orc_estimate_coverage(ce_acc, ce_min, n_left);
        if (iter_est) iter_est[n_iter] = last;
        ++n_iter;
        if (last > epsilon) stop = 1;
    }
    for (int32_t i = 0; i < d; ++i) out[i] = acc.out[i] / acc.exp_sum; /* finalize */
    res->blocks_processed = cursor;
    res->total_blocks = n;
    res->n_iterations = n_iter;
    res->estimated_coverage = last;
    res->terminated_early = topk ? (take < n) : (cursor < n);
    if (processed_ids)
        for (size_t r = 0; r < cursor; ++r) processed_ids[r] = blk->ids[ranked[r]];
    if (cfg_in->audit_coverage) { /* engine.cpp:140-145 */
        double s = -INFINITY;
        for (size_t r = 0; r < cursor; ++r) s = log_add_exp(s, orc[r]);
        res->true_coverage = exp(s - total_log_as);
    }
    free(acc.out);
    free(p_out);
    free(ranked);
    free(orc);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Fast-tier cache model (src/store.cpp:11-124).                             */
/* Front of the recency list = most recent; eviction takes the back.         */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t id;
    int32_t prev, next;
    int32_t used;
} orc_node;

typedef struct {
    int64_t capacity;
    int64_t size;
    int32_t head, tail; /* node indices, -1 if empty */
} orc_domain;

struct orc_cache {
    int32_t n_domains;
    int32_t fifo;
    orc_domain* dom;
    orc_node* nodes;
    int64_t n_nodes, cap_nodes;
    /* open-addressing map id -> node (per cache; ids are globally unique) */
    int64_t* keys;
    int32_t* vals;
    int64_t map_cap;
    int64_t map_count;
    uint64_t hits, misses, evictions, bytes;
};

static uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    return x;
}

#define EMPTY_KEY INT64_MIN
#define TOMB_VAL (-2)

static void map_init(orc_cache* c, int64_t cap) {
    c->map_cap = cap;
    c->keys = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
    c->vals = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
    for (int64_t i = 0; i < cap; ++i) {
        c->keys[i] = EMPTY_KEY;
        c->vals[i] = -1;
    }
}

static int64_t map_find(const orc_cache* c, int64_t id) {
    int64_t i = (int64_t)(mix((uint64_t)id) & (uint64_t)(c->map_cap - 1));
    while (c->keys[i] != EMPTY_KEY) {
        if (c->keys[i] == id && c->vals[i] != TOMB_VAL) return i;
        i = (i + 1) & (c->map_cap - 1);
    }
    return -1;
}

static void map_insert(orc_cache* c, int64_t id, int32_t node);

static void map_grow(orc_cache* c) {
    int64_t* ok = c->keys;
    int32_t* ov = c->vals;
    const int64_t oc = c->map_cap;
    map_init(c, oc * 2);
    for (int64_t i = 0; i < oc; ++i)
        if (ok[i] != EMPTY_KEY && ov[i] >= 0) map_insert(c, ok[i], ov[i]);
    free(ok);
    free(ov);
}

static void map_insert(orc_cache* c, int64_t id, int32_t node) {
    if ((c->map_count + 1) * 2 > c->map_cap) {
        c->map_count = 0;
        map_grow(c);
    }
    int64_t i = (int64_t)(mix((uint64_t)id) & (uint64_t)(c->map_cap - 1));
    while (c->keys[i] != EMPTY_KEY) i = (i + 1) & (c->map_cap - 1);
    c->keys[i] = id;
    c->vals[i] = node;
    ++c->map_count;
}

static void map_erase(orc_cache* c, int64_t id) {
    const int64_t i = map_find(c, id);
    if (i >= 0) c->vals[i] = TOMB_VAL;
}

orc_cache* orc_cache_create(int64_t capacity, int32_t n_layers, int32_t partitioned, int32_t fifo) {
    if (n_layers <= 0 || capacity < 0) return NULL;
    orc_cache* c = (orc_cache*)calloc(1, sizeof(orc_cache));
    c->fifo = fifo;
    c->n_domains = partitioned ? n_layers : 1;
    c->dom = (orc_domain*)calloc((size_t)c->n_domains, sizeof(orc_domain));
    for (int32_t i = 0; i < c->n_domains; ++i) {
        c->dom[i].capacity = partitioned ? capacity / n_layers : capacity; /* store.cpp:13-21 */
        c->dom[i].head = c->dom[i].tail = -1;
    }
    c->cap_nodes = 64;
    c->nodes = (orc_node*)malloc(sizeof(orc_node) * (size_t)c->cap_nodes);
    c->map_count = 0;
    map_init(c, 1 << 10);
    return c;
}

void orc_cache_destroy(orc_cache* c) {
    if (!c) return;
    free(c->dom);
    free(c->nodes);
    free(c->keys);
    free(c->vals);
    free(c);
}

static orc_domain* domain_for(orc_cache* c, int32_t layer) {
    return c->n_domains == 1 ? &c->dom[0] : &c->dom[layer];
}

static void unlink_node(orc_domain* dm, orc_node* nodes, int32_t x) {
    orc_node* nd = &nodes[x];
    if (nd->prev >= 0) nodes[nd->prev].next = nd->next; else dm->head = nd->next;
    if (nd->next >= 0) nodes[nd->next].prev = nd->prev; else dm->tail = nd->prev;
    nd->prev = nd->next = -1;
}

static void push_front(orc_domain* dm, orc_node* nodes, int32_t x) {
    nodes[x].prev = -1;
    nodes[x].next = dm->head;
    if (dm->head >= 0) nodes[dm->head].prev = x; else dm->tail = x;
    dm->head = x;
}

/* insert_fast (store.cpp:37-50) */
static void insert_fast(orc_cache* c, orc_domain* dm, int64_t id, int64_t* evicted_id) {
    *evicted_id = -1;
    if (dm->capacity == 0) return;
    if (dm->size == dm->capacity) {
        const int32_t v = dm->tail;
        *evicted_id = c->nodes[v].id;
        unlink_node(dm, c->nodes, v);
        map_erase(c, c->nodes[v].id);
        c->nodes[v].used = 0;
        dm->size--;
        c->evictions++;
    }
    if (c->n_nodes == c->cap_nodes) {
        c->cap_nodes *= 2;
        c->nodes = (orc_node*)realloc(c->nodes, sizeof(orc_node) * (size_t)c->cap_nodes);
    }
    const int32_t x = (int32_t)c->n_nodes++;
    c->nodes[x].id = id;
    c->nodes[x].used = 1;
    push_front(dm, c->nodes, x);
    map_insert(c, id, x);
    dm->size++;
}

int orc_cache_put(orc_cache* c, int64_t id, int32_t layer, int64_t* evicted_id) {
    insert_fast(c, domain_for(c, layer), id, evicted_id);
    return 0;
}

int orc_cache_load(orc_cache* c, int64_t id, int32_t layer, uint64_t payload_bytes, int64_t* evicted_id) {
    orc_domain* dm = domain_for(c, layer);
    *evicted_id = -1;
    const int64_t slot = map_find(c, id);
    if (slot >= 0) { /* hit: store.cpp:97-103 */
        c->hits++;
        if (!c->fifo) {
            const int32_t x = c->vals[slot];
            unlink_node(dm, c->nodes, x);
            push_front(dm, c->nodes, x);
        }
        return 1;
    }
    c->misses++; /* miss: store.cpp:104-110 */
    c->bytes += payload_bytes;
    insert_fast(c, dm, id, evicted_id);
    return 0;
}

void orc_cache_release(orc_cache* c, int64_t id, int32_t layer) { /* store.cpp:152-170 */
    const int64_t slot = map_find(c, id);
    if (slot < 0) return;
    orc_domain* dm = domain_for(c, layer);
    const int32_t x = c->vals[slot];
    unlink_node(dm, c->nodes, x);
    c->nodes[x].used = 0;
    map_erase(c, id);
    dm->size--;
}

int orc_cache_resident(orc_cache* c, int64_t id, int32_t layer) {
    (void)layer;
    return map_find(c, id) >= 0;
}

void orc_cache_stats(orc_cache* c, uint64_t* out) {
    out[0] = c->hits;
    out[1] = c->misses;
    out[2] = c->evictions;
    out[3] = c->bytes;
}
