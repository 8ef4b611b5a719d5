// TEST INFRASTRUCTURE — a thin C shim over the UNMODIFIED reference C++ library
// (oracle/_ref/libpsattn_ref.so, built from /root/reference/proj/src by oracle/Makefile).
//
// The reference's own C ABI (psattn.h) does not return processed ids, iteration
// estimates, the multi-head union or the per-layer cache trace; the parity tests
// and the CPU baseline of bench.py need those, so this file exposes them by
// calling the reference's public C++ entry points:
//   psattn::psa_attention            engine.cpp:162-171
//   psattn::topk_attention           engine.cpp:211-231
//   psattn::psa_attention_multi_head engine.cpp:240-260
//   psattn::psa_attention_batched    engine.cpp:173-209
//   psattn::run_pipelined            pipeline.cpp:72-151
//   psattn::TieredBlockStore         store.cpp:11-205
// Only tests/, bench.py's reference arm and __graft_entry__.smoke() load this.
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "psattn.h"
#include "psattn/attention.hpp"
#include "psattn/engine.hpp"
#include "psattn/metadata.hpp"
#include "psattn/pipeline.hpp"
#include "psattn/scenario.hpp"
#include "psattn/store.hpp"
#include "psattn/workload.hpp"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& fn) {
    try {
        return fn();
    } catch (const psattn::NotFoundError& e) {
        g_err = e.what();
        return 2;
    } catch (const psattn::ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

struct Store {
    psattn::TieredBlockStore impl;
    std::ostringstream trace;
    explicit Store(const psattn::StoreOptions& o) : impl(o) {}
};

psattn::PSAConfig to_cpp(const psattn_config& c) {
    psattn::PSAConfig cfg;
    cfg.epsilon = c.epsilon;
    cfg.microbatch_size = c.microbatch_size;
    cfg.block_size = c.block_size;
    cfg.estimator = static_cast<psattn::Estimator>(c.estimator);
    cfg.ranking_mode = c.ranking_mode == PSATTN_RANK_ORACLE ? psattn::RankingMode::Oracle
                                                            : psattn::RankingMode::Estimated;
    cfg.audit_coverage = c.audit_coverage != 0;
    cfg.scale_override = c.scale_override;
    return cfg;
}

struct ResultOut {
    float* out;
    uint64_t* stats_u64;   // [blocks_processed, total_blocks, n_iterations]
    double* stats_f64;     // [estimated_coverage, true_coverage (-1 if none)]
    int32_t* terminated;
    int64_t* processed_ids;  // capacity n (may be null)
    double* iter_est;        // capacity n (may be null)
};

void write_result(const psattn::PSAResult& r, const ResultOut& o) {
    std::memcpy(o.out, r.output.data(), r.output.size() * sizeof(float));
    o.stats_u64[0] = r.blocks_processed;
    o.stats_u64[1] = r.total_blocks;
    o.stats_u64[2] = r.iterations.size();
    o.stats_f64[0] = r.estimated_coverage;
    o.stats_f64[1] = r.true_coverage.value_or(-1.0);
    *o.terminated = r.terminated_early ? 1 : 0;
    if (o.processed_ids)
        for (std::size_t i = 0; i < r.processed_ids.size(); ++i) o.processed_ids[i] = r.processed_ids[i];
    if (o.iter_est)
        for (std::size_t i = 0; i < r.iterations.size(); ++i) o.iter_est[i] = r.iterations[i].estimated_coverage;
}

}  // namespace

extern "C" {

const char* refdrv_last_error(void) { return g_err.c_str(); }

void* refdrv_store_create(int64_t cap, int32_t n_layers, int32_t policy, int32_t evict,
                          double miss_ms) {
    psattn::StoreOptions o;
    o.fast_capacity_slots = static_cast<std::size_t>(cap);
    o.n_layers = n_layers;
    o.policy = policy ? psattn::PoolPolicy::LayerPartitioned : psattn::PoolPolicy::Unified;
    o.eviction = evict ? psattn::EvictionPolicy::FIFO : psattn::EvictionPolicy::LRU;
    o.miss_sleep_ms = miss_ms;
    try {
        return new Store(o);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void refdrv_store_destroy(void* s) { delete static_cast<Store*>(s); }

int refdrv_put(void* s, int64_t id, int32_t layer, int64_t owner, int32_t ntok, int32_t d,
               const float* k, const float* v) {
    return guarded([&] {
        auto b = std::make_shared<psattn::KVBlock>();
        b->block_id = id;
        b->layer_id = layer;
        b->n_tokens = ntok;
        b->dim = d;
        const std::size_t n = static_cast<std::size_t>(ntok) * static_cast<std::size_t>(d);
        b->keys.assign(k, k + n);
        b->values.assign(v, v + n);
        static_cast<Store*>(s)->impl.put_block(std::move(b), owner);
        return 0;
    });
}

// n blocks of ntok x d each, ids first_id.., keys/values [n][ntok][d] (setup helper).
int refdrv_put_many(void* s, int64_t n, int64_t first_id, int32_t layer, int64_t owner, int32_t ntok, int32_t d,
                    const float* k, const float* v) {
    const std::size_t per = static_cast<std::size_t>(ntok) * static_cast<std::size_t>(d);
    for (int64_t i = 0; i < n; ++i) {
        const int rc = refdrv_put(s, first_id + i, layer, owner, ntok, d, k + per * i, v + per * i);
        if (rc) return rc;
    }
    return 0;
}

int refdrv_release(void* s, int64_t owner) {
    return guarded([&] {
        static_cast<Store*>(s)->impl.release_request(owner);
        return 0;
    });
}

// out: [hits, misses, evictions, bytes_transferred]
int refdrv_stats(void* s, uint64_t* out) {
    const auto st = static_cast<Store*>(s)->impl.stats();
    out[0] = st.hits;
    out[1] = st.misses;
    out[2] = st.evictions;
    out[3] = st.bytes_transferred;
    return 0;
}

int refdrv_layer_stats(void* s, int32_t layer, uint64_t* out) {
    const auto st = static_cast<Store*>(s)->impl.stats();
    if (layer < 0 || static_cast<std::size_t>(layer) >= st.per_layer.size()) return 1;
    const auto& l = st.per_layer[static_cast<std::size_t>(layer)];
    out[0] = l.hits;
    out[1] = l.misses;
    out[2] = l.evictions;
    out[3] = l.bytes_transferred;
    return 0;
}

int refdrv_contains(void* s, int64_t id, int32_t* resident_fast) {
    auto* st = static_cast<Store*>(s);
    if (!st->impl.contains(id)) return 2;
    *resident_fast = st->impl.resident_fast(id) ? 1 : 0;
    return 0;
}

void refdrv_enable_trace(void* s) {
    auto* st = static_cast<Store*>(s);
    st->impl.enable_trace(&st->trace);
}

// Copies the accumulated trace text; returns its full length.
int64_t refdrv_trace(void* s, char* buf, int64_t cap) {
    const std::string t = static_cast<Store*>(s)->trace.str();
    if (buf && cap > 0) {
        const std::size_t n = std::min<std::size_t>(t.size(), static_cast<std::size_t>(cap - 1));
        std::memcpy(buf, t.data(), n);
        buf[n] = 0;
    }
    return static_cast<int64_t>(t.size());
}

// One psa_attention (topk == 0) or topk_attention (topk > 0) call.
int refdrv_query(void* s, const float* q, int32_t d, const int64_t* ids, uint64_t n,
                 const psattn_config* cfg, uint64_t topk, float* out, uint64_t* stats_u64,
                 double* stats_f64, int32_t* terminated, int64_t* processed_ids,
                 double* iter_est) {
    return guarded([&] {
        const psattn::PSAConfig c = to_cpp(*cfg);
        std::span<const float> qs(q, static_cast<std::size_t>(d));
        std::span<const psattn::BlockId> is(ids, n);
        auto& store = static_cast<Store*>(s)->impl;
        const psattn::PSAResult r = topk ? psattn::topk_attention(qs, is, topk, c, store)
                                         : psattn::psa_attention(qs, is, c, store);
        write_result(r, {out, stats_u64, stats_f64, terminated, processed_ids, iter_est});
        return 0;
    });
}

// run_pipelined (pipelined != 0) or run_sequential; same outputs as refdrv_query.
int refdrv_pipeline(void* s, int32_t pipelined, const float* q, int32_t d, const int64_t* ids,
                    uint64_t n, const psattn_config* cfg, float* out, uint64_t* stats_u64,
                    double* stats_f64, int32_t* terminated, int64_t* processed_ids) {
    return guarded([&] {
        const psattn::PSAConfig c = to_cpp(*cfg);
        std::span<const float> qs(q, static_cast<std::size_t>(d));
        std::span<const psattn::BlockId> is(ids, n);
        auto& store = static_cast<Store*>(s)->impl;
        const auto r = pipelined ? psattn::run_pipelined(qs, is, c, store)
                                 : psattn::run_sequential(qs, is, c, store);
        write_result(r.result, {out, stats_u64, stats_f64, terminated, processed_ids, nullptr});
        return 0;
    });
}

// psa_attention_multi_head over hq query heads and hkv kv lists of n blocks each
// (ids laid out [hkv][n]). Per-head outputs [hq][d]; per-head stats_u64 [hq][3],
// stats_f64 [hq][2], terminated [hq]; processed ids [hq][n] (may be null);
// fetched union (capacity hkv*n) and its length.
int refdrv_multi_head(void* s, const float* qs, int32_t hq, int32_t d, const int64_t* ids,
                      int32_t hkv, uint64_t n, const psattn_config* cfg, float* outs,
                      uint64_t* stats_u64, double* stats_f64, int32_t* terminated,
                      int64_t* processed_ids, int64_t* union_ids, uint64_t* union_n) {
    return guarded([&] {
        const psattn::PSAConfig c = to_cpp(*cfg);
        std::vector<psattn::HeadVector> heads(static_cast<std::size_t>(hq));
        for (int32_t h = 0; h < hq; ++h)
            heads[static_cast<std::size_t>(h)].assign(qs + static_cast<std::size_t>(h) * d,
                                                      qs + static_cast<std::size_t>(h + 1) * d);
        std::vector<std::vector<psattn::BlockId>> lists(static_cast<std::size_t>(hkv));
        for (int32_t k = 0; k < hkv; ++k)
            lists[static_cast<std::size_t>(k)].assign(ids + static_cast<std::size_t>(k) * n,
                                                      ids + static_cast<std::size_t>(k + 1) * n);
        auto& store = static_cast<Store*>(s)->impl;
        const psattn::MultiHeadResult r = psattn::psa_attention_multi_head(heads, lists, c, store);
        for (int32_t h = 0; h < hq; ++h) {
            const std::size_t hh = static_cast<std::size_t>(h);
            write_result(r.per_head[hh],
                         {outs + hh * d, stats_u64 + hh * 3, stats_f64 + hh * 2, terminated + hh,
                          processed_ids ? processed_ids + hh * n : nullptr, nullptr});
        }
        if (union_ids)
            for (std::size_t i = 0; i < r.fetched_union.size(); ++i) union_ids[i] = r.fetched_union[i];
        *union_n = r.fetched_union.size();
        return 0;
    });
}

// psa_attention_batched over nq queries, each with its own list of n blocks ([nq][n]).
int refdrv_batched(void* s, const float* qs, int32_t nq, int32_t d, const int64_t* ids,
                   uint64_t n, const psattn_config* cfg, float* outs, uint64_t* stats_u64,
                   double* stats_f64, int32_t* terminated, uint64_t* n_rounds) {
    return guarded([&] {
        const psattn::PSAConfig c = to_cpp(*cfg);
        std::vector<psattn::HeadVector> qv(static_cast<std::size_t>(nq));
        std::vector<std::vector<psattn::BlockId>> lists(static_cast<std::size_t>(nq));
        for (int32_t i = 0; i < nq; ++i) {
            const std::size_t ii = static_cast<std::size_t>(i);
            qv[ii].assign(qs + ii * d, qs + (ii + 1) * d);
            lists[ii].assign(ids + ii * n, ids + (ii + 1) * n);
        }
        auto& store = static_cast<Store*>(s)->impl;
        const psattn::BatchResult r = psattn::psa_attention_batched(qv, lists, c, store);
        for (int32_t i = 0; i < nq; ++i) {
            const std::size_t ii = static_cast<std::size_t>(i);
            write_result(r.results[ii], {outs + ii * d, stats_u64 + ii * 3, stats_f64 + ii * 2,
                                         terminated + ii, nullptr, nullptr});
        }
        *n_rounds = r.rounds.size();
        return 0;
    });
}

// store.load_block for each id in order (cache accounting replay of a given load sequence).
int refdrv_load_ids(void* s, const int64_t* ids, int64_t n) {
    return guarded([&] {
        auto& store = static_cast<Store*>(s)->impl;
        for (int64_t i = 0; i < n; ++i) store.load_block(ids[i]);
        return 0;
    });
}

// psa_attention_batched over ragged lists: query i's blocks are ids[off[i] .. off[i+1]);
// processed ids of query i go to pids[off[i] ..] (count = blocks_processed).
int refdrv_batched_ragged(void* s, const float* qs, int32_t nq, int32_t d, const int64_t* ids, const int64_t* off,
                          const psattn_config* cfg, float* outs, uint64_t* stats_u64, double* stats_f64,
                          int32_t* terminated, int64_t* pids, uint64_t* n_rounds) {
    return guarded([&] {
        const psattn::PSAConfig c = to_cpp(*cfg);
        std::vector<psattn::HeadVector> qv(static_cast<std::size_t>(nq));
        std::vector<std::vector<psattn::BlockId>> lists(static_cast<std::size_t>(nq));
        for (int32_t i = 0; i < nq; ++i) {
            const std::size_t ii = static_cast<std::size_t>(i);
            qv[ii].assign(qs + ii * d, qs + (ii + 1) * d);
            lists[ii].assign(ids + off[i], ids + off[i + 1]);
        }
        auto& store = static_cast<Store*>(s)->impl;
        const psattn::BatchResult r = psattn::psa_attention_batched(qv, lists, c, store);
        for (int32_t i = 0; i < nq; ++i) {
            const std::size_t ii = static_cast<std::size_t>(i);
            write_result(r.results[ii], {outs + ii * d, stats_u64 + ii * 3, stats_f64 + ii * 2,
                                         terminated + ii, nullptr, nullptr});
            std::copy(r.results[ii].processed_ids.begin(), r.results[ii].processed_ids.end(), pids + off[i]);
        }
        *n_rounds = r.rounds.size();
        return 0;
    });
}

// Reference metadata for one block (metadata.cpp:8-34).
int refdrv_build_metadata(int32_t ntok, int32_t d, const float* k, float* mean, float* lo,
                          float* hi) {
    return guarded([&] {
        psattn::KVBlock b;
        b.n_tokens = ntok;
        b.dim = d;
        b.keys.assign(k, k + static_cast<std::size_t>(ntok) * d);
        b.values.assign(b.keys.size(), 0.0f);
        const auto m = psattn::build_metadata(b);
        std::memcpy(mean, m.mean_key.data(), sizeof(float) * d);
        std::memcpy(lo, m.lo.data(), sizeof(float) * d);
        std::memcpy(hi, m.hi.data(), sizeof(float) * d);
        return 0;
    });
}

// Reference criticality score (metadata.cpp:41-72).
double refdrv_criticality(const float* q, int32_t d, const float* mean, const float* lo,
                          const float* hi, int32_t estimator, double scale) {
    psattn::BlockMetadata m;
    m.mean_key.assign(mean, mean + d);
    m.lo.assign(lo, lo + d);
    m.hi.assign(hi, hi + d);
    return psattn::criticality_score(std::span<const float>(q, static_cast<std::size_t>(d)), m,
                                     static_cast<psattn::Estimator>(estimator), scale);
}

// Reference fp64 block mass (attention.cpp:65-79).
double refdrv_block_log_as_oracle(const float* q, int32_t d, int32_t ntok, const float* k,
                                  double scale) {
    psattn::KVBlock b;
    b.n_tokens = ntok;
    b.dim = d;
    b.keys.assign(k, k + static_cast<std::size_t>(ntok) * d);
    b.values.assign(b.keys.size(), 0.0f);
    return psattn::block_log_as_oracle(std::span<const float>(q, static_cast<std::size_t>(d)), b,
                                       scale);
}

// ---- attention.hpp templates (attention.hpp:39-109, attention.cpp:7-63): golden values for
// the C++ API parity test (tests/golden/make_attention_golden.py).
namespace {
psattn::KVBlock make_kv(int32_t ntok, int32_t d, const float* k, const float* v) {
    psattn::KVBlock b;
    b.n_tokens = ntok;
    b.dim = d;
    b.keys.assign(k, k + static_cast<std::size_t>(ntok) * d);
    b.values.assign(v, v + static_cast<std::size_t>(ntok) * d);
    return b;
}
}  // namespace

// stats: max score, exp sum, log mass. prec 0 = float, 1 = double (out/stats as double either way).
int refdrv_block_partial(int32_t prec, const float* q, int32_t d, int32_t ntok, const float* k, const float* v,
                         double scale, double* out, double* stats) {
    return guarded([&] {
        const psattn::KVBlock b = make_kv(ntok, d, k, v);
        const std::span<const float> qs(q, static_cast<std::size_t>(d));
        if (prec == 0) {
            const auto r = psattn::block_partial_attention(qs, b, static_cast<float>(scale));
            for (int32_t i = 0; i < d; ++i) out[i] = r.out_unnorm[i];
            stats[0] = r.max_score, stats[1] = r.exp_sum, stats[2] = r.log_as;
        } else {
            const auto r = psattn::block_partial_attention_t<double>(qs, b, scale);
            for (int32_t i = 0; i < d; ++i) out[i] = r.out_unnorm[i];
            stats[0] = r.max_score, stats[1] = r.exp_sum, stats[2] = r.log_as;
        }
        return 0;
    });
}

// n blocks of ntok tokens merged in order (merge_partial) then finalize; log_as_acc in stats[0].
int refdrv_merge_chain(int32_t prec, const float* q, int32_t d, int32_t n, int32_t ntok, const float* k,
                       const float* v, double scale, double* out, double* stats) {
    return guarded([&] {
        const std::span<const float> qs(q, static_cast<std::size_t>(d));
        const std::size_t per = static_cast<std::size_t>(ntok) * d;
        auto run = [&](auto zero) {
            using T = decltype(zero);
            psattn::SoftmaxAccumulatorT<T> acc;
            for (int32_t i = 0; i < n; ++i) {
                const psattn::KVBlock b = make_kv(ntok, d, k + per * i, v + per * i);
                psattn::merge_partial(acc, psattn::block_partial_attention_t<T>(qs, b, static_cast<T>(scale)));
            }
            const auto o = psattn::finalize(acc);
            for (int32_t i = 0; i < d; ++i) out[i] = o[i];
            stats[0] = acc.log_as_acc, stats[1] = acc.exp_sum, stats[2] = acc.max_score;
        };
        if (prec == 0) run(0.0f);
        else run(0.0);
        return 0;
    });
}

int refdrv_exact_attention_blocks(const float* q, int32_t d, int32_t n, int32_t ntok, const float* k, const float* v,
                                  double scale, double* out) {
    return guarded([&] {
        const std::size_t per = static_cast<std::size_t>(ntok) * d;
        std::vector<psattn::KVBlock> bs;
        for (int32_t i = 0; i < n; ++i) bs.push_back(make_kv(ntok, d, k + per * i, v + per * i));
        std::vector<const psattn::KVBlock*> ptrs;
        for (auto& b : bs) ptrs.push_back(&b);
        const auto o = psattn::exact_attention_blocks(std::span<const float>(q, static_cast<std::size_t>(d)), ptrs, scale);
        for (int32_t i = 0; i < d; ++i) out[i] = o[i];
        return 0;
    });
}

// ---- Reference workload generator (workload.cpp:49-153), exported so the GPU path can be fed the
// exact inputs of the reference's own scenarios (tradeoff / serving golden reports in proj/out).
void* refdrv_workload_create(int32_t n_requests, int32_t dim, int32_t block_size, int32_t n_layers,
                             int32_t context_min, int32_t context_max, int32_t decode_steps, double rho,
                             double skew, int32_t planted, int32_t planted_alt, uint64_t seed) {
    try {
        psattn::WorkloadSpec w;
        w.n_requests = n_requests;
        w.dim = dim;
        w.block_size = block_size;
        w.n_layers = n_layers;
        w.context_min = context_min;
        w.context_max = context_max;
        w.decode_steps = decode_steps;
        w.rho = rho;
        w.skew = skew;
        w.planted_blocks = planted;
        w.planted_blocks_alt = planted_alt;
        w.seed = seed;
        return new std::vector<psattn::Request>(psattn::generate_workload(w));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void refdrv_workload_destroy(void* w) { delete static_cast<std::vector<psattn::Request>*>(w); }
int32_t refdrv_workload_n_requests(void* w) {
    return static_cast<int32_t>(static_cast<std::vector<psattn::Request>*>(w)->size());
}
// info[0..3] = request_id, context_tokens, decode_steps, n_blocks (all layers); info[4] = blocks per layer
int refdrv_workload_request(void* w, int32_t r, int64_t* info) {
    const auto& q = static_cast<std::vector<psattn::Request>*>(w)->at(static_cast<std::size_t>(r));
    info[0] = q.request_id;
    info[1] = q.context_tokens;
    info[2] = q.decode_steps;
    info[3] = static_cast<int64_t>(q.blocks.size());
    info[4] = static_cast<int64_t>(q.blocks_per_layer());
    return 0;
}
// Blocks in the request's put order: ids, layers, n_tokens, K/V [n][block_size][dim] zero-padded.
int refdrv_workload_blocks(void* w, int32_t r, int32_t block_size, int64_t* ids, int32_t* layers,
                           int32_t* ntok, float* keys, float* values) {
    const auto& q = static_cast<std::vector<psattn::Request>*>(w)->at(static_cast<std::size_t>(r));
    for (std::size_t i = 0; i < q.blocks.size(); ++i) {
        const auto& b = *q.blocks[i];
        ids[i] = b.block_id;
        layers[i] = b.layer_id;
        ntok[i] = b.n_tokens;
        const std::size_t stride = static_cast<std::size_t>(block_size) * b.dim;
        std::memset(keys + i * stride, 0, stride * sizeof(float));
        std::memset(values + i * stride, 0, stride * sizeof(float));
        std::memcpy(keys + i * stride, b.keys.data(), b.keys.size() * sizeof(float));
        std::memcpy(values + i * stride, b.values.data(), b.values.size() * sizeof(float));
    }
    return 0;
}
int refdrv_workload_layer_list(void* w, int32_t r, int32_t layer, int64_t* ids) {
    const auto& q = static_cast<std::vector<psattn::Request>*>(w)->at(static_cast<std::size_t>(r));
    const auto& l = q.layer_blocks.at(static_cast<std::size_t>(layer));
    std::memcpy(ids, l.data(), l.size() * sizeof(int64_t));
    return 0;
}
int refdrv_workload_query(void* w, int32_t r, int32_t step, int32_t layer, float* out) {
    const auto& q = static_cast<std::vector<psattn::Request>*>(w)->at(static_cast<std::size_t>(r));
    const auto& v = q.step_queries.at(static_cast<std::size_t>(step)).at(static_cast<std::size_t>(layer));
    std::memcpy(out, v.data(), v.size() * sizeof(float));
    return 0;
}

}  // extern "C"
