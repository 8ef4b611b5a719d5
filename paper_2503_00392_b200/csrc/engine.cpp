// engine.cpp — psattn:: C++ entry points over the device path (B200 build).
//
// Every entry point resolves ids to pool slots and issues ONE device launch
// (TieredBlockStore::run_device -> psattn_run_batch: score -> order ->
// progressive kernel). Host work afterwards is bookkeeping only: result
// assembly, the fast-tier accounting replay in the reference's load order, and
// the injected miss latency.
#include "psattn/engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <semaphore>
#include <string>
#include <thread>

#include "device.h"
#include "engine_internal.h"
#include "psattn/pipeline.hpp"

namespace psattn {

namespace {

double log_add_exp(double a, double b) {
    if (a == -std::numeric_limits<double>::infinity()) return b;
    if (b == -std::numeric_limits<double>::infinity()) return a;
    const double hi = std::max(a, b), lo = std::min(a, b);
    return hi + std::log1p(std::exp(lo - hi));
}

// Microbatch sizes the reference consumes for a run that processed `bp` blocks
// of an n-block plan (engine.cpp:98-102, 219-227).
std::vector<std::size_t> microbatches(std::size_t bp, std::size_t n, std::size_t m, std::size_t take) {
    std::vector<std::size_t> out;
    std::size_t cur = 0;
    while (cur < bp) {
        std::size_t c = std::min(n - cur, m);
        if (take) c = std::min(c, take - cur);
        out.push_back(c);
        cur += c;
    }
    return out;
}

struct Built {
    PSAResult res;
    std::vector<std::size_t> mbs;
};

// Assembles query qi's PSAResult (accounting filled in later).
Built assemble(const detail::DeviceQueryResult& r, std::size_t qi, std::size_t n, const PSAConfig& cfg,
               std::size_t take) {
    Built b;
    PSAResult& res = b.res;
    const std::size_t d = static_cast<std::size_t>(r.dim);
    res.output.assign(r.out.begin() + qi * d, r.out.begin() + (qi + 1) * d);
    res.blocks_processed = static_cast<std::size_t>(r.blocks_processed[qi]);
    res.total_blocks = n;
    res.estimated_coverage = r.est[qi];
    if (cfg.audit_coverage) res.true_coverage = r.true_cov[qi];
    res.terminated_early = r.terminated[qi] != 0;
    res.processed_ids.assign(r.ranked_ids[qi].begin(), r.ranked_ids[qi].begin() + res.blocks_processed);
    b.mbs = microbatches(res.blocks_processed, n, static_cast<std::size_t>(cfg.microbatch_size), take);
    res.iterations.reserve(b.mbs.size());
    std::size_t cur = 0;
    for (std::size_t c : b.mbs) {
        cur += c;
        IterationStats it;
        it.blocks = c;
        it.estimated_coverage = r.iter_est[qi][cur - 1];
        res.iterations.push_back(it);
    }
    return b;
}

// Replays microbatch k of a result through the store accounting.
std::uint64_t account_mb(TieredBlockStore& store, Built& b, std::size_t k, std::size_t start) {
    auto& it = b.res.iterations[k];
    const auto hm = store.account_loads(
        std::span<const BlockId>(b.res.processed_ids.data() + start, b.mbs[k]));
    it.hits = hm.first;
    it.misses = hm.second;
    return hm.second;
}

// Replays every microbatch of a result (one store lock for the whole list).
std::uint64_t account_all(TieredBlockStore& store, Built& b) {
    std::vector<std::pair<std::uint64_t, std::uint64_t>> hm;
    store.account_runs(b.res.processed_ids, b.mbs, hm);
    std::uint64_t misses = 0;
    for (std::size_t k = 0; k < b.mbs.size(); ++k) {
        b.res.iterations[k].hits = hm[k].first;
        b.res.iterations[k].misses = hm[k].second;
        misses += hm[k].second;
    }
    return misses;
}

PSAResult single(std::span<const float> q, std::span<const BlockId> block_ids, const PSAConfig& cfg,
                 TieredBlockStore& store, std::size_t topk) {
    cfg.validate();
    if (block_ids.empty()) throw Error("plan_blocks: no blocks given");
    detail::DeviceQueryBatch qb;
    qb.lists.push_back(block_ids);
    qb.queries.push_back(q.data());
    qb.group = 1;
    qb.dim = static_cast<std::int32_t>(q.size());
    qb.cfg = cfg;
    qb.topk = topk;
    detail::DeviceQueryResult r;
    store.run_device(qb, r);
    const std::size_t take = topk ? std::min(topk, block_ids.size()) : 0;
    Built b = assemble(r, 0, block_ids.size(), cfg, take);
    store.inject_miss_latency(account_all(store, b));
    return std::move(b.res);
}

}  // namespace

void PSAConfig::validate() const {
    if (!(epsilon > 0.0) || epsilon > 1.0)
        throw Error("config: epsilon must be in (0, 1], got " + std::to_string(epsilon));
    if (microbatch_size < 1)
        throw Error("config: microbatch_size must be >= 1, got " + std::to_string(microbatch_size));
    if (block_size < 1) throw Error("config: block_size must be >= 1, got " + std::to_string(block_size));
}

void CoverageEstimator::observe(double log_as) {
    log_as_acc = log_add_exp(log_as_acc, log_as);
    log_as_min = std::min(log_as_min, log_as);
    if (n_left == 0) throw Error("coverage estimator: observed more blocks than planned");
    --n_left;
}

double estimate_coverage(const CoverageEstimator& ce) {
    if (!ce.any_processed()) throw Error("estimate_coverage: no blocks processed yet");
    if (ce.n_left == 0) return 1.0;
    const double ratio = static_cast<double>(ce.n_left) * std::exp(ce.log_as_min - ce.log_as_acc);
    return 1.0 / (1.0 + ratio);
}

RankedPlan plan_blocks(std::span<const float> q, std::span<const BlockId> block_ids, const PSAConfig& cfg,
                       const TieredBlockStore& store) {
    cfg.validate();
    if (block_ids.empty()) throw Error("plan_blocks: no blocks given");
    detail::DeviceQueryBatch qb;
    qb.lists.push_back(block_ids);
    qb.queries.push_back(q.data());
    qb.dim = static_cast<std::int32_t>(q.size());
    qb.cfg = cfg;
    qb.rank_only = true;  // every rank ordered on the device (psattn_rank_batch), no attention
    detail::DeviceQueryResult r;
    const_cast<TieredBlockStore&>(store).run_device(qb, r);
    RankedPlan plan;
    plan.scale = cfg.scale_for(q.size());
    plan.ranked_ids = r.ranked_ids[0];
    if (cfg.ranking_mode == RankingMode::Oracle || cfg.audit_coverage) {
        plan.oracle_log_as = r.oracle_ranked[0];
        double t = -std::numeric_limits<double>::infinity();
        for (double x : plan.oracle_log_as) t = log_add_exp(t, x);
        plan.total_log_as = t;
    }
    return plan;
}

PSAResult psa_attention(std::span<const float> q, std::span<const BlockId> block_ids, const PSAConfig& cfg,
                        TieredBlockStore& store) {
    return single(q, block_ids, cfg, store, 0);
}

PSAResult topk_attention(std::span<const float> q, std::span<const BlockId> block_ids, std::size_t k,
                         const PSAConfig& cfg, TieredBlockStore& store) {
    cfg.validate();
    if (block_ids.empty()) throw Error("plan_blocks: no blocks given");
    if (k == 0) throw Error("topk_attention: k must be >= 1");
    return single(q, block_ids, cfg, store, k);
}

PSAResult topk_attention(std::span<const float> q, std::span<const BlockId> block_ids, std::size_t k,
                         Estimator estimator, TieredBlockStore& store) {
    PSAConfig cfg;
    cfg.estimator = estimator;
    return topk_attention(q, block_ids, k, cfg, store);
}

BatchResult psa_attention_batched(std::span<const HeadVector> queries,
                                  std::span<const std::vector<BlockId>> per_query_blocks, const PSAConfig& cfg,
                                  TieredBlockStore& store) {
    if (queries.size() != per_query_blocks.size()) throw Error("batched attention: query/block list count mismatch");
    if (queries.empty()) throw Error("batched attention: empty batch");
    cfg.validate();
    detail::DeviceQueryBatch qb;
    qb.group = 1;
    qb.dim = static_cast<std::int32_t>(queries[0].size());
    qb.cfg = cfg;
    for (std::size_t i = 0; i < queries.size(); ++i) {
        check_dim(queries[i].size(), static_cast<std::size_t>(qb.dim), "batched attention");
        qb.lists.emplace_back(per_query_blocks[i]);
        qb.queries.push_back(queries[i].data());
    }
    detail::DeviceQueryResult r;
    store.run_device(qb, r);
    std::vector<Built> built;
    for (std::size_t i = 0; i < queries.size(); ++i) built.push_back(assemble(r, i, per_query_blocks[i].size(), cfg, 0));
    // Lockstep replay: round k advances every live query by one microbatch (engine.cpp:191-205).
    BatchResult out;
    std::vector<std::size_t> start(built.size(), 0);
    std::uint64_t misses = 0;
    for (std::size_t k = 0;; ++k) {
        IterationStats round;
        bool any = false;
        for (std::size_t i = 0; i < built.size(); ++i) {
            if (k >= built[i].mbs.size()) continue;
            any = true;
            misses += account_mb(store, built[i], k, start[i]);
            start[i] += built[i].mbs[k];
            const auto& it = built[i].res.iterations[k];
            round.blocks += it.blocks;
            round.hits += it.hits;
            round.misses += it.misses;
            round.estimated_coverage = it.estimated_coverage;
        }
        if (!any) break;
        out.rounds.push_back(round);
    }
    for (auto& b : built) out.results.push_back(std::move(b.res));
    store.inject_miss_latency(misses);
    return out;
}

MultiHeadResult psa_attention_multi_head(std::span<const HeadVector> head_queries,
                                         std::span<const std::vector<BlockId>> kv_head_blocks,
                                         const PSAConfig& cfg, TieredBlockStore& store) {
    if (head_queries.empty()) throw Error("multi-head attention: no query heads");
    if (kv_head_blocks.empty()) throw Error("multi-head attention: no kv heads");
    if (head_queries.size() % kv_head_blocks.size() != 0)
        throw Error("multi-head attention: query head count must be a multiple of kv head count");
    cfg.validate();
    const std::size_t group = head_queries.size() / kv_head_blocks.size();
    for (const auto& q : head_queries) check_dim(q.size(), head_queries[0].size(), "multi-head attention");
    MultiHeadResult out;
    detail::DeviceQueryResult r;
    if (group <= 8) {
        detail::DeviceQueryBatch qb;
        qb.group = static_cast<std::int32_t>(group);
        qb.dim = static_cast<std::int32_t>(head_queries[0].size());
        qb.cfg = cfg;
        qb.want_union = true;
        for (const auto& l : kv_head_blocks) qb.lists.emplace_back(l);
        for (const auto& q : head_queries) {
            check_dim(q.size(), static_cast<std::size_t>(qb.dim), "multi-head attention");
            qb.queries.push_back(q.data());
        }
        store.run_device(qb, r);
    } else {
        // groups wider than 8 run as independent lists (one per q-head)
        detail::DeviceQueryBatch qb;
        qb.group = 1;
        qb.dim = static_cast<std::int32_t>(head_queries[0].size());
        qb.cfg = cfg;
        qb.want_union = true;
        for (std::size_t h = 0; h < head_queries.size(); ++h) {
            qb.lists.emplace_back(kv_head_blocks[h / group]);
            qb.queries.push_back(head_queries[h].data());
        }
        store.run_device(qb, r);
    }
    static const bool prof = std::getenv("PSA_RUN_PROF") != nullptr;  // development: host post-processing time
    const auto t_post = std::chrono::steady_clock::now();
    std::uint64_t misses = 0;
    double t_asm = 0.0, t_acc = 0.0;
    auto lap = [](std::chrono::steady_clock::time_point& t) {
        const auto now = std::chrono::steady_clock::now();
        const double us = std::chrono::duration<double, std::micro>(now - t).count();
        t = now;
        return us;
    };
    auto t_lap = t_post;
    out.per_head.reserve(head_queries.size());
    for (std::size_t h = 0; h < head_queries.size(); ++h) {
        Built b = assemble(r, h, kv_head_blocks[h / group].size(), cfg, 0);
        if (prof) t_asm += lap(t_lap);
        misses += account_all(store, b);
        if (prof) t_acc += lap(t_lap);
        out.per_head.push_back(std::move(b.res));
    }
    out.fetched_union = std::move(r.union_ids);  // sorted, distinct (reference engine.cpp:255-258)
    if (prof)
        std::fprintf(stderr, "multi_head_prof post_us=%.1f assemble_us=%.1f account_us=%.1f\n",
                     std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_post).count(),
                     t_asm, t_acc);
    store.inject_miss_latency(misses);
    return out;
}

namespace detail {

std::size_t multi_head_into(const float* q, std::int32_t n_q_heads, std::int32_t dim, const BlockId* ids,
                            const std::int64_t* list_off, std::int32_t n_kv_heads, const PSAConfig& cfg,
                            TieredBlockStore& store, float* out, HeadStats* stats) {
    // the checks of psa_attention_multi_head above (reference engine.cpp:243-247)
    if (n_q_heads <= 0) throw Error("multi-head attention: no query heads");
    if (n_kv_heads <= 0) throw Error("multi-head attention: no kv heads");
    if (n_q_heads % n_kv_heads != 0)
        throw Error("multi-head attention: query head count must be a multiple of kv head count");
    cfg.validate();
    const int group = n_q_heads / n_kv_heads;
    DeviceQueryBatch qb;
    qb.dim = dim;
    qb.cfg = cfg;
    qb.want_union = true;
    auto list = [&](int k) {
        if (list_off[k + 1] < list_off[k]) throw ConfigError("psattn_run_multi_head: bad list offsets");
        return std::span<const BlockId>(ids + list_off[k], static_cast<std::size_t>(list_off[k + 1] - list_off[k]));
    };
    qb.group = group <= 8 ? group : 1;  // wider groups run as independent lists (one per q-head)
    for (int h = 0; h < n_q_heads; ++h) {
        if (group > 8 || h % group == 0) qb.lists.push_back(list(h / group));
        qb.queries.push_back(q + static_cast<std::size_t>(h) * dim);
    }
    DeviceQueryResult r;
    store.run_device(qb, r);
    std::uint64_t misses = 0;
    std::vector<std::pair<std::uint64_t, std::uint64_t>> hm;
    for (int h = 0; h < n_q_heads; ++h) {
        const std::size_t n = qb.lists[static_cast<std::size_t>(group > 8 ? h : h / group)].size();
        const auto bp = static_cast<std::size_t>(r.blocks_processed[h]);
        const auto mbs = microbatches(bp, n, static_cast<std::size_t>(cfg.microbatch_size), 0);
        store.account_runs(r.ranked_ids[h], mbs, hm);  // load_microbatch of every microbatch, in order
        for (const auto& x : hm) misses += x.second;
        std::copy(r.out.begin() + static_cast<std::ptrdiff_t>(h) * dim,
                  r.out.begin() + static_cast<std::ptrdiff_t>(h + 1) * dim, out + static_cast<std::size_t>(h) * dim);
        if (stats)
            stats[h] = HeadStats{bp, n, r.est[h], cfg.audit_coverage ? r.true_cov[h] : -1.0, r.terminated[h] != 0};
    }
    store.inject_miss_latency(misses);
    return r.union_ids.size();
}

}  // namespace detail

// ---- pipeline.hpp (reference pipeline.cpp:32-176) ----
namespace {
using WallClock = std::chrono::steady_clock;

double elapsed_ms(WallClock::time_point from, WallClock::time_point to) {
    return std::chrono::duration<double, std::milli>(to - from).count();
}

void compute_pad(double ms) {
    if (ms > 0.0) std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(ms));
}

void close_timings(PipelineTimings& t, WallClock::time_point start) {
    t.total_wall_ms = elapsed_ms(start, WallClock::now());
    double sum = 0.0;
    for (double x : t.load_ms) sum += x;
    for (double x : t.compute_ms) sum += x;
    t.sequential_equiv_ms = sum;
    t.overlap_efficiency = t.total_wall_ms > 0.0 ? sum / t.total_wall_ms : 1.0;
}

// Depth-1 hand-off between the loader thread and the computing thread, built on two
// semaphores: `vacant` (the loader must hold it before it starts a load, so at most one
// loaded microbatch can be waiting — and be discarded on stop) and `filled`.
class Handoff {
public:
    // loader side
    bool claim(const StopSignal& stop) {
        vacant_.acquire();
        return !stop.raised();
    }
    void publish(LoadedBatch&& b, double load_ms) {
        batch_ = std::move(b);
        load_ms_ = load_ms;
        filled_.release();
    }
    void fail(std::exception_ptr e) {
        error_ = e;
        filled_.release();
    }
    // computing side: the next batch (rethrows a loader failure); frees the slot at once
    LoadedBatch take(double& load_ms) {
        filled_.acquire();
        if (error_) std::rethrow_exception(error_);
        LoadedBatch b = std::move(batch_);
        load_ms = load_ms_;
        vacant_.release();
        return b;
    }
    // wake a loader blocked in claim() after the stop was raised
    void release_loader() { vacant_.release(); }

private:
    std::counting_semaphore<4> vacant_{1};  // release_loader may add one past a finished loader
    std::binary_semaphore filled_{0};
    LoadedBatch batch_;
    double load_ms_ = 0.0;
    std::exception_ptr error_;
};
}  // namespace

ExecutionResult run_sequential(std::span<const float> q, std::span<const BlockId> block_ids, const PSAConfig& cfg,
                               TieredBlockStore& store, const PipelineOptions& opts) {
    const RankedPlan plan = plan_blocks(q, block_ids, cfg, store);
    ProgressiveRun run(q, plan, cfg);
    ExecutionResult out;
    const auto start = WallClock::now();
    while (!run.finished()) {
        const auto t0 = WallClock::now();
        const LoadedBatch lb = load_microbatch(store, plan, run.cursor(), run.next_microbatch_size());
        const auto t1 = WallClock::now();
        run.consume(lb.blocks, lb.hits, lb.misses);
        compute_pad(opts.compute_pad_ms);
        out.timings.load_ms.push_back(elapsed_ms(t0, t1));
        out.timings.compute_ms.push_back(elapsed_ms(t1, WallClock::now()));
    }
    close_timings(out.timings, start);
    out.result = run.result();
    return out;
}

ExecutionResult run_pipelined(std::span<const float> q, std::span<const BlockId> block_ids, const PSAConfig& cfg,
                              TieredBlockStore& store, const PipelineOptions& opts) {
    const RankedPlan plan = plan_blocks(q, block_ids, cfg, store);
    ProgressiveRun run(q, plan, cfg);
    const std::size_t n = plan.ranked_ids.size();
    const std::size_t m = static_cast<std::size_t>(cfg.microbatch_size);
    Handoff slot;
    StopSignal stop;
    ExecutionResult out;
    const auto start = WallClock::now();
    // The loader walks the plan in microbatches of m (the sizes ProgressiveRun asks for); a
    // stop seen after a load completes drops that batch (the one allowed in-flight load).
    std::thread loader([&] {
        try {
            for (std::size_t cur = 0; cur < n;) {
                if (!slot.claim(stop)) return;
                const std::size_t cnt = std::min(m, n - cur);
                const auto t0 = WallClock::now();
                LoadedBatch lb = load_microbatch(store, plan, cur, cnt);
                const double ms = elapsed_ms(t0, WallClock::now());
                cur += cnt;
                if (stop.raised()) return;
                slot.publish(std::move(lb), ms);
            }
        } catch (...) {
            slot.fail(std::current_exception());
        }
    });
    try {
        while (!run.finished()) {
            double load_ms = 0.0;
            const LoadedBatch lb = slot.take(load_ms);
            const auto t0 = WallClock::now();
            run.consume(lb.blocks, lb.hits, lb.misses);
            compute_pad(opts.compute_pad_ms);
            out.timings.load_ms.push_back(load_ms);
            out.timings.compute_ms.push_back(elapsed_ms(t0, WallClock::now()));
        }
    } catch (...) {
        stop.raise();
        slot.release_loader();
        loader.join();
        throw;
    }
    stop.raise();
    slot.release_loader();
    loader.join();
    close_timings(out.timings, start);
    out.result = run.result();
    return out;
}

PipelineModel simulate_pipeline(std::span<const double> load_ms, std::span<const double> compute_ms) {
    if (load_ms.size() != compute_ms.size()) throw Error("simulate_pipeline: load/compute series length mismatch");
    PipelineModel pm;
    // t_take: when compute took the previous batch (the loader may then start the next load);
    // t_done: when compute finished the previous batch.
    double t_take = 0.0, t_done = 0.0;
    for (std::size_t i = 0; i < load_ms.size(); ++i) {
        const double loaded = t_take + load_ms[i];
        t_take = std::max(loaded, t_done);
        t_done = t_take + compute_ms[i];
        pm.sequential_ms += load_ms[i] + compute_ms[i];
    }
    pm.pipelined_ms = t_done;
    pm.overlap_efficiency = pm.pipelined_ms > 0.0 ? pm.sequential_ms / pm.pipelined_ms : 1.0;
    return pm;
}

// ---- ProgressiveRun / load_microbatch (reference engine.cpp:92-160) ----
namespace detail {
struct RunHandle {
    psa::RunState* s = nullptr;
    ~RunHandle() { psa::prun_destroy(s); }
};
}  // namespace detail

ProgressiveRun::ProgressiveRun(std::span<const float> q, const RankedPlan& plan, const PSAConfig& cfg)
    : q_(q), plan_(&plan), cfg_(&cfg), dev_(std::make_shared<detail::RunHandle>()) {
    if (psa::prun_create(q.data(), static_cast<int>(q.size()), &dev_->s) != PSATTN_OK) throw Error(psa::last_error());
    estimator_.n_left = plan.ranked_ids.size();
}

std::size_t ProgressiveRun::next_microbatch_size() const {
    if (finished()) return 0;
    const std::size_t remaining = plan_->ranked_ids.size() - cursor_;
    return std::min(remaining, static_cast<std::size_t>(cfg_->microbatch_size));
}

double ProgressiveRun::consume(std::span<const std::shared_ptr<const KVBlock>> microbatch, std::uint64_t hits,
                               std::uint64_t misses) {
    if (microbatch.empty()) throw Error("progressive run: empty microbatch");
    if (cursor_ + microbatch.size() > plan_->ranked_ids.size())
        throw Error("progressive run: more blocks fed than planned");
    const std::size_t n = microbatch.size();
    std::vector<std::int32_t> ntok(n);
    std::vector<const float*> ks(n), vs(n);
    for (std::size_t i = 0; i < n; ++i) {
        const KVBlock& b = *microbatch[i];
        if (b.block_id != plan_->ranked_ids[cursor_ + i]) throw Error("progressive run: block fed out of rank order");
        if (b.n_tokens <= 0) throw Error("block_partial_attention: empty block");
        check_dim(q_.size(), static_cast<std::size_t>(b.dim), "block_partial_attention");
        ntok[i] = b.n_tokens;
        ks[i] = b.keys.data();
        vs[i] = b.values.data();
    }
    std::vector<float> las(n);
    if (psa::prun_consume(dev_->s, static_cast<float>(plan_->scale), static_cast<int>(n), ntok.data(), ks.data(),
                          vs.data(), las.data()) != PSATTN_OK)
        throw Error(psa::last_error());
    for (std::size_t i = 0; i < n; ++i) {
        // oracle ranking: the stop rule uses the oracle masses (reference engine.cpp:116-121)
        estimator_.observe(plan_->has_oracle() ? plan_->oracle_log_as[cursor_] : static_cast<double>(las[i]));
        ++cursor_;
    }
    last_estimate_ = estimate_coverage(estimator_);
    iterations_.push_back({n, hits, misses, last_estimate_});
    if (last_estimate_ > cfg_->epsilon) stop_ = true;
    return last_estimate_;
}

PSAResult ProgressiveRun::result() const {
    if (cursor_ == 0) throw Error("progressive run: no blocks processed");
    PSAResult res;
    res.output.resize(q_.size());
    if (psa::prun_result(dev_->s, res.output.data()) != PSATTN_OK) throw Error(psa::last_error());
    res.blocks_processed = cursor_;
    res.total_blocks = plan_->ranked_ids.size();
    res.estimated_coverage = last_estimate_;
    res.terminated_early = cursor_ < plan_->ranked_ids.size();
    res.processed_ids.assign(plan_->ranked_ids.begin(),
                             plan_->ranked_ids.begin() + static_cast<std::ptrdiff_t>(cursor_));
    res.iterations = iterations_;
    if (cfg_->audit_coverage) {
        if (!plan_->has_oracle()) throw Error("progressive run: audit requested without oracle plan data");
        double mx = -std::numeric_limits<double>::infinity(), s = 0.0;
        for (std::size_t i = 0; i < cursor_; ++i) mx = std::max(mx, plan_->oracle_log_as[i]);
        for (std::size_t i = 0; i < cursor_; ++i) s += std::exp(plan_->oracle_log_as[i] - mx);
        res.true_coverage = std::exp(mx + std::log(s) - plan_->total_log_as);
    }
    return res;
}

LoadedBatch load_microbatch(TieredBlockStore& store, const RankedPlan& plan, std::size_t cursor,
                            std::size_t count) {
    LoadedBatch out;
    out.blocks.reserve(count);
    const CacheStats before = store.stats();
    for (std::size_t i = 0; i < count; ++i) out.blocks.push_back(store.load_block(plan.ranked_ids[cursor + i]));
    const CacheStats after = store.stats();
    out.hits = after.hits - before.hits;
    out.misses = after.misses - before.misses;
    return out;
}

// ---- metadata.hpp ----
BlockMetadata build_metadata(const KVBlock& block) {
    if (block.n_tokens <= 0) throw Error("build_metadata: empty block");
    psattn_pool_desc desc{};
    desc.dim = block.dim;
    desc.block_tokens = block.n_tokens;
    desc.kv_dtype = PSATTN_KV_F32;
    desc.n_slots = 1;
    psattn_pool* pool = nullptr;
    if (psattn_pool_create(&desc, &pool) != PSATTN_OK) throw Error(psa::last_error());
    const std::int32_t slot = 0, nt = block.n_tokens;
    BlockMetadata m;
    m.block_id = block.block_id;
    m.layer_id = block.layer_id;
    m.n_tokens = block.n_tokens;
    m.mean_key.resize(block.dim);
    m.lo.resize(block.dim);
    m.hi.resize(block.dim);
    int rc = psa::pool_put(pool, 1, &slot, &nt, block.keys.data(), block.values.data(), 0, nullptr);
    if (rc == PSATTN_OK) rc = psa::read_meta(pool, 0, m.mean_key.data(), m.lo.data(), m.hi.data());
    psattn_pool_destroy(pool);
    if (rc != PSATTN_OK) throw Error(psa::last_error());
    return m;
}

namespace {
// Device scores of every record (metadata_api.cu: psattn_criticality_scores).
std::vector<double> device_scores(std::span<const float> q, std::span<const BlockMetadata> metas, Estimator est,
                                  double scale, const char* what) {
    const std::size_t d = q.size(), n = metas.size();
    std::vector<float> mean(n * d), lo(n * d), hi(n * d);
    for (std::size_t i = 0; i < n; ++i) {
        check_dim(q.size(), metas[i].mean_key.size(), what);
        check_dim(q.size(), metas[i].lo.size(), what);
        check_dim(q.size(), metas[i].hi.size(), what);
        std::copy(metas[i].mean_key.begin(), metas[i].mean_key.end(), mean.begin() + i * d);
        std::copy(metas[i].lo.begin(), metas[i].lo.end(), lo.begin() + i * d);
        std::copy(metas[i].hi.begin(), metas[i].hi.end(), hi.begin() + i * d);
    }
    std::vector<double> s(n);
    if (psattn_criticality_scores(q.data(), static_cast<std::int32_t>(d), mean.data(), lo.data(), hi.data(),
                                  static_cast<std::int64_t>(n), static_cast<std::int32_t>(est), scale,
                                  s.data()) != PSATTN_OK)
        throw Error(psa::last_error());
    return s;
}
}  // namespace

double criticality_score(std::span<const float> q, const BlockMetadata& meta, Estimator estimator, double scale) {
    return device_scores(q, std::span<const BlockMetadata>(&meta, 1), estimator, scale, "criticality_score")[0];
}

std::vector<std::size_t> rank_by_scores(std::span<const double> scores, std::span<const BlockId> block_ids) {
    if (scores.size() != block_ids.size()) throw Error("rank_by_scores: scores and block ids differ in length");
    std::vector<std::int64_t> order(scores.size());
    if (!scores.empty() &&
        psattn_rank_by_scores(scores.data(), block_ids.data(), static_cast<std::int64_t>(scores.size()),
                              order.data()) != PSATTN_OK)
        throw Error(psa::last_error());
    return std::vector<std::size_t>(order.begin(), order.end());
}

std::vector<std::size_t> rank_blocks(std::span<const float> q, std::span<const BlockMetadata> metas,
                                     Estimator estimator, double scale) {
    if (metas.empty()) throw Error("rank_blocks: empty metadata list");
    const std::vector<double> s = device_scores(q, metas, estimator, scale, "criticality_score");
    std::vector<BlockId> ids(metas.size());
    for (std::size_t i = 0; i < metas.size(); ++i) ids[i] = metas[i].block_id;
    return rank_by_scores(s, ids);
}

}  // namespace psattn
