// C++ API test (GPU): re-states reference engine/store tests (test_engine.cpp,
// test_pipeline.cpp, test_store.cpp) against include/psattn/*.hpp, linked to
// libpsattn_b200.so. Prints "OK <n>" and exits 0 on success. Built by
// tests/test_gpu_cpp.py with g++ -std=c++20.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <random>
#include <set>
#include <sstream>
#include <vector>

#include "psattn/engine.hpp"
#include "psattn/pipeline.hpp"
#include "psattn/store.hpp"

using namespace psattn;

static int g_checks = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            std::exit(1);                                                     \
        }                                                                     \
    } while (0)

static std::shared_ptr<KVBlock> make_block(std::mt19937_64& rng, BlockId id, int layer, int nt, int d) {
    std::normal_distribution<float> nd;
    auto b = std::make_shared<KVBlock>();
    b->block_id = id;
    b->layer_id = layer;
    b->n_tokens = nt;
    b->dim = d;
    b->keys.resize(static_cast<std::size_t>(nt) * d);
    b->values.resize(b->keys.size());
    for (auto& x : b->keys) x = nd(rng);
    for (auto& x : b->values) x = nd(rng);
    return b;
}

static StoreOptions opts(std::size_t cap, int layers = 1) {
    StoreOptions o;
    o.fast_capacity_slots = cap;
    o.n_layers = layers;
    return o;
}

int main() {
    // --- metadata.hpp scoring / ranking (reference test_core.cpp:363-434) ---
    {
        KVBlock proto;
        proto.layer_id = 0;
        proto.n_tokens = 2;
        proto.dim = 2;
        proto.keys = {1.0f, 0.0f, 0.0f, 1.0f};
        proto.values = {0.0f, 0.0f, 0.0f, 0.0f};
        std::vector<BlockMetadata> metas;
        for (BlockId id : {7, 3, 5}) {
            KVBlock b = proto;
            b.block_id = id;
            metas.push_back(build_metadata(b));
        }
        const std::vector<float> q = {1.0f, 1.0f};
        const auto order = rank_blocks(q, metas, Estimator::CuboidMean, 1.0);
        CHECK(order.size() == 3);
        CHECK(metas[order[0]].block_id == 3 && metas[order[1]].block_id == 5 && metas[order[2]].block_id == 7);
        bool threw = false;
        try {
            (void)rank_blocks(q, std::span<const BlockMetadata>{}, Estimator::Mean, 1.0);
        } catch (const Error&) {
            threw = true;
        }
        CHECK(threw);
        const std::vector<double> scores = {1.0, 3.0, 3.0, -2.0, 0.5};
        const std::vector<BlockId> ids = {10, 9, 4, 2, 3};
        const auto o2 = rank_by_scores(scores, ids);
        CHECK(o2.size() == 5 && ids[o2[0]] == 4 && ids[o2[1]] == 9 && ids[o2[2]] == 10 && ids[o2[3]] == 3 &&
              ids[o2[4]] == 2);
        // the cuboid upper bound dominates every per-token score of the block
        std::mt19937_64 rng(707);
        for (int i = 0; i < 200; ++i) {
            const int d = 4 + (i % 5) * 7, nt = 1 + i % 24;
            auto blk = make_block(rng, i, 0, nt, d);
            const BlockMetadata m = build_metadata(*blk);
            std::vector<float> qq(static_cast<std::size_t>(d));
            std::normal_distribution<float> nd;
            for (auto& x : qq) x = nd(rng);
            const double bound = criticality_score(qq, m, Estimator::CuboidUpperBound, 0.5);
            for (int t = 0; t < nt; ++t) {
                double s = 0.0;
                for (int k = 0; k < d; ++k) s += (double)qq[k] * (double)blk->keys[(std::size_t)t * d + k];
                CHECK(s * 0.5 <= bound + std::ldexp(std::max(1.0, std::abs(bound)), -48));
            }
        }
    }
    // --- Fig. 4 walkthrough (reference test_engine.cpp:130-211) with iteration records ---
    {
        const std::vector<double> masses = {400, 330, 250, 55, 40, 30, 20, 14.08, 12, 10, 9, 5.848, 5, 4, 3, 2};
        TieredBlockStore store(opts(16));
        std::vector<double> realized;
        std::vector<BlockId> ids;
        for (std::size_t i = 0; i < masses.size(); ++i) {
            auto b = std::make_shared<KVBlock>();
            b->block_id = static_cast<BlockId>(i);
            b->n_tokens = 1;
            b->dim = 2;
            const float k0 = static_cast<float>(std::log(masses[i]) / 2.0);
            b->keys = {k0, 0.0f};
            b->values = {static_cast<float>(i + 1), static_cast<float>(2 * i + 1)};
            store.put_block(b);
            realized.push_back(std::exp(2.0 * k0));
            ids.push_back(static_cast<BlockId>(i));
        }
        const HeadVector q = {2.0f, 0.0f};
        PSAConfig cfg;
        cfg.epsilon = 0.98;
        cfg.microbatch_size = 4;
        cfg.block_size = 1;
        cfg.ranking_mode = RankingMode::Oracle;
        cfg.audit_coverage = true;
        cfg.scale_override = 1.0;
        const PSAResult r = psa_attention(q, ids, cfg, store);
        CHECK(r.blocks_processed == 12 && r.total_blocks == 16 && r.terminated_early);
        CHECK(r.iterations.size() == 3);
        double acc = 0, mn = 1e300;
        for (std::size_t i = 0; i < 12; ++i) {
            acc += realized[i];
            mn = std::min(mn, realized[i]);
            if ((i + 1) % 4 == 0) {
                const double cov = acc / (acc + mn * (16 - i - 1));
                CHECK(std::fabs(r.iterations[i / 4].estimated_coverage - cov) < 1e-9);
                CHECK(r.iterations[i / 4].blocks == 4);
            }
        }
        for (std::size_t i = 0; i < 12; ++i) CHECK(r.processed_ids[i] == static_cast<BlockId>(i));
        CHECK(r.true_coverage.has_value() && r.estimated_coverage <= *r.true_coverage + 1e-12);
        // plan_blocks in Oracle mode: descending oracle masses
        const RankedPlan plan = plan_blocks(q, ids, cfg, store);
        CHECK(plan.has_oracle() && plan.oracle_log_as.size() == 16);
        for (std::size_t i = 1; i < 16; ++i) CHECK(plan.oracle_log_as[i - 1] >= plan.oracle_log_as[i]);
    }
    // --- caller-driven ProgressiveRun + load_microbatch (reference engine.cpp:162-171's loop)
    //     reproduces psa_attention: same stop point, ids, iteration records, output ---
    {
        std::mt19937_64 rng(9090);
        const int d = 32;
        TieredBlockStore sa(opts(64)), sb(opts(64));
        std::vector<BlockId> ids;
        for (int i = 0; i < 40; ++i) {
            auto blk = make_block(rng, 100 + i, 0, 1 + i % 16, d);
            sa.put_block(blk);
            sb.put_block(blk);
            ids.push_back(100 + i);
        }
        std::normal_distribution<float> nd;
        for (int rep = 0; rep < 2; ++rep) {
            HeadVector q(d);
            for (auto& x : q) x = 2.0f * nd(rng);
            PSAConfig cfg;
            cfg.epsilon = 0.9;
            cfg.microbatch_size = 3;
            cfg.audit_coverage = rep == 1;
            if (rep == 1) cfg.ranking_mode = RankingMode::Oracle;
            const PSAResult want = psa_attention(q, ids, cfg, sa);
            const RankedPlan plan = plan_blocks(q, ids, cfg, sb);
            ProgressiveRun run(q, plan, cfg);
            while (!run.finished()) {
                LoadedBatch lb = load_microbatch(sb, plan, run.cursor(), run.next_microbatch_size());
                run.consume(lb.blocks, lb.hits, lb.misses);
            }
            const PSAResult got = run.result();
            CHECK(got.blocks_processed == want.blocks_processed && got.processed_ids == want.processed_ids);
            CHECK(got.terminated_early == want.terminated_early && got.iterations.size() == want.iterations.size());
            CHECK(std::fabs(got.estimated_coverage - want.estimated_coverage) < 1e-6);
            for (int k = 0; k < d; ++k) CHECK(std::fabs(got.output[k] - want.output[k]) < 1e-4f);
            if (rep == 1) CHECK(got.true_coverage && std::fabs(*got.true_coverage - *want.true_coverage) < 1e-9);
        }
        const PSAConfig dcfg;  // (ProgressiveRun keeps references to q, plan and cfg, like the reference)
        const HeadVector q1(d, 1.0f);
        const RankedPlan plan = plan_blocks(q1, ids, dcfg, sb);
        ProgressiveRun run(q1, plan, dcfg);
        bool threw = false;
        try {
            std::vector<std::shared_ptr<const KVBlock>> wrong = {sb.peek_block(plan.ranked_ids[1])};
            run.consume(wrong, 0, 0);
        } catch (const Error&) {
            threw = true;
        }
        CHECK(threw);
    }
    // --- batched == solo (test_engine.cpp:280-327) incl. lockstep round accounting ---
    {
        std::mt19937_64 rng(4242);
        const int d = 20;
        TieredBlockStore bs(opts(16)), ss(opts(16));
        std::vector<std::vector<BlockId>> lists;
        std::vector<HeadVector> qs;
        BlockId next = 0;
        std::normal_distribution<float> nd;
        for (int r = 0; r < 3; ++r) {
            std::vector<BlockId> l;
            for (int b = 0; b < 10 + r * 4; ++b, ++next) {
                auto blk = make_block(rng, next, 0, 5, d);
                bs.put_block(blk);
                ss.put_block(blk);
                l.push_back(next);
            }
            lists.push_back(l);
            HeadVector q(d);
            for (auto& x : q) x = nd(rng);
            qs.push_back(q);
        }
        PSAConfig cfg;
        cfg.epsilon = 0.9;
        cfg.microbatch_size = 3;
        cfg.block_size = 5;
        cfg.audit_coverage = true;
        const BatchResult br = psa_attention_batched(qs, lists, cfg, bs);
        std::size_t total = 0;
        for (int i = 0; i < 3; ++i) {
            const PSAResult solo = psa_attention(qs[i], lists[i], cfg, ss);
            CHECK(br.results[i].blocks_processed == solo.blocks_processed);
            CHECK(br.results[i].processed_ids == solo.processed_ids);
            CHECK(br.results[i].output == solo.output);
            CHECK(br.results[i].estimated_coverage == solo.estimated_coverage);
            total += solo.blocks_processed;
        }
        std::size_t rb = 0;
        for (const auto& r : br.rounds) rb += r.blocks;
        CHECK(rb == total);
        bool threw = false;
        try {
            (void)psa_attention_batched({}, {}, cfg, bs);
        } catch (const Error&) {
            threw = true;
        }
        CHECK(threw);
    }
    // --- top-k processes the k best-ranked blocks (test_engine.cpp:329-367) ---
    {
        std::mt19937_64 rng(555);
        const int d = 16;
        TieredBlockStore store(opts(64));
        std::vector<BlockId> ids;
        for (int i = 0; i < 20; ++i) {
            store.put_block(make_block(rng, i, 0, 4, d));
            ids.push_back(i);
        }
        HeadVector q(d, 0.3f);
        q[3] = -1.0f;
        PSAConfig cfg;
        cfg.microbatch_size = 4;
        const RankedPlan plan = plan_blocks(q, ids, cfg, store);
        for (std::size_t k : {std::size_t{1}, std::size_t{7}, std::size_t{20}, std::size_t{50}}) {
            const PSAResult r = topk_attention(q, ids, k, cfg, store);
            const std::size_t take = std::min<std::size_t>(k, 20);
            CHECK(r.blocks_processed == take && r.terminated_early == (take < 20));
            for (std::size_t i = 0; i < take; ++i) CHECK(r.processed_ids[i] == plan.ranked_ids[i]);
        }
        CHECK(topk_attention(q, ids, 5, Estimator::CuboidMean, store).blocks_processed == 5);
        bool threw = false;
        try {
            (void)topk_attention(q, ids, 0, cfg, store);
        } catch (const Error&) {
            threw = true;
        }
        CHECK(threw);
    }
    // --- GQA multi-head (test_engine.cpp:369-414) ---
    {
        std::mt19937_64 rng(31337);
        const int d = 12;
        TieredBlockStore store(opts(64)), ref(opts(64));
        std::vector<std::vector<BlockId>> kv;
        BlockId next = 0;
        for (int h = 0; h < 2; ++h) {
            std::vector<BlockId> l;
            for (int b = 0; b < 12; ++b, ++next) {
                auto blk = make_block(rng, next, 0, 4, d);
                store.put_block(blk);
                ref.put_block(blk);
                l.push_back(next);
            }
            kv.push_back(l);
        }
        std::vector<HeadVector> hq;
        std::normal_distribution<float> nd;
        for (int h = 0; h < 4; ++h) {
            HeadVector q(d);
            for (auto& x : q) x = nd(rng);
            hq.push_back(q);
        }
        PSAConfig cfg;
        cfg.epsilon = 0.85;
        cfg.microbatch_size = 2;
        const MultiHeadResult mh = psa_attention_multi_head(hq, kv, cfg, store);
        std::set<BlockId> uni;
        for (int h = 0; h < 4; ++h) {
            const PSAResult solo = psa_attention(hq[h], kv[h / 2], cfg, ref);
            CHECK(mh.per_head[h].processed_ids == solo.processed_ids);
            CHECK(mh.per_head[h].output == solo.output);
            for (BlockId id : solo.processed_ids) uni.insert(id);
        }
        CHECK(mh.fetched_union == std::vector<BlockId>(uni.begin(), uni.end()));
        std::vector<HeadVector> bad(hq.begin(), hq.begin() + 3);
        bool threw = false;
        try {
            (void)psa_attention_multi_head(bad, kv, cfg, store);
        } catch (const Error&) {
            threw = true;
        }
        CHECK(threw);
    }
    // --- pipelined == sequential == plain, bitwise (test_pipeline.cpp:48-92) ---
    {
        std::mt19937_64 rng(77);
        const int d = 32;
        TieredBlockStore a(opts(8)), b(opts(8)), c(opts(8));
        std::vector<BlockId> ids;
        for (int i = 0; i < 40; ++i) {
            auto blk = make_block(rng, i, 0, 8, d);
            a.put_block(blk);
            b.put_block(blk);
            c.put_block(blk);
            ids.push_back(i);
        }
        HeadVector q(d, 0.2f);
        PSAConfig cfg;
        cfg.epsilon = 0.9;
        cfg.microbatch_size = 3;
        const auto p = run_pipelined(q, ids, cfg, a);
        const auto s = run_sequential(q, ids, cfg, b);
        const auto plain = psa_attention(q, ids, cfg, c);
        CHECK(p.result.output == s.result.output && s.result.output == plain.output);
        CHECK(p.result.processed_ids == plain.processed_ids);
        CHECK(a.stats().hits == c.stats().hits && a.stats().misses == c.stats().misses);
        for (std::size_t i = 0; i < plain.iterations.size(); ++i) {
            CHECK(p.result.iterations[i].hits == plain.iterations[i].hits);
            CHECK(p.result.iterations[i].misses == plain.iterations[i].misses);
        }
    }
    // --- store: hand-walked LRU + exact trace text (test_store.cpp:108-132, 294-309) ---
    {
        std::mt19937_64 rng(1);
        TieredBlockStore st(opts(2));
        for (int i = 0; i < 3; ++i) st.put_block(make_block(rng, i, 0, 2, 4));  // puts 0,1,2: evicts 0
        CHECK(st.stats().evictions == 1);
        CHECK(!st.resident_fast(0) && st.resident_fast(1) && st.resident_fast(2));
        std::ostringstream tr;
        st.enable_trace(&tr);
        (void)st.load_block(1);  // hit, 1 becomes MRU
        (void)st.load_block(0);  // miss, evicts 2 (LRU)
        (void)st.load_block(2);  // miss, evicts 1
        CHECK(tr.str() == "0,0,1,hit,-\n1,0,0,miss,2\n2,0,2,miss,1\n");
        const CacheStats cs = st.stats();
        CHECK(cs.hits == 1 && cs.misses == 2 && cs.evictions == 3);
        CHECK(cs.bytes_transferred == 2 * (2 * 2 * 4 * 4));
        const auto blk = st.peek_block(0);
        CHECK(blk->n_tokens == 2 && blk->dim == 4 && blk->keys.size() == 8);
        const BlockMetadata m = st.metadata(0);
        for (int i = 0; i < 4; ++i) {
            CHECK(m.lo[i] == std::min(blk->keys[i], blk->keys[4 + i]));
            CHECK(m.hi[i] == std::max(blk->keys[i], blk->keys[4 + i]));
        }
        bool nf = false;
        try {
            (void)st.load_block(99);
        } catch (const NotFoundError&) {
            nf = true;
        }
        CHECK(nf);
        const BlockMetadata bm = build_metadata(*blk);
        CHECK(bm.mean_key == m.mean_key && bm.lo == m.lo && bm.hi == m.hi);
    }
    // --- plan_blocks over a long list (> the 512/1024-rank tranches the progressive kernels order
    //     lazily): every rank equals the reference ranking restated on the host (criticality_score
    //     in index order, metadata.cpp:41-72; score desc, block id asc, metadata.cpp:87-96);
    //     psa_attention on the same list agrees with the plan's prefix ---
    {
        std::mt19937_64 rng(4242);
        const int d = 128, T = 16, n = 3000;
        TieredBlockStore store(opts(0));
        std::vector<BlockId> ids;
        // ids deliberately not in ascending order of insertion: the tie rule is on block id
        std::shared_ptr<KVBlock> prev;
        for (int i = 0; i < n; ++i) {
            const BlockId id = static_cast<BlockId>((i * 7919) % 10007);
            auto blk = make_block(rng, id, 0, T, d);
            if (i % 100 == 1) {  // exact copy of the previous block: equal scores, ties resolved by id
                *blk = *prev;
                blk->block_id = id;
            }
            store.put_block(blk, 1);
            ids.push_back(id);
            prev = blk;
        }
        std::normal_distribution<float> nd;
        std::vector<float> q(d);
        for (auto& x : q) x = nd(rng);
        for (Estimator est : {Estimator::Mean, Estimator::CuboidUpperBound, Estimator::CuboidMean}) {
            PSAConfig cfg;
            cfg.estimator = est;
            const RankedPlan plan = plan_blocks(q, ids, cfg, store);
            CHECK(plan.ranked_ids.size() == static_cast<std::size_t>(n));
            const double scale = 1.0 / std::sqrt(static_cast<double>(d));
            std::vector<std::pair<double, BlockId>> ref;
            for (BlockId id : ids) {
                const BlockMetadata m = store.metadata(id);
                double am = 0.0, au = 0.0;
                for (int k = 0; k < d; ++k) {
                    const double qd = q[k];
                    am += qd * static_cast<double>(m.mean_key[k]);
                    au += std::max(qd * static_cast<double>(m.lo[k]), qd * static_cast<double>(m.hi[k]));
                }
                const double s = est == Estimator::Mean ? am * scale
                                 : est == Estimator::CuboidUpperBound ? au * scale
                                                                      : 0.5 * (am * scale + au * scale);
                ref.emplace_back(s, id);
            }
            std::vector<std::pair<double, BlockId>> sorted = ref;
            std::sort(sorted.begin(), sorted.end(), [](const auto& a, const auto& b) {
                return a.first != b.first ? a.first > b.first : a.second < b.second;
            });
            std::size_t mism = 0;
            for (int r = 0; r < n; ++r)
                if (plan.ranked_ids[r] != sorted[r].second) {
                    // only a near-tie (fp64 summation order, ~1e-16 relative) may swap neighbours:
                    // the swapped partner is the previous or the next rank
                    const double up = r > 0 ? std::fabs(sorted[r].first - sorted[r - 1].first) : INFINITY;
                    const double dn = r + 1 < n ? std::fabs(sorted[r].first - sorted[r + 1].first) : INFINITY;
                    const double gap = std::min(up, dn);
                    if (!(gap <= 1e-12 * std::max(1.0, std::fabs(sorted[r].first))))
                        std::fprintf(stderr, "rank %d: device id %lld, host id %lld (score %.17g), gap %.3g\n", r,
                                     (long long)plan.ranked_ids[r], (long long)sorted[r].second, sorted[r].first, gap);
                    CHECK(gap <= 1e-12 * std::max(1.0, std::fabs(sorted[r].first)));
                    ++mism;
                }
            CHECK(mism <= 4);
            std::set<BlockId> uniq(plan.ranked_ids.begin(), plan.ranked_ids.end());
            CHECK(uniq.size() == static_cast<std::size_t>(n));
            const PSAResult run = psa_attention(q, ids, cfg, store);
            for (std::size_t r = 0; r < run.blocks_processed; ++r) CHECK(run.processed_ids[r] == plan.ranked_ids[r]);
        }
    }
    std::printf("OK %d\n", g_checks);
    return 0;
}
