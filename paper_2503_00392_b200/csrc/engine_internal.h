// engine_internal.h — host-side request/response of one device launch.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "psattn/engine.hpp"

namespace psattn::detail {

// n_units block lists; `group` queries per list (GQA). queries[u*group + h] is
// a host pointer to dim floats.
struct DeviceQueryBatch {
    std::vector<std::span<const BlockId>> lists;
    std::vector<const float*> queries;
    std::int32_t group = 1;
    std::int32_t dim = 0;
    PSAConfig cfg;
    std::size_t topk = 0;  // 0: PSA threshold stop
    bool rank_only = false;  // plan_blocks: full ranking of every rank (psattn_rank_batch), no attention
    bool want_union = false; // fill DeviceQueryResult::union_ids
};

struct DeviceQueryResult {
    std::int32_t dim = 0;
    double scale = 0.0;
    std::vector<float> out;  // [nq][dim]
    std::vector<std::int64_t> blocks_processed;
    std::vector<double> est;
    std::vector<double> true_cov;
    std::vector<std::int32_t> terminated;
    std::vector<std::vector<BlockId>> ranked_ids;   // per query: ranks < blocks_processed (all with rank_only)
    std::vector<std::vector<double>> oracle_ranked; // per query, fp64 masses of those ranks (oracle/audit)
    std::vector<std::vector<double>> iter_est;      // per query, estimate at each rank (boundaries valid)
    std::vector<BlockId> union_ids;  // want_union: ascending distinct ids processed by any query
};

// Per-head statistics of a multi-head run (the C ABI's psattn_run_stats).
struct HeadStats {
    std::uint64_t blocks_processed = 0, total_blocks = 0;
    double estimated_coverage = 0.0, true_coverage = -1.0;  // -1: not audited
    bool terminated_early = false;
};

// psa_attention_multi_head for the C ABI (psattn_run_multi_head): the same launch, accounting and
// errors, reading the caller's arrays in place and writing outputs [n_q_heads][dim] and per-head
// statistics without materialising PSAResults. Returns the fetched-union size.
std::size_t multi_head_into(const float* q, std::int32_t n_q_heads, std::int32_t dim, const BlockId* ids,
                            const std::int64_t* list_off, std::int32_t n_kv_heads, const PSAConfig& cfg,
                            TieredBlockStore& store, float* out, HeadStats* stats);

}  // namespace psattn::detail
