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
};

}  // namespace psattn::detail
