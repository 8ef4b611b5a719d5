// tier.cpp — two-tier KV block store on B200: the paper's KV-cache
// manager with the reference TieredBlockStore's observable semantics (store.cpp:11-205):
//
//   backing tier  every block's K/V in pinned, device-mapped host memory (the reference's
//                 backing unordered_map, store.hpp:111-117);
//   fast tier     `fast_slots` HBM slots managed as one Unified LRU/FIFO domain shared by
//                 all layers, or LayerPartitioned floor(cap / L) slots per layer
//                 (store.cpp:11-22);
//   metadata      resident in HBM for every block (paper §3.1: the estimator runs on GPU).
//
// A batch runs the normal device path (score -> lazy order -> progressive) with a location
// table: blocks resident in the fast tier are read from HBM, the others over PCIe/C2C from
// the host tier. Afterwards the loads are accounted in psa_attention_batched's order
// (reference engine.cpp:173-209: lockstep rounds over the queries, one microbatch of ranks
// each) through the LRU/FIFO domains — hits, misses, evictions and bytes exactly as the
// reference counts them — and the blocks that entered the fast tier are installed into
// their HBM slots by one copy kernel on the caller's stream.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "device.h"
#include "fast_tier.h"
#include "kernels.cuh"
#include "psattn_b200.h"

struct psattn_tier {
    psattn_tier_desc desc{};
    psattn_pool* pool = nullptr;
    std::unique_ptr<psa::FastTier> fast;          // residency + counters (fast_tier.h)
    std::vector<std::vector<int32_t>> free_slots;  // free HBM slots per domain
    std::vector<int32_t> loc;    // host mirror of the device location table
    std::vector<int32_t> layer;  // -1 = no such block
    std::vector<int32_t> ntok;
    std::vector<int64_t> owner;
    std::unordered_map<int64_t, std::vector<int64_t>> owned;
    uint64_t h2d_bytes = 0;
    std::vector<int64_t> pending;  // blocks (re)inserted into the fast tier since the last install
    std::mutex mu;
};

namespace {

using psa::fail;

size_t domain_index(const psattn_tier* t, int32_t layer) {
    return t->desc.pool_policy == PSATTN_POOL_UNIFIED ? 0 : (size_t)layer;
}

// Slot bookkeeping after an admission into the fast tier: the new block takes the victim's
// HBM slot, or a free slot of its domain.
void place(psattn_tier* t, int64_t id, const std::optional<int64_t>& victim) {
    if (!t->fast->resident(id, t->layer[(size_t)id])) return;  // zero-capacity domain
    int32_t slot;
    if (victim) {
        slot = t->loc[(size_t)*victim];
        t->loc[(size_t)*victim] = -1;
    } else {
        auto& fl = t->free_slots[domain_index(t, t->layer[(size_t)id])];
        slot = fl.back();
        fl.pop_back();
    }
    t->loc[(size_t)id] = slot;
    t->pending.push_back(id);
}

int32_t layer_lookup(const psattn_tier* t, int64_t id) { return t->layer[(size_t)id]; }

// put_block's write-allocate (reference store.cpp:75-77).
void put_fast(psattn_tier* t, int64_t id) {
    place(t, id, t->fast->put(id, t->layer[(size_t)id], [t](int64_t v) { return layer_lookup(t, v); }));
}

// load_block's accounting (reference store.cpp:80-124); true on a hit.
bool load(psattn_tier* t, int64_t id) {
    const uint64_t bytes = 2ull * (uint64_t)t->ntok[(size_t)id] * (uint64_t)t->desc.dim * sizeof(float);
    const auto a = t->fast->access(id, t->layer[(size_t)id], bytes, [t](int64_t v) { return layer_lookup(t, v); });
    if (!a.hit) place(t, id, a.evicted);
    return a.hit;
}

psattn_cache_stats to_c(const psa::TierCounters& c) { return psattn_cache_stats{c.hits, c.misses, c.evictions, c.bytes}; }

// Installs every pending block that is still resident and publishes the location table.
int install_pending(psattn_tier* t, cudaStream_t st) {
    std::vector<int64_t> ids;
    std::vector<int32_t> dst;
    std::sort(t->pending.begin(), t->pending.end());
    t->pending.erase(std::unique(t->pending.begin(), t->pending.end()), t->pending.end());
    for (int64_t id : t->pending)
        if (t->loc[(size_t)id] >= 0) {
            ids.push_back(id);
            dst.push_back(t->loc[(size_t)id]);
        }
    t->pending.clear();
    const psa::PoolView& v = psa::pool_view(t->pool);
    cudaError_t e;
    if (!ids.empty()) {
        int64_t* d_ids = nullptr;
        if ((e = cudaMallocAsync(&d_ids, ids.size() * 12, st)) != cudaSuccess) return psa::cuda_fail(e, "tier install");
        int32_t* d_dst = reinterpret_cast<int32_t*>(d_ids + ids.size());
        cudaMemcpyAsync(d_ids, ids.data(), ids.size() * 8, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_dst, dst.data(), dst.size() * 4, cudaMemcpyHostToDevice, st);
        if ((e = psa::launch_install(v, d_ids, d_dst, (int64_t)ids.size(), st)) != cudaSuccess)
            return psa::cuda_fail(e, "tier install");
        cudaFreeAsync(d_ids, st);
        t->h2d_bytes += ids.size() * (uint64_t)v.slot_bytes;
    }
    cudaMemcpyAsync(psa::pool_loc(t->pool), t->loc.data(), t->loc.size() * 4, cudaMemcpyHostToDevice, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return psa::cuda_fail(e, "tier install");
    return PSATTN_OK;
}

}  // namespace

extern "C" {

int psattn_tier_create(const psattn_tier_desc* desc, psattn_tier** out) {
    if (!desc || !out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_create: null argument");
    if (desc->n_layers <= 0) return fail(PSATTN_ERR_INVALID_ARGUMENT, "TieredBlockStore: n_layers must be positive");
    if (desc->n_blocks <= 0 || desc->n_blocks > INT32_MAX)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_create: n_blocks must be in [1, 2^31)");
    if (desc->fast_slots < 0 || desc->fast_slots > INT32_MAX)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_create: fast_slots must be in [0, 2^31)");
    if (desc->pool_policy != PSATTN_POOL_UNIFIED && desc->pool_policy != PSATTN_POOL_LAYER_PARTITIONED)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_create: unknown pool policy");
    if (desc->eviction_policy != PSATTN_EVICT_LRU && desc->eviction_policy != PSATTN_EVICT_FIFO)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_create: unknown eviction policy");
    psattn_pool_desc pd{};
    pd.dim = desc->dim;
    pd.block_tokens = desc->block_tokens;
    pd.kv_dtype = desc->kv_dtype;
    psattn_pool* pool = nullptr;
    int rc = psa::pool_create_tiered(&pd, desc->n_blocks, desc->fast_slots, &pool);
    if (rc) return rc;
    auto* t = new psattn_tier();
    t->desc = *desc;
    t->pool = pool;
    const size_t nb = (size_t)desc->n_blocks;
    t->loc.assign(nb, -1);
    t->layer.assign(nb, -1);
    t->ntok.assign(nb, 0);
    t->owner.assign(nb, 0);
    const bool per_layer = desc->pool_policy != PSATTN_POOL_UNIFIED;
    t->fast = std::make_unique<psa::FastTier>((size_t)desc->fast_slots, desc->n_layers, per_layer,
                                              desc->eviction_policy == PSATTN_EVICT_LRU, (size_t)nb);
    // HBM slots: [0, cap) for the unified domain, [l*per, (l+1)*per) for layer l
    const size_t n_dom = per_layer ? (size_t)desc->n_layers : 1;
    const size_t per = per_layer ? (size_t)desc->fast_slots / (size_t)desc->n_layers : (size_t)desc->fast_slots;
    t->free_slots.assign(n_dom, {});
    for (size_t dd = 0; dd < n_dom; ++dd)
        for (size_t i = 0; i < per; ++i) t->free_slots[dd].push_back((int32_t)(dd * per + per - 1 - i));
    *out = t;
    return PSATTN_OK;
}

void psattn_tier_destroy(psattn_tier* t) {
    if (!t) return;
    psattn_pool_destroy(t->pool);
    delete t;
}

int psattn_tier_put_blocks(psattn_tier* t, int64_t n, const int64_t* blocks, const int32_t* layers,
                           const int32_t* ntok, const int64_t* owners, const float* keys, const float* values) {
    if (!t || !blocks || !layers || !ntok || !keys || !values)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_put_blocks: null argument");
    std::lock_guard<std::mutex> lk(t->mu);
    for (int64_t i = 0; i < n; ++i) {
        if (blocks[i] < 0 || blocks[i] >= t->desc.n_blocks)
            return fail(PSATTN_ERR_RUNTIME, "put_block: block index out of the backing tier's range");
        if (layers[i] < 0 || layers[i] >= t->desc.n_layers) return fail(PSATTN_ERR_RUNTIME, "put_block: layer_id out of range");
        if (ntok[i] <= 0) return fail(PSATTN_ERR_RUNTIME, "build_metadata: empty block");
        if (ntok[i] > t->desc.block_tokens) return fail(PSATTN_ERR_RUNTIME, "put_block: block larger than block_tokens");
        if (t->layer[(size_t)blocks[i]] >= 0)
            return fail(PSATTN_ERR_RUNTIME, "put_block: duplicate block id " + std::to_string(blocks[i]));
    }
    psa::pool_pack_into(t->pool, n, blocks, ntok, keys, values);
    const psa::PoolView& v = psa::pool_view(t->pool);
    cudaStream_t st = nullptr;
    std::vector<int32_t> idx32(blocks, blocks + n);
    int32_t* d_idx = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&d_idx, (size_t)n * 8 + 8)) != cudaSuccess) return psa::cuda_fail(e, "tier put");
    cudaMemcpy(d_idx, idx32.data(), (size_t)n * 4, cudaMemcpyHostToDevice);
    for (int64_t i = 0; i < n; ++i) {
        t->layer[(size_t)blocks[i]] = layers[i];
        t->ntok[(size_t)blocks[i]] = ntok[i];
        t->owner[(size_t)blocks[i]] = owners ? owners[i] : 0;
        t->owned[owners ? owners[i] : 0].push_back(blocks[i]);
    }
    cudaMemcpy(v.ntok, t->ntok.data(), t->ntok.size() * 4, cudaMemcpyHostToDevice);
    // metadata from the host copy (every new block is still non-resident in the device location table)
    e = psa::launch_meta_build(v, d_idx, 0, n, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    cudaFree(d_idx);
    if (e != cudaSuccess || e2 != cudaSuccess) return psa::cuda_fail(e != cudaSuccess ? e : e2, "tier metadata build");
    for (int64_t i = 0; i < n; ++i) put_fast(t, blocks[i]);  // write-allocate (store.cpp:75-77)
    return install_pending(t, st);
}

int psattn_tier_release_request(psattn_tier* t, int64_t owner) {
    if (!t) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_release_request: null tier");
    std::lock_guard<std::mutex> lk(t->mu);
    auto it = t->owned.find(owner);
    if (it == t->owned.end()) return fail(PSATTN_ERR_NOT_FOUND, "release_request: unknown request " + std::to_string(owner));
    for (int64_t id : it->second) {
        if (t->layer[(size_t)id] < 0) continue;
        if (t->fast->release(id, t->layer[(size_t)id])) {
            t->free_slots[domain_index(t, t->layer[(size_t)id])].push_back(t->loc[(size_t)id]);
            t->loc[(size_t)id] = -1;
        }
        t->layer[(size_t)id] = -1;
    }
    t->owned.erase(it);
    return install_pending(t, nullptr);
}

}  // extern "C"

namespace psa {

// One microbatch load's accounting (reference IterationStats, engine.hpp:57-62).
struct TierIter {
    int64_t blocks = 0, hits = 0, misses = 0;
};

// psattn_run_batch on the tier, then the load accounting. lockstep: psa_attention_batched's
// rounds (engine.cpp:173-209; one TierIter per round with blocks > 0); otherwise query by
// query like consecutive psa_attention / topk_attention calls (one TierIter per microbatch).
int tier_run_account(psattn_tier* t, const psattn_batch* b, void* workspace, cudaStream_t st, bool lockstep,
                     std::vector<TierIter>* iters) {
    static const bool prof = getenv("PSA_TIER_PROF") != nullptr;  // development: phase times to stderr
    const auto c0 = std::chrono::steady_clock::now();
    int rc = psattn_run_batch(t->pool, b, workspace, st);
    if (rc) return rc;
    if (prof) cudaStreamSynchronize(st);
    const auto c1 = std::chrono::steady_clock::now();
    const int64_t nq = (int64_t)b->n_units * b->group;
    const int64_t hbt = b->total_blocks * b->group;
    std::vector<int64_t> bp((size_t)nq), off((size_t)b->n_units + 1);
    std::vector<int32_t> rpos((size_t)hbt), slots((size_t)b->total_blocks);
    const int32_t* d_rpos = b->ranked_pos ? b->ranked_pos
                                          : reinterpret_cast<const int32_t*>(static_cast<char*>(workspace) +
                                                                             psa::ws_rpos_offset(b));
    cudaMemcpyAsync(bp.data(), b->blocks_processed, (size_t)nq * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(off.data(), b->list_off, off.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(rpos.data(), d_rpos, (size_t)hbt * 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(slots.data(), b->slots, (size_t)b->total_blocks * 4, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return psa::cuda_fail(e, "psattn_tier_run_batch");
    for (int32_t s : slots)
        if (s < 0 || s >= t->desc.n_blocks || t->layer[(size_t)s] < 0)
            return fail(PSATTN_ERR_NOT_FOUND, "load_block: unknown block id " + std::to_string(s));
    const int64_t m = std::max<int32_t>(b->microbatch_size, 1);
    std::vector<int64_t> cur((size_t)nq, 0);
    auto load_mb = [&](int64_t qi, TierIter& it) {  // next microbatch of query qi
        const int64_t u = qi / b->group, h = qi % b->group;
        const int64_t n = off[(size_t)u + 1] - off[(size_t)u];
        const int64_t end = std::min(cur[(size_t)qi] + m, bp[(size_t)qi]);
        const int64_t hb = off[(size_t)u] * b->group + h * n;
        for (int64_t r = cur[(size_t)qi]; r < end; ++r) {
            if (load(t, slots[(size_t)(off[(size_t)u] + rpos[(size_t)(hb + r)])])) ++it.hits;
            else ++it.misses;
            ++it.blocks;
        }
        cur[(size_t)qi] = end;
        return end < bp[(size_t)qi];
    };
    if (lockstep) {
        // rounds over the live queries in query order (psa_attention_batched, engine.cpp:188-207);
        // finished queries leave the list, so a round costs only its loads
        std::vector<int64_t> act;
        act.reserve((size_t)nq);
        for (int64_t qi = 0; qi < nq; ++qi)
            if (cur[(size_t)qi] < bp[(size_t)qi]) act.push_back(qi);
        while (!act.empty()) {
            TierIter round;
            size_t w = 0;
            for (size_t k = 0; k < act.size(); ++k)
                if (load_mb(act[k], round)) act[w++] = act[k];
            act.resize(w);
            if (iters && round.blocks > 0) iters->push_back(round);
        }
    } else {
        for (int64_t qi = 0; qi < nq; ++qi)
            for (bool more = cur[(size_t)qi] < bp[(size_t)qi]; more;) {
                TierIter it;
                more = load_mb(qi, it);
                if (iters) iters->push_back(it);
            }
    }
    const auto c2 = std::chrono::steady_clock::now();
    rc = install_pending(t, st);
    if (prof) {
        const auto c3 = std::chrono::steady_clock::now();
        auto ms = [](auto a, auto b2) { return std::chrono::duration<double, std::milli>(b2 - a).count(); };
        fprintf(stderr, "tier phases ms: batch %.3f  d2h+replay %.3f  install %.3f\n", ms(c0, c1), ms(c1, c2), ms(c2, c3));
    }
    return rc;
}

}  // namespace psa

extern "C" {

int psattn_tier_run_batch(psattn_tier* t, const psattn_batch* b, void* workspace, void* stream) {
    if (!t || !b) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_run_batch: null argument");
    std::lock_guard<std::mutex> lk(t->mu);
    return psa::tier_run_account(t, b, workspace, (cudaStream_t)stream, true, nullptr);
}

int psattn_tier_stats(psattn_tier* t, int32_t layer, psattn_cache_stats* out) {
    if (!t || !out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_stats: null argument");
    std::lock_guard<std::mutex> lk(t->mu);
    if (layer < -1 || layer >= t->desc.n_layers) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_stats: bad layer");
    *out = to_c(layer < 0 ? t->fast->total() : t->fast->layer(layer));
    return PSATTN_OK;
}

int psattn_tier_resident(psattn_tier* t, int64_t block, int32_t* out_slot) {
    if (!t || !out_slot) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_resident: null argument");
    std::lock_guard<std::mutex> lk(t->mu);
    if (block < 0 || block >= t->desc.n_blocks || t->layer[(size_t)block] < 0)
        return fail(PSATTN_ERR_NOT_FOUND, "unknown block id " + std::to_string(block));
    *out_slot = t->loc[(size_t)block];
    return PSATTN_OK;
}

int psattn_tier_h2d_bytes(psattn_tier* t, uint64_t* out) {
    if (!t || !out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_h2d_bytes: null argument");
    std::lock_guard<std::mutex> lk(t->mu);
    *out = t->h2d_bytes;
    return PSATTN_OK;
}

psattn_pool* psattn_tier_pool(psattn_tier* t) { return t ? t->pool : nullptr; }

}  // extern "C"

// =============================================================================
// Batched serving loop on the GPU path (reference run_serving,
// serving.cpp:100-229): FCFS head-only admission while one microbatch per live
// (request, layer) fits the fast tier, then one decode step for every live request
// layer by layer — each layer ONE device batch over the live requests through the
// two-tier store — retirement and release. The simulated TBT cost model
// (iteration_costs + simulate_pipeline, serving.cpp:85-96, pipeline.cpp:153-175)
// is reproduced from the device run's hit/miss series, so the reports compare with
// the reference's byte for byte; the device time of the attention launches is
// measured alongside (CUDA events).
// =============================================================================
namespace {

struct ServeRequest {
    int64_t id = 0;
    double arrival_s = 0.0;
    int32_t steps = 0;
    std::vector<std::vector<int64_t>> layer_blocks;  // per layer, block ids in sequence order
    std::vector<int64_t> ids;
    std::vector<int32_t> layers, ntok;
    std::vector<float> keys, values;  // [nb][B][d]
    std::vector<float> queries;       // [steps][L][d]
};

struct DevScratch {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t n) {
        if (n > cap) {
            cudaFree(p);
            p = nullptr;
            cap = 0;
            if (cudaMalloc(&p, n) != cudaSuccess) return nullptr;
            cap = n;
        }
        return p;
    }
    ~DevScratch() { cudaFree(p); }
};

double percentile_nr(std::vector<double> v, double p) {
    std::sort(v.begin(), v.end());
    if (p == 0.0) return v.front();
    const auto rank = static_cast<size_t>(std::ceil(p / 100.0 * static_cast<double>(v.size())));
    return v[rank - 1];
}

}  // namespace

struct psattn_serving {
    psattn_tier_desc store{};
    psattn_config engine{};
    psattn_serving_cost cost{};
    std::vector<ServeRequest> requests;
};

extern "C" {

int psattn_serving_create(const psattn_tier_desc* store, const psattn_config* engine, const psattn_serving_cost* cost,
                          psattn_serving** out) {
    if (!store || !engine || !cost || !out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_serving_create: null argument");
    auto* s = new psattn_serving();
    s->store = *store;
    s->engine = *engine;
    s->cost = *cost;
    *out = s;
    return PSATTN_OK;
}

void psattn_serving_destroy(psattn_serving* s) { delete s; }

int psattn_serving_add_request(psattn_serving* s, int64_t request_id, double arrival_s, int32_t decode_steps,
                               int32_t n_layers, int64_t blocks_per_layer, const int64_t* layer_blocks,
                               int64_t n_blocks, const int64_t* block_ids, const int32_t* block_layers,
                               const int32_t* ntok, const float* keys, const float* values, const float* queries) {
    if (!s || !layer_blocks || !block_ids || !block_layers || !ntok || !keys || !values || !queries)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_serving_add_request: null argument");
    if (n_layers != s->store.n_layers) return fail(PSATTN_ERR_RUNTIME, "serving: requests disagree on layer count");
    ServeRequest r;
    r.id = request_id;
    r.arrival_s = arrival_s;
    r.steps = decode_steps;
    const int64_t d = s->store.dim, B = s->store.block_tokens;
    for (int32_t l = 0; l < n_layers; ++l)
        r.layer_blocks.emplace_back(layer_blocks + l * blocks_per_layer, layer_blocks + (l + 1) * blocks_per_layer);
    r.ids.assign(block_ids, block_ids + n_blocks);
    r.layers.assign(block_layers, block_layers + n_blocks);
    r.ntok.assign(ntok, ntok + n_blocks);
    r.keys.assign(keys, keys + n_blocks * B * d);
    r.values.assign(values, values + n_blocks * B * d);
    r.queries.assign(queries, queries + (int64_t)decode_steps * n_layers * d);
    s->requests.push_back(std::move(r));
    return PSATTN_OK;
}

int psattn_serving_run(psattn_serving* s, int32_t method, double epsilon, int64_t k, psattn_serving_report* out) {
    if (!s || !out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_serving_run: null argument");
    if (s->requests.empty()) return fail(PSATTN_ERR_RUNTIME, "serving: empty request list");
    if (method < 0 || method > 2) return fail(PSATTN_ERR_INVALID_ARGUMENT, "serving: unknown method");
    if (method == 1 && k < 1) return fail(PSATTN_ERR_RUNTIME, "serving: top-k method needs k >= 1");
    psattn_config cfg = s->engine;
    if (method == 0) cfg.epsilon = epsilon;
    if (method == 2) cfg.epsilon = 1.0;
    if (!(cfg.epsilon > 0.0) || cfg.epsilon > 1.0) return fail(PSATTN_ERR_INVALID_ARGUMENT, "config: epsilon must be in (0, 1]");
    if (cfg.microbatch_size < 1) return fail(PSATTN_ERR_INVALID_ARGUMENT, "config: microbatch_size must be >= 1");
    const int32_t L = s->store.n_layers;
    const int64_t d = s->store.dim;
    // block id -> backing-tier index (every request's blocks, in request order)
    std::unordered_map<int64_t, int64_t> index;
    int64_t nb = 0;
    for (const auto& r : s->requests)
        for (int64_t id : r.ids) index.emplace(id, nb++);
    psattn_tier_desc td = s->store;
    td.n_blocks = nb;
    psattn_tier* t = nullptr;
    int rc = psattn_tier_create(&td, &t);
    if (rc) return rc;
    struct TierGuard {
        psattn_tier* t;
        ~TierGuard() { psattn_tier_destroy(t); }
    } guard{t};
    // Admission (serving.cpp:31-81)
    const size_t m = (size_t)cfg.microbatch_size, cap = (size_t)td.fast_slots;
    const bool unified = td.pool_policy == PSATTN_POOL_UNIFIED;
    const size_t layer_cap = cap / (unified ? 1 : (size_t)L);
    size_t reserved = 0;  // per layer in partitioned mode (all layers reserve alike)
    auto fits = [&] { return unified ? reserved * L + m * L <= cap : reserved + m <= layer_cap; };
    const bool solo = unified ? m * L <= cap : m <= layer_cap;
    for (const auto& r : s->requests)
        if (!solo)
            return fail(PSATTN_ERR_RUNTIME, "unschedulable request " + std::to_string(r.id) +
                                                ": one microbatch per layer does not fit the fast pool");
    std::vector<size_t> pending;
    for (size_t i = 0; i < s->requests.size(); ++i) pending.push_back(i);
    size_t ph = 0;
    struct Live {
        size_t r;
        int32_t step;
    };
    std::vector<Live> live;
    std::vector<double> tbt, blocks, cov;
    uint64_t blocks_sum = 0, total_sum = 0;
    double now = 0.0, model_seq = 0.0, model_pipe = 0.0, gpu_ms = 0.0;
    int64_t steps = 0, completed = 0, launches = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    DevScratch d_in, d_out, d_ws;
    std::vector<char> h_in;
    while (ph < pending.size() || !live.empty()) {
        while (ph < pending.size() && s->requests[pending[ph]].arrival_s * 1000.0 <= now && fits()) {
            const ServeRequest& r = s->requests[pending[ph++]];
            reserved += m;
            std::vector<int64_t> bi(r.ids.size()), own(r.ids.size(), r.id);
            for (size_t i = 0; i < r.ids.size(); ++i) bi[i] = index.at(r.ids[i]);
            if ((rc = psattn_tier_put_blocks(t, (int64_t)bi.size(), bi.data(), r.layers.data(), r.ntok.data(), own.data(),
                                             r.keys.data(), r.values.data())))
                return rc;
            live.push_back({(size_t)(&r - s->requests.data()), 0});
        }
        if (live.empty()) {
            if (ph >= pending.size()) break;
            now = std::max(now, s->requests[pending[ph]].arrival_s * 1000.0);
            continue;
        }
        double step_cost = 0.0;
        for (int32_t l = 0; l < L; ++l) {
            // one device batch: unit i = live request i's layer-l list (ascending id), its step query
            const int32_t nu = (int32_t)live.size();
            std::vector<std::vector<int64_t>> sorted(nu);
            std::vector<int64_t> off(nu + 1, 0);
            int64_t maxn = 0;
            for (int32_t i = 0; i < nu; ++i) {
                sorted[i] = s->requests[live[i].r].layer_blocks[l];
                std::sort(sorted[i].begin(), sorted[i].end());
                off[i + 1] = off[i] + (int64_t)sorted[i].size();
                maxn = std::max<int64_t>(maxn, (int64_t)sorted[i].size());
            }
            const int64_t tot = off[nu];
            const size_t qb = (size_t)nu * d * 4, sb = (size_t)tot * 4, ob = (size_t)(nu + 1) * 8;
            h_in.resize(qb + sb + ob);
            for (int32_t i = 0; i < nu; ++i) {
                const ServeRequest& r = s->requests[live[i].r];
                std::memcpy(h_in.data() + (size_t)i * d * 4, r.queries.data() + ((size_t)live[i].step * L + l) * d, d * 4);
                for (size_t j = 0; j < sorted[i].size(); ++j)
                    reinterpret_cast<int32_t*>(h_in.data() + qb)[off[i] + (int64_t)j] = (int32_t)index.at(sorted[i][j]);
            }
            std::memcpy(h_in.data() + qb + sb, off.data(), ob);
            char* din = static_cast<char*>(d_in.get(h_in.size()));
            const size_t oo = (size_t)nu * d * 4, o8 = (size_t)nu * 8, o4 = (size_t)nu * 4;
            char* dout = static_cast<char*>(d_out.get(oo + 3 * o8 + o4 + (size_t)tot * 4 + 64));
            if (!din || !dout) return fail(PSATTN_ERR_RUNTIME, "serving: device allocation failed");
            cudaMemcpyAsync(din, h_in.data(), h_in.size(), cudaMemcpyHostToDevice, st);
            psattn_batch b{};
            b.n_units = nu;
            b.group = 1;
            b.dim = (int32_t)d;
            b.max_blocks = (int32_t)maxn;
            b.total_blocks = tot;
            b.q = reinterpret_cast<const float*>(din);
            b.slots = reinterpret_cast<const int32_t*>(din + qb);
            b.list_off = reinterpret_cast<const int64_t*>(din + qb + sb);
            b.epsilon = method == 1 ? 1.0 : cfg.epsilon;
            b.microbatch_size = cfg.microbatch_size;
            b.estimator = cfg.estimator;
            b.ranking_mode = cfg.ranking_mode;
            b.audit_coverage = cfg.audit_coverage;
            b.scale_override = cfg.scale_override;
            b.topk = method == 1 ? k : 0;
            b.out = reinterpret_cast<float*>(dout);
            b.blocks_processed = reinterpret_cast<int64_t*>(dout + oo);
            b.est_coverage = reinterpret_cast<double*>(dout + oo + o8);
            b.true_coverage = reinterpret_cast<double*>(dout + oo + 2 * o8);
            b.terminated = reinterpret_cast<int32_t*>(dout + oo + 3 * o8);
            b.ranked_pos = reinterpret_cast<int32_t*>(dout + oo + 3 * o8 + o4);
            void* ws = d_ws.get(psattn_batch_workspace_bytes(&b));
            if (!ws) return fail(PSATTN_ERR_RUNTIME, "serving: device allocation failed");
            std::vector<psa::TierIter> iters;
            cudaEventRecord(e0, st);
            // top-k: consecutive topk_attention calls (serving.cpp:168-174); else psa_attention_batched
            if ((rc = psa::tier_run_account(t, &b, ws, st, method != 1, &iters))) return rc;
            float ms = 0.0f;
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            gpu_ms += ms;  // attention launches + the (tiny) install of newly cached blocks
            ++launches;
            std::vector<int64_t> bp(nu);
            std::vector<double> est(nu), tc(nu);
            cudaMemcpy(bp.data(), b.blocks_processed, o8, cudaMemcpyDeviceToHost);
            cudaMemcpy(est.data(), b.est_coverage, o8, cudaMemcpyDeviceToHost);
            cudaMemcpy(tc.data(), b.true_coverage, o8, cudaMemcpyDeviceToHost);
            // cost model (iteration_costs + simulate_pipeline)
            double lf = 0.0, cf = 0.0, freed = 0.0, seq = 0.0;
            for (size_t i = 0; i < iters.size(); ++i) {
                const double load_ms = (double)iters[i].misses * s->cost.miss_cost_ms + (double)iters[i].hits * s->cost.hit_cost_ms;
                const double comp_ms = (double)iters[i].blocks * s->cost.compute_cost_ms;
                lf = (i == 0 ? 0.0 : freed) + load_ms;
                const double cs = std::max(lf, cf);
                freed = cs;
                cf = cs + comp_ms;
                seq += load_ms + comp_ms;
            }
            model_seq += seq;
            model_pipe += cf;
            step_cost += s->cost.overlap ? cf : seq;
            for (int32_t i = 0; i < nu; ++i) {
                blocks.push_back((double)bp[i]);
                cov.push_back(cfg.audit_coverage ? tc[i] : est[i]);
                blocks_sum += (uint64_t)bp[i];
                total_sum += (uint64_t)(off[i + 1] - off[i]);
            }
        }
        now += step_cost;
        ++steps;
        for (auto& lr : live) {
            tbt.push_back(step_cost);
            ++lr.step;
        }
        for (auto it = live.begin(); it != live.end();) {
            if (it->step >= s->requests[it->r].steps) {
                if ((rc = psattn_tier_release_request(t, s->requests[it->r].id))) return rc;
                reserved -= m;
                ++completed;
                it = live.erase(it);
            } else {
                ++it;
            }
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (blocks.empty()) return fail(PSATTN_ERR_RUNTIME, "serving produced no attention calls");
    psattn_serving_report rep{};
    double bm = 0.0, cm = 0.0, cmin = std::numeric_limits<double>::infinity();
    for (double x : blocks) bm += x;
    for (double x : cov) {
        cm += x;
        cmin = std::min(cmin, x);
    }
    psattn_tier_stats(t, -1, &rep.store_stats);
    const uint64_t acc = rep.store_stats.hits + rep.store_stats.misses;
    rep.mean_blocks = bm / (double)blocks.size();
    rep.p99_blocks = percentile_nr(blocks, 99.0);
    rep.kv_fraction = (double)blocks_sum / (double)total_sum;
    rep.mean_coverage = cm / (double)cov.size();
    rep.min_coverage = cmin;
    rep.hit_ratio = acc ? (double)rep.store_stats.hits / (double)acc : 0.0;
    rep.tbt_p50_ms = percentile_nr(tbt, 50.0);
    rep.tbt_p99_ms = percentile_nr(tbt, 99.0);
    rep.overlap_eff = model_pipe > 0.0 ? model_seq / model_pipe : 1.0;
    rep.n_calls = (int64_t)blocks.size();
    rep.n_steps = steps;
    rep.completed_requests = completed;
    rep.sim_time_ms = now;
    rep.gpu_ms = gpu_ms;
    rep.device_batches = launches;
    *out = rep;
    return PSATTN_OK;
}

}  // extern "C"
