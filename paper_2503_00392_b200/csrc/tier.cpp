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
#include <cstring>
#include <list>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "device.h"
#include "kernels.cuh"
#include "psattn_b200.h"

struct psattn_tier {
    psattn_tier_desc desc{};
    psattn_pool* pool = nullptr;
    struct Domain {
        size_t capacity = 0;
        std::list<int64_t> order;  // front = most recent
        std::unordered_map<int64_t, std::list<int64_t>::iterator> pos;
        std::vector<int32_t> free_slots;
    };
    std::vector<Domain> domains;
    std::vector<int32_t> loc;    // host mirror of the device location table
    std::vector<int32_t> layer;  // -1 = no such block
    std::vector<int32_t> ntok;
    std::vector<int64_t> owner;
    std::unordered_map<int64_t, std::vector<int64_t>> owned;
    std::vector<psattn_cache_stats> per_layer;
    psattn_cache_stats total{};
    uint64_t h2d_bytes = 0;
    std::vector<int64_t> pending;  // blocks (re)inserted into the fast tier since the last install
    std::mutex mu;
};

namespace {

using psa::fail;

psattn_tier::Domain& domain_of(psattn_tier* t, int32_t layer) {
    return t->desc.pool_policy == PSATTN_POOL_UNIFIED ? t->domains[0] : t->domains[(size_t)layer];
}

// insert_fast (reference store.cpp:44-57): evicts the LRU/FIFO tail when full; the new
// block takes the victim's HBM slot (or a free one).
void insert_fast(psattn_tier* t, int64_t id) {
    psattn_tier::Domain& d = domain_of(t, t->layer[(size_t)id]);
    if (d.capacity == 0) return;
    int32_t slot;
    if (d.pos.size() == d.capacity) {
        const int64_t victim = d.order.back();
        d.order.pop_back();
        d.pos.erase(victim);
        slot = t->loc[(size_t)victim];
        t->loc[(size_t)victim] = -1;
        t->total.evictions += 1;
        t->per_layer[(size_t)t->layer[(size_t)victim]].evictions += 1;
    } else {
        slot = d.free_slots.back();
        d.free_slots.pop_back();
    }
    d.order.push_front(id);
    d.pos.emplace(id, d.order.begin());
    t->loc[(size_t)id] = slot;
    t->pending.push_back(id);
}

// load_block's accounting (reference store.cpp:80-124).
void load(psattn_tier* t, int64_t id) {
    const int32_t l = t->layer[(size_t)id];
    psattn_tier::Domain& d = domain_of(t, l);
    auto& ls = t->per_layer[(size_t)l];
    auto it = d.pos.find(id);
    if (it != d.pos.end()) {
        t->total.hits += 1;
        ls.hits += 1;
        if (t->desc.eviction_policy == PSATTN_EVICT_LRU) d.order.splice(d.order.begin(), d.order, it->second);
        return;
    }
    const uint64_t bytes = 2ull * (uint64_t)t->ntok[(size_t)id] * (uint64_t)t->desc.dim * sizeof(float);
    t->total.misses += 1;
    ls.misses += 1;
    t->total.bytes_transferred += bytes;
    ls.bytes_transferred += bytes;
    insert_fast(t, id);
}

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
    t->per_layer.assign((size_t)desc->n_layers, psattn_cache_stats{});
    if (desc->pool_policy == PSATTN_POOL_UNIFIED) {
        t->domains.resize(1);
        t->domains[0].capacity = (size_t)desc->fast_slots;
    } else {
        t->domains.resize((size_t)desc->n_layers);
        const size_t per = (size_t)desc->fast_slots / (size_t)desc->n_layers;
        for (auto& d : t->domains) d.capacity = per;
    }
    // HBM slots: [0, cap) for the unified domain, [l*per, (l+1)*per) for layer l
    int32_t next = 0;
    for (auto& d : t->domains) {
        for (size_t i = 0; i < d.capacity; ++i) d.free_slots.push_back(next + (int32_t)(d.capacity - 1 - i));
        next += (int32_t)d.capacity;
    }
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
    for (int64_t i = 0; i < n; ++i) insert_fast(t, blocks[i]);  // write-allocate (store.cpp:75-77)
    return install_pending(t, st);
}

int psattn_tier_release_request(psattn_tier* t, int64_t owner) {
    if (!t) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_release_request: null tier");
    std::lock_guard<std::mutex> lk(t->mu);
    auto it = t->owned.find(owner);
    if (it == t->owned.end()) return fail(PSATTN_ERR_NOT_FOUND, "release_request: unknown request " + std::to_string(owner));
    for (int64_t id : it->second) {
        if (t->layer[(size_t)id] < 0) continue;
        psattn_tier::Domain& d = domain_of(t, t->layer[(size_t)id]);
        auto p = d.pos.find(id);
        if (p != d.pos.end()) {
            d.order.erase(p->second);
            d.pos.erase(p);
            d.free_slots.push_back(t->loc[(size_t)id]);
            t->loc[(size_t)id] = -1;
        }
        t->layer[(size_t)id] = -1;
    }
    t->owned.erase(it);
    return install_pending(t, nullptr);
}

int psattn_tier_run_batch(psattn_tier* t, const psattn_batch* b, void* workspace, void* stream) {
    if (!t || !b) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_run_batch: null argument");
    std::lock_guard<std::mutex> lk(t->mu);
    cudaStream_t st = (cudaStream_t)stream;
    int rc = psattn_run_batch(t->pool, b, workspace, stream);
    if (rc) return rc;
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
    // lockstep rounds (psa_attention_batched): every live query loads its next microbatch
    const int64_t m = std::max<int32_t>(b->microbatch_size, 1);
    std::vector<int64_t> cur((size_t)nq, 0);
    for (bool live = true; live;) {
        live = false;
        for (int64_t qi = 0; qi < nq; ++qi) {
            const int64_t u = qi / b->group, h = qi % b->group;
            const int64_t n = off[(size_t)u + 1] - off[(size_t)u];
            const int64_t end = std::min(cur[(size_t)qi] + m, bp[(size_t)qi]);
            const int64_t hb = off[(size_t)u] * b->group + h * n;
            for (int64_t r = cur[(size_t)qi]; r < end; ++r) load(t, slots[(size_t)(off[(size_t)u] + rpos[(size_t)(hb + r)])]);
            cur[(size_t)qi] = end;
            if (end < bp[(size_t)qi]) live = true;
        }
    }
    return install_pending(t, st);
}

int psattn_tier_stats(psattn_tier* t, int32_t layer, psattn_cache_stats* out) {
    if (!t || !out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_stats: null argument");
    std::lock_guard<std::mutex> lk(t->mu);
    if (layer < -1 || layer >= t->desc.n_layers) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tier_stats: bad layer");
    *out = layer < 0 ? t->total : t->per_layer[(size_t)layer];
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
