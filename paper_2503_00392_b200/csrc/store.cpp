// store.cpp — TieredBlockStore over the device pool (B200 build).
//
// Blocks: one device pool per head dim (psattn_pool, slots shared by all layers). The
// fast-tier hit/miss/eviction/byte accounting with the reference's observable semantics
// (store.cpp:11-124 of the reference) is psa::FastTier (fast_tier.h), shared with the two-tier
// store (tier.cpp); this file adds the block records, the device copies and the access trace.
#include "psattn/store.hpp"

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>

#include <cuda_runtime.h>

#include "device.h"
#include "engine_internal.h"
#include "block_table.h"
#include "fast_tier.h"
#include "psattn_b200.h"

namespace psattn {

namespace {
[[noreturn]] void throw_last(int rc) {
    if (rc == PSATTN_ERR_NOT_FOUND) throw NotFoundError(psa::last_error());
    if (rc == PSATTN_ERR_INVALID_ARGUMENT) throw ConfigError(psa::last_error());
    throw Error(psa::last_error());
}
void check_rc(int rc) {
    if (rc != PSATTN_OK) throw_last(rc);
}
void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Growable device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t n) {
        if (n > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            check_cuda(cudaMalloc(&p, std::max<size_t>(n, 256)), "device buffer");
            cap = std::max<size_t>(n, 256);
        }
        return p;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// Growable pinned host buffer.
struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t n) {
        if (n > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            check_cuda(cudaMallocHost(&p, std::max<size_t>(n, 256)), "pinned buffer");
            cap = std::max<size_t>(n, 256);
        }
        return p;
    }
    ~HostBuf() {
        if (p) cudaFreeHost(p);
    }
};

size_t align256(size_t x) { return (x + 255) / 256 * 256; }
}  // namespace

struct TieredBlockStore::DevicePool {
    psattn_pool* pool = nullptr;
    bool bf16 = false;  // lossless bf16 storage: every block put so far is exactly representable
    std::int64_t next_slot = 0;
    std::vector<std::int64_t> free_slots;
    ~DevicePool() { psattn_pool_destroy(pool); }
};

struct TieredBlockStore::DeviceState {
    cudaStream_t stream = nullptr;
    DevBuf in, outb, ws;
    HostBuf h_in, h_out;
    // Captured launch sequences of recent query shapes (psattn_graph_*): a repeated call with the
    // same pool, batch descriptor (sizes, config, device buffers) and launch knobs replays its graph
    // instead of re-issuing ~15 launches and memsets.
    struct Graph {
        std::vector<unsigned char> key;
        psattn_graph* g = nullptr;
    };
    std::array<Graph, 4> graphs;
    std::size_t graph_next = 0;
    ~DeviceState() {
        for (auto& x : graphs) psattn_graph_destroy(x.g);
        if (stream) cudaStreamDestroy(stream);
    }
    int launch(psattn_pool* pool, const psattn_batch& b, void* ws_ptr) {
        const std::uint64_t gen = psa::launch_config_generation();
        if (gen == ~0ull) return psattn_run_batch(pool, &b, ws_ptr, stream);  // profiling: per-stage events
        psattn_pool_desc desc{};
        psattn_pool_get_desc(pool, &desc);
        std::vector<unsigned char> key(sizeof(pool) + sizeof(desc) + sizeof(b) + sizeof(ws_ptr) + sizeof(gen));
        unsigned char* k = key.data();
        auto put = [&k](const void* p, std::size_t n) {
            std::memcpy(k, p, n);
            k += n;
        };
        put(&pool, sizeof(pool));
        put(&desc, sizeof(desc));
        put(&b, sizeof(b));
        put(&ws_ptr, sizeof(ws_ptr));
        put(&gen, sizeof(gen));
        for (auto& x : graphs)
            if (x.g && x.key == key) return psattn_graph_launch(x.g, stream);
        Graph& slot = graphs[graph_next++ % graphs.size()];
        psattn_graph_destroy(slot.g);
        slot.g = nullptr;
        slot.key.clear();
        const int rc = psattn_graph_create(pool, &b, ws_ptr, stream, &slot.g);
        if (rc != PSATTN_OK) return rc;
        slot.key = std::move(key);
        return psattn_graph_launch(slot.g, stream);
    }
};

TieredBlockStore::TieredBlockStore(const StoreOptions& options) : options_(options) {
    if (options_.n_layers <= 0) throw Error("TieredBlockStore: n_layers must be positive");
    tier_ = std::make_unique<psa::FastTier>(options_.fast_capacity_slots, options_.n_layers,
                                            options_.policy == PoolPolicy::LayerPartitioned,
                                            options_.eviction == EvictionPolicy::LRU, /*dense_ids=*/1);
    blocks_ = std::make_unique<psa::BlockTable<BlockRec>>();
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw Error("TieredBlockStore: no CUDA device (the B200 PSA path has no CPU fallback)");
    dev_ = std::make_unique<DeviceState>();
    check_cuda(cudaStreamCreateWithFlags(&dev_->stream, cudaStreamNonBlocking), "stream");
}

TieredBlockStore::~TieredBlockStore() = default;

std::int32_t TieredBlockStore::layer_of_handle(std::int64_t handle) const {
    return blocks_->at(handle).layer;
}

namespace {
// true when every value is exactly a bf16 (low 16 bits of the fp32 pattern zero): the block is
// then stored losslessly in bf16 — half the HBM, and the bf16 production kernels
bool bf16_exact(const float* x, std::size_t n) {
    std::uint32_t acc = 0;
    for (std::size_t i = 0; i < n; ++i) {
        std::uint32_t b;
        std::memcpy(&b, x + i, 4);
        acc |= b;
    }
    return (acc & 0xFFFFu) == 0;
}

bool lossless_bf16_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PSA_STORE_F32_ONLY");  // development: keep every pool fp32
        return !(e && e[0] == '1');
    }();
    return on;
}
}  // namespace

TieredBlockStore::DevicePool& TieredBlockStore::pool_for(std::int32_t dim, std::int32_t n_tokens, bool exact_bf16) {
    auto it = pools_.find(dim);
    if (it == pools_.end()) {
        auto dp = std::make_unique<DevicePool>();
        psattn_pool_desc desc{};
        desc.dim = dim;
        desc.block_tokens = std::max(n_tokens, 16);
        // the C/C++ API hands fp32 blocks and keeps them exact: bf16 while every block is exactly
        // representable in bf16 (e.g. an upcast bf16 KV cache), fp32 otherwise
        dp->bf16 = exact_bf16 && lossless_bf16_enabled();
        desc.kv_dtype = dp->bf16 ? PSATTN_KV_BF16 : PSATTN_KV_F32;
        desc.n_slots = 256;
        check_rc(psattn_pool_create(&desc, &dp->pool));
        it = pools_.emplace(dim, std::move(dp)).first;
    }
    DevicePool& dp = *it->second;
    psattn_pool_desc desc{};
    psattn_pool_get_desc(dp.pool, &desc);
    if (dp.bf16 && !exact_bf16) {
        // first block that bf16 cannot hold exactly: move every stored block to an fp32 pool (same
        // slots, values and metadata unchanged: bf16 -> fp32 is exact)
        psattn_pool_desc fd = desc;
        fd.kv_dtype = PSATTN_KV_F32;
        fd.block_tokens = std::max(desc.block_tokens, n_tokens);
        psattn_pool* fp = nullptr;
        check_rc(psattn_pool_create(&fd, &fp));
        std::vector<float> k, v;
        int rc = PSATTN_OK;
        blocks_->for_each([&](BlockId, const BlockRec& r) {
            if (r.dim != dim || rc != PSATTN_OK) return;
            const std::size_t cnt = static_cast<std::size_t>(r.n_tokens) * static_cast<std::size_t>(dim);
            k.resize(cnt);
            v.resize(cnt);
            const std::int32_t s32 = static_cast<std::int32_t>(r.slot), nt = r.n_tokens;
            rc = psa::read_slot(dp.pool, r.slot, r.n_tokens, k.data(), v.data());
            if (rc == PSATTN_OK) rc = psa::pool_put(fp, 1, &s32, &nt, k.data(), v.data(), 0, dev_->stream);
        });
        if (rc != PSATTN_OK) {
            psattn_pool_destroy(fp);
            check_rc(rc);
        }
        psattn_pool_destroy(dp.pool);
        dp.pool = fp;
        dp.bf16 = false;
        psattn_pool_get_desc(dp.pool, &desc);
    }
    if (n_tokens > desc.block_tokens) check_rc(psa::pool_grow(dp.pool, desc.n_slots, n_tokens));
    return dp;
}

void TieredBlockStore::put_block(std::shared_ptr<const KVBlock> block, RequestId owner) {
    if (!block) throw Error("put_block: null block");
    if (block->n_tokens <= 0) throw Error("build_metadata: empty block");
    if (block->dim <= 0 || block->dim > 256) throw Error("put_block: dim must be in [1, 256] on the device pool");
    if (block->n_tokens > 128) throw Error("put_block: blocks of more than 128 tokens are not supported by the device pool");
    const std::size_t nelem = static_cast<std::size_t>(block->n_tokens) * static_cast<std::size_t>(block->dim);
    if (block->keys.size() < nelem || block->values.size() < nelem) throw Error("put_block: short key/value arrays");
    const bool exact = bf16_exact(block->keys.data(), nelem) && bf16_exact(block->values.data(), nelem);
    std::lock_guard lock(mutex_);
    if (block->layer_id < 0 || block->layer_id >= options_.n_layers) throw Error("put_block: layer_id out of range");
    if (blocks_->contains(block->block_id))
        throw Error("put_block: duplicate block id " + std::to_string(block->block_id));
    DevicePool& dp = pool_for(block->dim, block->n_tokens, exact);
    std::int64_t slot;
    if (!dp.free_slots.empty()) {
        slot = dp.free_slots.back();
        dp.free_slots.pop_back();
    } else {
        psattn_pool_desc desc{};
        psattn_pool_get_desc(dp.pool, &desc);
        if (dp.next_slot >= desc.n_slots) check_rc(psa::pool_grow(dp.pool, desc.n_slots * 2, desc.block_tokens));
        slot = dp.next_slot++;
    }
    const std::int32_t s32 = static_cast<std::int32_t>(slot);
    const std::int32_t nt = block->n_tokens;
    check_rc(psa::pool_put(dp.pool, 1, &s32, &nt, block->keys.data(), block->values.data(), 0, dev_->stream));
    const std::int64_t h =
        blocks_->insert(block->block_id, BlockRec{block->dim, block->layer_id, block->n_tokens, slot, owner});
    owned_[owner].push_back(block->block_id);
    tier_->grow(blocks_->handles());
    tier_->put(h, block->layer_id, [this](std::int64_t v) { return layer_of_handle(v); });
}

bool TieredBlockStore::account_locked(BlockId id, std::int64_t handle, const BlockRec& rec) {
    const std::uint64_t payload = 2ull * static_cast<std::uint64_t>(rec.n_tokens) * rec.dim * sizeof(float);
    const auto a = tier_->access(handle, rec.layer, payload, [this](std::int64_t v) { return layer_of_handle(v); });
    if (trace_)  // seq,layer_id,block_id,hit|miss,evicted_id|-
        *trace_ << trace_seq_++ << ',' << rec.layer << ',' << id << ',' << (a.hit ? "hit," : "miss,")
                << (a.evicted ? std::to_string(blocks_->id_of(*a.evicted)) : std::string("-")) << '\n';
    return !a.hit;
}

std::pair<std::uint64_t, std::uint64_t> TieredBlockStore::account_loads(std::span<const BlockId> ids) {
    std::vector<std::pair<std::uint64_t, std::uint64_t>> hm;
    const std::size_t run = ids.size();
    account_runs(ids, std::span<const std::size_t>(&run, 1), hm);
    return hm[0];
}

void TieredBlockStore::account_runs(std::span<const BlockId> ids, std::span<const std::size_t> runs,
                                    std::vector<std::pair<std::uint64_t, std::uint64_t>>& hits_misses) {
    std::lock_guard lock(mutex_);
    hits_misses.assign(runs.size(), {0, 0});
    std::size_t i = 0;
    for (std::size_t k = 0; k < runs.size(); ++k) {
        for (std::size_t e = i + runs[k]; i < e && i < ids.size(); ++i) {
            const BlockId id = ids[i];
            const std::int64_t h = blocks_->handle(id);
            if (h < 0) throw NotFoundError("load_block: unknown block id " + std::to_string(id));
            if (account_locked(id, h, blocks_->at(h))) ++hits_misses[k].second;
            else ++hits_misses[k].first;
        }
    }
}

void TieredBlockStore::inject_miss_latency(std::uint64_t misses) const {
    if (misses > 0 && options_.miss_sleep_ms > 0.0)
        std::this_thread::sleep_for(std::chrono::duration<double, std::milli>(options_.miss_sleep_ms * misses));
}

std::shared_ptr<const KVBlock> TieredBlockStore::copy_out(BlockId id, const BlockRec& rec) const {
    auto b = std::make_shared<KVBlock>();
    b->block_id = id;
    b->layer_id = rec.layer;
    b->n_tokens = rec.n_tokens;
    b->dim = rec.dim;
    const std::size_t n = static_cast<std::size_t>(rec.n_tokens) * rec.dim;
    b->keys.resize(n);
    b->values.resize(n);
    check_rc(psa::read_slot(pools_.at(rec.dim)->pool, rec.slot, rec.n_tokens, b->keys.data(), b->values.data()));
    return b;
}

std::shared_ptr<const KVBlock> TieredBlockStore::load_block(BlockId block_id, std::int32_t layer_id) {
    std::shared_ptr<const KVBlock> out;
    bool miss = false;
    {
        std::lock_guard lock(mutex_);
        const std::int64_t h = blocks_->handle(block_id);
        if (h < 0) throw NotFoundError("load_block: unknown block id " + std::to_string(block_id));
        const BlockRec& rec = blocks_->at(h);
        if (layer_id >= 0 && rec.layer != layer_id) throw Error("load_block: layer_id does not match block");
        miss = account_locked(block_id, h, rec);
        out = copy_out(block_id, rec);
    }
    if (miss) inject_miss_latency(1);
    return out;
}

std::shared_ptr<const KVBlock> TieredBlockStore::peek_block(BlockId block_id) const {
    std::lock_guard lock(mutex_);
    const BlockRec* rec = blocks_->find(block_id);
    if (!rec) throw NotFoundError("peek_block: unknown block id " + std::to_string(block_id));
    return copy_out(block_id, *rec);
}

BlockMetadata TieredBlockStore::metadata(BlockId block_id) const {
    std::lock_guard lock(mutex_);
    const BlockRec* rp = blocks_->find(block_id);
    if (!rp) throw NotFoundError("metadata: unknown block id " + std::to_string(block_id));
    const BlockRec& r = *rp;
    BlockMetadata m;
    m.block_id = block_id;
    m.layer_id = r.layer;
    m.n_tokens = r.n_tokens;
    m.mean_key.resize(r.dim);
    m.lo.resize(r.dim);
    m.hi.resize(r.dim);
    check_rc(psa::read_meta(pools_.at(r.dim)->pool, r.slot, m.mean_key.data(), m.lo.data(), m.hi.data()));
    return m;
}

std::vector<BlockMetadata> TieredBlockStore::metadata_for(std::span<const BlockId> ids) const {
    std::vector<BlockMetadata> out;
    out.reserve(ids.size());
    for (BlockId id : ids) out.push_back(metadata(id));
    return out;
}

void TieredBlockStore::release_request(RequestId request_id) {
    std::lock_guard lock(mutex_);
    auto it = owned_.find(request_id);
    if (it == owned_.end()) throw NotFoundError("release_request: unknown request " + std::to_string(request_id));
    for (BlockId id : it->second) {
        const std::int64_t h = blocks_->handle(id);
        if (h < 0) continue;
        const BlockRec& rec = blocks_->at(h);
        tier_->release(h, rec.layer);
        pools_.at(rec.dim)->free_slots.push_back(rec.slot);
        blocks_->erase(id);
    }
    owned_.erase(it);
}

bool TieredBlockStore::contains(BlockId block_id) const {
    std::lock_guard lock(mutex_);
    return blocks_->contains(block_id);
}

bool TieredBlockStore::resident_fast(BlockId block_id) const {
    std::lock_guard lock(mutex_);
    const std::int64_t h = blocks_->handle(block_id);
    if (h < 0) return false;
    return tier_->resident(h, blocks_->at(h).layer);
}

CacheStats TieredBlockStore::stats() const {
    std::lock_guard lock(mutex_);
    const auto& t = tier_->total();
    CacheStats out{t.hits, t.misses, t.evictions, t.bytes, {}};
    for (std::int32_t l = 0; l < tier_->n_layers(); ++l) {
        const auto& c = tier_->layer(l);
        out.per_layer.push_back(LayerCacheStats{c.hits, c.misses, c.evictions, c.bytes});
    }
    return out;
}

std::size_t TieredBlockStore::fast_occupancy() const {
    std::lock_guard lock(mutex_);
    return tier_->occupancy();
}

std::size_t TieredBlockStore::domain_capacity(std::int32_t layer_id) const {
    std::lock_guard lock(mutex_);
    if (layer_id < 0 || layer_id >= options_.n_layers) throw Error("TieredBlockStore: layer_id out of range");
    return tier_->capacity(layer_id);
}

void TieredBlockStore::enable_trace(std::ostream* sink) {
    std::lock_guard lock(mutex_);
    trace_ = sink;
}

// -----------------------------------------------------------------------------
// One device launch for a batch of progressive queries.
// -----------------------------------------------------------------------------
void TieredBlockStore::run_device(const detail::DeviceQueryBatch& qb, detail::DeviceQueryResult& res) {
    std::lock_guard lock(mutex_);
    static const bool prof = getenv("PSA_RUN_PROF") != nullptr;  // development: phase times to stderr
    using PClock = std::chrono::steady_clock;
    const auto t_begin = PClock::now();
    auto us_since = [](PClock::time_point a) {
        return std::chrono::duration<double, std::micro>(PClock::now() - a).count();
    };
    const int g = qb.group, d = qb.dim;
    const int n_units = static_cast<int>(qb.lists.size());
    if (n_units == 0) throw Error("batched attention: empty batch");
    auto pit = pools_.find(d);
    std::vector<std::int64_t> off(n_units + 1, 0);
    std::int64_t max_n = 0;
    for (int u = 0; u < n_units; ++u) {
        const auto m = static_cast<std::int64_t>(qb.lists[u].size());
        if (m == 0) throw Error("plan_blocks: no blocks given");
        off[u + 1] = off[u] + m;
        max_n = std::max(max_n, m);
    }
    const std::int64_t total = off[n_units];
    const std::int64_t nq = static_cast<std::int64_t>(n_units) * g;
    const std::int64_t hbt = total * g;

    // ---- host inputs: q | slots | list_off ----
    const size_t q_b = align256(static_cast<size_t>(nq) * d * 4);
    const size_t s_b = align256(static_cast<size_t>(total) * 4);
    const size_t o_b = align256(static_cast<size_t>(n_units + 1) * 8);
    char* hin = static_cast<char*>(dev_->h_in.get(q_b + s_b + o_b));
    auto* hs = reinterpret_cast<std::int32_t*>(hin + q_b);
    // Resolve ids -> slots straight into the staging buffer (one table index per id), ascending-id
    // order per list; lists that arrive sorted (the usual page-table order) are used in place.
    std::vector<std::vector<BlockId>> sorted_copy(n_units);
    std::vector<const BlockId*> sorted(n_units);
    for (int u = 0; u < n_units; ++u) {
        const auto& ids = qb.lists[u];
        if (std::is_sorted(ids.begin(), ids.end())) {
            sorted[u] = ids.data();
        } else {
            sorted_copy[u].assign(ids.begin(), ids.end());
            std::sort(sorted_copy[u].begin(), sorted_copy[u].end());
            sorted[u] = sorted_copy[u].data();
        }
        const BlockId* src = sorted[u];
        std::int32_t* dst = hs + off[u];
        for (std::int64_t i = 0, m = off[u + 1] - off[u]; i < m; ++i) {
            const BlockRec* rec = blocks_->find(src[i]);
            if (!rec) throw NotFoundError("metadata: unknown block id " + std::to_string(src[i]));
            if (rec->dim != d) check_dim(static_cast<std::size_t>(d), static_cast<std::size_t>(rec->dim), "criticality_score");
            dst[i] = static_cast<std::int32_t>(rec->slot);
        }
    }
    if (pit == pools_.end()) throw Error("no blocks of this dimension");
    psattn_pool* pool = pit->second->pool;
    for (std::int64_t i = 0; i < nq; ++i) std::memcpy(hin + static_cast<size_t>(i) * d * 4, qb.queries[i], d * 4);
    std::memcpy(hin + q_b + s_b, off.data(), (n_units + 1) * 8);
    const double t_resolve = prof ? us_since(t_begin) : 0.0;
    char* din = static_cast<char*>(dev_->in.get(q_b + s_b + o_b));
    check_cuda(cudaMemcpyAsync(din, hin, q_b + s_b + o_b, cudaMemcpyHostToDevice, dev_->stream), "H2D");

    // ---- device outputs: out | bp | est | tcov | term | rpos | iest | omass(copy) ----
    const size_t ob_out = align256(static_cast<size_t>(nq) * d * 4), ob_bp = align256(nq * 8),
                 ob_est = align256(nq * 8), ob_tc = align256(nq * 8), ob_term = align256(nq * 4),
                 ob_rpos = align256(static_cast<size_t>(hbt) * 4), ob_iest = align256(static_cast<size_t>(hbt) * 8);
    const size_t out_total = ob_out + ob_bp + ob_est + ob_tc + ob_term + ob_rpos + ob_iest;
    char* dout = static_cast<char*>(dev_->outb.get(out_total));

    psattn_batch b{};
    std::memset(&b, 0, sizeof(b));  // padding too: the descriptor is a graph-cache key
    b.n_units = n_units;
    b.group = g;
    b.dim = d;
    b.max_blocks = max_n;
    b.total_blocks = total;
    b.q = reinterpret_cast<const float*>(din);
    b.slots = reinterpret_cast<const std::int32_t*>(din + q_b);
    b.list_off = reinterpret_cast<const std::int64_t*>(din + q_b + s_b);
    b.epsilon = qb.cfg.epsilon;
    b.microbatch_size = qb.cfg.microbatch_size;
    b.estimator = static_cast<std::int32_t>(qb.cfg.estimator);
    b.ranking_mode = qb.cfg.ranking_mode == RankingMode::Oracle ? PSATTN_RANK_ORACLE : PSATTN_RANK_ESTIMATED;
    b.audit_coverage = qb.cfg.audit_coverage ? 1 : 0;
    b.scale_override = qb.cfg.scale_override;
    b.topk = static_cast<std::int64_t>(qb.topk);
    size_t o = 0;
    b.out = reinterpret_cast<float*>(dout + o); o += ob_out;
    b.blocks_processed = reinterpret_cast<std::int64_t*>(dout + o); o += ob_bp;
    b.est_coverage = reinterpret_cast<double*>(dout + o); o += ob_est;
    b.true_coverage = reinterpret_cast<double*>(dout + o); o += ob_tc;
    b.terminated = reinterpret_cast<std::int32_t*>(dout + o); o += ob_term;
    b.ranked_pos = reinterpret_cast<std::int32_t*>(dout + o); o += ob_rpos;
    b.iter_est = reinterpret_cast<double*>(dout + o); o += ob_iest;
    const size_t wsb = psattn_batch_workspace_bytes(&b);
    void* ws = dev_->ws.get(wsb);
    cudaEvent_t pev[3] = {nullptr, nullptr, nullptr};
    if (prof) {
        for (auto& e : pev) cudaEventCreate(&e);
        cudaEventRecord(pev[0], dev_->stream);
    }
    check_rc(qb.rank_only ? psattn_rank_batch(pool, &b, ws, dev_->stream) : dev_->launch(pool, b, ws));
    if (prof) cudaEventRecord(pev[1], dev_->stream);

    const bool has_oracle = b.ranking_mode == PSATTN_RANK_ORACLE || b.audit_coverage;
    const size_t om_b = has_oracle ? static_cast<size_t>(hbt) * 8 : 0;
    char* hout = static_cast<char*>(dev_->h_out.get(out_total + om_b + 256));
    // Compact read-back (equal-length lists, no oracle masses): the per-query scalars first, then
    // only ranks below the largest blocks_processed of the rank positions and estimates (one 2-D
    // copy each: rows of n entries, max_bp wide) instead of every rank of every list.
    bool compact = !has_oracle && !qb.rank_only;
    for (int u = 0; compact && u < n_units; ++u) compact = off[u + 1] - off[u] == max_n;
    const size_t head_b = ob_out + ob_bp + ob_est + ob_tc + ob_term;
    std::int64_t rows_w = 0;  // compact: entries kept per (unit, head) row
    check_cuda(cudaMemcpyAsync(hout, dout, compact ? head_b : out_total, cudaMemcpyDeviceToHost, dev_->stream), "D2H");
    if (has_oracle) {
        // workspace layout: keys | rpos | omass (psattn_batch_workspace_bytes)
        const size_t om_off = align256(static_cast<size_t>(hbt) * 8) + align256(static_cast<size_t>(hbt) * 4);
        check_cuda(cudaMemcpyAsync(hout + out_total, static_cast<char*>(ws) + om_off, om_b, cudaMemcpyDeviceToHost,
                                   dev_->stream),
                   "D2H");
    }
    if (compact) {
        check_cuda(cudaStreamSynchronize(dev_->stream), "PSA device launch");
        const auto* bp0 = reinterpret_cast<const std::int64_t*>(hout + ob_out);
        for (std::int64_t qi = 0; qi < nq; ++qi) rows_w = std::max(rows_w, std::clamp<std::int64_t>(bp0[qi], 0, max_n));
        if (rows_w > 0) {
            const size_t w4 = static_cast<size_t>(rows_w) * 4, w8 = static_cast<size_t>(rows_w) * 8;
            check_cuda(cudaMemcpy2DAsync(hout + head_b, w4, dout + head_b, static_cast<size_t>(max_n) * 4, w4,
                                         static_cast<size_t>(nq), cudaMemcpyDeviceToHost, dev_->stream),
                       "D2H");
            check_cuda(cudaMemcpy2DAsync(hout + head_b + ob_rpos, w8, dout + head_b + ob_rpos,
                                         static_cast<size_t>(max_n) * 8, w8, static_cast<size_t>(nq),
                                         cudaMemcpyDeviceToHost, dev_->stream),
                       "D2H");
        }
    }
    if (prof) cudaEventRecord(pev[2], dev_->stream);
    const double t_launched = prof ? us_since(t_begin) : 0.0;
    check_cuda(cudaStreamSynchronize(dev_->stream), "PSA device launch");
    const double t_synced = prof ? us_since(t_begin) : 0.0;

    // ---- unpack ----
    res.dim = d;
    res.scale = qb.cfg.scale_for(static_cast<std::size_t>(d));
    o = 0;
    res.out.assign(reinterpret_cast<float*>(hout), reinterpret_cast<float*>(hout) + nq * d); o += ob_out;
    const auto* bp = reinterpret_cast<const std::int64_t*>(hout + o); o += ob_bp;
    const auto* est = reinterpret_cast<const double*>(hout + o); o += ob_est;
    const auto* tc = reinterpret_cast<const double*>(hout + o); o += ob_tc;
    const auto* term = reinterpret_cast<const std::int32_t*>(hout + o); o += ob_term;
    const auto* rpos = reinterpret_cast<const std::int32_t*>(hout + o); o += ob_rpos;
    const auto* iest = reinterpret_cast<const double*>(hout + o); o += ob_iest;
    const auto* om = reinterpret_cast<const double*>(hout + out_total);
    res.blocks_processed.assign(bp, bp + nq);
    res.est.assign(est, est + nq);
    res.true_cov.assign(tc, tc + nq);
    res.terminated.assign(term, term + nq);
    res.ranked_ids.assign(nq, {});
    res.iter_est.assign(nq, {});
    res.oracle_ranked.assign(nq, {});
    res.union_ids.clear();
    std::vector<std::uint8_t> seen;  // want_union: list positions processed by any head of the unit
    for (int u = 0; u < n_units; ++u) {
        const std::int64_t n = off[u + 1] - off[u];
        if (qb.want_union) seen.assign(static_cast<std::size_t>(n), 0);
        for (int h = 0; h < g; ++h) {
            const std::int64_t qi = static_cast<std::int64_t>(u) * g + h;
            const std::int64_t hb = compact ? qi * rows_w : off[u] * g + h * n;  // row of query qi
            // psattn_run_batch defines ranks below blocks_processed only (it orders lazily)
            const std::int64_t nr = qb.rank_only ? n : std::clamp<std::int64_t>(bp[qi], 0, n);
            auto& ids = res.ranked_ids[qi];
            ids.resize(static_cast<std::size_t>(nr));
            for (std::int64_t r = 0; r < nr; ++r) {
                const std::int32_t pos = rpos[hb + r];
                if (pos < 0 || pos >= n) throw Error("device ranking: position out of range");
                ids[r] = sorted[u][pos];
                if (qb.want_union) seen[static_cast<std::size_t>(pos)] = 1;
            }
            if (!qb.rank_only) res.iter_est[qi].assign(iest + hb, iest + hb + nr);
            if (has_oracle) {
                auto& orr = res.oracle_ranked[qi];
                orr.resize(static_cast<std::size_t>(nr));
                for (std::int64_t r = 0; r < nr; ++r) orr[r] = om[hb + rpos[hb + r]];
            }
        }
        if (qb.want_union) {  // positions ascend with ids: the unit's union comes out sorted
            std::int64_t i = 0;
            for (; i + 8 <= n; i += 8) {  // 8 positions per word test (most are unprocessed)
                std::uint64_t w;
                std::memcpy(&w, seen.data() + i, 8);
                if (!w) continue;
                for (int j = 0; j < 8; ++j)
                    if (seen[static_cast<std::size_t>(i + j)]) res.union_ids.push_back(sorted[u][i + j]);
            }
            for (; i < n; ++i)
                if (seen[static_cast<std::size_t>(i)]) res.union_ids.push_back(sorted[u][i]);
        }
    }
    if (qb.want_union && !std::is_sorted(res.union_ids.begin(), res.union_ids.end()))
        std::sort(res.union_ids.begin(), res.union_ids.end());  // lists sharing ids: merge the runs
    if (qb.want_union)
        res.union_ids.erase(std::unique(res.union_ids.begin(), res.union_ids.end()), res.union_ids.end());
    if (prof) {
        float kms = 0.0f, cms = 0.0f;
        cudaEventElapsedTime(&kms, pev[0], pev[1]);
        cudaEventElapsedTime(&cms, pev[1], pev[2]);
        for (auto& e : pev) cudaEventDestroy(e);
        fprintf(stderr,
                "run_device_prof units=%d blocks=%lld resolve_us=%.1f launch_us=%.1f sync_us=%.1f unpack_us=%.1f "
                "device_kernels_us=%.1f d2h_us=%.1f\n",
                n_units, static_cast<long long>(total), t_resolve, t_launched - t_resolve, t_synced - t_launched,
                us_since(t_begin) - t_synced, kms * 1e3, cms * 1e3);
    }
}

}  // namespace psattn
