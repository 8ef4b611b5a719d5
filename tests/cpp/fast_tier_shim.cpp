// ctypes shim over csrc/fast_tier.h (+ csrc/block_table.h) for the CPU accounting test
// (tests/test_fast_tier.py). Table mode is the C/C++ store's layout: ids -> dense handles
// through BlockTable, array-backed chains indexed by handle and grown as handles are issued.
#include <cstdint>
#include <unordered_map>

#include "block_table.h"
#include "fast_tier.h"

namespace {
struct Shim {
    psa::FastTier tier;
    bool table;
    psa::BlockTable<std::int32_t> bt;               // table mode: id -> handle, record = layer
    std::unordered_map<std::int64_t, std::int32_t> layer;  // id mode
    Shim(std::size_t cap, int layers, bool per_layer, bool lru, std::size_t dense, bool tab)
        : tier(cap, layers, per_layer, lru, tab ? 1 : dense), table(tab) {}
    std::int64_t key(std::int64_t id) const { return table ? bt.handle(id) : id; }
    std::int32_t layer_of_key(std::int64_t k) const { return table ? bt.at(k) : layer.at(k); }
    std::int64_t id_of_key(std::int64_t k) const { return table ? bt.id_of(k) : k; }
};
}  // namespace

extern "C" {
void* ft_create(std::uint64_t cap, int n_layers, int per_layer, int lru, std::uint64_t dense_ids) {
    return new Shim(cap, n_layers, per_layer != 0, lru != 0, dense_ids, false);
}
void* ft_create_table(std::uint64_t cap, int n_layers, int per_layer, int lru) {
    return new Shim(cap, n_layers, per_layer != 0, lru != 0, 0, true);
}
void ft_destroy(void* h) { delete static_cast<Shim*>(h); }
std::int64_t ft_put(void* h, std::int64_t id, int layer) {
    auto* s = static_cast<Shim*>(h);
    std::int64_t k = id;
    if (s->table) {
        k = s->bt.insert(id, layer);
        s->tier.grow(s->bt.handles());
    } else {
        s->layer[id] = layer;
    }
    auto v = s->tier.put(k, layer, [s](std::int64_t x) { return s->layer_of_key(x); });
    return v ? s->id_of_key(*v) : psa::RecencyChain::kNone;
}
int ft_load(void* h, std::int64_t id, std::uint64_t bytes, std::int64_t* evicted) {
    auto* s = static_cast<Shim*>(h);
    const std::int64_t k = s->key(id);
    auto a = s->tier.access(k, s->layer_of_key(k), bytes, [s](std::int64_t x) { return s->layer_of_key(x); });
    *evicted = a.evicted ? s->id_of_key(*a.evicted) : psa::RecencyChain::kNone;
    return a.hit ? 1 : 0;
}
void ft_release(void* h, std::int64_t id) {
    auto* s = static_cast<Shim*>(h);
    const std::int64_t k = s->key(id);
    s->tier.release(k, s->layer_of_key(k));
    if (s->table) s->bt.erase(id);
}
int ft_resident(void* h, std::int64_t id) {
    auto* s = static_cast<Shim*>(h);
    const std::int64_t k = s->key(id);
    return s->tier.resident(k, s->layer_of_key(k)) ? 1 : 0;
}
void ft_stats(void* h, int layer, std::uint64_t* out) {
    auto* s = static_cast<Shim*>(h);
    const psa::TierCounters& c = layer < 0 ? s->tier.total() : s->tier.layer(layer);
    out[0] = c.hits;
    out[1] = c.misses;
    out[2] = c.evictions;
    out[3] = c.bytes;
}
}
