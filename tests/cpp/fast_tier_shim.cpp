// ctypes shim over csrc/fast_tier.h for the CPU accounting test (tests/test_fast_tier.py).
#include <cstdint>
#include <unordered_map>

#include "fast_tier.h"

namespace {
struct Shim {
    psa::FastTier tier;
    std::unordered_map<std::int64_t, std::int32_t> layer;
    Shim(std::size_t cap, int layers, bool per_layer, bool lru, std::size_t dense)
        : tier(cap, layers, per_layer, lru, dense) {}
};
}  // namespace

extern "C" {
void* ft_create(std::uint64_t cap, int n_layers, int per_layer, int lru, std::uint64_t dense_ids) {
    return new Shim(cap, n_layers, per_layer != 0, lru != 0, dense_ids);
}
void ft_destroy(void* h) { delete static_cast<Shim*>(h); }
std::int64_t ft_put(void* h, std::int64_t id, int layer) {
    auto* s = static_cast<Shim*>(h);
    s->layer[id] = layer;
    auto v = s->tier.put(id, layer, [s](std::int64_t x) { return s->layer.at(x); });
    return v ? *v : psa::RecencyChain::kNone;
}
int ft_load(void* h, std::int64_t id, std::uint64_t bytes, std::int64_t* evicted) {
    auto* s = static_cast<Shim*>(h);
    auto a = s->tier.access(id, s->layer.at(id), bytes, [s](std::int64_t x) { return s->layer.at(x); });
    *evicted = a.evicted ? *a.evicted : psa::RecencyChain::kNone;
    return a.hit ? 1 : 0;
}
void ft_release(void* h, std::int64_t id) {
    auto* s = static_cast<Shim*>(h);
    s->tier.release(id, s->layer.at(id));
}
int ft_resident(void* h, std::int64_t id) {
    auto* s = static_cast<Shim*>(h);
    return s->tier.resident(id, s->layer.at(id)) ? 1 : 0;
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
