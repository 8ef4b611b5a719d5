// fast_tier.h — fast-tier residency accounting shared by the C/C++ store (store.cpp) and the
// two-tier HBM/host store (tier.cpp).
//
// Observable semantics are the reference TieredBlockStore's (store.hpp:16-120,
// store.cpp:11-124): slot domains (one Unified domain of `capacity` slots, or
// floor(capacity / n_layers) slots per layer), write-allocate on put, a hit refreshes recency
// under LRU (FIFO keeps insertion order), a miss costs the block's fp32 payload in bytes and
// admits it (evicting the oldest entry of a full domain; the eviction is charged to the
// victim's layer), release drops entries without counting evictions.
//
// Representation: each domain is an intrusive doubly linked recency chain (id -> {older, newer}
// neighbour ids) with the newest / oldest ids at the ends, no per-entry list nodes: in a hash map
// for arbitrary ids (the C/C++ store), in two flat arrays for dense ids (the two-tier store's
// block indices: no hashing on the per-step accounting replay).
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <algorithm>
#include <unordered_map>
#include <vector>

namespace psa {

class RecencyChain {
public:
    static constexpr std::int64_t kNone = INT64_MIN;

    // dense_ids > 0: ids are known to lie in [0, dense_ids) (the two-tier store's block indices):
    // the links live in two flat arrays indexed by id instead of a hash map (no hashing per access).
    explicit RecencyChain(std::size_t capacity = 0, std::size_t dense_ids = 0)
        : cap_(capacity), dense_(dense_ids > 0) {
        if (dense_) {
            older_.assign(dense_ids, kNone);
            newer_.assign(dense_ids, kNone);
            in_.assign(dense_ids, 0);
        }
    }
    std::size_t capacity() const { return cap_; }
    // dense chains: extends the id range to at least [0, n) (geometric growth)
    void grow(std::size_t n) {
        if (!dense_ || n <= in_.size()) return;
        const std::size_t m = std::max(n, 2 * in_.size());
        older_.resize(m, kNone);
        newer_.resize(m, kNone);
        in_.resize(m, 0);
    }
    std::size_t size() const { return dense_ ? count_ : links_.size(); }
    bool contains(std::int64_t id) const {
        if (dense_) return id >= 0 && static_cast<std::size_t>(id) < in_.size() && in_[static_cast<std::size_t>(id)];
        return links_.count(id) != 0;
    }

    // Moves a present id to the newest end. Returns false when absent.
    bool refresh(std::int64_t id) {
        if (!contains(id)) return false;
        if (newest_ != id) {
            unlink(id);
            link_newest(id);
        }
        return true;
    }
    // Inserts an absent id as newest; returns the evicted oldest id when the chain was full.
    // A zero-capacity chain holds nothing (the id is not inserted, nothing is evicted).
    std::optional<std::int64_t> admit(std::int64_t id) {
        if (cap_ == 0) return std::nullopt;
        std::optional<std::int64_t> victim;
        if (size() == cap_) {
            victim = oldest_;
            erase(oldest_);
        }
        if (dense_) {
            in_[static_cast<std::size_t>(id)] = 1;
            ++count_;
        } else {
            links_[id] = Link{};
        }
        link_newest(id);
        return victim;
    }
    bool erase(std::int64_t id) {
        if (!contains(id)) return false;
        unlink(id);
        if (dense_) {
            in_[static_cast<std::size_t>(id)] = 0;
            --count_;
        } else {
            links_.erase(id);
        }
        return true;
    }

private:
    struct Link {
        std::int64_t older = kNone, newer = kNone;
    };
    std::int64_t& older(std::int64_t id) {
        return dense_ ? older_[static_cast<std::size_t>(id)] : links_.find(id)->second.older;
    }
    std::int64_t& newer(std::int64_t id) {
        return dense_ ? newer_[static_cast<std::size_t>(id)] : links_.find(id)->second.newer;
    }
    void unlink(std::int64_t id) {
        std::int64_t& o = older(id);
        std::int64_t& w = newer(id);
        if (o != kNone) newer(o) = w;
        else oldest_ = w;
        if (w != kNone) older(w) = o;
        else newest_ = o;
        o = w = kNone;
    }
    void link_newest(std::int64_t id) {
        older(id) = newest_;
        newer(id) = kNone;
        if (newest_ != kNone) newer(newest_) = id;
        newest_ = id;
        if (oldest_ == kNone) oldest_ = id;
    }

    std::size_t cap_;
    bool dense_;
    std::unordered_map<std::int64_t, Link> links_;
    std::vector<std::int64_t> older_, newer_;
    std::vector<std::uint8_t> in_;
    std::size_t count_ = 0;
    std::int64_t newest_ = kNone, oldest_ = kNone;
};

struct TierCounters {
    std::uint64_t hits = 0, misses = 0, evictions = 0, bytes = 0;
};

// Domains + counters of one store.
class FastTier {
public:
    struct Access {
        bool hit = false;
        std::optional<std::int64_t> evicted;  // victim of the admission (misses only)
    };

    // dense_ids > 0: every id lies in [0, dense_ids) (array-backed recency chains)
    FastTier(std::size_t capacity, std::int32_t n_layers, bool per_layer_domains, bool lru, std::size_t dense_ids = 0)
        : per_layer_domains_(per_layer_domains), lru_(lru), layers_(static_cast<std::size_t>(n_layers)) {
        if (n_layers <= 0) throw std::invalid_argument("fast tier: n_layers must be positive");
        if (per_layer_domains) domains_.assign(layers_.size(), RecencyChain(capacity / layers_.size(), dense_ids));
        else domains_.assign(1, RecencyChain(capacity, dense_ids));
    }

    // put_block's write-allocate (no hit/miss). `layer_of` resolves a victim's layer.
    template <typename LayerOf>
    std::optional<std::int64_t> put(std::int64_t id, std::int32_t layer, LayerOf&& layer_of) {
        auto victim = domain(layer).admit(id);
        if (victim) charge_eviction(layer_of(*victim));
        return victim;
    }
    // load_block's accounting: hit (LRU refresh) or miss (bytes + admission).
    template <typename LayerOf>
    Access access(std::int64_t id, std::int32_t layer, std::uint64_t payload_bytes, LayerOf&& layer_of) {
        RecencyChain& d = domain(layer);
        TierCounters& c = layers_.at(static_cast<std::size_t>(layer));
        Access a;
        if (lru_ ? d.refresh(id) : d.contains(id)) {
            a.hit = true;
            ++c.hits;
            ++total_.hits;
            return a;
        }
        ++c.misses;
        ++total_.misses;
        c.bytes += payload_bytes;
        total_.bytes += payload_bytes;
        a.evicted = d.admit(id);
        if (a.evicted) charge_eviction(layer_of(*a.evicted));
        return a;
    }
    bool release(std::int64_t id, std::int32_t layer) { return domain(layer).erase(id); }
    void grow(std::size_t dense_ids) {
        for (auto& d : domains_) d.grow(dense_ids);
    }
    bool resident(std::int64_t id, std::int32_t layer) const { return domain(layer).contains(id); }

    std::size_t capacity(std::int32_t layer) const { return domain(layer).capacity(); }
    std::size_t occupancy() const {
        std::size_t n = 0;
        for (const auto& d : domains_) n += d.size();
        return n;
    }
    const TierCounters& total() const { return total_; }
    const TierCounters& layer(std::int32_t l) const { return layers_.at(static_cast<std::size_t>(l)); }
    std::int32_t n_layers() const { return static_cast<std::int32_t>(layers_.size()); }

private:
    RecencyChain& domain(std::int32_t layer) {
        check(layer);
        return domains_[per_layer_domains_ ? static_cast<std::size_t>(layer) : 0];
    }
    const RecencyChain& domain(std::int32_t layer) const {
        check(layer);
        return domains_[per_layer_domains_ ? static_cast<std::size_t>(layer) : 0];
    }
    void check(std::int32_t layer) const {
        if (layer < 0 || static_cast<std::size_t>(layer) >= layers_.size())
            throw std::out_of_range("fast tier: layer out of range");
    }
    void charge_eviction(std::int32_t victim_layer) {
        ++total_.evictions;
        if (victim_layer >= 0 && static_cast<std::size_t>(victim_layer) < layers_.size())
            ++layers_[static_cast<std::size_t>(victim_layer)].evictions;
    }

    bool per_layer_domains_, lru_;
    std::vector<RecencyChain> domains_;
    std::vector<TierCounters> layers_;
    TierCounters total_;
};

}  // namespace psa
