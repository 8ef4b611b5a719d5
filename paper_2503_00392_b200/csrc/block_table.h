// block_table.h — the store's block-id -> record table.
//
// Every block gets a dense handle in [0, handles()) when it is put (freed handles are reused);
// records live in a flat vector indexed by handle, and the fast-tier recency chains are indexed by
// handle too (array-backed, fast_tier.h), so the per-query work — resolving a list of ids to device
// slots (run_device) and replaying the loads through the LRU/FIFO accounting — costs an array
// index per id instead of several hash lookups. Ids in [0, kDirect) (the usual page-table ids)
// resolve through a direct-indexed vector; other ids (negative or huge) through a hash map.
#pragma once

#include <algorithm>
#include <cstdint>
#include <unordered_map>
#include <vector>

namespace psa {

template <typename Rec>
class BlockTable {
public:
    static constexpr std::int64_t kDirect = std::int64_t{1} << 24;

    // handle of `id`, or -1
    std::int64_t handle(std::int64_t id) const {
        if (id >= 0 && id < kDirect) {
            const std::size_t i = static_cast<std::size_t>(id);
            return i < direct_.size() ? static_cast<std::int64_t>(direct_[i]) - 1 : -1;
        }
        auto it = sparse_.find(id);
        return it == sparse_.end() ? -1 : it->second;
    }
    Rec* find(std::int64_t id) {
        const std::int64_t h = handle(id);
        return h < 0 ? nullptr : &recs_[static_cast<std::size_t>(h)];
    }
    const Rec* find(std::int64_t id) const {
        const std::int64_t h = handle(id);
        return h < 0 ? nullptr : &recs_[static_cast<std::size_t>(h)];
    }
    bool contains(std::int64_t id) const { return handle(id) >= 0; }

    // Inserts an absent id; returns its handle.
    std::int64_t insert(std::int64_t id, const Rec& r) {
        std::int64_t h;
        if (!free_.empty()) {
            h = free_.back();
            free_.pop_back();
            recs_[static_cast<std::size_t>(h)] = r;
            ids_[static_cast<std::size_t>(h)] = id;
        } else {
            h = static_cast<std::int64_t>(recs_.size());
            recs_.push_back(r);
            ids_.push_back(id);
        }
        if (id >= 0 && id < kDirect) {
            const std::size_t i = static_cast<std::size_t>(id);
            if (i >= direct_.size()) direct_.resize(std::max<std::size_t>(i + 1, direct_.size() * 2), 0);
            direct_[i] = static_cast<std::int32_t>(h + 1);
        } else {
            sparse_[id] = h;
        }
        ++live_;
        return h;
    }
    // Removes a present id (its handle becomes reusable).
    void erase(std::int64_t id) {
        const std::int64_t h = handle(id);
        if (h < 0) return;
        if (id >= 0 && id < kDirect) direct_[static_cast<std::size_t>(id)] = 0;
        else sparse_.erase(id);
        free_.push_back(h);
        --live_;
    }

    std::int64_t id_of(std::int64_t h) const { return ids_[static_cast<std::size_t>(h)]; }
    // fn(id, rec) for every live block
    template <typename Fn>
    void for_each(Fn&& fn) const {
        for (std::size_t h = 0; h < recs_.size(); ++h)
            if (handle(ids_[h]) == static_cast<std::int64_t>(h)) fn(ids_[h], recs_[h]);
    }
    const Rec& at(std::int64_t h) const { return recs_[static_cast<std::size_t>(h)]; }
    std::size_t handles() const { return recs_.size(); }  // every handle ever issued is below this
    std::size_t size() const { return live_; }

private:
    std::vector<std::int32_t> direct_;  // id -> handle + 1 (0: absent)
    std::unordered_map<std::int64_t, std::int64_t> sparse_;
    std::vector<Rec> recs_;
    std::vector<std::int64_t> ids_;
    std::vector<std::int64_t> free_;
    std::size_t live_ = 0;
};

}  // namespace psa
