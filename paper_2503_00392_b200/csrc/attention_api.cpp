// attention_api.cpp — psattn:: attention.hpp entry points (reference include/psattn/attention.hpp:39-109,
// src/attention.cpp:7-79): argument checks and exceptions on the host, arithmetic on the device
// (attention_kernels.cu).
#include "psattn/attention.hpp"

#include <string>

#include "device.h"

namespace psattn {
namespace {

void check(int rc) {
    if (rc != PSATTN_OK) throw Error(psa::last_error());
}

// Tokens of a block sequence, packed contiguously (the device kernel reads one [n][d] array).
struct Packed {
    std::vector<float> k, v;
    std::int64_t n = 0;
};

}  // namespace

template <typename T>
T dot_scaled(std::span<const float> q, const float* k, T scale) {
    if (q.empty()) return T(0) * scale;
    T st[3];
    check(psa::seq_attention(q.data(), static_cast<int>(q.size()), k, nullptr, 1, scale, 0, nullptr, st));
    return st[0];  // the single token's score is the max
}

template <typename T>
ScoredBlockT<T> block_partial_attention_t(std::span<const float> q, const KVBlock& block, T scale) {
    if (block.n_tokens <= 0) throw Error("block_partial_attention: empty block");
    check_dim(q.size(), static_cast<std::size_t>(block.dim), "block_partial_attention");
    ScoredBlockT<T> r;
    r.out_unnorm.assign(q.size(), T{0});
    T st[3];
    check(psa::seq_attention(q.data(), block.dim, block.keys.data(), block.values.data(), block.n_tokens, scale, 0,
                             r.out_unnorm.data(), st));
    r.max_score = st[0];
    r.exp_sum = st[1];
    r.log_as = st[2];
    return r;
}

template <typename T>
void merge_partial(SoftmaxAccumulatorT<T>& acc, const ScoredBlockT<T>& part) {
    if (acc.empty()) {
        acc.out_unnorm = part.out_unnorm;
        acc.max_score = part.max_score;
        acc.exp_sum = part.exp_sum;
        acc.log_as_acc = part.log_as;
        return;
    }
    check_dim(part.out_unnorm.size(), acc.out_unnorm.size(), "merge_partial");
    T a[3] = {acc.max_score, acc.exp_sum, acc.log_as_acc};
    const T p[3] = {part.max_score, part.exp_sum, part.log_as};
    check(psa::softmax_merge(acc.out_unnorm.data(), a, part.out_unnorm.data(), p,
                             static_cast<int>(acc.out_unnorm.size())));
    acc.max_score = a[0];
    acc.exp_sum = a[1];
    acc.log_as_acc = a[2];
}

template <typename T>
std::vector<T> finalize(const SoftmaxAccumulatorT<T>& acc) {
    if (acc.empty()) throw Error("finalize: no blocks processed");
    std::vector<T> out(acc.out_unnorm.size());
    check(psa::softmax_finalize(acc.out_unnorm.data(), static_cast<int>(out.size()), acc.exp_sum, out.data()));
    return out;
}

std::vector<double> exact_attention(std::span<const float> q, std::span<const HeadVector> keys,
                                    std::span<const HeadVector> values, double scale) {
    if (keys.empty()) throw Error("exact_attention: empty context");
    if (keys.size() != values.size()) throw Error("exact_attention: keys/values length mismatch");
    const std::size_t d = q.size();
    Packed pk;
    pk.n = static_cast<std::int64_t>(keys.size());
    pk.k.reserve(keys.size() * d);
    pk.v.reserve(keys.size() * d);
    for (std::size_t t = 0; t < keys.size(); ++t) {
        check_dim(keys[t].size(), d, "exact_attention keys");
        check_dim(values[t].size(), d, "exact_attention values");
        pk.k.insert(pk.k.end(), keys[t].begin(), keys[t].end());
        pk.v.insert(pk.v.end(), values[t].begin(), values[t].end());
    }
    std::vector<double> out(d);
    double st[3];
    check(psa::seq_attention(q.data(), static_cast<int>(d), pk.k.data(), pk.v.data(), pk.n, scale, 1, out.data(), st));
    return out;
}

std::vector<double> exact_attention_blocks(std::span<const float> q, std::span<const KVBlock* const> blocks,
                                           double scale) {
    if (blocks.empty()) throw Error("exact_attention: empty context");
    const std::size_t d = q.size();
    Packed pk;
    for (const KVBlock* b : blocks) {
        check_dim(static_cast<std::size_t>(b->dim), d, "exact_attention blocks");
        const std::size_t cnt = static_cast<std::size_t>(b->n_tokens) * d;
        pk.k.insert(pk.k.end(), b->keys.begin(), b->keys.begin() + static_cast<std::ptrdiff_t>(cnt));
        pk.v.insert(pk.v.end(), b->values.begin(), b->values.begin() + static_cast<std::ptrdiff_t>(cnt));
        pk.n += b->n_tokens;
    }
    std::vector<double> out(d);
    double st[3];
    check(psa::seq_attention(q.data(), static_cast<int>(d), pk.k.data(), pk.v.data(), pk.n, scale, 1, out.data(), st));
    return out;
}

double block_log_as_oracle(std::span<const float> q, const KVBlock& block, double scale) {
    if (block.n_tokens <= 0) throw Error("block_log_as_oracle: empty block");
    check_dim(q.size(), static_cast<std::size_t>(block.dim), "block_log_as_oracle");
    double st[3];
    check(psa::seq_attention(q.data(), block.dim, block.keys.data(), nullptr, block.n_tokens, scale, 0, nullptr, st));
    return st[2];
}

template float dot_scaled<float>(std::span<const float>, const float*, float);
template double dot_scaled<double>(std::span<const float>, const float*, double);
template ScoredBlockT<float> block_partial_attention_t<float>(std::span<const float>, const KVBlock&, float);
template ScoredBlockT<double> block_partial_attention_t<double>(std::span<const float>, const KVBlock&, double);
template void merge_partial<float>(SoftmaxAccumulatorT<float>&, const ScoredBlockT<float>&);
template void merge_partial<double>(SoftmaxAccumulatorT<double>&, const ScoredBlockT<double>&);
template std::vector<float> finalize<float>(const SoftmaxAccumulatorT<float>&);
template std::vector<double> finalize<double>(const SoftmaxAccumulatorT<double>&);

}  // namespace psattn
