// psattn/attention.hpp — block partial attention, softmax merge and the fp64 oracles (B200 build).
// Source-compatible with the reference's include/psattn/attention.hpp:10-130: same structs,
// same function names, argument meaning and exceptions. The bodies are NOT host code here:
// every function runs on the device (csrc/attention_kernels.cu) with the reference's arithmetic
// order — sequential dot products over d, token-order exponent sums and weighted value sums,
// explicit (non-fused) rounding — so results match the reference to the last bit except where
// device exp/log differ from glibc by an ulp. Templates are instantiated for float and double
// (the two element types the reference uses).
//
// These are per-call API entry points (one block, one merge); the batched decode path
// (psattn_run_batch) runs the same arithmetic inside its progressive kernels.
#pragma once

#include <cmath>
#include <limits>
#include <span>
#include <vector>

#include "psattn/types.hpp"

namespace psattn {

// Partial attention over one block, carried as (max_score, exp_sum) with
// log_as = max_score + ln(exp_sum) (reference attention.hpp:12-24).
template <typename T>
struct ScoredBlockT {
    std::vector<T> out_unnorm;  // sum_i exp(score_i - max_score) * v_i
    T max_score = -std::numeric_limits<T>::infinity();
    T exp_sum = 0;
    T log_as = -std::numeric_limits<T>::infinity();
};

// Running merge state over blocks; exp_sum == 0 iff nothing accumulated (attention.hpp:26-37).
template <typename T>
struct SoftmaxAccumulatorT {
    std::vector<T> out_unnorm;
    T max_score = -std::numeric_limits<T>::infinity();
    T exp_sum = 0;
    T log_as_acc = -std::numeric_limits<T>::infinity();

    bool empty() const { return exp_sum == 0; }
};

using ScoredBlockResult = ScoredBlockT<float>;
using SoftmaxAccumulator = SoftmaxAccumulatorT<float>;

// (sum_i q_i * k_i in T, index order) * scale (attention.hpp:39-45). k has q.size() elements.
template <typename T>
T dot_scaled(std::span<const float> q, const float* k, T scale);

// Scores one block against q: max score, exponent sum, unnormalised weighted value sum
// (attention.hpp:47-77). Throws Error on an empty block or a dimension mismatch.
template <typename T>
ScoredBlockT<T> block_partial_attention_t(std::span<const float> q, const KVBlock& block, T scale);

inline ScoredBlockResult block_partial_attention(std::span<const float> q, const KVBlock& block, float scale) {
    return block_partial_attention_t<float>(q, block, scale);
}

// Folds a partial into the accumulator at the common max; an empty accumulator absorbs the
// partial unchanged (attention.hpp:79-101).
template <typename T>
void merge_partial(SoftmaxAccumulatorT<T>& acc, const ScoredBlockT<T>& part);

// out_unnorm / exp_sum; throws Error when nothing was accumulated (attention.hpp:103-109).
template <typename T>
std::vector<T> finalize(const SoftmaxAccumulatorT<T>& acc);

// fp64 attention over a token sequence (attention.cpp:7-34).
std::vector<double> exact_attention(std::span<const float> q, std::span<const HeadVector> keys,
                                    std::span<const HeadVector> values, double scale);

// Same over the tokens of a block sequence (attention.cpp:36-63).
std::vector<double> exact_attention_blocks(std::span<const float> q, std::span<const KVBlock* const> blocks,
                                           double scale);

// fp64 log of a block's unnormalised softmax mass (attention.cpp:65-79).
double block_log_as_oracle(std::span<const float> q, const KVBlock& block, double scale);

inline double default_scale(std::size_t dim) { return 1.0 / std::sqrt(static_cast<double>(dim)); }

extern template float dot_scaled<float>(std::span<const float>, const float*, float);
extern template double dot_scaled<double>(std::span<const float>, const float*, double);
extern template ScoredBlockT<float> block_partial_attention_t<float>(std::span<const float>, const KVBlock&, float);
extern template ScoredBlockT<double> block_partial_attention_t<double>(std::span<const float>, const KVBlock&, double);
extern template void merge_partial<float>(SoftmaxAccumulatorT<float>&, const ScoredBlockT<float>&);
extern template void merge_partial<double>(SoftmaxAccumulatorT<double>&, const ScoredBlockT<double>&);
extern template std::vector<float> finalize<float>(const SoftmaxAccumulatorT<float>&);
extern template std::vector<double> finalize<double>(const SoftmaxAccumulatorT<double>&);

}  // namespace psattn
