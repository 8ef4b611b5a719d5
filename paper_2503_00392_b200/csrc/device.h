// device.h — internal interface of the device layer for the C++ host code.
#pragma once

#include <atomic>
#include <string>

#include <cuda_runtime.h>
#include <stdint.h>

#include "psattn_b200.h"

namespace psa {

struct PoolView;

void set_error(const std::string& msg);
const char* last_error();
int fail(int code, const std::string& msg);

// Grows slot capacity and/or tokens-per-slot, preserving contents.
int pool_grow(psattn_pool* pool, int64_t n_slots, int32_t T);
// Host fp32 blocks -> slots (row_stride_floats between consecutive blocks' K), metadata built.
int pool_put(psattn_pool* pool, int64_t n, const int32_t* slots, const int32_t* ntok, const float* keys,
             const float* values, int64_t row_stride_floats, cudaStream_t st);
int read_slot(const psattn_pool* pool, int64_t slot, int32_t ntok, float* keys, float* values);
int read_meta(const psattn_pool* pool, int64_t slot, float* mean, float* lo, float* hi);
int cuda_fail(cudaError_t e, const char* what);
// Changes whenever a launch-shaping knob (psattn_set_*) changes; ~0 while profiling is on. A
// captured launch sequence is reusable while this and its inputs are unchanged.
uint64_t launch_config_generation();
// psattn_run_batch internals shared with the audit/tradeoff tooling (tradeoff.cu).
int validate_batch(const psattn_pool* pool, const psattn_batch* b);
size_t ws_omass_offset(const psattn_batch* b);
size_t ws_rpos_offset(const psattn_batch* b);
const PoolView& pool_view(const psattn_pool* pool);
// Two-tier pools (tier.cpp).
int pool_create_tiered(const psattn_pool_desc* desc, int64_t n_blocks, int64_t fast_slots, psattn_pool** out);
int32_t* pool_loc(psattn_pool* pool);
char* pool_host_kv(psattn_pool* pool);
void pool_pack_into(const psattn_pool* pool, int64_t n, const int64_t* blocks, const int32_t* ntok, const float* keys,
                    const float* values);

// ProgressiveRun device state (progressive_api.cu).
struct RunState;
int prun_create(const float* q, int d, RunState** out);
void prun_destroy(RunState* s);
// Folds n host blocks (in order) into the accumulator; log_as[b] = the block's log mass.
int prun_consume(RunState* s, float scale, int n, const int32_t* ntok, const float* const* keys,
                 const float* const* values, float* log_as);
int prun_result(const RunState* s, float* out);

// attention.hpp API (attention_kernels.cu): one token sequence K/V [n][d] (host fp32), the
// reference's arithmetic order. out [d] (unnormalised unless `normalize`; V may be null),
// stats [3] = max score, exponent sum, log mass.
int seq_attention(const float* q, int d, const float* K, const float* V, int64_t n, float scale, int normalize,
                  float* out, float* stats);
int seq_attention(const float* q, int d, const float* K, const float* V, int64_t n, double scale, int normalize,
                  double* out, double* stats);
// merge_partial on a non-empty accumulator: acc_stats/part_stats [3] = max, exponent sum, log mass.
int softmax_merge(float* acc_out, float* acc_stats, const float* part_out, const float* part_stats, int d);
int softmax_merge(double* acc_out, double* acc_stats, const double* part_out, const double* part_stats, int d);
int softmax_finalize(const float* acc_out, int d, float es, float* out);
int softmax_finalize(const double* acc_out, int d, double es, double* out);

}  // namespace psa
