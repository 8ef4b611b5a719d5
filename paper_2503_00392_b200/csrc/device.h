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

}  // namespace psa
