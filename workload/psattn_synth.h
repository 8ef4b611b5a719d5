/* psattn_synth.h — the seekable synthetic KV/query generator (benchmark + parity fixture).
 *
 * NOT part of the attention path or of libpsattn_b200.so. Two libraries are built from it
 * (workload/Makefile):
 *   libpsattn_synth_host.so  host generator only (g++, no CUDA): the reference arm of the
 *                            benchmark and the parity tests build their CPU inputs with it;
 *   libpsattn_synth_dev.so   the same + a device fill of a pool's slot image (nvcc). It does
 *                            not link the product library: callers pass the pool layout
 *                            (psattn_pool_get_layout) and rebuild metadata themselves
 *                            (psattn_pool_build_metadata).
 * Values are a pure function of (seed, unit_id, block, token, dim), identical on host and
 * device. Keys: approx-N(0,1) noise, plus skew*direction on planted blocks (pattern of the
 * reference workload generator, workload.cpp:84-122); values: per-block centroid + 0.25*noise. */
#ifndef PSATTN_SYNTH_H
#define PSATTN_SYNTH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t seed;
    int32_t dim;
    int32_t block_tokens;
    float skew;
    float planted_prob;   /* probability a block is planted (0 = isotropic keys) */
    int32_t round_bf16;   /* round K/V to bf16 values (what a bf16 pool stores) */
    int32_t reserved;
} psattn_synth_params;

/* Unit direction (dim floats) for unit_id. */
void psattn_synth_direction(const psattn_synth_params* p, int64_t unit_id, float* out);
/* Query of q-head `head` for unit_id: normalize(dir + 0.1*g_head) * sqrt(dim). */
void psattn_synth_query(const psattn_synth_params* p, int64_t unit_id, int32_t head, float* out);
/* Host copy of one unit's blocks [first_block, first_block+n_blocks): keys/values
 * [n_blocks][block_tokens][dim]; tokens past n_tokens_total are zero. */
void psattn_synth_unit_host(const psattn_synth_params* p, int64_t unit_id, int64_t first_block, int64_t n_blocks,
                            int64_t n_tokens_total, float* keys, float* values);
int psattn_synth_is_planted(const psattn_synth_params* p, int64_t unit_id, int64_t block);

/* Device fill (libpsattn_synth_dev.so only): for each unit u (host arrays of n_units entries),
 * blocks [0, ceil(tokens[u]/B)) are written into slots slot_off[u] + b of the slot image
 * kv ([n_slots][2][B][dim], kv_dtype 0 = f32, 1 = bf16; slot_bytes apart) and ntok[slot] is
 * set. Metadata is NOT built. Stream-ordered; returns 0 or a cudaError_t code. */
int psattn_synth_fill(const psattn_synth_params* p, void* kv, int32_t* ntok, int64_t slot_bytes, int32_t kv_dtype,
                      int64_t n_slots, int32_t n_units, const int64_t* unit_ids, const int64_t* slot_off,
                      const int64_t* tokens, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PSATTN_SYNTH_H */
