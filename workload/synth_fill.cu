// synth_fill.cu — device fill of a pool's slot image from the seekable generator
// (psattn_synth.h). Directions first (one thread per unit, sequential fp64 norm so the
// host copy is bit-identical), then every K/V element of every block.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "psattn_synth.h"
#include "synth.h"

namespace {

__global__ void synth_dir_kernel(uint64_t seed, int32_t d, int32_t n_units, const int64_t* unit_ids, float* dirs) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n_units) return;
    psa_synth::direction(seed, unit_ids[u], d, dirs + (size_t)u * d);
}

__device__ __forceinline__ void store_kv(float* p, float x) { *p = x; }
__device__ __forceinline__ void store_kv(__nv_bfloat16* p, float x) { *p = __float2bfloat16_rn(x); }

template <typename KV>
__global__ void synth_fill_kernel(psattn_synth_params prm, char* kv, int32_t* ntok, int64_t slot_bytes,
                                  const int64_t* unit_ids, const int64_t* slot_off, const int64_t* tokens,
                                  const float* dirs) {
    const int u = blockIdx.y;
    const int T = prm.block_tokens, d = prm.dim;
    const int64_t ntok_total = tokens[u];
    const int64_t nb = (ntok_total + T - 1) / T;
    const int64_t uid = unit_ids[u];
    const int64_t per_block = (int64_t)T * d;
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int64_t slot = slot_off[u] + b;
        const int planted = psa_synth::is_planted(prm.seed, prm.planted_prob, uid, b);
        KV* kp = reinterpret_cast<KV*>(kv + slot * slot_bytes);
        KV* vp = kp + per_block;
        for (int64_t e = threadIdx.x; e < per_block; e += blockDim.x) {
            const int64_t t = e / d;
            const int i = (int)(e - t * d);
            const int64_t tok = b * T + t;
            float kx = 0.0f, vx = 0.0f;
            if (tok < ntok_total) {
                kx = psa_synth::key_at(prm.seed, uid, tok, i, d, planted, prm.skew, dirs[(size_t)u * d + i]);
                vx = psa_synth::value_at(prm.seed, uid, b, tok, i, d);
                if (prm.round_bf16) {
                    kx = psa_synth::round_bf16(kx);
                    vx = psa_synth::round_bf16(vx);
                }
            }
            store_kv(kp + e, kx);
            store_kv(vp + e, vx);
        }
        if (threadIdx.x == 0) {
            const int64_t rem = ntok_total - b * T;
            ntok[slot] = (int32_t)(rem < T ? rem : T);
        }
    }
}

}  // namespace

extern "C" int psattn_synth_fill(const psattn_synth_params* p, void* kv, int32_t* ntok, int64_t slot_bytes,
                                 int32_t kv_dtype, int64_t n_slots, int32_t n_units, const int64_t* unit_ids,
                                 const int64_t* slot_off, const int64_t* tokens, void* stream) {
    if (!p || !kv || !ntok || !unit_ids || !slot_off || !tokens) return (int)cudaErrorInvalidValue;
    if (n_units <= 0) return 0;
    const int T = p->block_tokens;
    int64_t max_blocks = 0;
    for (int u = 0; u < n_units; ++u) {
        const int64_t nb = (tokens[u] + T - 1) / T;
        if (slot_off[u] < 0 || slot_off[u] + nb > n_slots) return (int)cudaErrorInvalidValue;
        max_blocks = std::max(max_blocks, nb);
    }
    cudaStream_t st = (cudaStream_t)stream;
    int64_t* d_arr = nullptr;
    float* d_dirs = nullptr;
    cudaError_t e;
    if ((e = cudaMallocAsync(&d_arr, (size_t)n_units * 24, st)) != cudaSuccess) return (int)e;
    if ((e = cudaMallocAsync(&d_dirs, (size_t)n_units * p->dim * 4, st)) != cudaSuccess) return (int)e;
    cudaMemcpyAsync(d_arr, unit_ids, (size_t)n_units * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_arr + n_units, slot_off, (size_t)n_units * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_arr + 2 * n_units, tokens, (size_t)n_units * 8, cudaMemcpyHostToDevice, st);
    synth_dir_kernel<<<(n_units + 127) / 128, 128, 0, st>>>(p->seed, p->dim, n_units, d_arr, d_dirs);
    const unsigned gx = (unsigned)(max_blocks < 4096 ? (max_blocks > 0 ? max_blocks : 1) : 4096);
    const dim3 grid(gx, (unsigned)n_units);
    if (kv_dtype == 0)
        synth_fill_kernel<float><<<grid, 256, 0, st>>>(*p, static_cast<char*>(kv), ntok, slot_bytes, d_arr,
                                                       d_arr + n_units, d_arr + 2 * n_units, d_dirs);
    else
        synth_fill_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(*p, static_cast<char*>(kv), ntok, slot_bytes, d_arr,
                                                               d_arr + n_units, d_arr + 2 * n_units, d_dirs);
    e = cudaGetLastError();
    cudaFreeAsync(d_arr, st);
    cudaFreeAsync(d_dirs, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return (int)e;
}
