// kernels_misc.cu — K1 metadata build, KV append, slot install/scatter (sm_100a).
#include <cuda_bf16.h>
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace psa {

// Specialised lane mappings for d = 64 and d = 128; every other d <= 256 runs
// the masked 8-dims-per-lane variant.
int dpl_for(int d) { return d == 128 ? 4 : d == 64 ? 2 : 8; }
int tok_for(int T) { return T <= 16 ? 16 : T <= 32 ? 32 : kMaxBlockTokens; }
int g_for(int g) { return g <= 4 ? 4 : 8; }

// =============================================================================
// K1: metadata build. One warp per slot; lane i covers dims i, i+32, ...
// lo/hi: elementwise min/max with std::min/std::max semantics; mean: fp64 sum
// in token order, divided by n, rounded to fp32 — bit-identical to the reference.
// =============================================================================
template <typename KV>
__global__ void meta_build_kernel(PoolView p, const int32_t* list, int64_t s0, int64_t s1) {
    const int lane = threadIdx.x & 31;
    const int64_t idx = s0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (idx >= s1) return;
    const int64_t slot = list ? (int64_t)list[idx] : idx;
    const int n = p.ntok[slot];
    const int d = p.d;
    const KV* k = kv_block<KV>(p, slot);
    char* rec = p.meta + slot * p.meta_bytes;
    float* mean = reinterpret_cast<float*>(rec);
    KV* lo = reinterpret_cast<KV*>(rec + (size_t)d * 4);
    KV* hi = reinterpret_cast<KV*>(rec + (size_t)d * 4 + (size_t)d * sizeof(KV));
    for (int i = lane; i < d; i += 32) {
        if (n <= 0) {
            mean[i] = 0.0f;
            lo[i] = KVT<KV>::from_f(0.0f);
            hi[i] = KVT<KV>::from_f(0.0f);
            continue;
        }
        float l = KVT<KV>::to_f(k[i]);
        float h = l;
        double s = l;
        for (int t = 1; t < n; ++t) {
            const float x = KVT<KV>::to_f(k[(size_t)t * d + i]);
            l = (x < l) ? x : l;
            h = (h < x) ? x : h;
            s = __dadd_rn(s, (double)x);
        }
        mean[i] = __double2float_rn(__ddiv_rn(s, (double)n));
        lo[i] = KVT<KV>::from_f(l);  // exact: l is a KV value
        hi[i] = KVT<KV>::from_f(h);
    }
}

cudaError_t launch_meta_build(const PoolView& p, const int32_t* list, int64_t s0, int64_t s1, cudaStream_t st) {
    if (s1 <= s0) return cudaSuccess;
    const int warps = 8;
    const int64_t blocks = (s1 - s0 + warps - 1) / warps;
    if (p.dtype == 0)
        meta_build_kernel<float><<<(unsigned)blocks, warps * 32, 0, st>>>(p, list, s0, s1);
    else
        meta_build_kernel<__nv_bfloat16><<<(unsigned)blocks, warps * 32, 0, st>>>(p, list, s0, s1);
    return cudaGetLastError();
}

// Decode-step KV append: sequence i writes one token's K and V
// (fp32, converted to the pool dtype) at row ntok[slot] of its tail slot, then
// the slot's metadata is rebuilt over its rows exactly like K1 (reference
// put_block -> build_metadata, store.cpp:59-78, metadata.cpp:8-34). One warp per
// sequence; rows past ntok stay zero so the progressive kernel's unmasked loads
// remain finite.
template <typename KV>
__global__ void append_tokens_kernel(PoolView p, int32_t n, const int32_t* __restrict__ slots,
                                     const float* __restrict__ keys, const float* __restrict__ values,
                                     int32_t* __restrict__ status) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= n) return;
    const int64_t slot = slots[i];
    const int d = p.d;
    const int row = p.ntok[slot];
    if (row >= p.T) {  // full block: the caller must open a new slot
        if (lane == 0) atomicExch(status, 1);
        return;
    }
    KV* k = reinterpret_cast<KV*>(p.kv + slot * p.slot_bytes);
    KV* v = k + (size_t)p.T * d;
    for (int j = lane; j < d; j += 32) {
        k[(size_t)row * d + j] = KVT<KV>::from_f(keys[(size_t)i * d + j]);
        v[(size_t)row * d + j] = KVT<KV>::from_f(values[(size_t)i * d + j]);
    }
    __syncwarp();
    const int nt = row + 1;
    char* rec = p.meta + slot * p.meta_bytes;
    float* mean = reinterpret_cast<float*>(rec);
    KV* lo = reinterpret_cast<KV*>(rec + (size_t)d * 4);
    KV* hi = reinterpret_cast<KV*>(rec + (size_t)d * 4 + (size_t)d * sizeof(KV));
    for (int j = lane; j < d; j += 32) {
        float l = KVT<KV>::to_f(k[j]);
        float h = l;
        double sm = l;
        for (int t = 1; t < nt; ++t) {
            const float x = KVT<KV>::to_f(k[(size_t)t * d + j]);
            l = (x < l) ? x : l;
            h = (h < x) ? x : h;
            sm = __dadd_rn(sm, (double)x);
        }
        mean[j] = __double2float_rn(__ddiv_rn(sm, (double)nt));
        lo[j] = KVT<KV>::from_f(l);
        hi[j] = KVT<KV>::from_f(h);
    }
    if (lane == 0) p.ntok[slot] = nt;
}

cudaError_t launch_append(const PoolView& p, int32_t n, const int32_t* slots, const float* keys,
                          const float* values, int32_t* status, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int warps = 8;
    if (p.dtype == 0)
        append_tokens_kernel<float><<<(n + warps - 1) / warps, warps * 32, 0, st>>>(p, n, slots, keys, values, status);
    else
        append_tokens_kernel<__nv_bfloat16><<<(n + warps - 1) / warps, warps * 32, 0, st>>>(p, n, slots, keys, values,
                                                                                              status);
    return cudaGetLastError();
}

// Copies n staged slot images ([2][T][d] in the pool dtype) into pool slots and sets ntok.
__global__ void scatter_slots_kernel(PoolView p, const char* __restrict__ staged, const int32_t* __restrict__ slots,
                                     const int32_t* __restrict__ ntok, int64_t n) {
    const int64_t i = blockIdx.x;
    if (i >= n) return;
    const int64_t slot = slots[i];
    const int4* src = reinterpret_cast<const int4*>(staged + i * p.slot_bytes);
    int4* dst = reinterpret_cast<int4*>(p.kv + slot * p.slot_bytes);
    for (int64_t e = threadIdx.x; e < p.slot_bytes / 16; e += blockDim.x) dst[e] = src[e];
    if (threadIdx.x == 0) p.ntok[slot] = ntok[i];
}

// Two-tier pools: installs blocks[i] from the pinned host backing tier into HBM slot dst[i]
// (reads over PCIe/C2C, 16-byte vectors; one CTA per block).
__global__ void install_blocks_kernel(PoolView p, const int64_t* __restrict__ blocks, const int32_t* __restrict__ dst,
                                      int64_t n) {
    const int64_t i = blockIdx.x;
    if (i >= n) return;
    const int4* src = reinterpret_cast<const int4*>(p.host_kv + blocks[i] * p.slot_bytes);
    int4* out = reinterpret_cast<int4*>(p.kv + (int64_t)dst[i] * p.slot_bytes);
    for (int64_t e = threadIdx.x; e < p.slot_bytes / 16; e += blockDim.x) out[e] = src[e];
}

cudaError_t launch_install(const PoolView& p, const int64_t* d_blocks, const int32_t* d_dst, int64_t n,
                           cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    install_blocks_kernel<<<(unsigned)n, 256, 0, st>>>(p, d_blocks, d_dst, n);
    return cudaGetLastError();
}

cudaError_t launch_scatter(const PoolView& p, const void* staged, const int32_t* d_slots, const int32_t* d_ntok,
                           int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    scatter_slots_kernel<<<(unsigned)n, 128, 0, st>>>(p, static_cast<const char*>(staged), d_slots, d_ntok, n);
    return cudaGetLastError();
}

}  // namespace psa
