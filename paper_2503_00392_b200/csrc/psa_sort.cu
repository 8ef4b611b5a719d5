// psa_sort.cu — segmented stable LSD radix sort of (uint64 key, int32 value) pairs on the device.
//
// Serves the full rankings the reference computes with std::sort (rank_by_scores,
// metadata.cpp:87-96; plan_blocks' ranked_ids, engine.cpp:75-88): the progressive path itself
// orders blocks lazily (a tranche at a time, psa_order.cuh), but a caller of plan_blocks /
// rank_by_scores gets every rank. Keys sort ascending; the sort is stable, so equal keys keep
// their input order — with keys = order-preserving transform of the score (descending) and the
// input in block-id order, the result is "score desc, block id asc" exactly.
//
// One CTA (1024 threads) per segment, 8-bit digits, 8 passes (a pass whose digit is the same
// for every key of the segment is skipped). Per pass: digit histogram, exclusive scan, then
// the segment is scattered tile by tile (1024 keys): a key's destination is its digit's base
// + the count of equal digits in earlier warps of the tile (per-warp counts, prefix over warps)
// + its rank among equal digits of its own warp (__match_any_sync), which keeps the order.
#include <cuda_runtime.h>
#include <stdint.h>

#include "device.h"
#include "kernels.cuh"

namespace psa {

namespace {
constexpr int kSortThreads = 1024;
constexpr int kSortWarps = kSortThreads / 32;

__device__ __forceinline__ void seg_bounds(const int64_t* list_off, int g, int s, int64_t& start, int64_t& len) {
    const int u = s / g, h = s % g;
    const int64_t o = list_off[u], n = list_off[u + 1] - o;
    start = o * g + (int64_t)h * n;
    len = n;
}

// vals_in == nullptr: the values are the positions 0..len-1 within the segment.
__global__ void __launch_bounds__(kSortThreads) seg_radix_sort_kernel(uint64_t* keys, const int32_t* vals_in,
                                                                      int32_t* vals_out, uint64_t* tk, int32_t* tv,
                                                                      int32_t* tv2, const int64_t* list_off, int g) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t base[256];
    __shared__ uint32_t tile_cnt[256];
    __shared__ uint16_t wcnt[kSortWarps][256];
    __shared__ int skip;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int64_t start, n;
    seg_bounds(list_off, g, blockIdx.x, start, n);
    uint64_t* ka = keys + start;
    uint64_t* kb = tk + start;
    int32_t* va = tv + start;
    int32_t* vb = tv2 + start;
    for (int64_t i = tid; i < n; i += kSortThreads) va[i] = vals_in ? vals_in[start + i] : (int32_t)i;
    const unsigned lt_mask = (1u << lane) - 1u;
    for (int shift = 0; shift < 64; shift += 8) {
        if (tid < 256) hist[tid] = 0;
        __syncthreads();
        for (int64_t i = tid; i < n; i += kSortThreads) atomicAdd(&hist[(ka[i] >> shift) & 255u], 1u);
        __syncthreads();
        if (tid == 0) skip = hist[(ka[0] >> shift) & 255u] == (uint32_t)n;
        if (tid < 32) {  // exclusive scan of 256 digit counts: 8 per lane
            uint32_t loc[8], s = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                loc[j] = s;
                s += hist[lane * 8 + j];
            }
            uint32_t inc = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            const uint32_t ex = inc - s;
#pragma unroll
            for (int j = 0; j < 8; ++j) base[lane * 8 + j] = ex + loc[j];
        }
        __syncthreads();
        if (skip) continue;  // every key has the same digit: the order is unchanged
        for (int64_t t0 = 0; t0 < n; t0 += kSortThreads) {
            const int64_t i = t0 + tid;
            const bool valid = i < n;
            const uint64_t k = valid ? ka[i] : 0ull;
            const int32_t v = valid ? va[i] : 0;
            const int dg = valid ? (int)((k >> shift) & 255u) : 256;
            const unsigned peers = __match_any_sync(0xffffffffu, dg);
            const int rank = __popc(peers & lt_mask);
            for (int j = tid; j < kSortWarps * 256; j += kSortThreads) (&wcnt[0][0])[j] = 0;
            __syncthreads();
            if (valid && rank == 0) wcnt[warp][dg] = (uint16_t)__popc(peers);
            __syncthreads();
            if (tid < 256) {
                uint32_t run = 0;
                for (int w = 0; w < kSortWarps; ++w) {
                    const uint32_t c = wcnt[w][tid];
                    wcnt[w][tid] = (uint16_t)run;
                    run += c;
                }
                tile_cnt[tid] = run;
            }
            __syncthreads();
            if (valid) {
                const uint32_t dst = base[dg] + wcnt[warp][dg] + (uint32_t)rank;
                kb[dst] = k;
                vb[dst] = v;
            }
            __syncthreads();
            if (tid < 256) base[tid] += tile_cnt[tid];
            __syncthreads();
        }
        uint64_t* kt = ka;
        ka = kb;
        kb = kt;
        int32_t* vt = va;
        va = vb;
        vb = vt;
    }
    // results are in (ka, va): keys back into `keys` if they ended in the scratch, values out
    for (int64_t i = tid; i < n; i += kSortThreads) {
        if (ka != keys + start) keys[start + i] = ka[i];
        vals_out[start + i] = va[i];
    }
}
}  // namespace

// Sorts every (unit, head) segment of a batch-shaped array (segment u*g + h starts at
// list_off[u]*g + h*n_u and holds n_u = list_off[u+1] - list_off[u] entries). keys are sorted in
// place; vals_out receives the values in key order (vals_in == nullptr: positions in segment).
// Scratch: tk (total*g keys), tv and tv2 (total*g values).
cudaError_t launch_seg_sort(uint64_t* keys, const int32_t* vals_in, int32_t* vals_out, uint64_t* tk, int32_t* tv,
                            int32_t* tv2, const int64_t* list_off, int n_units, int g, cudaStream_t st) {
    seg_radix_sort_kernel<<<(unsigned)(n_units * g), kSortThreads, 0, st>>>(keys, vals_in, vals_out, tk, tv, tv2,
                                                                           list_off, g);
    return cudaGetLastError();
}

}  // namespace psa
