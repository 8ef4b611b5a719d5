// kernels_rank.cu — K2 scoring, K6 oracle masses, K3 ordering, GQA union, batch dispatch.
#include <cuda_bf16.h>
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"
#include "synth.h"

namespace psa {

// =============================================================================
// K2: criticality scoring. Grid (x: block chunks, y: unit). One warp scores one
// metadata record against all G q-heads of the GQA group, so each record is read
// from HBM once per kv-head. Lane owns DPL contiguous dims. fp64 products of
// fp32 operands are exact; only the summation order differs from the
// reference's sequential loop (~1e-16 relative).
// =============================================================================
constexpr int kScoreWarps = 8;

template <typename KV, int G, int DPL>
__global__ void __launch_bounds__(kScoreWarps * 32) score_kernel(PoolView p, BatchView b) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int u = blockIdx.y;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int d = b.d;
    const int base = lane * DPL;
    const int lim = d - base;
    const bool full = (d == 32 * DPL);

    double qd[G][DPL];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        float qf[DPL];
        if (h < b.g)
            load_row<DPL>(b.q + ((size_t)u * b.g + h) * d + base, full, lim, qf);
        else
#pragma unroll
            for (int j = 0; j < DPL; ++j) qf[j] = 0.0f;
#pragma unroll
        for (int j = 0; j < DPL; ++j) qd[h][j] = (double)qf[j];
    }
    const int est = b.estimator;
    const double scale = b.scale;
    const int gsh = 5 - Log2<G>::v;  // lanes per head after reduce-scatter = 1 << gsh
    const int my_h = lane >> gsh;

    for (int64_t pos = (int64_t)blockIdx.x * kScoreWarps + warp; pos < n; pos += (int64_t)gridDim.x * kScoreWarps) {
        const int32_t slot = b.slots[off + pos];
        const char* rec = p.meta + (int64_t)slot * p.meta_bytes;
        float mf[DPL], lf[DPL], hf[DPL];
        load_row<DPL>(reinterpret_cast<const float*>(rec) + base, full, lim, mf);
        load_row<DPL>(reinterpret_cast<const KV*>(rec + (size_t)d * 4) + base, full, lim, lf);
        load_row<DPL>(reinterpret_cast<const KV*>(rec + (size_t)d * 4 + (size_t)d * sizeof(KV)) + base, full, lim, hf);
        double acc[G];
#pragma unroll
        for (int h = 0; h < G; ++h) acc[h] = 0.0;
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
            const double md = (double)mf[j], ld = (double)lf[j], hd = (double)hf[j];
#pragma unroll
            for (int h = 0; h < G; ++h) {
                const double qv = qd[h][j];
                if (est != 1) acc[h] = fma(qv, md, acc[h]);                 // mean_score
                if (est != 0) acc[h] = fma(qv, qv >= 0.0 ? hd : ld, acc[h]); // max(q*lo, q*hi)
            }
        }
        const double tot = reduce_scatter_d<G>(acc, lane);
        if ((lane & ((1 << gsh) - 1)) == 0 && my_h < b.g) {
            const double s = est == 2 ? 0.5 * (tot * scale) : tot * scale;
            b.keys[off * b.g + (int64_t)my_h * n + pos] = make_key(s, (uint32_t)pos, b.pos_bits);
        }
    }
}

// =============================================================================
// K6: fp64 block masses log(sum_t exp(q.k_t*scale)) for Oracle ranking and the
// coverage audit (reference engine.cpp:64-72 computes these in plan_blocks).
// =============================================================================
template <typename KV, int DPL>
__global__ void __launch_bounds__(kScoreWarps * 32) oracle_mass_kernel(PoolView p, BatchView b) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int u = blockIdx.y;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int d = b.d;
    const int base = lane * DPL;
    const int lim = d - base;
    const bool full = (d == 32 * DPL);
    for (int64_t pos = (int64_t)blockIdx.x * kScoreWarps + warp; pos < n; pos += (int64_t)gridDim.x * kScoreWarps) {
        const int32_t slot = b.slots[off + pos];
        const int nt = p.ntok[slot];
        const KV* k = reinterpret_cast<const KV*>(p.kv + (int64_t)slot * p.slot_bytes) + base;
        for (int h = 0; h < b.g; ++h) {
            float qf[DPL];
            load_row<DPL>(b.q + ((size_t)u * b.g + h) * d + base, full, lim, qf);
            double mx = -INFINITY, es = 0.0;
            // two passes like the reference: max, then sum of exp
            for (int pass = 0; pass < 2; ++pass) {
                for (int t = 0; t < nt; ++t) {
                    float kf[DPL];
                    load_row<DPL>(k + (size_t)t * d, full, lim, kf);
                    double a = 0.0;
#pragma unroll
                    for (int j = 0; j < DPL; ++j) a = fma((double)qf[j], (double)kf[j], a);
                    const double s = warp_sum_d(a) * b.scale;
                    if (pass == 0) mx = fmax(mx, s);
                    else es += exp(s - mx);
                }
            }
            const double la = mx + log(es);
            const int64_t idx = off * b.g + (int64_t)h * n + pos;
            if (lane == 0) {
                b.omass[idx] = la;
                if (b.rank_oracle) b.keys[idx] = make_key(la, (uint32_t)pos, b.pos_bits);
            }
        }
    }
}

// =============================================================================
// K3: ordering. One CTA per (unit, head): all-ascending bitonic network (the
// "flip" formulation, every compare-exchange puts the min at the lower index),
// so indices >= n behave as +inf and need no padding. Keys are unique (they
// carry the position), so the result is THE (score desc, id asc) order.
// Emits rank-ordered list positions and the matching pool slots.
// =============================================================================
constexpr int kSortThreads = 1024;
constexpr int kSmemSortMax = 16384;  // keys per head sorted in shared memory (128 KB)

__device__ __forceinline__ void bitonic_ascending(uint64_t* a, int64_t n, int64_t n2) {
    for (int64_t k = 2; k <= n2; k <<= 1) {
        for (int64_t j = k >> 1; j > 0; j >>= 1) {
            for (int64_t i = threadIdx.x; i < (n2 >> 1); i += blockDim.x) {
                const int64_t lo = ((i / j) * 2 * j) + (i % j);
                const int64_t hi = (j == (k >> 1)) ? (lo ^ (k - 1)) : (lo + j);
                if (hi < n) {
                    const uint64_t x = a[lo], y = a[hi];
                    if (x > y) {
                        a[lo] = y;
                        a[hi] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(kSortThreads) sort_kernel(BatchView b) {
    extern __shared__ uint64_t skeys[];
    const int qi = blockIdx.x;
    const int u = qi / b.g, h = qi % b.g;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int64_t hb = off * b.g + (int64_t)h * n;
    int64_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    const bool in_smem = b.max_n <= kSmemSortMax;  // smem sized for max_n by the launcher
    uint64_t* a = in_smem ? skeys : (b.keys + hb);
    if (in_smem)
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a[i] = b.keys[hb + i];
    __syncthreads();
    bitonic_ascending(a, n, n2);
    const uint64_t mask = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);
    for (int64_t r = threadIdx.x; r < n; r += blockDim.x) {
        const int32_t pos = (int32_t)(a[r] & mask);
        b.rpos[hb + r] = pos;
        b.rslot[hb + r] = b.slots[off + pos];
    }
}

// =============================================================================
// GQA union of processed blocks per unit (for the algorithmic byte count).
// =============================================================================
__global__ void union_kernel(BatchView b, int64_t* out) {
    extern __shared__ uint32_t bits[];
    const int u = blockIdx.x;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int64_t words = (n + 31) / 32;
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) bits[i] = 0;
    __syncthreads();
    for (int h = 0; h < b.g; ++h) {
        const int64_t hb = off * b.g + (int64_t)h * n;
        const int64_t bp = b.bp[(int64_t)u * b.g + h];
        for (int64_t r = threadIdx.x; r < bp; r += blockDim.x) {
            const int32_t pos = b.rpos[hb + r];
            atomicOr(&bits[pos >> 5], 1u << (pos & 31));
        }
    }
    __syncthreads();
    __shared__ unsigned long long total;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    unsigned long long c = 0;
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) c += __popc(bits[i]);
    atomicAdd(&total, c);
    __syncthreads();
    if (threadIdx.x == 0) out[u] = (int64_t)total;
}

cudaError_t launch_union(const BatchView& b, int64_t* out, cudaStream_t st) {
    const size_t smem = (size_t)((b.max_n + 31) / 32) * 4;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    if (smem > 48 * 1024) cudaFuncSetAttribute(union_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    union_kernel<<<b.n_units, 512, smem, st>>>(b, out);
    return cudaGetLastError();
}

// =============================================================================
// Launch dispatch
// =============================================================================
template <typename KV, int G>
static void launch_score_g(const PoolView& p, const BatchView& b, dim3 grid, cudaStream_t st) {
    switch (dpl_for(b.d)) {
        case 2: score_kernel<KV, G, 2><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
        case 4: score_kernel<KV, G, 4><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
        default: score_kernel<KV, G, 8><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
    }
}

template <typename KV>
static void launch_score(const PoolView& p, const BatchView& b, dim3 grid, cudaStream_t st) {
    if (g_for(b.g) == 4) launch_score_g<KV, 4>(p, b, grid, st);
    else launch_score_g<KV, 8>(p, b, grid, st);
}

template <typename KV>
static void launch_oracle(const PoolView& p, const BatchView& b, dim3 grid, cudaStream_t st) {
    switch (dpl_for(b.d)) {
        case 2: oracle_mass_kernel<KV, 2><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
        case 4: oracle_mass_kernel<KV, 4><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
        default: oracle_mass_kernel<KV, 8><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
    }
}

int launch_batch(const PoolView& p, const BatchView& b, cudaStream_t st, cudaEvent_t* marks) {
    // marks (optional, 5 events): start | oracle | score | order | progressive
    int launches = 0;
    if (marks) cudaEventRecord(marks[0], st);
    const int64_t chunks = (b.max_n + kScoreWarps - 1) / kScoreWarps;
    dim3 grid((unsigned)(chunks < 65535 ? (chunks > 0 ? chunks : 1) : 65535), (unsigned)b.n_units);
    if (b.has_oracle) {
        if (p.dtype == 0) launch_oracle<float>(p, b, grid, st);
        else launch_oracle<__nv_bfloat16>(p, b, grid, st);
        ++launches;
    }
    if (marks) cudaEventRecord(marks[1], st);
    if (!b.rank_oracle) {
        if (p.dtype == 0) launch_score<float>(p, b, grid, st);
        else launch_score<__nv_bfloat16>(p, b, grid, st);
        ++launches;
    }
    if (marks) cudaEventRecord(marks[2], st);
    const int nq = b.n_units * b.g;
    const size_t smem = (size_t)(b.max_n <= kSmemSortMax ? b.max_n : 0) * sizeof(uint64_t);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sort_kernel<<<nq, kSortThreads, smem, st>>>(b);
    ++launches;
    if (marks) cudaEventRecord(marks[3], st);
    launch_psa(p, b, st);
    ++launches;
    if (marks) cudaEventRecord(marks[4], st);
    if (cudaPeekAtLastError() != cudaSuccess) return -1;
    return launches;
}

}  // namespace psa
