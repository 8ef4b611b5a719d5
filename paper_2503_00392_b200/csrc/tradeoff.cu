// tradeoff.cu — GPU oracle/audit tooling around the PSA path:
//
//   psattn_exact_attention  fp64 exact attention over every block of a list
//                           (exact_attention_blocks, reference attention.cpp:36-63) —
//                           the error reference of the threshold / top-k sweep (config 3);
//   psattn_tradeoff         run_tradeoff (reference scenario.cpp:451-545): fp64 block masses,
//                           per-query coverage curves in mass order, the smallest uniform
//                           top-k meeting a coverage target for every query, and PSA at
//                           epsilon = target with the coverage audit.
//
// Test/report mode: these read every block of every list; they are not on the hot path.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "common.cuh"
#include "device.h"
#include "kernels.cuh"
#include "psattn_b200.h"

namespace psa {
namespace {

constexpr int kExactThreads = 256;

// One CTA per query (u, h): two passes over the list's tokens like the reference
// (max of the fp64 scores, then sum of exp and the exp-weighted values). Warps take
// tokens round-robin; lanes own dims. fp64 products of fp32/bf16 operands are exact,
// only the summation order differs from the reference's sequential loops.
template <typename KV>
__global__ void __launch_bounds__(kExactThreads) exact_attention_kernel(PoolView p, BatchView b, double* out) {
    __shared__ double red[kExactThreads / 32];
    __shared__ double acc_s[kExactThreads / 32][256];
    __shared__ double mx_s, sum_s;
    const int qi = blockIdx.x;
    const int u = qi / b.g;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int W = kExactThreads / 32;
    const int d = b.d;
    const int64_t off = b.list_off[u], n = b.list_off[u + 1] - off;
    const float* q = b.q + (size_t)qi * d;
    const int64_t voff = (int64_t)p.T * d;
    double qd[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) qd[j] = (lane + 32 * j < d) ? (double)q[lane + 32 * j] : 0.0;
    auto score = [&](const KV* krow) {
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (lane + 32 * j < d) a = fma(qd[j], (double)KVT<KV>::to_f(krow[lane + 32 * j]), a);
        return warp_sum_d(a) * b.scale;
    };
    double mx = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        const int32_t slot = b.slots[off + i];
        const int nt = p.ntok[slot];
        for (int t = warp; t < nt; t += W) mx = fmax(mx, score(kv_block<KV>(p, slot) + (int64_t)t * d));
    }
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = -INFINITY;
        for (int w = 0; w < W; ++w) m = fmax(m, red[w]);
        mx_s = m;
    }
    __syncthreads();
    mx = mx_s;
    double es = 0.0, o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const int32_t slot = b.slots[off + i];
        const int nt = p.ntok[slot];
        for (int t = warp; t < nt; t += W) {
            const double w = exp(score(kv_block<KV>(p, slot) + (int64_t)t * d) - mx);
            es += w;
            const KV* vrow = kv_block<KV>(p, slot) + voff + (int64_t)t * d;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (lane + 32 * j < d) o[j] = fma(w, (double)KVT<KV>::to_f(vrow[lane + 32 * j]), o[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (lane + 32 * j < d) acc_s[warp][lane + 32 * j] = o[j];
    if (lane == 0) red[warp] = es;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < W; ++w) s += red[w];
        sum_s = s;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < d; i += kExactThreads) {
        double s = 0.0;
        for (int w = 0; w < W; ++w) s += acc_s[w][i];
        out[(size_t)qi * d + i] = s / sum_s;
    }
}

// Coverage curve of one query in rank (= mass-descending) order: prefix log-sum-exp
// with the reference's log_add (scenario.cpp:428-433), sequential like the reference.
__global__ void coverage_curve_kernel(BatchView b, const int32_t* rpos, const double* omass, double* curve) {
    const int qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= b.n_units * b.g) return;
    const int u = qi / b.g, h = qi % b.g;
    const int64_t off = b.list_off[u], n = b.list_off[u + 1] - off;
    const int64_t hb = off * b.g + (int64_t)h * n;
    double acc = -INFINITY;
    for (int64_t r = 0; r < n; ++r) {
        const double x = omass[hb + rpos[hb + r]];
        if (acc == -INFINITY) acc = x;
        else if (x != -INFINITY) {
            const double hi = fmax(acc, x);
            acc = hi + log1p(exp(fmin(acc, x) - hi));
        }
        curve[hb + r] = acc;
    }
}

struct DevMem {
    std::vector<void*> ptrs;
    void* alloc(size_t n) {
        void* p = nullptr;
        if (cudaMalloc(&p, n < 256 ? 256 : n) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return p;
    }
    ~DevMem() {
        for (void* p : ptrs) cudaFree(p);
    }
};

// Outputs of one psattn_run_batch call into scratch memory.
bool alloc_outputs(DevMem& m, psattn_batch& b, bool ranked) {
    const size_t nq = (size_t)b.n_units * b.group;
    b.out = static_cast<float*>(m.alloc(nq * b.dim * 4));
    b.blocks_processed = static_cast<int64_t*>(m.alloc(nq * 8));
    b.est_coverage = static_cast<double*>(m.alloc(nq * 8));
    b.true_coverage = static_cast<double*>(m.alloc(nq * 8));
    b.terminated = static_cast<int32_t*>(m.alloc(nq * 4));
    b.ranked_pos = ranked ? static_cast<int32_t*>(m.alloc((size_t)b.total_blocks * b.group * 4)) : nullptr;
    b.iter_est = nullptr;
    return b.out && b.blocks_processed && b.est_coverage && b.true_coverage && b.terminated && (!ranked || b.ranked_pos);
}

// percentile (reference serving.cpp:12-20): nearest rank, ceil(p/100 * n).
double percentile(std::vector<double> v, double p) {
    std::sort(v.begin(), v.end());
    if (p == 0.0) return v.front();
    const auto rank = static_cast<size_t>(std::ceil(p / 100.0 * static_cast<double>(v.size())));
    return v[rank - 1];
}

}  // namespace
}  // namespace psa

using namespace psa;

extern "C" {

int psattn_exact_attention(psattn_pool* pool, const psattn_batch* b, double* out, void* stream) {
    int rc = validate_batch(pool, b);
    if (rc) return rc;
    if (!out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_exact_attention: null output");
    if (b->dim > 256) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_exact_attention: dim > 256");
    psattn_batch bb = *b;
    BatchView v{};
    v.n_units = bb.n_units;
    v.g = bb.group;
    v.d = bb.dim;
    v.q = bb.q;
    v.slots = bb.slots;
    v.list_off = bb.list_off;
    v.scale = bb.scale_override > 0.0 ? bb.scale_override : 1.0 / std::sqrt((double)bb.dim);
    const PoolView& p = pool_view(pool);
    const unsigned grid = (unsigned)(bb.n_units * bb.group);
    if (p.dtype == PSATTN_KV_F32)
        exact_attention_kernel<float><<<grid, kExactThreads, 0, (cudaStream_t)stream>>>(p, v, out);
    else
        exact_attention_kernel<__nv_bfloat16><<<grid, kExactThreads, 0, (cudaStream_t)stream>>>(p, v, out);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PSATTN_OK : cuda_fail(e, "psattn_exact_attention");
}

int psattn_tradeoff(psattn_pool* pool, const psattn_batch* b, double target, psattn_tradeoff_report* out,
                    void* stream) {
    if (!out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_tradeoff: null report");
    if (!(target > 0.0) || target > 1.0) return fail(PSATTN_ERR_INVALID_ARGUMENT, "tradeoff: target must be in (0, 1]");
    int rc = validate_batch(pool, b);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nq = (int64_t)b->n_units * b->group;
    const int64_t hbt = b->total_blocks * b->group;
    DevMem mem;

    // ---- 1. fp64 masses and the full mass-descending order of every query ----
    psattn_batch o = *b;
    o.ranking_mode = PSATTN_RANK_ORACLE;
    o.epsilon = 1.0;  // every rank is consumed, so the ranked positions cover the whole list
    o.topk = 0;
    o.audit_coverage = 0;
    if (!alloc_outputs(mem, o, true)) return fail(PSATTN_ERR_RUNTIME, "psattn_tradeoff: device allocation failed");
    const size_t wsb = psattn_batch_workspace_bytes(&o);
    char* ws = static_cast<char*>(mem.alloc(wsb));
    double* curve = static_cast<double*>(mem.alloc((size_t)hbt * 8));
    if (!ws || !curve) return fail(PSATTN_ERR_RUNTIME, "psattn_tradeoff: device allocation failed");
    if ((rc = psattn_run_batch(pool, &o, ws, stream))) return rc;
    BatchView v{};
    v.n_units = o.n_units;
    v.g = o.group;
    v.list_off = o.list_off;
    coverage_curve_kernel<<<(unsigned)((nq + 127) / 128), 128, 0, st>>>(
        v, o.ranked_pos, reinterpret_cast<const double*>(ws + ws_omass_offset(&o)), curve);
    std::vector<double> hcurve((size_t)hbt);
    std::vector<int64_t> hoff((size_t)b->n_units + 1);
    cudaMemcpyAsync(hcurve.data(), curve, (size_t)hbt * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hoff.data(), b->list_off, hoff.size() * 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "psattn_tradeoff: oracle pass");

    // ---- 2. smallest uniform top-k meeting the target for every query (host bisection,
    //         reference scenario.cpp:482-499) ----
    struct Curve {
        const double* prefix;
        int64_t n;
        double at(int64_t k) const {
            if (k == 0) return 0.0;
            if (k >= n) return 1.0;
            return std::exp(prefix[k - 1] - prefix[n - 1]);
        }
    };
    std::vector<Curve> curves;
    int64_t max_blocks = 0;
    for (int u = 0; u < b->n_units; ++u) {
        const int64_t n = hoff[u + 1] - hoff[u];
        for (int h = 0; h < b->group; ++h) curves.push_back(Curve{hcurve.data() + hoff[u] * b->group + h * n, n});
        max_blocks = std::max(max_blocks, n);
    }
    auto worst = [&](int64_t k) {
        double w = std::numeric_limits<double>::infinity();
        for (const auto& c : curves) w = std::min(w, c.at(std::min(k, c.n)));
        return w;
    };
    int64_t lo = 1, hi = max_blocks;
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (worst(mid) >= target) hi = mid;
        else lo = mid + 1;
    }
    const int64_t k_min = lo;
    if (worst(k_min) < target) return fail(PSATTN_ERR_RUNTIME, "tradeoff: bisection failed to reach the coverage target");

    // ---- 3. PSA at epsilon = target with the coverage audit (scenario.cpp:501-529) ----
    psattn_batch p2 = *b;
    p2.epsilon = target;
    p2.topk = 0;
    p2.audit_coverage = 1;
    if (!alloc_outputs(mem, p2, false)) return fail(PSATTN_ERR_RUNTIME, "psattn_tradeoff: device allocation failed");
    char* ws2 = static_cast<char*>(mem.alloc(psattn_batch_workspace_bytes(&p2)));
    if (!ws2) return fail(PSATTN_ERR_RUNTIME, "psattn_tradeoff: device allocation failed");
    if ((rc = psattn_run_batch(pool, &p2, ws2, stream))) return rc;
    std::vector<int64_t> bp((size_t)nq);
    std::vector<double> tc((size_t)nq);
    cudaMemcpyAsync(bp.data(), p2.blocks_processed, (size_t)nq * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(tc.data(), p2.true_coverage, (size_t)nq * 8, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "psattn_tradeoff: PSA pass");
    std::vector<double> samples(bp.begin(), bp.end());
    double mean_blocks = 0.0, cov = 0.0;
    for (double x : samples) mean_blocks += x;
    mean_blocks /= static_cast<double>(samples.size());
    for (double x : tc) cov += x;

    out->target_coverage = target;
    out->n_queries = nq;
    out->max_blocks = max_blocks;
    out->k_min = k_min;
    out->worst_coverage_at_kmin = worst(k_min);
    out->worst_coverage_below_kmin = k_min > 1 ? worst(k_min - 1) : 0.0;
    out->psa_mean_blocks = mean_blocks;
    out->psa_p99_blocks = percentile(samples, 99.0);
    out->psa_mean_coverage = cov / static_cast<double>(nq);
    out->block_access_ratio = static_cast<double>(k_min) / mean_blocks;
    return PSATTN_OK;
}

}  // extern "C"
