// metadata_api.cu — the reference's per-call scoring and ranking entry points on the device:
//   psattn_criticality_scores  criticality_score over a list of host metadata records
//                              (reference src/metadata.cpp:41-72), bit-identical;
//   psattn_rank_by_scores      rank_by_scores (metadata.cpp:87-96): descending score, ties by
//                              ascending block id.
// rank_blocks (metadata.cpp:74-85) is the composition of the two (include/psattn/metadata.hpp).
//
// These serve callers that hold BlockMetadata in host memory (the reference's C++ API); the
// progressive path itself scores and orders pool-resident metadata inside its own kernels
// (score_kernel_tma, first_tranche_kernel, dense_decide_kernel).
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "common.cuh"
#include "device.h"
#include "kernels.cuh"
#include "psattn_b200.h"

namespace psa {
namespace {

// One thread per record, dims in index order like the reference's loops. Products and sums
// are explicitly rounded (__dmul_rn / __dadd_rn: no FMA contraction), std::max(a, b) is
// (a < b ? b : a): every score is the reference's double bit for bit.
__global__ void criticality_kernel(const float* __restrict__ q, int d, const float* __restrict__ mean,
                                   const float* __restrict__ lo, const float* __restrict__ hi, int64_t n, int est,
                                   double scale, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* m = mean + i * d;
    const float* l = lo + i * d;
    const float* h = hi + i * d;
    double am = 0.0, au = 0.0;
    for (int k = 0; k < d; ++k) {
        const double qd = (double)q[k];
        if (est != 1) am = __dadd_rn(am, __dmul_rn(qd, (double)m[k]));
        if (est != 0) {
            const double a = __dmul_rn(qd, (double)l[k]), b = __dmul_rn(qd, (double)h[k]);
            au = __dadd_rn(au, a < b ? b : a);
        }
    }
    const double ms = __dmul_rn(am, scale), us = __dmul_rn(au, scale);
    out[i] = est == 0 ? ms : (est == 1 ? us : __dmul_rn(0.5, __dadd_rn(ms, us)));
}

// rank_by_scores keys: pass 1 sorts by block id (signed -> order-preserving unsigned), pass 2
// stably by descending score, so equal scores keep ascending block id (metadata.cpp:92-93).
__global__ void id_keys_kernel(const int64_t* __restrict__ ids, int64_t n, uint64_t* __restrict__ keys) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = (uint64_t)ids[i] ^ 0x8000000000000000ull;
}
__global__ void score_keys_kernel(const double* __restrict__ s, const int32_t* __restrict__ perm, int64_t n,
                                  uint64_t* __restrict__ keys) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = make_key_masked(s[perm[i]], 0u, 0ull);
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t n) { return cudaMalloc(&p, (n ? n : 1) * sizeof(T)); }
};

int need_device(const char* what) {
    int dev_count = 0;
    const cudaError_t e = cudaGetDeviceCount(&dev_count);
    if (e != cudaSuccess || dev_count == 0)
        return fail(PSATTN_ERR_RUNTIME, std::string(what) + ": no CUDA device (no CPU fallback)");
    return 0;
}

}  // namespace
}  // namespace psa

using namespace psa;

extern "C" int psattn_criticality_scores(const float* q, int32_t d, const float* mean, const float* lo,
                                         const float* hi, int64_t n, int32_t estimator, double scale,
                                         double* scores) {
    if (!q || !mean || !lo || !hi || !scores || d <= 0 || n < 0)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_criticality_scores: bad arguments");
    if (estimator < 0 || estimator > 2)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "criticality_score: unknown estimator");
    if (int rc = need_device("psattn_criticality_scores")) return rc;
    if (n == 0) return PSATTN_OK;
    const size_t nd = (size_t)n * (size_t)d;
    DevBuf<float> dq, dm, dl, dh;
    DevBuf<double> ds;
    cudaError_t e;
    if ((e = dq.alloc(d)) || (e = dm.alloc(nd)) || (e = dl.alloc(nd)) || (e = dh.alloc(nd)) || (e = ds.alloc(n)))
        return cuda_fail(e, "psattn_criticality_scores: alloc");
    if ((e = cudaMemcpy(dq.p, q, (size_t)d * 4, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dm.p, mean, nd * 4, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dl.p, lo, nd * 4, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(dh.p, hi, nd * 4, cudaMemcpyHostToDevice)))
        return cuda_fail(e, "psattn_criticality_scores: upload");
    criticality_kernel<<<(unsigned)((n + 127) / 128), 128>>>(dq.p, d, dm.p, dl.p, dh.p, n, estimator, scale, ds.p);
    if ((e = cudaGetLastError())) return cuda_fail(e, "psattn_criticality_scores: launch");
    if ((e = cudaMemcpy(scores, ds.p, (size_t)n * 8, cudaMemcpyDeviceToHost)))
        return cuda_fail(e, "psattn_criticality_scores: download");
    return PSATTN_OK;
}

extern "C" int psattn_rank_by_scores(const double* scores, const int64_t* block_ids, int64_t n, int64_t* order) {
    if (!scores || !block_ids || !order || n < 0)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_rank_by_scores: bad arguments");
    if (int rc = need_device("psattn_rank_by_scores")) return rc;
    if (n == 0) return PSATTN_OK;
    DevBuf<double> ds;
    DevBuf<int64_t> di;
    cudaError_t e;
    if ((e = ds.alloc(n)) || (e = di.alloc(n))) return cuda_fail(e, "psattn_rank_by_scores: alloc");
    if ((e = cudaMemcpy(ds.p, scores, (size_t)n * 8, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(di.p, block_ids, (size_t)n * 8, cudaMemcpyHostToDevice)))
        return cuda_fail(e, "psattn_rank_by_scores: upload");
    if (n > 0x7fffffffLL) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_rank_by_scores: too many blocks");
    DevBuf<uint64_t> keys, tk;
    DevBuf<int32_t> perm, ord32, tv, tv2;
    DevBuf<int64_t> off;
    if ((e = keys.alloc(n)) || (e = tk.alloc(n)) || (e = perm.alloc(n)) || (e = ord32.alloc(n)) || (e = tv.alloc(n)) || (e = tv2.alloc(n)) ||
        (e = off.alloc(2)))
        return cuda_fail(e, "psattn_rank_by_scores: alloc");
    const int64_t hoff[2] = {0, n};
    if ((e = cudaMemcpy(off.p, hoff, sizeof(hoff), cudaMemcpyHostToDevice)))
        return cuda_fail(e, "psattn_rank_by_scores: upload");
    const unsigned blocks = (unsigned)((n + 255) / 256);
    id_keys_kernel<<<blocks, 256>>>(di.p, n, keys.p);
    if ((e = launch_seg_sort(keys.p, nullptr, perm.p, tk.p, tv.p, tv2.p, off.p, 1, 1, 0)))
        return cuda_fail(e, "psattn_rank_by_scores: sort by id");
    score_keys_kernel<<<blocks, 256>>>(ds.p, perm.p, n, keys.p);
    if ((e = launch_seg_sort(keys.p, perm.p, ord32.p, tk.p, tv.p, tv2.p, off.p, 1, 1, 0)))
        return cuda_fail(e, "psattn_rank_by_scores: sort by score");
    std::vector<int32_t> ord((size_t)n);
    if ((e = cudaMemcpy(ord.data(), ord32.p, (size_t)n * 4, cudaMemcpyDeviceToHost)))
        return cuda_fail(e, "psattn_rank_by_scores: download");
    for (int64_t i = 0; i < n; ++i) order[i] = ord[(size_t)i];
    return PSATTN_OK;
}
