// progressive_api.cu — device side of psattn::ProgressiveRun (include/psattn/engine.hpp), the
// reference's compute-side state of one caller-driven progressive run (reference
// src/engine.cpp:92-147): each consume() folds a microbatch of host blocks, in rank order, into
// a device-resident softmax accumulator (block_partial_attention + merge_partial,
// attention.hpp:41-101) and returns the blocks' log masses for the host-side coverage
// estimator; result() finalizes on the device (finalize, attention.hpp:104-110).
//
// This serves callers that run their own executor over ProgressiveRun (the reference's
// run_sequential / run_pipelined do); psa_attention and the batched paths run the whole loop
// inside the progressive kernels instead.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "device.h"
#include "kernels.cuh"

namespace psa {

struct RunState {
    int d = 0;
    float* q = nullptr;      // [d]
    float* acc = nullptr;    // [d] out_unnorm, then max_score, exp_sum, log_as_acc
    float* kv = nullptr;     // staging: [cap][2][T][d]
    int32_t* ntok = nullptr;  // [cap]
    float* las = nullptr;    // [cap] per-block log_as
    float* host = nullptr;   // pinned staging of the same layout
    int64_t cap_floats = 0;
    int cap_blocks = 0;
};

namespace {

constexpr int kThreads = 256;  // >= d (<= 256) and >= tokens per block (<= kMaxBlockTokens)

// One CTA; blocks strictly in order like the reference. Token scores: one thread per token,
// dims in order with explicit rounding (the reference's dot_scaled<float>); max / exp-sum by
// one thread in token order; thread i owns dim i of the weighted value sum (token order).
__global__ void __launch_bounds__(kThreads) consume_kernel(const float* __restrict__ q, int d, float scale,
                                                           const float* __restrict__ kv, const int32_t* __restrict__ ntok,
                                                           int n, int T, float* __restrict__ acc,
                                                           float* __restrict__ las) {
    __shared__ float sc[kMaxBlockTokens], w[kMaxBlockTokens];
    __shared__ float fa, fp;
    const int i = threadIdx.x;
    float* mx = acc + d;
    float* sm = acc + d + 1;
    float* la = acc + d + 2;
    for (int b = 0; b < n; ++b) {
        const int nt = ntok[b];
        const float* K = kv + (size_t)b * 2 * T * d;
        const float* V = K + (size_t)T * d;
        if (i < nt) {
            float s = 0.0f;
            for (int k = 0; k < d; ++k) s = __fadd_rn(s, __fmul_rn(q[k], K[(size_t)i * d + k]));
            sc[i] = __fmul_rn(s, scale);
        }
        __syncthreads();
        if (i == 0) {
            float m = -INFINITY;
            for (int t = 0; t < nt; ++t) m = sc[t] > m ? sc[t] : m;
            float e = 0.0f;
            for (int t = 0; t < nt; ++t) {
                w[t] = expf(sc[t] - m);
                e = __fadd_rn(e, w[t]);
            }
            las[b] = m + logf(e);
            // merge_partial: an empty accumulator absorbs the partial unchanged
            if (*sm == 0.0f) {
                fa = 0.0f;
                fp = 1.0f;
                *mx = m;
                *sm = e;
            } else {
                const float mm = *mx > m ? *mx : m;
                fa = expf(*mx - mm);
                fp = expf(m - mm);
                *sm = __fadd_rn(__fmul_rn(*sm, fa), __fmul_rn(e, fp));
                *mx = mm;
            }
            *la = *mx + logf(*sm);
        }
        __syncthreads();
        if (i < d) {
            float o = 0.0f;
            for (int t = 0; t < nt; ++t) o = __fadd_rn(o, __fmul_rn(w[t], V[(size_t)t * d + i]));
            acc[i] = fa == 0.0f && fp == 1.0f ? o : __fadd_rn(__fmul_rn(acc[i], fa), __fmul_rn(o, fp));
        }
        __syncthreads();
    }
}

__global__ void finalize_kernel(const float* __restrict__ acc, int d, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < d) out[i] = acc[i] / acc[d + 1];
}

}  // namespace

int prun_create(const float* q, int d, RunState** out) {
    if (!q || !out || d <= 0 || d > 256) return fail(PSATTN_ERR_INVALID_ARGUMENT, "progressive run: dim must be in [1, 256]");
    int dev_count = 0;
    cudaError_t e = cudaGetDeviceCount(&dev_count);
    if (e != cudaSuccess || dev_count == 0)
        return fail(PSATTN_ERR_RUNTIME, "progressive run: no CUDA device (no CPU fallback)");
    auto* s = new RunState();
    s->d = d;
    if ((e = cudaMalloc(&s->q, (size_t)d * 4)) || (e = cudaMalloc(&s->acc, (size_t)(d + 3) * 4)) ||
        (e = cudaMemcpy(s->q, q, (size_t)d * 4, cudaMemcpyHostToDevice)) ||
        (e = cudaMemset(s->acc, 0, (size_t)(d + 3) * 4))) {
        prun_destroy(s);
        return cuda_fail(e, "progressive run: alloc");
    }
    *out = s;
    return PSATTN_OK;
}

void prun_destroy(RunState* s) {
    if (!s) return;
    cudaFree(s->q);
    cudaFree(s->acc);
    cudaFree(s->kv);
    cudaFree(s->ntok);
    cudaFree(s->las);
    cudaFreeHost(s->host);
    delete s;
}

int prun_consume(RunState* s, float scale, int n, const int32_t* ntok, const float* const* keys,
                 const float* const* values, float* log_as) {
    int T = 1;
    for (int b = 0; b < n; ++b) {
        if (ntok[b] <= 0 || ntok[b] > kMaxBlockTokens)
            return fail(PSATTN_ERR_INVALID_ARGUMENT, "progressive run: blocks must hold 1..128 tokens");
        T = ntok[b] > T ? ntok[b] : T;
    }
    const int64_t need = (int64_t)n * 2 * T * s->d;
    cudaError_t e;
    if (need > s->cap_floats || n > s->cap_blocks) {
        cudaFree(s->kv);
        cudaFree(s->ntok);
        cudaFree(s->las);
        cudaFreeHost(s->host);
        s->kv = s->host = s->las = nullptr;
        s->ntok = nullptr;
        s->cap_floats = need;
        s->cap_blocks = n;
        if ((e = cudaMalloc(&s->kv, (size_t)need * 4)) || (e = cudaMalloc(&s->ntok, (size_t)n * 4)) ||
            (e = cudaMalloc(&s->las, (size_t)n * 4)) || (e = cudaMallocHost(&s->host, (size_t)need * 4))) {
            s->cap_floats = 0;
            s->cap_blocks = 0;
            return cuda_fail(e, "progressive run: staging alloc");
        }
    }
    const size_t blk = (size_t)T * s->d;
    for (int b = 0; b < n; ++b) {
        const size_t nb = (size_t)ntok[b] * s->d;
        float* K = s->host + (size_t)b * 2 * blk;
        std::copy(keys[b], keys[b] + nb, K);
        std::copy(values[b], values[b] + nb, K + blk);
    }
    if ((e = cudaMemcpy(s->kv, s->host, (size_t)n * 2 * blk * 4, cudaMemcpyHostToDevice)) ||
        (e = cudaMemcpy(s->ntok, ntok, (size_t)n * 4, cudaMemcpyHostToDevice)))
        return cuda_fail(e, "progressive run: upload");
    consume_kernel<<<1, kThreads>>>(s->q, s->d, scale, s->kv, s->ntok, n, T, s->acc, s->las);
    if ((e = cudaGetLastError()) || (e = cudaMemcpy(log_as, s->las, (size_t)n * 4, cudaMemcpyDeviceToHost)))
        return cuda_fail(e, "progressive run: consume");
    return PSATTN_OK;
}

int prun_result(const RunState* s, float* out) {
    float* dout = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&dout, (size_t)s->d * 4))) return cuda_fail(e, "progressive run: alloc");
    finalize_kernel<<<1, 256>>>(s->acc, s->d, dout);
    e = cudaGetLastError();
    if (!e) e = cudaMemcpy(out, dout, (size_t)s->d * 4, cudaMemcpyDeviceToHost);
    cudaFree(dout);
    return e ? cuda_fail(e, "progressive run: finalize") : PSATTN_OK;
}

}  // namespace psa
