// kernels_psa.cu — K4/K5 progressive attention kernel (sm_100a).
#include <cuda_bf16.h>
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace psa {

// =============================================================================
// K4/K5: progressive attention. One CTA (4 warps) per (unit, q-head) query.
// The ranked list is consumed in chunks of 32 ranks:
//   1. K pass  — each warp scores 8 blocks of the chunk: fp32 q.k*scale per token
//                (attention.hpp:41-46), block max, exp-sum, log_as (:50-75);
//                per-token weights are staged in shared memory;
//   2. decide  — warp 0 scans the chunk in rank order in fp64: running
//                log-sum-exp and min of the block masses (CoverageEstimator,
//                engine.cpp:38-55), evaluates the estimate at every microbatch
//                boundary and finds the first boundary with est > eps
//                (engine.cpp:125) or the top-k budget (engine.cpp:221-227);
//   3. V pass  — only ranks before the stop point read V and are merged
//                (online softmax, attention.hpp:83-102).
// No host round trip: the stop decision lives in shared memory. K bytes of at
// most one partial chunk past the stop point are the speculative waste.
// =============================================================================
constexpr int kPsaWarps = 4;
constexpr int kChunk = 32;
constexpr int kBpw = kChunk / kPsaWarps;

template <typename KV, int DPL, int TOK>
__global__ void __launch_bounds__(kPsaWarps * 32) psa_kernel(PoolView p, BatchView b) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int qi = blockIdx.x;
    const int u = qi / b.g, h = qi % b.g;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int64_t hb = off * b.g + (int64_t)h * n;
    const int32_t* __restrict__ rslot = b.rslot + hb;
    const int64_t limit = b.topk > 0 ? (b.topk < n ? b.topk : n) : n;
    const double eps = b.topk > 0 ? 1.0 : b.eps;
    const int d = b.d;
    const int base = lane * DPL;
    const int lim = d - base;
    const bool full = (d == 32 * DPL);
    const float fscale = (float)b.scale;  // engine.cpp:113
    constexpr int TSH = 5 - Log2<TOK>::v;  // lanes per token after reduce-scatter = 1 << TSH
    const int my_tok = lane >> TSH;

    __shared__ __align__(16) float s_w[kPsaWarps][kBpw][TOK];  // per-token weights exp(s - m_b)
    __shared__ float s_mb[kPsaWarps][kBpw], s_lb[kPsaWarps][kBpw];
    __shared__ float s_la[kChunk];
    __shared__ int s_commit, s_final;
    __shared__ double s_est, s_acc;
    __shared__ float s_m[kPsaWarps], s_l[kPsaWarps];
    __shared__ float s_o[kPsaWarps][256];

    float q[DPL];
    load_row<DPL>(b.q + ((size_t)u * b.g + h) * d + base, full, lim, q);

    // warp-local online-softmax state
    float M = -INFINITY, L = 0.0f, O[DPL];
#pragma unroll
    for (int j = 0; j < DPL; ++j) O[j] = 0.0f;
    // coverage state (warp 0, lane-uniform)
    double acc = -INFINITY, mn = INFINITY;

    const double* omass = b.has_oracle ? (b.omass + hb) : nullptr;
    const int32_t* rpos = b.rpos + hb;
    const KV* kv = reinterpret_cast<const KV*>(p.kv);
    const int64_t slot_elems = p.slot_bytes / (int64_t)sizeof(KV);
    const int64_t v_off = (int64_t)p.T * d;

    for (int64_t cb = 0;; cb += kChunk) {
        const int cnt = (int)((limit - cb) < kChunk ? (limit - cb) : kChunk);
        // ---- 1. K pass ----
#pragma unroll 1
        for (int j = 0; j < kBpw; ++j) {
            const int rl = warp * kBpw + j;
            if (rl >= cnt) break;
            const int32_t slot = rslot[cb + rl];
            const int nt = p.ntok[slot];
            const KV* kp = kv + (int64_t)slot * slot_elems + base;
            float part[TOK];
#pragma unroll
            for (int t = 0; t < TOK; ++t) {
                float kr[DPL];
                if (t < nt) {
                    load_row<DPL>(kp + (size_t)t * d, full, lim, kr);
                } else {
#pragma unroll
                    for (int jj = 0; jj < DPL; ++jj) kr[jj] = 0.0f;
                }
                float a = 0.0f;
#pragma unroll
                for (int jj = 0; jj < DPL; ++jj) a = fmaf(q[jj], kr[jj], a);
                part[t] = a;
            }
            float s = reduce_scatter<TOK>(part, lane) * fscale;
            s = my_tok < nt ? s : -INFINITY;
            const float mb = warp_max(s);
            const float w = my_tok < nt ? expf(s - mb) : 0.0f;
            float lb = w;
#pragma unroll
            for (int o = 16; o >= (1 << TSH); o >>= 1) lb += __shfl_xor_sync(PSA_FULL, lb, o);
            if ((lane & ((1 << TSH) - 1)) == 0) s_w[warp][j][my_tok] = w;
            if (lane == 0) {
                s_mb[warp][j] = mb;
                s_lb[warp][j] = lb;
                s_la[rl] = mb + logf(lb);
            }
        }
        __syncthreads();
        // ---- 2. decide (warp 0) ----
        if (warp == 0) {
            const bool valid = lane < cnt;
            const int64_t r = cb + lane;
            double x = -INFINITY;
            if (valid) x = omass ? omass[rpos[r]] : (double)s_la[lane];
            double mx = warp_max_d(x);
            mx = fmax(mx, acc);
            double e = valid ? exp(x - mx) : 0.0;
            double mnv = valid ? x : INFINITY;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double ye = __shfl_up_sync(PSA_FULL, e, o);
                const double ym = __shfl_up_sync(PSA_FULL, mnv, o);
                if (lane >= o) {
                    e += ye;
                    mnv = fmin(mnv, ym);
                }
            }
            if (acc != -INFINITY) e += exp(acc - mx);
            const double acc_i = mx + log(e);
            const double mn_i = fmin(mnv, mn);
            const int64_t nl = n - (r + 1);
            const double est_i = nl == 0 ? 1.0 : 1.0 / (1.0 + (double)nl * exp(mn_i - acc_i));
            const bool boundary = valid && ((((r + 1) % b.m) == 0) || (r + 1 == limit));
            const bool stop = boundary && (est_i > eps || r + 1 == limit);
            const unsigned bal = __ballot_sync(PSA_FULL, stop);
            const int f = bal ? (__ffs(bal) - 1) : (cnt - 1);
            if (b.iest && boundary && lane <= f) b.iest[hb + r] = est_i;  // IterationStats::estimated_coverage
            acc = __shfl_sync(PSA_FULL, acc_i, f);
            mn = __shfl_sync(PSA_FULL, mn_i, f);
            const double e_f = __shfl_sync(PSA_FULL, est_i, f);
            if (lane == 0) {
                s_commit = f + 1;
                s_final = bal ? 1 : 0;
                s_est = e_f;
                s_acc = acc;
            }
        }
        __syncthreads();
        const int commit = s_commit;
        const int fin = s_final;
        // ---- 3. V pass over committed ranks ----
#pragma unroll 1
        for (int j = 0; j < kBpw; ++j) {
            const int rl = warp * kBpw + j;
            if (rl >= commit) break;
            const int32_t slot = rslot[cb + rl];
            const int nt = p.ntok[slot];
            const KV* vp = kv + (int64_t)slot * slot_elems + v_off + base;
            float ob[DPL];
#pragma unroll
            for (int jj = 0; jj < DPL; ++jj) ob[jj] = 0.0f;
#pragma unroll
            for (int t = 0; t < TOK; ++t) {
                if (t < nt) {
                    const float wt = s_w[warp][j][t];
                    float vr[DPL];
                    load_row<DPL>(vp + (size_t)t * d, full, lim, vr);
#pragma unroll
                    for (int jj = 0; jj < DPL; ++jj) ob[jj] = fmaf(wt, vr[jj], ob[jj]);
                }
            }
            const float mbj = s_mb[warp][j];
            const float mnew = fmaxf(M, mbj);
            const float a = expf(M - mnew);
            const float c = expf(mbj - mnew);
#pragma unroll
            for (int jj = 0; jj < DPL; ++jj) O[jj] = O[jj] * a + ob[jj] * c;
            L = L * a + s_lb[warp][j] * c;
            M = mnew;
        }
        if (fin) {
            if (threadIdx.x == 0) {
                const int64_t bp = cb + commit;
                b.bp[qi] = bp;
                b.est[qi] = s_est;
                b.term[qi] = b.topk > 0 ? (limit < n) : (bp < n);
            }
            break;
        }
        __syncthreads();  // s_w / s_la are rewritten by the next chunk's K pass
    }
    // ---- finalize: merge the warps' states (finalize, attention.hpp:104-110) ----
    if (lane == 0) {
        s_m[warp] = M;
        s_l[warp] = L;
    }
#pragma unroll
    for (int jj = 0; jj < DPL; ++jj)
        if (base + jj < d) s_o[warp][base + jj] = O[jj];
    __syncthreads();
    float Mt = -INFINITY;
#pragma unroll
    for (int w = 0; w < kPsaWarps; ++w) Mt = fmaxf(Mt, s_m[w]);
    float Lt = 0.0f, sc[kPsaWarps];
#pragma unroll
    for (int w = 0; w < kPsaWarps; ++w) {
        sc[w] = s_l[w] > 0.0f ? expf(s_m[w] - Mt) : 0.0f;
        Lt += s_l[w] * sc[w];
    }
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        float o = 0.0f;
#pragma unroll
        for (int w = 0; w < kPsaWarps; ++w) o += sc[w] > 0.0f ? s_o[w][i] * sc[w] : 0.0f;
        b.out[(size_t)qi * d + i] = o / Lt;
    }
    if (b.tcov && threadIdx.x == 0) {
        double tc = -1.0;
        if (b.audit) {
            // total mass over all n blocks (engine.cpp:88 total_log_as)
            double mx = -INFINITY;
            for (int64_t i = 0; i < n; ++i) mx = fmax(mx, omass[i]);
            double s = 0.0;
            for (int64_t i = 0; i < n; ++i) s += exp(omass[i] - mx);
            tc = exp(s_acc - (mx + log(s)));
        }
        b.tcov[qi] = tc;
    }
}

template <typename KV, int TOK>
static void launch_psa_t(const PoolView& p, const BatchView& b, int nq, cudaStream_t st) {
    switch (dpl_for(b.d)) {
        case 2: psa_kernel<KV, 2, TOK><<<nq, kPsaWarps * 32, 0, st>>>(p, b); break;
        case 4: psa_kernel<KV, 4, TOK><<<nq, kPsaWarps * 32, 0, st>>>(p, b); break;
        default: psa_kernel<KV, 8, TOK><<<nq, kPsaWarps * 32, 0, st>>>(p, b); break;
    }
}

void launch_psa(const PoolView& p, const BatchView& b, cudaStream_t st) {
    const int nq = b.n_units * b.g;
    if (p.dtype == 0) {
        if (tok_for(p.T) == 16) launch_psa_t<float, 16>(p, b, nq, st);
        else launch_psa_t<float, 32>(p, b, nq, st);
    } else {
        if (tok_for(p.T) == 16) launch_psa_t<__nv_bfloat16, 16>(p, b, nq, st);
        else launch_psa_t<__nv_bfloat16, 32>(p, b, nq, st);
    }
}

}  // namespace psa
