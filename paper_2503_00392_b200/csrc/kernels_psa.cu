// kernels_psa.cu — K3 ordering (lazy tranche selection) fused with K4/K5, the
// persistent progressive attention kernel (sm_100a).
#include <cuda_bf16.h>
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace psa {

// =============================================================================
// One CTA (8 warps) per (unit, q-head) query. Two interleaved loops:
//
// ORDER (K3, rank_by_scores, reference metadata.cpp:87-96) — lazily, in
// tranches: the next C <= 1024 ranks are the C smallest sort keys above the
// last consumed key (keys from score_kernel encode score desc / block id asc).
// A bucket select over the head's n keys (min/max, 2048-bin histogram,
// refinement) finds the cut, the survivors are gathered and bitonic-sorted in
// shared memory. The first tranche targets 512 ranks — enough for most planted
// queries — so a head that stops early never pays for a full sort of n keys.
//
// PROGRESS (K4/K5, ProgressiveRun::consume + psa_attention / topk_attention,
// reference engine.cpp:104-127, 162-171, 211-231) over chunks of 32 ranks:
//   1. K pass  — each warp scores 4 blocks: fp32 q.k*scale per token
//                (attention.hpp:41-46), block max, exp-sum, log_as (:50-75);
//   2. decide  — warp 0 scans the chunk in rank order in fp64: running
//                log-sum-exp and min of the block masses (CoverageEstimator,
//                engine.cpp:38-55), evaluates the estimate at every microbatch
//                boundary and finds the first boundary with est > eps
//                (engine.cpp:125) or the top-k budget (engine.cpp:221-227);
//   3. V pass  — only ranks before the stop point read V and are merged
//                (online softmax, attention.hpp:83-102).
// The stop decision never leaves shared memory: no host round trip. K bytes of
// at most one partial chunk past the stop point are the speculative waste.
// =============================================================================
constexpr int kPsaWarps = 8;
constexpr int kPsaThreads = kPsaWarps * 32;
constexpr int kChunk = 32;
constexpr int kBpw = kChunk / kPsaWarps;
constexpr int kTCap = 1024;
constexpr int kBins = 2048;
constexpr int kFirstTranche = 512;

template <int TOK>
struct PsaSmem {
    uint64_t tb[kTCap];       // sorted keys of the current tranche
    int32_t tslot[kTCap];     // their pool slots
    uint8_t tntok[kTCap];     // their valid token counts
    uint32_t hist[kBins];     // bucket-select histogram; reused for the final merge
    float w[kPsaWarps][kBpw][TOK];
    float mb[kPsaWarps][kBpw], lb[kPsaWarps][kBpw];
    float la[kChunk];
    unsigned long long red_min, red_max;
    unsigned int red_cnt, gcount, excl;
    int bstar;
    int commit, fin;
    double est, acc;
    float m[kPsaWarps], l[kPsaWarps];
};

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long x) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(PSA_FULL, x, o);
        x = y < x ? y : x;
    }
    return x;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long x) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(PSA_FULL, x, o);
        x = y > x ? y : x;
    }
    return x;
}

// All-ascending bitonic network on a[0, n) in shared memory (indices >= n act as +inf).
__device__ __forceinline__ void bitonic_smem(uint64_t* a, int n) {
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < (n2 >> 1); i += blockDim.x) {
                const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));  // j is a power of two
                const int hi = (j == (k >> 1)) ? (lo ^ (k - 1)) : (lo + j);
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

// Calls f(key) for every key of the head; 8 independent loads in flight per thread.
template <typename F>
__device__ __forceinline__ void scan_keys(const uint64_t* __restrict__ keys, int64_t n, F&& f) {
    constexpr int U = 8;
    for (int64_t i0 = threadIdx.x; i0 < n; i0 += (int64_t)U * kPsaThreads) {
        uint64_t k[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + (int64_t)u * kPsaThreads;
            k[u] = i < n ? __ldg(reinterpret_cast<const unsigned long long*>(keys) + i) : ~0ull;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + (int64_t)u * kPsaThreads < n) f(k[u]);
    }
}

// Next tranche: the C (<= kTCap, ~target) smallest keys greater than `last` (all keys if first).
template <int TOK>
__device__ int select_tranche(PsaSmem<TOK>& s, const uint64_t* __restrict__ keys, int64_t n, uint64_t last,
                              bool first, unsigned target) {
    const int tid = threadIdx.x, lane = tid & 31;
    unsigned long long lmin = ~0ull, lmax = 0;
    unsigned lcnt = 0;
    scan_keys(keys, n, [&](uint64_t k) {
        if (first || k > last) {
            lmin = k < lmin ? k : lmin;
            lmax = k > lmax ? k : lmax;
            ++lcnt;
        }
    });
    if (tid == 0) {
        s.red_min = ~0ull;
        s.red_max = 0;
        s.red_cnt = 0;
        s.gcount = 0;
    }
    __syncthreads();
    lmin = warp_min_u64(lmin);
    lmax = warp_max_u64(lmax);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) lcnt += __shfl_xor_sync(PSA_FULL, lcnt, o);
    if (lane == 0) {
        atomicMin(&s.red_min, lmin);
        atomicMax(&s.red_max, lmax);
        atomicAdd(&s.red_cnt, lcnt);
    }
    __syncthreads();
    const uint64_t kmax = s.red_max;
    uint64_t tau = kmax;
    if (s.red_cnt > (unsigned)kTCap) {
        uint64_t lo = s.red_min, hi = kmax;
        unsigned need = target, before = 0;
        for (int it = 0; it < 10; ++it) {
            const uint64_t span = hi - lo;
            const int bits = 64 - __clzll((long long)span);
            const int sh = bits > 11 ? bits - 11 : 0;
            for (int i = tid; i < kBins; i += kPsaThreads) s.hist[i] = 0;
            __syncthreads();
            scan_keys(keys, n, [&](uint64_t k) {
                if ((first || k > last) && k >= lo && k <= hi) atomicAdd(&s.hist[(k - lo) >> sh], 1u);
            });
            __syncthreads();
            // first bin b with cum(b) >= need: each thread owns 8 consecutive bins
            constexpr int per = kBins / kPsaThreads;
            unsigned loc = 0;
#pragma unroll
            for (int j = 0; j < per; ++j) loc += s.hist[tid * per + j];
            unsigned inc = loc;  // inclusive warp scan
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(PSA_FULL, inc, o);
                if (lane >= o) inc += y;
            }
            __shared__ unsigned wsum[kPsaWarps];
            if (lane == 31) wsum[tid >> 5] = inc;
            __syncthreads();
            unsigned wbase = 0;
            for (int w = 0; w < (tid >> 5); ++w) wbase += wsum[w];
            unsigned cum = wbase + inc - loc;  // exclusive prefix of this thread's bins
            if (cum < need && need <= cum + loc) {
#pragma unroll 1
                for (int j = 0; j < per; ++j) {
                    const unsigned c = s.hist[tid * per + j];
                    if (need <= cum + c) {
                        s.bstar = tid * per + j;
                        s.excl = cum;
                        break;
                    }
                    cum += c;
                }
            }
            __syncthreads();
            const int bs = s.bstar;
            const unsigned ex = s.excl, incl = ex + s.hist[bs];
            const uint64_t width_m1 = (sh >= 64) ? ~0ull : ((1ull << sh) - 1ull);
            const uint64_t bin_lo = lo + ((uint64_t)bs << sh);
            if (before + incl <= (unsigned)kTCap) {
                tau = (hi - bin_lo <= width_m1) ? hi : bin_lo + width_m1;
                break;
            }
            if (before + ex >= 32) {
                tau = bin_lo - 1;  // take the bins below bs
                break;
            }
            before += ex;
            need -= ex;
            lo = bin_lo;
            if (hi - lo > width_m1) hi = lo + width_m1;
            __syncthreads();
        }
    }
    // gather the survivors (warp-aggregated slot reservation)
    scan_keys(keys, n, [&](uint64_t k) {
        const bool take = (first || k > last) && k <= tau;
        const unsigned m = __ballot_sync(__activemask(), take);
        if (take) {
            const int leader = __ffs(m) - 1;
            unsigned basei = 0;
            if (lane == leader) basei = atomicAdd(&s.gcount, (unsigned)__popc(m));
            basei = __shfl_sync(m, basei, leader);
            const unsigned idx = basei + __popc(m & ((1u << lane) - 1u));
            if (idx < (unsigned)kTCap) s.tb[idx] = k;
        }
    });
    __syncthreads();
    const int C = (int)min(s.gcount, (unsigned)kTCap);
    bitonic_smem(s.tb, C);
    return C;
}

template <typename KV, int DPL, int TOK, bool FULL>
__global__ void __launch_bounds__(kPsaThreads, 3) psa_kernel(PoolView p, BatchView b) {
    __shared__ PsaSmem<TOK> s;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int qi = blockIdx.x;
    const int u = qi / b.g, h = qi % b.g;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int64_t hb = off * b.g + (int64_t)h * n;
    const uint64_t* keys = b.keys + hb;
    const int64_t limit = b.topk > 0 ? (b.topk < n ? b.topk : n) : n;
    const double eps = b.topk > 0 ? 1.0 : b.eps;
    const int d = FULL ? 32 * DPL : b.d;  // compile-time on the full-row paths: row offsets fold to immediates
    const int base = lane * DPL;
    const int lim = d - base;
    constexpr bool full = FULL;  // d == 32*DPL: vector loads, no bounds
    const float fscale = (float)b.scale;  // engine.cpp:113
    constexpr int TSH = 5 - Log2<TOK>::v;  // lanes per token after reduce-scatter = 1 << TSH
    const int my_tok = lane >> TSH;
    const uint64_t pmask = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);

    float q[DPL];
    load_row<DPL>(b.q + ((size_t)u * b.g + h) * d + base, full, lim, q);

    float M = -INFINITY, L = 0.0f, O[DPL];  // warp-local online-softmax state
#pragma unroll
    for (int j = 0; j < DPL; ++j) O[j] = 0.0f;
    double acc = -INFINITY, mn = INFINITY;  // coverage state (warp 0, lane-uniform)

    const double* omass = b.has_oracle ? (b.omass + hb) : nullptr;
    const KV* kv = reinterpret_cast<const KV*>(p.kv);
    const int64_t slot_elems = p.slot_bytes / (int64_t)sizeof(KV);
    const int64_t v_off = (int64_t)p.T * d;
    const int T = p.T;

    int64_t tr0 = 0;  // global rank of s.tb[0]
    int tc = 0;       // ranks in the current tranche
    uint64_t last = 0;
    for (int64_t cb = 0;;) {
        if (cb >= tr0 + tc) {  // ---- ORDER: next tranche ----
            tr0 += tc;
            tc = select_tranche(s, keys, n, last, tr0 == 0, tr0 == 0 ? kFirstTranche : kTCap);
            last = s.tb[tc - 1];
            for (int i = threadIdx.x; i < tc; i += kPsaThreads) {
                const int32_t pos = (int32_t)(s.tb[i] & pmask);
                b.rpos[hb + tr0 + i] = pos;
                const int32_t sl = b.slots[off + pos];
                s.tslot[i] = sl;
                s.tntok[i] = (uint8_t)p.ntok[sl];
            }
            __syncthreads();
        }
        const int64_t room = tr0 + tc - cb;
        int cnt = (int)((limit - cb) < kChunk ? (limit - cb) : kChunk);
        if (room < cnt) cnt = (int)room;
        const int ci = (int)(cb - tr0);
        // ---- 1. K pass ----
#pragma unroll 1
        for (int j = 0; j < kBpw; ++j) {
            const int rl = warp * kBpw + j;
            if (rl >= cnt) break;
            const int32_t slot = s.tslot[ci + rl];
            const int nt = s.tntok[ci + rl];
            const KV* kp = kv + (int64_t)slot * slot_elems + base;
            // Branch-free: rows in [ntok, T) are zero-filled in the pool and rows >= T
            // (TOK > T) re-read row T-1, so all TOK loads issue before the first use;
            // tokens >= ntok are masked below.
            float part[TOK];
            if (T == TOK) {
#pragma unroll
                for (int t = 0; t < TOK; ++t) {
                    float kr[DPL];
                    load_row<DPL>(kp + t * d, full, lim, kr);
                    float a = 0.0f;
#pragma unroll
                    for (int jj = 0; jj < DPL; ++jj) a = fmaf(q[jj], kr[jj], a);
                    part[t] = a;
                }
            } else {
#pragma unroll
                for (int t = 0; t < TOK; ++t) {
                    float kr[DPL];
                    load_row<DPL>(kp + (size_t)(t < T ? t : T - 1) * d, full, lim, kr);
                    float a = 0.0f;
#pragma unroll
                    for (int jj = 0; jj < DPL; ++jj) a = fmaf(q[jj], kr[jj], a);
                    part[t] = a;
                }
            }
            float sc = reduce_scatter<TOK>(part, lane) * fscale;
            sc = my_tok < nt ? sc : -INFINITY;
            const float mb = warp_max(sc);
            const float w = my_tok < nt ? expf(sc - mb) : 0.0f;
            float lb = w;
#pragma unroll
            for (int o = 16; o >= (1 << TSH); o >>= 1) lb += __shfl_xor_sync(PSA_FULL, lb, o);
            if ((lane & ((1 << TSH) - 1)) == 0) s.w[warp][j][my_tok] = w;
            if (lane == 0) {
                s.mb[warp][j] = mb;
                s.lb[warp][j] = lb;
                s.la[rl] = mb + logf(lb);
            }
        }
        __syncthreads();
        // ---- 2. decide (warp 0) ----
        if (warp == 0) {
            const bool valid = lane < cnt;
            const int64_t r = cb + lane;
            double x = -INFINITY;
            if (valid) x = omass ? omass[s.tb[ci + lane] & pmask] : (double)s.la[lane];
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
                s.commit = f + 1;
                s.fin = bal ? 1 : 0;
                s.est = e_f;
                s.acc = acc;
            }
        }
        __syncthreads();
        const int commit = s.commit;
        const int fin = s.fin;
        // ---- 3. V pass over committed ranks ----
#pragma unroll 1
        for (int j = 0; j < kBpw; ++j) {
            const int rl = warp * kBpw + j;
            if (rl >= commit) break;
            const int32_t slot = s.tslot[ci + rl];
            const int nt = s.tntok[ci + rl];
            const KV* vp = kv + (int64_t)slot * slot_elems + v_off + base;
            float ob[DPL];
#pragma unroll
            for (int jj = 0; jj < DPL; ++jj) ob[jj] = 0.0f;
            if (T == TOK) {
#pragma unroll
                for (int t = 0; t < TOK; ++t) {
                    const float wt = s.w[warp][j][t];  // 0 for t >= ntok
                    float vr[DPL];
                    load_row<DPL>(vp + t * d, full, lim, vr);
#pragma unroll
                    for (int jj = 0; jj < DPL; ++jj) ob[jj] = fmaf(wt, vr[jj], ob[jj]);
                }
            } else {
#pragma unroll
                for (int t = 0; t < TOK; ++t) {
                    const float wt = s.w[warp][j][t];  // 0 for t >= ntok (and hence for t >= T)
                    float vr[DPL];
                    load_row<DPL>(vp + (size_t)(t < T ? t : T - 1) * d, full, lim, vr);
#pragma unroll
                    for (int jj = 0; jj < DPL; ++jj) ob[jj] = fmaf(wt, vr[jj], ob[jj]);
                }
            }
            const float mbj = s.mb[warp][j];
            const float mnew = fmaxf(M, mbj);
            const float a = expf(M - mnew);
            const float c = expf(mbj - mnew);
#pragma unroll
            for (int jj = 0; jj < DPL; ++jj) O[jj] = O[jj] * a + ob[jj] * c;
            L = L * a + s.lb[warp][j] * c;
            M = mnew;
        }
        if (fin) {
            if (threadIdx.x == 0) {
                const int64_t bp = cb + commit;
                b.bp[qi] = bp;
                b.est[qi] = s.est;
                b.term[qi] = b.topk > 0 ? (limit < n) : (bp < n);
            }
            break;
        }
        cb += cnt;
        __syncthreads();  // s.w / s.la / s.tb are rewritten next
    }
    // ---- finalize: merge the warps' states (finalize, attention.hpp:104-110) ----
    float* so = reinterpret_cast<float*>(s.hist);  // [kPsaWarps][256]
    if (lane == 0) {
        s.m[warp] = M;
        s.l[warp] = L;
    }
#pragma unroll
    for (int jj = 0; jj < DPL; ++jj)
        if (base + jj < d) so[warp * 256 + base + jj] = O[jj];
    __syncthreads();
    float Mt = -INFINITY;
#pragma unroll
    for (int w = 0; w < kPsaWarps; ++w) Mt = fmaxf(Mt, s.m[w]);
    float Lt = 0.0f, sc[kPsaWarps];
#pragma unroll
    for (int w = 0; w < kPsaWarps; ++w) {
        sc[w] = s.l[w] > 0.0f ? expf(s.m[w] - Mt) : 0.0f;
        Lt += s.l[w] * sc[w];
    }
    for (int i = threadIdx.x; i < d; i += kPsaThreads) {
        float o = 0.0f;
#pragma unroll
        for (int w = 0; w < kPsaWarps; ++w) o += sc[w] > 0.0f ? so[w * 256 + i] * sc[w] : 0.0f;
        b.out[(size_t)qi * d + i] = o / Lt;
    }
    if (b.tcov && threadIdx.x == 0) {
        double tc2 = -1.0;
        if (b.audit) {
            // total mass over all n blocks (engine.cpp:88 total_log_as)
            double mx = -INFINITY;
            for (int64_t i = 0; i < n; ++i) mx = fmax(mx, omass[i]);
            double sm = 0.0;
            for (int64_t i = 0; i < n; ++i) sm += exp(omass[i] - mx);
            tc2 = exp(s.acc - (mx + log(sm)));
        }
        b.tcov[qi] = tc2;
    }
}

template <typename KV, int TOK>
static void launch_psa_t(const PoolView& p, const BatchView& b, int nq, cudaStream_t st) {
    switch (dpl_for(b.d)) {  // d=64 and d=128 are always "full"; other d use the masked 8-dim path
        case 2: psa_kernel<KV, 2, TOK, true><<<nq, kPsaThreads, 0, st>>>(p, b); break;
        case 4: psa_kernel<KV, 4, TOK, true><<<nq, kPsaThreads, 0, st>>>(p, b); break;
        default:
            if (b.d == 256) psa_kernel<KV, 8, TOK, true><<<nq, kPsaThreads, 0, st>>>(p, b);
            else psa_kernel<KV, 8, TOK, false><<<nq, kPsaThreads, 0, st>>>(p, b);
            break;
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
