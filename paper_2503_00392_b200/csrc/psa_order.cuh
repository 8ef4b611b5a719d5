// psa_order.cuh — ordering (lazy tranche selection) and the coverage decide
// step shared by the progressive kernels (kernels_psa.cu, kernels_gqa.cu).
#pragma once

#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace psa {

constexpr int kPsaWarps = 8;
constexpr int kPsaThreads = kPsaWarps * 32;
constexpr int kChunk = 32;
constexpr int kBins = 2048;
#ifndef PSA_SCAN_U
#define PSA_SCAN_U 8
#endif

// A group of whole warps cooperating on one selection: the full CTA (__syncthreads)
// or a sub-team synchronised by a named barrier (bar.sync id, size).
struct Team {
    int tid;   // thread index within the team
    int size;  // threads in the team (multiple of 32)
    int bar;   // named barrier id (0 = the CTA barrier)
};
__device__ __forceinline__ void team_sync(const Team& tm) {
    if (tm.bar == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(tm.bar), "r"(tm.size) : "memory");
}
__device__ __forceinline__ Team cta_team() { return Team{(int)threadIdx.x, (int)blockDim.x, 0}; }

struct SelScratch {
    unsigned long long red_min, red_max;
    unsigned int red_cnt, gcount, excl;
    int bstar;
    unsigned wsum[kPsaWarps];
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
// Steps whose partner distance is >= 32 exchange through shared memory (one team barrier
// each); the remaining steps of every stage (distance < 32: the partner sits in the same
// aligned 32-element group) run in registers, one warp per group, partners by shuffle —
// one barrier per stage instead of one per step.
#ifndef PSA_BITONIC_WARP
#define PSA_BITONIC_WARP 2  // 1: warp-shuffle steps; 2: + shared-memory steps grouped three at a time
#endif
// S consecutive shared-memory steps of one stage at once (partner masks m[0..S-1], the first
// possibly the stage's reversal mask k-1, the rest single bits): each thread owns groups of 2^S
// elements closed under the S partner maps, loads them once, runs the S compare-exchange
// layers in registers and stores them once — one barrier per S steps.
template <int S>
__device__ __forceinline__ void bitonic_group_steps(uint64_t* a, int n, int n2, const int (&m)[3], const int (&hb)[3],
                                                    const Team& tm) {
    for (int i = tm.tid; i < (n2 >> S); i += tm.size) {
        // base: i with zero bits inserted at the masks' top-bit positions (lowest first, so a
        // later insertion never moves an earlier one)
        int bse = i;
#pragma unroll
        for (int q = S - 1; q >= 0; --q) {
            const int lowm = hb[q] - 1;
            bse = ((bse & ~lowm) << 1) | (bse & lowm);
        }
        int idx[1 << S];
        unsigned long long v[1 << S];
#pragma unroll
        for (int t = 0; t < (1 << S); ++t) {
            int x = bse;
#pragma unroll
            for (int q = 0; q < S; ++q)
                if (t & (1 << q)) x ^= m[q];
            idx[t] = x;
            v[t] = x < n ? a[x] : ~0ull;
        }
#pragma unroll
        for (int q = 0; q < S; ++q)
#pragma unroll
            for (int t = 0; t < (1 << S); ++t)
                if (!(t & (1 << q))) {
                    const int u = t | (1 << q);
                    const bool tlow = (idx[t] & hb[q]) == 0;  // the lower index keeps the minimum
                    const unsigned long long x = v[t], y = v[u];
                    const unsigned long long mn = x < y ? x : y, mx = x < y ? y : x;
                    v[t] = tlow ? mn : mx;
                    v[u] = tlow ? mx : mn;
                }
#pragma unroll
        for (int t = 0; t < (1 << S); ++t)
            if (idx[t] < n) a[idx[t]] = v[t];
    }
}

__device__ __forceinline__ void bitonic_smem(uint64_t* a, int n, const Team& tm) {
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    const int lane = threadIdx.x & 31, wt = tm.tid >> 5, nw = tm.size >> 5;
    for (int k = 2; k <= n2; k <<= 1) {
        int j = k >> 1;
        if (PSA_BITONIC_WARP >= 2) {
            while (j >= 32) {
                int m[3] = {0, 0, 0}, hb[3] = {1, 1, 1}, s = 0;
                for (; s < 3 && j >= 32; ++s, j >>= 1) {
                    m[s] = (j == (k >> 1)) ? k - 1 : j;
                    hb[s] = j;
                }
                if (s == 3) bitonic_group_steps<3>(a, n, n2, m, hb, tm);
                else if (s == 2) bitonic_group_steps<2>(a, n, n2, m, hb, tm);
                else bitonic_group_steps<1>(a, n, n2, m, hb, tm);
                team_sync(tm);
            }
        }
        for (; j > 0 && (!PSA_BITONIC_WARP || j >= 32); j >>= 1) {
            for (int i = tm.tid; i < (n2 >> 1); i += tm.size) {
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
            team_sync(tm);
        }
        if (j == 0) continue;
        for (int g = wt; g * 32 < n2; g += nw) {
            const int idx = g * 32 + lane;
            unsigned long long x = idx < n ? a[idx] : ~0ull;
            for (int jj = j; jj > 0; jj >>= 1) {
                // the stage's first step pairs idx with idx ^ (k - 1), later ones with idx ^ jj;
                // either way the lower index of the pair has bit jj clear and keeps the minimum
                const unsigned long long y = __shfl_xor_sync(PSA_FULL, x, jj == (k >> 1) ? k - 1 : jj);
                x = ((lane & jj) == 0) == (x < y) ? x : y;
            }
            if (idx < n) a[idx] = x;
        }
        team_sync(tm);
    }
}

// Calls f(key) for every key of the head: 16-byte loads (two keys), 8 in flight per
// thread (the scan is latency-bound: a team of 64 threads keeps 8 KB in flight).
// Scalar head/tail keys are handled by team thread 0, so f must tolerate a partial warp.
template <typename F>
__device__ __forceinline__ void scan_keys(const uint64_t* __restrict__ keys, int64_t n, const Team& tm, F&& f) {
    constexpr int U = PSA_SCAN_U;
    const int64_t head = ((reinterpret_cast<uintptr_t>(keys) & 15) && n > 0) ? 1 : 0;
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys + head);
    const int64_t n2 = (n - head) >> 1;
    for (int64_t i0 = tm.tid; i0 < n2; i0 += (int64_t)U * tm.size) {
        ulonglong2 k[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + (int64_t)u * tm.size;
            k[u] = i < n2 ? __ldg(k2 + i) : make_ulonglong2(~0ull, ~0ull);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + (int64_t)u * tm.size < n2) {
                f(k[u].x);
                f(k[u].y);
            }
    }
    if (tm.tid == 0) {
        if (head) f(__ldg(reinterpret_cast<const unsigned long long*>(keys)));
        if ((n - head) & 1) f(__ldg(reinterpret_cast<const unsigned long long*>(keys) + n - 1));
    }
}

// Next tranche: the C (<= kTCap, ~target) smallest keys greater than `last` (all keys if first).
static __device__ __noinline__ int select_tranche(SelScratch& s, uint64_t* tb, int cap, uint32_t* hist, int nbins,
                                          const uint64_t* __restrict__ keys, int64_t n, uint64_t last, bool first,
                                          unsigned target, Team tm, const unsigned long long* bounds = nullptr,
                                          int64_t bstride = 0) {
    const int tid = tm.tid, lane = threadIdx.x & 31;
    unsigned long long lmin = ~0ull, lmax = 0;
    unsigned lcnt = 0;
    if (first && bounds) {  // min / max of all keys from the score kernel: no scan
        if (tid == 0) {
            lmin = bounds[0];
            lmax = bounds[bstride];
            lcnt = (unsigned)n;
        }
    } else {
        scan_keys(keys, n, tm, [&](uint64_t k) {
            if (first || k > last) {
                lmin = k < lmin ? k : lmin;
                lmax = k > lmax ? k : lmax;
                ++lcnt;
            }
        });
    }
    if (tid == 0) {
        s.red_min = ~0ull;
        s.red_max = 0;
        s.red_cnt = 0;
        s.gcount = 0;
    }
    team_sync(tm);
    lmin = warp_min_u64(lmin);
    lmax = warp_max_u64(lmax);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) lcnt += __shfl_xor_sync(PSA_FULL, lcnt, o);
    if (lane == 0) {
        atomicMin(&s.red_min, lmin);
        atomicMax(&s.red_max, lmax);
        atomicAdd(&s.red_cnt, lcnt);
    }
    team_sync(tm);
    const uint64_t kmax = s.red_max;
    uint64_t tau = kmax;
    if (s.red_cnt > (unsigned)cap) {
        uint64_t lo = s.red_min, hi = kmax;
        unsigned need = target, before = 0;
        for (int it = 0; it < 10; ++it) {
            const uint64_t span = hi - lo;
            const int bits = 64 - __clzll((long long)span);
            const int bbits = 31 - __clz(nbins);  // log2(nbins): bin index (k - lo) >> sh < nbins
            const int sh = bits > bbits ? bits - bbits : 0;
            for (int i = tid; i < nbins; i += tm.size) hist[i] = 0;
            team_sync(tm);
            scan_keys(keys, n, tm, [&](uint64_t k) {
                if ((first || k > last) && k >= lo && k <= hi) atomicAdd(&hist[(k - lo) >> sh], 1u);
            });
            team_sync(tm);
            // first bin b with cum(b) >= need: each thread owns nbins/size consecutive bins
            const int per = nbins / tm.size;
            unsigned loc = 0;
            for (int j = 0; j < per; ++j) loc += hist[tid * per + j];
            unsigned inc = loc;  // inclusive warp scan
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(PSA_FULL, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) s.wsum[tid >> 5] = inc;
            team_sync(tm);
            unsigned wbase = 0;
            for (int w = 0; w < (tid >> 5); ++w) wbase += s.wsum[w];
            unsigned cum = wbase + inc - loc;  // exclusive prefix of this thread's bins
            if (cum < need && need <= cum + loc) {
#pragma unroll 1
                for (int j = 0; j < per; ++j) {
                    const unsigned c = hist[tid * per + j];
                    if (need <= cum + c) {
                        s.bstar = tid * per + j;
                        s.excl = cum;
                        break;
                    }
                    cum += c;
                }
            }
            team_sync(tm);
            const int bs = s.bstar;
            const unsigned ex = s.excl, incl = ex + hist[bs];
            const uint64_t width_m1 = (sh >= 64) ? ~0ull : ((1ull << sh) - 1ull);
            const uint64_t bin_lo = lo + ((uint64_t)bs << sh);
            if (before + incl <= (unsigned)cap) {
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
            team_sync(tm);
        }
    }
    // gather the survivors (warp-aggregated slot reservation)
    scan_keys(keys, n, tm, [&](uint64_t k) {
        const bool take = (first || k > last) && k <= tau;
        const unsigned m = __ballot_sync(__activemask(), take);
        if (take) {
            const int leader = __ffs(m) - 1;
            unsigned basei = 0;
            if (lane == leader) basei = atomicAdd(&s.gcount, (unsigned)__popc(m));
            basei = __shfl_sync(m, basei, leader);
            const unsigned idx = basei + __popc(m & ((1u << lane) - 1u));
            if (idx < (unsigned)cap) tb[idx] = k;
        }
    });
    team_sync(tm);
    const int C = (int)min(s.gcount, (unsigned)cap);
    bitonic_smem(tb, C, tm);
    return C;
}


// Tranche page-table fill: ranked positions -> rpos output, slots and token counts into
// shared memory. The two dependent gathers (slot, then its token count) are batched
// 8 per thread so one thread keeps 8 loads in flight instead of 2 serial misses per entry.
__device__ __forceinline__ void fill_tranche(const uint64_t* tb, int tc, uint64_t pmask, int32_t* rpos_out,
                                             const int32_t* __restrict__ slots, const int32_t* ntok, int32_t* tslot,
                                             uint8_t* tntok, const Team& tm) {
    constexpr int U = PSA_SCAN_U;
    for (int i0 = tm.tid; i0 < tc; i0 += U * tm.size) {
        int32_t sl[U], nt[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int i = i0 + k * tm.size;
            sl[k] = 0;
            if (i < tc) {
                const int32_t pos = (int32_t)(tb[i] & pmask);
                rpos_out[i] = pos;
                sl[k] = slots[pos];
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) nt[k] = (i0 + k * tm.size < tc) ? ntok[sl[k]] : 0;
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int i = i0 + k * tm.size;
            if (i < tc) {
                tslot[i] = sl[k];
                tntok[i] = (uint8_t)nt[k];
            }
        }
    }
}

// Coverage decide step for one chunk of ranks [cb, cb+cnt), executed by ONE full
// warp: lane i holds x = log-mass of rank cb+i (valid for i < cnt). Running
// log-sum-exp and min (CoverageEstimator::observe, reference engine.cpp:38-46) are
// carried in acc/mn (lane-uniform). The estimate 1/(1 + n_left*exp(min - acc))
// (engine.cpp:48-55) is evaluated at every microbatch boundary; the first boundary
// with est > eps (engine.cpp:125), or the budget/end of the plan, stops the run.
struct Decision {
    int commit;  // ranks of this chunk that are processed
    int fin;     // run finished inside this chunk
    double est;  // estimate at the last evaluated boundary
};

__device__ __forceinline__ Decision decide_chunk(double x, int cnt, int64_t cb, int64_t n, int64_t limit, int m,
                                                 double eps, double& acc, double& mn, double* iest_head) {
    const int lane = threadIdx.x & 31;
    const bool valid = lane < cnt;
    const int64_t r = cb + lane;
    if (!valid) x = -INFINITY;
    double mx = warp_max_d(x);
    mx = fmax(mx, acc);
    double e = valid ? exp(x - mx) : 0.0;
    const double e0 = acc != -INFINITY ? exp(acc - mx) : 0.0;  // independent of the scan
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
    e += e0;  // S = sum exp(mass - mx) over everything observed up to this rank
    const double mn_i = fmin(mnv, mn);
    const int64_t nl = n - (r + 1);
    // est = 1 / (1 + nl * exp(min - acc)) with acc = mx + log S, i.e. S / (S + nl * exp(min - mx)):
    // the exp and the log (for the carried acc) are independent, so their latencies overlap.
    const double t = exp(mn_i - mx);
    const double acc_i = mx + log(e);
    const double est_i = nl == 0 ? 1.0 : (e > 0.0 ? e / fma((double)nl, t, e) : 0.0);
    const bool boundary = valid && (m == 1 || (((r + 1) % m) == 0) || (r + 1 == limit));
    const bool stop = boundary && (est_i > eps || r + 1 == limit);
    const unsigned bal = __ballot_sync(PSA_FULL, stop);
    const int f = bal ? (__ffs(bal) - 1) : (cnt - 1);
    if (iest_head && boundary && lane <= f) iest_head[r] = est_i;  // IterationStats::estimated_coverage
    acc = __shfl_sync(PSA_FULL, acc_i, f);
    mn = __shfl_sync(PSA_FULL, mn_i, f);
    Decision d;
    d.est = __shfl_sync(PSA_FULL, est_i, f);
    d.commit = f + 1;
    d.fin = bal ? 1 : 0;
    return d;
}

// Same decision with the in-chunk work in fp32 (MUFU exp, fp32 scans) and the running sum
// carried in fp64 as (M, S): log-sum-exp of everything observed = M + log S. The estimate
// est = S / (S + n_left * exp(min - M_i)) (the reference's 1 / (1 + n_left * exp(min - acc))
// with both sides scaled by exp(M_i - acc)) carries ~1e-7 relative error, so a decision can
// differ from the fp64 reference only within ~1e-7 of eps (the parity rule's tau is 1e-5).
// Returns false, leaving every argument untouched, when a chunk mass sits > 80 below the
// chunk maximum (fp32 exp would lose it): the caller then runs decide_chunk in fp64.
// PSA_DECIDE_FAST = 0 (default): the round and per-head kernels decide in fp64 throughout, so the
// reported estimated_coverage carries fp64 accuracy like the reference's CoverageEstimator;
// 1 = the fp32 chunk scan below (measured faster on the round kernel, ~1e-7 relative estimate).
#ifndef PSA_DECIDE_FAST
#define PSA_DECIDE_FAST 0
#endif
__device__ __forceinline__ bool decide_chunk_fast(float x, int cnt, int64_t cb, int64_t n, int64_t limit, int m,
                                                  double eps, double& M, double& S, double& mn, double* iest_head,
                                                  Decision& d) {
    const int lane = threadIdx.x & 31;
    const bool valid = lane < cnt;
    const int64_t r = cb + lane;
    const float xf = valid ? x : -INFINITY;
    float cmax = xf;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) cmax = fmaxf(cmax, __shfl_xor_sync(PSA_FULL, cmax, o));
    const float Mf = (float)M;  // M is a carried fp32 mass (or -inf)
    const float mx = fmaxf(cmax, Mf);
    const float dx = xf - mx;
    if (__any_sync(PSA_FULL, valid && dx < -80.0f)) return false;
    float e = valid ? expf(dx) : 0.0f;
    const double scale = M == -INFINITY ? 0.0 : (double)expf(Mf - mx);
    float mnv = valid ? xf : INFINITY;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float ye = __shfl_up_sync(PSA_FULL, e, o);
        const float ym = __shfl_up_sync(PSA_FULL, mnv, o);
        if (lane >= o) {
            e += ye;
            mnv = fminf(mnv, ym);
        }
    }
    const double Si = fma(S, scale, (double)e);  // sum exp(mass - mx) observed up to this rank
    const float mn_i = fminf(mnv, (float)mn);
    const int64_t nl = n - (r + 1);
    const float t = expf(mn_i - mx);
    const float sf = (float)Si;
    const float est_f = nl == 0 ? 1.0f : (sf > 0.0f ? sf / fmaf((float)nl, t, sf) : 0.0f);
    const double est_i = (double)est_f;
    const bool boundary = valid && (m == 1 || (((r + 1) % m) == 0) || (r + 1 == limit));
    const bool stop = boundary && (est_i > eps || r + 1 == limit);
    const unsigned bal = __ballot_sync(PSA_FULL, stop);
    const int f = bal ? (__ffs(bal) - 1) : (cnt - 1);
    if (iest_head && boundary && lane <= f) iest_head[r] = est_i;
    M = (double)mx;
    S = __shfl_sync(PSA_FULL, Si, f);
    mn = (double)__shfl_sync(PSA_FULL, mn_i, f);
    d.est = __shfl_sync(PSA_FULL, est_i, f);
    d.commit = f + 1;
    d.fin = bal ? 1 : 0;
    return true;
}

}  // namespace psa
