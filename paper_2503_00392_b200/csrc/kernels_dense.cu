// kernels_dense.cu — dense mode of the GQA progressive path (bf16 pool, d = 128, blocks <= 16
// tokens, group 2..4, estimated ranking).
//
// The round-based GQA kernel (kernels_gqa.cu) reads a block once per ROUND in which any head
// of the group reaches it. When the heads need many ranks (weakly skewed attention, e.g.
// isotropic keys: ~90% of the list at eps 0.95) their rank orders diverge and a block is
// K-scored in up to g different rounds. psa_gqa_kernel therefore hands a unit over to this
// path when one of its heads has consumed kDenseHandover (384) ranks without stopping, and the unit
// is redone:
//
//   dense_k_kernel           ONE K pass over every block of the list (tensor-core scores for
//                            all heads at once): per (head, block) the fp32 block mass
//                            la = m + log(l) (block_partial_attention's log_as, reference
//                            attention.hpp:73) and the normalised token weights p_t = w_t / l;
//   dense_decide_kernel      per head: its full rank order (bitonic sort of the head's keys in
//                            shared memory) and Algorithm 1's stop rule over the masses in rank
//                            order, evaluated for all ranks at once (per-thread online
//                            log-sum-exp, block scan, second walk: the first boundary with
//                            est > eps) -> blocks_processed, estimate, rank threshold key;
//   dense_v_kernel           ONE V pass over the union of the heads' processed sets: block b
//                            belongs to head h's set iff key_h(b) <= threshold_h (keys are
//                            unique and ordered), accumulated with mma.sync like the round
//                            kernel's V pass, merged with weight exp(la - M).
//
// Same processed sets and stop points as the round kernel (identical masses; the estimates
// differ only by rounding, ~1e-7); outputs differ only by fp32 summation order.
#include <cuda_bf16.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"
#include "mma.cuh"
#include "psa_order.cuh"

namespace psa {

constexpr int kDenseWarps = 8;
#ifndef PSA_DENSE_PF
#define PSA_DENSE_PF 2
#endif
constexpr int kDensePf = PSA_DENSE_PF;  // L2 prefetch distance (warp iterations)
#ifndef PSA_DENSE_VPF
#define PSA_DENSE_VPF 1  // V pass: L2 prefetch of the weights / masses with the V block
#endif

// q fragments of the K pass (see psa_gqa_kernel): columns = (head, split), 4 per head.
template <int G>
__device__ __forceinline__ void load_qg(const BatchView& b, int u, int lane, uint32_t (&qg)[8][(G * 4 + 7) / 8][2]) {
    constexpr int NT = (G * 4 + 7) / 8;
    const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
    for (int tile = 0; tile < NT; ++tile) {
        const int hq = tile * 2 + (gq >> 2), sp = gq & 3;
        const float* qrow = b.q + ((size_t)u * b.g + (hq < b.g ? hq : 0)) * 128;
#pragma unroll
        for (int st = 0; st < 8; ++st)
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                uint32_t packed = 0;
#pragma unroll
                for (int e2 = 0; e2 < 2; ++e2) {
                    const float x = hq < b.g ? bf16_split(qrow[32 * tq + 4 * st + 2 * hf + e2], sp) : 0.0f;
                    packed |= bf16_bits(x) << (16 * e2);
                }
                qg[st][tile][hf] = packed;
            }
    }
}

// Work items of the K and V passes: (handed-over unit, slice of kDenseSlice list positions), so a
// few long units still spread over every SM (the V pass merges the slices' partial states).
__device__ __forceinline__ int dense_slices(const BatchView& b) { return (int)((b.max_n + b.dense_slice - 1) / b.dense_slice); }
// The round's unit list: round 0 the hand-over list, round 1 the escalated units.
__device__ __forceinline__ const int32_t* dense_list(const BatchView& b) {
    return b.dense_round == 0 ? b.dense_flag : b.dense_esc;
}
__device__ __forceinline__ int dense_list_count(const BatchView& b) {
    return *(b.dense_round == 0 ? b.dense_count : b.dense_esc_count);
}
// Round 0 skips, after its decide, the units a head escalated (round 1 redoes them).
__device__ __forceinline__ bool dense_skip(const BatchView& b, int u) {
    return b.dense_round == 0 && b.dense_esc_mark[u] > 0;
}

template <int G>
__device__ __forceinline__ void dense_k_unit(const PoolView& p, const BatchView& b, int u, int64_t e_begin, int64_t e_end) {
    constexpr int NT = (G * 4 + 7) / 8;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int64_t off = b.list_off[u], n = b.list_off[u + 1] - off;
    const float fscale = (float)b.scale;
    const int T = p.T;
    uint32_t qg[8][NT][2];
    load_qg<G>(b, u, lane, qg);
    // the small dependent loads (page-table slot, its ntok, the prefetch target's slot) are
    // issued one iteration ahead so they never sit on the block's critical path
    constexpr int64_t kPfd = (int64_t)kDensePf * kDenseWarps;
    // blocks this round computes: round 0 = the heads' candidate prefixes (key <= dense_sel), round 1
    // = the rest; every block when a head's candidate threshold is ~0 (no key test)
    uint64_t sel[G];
    bool all_sel = true;
#pragma unroll
    for (int h = 0; h < G; ++h) {
        sel[h] = h < b.g ? b.dense_sel[(size_t)u * b.g + h] : 0ull;
        all_sel = all_sel && (h >= b.g || sel[h] == ~0ull);
    }
    const bool every = all_sel && b.dense_round == 0;
    auto wanted = [&](int64_t f) -> bool {
        if (f >= e_end) return false;
        if (every) return true;
        bool cand = false;
#pragma unroll
        for (int h = 0; h < G; ++h)
            if (h < b.g) cand = cand || b.keys[off * b.g + (int64_t)h * n + f] <= sel[h];
        return b.dense_round == 0 ? cand : !cand;
    };
    // one block: K tile -> tensor-core scores of every head -> mass la and token weights p_t
    auto block = [&](int64_t e, int32_t slot, int nt) {
        const __nv_bfloat16* kblk = kv_block<__nv_bfloat16>(p, slot);
        const int r0 = gq < T ? gq : T - 1, r1 = (gq + 8) < T ? (gq + 8) : T - 1;
        const uint4* p0 = reinterpret_cast<const uint4*>(kblk + (size_t)r0 * 128 + 32 * tq);
        const uint4* p1 = reinterpret_cast<const uint4*>(kblk + (size_t)r1 * 128 + 32 * tq);
        uint32_t w0[16], w1[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 x0 = __ldg(p0 + i), x1 = __ldg(p1 + i);
            w0[4 * i] = x0.x; w0[4 * i + 1] = x0.y; w0[4 * i + 2] = x0.z; w0[4 * i + 3] = x0.w;
            w1[4 * i] = x1.x; w1[4 * i + 1] = x1.y; w1[4 * i + 2] = x1.z; w1[4 * i + 3] = x1.w;
        }
        float c[NT][4];
#pragma unroll
        for (int tile = 0; tile < NT; ++tile) c[tile][0] = c[tile][1] = c[tile][2] = c[tile][3] = 0.f;
#pragma unroll
        for (int st = 0; st < 8; ++st)
#pragma unroll
            for (int tile = 0; tile < NT; ++tile)
                mma_bf16_16816(c[tile][0], c[tile][1], c[tile][2], c[tile][3], w0[2 * st], w1[2 * st], w0[2 * st + 1],
                               w1[2 * st + 1], qg[st][tile][0], qg[st][tile][1]);
#pragma unroll
        for (int tile = 0; tile < NT; ++tile) {
            float lo = c[tile][0] + c[tile][1], hi = c[tile][2] + c[tile][3];
            lo += __shfl_xor_sync(PSA_FULL, lo, 1);
            hi += __shfl_xor_sync(PSA_FULL, hi, 1);
            const int hq = tile * 2 + (tq >> 1);
            lo = (gq < nt) ? lo * fscale : -INFINITY;
            hi = (gq + 8 < nt) ? hi * fscale : -INFINITY;
            float mbv = fmaxf(lo, hi);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) mbv = fmaxf(mbv, __shfl_xor_sync(PSA_FULL, mbv, o));
            const float wlo = (gq < nt) ? expf(lo - mbv) : 0.0f;
            const float whi = (gq + 8 < nt) ? expf(hi - mbv) : 0.0f;
            float lbv = wlo + whi;
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) lbv += __shfl_xor_sync(PSA_FULL, lbv, o);
            if ((tq & 1) == 0 && hq < b.g) {
                const int64_t hb = off * b.g + (int64_t)hq * n;
                float* pw = b.dense_p + (hb + e) * 16;
                const float inv = 1.0f / lbv;
                pw[gq] = wlo * inv;
                pw[gq + 8] = whi * inv;
                if (gq == 0) b.dense_la[hb + e] = mbv + logf(lbv);
            }
        }
    };
    int64_t e = e_begin + warp;
    if (every) {  // whole list: the page-table loads one iteration ahead, L2 prefetch kDensePf ahead
        int32_t slot_n = e < e_end ? b.slots[off + e] : 0;
        int nt_n = e < e_end ? p.ntok[slot_n] : 0;
        int32_t sf_n = e + kPfd < e_end ? b.slots[off + e + kPfd] : -1;
        for (; e < e_end; e += kDenseWarps) {
            const int32_t slot = slot_n, sf = sf_n;
            const int nt = nt_n;
            const int64_t en = e + kDenseWarps;
            if (en < e_end) {
                slot_n = b.slots[off + en];
                nt_n = p.ntok[slot_n];
            }
            sf_n = en + kPfd < e_end ? b.slots[off + en + kPfd] : -1;
            if (lane == 0 && sf >= 0 && kv_resident(p, sf))
                prefetch_l2_bulk(kv_block<__nv_bfloat16>(p, sf), (uint32_t)(T * 128 * 2));
            block(e, slot, nt);
        }
        return;
    }
    // a subset of the list: the warp's positions e + 8j are tested 32 at a time (one lane each: keys,
    // then slot and token count of the wanted ones), a ballot gives the window's wanted blocks, and
    // the L2 prefetch runs kDensePf wanted blocks ahead across the window boundary
    constexpr int64_t kWin = 32 * (int64_t)kDenseWarps;
    auto window = [&](int64_t wb, uint32_t& m, int32_t& sl, int& ntk) {
        const int64_t f = wb + (int64_t)kDenseWarps * lane;
        const bool ok = wanted(f);
        sl = ok ? b.slots[off + f] : 0;
        ntk = ok ? p.ntok[sl] : 0;
        m = __ballot_sync(PSA_FULL, ok);
    };
    uint32_t mc, mn;
    int32_t sc, sn;
    int tc, tn;
    window(e, mc, sc, tc);
    window(e + kWin, mn, sn, tn);
    for (int64_t wb = e; wb < e_end; wb += kWin) {
        const uint64_t comb = (uint64_t)mc | ((uint64_t)mn << 32);
        uint32_t rem = mc;
        while (rem) {
            const int i = __ffs(rem) - 1;
            rem &= rem - 1;
            uint64_t ahead = comb & ~((2ull << i) - 1ull);  // wanted blocks after i
#pragma unroll
            for (int k = 1; k < kDensePf; ++k) ahead &= ahead - 1;
            if (ahead) {
                const int j = __ffsll((long long)ahead) - 1;
                const int32_t sf = __shfl_sync(PSA_FULL, j < 32 ? sc : sn, j & 31);
                if (lane == 0 && kv_resident(p, sf))
                    prefetch_l2_bulk(kv_block<__nv_bfloat16>(p, sf), (uint32_t)(T * 128 * 2));
            }
            block(wb + (int64_t)kDenseWarps * i, __shfl_sync(PSA_FULL, sc, i), __shfl_sync(PSA_FULL, tc, i));
        }
        mc = mn;
        sc = sn;
        tc = tn;
        window(wb + 2 * kWin, mn, sn, tn);
    }
}

template <int G>
__global__ void __launch_bounds__(kDenseWarps * 32) dense_k_kernel(PoolView p, BatchView b) {
    const int S = dense_slices(b);
    const int32_t* list = dense_list(b);
    for (int item = blockIdx.x; item < dense_list_count(b) * S; item += gridDim.x) {
        const int u = list[item / S];
        const int64_t n = b.list_off[u + 1] - b.list_off[u];
        const int64_t e0 = (int64_t)(item % S) * b.dense_slice, e1 = e0 + b.dense_slice < n ? e0 + b.dense_slice : n;
        if (e0 < n) dense_k_unit<G>(p, b, u, e0, e1);
    }
}

// One CTA per (flagged unit, head): the head's keys sorted in shared memory, then warp 0 runs
// the stop rule over the masses in rank order.
__device__ __forceinline__ void dense_decide_head(const BatchView& b, int u, int h, uint64_t* ks);

#ifndef PSA_DECIDE_THREADS
#define PSA_DECIDE_THREADS 256
#endif
constexpr int kDecideThreads = PSA_DECIDE_THREADS;
__global__ void __launch_bounds__(kDecideThreads) dense_decide_kernel(BatchView b) {
    extern __shared__ __align__(16) unsigned char dsm[];
    uint64_t* ks = reinterpret_cast<uint64_t*>(dsm);
    const int32_t* list = dense_list(b);
    for (int item = blockIdx.x; item < dense_list_count(b) * b.g; item += gridDim.x) {
        dense_decide_head(b, list[item / b.g], item % b.g, ks);
        __syncthreads();
    }
}

// Bucket sort of a head's keys in shared memory (n <= kBucketPerThread * blockDim.x): keys are
// binned linearly in their decoded score between the head's min and max (monotone in the key,
// so bins are ordered), scattered by a block-wide counting pass and each bin is finished by an
// insertion sort. Returns false, leaving ks untouched, when a bin holds more than kBucketMax keys
// (the caller then runs the bitonic network). Uses `hist` (nbins u32, nbins a power of two).
#ifndef PSA_DECIDE_BUCKET
#define PSA_DECIDE_BUCKET 1
#endif
#ifndef PSA_DECIDE_BINS
#define PSA_DECIDE_BINS 2048
#endif
#ifndef PSA_DECIDE_SCAN
#define PSA_DECIDE_SCAN 1
#endif
constexpr int kBucketPerThread = 32;
constexpr unsigned kBucketMax = 64;
__device__ bool bucket_sort_smem(uint64_t* ks, int n, uint64_t pmask, uint32_t* hist, int nbins) {
    __shared__ unsigned long long s_min, s_max;
    __shared__ unsigned s_big, wsum[32];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    uint64_t r[kBucketPerThread];
    unsigned long long lmin = ~0ull, lmax = 0;
#pragma unroll
    for (int k = 0; k < kBucketPerThread; ++k) {
        const int i = tid + k * nt;
        r[k] = i < n ? ks[i] : ~0ull;
        if (i < n) {
            lmin = r[k] < lmin ? r[k] : lmin;
            lmax = r[k] > lmax ? r[k] : lmax;
        }
    }
    if (tid == 0) {
        s_min = ~0ull;
        s_max = 0;
        s_big = 0;
    }
    for (int i = tid; i < nbins; i += nt) hist[i] = 0;
    __syncthreads();
    lmin = warp_min_u64(lmin);
    lmax = warp_max_u64(lmax);
    if (lane == 0) {
        atomicMin(&s_min, lmin);
        atomicMax(&s_max, lmax);
    }
    __syncthreads();
    const double smax = key_score(s_min, pmask), smin = key_score(s_max, pmask);  // smallest key = top score
    const double range = smax - smin;
    if (!(range < 1e300)) return false;  // inf / nan scores: leave it to the bitonic network (uniform)
    const double inv = range > 0.0 ? (double)(nbins - 1) / range : 0.0;
    auto bin_of = [&](uint64_t k) {
        const int bb = (int)((smax - key_score(k, pmask)) * inv);
        return bb < 0 ? 0 : (bb >= nbins ? nbins - 1 : bb);
    };
#pragma unroll
    for (int k = 0; k < kBucketPerThread; ++k)
        if (tid + k * nt < n) atomicAdd(&hist[bin_of(r[k])], 1u);
    __syncthreads();
    // exclusive scan of the bin counts: thread t owns bins [t*per, (t+1)*per)
    const int per = (nbins + nt - 1) / nt;
    const int b0 = tid * per, b1 = b0 + per < nbins ? b0 + per : nbins;
    unsigned loc = 0, mx = 0;
    for (int j = b0; j < b1; ++j) {
        const unsigned c = hist[j];
        loc += c;
        mx = c > mx ? c : mx;
    }
    unsigned inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(PSA_FULL, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    if (mx > kBucketMax) atomicOr(&s_big, 1u);
    __syncthreads();
    if (s_big) return false;
    unsigned run = inc - loc;
    for (int w = 0; w < warp; ++w) run += wsum[w];
    for (int j = b0; j < b1; ++j) {
        const unsigned c = hist[j];
        hist[j] = run;
        run += c;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kBucketPerThread; ++k)
        if (tid + k * nt < n) ks[atomicAdd(&hist[bin_of(r[k])], 1u)] = r[k];
    __syncthreads();
    // hist[j] is now the end of bin j; insertion sort inside each bin
    for (int j = tid; j < nbins; j += nt) {
        const int s0 = j ? (int)hist[j - 1] : 0, s1 = (int)hist[j];
        for (int i = s0 + 1; i < s1; ++i) {
            const uint64_t x = ks[i];
            int q = i - 1;
            while (q >= s0 && ks[q] > x) {
                ks[q + 1] = ks[q];
                --q;
            }
            ks[q + 1] = x;
        }
    }
    __syncthreads();
    return true;
}

__device__ __forceinline__ void dense_decide_head(const BatchView& b, int u, int h, uint64_t* ks) {
    const int qi = u * b.g + h;
    const int64_t off = b.list_off[u], n = b.list_off[u + 1] - off;
    const int64_t hb = off * b.g + (int64_t)h * n;
    const uint64_t pmask = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);
    const int64_t limit = b.topk > 0 ? (b.topk < n ? b.topk : n) : n;
    const double eps = b.topk > 0 ? 1.0 : b.eps;
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    // round 0 decides on the head's candidate prefix (keys <= sel: the top ranks, whatever their
    // order) and escalates the unit when the head does not stop inside it
    const uint64_t sel = b.dense_round == 0 ? b.dense_sel[qi] : ~0ull;
    __shared__ int s_nsel;
    int64_t ns = n;  // keys sorted and walked
    if (sel == ~0ull) {  // 8 loads in flight per thread (the loop is latency-bound otherwise)
        constexpr int U = 8;
        for (int64_t i0 = threadIdx.x; i0 < n2; i0 += (int64_t)U * blockDim.x) {
            uint64_t v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int64_t i = i0 + (int64_t)k * blockDim.x;
                v[k] = i < n ? __ldg(reinterpret_cast<const unsigned long long*>(b.keys) + hb + i) : ~0ull;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int64_t i = i0 + (int64_t)k * blockDim.x;
                if (i < n2) ks[i] = v[k];
            }
        }
    } else {  // compaction of the candidates (any order: they are sorted next)
        if (threadIdx.x == 0) s_nsel = 0;
        __syncthreads();
        const int lane = threadIdx.x & 31;
        constexpr int U = 8;
        for (int64_t i0 = threadIdx.x; i0 < n; i0 += (int64_t)U * blockDim.x) {
            uint64_t v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int64_t i = i0 + (int64_t)k * blockDim.x;
                v[k] = i < n ? __ldg(reinterpret_cast<const unsigned long long*>(b.keys) + hb + i) : ~0ull;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const bool take = v[k] <= sel;  // (~0 padding never passes: sel < ~0)
                const unsigned m = __ballot_sync(PSA_FULL, take);
                int base = 0;
                if (lane == 0 && m) base = atomicAdd(&s_nsel, __popc(m));
                base = __shfl_sync(PSA_FULL, base, 0);
                if (take) ks[base + __popc(m & ((1u << lane) - 1u))] = v[k];
            }
        }
        __syncthreads();
        ns = s_nsel;
    }
    __syncthreads();
    {
        // bins: the rank-order mass array's space (n2 floats) before it is filled
        const int nbins = n2 < PSA_DECIDE_BINS ? n2 : PSA_DECIDE_BINS;
        if (!(PSA_DECIDE_BUCKET && ns <= (int64_t)kBucketPerThread * blockDim.x &&
              bucket_sort_smem(ks, (int)ns, pmask, reinterpret_cast<uint32_t*>(ks + n2), nbins)))
            bitonic_smem(ks, (int)ns, cta_team());
    }
    const int64_t wl = limit < ns ? limit : ns;  // ranks walked: the budget, or the candidate prefix
    // every rank's list position (ranked_pos output) and mass, gathered by the whole CTA so the
    // sequential walk below reads shared memory only
    float* xs = reinterpret_cast<float*>(ks + n2);
    {
        constexpr int U = 8;
        for (int64_t r0 = threadIdx.x; r0 < wl; r0 += (int64_t)U * blockDim.x) {
            float v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int64_t r = r0 + (int64_t)k * blockDim.x;
                v[k] = r < wl ? __ldg(b.dense_la + hb + (int64_t)(ks[r] & pmask)) : 0.0f;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int64_t r = r0 + (int64_t)k * blockDim.x;
                if (r < wl) {
                    b.rpos[hb + r] = (int32_t)(ks[r] & pmask);
                    xs[r] = v[k];
                }
            }
        }
    }
    __syncthreads();
    // Algorithm 1's stop rule over all ranks at once (every mass is known): thread t owns ranks
    // [t*seg, (t+1)*seg). (1) online log-sum-exp (running max M, fp64 sum S relative to it, min)
    // of its segment; (2) its exclusive prefix over the other threads' triples; (3) a second walk from the
    // prefix evaluating est = S / (S + n_left * exp(min - M)) at every microbatch boundary (the
    // reference's 1 / (1 + n_left * exp(min - acc)), engine.cpp:48-55); (4) the first rank whose
    // boundary has est > eps (or reaches the limit) over the block is the stop point.
    __shared__ float tM[kDecideThreads], tmn[kDecideThreads];
    __shared__ double tS[kDecideThreads];
    __shared__ unsigned long long first_stop;
    const int tid = threadIdx.x;
    const int64_t seg = (wl + kDecideThreads - 1) / kDecideThreads;
    const int64_t r0 = (int64_t)tid * seg, r1 = r0 + seg < wl ? r0 + seg : wl;
    // (the walk uses fp32 exponentials; the reported estimate is recomputed in fp64 below)
    auto absorb = [](float x, float& M, double& S, float& mn) {
        if (x > M) {
            S = (M == -INFINITY) ? 1.0 : fma(S, (double)expf(M - x), 1.0);
            M = x;
        } else {
            S += (double)expf(x - M);
        }
        mn = fminf(mn, x);
    };
    auto combine = [](float Ma, double Sa, float mna, float& M, double& S, float& mn) {  // (a) then (M, S, mn)
        const float Mx = fmaxf(Ma, M);
        const double sa = Ma == -INFINITY ? 0.0 : Sa * (double)expf(Ma - Mx);
        const double sb = M == -INFINITY ? 0.0 : S * (double)expf(M - Mx);
        M = Mx;
        S = sa + sb;
        mn = fminf(mna, mn);
    };
    float M = -INFINITY, mn = INFINITY;
    double S = 0.0;
    for (int64_t r = r0; r < r1; ++r) absorb(xs[r], M, S, mn);
    float PM = -INFINITY, Pmn = INFINITY;
    double PS = 0.0;
#if PSA_DECIDE_SCAN
    // exclusive prefix of this thread (the triples of threads 0 .. tid-1): a shuffle scan inside
    // the warp, the totals of the earlier warps folded in order
    const int lane = tid & 31, wid = tid >> 5;
    {
        float wM = M, wmn = mn;
        double wS = S;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float Mo = __shfl_up_sync(PSA_FULL, wM, o), mno = __shfl_up_sync(PSA_FULL, wmn, o);
            const double So = __shfl_up_sync(PSA_FULL, wS, o);
            if (lane >= o) combine(Mo, So, mno, wM, wS, wmn);
        }
        if (lane == 31) {
            tM[wid] = wM;
            tS[wid] = wS;
            tmn[wid] = wmn;
        }
        if (tid == 0) first_stop = ~0ull;
        float eM = __shfl_up_sync(PSA_FULL, wM, 1), emn = __shfl_up_sync(PSA_FULL, wmn, 1);
        double eS = __shfl_up_sync(PSA_FULL, wS, 1);
        if (lane == 0) {
            eM = -INFINITY;
            eS = 0.0;
            emn = INFINITY;
        }
        __syncthreads();
        for (int w = 0; w < wid; ++w) {
            float m2 = tM[w], n2v = tmn[w];
            double s2 = tS[w];
            combine(PM, PS, Pmn, m2, s2, n2v);
            PM = m2;
            PS = s2;
            Pmn = n2v;
        }
        combine(PM, PS, Pmn, eM, eS, emn);
        PM = eM;
        PS = eS;
        Pmn = emn;
    }
#else
    // exclusive prefix of this thread: the triples of threads 0 .. tid-1, combined in order
    tM[tid] = M;
    tS[tid] = S;
    tmn[tid] = mn;
    if (tid == 0) first_stop = ~0ull;
    __syncthreads();
    for (int t = 0; t < tid; ++t) {
        float m2 = tM[t], n2v = tmn[t];
        double s2 = tS[t];
        combine(PM, PS, Pmn, m2, s2, n2v);
        PM = m2;
        PS = s2;
        Pmn = n2v;
    }
#endif
    // walk again from the prefix
    int64_t stop_r = -1;
    for (int64_t r = r0; r < r1; ++r) {
        absorb(xs[r], PM, PS, Pmn);
        const bool boundary = b.m == 1 || ((r + 1) % b.m) == 0 || (r + 1 == limit);
        if (!boundary) continue;
        const int64_t nl = n - (r + 1);
        const double est = nl == 0 ? 1.0 : PS / fma((double)nl, (double)expf(Pmn - PM), PS);
        if (b.iest) b.iest[hb + r] = est;
        if (est > eps || r + 1 == limit) {
            stop_r = r;
            break;
        }
    }
    if (stop_r >= 0) atomicMin(&first_stop, (unsigned long long)stop_r);
    __syncthreads();
    if (first_stop == ~0ull) {  // no stop inside the candidate prefix (wl < limit): round 1 redoes the unit
        if (tid == 0 && atomicAdd(&b.dense_esc_mark[u], 1) == 0) b.dense_esc[atomicAdd(b.dense_esc_count, 1)] = u;
        return;
    }
    // The reported estimate at the stop rank, recomputed in fp64 over the processed ranks (the
    // reference's CoverageEstimator precision, engine.cpp:38-55): max, then sum exp(x - max) and min.
    const int64_t last = (int64_t)first_stop;  // every head stops (at the limit at the latest)
    const int64_t q1 = r1 < last + 1 ? r1 : last + 1;
    float pm = -INFINITY, pmn = INFINITY;
    for (int64_t r = r0; r < q1; ++r) {
        pm = fmaxf(pm, xs[r]);
        pmn = fminf(pmn, xs[r]);
    }
    tM[tid] = pm;
    tmn[tid] = pmn;
    __syncthreads();
    __shared__ float Mfin, mnfin;
    __shared__ double S64s;
    if (tid < 32) {  // warp 0 reduces the per-thread max / min
        float a = -INFINITY, c = INFINITY;
        for (int t = tid; t < kDecideThreads; t += 32) {
            a = fmaxf(a, tM[t]);
            c = fminf(c, tmn[t]);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            a = fmaxf(a, __shfl_xor_sync(PSA_FULL, a, o));
            c = fminf(c, __shfl_xor_sync(PSA_FULL, c, o));
        }
        if (tid == 0) {
            Mfin = a;
            mnfin = c;
        }
    }
    __syncthreads();
    double ps = 0.0;
    for (int64_t r = r0; r < q1; ++r) ps += exp((double)xs[r] - (double)Mfin);
    tS[tid] = ps;
    __syncthreads();
    if (tid < 32) {
        double a = 0.0;
        for (int t = tid; t < kDecideThreads; t += 32) a += tS[t];
        a = warp_sum_d(a);
        if (tid == 0) S64s = a;
    }
    __syncthreads();
    if (stop_r >= 0 && (unsigned long long)stop_r == first_stop) {
        const int64_t cb = stop_r + 1;
        const double S64 = S64s;
        const int64_t nl = n - cb;
        b.bp[qi] = cb;
        b.est[qi] = nl == 0 ? 1.0 : S64 / fma((double)nl, exp((double)mnfin - (double)Mfin), S64);
        b.term[qi] = b.topk > 0 ? (limit < n) : (cb < n);
        b.dense_thr[qi] = ks[stop_r];
    }
}

template <int G>
__device__ __forceinline__ void dense_v_unit(const PoolView& p, const BatchView& b, int u, int slice, int64_t e_begin,
                                             int64_t e_end, float (&so)[kDenseWarps][G][128],
                                             float (&som)[kDenseWarps][G], float (&sol)[kDenseWarps][G]);

template <int G>
__global__ void __launch_bounds__(kDenseWarps * 32) dense_v_kernel(PoolView p, BatchView b) {
    __shared__ float so[kDenseWarps][G][128];
    __shared__ float som[kDenseWarps][G], sol[kDenseWarps][G];
    const int S = dense_slices(b);
    const int32_t* list = dense_list(b);
    for (int item = blockIdx.x; item < dense_list_count(b) * S; item += gridDim.x) {
        const int u = list[item / S];
        const int64_t n = b.list_off[u + 1] - b.list_off[u];
        const int64_t e0 = (int64_t)(item % S) * b.dense_slice, e1 = e0 + b.dense_slice < n ? e0 + b.dense_slice : n;
        if (e0 < n && !dense_skip(b, u)) dense_v_unit<G>(p, b, u, item % S, e0, e1, so, som, sol);
        __syncthreads();
    }
}

template <int G>
__device__ __forceinline__ void dense_v_unit(const PoolView& p, const BatchView& b, int u, int slice, int64_t e_begin,
                                             int64_t e_end, float (&so)[kDenseWarps][G][128],
                                             float (&som)[kDenseWarps][G], float (&sol)[kDenseWarps][G]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const int gq = lane >> 2, tq = lane & 3;
    const int g = b.g;
    const int64_t off = b.list_off[u], n = b.list_off[u + 1] - off;
    const int T = p.T;
    const int64_t v_off = (int64_t)T * 128;
    uint64_t thr[G];
#pragma unroll
    for (int h = 0; h < G; ++h) thr[h] = h < g ? b.dense_thr[(size_t)u * g + h] : 0;
    auto mask_of = [&](int64_t e) {
        uint32_t m = 0;
#pragma unroll
        for (int h = 0; h < G; ++h)
            if (h < g && b.keys[off * g + (int64_t)h * n + e] <= thr[h]) m |= 1u << h;
        return m;
    };
    float Oreg[16], Mreg = -INFINITY, Lreg = 0.0f;
#pragma unroll
    for (int j = 0; j < 16; ++j) Oreg[j] = 0.0f;
    constexpr int kD = kDensePf;
    constexpr int64_t kW = kDenseWarps;
    // L2 prefetch of a union block's V tile ...
    auto prefetch = [&](int64_t ef, uint32_t mf, int32_t sf) {
        if (lane == 0 && mf && kv_resident(p, sf))
            prefetch_l2_bulk(kv_block<__nv_bfloat16>(p, sf) + v_off, (uint32_t)(T * 128 * 2));
#if PSA_DENSE_VPF
        // ... with the committed heads' token weights (lanes 0..g-1, one 64 B row each) and block
        // masses (lanes 8..8+g-1): both come from dense_k's write-back in HBM, and loading them
        // cold would put two DRAM round trips on every block's critical path
        if (mf) {
            const int hl = lane & 7;
            if (lane < 16 && hl < g && ((mf >> hl) & 1u)) {
                const int64_t row = off * g + (int64_t)hl * n + ef;
                prefetch_l2_line(lane < 8 ? (const void*)(b.dense_p + row * 16) : (const void*)(b.dense_la + row));
            }
        }
#endif
    };
    // one union block: V tile x the committed heads' weights (tensor cores), merged per head
    auto block = [&](int64_t e, int32_t slot, uint32_t mask) {
        const bool mine = tq < g && ((mask >> tq) & 1u);  // this lane's merge head (tq) is committed
        const float la = mine ? __ldg(b.dense_la + off * g + (int64_t)tq * n + e) : 0.0f;  // exp(la - M) weight
        const __nv_bfloat16* vblk = kv_block<__nv_bfloat16>(p, slot) + v_off;
        uint32_t vw[4][8];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int tok = 2 * tq + (r & 1) + (r >> 1) * 8;
            const int row = tok < T ? tok : T - 1;
            const uint4* pv = reinterpret_cast<const uint4*>(vblk + (size_t)row * 128 + 16 * gq);
            const uint4 x0 = __ldg(pv), x1 = __ldg(pv + 1);
            vw[r][0] = x0.x; vw[r][1] = x0.y; vw[r][2] = x0.z; vw[r][3] = x0.w;
            vw[r][4] = x1.x; vw[r][5] = x1.y; vw[r][6] = x1.z; vw[r][7] = x1.w;
        }
        // B columns = (head, split): weights p_t of head hb (2-term bf16 split), zero if not committed
        const int hbq = gq >> 1, sb = gq & 1;
        const bool hon = hbq < g && (mask >> hbq) & 1u;
        uint32_t bfr[2];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            float2 wv = make_float2(0.0f, 0.0f);
            if (hon) wv = *reinterpret_cast<const float2*>(b.dense_p + ((off * g + (int64_t)hbq * n) + e) * 16 + 2 * tq + 8 * hf);
            bfr[hf] = pack_bf16x2_split(wv.x, wv.y, sb);
        }
        float ob[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
            mma_bf16_16816(c0, c1, c2, c3, __byte_perm(vw[0][i], vw[1][i], 0x5410), __byte_perm(vw[0][i], vw[1][i], 0x7632),
                           __byte_perm(vw[2][i], vw[3][i], 0x5410), __byte_perm(vw[2][i], vw[3][i], 0x7632), bfr[0], bfr[1]);
            ob[2 * i] = c0 + c1;
            ob[2 * i + 1] = c2 + c3;
        }
        if (mine) {  // block weight exp(la - M), sum_t p_t = 1
            const float mnew = fmaxf(Mreg, la);
            const float a = expf(Mreg - mnew);
            const float cc = expf(la - mnew);
#pragma unroll
            for (int j = 0; j < 16; ++j) Oreg[j] = Oreg[j] * a + ob[j] * cc;
            Lreg = Lreg * a + cc;
            Mreg = mnew;
        }
    };
    int64_t e = e_begin + warp;
    int64_t most = 0;  // the heads' processed counts: a sparse union takes the windowed walk
    for (int h = 0; h < g; ++h) most = b.bp[(int64_t)u * g + h] > most ? b.bp[(int64_t)u * g + h] : most;
    if (4 * most >= n) {
        // membership masks and slots run kDensePf iterations ahead of the V reads: the L2 prefetch (same
        // distance) touches only blocks of the union, so no V byte outside it is fetched
        auto slot_or = [&](int64_t f) { return f < e_end ? b.slots[off + f] : 0; };
        auto mask_or = [&](int64_t f) { return f < e_end ? mask_of(f) : 0u; };
        uint32_t mq[kD + 1];
        int32_t sq[kD + 1];
#pragma unroll
        for (int i = 0; i <= kD; ++i) {
            mq[i] = mask_or(e + i * kW);
            sq[i] = slot_or(e + i * kW);
        }
        for (; e < e_end; e += kW) {
            const uint32_t mask = mq[0];
            const int32_t slot = sq[0];
            if (mq[kD]) prefetch(e + kD * kW, mq[kD], sq[kD]);  // block e + kD*W, kD iterations ahead
#pragma unroll
            for (int i = 0; i < kD; ++i) {
                mq[i] = mq[i + 1];
                sq[i] = sq[i + 1];
            }
            mq[kD] = mask_or(e + (kD + 1) * kW);
            sq[kD] = slot_or(e + (kD + 1) * kW);
            if (mask) block(e, slot, mask);
        }
    } else {
        // sparse union: the warp's positions tested 32 at a time (one lane each), a ballot gives the
        // window's union blocks, the prefetch runs kDensePf union blocks ahead across windows
        constexpr int64_t kWin = 32 * kW;
        auto window = [&](int64_t wb, uint32_t& bal, uint32_t& ml, int32_t& sl) {
            const int64_t f = wb + kW * lane;
            ml = f < e_end ? mask_of(f) : 0u;
            sl = ml ? b.slots[off + f] : 0;
            bal = __ballot_sync(PSA_FULL, ml != 0u);
        };
        uint32_t bc, bn, mc, mn;
        int32_t sc, sn;
        window(e, bc, mc, sc);
        window(e + kWin, bn, mn, sn);
        for (int64_t wb = e; wb < e_end; wb += kWin) {
            const uint64_t comb = (uint64_t)bc | ((uint64_t)bn << 32);
            uint32_t rem = bc;
            while (rem) {
                const int i = __ffs(rem) - 1;
                rem &= rem - 1;
                uint64_t ahead = comb & ~((2ull << i) - 1ull);
#pragma unroll
                for (int k = 1; k < kD; ++k) ahead &= ahead - 1;
                if (ahead) {
                    const int j = __ffsll((long long)ahead) - 1;
                    const uint32_t mf = __shfl_sync(PSA_FULL, j < 32 ? mc : mn, j & 31);
                    const int32_t sf = __shfl_sync(PSA_FULL, j < 32 ? sc : sn, j & 31);
                    prefetch(wb + kW * j, mf, sf);
                }
                block(wb + kW * i, __shfl_sync(PSA_FULL, sc, i), __shfl_sync(PSA_FULL, mc, i));
            }
            bc = bn;
            mc = mn;
            sc = sn;
            window(wb + 2 * kWin, bn, mn, sn);
        }
    }
    if (tq < G) {
#pragma unroll
        for (int j = 0; j < 16; ++j) so[warp][tq][16 * gq + j] = Oreg[j];
        if (gq == 0) {
            som[warp][tq] = Mreg;
            sol[warp][tq] = Lreg;
        }
    }
    __syncthreads();
    for (int h = 0; h < g; ++h) {
        float Mt = -INFINITY;
#pragma unroll
        for (int w = 0; w < kDenseWarps; ++w) Mt = fmaxf(Mt, som[w][h]);
        float Lt = 0.0f, sc[kDenseWarps];
#pragma unroll
        for (int w = 0; w < kDenseWarps; ++w) {
            sc[w] = sol[w][h] > 0.0f ? expf(som[w][h] - Mt) : 0.0f;
            Lt += sol[w][h] * sc[w];
        }
        // this slice's partial state of head h: (max, sum, unnormalised output), merged by dense_merge_kernel
        const int64_t qi = (int64_t)u * g + h;
        float* part = b.dense_part + (qi * dense_slices(b) + slice) * kDensePart;
        for (int i = tid; i < 128; i += kDenseWarps * 32) {
            float o = 0.0f;
#pragma unroll
            for (int w = 0; w < kDenseWarps; ++w) o += sc[w] > 0.0f ? so[w][h][i] * sc[w] : 0.0f;
            part[i] = o;
        }
        if (tid == 0) {
            part[128] = Mt;
            part[129] = Lt;
        }
    }
}

// Round 0's candidate prefix of every (handed-over unit, head): a key threshold tau with between
// dense_sel_ranks / 2 and 2 * dense_sel_ranks keys <= tau (a prefix of the head's rank order, since
// keys order the ranking), found by histogram refinement in key space between the head's min and
// max key (from the score kernel). ~0 (every block) for short lists, partial mode off, and flat
// units (criticality within dense_early nats over the first tranche: they stop near the end of
// their lists). Also clears the unit's escalation mark.
constexpr int kSelBins = 1024;
constexpr int kSelThreads = 256;
__global__ void __launch_bounds__(kSelThreads) dense_select_kernel(BatchView b) {
    __shared__ uint32_t hist[kSelBins];
    __shared__ unsigned wsum[kSelThreads / 32];
    __shared__ int s_bstar;
    __shared__ unsigned s_excl;
    const int tid = threadIdx.x, lane = tid & 31;
    const uint64_t pm = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);
    const int64_t N = b.dense_sel_ranks;
    for (int item = blockIdx.x; item < *b.dense_count * b.g; item += gridDim.x) {
        const int u = b.dense_flag[item / b.g], h = item % b.g;
        const int64_t off = b.list_off[u], n = b.list_off[u + 1] - off;
        const int64_t qi = (int64_t)u * b.g + h;
        if (h == 0 && tid == 0) b.dense_esc_mark[u] = 0;
        bool full = N <= 0 || n <= 2 * N;
        if (!full && b.dense_early > 0.0f && b.ft_keys) {
            for (int h2 = 0; h2 < b.g; ++h2) {
                const int64_t q2 = (int64_t)u * b.g + h2;
                if (b.ft_count[q2] >= kDenseHandover) {
                    const double s0 = key_score(b.ft_keys[q2 * kFirstCap], pm);
                    const double s1 = key_score(b.ft_keys[q2 * kFirstCap + kDenseHandover - 1], pm);
                    full = full || s0 - s1 < (double)b.dense_early;
                }
            }
        }
        if (full) {
            if (tid == 0) b.dense_sel[qi] = ~0ull;
            continue;
        }
        const uint64_t* keys = b.keys + off * b.g + (int64_t)h * n;
        uint64_t lo = 0, hi = ~0ull;
        if (b.kminmax) {
            lo = b.kminmax[qi];
            hi = b.kminmax[qi + b.kmm_stride];
        }
        uint64_t tau = ~0ull;
        unsigned before = 0, need = (unsigned)N;
        for (int it = 0; it < 8; ++it) {
            const uint64_t span = hi - lo;
            const int bits = span ? 64 - __clzll((long long)span) : 0;
            constexpr int kLog = 10;  // log2(kSelBins)
            const int sh = bits > kLog ? bits - kLog : 0;
            for (int i = tid; i < kSelBins; i += kSelThreads) hist[i] = 0;
            __syncthreads();
            scan_keys(keys, n, cta_team(), [&](uint64_t k) {
                if (k >= lo && k <= hi) atomicAdd(&hist[(k - lo) >> sh], 1u);
            });
            __syncthreads();
            constexpr int per = kSelBins / kSelThreads;
            unsigned loc = 0;
#pragma unroll
            for (int j = 0; j < per; ++j) loc += hist[tid * per + j];
            unsigned inc = loc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(PSA_FULL, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) wsum[tid >> 5] = inc;
            __syncthreads();
            unsigned cum = inc - loc;
            for (int w = 0; w < (tid >> 5); ++w) cum += wsum[w];
            if (cum < need && need <= cum + loc) {
#pragma unroll 1
                for (int j = 0; j < per; ++j) {
                    const unsigned c = hist[tid * per + j];
                    if (need <= cum + c) {
                        s_bstar = tid * per + j;
                        s_excl = cum;
                        break;
                    }
                    cum += c;
                }
            }
            __syncthreads();
            const int bs = s_bstar;
            const unsigned ex = s_excl, c = hist[bs];
            const uint64_t width_m1 = (sh >= 64) ? ~0ull : ((1ull << sh) - 1ull);
            const uint64_t bin_lo = lo + ((uint64_t)bs << sh);
            const uint64_t bin_hi = (hi - bin_lo <= width_m1) ? hi : bin_lo + width_m1;
            __syncthreads();  // (s_bstar / hist reused by the next pass)
            if (before + ex + c <= (unsigned)(2 * N)) {
                tau = bin_hi;
                break;
            }
            if (before + ex >= (unsigned)(N / 2)) {
                tau = bin_lo - 1;  // the bins below bs (bin_lo > lo: before < N / 2 keys lie below lo)
                break;
            }
            before += ex;
            need -= ex;
            lo = bin_lo;
            hi = bin_hi;
        }
        if (tid == 0) b.dense_sel[qi] = tau;
    }
}

// Per (handed-over unit, head): the slices' partial states merged (finalize, attention.hpp:104-110).
__global__ void __launch_bounds__(128) dense_merge_kernel(BatchView b) {
    const int S = dense_slices(b);
    const int32_t* list = dense_list(b);
    for (int item = blockIdx.x; item < dense_list_count(b) * b.g; item += gridDim.x) {
        const int u = list[item / b.g], h = item % b.g;
        if (dense_skip(b, u)) continue;
        const int64_t n = b.list_off[u + 1] - b.list_off[u];
        const int ns = (int)((n + b.dense_slice - 1) / b.dense_slice);
        const int64_t qi = (int64_t)u * b.g + h;
        const float* part = b.dense_part + qi * S * kDensePart;
        float Mt = -INFINITY;
        for (int s = 0; s < ns; ++s)
            if (part[s * kDensePart + 129] > 0.0f) Mt = fmaxf(Mt, part[s * kDensePart + 128]);
        float Lt = 0.0f, o = 0.0f;
        for (int s = 0; s < ns; ++s) {
            const float L = part[s * kDensePart + 129];
            if (!(L > 0.0f)) continue;
            const float c = expf(part[s * kDensePart + 128] - Mt);
            Lt += L * c;
            o += part[s * kDensePart + threadIdx.x] * c;
        }
        b.out[qi * 128 + threadIdx.x] = o / Lt;
    }
}

bool dense_supported(const PoolView& p, const BatchView& b) {
    return p.dtype == 1 && b.d == 128 && p.T <= 16 && b.g >= 2 && b.g <= 4 && !b.has_oracle && b.dense_flag &&
           b.max_n <= kDenseMaxBlocks;
}

static int dense_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Persistent grids over the hand-over list (sized to the SMs: no cost when the list is empty).
static void launch_dense_round(const PoolView& p, const BatchView& b, cudaStream_t st);
static int g_dense_sel = 1024;
void set_dense_partial(int ranks) { g_dense_sel = ranks; }

void launch_dense(const PoolView& p, const BatchView& b_in, cudaStream_t st) {
    // a whole list per work item when the batch alone fills the GPU, else kDenseSlice positions
    BatchView b = b_in;
    b.dense_slice = b.n_units >= 2 * dense_sms() ? (b.max_n > 0 ? b.max_n : 1) : kDenseSlice;
    b.dense_sel_ranks = g_dense_sel;
    b.dense_round = 0;
    {
        const int items = b.n_units * b.g < 2 * dense_sms() ? b.n_units * b.g : 2 * dense_sms();
        dense_select_kernel<<<items, kSelThreads, 0, st>>>(b);
    }
    launch_dense_round(p, b, st);
    b.dense_round = 1;  // units a head escalated: the rest of the K pass, full decide, V
    launch_dense_round(p, b, st);
}

static void launch_dense_round(const PoolView& p, const BatchView& b, cudaStream_t st) {
    const int G = b.g <= 2 ? 2 : 4;
    const int64_t slices = (b.max_n + b.dense_slice - 1) / b.dense_slice;
    const int units = b.n_units * slices < 2 * dense_sms() ? (int)(b.n_units * slices) : 2 * dense_sms();
    if (G == 2) dense_k_kernel<2><<<units, kDenseWarps * 32, 0, st>>>(p, b);
    else dense_k_kernel<4><<<units, kDenseWarps * 32, 0, st>>>(p, b);
    int n2 = 1;
    while (n2 < b.max_n) n2 <<= 1;
    const size_t smem = (size_t)n2 * 12;  // sorted keys + masses in rank order
    const int per_sm = smem <= 70 * 1024 ? 3 : (smem <= 110 * 1024 ? 2 : 1);
    const int heads = b.n_units * b.g < per_sm * dense_sms() ? b.n_units * b.g : per_sm * dense_sms();
    cudaFuncSetAttribute(dense_decide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dense_decide_kernel<<<heads, kDecideThreads, smem, st>>>(b);
    if (G == 2) dense_v_kernel<2><<<units, kDenseWarps * 32, 0, st>>>(p, b);
    else dense_v_kernel<4><<<units, kDenseWarps * 32, 0, st>>>(p, b);
    dense_merge_kernel<<<heads, 128, 0, st>>>(b);
}

}  // namespace psa
