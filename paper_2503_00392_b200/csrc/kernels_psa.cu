// kernels_psa.cu — K3 ordering (lazy tranche selection) fused with K4/K5, the
// persistent progressive attention kernel (sm_100a).
#include <cuda_bf16.h>
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"
#include "mma.cuh"
#include "psa_order.cuh"

#include <type_traits>

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
constexpr int kBpw = kChunk / kPsaWarps;
constexpr int kTCap = 1024;
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
    SelScratch sel;
    int commit, fin;
    double est, acc;
    float m[kPsaWarps], l[kPsaWarps];
};

// ---- tensor-core K pass (bf16 pools, d = 128, 16-token blocks) -------------
// S[token][c] = sum_k K[token][k] * Qs[k][c] with Qs = [q1 q2 q3 0..] the exact
// 3-term bf16 split of the fp32 query (q1 = bf16(q), q2 = bf16(q - q1),
// q3 = bf16(q - q1 - q2), q1 + q2 + q3 == q): bf16 x bf16 products are exact in
// the fp32 accumulator, so one mma.sync.m16n8k16 per 16 dims replaces 16x16
// FFMAs, 64 bf16->fp32 conversions and the cross-lane reduction. Dims are
// permuted (the sum over k is order-free) so thread (g = lane/4, t = lane%4)
// owns dims [32t, 32t+32) of token rows g and g+8: 8 x 128-bit loads per block.
// B fragments of the split query for the 8 k-steps: qb[s][0] = (k 2t, 2t+1), qb[s][1] = (k 2t+8, 2t+9), col g.
__device__ __forceinline__ void build_q_frags(const float* __restrict__ qrow, int lane, uint32_t (&qb)[8][2]) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int st = 0; st < 8; ++st) {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            uint32_t packed = 0;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float x = qrow[32 * t + 4 * st + 2 * hf + e];
                const float x1 = __bfloat162float(__float2bfloat16_rn(x));
                const float r1 = x - x1;
                const float x2 = __bfloat162float(__float2bfloat16_rn(r1));
                const float r2 = r1 - x2;
                const float part = g == 0 ? x : (g == 1 ? r1 : (g == 2 ? r2 : 0.0f));
                packed |= bf16_bits(part) << (16 * e);
            }
            qb[st][hf] = packed;
        }
    }
}

// Scores of one 16-token block: returns (token g, token g+8) on lanes with t < 2.
__device__ __forceinline__ void block_scores_mma(const __nv_bfloat16* __restrict__ kblk, int T, int lane,
                                                 const uint32_t (&qb)[8][2], float& s_lo, float& s_hi) {
    const int g = lane >> 2, t = lane & 3;
    const int r0 = g < T ? g : T - 1, r1 = (g + 8) < T ? (g + 8) : T - 1;
    const uint4* p0 = reinterpret_cast<const uint4*>(kblk + (size_t)r0 * 128 + 32 * t);
    const uint4* p1 = reinterpret_cast<const uint4*>(kblk + (size_t)r1 * 128 + 32 * t);
    uint32_t w0[16], w1[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint4 a = __ldg(p0 + i), b = __ldg(p1 + i);
        w0[4 * i] = a.x; w0[4 * i + 1] = a.y; w0[4 * i + 2] = a.z; w0[4 * i + 3] = a.w;
        w1[4 * i] = b.x; w1[4 * i + 1] = b.y; w1[4 * i + 2] = b.z; w1[4 * i + 3] = b.w;
    }
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
#pragma unroll
    for (int st = 0; st < 8; ++st)
        mma_bf16_16816(c0, c1, c2, c3, w0[2 * st], w1[2 * st], w0[2 * st + 1], w1[2 * st + 1], qb[st][0], qb[st][1]);
    // columns 2t, 2t+1 are split terms: t=0 holds q1,q2 and t=1 holds q3 -> sum across the pair
    float lo = c0 + c1, hi = c2 + c3;
    lo += __shfl_xor_sync(PSA_FULL, lo, 1);
    hi += __shfl_xor_sync(PSA_FULL, hi, 1);
    s_lo = lo;
    s_hi = hi;
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
    constexpr int TSH = TOK <= 32 ? 5 - Log2<TOK <= 32 ? TOK : 32>::v : 0;  // lanes per token after reduce-scatter = 1 << TSH
    const int my_tok = lane >> TSH;
    const uint64_t pmask = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);

    float q[DPL];
    load_row<DPL>(b.q + ((size_t)u * b.g + h) * d + base, full, lim, q);
    constexpr bool kMma = std::is_same<KV, __nv_bfloat16>::value && DPL == 4 && TOK == 16 && FULL;
    uint32_t qb[8][2];
    if constexpr (kMma) build_q_frags(b.q + ((size_t)u * b.g + h) * d, lane, qb);

    float M = -INFINITY, L = 0.0f, O[DPL];  // warp-local online-softmax state
#pragma unroll
    for (int j = 0; j < DPL; ++j) O[j] = 0.0f;
    // coverage state (warp 0, lane-uniform): acc = log-sum-exp (oracle masses) or the running
    // max M of the fast decide, whose running sum S is ssum
    double acc = -INFINITY, mn = INFINITY, ssum = 0.0;

    const double* omass = b.has_oracle ? (b.omass + hb) : nullptr;
    const int64_t v_off = (int64_t)p.T * d;
    const int T = p.T;

    int64_t tr0 = 0;  // global rank of s.tb[0]
    int tc = 0;       // ranks in the current tranche
    uint64_t last = 0;
    for (int64_t cb = 0;;) {
        if (cb >= tr0 + tc) {  // ---- ORDER: next tranche ----
            tr0 += tc;
            tc = select_tranche(s.sel, s.tb, kTCap, s.hist, kBins, keys, n, last, tr0 == 0, tr0 == 0 ? kFirstTranche : kTCap,
                                cta_team(), b.kminmax ? b.kminmax + (size_t)u * b.g + h : nullptr,
                                b.kmm_stride);
            last = s.tb[tc - 1];
            fill_tranche(s.tb, tc, pmask, b.rpos + hb + tr0, b.slots + off, p.ntok, s.tslot, s.tntok, cta_team());
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
            if constexpr (kMma) {
                float slo, shi;
                block_scores_mma(kv_block<KV>(p, slot), T, lane, qb, slo, shi);
                const int g8 = lane >> 2;
                slo = (g8 < nt) ? slo * fscale : -INFINITY;
                shi = (g8 + 8 < nt) ? shi * fscale : -INFINITY;
                float mb = fmaxf(slo, shi);
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) mb = fmaxf(mb, __shfl_xor_sync(PSA_FULL, mb, o));
                const float wlo = (g8 < nt) ? expf(slo - mb) : 0.0f;
                const float whi = (g8 + 8 < nt) ? expf(shi - mb) : 0.0f;
                float lb = wlo + whi;
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) lb += __shfl_xor_sync(PSA_FULL, lb, o);
                if ((lane & 3) == 0) {
                    s.w[warp][j][g8] = wlo;
                    s.w[warp][j][g8 + 8] = whi;
                }
                if (lane == 0) {
                    s.mb[warp][j] = mb;
                    s.lb[warp][j] = lb;
                    s.la[rl] = mb + logf(lb);
                }
                continue;
            }
            if constexpr (TOK > 32) {
                // long blocks (32 < T <= TOK): 32-token chunks, each scored like a 32-token block,
                // folded into the block's (max, exp-sum) online; the token weights end up relative
                // to the block max (attention.hpp:55-73 over all the block's tokens)
                const KV* kp = kv_block<KV>(p, slot) + base;
                float mbk = -INFINITY, lbk = 0.0f, wc[TOK / 32], mc[TOK / 32];
#pragma unroll
                for (int c = 0; c < TOK / 32; ++c) {
                    wc[c] = 0.0f;
                    mc[c] = -INFINITY;
                    if (c * 32 >= nt) continue;
                    float part[32];
#pragma unroll
                    for (int t = 0; t < 32; ++t) {
                        const int row = c * 32 + t < T ? c * 32 + t : T - 1;
                        float kr[DPL];
                        load_row<DPL>(kp + (size_t)row * d, full, lim, kr);
                        float a = 0.0f;
#pragma unroll
                        for (int jj = 0; jj < DPL; ++jj) a = fmaf(q[jj], kr[jj], a);
                        part[t] = a;
                    }
                    float sc = reduce_scatter<32>(part, lane) * fscale;  // token c*32 + lane
                    sc = c * 32 + lane < nt ? sc : -INFINITY;
                    const float m = warp_max(sc);
                    const float w = c * 32 + lane < nt ? expf(sc - m) : 0.0f;
                    const float l = warp_sum(w);
                    const float mnew = fmaxf(mbk, m);
                    lbk = lbk * expf(mbk - mnew) + l * expf(m - mnew);
                    mbk = mnew;
                    wc[c] = w;
                    mc[c] = m;
                }
#pragma unroll
                for (int c = 0; c < TOK / 32; ++c)
                    if (c * 32 < nt) s.w[warp][j][c * 32 + lane] = wc[c] * expf(mc[c] - mbk);
                if (lane == 0) {
                    s.mb[warp][j] = mbk;
                    s.lb[warp][j] = lbk;
                    s.la[rl] = mbk + logf(lbk);
                }
                continue;
            }
            const KV* kp = kv_block<KV>(p, slot) + base;
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
            double x = -INFINITY;
            if (lane < cnt) x = omass ? omass[s.tb[ci + lane] & pmask] : (double)s.la[lane];
            Decision dc;
            if (omass) {
                dc = decide_chunk(x, cnt, cb, n, limit, b.m, eps, acc, mn, b.iest ? b.iest + hb : nullptr);
            } else if (!PSA_DECIDE_FAST || !decide_chunk_fast((float)x, cnt, cb, n, limit, b.m, eps, acc, ssum, mn,
                                          b.iest ? b.iest + hb : nullptr, dc)) {
                acc = ssum > 0.0 ? acc + log(ssum) : -INFINITY;  // fp64 fallback (see kernels_gqa.cu)
                dc = decide_chunk(x, cnt, cb, n, limit, b.m, eps, acc, mn, b.iest ? b.iest + hb : nullptr);
                ssum = 1.0;
            }
            if (lane == 0) {
                s.commit = dc.commit;
                s.fin = dc.fin;
                s.est = dc.est;
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
            const KV* vp = kv_block<KV>(p, slot) + v_off + base;
            float ob[DPL];
#pragma unroll
            for (int jj = 0; jj < DPL; ++jj) ob[jj] = 0.0f;
            if constexpr (TOK > 32) {
                for (int t = 0; t < nt; ++t) {
                    const float wt = s.w[warp][j][t];
                    float vr[DPL];
                    load_row<DPL>(vp + (size_t)t * d, full, lim, vr);
#pragma unroll
                    for (int jj = 0; jj < DPL; ++jj) ob[jj] = fmaf(wt, vr[jj], ob[jj]);
                }
            } else if (T == TOK) {
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

static int g_psa_choice = 0;
void set_psa_kernel_choice(int choice) { g_psa_choice = choice; }
int psa_kernel_choice() { return g_psa_choice; }

static int g_dense_mode = 0;
void set_dense_mode(int mode) { g_dense_mode = mode; }
static float g_dense_early = 2.0f;
void set_dense_early(float nats) { g_dense_early = nats; }

int launch_psa(const PoolView& p, const BatchView& b, cudaStream_t st) {
    if (g_psa_choice != 1 && gqa_supported(p, b)) {  // auto = GQA-group kernel where supported
        BatchView v = b;
        const bool dense = g_dense_mode == 0 && dense_supported(p, b);
        if (!dense) v.dense_flag = nullptr;
        v.dense_early = g_dense_early;
        if (dense) {
            cudaMemsetAsync(v.dense_count, 0, 4, st);
            cudaMemsetAsync(v.dense_esc_count, 0, 4, st);
        }
        const int n = launch_gqa(p, v, st);
        if (!dense) return n;
        launch_dense(p, v, st);  // units the GQA kernel handed over (others exit at once)
        return n + 9;  // select + two rounds of K / decide / V / merge
    }
    const int nq = b.n_units * b.g;
    if (p.dtype == 0) {
        if (tok_for(p.T) == 16) launch_psa_t<float, 16>(p, b, nq, st);
        else if (tok_for(p.T) == 32) launch_psa_t<float, 32>(p, b, nq, st);
        else launch_psa_t<float, kMaxBlockTokens>(p, b, nq, st);
    } else {
        if (tok_for(p.T) == 16) launch_psa_t<__nv_bfloat16, 16>(p, b, nq, st);
        else if (tok_for(p.T) == 32) launch_psa_t<__nv_bfloat16, 32>(p, b, nq, st);
        else launch_psa_t<__nv_bfloat16, kMaxBlockTokens>(p, b, nq, st);
    }
    return 1;
}

}  // namespace psa
