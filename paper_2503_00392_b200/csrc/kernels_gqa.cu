// kernels_gqa.cu — progressive attention for a whole GQA group in one CTA (sm_100a).
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
// psa_gqa_kernel: one CTA (8 warps) per (request, layer, kv-head) unit running
// the g q-heads of its GQA group together (psa_attention_multi_head, reference
// engine.cpp:240-260: every head keeps its OWN ranking and stop point, SPEC D6).
//
// Each round, every live head h contributes its next chunk of <= CH ranks (64 on the
// tensor-core path with the dense hand-over, else 32); the chunks are merged into a
// union U (hash on list position) so a block ranked by several heads is read ONCE:
//   1. ORDER   the first tranche comes from first_tranche_kernel; later tranches
//              (32-rank variant only) by bucket select + bitonic (psa_order.cuh);
//   2. K pass  each block of U: its K rows are loaded once and scored for all g
//              heads (fp32 q.k*scale, block max / exp-sum per head);
//   3. decide  warp h runs head h's coverage scan over its chunk in 32-rank pieces
//              (decide_chunk_fast, fp64 fallback), all heads in parallel;
//              committed (block, head) pairs are marked;
//   4. V pass  each block of U committed by >= 1 head: V rows loaded once,
//              accumulated into every committing head's online-softmax state.
// With correlated heads (the usual GQA case) U is ~1 chunk, so K/V bytes and
// the bf16->fp32 conversions are ~1/g of the per-head kernel's. A head reaching
// kDenseHandover ranks hands the unit over to the dense kernels (kernels_dense.cu).
// =============================================================================
constexpr int kGTCap = kFirstCap;  // tranche capacity per head
#ifndef PSA_KUNROLL
#define PSA_KUNROLL 1
#endif
#ifndef PSA_VUNROLL
#define PSA_VUNROLL 1
#endif
constexpr int kKUnroll = PSA_KUNROLL, kVUnroll = PSA_VUNROLL;  // K / V pass loop unroll (build knobs)
constexpr int kHash = 512;    // pos -> U index (>= 2 * G * kChunk)
constexpr int kGBins = 1024;  // bucket-select bins per head team

// CH: ranks per head per round. CH = 64 (tensor-core path with the dense hand-over) halves the
// rounds; it has no later-tranche selection (a head that exhausts its first tranche is handed
// over) and its per-warp output accumulators alias the token weights (both fit 2 CTAs / SM).
template <int TOK, int G, int CH = kChunk>
struct GqaSmem {
    static constexpr bool kWide = CH > kChunk;
    uint64_t tb[G][kGTCap];
    int32_t tslot[G][kGTCap];
    uint8_t tntok[G][kGTCap];
    uint32_t hist[kWide ? 1 : G][kWide ? 1 : kGBins];
    union alignas(16) {
        float w[G * CH][G][TOK];  // per (U entry, head) token weights exp(s - m)
        float o_alias[kWide ? kPsaWarps : 1][G][128];
    } wo;
    float mb[G * CH][G], lb[G * CH][G];  // block max and exp-sum (log_as = mb + log lb)
    float o_sep[kWide ? 1 : kPsaWarps][kWide ? 1 : G][kWide ? 1 : 128];  // per-warp, per-head output accumulators
    __device__ __forceinline__ float* o(int w_, int h_) { return kWide ? wo.o_alias[w_][h_] : o_sep[w_][h_]; }
    float om[kPsaWarps][G], ol[kPsaWarps][G];
    int32_t uslot[G * CH];
    int32_t upos[G * CH];
    uint8_t untok[G * CH];
    uint32_t umask[G * CH];
    int16_t cidx[G][CH];
    int32_t hkey[kHash];
    int32_t hfirst[kHash];
    int16_t hval[kHash];
    alignas(16) int wcnt[kPsaWarps];  // (16-byte aligned: the prefix loop reads it with 128-bit loads)
    int64_t tr0[G], cb[G];
    uint64_t last[G];
    double est[G], acc[G], mn[G], ssum[G];  // acc: log-sum-exp (oracle masses) or running max M (fast decide)
    int tc[G], cnt[G], commit[G], fin[G], live[G];
    int ucount, nlive;
    SelScratch sel[G];
};

#ifdef PSA_GQA_PROF
// Development-only phase timer (make PROF=1): SM cycles per phase summed over CTAs.
__device__ unsigned long long g_gqa_prof[12];
#define GQA_MARK(k)                                \
    do {                                           \
        if (tid == 0) {                            \
            const long long t_ = clock64();        \
            pc[k] += t_ - pt;                      \
            pt = t_;                               \
        }                                          \
    } while (0)
#else
#define GQA_MARK(k) \
    do {            \
    } while (0)
#endif

template <typename KV, int DPL, int TOK, bool FULL, int G, int CH>
__global__ void __launch_bounds__(kPsaThreads, 2) psa_gqa_kernel(PoolView p, BatchView b) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GqaSmem<TOK, G, CH>& s = *reinterpret_cast<GqaSmem<TOK, G, CH>*>(smem_raw);
    constexpr bool kWide = GqaSmem<TOK, G, CH>::kWide;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int u = blockIdx.x;
    const int g = b.g;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int64_t limit = b.topk > 0 ? (b.topk < n ? b.topk : n) : n;
    const double eps = b.topk > 0 ? 1.0 : b.eps;
    const int d = FULL ? 32 * DPL : b.d;
    const int base = lane * DPL;
    const int lim = d - base;
    constexpr bool full = FULL;
    const float fscale = (float)b.scale;
    constexpr int TSH = 5 - Log2<TOK>::v;
    const int my_tok = lane >> TSH;
    const uint64_t pmask = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);
    const int T = p.T;
    const int64_t v_off = (int64_t)T * d;
#ifdef PSA_GQA_PROF
    long long pt = clock64(), pc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif

    float q[G][DPL];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        if (h < g)
            load_row<DPL>(b.q + ((size_t)u * g + h) * d + base, full, lim, q[h]);
        else
#pragma unroll
            for (int j = 0; j < DPL; ++j) q[h][j] = 0.0f;
    }
    // Tensor-core K pass (bf16 pools, d = 128, blocks <= 16 tokens): columns of the
    // n8 tiles are (head, split) pairs, 4 per head (3 exact bf16 split terms + 0), so
    // ONE set of 8 x NT mma.sync scores a block for the whole group.
    constexpr bool kMma = std::is_same<KV, __nv_bfloat16>::value && DPL == 4 && TOK == 16 && FULL;
    constexpr int NT = (G * 4 + 7) / 8;  // n8 tiles
    uint32_t qg[8][NT][2];
    if constexpr (kMma) {
        const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
        for (int tile = 0; tile < NT; ++tile) {
            const int hq = tile * 2 + (gq >> 2), sp = gq & 3;
            const float* qrow = b.q + ((size_t)u * g + (hq < g ? hq : 0)) * d;
#pragma unroll
            for (int st = 0; st < 8; ++st)
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t packed = 0;
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        const float x = hq < g ? bf16_split(qrow[32 * tq + 4 * st + 2 * hf + e2], sp) : 0.0f;
                        packed |= bf16_bits(x) << (16 * e2);
                    }
                    qg[st][tile][hf] = packed;
                }
        }
    }
    float Oreg[16], Mreg = -INFINITY, Lreg = 0.0f;  // tensor-core V pass: head lane%4, dims [16*(lane/4), +16)
#pragma unroll
    for (int j = 0; j < 16; ++j) Oreg[j] = 0.0f;
    if (tid < G) {
        s.tr0[tid] = 0;
        s.cb[tid] = 0;
        s.tc[tid] = 0;
        s.last[tid] = 0;
        s.acc[tid] = -INFINITY;
        s.ssum[tid] = 0.0;
        s.mn[tid] = INFINITY;
        s.live[tid] = tid < g;
        s.est[tid] = 0.0;
    }
    for (int i = tid; i < kPsaWarps * G; i += kPsaThreads) {
        (&s.om[0][0])[i] = -INFINITY;
        (&s.ol[0][0])[i] = 0.0f;
    }
    if constexpr (!GqaSmem<TOK, G, CH>::kWide)
        for (int i = tid; i < kPsaWarps * G * 128; i += kPsaThreads) (&s.o_sep[0][0][0])[i] = 0.0f;
    __syncthreads();
    GQA_MARK(0);

    for (;;) {
        // ---- 1. ORDER: refill the tranche of every live head that consumed it; the
        //      heads' selections run concurrently, one team of kPsaWarps/G warps each ----
        {
            constexpr int W = kPsaWarps / G;
            const int h = warp / W;
            const Team tm{tid - h * W * 32, W * 32, 1 + h};
            const bool need = s.live[h] && s.cb[h] >= s.tr0[h] + s.tc[h];
            int tc = 0;
            int64_t t0 = 0;
            if (need && b.ft_keys && s.tr0[h] + s.tc[h] == 0) {
                // first tranche selected up front (first_tranche_kernel): copy it in
                const size_t qi = (size_t)u * g + h;
                tc = b.ft_count[qi];
                for (int i = tm.tid; i < tc; i += tm.size) {
                    s.tb[h][i] = b.ft_keys[qi * kGTCap + i];
                    s.tslot[h][i] = b.ft_slot[qi * kGTCap + i];
                    s.tntok[h][i] = b.ft_ntok[qi * kGTCap + i];
                }
            } else if (!kWide && need) {  // (the wide variant hands the unit over instead)
                const int64_t hb = off * g + (int64_t)h * n;
                t0 = s.tr0[h] + s.tc[h];
                tc = select_tranche(s.sel[h], s.tb[h], kGTCap, s.hist[h], kGBins, b.keys + hb, n, s.last[h], t0 == 0,
                                    kGTCap, tm, b.kminmax ? b.kminmax + (size_t)u * g + h : nullptr,
                                    b.kmm_stride);
                fill_tranche(s.tb[h], tc, pmask, b.rpos + hb + t0, b.slots + off, p.ntok, s.tslot[h], s.tntok[h], tm);
            }
            __syncthreads();
            if (need && tm.tid == 0) {
                s.tr0[h] = t0;
                s.tc[h] = tc;
                s.last[h] = s.tb[h][tc - 1];
            }
            __syncthreads();
        }
        GQA_MARK(1);
#ifdef PSA_GQA_PROF
        pc[8] += 1;
#endif
        // ---- 2. round: union of the live heads' next chunks ----
        // U entries are numbered by first occurrence in (head, rank) order so the
        // per-warp accumulation order, and hence every output bit, is deterministic.
        for (int i = tid; i < kHash; i += kPsaThreads) {
            s.hkey[i] = -1;
            s.hfirst[i] = 0x7fffffff;
        }
        if (tid < G) {
            int c = 0;
            if (s.live[tid]) {
                const int64_t room = s.tr0[tid] + s.tc[tid] - s.cb[tid];
                const int64_t left = limit - s.cb[tid];
                c = (int)(left < CH ? left : CH);
                if (room < c) c = (int)room;
            }
            s.cnt[tid] = c;
        }
        __syncthreads();
        static_assert(G * CH <= kPsaThreads && 2 * G * CH <= kHash, "one thread per (head, rank) of the round");
        const int hh = tid / CH, rr = tid % CH;  // one thread per (head, rank in chunk)
        const bool act = hh < G && rr < s.cnt[hh];
        int hs = -1, ci = 0;
        if (act) {
            ci = (int)(s.cb[hh] - s.tr0[hh]) + rr;
            const int32_t pos = (int32_t)(s.tb[hh][ci] & pmask);
            hs = (int)(((uint32_t)pos * 2654435761u) >> 23) & (kHash - 1);
            for (;;) {
                const int old = atomicCAS(&s.hkey[hs], -1, pos);
                if (old == -1 || old == pos) break;
                hs = (hs + 1) & (kHash - 1);
            }
            atomicMin(&s.hfirst[hs], tid);  // (head, rank) order == thread order
        }
        __syncthreads();
        const bool first = act && s.hfirst[hs] == tid;
        const unsigned fb = __ballot_sync(PSA_FULL, first);
        if (lane == 0) s.wcnt[warp] = __popc(fb);
        __syncthreads();
        if (first) {
            int e = __popc(fb & ((1u << lane) - 1u));
            for (int w = 0; w < warp; ++w) e += s.wcnt[w];
            s.hval[hs] = (int16_t)e;
            s.uslot[e] = s.tslot[hh][ci];
            s.untok[e] = s.tntok[hh][ci];
            s.upos[e] = (int32_t)(s.tb[hh][ci] & pmask);
            s.umask[e] = 0u;
        }
        if (tid == 0) {
            int t = 0;
            for (int w = 0; w < kPsaWarps; ++w) t += s.wcnt[w];
            s.ucount = t;
        }
        __syncthreads();
        if (act) s.cidx[hh][rr] = s.hval[hs];
        const int ucount = s.ucount;
#ifndef PSA_PF
#define PSA_PF 0
#endif
        if constexpr (kMma && (PSA_PF >= 1 || kWide)) {  // measured: helps 64-rank rounds (1.76 -> 1.70 ms), not 32
            // Bulk L2 prefetch of every U block's K (threads 0..) and V (threads 128..): the K pass
            // below then walks L2-resident blocks, and the V pass finds committed blocks in L2.
            const int e = tid & (G * CH - 1);
            if (e < ucount && tid < (PSA_PF == 3 ? 1 : 2) * G * CH && kv_resident(p, s.uslot[e]))
                prefetch_l2_bulk(kv_block<KV>(p, s.uslot[e]) + (tid >= G * CH ? v_off : 0),
                                 (uint32_t)(T * 128 * sizeof(KV)));
        }
        GQA_MARK(2);
        // ---- 3. K pass: every U block once, scored for all heads ----
#pragma unroll kKUnroll
        for (int e = warp; e < ucount; e += kPsaWarps) {
            const int32_t slot = s.uslot[e];
            const int nt = s.untok[e];
            if constexpr (kMma) {
                const int gq = lane >> 2, tq = lane & 3;
                const __nv_bfloat16* kblk = reinterpret_cast<const __nv_bfloat16*>(kv_block<KV>(p, slot));
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
                        mma_bf16_16816(c[tile][0], c[tile][1], c[tile][2], c[tile][3], w0[2 * st], w1[2 * st],
                                       w0[2 * st + 1], w1[2 * st + 1], qg[st][tile][0], qg[st][tile][1]);
#pragma unroll
                for (int tile = 0; tile < NT; ++tile) {
                    float lo = c[tile][0] + c[tile][1], hi = c[tile][2] + c[tile][3];
                    lo += __shfl_xor_sync(PSA_FULL, lo, 1);  // sum the split terms of (head, token)
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
                    if ((tq & 1) == 0 && hq < G) {
                        s.wo.w[e][hq][gq] = wlo;
                        s.wo.w[e][hq][gq + 8] = whi;
                        if (gq == 0) {
                            s.mb[e][hq] = mbv;
                            s.lb[e][hq] = lbv;
                        }
                    }
                }
                continue;
            }
            const KV* kp = kv_block<KV>(p, slot) + base;
            float kr[TOK][DPL];
#pragma unroll
            for (int t = 0; t < TOK; ++t) load_row<DPL>(kp + (size_t)(T == TOK ? t : (t < T ? t : T - 1)) * d, full, lim, kr[t]);
#pragma unroll
            for (int h = 0; h < G; ++h) {
                if (!s.live[h]) continue;  // uniform
                float part[TOK];
#pragma unroll
                for (int t = 0; t < TOK; ++t) {
                    float a = 0.0f;
#pragma unroll
                    for (int jj = 0; jj < DPL; ++jj) a = fmaf(q[h][jj], kr[t][jj], a);
                    part[t] = a;
                }
                float sc = reduce_scatter<TOK>(part, lane) * fscale;
                sc = my_tok < nt ? sc : -INFINITY;
                const float mbv = warp_max(sc);
                const float wv = my_tok < nt ? expf(sc - mbv) : 0.0f;
                float lbv = wv;
#pragma unroll
                for (int o = 16; o >= (1 << TSH); o >>= 1) lbv += __shfl_xor_sync(PSA_FULL, lbv, o);
                if ((lane & ((1 << TSH) - 1)) == 0) s.wo.w[e][h][my_tok] = wv;
                if (lane == 0) {
                    s.mb[e][h] = mbv;
                    s.lb[e][h] = lbv;
                }
            }
        }
#ifdef PSA_GQA_PROF
        if (tid == 0) pc[10] += clock64() - pt;  // warp 0's own K-pass work (rest = imbalance)
#endif
        __syncthreads();
        GQA_MARK(3);
        // ---- 4. decide: warp h for head h, all heads in parallel ----
        if (warp < G && s.live[warp]) {
            const int h = warp;
            const int cnt_all = s.cnt[h];
            const int64_t hb = off * g + (int64_t)h * n;
            double acc = s.acc[h], mn = s.mn[h], ssum = s.ssum[h];
#ifdef PSA_GQA_PROF
            const long long d0_ = clock64();
#endif
            Decision dc{};
            int committed = 0;
            // the head's chunk in 32-rank pieces (one piece unless CH = 64); stop at the first stop
            for (int c0 = 0; c0 < cnt_all; c0 += 32) {
                const int cnt = cnt_all - c0 < 32 ? cnt_all - c0 : 32;
                double x = -INFINITY;
                if (lane < cnt) {
                    const int e = s.cidx[h][c0 + lane];
                    x = b.has_oracle ? b.omass[hb + s.upos[e]] : (double)(s.mb[e][h] + logf(s.lb[e][h]));
                }
                const int64_t cb = s.cb[h] + c0;
                if (b.has_oracle) {
                    dc = decide_chunk(x, cnt, cb, n, limit, b.m, eps, acc, mn, b.iest ? b.iest + hb : nullptr);
                } else if (!PSA_DECIDE_FAST || !decide_chunk_fast((float)x, cnt, cb, n, limit, b.m, eps, acc, ssum, mn,
                                              b.iest ? b.iest + hb : nullptr, dc)) {
                    // fp64 fallback: carried (M, S) -> log-sum-exp and back (M' = lse, S' = 1)
                    acc = ssum > 0.0 ? acc + log(ssum) : -INFINITY;
                    dc = decide_chunk(x, cnt, cb, n, limit, b.m, eps, acc, mn, b.iest ? b.iest + hb : nullptr);
                    ssum = 1.0;
                }
                if (lane < dc.commit) atomicOr(&s.umask[s.cidx[h][c0 + lane]], 1u << h);
                committed = c0 + dc.commit;
                if (dc.fin) break;
            }
            dc.commit = committed;
#ifdef PSA_GQA_PROF
            if (tid == 0) pc[9] += clock64() - d0_;
#endif
            __syncwarp();  // every lane read the carried state above before lane 0 replaces it
            if (lane == 0) {
                s.commit[h] = dc.commit;
                s.fin[h] = dc.fin;
                s.est[h] = dc.est;
                s.acc[h] = acc;
                s.ssum[h] = ssum;
                s.mn[h] = mn;
            }
        }
        __syncthreads();
        if constexpr (kMma && PSA_PF >= 2) {
            // next round's chunk of every continuing head, while this round's V pass runs
            const int h = tid >> 5, r = tid & 31;
            if (h < G && s.live[h] && !s.fin[h]) {
                const int64_t idx = s.cb[h] + s.commit[h] - s.tr0[h] + r;
                if (idx < s.tc[h] && kv_resident(p, s.tslot[h][idx])) {
                    const KV* bp0 = kv_block<KV>(p, s.tslot[h][idx]);
                    prefetch_l2_bulk(bp0, (uint32_t)(T * 128 * sizeof(KV)));
                    prefetch_l2_bulk(bp0 + v_off, (uint32_t)(T * 128 * sizeof(KV)));
                }
            }
        }
        GQA_MARK(4);
        // ---- 5. V pass: committed U blocks once, into every committing head ----
#pragma unroll kVUnroll
        for (int e = warp; e < ucount; e += kPsaWarps) {
            const uint32_t mask = s.umask[e];
            if (!mask) continue;
            const int32_t slot = s.uslot[e];
            if constexpr (kMma) {
                // O^T[dim][(head, split)] += V^T[dim][token] * W^T[token][(head, split)]: 8 MMAs cover
                // 128 dims x all heads; W carries a 2-term bf16 split (16-bit weight precision).
                // Lane (g, t) owns head t, dims [16g, 16g+16): no cross-lane reduction.
                const int gq = lane >> 2, tq = lane & 3;
                const __nv_bfloat16* vblk =
                    reinterpret_cast<const __nv_bfloat16*>(kv_block<KV>(p, slot) + v_off);
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
                const int hb = gq >> 1, sb = gq & 1;  // B column = (head, split)
                const bool hon = hb < G && (mask >> hb) & 1u;
                uint32_t bfr[2];
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const float2 wv = hon ? *reinterpret_cast<const float2*>(&s.wo.w[e][hb][2 * tq + 8 * hf])
                                          : make_float2(0.0f, 0.0f);
                    bfr[hf] = pack_bf16x2_split(wv.x, wv.y, sb);
                }
                float ob[16];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
                    mma_bf16_16816(c0, c1, c2, c3, __byte_perm(vw[0][i], vw[1][i], 0x5410),
                                   __byte_perm(vw[0][i], vw[1][i], 0x7632), __byte_perm(vw[2][i], vw[3][i], 0x5410),
                                   __byte_perm(vw[2][i], vw[3][i], 0x7632), bfr[0], bfr[1]);
                    ob[2 * i] = c0 + c1;      // dim 16g + 2i
                    ob[2 * i + 1] = c2 + c3;  // dim 16g + 2i + 1
                }
                if (tq < G && ((mask >> tq) & 1u)) {
                    const float mbj = s.mb[e][tq];
                    const float mnew = fmaxf(Mreg, mbj);
                    const float a = expf(Mreg - mnew);
                    const float c = expf(mbj - mnew);
#pragma unroll
                    for (int j = 0; j < 16; ++j) Oreg[j] = Oreg[j] * a + ob[j] * c;
                    Lreg = Lreg * a + s.lb[e][tq] * c;
                    Mreg = mnew;
                }
                continue;
            }
            const KV* vp = kv_block<KV>(p, slot) + v_off + base;
            float vr[TOK][DPL];
#pragma unroll
            for (int t = 0; t < TOK; ++t) load_row<DPL>(vp + (size_t)(T == TOK ? t : (t < T ? t : T - 1)) * d, full, lim, vr[t]);
#pragma unroll
            for (int h = 0; h < G; ++h) {
                if (!(mask & (1u << h))) continue;  // uniform
                float ob[DPL];
#pragma unroll
                for (int jj = 0; jj < DPL; ++jj) ob[jj] = 0.0f;
#pragma unroll
                for (int t = 0; t < TOK; ++t) {
                    const float wt = s.wo.w[e][h][t];
#pragma unroll
                    for (int jj = 0; jj < DPL; ++jj) ob[jj] = fmaf(wt, vr[t][jj], ob[jj]);
                }
                const float mbj = s.mb[e][h];
                const float M = s.om[warp][h];
                const float mnew = fmaxf(M, mbj);
                const float a = expf(M - mnew);
                const float c = expf(mbj - mnew);
                float* op = s.o(warp, h) + base;
#pragma unroll
                for (int jj = 0; jj < DPL; ++jj)
                    if (base + jj < d) op[jj] = op[jj] * a + ob[jj] * c;
                __syncwarp();
                if (lane == 0) {
                    s.ol[warp][h] = s.ol[warp][h] * a + s.lb[e][h] * c;
                    s.om[warp][h] = mnew;
                }
                __syncwarp();
            }
        }
#ifdef PSA_GQA_PROF
        if (tid == 0) pc[11] += clock64() - pt;
#endif
        __syncthreads();
        GQA_MARK(5);
        // ---- 6. advance cursors, retire finished heads ----
        if (tid < G && s.live[tid]) {
            const int h = tid;
            s.cb[h] += s.commit[h];
            if (s.fin[h]) {
                s.live[h] = 0;
                const int64_t qi = (int64_t)u * g + h;
                b.bp[qi] = s.cb[h];
                b.est[qi] = s.est[h];
                b.term[qi] = b.topk > 0 ? (limit < n) : (s.cb[h] < n);
            }
        }
        __syncthreads();
        int live = 0;
#pragma unroll
        for (int h = 0; h < G; ++h) live += s.live[h];
        GQA_MARK(6);
        if (!live) break;
        if constexpr (kMma) {
            // Dense hand-over (kernels_dense.cu): a head that exhausted its first tranche needs
            // many ranks; the unit is redone by one K pass + per-head stop rule + one V pass.
            if (b.dense_flag) {
                bool handover = false;
#pragma unroll
                for (int h = 0; h < G; ++h)
                    handover |= s.live[h] && s.cb[h] < limit &&
                                (s.cb[h] >= kDenseHandover || (kWide && s.cb[h] >= s.tr0[h] + s.tc[h]));
                if (handover) {
                    if (tid == 0) b.dense_flag[atomicAdd(b.dense_count, 1)] = u;
                    return;
                }
            }
        }
        __syncthreads();
    }
    if constexpr (kMma) {  // registers -> the per-warp shared-memory accumulators
        const int gq = lane >> 2, tq = lane & 3;
        if (tq < G) {
#pragma unroll
            for (int j = 0; j < 16; ++j) s.o(warp, tq)[16 * gq + j] = Oreg[j];
            if (gq == 0) {
                s.om[warp][tq] = Mreg;
                s.ol[warp][tq] = Lreg;
            }
        }
        __syncthreads();
    }
    // ---- finalize: merge the warps' states per head (finalize, attention.hpp:104-110) ----
    for (int h = 0; h < g; ++h) {
        float Mt = -INFINITY;
#pragma unroll
        for (int w = 0; w < kPsaWarps; ++w) Mt = fmaxf(Mt, s.om[w][h]);
        float Lt = 0.0f, sc[kPsaWarps];
#pragma unroll
        for (int w = 0; w < kPsaWarps; ++w) {
            sc[w] = s.ol[w][h] > 0.0f ? expf(s.om[w][h] - Mt) : 0.0f;
            Lt += s.ol[w][h] * sc[w];
        }
        const int64_t qi = (int64_t)u * g + h;
        for (int i = tid; i < d; i += kPsaThreads) {
            float o = 0.0f;
#pragma unroll
            for (int w = 0; w < kPsaWarps; ++w) o += sc[w] > 0.0f ? s.o(w, h)[i] * sc[w] : 0.0f;
            b.out[qi * d + i] = o / Lt;
        }
        if (b.tcov && tid == 0) {
            double tcv = -1.0;
            if (b.audit) {
                const double* om = b.omass + off * g + (int64_t)h * n;
                double mx = -INFINITY;
                for (int64_t i = 0; i < n; ++i) mx = fmax(mx, om[i]);
                double sm = 0.0;
                for (int64_t i = 0; i < n; ++i) sm += exp(om[i] - mx);
                tcv = exp(s.acc[h] - (mx + log(sm)));
            }
            b.tcov[qi] = tcv;
        }
    }
#ifdef PSA_GQA_PROF
    GQA_MARK(7);
    if (tid == 0)
        for (int k = 0; k < 12; ++k) atomicAdd(&g_gqa_prof[k], (unsigned long long)pc[k]);
#endif
}

template <typename KV, int DPL, int TOK, bool FULL, int G, int CH>
static void launch_gqa_c(const PoolView& p, const BatchView& b, cudaStream_t st) {
    const size_t smem = sizeof(GqaSmem<TOK, G, CH>);
    cudaFuncSetAttribute(psa_gqa_kernel<KV, DPL, TOK, FULL, G, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    psa_gqa_kernel<KV, DPL, TOK, FULL, G, CH><<<b.n_units, kPsaThreads, smem, st>>>(p, b);
}

#ifndef PSA_WIDE_CHUNK
#define PSA_WIDE_CHUNK 64
#endif
template <typename KV, int DPL, int TOK, bool FULL, int G>
static void launch_gqa_t(const PoolView& p, const BatchView& b, cudaStream_t st) {
    // 64-rank rounds on the tensor-core path when the dense hand-over covers long heads
    constexpr bool kMmaPath = std::is_same<KV, __nv_bfloat16>::value && DPL == 4 && TOK == 16 && FULL;
    if constexpr (kMmaPath && PSA_WIDE_CHUNK > kChunk) {
        if (b.dense_flag) {
            launch_gqa_c<KV, DPL, TOK, FULL, G, PSA_WIDE_CHUNK>(p, b, st);
            return;
        }
    }
    launch_gqa_c<KV, DPL, TOK, FULL, G, kChunk>(p, b, st);
}

template <typename KV, int G>
static void launch_gqa_g(const PoolView& p, const BatchView& b, cudaStream_t st) {
    // d = 128 (DPL 4) and d = 64 (DPL 2), blocks of <= 16 tokens: the production shapes
    if (b.d == 128) launch_gqa_t<KV, 4, 16, true, G>(p, b, st);
    else launch_gqa_t<KV, 2, 16, true, G>(p, b, st);
}

// First tranche of every (unit, head) up front: one CTA per head, bandwidth-parallel across the
// batch instead of four 2-warp teams inside each progressive CTA (the same select_tranche /
// fill_tranche, so the tranche is identical). Writes the ranked positions of the tranche too.
__global__ void __launch_bounds__(kPsaThreads) first_tranche_kernel(PoolView p, BatchView b) {
    __shared__ SelScratch sel;
    __shared__ uint32_t hist[kGBins];
    __shared__ uint64_t tb[kGTCap];
    const int qi = blockIdx.x;
    const int u = qi / b.g, h = qi % b.g;
    const int64_t off = b.list_off[u], n = b.list_off[u + 1] - off;
    const int64_t hb = off * b.g + (int64_t)h * n;
    const uint64_t pmask = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);
    const Team tm = cta_team();
    const int tc = select_tranche(sel, tb, kGTCap, hist, kGBins, b.keys + hb, n, 0, true, kGTCap, tm,
                                  b.kminmax ? b.kminmax + qi : nullptr, b.kmm_stride);
    fill_tranche(tb, tc, pmask, b.rpos + hb, b.slots + off, p.ntok, b.ft_slot + (size_t)qi * kGTCap,
                 b.ft_ntok + (size_t)qi * kGTCap, tm);
    for (int i = threadIdx.x; i < tc; i += blockDim.x) b.ft_keys[(size_t)qi * kGTCap + i] = tb[i];
    if (threadIdx.x == 0) b.ft_count[qi] = tc;
}

bool gqa_supported(const PoolView& p, const BatchView& b) {
    return b.g >= 2 && b.g <= 4 && (b.d == 128 || b.d == 64) && p.T <= 16;
}

int launch_gqa(const PoolView& p, const BatchView& b, cudaStream_t st) {
    const int G = b.g <= 2 ? 2 : 4;
#ifndef PSA_FT_THREADS
#define PSA_FT_THREADS 128  // measured (progressive stage): 128 threads 1.65 ms, 256: 1.69, 64: 1.69
#endif
    if (b.ft_keys) first_tranche_kernel<<<b.n_units * b.g, PSA_FT_THREADS, 0, st>>>(p, b);
    const int launches = b.ft_keys ? 2 : 1;
    if (psa_kernel_choice() != 2 && stream_supported(p, b)) {  // the production shape
        launch_stream(p, b, st);
        return launches;
    }
    if (p.dtype == 0) {
        if (G == 2) launch_gqa_g<float, 2>(p, b, st);
        else launch_gqa_g<float, 4>(p, b, st);
    } else {
        if (G == 2) launch_gqa_g<__nv_bfloat16, 2>(p, b, st);
        else launch_gqa_g<__nv_bfloat16, 4>(p, b, st);
    }
    return launches;
}

}  // namespace psa

// Reads (and zeroes) the phase timer: init, order, union, K pass, decide, V pass,
// advance, finalize cycles and the round count. -1 when built without PROF=1.
extern "C" int psattn_debug_gqa_phases(unsigned long long* out12) {
#ifdef PSA_GQA_PROF
    if (cudaMemcpyFromSymbol(out12, psa::g_gqa_prof, sizeof(unsigned long long) * 12) != cudaSuccess) return -1;
    static const unsigned long long z[12] = {};
    cudaMemcpyToSymbol(psa::g_gqa_prof, z, sizeof(z));
    return 0;
#else
    (void)out12;
    return -1;
#endif
}
