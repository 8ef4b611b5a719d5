// kernels_stream.cu — progressive attention of one GQA group as a warp-specialised stream
// (sm_100a): TMA tensor loads of K/V tiles into shared-memory rings, mbarrier hand-offs,
// tensor-core K and V passes, a per-round fp64 coverage decide.
//
// Replaces the round kernel (kernels_gqa.cu) on the production shape: bf16 pool, d = 128,
// 16-token blocks, GQA group of 2..4, HBM-resident pool. Same semantics (reference
// engine.cpp:92-147 per head, psa_attention_multi_head engine.cpp:240-260 for the group):
// every head keeps its own ranking and stop point; a block ranked by several heads in the
// same round is read once.
//
// One CTA per (request, layer, kv-head) unit, 8 warps with fixed roles:
//   warp 0    PRODUCER  round r = the live heads' ranks [rC, rC+C) (C = 32 / G); a block is an
//                       ENTRY the first time any head's round reaches it (unit-wide dedup: a
//                       hash of list positions in shared memory), so its K tile is fetched once
//                       (two 2-D TMA boxes of 64 dims x 16 tokens, 128-byte swizzle) into the K
//                       ring, at most kLook rounds ahead of the last decided round; V tiles are
//                       fetched for the blocks the decider releases, each once, together with the
//                       block's token weights (1-D bulk copy) into the V ring;
//   warp 1    DECIDER   per round, one warp-wide segmented scan (C lanes per head) of the
//                       block masses in each head's rank order: CoverageEstimator::observe + the
//                       estimate at microbatch boundaries (engine.cpp:38-55, 109-125) in fp64,
//                       the first boundary with est > eps stops the head. A block is released to
//                       the V pass once every head has decided it (committed it, or stopped
//                       before reaching it);
//   warps 2-4 SCORERS   K pass: ldmatrix of the swizzled K tile, mma.sync bf16 with the
//                       query split into 3 exact bf16 terms (all heads of the group in the
//                       N dimension); per (block, head) max / exp-sum kept in shared memory for
//                       the whole unit, token weights written to a global scratch row;
//   warps 5-7 V         V pass: ldmatrix.trans of the V tile, mma.sync with the weights split
//                       into 3 exact bf16 terms (fp32-exact weights), online-softmax merge of the
//                       block into every head that committed it (merge_partial,
//                       attention.hpp:83-102); at the end the three warps' states merge
//                       (finalize, attention.hpp:104-110).
// Bytes: every block of the heads' union is fetched exactly once (K and V); speculation is
// K-only and bounded by kLook rounds; blocks no head commits are never V-fetched. Counters of
// fetched K / V tiles feed the benchmark's waste figure.
#include <cuda.h>
#include <cuda_bf16.h>
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "common.cuh"
#include "kernels.cuh"
#include "mma.cuh"
#include "tma.cuh"

namespace psa {

__device__ unsigned long long g_stream_stats[4];  // K tiles, V tiles, rounds, units (accumulating)
__device__ unsigned long long g_stream_prof[32];  // PSA_STREAM_PROF builds: [role][0 total, wait sites 1-5, idle, busy]
// Development builds (make STREAM_DEBUG=1): a wait that does not complete within ~2^22 polls
// writes the stuck warp's state into mapped host memory (readable after the trap) and traps.
__device__ int* g_stream_dbg = nullptr;

namespace stream {

#ifndef PSA_STREAM_NS
#define PSA_STREAM_NS 3
#endif
#ifndef PSA_STREAM_NV
#define PSA_STREAM_NV 3
#endif
#ifndef PSA_STREAM_MINB
#define PSA_STREAM_MINB 2
#endif
constexpr int kNS = PSA_STREAM_NS, kNV = PSA_STREAM_NV;  // scorer / V warps
constexpr int kThreads = (2 + kNS + kNV) * 32;
constexpr int kWS0 = 2, kWV0 = 2 + kNS;  // first scorer / V warp
#ifndef PSA_STREAM_RK
#define PSA_STREAM_RK 12  // measured: 12 > 9 (the exponent sums moved to the weights rows made room)
#endif
#ifndef PSA_STREAM_RV
#define PSA_STREAM_RV 9
#endif
#ifndef PSA_STREAM_LOOK
#define PSA_STREAM_LOOK 2
#endif
#ifndef PSA_STREAM_PF
#define PSA_STREAM_PF 0
#endif
#ifndef PSA_STREAM_PARK
#define PSA_STREAM_PARK 0  // producer park bound (ns) on the next decision when idle; 0 = nanosleep(64)
#endif
constexpr int kRK = PSA_STREAM_RK;  // K ring stages (4 KB K tile)
constexpr int kRV = PSA_STREAM_RV;  // V ring stages (4 KB V tile + the block's token weights)
constexpr int kLR = 8;              // round slots in flight
constexpr int kENT = kStreamEnt;    // distinct blocks per unit
#ifndef PSA_STREAM_HASH
#define PSA_STREAM_HASH (2 * kStreamEnt)
#endif
constexpr int kHash = PSA_STREAM_HASH;  // list position -> entry (open addressing), a power of two
static_assert((kHash & (kHash - 1)) == 0 && kHash >= kENT && kHash <= 2048, "hash size");
constexpr int kLook = PSA_STREAM_LOOK;
#ifndef PSA_STREAM_SPL
#define PSA_STREAM_SPL 1
#endif
constexpr int kSPL = PSA_STREAM_SPL;
#ifndef PSA_STREAM_SLEEP
#define PSA_STREAM_SLEEP 64  // producer back-off (ns) when nothing can be issued
#endif
#ifndef PSA_STREAM_PAIR
#define PSA_STREAM_PAIR 1
#endif
constexpr int kPair = PSA_STREAM_PAIR;  // entries a scorer warp handles together (1 or 2)  // rank slots per lane in a round: a round is 32*kSPL/G ranks per head
static_assert(kSPL == 1 || kSPL == 2, "1 or 2 rank slots per lane");
// V reference R of a head: its top criticality score + kVRef. Kept while the rank-0 block's max is
// at least R - kVLow and no scored block's max exceeds R + kVHigh; otherwise the unit is redone densely.
constexpr float kVRef = 8.0f, kVLow = 40.0f, kVHigh = 60.0f;
static_assert(kLook + 2 <= kLR, "round slots must cover the lookahead");
// Entry e is consumed by scorer e % kNS from K stage e % kRK (V item j: V warp j % kNV, stage
// j % kRV). With the ring a multiple of the consumer count, a stage's previous use belongs to
// the SAME consumer, which has already waited on it: a full-barrier wait can never pass on the
// parity of a stale phase (two uses back) while another consumer's load is still in flight.
static_assert(kRK % kNS == 0 && kRV % kNV == 0, "each consumer warp owns its ring stages");

template <int G>
struct Smem {
    alignas(1024) unsigned char kring[kRK][4096];
    alignas(1024) unsigned char vring[kRV][4096];
    alignas(16) float vw[kRV][G * 16 + 4];  // token weights beside each V tile, then the heads' exponent sums
    float em[kENT][G];                 // block log mass per (entry, head) (the stop rule's observation)
    int32_t eslot[kENT];
    int32_t epos[kENT];
    uint32_t vmask[kENT];  // heads that committed the entry (decider)
    uint8_t entok[kENT];
    uint8_t queued[kENT];
    int32_t hkey[kHash];
    int16_t hval[kHash];
    int16_t r_map[kLR][32 * kSPL];  // (head, rank-in-round) slot lane*kSPL+s -> entry, -1 none
    int32_t r_e0[kLR], r_cnt[kLR], r_flag[kLR];
    int32_t r_live[kLR], r_vc[kLR], r_stop[kLR];  // decider -> producer, per decided round
    int16_t vq[kENT + kNV];  // V items in creation order (entry), -1 = end
    int32_t handover;
    int32_t vref_bad;    // a head's V reference does not fit its blocks (extreme logits): dense redo
    int32_t rank0[G];    // entry of each head's rank-0 block (set with round 0)
    int32_t dbg_flag;
    float lpart[kNV][G];
    uint64_t kfull[kRK], kempty[kRK], vfull[kRV], vempty[kRV];
    uint64_t rpub[kLR], rscored[kLR], rdec[kLR];
};

#ifdef PSA_STREAM_DEBUG
__device__ __noinline__ void dbg_stuck(int site, int a0, int a1, int a2, int a3, int a4, int a5, int a6, int a7) {
    int* d = g_stream_dbg;
    if (d) {
        const int k = atomicAdd(d, 1);
        if (k < 256) {
            int* r = d + 16 + 16 * k;
            const int v[12] = {(int)blockIdx.x, (int)(threadIdx.x >> 5), (int)(threadIdx.x & 31), site, a0, a1, a2, a3,
                               a4, a5, a6, a7};
            for (int i = 0; i < 12; ++i) ((volatile int*)r)[i] = v[i];
            __threadfence_system();
        }
    }
    __trap();
}
__device__ __noinline__ void dbg_note(int site, int a0, int a1, int a2, int a3, int a4, int a5, int a6, int a7) {
    int* d = g_stream_dbg;
    if (d) {
        const int k = atomicAdd(d, 1);
        if (k < 256) {
            int* r = d + 16 + 16 * k;
            const int v[12] = {(int)blockIdx.x, (int)(threadIdx.x >> 5), (int)(threadIdx.x & 31), site, a0, a1, a2, a3,
                               a4, a5, a6, a7};
            for (int i = 0; i < 12; ++i) ((volatile int*)r)[i] = v[i];
            __threadfence_system();
        }
    }
}
// waits; when the producer flags a stall, a waiting lane 0 writes where it waits (once)
#define SWAIT(bar, ph, site, a0, a1, a2, a3, a4, a5, a6, a7)                                            \
    do {                                                                                               \
        bool noted_ = false;                                                                           \
        for (uint32_t it_ = 0; !mbar_try_wait((bar), (ph)); ++it_) {                                   \
            if (!noted_ && (it_ & 255) == 0 && *(volatile int*)&s.dbg_flag && (threadIdx.x & 31) == 0) { \
                noted_ = true;                                                                         \
                dbg_note((site), (a0), (a1), (a2), (a3), (int)(ph), (int)*(volatile uint32_t*)(bar),     \
                         (int)(*(volatile uint64_t*)(bar) >> 32), (a7));                               \
            }                                                                                          \
        }                                                                                              \
    } while (0)
#elif defined(PSA_STREAM_PROF)
// development builds (make EXTRA=-DPSA_STREAM_PROF): cycles each warp spends in each wait site
#define SWAIT(bar, ph, site, a0, a1, a2, a3, a4, a5, a6, a7) \
    do {                                                      \
        const long long t0_ = clock64();                      \
        mbar_wait((bar), (ph));                               \
        pw[(site)] += clock64() - t0_;                        \
    } while (0)
#else
#define SWAIT(bar, ph, site, a0, a1, a2, a3, a4, a5, a6, a7) mbar_wait((bar), (ph))
#endif

template <int G>
__global__ void __launch_bounds__(kThreads, PSA_STREAM_MINB) psa_stream_kernel(const __grid_constant__ CUtensorMap kvmap,
                                                                PoolView p, BatchView b) {
    constexpr int LPH = 32 / G;    // lanes per head (producer / decider)
    constexpr int C = LPH * kSPL;  // ranks per head per round
    constexpr int NT = G / 2;  // n8 tiles (4 columns per head: 3 split terms + 0)
    constexpr uint32_t kWB = (G * 16 + 4) * 4;  // weight bytes per entry (+ exponent sums)
    extern __shared__ unsigned char smem_raw[];
    Smem<G>& s = *reinterpret_cast<Smem<G>*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int u = blockIdx.x;
    const int g = b.g;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int64_t limit = b.topk > 0 ? (b.topk < n ? b.topk : n) : n;
    const int T2 = 2 * p.T;  // tensor-map rows per slot (K rows then V rows)
#ifdef PSA_STREAM_PROF
    long long pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long t_start = clock64();
#endif
    float* wg = b.stream_w + (size_t)u * kENT * kStreamWRow;  // this unit's weight rows

    if (tid == 0) {
        for (int i = 0; i < kRK; ++i) {
            mbar_init(&s.kfull[i], 1);
            mbar_init(&s.kempty[i], 1);
        }
        for (int i = 0; i < kRV; ++i) {
            mbar_init(&s.vfull[i], 1);
            mbar_init(&s.vempty[i], 1);
        }
        for (int i = 0; i < kLR; ++i) {
            mbar_init(&s.rpub[i], 1);
            mbar_init(&s.rscored[i], kNS);
            mbar_init(&s.rdec[i], 1);
        }
        s.handover = 0;
        s.vref_bad = 0;
        s.dbg_flag = 0;
        for (int h = 0; h < G; ++h) s.rank0[h] = -1;
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == 0) {
        // ================================ PRODUCER ================================
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&kvmap)) : "memory");
        for (int i = lane; i < kHash; i += 32) s.hkey[i] = -1;
        __syncwarp();
        const int h = lane / LPH, il = lane % LPH;  // head; the lane's slots are ranks il*kSPL + s of a round
        const bool hv = h < g;
        const size_t qi = (size_t)u * g + (hv ? h : 0);
        const int ftc = hv ? b.ft_count[qi] : 0;
        const uint64_t pmask = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);
        int k_pub = 0, E = 0, k_issue = 0, v_seen = 0, v_issued = 0, decided = -1, lm = (1 << g) - 1;
        bool stopped = false, closed = false;  // closed: no more rounds (entry table full)
        int32_t fpos[kSPL], fslot[kSPL], fnt[kSPL];
        auto fetch = [&](int k) {
#pragma unroll
            for (int sl = 0; sl < kSPL; ++sl) {
                const int64_t r = (int64_t)k * C + il * kSPL + sl;
                if (hv && r < ftc && r < limit) {
                    fpos[sl] = (int32_t)(b.ft_keys[qi * kFirstCap + r] & pmask);
                    fslot[sl] = b.ft_slot[qi * kFirstCap + r];
                    fnt[sl] = b.ft_ntok[qi * kFirstCap + r];
                } else {
                    fpos[sl] = -1;
                    fslot[sl] = 0;
                    fnt[sl] = 0;
                }
            }
        };
        fetch(0);
#ifdef PSA_STREAM_DEBUG
        int idle = 0;
#endif
        for (;;) {
            bool progress = false;
            // (1) decisions, in round order
            // (lane 0 tests, the warp follows: every lane must see the same decisions)
            while (__shfl_sync(PSA_FULL, lane == 0 && decided + 1 < k_pub &&
                                             mbar_test(&s.rdec[(decided + 1) % kLR], ((decided + 1) / kLR) & 1), 0)) {
                ++decided;
                const int rs = decided % kLR;  // values the decider published with this round
                lm = s.r_live[rs];
                v_seen = s.r_vc[rs];
                if (s.r_stop[rs]) stopped = true;
                progress = true;
            }
            // lane 0 acquired the decisions; order the warp's later shared reads (vq, r_*) after it
            if (progress) __syncwarp();
            // (2) publish the next round (speculative: heads live as of the last decided round)
            if (!stopped && !closed && k_pub <= decided + kLook) {
                const int rs = k_pub % kLR;
                const int e_round0 = E;
#pragma unroll
                for (int sl = 0; sl < kSPL; ++sl) {  // one pass per rank slot of the lanes
                    const bool valid = !closed && fpos[sl] >= 0 && ((lm >> h) & 1);
                    const unsigned peers = __match_any_sync(PSA_FULL, valid ? fpos[sl] : -1 - lane);
                    const int leader = __ffs(peers) - 1;
                    const bool lead = valid && leader == lane;
                    int hs = 0, ent = -1;
                    bool isnew = false;
                    if (lead) {  // unit-wide dedup: a block fetched in an earlier round is not fetched again
                        hs = (int)(((uint32_t)fpos[sl] * 2654435761u) >> 21) & (kHash - 1);
                        for (;;) {
                            const int kk = s.hkey[hs];
                            if (kk == fpos[sl]) {
                                ent = s.hval[hs];
                                break;
                            }
                            if (kk == -1) {
                                const int old = atomicCAS(&s.hkey[hs], -1, fpos[sl]);
                                if (old == -1) {
                                    isnew = true;
                                    break;
                                }
                                continue;  // another lane took the slot: look at it again
                            }
                            hs = (hs + 1) & (kHash - 1);
                        }
                    }
                    const unsigned nb = __ballot_sync(PSA_FULL, isnew);
                    const int cnt = __popc(nb);
                    if (closed || E + cnt > kENT) {
                        // more distinct blocks than the entry table holds: the decider hands the unit
                        // over (dense path) at this round; nothing more is published
                        s.r_map[rs][lane * kSPL + sl] = -1;
                        closed = true;
                    } else {
                        if (isnew) {
#if PSA_STREAM_PF
                            // the entry's K (PF=2) or K and V (PF=1, one contiguous slot) start towards L2
                            // now, kLook rounds before the K tile is needed: the K ring refills from L2
                            prefetch_l2_bulk(p.kv + (int64_t)fslot[sl] * p.slot_bytes,
                                             (uint32_t)(PSA_STREAM_PF == 2 ? p.slot_bytes / 2 : p.slot_bytes));
#endif
                            ent = E + __popc(nb & ((1u << lane) - 1u));
                            s.hval[hs] = (int16_t)ent;
                            s.eslot[ent] = fslot[sl];
                            s.epos[ent] = fpos[sl];
                            s.entok[ent] = (uint8_t)fnt[sl];
                            s.vmask[ent] = 0u;
                            s.queued[ent] = 0;
                        }
                        const int myent = __shfl_sync(PSA_FULL, ent, leader);
                        s.r_map[rs][lane * kSPL + sl] = (int16_t)(valid ? myent : -1);
                        if (k_pub == 0 && il == 0 && sl == 0 && valid) s.rank0[h] = myent;
                        E += cnt;
                    }
                }
                if (lane == 0) {
                    s.r_e0[rs] = e_round0;
                    s.r_cnt[rs] = E - e_round0;
                    s.r_flag[rs] = closed ? 1 : 0;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.rpub[rs]);
                ++k_pub;
                if (!closed) fetch(k_pub);
                progress = true;
            }
            // (3) K tiles of new entries, while K stages are free
            {
                const int e = k_issue + lane;
                const bool ok = e < E && (e < kRK || mbar_test(&s.kempty[e % kRK], ((e / kRK) - 1) & 1));
                const unsigned bal = __ballot_sync(PSA_FULL, ok);
                const int pc = bal == PSA_FULL ? 32 : __ffs(~bal) - 1;
                if (lane < pc) {
                    const int st = e % kRK;
                    const int y = s.eslot[e] * T2;
                    mbar_arrive_expect_tx(&s.kfull[st], 4096);
                    const uint32_t dst = smem_u32(s.kring[st]);
                    tma_tile(dst, &kvmap, 0, y, &s.kfull[st]);
                    tma_tile(dst + 2048, &kvmap, 64, y, &s.kfull[st]);
                }
                k_issue += pc;
                progress |= pc > 0;
            }
            // (4) V tiles (+ the block's token weights) of ready items, while V stages are free
            {
                const int it = v_issued + lane;
                const bool ok = it < v_seen && (it < kRV || mbar_test(&s.vempty[it % kRV], ((it / kRV) - 1) & 1));
                const unsigned bal = __ballot_sync(PSA_FULL, ok);
                const int pc = bal == PSA_FULL ? 32 : __ffs(~bal) - 1;
                if (lane < pc) {
                    const int st = it % kRV;
                    const int e = s.vq[it];
                    const int y = s.eslot[e] * T2 + p.T;
                    mbar_arrive_expect_tx(&s.vfull[st], 4096 + kWB);
                    const uint32_t dst = smem_u32(s.vring[st]);
                    tma_tile(dst, &kvmap, 0, y, &s.vfull[st]);
                    tma_tile(dst + 2048, &kvmap, 64, y, &s.vfull[st]);
                    bulk_g2s(smem_u32(&s.vw[st][0]), wg + (size_t)e * kStreamWRow, kWB, &s.vfull[st]);
                }
                v_issued += pc;
                progress |= pc > 0;
            }
            // (5) done: every published K tile and every V item issued after the last decision
            if (stopped && k_issue == E && v_issued == v_seen) {
                const int rs = k_pub % kLR;  // sentinel round for the scorers
                if (lane == 0) s.r_cnt[rs] = -1;
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.rpub[rs]);
                if (lane < kNV) {  // one end item per V warp
                    const int it = v_seen + lane;
                    if (it >= kRV)
                        SWAIT(&s.vempty[it % kRV], ((it / kRV) - 1) & 1, 1, it, v_seen, v_issued, E, k_issue, k_pub,
                              decided, 0);
                    s.vq[it] = -1;
                    mbar_arrive(&s.vfull[it % kRV]);
                }
                break;
            }
#ifdef PSA_STREAM_PROF
            ++pw[progress ? 7 : 6];
#endif
            if (!progress) {
#if PSA_STREAM_PARK
                // nothing to issue: park on the next round's decision (the usual next event) for a
                // bounded time instead of spinning through the loop
                if (decided + 1 < k_pub)
                    (void)__shfl_sync(PSA_FULL, lane == 0 ? (int)mbar_try_wait_for(&s.rdec[(decided + 1) % kLR],
                                                                                   ((decided + 1) / kLR) & 1, PSA_STREAM_PARK)
                                                          : 0, 0);
                else
                    __nanosleep(PSA_STREAM_SLEEP);
#else
                __nanosleep(PSA_STREAM_SLEEP);
#endif
#ifdef PSA_STREAM_DEBUG
                if (++idle == (1 << 22)) {
                    if (lane == 0) {
                        const int st = k_issue % kRK;
                        dbg_note(0, k_pub, E, k_issue, v_seen, v_issued, decided, (int)*(volatile uint32_t*)&s.kempty[st],
                                 (int)(*(volatile uint64_t*)&s.kempty[st] >> 32));
                        dbg_note(6, s.r_e0[0], s.r_e0[1], s.r_e0[2], s.r_e0[3], s.r_e0[4], s.r_e0[5], s.r_e0[6], s.r_e0[7]);
                        dbg_note(7, s.r_cnt[0], s.r_cnt[1], s.r_cnt[2], s.r_cnt[3], s.r_cnt[4], s.r_cnt[5], s.r_cnt[6], s.r_cnt[7]);
                        *(volatile int*)&s.dbg_flag = 1;
                    }
                }
                if (idle > (1 << 22) + (1 << 16)) dbg_stuck(99, 0, 0, 0, 0, 0, 0, 0, 0);
            } else {
                idle = 0;
#endif
            }
        }
        if (lane == 0) {
            atomicAdd(&g_stream_stats[0], (unsigned long long)E);
            atomicAdd(&g_stream_stats[1], (unsigned long long)v_seen);
            atomicAdd(&g_stream_stats[2], (unsigned long long)(decided + 1));
            atomicAdd(&g_stream_stats[3], 1ull);
        }
    } else if (warp == 1) {
        // ================================ DECIDER ================================
        const int h = lane / LPH, il = lane % LPH;  // head; the lane's slots are ranks il*kSPL + sl
        const bool hv = h < g;
        const int64_t qi = (int64_t)u * g + (hv ? h : 0);
        const int64_t hb = off * g + (int64_t)(hv ? h : 0) * n;
        const int ftc = hv ? b.ft_count[qi] : 0;
        const double eps = b.topk > 0 ? 1.0 : b.eps;
        const unsigned seg = (LPH == 32 ? PSA_FULL : ((1u << LPH) - 1u)) << (h * LPH);
        const uint32_t all = (1u << g) - 1u;
        bool live = hv;
        int64_t cb = 0;
        int vc = 0;  // V items created
        // a flat head (criticality within dense_early nats over its top kDenseHandover ranks, e.g.
        // isotropic keys) would consume the hand-over budget without stopping: the unit goes to the
        // dense kernels after its first round instead of after kDenseHandover ranks (performance
        // only: both paths produce the same processed sets)
        bool flat = false;
        if (b.dense_early > 0.0f && hv && il == 0 && ftc >= kDenseHandover && limit > kDenseHandover) {
            const uint64_t pm = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);
            const double s0 = key_score(b.ft_keys[qi * kFirstCap], pm);
            const double s1 = key_score(b.ft_keys[qi * kFirstCap + kDenseHandover - 1], pm);
            flat = s0 - s1 < (double)b.dense_early;
        }
        const bool flat_unit = __any_sync(PSA_FULL, flat);
        // CoverageEstimator state (engine.cpp:38-55) in fp64 about the running max M of the observed
        // masses: S = sum exp(mass - M), E = exp(min mass - M) (+inf before the first block)
        double M = -INFINITY, S = 0.0, E = INFINITY, est = 0.0;
        const double one_m_eps = 1.0 - eps;
        for (int k = 0;; ++k) {
            const int rs = k % kLR;
            SWAIT(&s.rscored[rs], (k / kLR) & 1, 2, k, (int)cb, vc, (int)live, 0, 0, 0, 0);
#ifdef PSA_STREAM_PROF
            const long long td0_ = clock64();
#endif
            const int e_end = s.r_e0[rs] + s.r_cnt[rs];  // entries published up to this round
            const bool overflow = s.r_flag[rs] == 1;
            int e[kSPL];
            int64_t r[kSPL];
            bool valid[kSPL];
            double x[kSPL];
            float xmax = -INFINITY;
            double xmaxd = -INFINITY;
#pragma unroll
            for (int sl = 0; sl < kSPL; ++sl) {
                e[sl] = s.r_map[rs][lane * kSPL + sl];
                r[sl] = cb + il * kSPL + sl;
                valid[sl] = live && e[sl] >= 0 && r[sl] < limit;
                x[sl] = -INFINITY;
                if (valid[sl]) {
                    if (!b.has_oracle) {
                        const float xf = s.em[e[sl]][h];
                        x[sl] = (double)xf;
                        xmax = fmaxf(xmax, xf);
                    } else {
                        x[sl] = b.omass[hb + s.epos[e[sl]]];
                        xmaxd = fmax(xmaxd, x[sl]);
                    }
                }
            }
            double mx;
            if (!b.has_oracle) {  // fp32 masses: the segment max is exact in fp32
#pragma unroll
                for (int o = LPH / 2; o >= 1; o >>= 1) xmax = fmaxf(xmax, __shfl_xor_sync(PSA_FULL, xmax, o));
                mx = (double)xmax;
            } else {
                mx = xmaxd;
#pragma unroll
                for (int o = LPH / 2; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(PSA_FULL, mx, o));
            }
            mx = fmax(mx, M);
            // carried state re-expressed about the new max (only when it moved: rare after round 0)
            double Sc = S, Ec = E;  // (M = -inf: S = 0, E = +inf, nothing to rescale)
            const bool moved = M != -INFINITY && mx != M;
            if (__any_sync(PSA_FULL, moved)) {
                const double fct = moved ? exp(M - mx) : 1.0;
                Sc = S * fct;
                Ec = E * fct;
            }
            // prefix sums / prefix mins of exp(mass - mx) in rank order: within the lane's slots, then a
            // segmented scan over the head's lanes; exp(min - mx) is the min of the exponentials (monotone)
            double ps[kSPL], pm_[kSPL];
            double run = 0.0, runm = INFINITY;
#pragma unroll
            for (int sl = 0; sl < kSPL; ++sl) {
                const double ev = valid[sl] ? exp(x[sl] - mx) : 0.0;
                run += ev;
                runm = fmin(runm, valid[sl] ? ev : INFINITY);
                ps[sl] = run;
                pm_[sl] = runm;
            }
            double incl = run, inclm = runm;
#pragma unroll
            for (int o = 1; o < LPH; o <<= 1) {
                const double ye = __shfl_up_sync(PSA_FULL, incl, o, LPH);
                const double ym = __shfl_up_sync(PSA_FULL, inclm, o, LPH);
                if (il >= o) {
                    incl += ye;
                    inclm = fmin(inclm, ym);
                }
            }
            const double excl = incl - run;  // sum over the head's earlier lanes
            double exclm = __shfl_up_sync(PSA_FULL, inclm, 1, LPH);
            if (il == 0) exclm = INFINITY;
            double Si[kSPL], Ei[kSPL], est_i[kSPL];
            bool boundary[kSPL], stop[kSPL];
            bool anystop = false;
#pragma unroll
            for (int sl = 0; sl < kSPL; ++sl) {
                Si[sl] = Sc + (excl + ps[sl]);        // sum exp(mass - mx) observed up to this rank
                Ei[sl] = fmin(Ec, fmin(exclm, pm_[sl]));  // exp(min mass - mx)
                const int64_t nl = n - (r[sl] + 1);
                const double D = (double)nl * Ei[sl];
                // est = Si / (Si + n_left exp(min - mx)) = 1 / (1 + n_left exp(min - acc)) (engine.cpp:48-55);
                // est > eps  <=>  Si (1 - eps) > eps D: the division runs only when a head may stop
                boundary[sl] = valid[sl] && (b.m == 1 || ((r[sl] + 1) % b.m) == 0 || r[sl] + 1 == limit);
                const bool over = nl == 0 ? eps < 1.0 : (Si[sl] > 0.0 && Si[sl] * one_m_eps > eps * D);
                stop[sl] = boundary[sl] && (over || r[sl] + 1 == limit);
                anystop |= stop[sl];
                est_i[sl] = 0.0;
            }
            if (b.iest || __any_sync(PSA_FULL, anystop)) {
#pragma unroll
                for (int sl = 0; sl < kSPL; ++sl) {
                    const int64_t nl = n - (r[sl] + 1);
                    est_i[sl] = nl == 0 ? 1.0 : (Si[sl] > 0.0 ? Si[sl] / (Si[sl] + (double)nl * Ei[sl]) : 0.0);
                }
            }
            // first stop in rank order (lane-major, slot-minor) and the head's valid ranks
            int f_stop = 1 << 30, nvalid = 0;
#pragma unroll
            for (int sl = 0; sl < kSPL; ++sl) {
                const unsigned sb_s = __ballot_sync(PSA_FULL, stop[sl]) & seg;
                const unsigned vb_s = __ballot_sync(PSA_FULL, valid[sl]) & seg;
                nvalid += __popc(vb_s);
                if (sb_s) f_stop = min(f_stop, (__ffs(sb_s) - 1 - h * LPH) * kSPL + sl);
            }
            const unsigned sb = f_stop < (1 << 30) ? 1u : 0u;  // (head stops in this round)
            const int f = sb ? f_stop : nvalid - 1;  // last committed rank of the head in this round
            bool committed[kSPL];
#pragma unroll
            for (int sl = 0; sl < kSPL; ++sl) {
                const int ri = il * kSPL + sl;
                committed[sl] = valid[sl] && ri <= f;
                if (b.iest && boundary[sl] && ri <= f) b.iest[hb + r[sl]] = est_i[sl];  // IterationStats
                if (committed[sl]) atomicOr(&s.vmask[e[sl]], 1u << h);
            }
            const int fr = f > 0 ? f : 0;
            const int src = h * LPH + fr / kSPL, fsl = fr % kSPL;
            double Sf = 0.0, Ef = 0.0, estf = 0.0;
#pragma unroll
            for (int sl = 0; sl < kSPL; ++sl) {
                const double a1 = __shfl_sync(PSA_FULL, Si[sl], src), a2 = __shfl_sync(PSA_FULL, Ei[sl], src);
                const double a3 = __shfl_sync(PSA_FULL, est_i[sl], src);
                if (sl == fsl) {
                    Sf = a1;
                    Ef = a2;
                    estf = a3;
                }
            }
            if (nvalid > 0) {
                M = mx;
                S = Sf;
                E = Ef;
                est = estf;
                cb += f + 1;
            }
            const bool fin_now = live && sb != 0;
            if (fin_now) {
                live = false;
                if (il == 0) {
                    b.bp[qi] = cb;
                    b.est[qi] = est;
                    b.term[qi] = b.topk > 0 ? (limit < n) : (cb < n);
                    if (b.tcov) {
                        double tcv = -1.0;
                        if (b.audit) {
                            const double* om = b.omass + hb;
                            double omx = -INFINITY;
                            for (int64_t j = 0; j < n; ++j) omx = fmax(omx, om[j]);
                            double sm = 0.0;
                            for (int64_t j = 0; j < n; ++j) sm += exp(om[j] - omx);
                            tcv = exp((M + log(S)) - (omx + log(sm)));
                        }
                        b.tcov[qi] = tcv;
                    }
                }
            }
            // a head that used up its first tranche (or kDenseHandover ranks), or a unit whose
            // distinct blocks overflow the entry table, is handed over to the dense kernels
            const bool ho = live && cb < limit && (cb >= kDenseHandover || cb >= ftc || overflow || flat_unit);
            const bool anyho = __any_sync(PSA_FULL, ho);
            const unsigned lb = __ballot_sync(PSA_FULL, live && il == 0);
            uint32_t lmask = 0;
#pragma unroll
            for (int hh = 0; hh < G; ++hh) lmask |= ((lb >> (hh * LPH)) & 1u) << hh;
            const bool done = anyho || lmask == 0;
            __syncwarp();  // this round's vmask bits are visible to every lane
            if (!anyho) {
                // V items: a block goes to the V pass once every head has decided it (committed it,
                // or stopped before reaching it), in a deterministic order
                const uint32_t stopped = all & ~lmask;
#pragma unroll
                for (int sl = 0; sl < kSPL; ++sl) {
                    const unsigned peers = __match_any_sync(PSA_FULL, committed[sl] ? e[sl] : -1 - lane);
                    const bool cand = committed[sl] && (__ffs(peers) - 1) == lane;
                    const bool ready = cand && ((s.vmask[e[sl]] | stopped) == all) && !s.queued[e[sl]];
                    const unsigned rb = __ballot_sync(PSA_FULL, ready);
                    if (ready) {
                        s.vq[vc + __popc(rb & ((1u << lane) - 1u))] = (int16_t)e[sl];
                        s.queued[e[sl]] = 1;
                    }
                    vc += __popc(rb);
                    __syncwarp();  // queued flags of this pass before the next slot's
                }
                if (__any_sync(PSA_FULL, fin_now)) {  // a head stopped: blocks waiting only on it are ready
                    __syncwarp();
                    for (int e0 = 0; e0 < e_end; e0 += 32) {
                        const int ee = e0 + lane;
                        const bool rd = ee < e_end && s.vmask[ee] != 0u && !s.queued[ee] && ((s.vmask[ee] | stopped) == all);
                        const unsigned b2 = __ballot_sync(PSA_FULL, rd);
                        if (rd) {
                            s.vq[vc + __popc(b2 & ((1u << lane) - 1u))] = (int16_t)ee;
                            s.queued[ee] = 1;
                        }
                        vc += __popc(b2);
                    }
                }
            }
            if (lane == 0) {
                s.r_vc[rs] = vc;
                s.r_live[rs] = (int32_t)lmask;
                s.r_stop[rs] = done;
                if (done) {
                    s.handover = anyho;
                    if (anyho) b.dense_flag[atomicAdd(b.dense_count, 1)] = u;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.rdec[rs]);
#ifdef PSA_STREAM_PROF
            pw[6] += clock64() - td0_;
#endif
            if (done) break;
        }
    } else if (warp < kWV0) {
        // ================================ SCORERS ================================
        const int sidx = warp - kWS0;
        const int gq = lane >> 2, tq = lane & 3;
        const float fscale = (float)b.scale;
        uint32_t qg[8][NT][2];  // B fragments: column (head 2t + gq/4, split gq%4), k = dims
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int hq = 2 * t + (gq >> 2), sp = gq & 3;
            const float* qrow = b.q + ((size_t)u * g + (hq < g ? hq : 0)) * 128;
#pragma unroll
            for (int st = 0; st < 8; ++st)
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const int d0 = 16 * st + 8 * hf + 2 * tq;
                    const float a = hq < g ? qrow[d0] : 0.0f, c = hq < g ? qrow[d0 + 1] : 0.0f;
                    qg[st][t][hf] = pack_split3(a, c, sp);
                }
        }
        // V reference of the epilogue's head (2t + tq/2): the token weights handed to the V pass are
        // exp(s - R_h) with one fixed R_h per head (its top criticality score + kVRef), so the V warps
        // accumulate every committed block as is. Deterministic; checked against the blocks' actual
        // maxima (the rank-0 block within kVLow below R_h, no block more than kVHigh above it), else
        // the unit is redone by the dense kernels (per-block maxima).
        float vref[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int hq = 2 * t + (tq >> 1);
            const size_t qh = (size_t)u * g + (hq < g ? hq : 0);
            const uint64_t pm = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);
            vref[t] = b.ft_count[qh] > 0 ? (float)key_score(b.ft_keys[qh * kFirstCap], pm) + kVRef : 0.0f;
        }
        for (int k = 0;; ++k) {
            const int rs = k % kLR;
            SWAIT(&s.rpub[rs], (k / kLR) & 1, 3, k, 0, 0, 0, 0, 0, 0, 0);
            const int cnt = s.r_cnt[rs];
            if (cnt < 0) break;
            const int e0 = s.r_e0[rs];
            // entries of this round owned by this scorer, kPair at a time: the MMA chains and the
            // epilogues of the pair are independent (latency overlap)
            auto score_tile = [&](int e, float (&c)[NT][4]) {
                const int st = e % kRK;
                SWAIT(&s.kfull[st], (e / kRK) & 1, 4, k, e, e0, cnt, 0, 0, 0, 0);
                const uint32_t kb = smem_u32(s.kring[st]);
                // two accumulator sets (even / odd k-steps): halves the dependent MMA chain
                float c2[NT][4];
#pragma unroll
                for (int t = 0; t < NT; ++t)
#pragma unroll
                    for (int r = 0; r < 4; ++r) c[t][r] = c2[t][r] = 0.0f;
#pragma unroll
                for (int kst = 0; kst < 8; ++kst) {
                    uint32_t a0, a1, a2, a3;
                    ldsm4(swz(kb, lane & 15, 2 * kst + (lane >> 4)), a0, a1, a2, a3);
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        float(&cc)[4] = (kst & 1) ? c2[t] : c[t];
                        mma_bf16_16816(cc[0], cc[1], cc[2], cc[3], a0, a1, a2, a3, qg[kst][t][0], qg[kst][t][1]);
                    }
                }
#pragma unroll
                for (int t = 0; t < NT; ++t)
#pragma unroll
                    for (int r = 0; r < 4; ++r) c[t][r] += c2[t][r];
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.kempty[st]);  // the tile is in registers: release it
            };
            auto epilogue = [&](int e, float (&c)[NT][4]) {
                const int nt = s.entok[e];
                float* we = wg + (size_t)e * kStreamWRow;
#pragma unroll
                for (int t = 0; t < NT; ++t) {
                    float lo = c[t][0] + c[t][1], hi = c[t][2] + c[t][3];
                    lo += __shfl_xor_sync(PSA_FULL, lo, 1);  // the 4 split columns of (token, head)
                    hi += __shfl_xor_sync(PSA_FULL, hi, 1);
                    const int hq = 2 * t + (tq >> 1);
                    lo = (gq < nt) ? lo * fscale : -INFINITY;
                    hi = (gq + 8 < nt) ? hi * fscale : -INFINITY;
                    // token weights straight against the head's V reference R (no block-max pass):
                    // w = exp(s - R), block exponent sum L = sum w, log mass = R + ln L (the reference's
                    // m + ln sum exp(s - m), attention.hpp:55-73, taken about R instead of m)
                    const float R = vref[t];
                    float wlo = expf(lo - R), whi = expf(hi - R);
                    float lbv = wlo + whi;
#pragma unroll
                    for (int o = 4; o < 32; o <<= 1) lbv += __shfl_xor_sync(PSA_FULL, lbv, o);
                    float la = R + __logf(lbv);  // MUFU lg2: ~1e-7 absolute, below fp32 ulp(la) at these magnitudes
                    if (__any_sync(PSA_FULL, !(lbv >= 1e-30f && lbv <= 1e30f))) {
                        // a block far below R (its fp32 terms would lose precision) or above it (could
                        // overflow): exact mass about its own max; above-R blocks flag the unit (dense redo)
                        float mbv = fmaxf(lo, hi);
#pragma unroll
                        for (int o = 4; o < 32; o <<= 1) mbv = fmaxf(mbv, __shfl_xor_sync(PSA_FULL, mbv, o));
                        float l2 = ((gq < nt) ? expf(lo - mbv) : 0.0f) + ((gq + 8 < nt) ? expf(hi - mbv) : 0.0f);
#pragma unroll
                        for (int o = 4; o < 32; o <<= 1) l2 += __shfl_xor_sync(PSA_FULL, l2, o);
                        la = mbv + logf(l2);
                        if (mbv > R + kVHigh) s.vref_bad = 1;
                        if (!(lbv <= 1e30f)) wlo = whi = lbv = 0.0f;
                    }
                    if (k == 0 && e == s.rank0[hq] && la < R - kVLow) s.vref_bad = 1;  // R far above the top block
                    if ((tq & 1) == 0) {
                        we[hq * 16 + gq] = wlo;
                        we[hq * 16 + gq + 8] = whi;
                        if (gq == 0) {
                            s.em[e][hq] = la;  // log_as (attention.hpp:73)
                            we[G * 16 + hq] = lbv;  // exponent sum about R_h (travels with the weights)
                        }
                    }
                }
            };
            for (int e = e0 + ((sidx - e0 % kNS) + kNS) % kNS; e < e0 + cnt; e += kNS * kPair) {
#ifdef PSA_STREAM_PROF
                const long long tq0_ = clock64();
#endif
                float c[kPair][NT][4];
                const bool two = kPair == 2 && e + kNS < e0 + cnt;
                score_tile(e, c[0]);
                if constexpr (kPair == 2)
                    if (two) score_tile(e + kNS, c[kPair - 1]);
#ifdef PSA_STREAM_PROF
                pw[6] += clock64() - tq0_;
#endif
                epilogue(e, c[0]);
                if constexpr (kPair == 2)
                    if (two) epilogue(e + kNS, c[kPair - 1]);
            }
            // the weights are read back by the async proxy (bulk copy beside the V tile)
#ifdef PSA_STREAM_PROF
            const long long tq1_ = clock64();
#endif
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.rscored[rs]);
#ifdef PSA_STREAM_PROF
            pw[7] += clock64() - tq1_;
#endif
        }
    } else {
        // ================================== V ==================================
        // The scorers hand over token weights exp(s - R_h) relative to one fixed reference per head,
        // so a committed block is accumulated as is: acc += V^T w (exact 3-term bf16 split of w,
        // mma.sync into fp32 accumulators, one column per split term, summed once at the end) and
        // L_h += its exponent sum. Heads that did not commit the block get zero weights.
        const int vidx = warp - kWV0;
        const int gq = lane >> 2, tq = lane & 3;
        float acc[NT][8][4];
        float Lh[G];
#pragma unroll
        for (int h = 0; h < G; ++h) Lh[h] = 0.0f;
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) acc[t][mt][0] = acc[t][mt][1] = acc[t][mt][2] = acc[t][mt][3] = 0.0f;
        const int tok = (lane & 7) + ((lane >> 4) << 3);  // ldmatrix.trans row (token) of this lane
        const int chi = (lane >> 3) & 1;                   // + dim chunk
        for (int j = vidx;; j += kNV) {
            const int st = j % kRV;
            SWAIT(&s.vfull[st], (j / kRV) & 1, 5, j, 0, 0, 0, 0, 0, 0, 0);
#ifdef PSA_STREAM_PROF
            const long long tp0_ = clock64();
#endif
            const int e = s.vq[j];
            if (e < 0) break;
            const uint32_t mask = s.vmask[e];
            const int nt = s.entok[e];
#pragma unroll
            for (int h = 0; h < G; ++h)
                if ((mask >> h) & 1u) Lh[h] += s.vw[st][G * 16 + h];
            uint32_t bw[NT][2];
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int hq = 2 * t + (gq >> 2), sp = gq & 3;
                const bool on = (mask >> hq) & 1u;
                const float2 wl = *reinterpret_cast<const float2*>(&s.vw[st][hq * 16 + 2 * tq]);
                const float2 wh = *reinterpret_cast<const float2*>(&s.vw[st][hq * 16 + 2 * tq + 8]);
                bw[t][0] = on ? pack_split3(wl.x, wl.y, sp) : 0u;
                bw[t][1] = on ? pack_split3(wh.x, wh.y, sp) : 0u;
            }
#ifdef PSA_STREAM_PROF
            const long long tp1_ = clock64();
            pw[6] += tp1_ - tp0_;
#endif
            const uint32_t vb = smem_u32(s.vring[st]);
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                uint32_t a0, a1, a2, a3;
                ldsm4t(swz(vb, tok, 2 * mt + chi), a0, a1, a2, a3);
                if (nt < 16) {  // rows past the block's tokens may hold stale data: zero them
                    const uint32_t m0 = (2 * tq < nt ? 0x0000FFFFu : 0u) | (2 * tq + 1 < nt ? 0xFFFF0000u : 0u);
                    const uint32_t m1 = (2 * tq + 8 < nt ? 0x0000FFFFu : 0u) | (2 * tq + 9 < nt ? 0xFFFF0000u : 0u);
                    a0 &= m0;
                    a1 &= m0;
                    a2 &= m1;
                    a3 &= m1;
                }
#pragma unroll
                for (int t = 0; t < NT; ++t)
                    mma_bf16_16816(acc[t][mt][0], acc[t][mt][1], acc[t][mt][2], acc[t][mt][3], a0, a1, a2, a3,
                                   bw[t][0], bw[t][1]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.vempty[st]);
#ifdef PSA_STREAM_PROF
            pw[7] += clock64() - tp1_;
#endif
        }
        // sum the split columns: lane pair (tq, tq^1) holds the 4 columns of head 2t + tq/2
        float O[NT][8];
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                const float x = (tq & 1) ? (acc[t][mt][0] + acc[t][mt][1]) : (acc[t][mt][2] + acc[t][mt][3]);
                const float y = __shfl_xor_sync(PSA_FULL, x, 1);
                O[t][mt] = ((tq & 1) ? (acc[t][mt][2] + acc[t][mt][3]) : (acc[t][mt][0] + acc[t][mt][1])) + y;
            }
        // ---- merge the V warps' states per head (finalize, attention.hpp:104-110) ----
        asm volatile("bar.sync 1, %0;" ::"r"(kNV * 32) : "memory");  // every V tile consumed
        float* part = reinterpret_cast<float*>(&s.vring[0][0]);     // [kNV][G][128]
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const int hq = 2 * t + (tq >> 1);
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) part[(vidx * G + hq) * 128 + 16 * mt + gq + 8 * (tq & 1)] = O[t][mt];
            if (gq == 0 && (tq & 1) == 0) s.lpart[vidx][hq] = (tq >> 1) ? Lh[2 * t + 1] : Lh[2 * t];
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kNV * 32) : "memory");
        if (!s.handover && s.vref_bad) {
            // extreme logits: a head's criticality-based reference does not fit its blocks' maxima
            // (fp32 weights could overflow or the dominant blocks underflow): the dense kernels redo it
            if (tid == kWV0 * 32) b.dense_flag[atomicAdd(b.dense_count, 1)] = u;
        } else if (!s.handover) {
            for (int idx = tid - kWV0 * 32; idx < g * 128; idx += kNV * 32) {
                const int hq = idx >> 7, dd = idx & 127;
                float Lt = 0.0f, o = 0.0f;  // every V warp's state shares the head's reference: plain sums
#pragma unroll
                for (int w = 0; w < kNV; ++w) {
                    Lt += s.lpart[w][hq];
                    o += part[(w * G + hq) * 128 + dd];
                }
                b.out[((size_t)u * g + hq) * 128 + dd] = o / Lt;  // finalize (attention.hpp:104-110)
            }
        }
    }
#ifdef PSA_STREAM_PROF
    {
        const int role = warp == 0 ? 0 : warp == 1 ? 1 : warp < kWV0 ? 2 : 3;
        pw[0] = clock64() - t_start;
        if (lane == 0)
            for (int i = 0; i < 8; ++i) atomicAdd(&g_stream_prof[role * 8 + i], (unsigned long long)pw[i]);
    }
#endif
}

}  // namespace stream

bool stream_supported(const PoolView& p, const BatchView& b) {
    return p.kv_tmap != nullptr && p.loc == nullptr && p.dtype == 1 && p.T == 16 && b.d == 128 && b.g >= 2 &&
           b.g <= 4 && b.ft_keys != nullptr && b.dense_flag != nullptr && b.stream_w != nullptr;
}

void launch_stream(const PoolView& p, const BatchView& b, cudaStream_t st) {
    const CUtensorMap& map = *static_cast<const CUtensorMap*>(p.kv_tmap);
    auto go = [&](auto kern, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<b.n_units, stream::kThreads, smem, st>>>(map, p, b);
    };
    if (b.g <= 2) go(stream::psa_stream_kernel<2>, sizeof(stream::Smem<2>) + 1024);
    else go(stream::psa_stream_kernel<4>, sizeof(stream::Smem<4>) + 1024);
}

}  // namespace psa

// K tiles fetched, V tiles fetched, rounds decided, units run by the stream kernel since the last
// call (accumulating device counters; reading zeroes them). Benchmark instrumentation.
// Development builds: attach a mapped host buffer (int[16 + 16*256]) that collects stuck-wait
// records; returns its host pointer (nullptr in normal builds).
extern "C" int* psattn_debug_stream_attach() {
#ifdef PSA_STREAM_DEBUG
    static int* host = nullptr;
    if (!host) {
        if (cudaHostAlloc((void**)&host, sizeof(int) * (16 + 16 * 256), cudaHostAllocMapped) != cudaSuccess) return nullptr;
        memset(host, 0, sizeof(int) * (16 + 16 * 256));
        int* dev = nullptr;
        if (cudaHostGetDevicePointer((void**)&dev, host, 0) != cudaSuccess) return nullptr;
        if (cudaMemcpyToSymbol(psa::g_stream_dbg, &dev, sizeof(dev)) != cudaSuccess) return nullptr;
    }
    return host;
#else
    return nullptr;
#endif
}

extern "C" int psattn_debug_stream_stats(unsigned long long* out4) {
    if (cudaMemcpyFromSymbol(out4, psa::g_stream_stats, sizeof(unsigned long long) * 4) != cudaSuccess) return -1;
    static const unsigned long long z[4] = {};
    return cudaMemcpyToSymbol(psa::g_stream_stats, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}

// PSA_STREAM_PROF builds: per role (producer, decider, scorers, V) summed over warps: total
// cycles, cycles waiting at sites 1-5 (1 V-ring drain, 2 round scored, 3 round published,
// 4 K tile, 5 V tile), producer idle / productive loop iterations. Reading zeroes them.
extern "C" int psattn_debug_stream_prof(unsigned long long* out32) {
    if (cudaMemcpyFromSymbol(out32, psa::g_stream_prof, sizeof(unsigned long long) * 32) != cudaSuccess) return -1;
    static const unsigned long long z[32] = {};
    return cudaMemcpyToSymbol(psa::g_stream_prof, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
