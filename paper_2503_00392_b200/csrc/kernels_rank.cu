// kernels_rank.cu — K2 criticality scoring, K6 oracle masses, GQA union, batch dispatch.
#include <cuda_bf16.h>
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

// score-kernel conversion variants (build knobs; defaults are the measured best)
#ifndef PSA_ALL_F2F
#define PSA_ALL_F2F 0
#endif

namespace psa {

static int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// =============================================================================
// K2: criticality scoring (criticality_score, reference metadata.cpp:41-72).
// Grid (x: warps sharing a unit, y: unit). A warp scores kRecs CONSECUTIVE list
// positions per iteration against all G q-heads of the GQA group: every
// metadata record (mean f32 | lo kv | hi kv, 1 KB for d=128 bf16) is read from
// HBM once per kv-head, the loads of all kRecs records are issued before any
// math, and the G*kRecs fp64 dot products are finished with ONE reduce-scatter
// so the keys of each head land as one contiguous 32 B store.
//
// Arithmetic (fp64, like the reference): products of fp32 operands are exact in
// fp64; only the summation order differs from the reference's sequential loop
// (~1e-16 relative). Issue slots are the limiter at the HBM rate (ncu: IPC 2.7,
// ALU and FP64 pipes ~45%), so:
//  * bf16 lo/hi -> fp64 are bit constructions scaled by 2^-896 (2-3 ALU slots); the
//    fp32 mean takes one F2F on the otherwise idle XU pipe (all three on the XU pipe
//    measured slower: its 16 lanes/clk become the limit);
//  * max(q*lo, q*hi) == q*c + |q|*r with c = (lo+hi)/2, r = (hi-lo)/2 (hi >= lo):
//    no per-head select, and with the factor 2 folded into the final scale the
//    shared per-dim work is lo+hi, hi-lo and 2m+(lo+hi) (3 fp64 ops), then
//    2 DFMA per head: acc = sum q(2m + lo + hi) + |q|(hi - lo) = 4 * CuboidMean.
// =============================================================================
constexpr int kScoreWarps = 8;
// records per warp iteration: 4 for the d=128 / g<=4 path, fewer where registers would spill
template <int G, int DPL> struct RecsPer {
    static constexpr int r = (G * DPL <= 16) ? 4 : (G * DPL <= 32) ? 2 : 1;
    static constexpr int v = (G * r <= 16) ? r : 16 / G;  // G*v <= 16: the reduction scratch fits
};

// fp32 bit pattern -> double scaled by 2^-896, exact: the fp64 exponent field equals
// the fp32 one, so the conversion is a shift and a mask on the ALU pipe (an F2F on the
// XU pipe measured slower: 3.82 vs 3.64 ms for the bench's score stage).
__device__ __forceinline__ double f32_scaled(uint32_t u) {
    return __hiloint2double((int)(((uint32_t)((int32_t)u >> 3)) & 0x8FFFFFFFu), (int)(u << 29));
}

template <typename KV> struct MetaRow;
template <> struct MetaRow<float> {
    template <int DPL> __host__ __device__ static constexpr int words() { return DPL; }
    template <int DPL>
    __device__ __forceinline__ static void load(const float* p, bool full, int lim, uint32_t (&w)[DPL]) {
        float f[DPL];
        load_row<DPL>(p, full, lim, f);
#pragma unroll
        for (int j = 0; j < DPL; ++j) w[j] = __float_as_uint(f[j]);
    }
    template <int W>
    __device__ __forceinline__ static double get(const uint32_t (&w)[W], int j) { return f32_scaled(w[j]); }
};
template <> struct MetaRow<__nv_bfloat16> {
    template <int DPL> __host__ __device__ static constexpr int words() { return (DPL + 1) / 2; }
    template <int DPL>
    __device__ __forceinline__ static void load(const __nv_bfloat16* p, bool full, int lim,
                                                uint32_t (&w)[(DPL + 1) / 2]) {
        if (full && DPL % 8 == 0) {
#pragma unroll
            for (int j = 0; j < DPL / 8; ++j) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + j);
                w[4 * j] = v.x; w[4 * j + 1] = v.y; w[4 * j + 2] = v.z; w[4 * j + 3] = v.w;
            }
        } else if (full && DPL % 4 == 0) {
#pragma unroll
            for (int j = 0; j < DPL / 4; ++j) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(p) + j);
                w[2 * j] = v.x; w[2 * j + 1] = v.y;
            }
        } else {
            const unsigned short* ps = reinterpret_cast<const unsigned short*>(p);
#pragma unroll
            for (int j = 0; j < (DPL + 1) / 2; ++j) {
                const uint32_t a = (2 * j < lim) ? ps[2 * j] : 0u;
                const uint32_t c = (2 * j + 1 < lim && 2 * j + 1 < DPL) ? ps[2 * j + 1] : 0u;
                w[j] = a | (c << 16);
            }
        }
    }
    template <int W>
    __device__ __forceinline__ static double get(const uint32_t (&w)[W], int j) {
        const uint32_t x = w[j >> 1];
        return f32_scaled((j & 1) ? (x & 0xFFFF0000u) : (x << 16));
    }
};

// Cross-lane reduction of N per-lane doubles through a shared-memory transpose
// (cheaper than a shuffle reduce-scatter: no selects, 2 wavefronts per 64-bit
// access is optimal anyway). red: this warp's 32*N-double scratch. Returns the
// warp total of value index lane / (32/N) (on all 32/N lanes that own it).
template <int N>
__device__ __forceinline__ double smem_reduce(double (&acc)[N], double* red, int lane) {
    constexpr int P = 32 / N;   // lanes per value
    constexpr int RS = N + 1;   // padded row: writes and reads both hit the 2-wavefront minimum
    __syncwarp();
#pragma unroll
    for (int i = 0; i < N; ++i) red[lane * RS + i] = acc[i];
    __syncwarp();
    const int v = lane / P, part = lane % P;
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) t += red[(part * N + k) * RS + v];
#pragma unroll
    for (int o = 1; o < P; o <<= 1) t += __shfl_xor_sync(PSA_FULL, t, o);
    return t;
}

// Same reduction with XOR-swizzled 16-double rows (no padding): 32 x 16 doubles =
// exactly 4 KB, so it fits in a consumed TMA stage buffer. Conflict-free (2 wavefronts
// per 64-bit access, the minimum) for both the row writes and the column reads.
// Column-major variant (the TMA kernel's): value i's 32 partials are written contiguously
// (red[i*32 + lane]: immediate offsets, conflict-free), and lane (v = lane & 15, part = lane >> 4)
// sums the partials of lanes [16*part, 16*part + 16) of value v in the XOR order k ^ v, so the
// 16 lanes of a half-warp hit 16 different 8-byte bank pairs; the address of read k is
// A ^ 8k (one LOP3). Returns the total of value (lane & 15) on lanes v and v + 16.
__device__ __forceinline__ double smem_reduce16_cm(double (&acc)[16], double* red, int lane) {
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 16; ++i) red[i * 32 + lane] = acc[i];
    __syncwarp();
    const int v = lane & 15, part = lane >> 4;
    const uint32_t a0 = smem_u32(red) + (uint32_t)(v * 256 + part * 128 + v * 8);
    double x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x[k]) : "r"(a0 ^ (uint32_t)(8 * k)));
    // x[k] is the partial of lane 16*part + (k ^ v). A balanced pairwise tree pairs indices that
    // differ in one bit, level by level, so it is invariant under the XOR permutation by v: every
    // value v sums its 16 partials with the same bracketing, and equal metadata records give
    // bit-equal scores wherever they sit in a group (exact ties then fall to the block-id rule).
#pragma unroll
    for (int w = 1; w < 16; w <<= 1)
#pragma unroll
        for (int k = 0; k < 16; k += 2 * w) x[k] += x[k + w];
    return x[0] + __shfl_xor_sync(PSA_FULL, x[0], 16);
}

__device__ __forceinline__ double smem_reduce16_swz(double (&acc)[16], double* red, int lane) {
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 16; ++i) red[lane * 16 + (i ^ (lane & 15))] = acc[i];
    __syncwarp();
    const int v = lane >> 1, part = lane & 1;
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int r = part * 16 + k;
        t += red[r * 16 + (v ^ (r & 15))];
    }
    t += __shfl_xor_sync(PSA_FULL, t, 1);
    return t;
}

template <typename KV, int G, int DPL, bool FULL>
__global__ void __launch_bounds__(kScoreWarps * 32, 2) score_kernel(PoolView p, BatchView b) {
    constexpr int kRecs = RecsPer<G, DPL>::v;
    constexpr int N = G * kRecs;
    constexpr int SH = 5 - Log2<N>::v;  // lanes per value after reduce-scatter = 1 << SH
    constexpr int WKV = MetaRow<KV>::template words<DPL>();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    __shared__ __align__(16) double red_all[kScoreWarps][32 * (N + 1)];
    double* red = red_all[warp];
    const int u = blockIdx.y;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int d = FULL ? 32 * DPL : b.d;  // compile-time on the full-row paths
    const int base = lane * DPL;
    const int lim = d - base;
    constexpr bool full = FULL;  // d == 32*DPL: vector loads, no bounds

    double qd[G][DPL];  // q * 2^896 (compensates the scaled metadata)
#pragma unroll
    for (int h = 0; h < G; ++h) {
        float qf[DPL];
        if (h < b.g)
            load_row<DPL>(b.q + ((size_t)u * b.g + h) * d + base, full, lim, qf);
        else
#pragma unroll
            for (int j = 0; j < DPL; ++j) qf[j] = 0.0f;
#pragma unroll
        for (int j = 0; j < DPL; ++j) qd[h][j] = (double)qf[j] * 0x1p896;
    }
    const int est = b.estimator;
    const double scale = b.scale;
    const int my_idx = lane >> SH;  // value index this lane owns after the reduce-scatter
    const int my_h = my_idx / kRecs, my_j = my_idx % kRecs;
    const bool writer = (lane & ((1 << SH) - 1)) == 0 && my_h < b.g;
    uint64_t* keys = b.keys + off * b.g + (int64_t)my_h * n;
    uint64_t kmin = ~0ull, kmax = 0;  // keys written by this lane (first-tranche bounds)

    const int64_t ngroups = (n + kRecs - 1) / kRecs;
    const int64_t nwarps = (int64_t)gridDim.x * kScoreWarps;
    int64_t grp = (int64_t)blockIdx.x * kScoreWarps + warp;
    // slot ids of the next group are fetched one iteration ahead (lanes 0..kRecs-1)
    int32_t nxt = (lane < kRecs && grp * kRecs + lane < n) ? b.slots[off + grp * kRecs + lane] : -1;
    for (; grp < ngroups; grp += nwarps) {
        const int64_t p0 = grp * kRecs;
        const int32_t my_slot = nxt;
        const int64_t pn = (grp + nwarps) * kRecs;
        nxt = (lane < kRecs && pn + lane < n) ? b.slots[off + pn + lane] : -1;
        const int32_t slot0 = __shfl_sync(PSA_FULL, my_slot, 0);  // p0 < n: always valid
        uint32_t mw[kRecs][DPL], lw[kRecs][WKV], hw[kRecs][WKV];
        // Branch-free: a record past the end re-reads record 0 (its key is never written),
        // so all 3*kRecs loads issue back to back before the first use.
#pragma unroll
        for (int j = 0; j < kRecs; ++j) {
            int32_t slot = __shfl_sync(PSA_FULL, my_slot, j);
            slot = slot >= 0 ? slot : slot0;
            const char* rec = p.meta + (int64_t)slot * p.meta_bytes;
            MetaRow<float>::load<DPL>(reinterpret_cast<const float*>(rec) + base, full, lim, mw[j]);
            MetaRow<KV>::template load<DPL>(reinterpret_cast<const KV*>(rec + (size_t)d * 4) + base, full, lim, lw[j]);
            MetaRow<KV>::template load<DPL>(reinterpret_cast<const KV*>(rec + (size_t)d * 4 + (size_t)d * sizeof(KV)) +
                                                base, full, lim, hw[j]);
        }
        double acc[N];
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] = 0.0;
#pragma unroll
        for (int j = 0; j < kRecs; ++j) {
#pragma unroll
            for (int jj = 0; jj < DPL; ++jj) {
                const double m = MetaRow<float>::get(mw[j], jj);
                const double lo = MetaRow<KV>::get(lw[j], jj);
                const double hi = MetaRow<KV>::get(hw[j], jj);
                double A, B = 0.0;
                if (est == 0) {
                    A = m;  // mean_score
                } else {
                    const double c2 = lo + hi;          // exact
                    B = hi - lo;                        // 2r, exact
                    A = est == 2 ? fma(2.0, m, c2) : c2;  // 2(m + c)  |  2c
                }
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    const double qv = qd[h][jj];
                    double a = fma(qv, A, acc[h * kRecs + j]);
                    if (est != 0) a = fma(fabs(qv), B, a);  // + |q| r  ==  max(q lo, q hi) - q c
                    acc[h * kRecs + j] = a;
                }
            }
        }
        const double tot = smem_reduce<N>(acc, red, lane);
        if (writer && p0 + my_j < n) {
            // acc = sum q(2m + lo + hi) + |q|(hi - lo) = 4 * CuboidMean / 2 * Upper; Mean: plain
            const double s = est == 2 ? 0.25 * (tot * scale) : (est == 1 ? 0.5 * (tot * scale) : tot * scale);
            const uint64_t key = make_key(s, (uint32_t)(p0 + my_j), b.pos_bits);
            keys[p0 + my_j] = key;
            kmin = key < kmin ? key : kmin;
            kmax = key > kmax ? key : kmax;
        }
    }
    if (b.kminmax && writer && kmax != 0) {
        atomicMin(b.kminmax + (size_t)u * b.g + my_h, (unsigned long long)kmin);
        atomicMax(b.kminmax + b.kmm_stride + (size_t)u * b.g + my_h, (unsigned long long)kmax);
    }
}

// -----------------------------------------------------------------------------
// K2 for d = 128 (the production shape): same arithmetic, but the metadata
// records are staged through shared memory with 1-D TMA bulk copies
// (cp.async.bulk + mbarrier transaction counts). Each warp owns a ring of S
// stages of kRecs records; lanes 0..kRecs-1 each issue one record copy (1 KB bf16
// / 1.5 KB fp32, L2 evict-first: metadata is streamed once per step) S groups
// ahead of the math, so memory-level parallelism no longer costs registers.
// -----------------------------------------------------------------------------
constexpr int kTmaBarBytes = 256;  // kScoreWarps x (<= 4 stages) x 8 B mbarriers
#ifndef PSA_SCORE_CHUNKED
#define PSA_SCORE_CHUNKED 1  // contiguous group runs per warp + windowed slot loads
#endif

template <typename KV, int G, int EST>
#ifndef PSA_SCORE_MINB
#define PSA_SCORE_MINB 2
#endif
#ifndef PSA_SCORE_SB
#define PSA_SCORE_SB 12288  // bytes of TMA stages per warp (3 x 4 KB records groups)
#endif
__global__ void __launch_bounds__(kScoreWarps * 32, PSA_SCORE_MINB) score_kernel_tma(PoolView p, BatchView b) {
    constexpr int DPL = 4, D = 128;
    constexpr int kRecs = RecsPer<G, DPL>::v;
    constexpr int N = G * kRecs;
    constexpr int SH = 5 - Log2<N>::v;
    constexpr int MB = D * 4 + 2 * D * (int)sizeof(KV);  // metadata record bytes (meta_bytes)
    constexpr int STAGE = kRecs * MB;
    constexpr bool kReuse = (N == 16 && STAGE >= 4096);  // reduction scratch lives in the consumed stage
    constexpr int SB = kReuse ? PSA_SCORE_SB : 8192;
    constexpr int S = (SB / STAGE) < 2 ? 2 : ((SB / STAGE) > 4 ? 4 : (SB / STAGE));  // 2 CTAs/SM
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    static_assert(kScoreWarps * S * 8 <= kTmaBarBytes, "mbarrier region too small");
    unsigned char* wbuf = smem + kTmaBarBytes + (size_t)warp * S * STAGE;
    uint64_t* wbar = bars + warp * S;
    if (lane == 0)
        for (int i = 0; i < S; ++i) mbar_init(&wbar[i], 1);
    fence_mbar_init();
    __syncwarp();

    const int u = blockIdx.y;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int base = lane * DPL;
    double qd[G][DPL];  // q * 2^896 (compensates the scaled metadata)
#pragma unroll
    for (int h = 0; h < G; ++h) {
        float qf[DPL];
        if (h < b.g)
            load_row<DPL>(b.q + ((size_t)u * b.g + h) * D + base, true, DPL, qf);
        else
#pragma unroll
            for (int j = 0; j < DPL; ++j) qf[j] = 0.0f;
#pragma unroll
        for (int j = 0; j < DPL; ++j) qd[h][j] = (double)qf[j] * (PSA_ALL_F2F && EST == 2 ? 1.0 : 0x1p896);
    }
    constexpr int est = EST;  // estimator as a template parameter: no per-record branches
    // acc = 4 CuboidMean / 2 Upper / Mean: the power-of-two factor folded into the scale (exact)
    const double kscale = est == 2 ? 0.25 * b.scale : (est == 1 ? 0.5 * b.scale : b.scale);
    const uint64_t kmask = (b.pos_bits >= 64) ? ~0ull : ((1ull << b.pos_bits) - 1ull);
    // value this lane owns after the reduction: lane & 15 (lanes 0-15 write) for the column-major
    // 16-value reduce, else lane >> SH
    constexpr bool kCM = (N == 16 && STAGE >= 4096);
    const int my_idx = kCM ? (lane & 15) : (lane >> SH);
    const int my_h = my_idx / kRecs, my_j = my_idx % kRecs;
    const bool writer = (kCM ? lane < 16 : (lane & ((1 << SH) - 1)) == 0) && my_h < b.g;
    uint64_t* keys = b.keys + off * b.g + (int64_t)my_h * n;
    uint64_t kmin = ~0ull, kmax = 0;  // keys written by this lane (first-tranche bounds)
    const uint64_t pol = policy_evict_first();

    const int64_t ngroups = (n + kRecs - 1) / kRecs;
    const int64_t nwarps = (int64_t)gridDim.x * kScoreWarps;
#if PSA_SCORE_CHUNKED
    // each warp owns a contiguous run of groups; the page-table slots of 32 consecutive records
    // (a window) arrive in one coalesced load, one window ahead, and reach the issuing lanes by shuffle
    const int64_t gpw = (ngroups + nwarps - 1) / nwarps;
    const int64_t g_begin = ((int64_t)blockIdx.x * kScoreWarps + warp) * gpw;
    const int64_t g_end = g_begin + gpw < ngroups ? g_begin + gpw : ngroups;
    constexpr int kWinGroups = 32 / kRecs;
    const int64_t rec_end = g_end * kRecs < n ? g_end * kRecs : n;
    auto win_load = [&](int64_t w) -> int32_t {
        const int64_t r = g_begin * kRecs + w * 32 + lane;
        return r < rec_end ? b.slots[off + r] : 0;
    };
    int32_t wcur = win_load(0), wnext = win_load(1);
    int64_t wi = 0;  // window held in wcur
    auto slot_at = [&](int64_t g) -> int32_t {  // lanes < kRecs: slots of group g (all lanes call)
        const int64_t k = g - g_begin;
        const int src = (int)(k % kWinGroups) * kRecs + (lane < kRecs ? lane : 0);
        const int32_t a = __shfl_sync(PSA_FULL, wcur, src), c = __shfl_sync(PSA_FULL, wnext, src);
        return (k / kWinGroups) == wi ? a : c;
    };
#else
    const int64_t grp0 = (int64_t)blockIdx.x * kScoreWarps + warp;
#endif
    auto issue = [&](int64_t grp, int stage, int32_t slot) {
        const int64_t p0 = grp * kRecs;
        const int cnt = (int)((n - p0) < kRecs ? (n - p0) : kRecs);
        if (lane == 0) mbar_arrive_expect_tx(&wbar[stage], (uint32_t)(cnt * MB));
        __syncwarp();
        // records in consecutive slots (the usual page-table layout) move as ONE bulk copy
        const int32_t slot0 = __shfl_sync(PSA_FULL, slot, 0);
        if (__all_sync(PSA_FULL, lane >= cnt || slot == slot0 + lane)) {
            if (lane == 0)
                tma_load_1d(wbuf + stage * STAGE, p.meta + (int64_t)slot0 * MB, (uint32_t)(cnt * MB), &wbar[stage], pol);
        } else if (lane < cnt) {
            tma_load_1d(wbuf + stage * STAGE + lane * MB, p.meta + (int64_t)slot * MB, MB, &wbar[stage], pol);
        }
    };
#if PSA_SCORE_CHUNKED
    // prologue: S groups in flight
#pragma unroll 1
    for (int st = 0; st < S; ++st) {
        const int64_t g = g_begin + st;
        const int32_t sl = slot_at(g);
        if (g < g_end) issue(g, st, sl);
    }
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t grp = g_begin; grp < g_end; ++grp) {
        const int64_t gn = grp + S;  // group that refills this stage
        if ((gn - g_begin) / kWinGroups != wi) {  // the refill enters the next window: slide
            wcur = wnext;
            ++wi;
            wnext = win_load(wi + 1);
        }
        const int32_t nslot = slot_at(gn);
        mbar_wait(&wbar[stage], phase);
#else
    // prologue: S groups in flight
#pragma unroll 1
    for (int st = 0; st < S; ++st) {
        const int64_t g = grp0 + st * nwarps;
        if (g < ngroups) {
            const int32_t sl = (lane < kRecs && g * kRecs + lane < n) ? b.slots[off + g * kRecs + lane] : 0;
            issue(g, st, sl);
        }
    }
    int stage = 0;
    uint32_t phase = 0;
    // slot ids of refill groups are fetched two iterations before their copies are issued
    auto slot_of = [&](int64_t g) -> int32_t {
        return (g < ngroups && lane < kRecs && g * kRecs + lane < n) ? b.slots[off + g * kRecs + lane] : 0;
    };
    int32_t pf0 = slot_of(grp0 + S * nwarps), pf1 = slot_of(grp0 + (S + 1) * nwarps);
    for (int64_t grp = grp0; grp < ngroups; grp += nwarps) {
        const int64_t gn = grp + S * nwarps;  // group that refills this stage
        const int32_t nslot = pf0;
        pf0 = pf1;
        pf1 = slot_of(grp + (S + 2) * nwarps);
        mbar_wait(&wbar[stage], phase);
#endif
        const unsigned char* sb = wbuf + stage * STAGE;
        double acc[N];
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] = 0.0;
#pragma unroll
        for (int j = 0; j < kRecs; ++j) {
            const unsigned char* rec = sb + j * MB;
            const uint4 mv = *reinterpret_cast<const uint4*>(rec + lane * 16);
            const uint32_t mw[4] = {mv.x, mv.y, mv.z, mv.w};
            uint32_t lw[4], hw[4];
            if constexpr (sizeof(KV) == 2) {
                const uint2 lv = *reinterpret_cast<const uint2*>(rec + D * 4 + lane * 8);
                const uint2 hv = *reinterpret_cast<const uint2*>(rec + D * 4 + D * 2 + lane * 8);
                lw[0] = lv.x << 16; lw[1] = lv.x & 0xFFFF0000u; lw[2] = lv.y << 16; lw[3] = lv.y & 0xFFFF0000u;
                hw[0] = hv.x << 16; hw[1] = hv.x & 0xFFFF0000u; hw[2] = hv.y << 16; hw[3] = hv.y & 0xFFFF0000u;
            } else {
                const uint4 lv = *reinterpret_cast<const uint4*>(rec + D * 4 + lane * 16);
                const uint4 hv = *reinterpret_cast<const uint4*>(rec + D * 8 + lane * 16);
                lw[0] = lv.x; lw[1] = lv.y; lw[2] = lv.z; lw[3] = lv.w;
                hw[0] = hv.x; hw[1] = hv.y; hw[2] = hv.z; hw[3] = hv.w;
            }
#pragma unroll
            for (int jj = 0; jj < DPL; ++jj) {
#ifndef PSA_MEAN_F2F
#define PSA_MEAN_F2F 1  // measured: score 3.42 -> 3.22-3.33 ms
#endif
                // CuboidMean with PSA_MEAN_F2F: the mean converts with one F2F on the otherwise idle
                // XU pipe (true value) and the 2^-896 metadata scale is folded into A's DFMA
                // (exact: a power of two, fp32 denormals stay exact fp64 values)
#ifndef PSA_LO_F2F
#define PSA_LO_F2F 0
#endif
                constexpr bool kAll = PSA_ALL_F2F && est == 2;  // every conversion on the XU pipe, true scale
                constexpr bool kF2F = PSA_MEAN_F2F && est == 2 && !kAll;
                constexpr bool kLoF2F = PSA_LO_F2F && est != 0 && !kAll;  // lo's scale folded into c2 / B
                double A, B = 0.0;
                if constexpr (kAll) {
                    const double m = (double)__uint_as_float(mw[jj]);
                    const double lo = (double)__uint_as_float(lw[jj]);
                    const double hi = (double)__uint_as_float(hw[jj]);
                    B = hi - lo;                 // exact (bf16 operands)
                    A = fma(2.0, m, lo + hi);    // lo + hi exact in fp64
                } else {
                const double m = kF2F ? (double)__uint_as_float(mw[jj]) : f32_scaled(mw[jj]);
                const double lo = kLoF2F ? (double)__uint_as_float(lw[jj]) : f32_scaled(lw[jj]);
                const double hi = f32_scaled(hw[jj]);
                if (est == 0) {
                    A = m;
                } else {
                    const double c2 = kLoF2F ? fma(0x1p-896, lo, hi) : lo + hi;  // exact
                    B = kLoF2F ? fma(-0x1p-896, lo, hi) : hi - lo;             // 2r, exact
                    A = est == 2 ? fma(kF2F ? 0x1p-895 : 2.0, m, c2) : c2;       // 2(m + c)  |  2c
                }
                }
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    const double qv = qd[h][jj];
                    double a = fma(qv, A, acc[h * kRecs + j]);
                    if (est != 0) a = fma(fabs(qv), B, a);
                    acc[h * kRecs + j] = a;
                }
            }
        }
        // The consumed stage doubles as the reduction scratch when it is large enough
        // (N = 16 doubles x 32 lanes = 4 KB = one bf16 stage); then it is refilled.
        double tot;
        if constexpr (N == 16 && STAGE >= 4096) {
            tot = smem_reduce16_cm(acc, reinterpret_cast<double*>(wbuf + stage * STAGE), lane);
        } else {
            tot = smem_reduce<N>(acc, reinterpret_cast<double*>(smem + kTmaBarBytes + (size_t)kScoreWarps * S * STAGE) +
                                          warp * 32 * (N + 1),
                                 lane);
        }
        // every lane's shared-memory accesses of this stage precede the refill (generic -> async proxy)
        fence_proxy_async();
        __syncwarp();
#if PSA_SCORE_CHUNKED
        if (gn < g_end) issue(gn, stage, nslot);
#else
        if (gn < ngroups) issue(gn, stage, nslot);
#endif
        const int64_t p0 = grp * kRecs;
        if (writer && p0 + my_j < n) {
            const uint64_t key = make_key_masked(tot * kscale, (uint32_t)(p0 + my_j), kmask);
            keys[p0 + my_j] = key;
            kmin = key < kmin ? key : kmin;
            kmax = key > kmax ? key : kmax;
        }
        if (++stage == S) {
            stage = 0;
            phase ^= 1u;
        }
    }
    if (b.kminmax && writer && kmax != 0) {
        atomicMin(b.kminmax + (size_t)u * b.g + my_h, (unsigned long long)kmin);
        atomicMax(b.kminmax + b.kmm_stride + (size_t)u * b.g + my_h, (unsigned long long)kmax);
    }
}

template <typename KV, int G>
static size_t tma_smem_bytes() {
    constexpr int kRecs = RecsPer<G, 4>::v;
    constexpr int STAGE = kRecs * (128 * 4 + 2 * 128 * (int)sizeof(KV));
    constexpr int N = G * kRecs;
    constexpr bool kReuse = (N == 16 && STAGE >= 4096);
    constexpr int SB = kReuse ? PSA_SCORE_SB : 8192;
    constexpr int S = (SB / STAGE) < 2 ? 2 : ((SB / STAGE) > 4 ? 4 : (SB / STAGE));
    return kTmaBarBytes + (size_t)kScoreWarps * S * STAGE + (kReuse ? 0 : (size_t)kScoreWarps * 32 * (N + 1) * 8);
}

static int g_score_choice = 0;
void set_score_kernel_choice(int choice) { g_score_choice = choice; }
// Dynamic shared memory floor of the score kernel. In the two-stream pipeline the score
// kernel is held to ONE CTA per SM (its ~98 KB ring padded past half of the SM's 228 KB)
// so a progressive CTA (~105 KB, 128 regs x 256) can be co-resident on every SM.
static size_t g_score_smem_floor = 0;

template <typename KV, int G>
static void launch_score_tma(const PoolView& p, const BatchView& b, dim3 grid, cudaStream_t st) {
    size_t smem = tma_smem_bytes<KV, G>();
    if (smem < g_score_smem_floor) smem = g_score_smem_floor;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, kScoreWarps * 32, smem, st>>>(p, b);
    };
    if (b.estimator == 0) go(score_kernel_tma<KV, G, 0>);
    else if (b.estimator == 1) go(score_kernel_tma<KV, G, 1>);
    else go(score_kernel_tma<KV, G, 2>);
}

// =============================================================================
// K6: fp64 block masses log(sum_t exp(q.k_t*scale)) for Oracle ranking and the
// coverage audit (reference engine.cpp:64-72 computes these in plan_blocks).
// Test/audit mode only; not on the benchmarked path.
// =============================================================================
template <typename KV, int DPL>
__global__ void __launch_bounds__(kScoreWarps * 32) oracle_mass_kernel(PoolView p, BatchView b) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int u = blockIdx.y;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int d = b.d;
    const int base = lane * DPL;
    const int lim = d - base;
    const bool full = (d == 32 * DPL);
    for (int64_t pos = (int64_t)blockIdx.x * kScoreWarps + warp; pos < n; pos += (int64_t)gridDim.x * kScoreWarps) {
        const int32_t slot = b.slots[off + pos];
        const int nt = p.ntok[slot];
        const KV* k = kv_block<KV>(p, slot) + base;
        for (int h = 0; h < b.g; ++h) {
            float qf[DPL];
            load_row<DPL>(b.q + ((size_t)u * b.g + h) * d + base, full, lim, qf);
            double mx = -INFINITY, es = 0.0;
            // two passes like the reference: max, then sum of exp
            for (int pass = 0; pass < 2; ++pass) {
                for (int t = 0; t < nt; ++t) {
                    float kf[DPL];
                    load_row<DPL>(k + (size_t)t * d, full, lim, kf);
                    double a = 0.0;
#pragma unroll
                    for (int j = 0; j < DPL; ++j) a = fma((double)qf[j], (double)kf[j], a);
                    const double s = warp_sum_d(a) * b.scale;
                    if (pass == 0) mx = fmax(mx, s);
                    else es += exp(s - mx);
                }
            }
            const double la = mx + log(es);
            const int64_t idx = off * b.g + (int64_t)h * n + pos;
            if (lane == 0) {
                b.omass[idx] = la;
                if (b.rank_oracle) b.keys[idx] = make_key(la, (uint32_t)pos, b.pos_bits);
            }
        }
    }
}

// =============================================================================
// GQA union of processed blocks per unit (for the algorithmic byte count).
// =============================================================================
__global__ void union_kernel(BatchView b, int64_t* out) {
    extern __shared__ uint32_t bits[];
    const int u = blockIdx.x;
    const int64_t off = b.list_off[u];
    const int64_t n = b.list_off[u + 1] - off;
    const int64_t words = (n + 31) / 32;
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) bits[i] = 0;
    __syncthreads();
    for (int h = 0; h < b.g; ++h) {
        const int64_t hb = off * b.g + (int64_t)h * n;
        const int64_t bp = b.bp[(int64_t)u * b.g + h];
        for (int64_t r = threadIdx.x; r < bp; r += blockDim.x) {
            const int32_t pos = b.rpos[hb + r];
            atomicOr(&bits[pos >> 5], 1u << (pos & 31));
        }
    }
    __syncthreads();
    __shared__ unsigned long long total;
    if (threadIdx.x == 0) total = 0;
    __syncthreads();
    unsigned long long c = 0;
    for (int64_t i = threadIdx.x; i < words; i += blockDim.x) c += __popc(bits[i]);
    atomicAdd(&total, c);
    __syncthreads();
    if (threadIdx.x == 0) out[u] = (int64_t)total;
}

cudaError_t launch_union(const BatchView& b, int64_t* out, cudaStream_t st) {
    const size_t smem = (size_t)((b.max_n + 31) / 32) * 4;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    if (smem > 48 * 1024) cudaFuncSetAttribute(union_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    union_kernel<<<b.n_units, 512, smem, st>>>(b, out);
    return cudaGetLastError();
}

// =============================================================================
// Launch dispatch
// =============================================================================
template <typename KV, int G>
static void launch_score_g(const PoolView& p, const BatchView& b, dim3 grid, cudaStream_t st) {
    switch (dpl_for(b.d)) {  // d=64 and d=128 are always "full"; other d use the masked 8-dim path
        case 2: score_kernel<KV, G, 2, true><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
        case 4: score_kernel<KV, G, 4, true><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
        default:
            if (b.d == 256) score_kernel<KV, G, 8, true><<<grid, kScoreWarps * 32, 0, st>>>(p, b);
            else score_kernel<KV, G, 8, false><<<grid, kScoreWarps * 32, 0, st>>>(p, b);
            break;
    }
}

template <typename KV>
static void launch_score(const PoolView& p, const BatchView& b, dim3 grid, cudaStream_t st) {
    if (g_score_choice != 1 && b.d == 128 && p.meta_bytes == 128 * 4 + 2 * 128 * (int64_t)sizeof(KV)) {  // TMA path
        if (g_for(b.g) == 4) launch_score_tma<KV, 4>(p, b, grid, st);
        else launch_score_tma<KV, 8>(p, b, grid, st);
        return;
    }
    if (g_for(b.g) == 4) launch_score_g<KV, 4>(p, b, grid, st);
    else launch_score_g<KV, 8>(p, b, grid, st);
}

template <typename KV>
static void launch_oracle(const PoolView& p, const BatchView& b, dim3 grid, cudaStream_t st) {
    switch (dpl_for(b.d)) {
        case 2: oracle_mass_kernel<KV, 2><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
        case 4: oracle_mass_kernel<KV, 4><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
        default: oracle_mass_kernel<KV, 8><<<grid, kScoreWarps * 32, 0, st>>>(p, b); break;
    }
}

static int g_pipeline = 0;  // 0 auto, 1 off, k > 1: k sub-batches
void set_pipeline_subbatches(int k) { g_pipeline = k; }

// Units [u0, u0 + cnt) of a batch: unit-indexed arrays are offset, the workspace
// (keys / ranked positions / masses, indexed by absolute list offsets) is shared.
static BatchView sub_view(const BatchView& b, int u0, int cnt, int idx) {
    BatchView v = b;
    const size_t qo = (size_t)u0 * b.g;
    v.n_units = cnt;
    v.q = b.q + qo * b.d;
    v.list_off = b.list_off + u0;
    v.out = b.out + qo * b.d;
    v.bp = b.bp + qo;
    v.est = b.est + qo;
    v.tcov = b.tcov ? b.tcov + qo : nullptr;
    v.term = b.term + qo;
    if (b.kminmax) v.kminmax = b.kminmax + qo;  // (the max half stays kmm_stride further)
    if (b.dense_flag) {  // each sub-batch keeps its own hand-over list and counter
        v.dense_flag = b.dense_flag + u0;
        v.dense_count = b.dense_count + idx;
        v.dense_thr = b.dense_thr + qo;
        v.dense_sel = b.dense_sel + qo;
        v.dense_esc = b.dense_esc + u0;
        v.dense_esc_count = b.dense_esc_count + idx;
        v.dense_esc_mark = b.dense_esc_mark + u0;
        // the workspace holds ceil(max_n / kDenseSlice) partial states per head (the most any slicing uses)
        v.dense_part = b.dense_part + qo * (size_t)((b.max_n + kDenseSlice - 1) / kDenseSlice) * kDensePart;
    }
    if (b.stream_w) v.stream_w = b.stream_w + (size_t)u0 * kStreamEnt * kStreamWRow;
    if (b.ft_keys) {  // head-indexed [n_units*g][kFirstCap]: offset to the sub-batch's heads
        v.ft_keys = b.ft_keys + qo * kFirstCap;
        v.ft_slot = b.ft_slot + qo * kFirstCap;
        v.ft_ntok = b.ft_ntok + qo * kFirstCap;
        v.ft_count = b.ft_count + qo;
    }
    return v;
}

static void launch_score_stage(const PoolView& p, const BatchView& b, cudaStream_t st) {
    // enough CTAs for ~2 waves of 2 CTAs/SM, never more warps than record groups
    const int64_t groups = (b.max_n + 3) / 4;
    int64_t gx = (2LL * 2 * num_sms() + b.n_units - 1) / b.n_units;
    const int64_t gx_max = (groups + kScoreWarps - 1) / kScoreWarps;
    if (gx > gx_max) gx = gx_max;
    if (gx < 1) gx = 1;
    dim3 grid((unsigned)gx, (unsigned)b.n_units);
    if (p.dtype == 0) launch_score<float>(p, b, grid, st);
    else launch_score<__nv_bfloat16>(p, b, grid, st);
}

struct PipeResources {
    cudaStream_t aux = nullptr;
    cudaEvent_t ev[17] = {};
    bool ok = false;
};

static PipeResources& pipe_resources() {
    static PipeResources r;
    if (!r.ok) {
        if (cudaStreamCreateWithFlags(&r.aux, cudaStreamNonBlocking) != cudaSuccess) return r;
        for (auto& e : r.ev)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return r;
        r.ok = true;
    }
    return r;
}

int launch_batch(const PoolView& p, const BatchView& b, cudaStream_t st, cudaEvent_t* marks) {
    // marks (optional, 5 events): start | oracle | score | order | progressive. Ordering is
    // fused into the progressive kernel (lazy tranche selection), so the "order" stage is empty.
    int launches = 0;
    int subs = g_pipeline == 0 ? 1 : g_pipeline;  // measured: overlap does not pay (both stages are SM-bound)
    if (subs > 16) subs = 16;
    if (subs > b.n_units) subs = b.n_units;
    if (marks) cudaEventRecord(marks[0], st);
    if (b.has_oracle || b.rank_oracle || subs <= 1 || !pipe_resources().ok) {
        if (b.has_oracle) {
            const int64_t chunks = (b.max_n + kScoreWarps - 1) / kScoreWarps;
            dim3 grid((unsigned)(chunks < 65535 ? (chunks > 0 ? chunks : 1) : 65535), (unsigned)b.n_units);
            if (p.dtype == 0) launch_oracle<float>(p, b, grid, st);
            else launch_oracle<__nv_bfloat16>(p, b, grid, st);
            ++launches;
        }
        if (marks) cudaEventRecord(marks[1], st);
        if (!b.rank_oracle) {
            if (b.kminmax) {
                const size_t nq = (size_t)b.n_units * b.g;
                cudaMemsetAsync(b.kminmax, 0xff, nq * 8, st);
                cudaMemsetAsync(b.kminmax + nq, 0, nq * 8, st);
            }
            launch_score_stage(p, b, st);
            ++launches;
        }
        if (marks) cudaEventRecord(marks[2], st);
        if (marks) cudaEventRecord(marks[3], st);
        launches += launch_psa(p, b, st);
        if (marks) cudaEventRecord(marks[4], st);
    } else {
        // Two-stream pipeline over sub-batches of units: score(i+1) streams metadata from HBM
        // on `st` while progressive(i) runs on the auxiliary stream. Stream-ordered (events),
        // no host synchronisation; the caller's stream joins the auxiliary one at the end.
        // The auxiliary stream, its events and the score kernel's smem floor are process-wide:
        // concurrent callers serialise their enqueues here.
        static std::mutex pipe_mutex;
        std::lock_guard<std::mutex> lock(pipe_mutex);
        PipeResources& r = pipe_resources();
        static const size_t floor_env = [] {
            const char* e = getenv("PSA_SCORE_SMEM_FLOOR");
            return e ? (size_t)atol(e) : (size_t)(116 * 1024);
        }();
        g_score_smem_floor = floor_env;
        if (marks) cudaEventRecord(marks[1], st);
        if (b.kminmax) {
            const size_t nq = (size_t)b.n_units * b.g;
            cudaMemsetAsync(b.kminmax, 0xff, nq * 8, st);
            cudaMemsetAsync(b.kminmax + nq, 0, nq * 8, st);
        }
        cudaEventRecord(r.ev[0], st);
        cudaStreamWaitEvent(r.aux, r.ev[0], 0);
        const int per = (b.n_units + subs - 1) / subs;
        int i = 0;
        for (int u0 = 0; u0 < b.n_units; u0 += per, ++i) {
            const int cnt = (b.n_units - u0) < per ? (b.n_units - u0) : per;
            const BatchView v = sub_view(b, u0, cnt, i);
            launch_score_stage(p, v, st);
            cudaEventRecord(r.ev[1 + i], st);
            cudaStreamWaitEvent(r.aux, r.ev[1 + i], 0);
            launches += 1 + launch_psa(p, v, r.aux);
        }
        g_score_smem_floor = 0;
        if (marks) cudaEventRecord(marks[2], st);  // score chain done (progressive overlapped)
        if (marks) cudaEventRecord(marks[3], st);
        cudaEventRecord(r.ev[0], r.aux);
        cudaStreamWaitEvent(st, r.ev[0], 0);
        if (marks) cudaEventRecord(marks[4], st);  // exposed progressive tail
    }
    if (cudaPeekAtLastError() != cudaSuccess) return -1;
    return launches;
}

// Sort keys of every (unit, head) for a full ranking (psattn_rank_batch): fp64 oracle masses
// (Oracle ranking / audit) and/or criticality scores, nothing else. Returns launches or -1.
int launch_rank_keys(const PoolView& p, const BatchView& b, cudaStream_t st) {
    int launches = 0;
    if (b.has_oracle) {
        const int64_t chunks = (b.max_n + kScoreWarps - 1) / kScoreWarps;
        dim3 grid((unsigned)(chunks < 65535 ? (chunks > 0 ? chunks : 1) : 65535), (unsigned)b.n_units);
        if (p.dtype == 0) launch_oracle<float>(p, b, grid, st);
        else launch_oracle<__nv_bfloat16>(p, b, grid, st);
        ++launches;
    }
    if (!b.rank_oracle) {
        launch_score_stage(p, b, st);
        ++launches;
    }
    return cudaPeekAtLastError() == cudaSuccess ? launches : -1;
}

}  // namespace psa
