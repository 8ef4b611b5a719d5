// common.cuh — device helpers shared by the PSA kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define PSA_FULL 0xffffffffu

namespace psa {

// ---- KV element types ------------------------------------------------------
template <typename KV> struct KVT;
template <> struct KVT<float> {
    static constexpr int kBytes = 4;
    __device__ __forceinline__ static float to_f(float x) { return x; }
    __device__ __forceinline__ static float from_f(float x) { return x; }
};
template <> struct KVT<__nv_bfloat16> {
    static constexpr int kBytes = 2;
    __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
    __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

// Loads DPL consecutive KV elements starting at p (lane-contiguous mapping) as
// floats. `full` = all DPL elements valid and the address is DPL-aligned; else
// element-wise with the [0, lim) bound.
template <int DPL>
__device__ __forceinline__ void load_row(const float* __restrict__ p, bool full, int lim, float (&o)[DPL]) {
    if (full) {
        if constexpr (DPL % 4 == 0) {
#pragma unroll
            for (int j = 0; j < DPL; j += 4) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(p + j));
                o[j] = v.x; o[j + 1] = v.y; o[j + 2] = v.z; o[j + 3] = v.w;
            }
        } else if constexpr (DPL == 2) {
            const float2 v = __ldg(reinterpret_cast<const float2*>(p));
            o[0] = v.x; o[1] = v.y;
        } else {
#pragma unroll
            for (int j = 0; j < DPL; ++j) o[j] = __ldg(p + j);
        }
    } else {
#pragma unroll
        for (int j = 0; j < DPL; ++j) o[j] = j < lim ? __ldg(p + j) : 0.0f;
    }
}

template <int DPL>
__device__ __forceinline__ void load_row(const __nv_bfloat16* __restrict__ p, bool full, int lim, float (&o)[DPL]) {
    if (full) {
        if constexpr (DPL % 8 == 0) {
#pragma unroll
            for (int j = 0; j < DPL; j += 8) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(p + j));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    o[j + 2 * k] = __uint_as_float(w[k] << 16);
                    o[j + 2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
                }
            }
        } else if constexpr (DPL % 4 == 0) {
#pragma unroll
            for (int j = 0; j < DPL; j += 4) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(p + j));
                o[j] = __uint_as_float(v.x << 16);
                o[j + 1] = __uint_as_float(v.x & 0xffff0000u);
                o[j + 2] = __uint_as_float(v.y << 16);
                o[j + 3] = __uint_as_float(v.y & 0xffff0000u);
            }
        } else {
#pragma unroll
            for (int j = 0; j < DPL; ++j) o[j] = __bfloat162float(p[j]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < DPL; ++j) o[j] = j < lim ? __bfloat162float(p[j]) : 0.0f;
    }
}

// ---- warp reductions --------------------------------------------------------
__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x = fmaxf(x, __shfl_xor_sync(PSA_FULL, x, o));
    return x;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(PSA_FULL, x, o);
    return x;
}
__device__ __forceinline__ double warp_max_d(double x) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x = fmax(x, __shfl_xor_sync(PSA_FULL, x, o));
    return x;
}
__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(PSA_FULL, x, o);
    return x;
}

// Reduce-scatter of N per-lane values (N power of two, <= 32) across the warp:
// returns the warp-wide total of index (lane >> (5 - log2 N)); every index ends
// on 32/N lanes. N-1 + log2(32/N) shuffles instead of 5N for N all-reduces.
template <int N>
__device__ __forceinline__ float reduce_scatter(float (&v)[N], int lane) {
    int o = 16;
#pragma unroll
    for (int n = N; n > 1; n >>= 1, o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            const float send = upper ? v[i] : v[i + n / 2];
            const float keep = upper ? v[i + n / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(PSA_FULL, send, o);
        }
    }
    float x = v[0];
#pragma unroll
    for (; o >= 1; o >>= 1) x += __shfl_xor_sync(PSA_FULL, x, o);
    return x;
}

template <int N>
__device__ __forceinline__ double reduce_scatter_d(double (&v)[N], int lane) {
    int o = 16;
#pragma unroll
    for (int n = N; n > 1; n >>= 1, o >>= 1) {
        const bool upper = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            const double send = upper ? v[i] : v[i + n / 2];
            const double keep = upper ? v[i + n / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(PSA_FULL, send, o);
        }
    }
    double x = v[0];
#pragma unroll
    for (; o >= 1; o >>= 1) x += __shfl_xor_sync(PSA_FULL, x, o);
    return x;
}

template <int N> struct Log2 { static constexpr int v = 1 + Log2<N / 2>::v; };
template <> struct Log2<1> { static constexpr int v = 0; };

// ---- sort keys ---------------------------------------------------------------
// Ascending key order == (score descending, list position ascending), with the
// low `pos_bits` bits carrying the list position: scores that agree in all but
// their last pos_bits key bits (relative 2^-(52-pos_bits)) compare by position,
// i.e. by block id — the reference's tie rule (metadata.cpp:92-93).
__device__ __forceinline__ uint64_t make_key_masked(double s, uint32_t pos, uint64_t mask) {
    s = s + 0.0;  // -0 -> +0: the reference compares doubles, where -0 == +0
    const uint64_t u = (uint64_t)__double_as_longlong(s);
    const uint64_t asc = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
    const uint64_t desc = ~asc;
    return (desc & ~mask) | ((uint64_t)pos & mask);  // mask == 0: the pure score key (full rankings)
}
__device__ __forceinline__ uint64_t make_key(double s, uint32_t pos, int pos_bits) {
    return make_key_masked(s, pos, (pos_bits >= 64) ? ~0ull : ((1ull << pos_bits) - 1ull));
}
// Inverse of make_key_masked up to the position bits: the score a key encodes (those bits set).
__device__ __forceinline__ double key_score(uint64_t k, uint64_t pmask) {
    const uint64_t asc = ~k | pmask;
    const uint64_t u = (asc >> 63) ? (asc & 0x7FFFFFFFFFFFFFFFull) : ~asc;
    return __longlong_as_double((long long)u);
}

}  // namespace psa

// ---- TMA bulk copies + mbarriers (sm_90+/sm_100a PTX) ----------------------
namespace psa {
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
// try_wait with a suspend-time hint: the waiting thread is suspended until the phase completes
// (or ~1 ms passes) instead of spinning, so waiting warps do not take issue slots from the warps
// doing the work (measured on the stream kernel: ~40% of its issued instructions were polls).
__device__ __forceinline__ bool mbar_try_wait_suspend(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase), "r"(1000000u)
        : "memory");
    return ok != 0;
}
// Same with a caller-chosen suspend bound (ns): a polling agent parks on its most likely next
// event without spinning.
__device__ __forceinline__ bool mbar_try_wait_for(uint64_t* bar, uint32_t phase, uint32_t ns) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase), "r"(ns)
        : "memory");
    return ok != 0;
}
#ifndef PSA_MBAR_SUSPEND
#define PSA_MBAR_SUSPEND 1
#endif
// Waits for the phase; traps (kernel error, never a silent hang) if it does not complete
// within ~2^13 suspended polls (seconds) / ~2^26 plain polls.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#if PSA_MBAR_SUSPEND
    for (uint32_t i = 0; !mbar_try_wait_suspend(bar, phase); ++i)
        if (i > (1u << 13)) __trap();
#else
    for (uint32_t i = 0; !mbar_try_wait(bar, phase); ++i)
        if (i > (1u << 26)) __trap();
#endif
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0, 16 B aligned).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                           uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// Bulk L2 prefetch of [p, p + bytes) (16 B aligned, bytes % 16 == 0): one instruction per block.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// L2 prefetch of the line holding p (one lane, one line).
__device__ __forceinline__ void prefetch_l2_line(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
}  // namespace psa
