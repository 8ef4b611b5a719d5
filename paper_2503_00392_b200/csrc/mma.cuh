// mma.cuh — warp-level tensor-core helpers (mma.sync, bf16 in / fp32 accumulate).
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace psa {

__device__ __forceinline__ void mma_bf16_16816(float& c0, float& c1, float& c2, float& c3, uint32_t a0, uint32_t a1,
                                               uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c0), "+f"(c1), "+f"(c2), "+f"(c3)
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t bf16_bits(float x) { return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x)); }

// Two fp32 -> packed bf16x2 (round to nearest even), element a in the low half: one cvt.
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&v);
}
// Packed 2-term split of a pair: part 0 = rn(x), part 1 = rn(x - rn(x)) (as bf16_split(x, 0/1)).
__device__ __forceinline__ uint32_t pack_bf16x2_split(float a, float b, int part) {
    const uint32_t p = pack_bf16x2(a, b);
    if (part == 0) return p;
    return pack_bf16x2(a - __uint_as_float(p << 16), b - __uint_as_float(p & 0xFFFF0000u));
}


// Term `part` (0..2) of the exact 3-term bf16 split of a and b, packed (a low); part 3 -> 0.
// Branch-free: every lane computes the three terms and selects its own (lanes hold different parts).
__device__ __forceinline__ uint32_t pack_split3(float a, float b, int part) {
    const uint32_t p1 = pack_bf16x2(a, b);
    const float a1 = a - __uint_as_float(p1 << 16), b1 = b - __uint_as_float(p1 & 0xFFFF0000u);
    const uint32_t p2 = pack_bf16x2(a1, b1);
    const float a2 = a1 - __uint_as_float(p2 << 16), b2 = b1 - __uint_as_float(p2 & 0xFFFF0000u);
    const uint32_t p3 = pack_bf16x2(a2, b2);
    return part == 0 ? p1 : part == 1 ? p2 : part == 2 ? p3 : 0u;
}

// Exact 3-term bf16 split of an fp32 value: x == x1 + x2 + x3 (split index 0..2; 3+ -> 0).
__device__ __forceinline__ float bf16_split(float x, int part) {
    const float x1 = __bfloat162float(__float2bfloat16_rn(x));
    const float r1 = x - x1;
    const float x2 = __bfloat162float(__float2bfloat16_rn(r1));
    const float r2 = r1 - x2;
    return part == 0 ? x : (part == 1 ? r1 : (part == 2 ? r2 : 0.0f));
}

}  // namespace psa
