// synth.h — seekable synthetic KV/query generator, identical on host and device.
//
// Workload fixture for the benchmark and the parity tests, NOT part of the
// attention path. It keeps the *pattern* of the reference generator
// (workload.cpp:84-148: planted blocks whose keys are skew*direction + noise,
// per-block value centroids + 0.25 noise, queries near the planted direction
// with norm sqrt(d)) but is counter-based, so any (unit, block, token, dim)
// can be produced independently — the reference's sequential mt19937_64 cannot
// generate a 128K x 32-layer slice without replaying everything before it.
//
// Bit-identity host <-> device: only integer hashing, int->float conversion and
// single IEEE-rounded float/double operations (no contraction: device code uses
// the explicit _rn intrinsics, host code is compiled with -ffp-contract=off).
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define PSA_HD __host__ __device__ __forceinline__
#else
#define PSA_HD static inline
#endif

namespace psa_synth {

PSA_HD uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

PSA_HD uint64_t hash4(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
    uint64_t h = mix64(seed ^ (stream * 0x9E3779B97F4A7C15ULL));
    h = mix64(h + a * 0xD1B54A32D192ED03ULL);
    return mix64(h ^ (b + 0x8CB92BA72F3D8DD7ULL));
}

PSA_HD float fmul(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fmul_rn(a, b);
#else
    return a * b;
#endif
}
PSA_HD float fadd(float a, float b) {
#if defined(__CUDA_ARCH__)
    return __fadd_rn(a, b);
#else
    return a + b;
#endif
}
PSA_HD double dmul(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
PSA_HD double dadd(double a, double b) {
#if defined(__CUDA_ARCH__)
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}

// Approximately N(0,1): centred sum of four 16-bit uniforms (Irwin-Hall, std 1,
// support +-3.46). Exact integer sum, one rounded multiply.
PSA_HD float normal_from(uint64_t h) {
    const int32_t s = (int32_t)(h & 0xFFFF) + (int32_t)((h >> 16) & 0xFFFF) +
                      (int32_t)((h >> 32) & 0xFFFF) + (int32_t)(h >> 48);
    return fmul((float)(s - 131070), 2.6428806e-05f);  // 1 / (65536/sqrt(3))
}

PSA_HD uint32_t f2u(float x) {
#if defined(__CUDA_ARCH__)
    return __float_as_uint(x);
#else
    uint32_t u;
    memcpy(&u, &x, 4);
    return u;
#endif
}
PSA_HD float u2f(uint32_t u) {
#if defined(__CUDA_ARCH__)
    return __uint_as_float(u);
#else
    float x;
    memcpy(&x, &u, 4);
    return x;
#endif
}

// Round-to-nearest-even to bf16, returned as the float it represents.
PSA_HD float round_bf16(float x) {
    uint32_t u = f2u(x);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return u2f(u & 0xFFFF0000u);
}

enum : uint64_t { S_KEY = 1, S_VAL = 2, S_CENTROID = 3, S_PLANT = 5, S_DIR = 6, S_QUERY = 7 };

PSA_HD int is_planted(uint64_t seed, float prob, int64_t unit, int64_t block) {
    if (!(prob > 0.0f)) return 0;
    const uint64_t h = hash4(seed, S_PLANT, (uint64_t)unit, (uint64_t)block);
    return fmul((float)(uint32_t)(h >> 40), 5.9604645e-08f) < prob;  // 24-bit uniform
}

// Unit-norm direction for a unit; sequential fp64 norm, correctly rounded sqrt/div.
PSA_HD void direction(uint64_t seed, int64_t unit, int32_t d, float* out) {
    double ss = 0.0;
    for (int32_t i = 0; i < d; ++i) {
        const float g = normal_from(hash4(seed, S_DIR, (uint64_t)unit, (uint64_t)i));
        out[i] = g;
        ss = dadd(ss, dmul((double)g, (double)g));
    }
#if defined(__CUDA_ARCH__)
    const double inv = __ddiv_rn(1.0, __dsqrt_rn(ss));
#else
    const double inv = 1.0 / __builtin_sqrt(ss);
#endif
    for (int32_t i = 0; i < d; ++i) out[i] = (float)dmul((double)out[i], inv);
}

// Key element (unit, token, dim) given the unit's direction value dir_i.
PSA_HD float key_at(uint64_t seed, int64_t unit, int64_t token, int32_t i, int32_t d, int planted,
                    float skew, float dir_i) {
    float x = normal_from(hash4(seed, S_KEY, (uint64_t)unit, (uint64_t)(token * d + i)));
    if (planted) x = fadd(x, fmul(skew, dir_i));
    return x;
}

PSA_HD float value_at(uint64_t seed, int64_t unit, int64_t block, int64_t token, int32_t i, int32_t d) {
    const float c = normal_from(hash4(seed, S_CENTROID, (uint64_t)unit, (uint64_t)(block * d + i)));
    const float e = normal_from(hash4(seed, S_VAL, (uint64_t)unit, (uint64_t)(token * d + i)));
    return fadd(c, fmul(0.25f, e));
}

}  // namespace psa_synth
