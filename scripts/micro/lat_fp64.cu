// Latency microbenchmark (development only): dependent-chain cycles of the fp64 /
// int64 operations the coverage decide step uses, on one warp.
#include <cstdio>
#include <cstdint>
#include "../../paper_2503_00392_b200/csrc/psa_order.cuh"

__global__ void lat(double* out, long long* cyc, int m, int64_t n) {
    double x = 0.001 * threadIdx.x, acc = -INFINITY, mn = INFINITY;
    long long t0, t1;
    const int R = 64;
    // exp chain
    t0 = clock64();
    for (int i = 0; i < R; ++i) x = exp(x) * 1e-3;
    t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / R;
    t0 = clock64();
    for (int i = 0; i < R; ++i) x = log(x + 2.0);
    t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / R;
    t0 = clock64();
    for (int i = 0; i < R; ++i) x = 1.0 / (x + 1.5);
    t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / R;
    int64_t r = threadIdx.x + n;
    t0 = clock64();
    for (int i = 0; i < R; ++i) r = r % m + n + (int64_t)x;
    t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / R;
    t0 = clock64();
    for (int i = 0; i < R; ++i) x = fma(x, 0.999, 1e-3);
    t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / R;
    float f = x;
    t0 = clock64();
    for (int i = 0; i < R; ++i) f = fmaf(f, 0.999f, 1e-3f);
    t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / R;
    t0 = clock64();
    for (int i = 0; i < R; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-3;
    t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / R;
    // decide_chunk chain
    int cb = 0;
    t0 = clock64();
    for (int i = 0; i < R; ++i) {
        psa::Decision d = psa::decide_chunk(-0.01 * (threadIdx.x + i) + x * 1e-9, 32, cb, n, n, m, 0.999999, acc, mn, nullptr);
        cb += d.commit;
    }
    t1 = clock64(); if (threadIdx.x == 0) cyc[7] = (t1 - t0) / R;
    out[threadIdx.x] = x + f + (double)r + acc + mn + cb;
}

int main() {
    double* o; long long* c;
    cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 16 * 8);
    for (int rep = 0; rep < 2; ++rep) lat<<<1, 32>>>(o, c, 1, 8192);
    long long h[16];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    const char* nm[] = {"exp_f64", "log_f64", "div_f64", "mod_i64", "dfma", "ffma", "shfl_f64+dadd", "decide_chunk"};
    for (int i = 0; i < 8; ++i) printf("%s %lld cycles\n", nm[i], h[i]);
    return 0;
}
