// attention_kernels.cu — device side of include/psattn/attention.hpp (reference
// include/psattn/attention.hpp:39-109 and src/attention.cpp:7-79): the per-call partial
// attention of one token sequence, the softmax merge and finalize, the fp64 oracles.
//
// One CTA per call, the reference's arithmetic order kept exactly: a token's score is the
// sequential sum over d of rounded products (no FMA contraction), times scale; the max is
// order-free; the token weights are independent exponentials; the exponent sum and every
// dim of the weighted value sum run in token order. Arbitrary token counts and dims (the
// scores live in a global scratch row). These serve API calls, not the batched decode step.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <string>

#include "device.h"

namespace psa {
namespace {

constexpr int kThreads = 256;

template <typename T>
struct Arith;
template <>
struct Arith<float> {
    static __device__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ float div(float a, float b) { return __fdiv_rn(a, b); }
    static __device__ float ex(float a) { return expf(a); }
    static __device__ float lg(float a) { return logf(a); }
};
template <>
struct Arith<double> {
    static __device__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ double div(double a, double b) { return __ddiv_rn(a, b); }
    static __device__ double ex(double a) { return exp(a); }
    static __device__ double lg(double a) { return log(a); }
};

// w: [n] scratch. out: [d] (unnormalised, or divided by the exponent sum when `normalize`).
// st: [3] = max score, exponent sum, log mass. With V == nullptr only the mass is computed.
template <typename T>
__global__ void __launch_bounds__(kThreads) seq_attention_kernel(const float* __restrict__ q, int d,
                                                                  const float* __restrict__ K,
                                                                  const float* __restrict__ V, int64_t n, T scale,
                                                                  int normalize, T* __restrict__ w, T* __restrict__ out,
                                                                  T* __restrict__ st) {
    using A = Arith<T>;
    __shared__ T red[kThreads / 32];
    __shared__ T s_max, s_sum;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    T mx = -INFINITY;
    for (int64_t t = tid; t < n; t += kThreads) {
        const float* k = K + t * d;
        T acc = 0;
        for (int i = 0; i < d; ++i) acc = A::add(acc, A::mul((T)q[i], (T)k[i]));
        const T s = A::mul(acc, scale);
        w[t] = s;
        mx = s > mx ? s : mx;
    }
    for (int o = 16; o; o >>= 1) {
        const T y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (tid == 0) {
        T m = red[0];
        for (int i = 1; i < kThreads / 32; ++i) m = red[i] > m ? red[i] : m;
        s_max = m;
    }
    __syncthreads();
    mx = s_max;
    for (int64_t t = tid; t < n; t += kThreads) w[t] = A::ex(w[t] - mx);  // token weights, own thread's rows
    __syncthreads();
    if (tid == 0) {
        T es = 0;
        for (int64_t t = 0; t < n; ++t) es = A::add(es, w[t]);
        s_sum = es;
        st[0] = mx;
        st[1] = es;
        st[2] = mx + A::lg(es);
    }
    if (V) {
        for (int i = tid; i < d; i += kThreads) {
            T o = 0;
            for (int64_t t = 0; t < n; ++t) o = A::add(o, A::mul(w[t], (T)V[t * d + i]));
            out[i] = o;
        }
    }
    __syncthreads();
    if (V && normalize)
        for (int i = tid; i < d; i += kThreads) out[i] = A::div(out[i], s_sum);
}

// merge_partial (attention.hpp:81-101) on a non-empty accumulator: both sides rescaled to the
// common max. in: acc_out[d], part_out[d]; sc: [6] = acc max, acc sum, part max, part sum.
template <typename T>
__global__ void __launch_bounds__(kThreads) merge_kernel(T* __restrict__ acc_out, const T* __restrict__ part_out, int d,
                                                        T* __restrict__ sc) {
    using A = Arith<T>;
    const T am = sc[0], as = sc[1], pm = sc[2], ps = sc[3];
    const T m = am > pm ? am : pm;
    const T fa = A::ex(am - m), fp = A::ex(pm - m);
    for (int i = threadIdx.x; i < d; i += kThreads) acc_out[i] = A::add(A::mul(acc_out[i], fa), A::mul(part_out[i], fp));
    if (threadIdx.x == 0) {
        const T es = A::add(A::mul(as, fa), A::mul(ps, fp));
        sc[0] = m;
        sc[1] = es;
        sc[4] = m + A::lg(es);
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) finalize_kernel(const T* __restrict__ acc_out, int d, T es, T* __restrict__ out) {
    for (int i = threadIdx.x; i < d; i += kThreads) out[i] = Arith<T>::div(acc_out[i], es);
}

// Device buffers of one call, released on every path.
struct Scratch {
    void* p = nullptr;
    ~Scratch() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t bytes) { return cudaMalloc(&p, bytes ? bytes : 1); }
};

int have_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        return fail(PSATTN_ERR_RUNTIME, "attention API: no CUDA device (no CPU fallback)");
    return PSATTN_OK;
}

template <typename T>
int seq_attention_impl(const float* q, int d, const float* K, const float* V, int64_t n, T scale, int normalize,
                       T* out, T* stats) {
    if (int rc = have_device()) return rc;
    const size_t kv = (size_t)n * d * sizeof(float);
    const size_t bytes = d * sizeof(float) + (V ? 2 : 1) * kv + (size_t)n * sizeof(T) + (d + 3) * sizeof(T) + 64;
    Scratch s;
    cudaError_t e = s.alloc(bytes);
    if (e != cudaSuccess) return cuda_fail(e, "attention API: allocation");
    char* base = static_cast<char*>(s.p);
    T* w = reinterpret_cast<T*>(base);
    T* o = w + n;
    T* st = o + d;
    float* dq = reinterpret_cast<float*>(st + 3);
    float* dk = dq + d;
    float* dv = V ? dk + (size_t)n * d : nullptr;
    e = cudaMemcpy(dq, q, d * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dk, K, kv, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && V) e = cudaMemcpy(dv, V, kv, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "attention API: upload");
    seq_attention_kernel<T><<<1, kThreads>>>(dq, d, dk, dv, n, scale, normalize, w, o, st);
    e = cudaGetLastError();
    if (e == cudaSuccess && V) e = cudaMemcpy(out, o, d * sizeof(T), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(stats, st, 3 * sizeof(T), cudaMemcpyDeviceToHost);
    return e == cudaSuccess ? PSATTN_OK : cuda_fail(e, "attention API: kernel");
}

template <typename T>
int merge_impl(T* acc_out, T* acc_stats, const T* part_out, const T* part_stats, int d) {
    if (int rc = have_device()) return rc;
    Scratch s;
    cudaError_t e = s.alloc((2 * (size_t)d + 6) * sizeof(T));
    if (e != cudaSuccess) return cuda_fail(e, "merge_partial: allocation");
    T* a = static_cast<T*>(s.p);
    T* pp = a + d;
    T* sc = pp + d;
    const T host_sc[6] = {acc_stats[0], acc_stats[1], part_stats[0], part_stats[1], 0, 0};
    e = cudaMemcpy(a, acc_out, d * sizeof(T), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(pp, part_out, d * sizeof(T), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(sc, host_sc, sizeof(host_sc), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "merge_partial: upload");
    merge_kernel<T><<<1, kThreads>>>(a, pp, d, sc);
    e = cudaGetLastError();
    T back[6];
    if (e == cudaSuccess) e = cudaMemcpy(acc_out, a, d * sizeof(T), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(back, sc, sizeof(back), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "merge_partial: kernel");
    acc_stats[0] = back[0];
    acc_stats[1] = back[1];
    acc_stats[2] = back[4];
    return PSATTN_OK;
}

template <typename T>
int finalize_impl(const T* acc_out, int d, T es, T* out) {
    if (int rc = have_device()) return rc;
    Scratch s;
    cudaError_t e = s.alloc(2 * (size_t)d * sizeof(T));
    if (e != cudaSuccess) return cuda_fail(e, "finalize: allocation");
    T* a = static_cast<T*>(s.p);
    e = cudaMemcpy(a, acc_out, d * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "finalize: upload");
    finalize_kernel<T><<<1, kThreads>>>(a, d, es, a + d);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out, a + d, d * sizeof(T), cudaMemcpyDeviceToHost);
    return e == cudaSuccess ? PSATTN_OK : cuda_fail(e, "finalize: kernel");
}

}  // namespace

int seq_attention(const float* q, int d, const float* K, const float* V, int64_t n, float scale, int normalize,
                  float* out, float* stats) {
    return seq_attention_impl<float>(q, d, K, V, n, scale, normalize, out, stats);
}
int seq_attention(const float* q, int d, const float* K, const float* V, int64_t n, double scale, int normalize,
                  double* out, double* stats) {
    return seq_attention_impl<double>(q, d, K, V, n, scale, normalize, out, stats);
}
int softmax_merge(float* acc_out, float* acc_stats, const float* part_out, const float* part_stats, int d) {
    return merge_impl<float>(acc_out, acc_stats, part_out, part_stats, d);
}
int softmax_merge(double* acc_out, double* acc_stats, const double* part_out, const double* part_stats, int d) {
    return merge_impl<double>(acc_out, acc_stats, part_out, part_stats, d);
}
int softmax_finalize(const float* acc_out, int d, float es, float* out) { return finalize_impl<float>(acc_out, d, es, out); }
int softmax_finalize(const double* acc_out, int d, double es, double* out) {
    return finalize_impl<double>(acc_out, d, es, out);
}

}  // namespace psa
