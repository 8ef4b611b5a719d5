// device.cu — the device layer behind psattn_b200.h: HBM block pool, batched
// launch and workspace carving.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <mutex>
#include <cmath>
#include <string>
#include <vector>

#include "device.h"
#include "kernels.cuh"
#include "psattn_b200.h"

struct psattn_pool {
    psattn_pool_desc desc{};
    psa::PoolView v{};
    // two-tier pools only (psattn_tier): pinned host backing tier + HBM location table
    char* host_kv = nullptr;
    int32_t* loc = nullptr;
    // 2-D TMA descriptor of the K/V slots (rows of d bf16, 2T rows per slot) for the stream kernel
    CUtensorMap kv_tmap;
};

namespace psa {

namespace {
thread_local std::string g_err = "";
std::atomic<int> g_last_launches{0};

// Stage timing (benchmark instrumentation): events recorded around each kernel
// of psattn_run_batch on the launching stream; read back on request.
struct Profiler {
    std::mutex mu;
    bool on = false;
    std::vector<std::array<cudaEvent_t, 5>> pending;
    double ms[4] = {0, 0, 0, 0};
    int64_t count[4] = {0, 0, 0, 0};
};
Profiler g_prof;
std::atomic<uint64_t> g_knob_gen{0};  // bumped by every psattn_set_* / psattn_profile_enable

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }

int fail(int code, const std::string& msg) {
    set_error(msg);
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(PSATTN_ERR_RUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}

static int64_t slot_bytes_for(int d, int T, int dtype) {
    const int e = dtype == PSATTN_KV_F32 ? 4 : 2;
    return (int64_t)align_up((size_t)2 * T * d * e, 16);
}
static int64_t meta_bytes_for(int d, int dtype) {
    const int e = dtype == PSATTN_KV_F32 ? 4 : 2;
    return (int64_t)align_up((size_t)d * 4 + (size_t)2 * d * e, 16);
}

const PoolView& pool_view(const psattn_pool* p) { return p->v; }

// The stream kernel (kernels_stream.cu) loads K / V tiles with 2-D TMA: the pool's K/V array
// viewed as rows of 128 bf16 (256 B), 32 rows per slot (16 K rows, then 16 V rows); boxes of
// 64 dims x 16 rows with the 128-byte swizzle. Built for the production layout only (bf16,
// d = 128, 16-token slots); rebuilt whenever the pool's storage moves (pool_grow).
static void build_kv_tmap(psattn_pool* pool) {
    PoolView& v = pool->v;
    v.kv_tmap = nullptr;
    if (v.dtype != PSATTN_KV_BF16 || v.d != 128 || v.T != 16 || v.n_slots <= 0 || v.slot_bytes != 2 * 16 * 128 * 2)
        return;
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeFn>(nullptr);
        return reinterpret_cast<EncodeFn>(f);
    }();
    if (!fn || (uint64_t)v.n_slots * 32 > 0xFFFFFFFFull) return;
    const cuuint64_t dims[2] = {128, (cuuint64_t)v.n_slots * 32};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t box[2] = {64, 16};
    const cuuint32_t es[2] = {1, 1};
    if (fn(&pool->kv_tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, v.kv, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return;
    v.kv_tmap = &pool->kv_tmap;
}

int pool_grow(psattn_pool* pool, int64_t n_slots, int32_t T) {
    PoolView& v = pool->v;
    if (n_slots < v.n_slots) n_slots = v.n_slots;
    if (T < v.T) T = v.T;
    if (n_slots == v.n_slots && T == v.T) return PSATTN_OK;
    PoolView nv = v;
    nv.T = T;
    nv.n_slots = n_slots;
    nv.slot_bytes = slot_bytes_for(v.d, T, v.dtype);
    cudaError_t e;
    if ((e = cudaMalloc(&nv.kv, (size_t)(n_slots * nv.slot_bytes))) != cudaSuccess) return cuda_fail(e, "pool grow kv");
    if ((e = cudaMalloc(&nv.meta, (size_t)(n_slots * nv.meta_bytes))) != cudaSuccess) {
        cudaFree(nv.kv);
        return cuda_fail(e, "pool grow meta");
    }
    if ((e = cudaMalloc(&nv.ntok, (size_t)n_slots * 4)) != cudaSuccess) {
        cudaFree(nv.kv);
        cudaFree(nv.meta);
        return cuda_fail(e, "pool grow ntok");
    }
    cudaMemset(nv.kv, 0, (size_t)(n_slots * nv.slot_bytes));
    cudaMemset(nv.meta, 0, (size_t)(n_slots * nv.meta_bytes));
    cudaMemset(nv.ntok, 0, (size_t)n_slots * 4);
    if (v.n_slots > 0) {
        // K rows and V rows move to the new per-slot offsets (T may have grown).
        const size_t rows_old = (size_t)v.T * v.d * v.esize;
        const size_t rows_new = (size_t)T * v.d * v.esize;
        cudaMemcpy2D(nv.kv, nv.slot_bytes, v.kv, v.slot_bytes, rows_old, v.n_slots, cudaMemcpyDeviceToDevice);
        cudaMemcpy2D(nv.kv + rows_new, nv.slot_bytes, v.kv + rows_old, v.slot_bytes, rows_old, v.n_slots,
                     cudaMemcpyDeviceToDevice);
        cudaMemcpy(nv.meta, v.meta, (size_t)(v.n_slots * v.meta_bytes), cudaMemcpyDeviceToDevice);
        cudaMemcpy(nv.ntok, v.ntok, (size_t)v.n_slots * 4, cudaMemcpyDeviceToDevice);
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cuda_fail(e, "pool grow copy");
    cudaFree(v.kv);
    cudaFree(v.meta);
    cudaFree(v.ntok);
    v = nv;
    pool->desc.block_tokens = T;
    pool->desc.n_slots = n_slots;
    build_kv_tmap(pool);
    return PSATTN_OK;
}

// fp32 <-> bf16 bit patterns on the host (round to nearest even, like __float2bfloat16_rn)
static uint16_t f32_to_bf16_bits(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u);  // NaN stays NaN
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
static float bits_to_f32(uint32_t u) {
    float x;
    memcpy(&x, &u, 4);
    return x;
}

// Packs fp32 host blocks into the pool's slot image and converts to the pool dtype.
static void pack_host(const PoolView& v, int64_t n, const int32_t* ntok, const float* keys, const float* values,
                      int64_t row_stride_blocks, std::vector<char>& out) {
    out.assign((size_t)(n * v.slot_bytes), 0);
    const size_t per = (size_t)v.T * v.d;
    for (int64_t i = 0; i < n; ++i) {
        char* dst = out.data() + i * v.slot_bytes;
        const float* k = keys + (size_t)i * row_stride_blocks;
        const float* vv = values + (size_t)i * row_stride_blocks;
        const size_t cnt = (size_t)ntok[i] * v.d;
        if (v.dtype == PSATTN_KV_F32) {
            memcpy(dst, k, cnt * 4);
            memcpy(dst + per * 4, vv, cnt * 4);
        } else {
            uint16_t* dk = reinterpret_cast<uint16_t*>(dst);
            uint16_t* dv = dk + per;
            for (size_t j = 0; j < cnt; ++j) {
                dk[j] = (uint16_t)(f32_to_bf16_bits(k[j]));
                dv[j] = (uint16_t)(f32_to_bf16_bits(vv[j]));
            }
        }
    }
}

// Two-tier pool: metadata + ntok for n_blocks logical blocks in HBM, K/V of every block in
// pinned mapped host memory, `fast_slots` HBM K/V slots, loc[] = -1 (nothing resident).
int pool_create_tiered(const psattn_pool_desc* desc, int64_t n_blocks, int64_t fast_slots, psattn_pool** out) {
    psattn_pool_desc d = *desc;
    d.n_slots = 0;
    int rc = psattn_pool_create(&d, out);
    if (rc) return rc;
    psattn_pool* p = *out;
    PoolView& v = p->v;
    cudaError_t e;
    auto bail = [&](cudaError_t err, const char* what) {
        psattn_pool_destroy(p);
        *out = nullptr;
        return cuda_fail(err, what);
    };
    if ((e = cudaMalloc(&v.kv, (size_t)std::max<int64_t>(fast_slots, 1) * v.slot_bytes)) != cudaSuccess)
        return bail(e, "tier HBM slots");
    if ((e = cudaMalloc(&v.meta, (size_t)n_blocks * v.meta_bytes)) != cudaSuccess) return bail(e, "tier metadata");
    if ((e = cudaMalloc(&v.ntok, (size_t)n_blocks * 4)) != cudaSuccess) return bail(e, "tier ntok");
    if ((e = cudaMalloc(&p->loc, (size_t)n_blocks * 4)) != cudaSuccess) return bail(e, "tier location table");
    if ((e = cudaHostAlloc(&p->host_kv, (size_t)n_blocks * v.slot_bytes, cudaHostAllocMapped)) != cudaSuccess)
        return bail(e, "tier host backing store");
    void* dev_alias = nullptr;
    if ((e = cudaHostGetDevicePointer(&dev_alias, p->host_kv, 0)) != cudaSuccess) return bail(e, "tier host mapping");
    memset(p->host_kv, 0, (size_t)n_blocks * v.slot_bytes);
    cudaMemset(v.kv, 0, (size_t)std::max<int64_t>(fast_slots, 1) * v.slot_bytes);
    cudaMemset(v.meta, 0, (size_t)n_blocks * v.meta_bytes);
    cudaMemset(v.ntok, 0, (size_t)n_blocks * 4);
    cudaMemset(p->loc, 0xff, (size_t)n_blocks * 4);
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bail(e, "tier init");
    v.n_slots = n_blocks;
    v.loc = p->loc;
    v.host_kv = static_cast<const char*>(dev_alias);
    p->desc.n_slots = n_blocks;
    return PSATTN_OK;
}
int32_t* pool_loc(psattn_pool* pool) { return pool->loc; }
char* pool_host_kv(psattn_pool* pool) { return pool->host_kv; }

// Packs host fp32 blocks (rows past ntok zero) into the host backing tier in the pool dtype.
void pool_pack_into(const psattn_pool* pool, int64_t n, const int64_t* blocks, const int32_t* ntok, const float* keys,
                    const float* values) {
    const PoolView& v = pool->v;
    const size_t stride = (size_t)v.T * v.d;
    for (int64_t i = 0; i < n; ++i) {
        std::vector<char> img;
        pack_host(v, 1, ntok + i, keys + i * stride, values + i * stride, (int64_t)stride, img);
        memcpy(pool->host_kv + blocks[i] * v.slot_bytes, img.data(), (size_t)v.slot_bytes);
    }
}

int pool_put(psattn_pool* pool, int64_t n, const int32_t* slots, const int32_t* ntok, const float* keys,
             const float* values, int64_t row_stride_floats, cudaStream_t st) {
    if (n <= 0) return PSATTN_OK;
    const PoolView& v = pool->v;
    std::vector<char> img;
    pack_host(v, n, ntok, keys, values, row_stride_floats, img);
    char* d_img = nullptr;
    int32_t* d_idx = nullptr;
    // staging buffers are released on every path (stream-ordered frees, then one sync)
    auto finish = [&](cudaError_t err, const char* what) {
        if (d_img) cudaFreeAsync(d_img, st);
        if (d_idx) cudaFreeAsync(d_idx, st);
        const cudaError_t es = cudaStreamSynchronize(st);
        if (err != cudaSuccess) return cuda_fail(err, what);
        return es == cudaSuccess ? PSATTN_OK : cuda_fail(es, "put_blocks");
    };
    cudaError_t e;
    if ((e = cudaMallocAsync(&d_img, img.size(), st)) != cudaSuccess) return finish(e, "put staging");
    if ((e = cudaMallocAsync(&d_idx, (size_t)n * 8, st)) != cudaSuccess) return finish(e, "put staging");
    if ((e = cudaMemcpyAsync(d_img, img.data(), img.size(), cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return finish(e, "put upload");
    if ((e = cudaMemcpyAsync(d_idx, slots, (size_t)n * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return finish(e, "put upload");
    if ((e = cudaMemcpyAsync(d_idx + n, ntok, (size_t)n * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess)
        return finish(e, "put upload");
    if ((e = launch_scatter(v, d_img, d_idx, d_idx + n, n, st)) != cudaSuccess) return finish(e, "put scatter");
    if ((e = launch_meta_build(v, d_idx, 0, n, st)) != cudaSuccess) return finish(e, "metadata build");
    return finish(cudaSuccess, "put_blocks");
}

int read_slot(const psattn_pool* pool, int64_t slot, int32_t ntok, float* keys, float* values) {
    const PoolView& v = pool->v;
    std::vector<char> img((size_t)v.slot_bytes);
    cudaError_t e = cudaMemcpy(img.data(), v.kv + slot * v.slot_bytes, (size_t)v.slot_bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "read slot");
    const size_t per = (size_t)v.T * v.d, cnt = (size_t)ntok * v.d;
    if (v.dtype == PSATTN_KV_F32) {
        memcpy(keys, img.data(), cnt * 4);
        memcpy(values, img.data() + per * 4, cnt * 4);
    } else {
        const uint16_t* k = reinterpret_cast<const uint16_t*>(img.data());
        for (size_t j = 0; j < cnt; ++j) {
            keys[j] = bits_to_f32((uint32_t)k[j] << 16);
            values[j] = bits_to_f32((uint32_t)k[per + j] << 16);
        }
    }
    return PSATTN_OK;
}

int read_meta(const psattn_pool* pool, int64_t slot, float* mean, float* lo, float* hi) {
    const PoolView& v = pool->v;
    std::vector<char> rec((size_t)v.meta_bytes);
    cudaError_t e = cudaMemcpy(rec.data(), v.meta + slot * v.meta_bytes, (size_t)v.meta_bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "read metadata");
    memcpy(mean, rec.data(), (size_t)v.d * 4);
    const char* lp = rec.data() + (size_t)v.d * 4;
    const char* hp = lp + (size_t)v.d * v.esize;
    for (int i = 0; i < v.d; ++i) {
        if (v.dtype == PSATTN_KV_F32) {
            memcpy(lo + i, lp + 4 * i, 4);
            memcpy(hi + i, hp + 4 * i, 4);
        } else {
            uint16_t a, b;
            memcpy(&a, lp + 2 * i, 2);
            memcpy(&b, hp + 2 * i, 2);
            lo[i] = bits_to_f32((uint32_t)a << 16);
            hi[i] = bits_to_f32((uint32_t)b << 16);
        }
    }
    return PSATTN_OK;
}

// ---- workspace carving ----
struct WsLayout {
    size_t keys, rpos, omass, kmm, dflag, dla, dp, dthr, dpart, dsel, ft, sw, total;
};

static WsLayout ws_layout(const psattn_batch* b) {
    const size_t hb = (size_t)b->total_blocks * (size_t)b->group;
    WsLayout l{};
    size_t o = 0;
    l.keys = o;
    o += align_up(hb * 8, 256);
    l.rpos = o;
    o += align_up(hb * 4, 256);
    l.omass = o;
    if (b->ranking_mode == PSATTN_RANK_ORACLE || b->audit_coverage) o += align_up(hb * 8, 256);
    l.kmm = o;
    o += align_up((size_t)b->n_units * b->group * 16, 256);
    // dense hand-over scratch (GQA shapes with the estimated ranking: d = 128, group 2..4)
    l.dflag = l.dla = l.dp = l.dthr = l.dpart = l.dsel = 0;
    if (b->dim == 128 && b->group >= 2 && b->group <= 4 && b->ranking_mode != PSATTN_RANK_ORACLE &&
        !b->audit_coverage && b->max_blocks <= kDenseMaxBlocks) {
        l.dflag = o;
        o += 256 + align_up((size_t)b->n_units * 4, 256);  // counts (hand-over [0,32), escalated [32,64)) | unit list
        l.dsel = o;  // candidate thresholds | escalated list | escalation marks
        o += align_up((size_t)b->n_units * b->group * 8, 256) + 2 * align_up((size_t)b->n_units * 4, 256);
        l.dla = o;
        o += align_up(hb * 4, 256);
        l.dp = o;
        o += align_up(hb * 64, 256);
        l.dthr = o;
        o += align_up((size_t)b->n_units * b->group * 8, 256);
        l.dpart = o;
        o += align_up((size_t)b->n_units * b->group * ((b->max_blocks + kDenseSlice - 1) / kDenseSlice) * kDensePart * 4, 256);
        // stream kernel: token weights of every fetched block, [unit][kStreamEnt][4 heads][16] fp32
        l.sw = o;
        o += align_up((size_t)b->n_units * kStreamEnt * kStreamWRow * 4, 256);
    }
    // first tranche of every head (GQA shapes): keys | slots | ntok | count
    l.ft = 0;
    if ((b->dim == 128 || b->dim == 64) && b->group >= 2 && b->group <= 4) {
        const size_t hq = (size_t)b->n_units * b->group;
        l.ft = o;
        o += align_up(hq * kFirstCap * 8, 256) + align_up(hq * kFirstCap * 4, 256) + align_up(hq * kFirstCap, 256) +
             align_up(hq * 4, 256);
    }
    l.total = o;
    return l;
}

size_t ws_omass_offset(const psattn_batch* b) { return ws_layout(b).omass; }
size_t ws_rpos_offset(const psattn_batch* b) { return ws_layout(b).rpos; }

int validate_batch(const psattn_pool* pool, const psattn_batch* b) {
    if (!pool || !b) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_run_batch: null argument");
    if (b->n_units < 1 || b->group < 1 || b->group > 8)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_run_batch: need n_units >= 1 and 1 <= group <= 8");
    if (b->dim != pool->v.d)
        return fail(PSATTN_ERR_RUNTIME, "psattn_run_batch: dimension mismatch (" + std::to_string(b->dim) + " vs " +
                                            std::to_string(pool->v.d) + ")");
    if (!(b->epsilon > 0.0) || b->epsilon > 1.0)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "config: epsilon must be in (0, 1]");
    if (b->microbatch_size < 1) return fail(PSATTN_ERR_INVALID_ARGUMENT, "config: microbatch_size must be >= 1");
    if (b->estimator < 0 || b->estimator > 2) return fail(PSATTN_ERR_INVALID_ARGUMENT, "config: unknown estimator code");
    if (b->ranking_mode < 0 || b->ranking_mode > 1)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "config: unknown ranking mode code");
    if (b->topk < 0) return fail(PSATTN_ERR_INVALID_ARGUMENT, "topk must be >= 0");
    if (b->max_blocks < 1 || b->total_blocks < 1)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_run_batch: empty block lists");
    if (!b->q || !b->slots || !b->list_off || !b->out || !b->blocks_processed || !b->est_coverage || !b->terminated)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_run_batch: null device pointer");
    return PSATTN_OK;
}

BatchView make_view(const psattn_pool* pool, const psattn_batch* b, void* workspace) {
    const WsLayout l = ws_layout(b);
    char* ws = static_cast<char*>(workspace);
    BatchView v{};
    v.n_units = b->n_units;
    v.g = b->group;
    v.d = b->dim;
    v.max_n = b->max_blocks;
    v.total = b->total_blocks;
    int pb = 1;
    while (pb < 62 && (int64_t(1) << pb) < b->max_blocks) ++pb;
    v.pos_bits = pb;
    v.q = b->q;
    v.slots = b->slots;
    v.list_off = b->list_off;
    v.eps = b->epsilon;
    v.m = b->microbatch_size;
    v.estimator = b->estimator;
    v.rank_oracle = b->ranking_mode == PSATTN_RANK_ORACLE;
    v.audit = b->audit_coverage != 0;
    v.has_oracle = v.rank_oracle || v.audit;
    v.scale = b->scale_override > 0.0 ? b->scale_override : 1.0 / std::sqrt((double)b->dim);
    v.topk = b->topk;
    v.out = b->out;
    v.bp = b->blocks_processed;
    v.est = b->est_coverage;
    v.tcov = b->true_coverage;
    v.term = b->terminated;
    v.keys = reinterpret_cast<uint64_t*>(ws + l.keys);
    v.rpos = b->ranked_pos ? b->ranked_pos : reinterpret_cast<int32_t*>(ws + l.rpos);
    v.omass = v.has_oracle ? reinterpret_cast<double*>(ws + l.omass) : nullptr;
    v.iest = b->iter_est;
    v.kminmax = v.rank_oracle ? nullptr : reinterpret_cast<unsigned long long*>(ws + l.kmm);
    v.kmm_stride = (int64_t)b->n_units * b->group;
    v.dense_count = l.dflag ? reinterpret_cast<int32_t*>(ws + l.dflag) : nullptr;
    v.dense_flag = l.dflag ? reinterpret_cast<int32_t*>(ws + l.dflag + 256) : nullptr;
    v.dense_la = l.dflag ? reinterpret_cast<float*>(ws + l.dla) : nullptr;
    v.dense_p = l.dflag ? reinterpret_cast<float*>(ws + l.dp) : nullptr;
    v.dense_thr = l.dflag ? reinterpret_cast<unsigned long long*>(ws + l.dthr) : nullptr;
    v.dense_part = l.dflag ? reinterpret_cast<float*>(ws + l.dpart) : nullptr;
    v.dense_esc_count = l.dflag ? reinterpret_cast<int32_t*>(ws + l.dflag) + 32 : nullptr;
    v.dense_sel = l.dflag ? reinterpret_cast<unsigned long long*>(ws + l.dsel) : nullptr;
    v.dense_esc = l.dflag ? reinterpret_cast<int32_t*>(ws + l.dsel + align_up((size_t)b->n_units * b->group * 8, 256))
                          : nullptr;
    v.dense_esc_mark = l.dflag ? v.dense_esc + align_up((size_t)b->n_units * 4, 256) / 4 : nullptr;
    v.stream_w = l.sw ? reinterpret_cast<float*>(ws + l.sw) : nullptr;
    if (l.ft) {
        const size_t hq = (size_t)b->n_units * b->group;
        char* f = ws + l.ft;
        v.ft_keys = reinterpret_cast<unsigned long long*>(f);
        f += align_up(hq * kFirstCap * 8, 256);
        v.ft_slot = reinterpret_cast<int32_t*>(f);
        f += align_up(hq * kFirstCap * 4, 256);
        v.ft_ntok = reinterpret_cast<uint8_t*>(f);
        f += align_up(hq * kFirstCap, 256);
        v.ft_count = reinterpret_cast<int32_t*>(f);
    }
    (void)pool;
    return v;
}

}  // namespace psa

using namespace psa;

extern "C" {

int psattn_pool_create(const psattn_pool_desc* desc, psattn_pool** out_pool) {
    if (!desc || !out_pool) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_create: null argument");
    if (desc->dim < 1 || desc->dim > 256)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_create: dim must be in [1, 256]");
    if (desc->block_tokens < 1 || desc->block_tokens > kMaxBlockTokens)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_create: block_tokens must be in [1, 128]");
    if (desc->kv_dtype != PSATTN_KV_F32 && desc->kv_dtype != PSATTN_KV_BF16)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_create: unknown kv dtype");
    if (desc->n_slots < 0) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_create: n_slots must be >= 0");
    int dev_count = 0;
    cudaError_t e = cudaGetDeviceCount(&dev_count);
    if (e != cudaSuccess || dev_count == 0)
        return fail(PSATTN_ERR_RUNTIME, std::string("no CUDA device: the PSA path has no CPU fallback (") +
                                            cudaGetErrorString(e) + ")");
    auto* p = new psattn_pool();
    p->desc = *desc;
    p->desc.n_slots = 0;
    PoolView& v = p->v;
    v.d = desc->dim;
    v.T = desc->block_tokens;
    v.dtype = desc->kv_dtype;
    v.esize = desc->kv_dtype == PSATTN_KV_F32 ? 4 : 2;
    v.slot_bytes = slot_bytes_for(v.d, v.T, v.dtype);
    v.meta_bytes = meta_bytes_for(v.d, v.dtype);
    v.n_slots = 0;
    if (desc->n_slots > 0) {
        const int rc = pool_grow(p, desc->n_slots, v.T);
        if (rc) {
            delete p;
            return rc;
        }
    }
    *out_pool = p;
    return PSATTN_OK;
}

void psattn_pool_destroy(psattn_pool* pool) {
    if (!pool) return;
    if (pool->host_kv) cudaFreeHost(pool->host_kv);
    if (pool->loc) cudaFree(pool->loc);
    cudaFree(pool->v.kv);
    cudaFree(pool->v.meta);
    cudaFree(pool->v.ntok);
    delete pool;
}

int psattn_pool_get_desc(const psattn_pool* pool, psattn_pool_desc* out) {
    if (!pool || !out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_get_desc: null argument");
    *out = pool->desc;
    return PSATTN_OK;
}

int psattn_pool_get_layout(const psattn_pool* pool, psattn_pool_layout* out) {
    if (!pool || !out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_get_layout: null argument");
    out->kv = pool->v.kv;
    out->meta = pool->v.meta;
    out->ntok = pool->v.ntok;
    out->slot_bytes = pool->v.slot_bytes;
    out->meta_bytes = pool->v.meta_bytes;
    return PSATTN_OK;
}

int psattn_pool_put_blocks(psattn_pool* pool, int64_t n, const int32_t* slots, const int32_t* ntok, const float* keys,
                           const float* values) {
    if (!pool || !slots || !ntok || !keys || !values)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_put_blocks: null argument");
    for (int64_t i = 0; i < n; ++i) {
        if (slots[i] < 0 || slots[i] >= pool->v.n_slots)
            return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_put_blocks: slot out of range");
        if (ntok[i] < 1 || ntok[i] > pool->v.T)
            return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_put_blocks: ntok out of range");
    }
    return pool_put(pool, n, slots, ntok, keys, values, (int64_t)pool->v.T * pool->v.d, 0);
}

int psattn_pool_build_metadata(psattn_pool* pool, int64_t slot_begin, int64_t slot_end, void* stream) {
    if (!pool) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_build_metadata: null pool");
    if (slot_begin < 0 || slot_end > pool->v.n_slots)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_build_metadata: slot range out of bounds");
    cudaError_t e = launch_meta_build(pool->v, nullptr, slot_begin, slot_end, (cudaStream_t)stream);
    return e == cudaSuccess ? PSATTN_OK : cuda_fail(e, "metadata build");
}

int psattn_pool_append_tokens(psattn_pool* pool, int32_t n, const int32_t* tail_slots, const float* keys,
                              const float* values, int32_t* status, void* stream) {
    if (!pool || !tail_slots || !keys || !values || !status)
        return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_append_tokens: null argument");
    if (n < 0) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_append_tokens: n must be >= 0");
    cudaError_t e = launch_append(pool->v, n, tail_slots, keys, values, status, (cudaStream_t)stream);
    return e == cudaSuccess ? PSATTN_OK : cuda_fail(e, "append tokens");
}

int psattn_pool_read_metadata(psattn_pool* pool, int64_t slot, float* mean, float* lo, float* hi) {
    if (!pool || !mean || !lo || !hi) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_pool_read_metadata: null");
    if (slot < 0 || slot >= pool->v.n_slots) return fail(PSATTN_ERR_INVALID_ARGUMENT, "slot out of range");
    return read_meta(pool, slot, mean, lo, hi);
}

size_t psattn_batch_workspace_bytes(const psattn_batch* b) { return b ? ws_layout(b).total : 0; }

int psattn_run_batch(psattn_pool* pool, const psattn_batch* b, void* workspace, void* stream) {
    int rc = validate_batch(pool, b);
    if (rc) return rc;
    if (!workspace) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_run_batch: null workspace");
    const BatchView v = make_view(pool, b, workspace);
    std::array<cudaEvent_t, 5> ev{};
    bool prof = false;
    {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        prof = g_prof.on;
    }
    if (prof)
        for (auto& e : ev) cudaEventCreate(&e);
    const int n = launch_batch(pool->v, v, (cudaStream_t)stream, prof ? ev.data() : nullptr);
    if (n < 0) return cuda_fail(cudaGetLastError(), "psattn_run_batch launch");
    if (prof) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.pending.push_back(ev);
        g_prof.count[1] += v.rank_oracle ? 0 : 1;
        g_prof.count[0] += v.has_oracle ? 1 : 0;
        g_prof.count[2] += 1;
        g_prof.count[3] += 1;
    }
    g_last_launches.store(n);
    return PSATTN_OK;
}

int psattn_rank_batch(psattn_pool* pool, const psattn_batch* b, void* workspace, void* stream) {
    int rc = validate_batch(pool, b);
    if (rc) return rc;
    if (!workspace) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_rank_batch: null workspace");
    BatchView v = make_view(pool, b, workspace);
    v.pos_bits = 0;        // compare full scores; ties fall to the stable sort (input = block-id order)
    v.kminmax = nullptr;   // no tranche selection follows
    const cudaStream_t st = (cudaStream_t)stream;
    if (launch_rank_keys(pool->v, v, st) < 0) return cuda_fail(cudaGetLastError(), "psattn_rank_batch: keys");
    const size_t hb = (size_t)b->total_blocks * (size_t)b->group;
    void* tmp = nullptr;
    cudaError_t e = cudaMallocAsync(&tmp, align_up(hb * 8, 256) + 2 * align_up(hb * 4, 256), st);
    if (e != cudaSuccess) return cuda_fail(e, "psattn_rank_batch: scratch");
    char* t = static_cast<char*>(tmp);
    uint64_t* tk = reinterpret_cast<uint64_t*>(t);
    int32_t* tv = reinterpret_cast<int32_t*>(t + align_up(hb * 8, 256));
    int32_t* tv2 = reinterpret_cast<int32_t*>(t + align_up(hb * 8, 256) + align_up(hb * 4, 256));
    e = launch_seg_sort(v.keys, nullptr, v.rpos, tk, tv, tv2, b->list_off, b->n_units, b->group, st);
    const cudaError_t e2 = cudaFreeAsync(tmp, st);
    if (e != cudaSuccess) return cuda_fail(e, "psattn_rank_batch: sort");
    if (e2 != cudaSuccess) return cuda_fail(e2, "psattn_rank_batch: scratch free");
    return PSATTN_OK;
}

int psattn_set_progressive_kernel(int32_t mode) {
    if (mode < 0 || mode > 3) return fail(PSATTN_ERR_INVALID_ARGUMENT, "progressive kernel mode must be 0, 1, 2 or 3");
    set_psa_kernel_choice(mode);
    g_knob_gen.fetch_add(1);
    return PSATTN_OK;
}

}  // extern "C"

namespace psa {
uint64_t launch_config_generation() {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    return g_prof.on ? ~0ull : g_knob_gen.load();  // ~0: profiling (no graph reuse)
}
}  // namespace psa

struct psattn_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
};

extern "C" {

int psattn_graph_create(psattn_pool* pool, const psattn_batch* b, void* workspace, void* stream, psattn_graph** out) {
    if (!out) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_graph_create: null output");
    int rc = validate_batch(pool, b);
    if (rc) return rc;
    if (!workspace) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_graph_create: null workspace");
    cudaStream_t st = (cudaStream_t)stream, own = nullptr;
    if (!st) {
        cudaError_t e = cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_fail(e, "psattn_graph_create: stream");
        st = own;
    }
    auto* g = new psattn_graph();
    cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
        const BatchView v = make_view(pool, b, workspace);
        g->launches = launch_batch(pool->v, v, st, nullptr);
        e = cudaStreamEndCapture(st, &g->graph);
        if (e == cudaSuccess && g->launches < 0) e = cudaErrorUnknown;
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (own) cudaStreamDestroy(own);
    if (e != cudaSuccess) {
        psattn_graph_destroy(g);
        return cuda_fail(e, "psattn_graph_create: capture");
    }
    *out = g;
    return PSATTN_OK;
}

int psattn_graph_launch(psattn_graph* g, void* stream) {
    if (!g) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_graph_launch: null graph");
    const cudaError_t e = cudaGraphLaunch(g->exec, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "psattn_graph_launch");
    g_last_launches.store(g->launches);
    return PSATTN_OK;
}

void psattn_graph_destroy(psattn_graph* g) {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
}

int psattn_set_dense(int32_t mode) {
    if (mode < 0 || mode > 1) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_set_dense: mode must be 0 or 1");
    set_dense_mode(mode);
    g_knob_gen.fetch_add(1);
    return PSATTN_OK;
}

int psattn_set_dense_early(float nats) {
    if (!(nats >= 0.0f)) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_set_dense_early: threshold must be >= 0");
    set_dense_early(nats);
    g_knob_gen.fetch_add(1);
    return PSATTN_OK;
}

int psattn_set_dense_partial(int32_t ranks) {
    if (ranks < 0) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_set_dense_partial: ranks must be >= 0");
    set_dense_partial(ranks);
    g_knob_gen.fetch_add(1);
    return PSATTN_OK;
}

int psattn_set_score_kernel(int32_t mode) {
    if (mode < 0 || mode > 3) return fail(PSATTN_ERR_INVALID_ARGUMENT, "score kernel mode must be 0..3");
    set_score_kernel_choice(mode);
    g_knob_gen.fetch_add(1);
    return PSATTN_OK;
}

int psattn_set_pipeline(int32_t sub_batches) {
    if (sub_batches < 0 || sub_batches > 16) return fail(PSATTN_ERR_INVALID_ARGUMENT, "sub_batches must be in [0, 16]");
    set_pipeline_subbatches(sub_batches);
    g_knob_gen.fetch_add(1);
    return PSATTN_OK;
}

int psattn_profile_enable(int32_t enable) {
    g_knob_gen.fetch_add(1);
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = enable != 0;
    return PSATTN_OK;
}

int psattn_profile_read(double* ms, int64_t* count, int32_t reset) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (auto& ev : g_prof.pending) {
        cudaError_t e = cudaEventSynchronize(ev[4]);
        if (e != cudaSuccess) return cuda_fail(e, "profile read");
        for (int s = 0; s < 4; ++s) {
            float t = 0.f;
            cudaEventElapsedTime(&t, ev[s], ev[s + 1]);
            g_prof.ms[s] += t;
        }
        for (auto& x : ev) cudaEventDestroy(x);
    }
    g_prof.pending.clear();
    for (int s = 0; s < 4; ++s) {
        if (ms) ms[s] = g_prof.ms[s];
        if (count) count[s] = g_prof.count[s];
    }
    if (reset) {
        for (int s = 0; s < 4; ++s) {
            g_prof.ms[s] = 0;
            g_prof.count[s] = 0;
        }
    }
    return PSATTN_OK;
}

int psattn_batch_union_blocks(const psattn_batch* b, void* workspace, int64_t* out_union, void* stream) {
    if (!b || !workspace || !out_union) return fail(PSATTN_ERR_INVALID_ARGUMENT, "psattn_batch_union_blocks: null");
    const BatchView v = make_view(nullptr, b, workspace);
    cudaError_t e = launch_union(v, out_union, (cudaStream_t)stream);
    return e == cudaSuccess ? PSATTN_OK : cuda_fail(e, "union kernel");
}

int psattn_batch_last_launches(int32_t* out_count) {
    if (!out_count) return fail(PSATTN_ERR_INVALID_ARGUMENT, "null");
    *out_count = g_last_launches.load();
    return PSATTN_OK;
}

}  // extern "C"
