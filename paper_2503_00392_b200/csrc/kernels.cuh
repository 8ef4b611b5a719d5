// kernels.cuh — device-side views and launcher declarations of the PSA path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace psa {

// Unified paged KV block pool in HBM (one per head dim). Slot s holds one
// (layer, kv-head) block of up to T tokens: K rows [T][d] then V rows [T][d].
// Its metadata record (reference BlockMetadata, types.hpp:52-59) lives at
// meta + s*meta_bytes: mean[d] fp32 | lo[d] kv | hi[d] kv.
struct PoolView {
    int32_t d;
    int32_t T;
    int32_t dtype;  // 0 f32, 1 bf16
    int32_t esize;
    char* kv;
    char* meta;
    int32_t* ntok;
    int64_t slot_bytes;
    int64_t meta_bytes;
    int64_t n_slots;
    // Two-tier pools (psattn_tier): slot indices name LOGICAL blocks (metadata, ntok);
    // loc[s] >= 0 is the HBM slot holding block s's K/V, loc[s] < 0 means it is read
    // from the pinned host backing tier at host_kv + s*slot_bytes (zero-copy over
    // PCIe/C2C). loc == nullptr: the plain HBM pool, K/V of slot s at kv + s*slot_bytes.
    const int32_t* loc;
    const char* host_kv;
    // Host pointer to the pool's CUtensorMap (2-D view of the K/V rows) or nullptr; passed by
    // value to the stream kernel as a __grid_constant__ parameter, never read on the device.
    const void* kv_tmap;
};

#ifdef __CUDACC__
// K rows (then V rows at + T*d) of block s.
template <typename KV>
__device__ __forceinline__ const KV* kv_block(const PoolView& p, int64_t s) {
    if (p.loc) {
        const int32_t l = __ldg(p.loc + s);
        if (l < 0) return reinterpret_cast<const KV*>(p.host_kv + s * p.slot_bytes);
        s = l;
    }
    return reinterpret_cast<const KV*>(p.kv + s * p.slot_bytes);
}
// HBM-resident (bulk L2 prefetch is issued only for device memory).
__device__ __forceinline__ bool kv_resident(const PoolView& p, int64_t s) { return !p.loc || __ldg(p.loc + s) >= 0; }
#endif

// One batched launch: n_units block lists (page tables of slots, ascending
// block id), g q-heads per list. Workspace arrays are indexed per head at
// hb = list_off[u]*g + h*n_u.
struct BatchView {
    int32_t n_units, g, d, pos_bits;
    int64_t max_n, total;
    const float* q;
    const int32_t* slots;
    const int64_t* list_off;
    double eps;
    int32_t m, estimator, rank_oracle, has_oracle, audit;
    double scale;
    int64_t topk;
    float* out;
    int64_t* bp;
    double* est;
    double* tcov;
    int32_t* term;
    // workspace
    uint64_t* keys;
    int32_t* rpos;
    double* omass;
    double* iest;  // optional per-rank estimate at microbatch boundaries
    // optional [2][n_units*g]: per-head min / max sort key, produced by the score kernel so the
    // first tranche selection skips its min/max scan (nullptr: the selection scans)
    unsigned long long* kminmax;
    int64_t kmm_stride;  // offset of the max half of kminmax (the full batch's n_units * g)
    // dense hand-over (kernels_dense.cu); dense_flag == nullptr disables it
    int32_t* dense_flag;            // [n_units] list of handed-over units (dense_count entries)
    float dense_early;              // hand a unit over before its first round when a head's criticality
                                    // scores at ranks 0 and kDenseHandover-1 differ by less than this (0: off)
    int32_t* dense_count;
    float* dense_la;                // [total*g] fp32 block masses
    float* dense_p;                 // [total*g][16] normalised token weights
    unsigned long long* dense_thr;  // [n_units*g] rank-threshold key of each head's processed set
    float* dense_part;              // [n_units*g][slices][kDensePart] per-slice V-pass partial states
    int64_t dense_slice;            // list positions per dense work item (set by launch_dense)
    // partial dense mode: round 0 computes the masses of each head's candidate prefix only (keys <=
    // dense_sel, about dense_sel_ranks ranks) and decides on it; heads that do not stop inside it send
    // their unit to round 1 (dense_esc list), which completes the K pass on the rest and decides in full
    unsigned long long* dense_sel;  // [n_units*g] candidate threshold key per head (~0: every block)
    int32_t* dense_esc;             // [n_units] escalated units (dense_esc_count entries)
    int32_t* dense_esc_count;
    int32_t* dense_esc_mark;        // [n_units] per unit: > 0 once a head escalated it
    int32_t dense_sel_ranks;        // candidate prefix size (0: partial mode off)
    int32_t dense_round;            // 0: the hand-over list, 1: the escalated list (set by launch_dense)
    // first tranche of every head, selected up front by first_tranche_kernel (nullptr: the
    // progressive kernel selects it itself): [n_units*g][kFirstCap] sorted keys, slots, ntok, count
    unsigned long long* ft_keys;
    int32_t* ft_slot;
    uint8_t* ft_ntok;
    int32_t* ft_count;
    // stream kernel (kernels_stream.cu): token weights of every fetched block of a unit,
    // [n_units][kStreamEnt][kStreamWRow] fp32, bulk-copied back beside the block's V tile
    float* stream_w;
};
constexpr int kMaxBlockTokens = 128;  // longest block (tokens) a pool slot holds; > 32 runs the chunked per-head kernel
constexpr int kFirstCap = 512;   // == the GQA kernel's tranche capacity
#ifndef PSA_STREAM_ENT
#define PSA_STREAM_ENT 512
#endif
constexpr int kStreamEnt = PSA_STREAM_ENT;  // distinct blocks one unit may fetch on the stream kernel (else hand-over)
constexpr int kStreamWRow = 68;  // floats per fetched block: token weights [4 heads][16] + 4 exponent sums
constexpr int64_t kDenseMaxBlocks = 16384;  // decide smem: 12 B per rank (196 KB)
constexpr int64_t kDenseHandover = 384;     // ranks a head consumes on the round kernel before the hand-over
constexpr int64_t kDenseSlice = 512;        // list positions per dense K / V work item
constexpr int kDensePart = 132;             // partial state: out[128], max, sum (+ pad)

int dpl_for(int d);
int tok_for(int T);
int g_for(int g);

cudaError_t launch_meta_build(const PoolView& p, const int32_t* list, int64_t s0, int64_t s1, cudaStream_t st);
cudaError_t launch_append(const PoolView& p, int32_t n, const int32_t* slots, const float* keys,
                          const float* values, int32_t* status, cudaStream_t st);
cudaError_t launch_install(const PoolView& p, const int64_t* d_blocks, const int32_t* d_dst, int64_t n,
                           cudaStream_t st);
cudaError_t launch_scatter(const PoolView& p, const void* staged, const int32_t* d_slots, const int32_t* d_ntok,
                           int64_t n, cudaStream_t st);
int launch_psa(const PoolView& p, const BatchView& b, cudaStream_t st);  // returns kernels launched
bool gqa_supported(const PoolView& p, const BatchView& b);
bool stream_supported(const PoolView& p, const BatchView& b);
void launch_stream(const PoolView& p, const BatchView& b, cudaStream_t st);  // kernels_stream.cu
int launch_gqa(const PoolView& p, const BatchView& b, cudaStream_t st);  // returns kernels launched
// 0 = auto (stream kernel, else the GQA round kernel where supported), 1 = per-query kernel,
// 2 = GQA round kernel, 3 = stream kernel (kernels_stream.cu) where supported
int psa_kernel_choice();
void set_psa_kernel_choice(int choice);
void set_score_kernel_choice(int choice);
void set_pipeline_subbatches(int k);
void set_dense_mode(int mode);  // 0 auto (hand-over enabled), 1 off
void set_dense_partial(int ranks);  // dense hand-over: candidate prefix of round 0 (0: off)
void set_dense_early(float nats);  // stream kernel: early hand-over threshold (0 off)
bool dense_supported(const PoolView& p, const BatchView& b);
void launch_dense(const PoolView& p, const BatchView& b, cudaStream_t st);
// Returns the number of kernel launches issued, or -1 on error (cudaGetLastError has it).
int launch_batch(const PoolView& p, const BatchView& b, cudaStream_t st, cudaEvent_t* marks = nullptr);
cudaError_t launch_union(const BatchView& b, int64_t* out_union, cudaStream_t st);
int launch_rank_keys(const PoolView& p, const BatchView& b, cudaStream_t st);  // oracle masses / scores only
cudaError_t launch_seg_sort(uint64_t* keys, const int32_t* vals_in, int32_t* vals_out, uint64_t* tk, int32_t* tv,
                            int32_t* tv2, const int64_t* list_off, int n_units, int g, cudaStream_t st);

}  // namespace psa
