// internal.h — launch parameters shared by the host runtime (delta_api.cpp) and the
// sm_100a kernels.  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace delta {

// Per-device one-time kernel setup (cudaFuncSetAttribute opt-ins are per device context): the
// cached value (> 0) of init() for the current device; init() returning <= 0 is not cached.
constexpr int kMaxDevices = 64;
template <typename F>
int per_device_once(std::atomic<int>* cache, F init) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
        cudaGetLastError();
        dev = 0;
    }
    int v = cache[dev].load(std::memory_order_acquire);
    if (v <= 0) {
        v = init();  // idempotent: a racing first call repeats it and stores the same value
        if (v > 0) cache[dev].store(v, std::memory_order_release);
    }
    return v;
}

enum Role : int { kRoleFull = 0, kRoleSelect = 1, kRoleSparse = 2, kRoleQuest = 3, kRoleRaas = 4 };  // 3, 4: host only
enum DevErr : int { kDevOk = 0, kDevUsage = 2, kDevNumeric = 3, kDevCapacity = 4 };

constexpr int kPage = 16;        // P
constexpr int kMaxGs = 16;       // query heads per KV group handled by one MMA row tile
constexpr int kMaxSplit = 16;    // split-K CTAs per (sequence, kv head) = one thread-block cluster
constexpr int kSelSmemUnits = 16384;  // select: unit keys cached in shared memory up to this many
constexpr int kMaxSplitG = 64;   // split-K CTAs per (sequence, kv head) with the global merge
// Floats of one split's partial in the global-merge buffer: O rows [kMaxGs][d] then (M, L) pairs.
__host__ __device__ constexpr int gpart_floats(int d) { return kMaxGs * d + 2 * kMaxGs; }

// Row (of d elements) holding slot `slot` of the K head-page of (layer_page, head h), where
// layer_page = layer * num_phys + physical page; the matching V row is kv_row(...) + kPage.
// Pool layout [L][num_phys][g][2][P][d]: one (page, head) is 2P contiguous rows (K then V),
// so a single 4-8 KiB TMA request fetches both (per-SM TMA throughput is request-bound).
__host__ __device__ __forceinline__ size_t kv_row(size_t layer_page, int g, int h, int slot) {
    return ((layer_page * (size_t)g + (size_t)h) * 2) * kPage + (size_t)slot;
}

// One decode-attention launch (one layer, sequences [0, batch)).
struct AttnParams {
    int m, g, gs, d;
    int layer, batch, nsplit, role;
    int num_phys;       // pages per layer in each pool
    int bt_stride;      // block-table row stride (pages per sequence)
    int max_batch, max_seq;
    int sel_block;      // SPARSE: 1 = token plan, P = page plan
    int plan_cap;       // plan row stride (units)
    int fuse_append;    // 1: append k_new/v_new at position seq_len (pre) in this launch
    int deep;           // 1: one CTA per SM with the deep TMA ring (few CTAs), 0: shallow ring
    int prewait;        // 1: start geometry + KV stream before griddepcontrol.wait (see attn_tc.cu)
    int early_trigger;  // 1: launch_dependents right after the wait (else after the main loop)
    int cluster_policy; // cudaClusterSchedulingPolicy for the split-K cluster (0 = default)
    int emit_logits;    // 1: write the scaled logits of the attended tokens and the LSE (SELECT, RaaS)
    int gmerge;         // 1: no cluster; one CTA per SM; splits merged through global memory by
                        //    the last-arriving CTA of each (sequence, kv head) (combine.cuh)
    int q_prefetch;     // 1: prefetch this CTA's q rows into L2 before griddepcontrol.wait
    int sparse_lat;     // host: SPARSE layer takes the latency kernel (attn_sparse.cu)
    int gm_shallow;     // gmerge: 1 = shallow ring (two CTAs per SM: the next layer's CTAs co-reside
                        //    and prefetch during this one), 0 = deep ring (one CTA per SM)
    int fixed_part;     // FULL / SELECT: fixed page partition when the cache is >= 15/16 full (split_geometry)
    int gll;            // gmerge: 1 = partials as LL (value, flag) words polled by the merging CTAs
    float* gpart;       // gmerge: [batch][g][nsplit][gpart_floats(d)] split partials (x2 words with gll)
    unsigned long long* gcnt;  // gmerge: [max_batch][g][kMaxSplitG] ticket counters, by split count
    float scale;        // softmax scale (natural units)
    float scale_log2;   // scale * log2(e)
    const void* q;      // [batch][m][d]
    const void* k_new;  // [batch][g][d] (fuse_append)
    const void* v_new;
    void* kv_pool;      // [L][num_phys][g][2][P][d]: K rows then V rows of each (page, head)
    const int32_t* block_table;   // [max_batch][bt_stride]
    int32_t* seq_len;   // [L][max_batch] raw length counters: n * g (see combine.cuh)
    float* out;         // [batch][m][d]
    float* lse_out;     // [batch][m] or null
    float* logits;      // SELECT: [max_batch][max_seq][m] (natural units, scaled)
    float* lse_buf;     // SELECT: [max_batch][m] natural-log LSE for the score pass
    const int32_t* plan_idx;    // SPARSE: [max_batch][plan_cap] unit ids (pages or tokens)
    const int32_t* plan_phys;   // SPARSE: same shape: physical page (page plan) or page*P+slot (token plan)
    const int32_t* plan_count;  // [max_batch]
    const int32_t* plan_stamp;  // [max_batch]
    int32_t* err;
    // sequence sharding / fixed chunks (R21): attention covers pages [page_lo, page_hi) of
    // every sequence, and with part_o set the epilogue writes that range's partial (normalised
    // o, natural-log lse) instead of the outputs, for the LSE merge (shard.cu).
    int page_lo, page_hi;
    const int32_t* plan_lo;     // SPARSE, sharded: [max_batch] the range's plan entries [lo, hi)
    const int32_t* plan_hi;
    float* part_o;              // [batch][m][d], or null: write out / lse_out
    float* part_lse;            // [batch][m]
};

// Score + top-k selection launch (one Delta layer).
struct SelectParams {
    int m, g, layer, batch, nchunk;
    int sel_block, n_sink, n_window, k_units;
    int max_batch, max_seq, max_units, plan_cap;
    int32_t* seq_len;           // [L][max_batch] raw counters n * g (written by a Quest append)
    const float* logits;        // [max_batch][max_seq][m]
    const float* lse_buf;       // [max_batch][m]
    const float* keys_override; // [batch][ceil(s/sel_block)] or null
    float* keys;                // [max_batch][max_units] scratch
    int32_t* plan_idx;          // [max_batch][plan_cap]
    int32_t* plan_phys;         // [max_batch][plan_cap] physical page / page*P+slot of each unit
    const int32_t* block_table; // [max_batch][bt_stride]
    int bt_stride;
    int32_t* plan_count;
    int32_t* plan_stamp;
    int32_t* idx_out;           // optional [batch][plan_cap]
    int32_t* count_out;         // optional [batch]
    int32_t* cnt;               // [max_batch] arrival counters (this layer)
    // LL hand-off (ll = 1): phase-A CTAs also publish each unit key as a (key bits, flag) word;
    // CTA 0 polls them instead of an arrival election (flag = epoch[b] + 1, epoch bumped by CTA 0)
    int ll;
    uint2* keys_ll;             // [max_batch][max_units]
    int32_t* epoch;             // [max_batch] (every layer: the flags must differ across layers too)
    int32_t* err;
    // sequence sharding: mode 0 = unsharded; 1 = local (keys of own units only; export the
    // rank's top-k candidates to cand_out); 2 = global merge (keys_override = the dense keys
    // scattered from all ranks' candidates)
    int shard_mode, page_lo, page_hi;
    // plan ranges (modes 2, and 0 with fixed chunks): for c < range_n, the plan entries on pages
    // [range_first + c * range_step, + range_step) -> plan_lo/plan_hi[c * max_batch + b]
    int range_n, range_first, range_step;
    uint2* cand_out;            // mode 1: [batch][k_units] (order-preserving key bits, unit)
    int late_trigger;           // 1: launch dependents after the plan is written (else at entry)
    // Quest layers: this launch also performs the layer's Eq.7 append of one token (pool rows,
    // page representatives, length counter) before ranking — k_new null otherwise
    const void* k_new;          // [batch][g][d] bf16
    const void* v_new;
    void* kv_pool;              // [L][num_phys][g][2][P][d]
    void* reps;                 // [L][num_phys][g][2][d]
    int d, num_phys;
    int hist_mode;              // radix histogram: 0 per-warp private, 1 warp-aggregated shared
    int32_t* plan_lo;           // [range_n][max_batch]
    int32_t* plan_hi;
};

// Cross-rank merge of attention partials (sequence sharding): recv [W][batch][m][d] o and
// [W][batch][m] lse (natural), fixed rank order.
struct ShardMergeParams {
    int world, batch, m, d, role;
    const float* recv_o;        // [W][batch][m][d]
    const float* recv_lse;      // [W][batch][m]
    size_t o_stride, lse_stride;  // floats between ranks
    float* out;                 // [batch][m][d]
    float* lse_out;             // [batch][m] or null
    float* lse_buf;             // SELECT: [max_batch][m]
    int32_t* err;
};

struct AppendParams {
    int g, d, layer, batch, ntok, num_phys, bt_stride, max_batch, max_seq, elem_bytes;
    void* reps;         // Quest layers: [L][num_phys][g][2][d] bf16 page min/max, updated per token
    int32_t* ticket;    // [L][max_batch] arrival tickets of multi-CTA appends (reset by the last)
    int page_lo, page_hi;  // sequence sharding: this rank writes rows on its pages only
    const void* k_new;  // [batch][ntok][g][d]
    const void* v_new;
    void* kv_pool;
    const int32_t* block_table;
    int32_t* seq_len;
    int32_t* err;
};

// Quest policy (quest.cu): page representatives and page keys of one layer.
struct QuestParams {
    int m, g, d, layer, batch, num_phys, bt_stride, max_batch, max_units;
    const void* kv_pool;        // [L][num_phys][g][2][P][d] bf16
    void* reps;                 // [L][num_phys][g][2][d] bf16 (min row, max row)
    const int32_t* block_table;
    const int32_t* seq_len;     // raw counters n * g
    const void* q;              // [batch][m][d] bf16
    float* keys;                // [max_batch][max_units] page keys
    int prewait;                // 1: length counter and reps read before griddepcontrol.wait (see quest.cu)
};
cudaError_t launch_quest_reps(const QuestParams& p, int max_pages, cudaStream_t st, bool pdl);
cudaError_t launch_quest_score(const QuestParams& p, int max_pages, int sms, cudaStream_t st, bool pdl);

// Attention recall (recall.cu, Eq.9) of one layer's plan against its full-attention probe.
struct RecallParams {
    int m, g, layer, batch, max_batch, max_seq, plan_cap, sel_block;
    const int32_t* seq_len;     // raw counters n * g
    const float* logits;        // [max_batch][max_seq][m] scaled logits of the probe
    const float* lse;           // [max_batch][m] natural-log LSE of the probe
    const int32_t* plan_idx;    // [max_batch][plan_cap] units
    const int32_t* plan_count;  // [max_batch]
    float* recall_out;          // [batch][m]
};
cudaError_t launch_recall(const RecallParams& p, cudaStream_t st, bool pdl);

// Chunked prefill (prefill.cu): causal attention of ntok appended tokens per sequence.
struct PrefillParams {
    int m, g, gs, d, layer, batch, ntok, num_phys, bt_stride, max_batch;
    float scale_log2;
    const void* q;              // [batch][ntok][m][d] bf16
    const void* kv_pool;
    const int32_t* block_table;
    const int32_t* seq_len;     // raw counters n * g, AFTER the chunk's append
    float* out;                 // [batch][ntok][m][d]
    float* lse_out;             // [batch][ntok][m] or null
    int32_t* err;
};
cudaError_t launch_prefill(const PrefillParams& p, cudaStream_t st, bool pdl);
cudaError_t launch_prefill_umma(const PrefillParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl);
cudaError_t launch_prefill_umma2(const PrefillParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl);
cudaError_t launch_prefill_umma3(const PrefillParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl);
bool prefill_umma_supported(const PrefillParams& p);
size_t prefill_smem_bytes(int d, int gs);

// RaaS policy (raas.cu): retained-set reset and the per-step refresh / eviction.
struct RaasParams {
    int m, g, layer, batch, max_batch, max_seq, max_pages, plan_cap, n_sink, n_window, k_pages;
    int32_t* seq_len;           // raw counters n * g
    const float* logits;        // [max_batch][max_seq][m] of the layer's attention this step
    const float* lse;           // [max_batch][m]
    int32_t* plan_idx;          // [max_batch][plan_cap] retained pages, ascending (this layer's slot)
    int32_t* plan_phys;
    int32_t* plan_count;
    int32_t* plan_stamp;
    int32_t* last;              // [max_batch][max_pages] last-salient step (this layer)
    float* scores;              // [max_batch][max_units] page scores (exported)
    int max_units;
    const int32_t* block_table;
    int bt_stride;
    int32_t* ticket;            // [L][max_batch] arrival tickets (shared with the multi-CTA append)
};
cudaError_t launch_raas_reset(const RaasParams& p, cudaStream_t st, bool pdl);
cudaError_t launch_raas_update(const RaasParams& p, cudaStream_t st, bool pdl);

// Launchers (attn_tc.cu / attn_simt.cu / select.cu / append.cu).  Each returns the
// cudaError_t of the launch.  `pdl` enables programmatic dependent launch.
cudaError_t launch_attn_tc(const AttnParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl);
cudaError_t launch_read_probe(const void* buf, size_t bytes, float* sink, int sms, cudaStream_t st);
cudaError_t launch_attn_sparse_lat(const AttnParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl);
int sparse_lat_max_tiles();        // resident tiles per CTA of the latency kernel
int sparse_lat_max_split(int d);   // largest co-resident cluster (split count) of the latency kernel
cudaError_t launch_attn_umma(const AttnParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl);
bool umma_supported(const AttnParams& p);
cudaError_t launch_attn_simt(const AttnParams& p, bool bf16, cudaStream_t st, bool pdl);
cudaError_t launch_select(const SelectParams& p, cudaStream_t st, bool pdl);
cudaError_t launch_append(const AppendParams& p, cudaStream_t st, bool pdl);
size_t select_smem_bytes(int max_units);
cudaError_t launch_shard_merge(const ShardMergeParams& p, cudaStream_t st, bool pdl);
// scatter W x k candidates (uint2 key bits / unit) into dense fp32 keys (-inf elsewhere)
cudaError_t launch_cand_scatter(const uint2* recv, int world, int batch, int k_units, size_t rank_stride,
                                float* keys, int max_units, const int32_t* seq_len, int layer, int max_batch,
                                int g, int sel_block, cudaStream_t st, bool pdl);
// Largest cluster size (16, 8, 4, 2 or 1) with which `kern` can be resident (delta_api.cu).
int cluster_limit(const void* kern, int threads, int smem_bytes);

}  // namespace delta
