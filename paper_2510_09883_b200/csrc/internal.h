// internal.h — launch parameters shared by the host runtime (delta_api.cpp) and the
// sm_100a kernels.  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace delta {

enum Role : int { kRoleFull = 0, kRoleSelect = 1, kRoleSparse = 2 };
enum DevErr : int { kDevOk = 0, kDevUsage = 2, kDevNumeric = 3, kDevCapacity = 4 };

constexpr int kPage = 16;        // P
constexpr int kMaxGs = 16;       // query heads per KV group handled by one MMA row tile
constexpr int kMaxSplit = 64;    // split-K partials per (sequence, kv head)

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
    float scale;        // softmax scale (natural units)
    float scale_log2;   // scale * log2(e)
    const void* q;      // [batch][m][d]
    const void* k_new;  // [batch][g][d] (fuse_append)
    const void* v_new;
    void* k_pool;       // [L][num_phys][g][P][d]
    void* v_pool;
    const int32_t* block_table;   // [max_batch][bt_stride]
    int32_t* seq_len;   // [L][max_batch]
    float* out;         // [batch][m][d]
    float* lse_out;     // [batch][m] or null
    float* part_o;      // [batch][g][nsplit][gs][d]
    float* part_lse;    // [batch][g][nsplit][gs]  (log2 units)
    int32_t* cnt_head;  // [max_batch][g] (this layer)
    int32_t* cnt_seq;   // [max_batch]    (this layer)
    float* logits;      // SELECT: [max_batch][max_seq][m] (natural units, scaled)
    float* lse_buf;     // SELECT: [max_batch][m] natural-log LSE for the score pass
    const int32_t* plan_idx;    // SPARSE: [max_batch][plan_cap]
    const int32_t* plan_count;  // [max_batch]
    const int32_t* plan_stamp;  // [max_batch]
    int32_t* err;
};

// Score + top-k selection launch (one Delta layer).
struct SelectParams {
    int m, layer, batch, nchunk;
    int sel_block, n_sink, n_window, k_units;
    int max_batch, max_seq, max_units, plan_cap;
    const int32_t* seq_len;     // [L][max_batch]
    const float* logits;        // [max_batch][max_seq][m]
    const float* lse_buf;       // [max_batch][m]
    const float* keys_override; // [batch][ceil(s/sel_block)] or null
    float* keys;                // [max_batch][max_units] scratch
    int32_t* plan_idx;          // [max_batch][plan_cap]
    int32_t* plan_count;
    int32_t* plan_stamp;
    int32_t* idx_out;           // optional [batch][plan_cap]
    int32_t* count_out;         // optional [batch]
    int32_t* cnt;               // [max_batch] arrival counters (this layer)
    int32_t* err;
};

struct AppendParams {
    int g, d, layer, batch, ntok, num_phys, bt_stride, max_batch, max_seq, elem_bytes;
    const void* k_new;  // [batch][ntok][g][d]
    const void* v_new;
    void* k_pool;
    void* v_pool;
    const int32_t* block_table;
    int32_t* seq_len;
    int32_t* err;
};

// Launchers (attn_tc.cu / attn_simt.cu / select.cu / append.cu).  Each returns the
// cudaError_t of the launch.  `pdl` enables programmatic dependent launch.
cudaError_t launch_attn_tc(const AttnParams& p, const CUtensorMap* tm_k, const CUtensorMap* tm_v,
                           cudaStream_t st, bool pdl);
cudaError_t launch_attn_simt(const AttnParams& p, bool bf16, cudaStream_t st, bool pdl);
cudaError_t launch_select(const SelectParams& p, cudaStream_t st, bool pdl);
cudaError_t launch_append(const AppendParams& p, cudaStream_t st, bool pdl);
size_t select_smem_bytes(int max_units);

}  // namespace delta
