// delta_api.cu — host runtime behind include/delta.h: configuration validation and the
// three-tier schedule, workspace carving,
// TMA descriptors, launch sizing, call-order (plan freshness) tracking, and the CUDA-graph
// step driver.  All device work is in the kernels; this file only marshals and launches.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/delta.h"
#include "internal.h"

using namespace delta;

namespace {

thread_local std::string g_msg;

// NVTX range per enqueued layer role (header-only NVTX v3: a no-op unless a profiler injects
// itself), so nsys / ncu timelines of eager calls and graph captures show layer and role.
struct NvtxRange {
    explicit NvtxRange(const char* role, int layer) {
        char buf[48];
        snprintf(buf, sizeof buf, "delta L%d %s", layer, role);
        nvtxRangePushA(buf);
    }
    ~NvtxRange() { nvtxRangePop(); }
};
const char* role_name(int r) {
    switch (r) {
        case kRoleFull: return "FULL";
        case kRoleSelect: return "SELECT";
        case kRoleSparse: return "SPARSE";
        case kRoleQuest: return "QUEST";
        case kRoleRaas: return "RAAS";
        default: return "?";
    }
}

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Layout {
    size_t seq_len, err, cnt_sel, sel_epoch, keys_ll, logits, lse_buf, keys, plan_idx, plan_phys, plan_count, plan_stamp, plan_lo, plan_hi,
        shard_send, shard_recv, cand_send, cand_recv, stage_q, stage_k, stage_v, stage_out, gpart, gcnt, reps, ticket,
        raas_last,
        reps_bytes, total;
    int gslots;  // split partial slots of the global-merge kernels
    size_t shard_block, cand_block;  // bytes of one rank's attention partial(s) / candidate block
    size_t part_bytes;               // one attention partial (o [batch][m][d], lse [batch][m])
    int det_chunks, chunk_pages;     // R21 fixed chunks (0 = off) and pages per chunk
    int max_units, plan_cap, n_delta, max_pages;
};

int num_sms_current() {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
    }
    cudaGetLastError();  // no device (CPU-only host) -> keep the B200 default
    return sms > 0 ? sms : 148;
}

// Split-K CTAs per (sequence, kv head) = cluster size: as many as fit in ONE wave of two CTAs
// per SM (the shallow-ring kernel fits two per SM), at most 16 (one cluster).  Rounding down
// matters: at batch 8 x 8 heads, 5 splits (320 CTAs > 296 slots) leave a second, under-occupied
// wave — measured 190 us vs 161 us for 4 splits on a 32K full layer, 25 vs 18 us sparse.
int nsplit_full(int batch, int g, int sms, int max_pages) {
    const int heads = std::max(1, batch * g);
    int n = (2 * sms) / heads;
    n = std::max(1, std::min(n, kMaxSplit));
    return std::min(n, std::max(1, max_pages));
}

int plan_tiles(const delta_config& c, int plan_cap) {
    return c.select_block == 1 ? (plan_cap + 15) / 16 : plan_cap;
}

int nsplit_sparse(const delta_config& c, int batch, int sms, int max_pages, int plan_cap) {
    const int full = nsplit_full(batch, c.num_kv_heads, sms, max_pages);
    // ~12 tiles per CTA (two rounds of the six consumer warps): fewer, fuller CTAs shorten the
    // latency-bound cluster epilogue.  C1 (133 plan tiles): 16 splits 366 us/step, 12 splits 354,
    // 8 splits 383 (a third round per warp).
    const int by_tiles = std::max(1, (plan_tiles(c, plan_cap) + 11) / 12);
    return std::max(1, std::min(full, by_tiles));
}

// Global-merge kernels (no cluster, one CTA per SM): used when every (sequence, kv head) gets
// at least one CTA in a single wave, i.e. batch * g <= SMs.  Splits per (b, h) = SMs / (b g)
// (C1: 18 -> 144 CTAs), for a sparse layer at most one per ~4 plan tiles (nine consumer warps).
bool use_gmerge(int batch, int g, int sms) { return batch * g <= sms; }

int nsplit_gmerge(int batch, int g, int sms, int items) {
    int n = sms / std::max(1, batch * g);
    n = std::max(1, std::min(n, kMaxSplitG));
    return std::min(n, std::max(1, items));
}

// The deep-ring variant (one CTA per SM) is kept for experiments (DELTA_TUNE deep=1).
bool deep_ring(int, int, int, int) { return false; }

int elem_bytes(const delta_config& c) { return c.kv_dtype == DELTA_BF16 ? 2 : 4; }

// Validation (returns empty string if OK), following SPEC.md:378-386.
std::string validate(const delta_config& c, std::vector<int>& role, std::vector<int>& gov) {
    char buf[256];
    if (c.num_layers < 1) return "num_layers must be >= 1";
    if (c.num_q_heads < 1 || c.num_kv_heads < 1 || c.num_q_heads % c.num_kv_heads != 0)
        return "num_kv_heads must divide num_q_heads";
    if (c.num_q_heads / c.num_kv_heads > kMaxGs) return "num_q_heads / num_kv_heads must be <= 16";
    if (c.num_q_heads > 256) return "num_q_heads must be <= 256";
    if (c.head_dim != 64 && c.head_dim != 128) return "head_dim must be 64 or 128";
    if (c.max_batch < 1 || c.max_seq_len < 1) return "max_batch and max_seq_len must be >= 1";
    if (c.page_size != kPage) return "page_size must be 16 (PAPER.md:196)";
    if (c.kv_dtype != DELTA_BF16 && c.kv_dtype != DELTA_FP32) return "kv_dtype must be BF16 or FP32";
    if (c.num_full_prefix < 0 || c.num_full_prefix > c.num_layers) return "num_full_prefix out of range";
    if (c.num_select_layers < 0 || (c.num_select_layers > 0 && !c.select_layers))
        return "select_layers missing";
    if (c.budget_k < 0 || c.n_sink < 0 || c.n_window < 0) return "budget_k, n_sink, n_window must be >= 0";
    if (c.select_block != 1 && c.select_block != c.page_size) return "select_block must be 1 or page_size";
    if (c.select_block == c.page_size && c.budget_k % c.page_size != 0)
        return "page-level selection needs budget_k % page_size == 0 (R6)";
    if (c.shard_world < 1 || c.shard_world > 64 || c.shard_rank < 0 || c.shard_rank >= c.shard_world)
        return "shard_world must be in [1, 64] and 0 <= shard_rank < shard_world";
    if (c.det_chunks < 0 || c.det_chunks > 64 || (c.det_chunks > 0 && c.det_chunks % std::max(1, c.shard_world) != 0))
        return "det_chunks must be 0 or a multiple of shard_world in [1, 64]";
    if (c.det_chunks > 0 && c.policy != DELTA_POLICY_DELTA) return "det_chunks needs the DELTA policy";
    if (c.softmax_scale < 0.f || !std::isfinite(c.softmax_scale)) return "softmax_scale must be finite and >= 0";
    if (c.policy != DELTA_POLICY_DELTA && c.policy != DELTA_POLICY_QUEST && c.policy != DELTA_POLICY_RAAS)
        return "policy must be DELTA, QUEST or RAAS";
    if (c.policy != DELTA_POLICY_DELTA) {
        // Quest / RaaS: every layer >= F selects (Q1-Q3) or evicts (RS1-RS4) its own pages
        if (c.num_select_layers != 0) return "QUEST / RAAS policies take no Delta layers";
        if (c.select_block != c.page_size) return "QUEST / RAAS work on pages: select_block must be page_size";
        if (c.kv_dtype != DELTA_BF16) return "QUEST / RAAS need bf16 KV";
        if (c.shard_world != 1) return "QUEST / RAAS are not sequence-sharded";
        // raas_update stages 16 B per page of a sequence in shared memory (opt-in limit 200 KiB)
        if (c.policy == DELTA_POLICY_RAAS && 16LL * ((c.max_seq_len + kPage - 1) / kPage + 1) > 200 * 1024)
            return "RAAS: max_seq_len too large for the eviction kernel's shared memory (<= 204,784 tokens)";
        role.assign(c.num_layers, c.policy == DELTA_POLICY_QUEST ? kRoleQuest : kRoleRaas);
        gov.assign(c.num_layers, 0);
        for (int l = 0; l < c.num_layers; ++l) {
            if (l < c.num_full_prefix) role[l] = kRoleFull;
            gov[l] = l;
        }
        return "";
    }
    role.assign(c.num_layers, kRoleSparse);
    gov.assign(c.num_layers, -1);
    for (int i = 0; i < c.num_select_layers; ++i) {
        const int l = c.select_layers[i];
        if (l < c.num_full_prefix || l >= c.num_layers) {
            snprintf(buf, sizeof buf, "Delta layer %d inside the full prefix or out of range", l);
            return buf;
        }
        if (i > 0 && l <= c.select_layers[i - 1]) return "select_layers must be strictly ascending";
    }
    int current = -1, next = 0;
    for (int l = 0; l < c.num_layers; ++l) {
        if (l < c.num_full_prefix) {
            role[l] = kRoleFull; gov[l] = l;
        } else if (next < c.num_select_layers && c.select_layers[next] == l) {
            role[l] = kRoleSelect; gov[l] = l; current = l; ++next;
        } else {
            if (current < 0) {
                snprintf(buf, sizeof buf, "layer %d has no Delta layer at or below it (SPEC.md:382)", l);
                return buf;
            }
            role[l] = kRoleSparse; gov[l] = current;
        }
    }
    return "";
}

Layout layout(const delta_config& c, int sms) {
    Layout L = {};
    const int m = c.num_q_heads, g = c.num_kv_heads, D = c.head_dim;
    const size_t e = elem_bytes(c);
    L.max_pages = (c.max_seq_len + kPage - 1) / kPage;
    L.max_units = (c.max_seq_len + c.select_block - 1) / c.select_block;
    L.n_delta = c.num_select_layers;
    {   // plan capacity in units: salient k/block + max sink units + max window units
        const int blk = c.select_block;
        const int k_units = c.budget_k / blk;
        const int sink_units = c.n_sink > 0 ? (c.n_sink + blk - 1) / blk : 0;
        const int win_units = c.n_window > 0 ? (blk == 1 ? c.n_window : (c.n_window - 1) / blk + 2) : 0;
        L.plan_cap = std::max(1, std::min(L.max_units, k_units + sink_units + win_units));
        if (c.policy == DELTA_POLICY_RAAS) L.plan_cap = L.max_pages + 1;  // starts with every page retained
    }
    const bool has_sel = c.num_select_layers > 0 || c.policy != DELTA_POLICY_DELTA;  // logits, keys, plans
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + std::max<size_t>(bytes, 1)); return o; };
    L.seq_len = take((size_t)c.num_layers * c.max_batch * 4);
    L.err = take(16);
    L.cnt_sel = take((size_t)c.num_layers * c.max_batch * 4);
    L.ticket = take((size_t)c.num_layers * c.max_batch * 4);
    L.raas_last = take(c.policy == DELTA_POLICY_RAAS ? (size_t)c.num_layers * c.max_batch * L.max_pages * 4 : 0);
    L.logits = take(has_sel ? (size_t)c.max_batch * c.max_seq_len * m * 4 : 0);
    L.lse_buf = take((size_t)c.max_batch * m * 4);
    L.keys = take(has_sel ? (size_t)c.max_batch * L.max_units * 4 : 0);
    L.keys_ll = take(has_sel ? (size_t)c.max_batch * L.max_units * 8 : 0);
    L.sel_epoch = take((size_t)c.num_layers * c.max_batch * 4);
    // plan slots: one per Delta layer; QUEST: slot 0 = the current layer's plan; RAAS: one per layer
    const int nd = c.policy == DELTA_POLICY_RAAS ? c.num_layers : std::max(1, L.n_delta);
    L.plan_idx = take((size_t)nd * c.max_batch * L.plan_cap * 4);
    L.plan_phys = take((size_t)nd * c.max_batch * L.plan_cap * 4);
    L.plan_count = take((size_t)nd * c.max_batch * 4);
    L.plan_stamp = take((size_t)nd * c.max_batch * 4);
    L.det_chunks = c.det_chunks;
    L.chunk_pages = c.det_chunks > 0 ? (L.max_pages + c.det_chunks - 1) / c.det_chunks : 0;
    const int nranges = std::max(1, c.det_chunks);  // plan ranges per slot: one per chunk
    L.plan_lo = take((size_t)nd * nranges * c.max_batch * 4);
    L.plan_hi = take((size_t)nd * nranges * c.max_batch * 4);
    {   // sequence sharding exchange buffers: partials (o [B][m][d], lse [B][m]) and candidates;
        // with R21 chunks a rank sends its det_chunks / W chunk partials
        const int W = std::max(1, c.shard_world);
        const bool parts = W > 1 || c.det_chunks > 0;
        L.part_bytes = parts ? align_up((size_t)c.max_batch * m * (D + 1) * 4) : 0;
        L.shard_block = L.part_bytes * (c.det_chunks > 0 ? c.det_chunks / W : 1);
        L.cand_block = W > 1 && has_sel ? align_up((size_t)c.max_batch * L.plan_cap * 8) : 0;
        L.shard_send = take(L.shard_block);
        L.shard_recv = take(W > 1 ? L.shard_block * W : 0);
        L.cand_send = take(L.cand_block);
        L.cand_recv = take(L.cand_block * W);
    }
    // host-path staging, two slots (consecutive delta_decode_step_host calls overlap)
    L.stage_q = take(2 * (size_t)c.num_layers * c.max_batch * m * D * e);
    L.stage_k = take(2 * (size_t)c.num_layers * c.max_batch * g * D * e);
    L.stage_v = take(2 * (size_t)c.num_layers * c.max_batch * g * D * e);
    L.stage_out = take(2 * (size_t)c.num_layers * c.max_batch * m * D * 4);
    L.gslots = std::max(sms, 1) * 2;  // batch * g * nsplit <= sms for every gmerge launch
    L.gpart = take((size_t)L.gslots * gpart_floats(D) * 8);  // LL words (value, flag) with gll
    L.gcnt = take((size_t)c.max_batch * g * kMaxSplitG * 8);  // ticket counter per (b, h, split count)
    {   // Quest page representatives [L][num_phys][g][2][d] bf16
        const long long phys = c.num_phys_pages > 0 ? c.num_phys_pages : (long long)c.max_batch * L.max_pages;
        L.reps_bytes = c.policy == DELTA_POLICY_QUEST ? (size_t)c.num_layers * phys * g * 2 * D * 2 : 0;
        L.reps = take(L.reps_bytes);
    }
    L.total = off;
    return L;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

// NCCL, loaded at run time (the library has no link-time NCCL dependency; in a torch process
// dlopen finds the libnccl.so.2 torch already loaded, else DELTA_NCCL_LIB names it).
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
};

std::string g_nccl_path;  // delta_set_nccl_library (before the first NCCL use)

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);  // the copy already loaded, if any
        if (!lib && !g_nccl_path.empty()) lib = dlopen(g_nccl_path.c_str(), RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            a.why = "libnccl.so.2 not found (delta_set_nccl_library)";
            return a;
        }
        a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(lib, "ncclGetUniqueId"));
        a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(lib, "ncclCommInitRank"));
        a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(lib, "ncclAllGather"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(lib, "ncclCommDestroy"));
        a.getErrorString = reinterpret_cast<decltype(a.getErrorString)>(dlsym(lib, "ncclGetErrorString"));
        a.commGetAsyncError = reinterpret_cast<decltype(a.commGetAsyncError)>(dlsym(lib, "ncclCommGetAsyncError"));
        a.ok = a.getUniqueId && a.commInitRank && a.allGather && a.commDestroy && a.getErrorString;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

// Static page range of a rank: contiguous, page-aligned shares of the max_seq_len pages.
// With R21 chunks a rank's range is the union of its det_chunks / W consecutive chunks.
void shard_pages(const delta_config& c, int rank, int* lo, int* hi) {
    const int max_pages = (c.max_seq_len + kPage - 1) / kPage;
    const int W = std::max(1, c.shard_world);
    const int per = c.det_chunks > 0 ? (max_pages + c.det_chunks - 1) / c.det_chunks * (c.det_chunks / W)
                                      : (max_pages + W - 1) / W;
    *lo = std::min(max_pages, rank * per);
    *hi = std::min(max_pages, (rank + 1) * per);
    if (W == 1) { *lo = 0; *hi = 0x7fffffff; }
}

namespace delta {
int cluster_limit(const void* kern, int threads, int smem_bytes) {
    for (int cs = kMaxSplit; cs > 1; cs /= 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs, 1, 1);
        cfg.blockDim = dim3(threads, 1, 1);
        cfg.dynamicSmemBytes = smem_bytes;
        cudaLaunchAttribute a;
        a.id = cudaLaunchAttributeClusterDimension;
        a.val.clusterDim.x = cs;
        a.val.clusterDim.y = 1;
        a.val.clusterDim.z = 1;
        cfg.attrs = &a;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) return cs;
        cudaGetLastError();
    }
    return 1;
}
}  // namespace delta

struct delta_ctx {
    delta_config cfg;
    std::vector<int32_t> select_layers;
    std::vector<int> role, gov, slot;  // slot: Delta layer -> plan index
    Layout L;
    int sms = 148, gs = 1;
    uint8_t* ws = nullptr;
    void* kv_pool = nullptr;
    const int32_t* block_table = nullptr;
    CUtensorMap tm_kv;
    CUtensorMap tm_kvp;  // prefill: one box = 16 rows (K or V of a (page, head)) x one 64-column half
    bool use_tc = false;
    float scale = 0.f;
    std::vector<long long> step, dec_step, sel_step;
    // graph cache for delta_decode_step
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        const void* key[7] = {};
        int batch = -1;
        uint64_t kernels = 0;
    } graphs[3];  // the caller's step + the two host-path staging slots
    int graph_next = 0;  // round-robin replacement
    // delta_decode_step_host pipeline: copy-in, compute and copy-out streams, per staging slot
    // events (inputs landed, step done, outputs read)
    bool host_init = false, host_pending = false;
    int host_slot = 0;
    cudaStream_t hs_in = nullptr, hs_comp = nullptr, hs_out = nullptr;
    cudaEvent_t hev_in[2] = {}, hev_done[2] = {}, hev_out[2] = {}, hev_join = nullptr;
    uint64_t launches = 0;
    uint64_t captures = 0;  // decode-step graph captures (a timed loop of replays must not add any)
    bool pdl = true;
    int tune_nsplit = 0, tune_deep = -1;  // DELTA_TUNE overrides (0 / -1 = automatic)
    int tune_snsplit = 0;                 // sparse layers only
    // tcgen05 kernel (attn_umma.cu): correct, but one tcgen05.mma of a 16-token tile costs ~48
    // cycles to issue (tools/umma_test.cu), so 10 per tile lose to the mma.sync kernel here;
    // kept selectable (DELTA_TUNE umma=1) and parity-tested.
    int tune_prewait = 1, tune_early = 1, tune_umma = 0, tune_policy = 0;
    int tune_seltrig = 0, tune_selhist = 0, tune_gmerge = 1, tune_gm2 = 0, tune_lat = 1, tune_qpf = 1, tune_pfumma = 3, tune_gll = 1, tune_selll = 1, tune_gfix = 1;
    // sequence sharding
    int world = 1, rank = 0, page_lo = 0, page_hi = 0x7fffffff;
    ncclComm_t comm = nullptr;  // null with world > 1: the caller exchanges (delta_shard_* calls)
    // the previous kernel this handle enqueued (decides whether the next attention kernel
    // may start its KV stream before griddepcontrol.wait; see attn_tc.cu)
    enum { kLastNone, kLastAttn, kLastSelect, kLastAppend } last_kind = kLastNone;
    int last_layer = -1;
    std::string msg;

    template <typename T>
    T* at(size_t off) const { return reinterpret_cast<T*>(ws + off); }
};

namespace {

delta_status fail(delta_ctx* h, delta_status st, const std::string& m) {
    if (h) h->msg = m; else g_msg = m;
    return st;
}

delta_status cuda_fail(delta_ctx* h, cudaError_t e, const char* what) {
    return fail(h, DELTA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Work of earlier delta_decode_step_host calls runs on the handle's internal streams: order the
// caller's stream after it before any other call enqueues work there.
delta_status join_host(delta_ctx* h, cudaStream_t st) {
    if (!h || !h->host_pending) return DELTA_OK;
    cudaError_t e = cudaEventRecord(h->hev_join, h->hs_comp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, h->hev_join, 0);
    if (e != cudaSuccess) return cuda_fail(h, e, "join host pipeline");
    h->host_pending = false;
    return DELTA_OK;
}

AttnParams attn_params(delta_ctx* h, int layer, int batch, int role_override = -1) {
    const delta_config& c = h->cfg;
    AttnParams p = {};
    const int hrole = role_override >= 0 ? role_override : h->role[layer];
    p.m = c.num_q_heads; p.g = c.num_kv_heads; p.gs = h->gs; p.d = c.head_dim;
    p.layer = layer; p.batch = batch;
    p.role = (hrole == kRoleQuest || hrole == kRoleRaas) ? kRoleSparse : hrole;  // they attend their plan
    p.emit_logits = (hrole == kRoleSelect || hrole == kRoleRaas) ? 1 : 0;
    p.num_phys = c.num_phys_pages; p.bt_stride = h->L.max_pages;
    p.max_batch = c.max_batch; p.max_seq = c.max_seq_len;
    p.sel_block = c.select_block; p.plan_cap = h->L.plan_cap;
    p.scale = h->scale; p.scale_log2 = (float)((double)h->scale * 1.4426950408889634);
    p.kv_pool = h->kv_pool; p.block_table = h->block_table;
    p.seq_len = h->at<int32_t>(h->L.seq_len);
    p.logits = h->at<float>(h->L.logits); p.lse_buf = h->at<float>(h->L.lse_buf);
    p.err = h->at<int32_t>(h->L.err);
    if (p.role == kRoleSparse) {
        const int sl = h->slot[h->gov[layer]];
        p.plan_idx = h->at<int32_t>(h->L.plan_idx) + (size_t)sl * c.max_batch * h->L.plan_cap;
        p.plan_phys = h->at<int32_t>(h->L.plan_phys) + (size_t)sl * c.max_batch * h->L.plan_cap;
        p.plan_count = h->at<int32_t>(h->L.plan_count) + (size_t)sl * c.max_batch;
        p.plan_stamp = h->at<int32_t>(h->L.plan_stamp) + (size_t)sl * c.max_batch;
        p.nsplit = nsplit_sparse(c, batch, h->sms, h->L.max_pages, h->L.plan_cap);
    } else {
        p.nsplit = nsplit_full(batch, c.num_kv_heads, h->sms, h->L.max_pages);
    }
    p.page_lo = h->page_lo;
    p.page_hi = h->page_hi;
    if (h->world > 1 || h->L.det_chunks) {  // partials for the merge (launch_decode sets each chunk's)
        p.part_o = h->at<float>(h->L.shard_send);
        p.part_lse = p.part_o + (size_t)batch * c.num_q_heads * c.head_dim;
        if (p.role == kRoleSparse) {
            const int sl = h->slot[h->gov[layer]];
            const size_t nr = std::max(1, h->L.det_chunks);
            p.plan_lo = h->at<int32_t>(h->L.plan_lo) + (size_t)sl * nr * c.max_batch;
            p.plan_hi = h->at<int32_t>(h->L.plan_hi) + (size_t)sl * nr * c.max_batch;
        }
    }
    // (the tcgen05 and fp32 kernels keep the cluster merge)
    //  tune_gmerge: 0 never, 1 full-cache layers (FULL / SELECT), 2 every role
    const bool gm_role = h->tune_gmerge == 2 || (h->tune_gmerge == 1 && p.role != kRoleSparse);
    p.gmerge = (gm_role && h->use_tc && !h->tune_umma && use_gmerge(batch, c.num_kv_heads, h->sms)) ? 1 : 0;
    if (p.gmerge) {
        const int items = p.role == kRoleSparse ? (plan_tiles(c, h->L.plan_cap) + 3) / 4 : h->L.max_pages;
        p.nsplit = nsplit_gmerge(batch, c.num_kv_heads, h->sms, items);
        p.gpart = h->at<float>(h->L.gpart);
        p.gcnt = h->at<unsigned long long>(h->L.gcnt);
        p.gm_shallow = h->tune_gm2;
        p.gll = h->tune_gll;
        p.fixed_part = (p.role != kRoleSparse && h->world == 1 && !h->L.det_chunks) ? h->tune_gfix : 0;
    }
    const int cap = p.gmerge ? std::min(kMaxSplitG, h->L.gslots / std::max(1, batch * c.num_kv_heads)) : kMaxSplit;
    if (h->tune_nsplit > 0) p.nsplit = std::min(h->tune_nsplit, cap);
    if (h->tune_snsplit > 0 && p.role == kRoleSparse) p.nsplit = std::min(h->tune_snsplit, cap);
    // SPARSE page plans at small batch: the latency kernel (attn_sparse.cu) when every split's
    // share of the plan fits its resident tiles and two layers' CTAs fit one wave
    if (p.role == kRoleSparse && !p.emit_logits && h->use_tc && !h->tune_umma && h->tune_lat &&
        c.select_block == kPage && h->world == 1 && !h->L.det_chunks && h->gs <= 8) {
        const int lim = sparse_lat_max_split(c.head_dim);
        int ns = h->tune_snsplit > 0 ? h->tune_snsplit : 12;
        ns = std::min(ns, lim);
        const int tiles = plan_tiles(c, h->L.plan_cap);
        if (ns >= 1 && (tiles + ns - 1) / ns <= sparse_lat_max_tiles() && batch * c.num_kv_heads * ns <= h->sms) {
            p.sparse_lat = 1;
            p.gmerge = 0;
            p.nsplit = ns;
        }
    }
    p.deep = deep_ring(batch, c.num_kv_heads, p.nsplit, h->sms) ? 1 : 0;
    if (h->tune_deep >= 0) p.deep = h->tune_deep;
    return p;
}

delta_status check_layer_batch(delta_ctx* h, int layer, int batch) {
    if (!h) return fail(nullptr, DELTA_ERR_USAGE, "null handle");
    if (layer < 0 || layer >= h->cfg.num_layers) return fail(h, DELTA_ERR_USAGE, "layer out of range");
    if (batch < 1 || batch > h->cfg.max_batch) return fail(h, DELTA_ERR_USAGE, "batch out of range");
    return DELTA_OK;
}

// host-side plan freshness: a SPARSE layer may only run after its governing
// Delta layer selected at THIS step (R13).
delta_status check_sparse_fresh(delta_ctx* h, int layer, bool appending) {
    if (h->role[layer] != kRoleSparse) return DELTA_OK;
    const int d = h->gov[layer];
    const long long my_step = h->step[layer] + (appending ? 1 : 0);
    if (h->sel_step[h->slot[d]] != h->step[d] || my_step != h->step[d])
        return fail(h, DELTA_ERR_USAGE,
                    "stale plan: layer " + std::to_string(layer) + " needs delta_select on Delta layer " +
                        std::to_string(d) + " at this step (PAPER.md:160-161)");
    return DELTA_OK;
}

delta_status shard_allgather(delta_ctx* h, size_t send_off, size_t recv_off, size_t bytes, cudaStream_t st) {
    ncclResult_t r = nccl().allGather(h->ws + send_off, h->ws + recv_off, bytes, ncclUint8, h->comm, st);
    if (r != ncclSuccess) return fail(h, DELTA_ERR_NCCL, std::string("ncclAllGather: ") + nccl().getErrorString(r));
    return DELTA_OK;
}

// Cross-rank LSE merge of the attention partials (shard.cu) -> out, lse_out (and the Delta
// layer's global LSE for scoring).
delta_status launch_merge(delta_ctx* h, int layer, int batch, float* out, float* lse_out, cudaStream_t st) {
    const delta_config& c = h->cfg;
    ShardMergeParams mp = {};
    // R21 chunks: the det_chunks partials in chunk order (one rank: its own send block), merged
    // by the same fixed left fold whatever W is -> bitwise identical across W
    mp.world = h->L.det_chunks ? h->L.det_chunks : h->world;
    mp.batch = batch; mp.m = c.num_q_heads; mp.d = c.head_dim; mp.role = h->role[layer];
    mp.recv_o = h->at<float>(h->world > 1 ? h->L.shard_recv : h->L.shard_send);
    mp.recv_lse = mp.recv_o + (size_t)batch * c.num_q_heads * c.head_dim;
    mp.o_stride = mp.lse_stride = h->L.part_bytes / 4;
    mp.out = out; mp.lse_out = lse_out; mp.lse_buf = h->at<float>(h->L.lse_buf);
    mp.err = h->at<int32_t>(h->L.err);
    cudaError_t e = launch_shard_merge(mp, st, h->pdl);
    if (e != cudaSuccess) return cuda_fail(h, e, "shard merge launch");
    ++h->launches;
    h->last_kind = delta_ctx::kLastAttn;
    h->last_layer = layer;
    return DELTA_OK;
}

QuestParams quest_params(delta_ctx* h, int layer, int batch, const void* q) {
    const delta_config& c = h->cfg;
    QuestParams p = {};
    p.m = c.num_q_heads; p.g = c.num_kv_heads; p.d = c.head_dim; p.layer = layer; p.batch = batch;
    p.num_phys = c.num_phys_pages; p.bt_stride = h->L.max_pages; p.max_batch = c.max_batch;
    p.max_units = h->L.max_units;
    p.kv_pool = h->kv_pool; p.reps = h->ws + h->L.reps; p.block_table = h->block_table;
    p.seq_len = h->at<int32_t>(h->L.seq_len); p.q = q; p.keys = h->at<float>(h->L.keys);
    return p;
}

delta_status launch_append_impl(delta_ctx* h, int layer, int batch, int ntok, const void* k_new, const void* v_new,
                                cudaStream_t st) {
    AppendParams p = {};
    p.g = h->cfg.num_kv_heads; p.d = h->cfg.head_dim; p.layer = layer; p.batch = batch; p.ntok = ntok;
    p.num_phys = h->cfg.num_phys_pages; p.bt_stride = h->L.max_pages; p.max_batch = h->cfg.max_batch;
    p.max_seq = h->cfg.max_seq_len; p.elem_bytes = elem_bytes(h->cfg);
    p.k_new = k_new; p.v_new = v_new; p.kv_pool = h->kv_pool;
    p.reps = h->role[layer] == kRoleQuest ? h->ws + h->L.reps : nullptr;
    p.ticket = h->at<int32_t>(h->L.ticket);
    p.block_table = h->block_table; p.seq_len = h->at<int32_t>(h->L.seq_len); p.err = h->at<int32_t>(h->L.err);
    p.page_lo = h->page_lo; p.page_hi = h->page_hi;
    cudaError_t e = launch_append(p, st, h->pdl);
    if (e != cudaSuccess) return cuda_fail(h, e, "append launch");
    ++h->launches;
    h->last_kind = delta_ctx::kLastAppend;
    h->last_layer = layer;
    return DELTA_OK;
}

delta_status launch_sel(delta_ctx* h, int layer, int batch, const float* keys_override, int32_t* idx_out,
                        int32_t* count_out, cudaStream_t st, int shard_mode, const void* k_new = nullptr,
                        const void* v_new = nullptr);

// A Quest layer before its attention: page keys over the pages before this step's token (its
// page is a forced window page), then one launch that appends the token (pool rows, reps,
// length) and ranks the pages -> plan slot 0.
delta_status launch_quest_select(delta_ctx* h, int layer, int batch, const void* k_new, const void* v_new,
                                 const void* q, cudaStream_t st, bool in_step) {
    QuestParams qp = quest_params(h, layer, batch, q);
    // early reads only inside a captured step, and only if the previous kernel is another
    // layer's (an append, attention or reps rebuild of this layer writes its counter / reps)
    qp.prewait = (in_step && h->tune_prewait && h->last_kind != delta_ctx::kLastNone && h->last_layer != layer) ? 1 : 0;
    cudaError_t e = launch_quest_score(qp, h->L.max_pages, h->sms, st, h->pdl);
    if (e != cudaSuccess) return cuda_fail(h, e, "quest score launch");
    ++h->launches;
    return launch_sel(h, layer, batch, h->at<float>(h->L.keys), nullptr, nullptr, st, 0, k_new, v_new);
}

RaasParams raas_params(delta_ctx* h, int layer, int batch) {
    const delta_config& c = h->cfg;
    RaasParams p = {};
    const int sl = h->slot[layer];
    p.m = c.num_q_heads; p.g = c.num_kv_heads; p.layer = layer; p.batch = batch; p.max_batch = c.max_batch;
    p.max_seq = c.max_seq_len; p.max_pages = h->L.max_pages; p.plan_cap = h->L.plan_cap;
    p.n_sink = c.n_sink; p.n_window = c.n_window; p.k_pages = c.budget_k / c.page_size;
    p.seq_len = h->at<int32_t>(h->L.seq_len);
    p.logits = h->at<float>(h->L.logits); p.lse = h->at<float>(h->L.lse_buf);
    p.plan_idx = h->at<int32_t>(h->L.plan_idx) + (size_t)sl * c.max_batch * h->L.plan_cap;
    p.plan_phys = h->at<int32_t>(h->L.plan_phys) + (size_t)sl * c.max_batch * h->L.plan_cap;
    p.plan_count = h->at<int32_t>(h->L.plan_count) + (size_t)sl * c.max_batch;
    p.plan_stamp = h->at<int32_t>(h->L.plan_stamp) + (size_t)sl * c.max_batch;
    p.last = h->at<int32_t>(h->L.raas_last) + (size_t)layer * c.max_batch * h->L.max_pages;
    p.scores = h->at<float>(h->L.keys); p.max_units = h->L.max_units;
    p.block_table = h->block_table; p.bt_stride = h->L.max_pages;
    p.ticket = h->at<int32_t>(h->L.ticket);
    return p;
}

delta_status launch_decode(delta_ctx* h, int layer, int batch, const void* k_new, const void* v_new,
                           const void* q, float* out, float* lse_out, cudaStream_t st, bool in_step = false) {
    NvtxRange nv(role_name(h->role[layer]), layer);
    if (h->role[layer] == kRoleQuest) {
        delta_status s = launch_quest_select(h, layer, batch, k_new, v_new, q, st, in_step);
        if (s != DELTA_OK) return s;
        k_new = v_new = nullptr;  // appended above
    }
    AttnParams p = attn_params(h, layer, batch);
    p.q = q; p.out = out; p.lse_out = lse_out;
    p.fuse_append = (k_new != nullptr);
    p.k_new = k_new; p.v_new = v_new;
    // May the kernel read its length counter, block table and plan before the previous kernel
    // completes?  Not if that kernel is this layer's own (append / attention: the counter) or
    // the select that wrote this sparse layer's plan.
    // Only inside a captured step, where every kernel on the stream is this handle's and in
    // this order; eager calls may follow other work on the stream.
    p.prewait = (in_step && h->tune_prewait) ? 1 : 0;
    p.early_trigger = h->tune_early;
    p.q_prefetch = h->tune_qpf;
    p.cluster_policy = h->tune_policy;
    if (h->last_kind == delta_ctx::kLastNone) p.prewait = 0;
    if (h->last_layer == layer && (h->last_kind == delta_ctx::kLastAppend || h->last_kind == delta_ctx::kLastAttn))
        p.prewait = 0;
    if (p.role == kRoleSparse && h->last_kind == delta_ctx::kLastSelect && h->last_layer == h->gov[layer])
        p.prewait = 0;
    // bf16: the tcgen05/TMEM kernel for GQA groups of <= 8 heads, the mma.sync kernel otherwise;
    // fp32 caches: the CUDA-core kernel (no tensor-core rounding of fp32 inputs).
    auto launch_attn = [&](const AttnParams& ap) {
        return !h->use_tc ? launch_attn_simt(ap, h->cfg.kv_dtype == DELTA_BF16, st, h->pdl)
               : ap.sparse_lat ? launch_attn_sparse_lat(ap, &h->tm_kv, st, h->pdl)
               : (h->tune_umma && umma_supported(ap)) ? launch_attn_umma(ap, &h->tm_kv, st, h->pdl)
                                                      : launch_attn_tc(ap, &h->tm_kv, st, h->pdl);
    };
    cudaError_t e = cudaSuccess;
    if (h->L.det_chunks) {
        // R21 fixed chunks: the token is appended first (the rank's pages), then one launch per
        // chunk this rank holds, each over exactly that chunk's pages (or its plan entries) with
        // the W-independent split count, into the chunk's slot of the send block
        if (k_new) {
            delta_status s = launch_append_impl(h, layer, batch, 1, k_new, v_new, st);
            if (s != DELTA_OK) return s;
        }
        p.fuse_append = 0; p.k_new = p.v_new = nullptr;
        p.prewait = 0;
        const int per_rank = h->L.det_chunks / h->world;
        const size_t mb = h->cfg.max_batch;
        const int32_t* lo0 = p.plan_lo;
        const int32_t* hi0 = p.plan_hi;
        for (int i = 0; i < per_rank && e == cudaSuccess; ++i) {
            const int chunk = h->rank * per_rank + i;
            AttnParams cp = p;
            cp.page_lo = chunk * h->L.chunk_pages;
            cp.page_hi = cp.page_lo + h->L.chunk_pages;
            cp.part_o = h->at<float>(h->L.shard_send + (size_t)i * h->L.part_bytes);
            cp.part_lse = cp.part_o + (size_t)batch * h->cfg.num_q_heads * h->cfg.head_dim;
            if (lo0) { cp.plan_lo = lo0 + chunk * mb; cp.plan_hi = hi0 + chunk * mb; }
            e = launch_attn(cp);
            if (e == cudaSuccess) ++h->launches;
        }
    } else {
        e = launch_attn(p);
        if (e == cudaSuccess) ++h->launches;
    }
    if (e != cudaSuccess) return cuda_fail(h, e, "decode launch");
    h->last_kind = delta_ctx::kLastAttn;
    h->last_layer = layer;
    if (h->role[layer] == kRoleRaas) {  // refresh + evict -> the retained set of the next step
        e = launch_raas_update(raas_params(h, layer, batch), st, h->pdl);
        if (e != cudaSuccess) return cuda_fail(h, e, "raas update launch");
        ++h->launches;
    }
    if (h->world > 1 && h->comm) {  // sequence sharding: all-gather the partials, then merge
        delta_status s2 = shard_allgather(h, h->L.shard_send, h->L.shard_recv, h->L.shard_block, st);
        if (s2 != DELTA_OK) return s2;
        return launch_merge(h, layer, batch, out, lse_out, st);
    }
    if (h->world == 1 && h->L.det_chunks) return launch_merge(h, layer, batch, out, lse_out, st);
    return DELTA_OK;
}

delta_status launch_sel(delta_ctx* h, int layer, int batch, const float* keys_override, int32_t* idx_out,
                        int32_t* count_out, cudaStream_t st, int shard_mode, const void* k_new, const void* v_new) {
    NvtxRange nv(k_new ? "QUEST select+append" : "score+top-k", layer);
    const delta_config& c = h->cfg;
    SelectParams p = {};
    p.k_new = k_new; p.v_new = v_new; p.kv_pool = h->kv_pool; p.reps = h->ws + h->L.reps;
    p.d = c.head_dim; p.num_phys = c.num_phys_pages;
    const int sl = h->slot[layer];
    p.m = c.num_q_heads; p.g = c.num_kv_heads; p.layer = layer; p.batch = batch;
    p.nchunk = std::max(1, std::min((h->L.max_units + 15) / 16, (2 * h->sms + batch - 1) / batch));
    p.late_trigger = h->tune_seltrig;
    p.hist_mode = h->tune_selhist;
    p.sel_block = c.select_block; p.n_sink = c.n_sink; p.n_window = c.n_window;
    p.k_units = c.budget_k / c.select_block;
    p.max_batch = c.max_batch; p.max_seq = c.max_seq_len; p.max_units = h->L.max_units; p.plan_cap = h->L.plan_cap;
    p.seq_len = h->at<int32_t>(h->L.seq_len);
    p.logits = h->at<float>(h->L.logits); p.lse_buf = h->at<float>(h->L.lse_buf);
    p.keys_override = keys_override; p.keys = h->at<float>(h->L.keys);
    p.plan_idx = h->at<int32_t>(h->L.plan_idx) + (size_t)sl * c.max_batch * h->L.plan_cap;
    p.plan_phys = h->at<int32_t>(h->L.plan_phys) + (size_t)sl * c.max_batch * h->L.plan_cap;
    p.block_table = h->block_table; p.bt_stride = h->L.max_pages;
    p.plan_count = h->at<int32_t>(h->L.plan_count) + (size_t)sl * c.max_batch;
    p.plan_stamp = h->at<int32_t>(h->L.plan_stamp) + (size_t)sl * c.max_batch;
    p.idx_out = idx_out; p.count_out = count_out;
    p.cnt = h->at<int32_t>(h->L.cnt_sel) + (size_t)layer * c.max_batch;
    p.ll = (h->tune_selll && shard_mode == 0 && !keys_override && !k_new && h->L.max_units <= kSelSmemUnits) ? 1 : 0;
    p.keys_ll = h->at<uint2>(h->L.keys_ll);
    p.epoch = h->at<int32_t>(h->L.sel_epoch);  // one epoch per sequence: keys_ll is shared by the layers
    p.shard_mode = shard_mode;
    p.page_lo = h->page_lo; p.page_hi = h->page_hi;
    p.cand_out = h->at<uint2>(h->L.cand_send);
    {   // plan ranges for the sharded attention: each R21 chunk, else this rank's pages
        const size_t nr = std::max(1, h->L.det_chunks);
        p.plan_lo = h->at<int32_t>(h->L.plan_lo) + (size_t)sl * nr * c.max_batch;
        p.plan_hi = h->at<int32_t>(h->L.plan_hi) + (size_t)sl * nr * c.max_batch;
        if (h->L.det_chunks && shard_mode != 1) {
            p.range_n = h->L.det_chunks; p.range_first = 0; p.range_step = h->L.chunk_pages;
        } else if (shard_mode == 2) {
            p.range_n = 1; p.range_first = h->page_lo; p.range_step = h->page_hi - h->page_lo;
        }
    }
    p.err = h->at<int32_t>(h->L.err);
    cudaError_t e = launch_select(p, st, h->pdl);
    if (e != cudaSuccess) return cuda_fail(h, e, "select launch");
    ++h->launches;
    h->last_kind = delta_ctx::kLastSelect;
    h->last_layer = layer;
    return DELTA_OK;
}

// Global selection merge (sequence sharding): dense keys from every rank's candidates, then
// the unchanged forced-union + top-k (select.cu shard_mode 2).
delta_status launch_sel_merge(delta_ctx* h, int layer, int batch, int32_t* idx_out, int32_t* count_out,
                              cudaStream_t st) {
    const delta_config& c = h->cfg;
    float* keys = h->at<float>(h->L.keys);
    cudaError_t e = launch_cand_scatter(h->at<uint2>(h->L.cand_recv), h->world, batch, h->L.plan_cap,
                                        h->L.cand_block / 8, keys, h->L.max_units, h->at<int32_t>(h->L.seq_len),
                                        layer, c.max_batch, c.num_kv_heads, c.select_block, st, h->pdl);
    if (e != cudaSuccess) return cuda_fail(h, e, "candidate scatter launch");
    ++h->launches;
    return launch_sel(h, layer, batch, keys, idx_out, count_out, st, 2);
}

// Sharded selection: local candidates, exchange, merge (or stop after the local pass when the
// caller runs the exchange itself).
delta_status launch_sel_sharded(delta_ctx* h, int layer, int batch, int32_t* idx_out, int32_t* count_out,
                                cudaStream_t st) {
    delta_status s = launch_sel(h, layer, batch, nullptr, nullptr, nullptr, st, 1);
    if (s != DELTA_OK || !h->comm) return s;
    s = shard_allgather(h, h->L.cand_send, h->L.cand_recv, h->L.cand_block, st);
    if (s != DELTA_OK) return s;
    return launch_sel_merge(h, layer, batch, idx_out, count_out, st);
}

// enqueue one whole step (fused append + decode per layer, select after Delta layers)
delta_status enqueue_step(delta_ctx* h, int batch, const void* q_all, const void* k_all, const void* v_all,
                          float* out_all, float* lse_all, cudaStream_t st) {
    const delta_config& c = h->cfg;
    const size_t e = elem_bytes(c);
    const size_t q_l = (size_t)batch * c.num_q_heads * c.head_dim;
    const size_t kv_l = (size_t)batch * c.num_kv_heads * c.head_dim;
    for (int l = 0; l < c.num_layers; ++l) {
        const uint8_t* q = static_cast<const uint8_t*>(q_all) + l * q_l * e;
        const uint8_t* k = static_cast<const uint8_t*>(k_all) + l * kv_l * e;
        const uint8_t* v = static_cast<const uint8_t*>(v_all) + l * kv_l * e;
        if (l == 0) h->last_kind = delta_ctx::kLastNone;  // first node: its predecessor is outside the step
        delta_status s = launch_decode(h, l, batch, k, v, q, out_all + l * q_l,
                                       lse_all ? lse_all + (size_t)l * batch * c.num_q_heads : nullptr, st, true);
        if (s != DELTA_OK) return s;
        if (h->role[l] == kRoleSelect) {
            s = h->world > 1 ? launch_sel_sharded(h, l, batch, nullptr, nullptr, st)
                             : launch_sel(h, l, batch, nullptr, nullptr, nullptr, st, 0);
            if (s != DELTA_OK) return s;
        }
    }
    return DELTA_OK;
}

void mark_step_done(delta_ctx* h) {
    for (int l = 0; l < h->cfg.num_layers; ++l) {
        h->step[l] += 1;
        h->dec_step[l] = h->step[l];
        if (h->role[l] == kRoleSelect) h->sel_step[h->slot[l]] = h->step[l];
    }
}

}  // namespace

extern "C" {

const char* delta_version(void) { return "delta-b200 0.1 (sm_100a)"; }

delta_status delta_query_sizes(const delta_config* cfg, size_t* kv_pool_bytes, size_t* workspace_bytes) {
    if (!cfg) return fail(nullptr, DELTA_ERR_CONFIG, "null config");
    std::vector<int> role, gov;
    std::string err = validate(*cfg, role, gov);
    if (!err.empty()) return fail(nullptr, DELTA_ERR_CONFIG, err);
    delta_config c = *cfg;
    const int max_pages = (c.max_seq_len + kPage - 1) / kPage;
    const long long phys = c.num_phys_pages > 0 ? c.num_phys_pages : (long long)c.max_batch * max_pages;
    if (kv_pool_bytes)
        *kv_pool_bytes = (size_t)c.num_layers * phys * c.num_kv_heads * 2 * kPage * c.head_dim * elem_bytes(c);
    if (workspace_bytes) *workspace_bytes = layout(c, num_sms_current()).total;
    return DELTA_OK;
}

delta_status delta_create(const delta_config* cfg, const delta_buffers* bufs, delta_t* out) {
    if (!cfg || !bufs || !out) return fail(nullptr, DELTA_ERR_USAGE, "null argument");
    *out = nullptr;
    std::vector<int> role, gov;
    std::string err = validate(*cfg, role, gov);
    if (!err.empty()) return fail(nullptr, DELTA_ERR_CONFIG, err);
    delta_ctx* h = new delta_ctx();
    h->cfg = *cfg;
    h->select_layers.assign(cfg->select_layers, cfg->select_layers + cfg->num_select_layers);
    h->cfg.select_layers = h->select_layers.data();
    const int max_pages = (cfg->max_seq_len + kPage - 1) / kPage;
    if (h->cfg.num_phys_pages <= 0) h->cfg.num_phys_pages = cfg->max_batch * max_pages;
    h->role = role; h->gov = gov;
    h->slot.assign(cfg->num_layers, -1);
    for (int i = 0; i < cfg->num_select_layers; ++i) h->slot[cfg->select_layers[i]] = i;
    for (int l = 0; l < cfg->num_layers; ++l)
        if (h->role[l] == kRoleQuest) h->slot[l] = 0;  // each Quest layer's own plan, consumed at once
        else if (h->role[l] == kRoleRaas) h->slot[l] = l;  // each RaaS layer's persistent retained set
    h->sms = num_sms_current();
    h->gs = cfg->num_q_heads / cfg->num_kv_heads;
    h->L = layout(h->cfg, h->sms);
    h->scale = cfg->softmax_scale > 0.f ? cfg->softmax_scale : (float)(1.0 / std::sqrt((double)cfg->head_dim));
    if (!bufs->kv_pool || !bufs->block_table || !bufs->workspace) {
        delete h;
        return fail(nullptr, DELTA_ERR_USAGE, "null buffer");
    }
    if (bufs->workspace_bytes < h->L.total) {
        delete h;
        return fail(nullptr, DELTA_ERR_CAPACITY, "workspace too small: need " + std::to_string(h->L.total));
    }
    if (reinterpret_cast<uintptr_t>(bufs->workspace) % kAlign || reinterpret_cast<uintptr_t>(bufs->kv_pool) % 1024) {
        delete h;
        return fail(nullptr, DELTA_ERR_USAGE, "workspace must be 256-byte and kv_pool 1024-byte aligned");
    }
    h->ws = static_cast<uint8_t*>(bufs->workspace);
    h->kv_pool = bufs->kv_pool; h->block_table = bufs->block_table;
    h->use_tc = (cfg->kv_dtype == DELTA_BF16);
    if (h->use_tc) {
        const unsigned long long rows =  // rows of d elements in the pool (K and V rows)
            (unsigned long long)cfg->num_layers * h->cfg.num_phys_pages * cfg->num_kv_heads * 2 * kPage;
        if (rows >= (1ull << 31)) {
            delete h;
            return fail(nullptr, DELTA_ERR_CONFIG, "pool too large for 32-bit TMA row coordinates");
        }
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || !fn || q != cudaDriverEntryPointSuccess) {
            delete h;
            return fail(nullptr, DELTA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        }
        auto encode = reinterpret_cast<PFN_encodeTiled>(fn);
        // One box = one (page, head): its P K rows and P V rows (2P rows x d), i.e. one 4 KiB
        // (d = 64) or 8 KiB (d = 128) request.  d = 64: 2-D {64, rows}.  d = 128: 3-D
        // {64, rows, 2 halves} so a single request covers both 128-byte halves of each row under
        // the 128B swizzle (inner box extent <= 128 bytes) and lands as [half][row][128 B], the
        // canonical tcgen05 SW128 operand layout (combine.cuh TileLayout).
        const bool d128 = cfg->head_dim == 128;
        const cuuint32_t rank = d128 ? 3 : 2;
        const cuuint64_t dims[3] = {64, (cuuint64_t)rows, 2};
        const cuuint64_t strides[2] = {d128 ? 256ull : 128ull, 128ull};
        const cuuint32_t box[3] = {64, (cuuint32_t)(2 * kPage), 2};
        const cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode(&h->tm_kv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, bufs->kv_pool, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        // prefill_umma.cu: the K rows and the V rows of a (page, head) as separate boxes, one
        // 64-column half each, so 4 pages land as one uniformly strided [half][64 rows][128 B]
        const cuuint32_t boxp[3] = {64, (cuuint32_t)kPage, 1};
        if (r == CUDA_SUCCESS)
            r = encode(&h->tm_kvp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, bufs->kv_pool, dims, strides, boxp, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            delete h;
            return fail(nullptr, DELTA_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
        }
    }
    cudaError_t e = cudaMemset(h->ws, 0, h->L.total);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        std::string m = std::string("workspace init: ") + cudaGetErrorString(e);
        delete h;
        return fail(nullptr, DELTA_ERR_CUDA, m);
    }
    h->world = std::max(1, cfg->shard_world);
    h->rank = cfg->shard_rank;
    shard_pages(h->cfg, h->rank, &h->page_lo, &h->page_hi);
    if (h->world > 1 && cfg->nccl_id) {
        const NcclApi& api = nccl();
        if (!api.ok) {
            std::string m = api.why;
            delete h;
            return fail(nullptr, DELTA_ERR_NCCL, m);
        }
        ncclUniqueId id;
        std::memcpy(&id, cfg->nccl_id, sizeof id);
        ncclResult_t r = api.commInitRank(&h->comm, h->world, id, h->rank);
        if (r != ncclSuccess) {
            std::string m = std::string("ncclCommInitRank: ") + api.getErrorString(r);
            delete h;
            return fail(nullptr, DELTA_ERR_NCCL, m);
        }
    }
    h->step.assign(cfg->num_layers, 0);
    h->dec_step.assign(cfg->num_layers, -1);
    h->sel_step.assign(std::max(1, cfg->num_select_layers), -1);
    *out = h;
    return DELTA_OK;
}

delta_status delta_destroy(delta_t h) {
    if (!h) return DELTA_ERR_USAGE;
    for (auto& g : h->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (h->host_init) {
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(h->hev_in[i]);
            cudaEventDestroy(h->hev_done[i]);
            cudaEventDestroy(h->hev_out[i]);
        }
        cudaEventDestroy(h->hev_join);
        cudaStreamDestroy(h->hs_in);
        cudaStreamDestroy(h->hs_comp);
        cudaStreamDestroy(h->hs_out);
    }
    if (h->comm) nccl().commDestroy(h->comm);
    delete h;
    return DELTA_OK;
}

delta_status delta_set_seq_lens(delta_t h, int32_t layer, int32_t batch, const int32_t* lens_host,
                                cudaStream_t stream) {
    if (!h) return fail(nullptr, DELTA_ERR_USAGE, "null handle");
    { delta_status j = join_host(h, stream); if (j != DELTA_OK) return j; }
    if (batch < 1 || batch > h->cfg.max_batch || !lens_host) return fail(h, DELTA_ERR_USAGE, "bad batch/lens");
    if (layer < -1 || layer >= h->cfg.num_layers) return fail(h, DELTA_ERR_USAGE, "layer out of range");
    for (int b = 0; b < batch; ++b)
        if (lens_host[b] < 0 || lens_host[b] > h->cfg.max_seq_len)
            return fail(h, DELTA_ERR_CAPACITY, "length exceeds max_seq_len");
    int32_t* sl = h->at<int32_t>(h->L.seq_len);
    std::vector<int32_t> raw(lens_host, lens_host + batch);  // device counters hold n * g (combine.cuh)
    for (auto& x : raw) x *= h->cfg.num_kv_heads;
    const int l0 = layer < 0 ? 0 : layer, l1 = layer < 0 ? h->cfg.num_layers : layer + 1;
    for (int l = l0; l < l1; ++l) {
        cudaError_t e = cudaMemcpyAsync(sl + (size_t)l * h->cfg.max_batch, raw.data(), sizeof(int32_t) * batch,
                                        cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) return cuda_fail(h, e, "set_seq_lens");
    }
    cudaError_t e = cudaStreamSynchronize(stream);  // lens_host may be freed by the caller after return
    if (e != cudaSuccess) return cuda_fail(h, e, "set_seq_lens");
    std::fill(h->step.begin(), h->step.end(), 0);
    std::fill(h->dec_step.begin(), h->dec_step.end(), -1);
    std::fill(h->sel_step.begin(), h->sel_step.end(), -1);
    return DELTA_OK;
}

delta_status delta_append_kv(delta_t h, int32_t layer, int32_t batch, int32_t ntok, const void* k_new,
                             const void* v_new, cudaStream_t stream) {
    delta_status s = check_layer_batch(h, layer, batch);
    if (s != DELTA_OK) return s;
    s = join_host(h, stream);
    if (s != DELTA_OK) return s;
    if (ntok < 1 || !k_new || !v_new) return fail(h, DELTA_ERR_USAGE, "bad ntok or null k_new/v_new");
    s = launch_append_impl(h, layer, batch, ntok, k_new, v_new, stream);
    if (s == DELTA_OK) h->step[layer] += 1;
    return s;
}

delta_status delta_decode_layer(delta_t h, int32_t layer, int32_t batch, const void* q, float* out,
                                float* lse_out, cudaStream_t stream) {
    delta_status s = check_layer_batch(h, layer, batch);
    if (s != DELTA_OK) return s;
    s = join_host(h, stream);
    if (s != DELTA_OK) return s;
    if (!q || !out) return fail(h, DELTA_ERR_USAGE, "null q/out");
    s = check_sparse_fresh(h, layer, false);
    if (s != DELTA_OK) return s;
    s = launch_decode(h, layer, batch, nullptr, nullptr, q, out, lse_out, stream);
    if (s == DELTA_OK) h->dec_step[layer] = h->step[layer];
    return s;
}

delta_status delta_append_decode_layer(delta_t h, int32_t layer, int32_t batch, const void* k_new,
                                       const void* v_new, const void* q, float* out, float* lse_out,
                                       cudaStream_t stream) {
    delta_status s = check_layer_batch(h, layer, batch);
    if (s != DELTA_OK) return s;
    s = join_host(h, stream);
    if (s != DELTA_OK) return s;
    if (!q || !out || !k_new || !v_new) return fail(h, DELTA_ERR_USAGE, "null pointer");
    s = check_sparse_fresh(h, layer, true);
    if (s != DELTA_OK) return s;
    s = launch_decode(h, layer, batch, k_new, v_new, q, out, lse_out, stream);
    if (s == DELTA_OK) {
        h->step[layer] += 1;
        h->dec_step[layer] = h->step[layer];
    }
    return s;
}

delta_status delta_select(delta_t h, int32_t layer, int32_t batch, const float* keys_override, int32_t* idx_out,
                          int32_t* count_out, cudaStream_t stream) {
    delta_status s = check_layer_batch(h, layer, batch);
    if (s != DELTA_OK) return s;
    s = join_host(h, stream);
    if (s != DELTA_OK) return s;
    if (h->role[layer] != kRoleSelect) return fail(h, DELTA_ERR_USAGE, "delta_select on a non-Delta layer");
    if (!keys_override && h->dec_step[layer] != h->step[layer])
        return fail(h, DELTA_ERR_USAGE, "delta_select needs this layer's decode at the current step");
    if (h->world > 1)  // sharded: local candidates + exchange + global merge (a key override is global)
        s = keys_override ? launch_sel(h, layer, batch, keys_override, idx_out, count_out, stream, 2)
                          : launch_sel_sharded(h, layer, batch, idx_out, count_out, stream);
    else
        s = launch_sel(h, layer, batch, keys_override, idx_out, count_out, stream, 0);
    if (s == DELTA_OK) h->sel_step[h->slot[layer]] = h->step[layer];
    return s;
}

delta_status delta_decode_step(delta_t h, int32_t batch, const void* q_all, const void* k_all, const void* v_all,
                               float* out_all, float* lse_all, cudaStream_t stream) {
    if (!h) return fail(nullptr, DELTA_ERR_USAGE, "null handle");
    if (h->world > 1 && !h->comm)
        return fail(h, DELTA_ERR_USAGE, "sharded handle without NCCL: drive layers with the delta_shard_* calls");
    if (batch < 1 || batch > h->cfg.max_batch) return fail(h, DELTA_ERR_USAGE, "batch out of range");
    if (!q_all || !k_all || !v_all || !out_all) return fail(h, DELTA_ERR_USAGE, "null pointer");
    { delta_status j = join_host(h, stream); if (j != DELTA_OK) return j; }
    const bool legacy = (stream == 0 || stream == cudaStreamLegacy || stream == cudaStreamPerThread);
    if (legacy) {  // default streams cannot be captured: run eagerly
        delta_status s = enqueue_step(h, batch, q_all, k_all, v_all, out_all, lse_all, stream);
        if (s == DELTA_OK) mark_step_done(h);
        return s;
    }
    const void* key[7] = {q_all, k_all, v_all, out_all, lse_all, (const void*)stream, nullptr};
    delta_ctx::GraphEntry* ge = nullptr;
    for (auto& g : h->graphs)
        if (g.exec && g.batch == batch && std::memcmp(key, g.key, sizeof key) == 0) ge = &g;
    if (!ge) {
        ge = &h->graphs[h->graph_next];
        h->graph_next = (h->graph_next + 1) % 3;
        if (ge->exec) { cudaGraphExecDestroy(ge->exec); ge->exec = nullptr; }
        for (int attempt = 0; attempt < 2 && !ge->exec; ++attempt) {
            const uint64_t before = h->launches;
            cudaError_t e = cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal);
            if (e != cudaSuccess) return cuda_fail(h, e, "graph capture begin");
            delta_status s = enqueue_step(h, batch, q_all, k_all, v_all, out_all, lse_all, stream);
            cudaGraph_t graph = nullptr;
            e = cudaStreamEndCapture(stream, &graph);
            if (s != DELTA_OK) { if (graph) cudaGraphDestroy(graph); return s; }
            if (e != cudaSuccess) return cuda_fail(h, e, "graph capture end");
            ge->kernels = h->launches - before;
            ++h->captures;
            h->launches = before;
            e = cudaGraphInstantiate(&ge->exec, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) {
                cudaGetLastError();
                ge->exec = nullptr;
                if (!h->pdl) return cuda_fail(h, e, "graph instantiate");
                h->pdl = false;  // retry without programmatic edges
            }
        }
        std::memcpy(ge->key, key, sizeof key);
        ge->batch = batch;
    }
    cudaError_t e = cudaGraphLaunch(ge->exec, stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "graph launch");
    h->launches += ge->kernels;
    mark_step_done(h);
    return DELTA_OK;
}

// Host-buffer step, pipelined over two staging slots and three internal streams: step i's
// H2D (copy-in stream) overlaps step i-1's graph (compute stream), and its D2H (copy-out
// stream) overlaps step i+1's graph.  Each step still moves its own inputs and outputs.  The
// caller's stream waits for this step's D2H, so synchronising it makes out_all_host valid.
delta_status delta_decode_step_host(delta_t h, int32_t batch, const void* q_all_host, const void* k_all_host,
                                    const void* v_all_host, float* out_all_host, cudaStream_t stream) {
    if (!h) return fail(nullptr, DELTA_ERR_USAGE, "null handle");
    if (batch < 1 || batch > h->cfg.max_batch) return fail(h, DELTA_ERR_USAGE, "batch out of range");
    const delta_config& c = h->cfg;
    cudaError_t err = cudaSuccess;
    if (!h->host_init) {
        err = cudaStreamCreateWithFlags(&h->hs_in, cudaStreamNonBlocking);
        if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&h->hs_comp, cudaStreamNonBlocking);
        if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&h->hs_out, cudaStreamNonBlocking);
        for (int i = 0; i < 2 && err == cudaSuccess; ++i) {
            err = cudaEventCreateWithFlags(&h->hev_in[i], cudaEventDisableTiming);
            if (err == cudaSuccess) err = cudaEventCreateWithFlags(&h->hev_done[i], cudaEventDisableTiming);
            if (err == cudaSuccess) err = cudaEventCreateWithFlags(&h->hev_out[i], cudaEventDisableTiming);
        }
        if (err == cudaSuccess) err = cudaEventCreateWithFlags(&h->hev_join, cudaEventDisableTiming);
        if (err != cudaSuccess) return cuda_fail(h, err, "step_host streams");
        h->host_init = true;
    }
    const size_t e = elem_bytes(c);
    const size_t qb = (size_t)c.num_layers * batch * c.num_q_heads * c.head_dim * e;
    const size_t kb = (size_t)c.num_layers * batch * c.num_kv_heads * c.head_dim * e;
    const size_t ob = (size_t)c.num_layers * batch * c.num_q_heads * c.head_dim * 4;
    const size_t qs = (size_t)c.num_layers * c.max_batch * c.num_q_heads * c.head_dim * e;  // slot strides
    const size_t ks = (size_t)c.num_layers * c.max_batch * c.num_kv_heads * c.head_dim * e;
    const size_t os = (size_t)c.num_layers * c.max_batch * c.num_q_heads * c.head_dim;
    const int slot = h->host_slot;
    h->host_slot ^= 1;
    uint8_t* dq = h->at<uint8_t>(h->L.stage_q) + slot * qs;
    uint8_t* dk = h->at<uint8_t>(h->L.stage_k) + slot * ks;
    uint8_t* dv = h->at<uint8_t>(h->L.stage_v) + slot * ks;
    float* dout = h->at<float>(h->L.stage_out) + slot * os;
    if (!h->host_pending) {  // first of a run of host steps: after the caller's prior work
        err = cudaEventRecord(h->hev_out[slot ^ 1], stream);
        if (err == cudaSuccess) err = cudaStreamWaitEvent(h->hs_in, h->hev_out[slot ^ 1], 0);
        if (err == cudaSuccess) err = cudaStreamWaitEvent(h->hs_comp, h->hev_out[slot ^ 1], 0);
        if (err != cudaSuccess) return cuda_fail(h, err, "step_host join");
    }
    // copy-in: the slot is free once step i-2's graph and D2H are done with it
    err = cudaStreamWaitEvent(h->hs_in, h->hev_done[slot], 0);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(h->hs_in, h->hev_out[slot], 0);
    if (err == cudaSuccess) err = cudaMemcpyAsync(dq, q_all_host, qb, cudaMemcpyHostToDevice, h->hs_in);
    if (err == cudaSuccess) err = cudaMemcpyAsync(dk, k_all_host, kb, cudaMemcpyHostToDevice, h->hs_in);
    if (err == cudaSuccess) err = cudaMemcpyAsync(dv, v_all_host, kb, cudaMemcpyHostToDevice, h->hs_in);
    if (err == cudaSuccess) err = cudaEventRecord(h->hev_in[slot], h->hs_in);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(h->hs_comp, h->hev_in[slot], 0);
    if (err != cudaSuccess) return cuda_fail(h, err, "step_host H2D");
    h->host_pending = false;  // the compute stream is ordered after everything above
    delta_status s = delta_decode_step(h, batch, dq, dk, dv, dout, nullptr, h->hs_comp);
    if (s != DELTA_OK) return s;
    h->host_pending = true;
    err = cudaEventRecord(h->hev_done[slot], h->hs_comp);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(h->hs_out, h->hev_done[slot], 0);
    if (err == cudaSuccess) err = cudaMemcpyAsync(out_all_host, dout, ob, cudaMemcpyDeviceToHost, h->hs_out);
    if (err == cudaSuccess) err = cudaEventRecord(h->hev_out[slot], h->hs_out);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(stream, h->hev_out[slot], 0);
    if (err != cudaSuccess) return cuda_fail(h, err, "step_host D2H");
    return DELTA_OK;
}

delta_status delta_quest_build_reps(delta_t h, int32_t layer, int32_t batch, cudaStream_t stream) {
    if (!h) return fail(nullptr, DELTA_ERR_USAGE, "null handle");
    if (h->cfg.policy != DELTA_POLICY_QUEST) return fail(h, DELTA_ERR_USAGE, "not a QUEST handle");
    { delta_status j = join_host(h, stream); if (j != DELTA_OK) return j; }
    if (batch < 1 || batch > h->cfg.max_batch) return fail(h, DELTA_ERR_USAGE, "batch out of range");
    if (layer < -1 || layer >= h->cfg.num_layers) return fail(h, DELTA_ERR_USAGE, "layer out of range");
    const int l0 = layer < 0 ? 0 : layer, l1 = layer < 0 ? h->cfg.num_layers : layer + 1;
    for (int l = l0; l < l1; ++l) {
        if (h->role[l] != kRoleQuest) continue;
        cudaError_t e = launch_quest_reps(quest_params(h, l, batch, nullptr), h->L.max_pages, stream, h->pdl);
        if (e != cudaSuccess) return cuda_fail(h, e, "quest reps launch");
        ++h->launches;
        h->last_kind = delta_ctx::kLastAppend;
        h->last_layer = l;
    }
    return DELTA_OK;
}

delta_status delta_copy_plan(delta_t h, int32_t layer, int32_t batch, int32_t* idx_out, int32_t* count_out,
                             cudaStream_t stream) {
    delta_status s = check_layer_batch(h, layer, batch);
    if (s != DELTA_OK) return s;
    s = join_host(h, stream);
    if (s != DELTA_OK) return s;
    if (h->role[layer] == kRoleFull) return fail(h, DELTA_ERR_USAGE, "a FULL layer has no plan");
    const int sl = h->slot[h->gov[layer]];
    const size_t cap = h->L.plan_cap, mb = h->cfg.max_batch;
    cudaError_t e = cudaSuccess;
    if (idx_out)
        e = cudaMemcpyAsync(idx_out, h->at<int32_t>(h->L.plan_idx) + sl * mb * cap, batch * cap * 4,
                            cudaMemcpyDeviceToDevice, stream);
    if (e == cudaSuccess && count_out)
        e = cudaMemcpyAsync(count_out, h->at<int32_t>(h->L.plan_count) + sl * mb, batch * 4, cudaMemcpyDeviceToDevice,
                            stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "copy_plan");
    h->last_kind = delta_ctx::kLastNone;  // a copy node sits between kernels
    return DELTA_OK;
}

delta_status delta_attention_recall(delta_t h, int32_t layer, int32_t batch, const void* q, float* recall_out,
                                   cudaStream_t stream) {
    delta_status s = check_layer_batch(h, layer, batch);
    if (s != DELTA_OK) return s;
    s = join_host(h, stream);
    if (s != DELTA_OK) return s;
    if (!q || !recall_out) return fail(h, DELTA_ERR_USAGE, "null q/recall_out");
    if (h->role[layer] == kRoleFull) return fail(h, DELTA_ERR_USAGE, "a FULL layer attends everything (R = 1)");
    if (h->world > 1) return fail(h, DELTA_ERR_USAGE, "attention recall is not sequence-sharded");
    const delta_config& c = h->cfg;
    // 1. full-attention probe of the layer (SELECT role: logits + LSE into the Delta buffers)
    AttnParams p = attn_params(h, layer, batch, kRoleSelect);
    p.q = q;
    p.out = h->at<float>(h->L.stage_out) + (size_t)layer * c.max_batch * c.num_q_heads * c.head_dim;
    p.lse_out = nullptr;
    p.fuse_append = 0;
    p.prewait = 0;
    p.early_trigger = h->tune_early;
    cudaError_t e = !h->use_tc ? launch_attn_simt(p, c.kv_dtype == DELTA_BF16, stream, h->pdl)
                               : launch_attn_tc(p, &h->tm_kv, stream, h->pdl);
    if (e != cudaSuccess) return cuda_fail(h, e, "recall probe launch");
    ++h->launches;
    // 2. Eq.9 over the layer's plan
    RecallParams rp = {};
    const int sl = h->slot[h->gov[layer]];
    rp.m = c.num_q_heads; rp.g = c.num_kv_heads; rp.layer = layer; rp.batch = batch; rp.max_batch = c.max_batch;
    rp.max_seq = c.max_seq_len; rp.plan_cap = h->L.plan_cap; rp.sel_block = c.select_block;
    rp.seq_len = h->at<int32_t>(h->L.seq_len);
    rp.logits = h->at<float>(h->L.logits); rp.lse = h->at<float>(h->L.lse_buf);
    rp.plan_idx = h->at<int32_t>(h->L.plan_idx) + (size_t)sl * c.max_batch * h->L.plan_cap;
    rp.plan_count = h->at<int32_t>(h->L.plan_count) + (size_t)sl * c.max_batch;
    rp.recall_out = recall_out;
    if (c.num_q_heads > 256) return fail(h, DELTA_ERR_USAGE, "recall supports m <= 256");
    e = launch_recall(rp, stream, h->pdl);
    if (e != cudaSuccess) return cuda_fail(h, e, "recall launch");
    ++h->launches;
    h->last_kind = delta_ctx::kLastAttn;
    h->last_layer = layer;
    return DELTA_OK;
}

delta_status delta_prefill(delta_t h, int32_t layer, int32_t batch, int32_t ntok, const void* q, const void* k_new,
                           const void* v_new, float* out, float* lse_out, cudaStream_t stream) {
    delta_status s = check_layer_batch(h, layer, batch);
    if (s != DELTA_OK) return s;
    s = join_host(h, stream);
    if (s != DELTA_OK) return s;
    if (ntok < 1 || !q || !k_new || !v_new || !out) return fail(h, DELTA_ERR_USAGE, "bad ntok or null pointer");
    if (!h->use_tc) return fail(h, DELTA_ERR_USAGE, "prefill needs bf16 KV");
    if (h->world > 1) return fail(h, DELTA_ERR_USAGE, "prefill is not sequence-sharded");
    const delta_config& c = h->cfg;
    s = launch_append_impl(h, layer, batch, ntok, k_new, v_new, stream);  // Eq.7 for the chunk (+ Quest reps)
    if (s != DELTA_OK) return s;
    PrefillParams p = {};
    p.m = c.num_q_heads; p.g = c.num_kv_heads; p.gs = h->gs; p.d = c.head_dim; p.layer = layer; p.batch = batch;
    p.ntok = ntok; p.num_phys = c.num_phys_pages; p.bt_stride = h->L.max_pages; p.max_batch = c.max_batch;
    p.scale_log2 = (float)((double)h->scale * 1.4426950408889634);
    p.q = q; p.kv_pool = h->kv_pool; p.block_table = h->block_table; p.seq_len = h->at<int32_t>(h->L.seq_len);
    p.out = out; p.lse_out = lse_out; p.err = h->at<int32_t>(h->L.err);
    // tcgen05 / TMEM kernel (prefill_umma.cu); the mma.sync kernel stays selectable (pfumma=0)
    cudaError_t e = (h->tune_pfumma == 3 && prefill_umma_supported(p)) ? launch_prefill_umma3(p, &h->tm_kvp, stream, h->pdl)
                    : (h->tune_pfumma == 2 && prefill_umma_supported(p)) ? launch_prefill_umma2(p, &h->tm_kvp, stream, h->pdl)
                    : (h->tune_pfumma && prefill_umma_supported(p)) ? launch_prefill_umma(p, &h->tm_kvp, stream, h->pdl)
                                                                      : launch_prefill(p, stream, h->pdl);
    if (e != cudaSuccess) return cuda_fail(h, e, "prefill launch");
    ++h->launches;
    h->last_kind = delta_ctx::kLastAttn;
    h->last_layer = layer;
    h->step[layer] += 1;
    return DELTA_OK;
}

delta_status delta_raas_reset(delta_t h, int32_t layer, int32_t batch, cudaStream_t stream) {
    if (!h) return fail(nullptr, DELTA_ERR_USAGE, "null handle");
    if (h->cfg.policy != DELTA_POLICY_RAAS) return fail(h, DELTA_ERR_USAGE, "not a RAAS handle");
    if (batch < 1 || batch > h->cfg.max_batch) return fail(h, DELTA_ERR_USAGE, "batch out of range");
    if (layer < -1 || layer >= h->cfg.num_layers) return fail(h, DELTA_ERR_USAGE, "layer out of range");
    { delta_status j = join_host(h, stream); if (j != DELTA_OK) return j; }
    const int l0 = layer < 0 ? 0 : layer, l1 = layer < 0 ? h->cfg.num_layers : layer + 1;
    for (int l = l0; l < l1; ++l) {
        if (h->role[l] != kRoleRaas) continue;
        cudaError_t e = launch_raas_reset(raas_params(h, l, batch), stream, h->pdl);
        if (e != cudaSuccess) return cuda_fail(h, e, "raas reset launch");
        ++h->launches;
        h->last_kind = delta_ctx::kLastAppend;
        h->last_layer = l;
    }
    return DELTA_OK;
}

delta_status delta_workspace_region(delta_t h, int32_t which, void** ptr, size_t* bytes) {
    if (!h || !ptr || !bytes) return fail(h, DELTA_ERR_USAGE, "null argument");
    if (which == 0) {
        *ptr = h->ws + h->L.keys;
        *bytes = (size_t)h->cfg.max_batch * h->L.max_units * 4;
    } else if (which == 1) {
        *ptr = h->ws + h->L.reps;
        *bytes = h->L.reps_bytes;
    } else if (which == 2) {
        *ptr = h->ws + h->L.raas_last;
        *bytes = h->cfg.policy == DELTA_POLICY_RAAS ? (size_t)h->cfg.num_layers * h->cfg.max_batch * h->L.max_pages * 4 : 0;
    } else {
        return fail(h, DELTA_ERR_USAGE, "unknown workspace region");
    }
    return DELTA_OK;
}

delta_status delta_get_error(delta_t h, cudaStream_t stream, delta_status* sticky) {
    { delta_status j = join_host(h, stream); if (j != DELTA_OK) return j; }
    if (!h || !sticky) return fail(h, DELTA_ERR_USAGE, "null argument");
    cudaError_t e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "get_error sync");
    int32_t v = 0;
    int32_t* dev = h->at<int32_t>(h->L.err);
    e = cudaMemcpy(&v, dev, sizeof v, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemset(dev, 0, sizeof v);
    if (e != cudaSuccess) return cuda_fail(h, e, "get_error read");
    *sticky = (delta_status)v;
    // sequence sharding with the library's communicator: surface asynchronous NCCL failures
    // (a peer that died, a network error) — they would otherwise only show as a hang
    if (h->comm && nccl().commGetAsyncError) {
        ncclResult_t ar = ncclSuccess;
        const ncclResult_t r = nccl().commGetAsyncError(h->comm, &ar);
        if (r != ncclSuccess) return fail(h, DELTA_ERR_NCCL, std::string("ncclCommGetAsyncError: ") + nccl().getErrorString(r));
        if (ar != ncclSuccess && ar != ncclInProgress) {
            *sticky = DELTA_ERR_NCCL;
            return fail(h, DELTA_ERR_NCCL, std::string("NCCL async error: ") + nccl().getErrorString(ar));
        }
    }
    return DELTA_OK;
}

delta_status delta_set_nccl_library(const char* path) {
    if (!path) return fail(nullptr, DELTA_ERR_USAGE, "null path");
    g_nccl_path = path;
    return DELTA_OK;
}

delta_role delta_layer_role(delta_t h, int32_t layer) {
    if (!h || layer < 0 || layer >= h->cfg.num_layers) return (delta_role)-1;
    return (delta_role)h->role[layer];
}

int32_t delta_governing_layer(delta_t h, int32_t layer) {
    if (!h || layer < 0 || layer >= h->cfg.num_layers) return -1;
    return h->gov[layer];
}

int32_t delta_plan_capacity(delta_t h) { return h ? h->L.plan_cap : -1; }

const char* delta_last_error_message(delta_t h) { return h ? h->msg.c_str() : g_msg.c_str(); }

uint64_t delta_kernels_launched(delta_t h) { return h ? h->launches : 0; }

uint64_t delta_graph_captures(delta_t h) { return h ? h->captures : 0; }

const char* delta_layer_kernel_name(delta_t h, int32_t layer, int32_t batch) {
    if (!h || layer < 0 || layer >= h->cfg.num_layers || batch < 1 || batch > h->cfg.max_batch) return "";
    const AttnParams p = attn_params(h, layer, batch);
    if (!h->use_tc) return "attn_simt_kernel (fp32, cluster split-K merge)";
    if (h->tune_umma && umma_supported(p)) return "attn_umma_kernel (tcgen05, cluster split-K merge)";
    if (p.sparse_lat) return "sparse_lat_kernel (resident plan tiles, cluster DSMEM split-K merge)";
    if (p.gmerge) return p.gll ? "attn_tc_kernel (one CTA per SM, global split-K merge over LL words)"
                               : "attn_tc_kernel (one CTA per SM, global split-K merge)";
    return "attn_tc_kernel (cluster DSMEM split-K merge)";
}

delta_status delta_set_tuning(delta_t h, const char* key, int32_t value) {
    if (!h || !key) return fail(h, DELTA_ERR_USAGE, "null handle or key");
    struct Knob { const char* name; int* field; };
    const Knob knobs[] = {
        {"nsplit", &h->tune_nsplit}, {"snsplit", &h->tune_snsplit}, {"deep", &h->tune_deep},
        {"prewait", &h->tune_prewait}, {"early", &h->tune_early}, {"umma", &h->tune_umma},
        {"policy", &h->tune_policy}, {"seltrig", &h->tune_seltrig}, {"selhist", &h->tune_selhist},
        {"gmerge", &h->tune_gmerge}, {"gm2", &h->tune_gm2}, {"lat", &h->tune_lat}, {"qpf", &h->tune_qpf}, {"pfumma", &h->tune_pfumma}, {"gll", &h->tune_gll}, {"selll", &h->tune_selll}, {"gfix", &h->tune_gfix}};
    for (const Knob& k : knobs)
        if (std::strcmp(k.name, key) == 0) {
            *k.field = value;
            for (auto& g : h->graphs)  // captured steps baked the old setting in
                if (g.exec) { cudaGraphExecDestroy(g.exec); g.exec = nullptr; }
            return DELTA_OK;
        }
    return fail(h, DELTA_ERR_CONFIG, std::string("unknown tuning key: ") + key);
}

delta_status delta_read_bandwidth_probe(const void* buf, size_t bytes, float* sink, cudaStream_t stream) {
    if (!buf || !sink) return fail(nullptr, DELTA_ERR_USAGE, "null buffer");
    cudaError_t e = launch_read_probe(buf, bytes, sink, num_sms_current(), stream);
    if (e != cudaSuccess) return fail(nullptr, DELTA_ERR_CUDA, std::string("read probe: ") + cudaGetErrorString(e));
    return DELTA_OK;
}

delta_status delta_nccl_get_unique_id(void* out_128_bytes) {
    if (!out_128_bytes) return fail(nullptr, DELTA_ERR_USAGE, "null argument");
    const NcclApi& api = nccl();
    if (!api.ok) return fail(nullptr, DELTA_ERR_NCCL, api.why);
    ncclUniqueId id;
    ncclResult_t r = api.getUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, DELTA_ERR_NCCL, std::string("ncclGetUniqueId: ") + api.getErrorString(r));
    std::memcpy(out_128_bytes, &id, sizeof id);
    return DELTA_OK;
}

delta_status delta_shard_range(const delta_config* cfg, int32_t* page_lo, int32_t* page_hi) {
    if (!cfg || !page_lo || !page_hi) return fail(nullptr, DELTA_ERR_USAGE, "null argument");
    std::vector<int> role, gov;
    std::string err = validate(*cfg, role, gov);
    if (!err.empty()) return fail(nullptr, DELTA_ERR_CONFIG, err);
    int lo, hi;
    shard_pages(*cfg, cfg->shard_rank, &lo, &hi);
    const int max_pages = (cfg->max_seq_len + kPage - 1) / kPage;
    *page_lo = cfg->shard_world > 1 ? lo : 0;
    *page_hi = cfg->shard_world > 1 ? hi : max_pages;
    return DELTA_OK;
}

delta_status delta_shard_exchange_buffers(delta_t h, int32_t which, void** send, void** recv, size_t* block_bytes) {
    if (!h || !send || !recv || !block_bytes) return fail(h, DELTA_ERR_USAGE, "null argument");
    if (h->world < 2) return fail(h, DELTA_ERR_USAGE, "not a sharded handle");
    if (which != 0 && which != 1) return fail(h, DELTA_ERR_USAGE, "which must be 0 (attention) or 1 (candidates)");
    *send = h->ws + (which == 0 ? h->L.shard_send : h->L.cand_send);
    *recv = h->ws + (which == 0 ? h->L.shard_recv : h->L.cand_recv);
    *block_bytes = which == 0 ? h->L.shard_block : h->L.cand_block;
    return DELTA_OK;
}

delta_status delta_shard_merge(delta_t h, int32_t layer, int32_t batch, float* out, float* lse_out,
                               cudaStream_t stream) {
    delta_status s = check_layer_batch(h, layer, batch);
    if (s != DELTA_OK) return s;
    s = join_host(h, stream);
    if (s != DELTA_OK) return s;
    if (h->world < 2 || h->comm) return fail(h, DELTA_ERR_USAGE, "delta_shard_merge needs a sharded handle without NCCL");
    if (!out) return fail(h, DELTA_ERR_USAGE, "null out");
    return launch_merge(h, layer, batch, out, lse_out, stream);
}

delta_status delta_shard_select_merge(delta_t h, int32_t layer, int32_t batch, int32_t* idx_out,
                                      int32_t* count_out, cudaStream_t stream) {
    delta_status s = check_layer_batch(h, layer, batch);
    if (s != DELTA_OK) return s;
    s = join_host(h, stream);
    if (s != DELTA_OK) return s;
    if (h->world < 2 || h->comm) return fail(h, DELTA_ERR_USAGE, "delta_shard_select_merge needs a sharded handle without NCCL");
    if (h->role[layer] != kRoleSelect) return fail(h, DELTA_ERR_USAGE, "not a Delta layer");
    return launch_sel_merge(h, layer, batch, idx_out, count_out, stream);
}

}  // extern "C"
