/*
 * delta.h — C ABI of the B200-native DELTA decode-step attention stack
 * (DELTA: Dynamic Layer-Aware Token Attention, arXiv 2510.09883).
 *
 * The library implements ONE step of decoding through the three-tier attention
 * stack of PAPER.md §4 (lines 157-185): FULL layers attend to the whole paged KV
 * cache; Delta (SELECT) layers attend to the whole cache, score every token by its
 * maximum normalised attention weight over all query heads and pick the top-k
 * salient units plus the sink and recency window; SPARSE layers attend only to the
 * units chosen by the nearest Delta layer below them, at this step.
 *
 * Citations: "PAPER.md:L" = line L of the paper's LaTeX (§, Eq.); "R#" = the reading
 * of an ambiguous passage listed in DESIGN.md §3.  Index base is 0 (R25).
 *
 * Conventions (all entry points):
 *  - Every device pointer is CALLER-OWNED (e.g. torch tensors).  The library never
 *    allocates device memory after delta_create and never frees caller memory.
 *  - Hot-path calls (append / decode / select / step) are asynchronous on the given
 *    stream and never synchronise the host; their return value is host-side argument
 *    and call-order validation only.  Device-side faults (NaN/Inf in an output,
 *    a stale plan under graph replay) set a STICKY device flag read by delta_get_error.
 *  - One writer per handle (calls on one handle must be ordered by the caller).
 *  - All calls may be captured into a CUDA graph (no host syncs, device-resident
 *    sequence lengths, fixed grids).
 *  - Sizes: m = num_q_heads, g = num_kv_heads, gs = m/g, d = head_dim, P = page_size.
 */
#ifndef DELTA_H
#define DELTA_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct delta_ctx* delta_t;

typedef enum {
    DELTA_OK = 0,
    DELTA_ERR_CONFIG = 1,   /* invalid shapes / schedule / budget (SPEC "configuration error") */
    DELTA_ERR_USAGE = 2,    /* bad layer or batch, call-order violation, stale plan */
    DELTA_ERR_NUMERIC = 3,  /* NaN/Inf produced on device (sticky, via delta_get_error) */
    DELTA_ERR_CAPACITY = 4, /* append past max_seq_len / pool too small */
    DELTA_ERR_CUDA = 5,     /* a CUDA runtime call failed (message in delta_last_error_message) */
    DELTA_ERR_NCCL = 6      /* collective failure (sequence-sharded mode) */
} delta_status;

typedef enum { DELTA_BF16 = 0, DELTA_FP32 = 1 } delta_dtype;

typedef enum { DELTA_ROLE_FULL = 0, DELTA_ROLE_SELECT = 1, DELTA_ROLE_SPARSE = 2, DELTA_ROLE_QUEST = 3,
               DELTA_ROLE_RAAS = 4 } delta_role;

/* Selection policy of the layers >= F.
 *  DELTA: the paper's three-tier schedule (Delta layers select, sparse layers reuse).
 *  QUEST: the paper's comparison system Quest: every layer >= F
 *         (role QUEST) keeps the element-wise min/max of the keys of each (page, kv head) and, at
 *         every decode, scores each page by max_j sum_e max(q_j[e] min[e], q_j[e] max[e]) (Q1, Q2:
 *         an upper bound of q_j . k over the page), selects the forced sink/window pages plus the
 *         top budget_k/P candidate pages with the same rule as DELTA (Q3) and attends to them.
 *         Needs num_select_layers == 0, select_block == page_size, kv_dtype BF16, shard_world 1. */
/*  RAAS:  the paper's eviction baseline RaaS (readings RS1-RS4):
 *         every layer >= F (role RAAS) attends its own retained page set, then scores the
 *         retained pages with its attention weights (S_u = sum_{t in u} max_j alpha_j(t)),
 *         refreshes pages with S_u >= P / |attended tokens|, and permanently evicts the least
 *         recently salient non-exempt pages beyond budget_k/P (sink and recency pages exempt).
 *         Same restrictions as QUEST.  delta_raas_reset starts every sequence with all pages
 *         retained. */
typedef enum { DELTA_POLICY_DELTA = 0, DELTA_POLICY_QUEST = 1, DELTA_POLICY_RAAS = 2 } delta_policy;

/* Problem statement of the method (PAPER.md:157-158 schedule, 168-171/185 budget and
 * window, 180-181/196 paged layout). */
typedef struct {
    int32_t num_layers;        /* L */
    int32_t num_q_heads;       /* m */
    int32_t num_kv_heads;      /* g, g | m; head j reads group phi(j) = j / (m/g) (R15) */
    int32_t head_dim;          /* d in {64, 128} */
    int32_t max_batch;         /* sequences per call, >= 1 */
    int32_t max_seq_len;       /* cache capacity per sequence, tokens */
    int32_t page_size;         /* P; PAPER.md:196 uses 16.  Must be 16. */
    int32_t num_phys_pages;    /* pages per layer in each pool; 0 -> max_batch*ceil(max_seq_len/P) */
    int32_t num_full_prefix;   /* F: layers [0, F) are FULL */
    int32_t num_select_layers; /* |Delta| */
    const int32_t* select_layers; /* host array, strictly ascending, each >= F; every layer >= F
                                     must have a Delta layer <= it */
    int32_t budget_k;          /* k: salient TOKENS selected beyond sink and window (R1) */
    int32_t n_sink;            /* S: first S tokens always kept (R2) */
    int32_t n_window;          /* L: last L tokens (incl. this step's) always kept (R3) */
    int32_t select_block;      /* 1 = token-level selection,
                                  P = page-level; page mode needs P | k (R6) */
    delta_dtype kv_dtype;      /* dtype of K/V pools, q, k_new, v_new.  Outputs are fp32. */
    float softmax_scale;       /* 0 -> (float)(1/sqrt(d))  (Eq.4, R16) */
    int32_t shard_world;       /* W: sequence sharding across W GPUs (1 = off).  Rank r holds the
                                  contiguous page range delta_shard_range() returns of EVERY
                                  sequence (its kv_pool / block table need only those pages);
                                  every layer all-gathers the per-rank (o, lse) partials and
                                  LSE-merges them, every Delta layer also all-gathers its top-k
                                  candidates.  All ranks make the same calls. */
    int32_t shard_rank;        /* r in [0, W) */
    const void* nccl_id;       /* W > 1: 128-byte ncclUniqueId (delta_nccl_get_unique_id on rank 0,
                                  broadcast by the caller) -> the library owns an NCCL communicator
                                  and runs both exchanges itself, on the call's stream (graph-
                                  capturable).  NULL -> "external exchange": decode/select stop
                                  after the local pass and the caller moves the bytes itself
                                  (delta_shard_exchange_buffers) and calls delta_shard_merge /
                                  delta_shard_select_merge (used for single-GPU simulation). */
    int32_t policy;            /* delta_policy (0 = DELTA) */
    int32_t det_chunks;        /* C: 0 = off.  R21 run-to-run AND cross-W determinism: the pages
                                  [0, ceil(max_seq_len/P)) are cut into C fixed chunks of
                                  ceil(pages/C) pages; every layer attends each chunk separately
                                  (same kernel and split count whatever W is) and LSE-merges the
                                  C chunk partials in chunk order, Delta plans are ranged per
                                  chunk — so outputs, LSEs and plans are bitwise identical for
                                  every W dividing C (rank r holds chunks [r C/W, (r+1) C/W)).
                                  Costs C/W attention launches + 1 merge per layer.  DELTA
                                  policy only; C % W == 0, C <= 64. */
} delta_config;

/* Caller-owned device buffers.  Sizes from delta_query_sizes. */
typedef struct {
    void* kv_pool;             /* [L][num_phys_pages][g][2][P][d] kv_dtype, 1024-byte aligned:
                                  for every (layer, page, kv head) the P key rows then the P
                                  value rows, 2*P*d contiguous elements, so one request moves
                                  a head's K and V of a page (PAPER.md:180-181 paging, P = 16) */
    const int32_t* block_table;/* [max_batch][ceil(max_seq_len/P)] int32 physical page ids,
                                  shared by all layers: token t of sequence b lives in page
                                  block_table[b][t/P], slot t%P (PAPER.md:181 p(t)) */
    void* workspace;           /* >= workspace_bytes, 256-byte aligned, zero-initialised
                                  by delta_create */
    size_t workspace_bytes;
} delta_buffers;

/* Byte sizes of kv_pool and of the workspace for this config on the CURRENT device.
 * CONFIG error if the config is invalid. */
delta_status delta_query_sizes(const delta_config* cfg, size_t* kv_pool_bytes,
                               size_t* workspace_bytes);

/* Validate the config (shapes, schedule as in SPEC.md:378-386, budget), compute each
 * layer's role and governing Delta layer, carve the workspace, build TMA descriptors.
 * Sets every cache length to 0.  Synchronous (host + one memset). */
delta_status delta_create(const delta_config* cfg, const delta_buffers* bufs, delta_t* out);

/* Set cache lengths (tokens already stored, e.g. after an external prefill) of
 * sequences [0, batch) for one layer (layer >= 0) or all layers (layer == -1).
 * lens_host: host array [batch].  CAPACITY if a length exceeds max_seq_len.
 * Resets host-side call-order tracking. */
delta_status delta_set_seq_lens(delta_t h, int32_t layer, int32_t batch,
                                const int32_t* lens_host, cudaStream_t stream);

/* Eq.7 KV append for one layer: K <- [K; k_new], V <- [V; v_new].
 * k_new, v_new: device [batch][ntok][g][d] kv_dtype.  Token i of sequence b goes to
 * position n_b + i (n_b = current length); lengths grow by ntok.  Never evicts
 * (PAPER.md:161).  CAPACITY error is detected on device (sticky) if n_b+ntok > max. */
delta_status delta_append_kv(delta_t h, int32_t layer, int32_t batch, int32_t ntok,
                             const void* k_new, const void* v_new, cudaStream_t stream);

/* Decode attention of one layer for sequences [0, batch), dispatched on the layer's role:
 *  FULL   : Eq.4 over all s cached tokens.
 *  SELECT : Eq.4 over all s tokens (R11: the Delta layer's own output is full attention),
 *           and records the logits needed by delta_select.
 *  SPARSE : Eq.4 over tokens(rho) of the governing Delta layer's plan from THIS step,
 *           softmax renormalised over rho (R10, R13).  USAGE error if
 *           that plan is stale (host check) — under graph replay the device check sets
 *           the sticky USAGE flag and writes NaN outputs.
 *  QUEST  : page keys from the layer's min/max representatives and q, top-k pages, Eq.4 over
 *           them (policy QUEST, see below).
 *  RAAS   : Eq.4 over the layer's retained pages, then refresh / eviction for the next step
 *           (policy RAAS, see below).
 * q: device [batch][m][d] kv_dtype.  out: device [batch][m][d] fp32.
 * lse_out: optional device [batch][m] fp32 natural-log LSE of each head's logits over
 * the attended set (NULL to skip). */
delta_status delta_decode_layer(delta_t h, int32_t layer, int32_t batch, const void* q,
                                float* out, float* lse_out, cudaStream_t stream);

/* Fused Eq.7 append of ONE token (k_new, v_new: [batch][g][d]) + delta_decode_layer,
 * in a single launch: the new row is written to the pool and used from the input
 * directly.  Same semantics as delta_append_kv(ntok=1) followed by delta_decode_layer. */
delta_status delta_append_decode_layer(delta_t h, int32_t layer, int32_t batch,
                                       const void* k_new, const void* v_new, const void* q,
                                       float* out, float* lse_out, cudaStream_t stream);

/* Selection at a Delta layer (PAPER.md:163-171 token form, 180-185 page form), after
 * that layer's decode in the same step.  Per sequence:
 *   key_t = max_j (a_j(t) - LSE_j) in fp32 (log of s_t = max_j alpha_j(t), R7/R8);
 *   page mode: S_u = sum_{t in u} exp(key_t) in ascending t (fp32);
 *   rho = forced (sink, window units) U top-(k/block) candidates by (key desc, index asc)
 *   (R1-R6, R9, R12); all units if the candidates fit the budget.
 * The plan (ascending unit ids, count, stamp = s) is kept in the workspace for the
 * sparse layers this Delta layer governs.
 * keys_override: NULL, or device [batch][ceil(s/select_block)] fp32 unit keys to rank
 *   instead of this layer's scores (test hook; ranking and plan are identical code).
 * idx_out / count_out: optional device copies of the plan, [batch][plan_capacity] int32
 *   (entries past count are -1) and [batch] int32. */
delta_status delta_select(delta_t h, int32_t layer, int32_t batch, const float* keys_override,
                          int32_t* idx_out, int32_t* count_out, cudaStream_t stream);

/* One whole decode step of the stack: for every layer l in order, fused append of
 * k_all[l] / v_all[l] and decode with q_all[l], plus selection after each Delta layer.
 * q_all: [L][batch][m][d]; k_all, v_all: [L][batch][g][d] (kv_dtype); out_all:
 * [L][batch][m][d] fp32; lse_all: optional [L][batch][m] fp32.  The launch sequence
 * is captured once into a CUDA graph per (batch, pointers, stream) and replayed. */
delta_status delta_decode_step(delta_t h, int32_t batch, const void* q_all, const void* k_all,
                               const void* v_all, float* out_all, float* lse_all,
                               cudaStream_t stream);

/* delta_decode_step with HOST buffers (pinned recommended): copies the step's inputs
 * host->device into workspace staging, runs the step, copies out_all device->host.
 * Pipelined: two staging slots and three handle-internal streams (copy-in, compute,
 * copy-out), so step i's H2D overlaps step i-1's compute and its D2H overlaps step i+1's;
 * every step still moves its own inputs and outputs.  The first call of a run is ordered
 * after the work already on `stream`; `stream` waits for each call's D2H, so synchronising
 * it makes out_all_host valid, and any other call on the handle is ordered after the run.
 * The host buffers of a call must stay valid until `stream` is synchronised. */
delta_status delta_decode_step_host(delta_t h, int32_t batch, const void* q_all_host,
                                    const void* k_all_host, const void* v_all_host,
                                    float* out_all_host, cudaStream_t stream);

/* ---- Quest policy (policy == DELTA_POLICY_QUEST) ------------------------------------
 * Page representatives are kept in the workspace, [L][num_phys_pages][g][2][d] bf16 (min row,
 * then max row, of the keys of each (physical page, kv head)), updated by every append
 * (delta_append_kv / the append inside delta_append_decode_layer / delta_decode_step).  After
 * filling the pool some other way (external prefill), rebuild them for pages < ceil(n_b/P) of
 * sequences [0, batch) of one layer (layer >= 0) or of every QUEST layer (layer == -1).
 * A QUEST layer's delta_decode_layer / delta_append_decode_layer runs: [append + reps update],
 * page keys, top-k (select.cu), sparse attention over the plan — four launches. */
delta_status delta_quest_build_reps(delta_t h, int32_t layer, int32_t batch, cudaStream_t stream);

/* RaaS policy: (re)start the retained sets of sequences [0, batch) of one RAAS layer (or all,
 * layer == -1) at their current length n: every page < ceil(n/P) retained with last-salient
 * step 0 (plus the page of position n if n is page-aligned).  Call after filling the cache. */
delta_status delta_raas_reset(delta_t h, int32_t layer, int32_t batch, cudaStream_t stream);

/* Test hook: device copy of the plan that `layer` attends (a Delta layer's plan, the plan of
 * the governing Delta layer of a SPARSE layer, or a QUEST layer's own plan from its latest
 * decode): idx_out [batch][plan_capacity] (entries past count unspecified), count_out [batch]. */
delta_status delta_copy_plan(delta_t h, int32_t layer, int32_t batch, int32_t* idx_out, int32_t* count_out,
                             cudaStream_t stream);

/* Attention recall, Eq.9, a diagnostic (NEXT-2) for a SELECT, SPARSE or
 * QUEST layer after its decode at this step: R_j = sum_{t in tokens(rho)} alpha_j(t) /
 * sum_{t < s} alpha_j(t), alpha_j = the layer's exact full-attention weights for its query q
 * ([batch][m][d] kv_dtype, the same q as the decode), rho = the plan the layer attended (its
 * own, the governing Delta layer's, — QUEST — the plan of the latest decoded QUEST layer, so
 * call it right after that layer, or — RAAS — the layer's retained set after this step's
 * eviction).  Runs a full-attention probe of the layer, which
 * overwrites the Delta-layer logits / LSE buffers: call it after the step's delta_select
 * calls.  recall_out: device [batch][m] fp32.  Not sequence-sharded. */
delta_status delta_attention_recall(delta_t h, int32_t layer, int32_t batch, const void* q, float* recall_out,
                                   cudaStream_t stream);

/* Chunked prefill (NEXT-3; the step before the decode path, PAPER.md:34-45 over a prompt,
 * SPEC.md:387-395): appends ntok tokens per sequence (Eq.7, as delta_append_kv; Quest reps
 * too), then for each new token i at position n_b + i computes Eq.4 over tokens t <= n_b + i
 * (causal), every head j against group phi(j).  q: device [batch][ntok][m][d] bf16; k_new,
 * v_new: [batch][ntok][g][d] bf16; out: [batch][ntok][m][d] fp32; lse_out: optional
 * [batch][ntok][m] fp32.  bf16 KV only; not sequence-sharded.  Two launches. */
delta_status delta_prefill(delta_t h, int32_t layer, int32_t batch, int32_t ntok, const void* q, const void* k_new,
                           const void* v_new, float* out, float* lse_out, cudaStream_t stream);

/* Test hook: device pointers into the workspace.  which = 0: unit keys of the latest selection
 * [max_batch][ceil(max_seq_len/select_block)] fp32 (RAAS: the page scores of the latest RAAS
 * layer's update, by page); which = 1: Quest page representatives (layout above); which = 2:
 * RaaS last-salient steps [L][max_batch][ceil(max_seq_len/P)] int32.  *bytes = region size. */
delta_status delta_workspace_region(delta_t h, int32_t which, void** ptr, size_t* bytes);

/* Synchronises `stream`, reads and clears the sticky device error flag.
 * *sticky = DELTA_OK or the first device-side error recorded. The only syncing call. */
delta_status delta_get_error(delta_t h, cudaStream_t stream, delta_status* sticky);

/* ---- sequence sharding (shard_world > 1) -------------------------------------------
 * Rank 0 calls delta_nccl_get_unique_id; the 128 bytes are broadcast to all ranks (e.g. with
 * torch.distributed) and passed as delta_config.nccl_id.  NCCL is loaded at run time
 * (libnccl.so.2 already in the process, else $DELTA_NCCL_LIB).  DELTA_ERR_NCCL if absent. */
/* Where to dlopen NCCL from if no libnccl.so.2 is loaded or on the loader path (e.g. the copy
 * torch ships); call before the first NCCL use.  The library reads no environment variables. */
delta_status delta_set_nccl_library(const char* path);
delta_status delta_nccl_get_unique_id(void* out_128_bytes);

/* Host-only: the page range [*page_lo, *page_hi) of every sequence that rank cfg->shard_rank
 * holds (contiguous, page-aligned shares of ceil(max_seq_len/P) pages); [0, pages) if W = 1. */
delta_status delta_shard_range(const delta_config* cfg, int32_t* page_lo, int32_t* page_hi);

/* External-exchange mode (nccl_id == NULL).  which = 0: attention partials (after every
 * delta_decode_layer / delta_append_decode_layer), 1: Delta-layer candidates (after
 * delta_select).  The caller must make recv = the concatenation, in rank order, of every
 * rank's send block (block_bytes each): an all-gather.  Device pointers into the workspace. */
delta_status delta_shard_exchange_buffers(delta_t h, int32_t which, void** send, void** recv,
                                          size_t* block_bytes);
/* After the attention exchange: LSE-merge the ranks' partials in rank order -> out [batch][m][d],
 * lse_out (optional) — identical on every rank.  PAPER.md:61-67 (any partition of the attended
 * set gives the same softmax). */
delta_status delta_shard_merge(delta_t h, int32_t layer, int32_t batch, float* out, float* lse_out,
                               cudaStream_t stream);
/* After the candidate exchange: global top-k over all ranks' candidates + the forced units ->
 * the plan (and optional idx_out / count_out as in delta_select). */
delta_status delta_shard_select_merge(delta_t h, int32_t layer, int32_t batch, int32_t* idx_out,
                                      int32_t* count_out, cudaStream_t stream);

delta_role   delta_layer_role(delta_t h, int32_t layer);        /* -1 cast if out of range */
int32_t      delta_governing_layer(delta_t h, int32_t layer);  /* Delta layer of a SPARSE layer */
int32_t      delta_plan_capacity(delta_t h);                   /* max |rho| in units */
const char*  delta_last_error_message(delta_t h);              /* NULL handle: global message */
const char*  delta_version(void);
delta_status delta_destroy(delta_t h);

/* Launch statistics for the benchmark contract: number of kernels this handle has
 * enqueued since creation (graph replays count their kernels). */
uint64_t     delta_kernels_launched(delta_t h);

/* Number of CUDA-graph captures delta_decode_step has made (one per distinct input pointer
 * set / stream / batch; replays add none) — lets a timing loop assert it measured pure replays. */
uint64_t     delta_graph_captures(delta_t h);

/* Which attention kernel variant a decode of `layer` at `batch` launches (for reports); "" for
 * a bad handle / layer / batch.  The string is static. */
const char*  delta_layer_kernel_name(delta_t h, int32_t layer, int32_t batch);

/* Experiment hook (tools/, never needed for correct results): override one kernel-variant knob
 * of a handle (nsplit, snsplit, deep, prewait, early, umma, policy, seltrig, selhist, gmerge,
 * gm2, lat, qpf, pfumma — see DESIGN.md §7).  Drops the handle's captured step graphs.  CONFIG
 * for an unknown key, USAGE for a null handle.  The library reads no environment variables. */
delta_status delta_set_tuning(delta_t h, const char* key, int32_t value);

/* Measurement utility, not part of the method (SURVEY §8(d) "K10"): streams `bytes` of the
 * device buffer `buf` once with 16-byte loads (a pure-read roofline reference measured in the
 * same run as the decode kernels).  `sink` is a device float the kernel may write.  Enqueued on
 * `stream`; returns USAGE for null pointers, CUDA on a launch failure. */
delta_status delta_read_bandwidth_probe(const void* buf, size_t bytes, float* sink, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* DELTA_H */
