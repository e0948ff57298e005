/*
 * delta_oracle.h — ORACLE for DELTA decode-step attention (arXiv 2510.09883).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or call anything in oracle/.
 * The product path (paper_2510_09883_b200/, libdelta.so) never links, imports
 * or executes this code, and this code shares nothing with it: no headers, no
 * helpers, no constants, no generators.
 *
 * Plain, slow, obviously-correct fp64 C.  Every function follows the plain
 * definition in the paper (the method reaches its defined result exactly; there
 * is no approximation on the path), in the paper's order and notation.
 * Readings of ambiguous passages are the SURVEY.md §8(c) readings R1..R28,
 * collected in DESIGN.md §3.  Citations: "PAPER.md:L" is a line of the paper's
 * LaTeX in /root/reference; "SPEC.md:L" a line of the companion CPU-program spec.
 *
 * Index base is 0 everywhere (R25).  Status codes mirror the SPEC error classes:
 *   0 ok, 1 configuration error, 2 usage error, 3 numeric error (NaN/Inf).
 *
 * Parity pins (tests/test_oracle_pins.py) fix every function below against the
 * paper's worked values, closed forms, brute force and library routines.  No
 * function here is "parity unpinned".
 */
#ifndef DELTA_ORACLE_H
#define DELTA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_CONFIG 1
#define ORACLE_ERR_USAGE 2
#define ORACLE_ERR_NUMERIC 3

/* One sequence's paged K/V for one layer.  Pools are [phys_pages][g][P][d]
 * (page-major, then KV group, then slot, then dim), values widened EXACTLY
 * from the stored dtype (bf16 or fp32) to float.  block_table maps the
 * sequence's logical page u to a physical page ("fixed-size
 * pages of P tokens", p(t) maps token t to its page). */
typedef struct {
    int32_t P;                  /* page size (P = 16)            */
    int32_t g;                  /* KV groups                                   */
    int32_t d;                  /* head dim d_head                             */
    const float* k_pool;
    const float* v_pool;
    const int32_t* block_table;
} oracle_seq_kv;

/* p(t) = floor(t / P), 0-based. */
int64_t oracle_page_of(int64_t t, int32_t P);

/* Pointer to K (or V) row of token t, KV group grp (PAPER.md:53-56 K_l). */
const float* oracle_k_row(const oracle_seq_kv* kv, int64_t t, int32_t grp);
const float* oracle_v_row(const oracle_seq_kv* kv, int64_t t, int32_t grp);

/* KV append, Eq.7: K <- [K; k_new], V <- [V; v_new].
 * Writes token position n (= tokens already stored) into page p(n), slot
 * n mod P, for every group.  k_new/v_new are [g][d].  Pools are writable here. */
int oracle_append(float* k_pool, float* v_pool, const int32_t* block_table,
                  int32_t P, int32_t g, int32_t d, int64_t n,
                  const float* k_new, const float* v_new);

/* softmax (Eq.4's softmax): two-pass with max subtraction.
 * alpha[t] = exp(a[t] - LSE), LSE = M + log(sum_t exp(a[t] - M)).
 * n == 0 -> usage error; NaN/Inf in a -> numeric error. */
int oracle_softmax(const double* a, int64_t n, double* alpha, double* lse);

/* Scaled dot-product attention for ONE query head over an ordered token set
 * (Eq.4):  a_t = scale * (q . k_{grp,t});  alpha = softmax(a);
 * out = sum_t alpha_t v_{grp,t}.  When tokens is a strict subset of the cache
 * the softmax renormalises over that subset only (reading R10).
 * tokens == NULL means t = 0..ntok-1 (the whole cache).  q is [d].
 * alpha (optional, may be NULL) receives [ntok] weights in token-list order. */
int oracle_attend(const float* q, const oracle_seq_kv* kv, int32_t grp,
                  const int64_t* tokens, int64_t ntok, double scale,
                  double* out, double* lse, double* alpha);

/* All m query heads of one sequence/layer.  GQA group map phi(j) = floor(j/(m/g))
 * ("each query head j is assigned to one KV group"; SPEC.md:73;
 * reading R15 contiguous groups).  q is [m][d]; out [m][d]; lse [m];
 * alpha (optional) [m][ntok].  OpenMP over heads (nthreads <= 0: default). */
int oracle_decode_heads(const float* q, int32_t m, const oracle_seq_kv* kv,
                        const int64_t* tokens, int64_t ntok, double scale,
                        double* out, double* lse, double* alpha, int nthreads);

/* Token importance s_t = max_{j=1..m} alpha_j(t) (R7:
 * max over ALL m query heads of the normalised weight).  alpha is [m][s]. */
int oracle_token_scores(const double* alpha, int32_t m, int64_t s, double* s_t);

/* Page score S_u = sum_{t: p(t)=u} s_t; a partial last page
 * sums only its filled slots.  Output [ceil(s/P)]. */
int oracle_page_scores(const double* s_t, int64_t s, int32_t P, double* S_u);

/* Selection (PAPER.md:168-171 token form; PAPER.md:185 page form), with the
 * readings R1-R6, R9, R12, R23:
 *   units are tokens (block == 1) or pages (block == P), n_units = ceil(s/block);
 *   forced F = units overlapping the sink [0, n_sink) and the recency window
 *   [s - n_window, s);  candidates C = all units \ F;
 *   if |C| <= k_units: rho = all units;
 *   else rho = F  U  the first k_units of C sorted by (key desc, index asc).
 * unit_keys is [n_units] (entries of forced units are ignored).
 * units_out receives rho ascending; returns |rho| (or -1 on a usage error). */
int64_t oracle_select(const double* unit_keys, int64_t s, int32_t block,
                      int32_t n_sink, int32_t n_window, int64_t k_units,
                      int64_t* units_out);

/* tokens(rho): the ascending tokens t < s whose unit is in rho.  Returns count. */
int64_t oracle_units_to_tokens(const int64_t* units, int64_t n_units_sel,
                               int32_t block, int64_t s, int64_t* tokens_out);

/* Three-tier schedule:
 * layers [0,F) FULL (role 0); Delta layers SELECT (role 1); every other layer
 * SPARSE (role 2) governed by the nearest Delta layer below it.
 * Config error if a Delta layer lies inside the full prefix, Delta layers are
 * not strictly ascending / out of range, or a layer >= F has no Delta <= it.
 * governing_out[l] = l for FULL/SELECT layers, the governing Delta otherwise. */
int oracle_validate_tiers(int32_t num_layers, int32_t num_full_prefix,
                          int32_t n_delta, const int32_t* delta_layers,
                          int32_t* role_out, int32_t* governing_out);

/* KV bytes = Layers x s x b x g x d_head x 2 (K and V) x bytes/scalar
 * (PAPER.md:11 footnote). */
uint64_t oracle_kv_bytes(uint64_t num_layers, uint64_t seq_len, uint64_t batch,
                         uint64_t kv_heads, uint64_t head_dim, uint64_t bytes_per_scalar);

/* Attention recall R = sum_{u in rho} alpha(u) / sum_u alpha(u) (Eq.9,
 * PAPER.md:112-117).  rho holds token indices into alpha[0..s). */
double oracle_attention_recall(const double* alpha, int64_t s,
                               const int64_t* rho, int64_t n_rho);

/* ---------------------------------------------------------------- Quest (NEXT-1)
 * The paper's comparison policy Quest ("compresses each KV page into two
 * representative vectors (element-wise min/max of keys), scores pages against the current
 * query, and retrieves the top-k for attention").  Readings:
 *   Q1 score of page u for head j = sum_e max(q_j[e] min_u[e], q_j[e] max_u[e]) with the reps
 *      of group phi(j) (the upper bound of q . k over the page's keys; no
 *      softmax scale — a positive factor does not change the ranking);
 *   Q2 page key = max over the m query heads (SPEC.md:347 ledger, mirroring R7);
 *   Q3 selection = oracle_select on the page keys (same forced sink/window pages, budget
 *      k / P candidate pages, ties to the lowest index R9) so Quest and DELTA attend the same
 *      number of tokens; every layer >= F selects its own pages from its own reps. */

/* Page representatives: for page u < ceil(s/P) and group grp, min/max over the page's
 * filled slots t < s of K[t][grp][e].  reps is [n_pages][g][2][d]
 * (min row, then max row). */
int oracle_quest_reps(const oracle_seq_kv* kv, int64_t s, double* reps);

/* Page keys (Q1, Q2): out[u] = max_j sum_e max(q[j][e] min, q[j][e] max), q [m][d]. */
int oracle_quest_scores(const float* q, int32_t m, int32_t g, int32_t d,
                        const double* reps, int64_t n_pages, double* out);

/* ---------------------------------------------------------------- RaaS (NEXT-4)
 * The paper's eviction baseline RaaS ("an eviction-based method that removes
 * pages with consistently low attention scores ... risking the loss of tokens that may later
 * become important").  Readings RS1-RS4: one step of the
 * threshold-refresh / least-recently-salient rule for ONE (layer, sequence):
 *   1. retained pages u with S[u] >= threshold get last[u] = current_step;
 *   2. while more than `capacity` retained pages are not exempt: evict the non-exempt retained
 *      page with the smallest (last[u], u) — retained[u] = 0 for good.
 * S: [n_pages] scores (entries of non-retained pages ignored); exempt, retained: [n_pages]
 * 0/1; last: [n_pages].  evicted_out receives the evicted pages in eviction order; returns
 * their number. */
int64_t oracle_raas_step(int64_t n_pages, const double* S, int64_t current_step, double threshold,
                         const char* exempt, int64_t capacity, char* retained, int64_t* last,
                         int64_t* evicted_out);

#ifdef __cplusplus
}
#endif
#endif
