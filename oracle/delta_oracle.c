/*
 * delta_oracle.c — ORACLE (test infrastructure only; see delta_oracle.h).
 *
 * Plain fp64 C, compiled with -O2 -ffp-contract=off and no fast-math so every
 * multiply and add is a separately rounded IEEE double operation.  Loops follow
 * the paper's formulas term by term; no blocking, no fusion, no reordering.
 */
#include "delta_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int64_t oracle_page_of(int64_t t, int32_t P) { return t / (int64_t)P; }

static const float* row_of(const float* pool, const oracle_seq_kv* kv, int64_t t, int32_t grp) {
    /* pool layout [phys_pages][g][P][d]; token t lives in logical page p(t),
     * slot t mod P. */
    int64_t page = oracle_page_of(t, kv->P);
    int64_t slot = t - page * kv->P;
    int64_t phys = kv->block_table[page];
    return pool + (((phys * kv->g + grp) * kv->P + slot) * kv->d);
}

const float* oracle_k_row(const oracle_seq_kv* kv, int64_t t, int32_t grp) {
    return row_of(kv->k_pool, kv, t, grp);
}
const float* oracle_v_row(const oracle_seq_kv* kv, int64_t t, int32_t grp) {
    return row_of(kv->v_pool, kv, t, grp);
}

int oracle_append(float* k_pool, float* v_pool, const int32_t* block_table,
                  int32_t P, int32_t g, int32_t d, int64_t n,
                  const float* k_new, const float* v_new) {
    /* Eq.7: the new token takes position n = current length. */
    if (n < 0 || P < 1 || g < 1 || d < 1) return ORACLE_ERR_USAGE;
    int64_t page = oracle_page_of(n, P);
    int64_t slot = n - page * P;
    int64_t phys = block_table[page];
    for (int32_t grp = 0; grp < g; ++grp) {
        float* kr = k_pool + ((phys * g + grp) * P + slot) * d;
        float* vr = v_pool + ((phys * g + grp) * P + slot) * d;
        for (int32_t e = 0; e < d; ++e) {
            kr[e] = k_new[grp * d + e];
            vr[e] = v_new[grp * d + e];
        }
    }
    return ORACLE_OK;
}

int oracle_softmax(const double* a, int64_t n, double* alpha, double* lse) {
    if (n <= 0) return ORACLE_ERR_USAGE;
    /* pass 1: M = max_t a_t */
    double M = a[0];
    for (int64_t t = 0; t < n; ++t) {
        if (!isfinite(a[t])) return ORACLE_ERR_NUMERIC;
        if (a[t] > M) M = a[t];
    }
    /* pass 2: Z = sum_t exp(a_t - M), LSE = M + log Z */
    double Z = 0.0;
    for (int64_t t = 0; t < n; ++t) Z += exp(a[t] - M);
    double L = M + log(Z);
    /* alpha_t = exp(a_t - LSE) */
    if (alpha)
        for (int64_t t = 0; t < n; ++t) alpha[t] = exp(a[t] - L);
    if (lse) *lse = L;
    return ORACLE_OK;
}

int oracle_attend(const float* q, const oracle_seq_kv* kv, int32_t grp,
                  const int64_t* tokens, int64_t ntok, double scale,
                  double* out, double* lse, double* alpha) {
    if (ntok <= 0) return ORACLE_ERR_USAGE;
    const int32_t d = kv->d;
    double* a = (double*)malloc(sizeof(double) * (size_t)ntok);
    double* w = alpha ? alpha : (double*)malloc(sizeof(double) * (size_t)ntok);
    if (!a || !w) { free(a); if (!alpha) free(w); return ORACLE_ERR_USAGE; }
    /* A_j = Q_j K_phi(j)^T / sqrt(d)   (Eq.4) */
    for (int64_t i = 0; i < ntok; ++i) {
        int64_t t = tokens ? tokens[i] : i;
        const float* k = oracle_k_row(kv, t, grp);
        double dot = 0.0;
        for (int32_t e = 0; e < d; ++e) dot += (double)q[e] * (double)k[e];
        a[i] = scale * dot;
    }
    /* alpha_j = softmax(A_j) */
    int st = oracle_softmax(a, ntok, w, lse);
    if (st == ORACLE_OK) {
        /* O_j = softmax(A_j) V_phi(j) */
        for (int32_t e = 0; e < d; ++e) out[e] = 0.0;
        for (int64_t i = 0; i < ntok; ++i) {
            int64_t t = tokens ? tokens[i] : i;
            const float* v = oracle_v_row(kv, t, grp);
            for (int32_t e = 0; e < d; ++e) out[e] += w[i] * (double)v[e];
        }
    }
    free(a);
    if (!alpha) free(w);
    return st;
}

int oracle_decode_heads(const float* q, int32_t m, const oracle_seq_kv* kv,
                        const int64_t* tokens, int64_t ntok, double scale,
                        double* out, double* lse, double* alpha, int nthreads) {
    if (m < 1 || kv->g < 1 || m % kv->g != 0) return ORACLE_ERR_CONFIG;
    const int32_t gs = m / kv->g; /* query heads per KV group */
    const int32_t d = kv->d;
    int status = ORACLE_OK;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
    for (int32_t j = 0; j < m; ++j) {
        int32_t grp = j / gs; /* phi(j), R15 */
        int st = oracle_attend(q + (int64_t)j * d, kv, grp, tokens, ntok, scale,
                               out + (int64_t)j * d, lse + j,
                               alpha ? alpha + (int64_t)j * ntok : NULL);
        if (st != ORACLE_OK) {
#ifdef _OPENMP
#pragma omp critical
#endif
            status = st;
        }
    }
    (void)nthreads;
    return status;
}

int oracle_token_scores(const double* alpha, int32_t m, int64_t s, double* s_t) {
    if (m < 1 || s < 0) return ORACLE_ERR_USAGE;
    for (int64_t t = 0; t < s; ++t) {
        double best = alpha[t]; /* head j = 0 */
        for (int32_t j = 1; j < m; ++j) {
            double v = alpha[(int64_t)j * s + t];
            if (v > best) best = v;
        }
        s_t[t] = best;
    }
    return ORACLE_OK;
}

int oracle_page_scores(const double* s_t, int64_t s, int32_t P, double* S_u) {
    if (P < 1 || s < 0) return ORACLE_ERR_USAGE;
    int64_t n_pages = (s + P - 1) / P;
    for (int64_t u = 0; u < n_pages; ++u) S_u[u] = 0.0;
    for (int64_t t = 0; t < s; ++t) S_u[oracle_page_of(t, P)] += s_t[t];
    return ORACLE_OK;
}

/* candidate ordering: key descending, then index ascending (reading R9) */
typedef struct { double key; int64_t idx; } cand_t;
static int cand_cmp(const void* x, const void* y) {
    const cand_t* a = (const cand_t*)x;
    const cand_t* b = (const cand_t*)y;
    if (a->key > b->key) return -1;
    if (a->key < b->key) return 1;
    if (a->idx < b->idx) return -1;
    if (a->idx > b->idx) return 1;
    return 0;
}
static int cmp_i64(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    return (a > b) - (a < b);
}

int64_t oracle_select(const double* unit_keys, int64_t s, int32_t block,
                      int32_t n_sink, int32_t n_window, int64_t k_units,
                      int64_t* units_out) {
    if (s < 0 || block < 1 || n_sink < 0 || n_window < 0 || k_units < 0) return -1;
    if (s == 0) return 0;
    int64_t n_units = (s + block - 1) / block;
    /* forced set F: units overlapping [0, n_sink) and [s - n_window, s)  (R2, R3, R6) */
    char* forced = (char*)calloc((size_t)n_units, 1);
    if (!forced) return -1;
    if (n_sink > 0) {
        int64_t last_tok = (n_sink < s ? n_sink : s) - 1;
        for (int64_t u = 0; u <= last_tok / block; ++u) forced[u] = 1;
    }
    if (n_window > 0) {
        int64_t first_tok = s - n_window;
        if (first_tok < 0) first_tok = 0;
        for (int64_t u = first_tok / block; u < n_units; ++u) forced[u] = 1;
    }
    /* candidates C = units \ F  (R4) */
    int64_t n_cand = 0;
    for (int64_t u = 0; u < n_units; ++u) n_cand += !forced[u];
    int64_t n_out = 0;
    if (n_cand <= k_units) {
        /* budget covers every candidate: rho = all units (R12) */
        for (int64_t u = 0; u < n_units; ++u) units_out[n_out++] = u;
    } else {
        cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)n_cand);
        if (!c) { free(forced); return -1; }
        int64_t i = 0;
        for (int64_t u = 0; u < n_units; ++u)
            if (!forced[u]) { c[i].key = unit_keys[u]; c[i].idx = u; ++i; }
        /* Topk({s_t : t in C}, k) — sort by (key desc, index asc) and take k */
        qsort(c, (size_t)n_cand, sizeof(cand_t), cand_cmp);
        for (int64_t u = 0; u < n_units; ++u)
            if (forced[u]) units_out[n_out++] = u;
        for (int64_t r = 0; r < k_units; ++r) units_out[n_out++] = c[r].idx;
        free(c);
        qsort(units_out, (size_t)n_out, sizeof(int64_t), cmp_i64); /* ascending */
    }
    free(forced);
    return n_out;
}

int64_t oracle_units_to_tokens(const int64_t* units, int64_t n_units_sel,
                               int32_t block, int64_t s, int64_t* tokens_out) {
    int64_t n = 0;
    for (int64_t i = 0; i < n_units_sel; ++i) {
        int64_t u = units[i];
        for (int64_t t = u * block; t < (u + 1) * block && t < s; ++t) tokens_out[n++] = t;
    }
    return n;
}

int oracle_validate_tiers(int32_t num_layers, int32_t num_full_prefix,
                          int32_t n_delta, const int32_t* delta_layers,
                          int32_t* role_out, int32_t* governing_out) {
    if (num_layers < 1 || num_full_prefix < 0 || num_full_prefix > num_layers || n_delta < 0)
        return ORACLE_ERR_CONFIG;
    for (int32_t i = 0; i < n_delta; ++i) {
        if (delta_layers[i] < num_full_prefix || delta_layers[i] >= num_layers)
            return ORACLE_ERR_CONFIG; /* Delta inside the full prefix / out of range */
        if (i > 0 && delta_layers[i] <= delta_layers[i - 1]) return ORACLE_ERR_CONFIG;
    }
    int32_t current = -1; /* governing Delta layer for the group being walked */
    int32_t next = 0;
    for (int32_t l = 0; l < num_layers; ++l) {
        if (l < num_full_prefix) {
            role_out[l] = 0;
            governing_out[l] = l;
        } else if (next < n_delta && delta_layers[next] == l) {
            role_out[l] = 1;
            governing_out[l] = l;
            current = l;
            ++next;
        } else {
            if (current < 0) return ORACLE_ERR_CONFIG; /* sparse layer with no Delta below */
            role_out[l] = 2;
            governing_out[l] = current;
        }
    }
    return ORACLE_OK;
}

uint64_t oracle_kv_bytes(uint64_t num_layers, uint64_t seq_len, uint64_t batch,
                         uint64_t kv_heads, uint64_t head_dim, uint64_t bytes_per_scalar) {
    return num_layers * seq_len * batch * kv_heads * head_dim * 2ull * bytes_per_scalar;
}

double oracle_attention_recall(const double* alpha, int64_t s,
                               const int64_t* rho, int64_t n_rho) {
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < n_rho; ++i) {
        if (rho[i] < 0 || rho[i] >= s) return NAN;
        num += alpha[rho[i]];
    }
    for (int64_t t = 0; t < s; ++t) den += alpha[t];
    return num / den;
}

/* ---------------------------------------------------------------- Quest (NEXT-1) */

int oracle_quest_reps(const oracle_seq_kv* kv, int64_t s, double* reps) {
    if (!kv || s < 0) return ORACLE_ERR_USAGE;
    const int64_t n_pages = (s + kv->P - 1) / kv->P;
    for (int64_t u = 0; u < n_pages; ++u) {
        for (int32_t grp = 0; grp < kv->g; ++grp) {
            double* mn = reps + ((size_t)u * kv->g + grp) * 2 * kv->d;
            double* mx = mn + kv->d;
            /* element-wise extrema over the keys of page u ("element-wise min/max") */
            for (int64_t t = u * kv->P; t < (u + 1) * kv->P && t < s; ++t) {
                const float* k = oracle_k_row(kv, t, grp);
                for (int32_t e = 0; e < kv->d; ++e) {
                    if (t == u * kv->P || (double)k[e] < mn[e]) mn[e] = (double)k[e];
                    if (t == u * kv->P || (double)k[e] > mx[e]) mx[e] = (double)k[e];
                }
            }
        }
    }
    return ORACLE_OK;
}

int oracle_quest_scores(const float* q, int32_t m, int32_t g, int32_t d,
                        const double* reps, int64_t n_pages, double* out) {
    if (m < 1 || g < 1 || m % g != 0 || d < 1) return ORACLE_ERR_USAGE;
    const int32_t gs = m / g;
    for (int64_t u = 0; u < n_pages; ++u) {
        double best = 0.0;
        for (int32_t j = 0; j < m; ++j) {
            const int32_t grp = j / gs; /* phi(j), R15 */
            const double* mn = reps + ((size_t)u * g + grp) * 2 * d;
            const double* mx = mn + d;
            /* Q1: sum_e max(q_e min_e, q_e max_e) >= q . k for every key of the page */
            double sc = 0.0;
            for (int32_t e = 0; e < d; ++e) {
                const double a = (double)q[(size_t)j * d + e] * mn[e];
                const double b = (double)q[(size_t)j * d + e] * mx[e];
                sc += a > b ? a : b;
            }
            if (j == 0 || sc > best) best = sc; /* Q2: max over heads */
        }
        out[u] = best;
    }
    return ORACLE_OK;
}

/* ---------------------------------------------------------------- RaaS (NEXT-4) */

int64_t oracle_raas_step(int64_t n_pages, const double* S, int64_t current_step, double threshold,
                         const char* exempt, int64_t capacity, char* retained, int64_t* last,
                         int64_t* evicted_out) {
    if (n_pages < 0 || capacity < 0) return -1;
    /* 1. refresh: "pages with S_u >= threshold get last_salient_step := current_step" */
    for (int64_t u = 0; u < n_pages; ++u)
        if (retained[u] && S[u] >= threshold) last[u] = current_step;
    /* 2. evict the least recently salient non-exempt pages until `capacity` remain */
    int64_t n_evicted = 0;
    for (;;) {
        int64_t count = 0, victim = -1;
        for (int64_t u = 0; u < n_pages; ++u) {
            if (!retained[u] || exempt[u]) continue;
            ++count;
            if (victim < 0 || last[u] < last[victim]) victim = u; /* ties: lowest index (scan order) */
        }
        if (count <= capacity) break;
        retained[victim] = 0;
        evicted_out[n_evicted++] = victim;
    }
    return n_evicted;
}
