// combine.cuh — split-K (flash-decoding) merge used by every attention kernel.
//
// Within a CTA, each warp keeps an online-softmax state (running max m in log2 units,
// running sum l, unnormalised O) over the tokens it processed.  cta_merge() folds the
// warps' states (fixed warp order) into ONE partial (o normalised, lse in log2 units)
// per (sequence, kv head, split, query head).  grid_combine() then elects the last CTA
// of each (sequence, kv head) with an arrival counter ("last block done"), which merges
// all splits in ascending split order — a fixed order, so results are deterministic —
// and writes O, LSE.  This is the identity LSE = log sum_s exp(lse_s),
// O = sum_s exp(lse_s - LSE) o_s (any partition of the token set gives the same
// attention, Eq.4).
#pragma once
#include "internal.h"
#include "ptx.cuh"

namespace delta {

constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ void consumer_bar(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ void set_err(int32_t* err, int code) {
    if (err) atomicCAS(err, 0, code);
}

// smem layout for the per-warp states: ms[NW][16], ls[NW][16], os[NW][16][D]
template <int D>
__device__ __forceinline__ void cta_merge(const AttnParams& p, const float* ms, const float* ls,
                                          const float* os, int nw, int b, int h, int split,
                                          int tid, int nthreads) {
    const int gs = p.gs;
    for (int idx = tid; idx < gs * D; idx += nthreads) {
        const int row = idx / D, col = idx - row * D;
        float M = -INFINITY;
        for (int w = 0; w < nw; ++w) M = fmaxf(M, ms[w * 16 + row]);
        float L = 0.f, o = 0.f;
        if (M != -INFINITY) {
            for (int w = 0; w < nw; ++w) {
                const float mw = ms[w * 16 + row];
                const float f = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
                L += ls[w * 16 + row] * f;
                o += os[(w * 16 + row) * D + col] * f;
            }
        }
        const size_t prow = ((size_t)(b * p.g + h) * p.nsplit + split) * gs + row;
        p.part_o[prow * D + col] = (L > 0.f) ? o / L : 0.f;
        if (col == 0) p.part_lse[prow] = (L > 0.f) ? M + log2f(L) : -INFINITY;
    }
}

// Called by `nthreads` threads (named barrier 1) after cta_merge.  s_post: cache length
// after this launch (used to bump seq_len when the launch fused the append).
template <int D>
__device__ __forceinline__ void grid_combine(const AttnParams& p, int b, int h, int s_post, bool stale,
                                             bool capacity_err, int tid, int nthreads, int* sflag) {
    __threadfence();
    consumer_bar(nthreads);
    if (tid == 0) {
        const int t = atomicAdd(&p.cnt_head[b * p.g + h], 1);
        *sflag = (t == p.nsplit - 1);
    }
    consumer_bar(nthreads);
    if (!*sflag) return;
    __threadfence();
    const int gs = p.gs;
    const size_t base = (size_t)(b * p.g + h) * p.nsplit;
    bool bad = false;
    for (int idx = tid; idx < gs * D; idx += nthreads) {
        const int row = idx / D, col = idx - row * D;
        float M = -INFINITY;
        for (int sp = 0; sp < p.nsplit; ++sp) M = fmaxf(M, __ldcg(&p.part_lse[(base + sp) * gs + row]));
        float L2 = -INFINITY, o = 0.f;
        if (M != -INFINITY) {
            float W = 0.f;
            for (int sp = 0; sp < p.nsplit; ++sp) {
                const float l = __ldcg(&p.part_lse[(base + sp) * gs + row]);
                if (l != -INFINITY) W += exp2f(l - M);
            }
            L2 = M + log2f(W);
            for (int sp = 0; sp < p.nsplit; ++sp) {
                const float l = __ldcg(&p.part_lse[(base + sp) * gs + row]);
                if (l != -INFINITY) o += exp2f(l - L2) * __ldcg(&p.part_o[((base + sp) * gs + row) * D + col]);
            }
        }
        if (stale) o = __int_as_float(0x7fc00000);  // NaN: stale plan must be loud
        else if (!isfinite(o)) bad = true;
        const int j = h * gs + row;
        p.out[((size_t)b * p.m + j) * D + col] = o;
        if (col == 0) {
            const float lse = (L2 == -INFINITY) ? -INFINITY : L2 * kLn2;
            if (p.lse_out) p.lse_out[(size_t)b * p.m + j] = lse;
            if (p.role == kRoleSelect) p.lse_buf[(size_t)b * p.m + j] = lse;
        }
    }
    if (bad) set_err(p.err, kDevNumeric);
    consumer_bar(nthreads);
    if (tid == 0) {
        if (stale) set_err(p.err, kDevUsage);
        if (capacity_err) set_err(p.err, kDevCapacity);
        if (s_post <= 0) set_err(p.err, kDevUsage);  // attention over an empty cache
        p.cnt_head[b * p.g + h] = 0;
        __threadfence();
        const int t2 = atomicAdd(&p.cnt_seq[b], 1);
        if (t2 == p.g - 1) {
            if (p.fuse_append && !capacity_err) p.seq_len[p.layer * p.max_batch + b] = s_post;
            p.cnt_seq[b] = 0;
        }
    }
}

}  // namespace delta
