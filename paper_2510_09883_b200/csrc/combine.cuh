// combine.cuh — split-K (flash-decoding) merge used by every attention kernel, done inside
// a thread-block cluster through distributed shared memory (no global partials, no
// arrival counters, no grid-wide fences).
//
// Within a CTA, each warp keeps an online-softmax state (running max m in log2 units,
// running sum l, unnormalised O) over the tokens it processed.
#pragma once
#include <cooperative_groups.h>

#include "internal.h"
#include "ptx.cuh"

namespace delta {

constexpr float kLn2 = 0.6931471805599453f;

// Dedicated shared-memory staging that cluster peers push into (must not overlap anything
// the owning CTA still uses while peers may be writing, e.g. its TMA ring).
template <int D>
struct ClusterStage {
    static constexpr int kO4 = 16 * D / 4 + kMaxSplit;            // float4 slots: sO[rank * per + k]
    static constexpr int kFloats = kO4 * 4 + 2 * kMaxSplit * 16;  // + sM[rank][16], sL[rank][16]
    static constexpr int kBytes = kFloats * 4;
};

// Row stride (floats) of the per-warp O states: D + 4 makes the fragment-order stores of
// the MMA accumulators bank-conflict free and keeps float4 rows aligned.
template <int D>
constexpr int os_stride() { return D + 4; }

__device__ __forceinline__ void consumer_bar(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ void set_err(int32_t* err, int code) {
    if (err) atomicCAS(err, 0, code);
}

// Shared-memory image of one (page, kv head) tile as the TMA box {64, 2P rows, D/64 halves}
// with SWIZZLE_128B writes it: [half][row][128 B]; rows 0..P-1 are K, rows P..2P-1 are V.
// Each 64-element half of all 2P rows is a run of 128-byte lines (the canonical UMMA SW128
// layout: K-major for K, MN-major for V).
template <int D>
struct TileLayout {
    static constexpr int kHalfBytes = 2 * kPage * 128;    // 4096: one half of the 32 rows
    static constexpr int kVOff = kPage * 128;             // 2048: first V row
    static constexpr int kBytes = (D / 64) * kHalfBytes;  // 8192 (d = 128) / 4096 (d = 64)
};
// Byte offset of 16-byte chunk c (0..D/8-1) of row r (K rows from the tile base, V rows from
// base + kVOff): the 128B swizzle XORs the chunk with the line index mod 8.
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
    return (uint32_t)((c >> 3) * TileLayout<D>::kHalfBytes + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// Does this rank hold logical page u (sequence sharding; always true when unsharded)?
__device__ __forceinline__ bool owns_page(const AttnParams& p, int u) { return u >= p.page_lo && u < p.page_hi; }

// The units this CTA (split `split` of the nsplit CTAs of one (sequence, kv head)) attends:
//  FULL / SELECT: pages [unit0, unit0 + n_items) of this rank's share of [0, ceil(s/P));
//  SPARSE: plan entries [unit0, e_end) of this rank's share of the plan (n_items tiles of
//  16 entries for a token plan); a stale plan (stamp != s) attends nothing (NaN outputs).
__device__ __forceinline__ void split_geometry(const AttnParams& p, int b, int split, int s, bool token_plan,
                                               int& unit0, int& n_items, int& e_end, bool& stale) {
    if (p.role != kRoleSparse) {
        const int npages = (s + kPage - 1) / kPage;
        const int lo = max(0, p.page_lo), hi = min(npages, p.page_hi), n = max(0, hi - lo);
        unit0 = lo + (int)((long long)split * n / p.nsplit);
        n_items = lo + (int)((long long)(split + 1) * n / p.nsplit) - unit0;
    } else {
        stale = p.plan_stamp[b] != s;
        const int cnt = stale ? 0 : p.plan_count[b];
        const int elo = (p.plan_lo && !stale) ? p.plan_lo[b] : 0;
        const int ehi = (p.plan_hi && !stale) ? p.plan_hi[b] : cnt;
        const int n = max(0, ehi - elo);
        unit0 = elo + (int)((long long)split * n / p.nsplit);
        e_end = elo + (int)((long long)(split + 1) * n / p.nsplit);
        n_items = token_plan ? (e_end - unit0 + 15) / 16 : e_end - unit0;
    }
}

// Cluster split-K epilogue, called by EVERY thread of every CTA of the cluster (the
// cluster = the `nsplit` CTAs of one (sequence, kv head); rank = split).  Push model, one
// cluster barrier:
//  1. each thread folds the warps' states (ms[w*16+row] running max in log2 units, ls
//     running sum, os[(w*OSROWS+row)*OS+col] unnormalised O) in fixed warp order into this CTA's
//     (M_c, L_c, O_c) for its float4 of the gs x D output, and stores it straight into the
//     shared staging of the CTA that owns that output slice (distributed shared memory);
//  2. cluster barrier (release / acquire): every pushed value is visible to its owner;
//  3. the owner of a slice merges the ns partials from its own shared memory in ascending
//     rank order: M = max_c M_c, w_c = exp2(M_c - M), L = sum_c w_c L_c,
//     O = sum_c w_c O_c / L, LSE = (M + log2 L) ln 2 — the identity that any partition of
//     the attended token set gives the same softmax (Eq.4).  Fixed order:
//     deterministic.  No CTA touches a peer's memory after the barrier.
//  Rank 0 then reports device errors and, for a fused append, adds 1 to the length counter.
//
// Length counter encoding: seq_len_raw[l][b] = n * g.  Each of the g head clusters of a
// fused append+decode adds 1 when it is done; every reader takes raw / g, which is exact
// because a reader's own cluster has not yet added, so at most g - 1 additions precede it.
template <int D, int NW, int OSROWS = 16>
__device__ __forceinline__ void cluster_epilogue(const AttnParams& p, const float* ms, const float* ls,
                                                 const float* os, float* stage, int b, int h, bool stale,
                                                 bool cap_err, int s_post) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int tid = threadIdx.x, nthreads = blockDim.x;
    const int gs = p.gs;
    const int ns = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    constexpr int C4 = D / 4, OS = os_stride<D>();
    const int total = gs * C4;
    const int per = (total + ns - 1) / ns;
    float4* sO = reinterpret_cast<float4*>(stage);
    float* sM = stage + ClusterStage<D>::kO4 * 4;
    float* sL = sM + kMaxSplit * 16;
    // 1. push: each thread folds the NW warp states of one float4 (fixed warp order, fully
    //    unrolled so every shared load is in flight at once) and stores it into the owner's
    //    staging; the c4 == 0 thread of a row also pushes the row's (M_c, L_c) to every owner.
    for (int idx = tid; idx < total; idx += nthreads) {
        const int row = idx / C4, c4 = idx - row * C4;
        float mw[NW];
        float4 v[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            mw[w] = ms[w * 16 + row];
            v[w] = reinterpret_cast<const float4*>(os + (w * OSROWS + row) * OS)[c4];
        }
        float M = mw[0];
#pragma unroll
        for (int w = 1; w < NW; ++w) M = fmaxf(M, mw[w]);
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        float f[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            f[w] = (M == -INFINITY || mw[w] == -INFINITY) ? 0.f : exp2f(mw[w] - M);
            o.x += f[w] * v[w].x; o.y += f[w] * v[w].y; o.z += f[w] * v[w].z; o.w += f[w] * v[w].w;
        }
        const int r = idx / per, k = idx - r * per;
        cl.map_shared_rank(sO, r)[rank * per + k] = o;
        if (c4 == 0) {
            float L = 0.f;
#pragma unroll
            for (int w = 0; w < NW; ++w) L += ls[w * 16 + row] * f[w];
            for (int rr = 0; rr < ns; ++rr) {
                cl.map_shared_rank(sM, rr)[rank * 16 + row] = M;
                cl.map_shared_rank(sL, rr)[rank * 16 + row] = L;
            }
        }
    }
    if (tid == 0) DTRACE(5);
    cl.sync();  // release / acquire: every pushed value is visible to its owner
    if (tid == 0) DTRACE(7);
    // 2. owner: 16 lanes per owned float4, lane c holds rank c's partial; max, weights and
    //    sums are fixed shuffle trees over the 16 lanes (deterministic).
    bool bad = false;
    const int grp = tid >> 4, c = tid & 15, ngrp = nthreads >> 4;
    for (int k0 = 0; k0 < per; k0 += ngrp) {
        const int k = k0 + grp;
        const int idx = rank * per + k;
        const bool live = k < per && idx < total;
        const int row = live ? idx / C4 : 0, c4 = live ? idx - row * C4 : 0;
        const bool mine = live && c < ns;
        float mc = mine ? sM[c * 16 + row] : -INFINITY;
        float lc = mine ? sL[c * 16 + row] : 0.f;
        float4 x = mine ? sO[c * per + k] : make_float4(0.f, 0.f, 0.f, 0.f);
        float M = mc;
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
        const float f = (M == -INFINITY || mc == -INFINITY) ? 0.f : exp2f(mc - M);
        float L = f * lc;
        float4 v = make_float4(f * x.x, f * x.y, f * x.z, f * x.w);
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) {
            L += __shfl_xor_sync(0xffffffffu, L, off);
            v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
            v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
            v.z += __shfl_xor_sync(0xffffffffu, v.z, off);
            v.w += __shfl_xor_sync(0xffffffffu, v.w, off);
        }
        if (live && c == 0) {
            const float inv = (L > 0.f) ? 1.f / L : 0.f;
            float4 o = make_float4(v.x * inv, v.y * inv, v.z * inv, v.w * inv);
            if (stale) {
                const float qn = __int_as_float(0x7fc00000);  // NaN: stale plan must be loud
                o = make_float4(qn, qn, qn, qn);
            } else if (!(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w))) {
                bad = true;
            }
            const int j = h * gs + row;
            const bool shard = p.shard_world > 1;  // the rank's partial; shard.cu merges the ranks
            reinterpret_cast<float4*>((shard ? p.part_o : p.out) + ((size_t)b * p.m + j) * D)[c4] = o;
            if (c4 == 0) {
                const float lse = (L > 0.f) ? (M + log2f(L)) * kLn2 : -INFINITY;
                if (shard) {
                    p.part_lse[(size_t)b * p.m + j] = lse;
                } else {
                    if (p.lse_out) p.lse_out[(size_t)b * p.m + j] = lse;
                    if (p.role == kRoleSelect) p.lse_buf[(size_t)b * p.m + j] = lse;
                }
            }
        }
    }
    if (tid == 0) DTRACE(9);
    if (bad) set_err(p.err, kDevNumeric);
    if (rank == 0 && tid == 0) {
        if (stale) set_err(p.err, kDevUsage);
        if (cap_err) set_err(p.err, kDevCapacity);
        if (s_post <= 0) set_err(p.err, kDevUsage);  // attention over an empty cache
        if (p.fuse_append && !cap_err) atomicAdd(&p.seq_len[p.layer * p.max_batch + b], 1);
    }
}

}  // namespace delta
