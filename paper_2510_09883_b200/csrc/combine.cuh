// combine.cuh — split-K (flash-decoding) merge used by every attention kernel, done inside
// a thread-block cluster through distributed shared memory (no global partials, no
// arrival counters, no grid-wide fences).
//
// Within a CTA, each warp keeps an online-softmax state (running max m in log2 units,
// running sum l, unnormalised O) over the tokens it processed.
#pragma once
#include "internal.h"
#include "ptx.cuh"

namespace delta {

constexpr float kLn2 = 0.6931471805599453f;

// Dedicated shared-memory staging that cluster peers push into (must not overlap anything
// the owning CTA still uses while peers may be writing, e.g. its TMA ring).
template <int D>
struct ClusterStage {
    static constexpr int kO4 = 16 * D / 4 + kMaxSplit;            // float4 slots: sO[rank * per + k]
    static constexpr int kFloats = kO4 * 4 + 2 * kMaxSplit * 16;  // + (M, L) pairs [rank][16]
    static constexpr int kBarOff = kFloats * 4;                   // + the arrival mbarrier (8 B)
    static constexpr int kBytes = kBarOff + 16;
};

__device__ __forceinline__ uint32_t cluster_nranks() {
    uint32_t n;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(n));
    return n;
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// Address of the same shared variable in cluster CTA `rank` (shared::cluster window).
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// Remote stores that complete bytes on the destination CTA's mbarrier: no fence and no
// cluster barrier on the push path (the owner waits on its own mbarrier for the bytes).
__device__ __forceinline__ void st_async_v4(uint32_t dst, float4 v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                 ::"r"(dst), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar) : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t dst, float a, float b, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
                 ::"r"(dst), "f"(a), "f"(b), "r"(bar) : "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// Output slice of the gs x D float4s that cluster rank `r` merges: [r * per, min(total, (r + 1) * per)).
struct EpiSlice {
    int total, per, lo, n4, rows;
    __device__ EpiSlice(int gs, int c4s, int ns, int r) {
        total = gs * c4s;
        per = (total + ns - 1) / ns;
        lo = r * per;
        n4 = max(0, min(total, lo + per) - lo);
        rows = n4 > 0 ? (lo + n4 - 1) / c4s - lo / c4s + 1 : 0;
    }
};

// Kernel prologue half of the cluster epilogue (thread 0, with the kernel's other mbarrier
// inits, before fence_mbar_init): the arrival barrier expects, from each of the ns ranks, one
// float4 per owned output element and one (M, L) pair per owned row.
template <int D>
__device__ __forceinline__ void cluster_stage_init(float* stage, int gs) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stage) + ClusterStage<D>::kBarOff);
    const int ns = (int)cluster_nranks();
    const EpiSlice sl(gs, D / 4, ns, (int)cluster_rank());
    mbar_init(bar, 1);
    mbar_arrive_expect_tx(bar, (uint32_t)(ns * (sl.n4 * 16 + sl.rows * 8)));
}

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

// fixed_part geometry (FULL / SELECT): pages per split of the rank's maximum range, so split c
// starts at page lo + c * fixed_pages(p) whatever the length (split_geometry, attn_tc.cu)
__device__ __forceinline__ int fixed_pages(const AttnParams& p) {
    const int lo = max(0, p.page_lo), maxr = max(0, min(p.bt_stride, p.page_hi) - lo);
    return (maxr + p.nsplit - 1) / p.nsplit;
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
        const int maxr = max(0, min(p.bt_stride, p.page_hi) - lo), pf = fixed_pages(p);
        if (p.fixed_part && n * 16 >= maxr * 15) {
            // fixed_part: split c starts at page c * ceil(max / nsplit) whatever s is (while the
            // cache is at least 15/16 full), so a producer can load its first block-table entries
            // together with the length counter instead of after it (attn_tc.cu)
            unit0 = lo + min(n, split * pf);
            n_items = lo + min(n, (split + 1) * pf) - unit0;
        } else {
            unit0 = lo + (int)((long long)split * n / p.nsplit);
            n_items = lo + (int)((long long)(split + 1) * n / p.nsplit) - unit0;
        }
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
// cluster = the `nsplit` CTAs of one (sequence, kv head); rank = split).  Push model over
// st.async: the kernel called cluster_stage_init (thread 0) and cluster_arrive_relaxed (all
// threads, after its __syncthreads) at entry, so every peer's arrival mbarrier is live by now.
//  1. each thread folds the warps' states (ms[w*16+row] running max in log2 units, ls
//     running sum, os[(w*OSROWS+row)*OS+col] unnormalised O) in fixed warp order into this CTA's
//     (M_c, L_c, O_c) for its float4 of the gs x D output and st.async-stores it straight into
//     the shared staging of the CTA that owns that output slice; the thread holding a row's
//     first float4 in an owner's range also sends the row's (M_c, L_c) pair;
//  2. the owner waits on its own arrival mbarrier until all ns ranks' bytes have landed (no
//     cluster barrier, no GPU-scope fence), then merges the ns partials in ascending rank
//     order: M = max_c M_c, w_c = exp2(M_c - M), L = sum_c w_c L_c, O = sum_c w_c O_c / L,
//     LSE = (M + log2 L) ln 2 — the identity that any partition of the attended token set
//     gives the same softmax (Eq.4).  Fixed order: deterministic.
//  A CTA exits once its own slice is written: nobody writes into its shared memory after its
//  barrier completed (the expected byte count is exact), and it never reads a peer's.
//  Rank 0 then reports device errors and, for a fused append, adds 1 to the length counter.
//
// Length counter encoding: seq_len_raw[l][b] = n * g.  Each of the g head clusters of a
// fused append+decode adds 1 when it is done; every reader takes raw / g, which is exact
// because a reader's own cluster has not yet added, so at most g - 1 additions precede it.
template <int D, int NW, int OSROWS = 16>
__device__ __forceinline__ void cluster_epilogue(const AttnParams& p, const float* ms, const float* ls,
                                                 const float* os, float* stage, int b, int h, bool stale,
                                                 bool cap_err, int s_post) {
    const int tid = threadIdx.x, nthreads = blockDim.x;
    const int gs = p.gs;
    const int ns = (int)cluster_nranks(), rank = (int)cluster_rank();
    constexpr int C4 = D / 4, OS = os_stride<D>();
    const EpiSlice mine(gs, C4, ns, rank);
    const int total = mine.total, per = mine.per;
    float4* sO = reinterpret_cast<float4*>(stage);
    float* sM = stage + ClusterStage<D>::kO4 * 4;  // float2 (M_c, L_c) per [rank][row]
    uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stage) + ClusterStage<D>::kBarOff);
    const uint32_t sO_u = smem_u32(sO), sM_u = smem_u32(sM), bar_u = smem_u32(bar);
    cluster_wait();  // pairs with the entry arrive: every peer's barrier is initialised
    if (ns == 1) {
        // a cluster of one CTA (one split): st.async needs a peer CTA, so fold the warp states
        // and write the outputs directly
        bool bad1 = false;
        for (int idx = tid; idx < total; idx += nthreads) {
            const int row = idx / C4, c4 = idx - row * C4;
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < NW; ++w) M = fmaxf(M, ms[w * 16 + row]);
            float L = 0.f;
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const float mw = ms[w * 16 + row];
                const float f = (M == -INFINITY || mw == -INFINITY) ? 0.f : exp2f(mw - M);
                const float4 v = reinterpret_cast<const float4*>(os + (w * OSROWS + row) * OS)[c4];
                o.x += f * v.x; o.y += f * v.y; o.z += f * v.z; o.w += f * v.w;
                L += ls[w * 16 + row] * f;
            }
            const float inv = (L > 0.f) ? __frcp_rn(L) : 0.f;
            o = make_float4(o.x * inv, o.y * inv, o.z * inv, o.w * inv);
            if (stale) {
                const float qn = __int_as_float(0x7fc00000);  // NaN: stale plan must be loud
                o = make_float4(qn, qn, qn, qn);
            } else if (!(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w))) {
                bad1 = true;
            }
            const int j = h * gs + row;
            const bool shard = p.part_o != nullptr;
            reinterpret_cast<float4*>((shard ? p.part_o : p.out) + ((size_t)b * p.m + j) * D)[c4] = o;
            if (c4 == 0) {
                const float lse = (L > 0.f) ? (M + log2f(L)) * kLn2 : -INFINITY;
                if (shard) {
                    p.part_lse[(size_t)b * p.m + j] = lse;
                } else {
                    if (p.lse_out) p.lse_out[(size_t)b * p.m + j] = lse;
                    if (p.emit_logits) p.lse_buf[(size_t)b * p.m + j] = lse;
                }
            }
        }
        if (bad1) set_err(p.err, kDevNumeric);
        if (tid == 0) {
            if (stale) set_err(p.err, kDevUsage);
            if (cap_err) set_err(p.err, kDevCapacity);
            if (s_post <= 0) set_err(p.err, kDevUsage);  // attention over an empty cache
            if (p.fuse_append && !cap_err) atomicAdd(&p.seq_len[p.layer * p.max_batch + b], 1);
        }
        return;
    }
    // 1. push
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
        const uint32_t rbar = mapa_u32(bar_u, (uint32_t)r);
        st_async_v4(mapa_u32(sO_u + (uint32_t)(rank * per + k) * 16u, (uint32_t)r), o, rbar);
        if (c4 == 0 || k == 0) {  // first float4 of this row in owner r's range: r needs (M, L)
            float L = 0.f;
#pragma unroll
            for (int w = 0; w < NW; ++w) L += ls[w * 16 + row] * f[w];
            st_async_v2(mapa_u32(sM_u + (uint32_t)(rank * 16 + row) * 8u, (uint32_t)r), M, L, rbar);
        }
    }
    if (tid == 0) DTRACE(5);
    // 2. owner: 16 lanes per owned float4, lane c holds rank c's partial; max, weights and
    //    sums are fixed shuffle trees over the 16 lanes (deterministic).
    bool bad = false;
    if (mine.n4 > 0) {
        mbar_wait(bar, 0);
        if (tid == 0) DTRACE(7);
        const int grp = tid >> 4, c = tid & 15, ngrp = nthreads >> 4;
        const float2* sML = reinterpret_cast<const float2*>(sM);
        for (int k0 = 0; k0 < per; k0 += ngrp) {
            const int k = k0 + grp;
            const int idx = rank * per + k;
            const bool live = k < per && idx < total;
            const int row = live ? idx / C4 : 0, c4 = live ? idx - row * C4 : 0;
            const bool have = live && c < ns;
            const float2 ml = have ? sML[c * 16 + row] : make_float2(-INFINITY, 0.f);
            const float mc = ml.x, lc = ml.y;
            float4 x = have ? sO[c * per + k] : make_float4(0.f, 0.f, 0.f, 0.f);
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
                const float inv = (L > 0.f) ? __frcp_rn(L) : 0.f;
                float4 o = make_float4(v.x * inv, v.y * inv, v.z * inv, v.w * inv);
                if (stale) {
                    const float qn = __int_as_float(0x7fc00000);  // NaN: stale plan must be loud
                    o = make_float4(qn, qn, qn, qn);
                } else if (!(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w))) {
                    bad = true;
                }
                const int j = h * gs + row;
                const bool shard = p.part_o != nullptr;  // the rank's partial; shard.cu merges the ranks
                reinterpret_cast<float4*>((shard ? p.part_o : p.out) + ((size_t)b * p.m + j) * D)[c4] = o;
                if (c4 == 0) {
                    const float lse = (L > 0.f) ? (M + log2f(L)) * kLn2 : -INFINITY;
                    if (shard) {
                        p.part_lse[(size_t)b * p.m + j] = lse;
                    } else {
                        if (p.lse_out) p.lse_out[(size_t)b * p.m + j] = lse;
                        if (p.emit_logits) p.lse_buf[(size_t)b * p.m + j] = lse;
                    }
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

// Split-K epilogue without a cluster (AttnParams::gmerge), called by every thread of the CTA
// after the warp states are complete in shared memory:
//  1. fold the NW warp states in fixed warp order into this CTA's (M_c, L_c, O_c) (as in
//     cluster_epilogue step 1); with one split the CTA normalises and writes the outputs itself;
//  2. otherwise store the partial to its slot in p.gpart and draw a ticket from the (b, h, ns)
//     counter with one acq_rel atomic (the barrier before it puts every thread's stores in the
//     release); wait until the ns tickets of this launch are drawn (every CTA of a launch is
//     resident or will be: the grid is at most one wave, and nothing it waits on waits on it);
//  3. like the cluster owners, CTA `split` merges its slice of the gs x D outputs from all ns
//     partials in ascending split order (deterministic): one round of loads into shared memory,
//     then M = max_c M_c, w_c = exp2(M_c - M), L = sum_c w_c L_c, O = sum_c w_c O_c / L.
//  Split 0 does the once-per-(b, h) duties (error flags, fused-append counter).
__device__ __forceinline__ int atom_add_acq_rel_gpu(int32_t* a, int v) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(a), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned long long atom_add_acq_rel_gpu_u64(unsigned long long* a, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.u64 %0, [%1], %2;" : "=l"(old) : "l"(a), "l"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire_gpu(const int32_t* a) {
    int v;
    asm volatile("ld.acquire.gpu.s32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int32_t* a, int v) {
    asm volatile("st.release.gpu.s32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

// Low-latency (LL) words of the gmerge partials (AttnParams::gll): every 8-byte word carries
// (value, flag), written by one 8-byte-aligned store (single-copy atomic), so a reader that sees
// the flag of this launch also sees the value — the merging CTAs poll the partials themselves
// instead of drawing a ticket, waiting for the last one and then loading (two global round trips
// fewer on the critical path).  The flag identifies the launch: ((E + 1) << 6) | (ns - 1) with
// E = floor(gcnt[b][h][ns - 1] / ns) read after griddepcontrol.wait (every CTA adds 1 to that
// counter with a fire-and-forget red, so E is the same for all CTAs of a launch whichever has
// already added, and grows by one per launch with this split count).
__device__ __forceinline__ void st_ll2(void* a, float v0, float v1, uint32_t f) {
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(a), "r"(__float_as_uint(v0)), "r"(f),
                 "r"(__float_as_uint(v1)), "r"(f)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_ll2(const void* a) {
    uint4 r;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(a)
                 : "memory");
    return r;
}
__device__ __forceinline__ uint32_t ll_flag(const AttnParams& p, int b, int h, int ns) {
    const unsigned long long* cnt = p.gcnt + ((size_t)b * p.g + h) * kMaxSplitG + (ns - 1);
    unsigned long long c;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(cnt) : "memory");
    return (uint32_t)(((c / (unsigned long long)ns + 1ull) << 6) | (unsigned long long)(ns - 1));
}

template <int D, int NW, int OSROWS>
__device__ __forceinline__ void global_epilogue(const AttnParams& p, const float* ms, const float* ls,
                                                const float* os, float* scratch, int b, int h, int split,
                                                bool stale, bool cap_err, int s_post, uint32_t llf = 0) {
    const int tid = threadIdx.x, nthreads = blockDim.x;
    const int gs = p.gs, ns = p.nsplit;
    constexpr int C4 = D / 4, OS = os_stride<D>();
    const int total = gs * C4;
    const size_t rec = (size_t)gpart_floats(D);
    float* my = p.gpart + (((size_t)b * p.g + h) * ns + split) * rec;
    const bool shard = p.part_o != nullptr;
    bool bad = false;
    auto emit = [&](int row, int c4, float M, float L, float4 v) {
        const float inv = (L > 0.f) ? __frcp_rn(L) : 0.f;
        float4 o = make_float4(v.x * inv, v.y * inv, v.z * inv, v.w * inv);
        if (stale) {
            const float qn = __int_as_float(0x7fc00000);  // NaN: stale plan must be loud
            o = make_float4(qn, qn, qn, qn);
        } else if (!(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w))) {
            bad = true;
        }
        const int j = h * gs + row;
        reinterpret_cast<float4*>((shard ? p.part_o : p.out) + ((size_t)b * p.m + j) * D)[c4] = o;
        if (c4 == 0) {
            const float lse = (L > 0.f) ? (M + log2f(L)) * kLn2 : -INFINITY;
            if (shard) {
                p.part_lse[(size_t)b * p.m + j] = lse;
            } else {
                if (p.lse_out) p.lse_out[(size_t)b * p.m + j] = lse;
                if (p.emit_logits) p.lse_buf[(size_t)b * p.m + j] = lse;
            }
        }
    };
    // 1. this CTA's state
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
        float L = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float f = (M == -INFINITY || mw[w] == -INFINITY) ? 0.f : exp2f(mw[w] - M);
            o.x += f * v[w].x; o.y += f * v[w].y; o.z += f * v[w].z; o.w += f * v[w].w;
            L += ls[w * 16 + row] * f;
        }
        if (ns == 1) {
            emit(row, c4, M, L, o);
        } else if (p.gll) {  // LL words: slot of 2 * gpart_floats words (value, flag)
            uint32_t* w = reinterpret_cast<uint32_t*>(p.gpart) + (((size_t)b * p.g + h) * ns + split) * 2 * rec;
            st_ll2(w + ((size_t)row * D + c4 * 4) * 2, o.x, o.y, llf);
            st_ll2(w + ((size_t)row * D + c4 * 4 + 2) * 2, o.z, o.w, llf);
            if (c4 == 0) st_ll2(w + ((size_t)kMaxGs * D + 2 * row) * 2, M, L, llf);
        } else {
            reinterpret_cast<float4*>(my + (size_t)row * D)[c4] = o;
            if (c4 == 0) reinterpret_cast<float2*>(my + kMaxGs * D)[row] = make_float2(M, L);
        }
    }
    if (ns > 1 && p.gll) {
        // 2'. this launch's ticket (fire and forget: only keeps the epoch counter moving), then
        //     poll this CTA's slice of the ns partials until every word carries this launch's flag
        if (tid == 0) {
            unsigned long long* cnt = p.gcnt + ((size_t)b * p.g + h) * kMaxSplitG + (ns - 1);
            asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");
        }
        const int per = (total + ns - 1) / ns, lo = split * per, n = max(0, min(total, lo + per) - lo);
        const uint32_t* wb = reinterpret_cast<const uint32_t*>(p.gpart) + ((size_t)b * p.g + h) * ns * 2 * rec;
        float4* sx = reinterpret_cast<float4*>(scratch);
        float2* sml = reinterpret_cast<float2*>(sx + per * ns);
        for (int i = tid; i < n * ns; i += nthreads) {
            const int k = i / ns, c = i - k * ns;
            const int idx = lo + k, row = idx / C4, c4 = idx - row * C4;
            const uint32_t* w = wb + (size_t)c * 2 * rec;
            const uint32_t* a0 = w + ((size_t)row * D + c4 * 4) * 2;
            const uint32_t* a2 = w + ((kMaxGs * D) + 2 * row) * 2;
            uint4 x0, x1, y;
            do {
                x0 = ld_ll2(a0);
                x1 = ld_ll2(a0 + 4);
                y = ld_ll2(a2);
            } while (x0.y != llf || x0.w != llf || x1.y != llf || x1.w != llf || y.y != llf || y.w != llf);
            sx[i] = make_float4(__uint_as_float(x0.x), __uint_as_float(x0.z), __uint_as_float(x1.x),
                                __uint_as_float(x1.z));
            sml[i] = make_float2(__uint_as_float(y.x), __uint_as_float(y.z));
        }
        __syncthreads();
        if (tid == 0) DTRACE(9);
    }
    if (ns > 1 && !p.gll) {
        // 2. arrive (ticket on the (b, h, ns) 64-bit counter: launches with this split count
        //    always add exactly ns, so the counter is a multiple of ns between launches) and
        //    wait until all ns tickets of this launch are drawn
        __syncthreads();
        if (tid == 0) DTRACE(5);
        if (tid == 0) {
            unsigned long long* cnt = p.gcnt + ((size_t)b * p.g + h) * kMaxSplitG + (ns - 1);
            const unsigned long long old = atom_add_acq_rel_gpu_u64(cnt, 1ull);
            const unsigned long long target = old - old % (unsigned long long)ns + (unsigned long long)ns;
            if (old + 1 != target) {
                while (ld_acquire_gpu_u64(cnt) < target) {
                }
            }
            DTRACE(7);
        }
        __syncthreads();
        // 3. merge this CTA's slice [lo, lo + n) of the outputs: one round of loads into shared
        //    memory, then one warp per output, split c on lane c (and c - 32), fixed xor trees
        const int per = (total + ns - 1) / ns, lo = split * per, n = max(0, min(total, lo + per) - lo);
        const float* base = p.gpart + ((size_t)b * p.g + h) * ns * rec;
        float4* sx = reinterpret_cast<float4*>(scratch);          // [n][ns] partial O
        float2* sml = reinterpret_cast<float2*>(sx + per * ns);   // [n][ns] (M_c, L_c) of the row
        for (int i = tid; i < n * ns; i += nthreads) {
            const int k = i / ns, c = i - k * ns;
            const int idx = lo + k, row = idx / C4, c4 = idx - row * C4;
            sx[i] = __ldcg(reinterpret_cast<const float4*>(base + c * rec + (size_t)row * D) + c4);
            sml[i] = __ldcg(reinterpret_cast<const float2*>(base + c * rec + kMaxGs * D) + row);
        }
        __syncthreads();
        if (tid == 0) DTRACE(9);
    }
    if (ns > 1) {
        const int per = (total + ns - 1) / ns, lo = split * per, n = max(0, min(total, lo + per) - lo);
        const float4* sx = reinterpret_cast<const float4*>(scratch);
        const float2* sml = reinterpret_cast<const float2*>(sx + per * ns);
        const int lane = tid & 31, warp = tid >> 5, nwarps = nthreads >> 5;
        for (int k = warp; k < n; k += nwarps) {
            const int idx = lo + k, row = idx / C4, c4 = idx - row * C4;
            float2 ml[2];
            float4 x[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int c = lane + 32 * j;
                ml[j] = c < ns ? sml[k * ns + c] : make_float2(-INFINITY, 0.f);
                x[j] = c < ns ? sx[k * ns + c] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            float M = fmaxf(ml[0].x, ml[1].x);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
            float L = 0.f;
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const float f = (M == -INFINITY || ml[j].x == -INFINITY) ? 0.f : exp2f(ml[j].x - M);
                L += f * ml[j].y;
                o.x += f * x[j].x; o.y += f * x[j].y; o.z += f * x[j].z; o.w += f * x[j].w;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                L += __shfl_xor_sync(0xffffffffu, L, off);
                o.x += __shfl_xor_sync(0xffffffffu, o.x, off);
                o.y += __shfl_xor_sync(0xffffffffu, o.y, off);
                o.z += __shfl_xor_sync(0xffffffffu, o.z, off);
                o.w += __shfl_xor_sync(0xffffffffu, o.w, off);
            }
            if (lane == 0) emit(row, c4, M, L, o);
        }
    }
    if (bad) set_err(p.err, kDevNumeric);
    if (split == 0 && tid == 0) {
        if (stale) set_err(p.err, kDevUsage);
        if (cap_err) set_err(p.err, kDevCapacity);
        if (s_post <= 0) set_err(p.err, kDevUsage);  // attention over an empty cache
        // after the wait: every CTA of (b, h) has read the length counter
        if (p.fuse_append && !cap_err) atomicAdd(&p.seq_len[p.layer * p.max_batch + b], 1);
    }
}

}  // namespace delta
