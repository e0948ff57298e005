// attn_tc.cu — bf16 paged decode attention for sm_100a (FULL / SELECT / SPARSE roles).
//
// Eq.4 for one decode query per head, GQA group phi(j) = j / gs (R15),
// over the paged cache of PAPER.md:180-181 (P = 16):
//   a_t = scale * q_j . k_{phi(j),t};  O_j = sum_t softmax(a)_t v_{phi(j),t}
// over all s tokens (FULL, SELECT — R11) or over tokens(rho) of the governing Delta
// layer's plan (SPARSE — PAPER.md:152,158; softmax renormalised over rho, R10).
//
// CTA = (split, kv head h, sequence b); split-K over the sequence (flash-decoding):
//  * warp NCW (producer): streams head-pages (16 tokens x d bf16 = 4 KiB for d=128)
//    of K and V into an NSTAGE-deep shared-memory ring with TMA (2-D tensor map,
//    128-byte swizzle, L2 evict-first) — page mode; or with 16-byte cp.async row
//    gathers tracked by the same mbarriers — token-mode sparse plans.
//  * warps 0..NCW-1 (consumers): each takes one head-page per stage; QK^T and PV on
//    tensor cores with mma.sync m16n8k16 (rows = the gs query heads of the group,
//    padded to 16; K fragments via ldmatrix, V via ldmatrix.trans, conflict-free
//    thanks to the swizzle), online softmax in fp32 registers (exp2 domain).
//    P is fed to PV as bf16 hi + bf16 lo (two MMAs) so probabilities keep ~16
//    mantissa bits (bf16-rounded P breaks the 2e-3 bound).
//  * SELECT additionally writes the scaled logits a_j(t) for the score pass.
//  * fused append (Eq.7): split 0 writes the new K/V row to the pool;
//    the warp whose tile holds token s-1 patches it into shared memory from the input.
//  * end: warps merge (cta_merge), last CTA per (b, h) merges splits (grid_combine).
#include <algorithm>

#include "combine.cuh"

#ifdef DELTA_TRACE
extern "C" int delta_trace_read(void* host, size_t bytes) {  // copies then clears the stamps
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess)
        e = cudaMemcpyFromSymbol(host, g_delta_trace, bytes < sizeof(g_delta_trace) ? bytes : sizeof(g_delta_trace));
    void* dev = nullptr;
    if (e == cudaSuccess) e = cudaGetSymbolAddress(&dev, g_delta_trace);
    if (e == cudaSuccess) e = cudaMemset(dev, 0, sizeof(g_delta_trace));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return (int)e;
}
extern "C" int delta_trace_read_smid(void* host, size_t bytes) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess)
        e = cudaMemcpyFromSymbol(host, g_delta_smid, bytes < sizeof(g_delta_smid) ? bytes : sizeof(g_delta_smid));
    return (int)e;
}
#endif

namespace delta {
namespace {

constexpr int NT = 3;            // tiles per ring stage; a group of NT consumer warps takes a stage
constexpr int kBatch = (32 / NT) * NT;  // tiles whose page ids the producer resolves at once
// Consumer groups NG (ring slot i is always consumed by group i % NG) and ring depth NSTAGE
// (stages of NT tiles; a multiple of NG, so a group consumes the same slots in consecutive
// rounds and its mbarrier parity waits can never alias a round it skipped):
//  * full-cache layers: NG = 2 (6 consumer warps), NSTAGE = 4 (96 KiB in flight) — or 8 with
//    one CTA per SM (deep);
//  (NG = 3 with NSTAGE = 3 — nine warps, one tile each for a sparse layer's ~8 tiles per CTA —
//  measured no faster at C1: the sparse layer is bound by its fixed latencies.)
constexpr int kDeep = 8, kShallow = 4;
template <int NG>
constexpr int cta_threads() { return (NT * NG + 1) * 32; }

template <int D, int NSTAGE>
struct TcCfg {
    static constexpr int kHalf = TileLayout<D>::kVOff;   // K rows -> V rows of a tile
    static constexpr int kTile = TileLayout<D>::kBytes;  // K and V of one (page, head): one TMA request
    static constexpr int kRing = NSTAGE * NT * kTile;
    static constexpr int kRowTok = NSTAGE * NT * kPage;  // token id of every ring row (-1 = none)
    static constexpr int kSmem = 1024 + kRing + ClusterStage<D>::kBytes + 2 * NSTAGE * 8 + kRowTok * 4 + 16;
};

template <int D, bool TOKEN_PLAN, int NSTAGE, int NH, int NG, bool CL>
__global__ void __launch_bounds__(cta_threads<NG>(), (NH == 1 && (CL || NSTAGE == kShallow)) ? 2 : 1)  // two CTAs per SM
attn_tc_kernel(const __grid_constant__ CUtensorMap tm_kv, const AttnParams p) {
    static_assert(NSTAGE % NG == 0, "ring slots must map to fixed consumer groups");
    constexpr int NCW = NT * NG;  // consumer warps; warp NCW is the producer
    constexpr int NGRP = NG;
    using C = TcCfg<D, NSTAGE>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring = base;  // [NSTAGE][NT] tiles of kTile bytes: K rows then V rows
    float* cstage = reinterpret_cast<float*>(ring + C::kRing);  // peers push partials here
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + C::kRing + ClusterStage<D>::kBytes);
    uint64_t* empty = full + NSTAGE;
    int* rowtok = reinterpret_cast<int*>(empty + NSTAGE);  // [NSTAGE][NT][P], written by the producer
    int* sflag = rowtok + C::kRowTok;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;

    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&full[i], 32);  // every producer lane (it wrote row-token entries)
            // every consumer LANE arrives on `empty` (and every producer lane on `full`): each
            // lane reads / writes row-token entries of the stage, so each lane's accesses are
            // ordered by its own release/acquire pair (one arrival per warp after __syncwarp is
            // also correct under the PTX model, but racecheck does not follow the warp barrier)
            mbar_init(&empty[i], NT * 32);
        }
        if (CL) cluster_stage_init<D>(cstage, p.gs);
        fence_mbar_init();
    }
    if (!TOKEN_PLAN && warp == NCW && lane == 0) {
        tma_prefetch_desc(&tm_kv);
    }
    __syncthreads();
    if (CL) cluster_arrive_relaxed();  // peers may push into cstage once they pass the matching wait
    if (tid == 0) DTRACE(0);
    // Programmatic dependent launch: without `prewait` everything waits for the previous
    // kernel here.  With `prewait` (the host knows the previous kernel of this handle wrote
    // neither this layer's length counter nor the plan read here) the geometry and the KV
    // stream start before the wait — the cache rows < s-1, the block table and the plan are
    // then at least two kernels old, hence complete — and only the consumers (q, k_new, v_new,
    // outputs) wait, so the first stages land while the previous layer finishes.
    // the consumers' q rows (read right after the wait): warm L2 and the translation before it
    if (p.q_prefetch && warp == 0 && lane < (p.gs * D * 2 + 127) / 128) {
        const char* qrow = reinterpret_cast<const char*>(p.q) + ((size_t)b * p.m + h * p.gs) * D * 2;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(qrow + lane * 128));
    }
    if (!p.prewait) pdl_wait();
    if (tid == 0) DTRACE(1);

    // ---------------------------------------------------------------- geometry
    // fixed_part: the producer's first block-table entries do not depend on the length, so they
    // are loaded in the same round trip as the length counter (used if the geometry agrees)
    int spec_phys = 0;
    const int spec_u0 = max(0, p.page_lo) + split * fixed_pages(p);
    if (!TOKEN_PLAN && p.fixed_part && p.role != kRoleSparse && warp == NCW && lane < kBatch &&
        spec_u0 + lane < p.bt_stride)
        spec_phys = p.block_table[(size_t)b * p.bt_stride + spec_u0 + lane];
    const int n_old = p.seq_len[p.layer * p.max_batch + b] / p.g;  // raw counter = n * g
    const int s = p.fuse_append ? n_old + 1 : n_old;
    const bool cap_err = s > p.max_seq;
    bool stale = false;
    int n_items = 0, unit0 = 0, e_end = 0;
    if (!cap_err) split_geometry(p, b, split, s, TOKEN_PLAN, unit0, n_items, e_end, stale);
    const int32_t* bt = p.block_table + (size_t)b * p.bt_stride;
    const int32_t* plan = p.plan_idx + (size_t)b * p.plan_cap;
    const int32_t* plan_phys = p.plan_phys + (size_t)b * p.plan_cap;
    const size_t layer_ph = (size_t)p.layer * p.num_phys;
    if (p.prewait && warp != NCW) pdl_wait();
    if (!CL && p.gll && tid == 0) sflag[0] = (int)ll_flag(p, b, h, p.nsplit);  // after the wait (combine.cuh)
    // Every CTA has passed its wait here (the producer never reads upstream outputs), so the
    // previous kernel is complete: let the next layer's kernel launch now — its CTAs co-reside
    // (two per SM), resolve their geometry and start their KV stream during this kernel.
    if (p.early_trigger && warp == 0) pdl_launch_dependents();
    const __nv_bfloat16* k_new = reinterpret_cast<const __nv_bfloat16*>(p.k_new) + ((size_t)b * p.g + h) * D;
    const __nv_bfloat16* v_new = reinterpret_cast<const __nv_bfloat16*>(p.v_new) + ((size_t)b * p.g + h) * D;

    // fused append: split 0 writes the new row of head h to the pool (Eq.7)
    if (p.fuse_append && !cap_err && split == 0 && warp == 0 && owns_page(p, (s - 1) / kPage)) {
        constexpr int kChunks = D / 8;
        const int t = s - 1;
        const size_t krow = kv_row(layer_ph + bt[t / kPage], p.g, h, t % kPage);
        __nv_bfloat16* pool = reinterpret_cast<__nv_bfloat16*>(p.kv_pool);
        if (lane < kChunks) {
            reinterpret_cast<uint4*>(pool + krow * D)[lane] = reinterpret_cast<const uint4*>(k_new)[lane];
        } else if (lane < 2 * kChunks) {
            reinterpret_cast<uint4*>(pool + (krow + kPage) * D)[lane - kChunks] =
                reinterpret_cast<const uint4*>(v_new)[lane - kChunks];
        }
    }

    // warp states for the epilogue live in the ring once every consumer is done with it
    float* ms = reinterpret_cast<float*>(ring);
    float* ls = ms + NCW * 16;
    float* os = ls + NCW * 16;
    constexpr int OSR = 8 * NH;  // O rows kept per warp (the group's heads, gs <= 8 * NH)
    static_assert((2 * NCW * 16 + NCW * OSR * os_stride<D>()) * 4 <= TcCfg<D, NSTAGE>::kRing,
                  "epilogue state must fit in the K ring");
    // global-merge scratch (weights, L_c, merged M/L) in the ring past the warp states
    constexpr int kMergeScratch = 2 * NCW * 16 + NCW * OSR * os_stride<D>();
    // (n outputs of the slice x ns partials, float4 O + float2 (M, L) each; n * ns <= total + ns)
    static_assert(CL || (kMergeScratch + 6 * (kMaxGs * D / 4 + kMaxSplitG) + 64) * 4 <= TcCfg<D, NSTAGE>::kRing,
                  "merge scratch must fit in the ring");

    if (warp == NCW) {
        // ============================================================ producer
        // The whole warp resolves up to 32 tiles' page ids (or 64 rows' token ids) with
        // independent loads, so the dependent plan -> block-table -> copy chain costs two
        // L2 round trips per batch rather than per tile.  The token id of every ring row is
        // handed to the consumers through shared memory (published by the stage barrier).
        if (!TOKEN_PLAN) {
            // page ids of one batch of tiles (lane i: tile base + i)
            auto resolve = [&](int base, int& lp, int& phys) {
                lp = -1;
                phys = 0;
                if (lane < kBatch && base + lane < n_items) {
                    if (p.role == kRoleSparse) {  // logical and physical page: independent loads
                        lp = plan[unit0 + base + lane];
                        phys = plan_phys[unit0 + base + lane];
                    } else {
                        lp = unit0 + base + lane;
                        phys = bt[lp];
                    }
                }
            };
            int my_lp, my_phys;
            if (p.fixed_part && p.role != kRoleSparse && unit0 == spec_u0) {  // the speculative entries
                my_lp = (lane < kBatch && lane < n_items) ? unit0 + lane : -1;
                my_phys = my_lp >= 0 ? spec_phys : 0;
            } else {
                resolve(0, my_lp, my_phys);
            }
            for (int base = 0; base < n_items; base += kBatch) {
                if (base > 0) resolve(base, my_lp, my_phys);
                const int nb = min(kBatch, n_items - base);
                for (int j = 0; j < nb; j += NT) {
                    const int iter = (base + j) / NT;
                    const int stg = iter % NSTAGE, round = iter / NSTAGE;
                    if (round > 0) mbar_wait(&empty[stg], (round - 1) & 1);
                    const int valid = min(NT, nb - j);
#pragma unroll
                    for (int k = 0; k < (NT * kPage + 31) / 32; ++k) {
                        const int rr = lane + 32 * k, w = rr / kPage, r = rr % kPage;
                        const int lp_w = __shfl_sync(0xffffffffu, my_lp, min(j + w, 31));
                        int t = -1;
                        if (w < valid) {
                            t = lp_w * kPage + r;
                            if (t >= s) t = -1;
                        }
                        if (rr < NT * kPage) rowtok[(stg * NT + w) * kPage + r] = t;
                    }
                    const int phys_w = __shfl_sync(0xffffffffu, my_phys, j + (lane % NT));
                    __syncwarp();
                    if (lane == 0) mbar_arrive_expect_tx(&full[stg], valid * C::kTile);
                    else mbar_arrive(&full[stg]);
                    __syncwarp();
                    if (lane < valid) {  // one 2P-row box: this head's K and V rows of the page
                        const int row0 = (int)kv_row(layer_ph + phys_w, p.g, h, 0);
                        uint8_t* dst = ring + (stg * NT + lane) * C::kTile;
                        if (D == 64) tma_load_2d(dst, &tm_kv, &full[stg], 0, row0, kEvictFirst);
                        else tma_load_3d(dst, &tm_kv, &full[stg], 0, row0, 0, kEvictFirst);
                    }
                }
            }
        } else {
            const __nv_bfloat16* pool = reinterpret_cast<const __nv_bfloat16*>(p.kv_pool);
            constexpr int kChunks = D / 8;
            constexpr int kRowsPerStage = NT * kPage;
            constexpr int kRowIt = (kRowsPerStage + 31) / 32;  // rows per lane
            for (int it = 0, iter = 0; it < n_items; it += NT, ++iter) {
                const int stg = iter % NSTAGE, round = iter / NSTAGE;
                // resolve the stage's rows: lane owns rows lane + 32k (token -> pool row)
                long long my_row[kRowIt];
                int my_t[kRowIt];
#pragma unroll
                for (int k = 0; k < kRowIt; ++k) {  // token and its physical slot: independent loads
                    const int rr = lane + 32 * k, w = rr / kPage, r = rr % kPage;
                    const int e = unit0 + (it + w) * kPage + r;
                    const bool ok = rr < kRowsPerStage && it + w < n_items && e < e_end;
                    my_t[k] = ok ? plan[e] : -1;
                    const int ps = ok ? plan_phys[e] : 0;  // phys_page * P + slot
                    my_row[k] = ok ? (long long)kv_row(layer_ph + ps / kPage, p.g, h, ps % kPage) : -1ll;
                }
                if (round > 0) mbar_wait(&empty[stg], (round - 1) & 1);
#pragma unroll
                for (int k = 0; k < kRowIt; ++k)
                    if (lane + 32 * k < kRowsPerStage) rowtok[stg * kRowsPerStage + lane + 32 * k] = my_t[k];
                for (int w = 0; w < NT; ++w) {
                    if (it + w >= n_items) break;
                    uint8_t* kd = ring + (stg * NT + w) * C::kTile;
                    uint8_t* vd = kd + C::kHalf;
                    for (int ci = lane; ci < kPage * kChunks; ci += 32) {
                        const int r = ci / kChunks, c = ci - r * kChunks;
                        const int rr = w * kPage + r;
                        long long row = -1;
#pragma unroll
                        for (int k = 0; k < kRowIt; ++k) {
                            const long long x = __shfl_sync(0xffffffffu, my_row[k], rr & 31);
                            if ((rr >> 5) == k) row = x;
                        }
                        if (row >= 0) {
                            cp_async16(kd + swz<D>(r, c), pool + row * D + c * 8);
                            cp_async16(vd + swz<D>(r, c), pool + (row + kPage) * D + c * 8);
                        }
                    }
                }
                cp_async_mbar_arrive_noinc(&full[stg]);
            }
        }
    } else {
        // ============================================================ consumers
        // "Swapped" GQA tile: tokens are the MMA M dimension and the group's query heads the
        // N dimension (NH tiles of 8), so no MMA row is spent on padding heads:
        //   S^T[16 tok x 8 heads] = K[16 x D] . Q^T[D x 8]          (D/16 MMAs)
        //   O^T[D x 8 heads]     += V^T[D x 16 tok] . P^T[16 x 8]   (2 x D/16 MMAs: P hi + lo)
        // The S^T accumulator becomes the P^T operand with two movmatrix transposes per half.
        // Lane (g4 = lane/4, t4 = lane%4) owns heads 2*t4, 2*t4+1 of each head tile, tokens g4
        // and g4+8 of S^T, and rows d = 16*mt + g4 (+8) of O^T.
        // NH = head tiles of 8 (1: gs <= 8, 2: gs <= 16); tiles past gs are skipped
        const int g4 = lane >> 2, t4 = lane & 3;
        const int gs = p.gs;
        const int nh_used = (gs + 7) / 8;
        // Q^T fragments (B operand): qb[nh][kc] = Q[head nh*8+g4][16kc + 2t4 (+1)], [.. + 8 (+9)]
        uint32_t qb[NH][D / 16][2];
        {
            const __nv_bfloat16* qp = reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)b * p.m + h * gs) * D;
#pragma unroll
            for (int nh = 0; nh < NH; ++nh) {
                const int hq = nh * 8 + g4;
                const uint32_t* qr = reinterpret_cast<const uint32_t*>(qp + (size_t)hq * D);
#pragma unroll
                for (int kc = 0; kc < D / 16; ++kc) {
                    qb[nh][kc][0] = hq < gs ? qr[(kc * 16 + 2 * t4) >> 1] : 0u;
                    qb[nh][kc][1] = hq < gs ? qr[(kc * 16 + 2 * t4 + 8) >> 1] : 0u;
                }
            }
        }
        float o[NH][D / 16][4];
        float mh[NH][2], lh[NH][2];
#pragma unroll
        for (int nh = 0; nh < NH; ++nh) {
            mh[nh][0] = mh[nh][1] = -INFINITY;
            lh[nh][0] = lh[nh][1] = 0.f;
#pragma unroll
            for (int mt = 0; mt < D / 16; ++mt) o[nh][mt][0] = o[nh][mt][1] = o[nh][mt][2] = o[nh][mt][3] = 0.f;
        }
        const float sl2 = p.scale_log2;

        const int grp = warp / NT, wt = warp % NT;  // consumer group, tile within the stage
        for (int iter = grp; iter * NT < n_items; iter += NGRP) {
            const int it = iter * NT;
            const int stg = iter % NSTAGE, round = iter / NSTAGE;
            mbar_wait(&full[stg], round & 1);
            if (iter == 0 && tid == 0) DTRACE(2);
            const int item = it + wt;
            if (item < n_items) {
                uint8_t* kt = ring + (stg * NT + wt) * C::kTile;
                uint8_t* vt = kt + C::kHalf;
                const int* rt = rowtok + (stg * NT + wt) * kPage;
                const int my_tok = (lane < kPage) ? rt[lane] : -1;  // token of ring row `lane`
                const int tok0 = rt[g4], tok1 = rt[g4 + 8];         // tokens of this lane's S^T rows
                // fused append: patch row holding token s-1 from the inputs
                if (p.fuse_append) {
                    const unsigned pm = __ballot_sync(0xffffffffu, my_tok == s - 1);
                    if (pm) {
                        const int r = __ffs(pm) - 1;
                        constexpr int kChunks = D / 8;
                        if (lane < kChunks)
                            *reinterpret_cast<uint4*>(kt + swz<D>(r, lane)) = reinterpret_cast<const uint4*>(k_new)[lane];
                        else if (lane < 2 * kChunks)
                            *reinterpret_cast<uint4*>(vt + swz<D>(r, lane - kChunks)) =
                                reinterpret_cast<const uint4*>(v_new)[lane - kChunks];
                    }
                }
                // rows without a token: zero V (0 * garbage must not produce NaN)
                bool wrote_smem = p.fuse_append != 0;
                {
                    unsigned inval = __ballot_sync(0xffffffffu, lane < 16 && my_tok < 0);
                    wrote_smem |= inval != 0;
                    while (inval) {
                        const int r = __ffs(inval) - 1;
                        inval &= inval - 1;
                        if (lane < D / 8) *reinterpret_cast<uint4*>(vt + swz<D>(r, lane)) = make_uint4(0, 0, 0, 0);
                    }
                }
                __syncwarp();
                const uint32_t kt_u = smem_u32(kt), vt_u = smem_u32(vt);
#ifndef EXP_TCNOMATH  // experiment builds: consumers skip the tile math (stream-only timing)
                {
                // ---- S^T = K Q^T: two accumulator chains (even / odd k-chunks)
                float acc[NH][4], acc2[NH][4];
#pragma unroll
                for (int nh = 0; nh < NH; ++nh)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[nh][i] = acc2[nh][i] = 0.f;
#pragma unroll
                for (int kc = 0; kc < D / 16; ++kc) {
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4(kt_u + swz<D>((lane & 7) + 8 * ((lane >> 3) & 1), kc * 2 + (lane >> 4)), a0, a1, a2, a3);
                    const uint32_t af[4] = {a0, a1, a2, a3};
#pragma unroll
                    for (int nh = 0; nh < NH; ++nh) {
                        if (nh < nh_used) {
                            if (kc & 1) mma_bf16_16816(acc2[nh], af, qb[nh][kc][0], qb[nh][kc][1]);
                            else mma_bf16_16816(acc[nh], af, qb[nh][kc][0], qb[nh][kc][1]);
                        }
                    }
                }
                uint32_t bhi[NH][2], blo[NH][2];
#pragma unroll
                for (int nh = 0; nh < NH; ++nh) {
                    if (nh >= nh_used) continue;
                    float c[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) c[i] = acc[nh][i] + acc2[nh][i];
                    // c[0],c[1]: token tok0, heads 2t4, 2t4+1; c[2],c[3]: token tok1
                    if (p.emit_logits) {
                        float* lg = p.logits + (size_t)b * p.max_seq * p.m + h * gs;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int hq = nh * 8 + 2 * t4 + (i & 1);
                            const int t = (i < 2) ? tok0 : tok1;
                            if (hq < gs && t >= 0) lg[(size_t)t * p.m + hq] = c[i] * p.scale;
                        }
                    }
                    // ---- softmax per head column (log2 domain) with a lazily raised stabiliser:
                    // p = exp2(x - m) for ANY m gives the same normalised softmax (the
                    // epilogue divides by the same sums), so m is only moved -- with the
                    // cross-lane max and the rescale of O -- when a logit exceeds it by more
                    // than kHeadroom (p then stays <= 2^kHeadroom, far inside fp32/bf16
                    // range; logits far below m underflow only below 2^-126 relative).
                    // The first valid tile of a warp always sets m.  Deterministic: m depends
                    // only on the data, in a fixed order.
                    constexpr float kHeadroom = 16.f;
                    float x[4];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        x[e] = tok0 >= 0 ? c[e] * sl2 : -INFINITY;
                        x[2 + e] = tok1 >= 0 ? c[2 + e] * sl2 : -INFINITY;
                    }
                    const bool raise = fmaxf(x[0], x[2]) > mh[nh][0] + kHeadroom ||
                                       fmaxf(x[1], x[3]) > mh[nh][1] + kHeadroom;
                    if (__any_sync(0xffffffffu, raise)) {  // rare after the first tile
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            float mx = fmaxf(x[e], x[2 + e]);
                            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
                            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
                            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
                            const float mn = fmaxf(mh[nh][e], mx);
                            if (mn > mh[nh][e]) {
                                const float al = ex2(mh[nh][e] - mn);  // mh = -inf -> 0
                                lh[nh][e] *= al;
#pragma unroll
                                for (int mt = 0; mt < D / 16; ++mt) {
                                    o[nh][mt][e] *= al;
                                    o[nh][mt][2 + e] *= al;
                                }
                                mh[nh][e] = mn;
                            }
                        }
                    }
                    float pr[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {  // x = -inf -> 0 (m = -inf only while every x is -inf)
                        const float m = mh[nh][i & 1];
                        pr[i] = ex2(x[i] - (m == -INFINITY ? 0.f : m));
                    }
                    lh[nh][0] += pr[0] + pr[2];
                    lh[nh][1] += pr[1] + pr[3];
                    // ---- P^T operand: bf16 hi + lo (P keeps ~16 mantissa bits), transposed
                    const __nv_bfloat162 h01 = __floats2bfloat162_rn(pr[0], pr[1]);
                    const __nv_bfloat162 h23 = __floats2bfloat162_rn(pr[2], pr[3]);
                    const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
                    bhi[nh][0] = movmatrix_trans(*reinterpret_cast<const uint32_t*>(&h01));
                    bhi[nh][1] = movmatrix_trans(*reinterpret_cast<const uint32_t*>(&h23));
                    blo[nh][0] = movmatrix_trans(pack_bf16(pr[0] - f01.x, pr[1] - f01.y));
                    blo[nh][1] = movmatrix_trans(pack_bf16(pr[2] - f23.x, pr[3] - f23.y));
                }
                // ---- O^T += V^T P^T
                constexpr int kPvTiles = D / 16;
#pragma unroll
                for (int mt = 0; mt < kPvTiles; ++mt) {
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4_t(vt_u + swz<D>((lane & 7) + 8 * (lane >> 4), mt * 2 + ((lane >> 3) & 1)), a0, a1, a2, a3);
                    const uint32_t af[4] = {a0, a1, a2, a3};
#pragma unroll
                    for (int nh = 0; nh < NH; ++nh) {
                        if (nh < nh_used) {
                            mma_bf16_16816(o[nh][mt], af, bhi[nh][0], bhi[nh][1]);
                            mma_bf16_16816(o[nh][mt], af, blo[nh][0], blo[nh][1]);
                        }
                    }
                }
                }
#else
                (void)kt_u; (void)vt_u;
#endif
                // generic-proxy smem writes must be ordered before the next TMA refill
                if (wrote_smem) fence_proxy_async_smem();
            }
            mbar_arrive(&empty[stg]);
        }

        // ---------------------------------------------------------------- warp states
        if (tid == 0) DTRACE(3);
        if (tid == (NCW - 1) * 32) DTRACE(11);
        consumer_bar(NCW * 32);  // every consumer is done reading the ring
        if (tid == 0) DTRACE(8);
#pragma unroll
        for (int nh = 0; nh < NH; ++nh) {
            if (nh >= nh_used) continue;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                float l = lh[nh][e];  // column sum over the 8 token-row groups
                l += __shfl_xor_sync(0xffffffffu, l, 4);
                l += __shfl_xor_sync(0xffffffffu, l, 8);
                l += __shfl_xor_sync(0xffffffffu, l, 16);
                const int hq = nh * 8 + 2 * t4 + e;
                if (g4 == 0 && hq < gs) {
                    ms[warp * 16 + hq] = mh[nh][e];
                    ls[warp * 16 + hq] = l;
                }
            }
#pragma unroll
            for (int mt = 0; mt < D / 16; ++mt)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int hq = nh * 8 + 2 * t4 + (i & 1);
                    const int dd = mt * 16 + g4 + 8 * (i >> 1);
                    if (hq < gs) os[(warp * OSR + hq) * os_stride<D>() + dd] = o[nh][mt][i];
                }
        }
    }
    if (tid == 0) DTRACE(10);
    __syncthreads();  // producer joins: warp states complete
    if (!p.early_trigger) pdl_launch_dependents();
    if (tid == 0) DTRACE(4);
    if (CL) cluster_epilogue<D, NCW, OSR>(p, ms, ls, os, cstage, b, h, stale, cap_err, s);
    else global_epilogue<D, NCW, OSR>(p, ms, ls, os, reinterpret_cast<float*>(ring) + kMergeScratch, b, h, split,
                                       stale, cap_err, s, (uint32_t)sflag[0]);
    if (tid == 0) DTRACE(6);
}

template <int D, bool TOKEN_PLAN, int NST, int NH, int NG, bool CL = true>
cudaError_t launch_impl(const AttnParams& p0, const CUtensorMap* tm_kv,
                        cudaStream_t st, bool pdl) {
    auto kern = attn_tc_kernel<D, TOKEN_PLAN, NST, NH, NG, CL>;
    constexpr int kThreads = cta_threads<NG>();
    constexpr int smem = TcCfg<D, NST>::kSmem;
    // largest feasible cluster for this instantiation, per device (attribute opt-ins are per context)
    static std::atomic<int> cache[kMaxDevices];
    const int max_cluster = per_device_once(cache, [&] {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
            (CL && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess))
            return -1;
        return CL ? cluster_limit((const void*)kern, kThreads, smem) : kMaxSplitG;
    });
    if (max_cluster < 1) return cudaErrorInvalidConfiguration;
    AttnParams p = p0;
    p.nsplit = std::min(p.nsplit, max_cluster);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.nsplit, p.g, p.batch);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[3];
    int na = 0;
    if (CL) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = p.nsplit;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (CL && p.cluster_policy) {
        attr[na].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
        attr[na].val.clusterSchedulingPolicyPreference = (cudaClusterSchedulingPolicy)p.cluster_policy;
        ++na;
    }
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, *tm_kv, p);
}

// Global-merge variant: one CTA per SM, nine consumer warps (a sparse layer's ~8 tiles per CTA
// in one round), six ring stages of three tiles (144 KiB in flight per SM).
constexpr int kGStage = 6, kGGroups = 3;

template <int D, bool TOKEN_PLAN>
cudaError_t launch_stages(const AttnParams& p, const CUtensorMap* tm_kv, cudaStream_t st,
                          bool pdl) {
    if (p.gmerge && p.gm_shallow && p.gs <= 8) return launch_impl<D, TOKEN_PLAN, kShallow, 1, 2, false>(p, tm_kv, st, pdl);
    if (p.gmerge)
        return p.gs <= 8 ? launch_impl<D, TOKEN_PLAN, kGStage, 1, kGGroups, false>(p, tm_kv, st, pdl)
                         : launch_impl<D, TOKEN_PLAN, kGStage, 2, kGGroups, false>(p, tm_kv, st, pdl);
    if (p.gs <= 8)
        return p.deep ? launch_impl<D, TOKEN_PLAN, kDeep, 1, 2>(p, tm_kv, st, pdl)
                      : launch_impl<D, TOKEN_PLAN, kShallow, 1, 2>(p, tm_kv, st, pdl);
    return p.deep ? launch_impl<D, TOKEN_PLAN, kDeep, 2, 2>(p, tm_kv, st, pdl)
                  : launch_impl<D, TOKEN_PLAN, kShallow, 2, 2>(p, tm_kv, st, pdl);
}

}  // namespace

#ifdef DELTA_TRACE
// trace builds: max co-resident clusters of the real kernel for a cluster size
extern "C" int delta_debug_cluster_occupancy(int deep, int cs) {
    auto kern = deep ? attn_tc_kernel<128, false, kDeep, 1, 2, true> : attn_tc_kernel<128, false, kShallow, 1, 2, true>;
    const int smem = deep ? TcCfg<128, kDeep>::kSmem : TcCfg<128, kShallow>::kSmem;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 8, 1);
    cfg.blockDim = dim3(cta_threads<2>());
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a;
    a.id = cudaLaunchAttributeClusterDimension;
    a.val.clusterDim.x = cs; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
    cfg.attrs = &a; cfg.numAttrs = 1;
    int n = -1;
    if (cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &cfg) != cudaSuccess) { cudaGetLastError(); return -2; }
    return n;
}
#endif

cudaError_t launch_attn_tc(const AttnParams& p, const CUtensorMap* tm_kv,
                           cudaStream_t st, bool pdl) {
    const bool tok = (p.role == kRoleSparse) && p.sel_block == 1;
    if (p.d == 128)
        return tok ? launch_stages<128, true>(p, tm_kv, st, pdl) : launch_stages<128, false>(p, tm_kv, st, pdl);
    if (p.d == 64)
        return tok ? launch_stages<64, true>(p, tm_kv, st, pdl) : launch_stages<64, false>(p, tm_kv, st, pdl);
    return cudaErrorInvalidValue;
}

}  // namespace delta
