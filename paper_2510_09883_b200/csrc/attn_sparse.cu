// attn_sparse.cu — latency-specialised SPARSE decode for small batches (sparse layers of
// Eq.4 over tokens(rho) of the governing Delta layer's page plan, softmax
// renormalised over rho, R10).
//
// At batch 1 a sparse layer moves ~8.6 MB (C1), 1.3 us of HBM time, so its cost is latency:
// the dependency release of the previous layer, the q load, the tile math and the split-K
// merge.  Measured on B200 (tools/latency_floor.cu, a chain of 100 PDL kernels in a graph):
// an empty kernel costs 0.45-0.66 us, + a dependent q load 1.0 us; a split-K merge through
// global memory (acq_rel ticket + spin, or LL flags) 2.3-4.6 us; through distributed shared
// memory (st.async into the owner CTA, mbarrier complete_tx) 1.5 us — and only 1.0 us less
// when consecutive kernels' CTAs cannot co-reside (one CTA per SM).  Hence:
//  * the CTAs of one (sequence, kv head) form a thread-block cluster; the split partials are
//    merged in DSMEM (combine.cuh cluster_epilogue: push model, fixed rank order);
//  * every tile of the CTA's share of the plan is resident at once (no ring reuse, one
//    mbarrier per tile), and <= 112 KiB of shared memory + 8 warps keep two CTAs per SM, so
//    the next layer's CTAs launch during this one (PDL early trigger) and, with `prewait`,
//    their whole KV share lands before griddepcontrol.wait returns — the plan and the cache
//    rows are >= two kernels old, the appended row is patched from the input after the wait;
//  * all 8 warps consume (the TMA requests are issued by warp 0 in the prologue).
// Math per 16-token tile: the swapped GQA tile of attn_tc.cu (S^T = K Q^T, P^T split into
// bf16 hi + lo for O^T += V^T P^T; fp32 online softmax with the lazily raised stabiliser).
#include <algorithm>

#include "combine.cuh"

#ifdef DELTA_TRACE
// per-warp %globaltimer stamps of the latest launch of each layer: [layer][cta][warp][event]
static __device__ unsigned long long g_sp_trace[64 * 128 * 8 * 16];
extern "C" int delta_trace_read_sparse(void* host, size_t bytes) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess)
        e = cudaMemcpyFromSymbol(host, g_sp_trace, bytes < sizeof(g_sp_trace) ? bytes : sizeof(g_sp_trace));
    void* dev = nullptr;
    if (e == cudaSuccess) e = cudaGetSymbolAddress(&dev, g_sp_trace);
    if (e == cudaSuccess) e = cudaMemset(dev, 0, sizeof(g_sp_trace));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return (int)e;
}
#define SPTRACE(ev)                                                                                 \
    do {                                                                                            \
        const int cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);           \
        if (lane == 0 && cta_ < 128 && p.layer < 64) {                                              \
            unsigned long long t_;                                                                  \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
            g_sp_trace[((p.layer * 128 + cta_) * 8 + warp) * 16 + (ev)] = t_;                       \
        }                                                                                           \
    } while (0)
// SM clock (cycles) of the warp at an epilogue point (events 7..11, 14, 15)
#define SPCLK(ev)                                                                                   \
    do {                                                                                            \
        const int cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);           \
        if (lane == 0 && cta_ < 128 && p.layer < 64)                                                \
            g_sp_trace[((p.layer * 128 + cta_) * 8 + warp) * 16 + (ev)] = clock64();                \
    } while (0)
#else
#define SPTRACE(ev) do {} while (0)
#define SPCLK(ev) do {} while (0)
#endif

namespace delta {
namespace {

constexpr int kSpWarps = 8;      // all consumers
constexpr int kSpMaxTiles = 12;  // resident (page, head) tiles per CTA: 96 KiB at d = 128

template <int D>
constexpr int sp_smem() {
    return 1024 + kSpMaxTiles * TileLayout<D>::kBytes + ClusterStage<D>::kBytes + kSpMaxTiles * 8 + kSpMaxTiles * 4 + 16;
}

// One group of NT (1 or 2) resident (page, head) tiles of a warp, processed together so their
// MMA chains interleave: the swapped GQA tile of attn_tc.cu — S^T[16 tok x 8 heads] = K Q^T,
// O^T[D x 8] += V^T P^T with P^T as bf16 hi + lo (~16-bit probabilities).
// Lane (g4, t4) owns tokens g4, g4 + 8 of each tile and heads 2 t4, 2 t4 + 1 (its "columns").
// Stabiliser mh (log2 units) starts at 0 and only moves when needed, decided with ballots
// instead of cross-lane max shuffles on every tile:
//  * raise: a logit exceeds mh + 16 in the column -> mh = column max, rescale o, l (p <= 2^16);
//  * rebase: a column with tokens has no positive probability yet (every logit so far more than
//    ~126 below mh, only possible for extreme logits) -> mh = column max (o, l are still 0).
// p = exp2(x - mh) for any mh gives the same normalised softmax (the epilogue divides by the
// same sums), so the output is Eq.4 whatever mh is; mh depends only on the data (deterministic).
template <int D, int NT>
__device__ __forceinline__ void sp_tiles(const uint32_t (&ku)[NT], const uint32_t (&vu)[NT], const int (&nv)[NT],
                                         const uint32_t (&qb)[D / 16][2], float (&o)[D / 16][4], float (&mh)[2],
                                         float (&lh)[2], float sl2, int lane) {
    constexpr int CH = 4 / NT;  // independent accumulator chains per tile
    const int g4 = lane >> 2, t4 = lane & 3;
    float acc[NT][CH][4];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[t][c][0] = acc[t][c][1] = acc[t][c][2] = acc[t][c][3] = 0.f;
#pragma unroll
    for (int kc = 0; kc < D / 16; ++kc)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4(ku[t] + swz<D>((lane & 7) + 8 * ((lane >> 3) & 1), kc * 2 + (lane >> 4)), a0, a1, a2, a3);
            const uint32_t af[4] = {a0, a1, a2, a3};
            mma_bf16_16816(acc[t][kc % CH], af, qb[kc][0], qb[kc][1]);
        }
    float x[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float v = acc[t][0][i];
#pragma unroll
            for (int c = 1; c < CH; ++c) v += acc[t][c][i];
            x[t][i] = ((i < 2 ? g4 : g4 + 8) < nv[t]) ? v * sl2 : -INFINITY;
        }
    auto colmax = [&](int e) {
        float mx = -INFINITY;
#pragma unroll
        for (int t = 0; t < NT; ++t) mx = fmaxf(mx, fmaxf(x[t][e], x[t][2 + e]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        return mx;
    };
    constexpr float kHeadroom = 16.f;
    bool up = false;
#pragma unroll
    for (int t = 0; t < NT; ++t)
        up |= fmaxf(x[t][0], x[t][2]) > mh[0] + kHeadroom || fmaxf(x[t][1], x[t][3]) > mh[1] + kHeadroom;
    if (__ballot_sync(0xffffffffu, up)) {  // rare: raise the stabiliser of the columns that need it
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const float mn = fmaxf(mh[e], colmax(e));
            if (mn > mh[e] + kHeadroom) {
                const float al = ex2(mh[e] - mn);
                lh[e] *= al;
#pragma unroll
                for (int mt = 0; mt < D / 16; ++mt) {
                    o[mt][e] *= al;
                    o[mt][2 + e] *= al;
                }
                mh[e] = mn;
            }
        }
    }
    float pr[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int i = 0; i < 4; ++i) pr[t][i] = ex2(x[t][i] - mh[i & 1]);
    {
        bool pos0 = lh[0] > 0.f, pos1 = lh[1] > 0.f, tok = false;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            pos0 |= pr[t][0] > 0.f || pr[t][2] > 0.f;
            pos1 |= pr[t][1] > 0.f || pr[t][3] > 0.f;
            tok |= nv[t] > 0;
        }
        const unsigned col = 0x11111111u << t4;
        const unsigned b0 = __ballot_sync(0xffffffffu, pos0), b1 = __ballot_sync(0xffffffffu, pos1);
        const bool dead0 = tok && (b0 & col) == 0, dead1 = tok && (b1 & col) == 0;
        if (__any_sync(0xffffffffu, dead0 || dead1)) {  // rare: rebase the dead columns
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float mx = colmax(e);
                if ((e == 0 ? dead0 : dead1) && mx > -INFINITY) {
                    mh[e] = mx;
#pragma unroll
                    for (int t = 0; t < NT; ++t) {
                        pr[t][e] = ex2(x[t][e] - mx);
                        pr[t][2 + e] = ex2(x[t][2 + e] - mx);
                    }
                }
            }
        }
    }
    uint32_t bhi[NT][2], blo[NT][2];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        lh[0] += pr[t][0] + pr[t][2];
        lh[1] += pr[t][1] + pr[t][3];
        const __nv_bfloat162 h01 = __floats2bfloat162_rn(pr[t][0], pr[t][1]);
        const __nv_bfloat162 h23 = __floats2bfloat162_rn(pr[t][2], pr[t][3]);
        const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
        bhi[t][0] = movmatrix_trans(*reinterpret_cast<const uint32_t*>(&h01));
        bhi[t][1] = movmatrix_trans(*reinterpret_cast<const uint32_t*>(&h23));
        blo[t][0] = movmatrix_trans(pack_bf16(pr[t][0] - f01.x, pr[t][1] - f01.y));
        blo[t][1] = movmatrix_trans(pack_bf16(pr[t][2] - f23.x, pr[t][3] - f23.y));
    }
#pragma unroll
    for (int mt = 0; mt < D / 16; ++mt)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4_t(vu[t] + swz<D>((lane & 7) + 8 * (lane >> 4), mt * 2 + ((lane >> 3) & 1)), a0, a1, a2, a3);
            const uint32_t af[4] = {a0, a1, a2, a3};
            mma_bf16_16816(o[mt], af, bhi[t][0], bhi[t][1]);
            mma_bf16_16816(o[mt], af, blo[t][0], blo[t][1]);
        }
}

// Split-K merge of one (sequence, kv head) across its cluster (push model, as combine.cuh's
// cluster_epilogue, with the owner merge done per output float4 by one thread looping over the
// ranks in ascending order — no shuffle trees on the critical path):
//  1. thread idx < gs * D/4 folds the NW warp states of its float4 (fixed warp order) into this
//     CTA's (M_c, L_c, O_c) and st.async-stores it into the owner's staging (DSMEM, completes
//     bytes on the owner's mbarrier; the first float4 of a row in an owner's range also sends
//     the row's (M_c, L_c));
//  2. the owner waits on its own mbarrier, then M = max_c M_c, w_c = 2^(M_c - M),
//     O = sum_c w_c O_c / sum_c w_c L_c, LSE = (M + log2 L) ln 2 — Eq.4's softmax over the
//     union of the splits' token sets; deterministic (fixed orders).
template <int D, int NW, int OSROWS>
__device__ __forceinline__ void sp_epilogue(const AttnParams& p, const float* ms, const float* ls, const float* os,
                                            float* stage, int b, int h, bool stale, bool cap_err, int s_post,
                                            int warp, int lane) {
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
    const bool shard = p.part_o != nullptr;
    bool bad = false;
    auto emit = [&](int row, int c4, float M, float L, float4 v) {
        const float inv = (L > 0.f) ? __frcp_rn(L) : 0.f;
        float4 o = make_float4(v.x * inv, v.y * inv, v.z * inv, v.w * inv);
        if (stale) {
            const float qn = __int_as_float(0x7fc00000);  // NaN: a stale plan must be loud
            o = make_float4(qn, qn, qn, qn);
        } else if (!(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w))) {
            bad = true;
        }
        const int j = h * gs + row;
        reinterpret_cast<float4*>((shard ? p.part_o : p.out) + ((size_t)b * p.m + j) * D)[c4] = o;
        if (c4 == 0) {
            const float lse = (L > 0.f) ? (M + log2f(L)) * kLn2 : -INFINITY;
            if (shard) p.part_lse[(size_t)b * p.m + j] = lse;
            else if (p.lse_out) p.lse_out[(size_t)b * p.m + j] = lse;
        }
    };
    // (the kernel passed barrier.cluster.wait after issuing its q loads: peers' barriers are live)
    // 1. fold + push (or, with one split, emit)
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
            const float f = ex2(mw[w] - M);  // warp stabilisers are finite
            o.x += f * v[w].x; o.y += f * v[w].y; o.z += f * v[w].z; o.w += f * v[w].w;
            L += f * ls[w * 16 + row];
        }
#ifdef EXP_NOEPI
        if (true) {
#else
        if (ns == 1) {
#endif
            emit(row, c4, M, L, o);
            continue;
        }
        const int r = idx / per, k = idx - r * per;
        const uint32_t rbar = mapa_u32(bar_u, (uint32_t)r);
        st_async_v4(mapa_u32(sO_u + (uint32_t)(rank * per + k) * 16u, (uint32_t)r), o, rbar);
        if (c4 == 0 || k == 0) st_async_v2(mapa_u32(sM_u + (uint32_t)(rank * 16 + row) * 8u, (uint32_t)r), M, L, rbar);
    }
    SPTRACE(12);
    SPCLK(10);
    // 2. owner merge: one thread per owned float4, ranks in ascending order
    // only the threads that merge wait on the staging barrier (the others exit)
#ifdef EXP_NOEPI
    if (false) {
#else
    if (ns > 1 && tid < mine.n4) {
#endif
        mbar_wait(bar, 0);
        SPTRACE(13);
        SPCLK(11);
        const float2* sML = reinterpret_cast<const float2*>(sM);
        {
            const int k = tid;
            const int idx = rank * per + k, row = idx / C4, c4 = idx - row * C4;
            float2 ml[kMaxSplit];
            float4 xo[kMaxSplit];
#pragma unroll
            for (int c = 0; c < kMaxSplit; ++c) {  // one round of independent loads
                ml[c] = c < ns ? sML[c * 16 + row] : make_float2(-INFINITY, 0.f);
                xo[c] = c < ns ? sO[c * per + k] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            float M = -INFINITY;
#pragma unroll
            for (int c = 0; c < kMaxSplit; ++c) M = fmaxf(M, ml[c].x);
            float L = 0.f;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int c = 0; c < kMaxSplit; ++c) {  // ascending rank order
                const float f = c < ns ? ex2(ml[c].x - M) : 0.f;
                L += f * ml[c].y;
                v.x += f * xo[c].x; v.y += f * xo[c].y; v.z += f * xo[c].z; v.w += f * xo[c].w;
            }
            emit(row, c4, M, L, v);
        }
    }
    SPCLK(14);
    if (bad) set_err(p.err, kDevNumeric);
    if (rank == 0 && tid == 0) {
        if (stale) set_err(p.err, kDevUsage);
        if (cap_err) set_err(p.err, kDevCapacity);
        if (s_post <= 0) set_err(p.err, kDevUsage);  // attention over an empty cache
        // length counter n * g: each head's cluster adds 1 (readers take raw / g, combine.cuh)
        if (p.fuse_append && !cap_err) atomicAdd(&p.seq_len[p.layer * p.max_batch + b], 1);
    }
}

template <int D>
__global__ void __launch_bounds__(kSpWarps * 32, 2)
sparse_lat_kernel(const __grid_constant__ CUtensorMap tm_kv, const AttnParams p) {
    constexpr int NW = kSpWarps, MT = kSpMaxTiles;
    constexpr int kTile = TileLayout<D>::kBytes, kHalf = TileLayout<D>::kVOff;
    constexpr int OSR = 8;  // O rows kept per warp (gs <= 8)
    extern __shared__ __align__(16) uint8_t smem_raw[];
    // 1024-byte alignment (TMA 128B swizzle) by an integer offset, so every pointer below stays
    // visibly in the shared window (LDS/STS rather than generic loads)
    uint8_t* tiles = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    float* cstage = reinterpret_cast<float*>(tiles + MT * kTile);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(cstage) + ClusterStage<D>::kBytes);
    int* tlp = reinterpret_cast<int*>(bars + MT);  // logical page of each resident tile
    static_assert((2 * NW * 16 + NW * OSR * os_stride<D>()) * 4 <= MT * kTile, "epilogue state must fit the tiles");

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    SPTRACE(0);
    if (!p.prewait) pdl_wait();
    // ------------------------------------------------ geometry + the whole KV share in flight
    // Fixed quota of T plan entries per split (split c: entries [c T, c T + T) of the plan,
    // trimmed by its count), so the plan loads do not wait for the count: the length counter,
    // the plan's count and stamp and this split's plan entries are independent loads, issued
    // before the barrier set-up.
    const int T = (p.plan_cap + p.nsplit - 1) / p.nsplit, e0 = split * T;
    const int raw_len = p.seq_len[p.layer * p.max_batch + b];  // raw counter = n * g
    const int plan_cnt = p.plan_count[b], plan_stamp = p.plan_stamp[b];
    int lp = 0, phys = 0;
    if (warp == 0 && lane < min(T, MT) && e0 + lane < p.plan_cap) {
        const size_t e = (size_t)b * p.plan_cap + e0 + lane;
        lp = p.plan_idx[e];
        phys = p.plan_phys[e];
    }
    // the tiles' logical pages for the consumers, published by the CTA barrier below (the TMA
    // barriers would order it too, but racecheck does not follow a tx-completed phase)
    if (warp == 0 && lane < MT) tlp[lane] = lp;
    if (tid == 0) {
        for (int i = 0; i < MT; ++i) mbar_init(&bars[i], 1);
        cluster_stage_init<D>(cstage, p.gs);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) tma_prefetch_desc(&tm_kv);
    __syncthreads();
    cluster_arrive_relaxed();  // peers may push into cstage once they pass the matching wait

    const int n_old = raw_len / p.g;
    const int s = p.fuse_append ? n_old + 1 : n_old;
    const bool cap_err = s > p.max_seq;
    const bool stale = plan_stamp != s;  // R13: a plan is valid for the step it was made at
    const int cnt = (cap_err || stale) ? 0 : plan_cnt;
    const int n_items = max(0, min(min(T, MT), cnt - e0));  // the launcher guarantees T <= MT
#ifdef EXP_NOTMA
    if (false) {
#else
    if (warp == 0 && lane < n_items) {
#endif
        mbar_arrive_expect_tx(&bars[lane], kTile);
        const int row0 = (int)kv_row((size_t)p.layer * p.num_phys + phys, p.g, h, 0);
        uint8_t* dst = tiles + lane * kTile;
        if (D == 64) tma_load_2d(dst, &tm_kv, &bars[lane], 0, row0, kEvictFirst);
        else tma_load_3d(dst, &tm_kv, &bars[lane], 0, row0, 0, kEvictFirst);
    }
    // Warm L2 (and the TLB) for this CTA's q rows: a prefetch is not a read — the q values are
    // loaded after the wait; L2 is the coherence point, so a line the previous kernel writes
    // afterwards is simply updated there (a real decoder's q was just written: L2-hot anyway).
    if (p.q_prefetch && warp == 1 && lane < (p.gs * D * 2 + 127) / 128) {
        const char* qrow = reinterpret_cast<const char*>(p.q) + ((size_t)b * p.m + h * p.gs) * D * 2;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(qrow + lane * 128));
    }
    if (p.prewait) pdl_wait();
    SPTRACE(1);
    // every CTA is past its wait: the next layer may launch (its CTAs co-reside, two per SM)
    if (p.early_trigger && warp == 0) pdl_launch_dependents();
#ifdef EXP_EMPTY
    return;
#endif

    const __nv_bfloat16* k_new = reinterpret_cast<const __nv_bfloat16*>(p.k_new) + ((size_t)b * p.g + h) * D;
    const __nv_bfloat16* v_new = reinterpret_cast<const __nv_bfloat16*>(p.v_new) + ((size_t)b * p.g + h) * D;
    constexpr int kChunks = D / 8;  // 16-byte chunks per row
    // Fused append (Eq.7).  The plan is ascending and always holds the window pages, so its last
    // entry is the page of token s-1: the CTA holding it loads the new row right after
    // the wait (lane c < kChunks: K chunk c, lane kChunks + c: V chunk c), patches it into the
    // resident tile and writes it to the pool after the tile math (off the critical path).
#ifdef EXP_NOAPPEND
    const bool row_cta = false;
#else
    const bool row_cta = p.fuse_append && !cap_err && cnt > 0 && split == (cnt - 1) / T;
#endif
    uint4 new_row = make_uint4(0, 0, 0, 0);
    int new_phys = 0;
    if (row_cta) {
        if (lane < kChunks) new_row = reinterpret_cast<const uint4*>(k_new)[lane];
        else if (lane < 2 * kChunks) new_row = reinterpret_cast<const uint4*>(v_new)[lane - kChunks];
        if (warp == 0) new_phys = p.block_table[(size_t)b * p.bt_stride + (s - 1) / kPage];
    }

    // ------------------------------------------------ consumers: swapped GQA tile (attn_tc.cu)
    const int g4 = lane >> 2, t4 = lane & 3;
    const int gs = p.gs;
    uint32_t qb[D / 16][2];
    {
        const uint32_t* qr = reinterpret_cast<const uint32_t*>(reinterpret_cast<const __nv_bfloat16*>(p.q) +
                                                               ((size_t)b * p.m + h * gs + g4) * D);
#pragma unroll
        for (int kc = 0; kc < D / 16; ++kc) {
#ifdef EXP_NOQ
            qb[kc][0] = qb[kc][1] = (uint32_t)kc * 0x3f803f80u + (uint32_t)(size_t)qr;
#else
            qb[kc][0] = g4 < gs ? qr[(kc * 16 + 2 * t4) >> 1] : 0u;
            qb[kc][1] = g4 < gs ? qr[(kc * 16 + 2 * t4 + 8) >> 1] : 0u;
#endif
        }
    }
    cluster_wait();  // pairs with the entry arrive: every peer's staging barrier is initialised
    SPTRACE(2);
    float o[D / 16][4];
    float mh[2] = {0.f, 0.f}, lh[2] = {0.f, 0.f};  // stabiliser starts at 0 (log2 units), see sp_tiles
#pragma unroll
    for (int mt = 0; mt < D / 16; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    const float sl2 = p.scale_log2;

    // wait for a resident tile, patch the appended row, zero V rows past s; returns valid rows
    auto prepare = [&](int it) -> int {
#ifndef EXP_NOTMA
        mbar_wait(&bars[it], 0);
#endif
        if (it == warp) SPTRACE(3);
        uint8_t* kt = tiles + it * kTile;
        uint8_t* vt = kt + kHalf;
#ifdef EXP_NOTMA
        const int tbase = 0;
#else
        const int tbase = tlp[it] * kPage;
#endif
        const int nvalid = min(kPage, s - tbase);  // rows past s hold no token (partial last page)
#ifdef EXP_NOAPPEND
        if (false) {
#else
        if (p.fuse_append && s - 1 >= tbase && s - 1 < tbase + kPage) {  // patch the appended row
#endif
            const int r = s - 1 - tbase;
            uint4 x = new_row;
            if (!row_cta) {  // not the expected split (cannot happen for a fresh plan): load it now
                if (lane < kChunks) x = reinterpret_cast<const uint4*>(k_new)[lane];
                else if (lane < 2 * kChunks) x = reinterpret_cast<const uint4*>(v_new)[lane - kChunks];
            }
            if (lane < kChunks) *reinterpret_cast<uint4*>(kt + swz<D>(r, lane)) = x;
            else if (lane < 2 * kChunks) *reinterpret_cast<uint4*>(vt + swz<D>(r, lane - kChunks)) = x;
        }
        for (int r = nvalid; r < kPage; ++r)  // 0 * garbage must not be NaN
            if (lane < kChunks) *reinterpret_cast<uint4*>(vt + swz<D>(r, lane)) = make_uint4(0, 0, 0, 0);
        return nvalid;
    };
    // a warp takes tiles warp, warp + NW, ...: two at a time (their MMA chains interleave)
    int it = warp;
    for (; it + NW < n_items; it += 2 * NW) {
        const int nv[2] = {prepare(it), prepare(it + NW)};
        __syncwarp();
        const uint32_t ku[2] = {smem_u32(tiles + it * kTile), smem_u32(tiles + (it + NW) * kTile)};
        const uint32_t vu[2] = {ku[0] + kHalf, ku[1] + kHalf};
#ifndef EXP_NOMATH
        sp_tiles<D, 2>(ku, vu, nv, qb, o, mh, lh, sl2, lane);
#endif
    }
    if (it < n_items) {
        const int nv[1] = {prepare(it)};
        __syncwarp();
        const uint32_t ku[1] = {smem_u32(tiles + it * kTile)};
        const uint32_t vu[1] = {ku[0] + kHalf};
#ifndef EXP_NOMATH
        sp_tiles<D, 1>(ku, vu, nv, qb, o, mh, lh, sl2, lane);
#endif
    }
    SPTRACE(4);
    SPCLK(7);
    if (row_cta && warp == 0 && owns_page(p, (s - 1) / kPage)) {  // Eq.7: the new row into the pool
        const size_t krow = kv_row((size_t)p.layer * p.num_phys + new_phys, p.g, h, (s - 1) % kPage);
        uint4* pool = reinterpret_cast<uint4*>(p.kv_pool);
        if (lane < kChunks) pool[krow * kChunks + lane] = new_row;
        else if (lane < 2 * kChunks) pool[(krow + kPage) * kChunks + lane - kChunks] = new_row;
    }

    // ------------------------------------------------ warp states -> shared memory (tile area)
    __syncthreads();  // every warp is done reading the tiles
    SPCLK(8);
    float* ms = reinterpret_cast<float*>(tiles);
    float* ls = ms + NW * 16;
    float* os = ls + NW * 16;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        float l = lh[e];  // column sum over the 8 token-row groups
        l += __shfl_xor_sync(0xffffffffu, l, 4);
        l += __shfl_xor_sync(0xffffffffu, l, 8);
        l += __shfl_xor_sync(0xffffffffu, l, 16);
        const int hq = 2 * t4 + e;
        if (g4 == 0 && hq < gs) {
            ms[warp * 16 + hq] = mh[e];
            ls[warp * 16 + hq] = l;
        }
    }
#pragma unroll
    for (int mt = 0; mt < D / 16; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int hq = 2 * t4 + (i & 1);
            if (hq < gs) os[(warp * OSR + hq) * os_stride<D>() + mt * 16 + g4 + 8 * (i >> 1)] = o[mt][i];
        }
    __syncthreads();
    SPTRACE(5);
    SPCLK(9);
    sp_epilogue<D, NW, OSR>(p, ms, ls, os, cstage, b, h, stale, cap_err, s, warp, lane);
    SPTRACE(6);
    SPCLK(15);
    if (!p.early_trigger) pdl_launch_dependents();
}

}  // namespace

// Per-device attribute setup (dynamic shared memory opt-in, non-portable clusters) and the
// largest co-resident cluster size for this kernel; cached per device ordinal.
template <int D>
static int sparse_lat_cluster_limit() {
    static std::atomic<int> cache[kMaxDevices];
    return per_device_once(cache, [] {
        auto kern = sparse_lat_kernel<D>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sp_smem<D>()) != cudaSuccess ||
            cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
        return cluster_limit((const void*)kern, kSpWarps * 32, sp_smem<D>());
    });
}

int sparse_lat_max_tiles() { return kSpMaxTiles; }

int sparse_lat_max_split(int d) {
    const int c = d == 128 ? sparse_lat_cluster_limit<128>() : sparse_lat_cluster_limit<64>();
    return c < 1 ? 0 : c;
}

cudaError_t launch_attn_sparse_lat(const AttnParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl) {
    const int lim = sparse_lat_max_split(p.d);
    if (lim < 1 || p.nsplit > lim || p.nsplit < 1 || p.gs > 8) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.nsplit, p.g, p.batch);
    cfg.blockDim = dim3(kSpWarps * 32);
    cfg.dynamicSmemBytes = p.d == 128 ? sp_smem<128>() : sp_smem<64>();
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = p.nsplit;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    if (p.d == 128) return cudaLaunchKernelEx(&cfg, sparse_lat_kernel<128>, *tm_kv, p);
    if (p.d == 64) return cudaLaunchKernelEx(&cfg, sparse_lat_kernel<64>, *tm_kv, p);
    return cudaErrorInvalidValue;
}

}  // namespace delta
