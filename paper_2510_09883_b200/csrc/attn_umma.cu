// attn_umma.cu — bf16 paged decode attention on the 5th-generation tensor cores (tcgen05 +
// TMEM), FULL / SELECT / SPARSE roles, for GQA groups of gs <= 8 query heads.
//
// Eq.4 for one decode query per head, GQA group phi(j) = j / gs (R15), over
// the paged cache (P = 16), split-K over a thread-block cluster exactly as
// attn_tc.cu; what changes is who does the math:
//  * warp 2, producer: one TMA request per (page, head) tile (K rows + V rows, 8 KiB) into a
//    ring of NR tiles with per-tile full / empty mbarriers (token plans: cp.async gathers).
//  * warp 1, MMA issuer (one lane): per tile, 8 x tcgen05.mma (M=128, N=16, K=16)
//        S[heads x 16 tok] = Q . K^T  into a double-buffered TMEM block, A = Q (8 real rows,
//        the other 120 aliased through a zero stride-byte-offset), B = the K rows in place;
//    then, once the softmax has written P, 2 x tcgen05.mma (M=128, N=8, K=16)
//        O^T[d x heads] += V^T . P^T   (P as bf16 hi + bf16 lo, ~16-bit probabilities),
//    A = the V rows in place (MN-major), accumulating in TMEM; tcgen05.commit frees the ring
//    slot and the P buffer.  It also patches the tile holding token s-1 (fused append) and
//    zeroes V rows without a token before the MMAs read them.
//  * warp 0, softmax: lane j (< gs) owns query head j: tcgen05.ld of its 16 logits, mask,
//    SELECT logits to global, exp2 with a lazily raised stabiliser, row sums, P to smem.  A
//    stabiliser raise after P has been accumulated opens a new TMEM accumulator "epoch"
//    (O^T columns 32 + 8e), so the tensor core never waits for a rescale; the epilogue folds
//    the epochs with their stabilisers.
//  * epilogue: the 4 warps read O^T (lane = d) and hand one state per CTA to the cluster merge
//    (combine.cuh).
// Per tile the SM issues ~10 tensor instructions and ~60 softmax instructions instead of
// ~400 mma.sync-path instructions, so one CTA streams its share at TMA speed.
#include <algorithm>

#include "combine.cuh"
#include "umma.cuh"

#ifdef DELTA_TRACE
// per-tile event stamps of CTA (0,0,0) (trace builds): [tile][event]
static __device__ unsigned long long g_tile_trace[64 * 8];
#define TTRACE(tile, ev)                                                                                   \
    do {                                                                                                   \
        if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (tile) < 64) {                        \
            unsigned long long t_;                                                                         \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                         \
            g_tile_trace[(tile) * 8 + (ev)] = t_;                                                          \
        }                                                                                                  \
    } while (0)
extern "C" int delta_trace_read_tiles(void* host) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(host, g_tile_trace, sizeof(g_tile_trace));
    return (int)e;
}
#else
#define TTRACE(tile, ev) do {} while (0)
#endif

namespace delta {
namespace {

constexpr int kUThreads = 128;
constexpr int kNS = 8;                                  // S buffers (tiles the QKs run ahead of the softmax)
constexpr int kLA = kNS - 1;                            // PV(i - kLA) is issued after QK(i)
constexpr int kTmemCols = 256;                          // S: kNS x 16 columns, then O^T epochs: 8 each
constexpr int kSCol = 0;
constexpr int kOCol = kNS * 16;
constexpr int kMaxEpoch = (kTmemCols - kOCol) / 8;      // 16
constexpr float kRaise = 64.f;                          // log2 headroom before the stabiliser moves

template <int D, int NR>
struct UCfg {
    static constexpr int kTile = TileLayout<D>::kBytes;
    static constexpr int kRing = NR * kTile;
    static constexpr int kQBytes = (D / 64) * 1024;     // 8 rows x D bf16, SW128 K-major atoms
    static constexpr int oQ = kRing;
    static constexpr int oP = oQ + kQBytes;             // kNS buffers x (hi 256 B + lo 256 B)
    static constexpr int oStage = oP + kNS * 512;
    static constexpr int oBar = oStage + ClusterStage<D>::kBytes;
    static constexpr int nBar = 2 * NR + 3 * kNS + 1;   // full, empty, s_full, p_full, p_free [kNS], o_done
    static constexpr int oRowTok = oBar + (nBar * 8 + 15) / 16 * 16;  // 16-byte aligned (int4 reads)
    static constexpr int oMisc = oRowTok + NR * kPage * 4;
    static constexpr int kMisc = 16 + (kNS + 4) * 4 + 2 * kMaxEpoch * 8 * 4;
    static constexpr int kSmem = 1024 + oMisc + kMisc;
};

template <int D, bool TOKEN_PLAN, int NR>
__global__ void __launch_bounds__(kUThreads, 2)
attn_umma_kernel(const __grid_constant__ CUtensorMap tm_kv, const AttnParams p) {
    using C = UCfg<D, NR>;
    constexpr int kChunks = D / 8;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring = base;
    uint8_t* qs = base + C::oQ;
    uint8_t* ps = base + C::oP;
    float* cstage = reinterpret_cast<float*>(base + C::oStage);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + C::oBar);
    uint64_t* empty = full + NR;
    uint64_t* s_full = empty + NR;
    uint64_t* p_full = s_full + kNS;
    uint64_t* p_free = p_full + kNS;
    uint64_t* o_done = p_free + kNS;
    int* rowtok = reinterpret_cast<int*>(base + C::oRowTok);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + C::oMisc);
    int* tile_epoch = reinterpret_cast<int*>(base + C::oMisc + 16);  // [kNS]: epoch of each P; [kNS]: count
    float* ep_m = reinterpret_cast<float*>(base + C::oMisc + 16 + (kNS + 4) * 4);  // [kMaxEpoch][8]
    float* ep_l = ep_m + kMaxEpoch * 8;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int gs = p.gs;

    if (tid == 0) {
        for (int i = 0; i < NR; ++i) {
            mbar_init(&full[i], TOKEN_PLAN ? 32 : 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < kNS; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 1);
            mbar_init(&p_free[i], 1);
        }
        mbar_init(o_done, 1);
        cluster_stage_init<D>(cstage, gs);
        fence_mbar_init();
    }
    if (!TOKEN_PLAN && warp == 2 && lane == 0) tma_prefetch_desc(&tm_kv);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    cluster_arrive_relaxed();
    const uint32_t tbase = *tmem_slot;
    if (tid == 0) DTRACE(0);
    if (!p.prewait) pdl_wait();
    if (tid == 0) DTRACE(1);

    // ---------------------------------------------------------------- geometry
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
    const __nv_bfloat16* k_new = reinterpret_cast<const __nv_bfloat16*>(p.k_new) + ((size_t)b * p.g + h) * D;
    const __nv_bfloat16* v_new = reinterpret_cast<const __nv_bfloat16*>(p.v_new) + ((size_t)b * p.g + h) * D;
    if (p.prewait && warp != 2) pdl_wait();
    if (p.early_trigger && warp == 0) pdl_launch_dependents();  // see attn_tc.cu

    if (warp == 3) {
        // fused append: split 0 writes the new row of head h to the pool (Eq.7)
        if (p.fuse_append && !cap_err && split == 0 && owns_page(p, (s - 1) / kPage)) {
            const int t = s - 1;
            const size_t krow = kv_row(layer_ph + bt[t / kPage], p.g, h, t % kPage);
            __nv_bfloat16* pool = reinterpret_cast<__nv_bfloat16*>(p.kv_pool);
            if (lane < kChunks)
                reinterpret_cast<uint4*>(pool + krow * D)[lane] = reinterpret_cast<const uint4*>(k_new)[lane];
            else if (lane < 2 * kChunks)
                reinterpret_cast<uint4*>(pool + (krow + kPage) * D)[lane - kChunks] =
                    reinterpret_cast<const uint4*>(v_new)[lane - kChunks];
        }
    } else if (warp == 2) {
        // ============================================================ producer
        if (!TOKEN_PLAN) {
            for (int base_i = 0; base_i < n_items; base_i += 32) {
                int my_lp = -1, my_phys = 0;
                if (base_i + lane < n_items) {
                    if (p.role == kRoleSparse) {
                        my_lp = plan[unit0 + base_i + lane];
                        my_phys = plan_phys[unit0 + base_i + lane];
                    } else {
                        my_lp = unit0 + base_i + lane;
                        my_phys = bt[my_lp];
                    }
                }
                const int nb = min(32, n_items - base_i);
                for (int j = 0; j < nb; ++j) {
                    const int i = base_i + j, slot = i % NR, round = i / NR;
                    if (round > 0) mbar_wait(&empty[slot], (round - 1) & 1);
                    const int lp = __shfl_sync(0xffffffffu, my_lp, j);
                    const int ph = __shfl_sync(0xffffffffu, my_phys, j);
                    if (lane < kPage) {
                        const int t = lp * kPage + lane;
                        rowtok[slot * kPage + lane] = t < s ? t : -1;
                    }
                    __syncwarp();
                    if (lane == 0) {
                        TTRACE(i, 0);
                        mbar_arrive_expect_tx(&full[slot], C::kTile);
                        const int row0 = (int)kv_row(layer_ph + ph, p.g, h, 0);
                        uint8_t* dst = ring + slot * C::kTile;
                        if (D == 64) tma_load_2d(dst, &tm_kv, &full[slot], 0, row0, kEvictFirst);
                        else tma_load_3d(dst, &tm_kv, &full[slot], 0, row0, 0, kEvictFirst);
                    }
                }
            }
        } else {
            const __nv_bfloat16* pool = reinterpret_cast<const __nv_bfloat16*>(p.kv_pool);
            for (int i = 0; i < n_items; ++i) {
                const int slot = i % NR, round = i / NR;
                int t = -1;
                long long row = -1;
                if (lane < kPage) {
                    const int e = unit0 + i * kPage + lane;
                    if (e < e_end) {
                        t = plan[e];
                        const int pp = plan_phys[e];  // phys_page * P + slot
                        row = (long long)kv_row(layer_ph + pp / kPage, p.g, h, pp % kPage);
                    }
                }
                if (round > 0) mbar_wait(&empty[slot], (round - 1) & 1);
                if (lane < kPage) rowtok[slot * kPage + lane] = t;
                uint8_t* kd = ring + slot * C::kTile;
                for (int ci = lane; ci < kPage * kChunks; ci += 32) {
                    const int r = ci / kChunks, c = ci - r * kChunks;
                    const long long rr = __shfl_sync(0xffffffffu, row, r);
                    if (rr >= 0) {
                        cp_async16(kd + swz<D>(r, c), pool + rr * D + c * 8);
                        cp_async16(kd + TileLayout<D>::kVOff + swz<D>(r, c), pool + (rr + kPage) * D + c * 8);
                    }
                }
                cp_async_mbar_arrive_noinc(&full[slot]);
            }
        }
    } else if (warp == 1) {
        // ============================================================ MMA issuer
        {   // Q of the group: rows = heads (zero past gs), SW128 K-major 8-row atoms per half
            const __nv_bfloat16* qp = reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)b * p.m + h * gs) * D;
            for (int i = lane; i < 8 * kChunks; i += 32) {
                const int r = i / kChunks, c = i - r * kChunks;
                const uint4 v = r < gs ? reinterpret_cast<const uint4*>(qp + (size_t)r * D)[c] : make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4*>(qs + (c >> 3) * 1024 + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
            }
            fence_proxy_async_smem();
            __syncwarp();
        }
        constexpr uint32_t kIdQK = umma_idesc(128, 16, 0, 0);
        constexpr uint32_t kIdPV = umma_idesc(128, 8, 1, 0);
        const uint32_t ring_u = smem_u32(ring), qs_u = smem_u32(qs), ps_u = smem_u32(ps);
        int cur_epoch = -1;
        auto issue_pv = [&](int j) {
            mbar_wait(&p_full[j % kNS], (j / kNS) & 1);
            tc_fence_after();
            const int ep = tile_epoch[j % kNS];
            if (lane == 0) {
                const uint32_t vt = ring_u + (j % NR) * C::kTile + TileLayout<D>::kVOff;
                const uint64_t a = umma_desc(vt, D == 128 ? TileLayout<D>::kHalfBytes : 0, 1024, kLayoutSW128);
                const uint32_t pb = ps_u + (j % kNS) * 512;
                const uint32_t td = tbase + kOCol + 8 * ep;
                umma(td, a, umma_desc(pb, 128, 0, kLayoutNone), kIdPV, ep == cur_epoch ? 1u : 0u);
                umma(td, a, umma_desc(pb + 256, 128, 0, kLayoutNone), kIdPV, 1u);
                umma_commit(&empty[j % NR]);
                umma_commit(&p_free[j % kNS]);
                TTRACE(j, 5);
            }
            cur_epoch = ep;
            __syncwarp();
        };
        // QK runs up to kLA tiles ahead of PV, so the tensor core, the softmax warp and the TMA
        // stream overlap; S buffer i % kNS is free again once PV(i - kNS) was issued (its
        // softmax is done).
        for (int i = 0; i < n_items + kLA; ++i) {
            if (i < n_items) {
                const int slot = i % NR;
                mbar_wait(&full[slot], (i / NR) & 1);
                if (lane == 0) TTRACE(i, 1);
                if (i == 0 && tid == 32) DTRACE(2);
                // tiles with a row to patch: the fused-append token s-1, rows without a token
                const int tok = lane < kPage ? rowtok[slot * kPage + lane] : -1;
                const unsigned inval = __ballot_sync(0xffffffffu, lane < kPage && tok < 0);
                const unsigned fused = p.fuse_append ? __ballot_sync(0xffffffffu, lane < kPage && tok == s - 1) : 0u;
                if (inval | fused) {
                    uint8_t* kt = ring + slot * C::kTile;
                    uint8_t* vt = kt + TileLayout<D>::kVOff;
                    if (fused) {
                        const int r = __ffs(fused) - 1;
                        if (lane < kChunks)
                            *reinterpret_cast<uint4*>(kt + swz<D>(r, lane)) = reinterpret_cast<const uint4*>(k_new)[lane];
                        else if (lane < 2 * kChunks)
                            *reinterpret_cast<uint4*>(vt + swz<D>(r, lane - kChunks)) =
                                reinterpret_cast<const uint4*>(v_new)[lane - kChunks];
                    }
                    for (unsigned mm = inval; mm; mm &= mm - 1) {  // 0 * garbage must not make NaN
                        const int r = __ffs(mm) - 1;
                        if (lane < kChunks) *reinterpret_cast<uint4*>(vt + swz<D>(r, lane)) = make_uint4(0, 0, 0, 0);
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                }
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t kt = ring_u + slot * C::kTile;
                    const uint32_t td = tbase + kSCol + 16 * (i % kNS);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = (kk >> 2) * 1024 + (kk & 3) * 32;
                        const uint64_t a = umma_desc(qs_u + off, 16, 0, kLayoutSW128);  // SBO 0: rows alias 0..7
                        const uint64_t bk = umma_desc(kt + (kk >> 2) * TileLayout<D>::kHalfBytes + (kk & 3) * 32, 16,
                                                      1024, kLayoutSW128);
                        umma(td, a, bk, kIdQK, kk > 0 ? 1u : 0u);
                    }
                    umma_commit(&s_full[i % kNS]);
                    TTRACE(i, 2);
                }
                __syncwarp();
            }
            if (i - kLA >= 0) issue_pv(i - kLA);
        }
        if (lane == 0) umma_commit(o_done);  // arrives once every MMA above has completed
        __syncwarp();
    } else {
        // ============================================================ softmax (warp 0)
        // S rows r >= 8 duplicate row r % 8 (Q rows alias through SBO 0), so lane L holds head
        // hq = L % 8's 16 logits; it handles that head's tokens 4q..4q+3, q = L / 8.
        const int hq = lane & 7, q = lane >> 3;
        const bool active = hq < gs;
        const float sl2 = p.scale_log2;
        float m = -INFINITY, l = 0.f;  // l: this lane's partial sum (4 of the 16 tokens per tile)
        int epoch = 0;
        bool used = false;
        float* lg = p.logits + (size_t)b * p.max_seq * p.m + h * gs + hq;
        for (int i = 0; i < n_items; ++i) {
            mbar_wait(&full[i % NR], (i / NR) & 1);  // rowtok of the tile is published (slot not yet reused)
            mbar_wait(&s_full[i % kNS], (i / kNS) & 1);
            if (lane == 0) TTRACE(i, 3);
            tc_fence_after();
            uint32_t v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(tbase + kSCol + 16 * (i % kNS)));
            const int4 t4 = reinterpret_cast<const int4*>(rowtok + (i % NR) * kPage)[q];
            const int tk[4] = {t4.x, t4.y, t4.z, t4.w};
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            float a4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {  // select this lane's 4 columns (register-indexed by q)
                float x = __uint_as_float(v[j]);
                x = q == 1 ? __uint_as_float(v[4 + j]) : x;
                x = q == 2 ? __uint_as_float(v[8 + j]) : x;
                x = q == 3 ? __uint_as_float(v[12 + j]) : x;
                a4[j] = x;
            }
            float x[4];
            float tmax = -INFINITY;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                x[j] = (active && tk[j] >= 0) ? a4[j] * sl2 : -INFINITY;
                tmax = fmaxf(tmax, x[j]);
                if (p.role == kRoleSelect && active && tk[j] >= 0) lg[(size_t)tk[j] * p.m] = a4[j] * p.scale;
            }
            if (__any_sync(0xffffffffu, tmax > m + kRaise)) {  // stabiliser must move (rare after tile 0)
                tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
                tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
                if (used) {
                    if (epoch + 1 < kMaxEpoch) {  // close this accumulator epoch, open the next
                        float lt = l;
                        lt += __shfl_xor_sync(0xffffffffu, lt, 8);
                        lt += __shfl_xor_sync(0xffffffffu, lt, 16);
                        if (lane < 8) { ep_m[epoch * 8 + lane] = m; ep_l[epoch * 8 + lane] = lt; }
                        ++epoch;
                        l = 0.f;
                        used = false;
                        m = fmaxf(m, tmax);
                    } else if (lane == 0) {
                        set_err(p.err, kDevNumeric);  // logit range beyond kMaxEpoch x 64 log2 units
                    }
                } else {
                    m = fmaxf(m, tmax);
                }
            }
            const float msafe = m == -INFINITY ? 0.f : m;
            float pr[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                pr[j] = ex2(x[j] - msafe);  // -inf -> 0
                l += pr[j];
            }
            used = true;
            if (i >= kNS) mbar_wait(&p_free[i % kNS], ((i - kNS) / kNS) & 1);  // P buffer read by PV(i - kNS)
            {   // P row hq, tokens 4q..4q+3: core matrix q / 2, bytes (q % 2) * 8 of the 16-byte row
                const __nv_bfloat162 h01 = __floats2bfloat162_rn(pr[0], pr[1]);
                const __nv_bfloat162 h23 = __floats2bfloat162_rn(pr[2], pr[3]);
                const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
                uint8_t* pb = ps + (i % kNS) * 512 + (q >> 1) * 128 + hq * 16 + (q & 1) * 8;
                *reinterpret_cast<uint2*>(pb) =
                    make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
                *reinterpret_cast<uint2*>(pb + 256) =
                    make_uint2(pack_bf16(pr[0] - f01.x, pr[1] - f01.y), pack_bf16(pr[2] - f23.x, pr[3] - f23.y));
            }
            if (lane == 0) tile_epoch[i % kNS] = epoch;
            fence_proxy_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[i % kNS]);
            if (lane == 0) TTRACE(i, 4);
        }
        float lt = l;
        lt += __shfl_xor_sync(0xffffffffu, lt, 8);
        lt += __shfl_xor_sync(0xffffffffu, lt, 16);
        if (lane < 8) { ep_m[epoch * 8 + lane] = m; ep_l[epoch * 8 + lane] = lt; }
        if (lane == 0) tile_epoch[kNS] = epoch + 1;
    }

    // ---------------------------------------------------------------- epilogue
    if (tid == 0) DTRACE(3);
    mbar_wait(o_done, 0);
    tc_fence_after();
    __syncthreads();  // epoch tables, every MMA complete
    float* ms = reinterpret_cast<float*>(ring);  // the ring is idle now
    float* ls = ms + 16;
    float* os = ls + 16;
    const int n_ep = tile_epoch[kNS];
    float Mh[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float M = -INFINITY;
        for (int e = 0; e < n_ep; ++e) M = fmaxf(M, ep_m[e * 8 + j]);
        Mh[j] = M;
    }
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = 0.f;
    for (int e = 0; e < n_ep; ++e) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tbase + ((uint32_t)(warp * 32) << 16) + kOCol + 8 * e));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float me = ep_m[e * 8 + j];
            const float w = (Mh[j] == -INFINITY || me == -INFINITY) ? 0.f : exp2f(me - Mh[j]);
            if (w > 0.f) o[j] += w * __uint_as_float(v[j]);  // an epoch no tile reached is never read
        }
    }
    const int d = warp * 32 + lane;
    if (d < D) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j < gs) os[j * os_stride<D>() + d] = o[j];
    }
    if (tid < gs) {
        float L = 0.f;
        for (int e = 0; e < n_ep; ++e) {
            const float me = ep_m[e * 8 + tid];
            L += (Mh[tid] == -INFINITY || me == -INFINITY) ? 0.f : exp2f(me - Mh[tid]) * ep_l[e * 8 + tid];
        }
        ms[tid] = Mh[tid];
        ls[tid] = L;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols));
    if (tid == 0) DTRACE(4);
    cluster_epilogue<D, 1>(p, ms, ls, os, cstage, b, h, stale, cap_err, s);
    if (tid == 0) DTRACE(6);
}

template <int D, bool TOKEN_PLAN, int NR>
cudaError_t launch_impl(const AttnParams& p0, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl) {
    auto kern = attn_umma_kernel<D, TOKEN_PLAN, NR>;
    constexpr int smem = UCfg<D, NR>::kSmem;
    static std::atomic<int> cache[kMaxDevices];  // per device: attribute opt-ins are per context
    const int max_cluster = per_device_once(cache, [&] {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess ||
            cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
            return -1;
        return cluster_limit((const void*)kern, kUThreads, smem);
    });
    if (max_cluster < 1) return cudaErrorInvalidConfiguration;
    AttnParams p = p0;
    p.nsplit = std::min(p.nsplit, max_cluster);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.nsplit, p.g, p.batch);
    cfg.blockDim = dim3(kUThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.nsplit;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, *tm_kv, p);
}

template <int D, bool TOKEN_PLAN>
cudaError_t launch_ring(const AttnParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl) {
    return p.deep ? launch_impl<D, TOKEN_PLAN, 24>(p, tm_kv, st, pdl) : launch_impl<D, TOKEN_PLAN, 11>(p, tm_kv, st, pdl);
}

}  // namespace

bool umma_supported(const AttnParams& p) { return p.gs <= 8 && (p.d == 64 || p.d == 128); }

cudaError_t launch_attn_umma(const AttnParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl) {
    const bool tok = (p.role == kRoleSparse) && p.sel_block == 1;
    if (p.d == 128) return tok ? launch_ring<128, true>(p, tm_kv, st, pdl) : launch_ring<128, false>(p, tm_kv, st, pdl);
    if (p.d == 64) return tok ? launch_ring<64, true>(p, tm_kv, st, pdl) : launch_ring<64, false>(p, tm_kv, st, pdl);
    return cudaErrorInvalidValue;
}

}  // namespace delta
