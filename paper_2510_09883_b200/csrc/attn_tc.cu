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
#include "combine.cuh"

namespace delta {
namespace {

constexpr int NCW = 4;      // consumer warps
constexpr int NSTAGE = 3;   // pipeline depth (stages of NCW head-pages)
constexpr int kThreads = (NCW + 1) * 32;

template <int D>
struct TcCfg {
    static constexpr int kTile = kPage * D * 2;        // bytes of one head-page
    static constexpr int kStageBytes = NCW * kTile;    // per tensor per stage
    static constexpr int kRing = NSTAGE * kStageBytes; // per tensor
    static constexpr int kSmem = 1024 + 2 * kRing + 2 * NSTAGE * 8 + 16;
};

// byte offset of 16-byte chunk c (0..D/8-1) of row r inside a 128B-swizzled head-page
__device__ __forceinline__ uint32_t swz(int r, int c) {
    return (uint32_t)((c >> 3) * (kPage * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

template <int D, bool TOKEN_PLAN>
__global__ void __launch_bounds__(kThreads, 2)
attn_tc_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
               const AttnParams p) {
    using C = TcCfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* kbuf = base;
    uint8_t* vbuf = base + C::kRing;
    uint64_t* full = reinterpret_cast<uint64_t*>(vbuf + C::kRing);
    uint64_t* empty = full + NSTAGE;
    int* sflag = reinterpret_cast<int*>(empty + NSTAGE);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;

    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&full[i], TOKEN_PLAN ? 32 : 1);
            mbar_init(&empty[i], NCW);
        }
        fence_mbar_init();
    }
    if (!TOKEN_PLAN && warp == NCW && lane == 0) {
        tma_prefetch_desc(&tm_k);
        tma_prefetch_desc(&tm_v);
    }
    __syncthreads();
    pdl_wait();  // everything below reads state written by earlier launches

    // ---------------------------------------------------------------- geometry
    const int n_old = p.seq_len[p.layer * p.max_batch + b];
    const int s = p.fuse_append ? n_old + 1 : n_old;
    const bool cap_err = s > p.max_seq;
    bool stale = false;
    int n_items = 0, unit0 = 0, e_end = 0;
    if (!cap_err) {
        if (p.role != kRoleSparse) {
            const int npages = (s + kPage - 1) / kPage;
            unit0 = (int)((long long)split * npages / p.nsplit);
            n_items = (int)((long long)(split + 1) * npages / p.nsplit) - unit0;
        } else {
            stale = p.plan_stamp[b] != s;
            const int cnt = stale ? 0 : p.plan_count[b];
            unit0 = (int)((long long)split * cnt / p.nsplit);
            e_end = (int)((long long)(split + 1) * cnt / p.nsplit);
            n_items = TOKEN_PLAN ? (e_end - unit0 + 15) / 16 : e_end - unit0;
        }
    }
    const int32_t* bt = p.block_table + (size_t)b * p.bt_stride;
    const int32_t* plan = p.plan_idx + (size_t)b * p.plan_cap;
    const size_t layer_ph = (size_t)p.layer * p.num_phys;
    const __nv_bfloat16* k_new = reinterpret_cast<const __nv_bfloat16*>(p.k_new) + ((size_t)b * p.g + h) * D;
    const __nv_bfloat16* v_new = reinterpret_cast<const __nv_bfloat16*>(p.v_new) + ((size_t)b * p.g + h) * D;

    // fused append: split 0 writes the new row of head h to the pools (Eq.7)
    if (p.fuse_append && !cap_err && split == 0 && warp == 0) {
        constexpr int kChunks = D / 8;
        const int t = s - 1;
        const size_t row = ((layer_ph + bt[t / kPage]) * p.g + h) * kPage + (t % kPage);
        if (lane < kChunks) {
            reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.k_pool) + row * D)[lane] =
                reinterpret_cast<const uint4*>(k_new)[lane];
        } else if (lane < 2 * kChunks) {
            reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.v_pool) + row * D)[lane - kChunks] =
                reinterpret_cast<const uint4*>(v_new)[lane - kChunks];
        }
    }

    if (warp == NCW) {
        // ============================================================ producer
        if (!TOKEN_PLAN) {
            if (lane == 0) {
                for (int it = 0, iter = 0; it < n_items; it += NCW, ++iter) {
                    const int stg = iter % NSTAGE, round = iter / NSTAGE;
                    if (round > 0) mbar_wait(&empty[stg], (round - 1) & 1);
                    const int valid = min(NCW, n_items - it);
                    mbar_arrive_expect_tx(&full[stg], valid * 2 * C::kTile);
                    for (int w = 0; w < valid; ++w) {
                        const int item = it + w;
                        const int lp = (p.role == kRoleSparse) ? plan[unit0 + item] : unit0 + item;
                        const int row0 = (int)(((layer_ph + bt[lp]) * p.g + h) * kPage);
                        uint8_t* kd = kbuf + (stg * NCW + w) * C::kTile;
                        uint8_t* vd = vbuf + (stg * NCW + w) * C::kTile;
#pragma unroll
                        for (int half = 0; half < D / 64; ++half) {
                            tma_load_2d(kd + half * kPage * 128, &tm_k, &full[stg], half * 64, row0, kEvictFirst);
                            tma_load_2d(vd + half * kPage * 128, &tm_v, &full[stg], half * 64, row0, kEvictFirst);
                        }
                    }
                }
            }
        } else {
            const __nv_bfloat16* kp = reinterpret_cast<const __nv_bfloat16*>(p.k_pool);
            const __nv_bfloat16* vp = reinterpret_cast<const __nv_bfloat16*>(p.v_pool);
            constexpr int kChunks = D / 8;
            for (int it = 0, iter = 0; it < n_items; it += NCW, ++iter) {
                const int stg = iter % NSTAGE, round = iter / NSTAGE;
                if (round > 0) mbar_wait(&empty[stg], (round - 1) & 1);
                for (int w = 0; w < NCW; ++w) {
                    const int item = it + w;
                    if (item >= n_items) break;
                    // lane r < 16 resolves row r of this tile: token -> pool row
                    long long my_row = -1;
                    if (lane < 16) {
                        const int e = unit0 + item * 16 + lane;
                        if (e < e_end) {
                            const int t = plan[e];
                            my_row = (long long)(((layer_ph + bt[t / kPage]) * p.g + h) * kPage + (t % kPage));
                        }
                    }
                    uint8_t* kd = kbuf + (stg * NCW + w) * C::kTile;
                    uint8_t* vd = vbuf + (stg * NCW + w) * C::kTile;
                    for (int ci = lane; ci < 16 * kChunks; ci += 32) {
                        const int r = ci / kChunks, c = ci - r * kChunks;
                        const long long row = __shfl_sync(0xffffffffu, my_row, r);
                        if (row >= 0) {
                            cp_async16(kd + swz(r, c), kp + row * D + c * 8);
                            cp_async16(vd + swz(r, c), vp + row * D + c * 8);
                        }
                    }
                }
                cp_async_mbar_arrive_noinc(&full[stg]);
            }
        }
    } else {
        // ============================================================ consumers
        const int g4 = lane >> 2, t4 = lane & 3;
        const int gs = p.gs;
        // Q fragments (A operand, rows = query heads of the group, zero-padded to 16)
        uint32_t qa[D / 16][4];
        {
            const __nv_bfloat16* qp = reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)b * p.m + h * gs) * D;
            const uint32_t* q0 = reinterpret_cast<const uint32_t*>(qp + (size_t)g4 * D);
            const uint32_t* q1 = reinterpret_cast<const uint32_t*>(qp + (size_t)(g4 + 8) * D);
            const bool v0 = g4 < gs, v1 = g4 + 8 < gs;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                const int c = (kk * 16 + t4 * 2) >> 1;
                qa[kk][0] = v0 ? q0[c] : 0u;
                qa[kk][1] = v1 ? q1[c] : 0u;
                qa[kk][2] = v0 ? q0[c + 4] : 0u;
                qa[kk][3] = v1 ? q1[c + 4] : 0u;
            }
        }
        float o[D / 8][4];
#pragma unroll
        for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
        const float sl2 = p.scale_log2;

        for (int it = 0, iter = 0; it < n_items; it += NCW, ++iter) {
            const int stg = iter % NSTAGE, round = iter / NSTAGE;
            mbar_wait(&full[stg], round & 1);
            const int item = it + warp;
            if (item < n_items) {
                uint8_t* kt = kbuf + (stg * NCW + warp) * C::kTile;
                uint8_t* vt = vbuf + (stg * NCW + warp) * C::kTile;
                // token of row `lane` (lanes 0..15); -1 = no token
                int my_tok = -1;
                if (lane < 16) {
                    if (!TOKEN_PLAN) {
                        const int lp = (p.role == kRoleSparse) ? plan[unit0 + item] : unit0 + item;
                        const int t = lp * kPage + lane;
                        my_tok = (t < s) ? t : -1;
                    } else {
                        const int e = unit0 + item * 16 + lane;
                        my_tok = (e < e_end) ? plan[e] : -1;
                    }
                }
                // fused append: patch row holding token s-1 from the inputs
                if (p.fuse_append) {
                    const unsigned pm = __ballot_sync(0xffffffffu, my_tok == s - 1);
                    if (pm) {
                        const int r = __ffs(pm) - 1;
                        constexpr int kChunks = D / 8;
                        if (lane < kChunks)
                            *reinterpret_cast<uint4*>(kt + swz(r, lane)) = reinterpret_cast<const uint4*>(k_new)[lane];
                        else if (lane < 2 * kChunks)
                            *reinterpret_cast<uint4*>(vt + swz(r, lane - kChunks)) =
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
                        if (lane < D / 8) *reinterpret_cast<uint4*>(vt + swz(r, lane)) = make_uint4(0, 0, 0, 0);
                    }
                }
                __syncwarp();
                // ---- S = Q K^T (16 q rows x 16 tokens)
                float acc[2][4];
                const uint32_t kt_u = smem_u32(kt), vt_u = smem_u32(vt);
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
                    for (int kc = 0; kc < D / 32; ++kc) {
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4(kt_u + swz(nt * 8 + (lane & 7), kc * 4 + (lane >> 3)), b0, b1, b2, b3);
                        mma_bf16_16816(acc[nt], qa[2 * kc], b0, b1);
                        mma_bf16_16816(acc[nt], qa[2 * kc + 1], b2, b3);
                    }
                }
                // tokens of this lane's accumulator columns: col = nt*8 + 2*t4 + (i&1)
                int tk[2][2];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) tk[nt][e] = __shfl_sync(0xffffffffu, my_tok, nt * 8 + 2 * t4 + e);
                if (p.role == kRoleSelect) {
                    float* lg = p.logits + (size_t)b * p.max_seq * p.m + h * gs;
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const int row = (i < 2) ? g4 : g4 + 8;
                            const int t = tk[nt][i & 1];
                            if (row < gs && t >= 0) lg[(size_t)t * p.m + row] = acc[nt][i] * p.scale;
                        }
                }
                // ---- online softmax (log2 domain)
                float x[2][4];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                    for (int i = 0; i < 4; ++i) x[nt][i] = (tk[nt][i & 1] >= 0) ? acc[nt][i] * sl2 : -INFINITY;
                float mx0 = fmaxf(fmaxf(x[0][0], x[0][1]), fmaxf(x[1][0], x[1][1]));
                float mx1 = fmaxf(fmaxf(x[0][2], x[0][3]), fmaxf(x[1][2], x[1][3]));
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
                mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
                mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
                const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
                const float ms0 = (mn0 == -INFINITY) ? 0.f : mn0;
                const float ms1 = (mn1 == -INFINITY) ? 0.f : mn1;
                const float a0 = ex2(m0 - ms0), a1 = ex2(m1 - ms1);
                float pr[2][4];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    pr[nt][0] = ex2(x[nt][0] - ms0);
                    pr[nt][1] = ex2(x[nt][1] - ms0);
                    pr[nt][2] = ex2(x[nt][2] - ms1);
                    pr[nt][3] = ex2(x[nt][3] - ms1);
                }
                l0 = l0 * a0 + (pr[0][0] + pr[0][1] + pr[1][0] + pr[1][1]);
                l1 = l1 * a1 + (pr[0][2] + pr[0][3] + pr[1][2] + pr[1][3]);
                m0 = mn0;
                m1 = mn1;
#pragma unroll
                for (int n = 0; n < D / 8; ++n) {
                    o[n][0] *= a0; o[n][1] *= a0; o[n][2] *= a1; o[n][3] *= a1;
                }
                // ---- O += P V, P split into bf16 hi + lo
                uint32_t ahi[4], alo[4];
                {
                    const float* f[4] = {&pr[0][0], &pr[0][2], &pr[1][0], &pr[1][2]};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const __nv_bfloat162 hv = __floats2bfloat162_rn(f[i][0], f[i][1]);
                        const float2 hf = __bfloat1622float2(hv);
                        ahi[i] = *reinterpret_cast<const uint32_t*>(&hv);
                        alo[i] = pack_bf16(f[i][0] - hf.x, f[i][1] - hf.y);
                    }
                }
#pragma unroll
                for (int vc = 0; vc < D / 16; ++vc) {
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4_t(vt_u + swz(((lane >> 3) & 1) * 8 + (lane & 7), vc * 2 + (lane >> 4)), b0, b1, b2, b3);
                    mma_bf16_16816(o[2 * vc], ahi, b0, b1);
                    mma_bf16_16816(o[2 * vc], alo, b0, b1);
                    mma_bf16_16816(o[2 * vc + 1], ahi, b2, b3);
                    mma_bf16_16816(o[2 * vc + 1], alo, b2, b3);
                }
                // generic-proxy smem writes must be ordered before the next TMA refill
                if (wrote_smem) fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
        }
        // quad-reduce the row sums
        l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
        l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 2);

        // ---------------------------------------------------------------- merge
        consumer_bar(NCW * 32);  // every consumer is done reading the ring
        float* ms = reinterpret_cast<float*>(kbuf);
        float* ls = ms + NCW * 16;
        float* os = ls + NCW * 16;
        if (t4 == 0) {
            ms[warp * 16 + g4] = m0; ls[warp * 16 + g4] = l0;
            ms[warp * 16 + g4 + 8] = m1; ls[warp * 16 + g4 + 8] = l1;
        }
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
            const int col = n * 8 + 2 * t4;
            if (g4 < gs) {
                os[(warp * 16 + g4) * D + col] = o[n][0];
                os[(warp * 16 + g4) * D + col + 1] = o[n][1];
            }
            if (g4 + 8 < gs) {
                os[(warp * 16 + g4 + 8) * D + col] = o[n][2];
                os[(warp * 16 + g4 + 8) * D + col + 1] = o[n][3];
            }
        }
        consumer_bar(NCW * 32);
        pdl_launch_dependents();
        cta_merge<D>(p, ms, ls, os, NCW, b, h, split, tid, NCW * 32);
        grid_combine<D>(p, b, h, s, stale, cap_err, tid, NCW * 32, sflag);
    }
}

template <int D, bool TOKEN_PLAN>
cudaError_t launch_impl(const AttnParams& p, const CUtensorMap* tm_k, const CUtensorMap* tm_v,
                        cudaStream_t st, bool pdl) {
    auto kern = attn_tc_kernel<D, TOKEN_PLAN>;
    constexpr int smem = TcCfg<D>::kSmem;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.nsplit, p.g, p.batch);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, *tm_k, *tm_v, p);
}

}  // namespace

cudaError_t launch_attn_tc(const AttnParams& p, const CUtensorMap* tm_k, const CUtensorMap* tm_v,
                           cudaStream_t st, bool pdl) {
    const bool tok = (p.role == kRoleSparse) && p.sel_block == 1;
    if (p.d == 128) return tok ? launch_impl<128, true>(p, tm_k, tm_v, st, pdl) : launch_impl<128, false>(p, tm_k, tm_v, st, pdl);
    if (p.d == 64) return tok ? launch_impl<64, true>(p, tm_k, tm_v, st, pdl) : launch_impl<64, false>(p, tm_k, tm_v, st, pdl);
    return cudaErrorInvalidValue;
}

}  // namespace delta
