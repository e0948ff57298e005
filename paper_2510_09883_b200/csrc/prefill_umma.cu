// prefill_umma.cu — chunked prefill (NEXT-3; Eq.4 with the causal mask over a
// prompt chunk) on the 5th-generation tensor cores: tcgen05.mma with the
// accumulators in TMEM, operands in shared memory, K/V pages streamed by TMA.
//
// Query i of the chunk sits at position n0 + i and attends tokens t <= n0 + i; GQA head j
// reads group phi(j) = j / gs (R15).  CTA = (tile of T = 128 / gs query tokens, kv head h,
// sequence b): its 128 MMA rows are the (head j, token i) pairs of the group, row = j T + i.
// Per KV block of KB = 4 pages (64 tokens):
//   S[128 x 64]  = Q . K^T           D/16 MMAs M=128 N=64  K=16   (TMEM, double-buffered)
//   P = exp2(S * scale * log2 e - m) (online softmax, one thread per row, lazily raised m)
//   O[128 x D]  += P . V             per page: P_hi . V and P_lo . V, M=128 N=D K=16 (TMEM)
// P enters as bf16 hi + lo (~16-bit probabilities, R18 as in the decode kernels).
// Measured on this B200 (tools/umma_rate.cu): a tcgen05.mma costs ~46 cycles whatever its N up
// to N = 32, 48 at N = 64 and 64 at N = 128 — so S is issued over 64-token blocks.  The K rows
// and the V rows of a block's 4 pages arrive as separate TMA boxes (16 rows x 128 B of one
// 64-column half each: the pool interleaves K and V per (page, head), so only per-page boxes
// give a uniformly strided [half][64 rows][128 B] operand) into their own 4-deep rings: a K
// block is released by its S MMAs, a V block by its PV MMAs, and no warp copies operands.
// Warps: 0-3 softmax + epilogue (thread = row), 4 K producer, 5 MMA issuer, 6 V producer (and
// the zeroing of V rows past the end in the last page), 7 idle.
#include <algorithm>

#include "combine.cuh"
#include "umma.cuh"

namespace delta {
namespace {

constexpr int kPuThreads = 256;
constexpr int kPuKB = 4;                  // pages per KV block (64 tokens)
constexpr int kPuNB = 4;                  // blocks in the K ring and in the V ring
constexpr int kPuBT = kPuKB * kPage;      // tokens per block
constexpr float kPuRaise = 8.f;           // log2 headroom before the running max moves

template <int D>
struct PuCfg {
    static constexpr int kHalves = D / 64;
    static constexpr int kQ = kHalves * 128 * 128;               // Q: [half][128 rows][128 B]
    static constexpr int kBlk = kHalves * kPuBT * 128;           // K or V block: [half][64 rows][128 B]
    static constexpr int kP = 128 * 128;                         // P: [128 rows][64 tok bf16]
    static constexpr int oQ = 0;
    static constexpr int oK = oQ + kQ;                           // K ring
    static constexpr int oV = oK + kPuNB * kBlk;                 // V ring
    static constexpr int oP = oV + kPuNB * kBlk;                 // 2 x (hi, lo)
    static constexpr int oBar = oP + 4 * kP;
    static constexpr int nBar = 4 * kPuNB + 1 + 2 * 4;
    static constexpr int kSmem = 1024 + oBar + nBar * 8 + 16;
    static constexpr int kTmemCols = 256;                        // S: 2 x 64 columns, O: D columns at 128
    static constexpr int kOCol = 128;
};

template <int D>
__global__ void __launch_bounds__(kPuThreads, 1)
prefill_umma_kernel(const __grid_constant__ CUtensorMap tm_kv, const PrefillParams p) {
    using C = PuCfg<D>;
    extern __shared__ __align__(16) uint8_t pu_smem[];
    uint8_t* base = pu_smem + ((1024u - (smem_u32(pu_smem) & 1023u)) & 1023u);
    uint8_t* qs = base + C::oQ;
    uint8_t* kring = base + C::oK;
    uint8_t* vring = base + C::oV;
    uint8_t* pbuf = base + C::oP;  // [2][hi, lo][kP]
    uint64_t* k_full = reinterpret_cast<uint64_t*>(base + C::oBar);
    uint64_t* k_empty = k_full + kPuNB;
    uint64_t* v_full = k_empty + kPuNB;
    uint64_t* v_empty = v_full + kPuNB;
    uint64_t* vz_done = v_empty + kPuNB;  // the last page's V rows past the end are zeroed
    uint64_t* s_full = vz_done + 1;
    uint64_t* s_free = s_full + 2;
    uint64_t* p_full = s_free + 2;
    uint64_t* p_free = p_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_free + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gs = p.gs, T = 128 / gs;
    const int tile = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, b = blockIdx.z;  // longest rows first
    const int t0 = tile * T;

    if (tid == 0) {
        for (int i = 0; i < kPuNB; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);  // the block's S MMAs completed
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);  // the block's PV MMAs completed
        }
        mbar_init(vz_done, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 4);    // the four softmax warps
            mbar_init(&p_full[i], 4);
            mbar_init(&p_free[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp == 4 && lane == 0) tma_prefetch_desc(&tm_kv);
    pdl_wait();  // the chunk's append (previous kernel) wrote the pool rows and the length
    const int s_tot = p.seq_len[p.layer * p.max_batch + b] / p.g;  // raw counter = n * g
    const int n0 = s_tot - p.ntok;
    const int t_hi = min(p.ntok, t0 + T);                 // tokens [t0, t_hi) of the chunk
    const int kv_end = n0 + t_hi;                         // keys [0, kv_end) are needed
    const int n_pages = (kv_end + kPage - 1) / kPage;
    const int nblk = (n_pages + kPuKB - 1) / kPuKB;
    // Q rows (warps 0-3: thread = row), K-major SW128: 16-byte chunk c of row r at
    // half (c / 8) * 16 KiB + r * 128 + ((c % 8) ^ (r % 8)) * 16
    if (warp < 4) {
        const int r = tid, j = r / T, i = r - j * T;
        const bool valid = j < gs && t0 + i < p.ntok;
        const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.q) +
                                                          (((size_t)b * p.ntok + t0 + i) * p.m + h * gs + j) * D);
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
            const uint4 v = valid ? src[c] : make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(qs + (c >> 3) * 16384 + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_launch_dependents();
    const uint32_t tbase = *tmem_slot;
    const size_t layer_ph = (size_t)p.layer * p.num_phys;
    const int32_t* bt = p.block_table + (size_t)b * p.bt_stride;

    // per block: the pages it holds and the TMA bytes of its K (or V) boxes
    auto block_pages = [&](int i) { return min(kPuKB, n_pages - i * kPuKB); };
    const bool tail = (kv_end % kPage) != 0;  // the last page holds rows past the end
    if (warp == 4 || warp == 6) {
        // ============================================================ TMA producers: K (warp 4)
        // and V (warp 6), one 16-row box per (page, half) into the block's [half][64 rows][128 B]
        const bool is_v = warp == 6;
        uint8_t* ring = is_v ? vring : kring;
        uint64_t* fullb = is_v ? v_full : k_full;
        uint64_t* emptyb = is_v ? v_empty : k_empty;
        if (lane == 0) {
            for (int i = 0; i < nblk; ++i) {
                const int slot = i % kPuNB, round = i / kPuNB;
                if (round > 0) mbar_wait(&emptyb[slot], (round - 1) & 1);
                const int np = block_pages(i);
#ifdef EXP_PFNOLOAD
                mbar_arrive(&fullb[slot]);
                continue;
#endif
                mbar_arrive_expect_tx(&fullb[slot], np * C::kHalves * kPage * 128);
                for (int q = 0; q < np; ++q) {
                    const int row0 = (int)kv_row(layer_ph + bt[i * kPuKB + q], p.g, h, 0) + (is_v ? kPage : 0);
#pragma unroll
                    for (int hf = 0; hf < C::kHalves; ++hf) {
                        uint8_t* dst = ring + slot * C::kBlk + hf * (kPuBT * 128) + q * kPage * 128;
                        if (D == 64) tma_load_2d(dst, &tm_kv, &fullb[slot], 0, row0, kEvictNormal);
                        else tma_load_3d(dst, &tm_kv, &fullb[slot], 0, row0, hf, kEvictNormal);
                    }
                }
            }
        }
        // (a parity wait names one of two phases: the other lanes may wait for the last block only
        // once lane 0 has issued it, i.e. its slot's barrier is in that block's phase)
        __syncwarp();
        if (is_v && tail && nblk > 0) {
            // V rows past the end in the last page: 0 (P is 0 there, but 0 * garbage may be NaN)
            const int i = nblk - 1, slot = i % kPuNB, q = block_pages(i) - 1, r0 = kv_end % kPage;
            mbar_wait(&v_full[slot], (i / kPuNB) & 1);
            uint8_t* vb = vring + slot * C::kBlk;
            for (int ch = lane; ch < C::kHalves * (kPage - r0) * 8; ch += 32) {
                const int hf = ch / ((kPage - r0) * 8), rem = ch - hf * (kPage - r0) * 8;
                const int r = q * kPage + r0 + rem / 8, c = rem % 8;
                *reinterpret_cast<uint4*>(vb + hf * (kPuBT * 128) + r * 128 + ((c ^ (r & 7)) << 4)) = make_uint4(0, 0, 0, 0);
            }
            fence_proxy_async_smem();  // generic stores -> the tensor core's async-proxy reads
            __syncwarp();
            if (lane == 0) mbar_arrive(vz_done);
        }
    } else if (warp == 5) {
        // ============================================================ MMA issuer (one lane)
        constexpr uint32_t kIdS = umma_idesc(128, kPuBT, 0, 0);  // A = Q K-major, B = K rows K-major
        constexpr uint32_t kIdPV = umma_idesc(128, D, 0, 1);     // A = P K-major, B = V MN-major
        const uint32_t qs_u = smem_u32(qs), k_u = smem_u32(kring), v_u = smem_u32(vring), p_u = smem_u32(pbuf);
        for (int i = 0; i <= nblk; ++i) {
            if (i < nblk) {  // S(i)
                mbar_wait(&k_full[i % kPuNB], (i / kPuNB) & 1);
                if (i >= 2) mbar_wait(&s_free[i & 1], ((i - 2) >> 1) & 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t kb = k_u + (i % kPuNB) * C::kBlk;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint64_t a = umma_desc(qs_u + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, kLayoutSW128);
                        const uint64_t bk = umma_desc(kb + (kk >> 2) * (kPuBT * 128) + (kk & 3) * 32, 16, 1024, kLayoutSW128);
                        umma(tbase + (i & 1) * kPuBT, a, bk, kIdS, kk > 0 ? 1u : 0u);
                    }
                    umma_commit(&s_full[i & 1]);
                    umma_commit(&k_empty[i % kPuNB]);
                }
                __syncwarp();
            }
            if (i >= 1) {  // PV(i - 1), after its softmax wrote P
                const int j = i - 1;
                mbar_wait(&p_full[j & 1], (j >> 1) & 1);
                mbar_wait(&v_full[j % kPuNB], (j / kPuNB) & 1);
                if (tail && j == nblk - 1) mbar_wait(vz_done, 0);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t ph = p_u + (j & 1) * 2 * C::kP, pl = ph + C::kP;
                    const uint32_t vb = v_u + (j % kPuNB) * C::kBlk;
                    const int np = block_pages(j);
                    for (int q = 0; q < np; ++q) {
                        // V rows of page q: MN-major, the two d halves kPuBT * 128 bytes apart
                        const uint64_t bv = umma_desc(vb + q * kPage * 128, D == 128 ? kPuBT * 128 : 0, 1024, kLayoutSW128);
                        umma(tbase + C::kOCol, umma_desc(ph + q * 32, 16, 1024, kLayoutSW128), bv, kIdPV,
                             (j > 0 || q > 0) ? 1u : 0u);
                        umma(tbase + C::kOCol, umma_desc(pl + q * 32, 16, 1024, kLayoutSW128), bv, kIdPV, 1u);
                    }
                    umma_commit(&v_empty[j % kPuNB]);
                    umma_commit(&p_free[j & 1]);
                }
                __syncwarp();
            }
        }
    } else if (warp < 4) {
        // ============================================================ softmax (thread = row)
        const int r = tid, j = r / T, i_tok = r - j * T;
        const bool valid = j < gs && t0 + i_tok < p.ntok;
        const int pos = n0 + t0 + i_tok;   // keys t <= pos
        const float sl2 = p.scale_log2;
        const uint32_t lane_base = tbase + ((uint32_t)(warp * 32) << 16);
        float m = -INFINITY, l = 0.f;
        for (int i = 0; i < nblk; ++i) {
            mbar_wait(&s_full[i & 1], (i >> 1) & 1);
            tc_fence_after();
            float x[kPuBT];
            {
                uint32_t v0[32], v1[32];
                tmem_ld32(lane_base + (i & 1) * kPuBT, v0);
                tmem_ld32(lane_base + (i & 1) * kPuBT + 32, v1);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    x[c] = __uint_as_float(v0[c]);
                    x[32 + c] = __uint_as_float(v1[c]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_free[i & 1]);
            float bmax = -INFINITY;
            const int tk0 = i * kPuBT;
#pragma unroll
            for (int c = 0; c < kPuBT; ++c) {
                x[c] = (valid && tk0 + c <= pos) ? x[c] * sl2 : -INFINITY;
                bmax = fmaxf(bmax, x[c]);
            }
            // raise the running max only when a logit exceeds it by the headroom (p <= 2^8)
            const bool raise = bmax > m + kPuRaise || (m == -INFINITY && bmax > -INFINITY);
            const float m_new = raise ? fmaxf(m, bmax) : m;
            const bool rescale = raise && l > 0.f;
            if (__any_sync(0xffffffffu, rescale)) {
                // O rows of this warp hold earlier blocks' contributions: wait for PV(i - 1),
                // then scale them in TMEM (warp-wide: tcgen05.ld / st are .sync.aligned)
                mbar_wait(&p_free[(i - 1) & 1], ((i - 1) >> 1) & 1);
                tc_fence_after();
                const float al = rescale ? ex2(m - m_new) : 1.f;
#pragma unroll
                for (int c0 = 0; c0 < D; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(lane_base + C::kOCol + c0, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(__uint_as_float(v[c]) * al);
                    tmem_st32(lane_base + C::kOCol + c0, v);
                }
                tmem_wait_st();
                l *= al;
            }
            m = m_new;
            const float msafe = m == -INFINITY ? 0.f : m;
            if (i >= 2) mbar_wait(&p_free[i & 1], ((i - 2) >> 1) & 1);  // PV(i - 2) done with this P buffer
            uint8_t* ph = pbuf + (i & 1) * 2 * C::kP;
            uint8_t* pl = ph + C::kP;
#pragma unroll
            for (int c16 = 0; c16 < kPuBT / 8; ++c16) {  // 8 tokens per 16-byte chunk
                uint32_t hw[4], lw[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
#ifdef EXP_PFNOEXP
                    const float p0 = x[c16 * 8 + 2 * e] - msafe, p1 = x[c16 * 8 + 2 * e + 1] - msafe;
#else
                    const float p0 = ex2(x[c16 * 8 + 2 * e] - msafe), p1 = ex2(x[c16 * 8 + 2 * e + 1] - msafe);
#endif
                    l += p0 + p1;
                    const __nv_bfloat162 hv = __floats2bfloat162_rn(p0, p1);
                    const float2 hf = __bfloat1622float2(hv);
                    hw[e] = *reinterpret_cast<const uint32_t*>(&hv);
                    lw[e] = pack_bf16(p0 - hf.x, p1 - hf.y);
                }
                const int off = r * 128 + ((c16 ^ (r & 7)) << 4);
                *reinterpret_cast<uint4*>(ph + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                *reinterpret_cast<uint4*>(pl + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
            fence_proxy_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[i & 1]);
        }
        // ------------------------------------------------------------ epilogue: O / l
        if (nblk > 0) mbar_wait(&p_free[(nblk - 1) & 1], ((nblk - 1) >> 1) & 1);  // the last PV completed
        tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        float* dst = p.out + (((size_t)b * p.ntok + t0 + i_tok) * p.m + h * gs + j) * D;
        bool bad = false;
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(lane_base + C::kOCol + c0, v);
            tmem_wait_ld();
            if (valid) {
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    const float4 o = make_float4(__uint_as_float(v[c]) * inv, __uint_as_float(v[c + 1]) * inv,
                                                 __uint_as_float(v[c + 2]) * inv, __uint_as_float(v[c + 3]) * inv);
                    bad |= !(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w));
                    *reinterpret_cast<float4*>(dst + c0 + c) = o;
                }
            }
        }
        if (valid && p.lse_out)
            p.lse_out[((size_t)b * p.ntok + t0 + i_tok) * p.m + h * gs + j] =
                l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
        if (bad) set_err(p.err, kDevNumeric);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::kTmemCols));
}

// ================================================================================================
// Operands in TMEM (pfumma = 2): Q and P are the A operands of the two MMAs, and both live in
// tensor memory instead of shared memory — tcgen05.mma [d], [a_tmem], b_desc — so the tensor
// core reads only K (for S) and V (for PV) from shared memory.  Measured reason: the one-tile
// kernel takes ~2500 cycles per 64-token block against ~900 cycles of MMA time, and is neither
// TMA nor MUFU bound (EXP_PFNOLOAD / EXP_PFNOEXP) nor softmax-latency bound (two query tiles
// per CTA ping-ponging the tensor core: no change) — its shared memory moves ~176 KB per block
// (TMA K/V 32, Q 32 + K 16 for S, P 32 + V 32 for PV, P stores 32) against ~128 B/clock; with Q
// and P in TMEM it moves ~80 KB.  Q is written once per CTA (tcgen05.st, thread = row); P is
// written by the softmax threads with tcgen05.st (32 columns of bf16 pairs per hi / lo) instead
// of swizzled shared-memory stores.  TMEM columns (D = 128): Q [0, 64), S [64, 192) (two
// buffers), P [192, 320) (two buffers of hi, lo), O [320, 448).
template <int D>
struct Pu2Cfg {
    static constexpr int kHalves = D / 64;
    static constexpr int kBlk = kHalves * kPuBT * 128;           // K or V block: [half][64 rows][128 B]
    static constexpr int oK = 0;
    static constexpr int oV = oK + kPuNB * kBlk;
    static constexpr int oBar = oV + kPuNB * kBlk;
    static constexpr int nBar = 4 * kPuNB + 1 + 2 * 4;
    static constexpr int kSmem = 1024 + oBar + nBar * 8 + 16;
    static constexpr int kTmemCols = 512;
    static constexpr int kQCol = 0;
    static constexpr int kSCol = 64;                              // + buffer * 64
    static constexpr int kPCol = 192;                             // + buffer * 64: hi [0, 32), lo [32, 64)
    static constexpr int kOCol = 320;
};

// Issued by the whole (converged) warp: one lane, elected inside the asm, issues the MMA — no
// divergent `if (lane == 0)` around it, so the operands can stay in uniform registers instead
// of the per-MMA elect / broadcast loop the compiler wraps around divergent tcgen05 issue.
__device__ __forceinline__ void umma_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_w(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
        : "memory");
}

template <int D>
__global__ void __launch_bounds__(kPuThreads, 1)
prefill_umma2_kernel(const __grid_constant__ CUtensorMap tm_kv, const PrefillParams p) {
    using C = Pu2Cfg<D>;
    extern __shared__ __align__(16) uint8_t pu_smem[];
    uint8_t* base = pu_smem + ((1024u - (smem_u32(pu_smem) & 1023u)) & 1023u);
    uint8_t* kring = base + C::oK;
    uint8_t* vring = base + C::oV;
    uint64_t* k_full = reinterpret_cast<uint64_t*>(base + C::oBar);
    uint64_t* k_empty = k_full + kPuNB;
    uint64_t* v_full = k_empty + kPuNB;
    uint64_t* v_empty = v_full + kPuNB;
    uint64_t* vz_done = v_empty + kPuNB;
    uint64_t* s_full = vz_done + 1;
    uint64_t* s_free = s_full + 2;
    uint64_t* p_full = s_free + 2;
    uint64_t* p_free = p_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_free + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gs = p.gs, T = 128 / gs;
    const int tile = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, b = blockIdx.z;  // longest rows first
    const int t0 = tile * T;

    if (tid == 0) {
        for (int i = 0; i < kPuNB; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
        }
        mbar_init(vz_done, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 4);
            mbar_init(&p_full[i], 4);
            mbar_init(&p_free[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp == 4 && lane == 0) tma_prefetch_desc(&tm_kv);
    pdl_wait();  // the chunk's append (previous kernel) wrote the pool rows and the length
    const int s_tot = p.seq_len[p.layer * p.max_batch + b] / p.g;  // raw counter = n * g
    const int n0 = s_tot - p.ntok;
    const int t_hi = min(p.ntok, t0 + T);
    const int kv_end = n0 + t_hi;
    const int n_pages = (kv_end + kPage - 1) / kPage;
    const int nblk = (n_pages + kPuKB - 1) / kPuKB;
    __syncthreads();  // the TMEM allocation is visible
    const uint32_t tbase = *tmem_slot;
    if (warp < 4) {  // Q row r (thread = row) into TMEM lane r, two bf16 per column
        const int r = tid, j = r / T, i = r - j * T;
        const bool valid = j < gs && t0 + i < p.ntok;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(reinterpret_cast<const __nv_bfloat16*>(p.q) +
                                                                (((size_t)b * p.ntok + t0 + i) * p.m + h * gs + j) * D);
        const uint32_t lb = tbase + ((uint32_t)(warp * 32) << 16);
#pragma unroll
        for (int c0 = 0; c0 < D / 2; c0 += 32) {
            uint32_t v[32];
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
                const uint4 x = valid ? reinterpret_cast<const uint4*>(src + c0)[c / 4] : make_uint4(0, 0, 0, 0);
                v[c] = x.x; v[c + 1] = x.y; v[c + 2] = x.z; v[c + 3] = x.w;
            }
            tmem_st32(lb + C::kQCol + c0, v);
        }
        tmem_wait_st();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_launch_dependents();
    const size_t layer_ph = (size_t)p.layer * p.num_phys;
    const int32_t* bt = p.block_table + (size_t)b * p.bt_stride;
    auto block_pages = [&](int i) { return min(kPuKB, n_pages - i * kPuKB); };
    const bool tail = (kv_end % kPage) != 0;
    if (warp == 4 || warp == 6) {
        // ============================================================ TMA producers: K (4), V (6)
        const bool is_v = warp == 6;
        uint8_t* ring = is_v ? vring : kring;
        uint64_t* fullb = is_v ? v_full : k_full;
        uint64_t* emptyb = is_v ? v_empty : k_empty;
        if (lane == 0) {
            for (int i = 0; i < nblk; ++i) {
                const int slot = i % kPuNB, round = i / kPuNB;
                if (round > 0) mbar_wait(&emptyb[slot], (round - 1) & 1);
                const int np = block_pages(i);
                mbar_arrive_expect_tx(&fullb[slot], np * C::kHalves * kPage * 128);
                for (int q = 0; q < np; ++q) {
                    const int row0 = (int)kv_row(layer_ph + bt[i * kPuKB + q], p.g, h, 0) + (is_v ? kPage : 0);
#pragma unroll
                    for (int hf = 0; hf < C::kHalves; ++hf) {
                        uint8_t* dst = ring + slot * C::kBlk + hf * (kPuBT * 128) + q * kPage * 128;
                        if (D == 64) tma_load_2d(dst, &tm_kv, &fullb[slot], 0, row0, kEvictNormal);
                        else tma_load_3d(dst, &tm_kv, &fullb[slot], 0, row0, hf, kEvictNormal);
                    }
                }
            }
        }
        __syncwarp();
        if (is_v && tail && nblk > 0) {  // V rows past the end in the last page: 0
            const int i = nblk - 1, slot = i % kPuNB, q = block_pages(i) - 1, r0 = kv_end % kPage;
            mbar_wait(&v_full[slot], (i / kPuNB) & 1);
            uint8_t* vb = vring + slot * C::kBlk;
            for (int ch = lane; ch < C::kHalves * (kPage - r0) * 8; ch += 32) {
                const int hf = ch / ((kPage - r0) * 8), rem = ch - hf * (kPage - r0) * 8;
                const int r = q * kPage + r0 + rem / 8, c = rem % 8;
                *reinterpret_cast<uint4*>(vb + hf * (kPuBT * 128) + r * 128 + ((c ^ (r & 7)) << 4)) = make_uint4(0, 0, 0, 0);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(vz_done);
        }
    } else if (warp == 5) {
        // ============================================================ MMA issuer (converged warp)
        constexpr uint32_t kIdS = umma_idesc(128, kPuBT, 0, 0);  // A = Q (TMEM), B = K rows K-major
        constexpr uint32_t kIdPV = umma_idesc(128, D, 0, 1);     // A = P (TMEM), B = V MN-major
        const uint32_t tb = __shfl_sync(0xffffffffu, tbase, 0);
        const uint64_t k_d0 = umma_desc(smem_u32(kring), 16, 1024, kLayoutSW128);
        const uint64_t v_d0 = umma_desc(smem_u32(vring), D == 128 ? kPuBT * 128 : 0, 1024, kLayoutSW128);
        for (int i = 0; i <= nblk; ++i) {
            if (i < nblk) {  // S(i)
                mbar_wait(&k_full[i % kPuNB], (i / kPuNB) & 1);
                if (i >= 2) mbar_wait(&s_free[i & 1], ((i - 2) >> 1) & 1);
                tc_fence_after();
                const uint64_t kd = k_d0 + (uint64_t)(((i % kPuNB) * C::kBlk) >> 4);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk)
                    umma_ts_w(tb + C::kSCol + (i & 1) * kPuBT, tb + C::kQCol + kk * 8,
                              kd + (uint64_t)((((kk >> 2) * (kPuBT * 128)) + (kk & 3) * 32) >> 4), kIdS, kk > 0 ? 1u : 0u);
                umma_commit_w(&s_full[i & 1]);
                umma_commit_w(&k_empty[i % kPuNB]);
            }
            if (i >= 1) {  // PV(i - 1), after its softmax wrote P
                const int j = i - 1;
                mbar_wait(&p_full[j & 1], (j >> 1) & 1);
                mbar_wait(&v_full[j % kPuNB], (j / kPuNB) & 1);
                if (tail && j == nblk - 1) mbar_wait(vz_done, 0);
                tc_fence_after();
                const uint32_t pc = tb + C::kPCol + (j & 1) * 64;
                const uint64_t vd = v_d0 + (uint64_t)(((j % kPuNB) * C::kBlk) >> 4);
                const int np = block_pages(j);
#pragma unroll
                for (int q = 0; q < kPuKB; ++q) {
                    if (q < np) {
                        const uint64_t bv = vd + (uint64_t)((q * kPage * 128) >> 4);
                        umma_ts_w(tb + C::kOCol, pc + q * 8, bv, kIdPV, (j > 0 || q > 0) ? 1u : 0u);
                        umma_ts_w(tb + C::kOCol, pc + 32 + q * 8, bv, kIdPV, 1u);
                    }
                }
                umma_commit_w(&v_empty[j % kPuNB]);
                umma_commit_w(&p_free[j & 1]);
            }
        }
} else if (warp < 4) {
        // ============================================================ softmax (thread = row)
        const int r = tid, j = r / T, i_tok = r - j * T;
        const bool valid = j < gs && t0 + i_tok < p.ntok;
        const int pos = n0 + t0 + i_tok;
        const float sl2 = p.scale_log2;
        const uint32_t lane_base = tbase + ((uint32_t)(warp * 32) << 16);
        float m = -INFINITY, l = 0.f;
        for (int i = 0; i < nblk; ++i) {
            mbar_wait(&s_full[i & 1], (i >> 1) & 1);
            tc_fence_after();
            float x[kPuBT];
            {
                uint32_t v0[32], v1[32];
                tmem_ld32(lane_base + C::kSCol + (i & 1) * kPuBT, v0);
                tmem_ld32(lane_base + C::kSCol + (i & 1) * kPuBT + 32, v1);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    x[c] = __uint_as_float(v0[c]);
                    x[32 + c] = __uint_as_float(v1[c]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_free[i & 1]);
#ifdef EXP_PFNOSM
            if (i >= 2) mbar_wait(&p_free[i & 1], ((i - 2) >> 1) & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[i & 1]);
            continue;
#endif
            float bmax = -INFINITY;
            const int tk0 = i * kPuBT;
#pragma unroll
            for (int c = 0; c < kPuBT; ++c) {
                x[c] = (valid && tk0 + c <= pos) ? x[c] * sl2 : -INFINITY;
                bmax = fmaxf(bmax, x[c]);
            }
            const bool raise = bmax > m + kPuRaise || (m == -INFINITY && bmax > -INFINITY);
            const float m_new = raise ? fmaxf(m, bmax) : m;
            const bool rescale = raise && l > 0.f;
            if (__any_sync(0xffffffffu, rescale)) {
                mbar_wait(&p_free[(i - 1) & 1], ((i - 1) >> 1) & 1);
                tc_fence_after();
                const float al = rescale ? ex2(m - m_new) : 1.f;
#pragma unroll
                for (int c0 = 0; c0 < D; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(lane_base + C::kOCol + c0, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(__uint_as_float(v[c]) * al);
                    tmem_st32(lane_base + C::kOCol + c0, v);
                }
                tmem_wait_st();
                l *= al;
            }
            m = m_new;
            const float msafe = m == -INFINITY ? 0.f : m;
            if (i >= 2) mbar_wait(&p_free[i & 1], ((i - 2) >> 1) & 1);  // PV(i - 2) done with this P buffer
            tc_fence_after();
            uint32_t hw[32], lw[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const float p0 = ex2(x[2 * c] - msafe), p1 = ex2(x[2 * c + 1] - msafe);
                l += p0 + p1;
                const __nv_bfloat162 hv = __floats2bfloat162_rn(p0, p1);
                const float2 hf = __bfloat1622float2(hv);
                hw[c] = *reinterpret_cast<const uint32_t*>(&hv);
                lw[c] = pack_bf16(p0 - hf.x, p1 - hf.y);
            }
            tmem_st32(lane_base + C::kPCol + (i & 1) * 64, hw);
            tmem_st32(lane_base + C::kPCol + (i & 1) * 64 + 32, lw);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[i & 1]);
        }
        // ------------------------------------------------------------ epilogue: O / l
        if (nblk > 0) mbar_wait(&p_free[(nblk - 1) & 1], ((nblk - 1) >> 1) & 1);  // the last PV completed
        tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        float* dst = p.out + (((size_t)b * p.ntok + t0 + i_tok) * p.m + h * gs + j) * D;
        bool bad = false;
#pragma unroll
        for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t v[32];
            tmem_ld32(lane_base + C::kOCol + c0, v);
            tmem_wait_ld();
            if (valid) {
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    const float4 o = make_float4(__uint_as_float(v[c]) * inv, __uint_as_float(v[c + 1]) * inv,
                                                 __uint_as_float(v[c + 2]) * inv, __uint_as_float(v[c + 3]) * inv);
                    bad |= !(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w));
                    *reinterpret_cast<float4*>(dst + c0 + c) = o;
                }
            }
        }
        if (valid && p.lse_out)
            p.lse_out[((size_t)b * p.ntok + t0 + i_tok) * p.m + h * gs + j] =
                l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
        if (bad) set_err(p.err, kDevNumeric);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::kTmemCols));
}

// ================================================================================================
// Two query tiles per CTA on the converged-issue pipeline (pfumma = 3): tiles A = 2c and B = 2c + 1
// of one (kv head, sequence) share every K / V block and alternate on the tensor core — S_A(i),
// S_B(i), then PV_A(i - 1), PV_B(i - 1) — so one tile's softmax runs while the other tile's MMAs
// execute.  TMEM budget (512 columns): per tile two 64-column S/P buffers — the softmax writes P(i)
// (hi [0, 32), lo [32, 64)) over the S(i) it has read — and O; Q of both tiles in shared memory.
// S_X(i) reuses the buffer of PV_X(i - 2): the MMA warp waits for that PV's completion first (an
// MMA writing TMEM columns an earlier MMA still reads is not ordered for us: without the wait the
// results were wrong), so the softmax never waits for the previous PV before writing its P.
constexpr int kPu3Threads = 352;  // softmax of A: warps 0-3, of B: 4-7; K producer 8, MMA 9, V producer 10

template <int D>
struct Pu3Cfg {
    static constexpr int kHalves = D / 64;
    static constexpr int kQ = kHalves * 128 * 128;               // one tile's Q: [half][128 rows][128 B]
    static constexpr int kBlk = kHalves * kPuBT * 128;
    static constexpr int oQ = 0;
    static constexpr int oK = oQ + 2 * kQ;
    static constexpr int oV = oK + kPuNB * kBlk;
    static constexpr int oBar = oV + kPuNB * kBlk;
    static constexpr int nBar = 4 * kPuNB + 1 + 3 * 4;
    static constexpr int kSmem = 1024 + oBar + nBar * 8 + 16;
    static constexpr int kTmemCols = 512;
    static constexpr int kTile = 256;                            // TMEM columns per tile: S/P 2 x 64, O at +128
};

__device__ __forceinline__ void umma_ss_w(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int D>
__global__ void __launch_bounds__(kPu3Threads, 1)
prefill_umma3_kernel(const __grid_constant__ CUtensorMap tm_kv, const PrefillParams p) {
    using C = Pu3Cfg<D>;
    extern __shared__ __align__(16) uint8_t pu_smem[];
    uint8_t* base = pu_smem + ((1024u - (smem_u32(pu_smem) & 1023u)) & 1023u);
    uint8_t* kring = base + C::oK;
    uint8_t* vring = base + C::oV;
    uint64_t* k_full = reinterpret_cast<uint64_t*>(base + C::oBar);
    uint64_t* k_empty = k_full + kPuNB;
    uint64_t* v_full = k_empty + kPuNB;
    uint64_t* v_empty = v_full + kPuNB;
    uint64_t* vz_done = v_empty + kPuNB;
    uint64_t* s_full = vz_done + 1;   // [tile][buffer]: S landed
    uint64_t* p_full = s_full + 4;    // [tile][buffer]: the softmax wrote P
    uint64_t* p_free = p_full + 4;    // [tile][buffer]: PV completed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_free + 4);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gs = p.gs, T = 128 / gs;
    const int ntiles = (p.ntok + T - 1) / T;
    const int pair = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, b = blockIdx.z;  // longest rows first
    const bool hasB = 2 * pair + 1 < ntiles;

    if (tid == 0) {
        for (int i = 0; i < kPuNB; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
        }
        mbar_init(vz_done, 1);
        for (int i = 0; i < 4; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);
            mbar_init(&p_free[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp == 8 && lane == 0) tma_prefetch_desc(&tm_kv);
    pdl_wait();  // the chunk's append (previous kernel) wrote the pool rows and the length
    const int s_tot = p.seq_len[p.layer * p.max_batch + b] / p.g;  // raw counter = n * g
    const int n0 = s_tot - p.ntok;
    auto tile_blocks = [&](int x) {
        const int kv_end = n0 + min(p.ntok, (2 * pair + x) * T + T);
        return ((kv_end + kPage - 1) / kPage + kPuKB - 1) / kPuKB;
    };
    const int nblkA = tile_blocks(0);
    const int nblk = hasB ? tile_blocks(1) : nblkA;
    const int kv_end = n0 + min(p.ntok, (2 * pair + (hasB ? 1 : 0)) * T + T);
    const int n_pages = (kv_end + kPage - 1) / kPage;
    if (warp < 8) {  // Q rows of tile warp / 4 (thread = row), K-major SW128
        const int x = warp >> 2, r = tid & 127, j = r / T, i = r - j * T;
        const int t0 = (2 * pair + x) * T;
        const bool valid = (x == 0 || hasB) && j < gs && t0 + i < p.ntok;
        const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.q) +
                                                          (((size_t)b * p.ntok + t0 + i) * p.m + h * gs + j) * D);
        uint8_t* qs = base + C::oQ + x * C::kQ;
#pragma unroll
        for (int c = 0; c < D / 8; ++c) {
            const uint4 v = valid ? src[c] : make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(qs + (c >> 3) * 16384 + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_launch_dependents();
    const uint32_t tbase = *tmem_slot;
    const size_t layer_ph = (size_t)p.layer * p.num_phys;
    const int32_t* bt = p.block_table + (size_t)b * p.bt_stride;
    auto block_pages = [&](int i) { return min(kPuKB, n_pages - i * kPuKB); };
    const bool tail = (kv_end % kPage) != 0;

    if (warp == 8 || warp == 10) {
        // ============================================================ TMA producers (K: 8, V: 10)
        const bool is_v = warp == 10;
        uint8_t* ring = is_v ? vring : kring;
        uint64_t* fullb = is_v ? v_full : k_full;
        uint64_t* emptyb = is_v ? v_empty : k_empty;
        if (lane == 0) {
            for (int i = 0; i < nblk; ++i) {
                const int slot = i % kPuNB, round = i / kPuNB;
                if (round > 0) mbar_wait(&emptyb[slot], (round - 1) & 1);
                const int np = block_pages(i);
                mbar_arrive_expect_tx(&fullb[slot], np * C::kHalves * kPage * 128);
                for (int q = 0; q < np; ++q) {
                    const int row0 = (int)kv_row(layer_ph + bt[i * kPuKB + q], p.g, h, 0) + (is_v ? kPage : 0);
#pragma unroll
                    for (int hf = 0; hf < C::kHalves; ++hf) {
                        uint8_t* dst = ring + slot * C::kBlk + hf * (kPuBT * 128) + q * kPage * 128;
                        if (D == 64) tma_load_2d(dst, &tm_kv, &fullb[slot], 0, row0, kEvictNormal);
                        else tma_load_3d(dst, &tm_kv, &fullb[slot], 0, row0, hf, kEvictNormal);
                    }
                }
            }
        }
        __syncwarp();
        if (is_v && tail && nblk > 0) {  // V rows past the end of the last page: 0
            const int i = nblk - 1, slot = i % kPuNB, q = block_pages(i) - 1, r0 = kv_end % kPage;
            mbar_wait(&v_full[slot], (i / kPuNB) & 1);
            uint8_t* vb = vring + slot * C::kBlk;
            for (int ch = lane; ch < C::kHalves * (kPage - r0) * 8; ch += 32) {
                const int hf = ch / ((kPage - r0) * 8), rem = ch - hf * (kPage - r0) * 8;
                const int r = q * kPage + r0 + rem / 8, c = rem % 8;
                *reinterpret_cast<uint4*>(vb + hf * (kPuBT * 128) + r * 128 + ((c ^ (r & 7)) << 4)) = make_uint4(0, 0, 0, 0);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(vz_done);
        }
    } else if (warp == 9) {
        // ============================================================ MMA issuer (converged warp)
        constexpr uint32_t kIdS = umma_idesc(128, kPuBT, 0, 0);  // A = Q (smem), B = K rows K-major
        constexpr uint32_t kIdPV = umma_idesc(128, D, 0, 1);     // A = P (TMEM), B = V MN-major
        const uint32_t tb = __shfl_sync(0xffffffffu, tbase, 0);
        const uint64_t k_d0 = umma_desc(smem_u32(kring), 16, 1024, kLayoutSW128);
        const uint64_t v_d0 = umma_desc(smem_u32(vring), D == 128 ? kPuBT * 128 : 0, 1024, kLayoutSW128);
        const uint64_t q_d0 = umma_desc(smem_u32(base + C::oQ), 16, 1024, kLayoutSW128);
        for (int i = 0; i <= nblk; ++i) {
            if (i < nblk) {  // S_A(i), S_B(i)
                mbar_wait(&k_full[i % kPuNB], (i / kPuNB) & 1);
                tc_fence_after();
                const uint64_t kd = k_d0 + (uint64_t)(((i % kPuNB) * C::kBlk) >> 4);
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    if (x == 0 ? i >= nblkA : !hasB) continue;
                    if (i >= 2) {
                        mbar_wait(&p_free[x * 2 + (i & 1)], ((i - 2) >> 1) & 1);  // PV_X(i - 2) left the buffer
                        tc_fence_after();
                    }
                    const uint64_t qd = q_d0 + (uint64_t)((x * C::kQ) >> 4);
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = (uint32_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
                        const uint32_t offk = (uint32_t)((((kk >> 2) * (kPuBT * 128)) + (kk & 3) * 32) >> 4);
                        umma_ss_w(tb + x * C::kTile + (i & 1) * 64, qd + off, kd + offk, kIdS, kk > 0 ? 1u : 0u);
                    }
                    umma_commit_w(&s_full[x * 2 + (i & 1)]);
                }
                umma_commit_w(&k_empty[i % kPuNB]);
            }
            if (i >= 1) {  // PV_A(i - 1), PV_B(i - 1), each after its softmax wrote P over its S
                const int j = i - 1;
                mbar_wait(&v_full[j % kPuNB], (j / kPuNB) & 1);
                if (tail && j == nblk - 1) mbar_wait(vz_done, 0);
                const uint64_t vd = v_d0 + (uint64_t)(((j % kPuNB) * C::kBlk) >> 4);
                const int np = block_pages(j);
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    if (x == 0 ? j >= nblkA : !hasB) continue;
                    mbar_wait(&p_full[x * 2 + (j & 1)], (j >> 1) & 1);
                    tc_fence_after();
                    const uint32_t pc = tb + x * C::kTile + (j & 1) * 64;
#pragma unroll
                    for (int q = 0; q < kPuKB; ++q) {
                        if (q < np) {
                            const uint64_t bv = vd + (uint64_t)((q * kPage * 128) >> 4);
                            umma_ts_w(tb + x * C::kTile + 128, pc + q * 8, bv, kIdPV, (j > 0 || q > 0) ? 1u : 0u);
                            umma_ts_w(tb + x * C::kTile + 128, pc + 32 + q * 8, bv, kIdPV, 1u);
                        }
                    }
                    umma_commit_w(&p_free[x * 2 + (j & 1)]);
                }
                umma_commit_w(&v_empty[j % kPuNB]);
            }
        }
    } else if (warp < 8) {
        // ============================================================ softmax (thread = row of tile x)
        const int x = warp >> 2, qd = warp & 3, r = qd * 32 + lane, j = r / T, i_tok = r - j * T;
        const int t0 = (2 * pair + x) * T;
        const bool present = x == 0 || hasB;
        const bool valid = present && j < gs && t0 + i_tok < p.ntok;
        const int nb = present ? (x == 0 ? nblkA : nblk) : 0;
        const int pos = n0 + t0 + i_tok;
        const float sl2 = p.scale_log2;
        const uint32_t lane_base = tbase + ((uint32_t)(qd * 32) << 16) + x * C::kTile;
        float m = -INFINITY, l = 0.f;
        for (int i = 0; i < nb; ++i) {
            mbar_wait(&s_full[x * 2 + (i & 1)], (i >> 1) & 1);
            tc_fence_after();
            float xs[kPuBT];
            {
                uint32_t v0[32], v1[32];
                tmem_ld32(lane_base + (i & 1) * 64, v0);
                tmem_ld32(lane_base + (i & 1) * 64 + 32, v1);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    xs[c] = __uint_as_float(v0[c]);
                    xs[32 + c] = __uint_as_float(v1[c]);
                }
            }
            float bmax = -INFINITY;
            const int tk0 = i * kPuBT;
#pragma unroll
            for (int c = 0; c < kPuBT; ++c) {
                xs[c] = (valid && tk0 + c <= pos) ? xs[c] * sl2 : -INFINITY;
                bmax = fmaxf(bmax, xs[c]);
            }
            const bool raise = bmax > m + kPuRaise || (m == -INFINITY && bmax > -INFINITY);
            const float m_new = raise ? fmaxf(m, bmax) : m;
            const bool rescale = raise && l > 0.f;
            if (__any_sync(0xffffffffu, rescale)) {  // O holds earlier blocks: wait for PV(i - 1)
                mbar_wait(&p_free[x * 2 + ((i - 1) & 1)], ((i - 1) >> 1) & 1);
                tc_fence_after();
                const float al = rescale ? ex2(m - m_new) : 1.f;
#pragma unroll
                for (int c0 = 0; c0 < D; c0 += 32) {
                    uint32_t v[32];
                    tmem_ld32(lane_base + 128 + c0, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(__uint_as_float(v[c]) * al);
                    tmem_st32(lane_base + 128 + c0, v);
                }
                tmem_wait_st();
                l *= al;
            }
            m = m_new;
            const float msafe = m == -INFINITY ? 0.f : m;
            uint32_t hw[32], lw[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const float p0 = ex2(xs[2 * c] - msafe), p1 = ex2(xs[2 * c + 1] - msafe);
                l += p0 + p1;
                const __nv_bfloat162 hv = __floats2bfloat162_rn(p0, p1);
                const float2 hf = __bfloat1622float2(hv);
                hw[c] = *reinterpret_cast<const uint32_t*>(&hv);
                lw[c] = pack_bf16(p0 - hf.x, p1 - hf.y);
            }
            tmem_st32(lane_base + (i & 1) * 64, hw);  // P over the S it was computed from
            tmem_st32(lane_base + (i & 1) * 64 + 32, lw);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[x * 2 + (i & 1)]);
        }
        // ------------------------------------------------------------ epilogue: O / l
        if (nb > 0) mbar_wait(&p_free[x * 2 + ((nb - 1) & 1)], ((nb - 1) >> 1) & 1);
        tc_fence_after();
        const float inv = l > 0.f ? 1.f / l : 0.f;
        float* dst = p.out + (((size_t)b * p.ntok + t0 + i_tok) * p.m + h * gs + j) * D;
        bool bad = false;
        if (present) {
#pragma unroll
            for (int c0 = 0; c0 < D; c0 += 32) {
                uint32_t v[32];
                tmem_ld32(lane_base + 128 + c0, v);
                tmem_wait_ld();
                if (valid) {
#pragma unroll
                    for (int c = 0; c < 32; c += 4) {
                        const float4 o = make_float4(__uint_as_float(v[c]) * inv, __uint_as_float(v[c + 1]) * inv,
                                                     __uint_as_float(v[c + 2]) * inv, __uint_as_float(v[c + 3]) * inv);
                        bad |= !(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w));
                        *reinterpret_cast<float4*>(dst + c0 + c) = o;
                    }
                }
            }
        }
        if (valid && p.lse_out)
            p.lse_out[((size_t)b * p.ntok + t0 + i_tok) * p.m + h * gs + j] =
                l > 0.f ? (m + log2f(l)) * kLn2 : -INFINITY;
        if (bad) set_err(p.err, kDevNumeric);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::kTmemCols));
}

}  // namespace

bool prefill_umma_supported(const PrefillParams& p) { return (p.d == 128 || p.d == 64) && p.gs <= 16; }

cudaError_t launch_prefill_umma2(const PrefillParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl) {
    const void* fn = p.d == 128 ? (const void*)prefill_umma2_kernel<128> : (const void*)prefill_umma2_kernel<64>;
    const int smem = p.d == 128 ? Pu2Cfg<128>::kSmem : Pu2Cfg<64>::kSmem;
    static std::atomic<int> cache[kMaxDevices * 2];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    const int slot = dev * 2 + (p.d == 128 ? 0 : 1);
    if (cache[slot].load(std::memory_order_acquire) == 0) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        cache[slot].store(1, std::memory_order_release);
    }
    const int T = 128 / p.gs;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((p.ntok + T - 1) / T, p.g, p.batch);
    cfg.blockDim = dim3(kPuThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    void* args[] = {const_cast<CUtensorMap*>(tm_kv), const_cast<PrefillParams*>(&p)};
    return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_prefill_umma3(const PrefillParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl) {
    const void* fn = p.d == 128 ? (const void*)prefill_umma3_kernel<128> : (const void*)prefill_umma3_kernel<64>;
    const int smem = p.d == 128 ? Pu3Cfg<128>::kSmem : Pu3Cfg<64>::kSmem;
    static std::atomic<int> cache[kMaxDevices * 2];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    const int slot = dev * 2 + (p.d == 128 ? 0 : 1);
    if (cache[slot].load(std::memory_order_acquire) == 0) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        cache[slot].store(1, std::memory_order_release);
    }
    const int T = 128 / p.gs, ntiles = (p.ntok + T - 1) / T;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((ntiles + 1) / 2, p.g, p.batch);
    cfg.blockDim = dim3(kPu3Threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    void* args[] = {const_cast<CUtensorMap*>(tm_kv), const_cast<PrefillParams*>(&p)};
    return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_prefill_umma(const PrefillParams& p, const CUtensorMap* tm_kv, cudaStream_t st, bool pdl) {
    const void* fn = p.d == 128 ? (const void*)prefill_umma_kernel<128> : (const void*)prefill_umma_kernel<64>;
    const int smem = p.d == 128 ? PuCfg<128>::kSmem : PuCfg<64>::kSmem;
    static std::atomic<int> cache[kMaxDevices * 2];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    const int slot = dev * 2 + (p.d == 128 ? 0 : 1);
    if (cache[slot].load(std::memory_order_acquire) == 0) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        cache[slot].store(1, std::memory_order_release);
    }
    const int T = 128 / p.gs;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((p.ntok + T - 1) / T, p.g, p.batch);
    cfg.blockDim = dim3(kPuThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    void* args[] = {const_cast<CUtensorMap*>(tm_kv), const_cast<PrefillParams*>(&p)};
    return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace delta
