// append.cu — Eq.7 KV append: K <- [K; k_new], V <- [V; v_new] for one
// layer; token i of sequence b goes to position n_b + i = page block_table[b][pos/P],
// slot pos % P, then seq_len[b] grows by ntok.  The cache is append-only.
// One CTA per sequence, 16-byte vector copies.
#include "combine.cuh"

namespace delta {
namespace {

// CTA (c, b) handles the pages [n/P + c*kPagesPerCta, ... + kPagesPerCta) of the chunk of
// sequence b (a page is never split between CTAs, so the Quest reps fold stays sequential per
// page); with several CTAs the last to arrive (ticket) publishes the new length, after every
// CTA has read the old one.
constexpr int kPagesPerCta = 4;

__global__ void __launch_bounds__(256) append_kernel(const AppendParams p) {
    const int c = blockIdx.x, b = blockIdx.y;
    pdl_wait();
    pdl_launch_dependents();
    const int n = p.seq_len[p.layer * p.max_batch + b] / p.g;  // raw counter = n * g
    if (n + p.ntok > p.max_seq) {
        if (threadIdx.x == 0 && c == 0) set_err(p.err, kDevCapacity);
        return;
    }
    const int u_lo = n / kPage + c * kPagesPerCta;
    const int t_lo = max(n, u_lo * kPage), t_hi = min(n + p.ntok, (u_lo + kPagesPerCta) * kPage);
    const int row_bytes = p.d * p.elem_bytes;        // one head row
    const int chunks = row_bytes / 16;               // 16-byte chunks per row
    const uint8_t* __restrict__ ks = reinterpret_cast<const uint8_t*>(p.k_new) + (size_t)b * p.ntok * p.g * row_bytes;
    const uint8_t* __restrict__ vs = reinterpret_cast<const uint8_t*>(p.v_new) + (size_t)b * p.ntok * p.g * row_bytes;
    const int32_t* __restrict__ bt = p.block_table + (size_t)b * p.bt_stride;
    uint8_t* pool = reinterpret_cast<uint8_t*>(p.kv_pool);
    if (t_lo < t_hi) {
        const int total = (t_hi - t_lo) * p.g * chunks;
        constexpr int kUnroll = 4;  // independent 16-byte loads in flight per thread
        for (int i0 = threadIdx.x; i0 < total; i0 += kUnroll * blockDim.x) {
            uint4 kx[kUnroll], vx[kUnroll];
            size_t dst[kUnroll];
#pragma unroll
            for (int r = 0; r < kUnroll; ++r) {
                const int i = i0 + r * blockDim.x;
                if (i < total) {
                    const int cc = i % chunks;
                    const int hh = (i / chunks) % p.g;
                    const int t = t_lo + i / (chunks * p.g);
                    const size_t src_off = ((size_t)(t - n) * p.g + hh) * row_bytes + (size_t)cc * 16;
                    kx[r] = *reinterpret_cast<const uint4*>(ks + src_off);
                    vx[r] = *reinterpret_cast<const uint4*>(vs + src_off);
                    const bool own = t / kPage >= p.page_lo && t / kPage < p.page_hi;  // sequence sharding
                    dst[r] = own ? kv_row((size_t)p.layer * p.num_phys + bt[t / kPage], p.g, hh, t % kPage) * row_bytes +
                                       (size_t)cc * 16
                                 : ~size_t(0);
                }
            }
#pragma unroll
            for (int r = 0; r < kUnroll; ++r) {
                const int i = i0 + r * blockDim.x;
                if (i < total && dst[r] != ~size_t(0)) {
                    *reinterpret_cast<uint4*>(pool + dst[r]) = kx[r];
                    *reinterpret_cast<uint4*>(pool + dst[r] + (size_t)kPage * row_bytes) = vx[r];
                }
            }
        }
        // Quest page representatives (quest.cu): thread owns (head, bf16 pair) and folds this
        // CTA's tokens in order; a token in slot 0 starts its page's min/max.
        if (p.reps) {
            const int pairs = p.d / 2;
            const __nv_bfloat162* kn = reinterpret_cast<const __nv_bfloat162*>(ks);
            for (int i = threadIdx.x; i < p.g * pairs; i += blockDim.x) {
                const int hh = i / pairs, e2 = i - hh * pairs;
                int cur = -1;
                __nv_bfloat162 mn, mx;
                __nv_bfloat162* rep = nullptr;
                for (int t = t_lo; t < t_hi; ++t) {
                    const int u = t / kPage;
                    if (u < p.page_lo || u >= p.page_hi) continue;
                    const __nv_bfloat162 k = kn[((size_t)(t - n) * p.g + hh) * pairs + e2];
                    if (u != cur) {
                        if (rep) { rep[e2] = mn; rep[pairs + e2] = mx; }
                        rep = reinterpret_cast<__nv_bfloat162*>(p.reps) +
                              (((size_t)p.layer * p.num_phys + bt[u]) * p.g + hh) * p.d;
                        cur = u;
                        if (t % kPage == 0) { mn = k; mx = k; }
                        else { mn = __hmin2(rep[e2], k); mx = __hmax2(rep[pairs + e2], k); }
                    } else {
                        mn = __hmin2(mn, k);
                        mx = __hmax2(mx, k);
                    }
                }
                if (rep) { rep[e2] = mn; rep[pairs + e2] = mx; }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (gridDim.x == 1) {
            p.seq_len[p.layer * p.max_batch + b] = (n + p.ntok) * p.g;
        } else {
            int32_t* ticket = p.ticket + (size_t)p.layer * p.max_batch + b;
            int old;
            asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(ticket) : "memory");
            if (old == (int)gridDim.x - 1) {  // every CTA has read the old length
                *ticket = 0;
                p.seq_len[p.layer * p.max_batch + b] = (n + p.ntok) * p.g;
            }
        }
    }
}

}  // namespace

cudaError_t launch_append(const AppendParams& p, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    // pages a chunk of ntok tokens can touch: ceil(ntok / P) + 1
    const int pages = (p.ntok + kPage - 1) / kPage + 1;
    cfg.gridDim = dim3(p.ntok == 1 ? 1 : (pages + kPagesPerCta - 1) / kPagesPerCta, p.batch);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, append_kernel, p);
}

}  // namespace delta
