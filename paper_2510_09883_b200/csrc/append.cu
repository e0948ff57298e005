// append.cu — Eq.7 KV append: K <- [K; k_new], V <- [V; v_new] for one
// layer; token i of sequence b goes to position n_b + i = page block_table[b][pos/P],
// slot pos % P, then seq_len[b] grows by ntok.  The cache is append-only.
// One CTA per sequence, 16-byte vector copies.
#include "combine.cuh"

namespace delta {
namespace {

__global__ void __launch_bounds__(256) append_kernel(const AppendParams p) {
    const int b = blockIdx.x;
    pdl_wait();
    pdl_launch_dependents();
    const int n = p.seq_len[p.layer * p.max_batch + b] / p.g;  // raw counter = n * g
    if (n + p.ntok > p.max_seq) {
        if (threadIdx.x == 0) set_err(p.err, kDevCapacity);
        return;
    }
    const int row_bytes = p.d * p.elem_bytes;        // one head row
    const int chunks = row_bytes / 16;               // 16-byte chunks per row
    const int total = p.ntok * p.g * chunks;
    const uint8_t* ks = reinterpret_cast<const uint8_t*>(p.k_new) + (size_t)b * p.ntok * p.g * row_bytes;
    const uint8_t* vs = reinterpret_cast<const uint8_t*>(p.v_new) + (size_t)b * p.ntok * p.g * row_bytes;
    const int32_t* bt = p.block_table + (size_t)b * p.bt_stride;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
        const int c = i % chunks;
        const int hh = (i / chunks) % p.g;
        const int tok = i / (chunks * p.g);
        const int t = n + tok;
        if (t / kPage < p.page_lo || t / kPage >= p.page_hi) continue;  // another rank's page
        const size_t row = kv_row((size_t)p.layer * p.num_phys + bt[t / kPage], p.g, hh, t % kPage);
        const size_t src_off = ((size_t)tok * p.g + hh) * row_bytes + (size_t)c * 16;
        const size_t dst_off = row * row_bytes + (size_t)c * 16;
        uint8_t* pool = reinterpret_cast<uint8_t*>(p.kv_pool);
        *reinterpret_cast<uint4*>(pool + dst_off) = *reinterpret_cast<const uint4*>(ks + src_off);
        *reinterpret_cast<uint4*>(pool + dst_off + (size_t)kPage * row_bytes) =
            *reinterpret_cast<const uint4*>(vs + src_off);
    }
    // Quest page representatives (quest.cu): thread owns (head, bf16 pair) and folds the
    // appended tokens in order; a token in slot 0 starts its page's min/max.
    if (p.reps) {
        const int pairs = p.d / 2;
        const __nv_bfloat162* kn = reinterpret_cast<const __nv_bfloat162*>(ks);
        for (int i = threadIdx.x; i < p.g * pairs; i += blockDim.x) {
            const int hh = i / pairs, e2 = i - hh * pairs;
            int cur = -1;
            __nv_bfloat162 mn, mx;
            __nv_bfloat162* rep = nullptr;
            for (int tok = 0; tok < p.ntok; ++tok) {
                const int t = n + tok, u = t / kPage;
                if (u < p.page_lo || u >= p.page_hi) continue;
                const __nv_bfloat162 k = kn[((size_t)tok * p.g + hh) * pairs + e2];
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
    __syncthreads();
    if (threadIdx.x == 0) p.seq_len[p.layer * p.max_batch + b] = (n + p.ntok) * p.g;
}

}  // namespace

cudaError_t launch_append(const AppendParams& p, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.batch);
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
