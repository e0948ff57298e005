// shard.cu — sequence sharding across GPUs: the cross-rank merges.
//
// Each rank holds a contiguous, page-aligned share of every sequence's KV pages and runs the
// same decode kernels over its share.  Two exchanges per Delta layer, one per other layer:
//  1. LSE merge.  Every rank's attention kernel leaves a partial (o_r normalised over the
//     rank's tokens, lse_r = log of its softmax denominator); after an all-gather,
//     shard_merge_kernel forms, in fixed rank order,
//         LSE = log sum_r exp(lse_r),   O = sum_r exp(lse_r - LSE) o_r
//     — the identity that any partition of the attended set gives the same softmax (Eq.4,
//     PAPER.md:61-67).  Every rank ends with identical O and LSE.
//  2. Global top-k.  Scores need the global LSE, so each rank scores its own units after (1),
//     exports its local top-k candidates (select.cu, shard_mode 1), and after an all-gather
//     cand_scatter_kernel rebuilds a dense key array (-inf for units no rank proposed);
//     select.cu (shard_mode 2) then runs the unchanged forced-union + top-k on it.  Exact:
//     every member of the global top-k is in its own rank's local top-k, and both use the
//     same (key desc, index asc) order (R9).
#include "combine.cuh"

namespace delta {
namespace {

__global__ void __launch_bounds__(128) shard_merge_kernel(const ShardMergeParams p) {
    pdl_wait();
    pdl_launch_dependents();
    const int bj = blockIdx.x;  // b * m + j
    const int b = bj / p.m, j = bj - b * p.m;
    float M = -INFINITY;
    for (int r = 0; r < p.world; ++r) M = fmaxf(M, p.recv_lse[r * p.lse_stride + bj]);
    float L = 0.f;
    for (int r = 0; r < p.world; ++r) {
        const float l = p.recv_lse[r * p.lse_stride + bj];
        L += (M == -INFINITY || l == -INFINITY) ? 0.f : expf(l - M);
    }
    const float LSE = (L > 0.f) ? M + logf(L) : -INFINITY;
    bool bad = false;
    for (int c4 = threadIdx.x; c4 < p.d / 4; c4 += blockDim.x) {
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 0; r < p.world; ++r) {
            const float l = p.recv_lse[r * p.lse_stride + bj];
            const float w = (LSE == -INFINITY || l == -INFINITY) ? 0.f : expf(l - LSE);
            const float4 v = reinterpret_cast<const float4*>(p.recv_o + r * p.o_stride + (size_t)bj * p.d)[c4];
            o.x += w * v.x; o.y += w * v.y; o.z += w * v.z; o.w += w * v.w;
        }
        bad |= !(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(o.w));
        reinterpret_cast<float4*>(p.out + (size_t)bj * p.d)[c4] = o;
    }
    if (threadIdx.x == 0) {
        if (p.lse_out) p.lse_out[(size_t)b * p.m + j] = LSE;
        if (p.role == kRoleSelect) p.lse_buf[(size_t)b * p.m + j] = LSE;
    }
    if (bad) set_err(p.err, kDevNumeric);
}

__global__ void __launch_bounds__(256) cand_scatter_kernel(const uint2* __restrict__ recv, int world, int k_slots,
                                                           size_t rank_stride, float* keys, int max_units,
                                                           const int32_t* seq_len, int layer, int max_batch,
                                                           int g, int sel_block) {
    pdl_wait();
    const int b = blockIdx.x;
    const int s = seq_len[layer * max_batch + b] / g;  // raw counter = n * g
    const int n_units = (s + sel_block - 1) / sel_block;
    float* kb = keys + (size_t)b * max_units;
    for (int u = threadIdx.x; u < n_units; u += blockDim.x) kb[u] = -INFINITY;
    __syncthreads();
    for (int r = 0; r < world; ++r) {
        const uint2* c = recv + r * rank_stride + (size_t)b * k_slots;
        for (int i = threadIdx.x; i < k_slots; i += blockDim.x) {
            const uint2 v = c[i];
            if ((int)v.y >= 0 && (int)v.y < n_units) kb[v.y] = __uint_as_float(v.x);  // each unit: one owner
        }
    }
    __syncthreads();
    pdl_launch_dependents();
}

}  // namespace

cudaError_t launch_shard_merge(const ShardMergeParams& p, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.batch * p.m);
    cfg.blockDim = dim3(32);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, shard_merge_kernel, p);
}

cudaError_t launch_cand_scatter(const uint2* recv, int world, int batch, int k_slots, size_t rank_stride, float* keys,
                                int max_units, const int32_t* seq_len, int layer, int max_batch, int g, int sel_block,
                                cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(batch);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, cand_scatter_kernel, recv, world, k_slots, rank_stride, keys, max_units, seq_len,
                              layer, max_batch, g, sel_block);
}

}  // namespace delta
