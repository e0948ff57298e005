// recall.cu — attention recall, Eq.9: for head j of layer i,
//   R_j = sum_{u in rho} alpha_j(u) / sum_{u=1..s} alpha_j(u),  alpha_j = softmax(A_j),
// the fraction of the layer's exact full-attention mass that its selected set keeps (NEXT-2,
// a diagnostic pass, not part of the timed step).  alpha_j(t) = exp(a_j(t) - LSE_j) from the
// scaled logits and LSE of a full-attention probe of the layer (attn kernels, SELECT role).
// rho = the plan the layer attends (page or token units -> tokens t < s).
// One CTA per sequence; thread (head j = tid % m, lane group r = tid / m) sums a fixed strided
// share of the tokens in ascending order, then the groups are added in fixed order:
// deterministic.
#include "combine.cuh"

namespace delta {
namespace {

__global__ void __launch_bounds__(256) recall_kernel(const RecallParams p) {
    extern __shared__ float sred[];  // [2][groups][m]
    const int b = blockIdx.x, tid = threadIdx.x;
    pdl_wait();
    const int s = p.seq_len[p.layer * p.max_batch + b] / p.g;
    const int groups = blockDim.x / p.m;
    const int j = tid % p.m, r = tid / p.m;
    const float* lg = p.logits + (size_t)b * p.max_seq * p.m;
    const float lse = p.lse[(size_t)b * p.m + j];
    float num = 0.f, den = 0.f;
    if (r < groups) {
        for (int t = r; t < s; t += groups) den += expf(lg[(size_t)t * p.m + j] - lse);
        const int cnt = p.plan_count[b];
        const int32_t* plan = p.plan_idx + (size_t)b * p.plan_cap;
        for (int i = r; i < cnt; i += groups) {
            const int u = plan[i];
            for (int t = u * p.sel_block; t < (u + 1) * p.sel_block && t < s; ++t)
                num += expf(lg[(size_t)t * p.m + j] - lse);
        }
        sred[r * p.m + j] = num;
        sred[(groups + r) * p.m + j] = den;
    }
    __syncthreads();
    if (tid < p.m) {
        float n = 0.f, d = 0.f;
        for (int k = 0; k < groups; ++k) {
            n += sred[k * p.m + tid];
            d += sred[(groups + k) * p.m + tid];
        }
        p.recall_out[(size_t)b * p.m + tid] = d > 0.f ? n / d : 0.f;
    }
}

}  // namespace

cudaError_t launch_recall(const RecallParams& p, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.batch);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 2 * 256 * sizeof(float);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, recall_kernel, p);
}

}  // namespace delta
