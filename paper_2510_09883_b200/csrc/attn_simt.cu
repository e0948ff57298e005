// attn_simt.cu — CUDA-core paged decode attention (FULL / SELECT / SPARSE roles) for
// fp32 KV caches (the tiny oracle configuration C0 is fp32) — same math, partials and
// grid combine as attn_tc.cu, but dot products on the FP32 pipe so fp32 inputs are not
// rounded to a tensor-core input type.
//
// CTA = (split, kv head h, sequence b), 4 warps; warp w takes tiles w, w+4, ... of the
// CTA's range (a tile = one 16-token page, or 16 consecutive token-plan entries).
// Lane l owns dims [l*VPL, (l+1)*VPL) of d (VPL = d/32) and the gs query heads of
// the group: per token, partial dots -> warp all-reduce -> online softmax per head
// (log2 domain) -> O_j += p_j v_t.
#include "combine.cuh"

namespace delta {
namespace {

constexpr int NW = 4;

template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

template <typename T, int D>
__global__ void __launch_bounds__(NW * 32) attn_simt_kernel(const AttnParams p) {
    constexpr int VPL = D / 32;
    __shared__ float ms[NW * 16], ls[NW * 16];
    __shared__ __align__(16) float os[NW * 16 * os_stride<D>()];
    __shared__ __align__(16) float cstage[ClusterStage<D>::kBytes / 4];  // peers push partials here

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int split = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    const int gs = p.gs;
    if (tid == 0) {
        cluster_stage_init<D>(cstage, gs);
        fence_mbar_init();
    }
    __syncthreads();
    cluster_arrive_relaxed();
    pdl_wait();
    pdl_launch_dependents();  // after the wait: the next kernel may launch (see attn_tc.cu)

    const int n_old = p.seq_len[p.layer * p.max_batch + b] / p.g;  // raw counter = n * g
    const int s = p.fuse_append ? n_old + 1 : n_old;
    const bool cap_err = s > p.max_seq;
    const bool token_plan = (p.role == kRoleSparse) && p.sel_block == 1;
    bool stale = false;
    int n_items = 0, unit0 = 0, e_end = 0;
    if (!cap_err) split_geometry(p, b, split, s, token_plan, unit0, n_items, e_end, stale);
    const int32_t* bt = p.block_table + (size_t)b * p.bt_stride;
    const int32_t* plan = p.plan_idx + (size_t)b * p.plan_cap;
    const size_t layer_ph = (size_t)p.layer * p.num_phys;
    const T* pool = reinterpret_cast<const T*>(p.kv_pool);
    const T* k_new = reinterpret_cast<const T*>(p.k_new) + ((size_t)b * p.g + h) * D;
    const T* v_new = reinterpret_cast<const T*>(p.v_new) + ((size_t)b * p.g + h) * D;

    if (p.fuse_append && !cap_err && split == 0 && warp == 0 && owns_page(p, (s - 1) / kPage)) {  // Eq.7 append of head h
        const int t = s - 1;
        const size_t row = kv_row(layer_ph + bt[t / kPage], p.g, h, t % kPage);
        T* kd = reinterpret_cast<T*>(p.kv_pool) + row * D;
        T* vd = kd + kPage * D;
        for (int e = lane; e < D; e += 32) { kd[e] = k_new[e]; vd[e] = v_new[e]; }
    }

    float q[kMaxGs][VPL];
    const T* qp = reinterpret_cast<const T*>(p.q) + ((size_t)b * p.m + h * gs) * D;
#pragma unroll
    for (int j = 0; j < kMaxGs; ++j)
#pragma unroll
        for (int v = 0; v < VPL; ++v) q[j][v] = (j < gs) ? ldf(qp + (size_t)j * D + lane * VPL + v) : 0.f;
    float o[kMaxGs][VPL];
    float mj[kMaxGs], lj[kMaxGs];
#pragma unroll
    for (int j = 0; j < kMaxGs; ++j) {
        mj[j] = -INFINITY; lj[j] = 0.f;
#pragma unroll
        for (int v = 0; v < VPL; ++v) o[j][v] = 0.f;
    }

    for (int item = warp; item < n_items; item += NW) {
        for (int r = 0; r < 16; ++r) {
            int t;
            if (!token_plan) {
                const int lp = (p.role == kRoleSparse) ? plan[unit0 + item] : unit0 + item;
                t = lp * kPage + r;
                if (t >= s) break;
            } else {
                const int e = unit0 + item * 16 + r;
                if (e >= e_end) break;
                t = plan[e];
            }
            const T* kr;
            const T* vr;
            if (p.fuse_append && t == s - 1) {
                kr = k_new; vr = v_new;
            } else {
                const size_t row = kv_row(layer_ph + bt[t / kPage], p.g, h, t % kPage);
                kr = pool + row * D; vr = kr + kPage * D;
            }
            float kv[VPL], vv[VPL];
#pragma unroll
            for (int v = 0; v < VPL; ++v) { kv[v] = ldf(kr + lane * VPL + v); vv[v] = ldf(vr + lane * VPL + v); }
#pragma unroll
            for (int j = 0; j < kMaxGs; ++j) {
                if (j >= gs) break;
                float dot = 0.f;
#pragma unroll
                for (int v = 0; v < VPL; ++v) dot = fmaf(q[j][v], kv[v], dot);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, off);
                const float a = dot * p.scale;
                if (p.role == kRoleSelect && lane == 0)
                    p.logits[((size_t)b * p.max_seq + t) * p.m + h * gs + j] = a;
                const float x = dot * p.scale_log2;
                const float mn = fmaxf(mj[j], x);
                const float al = exp2f(mj[j] - mn);  // mj = -inf -> 0
                const float pr = exp2f(x - mn);
                lj[j] = lj[j] * al + pr;
                mj[j] = mn;
#pragma unroll
                for (int v = 0; v < VPL; ++v) o[j][v] = fmaf(pr, vv[v], o[j][v] * al);
            }
        }
    }
    // per-warp states -> smem (m, l replicated across lanes; lane 0 writes them)
#pragma unroll
    for (int j = 0; j < kMaxGs; ++j) {
        if (j >= gs) break;
        if (lane == 0) { ms[warp * 16 + j] = mj[j]; ls[warp * 16 + j] = lj[j]; }
#pragma unroll
        for (int v = 0; v < VPL; ++v) os[(warp * 16 + j) * os_stride<D>() + lane * VPL + v] = o[j][v];
    }
    __syncthreads();
    cluster_epilogue<D, NW>(p, ms, ls, os, cstage, b, h, stale, cap_err, s);
}

template <typename T, int D>
cudaError_t launch_impl(const AttnParams& p0, cudaStream_t st, bool pdl) {
    auto kern = attn_simt_kernel<T, D>;
    static std::atomic<int> cache[kMaxDevices];  // per device: attribute opt-ins are per context
    const int max_cluster = per_device_once(cache, [&] {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) return -1;
        return cluster_limit((const void*)kern, NW * 32, 0);
    });
    if (max_cluster < 1) return cudaErrorInvalidConfiguration;
    AttnParams p = p0;
    p.nsplit = p.nsplit < max_cluster ? p.nsplit : max_cluster;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.nsplit, p.g, p.batch);
    cfg.blockDim = dim3(NW * 32);
    cfg.dynamicSmemBytes = 0;
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
    return cudaLaunchKernelEx(&cfg, kern, p);
}

}  // namespace

cudaError_t launch_attn_simt(const AttnParams& p, bool bf16, cudaStream_t st, bool pdl) {
    if (bf16) {
        if (p.d == 128) return launch_impl<__nv_bfloat16, 128>(p, st, pdl);
        if (p.d == 64) return launch_impl<__nv_bfloat16, 64>(p, st, pdl);
    } else {
        if (p.d == 128) return launch_impl<float, 128>(p, st, pdl);
        if (p.d == 64) return launch_impl<float, 64>(p, st, pdl);
    }
    return cudaErrorInvalidValue;
}

}  // namespace delta
