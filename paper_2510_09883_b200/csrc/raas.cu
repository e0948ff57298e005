// raas.cu — the RaaS eviction policy (NEXT-4; "removes pages with consistently low
// attention scores"; readings RS1-RS4 in DESIGN.md §3) for one layer:
//  * reset: every page < ceil(n/P) retained, last-salient step 0;
//  * update (after the layer attended its retained pages at length s, logits + LSE recorded):
//      S_u = sum_{t in u, t < s} max_j exp(a_j(t) - LSE_j)   (weights renormalised over the
//            attended tokens, R7's max over heads, ascending t, fixed lane order)
//      refresh: S_u >= P / |attended tokens| -> last[u] = s
//      evict:   while more than k/P retained pages are not exempt (sink pages, pages overlapping
//               [s - L, s)): drop the smallest (last[u], u) — for good
//      the page of position s joins when s opens a page (last = s + 1, its creation step);
//    the new ascending retained list is the plan the next step attends (stamp s + 1).
#include "combine.cuh"

namespace delta {
namespace {

constexpr int kRaasThreads = 512;
constexpr int kRaasWarps = kRaasThreads / 32;

__global__ void __launch_bounds__(256) raas_reset_kernel(const RaasParams p) {
    const int b = blockIdx.x;
    pdl_wait();
    const int n = p.seq_len[p.layer * p.max_batch + b] / p.g;
    const int n_pages = (n + kPage - 1) / kPage;
    const int cnt = n_pages + ((n % kPage == 0) ? 1 : 0);  // + the page position n opens
    int32_t* plan = p.plan_idx + (size_t)b * p.plan_cap;
    int32_t* phys = p.plan_phys + (size_t)b * p.plan_cap;
    int32_t* last = p.last + (size_t)b * p.max_pages;
    const int32_t* bt = p.block_table + (size_t)b * p.bt_stride;
    for (int u = threadIdx.x; u < p.max_pages; u += blockDim.x) {
        if (u < cnt && u < p.plan_cap) {
            plan[u] = u;
            phys[u] = bt[u];
        }
        last[u] = (u < n_pages) ? 0 : -1;
    }
    if (threadIdx.x == 0) {
        if (n % kPage == 0 && n_pages < p.max_pages) last[n_pages] = n + 1;
        p.plan_count[b] = min(cnt, p.plan_cap);
        p.plan_stamp[b] = n + 1;
    }
}

// Phase A (kRaasCtas CTAs per sequence): a warp per retained page computes S_u and refreshes
// last[u] in global memory; the CTAs then draw arrival tickets and the last one runs phase B:
// the eviction ranking and the compaction (physical pages from the old plan, no block-table
// loads) for the whole retained set.
constexpr int kRaasCtas = 16;

__global__ void __launch_bounds__(kRaasThreads) raas_update_kernel(const RaasParams p) {
    extern __shared__ int32_t sm[];  // [plan_cap] pages, [plan_cap] last, [plan_cap] phys, [plan_cap] keep
    __shared__ int s_scan[kRaasWarps + 1];
    __shared__ int s_last_cta;
    __shared__ float s_lse[256];  // m <= 256
    const int b = blockIdx.y, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    pdl_wait();
    const int s = p.seq_len[p.layer * p.max_batch + b] / p.g;
    const int cnt = p.plan_count[b];
    int32_t* plan = p.plan_idx + (size_t)b * p.plan_cap;
    int32_t* phys = p.plan_phys + (size_t)b * p.plan_cap;
    int32_t* last = p.last + (size_t)b * p.max_pages;
    // ---- phase A: attended tokens (threshold P / |attended|), scores, refresh
    int nt = 0;
    for (int i = tid; i < cnt; i += kRaasThreads) nt += max(0, min(kPage, s - plan[i] * kPage));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) nt += __shfl_xor_sync(0xffffffffu, nt, off);
    if (lane == 0) s_scan[warp] = nt;
    for (int j = tid; j < p.m; j += kRaasThreads) s_lse[j] = p.lse[(size_t)b * p.m + j];
    __syncthreads();
    int ntok = 0;
    for (int w = 0; w < kRaasWarps; ++w) ntok += s_scan[w];
    const float thr = ntok > 0 ? (float)kPage / (float)ntok : INFINITY;
    const float* lg = p.logits + (size_t)b * p.max_seq * p.m;
    const int jr = lane >> 1, hh = lane & 1;
    for (int i = blockIdx.x * kRaasWarps + warp; i < cnt; i += gridDim.x * kRaasWarps) {
        const int u = plan[i];
        const int t = u * kPage + jr;
        float mx = -INFINITY;
        if (t < s) {
            const float* row = lg + (size_t)t * p.m;
            for (int j0 = hh; j0 < p.m; j0 += 16) {  // 8 independent loads in flight per lane
                float v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = (j0 + 2 * k < p.m) ? __ldcg(row + j0 + 2 * k) : -INFINITY;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (j0 + 2 * k < p.m) mx = fmaxf(mx, v[k] - s_lse[j0 + 2 * k]);
            }
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        const float e = (t < s) ? expf(mx) : 0.f;
        float sum = 0.f;
#pragma unroll
        for (int r = 0; r < kPage; ++r) sum += __shfl_sync(0xffffffffu, e, 2 * r);  // ascending t
        if (lane == 0) {
            p.scores[(size_t)b * p.max_units + u] = sum;
            if (sum >= thr) last[u] = s;
        }
    }
    // ---- arrival: the last CTA of the sequence runs phase B
    __syncthreads();
    if (tid == 0) {
        int old;
        int32_t* ticket = p.ticket + (size_t)p.layer * p.max_batch + b;
        asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(ticket) : "memory");
        s_last_cta = (old == (int)gridDim.x - 1);
        if (s_last_cta) *ticket = 0;
    }
    __syncthreads();
    if (!s_last_cta) return;
    int32_t* s_pg = sm;
    int32_t* s_lst = sm + p.plan_cap;
    int32_t* s_phys = sm + 2 * p.plan_cap;
    int32_t* s_keep = sm + 3 * p.plan_cap;
    for (int i = tid; i < cnt; i += kRaasThreads) {
        const int u = __ldcg(plan + i);
        s_pg[i] = u;
        s_lst[i] = __ldcg(last + u);
        s_phys[i] = __ldcg(phys + i);
    }
    __syncthreads();
    // eviction: rank the non-exempt retained pages by (last, page); keep the newest k_pages
    const int sink_hi = (p.n_sink > 0 && s > 0) ? (min(p.n_sink, s) - 1) / kPage + 1 : 0;
    const int win_lo = (p.n_window > 0) ? max(0, s - p.n_window) / kPage : 0x7fffffff;
    auto exempt = [&](int u) { return u < sink_hi || u >= win_lo; };
    int n_ne = 0;
    {
        int c = 0;
        for (int i = tid; i < cnt; i += kRaasThreads) c += !exempt(s_pg[i]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
        if (lane == 0) s_scan[warp] = c;
        __syncthreads();
        for (int w = 0; w < kRaasWarps; ++w) n_ne += s_scan[w];
        __syncthreads();
    }
    const int n_evict = max(0, n_ne - p.k_pages);
    for (int i = tid; i < cnt; i += kRaasThreads) {
        const int u = s_pg[i];
        bool keep = true;
        if (n_evict > 0 && !exempt(u)) {
            const int li = s_lst[i];
            int rank = 0;  // non-exempt pages strictly before (last, page) order
            for (int j = 0; j < cnt; ++j) {
                const int v = s_pg[j];
                if (exempt(v)) continue;
                const int lj = s_lst[j];
                rank += (lj < li) || (lj == li && v < u);
            }
            keep = rank >= n_evict;
        }
        s_keep[i] = keep;
        if (!keep) last[u] = -1;  // evicted for good
    }
    __syncthreads();
    // compaction (ascending) + the page position s opens
    if (warp == 0) {
        int pos = 0;
        for (int i0 = 0; i0 < cnt; i0 += 32) {
            const int i = i0 + lane;
            const bool k = i < cnt && s_keep[i];
            const unsigned m = __ballot_sync(0xffffffffu, k);
            if (k) {
                const int at = pos + __popc(m & ((1u << lane) - 1u));
                plan[at] = s_pg[i];
                phys[at] = s_phys[i];
            }
            pos += __popc(m);
        }
        if (lane == 0) {
            if (s % kPage == 0 && s / kPage < p.max_pages && pos < p.plan_cap) {
                const int un = s / kPage;
                plan[pos] = un;
                phys[pos] = p.block_table[(size_t)b * p.bt_stride + un];
                last[un] = s + 1;
                ++pos;
            }
            p.plan_count[b] = pos;
            p.plan_stamp[b] = s + 1;
        }
    }
}

}  // namespace

cudaError_t launch_raas_reset(const RaasParams& p, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.batch);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, raas_reset_kernel, p);
}

cudaError_t launch_raas_update(const RaasParams& p, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kRaasCtas, p.batch);
    cfg.blockDim = dim3(kRaasThreads);
    cfg.dynamicSmemBytes = (size_t)4 * p.plan_cap * sizeof(int32_t);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    static std::atomic<int> cache[kMaxDevices];  // per device: attribute opt-ins are per context
    if (per_device_once(cache, [] {
            return cudaFuncSetAttribute(raas_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) ==
                           cudaSuccess ? 1 : -1;
        }) < 0)
        return cudaErrorInvalidConfiguration;
    return cudaLaunchKernelEx(&cfg, raas_update_kernel, p);
}

}  // namespace delta
