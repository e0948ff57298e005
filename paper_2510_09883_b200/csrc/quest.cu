// quest.cu — the Quest selection policy (readings Q1-Q3 in
// DESIGN.md §3), the paper's main comparison system, as a kernel-level policy of this library:
//  * page representatives: element-wise min / max of the keys of every (page, kv head),
//    [L][num_phys][g][2][d] bf16 (exact: min/max of bf16 values), rebuilt from the pool by
//    quest_reps_kernel and maintained on append by append.cu;
//  * page key (Q1, Q2): max over the m query heads j of sum_e max(q_j[e] min[e], q_j[e] max[e])
//    with the reps of group phi(j) — an upper bound of q_j . k over the page's keys;
//  * the page plan comes from the unchanged radix top-k (select.cu, keys precomputed) and the
//    sparse attention kernel reads it (Q3: same forced pages and page budget as DELTA).
#include <type_traits>

#include "combine.cuh"

namespace delta {
namespace {

// Rebuild: one CTA per (logical page u, kv head h, sequence b); thread i owns the bf16 pair
// (2i, 2i+1) of the d-vector and folds the page's filled slots t < n in ascending order.
__global__ void __launch_bounds__(64) quest_reps_kernel(const QuestParams p) {
    const int u = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
    pdl_wait();
    const int n = p.seq_len[p.layer * p.max_batch + b] / p.g;  // raw counter = n * g
    if (u * kPage >= n) return;
    const int filled = min(kPage, n - u * kPage);
    const int phys = p.block_table[(size_t)b * p.bt_stride + u];
    const __nv_bfloat162* rows = reinterpret_cast<const __nv_bfloat162*>(p.kv_pool) +
                                 kv_row((size_t)p.layer * p.num_phys + phys, p.g, h, 0) * (p.d / 2);
    __nv_bfloat162* rep = reinterpret_cast<__nv_bfloat162*>(p.reps) +
                          (((size_t)p.layer * p.num_phys + phys) * p.g + h) * p.d;  // 2 rows of d/2 pairs
    for (int i = threadIdx.x; i < p.d / 2; i += blockDim.x) {
        __nv_bfloat162 mn = rows[i], mx = mn;
        for (int r = 1; r < filled; ++r) {
            const __nv_bfloat162 k = rows[(size_t)r * (p.d / 2) + i];
            mn = __hmin2(mn, k);
            mx = __hmax2(mx, k);
        }
        rep[i] = mn;
        rep[p.d / 2 + i] = mx;
    }
}

// Page keys: one warp per page (8 pages per CTA); q of the sequence staged in shared memory as
// fp32.  Lane l owns the E = D/32 consecutive elements [l*E, l*E + E).  All G groups' min/max
// slices of the page are loaded up front (one independent 8- or 4-byte load each), then per
// head the lane's partial sum (ascending e) is reduced over the warp with a fixed xor tree:
// deterministic.
template <int D, int G>
__global__ void __launch_bounds__(256) quest_score_kernel(const QuestParams p) {
    constexpr int E = D / 32;
    using Vec = typename std::conditional<E == 4, uint2, uint32_t>::type;  // E bf16
    extern __shared__ float sq[];  // [m][D]
    const int b = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // With `prewait` (set by the host only inside a captured step, when the previous kernel is
    // another layer's: it wrote neither this layer's length counter nor its reps) the length and
    // the first page's reps stream in before the dependency wait; otherwise (eager calls, e.g.
    // delta_append_kv of this layer right before) everything is read after it.
    if (!p.prewait) pdl_wait();
    const int n = p.seq_len[p.layer * p.max_batch + b] / p.g;
    const int n_pages = (n + kPage - 1) / kPage;
    const int gs = p.m / p.g;
    auto load_reps = [&](int u, Vec* vmn, Vec* vmx) {
        const int phys = p.block_table[(size_t)b * p.bt_stride + u];
        const Vec* rep = reinterpret_cast<const Vec*>(reinterpret_cast<const __nv_bfloat16*>(p.reps) +
                                                      ((size_t)p.layer * p.num_phys + phys) * p.g * 2 * D);
#pragma unroll
        for (int h = 0; h < G; ++h) {
            if (h < p.g) {
                vmn[h] = rep[(size_t)h * 2 * (D / E) + lane];
                vmx[h] = rep[(size_t)h * 2 * (D / E) + D / E + lane];
            }
        }
    };
    Vec vmn[G], vmx[G];
    int u = blockIdx.x * 8 + warp;
    if (u < n_pages) load_reps(u, vmn, vmx);
    if (p.prewait) pdl_wait();
    pdl_launch_dependents();
    {   // 16-byte loads of q (all issued before the first store)
        const uint4* q8 = reinterpret_cast<const uint4*>(p.q) + (size_t)b * p.m * D / 8;
        constexpr int kPer = 4;
        for (int i0 = threadIdx.x; i0 < p.m * D / 8; i0 += kPer * blockDim.x) {
            uint4 x[kPer];
#pragma unroll
            for (int r = 0; r < kPer; ++r) {
                const int i = i0 + r * blockDim.x;
                if (i < p.m * D / 8) x[r] = q8[i];
            }
#pragma unroll
            for (int r = 0; r < kPer; ++r) {
                const int i = i0 + r * blockDim.x;
                if (i < p.m * D / 8) {
                    const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&x[r]);
#pragma unroll
                    for (int e = 0; e < 8; ++e) sq[i * 8 + e] = __bfloat162float(hv[e]);
                }
            }
        }
    }
    __syncthreads();
    for (; u < n_pages; u += gridDim.x * 8) {
        if (u != blockIdx.x * 8 + warp) load_reps(u, vmn, vmx);
        float best = -INFINITY;
#pragma unroll
        for (int h = 0; h < G; ++h) {
            if (h >= p.g) break;
            float mn[E], mx[E];
            const __nv_bfloat16* pn = reinterpret_cast<const __nv_bfloat16*>(&vmn[h]);
            const __nv_bfloat16* px = reinterpret_cast<const __nv_bfloat16*>(&vmx[h]);
#pragma unroll
            for (int i = 0; i < E; ++i) {
                mn[i] = __bfloat162float(pn[i]);
                mx[i] = __bfloat162float(px[i]);
            }
            for (int jj = 0; jj < gs; ++jj) {
                const float* qj = sq + (size_t)(h * gs + jj) * D + lane * E;
                float acc = 0.f;
#pragma unroll
                for (int i = 0; i < E; ++i) acc += fmaxf(qj[i] * mn[i], qj[i] * mx[i]);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
                best = fmaxf(best, acc);
            }
        }
        if (lane == 0) p.keys[(size_t)b * p.max_units + u] = best;
    }
}

}  // namespace

cudaError_t launch_quest_reps(const QuestParams& p, int max_pages, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(max_pages, p.g, p.batch);
    cfg.blockDim = dim3(64);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, quest_reps_kernel, p);
}

cudaError_t launch_quest_score(const QuestParams& p, int max_pages, int sms, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    const int per_seq = std::max(1, std::min((max_pages + 7) / 8, (2 * sms + p.batch - 1) / p.batch));
    cfg.gridDim = dim3(per_seq, p.batch);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = (size_t)p.m * p.d * sizeof(float);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (p.g > 16) return cudaErrorInvalidValue;
    const void* fn = p.d == 128 ? (p.g <= 8 ? (const void*)quest_score_kernel<128, 8> : (const void*)quest_score_kernel<128, 16>)
                   : p.d == 64  ? (p.g <= 8 ? (const void*)quest_score_kernel<64, 8> : (const void*)quest_score_kernel<64, 16>)
                                : nullptr;
    if (!fn) return cudaErrorInvalidValue;
    static std::atomic<int> cache[kMaxDevices * 4];  // per (device, instantiation)
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    const int slot = dev * 4 + (p.d == 128 ? 0 : 2) + (p.g <= 8 ? 0 : 1);
    if (cache[slot].load(std::memory_order_acquire) == 0) {  // opt in to the dynamic shared memory
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 128 * 4);
        if (e != cudaSuccess) return e;
        cache[slot].store(1, std::memory_order_release);
    }
    void* args[] = {const_cast<QuestParams*>(&p)};
    return cudaLaunchKernelExC(&cfg, fn, args);
    return cudaErrorInvalidValue;
}

}  // namespace delta
