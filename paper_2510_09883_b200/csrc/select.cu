// select.cu — Delta-layer scoring and top-k selection.
//
// Phase A (grid of CTAs per sequence): with the layer's global per-head LSE_j (written by
// the decode combine) and its scaled logits a_j(t):
//   key_t = max_j (a_j(t) - LSE_j)                      = log s_t,  s_t = max_j alpha_j(t)
//   token mode: unit key = key_t                         (rank-equivalent to s_t, R8)
//   page mode : unit key = S_u = sum_{t in u} exp(key_t), ascending t, fp32 (R8)
// Phase B (the last CTA of each sequence, elected with an arrival counter):
//   forced F = units overlapping [0, S) and [s-L, s); candidates C = the rest;
//   if |C| <= k: rho = all units; else a 4-pass MSB-first radix select (8-bit digits) on
//   the order-preserving uint32 image of the fp32 keys finds the k-th largest key T; the
//   plan is F U {key > T} U {the lowest-index (k - #{key > T}) keys == T}  — i.e. the top
//   k by (key desc, index asc) (R9) — compacted in ascending unit order with block scans.
// Integer radix + fixed-order float sums: deterministic, bit-exact to any correct top-k on
// the same fp32 key buffer.
#include "combine.cuh"

namespace delta {
namespace {

constexpr int kSelThreads = 512;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSmemUnits = 16384;  // keys cached in shared memory up to this many units

__device__ __forceinline__ uint32_t key_bits(float f) {
    f = (f == 0.0f) ? 0.0f : f;  // -0 and +0 rank equal
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Exclusive block-wide prefix sum over kSelThreads threads; returns the exclusive value and
// writes the block total to *total.  `scratch` holds kSelWarps + 1 ints.
__device__ __forceinline__ int block_excl_scan(int v, int* scratch, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = (lane < kSelWarps) ? scratch[lane] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += y;
        }
        if (lane < kSelWarps) scratch[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const int warp_excl = (warp == 0) ? 0 : scratch[warp - 1];
    *total = scratch[kSelWarps - 1];
    __syncthreads();
    return warp_excl + x - v;
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(const SelectParams p) {
    extern __shared__ uint32_t sm_keys[];  // [kSmemUnits] (only when it fits)
    __shared__ float lse_s[256];
    __shared__ int scratch[kSelWarps + 1];
    __shared__ int hist[256];
    __shared__ int s_flag, s_bin, s_rem;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int b = blockIdx.y;
    pdl_wait();

    const int s = p.seq_len[p.layer * p.max_batch + b];
    const int block = p.sel_block;
    const int n_units = (s + block - 1) / block;
    float* keys_b = p.keys + (size_t)b * p.max_units;
    const float* src = p.keys_override ? p.keys_override + (size_t)b * p.max_units : keys_b;

    // ------------------------------------------------------------ phase A: scores
    if (!p.keys_override) {
        for (int j = tid; j < p.m; j += kSelThreads) lse_s[j] = p.lse_buf[(size_t)b * p.m + j];
        __syncthreads();
        const int per = (n_units + p.nchunk - 1) / p.nchunk;
        const int u_lo = blockIdx.x * per, u_hi = min(n_units, u_lo + per);
        const float* lg = p.logits + (size_t)b * p.max_seq * p.m;
        const int half_m = (p.m + 1) >> 1;
        const int jr = lane >> 1, hh = lane & 1;
        const int j0 = hh * half_m, j1 = min(p.m, j0 + half_m);
        // a warp handles 16 consecutive tokens: lane = 2*token + half-of-heads
        if (block == kPage) {
            for (int u = u_lo + warp; u < u_hi; u += kSelWarps) {
                const int t = u * kPage + jr;
                float mx = -INFINITY;
                if (t < s)
                    for (int j = j0; j < j1; ++j) mx = fmaxf(mx, lg[(size_t)t * p.m + j] - lse_s[j]);
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                const float e = (t < s) ? expf(mx) : 0.f;
                float sum = 0.f;
#pragma unroll
                for (int r = 0; r < kPage; ++r) sum += __shfl_sync(0xffffffffu, e, 2 * r);  // ascending t
                if (lane == 0) keys_b[u] = sum;
            }
        } else {
            const int t_lo = u_lo, t_hi = u_hi;  // block == 1: units are tokens
            for (int t0 = t_lo + warp * 16; t0 < t_hi; t0 += kSelWarps * 16) {
                const int t = t0 + jr;
                float mx = -INFINITY;
                if (t < t_hi)
                    for (int j = j0; j < j1; ++j) mx = fmaxf(mx, lg[(size_t)t * p.m + j] - lse_s[j]);
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                if (t < t_hi && hh == 0) keys_b[t] = mx;
            }
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) s_flag = (atomicAdd(&p.cnt[b], 1) == p.nchunk - 1);
        __syncthreads();
        if (!s_flag) return;
        __threadfence();
        if (tid == 0) p.cnt[b] = 0;
    }
    pdl_launch_dependents();

    // ------------------------------------------------------------ phase B: top-k
    int32_t* plan = p.plan_idx + (size_t)b * p.plan_cap;
    const int S = p.n_sink, L = p.n_window;
    const int sink_hi = (S > 0 && s > 0) ? (min(S, s) - 1) / block + 1 : 0;
    const int win_lo = (L > 0) ? max(0, s - L) / block : n_units;
    auto forced = [&](int u) { return u < sink_hi || u >= win_lo; };
    const int n_forced = sink_hi + (n_units - win_lo) - max(0, sink_hi - win_lo);
    const int n_cand = n_units - n_forced;
    int count = 0;

    if (n_cand <= p.k_units) {
        for (int u = tid; u < n_units; u += kSelThreads) plan[u] = u;  // R12: budget covers all
        count = n_units;
    } else {
        const bool cached = n_units <= kSmemUnits;
        bool bad = false;
        if (cached) {
            for (int u = tid; u < n_units; u += kSelThreads) {
                const float f = __ldcg(src + u);
                bad |= isnan(f);
                sm_keys[u] = key_bits(f);
            }
        } else {
            for (int u = tid; u < n_units; u += kSelThreads) bad |= isnan(__ldcg(src + u));
        }
        if (bad) set_err(p.err, kDevNumeric);
        __syncthreads();
        auto K = [&](int u) -> uint32_t { return cached ? sm_keys[u] : key_bits(__ldcg(src + u)); };

        uint32_t prefix = 0, maskbits = 0;
        int remaining = p.k_units;
        if (remaining > 0) {
            for (int pass = 0; pass < 4; ++pass) {
                const int shift = 24 - 8 * pass;
                if (tid < 256) hist[tid] = 0;
                __syncthreads();
                for (int u = tid; u < n_units; u += kSelThreads) {
                    if (forced(u)) continue;
                    const uint32_t v = K(u);
                    if ((v & maskbits) == prefix) atomicAdd(&hist[(v >> shift) & 255], 1);
                }
                __syncthreads();
                const int c = (tid < 256) ? hist[255 - tid] : 0;  // bins in descending order
                int tot;
                const int excl = block_excl_scan(c, scratch, &tot);
                if (tid < 256 && excl < remaining && excl + c >= remaining) {
                    s_bin = 255 - tid;
                    s_rem = remaining - excl;
                }
                __syncthreads();
                prefix |= (uint32_t)s_bin << shift;
                maskbits |= 0xFFu << shift;
                remaining = s_rem;
                __syncthreads();
            }
        }
        const uint32_t T = prefix;
        const int need_eq = remaining;  // keys equal to T still to take (lowest index first)
        const bool take_any = p.k_units > 0;
        int carry_eq = 0, carry_pos = 0;
        for (int base = 0; base < n_units; base += kSelThreads) {
            const int u = base + tid;
            const bool valid = u < n_units;
            const bool f = valid && forced(u);
            uint32_t v = 0;
            if (valid && !f) v = K(u);
            const bool cand = valid && !f && take_any;
            const bool is_gt = cand && v > T;
            const bool is_eq = cand && v == T;
            int tot_eq, tot_sel;
            const int eq_rank = block_excl_scan(is_eq ? 1 : 0, scratch, &tot_eq) + carry_eq;
            const bool sel = f || is_gt || (is_eq && eq_rank < need_eq);
            const int pos = block_excl_scan(sel ? 1 : 0, scratch, &tot_sel) + carry_pos;
            if (sel && pos < p.plan_cap) plan[pos] = u;
            carry_eq += tot_eq;
            carry_pos += tot_sel;
        }
        count = carry_pos;
        if (count > p.plan_cap) set_err(p.err, kDevUsage);
    }
    __syncthreads();
    if (tid == 0) {
        p.plan_count[b] = min(count, p.plan_cap);
        p.plan_stamp[b] = s;
        if (p.count_out) p.count_out[b] = min(count, p.plan_cap);
    }
    if (p.idx_out) {
        __syncthreads();
        for (int i = tid; i < p.plan_cap; i += kSelThreads)
            p.idx_out[(size_t)b * p.plan_cap + i] = (i < count) ? plan[i] : -1;
    }
}

}  // namespace

size_t select_smem_bytes(int max_units) {
    return (size_t)min(max_units, kSmemUnits) * sizeof(uint32_t);
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t st, bool pdl) {
    const size_t smem = select_smem_bytes(p.max_units);
    static size_t configured = 0;
    if (smem > 48 * 1024 && configured < smem) {
        cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.keys_override ? 1 : p.nchunk, p.batch);
    cfg.blockDim = dim3(kSelThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, select_kernel, p);
}

}  // namespace delta
