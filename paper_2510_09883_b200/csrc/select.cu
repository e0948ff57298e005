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
#define DTRACE_LAYER_OFF 32  // trace builds: select stamps go to layer slot + 32
#include "combine.cuh"

#ifdef DELTA_TRACE
// per-warp SM-clock stamps of phase A (trace builds): [layer][cta][warp][8]
static __device__ long long g_sel_clk[64 * 160 * 16 * 8];
extern "C" int delta_trace_read_select_clk(void* host, size_t bytes) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess)
        e = cudaMemcpyFromSymbol(host, g_sel_clk, bytes < sizeof(g_sel_clk) ? bytes : sizeof(g_sel_clk));
    void* dev = nullptr;
    if (e == cudaSuccess) e = cudaGetSymbolAddress(&dev, g_sel_clk);
    if (e == cudaSuccess) e = cudaMemset(dev, 0, sizeof(g_sel_clk));
    return (int)e;
}
#define SELCLK(ev)                                                                                       \
    do {                                                                                                 \
        if ((threadIdx.x & 31) == 0 && blockIdx.x < 160 && p.layer < 64 && blockIdx.y == 0)              \
            g_sel_clk[((p.layer * 160 + blockIdx.x) * 16 + (threadIdx.x >> 5)) * 8 + (ev)] = clock64(); \
    } while (0)
#else
#define SELCLK(ev) do {} while (0)
#endif

namespace delta {
namespace {

#ifndef DELTA_SEL_THREADS
#define DELTA_SEL_THREADS 512
#endif
constexpr int kSelThreads = DELTA_SEL_THREADS;  // 1024 measured: C1 select 10.8 vs 9.0 us, C3 equal
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSmemUnits = 16384;  // keys cached in shared memory up to this many units

// LL unit keys (SelectParams::ll): one 8-byte (key bits, flag) word per unit, single-copy atomic
__device__ __forceinline__ void st_key_ll(uint2* a, float key, uint32_t flag) {
    asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1, %2};" ::"l"(a), "r"(__float_as_uint(key)), "r"(flag)
                 : "memory");
}
__device__ __forceinline__ uint2 ld_key_ll(const uint2* a) {
    uint2 w;
    asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];" : "=r"(w.x), "=r"(w.y) : "l"(a) : "memory");
    return w;
}
__device__ __forceinline__ float poll_key_ll(const uint2* a, uint32_t flag) {
    uint2 w = ld_key_ll(a);
    while (w.y != flag) w = ld_key_ll(a);
    return __uint_as_float(w.x);
}

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

// Exclusive block-wide prefix sum with ONE barrier: warp totals go to scratch[0..kSelWarps),
// then every warp sums the totals below it itself.  `scratch` must not be reused before
// the next barrier.
__device__ __forceinline__ int block_excl_scan1(int v, int* scratch, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    const int t = lane < kSelWarps ? scratch[lane] : 0;
    int below = lane < warp ? t : 0, all = t;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        below += __shfl_xor_sync(0xffffffffu, below, off);
        all += __shfl_xor_sync(0xffffffffu, all, off);
    }
    *total = all;
    return below + x - v;
}

// max_j (a_j(t) - LSE_j) over the heads j this lane owns: lane pair (hh = 0, 1) splits the m
// heads of token t; lane hh owns the 16-byte head groups q = hh, hh+2, ... (m % 4 == 0; the
// row is 16-byte aligned because the logits are [s][m] fp32).  `lse4` holds this lane's LSE
// groups in registers.  Max is exact, so the split and the order do not change the result.
struct LseLane {
    float4 v[4];  // q = hh + 2i, i < 4 (m <= 32); larger m falls back to global loads
};

__device__ __forceinline__ float head_max(const float* __restrict__ row, const LseLane& ls,
                                          const float* __restrict__ lse_g, int m, int hh) {
    float mx = -INFINITY;
    if ((m & 3) == 0) {
        const float4* r4 = reinterpret_cast<const float4*>(row);
        const int n4 = m >> 2;
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int q = hh + 2 * i;
            v[i] = q < n4 ? r4[q] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int q = hh + 2 * i;
            if (q < n4) {
                const float4 l = ls.v[i];
                mx = fmaxf(mx, fmaxf(fmaxf(v[i].x - l.x, v[i].y - l.y), fmaxf(v[i].z - l.z, v[i].w - l.w)));
            }
        }
        const float4* l4 = reinterpret_cast<const float4*>(lse_g);
        for (int q = hh + 8; q < n4; q += 2) {
            const float4 w = r4[q], l = l4[q];
            mx = fmaxf(mx, fmaxf(fmaxf(w.x - l.x, w.y - l.y), fmaxf(w.z - l.z, w.w - l.w)));
        }
    } else {
#pragma unroll 8
        for (int j = hh; j < m; j += 2) mx = fmaxf(mx, row[j] - lse_g[j]);
    }
    return mx;
}

// Register-resident top-k (phase B) for n_units <= kSelThreads * IPT: thread t holds units
// [t*IPT, t*IPT + IPT) — keys, candidate flags — loaded with one round of independent loads;
// the radix passes and the compaction then run on-chip (2 barriers per pass).  Returns the
// plan length.  Instantiated for IPT = 4 / 8 / 16 so no predicated-off slots are executed.
template <int IPT>
__device__ __forceinline__ int topk_regs(const SelectParams& p, int n_units, int sink_hi, int win_lo, int block,
                                      const float* __restrict__ src, const int32_t* __restrict__ bt,
                                      int32_t* plan, int32_t* plan_phys, uint32_t* sm_keys, int* hist2,
                                      int* scratch, uint32_t& s_and, uint32_t& s_or, int& s_bin, int& s_rem,
                                      int& s_cnt, const uint2* kll, uint32_t llf) {
    const int tid = threadIdx.x, lane = tid & 31;
    auto forced = [&](int u) { return u < sink_hi || u >= win_lo; };
    auto phys_of = [&](int u) -> int32_t { return block == 1 ? bt[u / kPage] * kPage + (u % kPage) : bt[u]; };
    // ---- register-resident path: thread t holds units [t*ipt, t*ipt + ipt) — keys,
    // candidate flags and physical locations — loaded with one round of independent loads;
    // the radix passes and the compaction then run on-chip (2 barriers per pass).
    const int ipt = IPT;
    const int u0 = tid * ipt;
    uint32_t key[IPT];
    // coalesced staging (unit u = i * kSelThreads + tid) of the keys' order-preserving bits and
    // the units' physical locations into shared memory, then contiguous ownership for the scan
    uint32_t* s_key = sm_keys;                                                  // [n_units]
    int32_t* s_phys = reinterpret_cast<int32_t*>(sm_keys + n_units);            // [n_units]
    bool bad = false;
    // the units' physical locations first: independent loads in flight before the key polls (a
    // block-table load after each poll — asm volatile with a memory clobber — would serialise:
    // one L2 round trip per unit per thread, ~7 us at 16 units per thread)
    // (in groups of at most 8 units, so the in-flight words stay in registers: 64 per thread)
    constexpr int GS = IPT < 8 ? IPT : 8;
#pragma unroll
    for (int g0 = 0; g0 < IPT; g0 += GS) {
        int32_t ph[GS];
#pragma unroll
        for (int i = 0; i < GS; ++i) {
            const int u = (g0 + i) * kSelThreads + tid;
            ph[i] = u < n_units ? phys_of(u) : 0;
        }
        uint2 w[GS];  // LL: one round of independent loads, then re-poll the words not yet published
        if (kll) {
#pragma unroll
            for (int i = 0; i < GS; ++i) {
                const int u = (g0 + i) * kSelThreads + tid;
                if (u < n_units) w[i] = ld_key_ll(kll + u);
            }
        }
#pragma unroll
        for (int i = 0; i < GS; ++i) {
            const int u = (g0 + i) * kSelThreads + tid;
            if (u < n_units) {
                float f;
                if (kll) {
                    while (w[i].y != llf) w[i] = ld_key_ll(kll + u);
                    f = __uint_as_float(w[i].x);
                } else {
                    f = __ldcg(src + u);
                }
                s_key[u] = key_bits(f);
                s_phys[u] = ph[i];
                bad |= isnan(f);
            }
        }
    }
    __syncthreads();
    if (tid == 0) DTRACE(11);
    uint32_t cand = 0, live = 0;
    if (u0 + IPT <= n_units) {  // 16-byte loads: scalar ones at a stride of IPT words conflict IPT-way
#pragma unroll
        for (int j = 0; j < IPT / 4; ++j) {
            const uint4 x = reinterpret_cast<const uint4*>(s_key + u0)[j];
            key[4 * j] = x.x; key[4 * j + 1] = x.y; key[4 * j + 2] = x.z; key[4 * j + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < IPT; ++i) key[i] = u0 + i < n_units ? s_key[u0 + i] : 0u;
    }
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const int u = u0 + i;
        const bool in = i < ipt && u < n_units;
        if (!in) key[i] = 0u;
        if (in) live |= 1u << i;
        if (in && !forced(u)) cand |= 1u << i;
    }
    if (bad) set_err(p.err, kDevNumeric);
    // leading bits every candidate shares (block AND / OR): the radix passes start at the
    // first byte where the candidates differ
    uint32_t kand = 0xffffffffu, kor = 0u;
#pragma unroll
    for (int i = 0; i < IPT; ++i)
        if (cand & (1u << i)) {
            kand &= key[i];
            kor |= key[i];
        }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        kand &= __shfl_xor_sync(0xffffffffu, kand, off);
        kor |= __shfl_xor_sync(0xffffffffu, kor, off);
    }
    if (lane == 0) {
        atomicAnd(&s_and, kand);
        atomicOr(&s_or, kor);
    }
    __syncthreads();
    if (tid == 0) DTRACE(6);
    const uint32_t same = ~(s_and ^ s_or);
    int first_pass = 0;
    while (first_pass < 3 && ((same >> (24 - 8 * first_pass)) & 0xFFu) == 0xFFu) ++first_pass;
    uint32_t maskbits = first_pass == 0 ? 0u : ~((1u << (32 - 8 * first_pass)) - 1u);
    uint32_t prefix = s_and & maskbits;
    int remaining = p.k_units, bin_cnt = 0;
    // One barrier per pass: every warp walks the histogram itself (same result in every warp).
    // Four buffers: pass p fills buffer p % 4 (zeroed during pass p - 2, before that pass's
    // barrier) and zeroes buffer (p + 2) % 4, last read in pass p - 2's walk, which every warp
    // finished before it could arrive at pass p - 1's barrier.
    for (int pass = p.k_units > 0 ? first_pass : 4; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        int* h = hist2 + (pass & 3) * 256;
#pragma unroll
        for (int i = 0; i < IPT; ++i)
            if ((cand & (1u << i)) && (key[i] & maskbits) == prefix) atomicAdd(&h[(key[i] >> shift) & 255u], 1);
        if (tid < 256) hist2[((pass + 2) & 3) * 256 + tid] = 0;
        __syncthreads();
        // walk the 256 bins in descending order: lane owns bins 255 - 8 lane - k
        int c[8], sum = 0;
        {
            const int4* h4 = reinterpret_cast<const int4*>(h + 248 - 8 * lane);
            const int4 x = h4[0], y = h4[1];  // bins 248-8l .. 255-8l ascending
            c[0] = y.w; c[1] = y.z; c[2] = y.y; c[3] = y.x; c[4] = x.w; c[5] = x.z; c[6] = x.y; c[7] = x.x;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) sum += c[k];
        int incl = sum;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        int excl = incl - sum, bin = 0, rem = 0, cnt = 0;
        const bool mine = excl < remaining && incl >= remaining;
        if (mine) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (excl + c[k] >= remaining) {
                    bin = 255 - (lane * 8 + k);
                    rem = remaining - excl;
                    cnt = c[k];
                    break;
                }
                excl += c[k];
            }
        }
        const int src_lane = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        bin = __shfl_sync(0xffffffffu, bin, src_lane);
        rem = __shfl_sync(0xffffffffu, rem, src_lane);
        cnt = __shfl_sync(0xffffffffu, cnt, src_lane);
        prefix |= (uint32_t)bin << shift;
        maskbits |= 0xFFu << shift;
        remaining = rem;
        bin_cnt = cnt;
        if (tid == 0) DTRACE(7 + pass);
        // every candidate of the bin is taken: T = the bin's lowest key image (prefix, low bits
        // 0), so {key > T} U {key == T} is exactly the higher bins plus this whole bin — the
        // remaining digits cannot change the selection (typically after the second digit, where
        // the k-th key's bin holds that key alone)
        if (cnt == rem) break;
    }
    if (tid == 0) DTRACE(4);
    // selection: forced, key > T, and the lowest-index `remaining` of the keys == T
    // (all of them when no tie straddles the boundary: one scan instead of two)
    const uint32_t T = prefix;
    uint32_t fl_sel = live & ~cand, fl_eq = 0;
    if (p.k_units == 0) cand = 0;  // forced units only
#pragma unroll
    for (int i = 0; i < IPT; ++i)
        if (cand & (1u << i)) {
            if (key[i] > T) fl_sel |= 1u << i;
            else if (key[i] == T) fl_eq |= 1u << i;
        }
    int tot;
    if (remaining < bin_cnt) {  // ties at T: rank the equal keys by index
        int eq_rank = block_excl_scan1(__popc(fl_eq), scratch, &tot);
#pragma unroll
        for (int i = 0; i < IPT; ++i)
            if (fl_eq & (1u << i)) {
                if (eq_rank < remaining) fl_sel |= 1u << i;
                ++eq_rank;
            }
        __syncthreads();  // scratch reuse
    } else {
        fl_sel |= fl_eq;
    }
    int pos = block_excl_scan1(__popc(fl_sel), scratch + kSelWarps, &tot);
#pragma unroll
    for (int i = 0; i < IPT; ++i)
        if (fl_sel & (1u << i)) {
            if (pos < p.plan_cap) {
                plan[pos] = u0 + i;
                plan_phys[pos] = s_phys[u0 + i];
            }
            ++pos;
        }
    if (tot > p.plan_cap) set_err(p.err, kDevUsage);
    return tot;
}

__global__ void __launch_bounds__(kSelThreads, 1024 / kSelThreads) select_kernel(const SelectParams p) {
    extern __shared__ uint32_t sm_keys[];  // [kSmemUnits] (only when it fits)
    __shared__ int scratch[2 * kSelWarps + 1];
    __shared__ __align__(16) int hist2[4 * 256];  // radix histograms (4 buffers, see topk_regs)
    __shared__ int whist[kSelWarps * 256];
    __shared__ int s_flag, s_bin, s_rem, s_cnt;
    __shared__ uint32_t s_and, s_or;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int b = blockIdx.y;
    if (tid == 0) DTRACE(0);
    // warm the address translation (and L2) of the words read right after the wait: a prefetch
    // reads nothing, so it may precede griddepcontrol.wait
    if (tid < 8) {
        const char* a = nullptr;
        if (tid == 0) a = reinterpret_cast<const char*>(p.seq_len + p.layer * p.max_batch + b);
        if (tid == 1) a = reinterpret_cast<const char*>(p.lse_buf + (size_t)b * p.m);
        if (tid == 2 && p.ll) a = reinterpret_cast<const char*>(p.epoch + b);
        if (tid == 3 && p.ll) a = reinterpret_cast<const char*>(p.keys_ll + (size_t)b * p.max_units);
        if (tid >= 4) a = reinterpret_cast<const char*>(p.logits + ((size_t)b * p.max_seq +
                          (size_t)(tid - 4) * (p.max_seq / 4) + (size_t)blockIdx.x * p.max_seq / (4 * gridDim.x)) * p.m);
        if (a && !p.keys_override && !p.k_new) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
    pdl_wait();
    if (!p.late_trigger) pdl_launch_dependents();  // the next kernel's reads of this plan come after its own wait
    if (tid == 0) DTRACE(1);

    SELCLK(0);
    // Per-CTA broadcast of the values every warp needs (length counter, the LSE row): every
    // warp of every CTA loading the same words makes an L2 hot spot (measured: ~1850 cycles for
    // the length load, ~2800 for the LSE + logits, against ~300 for an uncontended L2 hit)
    __shared__ int s_len;
    __shared__ __align__(16) float s_lse[256];
    __shared__ uint32_t s_llf;
    if (tid == 0) {
        s_len = p.seq_len[p.layer * p.max_batch + b];
        if (p.ll) s_llf = (uint32_t)p.epoch[b] + 1u;  // this launch's LL flag (same round trip)
    }
    if (!p.keys_override && !p.k_new && tid < p.m) s_lse[tid] = p.lse_buf[(size_t)b * p.m + tid];
    __syncthreads();
    int s = s_len / p.g;  // raw counter = n * g
    const uint32_t llf = p.ll ? s_llf : 0u;
    const uint2* kll = p.ll ? p.keys_ll + (size_t)b * p.max_units : nullptr;
    if (p.k_new) {
        // Quest layer: Eq.7 append of this step's token at position s, then
        // fold it into its page's min/max representatives (quest.cu); a token in slot 0 starts
        // the page.  One thread per 16-byte chunk of the K and V rows, one per bf16 pair of reps.
        const int t = s;
        if (t + 1 > p.max_seq) {
            if (tid == 0) set_err(p.err, kDevCapacity);
            return;
        }
        const int32_t* btb = p.block_table + (size_t)b * p.bt_stride;
        const size_t lp = (size_t)p.layer * p.num_phys + btb[t / kPage];
        const int chunks = p.d / 8;
        __nv_bfloat16* pool = reinterpret_cast<__nv_bfloat16*>(p.kv_pool);
        const uint4* kn = reinterpret_cast<const uint4*>(p.k_new) + (size_t)b * p.g * chunks;
        const uint4* vn = reinterpret_cast<const uint4*>(p.v_new) + (size_t)b * p.g * chunks;
        for (int i = tid; i < p.g * chunks; i += kSelThreads) {
            const int hh = i / chunks, c = i - hh * chunks;
            const size_t row = kv_row(lp, p.g, hh, t % kPage);
            reinterpret_cast<uint4*>(pool + row * p.d)[c] = kn[i];
            reinterpret_cast<uint4*>(pool + (row + kPage) * p.d)[c] = vn[i];
        }
        const int pairs = p.d / 2;
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(p.k_new) + (size_t)b * p.g * pairs;
        for (int i = tid; i < p.g * pairs; i += kSelThreads) {
            const int hh = i / pairs, e2 = i - hh * pairs;
            __nv_bfloat162* rep = reinterpret_cast<__nv_bfloat162*>(p.reps) + (lp * p.g + hh) * p.d;
            const __nv_bfloat162 k = k2[i];
            if (t % kPage == 0) {
                rep[e2] = k;
                rep[pairs + e2] = k;
            } else {
                rep[e2] = __hmin2(rep[e2], k);
                rep[pairs + e2] = __hmax2(rep[pairs + e2], k);
            }
        }
        __syncthreads();
        if (tid == 0) p.seq_len[p.layer * p.max_batch + b] = (t + 1) * p.g;
        s = t + 1;
    }
    const int block = p.sel_block;
    const int n_units = (s + block - 1) / block;
    float* keys_b = p.keys + (size_t)b * p.max_units;
    const float* src = p.keys_override ? p.keys_override + (size_t)b * p.max_units : keys_b;

    // ------------------------------------------------------------ phase A: scores
    if (!p.keys_override) {
        const float* lse_g = s_lse;  // broadcast above (m <= 256)
        LseLane lsl;
        {
            const int hh0 = lane & 1, n4 = p.m >> 2;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int q = hh0 + 2 * i;
                lsl.v[i] = ((p.m & 3) == 0 && q < n4) ? reinterpret_cast<const float4*>(lse_g)[q]
                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        const int per = (n_units + p.nchunk - 1) / p.nchunk;
        const int u_lo = blockIdx.x * per, u_hi = min(n_units, u_lo + per);
#ifdef DELTA_TRACE
        if (u_hi == -12345) lsl.v[0].x += 1.f;  // orders the stamp after the length load
#endif
        SELCLK(1);
        const float* lg = p.logits + (size_t)b * p.max_seq * p.m;
        const int jr = lane >> 1, hh = lane & 1;
        // a warp handles 16 consecutive tokens: lane = 2*token + half-of-heads
        // sequence-sharded local pass: only this rank's pages carry logits; the other units'
        // keys are -inf (never a candidate of this rank)
        const int own_lo = p.shard_mode == 1 ? p.page_lo * kPage : 0;
        const int own_hi = p.shard_mode == 1 ? p.page_hi * kPage : 0x7fffffff;
        if (block == kPage) {
            for (int u = u_lo + warp; u < u_hi; u += kSelWarps) {
                const int t = u * kPage + jr;
                const bool own = t >= own_lo && t < own_hi;
                float mx = -INFINITY;
                if (t < s && own) mx = head_max(lg + (size_t)t * p.m, lsl, lse_g, p.m, hh);
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                if (u == u_lo + warp) SELCLK(2);
                const float e = (t < s) ? expf(mx) : 0.f;
                float sum = 0.f;
#pragma unroll
                for (int r = 0; r < kPage; ++r) sum += __shfl_sync(0xffffffffu, e, 2 * r);  // ascending t
                if (lane == 0) {
                    const float key = (u * kPage >= own_lo && u * kPage < own_hi) ? sum : -INFINITY;
                    keys_b[u] = key;
                    if (p.ll) st_key_ll(p.keys_ll + (size_t)b * p.max_units + u, key, llf);
                }
                if (u == u_lo + warp) SELCLK(3);
            }
        } else {
            const int t_lo = u_lo, t_hi = u_hi;  // block == 1: units are tokens
            for (int t0 = t_lo + warp * 16; t0 < t_hi; t0 += kSelWarps * 16) {
                const int t = t0 + jr;
                const bool own = t >= own_lo && t < own_hi;
                float mx = -INFINITY;
                if (t < t_hi && own) mx = head_max(lg + (size_t)t * p.m, lsl, lse_g, p.m, hh);
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                if (t < t_hi && hh == 0) {
                    keys_b[t] = mx;
                    if (p.ll) st_key_ll(p.keys_ll + (size_t)b * p.max_units + t, mx, llf);
                }
            }
        }
        // arrival: the barrier puts every thread's key stores before thread 0's acq_rel atomic
        // (release, cumulative); the last arrival's acquire + the barrier order its threads'
        // key loads after every other CTA's stores — no per-thread fences
        SELCLK(4);
        if (p.ll) {  // LL hand-off: CTA 0 ranks, polling the published keys; the others are done
            SELCLK(5);
            if (tid == 0) DTRACE(2);
            if (blockIdx.x != 0) return;
            goto phase_b;
        }
        __syncthreads();
        if (tid == 0) DTRACE(2);
        if (tid == 0) {
            int old;
            asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(p.cnt + b) : "memory");
            s_flag = (old == p.nchunk - 1);
        }
        __syncthreads();
#ifdef DELTA_TRACE
        if (s_flag == 7) s = 0;  // orders the stamp after the election
#endif
        SELCLK(5);
        if (!s_flag) return;
        if (tid == 0) DTRACE(3);
        if (tid == 0) p.cnt[b] = 0;
    }

    // ------------------------------------------------------------ phase B: top-k
phase_b:
    int32_t* plan = p.plan_idx + (size_t)b * p.plan_cap;
    int32_t* plan_phys = p.plan_phys + (size_t)b * p.plan_cap;
    const int32_t* bt = p.block_table + (size_t)b * p.bt_stride;
    // physical location of a unit for the sparse kernels: page id, or page * P + slot (tokens)
    auto phys_of = [&](int u) -> int32_t { return block == 1 ? bt[u / kPage] * kPage + (u % kPage) : bt[u]; };
    const int S = p.n_sink, L = p.n_window;
    const int sink_hi = (S > 0 && s > 0) ? (min(S, s) - 1) / block + 1 : 0;
    const int win_lo = (L > 0) ? max(0, s - L) / block : n_units;
    auto forced = [&](int u) { return u < sink_hi || u >= win_lo; };
    const int n_forced = sink_hi + (n_units - win_lo) - max(0, sink_hi - win_lo);
    const int n_cand = n_units - n_forced;
    int count = 0;
    constexpr int IPT = 8;  // old path: consecutive units per thread, one chunk = 4096 units
    for (int i = tid; i < 4 * 256; i += kSelThreads) hist2[i] = 0;
    if (tid == 0) {
        s_and = 0xffffffffu;
        s_or = 0u;
    }

    if (n_cand <= p.k_units) {
        if (kll)  // the epoch may only move once every phase-A CTA has published (hence read it)
            for (int u = tid; u < n_units; u += kSelThreads) (void)poll_key_ll(kll + u, llf);
        for (int u = tid; u < n_units; u += kSelThreads) {  // R12: budget covers all
            plan[u] = u;
            plan_phys[u] = phys_of(u);
        }
        count = n_units;
    } else if (n_units <= kSelThreads * 16) {
        const int ipt = (n_units + kSelThreads - 1) / kSelThreads;
        if (ipt <= 4)
            count = topk_regs<4>(p, n_units, sink_hi, win_lo, block, src, bt, plan, plan_phys, sm_keys, hist2,
                                 scratch, s_and, s_or, s_bin, s_rem, s_cnt, kll, llf);
        else if (ipt <= 8)
            count = topk_regs<8>(p, n_units, sink_hi, win_lo, block, src, bt, plan, plan_phys, sm_keys, hist2,
                                 scratch, s_and, s_or, s_bin, s_rem, s_cnt, kll, llf);
        else
            count = topk_regs<16>(p, n_units, sink_hi, win_lo, block, src, bt, plan, plan_phys, sm_keys, hist2,
                                  scratch, s_and, s_or, s_bin, s_rem, s_cnt, kll, llf);
    } else {
        const bool cached = n_units <= kSmemUnits;
        bool bad = false;
        if (cached) {
            for (int u = tid; u < n_units; u += kSelThreads) {
                const float f = kll ? poll_key_ll(kll + u, llf) : __ldcg(src + u);
                bad |= isnan(f);
                sm_keys[u] = key_bits(f);
            }
        } else {
            for (int u = tid; u < n_units; u += kSelThreads) bad |= isnan(__ldcg(src + u));
        }
        if (bad) set_err(p.err, kDevNumeric);
        __syncthreads();
        auto K = [&](int u) -> uint32_t { return cached ? sm_keys[u] : key_bits(__ldcg(src + u)); };

        if (tid == 0) DTRACE(6);
        // Leading digits every candidate shares (block AND / OR of the candidate keys): those
        // bits of the k-th key are known, so the radix passes start at the first byte where
        // the candidates differ (page sums share sign and most exponent bits).
        uint32_t kand = 0xffffffffu, kor = 0u;
        for (int u = tid; u < n_units; u += kSelThreads) {
            if (forced(u)) continue;
            const uint32_t v = K(u);
            kand &= v;
            kor |= v;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            kand &= __shfl_xor_sync(0xffffffffu, kand, off);
            kor |= __shfl_xor_sync(0xffffffffu, kor, off);
        }
        if (lane == 0) {
            atomicAnd(&s_and, kand);
            atomicOr(&s_or, kor);
        }
        __syncthreads();
        const uint32_t same = ~(s_and ^ s_or);  // bit set: identical in every candidate
        int first_pass = 0;
        while (first_pass < 3 && ((same >> (24 - 8 * first_pass)) & 0xFFu) == 0xFFu) ++first_pass;
        uint32_t maskbits = first_pass == 0 ? 0u : ~((1u << (32 - 8 * first_pass)) - 1u);
        uint32_t prefix = s_and & maskbits;
        int remaining = p.k_units;
        if (remaining > 0) {
            for (int pass = first_pass; pass < 4; ++pass) {
                const int shift = 24 - 8 * pass;
                int* h = hist2 + (pass & 1) * 256;  // the other buffer was zeroed last pass
                if (p.hist_mode == 1) {
                    // warp-aggregated histogram: lanes with the same digit add once
                    for (int u0 = warp * 32; u0 < n_units; u0 += kSelThreads) {
                        const int u = u0 + lane;
                        int bin = -1;
                        if (u < n_units && !forced(u)) {
                            const uint32_t v = K(u);
                            if ((v & maskbits) == prefix) bin = (int)((v >> shift) & 255u);
                        }
                        const unsigned peers = __match_any_sync(0xffffffffu, bin);
                        if (bin >= 0 && lane == __ffs(peers) - 1) atomicAdd(&h[bin], __popc(peers));
                    }
                    if (tid < 256) hist2[((pass + 1) & 1) * 256 + tid] = 0;
                    __syncthreads();
                } else {
                    // per-warp private histograms (keys sharing digits do not serialise warps
                    // on the same bins), then one reduction per bin
                    for (int i = tid; i < kSelWarps * 256; i += kSelThreads) whist[i] = 0;
                    __syncthreads();
                    int* myh = whist + warp * 256;
                    for (int u = tid; u < n_units; u += kSelThreads) {
                        if (forced(u)) continue;
                        const uint32_t v = K(u);
                        if ((v & maskbits) == prefix) atomicAdd(&myh[(v >> shift) & 255], 1);
                    }
                    __syncthreads();
                    if (tid < 256) {
                        int c = 0;
#pragma unroll
                        for (int w = 0; w < kSelWarps; ++w) c += whist[w * 256 + tid];
                        h[tid] = c;
                    }
                    __syncthreads();
                }
                if (warp == 0) {  // one warp walks the 256 bins in descending order
                    int c[8], sum = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        c[k] = h[255 - (lane * 8 + k)];
                        sum += c[k];
                    }
                    int incl = sum;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, off);
                        if (lane >= off) incl += y;
                    }
                    int excl = incl - sum;
                    if (excl < remaining && incl >= remaining) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            if (excl + c[k] >= remaining) {
                                s_bin = 255 - (lane * 8 + k);
                                s_rem = remaining - excl;
                                break;
                            }
                            excl += c[k];
                        }
                    }
                }
                __syncthreads();
                prefix |= (uint32_t)s_bin << shift;
                maskbits |= 0xFFu << shift;
                remaining = s_rem;
                if (tid == 0) DTRACE(7 + pass);
            }
        }
        if (tid == 0) DTRACE(4);
        const uint32_t T = prefix;
        const int need_eq = remaining;  // keys equal to T still to take (lowest index first)
        const bool take_any = p.k_units > 0;
        int carry_eq = 0, carry_pos = 0;
        for (int base = 0; base < n_units; base += kSelThreads * IPT) {
            const int u0 = base + tid * IPT;
            // physical locations of this thread's units, loaded before the scans (overlap)
            int32_t phys[IPT];
            if (block == 1) {
                const int32_t pg = u0 < n_units ? bt[u0 / kPage] : 0;  // u0..u0+7 share a page
#pragma unroll
                for (int i = 0; i < IPT; ++i) phys[i] = pg * kPage + ((u0 + i) % kPage);
            } else {
#pragma unroll
                for (int i = 0; i < IPT; ++i) phys[i] = (u0 + i < n_units) ? bt[u0 + i] : 0;
            }
            uint32_t fl_f = 0, fl_gt = 0, fl_eq = 0;  // bit i: unit u0 + i is forced / > T / == T
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const int u = u0 + i;
                if (u < n_units) {
                    if (forced(u)) {
                        fl_f |= 1u << i;
                    } else if (take_any) {
                        const uint32_t v = K(u);
                        if (v > T) fl_gt |= 1u << i;
                        else if (v == T) fl_eq |= 1u << i;
                    }
                }
            }
            int tot_eq, tot_sel;
            int eq_rank = block_excl_scan(__popc(fl_eq), scratch, &tot_eq) + carry_eq;
            uint32_t fl_sel = fl_f | fl_gt;
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                if (fl_eq & (1u << i)) {
                    if (eq_rank < need_eq) fl_sel |= 1u << i;
                    ++eq_rank;
                }
            }
            int pos = block_excl_scan(__popc(fl_sel), scratch, &tot_sel) + carry_pos;
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                if (fl_sel & (1u << i)) {
                    if (pos < p.plan_cap) {
                        plan[pos] = u0 + i;
                        plan_phys[pos] = phys[i];
                    }
                    ++pos;
                }
            }
            carry_eq += tot_eq;
            carry_pos += tot_sel;
        }
        count = carry_pos;
        if (count > p.plan_cap) set_err(p.err, kDevUsage);
    }
    __syncthreads();
    if (tid == 0) DTRACE(5);
    const int n_plan = min(count, p.plan_cap);
    if (p.shard_mode == 1) {
        // export this rank's candidates: its non-forced plan units with a real key
        uint2* cand = p.cand_out + (size_t)b * p.plan_cap;
        for (int i = tid; i < p.plan_cap; i += kSelThreads) {
            uint2 c = make_uint2(0u, 0xffffffffu);  // (key bits, unit = -1): empty slot
            if (i < n_plan) {
                const int u = plan[i];
                const float key = __ldcg(src + u);
                if (!forced(u) && key != -INFINITY) c = make_uint2(__float_as_uint(key), (uint32_t)u);
            }
            cand[i] = c;
        }
        return;  // the global plan comes from the merge pass (shard_mode 2)
    }
    if (p.range_n > 0 && tid < 32) {
        // plan entries per page range (this rank's share, or each fixed chunk of R21): the
        // plan ascends, so range c holds entries [#(page < lo_c), #(page < hi_c))
        for (int c = 0; c < p.range_n; ++c) {
            const int plo = p.range_first + c * p.range_step, phi = plo + p.range_step;
            int below_lo = 0, below_hi = 0;
            for (int i = lane; i < n_plan; i += 32) {
                const int pg = block == 1 ? plan[i] / kPage : plan[i];
                below_lo += pg < plo;
                below_hi += pg < phi;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                below_lo += __shfl_xor_sync(0xffffffffu, below_lo, off);
                below_hi += __shfl_xor_sync(0xffffffffu, below_hi, off);
            }
            if (lane == 0) {
                p.plan_lo[(size_t)c * p.max_batch + b] = below_lo;
                p.plan_hi[(size_t)c * p.max_batch + b] = below_hi;
            }
        }
    }
    if (tid == 0) {
        if (kll) p.epoch[b] = (int32_t)llf;  // every phase-A CTA has read the old epoch
        p.plan_count[b] = n_plan;
        p.plan_stamp[b] = s;
        if (p.count_out) p.count_out[b] = n_plan;
    }
    if (p.idx_out) {
        __syncthreads();
        for (int i = tid; i < p.plan_cap; i += kSelThreads)
            p.idx_out[(size_t)b * p.plan_cap + i] = (i < count) ? plan[i] : -1;
    }
    if (p.late_trigger) pdl_launch_dependents();
}

}  // namespace

#ifdef DELTA_TRACE
extern "C" int delta_trace_read_select(void* host, size_t bytes) {  // this TU's copy of the stamps
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess)
        e = cudaMemcpyFromSymbol(host, g_delta_trace, bytes < sizeof(g_delta_trace) ? bytes : sizeof(g_delta_trace));
    void* dev = nullptr;
    if (e == cudaSuccess) e = cudaGetSymbolAddress(&dev, g_delta_trace);
    if (e == cudaSuccess) e = cudaMemset(dev, 0, sizeof(g_delta_trace));
    return (int)e;
}
#endif

size_t select_smem_bytes(int max_units) {
    // keys (and, on the register path, the units' physical locations: 2 x 4 B per unit)
    return (size_t)min(max_units, kSmemUnits) * sizeof(uint32_t) * 2;
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t st, bool pdl) {
    const size_t smem = select_smem_bytes(p.max_units);
    // static + dynamic shared memory exceeds the 48 KiB default; opt in once per device
    static std::atomic<int> cache[kMaxDevices];
    if (per_device_once(cache, [] {
            return cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(2 * kSmemUnits * sizeof(uint32_t))) == cudaSuccess ? 1 : -1;
        }) < 0)
        return cudaErrorInvalidConfiguration;
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
