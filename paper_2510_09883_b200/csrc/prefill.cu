// prefill.cu — chunked prefill (NEXT-3): causal attention of ntok new tokens per sequence over
// the paged cache that already holds them (appended by append.cu in the same call), the step
// before the decode path (Eq.1-4 over a prompt; "prefill").
// Query i of the chunk sits at position pos_i = n0 + i and attends tokens t <= pos_i (Eq.4 with
// the causal mask), GQA head j reads group phi(j) = j / gs (R15).
//
// CTA = (block of QB = 32 (gs <= 8) or 16 query tokens, kv head h, sequence b), latest blocks
// (longest causal rows) first; its rows are the QB x gs (token, head) pairs of the group, 16
// rows per warp.  The CTA streams the head's
// K|V pages (the decode kernels' 8 KiB (page, head) tile, 128-byte swizzle) through a
// double-buffered cp.async ring of two-page stages; per page and warp: S = Q K^T (m16n8k16, bf16 -> fp32,
// 2 token tiles x d/16), causal mask, online softmax in the exp2 domain, O += P V with P as
// bf16 hi + lo (two MMAs, ~16-bit probabilities as in the decode kernels, R18).
// Tensor cores on a dense contraction: mma.sync here; the tcgen05 version is the next step.
#include "combine.cuh"

namespace delta {
namespace {

// query tokens per CTA: QB x gs rows, 16 per warp (QB = 32 for gs <= 8, else 16: <= 16 warps)
__host__ __device__ constexpr int prefill_qb(int gs) { return gs <= 8 ? 32 : 16; }
constexpr int kPPS = 2;  // pages per ring stage (32 tokens between barriers)

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int D, int kQB>
__global__ void __launch_bounds__(512) prefill_kernel(const PrefillParams p) {
    constexpr int QS = D + 8;                     // padded Q row (bf16): conflict-free ldmatrix
    constexpr int kTile = TileLayout<D>::kBytes;  // K rows then V rows of one (page, head)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring = base;                                                         // [2][kPPS][kTile]
    __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(base + 2 * kPPS * kTile);  // [rows][QS]

    const int qb = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, b = blockIdx.z;  // longest rows first
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nthr = blockDim.x;
    const int g4 = lane >> 2, t4 = lane & 3;
    const int gs = p.gs, rows = kQB * gs;
    pdl_wait();
    const int n_after = p.seq_len[p.layer * p.max_batch + b] / p.g;  // raw counter n * g (append ran)
    const int n0 = n_after - p.ntok;
    const int i0 = qb * kQB;
    if (i0 >= p.ntok) return;
    const int pos_last = n0 + min(p.ntok, i0 + kQB) - 1;
    const int npages = pos_last / kPage + 1;
    const int32_t* bt = p.block_table + (size_t)b * p.bt_stride;
    const size_t layer_ph = (size_t)p.layer * p.num_phys;
    const __nv_bfloat16* pool = reinterpret_cast<const __nv_bfloat16*>(p.kv_pool);

    // Q tile: row r = (token i0 + r / gs, head h*gs + r % gs)
    {
        constexpr int C = D / 8;
        const __nv_bfloat16* q = reinterpret_cast<const __nv_bfloat16*>(p.q);
        for (int x = tid; x < rows * C; x += nthr) {
            const int r = x / C, c = x - r * C;
            const int i = i0 + r / gs, jj = r % gs;
            __nv_bfloat16* dst = sq + (size_t)r * QS + c * 8;
            if (i < p.ntok)
                cp_async16(dst, q + (((size_t)b * p.ntok + i) * p.m + h * gs + jj) * D + c * 8);
            else
                *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
        }
    }
    auto load_page = [&](int u, int slot) {
        const size_t row0 = kv_row(layer_ph + bt[u], p.g, h, 0);  // 2P contiguous rows: K then V
        uint8_t* dst = ring + slot * kTile;
        constexpr int C = D / 8;
        for (int x = tid; x < 2 * kPage * C; x += nthr) {
            const int r = x / C, c = x - r * C;  // r < P: K row r; r >= P: V row r - P
            const uint8_t* src = reinterpret_cast<const uint8_t*>(pool + (row0 + r) * D) + c * 16;
            uint8_t* d = (r < kPage) ? dst + swz<D>(r, c) : dst + TileLayout<D>::kVOff + swz<D>(r - kPage, c);
            cp_async16(d, src);
        }
    };
    for (int k = 0; k < kPPS && k < npages; ++k) load_page(k, k);
    cp_async_commit();

    // this warp's 16 rows: row g4 and g4 + 8 of the tile; their query positions
    const int r_lo = warp * 16 + g4, r_hi = r_lo + 8;
    const bool live_w = warp * 16 < rows;
    const int pos_lo = (r_lo < rows && i0 + r_lo / gs < p.ntok) ? n0 + i0 + r_lo / gs : -1;
    const int pos_hi = (r_hi < rows && i0 + r_hi / gs < p.ntok) ? n0 + i0 + r_hi / gs : -1;
    float o[D / 8][4];
#pragma unroll
    for (int dt = 0; dt < D / 8; ++dt) o[dt][0] = o[dt][1] = o[dt][2] = o[dt][3] = 0.f;
    float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;
    const float sl2 = p.scale_log2;
    uint32_t qa[D / 16][4];
    bool q_loaded = false;

    for (int u0 = 0; u0 < npages; u0 += kPPS) {
        const int buf = (u0 / kPPS) & 1;
        for (int k = 0; k < kPPS && u0 + kPPS + k < npages; ++k) load_page(u0 + kPPS + k, (buf ^ 1) * kPPS + k);
        cp_async_commit();
        cp_async_wait<1>();  // this stage's pages (and Q) landed
        __syncthreads();
        for (int sub = 0; sub < kPPS && u0 + sub < npages; ++sub) {
        const int u = u0 + sub;
        if (live_w) {
            if (!q_loaded) {
                const uint32_t qbase = smem_u32(sq + (size_t)(warp * 16) * QS);
#pragma unroll
                for (int kc = 0; kc < D / 16; ++kc)
                    ldsm_x4(qbase + (uint32_t)(((lane & 15) * QS + kc * 16 + (lane >> 4) * 8) * 2), qa[kc][0],
                            qa[kc][1], qa[kc][2], qa[kc][3]);
                q_loaded = true;
            }
            const uint32_t kt = smem_u32(ring + (buf * kPPS + sub) * kTile), vt = kt + TileLayout<D>::kVOff;
            // S[16 rows x 16 tokens] = Q K^T: token tile nt = tokens 8nt..8nt+7
            float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int kc = 0; kc < D / 16; ++kc) {
                uint32_t k0, k1, k2, k3;
                ldsm_x4(kt + swz<D>((lane & 7) + 8 * (lane >> 4), kc * 2 + ((lane >> 3) & 1)), k0, k1, k2, k3);
                mma_bf16_16816(sc[0], qa[kc], k0, k1);
                mma_bf16_16816(sc[1], qa[kc], k2, k3);
            }
            // causal mask + online softmax (log2 domain); lane holds rows g4 (c0, c1) and
            // g4 + 8 (c2, c3), tokens 8nt + 2t4 + {0, 1}
            const int tbase = u * kPage;
            float x[2][4];
            float mx_lo = -INFINITY, mx_hi = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int t = tbase + nt * 8 + 2 * t4 + e;
                    x[nt][e] = (t <= pos_lo) ? sc[nt][e] * sl2 : -INFINITY;
                    x[nt][2 + e] = (t <= pos_hi) ? sc[nt][2 + e] * sl2 : -INFINITY;
                    mx_lo = fmaxf(mx_lo, x[nt][e]);
                    mx_hi = fmaxf(mx_hi, x[nt][2 + e]);
                }
            mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
            mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
            mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
            mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
            const float mn_lo = fmaxf(m_lo, mx_lo), mn_hi = fmaxf(m_hi, mx_hi);
            const float al_lo = (mn_lo == -INFINITY) ? 1.f : ex2(m_lo - mn_lo);
            const float al_hi = (mn_hi == -INFINITY) ? 1.f : ex2(m_hi - mn_hi);
            m_lo = mn_lo;
            m_hi = mn_hi;
            l_lo *= al_lo;
            l_hi *= al_hi;
#pragma unroll
            for (int dt = 0; dt < D / 8; ++dt) {
                o[dt][0] *= al_lo; o[dt][1] *= al_lo;
                o[dt][2] *= al_hi; o[dt][3] *= al_hi;
            }
            float pr[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    pr[nt][e] = (m_lo == -INFINITY) ? 0.f : ex2(x[nt][e] - m_lo);
                    pr[nt][2 + e] = (m_hi == -INFINITY) ? 0.f : ex2(x[nt][2 + e] - m_hi);
                    l_lo += pr[nt][e];
                    l_hi += pr[nt][2 + e];
                }
            // P as the A operand of PV (rows x 16 tokens): hi + lo bf16 parts
            uint32_t ph[4], pl[4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const __nv_bfloat162 h01 = __floats2bfloat162_rn(pr[nt][0], pr[nt][1]);
                const __nv_bfloat162 h23 = __floats2bfloat162_rn(pr[nt][2], pr[nt][3]);
                const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
                ph[2 * nt] = *reinterpret_cast<const uint32_t*>(&h01);       // row g4, k 8nt + 2t4
                ph[2 * nt + 1] = *reinterpret_cast<const uint32_t*>(&h23);   // row g4 + 8
                pl[2 * nt] = pack_bf16(pr[nt][0] - f01.x, pr[nt][1] - f01.y);
                pl[2 * nt + 1] = pack_bf16(pr[nt][2] - f23.x, pr[nt][3] - f23.y);
            }
            const uint32_t pa_h[4] = {ph[0], ph[1], ph[2], ph[3]};
            const uint32_t pa_l[4] = {pl[0], pl[1], pl[2], pl[3]};
            // O[16 x D] += P V: B = V (k = token, n = d) via ldmatrix.trans, two d tiles per load
#pragma unroll
            for (int dp = 0; dp < D / 16; ++dp) {
                uint32_t v0, v1, v2, v3;
                ldsm_x4_t(vt + swz<D>((lane & 7) + 8 * ((lane >> 3) & 1), dp * 2 + (lane >> 4)), v0, v1, v2, v3);
                mma_bf16_16816(o[2 * dp], pa_h, v0, v1);
                mma_bf16_16816(o[2 * dp], pa_l, v0, v1);
                mma_bf16_16816(o[2 * dp + 1], pa_h, v2, v3);
                mma_bf16_16816(o[2 * dp + 1], pa_l, v2, v3);
            }
        }
        }
        __syncthreads();  // buffer buf is refilled by the next iteration's prefetch
    }
    if (!live_w) return;
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
    bool bad = false;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        const int r = half ? r_hi : r_lo;
        const int pos = half ? pos_hi : pos_lo;
        if (pos < 0) continue;
        const float l = half ? l_hi : l_lo;
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const int i = i0 + r / gs, j = h * gs + r % gs;
        float* out = p.out + (((size_t)b * p.ntok + i) * p.m + j) * D;
#pragma unroll
        for (int dt = 0; dt < D / 8; ++dt) {
            const float2 v = make_float2(o[dt][2 * half] * inv, o[dt][2 * half + 1] * inv);
            bad |= !(isfinite(v.x) && isfinite(v.y));
            *reinterpret_cast<float2*>(out + dt * 8 + 2 * t4) = v;
        }
        if (p.lse_out && t4 == 0) {
            const float m = half ? m_hi : m_lo;
            p.lse_out[((size_t)b * p.ntok + i) * p.m + j] = (l > 0.f) ? (m + log2f(l)) * kLn2 : -INFINITY;
        }
    }
    if (bad) set_err(p.err, kDevNumeric);
}

}  // namespace

size_t prefill_smem_bytes(int d, int gs) {
    return 1024 + 2 * kPPS * (size_t)(d == 128 ? TileLayout<128>::kBytes : TileLayout<64>::kBytes) +
           (size_t)prefill_qb(gs) * gs * (d + 8) * 2;
}

cudaError_t launch_prefill(const PrefillParams& p, cudaStream_t st, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    const int qb = prefill_qb(p.gs);
    cfg.gridDim = dim3((p.ntok + qb - 1) / qb, p.g, p.batch);
    cfg.blockDim = dim3(32 * p.gs * qb / 16);
    cfg.dynamicSmemBytes = prefill_smem_bytes(p.d, p.gs);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    const bool big = qb == 32;
    const void* fn = p.d == 128 ? (big ? (const void*)prefill_kernel<128, 32> : (const void*)prefill_kernel<128, 16>)
                   : p.d == 64  ? (big ? (const void*)prefill_kernel<64, 32> : (const void*)prefill_kernel<64, 16>)
                                : nullptr;
    if (!fn) return cudaErrorInvalidValue;
    static std::atomic<int> cache[kMaxDevices * 4];  // per (device, instantiation)
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
    const int slot = dev * 4 + (p.d == 128 ? 0 : 2) + (big ? 1 : 0);
    if (cache[slot].load(std::memory_order_acquire) == 0) {  // opt in to the dynamic shared memory
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max(prefill_smem_bytes(128, 8), prefill_smem_bytes(128, kMaxGs)));
        if (e != cudaSuccess) return e;
        cache[slot].store(1, std::memory_order_release);
    }
    void* args[] = {const_cast<PrefillParams*>(&p)};
    return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace delta
