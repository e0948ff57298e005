// Unit test of the tcgen05 (UMMA) operand descriptors used by the decode kernel, on one CTA:
//   QK: S[128 x 16] = Q[128 x 128] . K^T   A = Q (K-major SW128, 8 real rows aliased by SBO = 0)
//                                          B = K tile [16 tok][128 d] (K-major SW128, halves 4 KiB apart)
//   PV: O^T[128 x 8] = V^T[128 x 16] . P^T  A = V tile [16 tok][128 d] (MN-major SW128: LBO 4 KiB, SBO 1 KiB)
//                                          B = P [8 heads][16 tok] bf16 (K-major, no swizzle: LBO 128 B)
// Smem tile layout = what the TMA box {64, 32 rows, 2 halves} with SWIZZLE_128B writes: [half][row][128 B],
// 16-byte chunk c of row r at half*4096 + r*128 + ((c ^ (r & 7)) << 4); V rows are rows 16..31.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;               // version 1 (sm_100)
    d |= (uint64_t)(layout & 7) << 61;    // 0 none, 2 SW128
    return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, int acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d), "l"(a), "l"(b),
                 "r"(id), "r"(acc));
}

__global__ void umma_test(const __nv_bfloat16* gq, const __nv_bfloat16* gk, const __nv_bfloat16* gv,
                          const __nv_bfloat16* gp, float* s_out, float* o_out) {
    __shared__ __align__(1024) uint8_t tile[8192];   // [half][32 rows][128 B]: K rows 0-15, V rows 16-31
    __shared__ __align__(1024) uint8_t qs[2048];     // Q: 2 halves x 8 rows x 128 B (SW128)
    __shared__ __align__(128) uint8_t ps[256];       // P: 2 core matrices (tok 0-7, 8-15) x 8 rows x 16 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // stage operands with the TMA swizzle
    for (int i = tid; i < 32 * 16; i += blockDim.x) {  // rows 0..31 (K then V), 16 chunks of 8 bf16
        const int r = i / 16, c = i % 16;
        const __nv_bfloat16* src = (r < 16 ? gk + r * 128 : gv + (r - 16) * 128) + c * 8;
        *reinterpret_cast<uint4*>(tile + (c >> 3) * 4096 + r * 128 + (((c & 7) ^ (r & 7)) << 4)) =
            *reinterpret_cast<const uint4*>(src);
    }
    for (int i = tid; i < 8 * 16; i += blockDim.x) {
        const int r = i / 16, c = i % 16;
        *reinterpret_cast<uint4*>(qs + (c >> 3) * 1024 + r * 128 + (((c & 7) ^ (r & 7)) << 4)) =
            *reinterpret_cast<const uint4*>(gq + r * 128 + c * 8);
    }
    for (int i = tid; i < 8 * 2; i += blockDim.x) {  // P row h, tokens 8j..8j+7 -> core matrix j
        const int h = i / 2, j = i % 2;
        *reinterpret_cast<uint4*>(ps + j * 128 + h * 16) = *reinterpret_cast<const uint4*>(gp + h * 16 + j * 8);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base;
    const uint32_t tS = tbase, tO = tbase + 16;
    if (tid == 0) {
        // QK: 8 k-steps of 16 elements; 4 per 128-byte half
        const uint32_t iq = idesc_bf16(128, 16, 0, 0);
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 0 + (kk & 3) * 32;
            const uint64_t a = desc(su(qs) + (kk >> 2) * 1024 + (kk & 3) * 32, 16, 0, 2);
            const uint64_t b = desc(su(tile) + (kk >> 2) * 4096 + (kk & 3) * 32, 16, 1024, 2);
            (void)off;
            mma(tS, a, b, iq, kk > 0);
        }
        // PV: A = V^T (MN-major SW128), B = P (K-major, no swizzle)
        const uint32_t ip = idesc_bf16(128, 8, 1, 0);
        const uint64_t a = desc(su(tile) + 2048, 4096, 1024, 2);
        const uint64_t b = desc(su(ps), 128, 0, 0);
        mma(tO, a, b, ip, 0);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
    }
    __syncwarp();
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0; @!P bra W;}" ::"r"(su(&bar)));
    if (tid == 0) {
        const uint32_t iq = idesc_bf16(128, 16, 0, 0);
        const uint32_t ip = idesc_bf16(128, 8, 1, 0);
        long long t_issue = 0, t_total = 0, t_pv = 0;
        for (int it = 0; it < 64; ++it) {
            const long long c0 = clock64();
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t a = desc(su(qs) + (kk >> 2) * 1024 + (kk & 3) * 32, 16, 0, 2);
                const uint64_t b = desc(su(tile) + (kk >> 2) * 4096 + (kk & 3) * 32, 16, 1024, 2);
                mma(tS, a, b, iq, kk > 0);
            }
            const long long c1 = clock64();
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
            asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(su(&bar)), "r"((it + 1) & 1));
            const long long c2 = clock64();
            t_issue += c1 - c0;
            t_total += c2 - c0;
        }
        for (int it = 0; it < 64; ++it) {
            const long long c0 = clock64();
            const uint64_t a = desc(su(tile) + 2048, 4096, 1024, 2);
            mma(tO, a, desc(su(ps), 128, 0, 0), ip, 1);
            mma(tO, a, desc(su(ps), 128, 0, 0), ip, 1);
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
            asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(su(&bar)), "r"((it + 65) & 1));
            t_pv += clock64() - c0;
        }
        printf("QK 8 MMAs: issue %lld cyc, issue+complete %lld cyc;  PV 2 MMAs issue+complete %lld cyc (avg of 64)\n",
               t_issue / 64, t_total / 64, t_pv / 64);
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- A from TMEM: Q rows (lane r holds head r % 8) packed 2 bf16 per 32-bit column at cols 128..191
    {
        const uint32_t tQ = tbase + 128 + ((uint32_t)(warp * 32) << 16);
        const uint32_t* qrow = reinterpret_cast<const uint32_t*>(gq + (lane % 8) * 128);
        uint32_t r[32];
        for (int half = 0; half < 2; ++half) {
            for (int j = 0; j < 32; ++j) r[j] = qrow[half * 32 + j];
            asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                         "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                         :: "r"(tQ + half * 32), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
                            "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
                            "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
                            "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]),
                            "r"(r[31]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) {
        const uint32_t iq = idesc_bf16(128, 16, 0, 0);
        long long t_issue = 0, t_total = 0;
        for (int it = 0; it < 65; ++it) {
            const long long c0 = clock64();
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t b = desc(su(tile) + (kk >> 2) * 4096 + (kk & 3) * 32, 16, 1024, 2);
                const uint32_t ta = tbase + 128 + kk * 8;
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tbase + 32), "r"(ta),
                             "l"(b), "r"(iq), "r"(kk > 0 ? 1 : 0));
            }
            const long long c1 = clock64();
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
            asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(su(&bar)), "r"((it + 129) & 1));
            const long long c2 = clock64();
            if (it > 0) { t_issue += c1 - c0; t_total += c2 - c0; }
        }
        printf("QK (A in TMEM) 8 MMAs: issue %lld cyc, issue+complete %lld cyc\n", t_issue / 64, t_total / 64);
        // interleave 4 independent accumulators (4 tiles): 32 MMAs
        for (int nd : {1, 2, 4}) {
            long long ti = 0, tt = 0;
            for (int it = 0; it < 65; ++it) {
                const long long c0 = clock64();
                for (int kk = 0; kk < 8; ++kk)
                    for (int dd = 0; dd < nd; ++dd) {
                        const uint64_t a = desc(su(qs) + (kk >> 2) * 1024 + (kk & 3) * 32, 16, 0, 2);
                        const uint64_t b = desc(su(tile) + (kk >> 2) * 4096 + (kk & 3) * 32, 16, 1024, 2);
                        mma(tbase + 48 + 16 * dd, a, b, iq, kk > 0);
                    }
                const long long c1 = clock64();
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
                asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(su(&bar)), "r"((it + 194 + (nd == 1 ? 0 : nd == 2 ? 65 : 130)) & 1));
                const long long c2 = clock64();
                if (it > 0) { ti += c1 - c0; tt += c2 - c0; }
            }
            printf("SS QK, %d independent accumulators x 8 MMAs: issue %lld cyc, issue+complete %lld cyc\n", nd, ti / 64, tt / 64);
        }
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    {   // compare S2 (cols 32..47) with S (cols 0..15)
        uint32_t a[16], c[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]),
                       "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15])
                     : "r"(tS + ((uint32_t)(warp * 32) << 16)));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]), "=r"(c[7]),
                       "=r"(c[8]), "=r"(c[9]), "=r"(c[10]), "=r"(c[11]), "=r"(c[12]), "=r"(c[13]), "=r"(c[14]), "=r"(c[15])
                     : "r"(tbase + 32 + ((uint32_t)(warp * 32) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        float md = 0.f;
        for (int j = 0; j < 16; ++j) md = fmaxf(md, fabsf(__uint_as_float(a[j]) - __uint_as_float(c[j])));
        for (int o = 16; o > 0; o >>= 1) md = fmaxf(md, __shfl_xor_sync(0xffffffffu, md, o));
        if (lane == 0 && warp == 0) printf("A-in-TMEM QK vs SS QK: max |diff| %g (S[0][0] %f vs %f)\n", md,
                                          __uint_as_float(a[0]), __uint_as_float(c[0]));
    }
    // S: lanes 0..127 x 16 columns (warp w reads lanes 32w..32w+31)
    uint32_t v[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(tS + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) s_out[(warp * 32 + lane) * 16 + j] = __uint_as_float(v[j]);
    uint32_t w8[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w8[0]), "=r"(w8[1]), "=r"(w8[2]), "=r"(w8[3]), "=r"(w8[4]), "=r"(w8[5]), "=r"(w8[6]), "=r"(w8[7])
                 : "r"(tO + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) o_out[(warp * 32 + lane) * 8 + j] = __uint_as_float(w8[j]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

static float bf(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }

int main() {
    const int nq = 8 * 128, nk = 16 * 128, np = 8 * 16;
    uint16_t hq[nq], hk[nk], hv[nk], hp[np];
    srand(5);
    auto rb = [] { float f = (rand() / (float)RAND_MAX - 0.5f) * 2.f; uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); };
    for (auto& x : hq) x = rb();
    for (auto& x : hk) x = rb();
    for (auto& x : hv) x = rb();
    for (auto& x : hp) x = rb();
    __nv_bfloat16 *dq, *dk, *dv, *dp;
    float *ds, *dout;
    cudaMalloc(&dq, sizeof hq); cudaMalloc(&dk, sizeof hk); cudaMalloc(&dv, sizeof hv); cudaMalloc(&dp, sizeof hp);
    cudaMalloc(&ds, 128 * 16 * 4); cudaMalloc(&dout, 128 * 8 * 4);
    cudaMemcpy(dq, hq, sizeof hq, cudaMemcpyHostToDevice); cudaMemcpy(dk, hk, sizeof hk, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, hv, sizeof hv, cudaMemcpyHostToDevice); cudaMemcpy(dp, hp, sizeof hp, cudaMemcpyHostToDevice);
    umma_test<<<1, 128>>>(dq, dk, dv, dp, ds, dout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    float hs[128 * 16], ho[128 * 8];
    cudaMemcpy(hs, ds, sizeof hs, cudaMemcpyDeviceToHost);
    cudaMemcpy(ho, dout, sizeof ho, cudaMemcpyDeviceToHost);
    double es = 0, eo = 0, es_alias = 0;
    for (int h = 0; h < 128; ++h)
        for (int t = 0; t < 16; ++t) {
            double ref = 0;
            for (int d = 0; d < 128; ++d) ref += (double)bf(hq[(h % 8) * 128 + d]) * bf(hk[t * 128 + d]);
            const double err = fabs(ref - hs[h * 16 + t]);
            if (h < 8) es = fmax(es, err); else es_alias = fmax(es_alias, err);
        }
    for (int d = 0; d < 128; ++d)
        for (int h = 0; h < 8; ++h) {
            double ref = 0;
            for (int t = 0; t < 16; ++t) ref += (double)bf(hv[t * 128 + d]) * bf(hp[h * 16 + t]);
            eo = fmax(eo, fabs(ref - ho[d * 8 + h]));
        }
    printf("QK max err rows 0-7: %.3g (aliased rows 8-127: %.3g)   PV max err: %.3g\n", es, es_alias, eo);
    printf("S[0][0..3] %f %f %f %f   O^T[0][0..3] %f %f %f %f\n", hs[0], hs[1], hs[2], hs[3], ho[0], ho[1], ho[2], ho[3]);
    return 0;
}
