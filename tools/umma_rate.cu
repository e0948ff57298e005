// tcgen05.mma (kind::f16, cta_group::1, SS operands) issue throughput on one CTA: R back-to-back
// MMAs M=128, K=16, N in {8, 16, 32, 64, 128, 256} accumulating into one TMEM tile, then commit
// + mbarrier wait; cycles per MMA (operand contents are irrelevant for the rate).  Compare with
// the guide's floor max(M,128) * N / 256 cycles.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void rate(long long* out, int R) {
    __shared__ __align__(1024) uint8_t a[16384];   // 128 rows x 128 B (one SW128 K-block of A)
    __shared__ __align__(1024) uint8_t bm[16384];  // 128 rows x 128 B (B rows alias past 128: rate only)
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 16384 / 16; i += blockDim.x) reinterpret_cast<uint4*>(a)[i] = make_uint4(0, 0, 0, 0);
    for (int i = tid; i < 16384 / 16; i += blockDim.x) reinterpret_cast<uint4*>(bm)[i] = make_uint4(0, 0, 0, 0);
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int Ns[6] = {8, 16, 32, 64, 128, 256};
    for (int ni = 0; ni < 6; ++ni) {
        const int N = Ns[ni];
        const uint32_t id = idesc(128, N);
        long long t0 = 0, t1 = 0;
        if (tid == 0) {
            const uint64_t da = desc(su(a), 16, 0), db = desc(su(bm), 16, 0);  // SBO 0: 8-row groups alias (rate only)
            t0 = clock64();
            for (int r = 0; r < R; ++r)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                             ::"r"(tbase), "l"(da), "l"(db), "r"(id), "r"(r > 0 ? 1 : 0));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar))
                         : "memory");
            asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                         "@!P1 bra W_%=;\n}" ::"r"(su(&bar)), "r"(ni & 1) : "memory");
            t1 = clock64();
            out[ni] = (t1 - t0);
        }
        __syncthreads();
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

int main() {
    long long* d;
    cudaMalloc(&d, 64 * sizeof(long long));
    for (int R : {64, 512}) {
        rate<<<1, 128>>>(d, R);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[6];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        const int Ns[6] = {8, 16, 32, 64, 128, 256};
        printf("R=%d (%s)\n", R, cudaGetErrorString(e));
        for (int i = 0; i < 6; ++i)
            printf("  M128 N%-3d K16: %7.1f cycles per MMA (floor %d)\n", Ns[i], (double)h[i] / R,
                   128 * Ns[i] / 256);
    }
    return 0;
}
