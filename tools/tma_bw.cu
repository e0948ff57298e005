// Per-SM ingest microbenchmark (B200): how fast can one CTA pull HBM data into shared memory?
//  mode 0: cp.async.bulk (1-D TMA) 4 KiB chunks, one producer thread, NST-deep ring
//  mode 1: LDG.128 by all warps into registers (sum to defeat DCE)
//  mode 2: cp.async.bulk with 16 KiB chunks
// Chunks are random 4 KiB pages of a 2 GiB buffer (like a paged KV cache).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include <cuda.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CHUNK, int NST>
__global__ void __launch_bounds__(160) bulk_kernel(const uint8_t* __restrict__ src, const int* __restrict__ pages,
                                                   int n_per_cta, float* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NST * CHUNK);
    uint64_t* empty = full + NST;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(su(&empty[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int* pg = pages + (size_t)blockIdx.x * n_per_cta;
    float acc = 0.f;
    if (warp == 4) {
        if (lane == 0) {
            for (int i = 0; i < n_per_cta; ++i) {
                const int st = i % NST, rnd = i / NST;
                if (rnd > 0) {
                    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}"
                                 ::"r"(su(&empty[st])), "r"((rnd - 1) & 1));
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(CHUNK));
                const uint8_t* g = src + (size_t)pg[i] * CHUNK;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su(sm + st * CHUNK)), "l"(g), "r"(CHUNK), "r"(su(&full[st])) : "memory");
            }
        }
    } else {
        for (int i = 0; i < n_per_cta; ++i) {
            const int st = i % NST, rnd = i / NST;
            asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}"
                         ::"r"(su(&full[st])), "r"(rnd & 1));
            acc += reinterpret_cast<const float*>(sm + st * CHUNK)[tid];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[st])));
        }
    }
    if (acc == 12345.f) sink[0] = acc;
}

template <int NST>
__global__ void __launch_bounds__(160) tensor_kernel(const __grid_constant__ CUtensorMap tm, const int* __restrict__ pages,
                                                     int n_per_cta, float* sink) {
    constexpr int CHUNK = 4096;
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NST * CHUNK);
    uint64_t* empty = full + NST;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(su(&empty[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int* pg = pages + (size_t)blockIdx.x * n_per_cta;
    float acc = 0.f;
    if (warp == 4) {
        if (lane == 0) {
            for (int i = 0; i < n_per_cta; ++i) {
                const int st = i % NST, rnd = i / NST;
                if (rnd > 0) {
                    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}"
                                 ::"r"(su(&empty[st])), "r"((rnd - 1) & 1));
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(CHUNK));
                const int row0 = pg[i] * 16;
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su(sm + st * CHUNK)),
                             "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su(&full[st])), "r"(0), "r"(0), "r"(row0)
                             : "memory");
            }
        }
    } else {
        for (int i = 0; i < n_per_cta; ++i) {
            const int st = i % NST, rnd = i / NST;
            asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}"
                         ::"r"(su(&full[st])), "r"(rnd & 1));
            acc += reinterpret_cast<const float*>(sm + st * CHUNK)[tid];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[st])));
        }
    }
    if (acc == 12345.f) sink[0] = acc;
}

// BOX boxes of 4 KiB per stage under one expect_tx; ISSUERS lanes issue them in parallel
template <int NST, int BOX, int ISSUERS, int BB = 4096>
__global__ void __launch_bounds__(160) tensor_multi(const __grid_constant__ CUtensorMap tm, const int* __restrict__ pages,
                                                    int n_per_cta, float* sink) {
    constexpr int CHUNK = BB * BOX;
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NST * CHUNK);
    uint64_t* empty = full + NST;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(su(&empty[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int* pg = pages + (size_t)blockIdx.x * n_per_cta;
    float acc = 0.f;
    const int nst = n_per_cta / BOX;
    if (warp == 4) {
        for (int i = 0; i < nst; ++i) {
            const int st = i % NST, rnd = i / NST;
            if (rnd > 0) {
                asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}"
                             ::"r"(su(&empty[st])), "r"((rnd - 1) & 1));
            }
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(CHUNK));
            __syncwarp();
            for (int bx = lane; bx < BOX; bx += ISSUERS) {
                if (lane >= ISSUERS) break;
                const int row0 = (pg[i * BOX + bx] % (int)(2147483648ull / BB)) * (BB / 256);
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                             " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su(sm + st * CHUNK + bx * BB)),
                             "l"(reinterpret_cast<uint64_t>(&tm)), "r"(su(&full[st])), "r"(0), "r"(0), "r"(row0)
                             : "memory");
            }
        }
    } else {
        for (int i = 0; i < nst; ++i) {
            const int st = i % NST, rnd = i / NST;
            asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}"
                         ::"r"(su(&full[st])), "r"(rnd & 1));
            acc += reinterpret_cast<const float*>(sm + st * CHUNK)[tid];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[st])));
        }
    }
    if (acc == 12345.f) sink[0] = acc;
}

__global__ void __launch_bounds__(256) ldg_kernel(const uint8_t* __restrict__ src, const int* __restrict__ pages,
                                                  int n_per_cta, float* sink) {
    const int* pg = pages + (size_t)blockIdx.x * n_per_cta;
    float acc = 0.f;
    // 256 threads x 16 B = 4 KiB = one page per iteration; unroll 8 pages for MLP
    for (int i = 0; i < n_per_cta; i += 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint4* g = reinterpret_cast<const uint4*>(src + (size_t)pg[min(i + u, n_per_cta - 1)] * 4096);
            v[u] = __ldg(g + threadIdx.x);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += __uint_as_float(v[u].x ^ v[u].y ^ v[u].z ^ v[u].w);
    }
    if (acc == 12345.f) sink[0] = acc;
}

int main() {
    const size_t bytes = 2ull << 30;
    uint8_t* src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    float* sink;
    cudaMalloc(&sink, 4);
    const int n_pages4k = bytes / 4096;
    const int per_cta = 2048;
    std::vector<int> h(148 * per_cta * 2);
    uint64_t x = 88172645463325252ull;
    auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
    int* dpages;
    cudaMalloc(&dpages, h.size() * 4);
    auto bulk4 = bulk_kernel<4096, 12>;
    auto bulk16 = bulk_kernel<16384, 6>;
    cudaFuncSetAttribute(bulk4, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 4096 + 256);
    cudaFuncSetAttribute(bulk16, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16384 + 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto bulk4d = bulk_kernel<4096, 48>;
    cudaFuncSetAttribute(bulk4d, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 4096 + 1024);
    auto tens = tensor_kernel<48>;
    cudaFuncSetAttribute(tens, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 4096 + 2048);
    CUtensorMap tm;
    {
        const cuuint64_t dims[3] = {64, 2, (cuuint64_t)(bytes / 256)};
        const cuuint64_t strides[2] = {128, 256};
        const cuuint32_t box[3] = {64, 2, 16};
        const cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, src, dims, strides, box, estr,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("encode %d\n", (int)r);
    }
    {
        const int npg = (int)(bytes / 4096);
        for (size_t i = 0; i < h.size(); ++i) h[i] = (int)(rnd() % npg);
        cudaMemcpy(dpages, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    }
    auto run = [&](auto kern, int smem, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int grid : {1, 16, 148}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                kern<<<grid, 160, smem>>>(tm, dpages, per_cta, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double b = (double)grid * per_cta * 4096;
            printf("%-28s grid %3d: %.1f GB/s total, %.1f GB/s per CTA\n", name, grid, b / ms / 1e6, b / ms / 1e6 / grid);
        }
    };
    run(tensor_multi<12, 4, 4>, 12 * 16384 + 2048, "4KB x4/stage");
    CUtensorMap tm8 = tm, tm16 = tm;
    for (int which = 0; which < 2; ++which) {
        const cuuint64_t dims[3] = {64, 2, (cuuint64_t)(bytes / 256)};
        const cuuint64_t strides[2] = {128, 256};
        const cuuint32_t box[3] = {64, 2, which == 0 ? 32u : 64u};
        const cuuint32_t estr[3] = {1, 1, 1};
        cuTensorMapEncodeTiled(which == 0 ? &tm8 : &tm16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, src, dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    auto run2 = [&](auto kern, const CUtensorMap& m, int smem, int bb, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int grid : {1, 16, 128, 148}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                kern<<<grid, 160, smem>>>(m, dpages, per_cta, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double b = (double)grid * per_cta * bb;
            printf("%-28s grid %3d: %.1f GB/s total, %.1f GB/s per CTA\n", name, grid, b / ms / 1e6, b / ms / 1e6 / grid);
        }
    };
    run2(tensor_multi<6, 4, 4, 8192>, tm8, 6 * 32768 + 2048, 8192, "8KB x4/stage");
    run2(tensor_multi<3, 4, 4, 16384>, tm16, 3 * 65536 + 2048, 16384, "16KB x4/stage");
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    (void)n_pages4k;
    return 0;
}
