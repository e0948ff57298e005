// Primitive latencies on this B200 (cycles, SM clock): dependent global loads that hit L2 or
// miss to HBM, __syncthreads at 256 / 1024 threads, shared atomics (spread / one address),
// __match_any_sync, a chain of dependent mma.sync m16n8k16 bf16, an ex2 chain, and the cost of
// reading %globaltimer.  One CTA unless stated; each figure is cycles per operation.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);             \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

__device__ long long g_out[64];
__device__ int g_sink;

__global__ void chase(const int* __restrict__ next, int n, int reps, int slot) {
    int i = 0;
    // warm: one pass
    for (int r = 0; r < n; ++r) i = __ldcg(next + i);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) i = __ldcg(next + i);
    const long long t1 = clock64();
    if (threadIdx.x == 0) { g_out[slot] = (t1 - t0) / reps; g_sink = i; }
}

__global__ void chase_cold(const int* __restrict__ next, int start, int reps, int slot) {
    int i = start;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) i = __ldcg(next + i);
    const long long t1 = clock64();
    if (threadIdx.x == 0) { g_out[slot] = (t1 - t0) / reps; g_sink = i; }
}

__global__ void bar_lat(int reps, int slot) {
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) g_out[slot] = (t1 - t0) / reps;
}

__global__ void atom_lat(int reps, int same, int slot) {
    __shared__ int h[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) atomicAdd(&h[same ? 0 : (threadIdx.x * 33) & 1023], 1);
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) { g_out[slot] = (t1 - t0) / reps; g_sink = h[0]; }
}

__global__ void match_lat(int reps, int slot) {
    int v = threadIdx.x & 7;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) v = (int)__match_any_sync(0xffffffffu, v) & 15;
    const long long t1 = clock64();
    if (threadIdx.x == 0) { g_out[slot] = (t1 - t0) / reps; g_sink = v; }
}

__global__ void shfl_lat(int reps, int slot) {
    float v = threadIdx.x;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1.f;
    const long long t1 = clock64();
    if (threadIdx.x == 0) { g_out[slot] = (t1 - t0) / reps; g_sink = (int)v; }
}

__global__ void mma_lat(int reps, int chains, int slot) {
    float d[4][4] = {};
    const uint32_t a[4] = {0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u};
    const uint32_t b0 = 0x3c003c00u, b1 = 0x3c003c00u;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (c < chains)
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) { g_out[slot] = (t1 - t0) / reps; g_sink = (int)(d[0][0] + d[1][0] + d[2][0] + d[3][0]); }
}

__global__ void ex2_lat(int reps, int slot) {
    float v = threadIdx.x * 1e-3f;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v));
    const long long t1 = clock64();
    if (threadIdx.x == 0) { g_out[slot] = (t1 - t0) / reps; g_sink = (int)v; }
}

__global__ void gt_lat(int reps, int slot) {
    unsigned long long acc = 0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        acc += t;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) { g_out[slot] = (t1 - t0) / reps; g_sink = (int)acc; }
}

int main() {
    const int n_l2 = 1 << 16;          // 256 KB ring, fully warmed: L2 resident
    const int n_hbm = 1 << 28;         // 1 GB ring: misses
    int *ring_l2, *ring_hbm;
    int idx_start = 0;
    CK(cudaMalloc(&ring_l2, (size_t)n_l2 * 4));
    CK(cudaMalloc(&ring_hbm, (size_t)n_hbm * 4));
    {   // random permutation cycles with a large stride (defeat prefetch)
        std::vector<int> h(n_l2);
        for (int i = 0; i < n_l2; ++i) h[i] = (i + 32 * 37) % n_l2;  // stride 37 lines: one 4096-hop cycle
        CK(cudaMemcpy(ring_l2, h.data(), (size_t)n_l2 * 4, cudaMemcpyHostToDevice));
        std::vector<int> g(n_hbm / 1024);
        // sparse chain in the big ring: element k*1024*stride hops
        CK(cudaMemset(ring_hbm, 0, (size_t)n_hbm * 4));
        idx_start = 0;
        std::vector<int> idx(4096);
        for (int k = 0; k < 4096; ++k) idx[k] = (int)(((long long)k * 2654435761ull) % (n_hbm / 4096)) * 4096 + (k & 1023) * 4;
        for (int k = 0; k < 4096; ++k) CK(cudaMemcpy(ring_hbm + idx[k], &idx[(k + 1) % 4096], 4, cudaMemcpyHostToDevice));
        idx_start = idx[0];
    }
    long long out[64];
    chase<<<1, 32>>>(ring_l2, 8192, 2000, 0);
    chase_cold<<<1, 32>>>(ring_hbm, idx_start, 2000, 1);
    bar_lat<<<1, 256>>>(1000, 2);
    bar_lat<<<1, 1024>>>(1000, 3);
    atom_lat<<<1, 1024>>>(200, 0, 4);
    atom_lat<<<1, 1024>>>(200, 1, 5);
    match_lat<<<1, 32>>>(1000, 6);
    shfl_lat<<<1, 32>>>(1000, 7);
    mma_lat<<<1, 32>>>(1000, 1, 8);
    mma_lat<<<1, 32>>>(1000, 4, 9);
    mma_lat<<<1, 128>>>(1000, 4, 10);
    mma_lat<<<1, 256>>>(1000, 4, 11);
    ex2_lat<<<1, 32>>>(1000, 12);
    gt_lat<<<1, 32>>>(1000, 13);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpyFromSymbol(out, g_out, sizeof out));
    const char* names[] = {"L2-hit dependent load (warmed 256 KB ring)", "HBM dependent load (TLB mostly hit)", "__syncthreads 256 thr",
                           "__syncthreads 1024 thr", "smem atomicAdd spread, 1024 thr (per round)",
                           "smem atomicAdd same addr, 1024 thr (per round)", "__match_any_sync", "shfl_xor + fadd",
                           "mma.sync m16n8k16 bf16, 1 chain (per mma)", "mma.sync 4 chains, 1 warp (per round of 4)",
                           "mma.sync 4 chains, 4 warps (per round)", "mma.sync 4 chains, 8 warps (per round)",
                           "ex2.approx chain", "read %globaltimer"};
    for (int i = 0; i < 14; ++i) printf("%-52s %6lld cycles\n", names[i], out[i]);
    return 0;
}
