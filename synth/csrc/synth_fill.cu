// synth_fill.cu — device implementation of the seeded input generator in synth/__init__.py
// (counter-based splitmix64 + integer Irwin-Hall(12) + bit-level bf16 RNE).  Bit-identical
// to the numpy implementation; holds none of DELTA's arithmetic.  Test/bench
// infrastructure: fills KV pools and per-step queries directly in HBM.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t tag, uint64_t layer, uint64_t seq,
                                                        uint64_t step) {
    uint64_t k = splitmix64(seed);
    k = splitmix64(k ^ tag);
    k = splitmix64(k ^ layer);
    k = splitmix64(k ^ seq);
    k = splitmix64(k ^ step);
    return k;
}

__device__ __forceinline__ float normal_f32(uint64_t key, uint64_t idx) {
    int64_t S = 0;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        const uint64_t w = splitmix64(key + idx * 3ull + (uint64_t)r);
#pragma unroll
        for (int c = 0; c < 4; ++c) S += (int64_t)((w >> (16 * c)) & 0xFFFFull);
    }
    return __fmul_rn((float)(S - 393210), 1.52587890625e-05f);  // exact: |S-mean| < 2^24
}

__device__ __forceinline__ float round_bf16(float x) {
    uint32_t u = __float_as_uint(x);
    const uint32_t lsb = (u >> 16) & 1u;
    u = (u + 0x7FFFu + lsb) & 0xFFFF0000u;
    return __uint_as_float(u);
}

// pool [L][num_phys][g][kv_slots][P][d]; fills logical rows t < s_fill of layers
// [layer0, layer0+nl), sequences [0, batch), into slot `kv_slot` (0 = K, 1 = V when the pool
// interleaves K and V per (page, head)).  plant_mask: [nl][batch][plant_stride].
__global__ void fill_pool_kernel(void* pool, int bf16, uint64_t seed, int tag, int layer0, int batch, int s_fill,
                                 int g, int d, int P, int num_phys, const int32_t* bt, int bt_stride,
                                 const uint8_t* plant_mask, int plant_block, int plant_stride, const float* sigma,
                                 float B, int kv_slots, int kv_slot) {
    const int ls = blockIdx.y;  // (layer offset, seq)
    const int li = ls / batch, b = ls % batch;
    const int layer = layer0 + li;
    const uint64_t key = stream_key(seed, (uint64_t)tag, (uint64_t)layer, (uint64_t)b, 0);
    const long long n = (long long)s_fill * g * d;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(i % d);
        const int h = (int)((i / d) % g);
        const int t = (int)(i / ((long long)d * g));
        float x = normal_f32(key, (uint64_t)i);
        const bool planted = plant_mask && plant_mask[((size_t)li * batch + b) * plant_stride + t / plant_block];
        if (bf16) x = round_bf16(x);
        if (planted) {
            x = __fadd_rn(x, __fmul_rn(B, sigma[((size_t)li * batch + b) * d + e]));
            if (bf16) x = round_bf16(x);
        }
        const size_t row =
            ((((size_t)layer * num_phys + bt[(size_t)b * bt_stride + t / P]) * g + h) * kv_slots + kv_slot) * P + (t % P);
        if (bf16)
            reinterpret_cast<__nv_bfloat16*>(pool)[row * d + e] = __float2bfloat16_rn(x);  // exact
        else
            reinterpret_cast<float*>(pool)[row * d + e] = x;
    }
}

// out [nl][batch][rows][d] contiguous: rows of a logical tensor (tag) at `step`,
// element index (row*d + e) + idx_offset;  tag Q: rows = m query heads, step = s.
// KV-row mode (tag K/V): rows = g heads of token `step`... handled by idx_offset.
__global__ void fill_rows_kernel(void* out, int bf16, uint64_t seed, int tag, int layer0, int batch,
                                 const int32_t* steps /*[batch]*/, int use_step_key, int rows, int d,
                                 const int64_t* idx_offset /*[batch] or null*/, const uint8_t* planted /*[nl][batch]*/,
                                 const float* sigma, float boost) {
    const int ls = blockIdx.y;
    const int li = ls / batch, b = ls % batch;
    const int layer = layer0 + li;
    const uint64_t key =
        stream_key(seed, (uint64_t)tag, (uint64_t)layer, (uint64_t)b, use_step_key ? (uint64_t)steps[b] : 0ull);
    const int n = rows * d;
    const int64_t off = idx_offset ? idx_offset[b] : 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int e = i % d;
        float x = normal_f32(key, (uint64_t)(off + i));
        const bool pl = planted && planted[(size_t)li * batch + b];
        if (bf16) x = round_bf16(x);
        if (pl) {
            x = __fadd_rn(x, __fmul_rn(boost, sigma[((size_t)li * batch + b) * d + e]));
            if (bf16) x = round_bf16(x);
        }
        const size_t o = ((size_t)ls * rows) * d + i;
        if (bf16)
            reinterpret_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16_rn(x);
        else
            reinterpret_cast<float*>(out)[o] = x;
    }
}

}  // namespace

extern "C" {

int synth_fill_pool(void* pool, int bf16, uint64_t seed, int tag, int layer0, int nl, int batch, int s_fill, int g,
                    int d, int P, int num_phys, const int32_t* bt, int bt_stride, const uint8_t* plant_mask,
                    int plant_block, int plant_stride, const float* sigma, float B, int kv_slots, int kv_slot,
                    cudaStream_t st) {
    if (s_fill <= 0) return 0;
    const long long n = (long long)s_fill * g * d;
    const int threads = 256;
    long long blocks = (n + threads - 1) / threads;
    if (blocks > 4096) blocks = 4096;
    dim3 grid((unsigned)blocks, (unsigned)(nl * batch));
    fill_pool_kernel<<<grid, threads, 0, st>>>(pool, bf16, seed, tag, layer0, batch, s_fill, g, d, P, num_phys, bt,
                                               bt_stride, plant_mask, plant_block, plant_stride, sigma, B,
                                               kv_slots, kv_slot);
    return (int)cudaGetLastError();
}

int synth_fill_rows(void* out, int bf16, uint64_t seed, int tag, int layer0, int nl, int batch, const int32_t* steps,
                    int use_step_key, int rows, int d, const int64_t* idx_offset, const uint8_t* planted,
                    const float* sigma, float boost, cudaStream_t st) {
    const int n = rows * d;
    const int threads = 256;
    int blocks = (n + threads - 1) / threads;
    if (blocks > 1024) blocks = 1024;
    dim3 grid((unsigned)blocks, (unsigned)(nl * batch));
    fill_rows_kernel<<<grid, threads, 0, st>>>(out, bf16, seed, tag, layer0, batch, steps, use_step_key, rows, d,
                                               idx_offset, planted, sigma, boost);
    return (int)cudaGetLastError();
}

}  // extern "C"
