// bw_probe.cu — the pure-read roofline kernel (SURVEY §8(d) "K10"): streams a device buffer
// once with 16-byte loads and reduces it to one float, so the benchmark can report the HBM
// read bandwidth measured in the same run beside the decode kernels' attended-KV GB/s.  Not
// part of the method; the decode kernels never call it.
#include "internal.h"

namespace delta {
namespace {

__global__ void __launch_bounds__(512) read_probe_kernel(const uint4* __restrict__ buf, size_t n16, float* sink) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    constexpr int kU = 8;  // independent 16-byte loads in flight per thread
    for (; i + (kU - 1) * stride < n16; i += kU * stride) {
        uint4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = __ldcs(buf + i + u * stride);
#pragma unroll
        for (int u = 0; u < kU; ++u) acc += __uint_as_float(v[u].x ^ v[u].y ^ v[u].z ^ v[u].w);
    }
    for (; i < n16; i += stride) {
        const uint4 v = __ldcs(buf + i);
        acc += __uint_as_float(v.x ^ v.y ^ v.z ^ v.w);
    }
    // keep the loads live: one store per CTA, only if the (never true in practice) sum is tiny
    if (acc == 1.2345e-30f) sink[0] = acc;
}

}  // namespace

cudaError_t launch_read_probe(const void* buf, size_t bytes, float* sink, int sms, cudaStream_t st) {
    const size_t n16 = bytes / 16;
    read_probe_kernel<<<sms * 4, 512, 0, st>>>(reinterpret_cast<const uint4*>(buf), n16, sink);
    return cudaGetLastError();
}

}  // namespace delta
