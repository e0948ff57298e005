// Latency floor of a chain of small dependent kernels on B200 (graph replay, PDL), and the
// cost of the split-K merge mechanisms a batch-1 decode layer can use:
//   empty    : griddepcontrol.wait + launch_dependents, nothing else
//   qout     : + a dependent global load (the layer's q) and a 2 KiB output per group
//   last     : each CTA stores a 2 KiB partial, one acq_rel ticket per group; the last
//              arriving CTA loads all partials of its group and writes the output
//   spin     : every CTA draws a ticket, spins until the group is complete, merges its slice
//   cpush    : thread-block cluster = group; st.async of each rank's slice into the owner's
//              shared memory (mbarrier complete_tx), owner merges and writes
//   cbar     : cluster; plain DSMEM stores + barrier.cluster release/acquire, owner merges
// Usage: latency_floor [groups=8] [group_size=18] [smem_kb=100] [threads=256]
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess) {                                                              \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);   \
            exit(1);                                                                          \
        }                                                                                     \
    } while (0)

constexpr int kPartFloats = 512;  // 2 KiB partial per CTA (4 heads x 128 floats)

struct Args {
    const float* q;
    float* part;                 // [groups][gsize][kPartFloats]
    float* out;                  // [groups][kPartFloats]
    unsigned long long* cnt;     // [groups] tickets (stride 64 B)
    int gsize;
};

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cl_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t x; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(x) : "r"(a), "r"(r)); return x;
}

template <int V>
__global__ void __launch_bounds__(256) chain_kernel(Args a) {
    extern __shared__ __align__(16) float sm[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int grp = blockIdx.x / a.gsize, rk = blockIdx.x % a.gsize;
    __shared__ uint64_t bar;
    __shared__ int last;
    if (V == 4) {
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
            // expect: every rank sends its slice of the owner: kPartFloats / gsize floats, 4 B each
            const int per = (kPartFloats + a.gsize - 1) / a.gsize;
            const int lo = rk * per, n = max(0, min(kPartFloats, lo + per) - lo);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                         "r"(n * 4 * a.gsize));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    }
    pdl_wait();
    pdl_trigger();
    if (V == 0) {
        if (tid == 0 && blockIdx.x == 0) a.out[0] = 1.f;
        return;
    }
    // the layer's input: one dependent load per thread
    const float qv = a.q[(blockIdx.x * nt + tid) & 8191];
    // this CTA's partial: kPartFloats values
    float* my = a.part + ((size_t)grp * a.gsize + rk) * kPartFloats;
    if (V == 1) {
        if (rk == 0)
            for (int i = tid; i < kPartFloats; i += nt) a.out[grp * kPartFloats + i] = qv + i;
        return;
    }
    if (V == 2 || V == 3) {
        for (int i = tid; i < kPartFloats; i += nt) my[i] = qv * (i + 1);
        __syncthreads();
        unsigned long long* c = a.cnt + grp * 8;
        if (tid == 0) {
            unsigned long long old;
            asm volatile("atom.add.acq_rel.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(c) : "memory");
            const unsigned long long target = old - old % a.gsize + a.gsize;
            last = (old + 1 == target);
            if (V == 3 && !last) {
                unsigned long long v;
                do {
                    asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(c) : "memory");
                } while (v < target);
            }
        }
        __syncthreads();
        const float* base = a.part + (size_t)grp * a.gsize * kPartFloats;
        if (V == 2) {
            if (!last) return;
            for (int i = tid; i < kPartFloats; i += nt) {
                float s = 0.f;
                for (int r = 0; r < a.gsize; ++r) s += __ldcg(base + (size_t)r * kPartFloats + i);
                a.out[grp * kPartFloats + i] = s;
            }
        } else {
            const int per = (kPartFloats + a.gsize - 1) / a.gsize;
            const int lo = rk * per, n = max(0, min(kPartFloats, lo + per) - lo);
            for (int i = tid; i < n * a.gsize; i += nt) sm[i] = __ldcg(base + (size_t)(i / n) * kPartFloats + lo + i % n);
            __syncthreads();
            for (int i = tid; i < n; i += nt) {
                float s = 0.f;
                for (int r = 0; r < a.gsize; ++r) s += sm[r * n + i];
                a.out[grp * kPartFloats + lo + i] = s;
            }
        }
        return;
    }
    if (V == 6) {
        // LL protocol: {value, flag} 8-byte stores (single-copy atomic), no fences or atomics;
        // the owner of slice r spins on the flags of its slice from every CTA, then clears them
        // (the next launch writes only after this one completed: PDL wait)
        uint2* myll = reinterpret_cast<uint2*>(a.part) + ((size_t)grp * a.gsize + rk) * kPartFloats;
        for (int i = tid; i < kPartFloats; i += nt) {
            const uint2 w = make_uint2(__float_as_uint(qv * (i + 1)), 1u);
            asm volatile("st.relaxed.gpu.global.v2.u32 [%0], {%1, %2};" ::"l"(myll + i), "r"(w.x), "r"(w.y) : "memory");
        }
        const int per = (kPartFloats + a.gsize - 1) / a.gsize;
        const int lo = rk * per, n = max(0, min(kPartFloats, lo + per) - lo);
        uint2* base = reinterpret_cast<uint2*>(a.part) + (size_t)grp * a.gsize * kPartFloats;
        for (int i = tid; i < n * a.gsize; i += nt) {
            uint2* src = base + (size_t)(i / n) * kPartFloats + lo + i % n;
            uint2 w;
            do {
                asm volatile("ld.relaxed.gpu.global.v2.u32 {%0, %1}, [%2];" : "=r"(w.x), "=r"(w.y) : "l"(src) : "memory");
            } while (w.y != 1u);
            sm[i] = __uint_as_float(w.x);
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(reinterpret_cast<uint32_t*>(src) + 1), "r"(0u) : "memory");
        }
        __syncthreads();
        for (int i = tid; i < n; i += nt) {
            float s = 0.f;
            for (int r = 0; r < a.gsize; ++r) s += sm[r * n + i];
            a.out[grp * kPartFloats + lo + i] = s;
        }
        return;
    }
    // cluster variants: owner r holds slice r of the output; stage[rank][n] floats
    const int per = (kPartFloats + a.gsize - 1) / a.gsize;
    if (V == 4) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every peer's barrier is live
    const uint32_t st_u = smem_u32(sm);
    for (int i = tid; i < kPartFloats; i += nt) {
        const int r = i / per, k = i - r * per;
        const float v = qv * (i + 1);
        const uint32_t dst = mapa(st_u + (uint32_t)(rk * per + k) * 4u, (uint32_t)r);
        if (V == 4) {
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                         ::"r"(dst), "r"(__float_as_uint(v)), "r"(mapa(smem_u32(&bar), (uint32_t)r)) : "memory");
        } else {
            asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst), "f"(v) : "memory");
        }
    }
    const int lo = rk * per, n = max(0, min(kPartFloats, lo + per) - lo);
    if (V == 4) {
        asm volatile(
            "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n}"
            ::"r"(smem_u32(&bar)) : "memory");
    } else {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    for (int i = tid; i < n; i += nt) {
        float s = 0.f;
        for (int r = 0; r < a.gsize; ++r) s += sm[r * per + i];
        a.out[grp * kPartFloats + lo + i] = s;
    }
    if (V == 5) {  // nobody may exit while a peer could still read its smem: not needed (owner reads own)
    }
}

template <int V>
float run(int groups, int gsize, int smem, int threads, bool pdl, bool cluster, const Args& a, cudaStream_t st,
          int chain) {
    auto k = chain_kernel<V>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (cluster) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(groups * gsize);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = gsize; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < chain; ++i) CK(cudaLaunchKernelEx(&cfg, k, a));
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(e0, st));
    const int reps = 10;
    for (int r = 0; r < reps; ++r) CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(g));
    return ms * 1e3f / (reps * chain);
}

int main(int argc, char** argv) {
    const int groups = argc > 1 ? atoi(argv[1]) : 8;
    const int gsize = argc > 2 ? atoi(argv[2]) : 18;
    const int smem = (argc > 3 ? atoi(argv[3]) : 100) * 1024;
    const int threads = argc > 4 ? atoi(argv[4]) : 256;
    Args a = {};
    float *q, *part, *out;
    unsigned long long* cnt;
    CK(cudaMalloc(&q, 8192 * 4));
    CK(cudaMalloc(&part, (size_t)groups * gsize * kPartFloats * 8));
    CK(cudaMemset(part, 0, (size_t)groups * gsize * kPartFloats * 8));
    CK(cudaMalloc(&out, (size_t)groups * kPartFloats * 4));
    CK(cudaMalloc(&cnt, groups * 64));
    CK(cudaMemset(q, 0, 8192 * 4));
    CK(cudaMemset(cnt, 0, groups * 64));
    a.q = q; a.part = part; a.out = out; a.cnt = cnt; a.gsize = gsize;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const int chain = 100;
    printf("groups %d x %d CTAs, %d threads, %d KiB smem: us per kernel in a graph of %d\n", groups, gsize, threads,
           smem / 1024, chain);
    for (int pdl = 1; pdl >= 0; --pdl) {
        printf(" pdl=%d  empty %6.2f  qout %6.2f  last %6.2f  spin %6.2f  ll %6.2f", pdl,
               run<0>(groups, gsize, smem, threads, pdl, false, a, st, chain),
               run<1>(groups, gsize, smem, threads, pdl, false, a, st, chain),
               run<2>(groups, gsize, smem, threads, pdl, false, a, st, chain),
               run<3>(groups, gsize, smem, threads, pdl, false, a, st, chain),
               run<6>(groups, gsize, smem, threads, pdl, false, a, st, chain));
        if (gsize <= 16)
            printf("  cpush %6.2f  cbar %6.2f  cempty %6.2f",
                   run<4>(groups, gsize, smem, threads, pdl, true, a, st, chain),
                   run<5>(groups, gsize, smem, threads, pdl, true, a, st, chain),
                   run<0>(groups, gsize, smem, threads, pdl, true, a, st, chain));
        printf("\n");
    }
    return 0;
}
