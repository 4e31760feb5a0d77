// DSMEM atomic throughput / latency microbenchmark (profiling aid, not part of the product).
// One cluster of 16 CTAs x 1024 threads; every thread does N atomicSub on random words of
// random CTAs' shared memory (remote), or of its own CTA's (local), or of a global array in
// L2; prints cycles per atomic per SM and the total time.
//
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dsmem_bench tools/dsmem_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int kWords = 32768;   // 128 KB of counters per CTA

__global__ void __launch_bounds__(1024, 1) bench(int mode, int n, int dep, unsigned *glob, unsigned long long *out) {
    extern __shared__ unsigned sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int S = cl.num_blocks();
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) sm[i] = 0xFFFFFFFFu;
    cl.sync();
    unsigned x = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u + 12345u;
    unsigned acc = 0;
    const unsigned long long t0 = gtimer();
    for (int i = 0; i < n; ++i) {
        x = x * 1664525u + 1013904223u;
        const int w = (x >> 8) % kWords;
        const int r = (x >> 3) % S;
        unsigned old;
        if (mode == 0) old = atomicSub(cl.map_shared_rank(sm, r) + w, 1u);        // remote DSMEM
        else if (mode == 1) old = atomicSub(sm + w, 1u);                          // local smem
        else old = atomicSub(glob + (int64_t)r * kWords + w, 1u);                 // global (L2)
        if (dep) x ^= old & 1u;   // dependent chain: the next address needs the result
        acc += old;
    }
    cl.sync();
    const unsigned long long t1 = gtimer();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    if (acc == 0x12345678u) out[1] = acc;
}

int main() {
    unsigned *glob;
    unsigned long long *out;
    cudaMalloc(&glob, 16 * kWords * 4);
    cudaMemset(glob, 0xFF, 16 * kWords * 4);
    cudaMalloc(&out, 16);
    cudaFuncSetAttribute(bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, kWords * 4);
    const char *names[] = {"remote DSMEM", "local smem", "global L2"};
    for (int dep = 0; dep < 2; ++dep)
        for (int mode = 0; mode < 3; ++mode)
            for (int n : {16, 64}) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(16);
                cfg.blockDim = dim3(1024);
                cfg.dynamicSmemBytes = kWords * 4;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 16;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, bench, mode, n, dep, glob, out);   // warm
                cudaLaunchKernelEx(&cfg, bench, mode, n, dep, glob, out);
                cudaError_t e = cudaDeviceSynchronize();
                unsigned long long ns = 0;
                cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
                const double per_sm = (double)n * 1024;   // atomics per SM
                printf("%-13s dep=%d n=%2d: %8.1f us total, %6.2f ns per atomic per SM (%s)\n", names[mode], dep, n,
                       ns / 1e3, ns / per_sm, cudaGetErrorString(e));
            }
    return 0;
}
