// Grid-barrier and dependent-round-trip microbenchmark for the persistent kernels
// (profiling aid, not part of the product).  One CTA of 1024 threads per SM, R rounds of
//   [optional L2 work: one dependent __ldcg chain of `chain` links per thread] + barrier
// timed with %globaltimer by CTA 0; prints ns per round for each barrier variant.
//
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/bb tools/barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t ld_acq(const uint32_t *a) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_rlx(const uint32_t *a) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel_add(uint32_t *a, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel(uint32_t *a, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

struct Args {
    uint32_t *ctr;     // [64] counters (spaced)
    uint32_t *flags;   // [G * 32] one line per CTA
    const int32_t *chain;  // pointer-chasing array
    int32_t chain_n;
    int links;
    int rounds;
    int variant;
    unsigned long long *out;
    int32_t *sink;
};

// variant 0: cg grid.sync
// variant 1: counter barrier, thread 0: fence + atomicAdd; poll volatile (cg-like, monotonic target)
// variant 2: counter barrier, red.release.gpu + ld.acquire poll
// variant 3: flag array: st.release own flag; warp 0 polls all flags (ld.relaxed) + fence
// variant 4: hierarchical: cluster barrier (8), cluster rank 0 arrives on counter, polls, cluster barrier
// variant 5: no barrier (__syncthreads only) -- floor of the work + loop
__global__ void __launch_bounds__(1024, 1) bench(Args a) {
    cg::grid_group grid = cg::this_grid();
    const int tid = threadIdx.x;
    const int G = gridDim.x;
    uint32_t epoch = 0;
    int32_t x = (blockIdx.x * 1024 + tid) % a.chain_n;
    int32_t acc = 0;
    unsigned long long t0 = 0;
    for (int r = 0; r < a.rounds + 8; ++r) {
        if (r == 8 && blockIdx.x == 0 && tid == 0) t0 = gtimer();
        for (int l = 0; l < a.links; ++l) x = __ldcg(a.chain + x);
        acc += x;
        ++epoch;
        switch (a.variant) {
            case 0: grid.sync(); break;
            case 1:
                __syncthreads();
                if (tid == 0) {
                    __threadfence();
                    atomicAdd(a.ctr, 1u);
                    while (*(volatile uint32_t *)a.ctr < epoch * G) {}
                    __threadfence();
                }
                __syncthreads();
                break;
            case 2:
                __syncthreads();
                if (tid == 0) {
                    red_rel_add(a.ctr, 1u);
                    while (ld_acq(a.ctr) < epoch * G) {}
                }
                __syncthreads();
                break;
            case 3:
                __syncthreads();
                if (tid < 32) {
                    if (tid == 0) st_rel(a.flags + blockIdx.x * 32, epoch);
                    for (int b = tid; b < G; b += 32)
                        while (ld_rlx(a.flags + b * 32) < epoch) {}
                    __syncwarp();
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
                __syncthreads();
                break;
            case 4: {
                cg::cluster_group cl = cg::this_cluster();
                cl.sync();
                if (cl.block_rank() == 0 && tid == 0) {
                    const uint32_t nc = G / cl.num_blocks();
                    red_rel_add(a.ctr, 1u);
                    while (ld_acq(a.ctr) < epoch * nc) {}
                }
                cl.sync();
                break;
            }
            case 5: __syncthreads(); break;
            case 6:
                __syncthreads();
                if (tid == 0) {
                    red_rel_add(a.ctr, 1u);
                    while (ld_acq(a.ctr) < epoch * G) __nanosleep(20);
                }
                __syncthreads();
                break;
            case 7:
                __syncthreads();
                if (tid == 0) {
                    uint32_t old;
                    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.ctr) : "memory");
                    if (old == epoch * G - 1) st_rel(a.ctr + 32, epoch);
                    else while (ld_acq(a.ctr + 32) < epoch) {}
                }
                __syncthreads();
                break;
            case 8:
                __syncthreads();
                if (tid == 0) {
                    red_rel_add(a.ctr, 1u);
                    while (ld_rlx(a.ctr) < epoch * G) {}
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
                __syncthreads();
                break;
            case 10:   // cg grid.sync + every CTA's thread 0 reads one hot counter line after it
            case 11:   // ... after each CTA's warps added to that line during the round
                if (a.variant == 11 && (tid & 31) == 0) atomicAdd(a.ctr + 256, 1u);
                grid.sync();
                {
                    __shared__ uint32_t sv;
                    if (tid == 0) sv = __ldcg(a.ctr + 256) + __ldcg(a.ctr + 257) + __ldcg(a.ctr + 258);
                    __syncthreads();
                    acc += sv;
                }
                break;
            case 9:   // two-level: 4 sub-counters (by blockIdx % 4), last arriver of each adds to top
                __syncthreads();
                if (tid == 0) {
                    uint32_t old;
                    const int sc = blockIdx.x & 3;
                    const uint32_t nsub = (G - sc + 3) / 4;
                    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.ctr + 64 + 32 * sc) : "memory");
                    if (old == epoch * nsub - 1) red_rel_add(a.ctr + 32, 1u);
                    while (ld_acq(a.ctr + 32) < epoch * 4) {}
                }
                __syncthreads();
                break;
        }
    }
    if (blockIdx.x == 0 && tid == 0) *a.out = gtimer() - t0;
    if (acc == 0x7fffffff) *a.sink = acc;
}

int main(int argc, char **argv) {
    int rounds = 2000;
    int G = 0;
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    G = prop.multiProcessorCount;
    uint32_t *ctr, *flags;
    int32_t *chain, *sink;
    unsigned long long *out;
    const int32_t chain_n = 1 << 20;
    cudaMalloc(&ctr, 512 * 4);
    cudaMalloc(&flags, G * 32 * 4);
    cudaMalloc(&chain, chain_n * 4);
    cudaMalloc(&sink, 4);
    cudaMalloc(&out, 8);
    std::vector<int32_t> h(chain_n);
    // random permutation cycle: a dependent chain that misses L1 (ldcg) but hits L2 (4 MB)
    for (int i = 0; i < chain_n; ++i) h[i] = i;
    uint64_t s = 88172645463325252ull;
    for (int i = chain_n - 1; i > 0; --i) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        int j = (int)(s % (uint64_t)(i + 1));
        std::swap(h[i], h[j]);
    }
    std::vector<int32_t> nxt(chain_n);
    for (int i = 0; i < chain_n; ++i) nxt[h[i]] = h[(i + 1) % chain_n];
    cudaMemcpy(chain, nxt.data(), chain_n * 4, cudaMemcpyHostToDevice);
    const char *names[] = {"cg grid.sync", "counter fence+atomicAdd", "counter red.release/ld.acquire",
                           "flag array", "cluster8 + counter", "syncthreads only", "counter + nanosleep poll", "last arriver flag", "counter relaxed poll + fence", "two-level 4 counters", "grid.sync + hot-line read", "grid.sync + atomics + hot-line read"};
    for (int links : {0, 1, 3}) {
        for (int v = 0; v < 12; ++v) {
            cudaMemset(ctr, 0, 512 * 4);
            cudaMemset(flags, 0, G * 32 * 4);
            Args a{ctr, flags, chain, chain_n, links, rounds, v, out, sink};
            cudaError_t e;
            if (v == 4) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(G - G % 8);
                cfg.blockDim = dim3(1024);
                cudaLaunchAttribute at[2];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 8;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int ncl = 0;
                cudaOccupancyMaxActiveClusters(&ncl, bench, &cfg);
                cfg.gridDim = dim3(ncl * 8);
                e = cudaLaunchKernelEx(&cfg, bench, a);
                if (links == 0) printf("(cluster variant: %d clusters of 8)\n", ncl);
            } else {
                void *args[] = {&a};
                e = cudaLaunchCooperativeKernel((void *)bench, dim3(G), dim3(1024), args, 0, 0);
            }
            cudaError_t e2 = cudaDeviceSynchronize();
            unsigned long long ns = 0;
            cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
            printf("links %d  %-32s %8.1f ns/round  (%s %s)\n", links, names[v], (double)ns / rounds,
                   cudaGetErrorString(e), cudaGetErrorString(e2));
        }
    }
    // single-thread dependent L2 latency
    return 0;
}
