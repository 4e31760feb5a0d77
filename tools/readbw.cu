// Read-stream ceiling on this GPU for the θ-pass load pattern (profiling aid, not product):
// persistent grid, int4 loads, U in flight per thread, trivial consume.  Prints GB/s for
// several (threads, U, load flavour) at 200 MB and 600 MB.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int4 ld_nc(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ int4 ld_lu(const int4 *p) {
    int4 r;
    asm volatile("ld.global.lu.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
// 256-bit load (sm_100: ld.global.v8.b32) of two consecutive int4; returns their XOR
__device__ __forceinline__ int4 ld_ef(const int4 *p) {
    int4 r, s;
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w), "=r"(s.x), "=r"(s.y), "=r"(s.z), "=r"(s.w) : "l"(p));
    r.x ^= s.x; r.y ^= s.y; r.z ^= s.z; r.w ^= s.w;
    return r;
}
__device__ __forceinline__ int4 ld_256(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int U, int F>
__global__ void rd(const int4 *a, long long n, int *out) {
    const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long G = (long long)gridDim.x * blockDim.x;
    int acc = 0;
    const long long lim0 = F == 2 ? n / 2 : n;
    for (long long i0 = g; i0 < lim0; i0 += G * U) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long i = i0 + u * G;
            const long long lim = F == 2 ? n / 2 : n;
            if (i < lim) v[u] = F == 0 ? ld_nc(a + i) : F == 1 ? ld_lu(a + i) : F == 2 ? ld_ef(a + 2 * i) : ld_256(a + i);
            else v[u] = make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678) out[0] = acc;
}

template <int U, int F>
float run(const int4 *a, long long n, int *out, int blocks, int threads, void *flush, size_t fb) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 8; ++it) {
        cudaMemsetAsync(flush, it, fb);
        cudaEventRecord(e0);
        rd<U, F><<<blocks, threads>>>(a, n, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it >= 2 && ms < best) best = ms;
    }
    return best;
}

int main() {
    const size_t maxb = 600ull << 20;
    int4 *a;
    int *out;
    void *flush;
    const size_t fb = 256ull << 20;
    cudaMalloc(&a, maxb);
    cudaMalloc(&out, 4);
    cudaMalloc(&flush, fb);
    cudaMemset(a, 1, maxb);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char *fl[] = {"nc.no_alloc", "lu", "nc.v8 (256-bit)", "nc.L2::256B"};
    for (size_t mb : {200, 600}) {
        const long long n = (long long)(mb << 20) / 16;
        for (int threads : {512, 1024}) {
            const int blocks = sms * (2048 / threads);
            for (int F = 0; F < 4; ++F) {
                float t4, t8, t16;
#define RUNF(UU, FF) run<UU, FF>(a, n, out, blocks, threads, flush, fb)
                switch (F) {
                    case 0: t4 = RUNF(4, 0); t8 = RUNF(8, 0); t16 = RUNF(16, 0); break;
                    case 1: t4 = RUNF(4, 1); t8 = RUNF(8, 1); t16 = RUNF(16, 1); break;
                    case 2: t4 = RUNF(4, 2); t8 = RUNF(8, 2); t16 = RUNF(16, 2); break;
                    default: t4 = RUNF(4, 3); t8 = RUNF(8, 3); t16 = RUNF(16, 3); break;
                }
                const double B = (double)n * 16;
                printf("%zu MB  %4d thr x %d blk  %-16s  U4 %6.0f  U8 %6.0f  U16 %6.0f GB/s\n", mb, threads,
                       blocks, fl[F], B / t4 / 1e6, B / t8 / 1e6, B / t16 / 1e6);
            }
        }
        // one CTA of 1024 per SM (the θ-pass configuration)
        for (int F = 0; F < 1; ++F) {
            const double B = (double)n * 16;
            float t8 = run<8, 0>(a, n, out, sms, 1024, flush, fb);
            float t16 = run<16, 0>(a, n, out, sms, 1024, flush, fb);
            printf("%zu MB  1024 thr x %d blk (1/SM)  nc.no_alloc  U8 %6.0f  U16 %6.0f GB/s\n", mb, sms, B / t8 / 1e6,
                   B / t16 / 1e6);
        }
    }
    return 0;
}
