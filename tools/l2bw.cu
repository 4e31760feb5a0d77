// L2 read bandwidth on this GPU (the roofline denominator of the L2-resident stable pass):
// a persistent 148 x 1024 grid streams a buffer that fits the 126 MB L2 (after one warm
// pass) with int4 loads, U in flight per thread, XOR-consumed.  Prints GB/s per size.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2bw tools/l2bw.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(1024, 1) rd(const int4 *a, long long n4, int rounds, int *out) {
    int x = 0;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x, G = (long long)gridDim.x * blockDim.x;
    for (int r = 0; r < rounds; ++r)
        for (long long i = g; i < n4; i += G * U) {
            int4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = i + u * G < n4 ? __ldcg(a + i + u * G) : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < U; ++u) x ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        }
    if (x == 0x12345678) out[0] = x;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int *out;
    cudaMalloc(&out, 4);
    const size_t sizes[] = {8u << 20, 32u << 20, 64u << 20, 96u << 20};
    for (size_t bytes : sizes) {
        int4 *a;
        cudaMalloc(&a, bytes);
        cudaMemset(a, 1, bytes);
        const long long n4 = (long long)(bytes / 16);
        const int rounds = (int)(4096ull * 1024 * 1024 / bytes);
        float best = 1e30f;
        for (int t = 0; t < 5; ++t) {
            rd<4><<<sms, 1024>>>(a, n4, 1, out);   // warm the L2
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            rd<4><<<sms, 1024>>>(a, n4, rounds, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("{\"bytes\": %zu, \"rounds\": %d, \"ms\": %.4f, \"gbs\": %.1f}\n", bytes, rounds, best,
               (double)bytes * rounds / (best * 1e-3) / 1e9);
        cudaFree(a);
    }
    return 0;
}
