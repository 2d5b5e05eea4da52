// Microbenchmark: streaming read bandwidth of an L2-resident vs HBM-resident
// buffer (sizes 8..128 MiB), float4 loads, grid = 148 x k.  Dev tool only.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const float4* __restrict__ a, size_t n4, float4* out) {
    float4 s = make_float4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = __ldcg(a + i);
        s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    if (s.x == 12345.f) out[0] = s;
}
__global__ void wr(float4* a, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        a[i] = make_float4(1, 2, 3, 4);
}

int main() {
    float4 *a, *flush, *out;
    size_t maxb = 128u << 20, fb = 512u << 20;
    cudaMalloc(&a, maxb);
    cudaMalloc(&flush, fb);
    cudaMalloc(&out, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (size_t mb : {8, 16, 32, 64, 96}) {
        size_t n4 = (mb << 20) / 16;
        for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
            float best_l2 = 1e9, best_dram = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                wr<<<148 * 8, 256>>>(a, n4);            // resident in L2 (dirty)
                rd<<<148 * 8, 256>>>(a, n4, out);       // and clean
                cudaEventRecord(e0);
                rd<<<blocks, 256>>>(a, n4, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best_l2) best_l2 = ms;
                wr<<<148 * 8, 256>>>(flush, fb / 16);   // evict
                cudaEventRecord(e0);
                rd<<<blocks, 256>>>(a, n4, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best_dram) best_dram = ms;
            }
            printf("%3zu MiB blocks %5d  L2-warm %7.2f us %6.0f GB/s   cold %7.2f us %6.0f GB/s\n", mb, blocks,
                   best_l2 * 1e3, (mb << 20) / (best_l2 * 1e-3) / 1e9, best_dram * 1e3,
                   (mb << 20) / (best_dram * 1e-3) / 1e9);
        }
    }
    return 0;
}
