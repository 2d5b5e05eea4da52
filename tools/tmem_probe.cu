// Microbenchmark (dev tool): can two co-resident CTAs of one SM each hold a
// tcgen05.alloc'd block of tensor memory at the same time, and what does a
// thread-private tcgen05.st / tcgen05.ld round trip (32x32b.x16) cost?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int COLS>
__global__ void __launch_bounds__(256, 2) k_alloc(unsigned long long* out, int spin_us, int clusterish) {
    extern __shared__ unsigned char dyn[];
    __shared__ uint32_t s_tmem;
    const int t = threadIdx.x;
    unsigned long long t0 = gtime();
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"((uint32_t)COLS) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    unsigned long long t1 = gtime();
    const int wp = t >> 5;
    const uint32_t tm = s_tmem + ((uint32_t)((wp & 3) * 32) << 16) + (uint32_t)((wp >> 2) * (COLS / 2));
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = t + i * 0.5f;
    // round trips
    long long c0 = clock64();
    float acc = 0.f;
    for (int it = 0; it < 256; ++it) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
                     ::"r"(tm), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
                       "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n\ttcgen05.wait::ld.sync.aligned;"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                       "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]) : "r"(tm) : "memory");
        acc += v[it & 15];
        v[it & 15] += 1.f;
    }
    long long c1 = clock64();
    // loads only
    for (int it = 0; it < 256; ++it) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n\ttcgen05.wait::ld.sync.aligned;"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                       "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]) : "r"(tm) : "memory");
        acc += v[it & 15];
    }
    long long c2 = clock64();
    while (gtime() - t1 < (unsigned long long)spin_us * 1000ull) {}
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"((uint32_t)COLS) : "memory");
    unsigned long long t2 = gtime();
    if (t == 0) {
        unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long* o = out + 8 * (size_t)blockIdx.x;
        o[0] = smid; o[1] = t0; o[2] = t1; o[3] = t2; o[4] = (unsigned long long)(c1 - c0); o[5] = (unsigned long long)(c2 - c1);
        o[6] = s_tmem; o[7] = (unsigned long long)acc;
    }
}

int main() {
    const int grid = 296;
    unsigned long long* d; cudaMalloc(&d, grid * 8 * sizeof(unsigned long long));
    std::vector<unsigned long long> h(grid * 8);
    for (int cols : {128, 256}) {
        for (size_t smem : {(size_t)1024, (size_t)100 * 1024}) {
            cudaMemset(d, 0, grid * 8 * sizeof(unsigned long long));
            if (cols == 128) {
                cudaFuncSetAttribute(k_alloc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_alloc<128><<<grid, 256, smem>>>(d, 300, 0);
            } else {
                cudaFuncSetAttribute(k_alloc<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k_alloc<256><<<grid, 256, smem>>>(d, 300, 0);
            }
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h.data(), d, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
            unsigned long long tmin = ~0ull;
            for (int b = 0; b < grid; ++b) tmin = std::min(tmin, h[8 * b + 1]);
            // CTAs whose alloc returned within 50 us of the kernel start
            int early = 0; double max_alloc = 0, rt = 0, ld = 0;
            for (int b = 0; b < grid; ++b) {
                const double a_us = (h[8 * b + 2] - tmin) / 1e3;
                if (a_us < 50) ++early;
                max_alloc = std::max(max_alloc, (h[8 * b + 2] - h[8 * b + 1]) / 1e3);
                rt += h[8 * b + 4] / 256.0; ld += h[8 * b + 5] / 256.0;
            }
            printf("cols %d smem %zu: %s; %d / %d CTAs allocated within 50 us of start (2 per SM expected), slowest alloc %.1f us; "
                   "st+ld round trip %.1f clk, ld %.1f clk (8 warps/CTA)\n", cols, smem, cudaGetErrorString(e), early, grid,
                   max_alloc, rt / grid, ld / grid);
            for (int b = 0; b < 4; ++b)
                printf("   cta %d sm %llu start %.1f alloc_done %.1f end %.1f taddr 0x%llx\n", b, h[8 * b], (h[8 * b + 1] - tmin) / 1e3,
                       (h[8 * b + 2] - tmin) / 1e3, (h[8 * b + 3] - tmin) / 1e3, h[8 * b + 6]);
        }
    }
    return 0;
}
