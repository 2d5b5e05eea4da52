// Microbenchmark (dev tool): issue throughput of FP32 scalar vs packed (f32x2)
// add / mul / fma on sm_100a, full occupancy, 8 independent chains per thread.
// Prints ops per SM per clock for each form.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048
__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
template <int KIND>
__global__ void k(float* out, float s0, float s1) {
    float a[8]; unsigned long long p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i; p[i] = pk(a[i], a[i] + 1.f); }
    const unsigned long long m = pk(s0, s1), c = pk(s1, s0);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(s0), "f"(s1));        // FFMA 3-reg
            if (KIND == 1) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(s0));                     // FADD
            if (KIND == 2) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(m), "l"(c));        // FFMA2
            if (KIND == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(m));                   // FADD2
            if (KIND == 4) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(m));                   // FMUL2
            if (KIND == 5) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3C000000;" : "+f"(a[i]));          // FFMA imm
            if (KIND == 6) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(s0));                     // FMUL
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { s += a[i]; float lo, hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[i])); s += lo + hi; }
    if (s == 1234.5f) out[0] = s;
}
template <int KIND>
void run(const char* name, int lanes_per_op) {
    float* out; cudaMalloc(&out, 4);
    int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 256;
    k<KIND><<<blocks, threads>>>(out, 1.0001f, 0.999f);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0); k<KIND><<<blocks, threads>>>(out, 1.0001f, 0.999f); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double instr = (double)blocks * threads / 32 * ITERS * 8;           // warp instructions
    double cycles = best * 1e-3 * 1965e6;                               // at max clock
    double per_smsp = instr / (148 * 4) / cycles;                        // warp-instr per SMSP per clock
    printf("%-10s %8.3f ms  %.3f warp-instr/SMSP/clk  (rt %.2f)  %.1f lane-ops/SM/clk\n", name, best, per_smsp,
           1.0 / per_smsp, per_smsp * 4 * 32 * lanes_per_op);
}
int main() {
    run<0>("FFMA", 1); run<5>("FFMA-imm", 1); run<1>("FADD", 1); run<6>("FMUL", 1);
    run<2>("FFMA2", 2); run<3>("FADD2", 2); run<4>("FMUL2", 2);
    return 0;
}
