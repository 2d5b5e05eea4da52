// common.cuh — shared device/host helpers for libptg (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "../../include/ptg.h"

namespace ptg {

// Programmatic dependent launch: wait until the preceding grid in the stream
// has completed and flushed (no-op when launched without the PDL attribute),
// then let the next grid start launching.
__device__ __forceinline__ void pdl_wait_and_trigger() {
#if defined(__CUDA_ARCH__)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// Status-carrying exception used inside the library; the C-ABI layer
// (capi.cu) converts it to an int status + ptg_last_error() string.
struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Status(code, msg); }

#define PTG_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            ::ptg::raise(PTG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define PTG_CHECK_LAUNCH() PTG_CUDA(cudaGetLastError())

// Complex scalar vector types: T = float (complex64) or double (complex128).
template <typename T> struct V2;
template <> struct V2<float> { using type = float2; };
template <> struct V2<double> { using type = double2; };
template <typename T> using cplx = typename V2<T>::type;

template <typename T>
__host__ __device__ __forceinline__ cplx<T> mk(T re, T im) {
    cplx<T> r;
    r.x = re;
    r.y = im;
    return r;
}
template <typename C>
__host__ __device__ __forceinline__ C cadd(C a, C b) { C r; r.x = a.x + b.x; r.y = a.y + b.y; return r; }
template <typename C>
__host__ __device__ __forceinline__ C csub(C a, C b) { C r; r.x = a.x - b.x; r.y = a.y - b.y; return r; }
template <typename C>
__host__ __device__ __forceinline__ C cmul(C a, C b) {
    C r;
    r.x = a.x * b.x - a.y * b.y;
    r.y = a.x * b.y + a.y * b.x;
    return r;
}
// conj(a) * b
template <typename C>
__host__ __device__ __forceinline__ C cmulc(C a, C b) {
    C r;
    r.x = a.x * b.x + a.y * b.y;
    r.y = a.x * b.y - a.y * b.x;
    return r;
}
template <typename C, typename S>
__host__ __device__ __forceinline__ C cscale(C a, S s) { C r; r.x = a.x * s; r.y = a.y * s; return r; }

// complex64 on sm_100: packed FP32 pairs (FADD2 / FMUL2 / FFMA2).  ptxas folds
// the swaps, negations and scalar broadcasts of complex arithmetic into the
// packed operand selectors, halving the FP32 instruction count of the FFTs.
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
__device__ __forceinline__ unsigned long long f2u(float2 a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 u2f(unsigned long long r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(make_float2(s, s))));
    return u2f(r);
}
// a * b = (ax bx, ax by) + (ay (-by), ay bx)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    unsigned long long t, r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2u(make_float2(a.x, a.x))), "l"(f2u(b)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(make_float2(a.y, a.y))),
        "l"(f2u(make_float2(-b.y, b.x))), "l"(t));
    return u2f(r);
}
// conj(a) * b = (ax bx, ax by) + (ay by, -ay bx)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    unsigned long long t, r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f2u(make_float2(a.x, a.x))), "l"(f2u(b)));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(make_float2(a.y, a.y))),
        "l"(f2u(make_float2(b.y, -b.x))), "l"(t));
    return u2f(r);
}
#endif

// Per-position contribution ("stash") rows have pitch >= w + 2, rounded up to
// even: the window row is stored at offset (col0 & 1) with zeros elsewhere, so
// every even-aligned pixel pair of the object maps to one aligned 16-byte
// (complex64) vector of the stash (plan.cu k_overlap_gather).
__host__ __device__ constexpr int stash_pitch(int w) { return (w + 3) & ~1; }

inline int ilog2(int n) { int l = 0; while ((1 << l) < n) ++l; return l; }
inline bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

}  // namespace ptg
