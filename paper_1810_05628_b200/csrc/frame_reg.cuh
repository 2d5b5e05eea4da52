// frame_reg.cuh — register-resident line FFT + TMA/mbarrier helpers (complex64).
//
// Same computation as frame_kernel<OP_DISTANCE/OP_INTENSITY> (frame_kernels.cuh;
// reference: objectives.cpp:59-103) but organised around the B200 register file:
//
//   * each thread owns one whole line (column, then row) of the M x M frame:
//     M complex values = 2M fp32 registers;
//   * a line FFT is a fully unrolled two-level Cooley-Tukey (8 x M/8) in
//     registers with compile-time twiddles (folded into FMUL/FFMA immediates):
//     no shared-memory traffic and no bit reversal inside a 1-D transform;
//   * the 2-D transform needs exactly two transposes through shared memory
//     (after the forward column pass, before the inverse column pass), with a
//     (M+2)-element row pitch so 64/128-bit accesses are bank-conflict free;
//   * global traffic is coalesced: the object window and probe are read
//     column-per-thread (lanes walk a row), the contribution is written the
//     same way; the per-pattern amplitudes sqrt(d_j) (the dominant HBM stream)
//     are fetched by TMA bulk copies (cp.async.bulk + mbarrier), one per row,
//     into padded rows of the (then idle) transpose buffer while the row FFT
//     runs, and read back with conflict-free 128-bit loads.
//
// Order: gather(col) -> FFT cols -> transpose -> FFT rows -> spectral op +
// fp64 misfit -> IFFT rows -> transpose -> IFFT cols -> conj(P) epilogue.
#pragma once

#include "fft.cuh"
#include "frame_kernels.cuh"
#include <utility>

// unroll factor as a macro argument (A/B variants of the pass loops)
#define PTG_PRAGMA_(x) _Pragma(#x)
#define PTG_UNROLL_N(n) PTG_PRAGMA_(unroll n)
// the four register-FFT passes of a frame kernel: 1 = one rolled loop (one
// copy of the body), 4 = unrolled (each pass specialised, the next pass's
// loads scheduled across the boundary).  Measured per kernel (round 2):
//   PTG_RMW_PASS_UNROLL (frame_rmw / frame_sc)  config 5   19.66 -> 18.84 ms  => 4
//   PTG_CL_PASS_UNROLL  (frame_cl)              config 3   0.1598 -> 0.1504 ms => 4
//   PTG_TMA_PASS_UNROLL (frame_tma)             config 2   0.0279 -> 0.0280 ms (254 registers) => 1
//   PTG_PIE_PASS_UNROLL (pie_reg)               PIE sweep  5.19 -> 6.48 ms => 1
#ifndef PTG_CL_PASS_UNROLL
#define PTG_CL_PASS_UNROLL 4
#endif
#ifndef PTG_TMA_PASS_UNROLL
#define PTG_TMA_PASS_UNROLL 1
#endif
#ifndef PTG_PIE_PASS_UNROLL
#define PTG_PIE_PASS_UNROLL 1
#endif

namespace ptg {

#ifdef ABL_TIMELINE   // diagnostic build: per-CTA globaltimer stamps (tools/timeline.py)
__device__ unsigned long long g_tl[8192 * 8];
__device__ __forceinline__ void tl_stamp(int k) {
    if (threadIdx.x == 0 && blockIdx.x < 8192) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_tl[blockIdx.x * 8 + k] = t;
        if (k == 0) g_tl[blockIdx.x * 8 + 7] = smid;
    }
}
#define TL(k) tl_stamp(k)
#else
#define TL(k)
#endif

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbarrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// read-only 64-bit load pinned in program order (volatile asm): bounds how
// many loads the compiler hoists while a whole line is live in registers
__device__ __forceinline__ float2 ldg_pinned(const float2* p) {
    float2 v;
    asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

// 1/sqrt(x) as one MUFU op (approximate, flush-to-zero; callers keep x normal)
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// epilogue value sc * conj(P) * IDFT_u(R) from x = conj(IDFT_u(R)):
// conj(P) (sc conj x), scalar FMAs with the signs in the operands
__device__ __forceinline__ float2 epi_contrib(float2 x, float2 P, float sc) {
    const float a = x.x * sc, b = x.y * sc;
    return make_float2(fmaf(P.x, a, -(P.y * b)), fmaf(-P.x, b, -(P.y * a)));
}
__device__ __forceinline__ float2 epi_contrib(float2 x, float sc) { return make_float2(x.x * sc, -x.y * sc); }
// the same with a pre-scaled, pre-conjugated probe Pc = conj(sc * P):
// conj(sc P x) = Pc * conj(x) = cmul((x.x, -x.y), Pc) -- the conj lands on the
// broadcast scalar, so the product is one FMUL2 + one FFMA2
__device__ __forceinline__ float2 epi_contrib_pre(float2 x, float2 Pc) {
    return cmul(make_float2(x.x, -x.y), Pc);
}

// ------------------------------------------------------ register line FFT
// Compile-time twiddles: Taylor series evaluated by the compiler (constexpr),
// argument reduced to [-pi, pi]; exact to ~1e-16, rounded once to fp32.
__host__ __device__ constexpr double ct_sin(double x) {
    double term = x, sum = x;
    for (int k = 1; k < 24; ++k) {
        term *= -x * x / ((2.0 * k) * (2.0 * k + 1.0));
        sum += term;
    }
    return sum;
}
__host__ __device__ constexpr double ct_cos(double x) {
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 24; ++k) {
        term *= -x * x / ((2.0 * k - 1.0) * (2.0 * k));
        sum += term;
    }
    return sum;
}
__host__ __device__ constexpr double ct_angle(int idx, int L) {   // 2 pi idx / L in [-pi, pi]
    const double pi = 3.14159265358979323846264338327950288;
    double th = 2.0 * pi * (double)(idx % L) / (double)L;
    return th > pi ? th - 2.0 * pi : th;
}

template <int N, class F, int... Is>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl<N>(f, std::make_integer_sequence<int, N>{});
}

// v * W_L^E (forward W = e^{-2 pi i / L}), E a template constant: the
// twiddle becomes FMUL/FFMA immediates; quarter turns are free swaps.
template <int L, bool INV, int E>
__device__ __forceinline__ float2 twiddle_mul(float2 v) {
    constexpr int e = E % L;
    if constexpr (e == 0) {
        return v;
    } else if constexpr (4 * e == L) {
        return mul_negi<INV>(v);
    } else if constexpr (2 * e == L) {
        return make_float2(-v.x, -v.y);
    } else if constexpr (4 * e == 3 * L) {
        return mul_negi<!INV>(v);
    } else {
        constexpr float c = (float)ct_cos(ct_angle(e, L));
        constexpr float s = INV ? (float)ct_sin(ct_angle(e, L)) : -(float)ct_sin(ct_angle(e, L));
        return cmul(make_float2(c, s), v);   // FMUL2 + FFMA2 with immediate operands
    }
}

// In-place DFT of L values held in registers (natural order in and out).
// L = A * B with A = 8:  n = B n1 + n2,  k = k1 + A k2.
template <int L, bool INV>
__device__ __forceinline__ void reg_fft(float2* x) {
    if constexpr (L == 1) {
    } else if constexpr (L == 2) {
        dft2<INV>(x[0], x[1]);
    } else if constexpr (L == 4) {
        dft4<INV>(x[0], x[1], x[2], x[3]);
    } else if constexpr (L == 8) {
        dft8<INV>(x);
    } else if constexpr (L == 16) {
        dft16<INV>(x);
    } else {
        constexpr int A = 8, B = L / 8;
        float2 y[L];
        static_for<B>([&](auto n2c) {
            constexpr int n2 = decltype(n2c)::value;
            float2 t[A];
#pragma unroll
            for (int n1 = 0; n1 < A; ++n1) t[n1] = x[B * n1 + n2];
            dft8<INV>(t);
            static_for<A>([&](auto k1c) {
                constexpr int k1 = decltype(k1c)::value;
                y[k1 * B + n2] = twiddle_mul<L, INV, n2 * k1>(t[k1]);
            });
        });
#pragma unroll
        for (int k1 = 0; k1 < A; ++k1) {
            float2 t[B];
#pragma unroll
            for (int n2 = 0; n2 < B; ++n2) t[n2] = y[k1 * B + n2];
            reg_fft<B, INV>(t);
#pragma unroll
            for (int k2 = 0; k2 < B; ++k2) x[k1 + A * k2] = t[k2];
        }
    }
}

}  // namespace ptg
