// frame_tma.cuh — the hot kernel: fused objective/gradient frame kernel for
// complex64 frames M in {16, 32, 64} with w == M (patch mode).
//
// Same computation as frame_kernel<OP_DISTANCE/OP_INTENSITY> (frame_kernels.cuh,
// reference objectives.cpp:59-103), organised for the B200:
//
//   * data movement by TMA: the M x M object window psi-source is ONE 2-D
//     tensor load (cp.async.bulk.tensor.2d) into shared memory, the pattern's
//     amplitudes sqrt(d_j) are 3-D tensor tiles with 128B (64B) swizzle so the
//     row-per-thread reads are bank-conflict free; both complete on mbarriers
//     and the amplitude load overlaps the row FFT;
//   * each thread owns one whole line (column, then row) in registers; a line
//     FFT is a fully unrolled 8 x (M/8) Cooley-Tukey with compile-time twiddle
//     immediates (frame_reg.cuh);
//   * all four line passes (fwd cols, fwd rows, inv rows, inv cols) run the
//     SAME forward-FFT code in a rolled loop: the inverse is taken as
//     IDFT(X) = conj(DFT(conj X)), and the two conjugations between the inverse
//     passes cancel, so the code footprint stays inside the instruction cache;
//   * two transposes through shared memory with an (M+2) pitch (conflict free);
//   * the probe products (P o x before, conj(P) o r after) run as cooperative
//     shared-memory passes when no line is live in registers, so the probe
//     loads (L2-resident) are deep in flight without register pressure.
//
// Timing-only build variants (tools/build_variant.sh, never the shipped
// library): ABL_NOPREF / ABL_NOSPEC / ABL_NOTRANS / ABL_NOSTORE remove one
// phase each (results invalid), ABL_TIMELINE records per-CTA %globaltimer
// stamps (tools/timeline.py).  profiles/r01_frame_analysis.txt has the numbers.
#pragma once

#include <cuda.h>

#include "frame_reg.cuh"

namespace ptg {

template <int M>
constexpr int tma_frames_per_cta() { return M == 64 ? 1 : M == 32 ? 4 : 8; }

// bytes of one frame's shared region: transpose buffer (pitch M+2), z tile
// (dense M x 2M floats) and amplitude tiles all alias; rounded to 1 KiB so
// swizzled TMA tiles keep their 1024-B alignment.
template <int M>
__host__ __device__ constexpr size_t tma_frame_bytes() {
    const size_t a = sizeof(float2) * (size_t)M * (M + 2);
    return (a + 1023) / 1024 * 1024;
}
template <int M>
__host__ __device__ constexpr size_t tma_smem_bytes() {
    return tma_frame_bytes<M>() * tma_frames_per_cta<M>() + 1024;   // + alignment slack
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}


template <int M, int OP, bool PROBE>
__global__ void __launch_bounds__(M * tma_frames_per_cta<M>(), M == 64 ? 6 : 3)
    frame_tma_kernel(FrameArgs<float> a, int count, const __grid_constant__ CUtensorMap tm_z,
                     const __grid_constant__ CUtensorMap tm_amp, const __grid_constant__ CUtensorMap tm_p) {
    constexpr int FPC = tma_frames_per_cta<M>();
    constexpr int S = M + 2;                    // float2 pitch of the transpose buffer
    constexpr int WPF = (M + 31) / 32;
    constexpr int AT = M < 32 ? M : 32;         // amplitude tile width (floats) = swizzle span
    constexpr int NAT = M / AT;                 // amplitude tiles per frame
    constexpr int SWZ = AT == 32 ? 7 : 3;       // 128B / 64B swizzle: chunk ^= (addr >> 7) & SWZ

    extern __shared__ unsigned char smem_tma[];
    __shared__ __align__(8) unsigned long long bar_z[FPC], bar_a[FPC], bar_p[FPC];
    __shared__ double red[FPC * WPF];

    TL(0);
    const int f = threadIdx.x / M;
    const int t = threadIdx.x % M;
    const int jl = blockIdx.x * FPC + f;
    const bool live = jl < count;
    const int j = a.first + (live ? jl : 0);
    // 1 KiB-align inside the dynamic buffer by offsetting the shared array itself
    // (keeps the shared address space visible to the compiler: LDS/STS, not LD/ST)
    const uint32_t pad = (1024u - (smem_u32(smem_tma) & 1023u)) & 1023u;
    unsigned char* fr = smem_tma + pad + (size_t)f * tma_frame_bytes<M>();
    float2* buf = reinterpret_cast<float2*>(fr);

    // The object window is loaded as an M x (M+2) box starting at the even
    // column below col0 (TMA box starts must be 16-B aligned); the tile pitch
    // is then S and column t of the window sits at t + (col0 & 1).
    const int2 pj = a.pos[j];
    const int odd = pj.y & 1;
    if (t == 0) {
        mbar_init(&bar_z[f], 1);
        mbar_init(&bar_a[f], 1);
        mbar_init(&bar_p[f], 1);
        fence_mbarrier_init();
        // PDL (solver graphs): the object is the predecessor's output
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (live) {   // object window -> [M][S] tile (out-of-range columns zero-filled)
            mbar_arrive_expect_tx(&bar_z[f], M * S * sizeof(float2));
            tma_load_2d(fr, &tm_z, 2 * (pj.y - odd), pj.x, &bar_z[f]);
        }
    }

    float2 x[M];
    const float2* __restrict__ probe = a.probe;
    // probe column t prefetched into the (not yet live) line registers while
    // the object tile is in flight: the L2 latency hides behind the TMA
    if constexpr (PROBE) {
#ifdef ABL_NOPREF   // ablation (timing only): no probe prefetch
#pragma unroll
        for (int r = 0; r < M; ++r) x[r] = make_float2(1.f + r * 1e-3f, 0.5f);
        (void)probe;
#else
#pragma unroll
        for (int r = 0; r < M; ++r) x[r] = __ldg(probe + r * M + t);
#endif
    }
    // the probe is immutable: its prefetch above may overlap the predecessor
    // grid; nothing written by it is read or overwritten before this point
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    if (live) mbar_wait(&bar_z[f], 0);
    TL(1);
#pragma unroll
    for (int r = 0; r < M; ++r) {   // psi = P o x, own column t
        if constexpr (PROBE) x[r] = cmul(x[r], buf[r * S + t + odd]);
        else x[r] = buf[r * S + t + odd];
    }
    __syncthreads();

    const float* amp_tile = reinterpret_cast<const float*>(fr);
    double acc = 0.0;
PTG_UNROLL_N(PTG_TMA_PASS_UNROLL)
    for (int pass = 0; pass < 4; ++pass) {
        reg_fft<M, false>(x);
        if (pass == 1) TL(2);
        if (pass == 0) {
            // columns -> rows
#ifndef ABL_NOTRANS
#pragma unroll
            for (int k = 0; k < M; ++k) buf[k * S + t] = x[k];
            __syncthreads();
#pragma unroll
            for (int c = 0; c < M; c += 2) {
                const float4 v = *reinterpret_cast<const float4*>(&buf[t * S + c]);
                x[c] = make_float2(v.x, v.y);
                x[c + 1] = make_float2(v.z, v.w);
            }
#endif
            __syncthreads();
            if (t == 0 && live) {   // amplitudes land while the row FFT runs
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&bar_a[f], M * M * sizeof(float));
#pragma unroll
                for (int h = 0; h < NAT; ++h)
                    tma_load_3d(fr + (size_t)h * AT * M * sizeof(float), &tm_amp, h * AT, 0, j, &bar_a[f]);
            }
        } else if (pass == 1) {
            // spectral operator on row t; x <- conj(R) feeds the inverse passes
            if (live) {
                mbar_wait(&bar_a[f], 0);
                // row misfit: four fp32 partial sums of non-negative terms (short
                // dependency chains), promoted to fp64 once per row
                float af[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < M; c += 4) {
                    const int h = c / AT, cc = c % AT;
                    const uint32_t off = (uint32_t)(t * AT + cc) * 4u;
                    const uint32_t sw = off ^ (((off >> 7) & SWZ) << 4);
                    const float4 A4 =
                        *reinterpret_cast<const float4*>(reinterpret_cast<const unsigned char*>(amp_tile) +
                                                         (size_t)h * AT * M * sizeof(float) + sw);
                    const float Av[4] = {A4.x, A4.y, A4.z, A4.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float2 W = x[c + q];
                        const float A = Av[q];
                        float2 R;
#ifdef ABL_NOSPEC   // ablation (timing only): trivial spectral operator
                        if (true) {
                            af[q] += A;
                            x[c + q] = make_float2(W.x * A, -W.y);
                            continue;
                        }
#endif
                        if constexpr (OP == OP_INTENSITY) {
                            const float r = (W.x * W.x + W.y * W.y) - A;
                            af[q] = fmaf(r, r, af[q]);
                            R = make_float2(W.x * r, W.y * r);
                        } else {
                            // |W|^2 below the smallest normal float is treated as W = 0
                            // (theta(0) = 0 branch: R = -A); this keeps the reciprocal
                            // square root a single flush-to-zero MUFU op
                            const float m2 = fmaf(W.x, W.x, W.y * W.y);
                            const bool nz = m2 >= 1.17549435e-38f;
                            const float inv = nz ? rsqrt_ftz(m2) : 0.f;   // 1/|W|, 0 for W = 0
                            const float dl = fmaf(m2, inv, -A);            // |W| - A
                            af[q] = fmaf(dl, dl, af[q]);
                            const float s = fmaf(-A, inv, 1.f);            // 1 - A/|W|
                            R = make_float2(fmaf(W.x, s, nz ? 0.f : -A), W.y * s);
                        }
                        x[c + q] = make_float2(R.x, -R.y);   // conj
                    }
                }
                acc = ((double)af[0] + (double)af[1]) + ((double)af[2] + (double)af[3]);
            }
        } else if (pass == 2) {
            // rows -> columns (x holds conj of the row-inverse; conjugations cancel)
            __syncthreads();   // amplitude reads done before the buffer is rewritten
#ifndef ABL_NOTRANS
#pragma unroll
            for (int c = 0; c < M; c += 2)
                *reinterpret_cast<float4*>(&buf[t * S + c]) = make_float4(x[c].x, x[c].y, x[c + 1].x, x[c + 1].y);
            __syncthreads();
#pragma unroll
            for (int r = 0; r < M; ++r) x[r] = buf[r * S + t];
#endif
            __syncthreads();
            if constexpr (PROBE) {
                // the buffer is idle during the last pass: TMA the probe tile in
                if (t == 0 && live) {
                    fence_proxy_async_smem();
                    mbar_arrive_expect_tx(&bar_p[f], M * M * sizeof(float2));
                    tma_load_2d(fr, &tm_p, 0, 0, &bar_p[f]);
                }
            }
        }
    }
    // x = conj(IDFT_unnormalised(R)) for column t

    // per-frame misfit (fixed shuffle tree + fixed warp order)
    if constexpr (M >= 32) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((t & 31) == 0) red[f * WPF + t / 32] = acc;
    } else {
#pragma unroll
        for (int o = M / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (t == 0) red[f] = acc;
    }
    __syncthreads();
    if (t == 0 && live) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < WPF; ++i) s += red[f * WPF + i];
        a.misfit[j] = (OP == OP_DISTANCE) ? s / (2.0 * (double)M * (double)M) : 0.5 * s;
    }
    // let the dependent gather kernel start launching (it waits on griddepcontrol.wait)
    TL(3);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // epilogue: contribution = sc * conj(P) o IDFT_u(R) = conj(sc P) o conj(x)
    if (live) {
        // stash row pitch M + 2, window row at offset (col0 & 1), zero pads (plan.cuh)
        const float sc = (OP == OP_DISTANCE) ? 1.f / (float(M) * float(M)) : 2.f;
        if constexpr (PROBE) mbar_wait(&bar_p[f], 0);
        if (a.planes) {   // colour plane: plain coalesced stores into the window
            float2* __restrict__ pl = a.planes + (size_t)a.color[j] * a.n * a.n + (size_t)pj.x * a.n + pj.y + t;
#pragma unroll
            for (int r = 0; r < M; ++r) {
                const float2 v = PROBE ? epi_contrib_pre(x[r], buf[r * M + t]) : epi_contrib(x[r], sc);
#ifdef ABL_NOSTORE   // ablation (timing only): no contribution stores
                if (v.x == 1234.5f)
#endif
                pl[(size_t)r * a.n] = v;
            }
            TL(4);
            return;
        }
        float2* __restrict__ out = a.stash + (size_t)j * M * S;
#pragma unroll
        for (int r = 0; r < M; ++r) {
            // pre-scaled conjugated probe tile conj(sc * P) (dense pitch M)
            const float2 v = PROBE ? epi_contrib_pre(x[r], buf[r * M + t]) : epi_contrib(x[r], sc);
            out[(size_t)r * S + odd + t] = v;
        }
        // the two zero pads of row t
        out[(size_t)t * S + (odd ? 0 : M)] = make_float2(0.f, 0.f);
        out[(size_t)t * S + M + 1] = make_float2(0.f, 0.f);
    }
}

}  // namespace ptg
