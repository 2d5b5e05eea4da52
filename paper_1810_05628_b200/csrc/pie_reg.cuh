// pie_reg.cuh — PIE sweep (solvers.cpp:229-265, Alg. 1 complex-probe weight)
// for complex64 frames M in {16, 32, 64} with w == M, latency-optimised.
//
// A sweep is strictly sequential (each projection reads the window the
// previous one updated), so its cost is the latency of one projection.  One
// CTA of M threads walks the scan with the register line FFT of the objective
// kernel (frame_reg.cuh): each thread owns one column, then one row, of the
// frame; the four line passes (forward columns / rows, inverse rows / columns
// as DFTs of the conjugate) run from one rolled loop; two transposes go
// through shared memory.  Everything position-independent stays resident in
// shared memory (probe, PIE weight), the next position's amplitudes arrive by
// a TMA bulk copy while the current position computes, and the window's old
// values are kept in shared memory for the update, so a position costs one
// L2 round trip for its window plus the arithmetic.
#pragma once

#include "frame_reg.cuh"

namespace ptg {

template <int M>
__host__ __device__ constexpr size_t pie_reg_smem_bytes() {
    // transpose buffer (M x (M+2)) + window (M x M) + probe + weight (M x M each)
    // + two amplitude tiles (M x M floats) + alignment slack
    return sizeof(float2) * ((size_t)M * (M + 2) + 3 * (size_t)M * M) + 2 * sizeof(float) * M * M + 128;
}

// z (n x n, updated in place), probe / wgt (M x M, either may be null:
// binary window / scalar damping), amp = sqrt(d) per position (N x M x M)
template <int M>
__global__ void __launch_bounds__(M, 1)
    k_pie_reg(float2* z, const float2* __restrict__ probe, const int2* __restrict__ pos,
              const float* __restrict__ amp, int N, int n, const float2* __restrict__ wgt, float damping) {
    constexpr int S = M + 2;
    extern __shared__ __align__(128) unsigned char pie_smem[];
    float* amp_s = reinterpret_cast<float*>(pie_smem);                  // [2][M*M], 16-B aligned for TMA
    float2* buf = reinterpret_cast<float2*>(amp_s + 2 * M * M);        // [M][S]
    float2* zw = buf + M * S;                                          // [M][M] window before the update
    float2* P = zw + M * M;                                            // [M][M]
    float2* Wt = P + M * M;                                            // [M][M]
    __shared__ __align__(8) unsigned long long bar[2];
    const int t = threadIdx.x;
    const bool has_p = probe != nullptr, has_w = wgt != nullptr;
    for (int i = t; i < M * M; i += M) {
        P[i] = has_p ? probe[i] : make_float2(1.f, 0.f);
        Wt[i] = has_w ? wgt[i] : make_float2(damping, 0.f);
    }
    if (t == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbarrier_init();
        mbar_arrive_expect_tx(&bar[0], M * M * sizeof(float));
        tma_bulk_g2s(amp_s, amp, M * M * sizeof(float), &bar[0]);
    }
    __syncthreads();
    const float inv = 1.f / (float(M) * float(M));
    float2 x[M];
    for (int k = 0; k < N; ++k) {
        const int2 p = pos[k];
        const int b = k & 1;
        if (t == 0 && k + 1 < N) {   // next position's amplitudes land during this one
            fence_proxy_async_smem();   // the previous reads of that tile precede the async write
            mbar_arrive_expect_tx(&bar[b ^ 1], M * M * sizeof(float));
            tma_bulk_g2s(amp_s + (b ^ 1) * M * M, amp + (size_t)(k + 1) * M * M, M * M * sizeof(float), &bar[b ^ 1]);
        }
        // window column t (L2: the previous positions' updates), psi = P o x
        const float2* zc = z + (size_t)p.x * n + p.y + t;
#pragma unroll
        for (int r = 0; r < M; ++r) x[r] = __ldcg(zc + (size_t)r * n);
#pragma unroll
        for (int r = 0; r < M; ++r) {
            zw[r * M + t] = x[r];
            x[r] = cmul(P[r * M + t], x[r]);
        }
PTG_UNROLL_N(PTG_PIE_PASS_UNROLL)
        for (int pass = 0; pass < 4; ++pass) {
            reg_fft<M, false>(x);
            if (pass == 0 || pass == 2) {   // transpose through shared memory
                if (pass == 0) {
#pragma unroll
                    for (int r = 0; r < M; ++r) buf[r * S + t] = x[r];
                } else {
#pragma unroll
                    for (int c = 0; c < M; c += 2)
                        *reinterpret_cast<float4*>(&buf[t * S + c]) = make_float4(x[c].x, x[c].y, x[c + 1].x, x[c + 1].y);
                }
                __syncthreads();
                if (pass == 0) {
#pragma unroll
                    for (int c = 0; c < M; c += 2) {
                        const float4 v = *reinterpret_cast<const float4*>(&buf[t * S + c]);
                        x[c] = make_float2(v.x, v.y);
                        x[c + 1] = make_float2(v.z, v.w);
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < M; ++r) x[r] = buf[r * S + t];
                }
                __syncthreads();
            } else if (pass == 1) {
                // projection of row t: R = A W/|W| (theta(0) = 0: W = 0 -> A); x <- conj(R)
                mbar_wait(&bar[b], (k >> 1) & 1);
                const float* A = amp_s + b * M * M + t * M;
#pragma unroll
                for (int c = 0; c < M; c += 4) {
                    const float4 A4 = *reinterpret_cast<const float4*>(A + c);
                    const float Av[4] = {A4.x, A4.y, A4.z, A4.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float2 W = x[c + u];
                        const float m2 = fmaf(W.x, W.x, W.y * W.y);
                        const bool nz = m2 >= 1.17549435e-38f;
                        const float s = nz ? Av[u] * rsqrt_ftz(m2) : 0.f;
                        const float2 R = make_float2(nz ? W.x * s : Av[u], W.y * s);
                        x[c + u] = make_float2(R.x, -R.y);
                    }
                }
            }
        }
        // x = conj(IDFT_u(R)) for column t: Pi(psi) = conj(x) / M^2;
        // window += wgt o (Pi(psi) - psi)   (solvers.cpp:247-250, Alg. 1)
        float2* zo = z + (size_t)p.x * n + p.y + t;
#pragma unroll
        for (int r = 0; r < M; ++r) {
            const float2 zo_v = zw[r * M + t];
            const float2 psi = cmul(P[r * M + t], zo_v);
            const float2 dl = make_float2(x[r].x * inv - psi.x, -x[r].y * inv - psi.y);
            zo[(size_t)r * n] = cadd(zo_v, cmul(Wt[r * M + t], dl));
        }
        __syncthreads();   // this window's stores before the next window's loads
    }
}

}  // namespace ptg
