// frame_kernels.cuh — fused per-scan-position kernels (one CTA per pattern).
//
// GPU restatement of the reference's per-probe loop bodies:
//   phiDistance          objectives.cpp:59-72  (+ projectModulus :42-50,
//                        replaceModulus :29-38 with the theta(0)=0 rule)
//   phiIntensityGaussian objectives.cpp:83-103
//   simulate             forward.cpp:46-52
// generalised to the patch model: psi_j = P o S_j x placed at the origin of an
// M x M frame (M >= w), complex probe P (or the reference's binary window).
//
// Per CTA: gather P o x-window -> smem frame -> 2-D FFT -> spectral operator
// with a deterministic fp64 block reduction of the misfit -> inverse 2-D FFT
// -> conj(P) epilogue -> per-pattern contribution "stash" (w x w).  The stash
// is summed into the gradient by the fixed-order gather in eval.cu, so no
// float atomics are used and results are bitwise reproducible.
#pragma once

#include "common.cuh"
#include "fft.cuh"

namespace ptg {

enum SpectralOp {
    OP_DISTANCE = 0, OP_INTENSITY = 1, OP_SIMULATE = 2, OP_PROJECT = 3,
    // plain 2-D transforms of the gathered frame (fft2 / ifft2, field.hpp:91-93):
    // the same smem FFT and 1/M^2 scaling as the projection's inverse, so
    // ifft2 of a projection's spectrum is bitwise the projection
    OP_FFT_FWD = 4, OP_FFT_INV = 5
};

template <typename T>
struct FrameArgs {
    const cplx<T>* z;        // object n x n
    const cplx<T>* probe;    // M x M, or nullptr (binary window)
    const int2* pos;         // (row0, col0) per pattern
    const T* amp;            // N x M x M: sqrt(d) (distance/project) or d (intensity)
    cplx<T>* stash;          // per-pattern contribution, w x w (distance / intensity)
    cplx<T>* frame_out;      // OP_PROJECT: M x M projection per pattern
    T* data_out;             // OP_SIMULATE: N x M x M intensities
    double* misfit;          // per-pattern objective contribution
    int n, w, first;         // pattern index = first + blockIdx.x
    // colour-plane overlap-add (plan.cuh): contribution of pattern j goes to
    // planes[color[j]] at its window (nullptr = stash mode)
    cplx<T>* planes;
    const int* color;
};

// Deterministic block reduction (fixed shuffle tree + fixed warp order).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    constexpr int NW = (NT + 31) / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NW; ++i) s += red[i];
    }
    __syncthreads();
    return s;
}

// value = sum_j misfit_j - sum_t dotp_t by NT threads: fixed contiguous
// partition + fixed shuffle tree + fixed warp order (deterministic).
// red needs NT / 32 doubles; the result is written by thread 0.
template <int NT>
__device__ __forceinline__ void finalize_value(const double* misfit, int N, const double* dotp, int ndot,
                                               double* out, double* red, int lin) {
    constexpr int NW = NT / 32;
    double m = 0.0, d = 0.0;
    const int cm = (N + NT - 1) / NT, cd = (ndot + NT - 1) / NT;
    const int m0 = lin * cm, me = min(m0 + cm, N), d0 = lin * cd, de = min(d0 + cd, ndot);
    // both partitions' loads batched ahead of the (in-order) sums: one L2 round
    // trip per B values of each
    constexpr int B = 16;
    for (int i = 0; i < cm || i < cd; i += B) {
        double tm[B], td[B];
#pragma unroll
        for (int u = 0; u < B; ++u) tm[u] = m0 + i + u < me ? __ldcg(misfit + m0 + i + u) : 0.0;
#pragma unroll
        for (int u = 0; u < B; ++u) td[u] = d0 + i + u < de ? __ldcg(dotp + d0 + i + u) : 0.0;
#pragma unroll
        for (int u = 0; u < B; ++u) m += tm[u];
#pragma unroll
        for (int u = 0; u < B; ++u) d += td[u];
    }
    double both[2] = {m, d};
    double res[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        double x = both[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        __syncthreads();
        if ((lin & 31) == 0) red[lin >> 5] = x;
        __syncthreads();
        double s = 0.0;
        if (lin == 0)
            for (int i = 0; i < NW; ++i) s += red[i];
        res[q] = s;
    }
    if (lin == 0) *out = res[0] - res[1];
}

template <typename T, int M>
__host__ __device__ constexpr size_t frame_smem_bytes(int NT) {
    return sizeof(cplx<T>) * ((size_t)M * frame_stride(M) + M) + sizeof(double) * ((NT + 31) / 32);
}

template <typename T, int M, int NT, int OP>
__global__ void __launch_bounds__(NT) frame_kernel(FrameArgs<T> a) {
    using C = cplx<T>;
    constexpr int S = frame_stride(M);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* buf = reinterpret_cast<C*>(smem_raw);
    C* tw = buf + M * S;
    double* red = reinterpret_cast<double*>(tw + M);

    const int j = a.first + blockIdx.x;
    const int2 p = a.pos[j];
    const int n = a.n, w = a.w;
    build_twiddles<T>(tw, M);

    // gather psi = P o S_j x into the frame origin, zero elsewhere (applyProbe)
    for (int idx = threadIdx.x; idx < M * M; idx += NT) {
        const int r = idx / M, c = idx % M;
        C v = mk<T>(T(0), T(0));
        if (r < w && c < w) {
            const C zz = a.z[(size_t)(p.x + r) * n + (p.y + c)];
            v = a.probe ? cmul(a.probe[idx], zz) : zz;
        }
        buf[r * S + c] = v;
    }
    __syncthreads();
    if constexpr (OP == OP_FFT_FWD || OP == OP_FFT_INV) {
        fft2d_smem<T, M, NT, OP == OP_FFT_INV>(buf, S, tw);
        C* out = a.frame_out + (size_t)j * M * M;
        const T sc = T(1) / (T(M) * T(M));
        for (int idx = threadIdx.x; idx < M * M; idx += NT) {
            const C v = buf[(idx / M) * S + idx % M];
            out[idx] = OP == OP_FFT_INV ? cscale(v, sc) : v;
        }
        return;
    }
    fft2d_smem<T, M, NT, false>(buf, S, tw);

    if constexpr (OP == OP_SIMULATE) {
        T* out = a.data_out + (size_t)j * M * M;
        for (int idx = threadIdx.x; idx < M * M; idx += NT) {
            const C W = buf[(idx / M) * S + idx % M];
            out[idx] = W.x * W.x + W.y * W.y;
        }
        return;
    } else {
        const T* amp = a.amp + (size_t)j * M * M;
        double acc = 0.0;
        for (int idx = threadIdx.x; idx < M * M; idx += NT) {
            C W = buf[(idx / M) * S + idx % M];
            const T A = amp[idx];
            C R;
            if constexpr (OP == OP_INTENSITY) {
                // r = |W|^2 - d ; value += r^2 / 2 ; spectral R = r W
                const T r = (W.x * W.x + W.y * W.y) - A;
                acc += (double)r * (double)r;
                R = cscale(W, r);
            } else {
                const T mag = sqrt(W.x * W.x + W.y * W.y);
                if constexpr (OP == OP_DISTANCE) {
                    // psi - Pi(psi) in frequency space: W (1 - A/|W|); W = 0 -> -A
                    const T dlt = mag - A;
                    acc += (double)dlt * (double)dlt;
                    R = mag > T(0) ? cscale(W, T(1) - A / mag) : mk<T>(-A, T(0));
                } else {   // OP_PROJECT: Pi(psi) = A W/|W|, W = 0 -> A
                    R = mag > T(0) ? cscale(W, A / mag) : mk<T>(A, T(0));
                }
            }
            buf[(idx / M) * S + idx % M] = R;
        }
        if constexpr (OP != OP_PROJECT) {
            const double s = block_sum<NT>(acc, red);   // includes __syncthreads
            if (threadIdx.x == 0)
                a.misfit[j] = (OP == OP_DISTANCE) ? s / (2.0 * (double)M * (double)M) : 0.5 * s;
        } else {
            __syncthreads();
        }
        fft2d_smem<T, M, NT, true>(buf, S, tw);

        if constexpr (OP == OP_PROJECT) {
            const T sc = T(1) / (T(M) * T(M));
            C* out = a.frame_out + (size_t)j * M * M;
            for (int idx = threadIdx.x; idx < M * M; idx += NT)
                out[idx] = cscale(buf[(idx / M) * S + idx % M], sc);
        } else {
            // epilogue: contribution ADDED to the gradient
            //   distance : conj(P) (psi - Pi(psi)) = conj(P) ifft2(R)           (x 1/M^2)
            //   intensity: 2 M^2 conj(P) ifft2(r W) = 2 conj(P) IDFT_unnorm(R)  (objectives.cpp:98-102)
            const T sc = (OP == OP_DISTANCE) ? T(1) / (T(M) * T(M)) : T(2);
            if (a.planes) {   // colour plane: plain stores into the window
                C* pl = a.planes + (size_t)a.color[j] * n * n + (size_t)p.x * n + p.y;
                for (int idx = threadIdx.x; idx < w * w; idx += NT) {
                    const int r = idx / w, c = idx % w;
                    C v = cscale(buf[r * S + c], sc);
                    if (a.probe) v = cmulc(a.probe[r * M + c], v);
                    pl[(size_t)r * n + c] = v;
                }
                return;
            }
            const int sp = stash_pitch(w), odd = p.y & 1;   // stash row pitch / parity shift
            C* out = a.stash + (size_t)j * w * sp;
            for (int idx = threadIdx.x; idx < w * sp; idx += NT) {
                const int r = idx / sp, e = idx % sp, c = e - odd;
                C v = mk<T>(T(0), T(0));
                if ((unsigned)c < (unsigned)w) {
                    v = cscale(buf[r * S + c], sc);
                    if (a.probe) v = cmulc(a.probe[r * M + c], v);
                }
                out[idx] = v;
            }
        }
    }
}

}  // namespace ptg
