// frame_multipass.cuh — per-position pipeline for frames too large for one
// CTA's shared memory (complex64 M = 256, complex128 M >= 128; M <= 512).
//
// Same computation as frame_kernel (frame_kernels.cuh; reference
// objectives.cpp:59-103, forward.cpp:46-52), split into three kernels over a
// chunk of positions with an L2-sized scratch of whole frames:
//   mp_rows_fwd   grid (frames, M/NL): gather P o x for NL rows, row FFTs
//   mp_cols       grid (frames, M/NL): NL columns: FFT, spectral op (+ fp64
//                 misfit partial per block), inverse FFT  [or |W|^2 for simulate]
//   mp_rows_inv   grid (frames, M/NL): inverse row FFTs, conj(P) epilogue ->
//                 per-position stash (distance / intensity) or projection
// Lines are transformed in shared memory by the Stockham engine (fft.cuh).
#pragma once

#include "fft.cuh"
#include "frame_kernels.cuh"

namespace ptg {

constexpr int kMpLines = 16;   // lines (rows or columns) per CTA

template <int M>
constexpr int mp_threads() { return M >= 512 ? 512 : 256; }

template <typename T, int M>
constexpr size_t mp_smem_bytes() {
    return sizeof(cplx<T>) * ((size_t)kMpLines * (M + 1) + M) + sizeof(double) * 32;
}

struct MpArgs {
    int first;            // global index of the chunk's first position
    int nblk;             // M / kMpLines
    double* misfit_part;  // [N][nblk] partial objective values (global j)
};

// 1. rows [r0, r0+NL) of psi_j = P o S_j x, forward row FFTs -> scratch
template <typename T, int M>
__global__ void __launch_bounds__(mp_threads<M>()) mp_rows_fwd(FrameArgs<T> a, MpArgs m, cplx<T>* scratch) {
    using C = cplx<T>;
    constexpr int NL = kMpLines, NT = mp_threads<M>(), S = M + 1;
    extern __shared__ __align__(16) unsigned char smem_mp[];
    C* buf = reinterpret_cast<C*>(smem_mp);
    C* tw = buf + NL * S;
    const int f = blockIdx.x, blk = blockIdx.y, r0 = blk * NL;
    const int j = m.first + f;
    const int2 p = a.pos[j];
    build_twiddles<T>(tw, M);
    for (int idx = threadIdx.x; idx < NL * M; idx += NT) {
        const int rl = idx / M, c = idx % M, r = r0 + rl;
        C v = mk<T>(T(0), T(0));
        if (r < a.w && c < a.w) {
            v = a.z[(size_t)(p.x + r) * a.n + (p.y + c)];
            if (a.probe) v = cmul(a.probe[(size_t)r * M + c], v);
        }
        buf[rl * S + c] = v;
    }
    __syncthreads();
    fft_lines<T, M, NL, NT, false, false>(buf, S, 1, tw);
    C* out = scratch + (size_t)f * M * M + (size_t)r0 * M;
    for (int idx = threadIdx.x; idx < NL * M; idx += NT) out[idx] = buf[(idx / M) * S + idx % M];
}

// 2. columns [c0, c0+NL): forward FFT, spectral op, inverse FFT (in place)
template <typename T, int M, int OP>
__global__ void __launch_bounds__(mp_threads<M>()) mp_cols(FrameArgs<T> a, MpArgs m, cplx<T>* scratch) {
    using C = cplx<T>;
    constexpr int NL = kMpLines, NT = mp_threads<M>(), S = M + 1;
    extern __shared__ __align__(16) unsigned char smem_mp[];
    C* buf = reinterpret_cast<C*>(smem_mp);       // column-major: line = column
    C* tw = buf + NL * S;
    double* red = reinterpret_cast<double*>(tw + M);
    const int f = blockIdx.x, blk = blockIdx.y, c0 = blk * NL;
    const int j = m.first + f;
    build_twiddles<T>(tw, M);
    C* fr = scratch + (size_t)f * M * M;
    for (int idx = threadIdx.x; idx < NL * M; idx += NT) {
        const int r = idx / NL, cl = idx % NL;
        buf[cl * S + r] = fr[(size_t)r * M + c0 + cl];
    }
    __syncthreads();
    fft_lines<T, M, NL, NT, false, false>(buf, S, 1, tw);
    if constexpr (OP == OP_SIMULATE) {
        T* out = a.data_out + (size_t)j * M * M;
        for (int idx = threadIdx.x; idx < NL * M; idx += NT) {
            const int r = idx / NL, cl = idx % NL;
            const C W = buf[cl * S + r];
            out[(size_t)r * M + c0 + cl] = W.x * W.x + W.y * W.y;
        }
        return;
    } else {
        const T* amp = a.amp + (size_t)j * M * M;
        double acc = 0.0;
        for (int idx = threadIdx.x; idx < NL * M; idx += NT) {
            const int r = idx / NL, cl = idx % NL;
            const C W = buf[cl * S + r];
            const T A = amp[(size_t)r * M + c0 + cl];
            C R;
            if constexpr (OP == OP_INTENSITY) {
                const T rr = (W.x * W.x + W.y * W.y) - A;
                acc += (double)rr * (double)rr;
                R = cscale(W, rr);
            } else {
                const T mag = sqrt(W.x * W.x + W.y * W.y);
                if constexpr (OP == OP_DISTANCE) {
                    const T dl = mag - A;
                    acc += (double)dl * (double)dl;
                    R = mag > T(0) ? cscale(W, T(1) - A / mag) : mk<T>(-A, T(0));
                } else {   // OP_PROJECT
                    R = mag > T(0) ? cscale(W, A / mag) : mk<T>(A, T(0));
                }
            }
            buf[cl * S + r] = R;
        }
        if constexpr (OP != OP_PROJECT) {
            const double s = block_sum<NT>(acc, red);
            if (threadIdx.x == 0)
                m.misfit_part[(size_t)j * m.nblk + blk] =
                    (OP == OP_DISTANCE) ? s / (2.0 * (double)M * (double)M) : 0.5 * s;
        } else {
            __syncthreads();
        }
        fft_lines<T, M, NL, NT, true, false>(buf, S, 1, tw);
        for (int idx = threadIdx.x; idx < NL * M; idx += NT) {
            const int r = idx / NL, cl = idx % NL;
            fr[(size_t)r * M + c0 + cl] = buf[cl * S + r];
        }
    }
}

// 3. rows [r0, r0+NL): inverse row FFTs, epilogue
template <typename T, int M, int OP>
__global__ void __launch_bounds__(mp_threads<M>()) mp_rows_inv(FrameArgs<T> a, MpArgs m, const cplx<T>* scratch) {
    using C = cplx<T>;
    constexpr int NL = kMpLines, NT = mp_threads<M>(), S = M + 1;
    extern __shared__ __align__(16) unsigned char smem_mp[];
    C* buf = reinterpret_cast<C*>(smem_mp);
    C* tw = buf + NL * S;
    const int f = blockIdx.x, blk = blockIdx.y, r0 = blk * NL;
    const int j = m.first + f;
    build_twiddles<T>(tw, M);
    const C* in = scratch + (size_t)f * M * M + (size_t)r0 * M;
    for (int idx = threadIdx.x; idx < NL * M; idx += NT) buf[(idx / M) * S + idx % M] = in[idx];
    __syncthreads();
    fft_lines<T, M, NL, NT, true, false>(buf, S, 1, tw);
    const T inv = T(1) / (T(M) * T(M));
    if constexpr (OP == OP_PROJECT) {
        C* out = a.frame_out + (size_t)j * M * M + (size_t)r0 * M;
        for (int idx = threadIdx.x; idx < NL * M; idx += NT) out[idx] = cscale(buf[(idx / M) * S + idx % M], inv);
    } else {
        const T sc = (OP == OP_DISTANCE) ? inv : T(2);
        const int w = a.w, sp = stash_pitch(w), odd = a.pos[j].y & 1;   // stash pitch / parity shift
        C* out = a.stash + (size_t)j * w * sp;
        for (int idx = threadIdx.x; idx < NL * sp; idx += NT) {
            const int rl = idx / sp, e = idx % sp, r = r0 + rl, c = e - odd;
            if (r >= w) continue;
            C v = mk<T>(T(0), T(0));
            if ((unsigned)c < (unsigned)w) {
                v = cscale(buf[rl * S + c], sc);
                if (a.probe) v = cmulc(a.probe[(size_t)r * M + c], v);
            }
            out[(size_t)r * sp + e] = v;
        }
    }
}

}  // namespace ptg
