// fft.cuh — CTA-cooperative shared-memory FFT engine (sm_100a).
//
// Replaces the reference's serial radix-2 fft1d / fft2Impl
// (/root/reference/proj/src/kernels.cpp:34-85) for the GPU hot path.  Same DFT
// convention (kernels.hpp:25-28): forward F[u] = sum f[r] e^{-2 pi i u r / L},
// unnormalised; the inverse here is ALSO unnormalised — callers fold the 1/L^2
// of the 2-D inverse into their epilogue.
//
// Algorithm: mixed-radix Stockham autosort (radix 2/4/8/16), one pass per
// radix.  A pass reads R elements of a line at stride L/R into registers,
// applies the inter-pass twiddles (from a per-CTA table in shared memory),
// runs an unrolled register DFT_R with compile-time constants, and writes the
// R results back at stride Ns (natural order after the last pass, so no
// bit-reversal step).  Lines are rows (elem_stride 1) or columns
// (line_stride 1) of a frame resident in shared memory.
#pragma once

#include "common.cuh"

namespace ptg {

// ---------------------------------------------------------------- planning
// radices per line length (product == L); index q = pass number
__host__ __device__ constexpr int fft_npass(int L) {
    return L <= 1 ? 0 : (L <= 8 ? 1 : (L <= 256 ? 2 : 3));
}
__host__ __device__ constexpr int fft_radix(int L, int q) {
    // 2:[2] 4:[4] 8:[8] 16:[4,4] 32:[4,8] 64:[8,8] 128:[8,16] 256:[16,16]
    // 512:[8,8,8] 1024:[16,8,8] 2048:[16,16,8] 4096:[16,16,16]
    return L <= 8 ? L
         : L == 16 ? 4
         : L == 32 ? (q == 0 ? 4 : 8)
         : L == 64 ? 8
         : L == 128 ? (q == 0 ? 8 : 16)
         : L == 256 ? 16
         : L == 512 ? 8
         : L == 1024 ? (q == 0 ? 16 : 8)
         : L == 2048 ? (q < 2 ? 16 : 8)
         : 16;
}
__host__ __device__ constexpr int fft_ns(int L, int q) {
    int ns = 1;
    for (int i = 0; i < q; ++i) ns *= fft_radix(L, i);
    return ns;
}

// ------------------------------------------------------ register DFT_R
template <bool INV, typename C>
__device__ __forceinline__ C mul_negi(C a) {   // a * (-i) forward, a * (+i) inverse
    C r;
    if (INV) { r.x = -a.y; r.y = a.x; } else { r.x = a.y; r.y = -a.x; }
    return r;
}

template <bool INV, typename C>
__device__ __forceinline__ void dft2(C& a, C& b) {
    C t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

template <bool INV, typename C>
__device__ __forceinline__ void dft4(C& a0, C& a1, C& a2, C& a3) {
    C t0 = cadd(a0, a2), t1 = csub(a0, a2);
    C t2 = cadd(a1, a3), t3 = mul_negi<INV>(csub(a1, a3));
    a0 = cadd(t0, t2);
    a2 = csub(t0, t2);
    a1 = cadd(t1, t3);
    a3 = csub(t1, t3);
}

// (x + iy) * W8^1 (forward W8 = (1 - i)/sqrt2; inverse conj), written as a
// complex add of the swapped/negated copy so packed FP32 folds it to 2 ops
template <bool INV, typename C>
__device__ __forceinline__ C mul_w8_1(C a) {
    using T = decltype(a.x);
    const T c = T(0.70710678118654752440084436210485);
    C sw;
    if (INV) { sw.x = -a.y; sw.y = a.x; }   // (x - y, y + x)
    else     { sw.x = a.y; sw.y = -a.x; }   // (x + y, y - x)
    return cscale(cadd(a, sw), c);
}
template <bool INV, typename C>
__device__ __forceinline__ C mul_w8_3(C a) {   // W8^3 = (-1 - i)/sqrt2 forward
    using T = decltype(a.x);
    const T c = T(0.70710678118654752440084436210485);
    C sw;
    if (INV) { sw.x = -a.y; sw.y = a.x; }   // (-y - x, x - y)
    else     { sw.x = a.y; sw.y = -a.x; }   // (y - x, -x - y)
    return cscale(csub(sw, a), c);
}

template <bool INV, typename C>
__device__ __forceinline__ void dft8(C* a) {
    // radix-2 DIT over two DFT4s (even / odd samples)
    dft4<INV>(a[0], a[2], a[4], a[6]);
    dft4<INV>(a[1], a[3], a[5], a[7]);
    C o1 = mul_w8_1<INV>(a[3]);
    C o2 = mul_negi<INV>(a[5]);
    C o3 = mul_w8_3<INV>(a[7]);
    C e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6], o0 = a[1];
    a[0] = cadd(e0, o0); a[4] = csub(e0, o0);
    a[1] = cadd(e1, o1); a[5] = csub(e1, o1);
    a[2] = cadd(e2, o2); a[6] = csub(e2, o2);
    a[3] = cadd(e3, o3); a[7] = csub(e3, o3);
}

template <bool INV, typename C>
__device__ __forceinline__ void dft16(C* a) {
    using T = decltype(a[0].x);
    C e[8], o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { e[i] = a[2 * i]; o[i] = a[2 * i + 1]; }
    dft8<INV>(e);
    dft8<INV>(o);
    // W16^k = exp(-+ i pi k / 8)
    const T c1 = T(0.92387953251128675612818318939679);   // cos(pi/8)
    const T s1 = T(0.38268343236508977172845998403040);   // sin(pi/8)
    const T c2 = T(0.70710678118654752440084436210485);
    const T sg = INV ? T(1) : T(-1);
    const T wr[8] = {T(1), c1, c2, s1, T(0), -s1, -c2, -c1};
    const T wi[8] = {T(0), s1, c2, c1, T(1), c1, c2, s1};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        C t;
        if (k == 0) {
            t = o[0];
        } else {
            C w;
            w.x = wr[k];
            w.y = sg * wi[k];
            t = cmul(o[k], w);
        }
        a[k] = cadd(e[k], t);
        a[k + 8] = csub(e[k], t);
    }
}

template <int R, bool INV, typename C>
__device__ __forceinline__ void dft(C* a) {
    if constexpr (R == 2) dft2<INV>(a[0], a[1]);
    else if constexpr (R == 4) dft4<INV>(a[0], a[1], a[2], a[3]);
    else if constexpr (R == 8) dft8<INV>(a);
    else if constexpr (R == 16) dft16<INV>(a);
}

// ----------------------------------------------------------- twiddle table
// tw[e] = exp(-2 pi i e / L), e in [0, L); built once per CTA in double.
template <typename T>
__device__ __forceinline__ void build_twiddles(cplx<T>* tw, int L) {
    for (int e = threadIdx.x; e < L; e += blockDim.x) {
        double s, c;
        sincospi(-2.0 * (double)e / (double)L, &s, &c);
        tw[e] = mk<T>(T(c), T(s));
    }
}

// ------------------------------------------------------------- line passes
// One Stockham pass Q over NLINES lines of length L held in shared memory.
// LANES_ON_LINES: consecutive threads take consecutive lines (column passes,
// coalesced across the row); otherwise consecutive threads walk one line.
template <typename T, int L, int NLINES, int NT, bool INV, bool LANES_ON_LINES, int Q>
__device__ __forceinline__ void fft_pass(cplx<T>* buf, int ls, int es, const cplx<T>* tw) {
    using C = cplx<T>;
    if constexpr (Q < fft_npass(L)) {
        constexpr int R = fft_radix(L, Q);
        constexpr int Ns = fft_ns(L, Q);
        constexpr int TL = L / R;             // tasks per line
        constexpr int TASKS = NLINES * TL;
        constexpr int K = (TASKS + NT - 1) / NT;
        C v[K][R];
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
            const int t = threadIdx.x + kk * NT;
            if (TASKS % NT == 0 || t < TASKS) {
                const int line = LANES_ON_LINES ? (t % NLINES) : (t / TL);
                const int j = LANES_ON_LINES ? (t / NLINES) : (t % TL);
                const C* base = buf + line * ls;
#pragma unroll
                for (int r = 0; r < R; ++r) v[kk][r] = base[(j + r * TL) * es];
                if constexpr (Ns > 1) {
                    const int e = (j % Ns) * (L / (Ns * R));
#pragma unroll
                    for (int r = 1; r < R; ++r) {
                        C w = tw[e * r];
                        if (INV) w.y = -w.y;
                        v[kk][r] = cmul(v[kk][r], w);
                    }
                }
                dft<R, INV>(v[kk]);
            }
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
            const int t = threadIdx.x + kk * NT;
            if (TASKS % NT == 0 || t < TASKS) {
                const int line = LANES_ON_LINES ? (t % NLINES) : (t / TL);
                const int j = LANES_ON_LINES ? (t / NLINES) : (t % TL);
                C* base = buf + line * ls;
                const int idxD = (j / Ns) * Ns * R + (j % Ns);
#pragma unroll
                for (int r = 0; r < R; ++r) base[(idxD + r * Ns) * es] = v[kk][r];
            }
        }
        __syncthreads();
        fft_pass<T, L, NLINES, NT, INV, LANES_ON_LINES, Q + 1>(buf, ls, es, tw);
    }
}

// 1-D transforms of NLINES lines (caller has synchronised the buffer).
template <typename T, int L, int NLINES, int NT, bool INV, bool LANES_ON_LINES>
__device__ __forceinline__ void fft_lines(cplx<T>* buf, int ls, int es, const cplx<T>* tw) {
    fft_pass<T, L, NLINES, NT, INV, LANES_ON_LINES, 0>(buf, ls, es, tw);
}

// Full 2-D M x M transform of a frame in shared memory, row stride S.
template <typename T, int M, int NT, bool INV>
__device__ __forceinline__ void fft2d_smem(cplx<T>* buf, int S, const cplx<T>* tw) {
    fft_lines<T, M, M, NT, INV, false>(buf, S, 1, tw);   // rows
    fft_lines<T, M, M, NT, INV, true>(buf, 1, S, tw);    // columns
}

// Row stride (in complex elements) of a frame in shared memory: one element of
// padding staggers rows across banks for the row passes.
__host__ __device__ constexpr int frame_stride(int M) { return M >= 8 ? M + 1 : M; }

}  // namespace ptg
