// frame_cl.cuh — cluster-split fused frame kernel for complex64 frames of
// side M = Q L (M = 128, 256; local line L = 32 or 64), w == M (patch mode).
//
// Same computation as frame_kernel<OP_DISTANCE/OP_INTENSITY> (frame_kernels.cuh,
// reference objectives.cpp:59-103).  A frame of M x M complex64 (128 / 512 KiB)
// is too large for one SM's registers or shared memory, so it is split over a
// thread-block cluster of Q CTAs: CTA q holds frame rows [Lq, Lq + L) in
// shared memory, and every line transform is one radix-Q butterfly stage
// plus Q independent L-point transforms, the latter done by the register
// line FFT of the M = 64 kernel (frame_reg.cuh: compile-time twiddles, one
// thread per L-point line):
//
//   columns (length M, split across the cluster):
//     forward  = DIF: radix-Q butterfly over the Q CTAs (distributed shared
//                memory) then FFT_L over each CTA's L rows; frequency
//                kr = Q k + q lands in CTA q, local row k;
//     inverse  = DIT: FFT_L over the local rows, pushed to the CTA owning the
//                output rows, then the radix-Q combine fused with the conj(P)
//                epilogue (global stores);
//   rows (length M, local to a CTA):
//     forward  = DIF butterfly in shared memory then FFT_L per row part,
//                spectral operator in registers (frequency kc = Q k + p),
//     inverse  = FFT_L of conj(R) in the same registers then the DIT combine.
//
// The inverse transforms use IDFT(X) = conj(DFT(conj X)) as in frame_tma.cuh,
// and all four FFT_L passes run from one rolled loop (one copy of the body in
// the instruction cache).  The spectral operator reads the amplitudes in the
// frequency order it produces them: the plan keeps a copy permuted to
// [j][q][r][p][k] = A_j[Q r + q][Q k + p] (k_perm_amp, plan.cu), so every
// thread streams L contiguous floats.  Per-CTA misfit partials go to
// misfit[j*M/32 + q] (fixed order, fp64).
#pragma once

#include <cooperative_groups.h>

#include "frame_reg.cuh"

namespace ptg {

// Q CTAs x L local rows, M = Q L.  The CTA's L amplitude rows are staged in
// shared memory by TMA bulk copies issued at kernel start (pitch M + 4
// floats: conflict-free 128-bit reads) when they fit next to the frame rows.
template <int Q, int L>
__host__ __device__ constexpr int cl_pitch() { return Q * L + 2; }   // complex elements per smem row
template <int Q, int L>
__host__ __device__ constexpr bool cl_amp_staged() { return !(Q == 2 && L == 64); }
template <int Q, int L>
__host__ __device__ constexpr int cl_amp_pitch() { return Q * L + 4; }
template <int Q, int L>
__host__ __device__ constexpr size_t cl_smem_bytes() {
    return sizeof(float2) * ((size_t)L * cl_pitch<Q, L>() + (size_t)Q * L)     // L rows + twiddle table
           + (cl_amp_staged<Q, L>() ? sizeof(float) * (size_t)L * cl_amp_pitch<Q, L>() : 0);
}
template <int Q, int L>
__host__ __device__ constexpr int cl_min_blocks() { return L == 32 ? (Q == 4 ? 4 : 2) : Q == 2 ? 2 : 1; }
// per-position misfit slots written by a cluster variant (one per CTA, at least M / 32)
__host__ __device__ constexpr int cl_mpp(int Q, int M) { return Q > M / 32 ? Q : M / 32; }

#ifndef PTG_CL_ASYNC_GATHER
#define PTG_CL_ASYNC_GATHER 1
#endif
// shared::cta address -> the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// 8-byte remote store completing 8 tx bytes on the receiver's mbarrier
__device__ __forceinline__ void st_async_f2(uint32_t raddr, float2 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "f"(v.x), "f"(v.y), "r"(rbar)
                 : "memory");
}

// forward DFT_Q in place, natural order
template <int Q>
__device__ __forceinline__ void dft_q(float2* v) {
    if constexpr (Q == 2) dft2<false>(v[0], v[1]);
    else if constexpr (Q == 4) dft4<false>(v[0], v[1], v[2], v[3]);
    else dft8<false>(v);
}

template <int Q, int L, int OP, bool PROBE>
__global__ void __launch_bounds__(Q * L, cl_min_blocks<Q, L>())
    frame_cl_kernel(FrameArgs<float> a, const float* __restrict__ amp_perm, const float2* __restrict__ tw_g,
                    const float2* __restrict__ probe_epi) {
    namespace cg = cooperative_groups;
    constexpr int M = Q * L, NT = M, PM = cl_pitch<Q, L>(), NPC = L / Q, AP = cl_amp_pitch<Q, L>();
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char cl_smem[];
    float2* buf = reinterpret_cast<float2*>(cl_smem);   // [L][PM]: frame rows Lq..Lq+L-1
    float2* tw = buf + L * PM;                           // W_M^i, i < M
    __shared__ double red[NT / 32];

    TL(0);
    const int q = (int)cl.block_rank();
    const int j = a.first + (int)(blockIdx.x / Q);
    const int t = threadIdx.x;
    const int2 pj = a.pos[j];
    const int n = a.n;
    float* amp_s = reinterpret_cast<float*>(tw + M);   // [L][M + 4] (staged variants)
    __shared__ __align__(8) unsigned long long bar_a;
#if PTG_CL_ASYNC_GATHER
    // gather exchange by st.async: every CTA's L x M rows arrive as remote
    // stores that complete_tx on the receiver's mbarrier (no cluster barrier,
    // no fence); initialised before the cluster start handshake below
    __shared__ __align__(8) unsigned long long bar_g;
    if (t == 0) {
        mbar_init(&bar_g, 1);
        fence_mbarrier_init();
        mbar_arrive_expect_tx(&bar_g, (uint32_t)(L * M * sizeof(float2)));
    }
    __syncthreads();
#endif
    // cluster start handshake, split: the wait sits before the first remote store
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    if constexpr (cl_amp_staged<Q, L>()) {
        if (t == 0) {
            mbar_init(&bar_a, 1);
            fence_mbarrier_init();
        }
        __syncthreads();
        if (t < 32) {   // this CTA's L permuted amplitude rows, one bulk copy per row
            const float* src = amp_perm + (size_t)j * M * M + (size_t)q * L * M;
            if (t == 0) mbar_arrive_expect_tx(&bar_a, L * M * sizeof(float));
            __syncwarp();
            for (int r = t; r < L; r += 32)
                tma_bulk_g2s(amp_s + r * AP, src + (size_t)r * M, M * sizeof(float), &bar_a);
        }
    }
    for (int i = t; i < M; i += NT) tw[i] = __ldg(tw_g + i);   // W_M^i (host fp64, rounded once)
    float2* rb[Q];   // every CTA's frame rows (distributed shared memory)
#pragma unroll
    for (int s = 0; s < Q; ++s) rb[s] = cl.map_shared_rank(buf, s);

    // gather fused with the column DIF butterflies: CTA q forms butterfly rows
    // r = q NPC + i (window rows r + 64 s, column t) straight from global memory
    // and stores output s into CTA s's row r
    float2 x[L];
    {
        // batches of BT butterflies: their Q z values and probe values in flight together
        constexpr int BT = 16 / Q;
        const float2* zc = a.z + (size_t)pj.x * n + pj.y + t;
#pragma unroll 1
        for (int b = 0; b < NPC; b += BT) {
            float2 zv[BT * Q], pv[BT * Q];
#pragma unroll
            for (int i = 0; i < BT; ++i)
#pragma unroll
                for (int s = 0; s < Q; ++s) {
                    const int row = q * NPC + b + i + L * s;
                    zv[i * Q + s] = zc[(size_t)row * n];
                    if constexpr (PROBE) pv[i * Q + s] = __ldg(a.probe + (size_t)row * M + t);
                }
            if (b == 0) {
                // the first batch's loads are in flight across the twiddle-table
                // sync and the cluster start handshake (needed only before the
                // first remote store)
                __syncthreads();                                              // twiddle table
                asm volatile("barrier.cluster.wait.aligned;" ::: "memory");   // every CTA of the cluster runs
            }
#pragma unroll
            for (int i = 0; i < BT; ++i) {
                const int r = q * NPC + b + i;
                float2 v[Q];
#pragma unroll
                for (int s = 0; s < Q; ++s) v[s] = PROBE ? cmul(pv[i * Q + s], zv[i * Q + s]) : zv[i * Q + s];
                dft_q<Q>(v);
#pragma unroll
                for (int s = 1; s < Q; ++s) v[s] = cmul(tw[r * s], v[s]);
#if PTG_CL_ASYNC_GATHER
#pragma unroll
                for (int s = 0; s < Q; ++s)
                    st_async_f2(mapa_u32(smem_u32(buf + r * PM + t), s), v[s], mapa_u32(smem_u32(&bar_g), s));
#else
#pragma unroll
                for (int s = 0; s < Q; ++s) rb[s][r * PM + t] = v[s];
#endif
            }
        }
    }
#if PTG_CL_ASYNC_GATHER
    mbar_wait(&bar_g, 0);   // all Q senders' rows have landed in this CTA
#else
    cl.sync();
#endif
    TL(1);

    // row-stage roles: butterflies (row g + Q i, element m); FFT64 quarter-rows (rr, qq)
    const int m = t % L, g = t / L;
    const int rr = t % L, qq = t / L;
    float2 rtw[Q];
#pragma unroll
    for (int s = 0; s < Q; ++s) rtw[s] = tw[m * s];
    const float* A = amp_perm + (size_t)j * M * M + ((size_t)q * L + rr) * M + (size_t)qq * L;
    double acc = 0.0;
PTG_UNROLL_N(PTG_CL_PASS_UNROLL)
    for (int pass = 0; pass < 4; ++pass) {
        if (pass == 0 || pass == 3) {   // column t of the local rows
#pragma unroll
            for (int k = 0; k < L; ++k) x[k] = buf[k * PM + t];
            // pass 3: this CTA's rows are consumed; the other CTAs may push into them
            if (pass == 3) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        } else if (pass == 1) {         // quarter qq of local row rr
#pragma unroll
            for (int c = 0; c < L; c += 2) {
                const float4 v = *reinterpret_cast<const float4*>(&buf[rr * PM + qq * L + c]);
                x[c] = make_float2(v.x, v.y);
                x[c + 1] = make_float2(v.z, v.w);
            }
        }
        reg_fft<L, false>(x);
        if (pass == 0) {
#pragma unroll
            for (int k = 0; k < L; ++k) buf[k * PM + t] = x[k];
            __syncthreads();
            // row DIF butterflies (local): elements m + 64 s of rows g + Q i
#pragma unroll 2
            for (int i = 0; i < NPC; ++i) {
                float2* row = buf + (g + Q * i) * PM + m;
                float2 v[Q];
#pragma unroll
                for (int s = 0; s < Q; ++s) v[s] = row[L * s];
                dft_q<Q>(v);
#pragma unroll
                for (int s = 1; s < Q; ++s) v[s] = cmul(rtw[s], v[s]);
#pragma unroll
                for (int s = 0; s < Q; ++s) row[L * s] = v[s];
            }
            __syncthreads();
        } else if (pass == 1) {
            // spectral operator at (kr, kc) = (Q rr + q, Q k + qq); x <- conj(R)
            float af[4] = {0.f, 0.f, 0.f, 0.f};
            if constexpr (cl_amp_staged<Q, L>()) mbar_wait(&bar_a, 0);
#pragma unroll
            for (int c = 0; c < L; c += 4) {
                const float4 A4 = cl_amp_staged<Q, L>()
                                      ? *reinterpret_cast<const float4*>(amp_s + rr * AP + qq * L + c)
                                      : __ldg(reinterpret_cast<const float4*>(A + c));
                const float Av[4] = {A4.x, A4.y, A4.z, A4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 W = x[c + u];
                    const float Am = Av[u];
                    float2 R;
                    if constexpr (OP == OP_INTENSITY) {
                        const float r = (W.x * W.x + W.y * W.y) - Am;
                        af[u] = fmaf(r, r, af[u]);
                        R = make_float2(W.x * r, W.y * r);
                    } else {
                        // |W|^2 below the smallest normal float is treated as W = 0 (frame_tma.cuh)
                        const float m2 = fmaf(W.x, W.x, W.y * W.y);
                        const bool nz = m2 >= 1.17549435e-38f;
                        const float inv = nz ? rsqrt_ftz(m2) : 0.f;
                        const float dl = fmaf(m2, inv, -Am);
                        af[u] = fmaf(dl, dl, af[u]);
                        const float s = fmaf(-Am, inv, 1.f);
                        R = make_float2(fmaf(W.x, s, nz ? 0.f : -Am), W.y * s);
                    }
                    x[c + u] = make_float2(R.x, -R.y);
                }
            }
            acc = ((double)af[0] + (double)af[1]) + ((double)af[2] + (double)af[3]);
            TL(2);
        } else if (pass == 2) {
#pragma unroll
            for (int c = 0; c < L; c += 2)
                *reinterpret_cast<float4*>(&buf[rr * PM + qq * L + c]) = make_float4(x[c].x, x[c].y, x[c + 1].x, x[c + 1].y);
            __syncthreads();
            // row DIT combine (local): out[m + 64 s] = DFT_Q_s(W_M^{m p} F_p[m])
#pragma unroll 2
            for (int i = 0; i < NPC; ++i) {
                float2* row = buf + (g + Q * i) * PM + m;
                float2 v[Q];
#pragma unroll
                for (int s = 0; s < Q; ++s) v[s] = row[L * s];
#pragma unroll
                for (int s = 1; s < Q; ++s) v[s] = cmul(rtw[s], v[s]);
                dft_q<Q>(v);
#pragma unroll
                for (int s = 0; s < Q; ++s) row[L * s] = v[s];
            }
            __syncthreads();
        } else {
            // push G_q[m] (column t) to the CTA that combines row m: its local row
            // (m % NPC) Q + q, so the combine reads only local shared memory
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < L; ++k) rb[k / NPC][((k % NPC) * Q + q) * PM + t] = x[k];
        }
    }
    // epilogue probe values conj(sc P) (rows q NPC + i + L s, column t) in
    // flight across the barrier
    if constexpr (PROBE) {
#pragma unroll
        for (int i = 0; i < NPC; ++i)
#pragma unroll
            for (int s = 0; s < Q; ++s) x[i * Q + s] = __ldg(probe_epi + (size_t)(q * NPC + i + L * s) * M + t);
    }

    // per-CTA misfit partial (fixed shuffle tree + fixed warp order)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((t & 31) == 0) red[t / 32] = acc;
    TL(3);
    cl.sync();   // every push has landed; no remote access after this point
    TL(4);
    if (t == 0) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < NT / 32; ++i) s += red[i];
        // misfit slots per position: M / 32 (the plan's layout for either split)
        constexpr int MPP = M / 32;
        a.misfit[(size_t)j * MPP + q] = (OP == OP_DISTANCE) ? s / (2.0 * (double)M * (double)M) : 0.5 * s;
        if constexpr (MPP > Q) a.misfit[(size_t)j * MPP + Q + q] = 0.0;
    }

    // column DIT combine over the cluster + epilogue: rows r + L s, column t.
    // One base pointer per CTA and 32-bit row offsets (rows r + L s of this
    // CTA, r = q NPC + i); stash rows have pitch SP with the window at
    // column (col0 & 1) and two zero pads (plan.cuh), written once below.
    const float sc = (OP == OP_DISTANCE) ? 1.f / (float(M) * float(M)) : 2.f;
    const int odd = pj.y & 1;
    constexpr int SP = stash_pitch(M);
    float2* __restrict__ base;
    unsigned rs;
    if (a.planes) {
        base = a.planes + (size_t)a.color[j] * n * n + (size_t)(pj.x + q * NPC) * n + pj.y + t;
        rs = (unsigned)n;
    } else {
        base = a.stash + (size_t)j * M * SP + (size_t)(q * NPC) * SP + odd + t;
        rs = (unsigned)SP;
    }
#pragma unroll   // x[] is indexed by i: full unroll keeps it in registers
    for (int i = 0; i < NPC; ++i) {
        const int r = q * NPC + i;
        float2 v[Q];
#pragma unroll
        for (int s = 0; s < Q; ++s) v[s] = buf[(i * Q + s) * PM + t];   // G_s[r], pushed by CTA s
#pragma unroll
        for (int s = 1; s < Q; ++s) v[s] = cmul(tw[r * s], v[s]);
        dft_q<Q>(v);
#pragma unroll
        for (int s = 0; s < Q; ++s) {
            const float2 val = PROBE ? epi_contrib_pre(v[s], x[i * Q + s]) : epi_contrib(v[s], sc);
            base[(unsigned)(i + L * s) * rs] = val;
        }
    }
    if (!a.planes && t < 2 * NPC * Q) {   // the zero pads of this CTA's stash rows
        const int k = t >> 1, row = q * NPC + k % NPC + L * (k / NPC);
        float2* out = a.stash + (size_t)j * M * SP + (size_t)row * SP;
        out[(t & 1) ? M + 1 : (odd ? 0 : M)] = make_float2(0.f, 0.f);
    }
    TL(5);
}

// [j][q][r][p][k] = A_j[Q r + q][Q k + p]: amplitudes in the order the cluster
// kernel's spectral operator consumes them
template <int Q, int L>
__global__ void k_perm_amp(const float* __restrict__ in, float* __restrict__ out, size_t total) {
    constexpr int M = Q * L;
    for (size_t o = blockIdx.x * (size_t)blockDim.x + threadIdx.x; o < total; o += (size_t)gridDim.x * blockDim.x) {
        const size_t jj = o / ((size_t)M * M);
        const int rem = (int)(o % ((size_t)M * M));
        const int k = rem % L, p = (rem / L) % Q, r = (rem / M) % L, q = rem / (L * M);
        out[o] = in[jj * M * M + (size_t)(Q * r + q) * M + Q * k + p];
    }
}

}  // namespace ptg
