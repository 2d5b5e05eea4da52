// frame_rmw2.cuh — the persistent RMW frame kernel (frame_rmw.cuh) for
// M = 256 with TWO threads per 32-point line: 512 threads per CTA, 64
// registers, so two CTAs of an SM hold 32 warps instead of 16.
//
// Same decomposition as frame_rmw_kernel<8, 32> (8-CTA clusters, 32 frame
// rows per CTA, radix-8 butterflies across the cluster / across row parts)
// and the same dependency-ordered read-modify-write of the gradient; what
// changes is the 32-point line transforms:
//   forward (columns in pass 0 / 3, row parts in pass 1): DIF split -- both
//     threads of a line read its 32 values, thread h forms
//     h = 0: a[n] = x[n] + x[n+16],  h = 1: a[n] = (x[n] - x[n+16]) W32^n,
//     and a DFT_16 of a gives X[2j + h];
//   inverse row parts (pass 2, on the spectral operator's output held in
//     that decimated order): DIT -- thread h's DFT_16 gives E (h = 0) or O
//     (h = 1), stored as E and W32^n O, and the row combine reads
//     Y[n] = E[n'] +- W32^n' O[n'].
// The amplitudes are permuted so each thread reads its 16 spectral samples
// contiguously ([j][q][r][p][h][j'] = A_j[8 r + q][8 (2 j' + h) + p]).
#pragma once

#include "frame_rmw.cuh"

namespace ptg {

// thread h's half of a forward DFT_32 (natural-order inputs ld(0..31)):
// y[j] = X[2 j + h]
template <class LD>
__device__ __forceinline__ void dft32_half(int h, const LD& ld, float2 (&y)[16]) {
    if (h == 0) {
        static_for<16>([&](auto nc) {
            constexpr int m = decltype(nc)::value;
            y[m] = cadd(ld(m), ld(m + 16));
        });
    } else {
        static_for<16>([&](auto nc) {
            constexpr int m = decltype(nc)::value;
            y[m] = twiddle_mul<32, false, m>(csub(ld(m), ld(m + 16)));
        });
    }
    reg_fft<16, false>(y);
}

template <int OP, bool PROBE>
__global__ void __launch_bounds__(512, 2)
    frame_rmw2_kernel(FrameArgs<float> a, const float* __restrict__ amp_perm, const float2* __restrict__ tw_g,
                      const float2* __restrict__ probe_epi, RmwArgs r) {
    namespace cg = cooperative_groups;
    constexpr int Q = 8, L = 32, M = Q * L, NT = 512, PM = cl_pitch<Q, L>(), NPC = L / Q, AP = cl_amp_pitch<Q, L>();
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char cl_smem[];
    float2* buf = reinterpret_cast<float2*>(cl_smem);   // [L][PM]: this CTA's frame rows
    float2* tw = buf + L * PM;                           // W_M^i, i < M
    float* amp_s = reinterpret_cast<float*>(tw + M);     // [L][AP] (split order within each 32-sample part)
    __shared__ double red[NT / 32];
    __shared__ __align__(8) unsigned long long bar_a, bar_g;
    __shared__ int4 s_item;

    const int q = (int)cl.block_rank();
    const int t = threadIdx.x;
    const int h = t >> 8, c = t & 255;         // line half, column / line index
    const int m = t % L, g = t / L;            // row-butterfly roles: element m, rows g + 16 i
    const int rr = c % L, qq = c / L;          // row-part roles: row rr, part qq
    const int n = a.n;
    if (t == 0) {
        mbar_init(&bar_g, 1);
        mbar_init(&bar_a, 1);
        fence_mbarrier_init();
    }
    for (int i = t; i < M; i += NT) tw[i] = __ldg(tw_g + i);
    const bool leader = q == 0 && t == 0;
    int4 next = make_int4(0, 0, 0, 0);
    if (leader) {
        next.x = r.kbeg + (int)atomicAdd(r.work, 1u);
        if (next.x < r.kend) {
            next.y = __ldg(r.order + next.x);
            const int2 pp = a.pos[next.y];
            next.z = pp.x;
            next.w = pp.y;
        }
    }
    __syncthreads();
    const uint32_t bar_g_u = smem_u32(&bar_g), buf_u = smem_u32(buf);
    uint32_t ph = 0;

#pragma unroll 1
    for (;;) {
        if (t == 0) mbar_arrive_expect_tx(&bar_g, (uint32_t)(L * M * sizeof(float2)));
        if (leader) {
#pragma unroll
            for (int s = 0; s < Q; ++s) {
                const uint32_t base = mapa_u32(smem_u32(&s_item), s);
                st_cluster_u32(base, (unsigned)next.x);
                st_cluster_u32(base + 4, (unsigned)next.y);
                st_cluster_u32(base + 8, (unsigned)next.z);
                st_cluster_u32(base + 12, (unsigned)next.w);
            }
            next.x = r.kbeg + (int)atomicAdd(r.work, 1u);
        }
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        const int4 it = s_item;
        const int k = it.x;
        if (k >= r.kend) break;
        const int j = it.y;
        const int2 pj = make_int2(it.z, it.w);

        if (t < 32) {
            const float* src = amp_perm + (size_t)j * M * M + (size_t)q * L * M;
            if (t == 0) mbar_arrive_expect_tx(&bar_a, L * M * sizeof(float));
            __syncwarp();
            for (int r2 = t; r2 < L; r2 += 32)
                tma_bulk_g2s(amp_s + r2 * AP, src + (size_t)r2 * M, M * sizeof(float), &bar_a);
        }

        // gather + column DIF butterflies: butterfly rows 2h, 2h + 1 of column c
        {
            const float2* zc = a.z + (size_t)pj.x * n + pj.y + c;
#pragma unroll 1
            for (int bb = 0; bb < 2; ++bb) {
                const int rw = q * NPC + 2 * h + bb;
                float2 v[Q];
                const float2* zp = zc + (size_t)rw * n;
                const float2* pp = a.probe + (size_t)rw * M + c;
#pragma unroll
                for (int s = 0; s < Q; ++s) {
                    const float2 zz = zp[(size_t)s * L * n];
                    v[s] = PROBE ? cmul(__ldg(pp + (size_t)s * L * M), zz) : zz;
                }
                dft_q<Q>(v);
#pragma unroll
                for (int s = 1; s < Q; ++s) v[s] = cmul(tw[rw * s], v[s]);
#pragma unroll
                for (int s = 0; s < Q; ++s)
                    st_async_f2(mapa_u32(smem_u32(buf + rw * PM + c), s), v[s], mapa_u32(bar_g_u, s));
            }
        }
        if (leader && next.x < r.kend) next.y = __ldg(r.order + next.x);
        mbar_wait(&bar_g, ph);

        float2 y[16];
        // pass 0: column c (local rows), forward, halves to rows 2j + h
        dft32_half(h, [&](int kk) { return buf[kk * PM + c]; }, y);
        __syncthreads();
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) buf[(2 * jj + h) * PM + c] = y[jj];
        __syncthreads();
        // row DIF butterflies: element m of the 8 parts of rows g, g + 16
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            float2* row = buf + (g + 16 * i) * PM + m;
            float2 v[Q];
#pragma unroll
            for (int s = 0; s < Q; ++s) v[s] = row[L * s];
            dft_q<Q>(v);
#pragma unroll
            for (int s = 1; s < Q; ++s) v[s] = cmul(tw[m * s], v[s]);
#pragma unroll
            for (int s = 0; s < Q; ++s) row[L * s] = v[s];
        }
        __syncthreads();
        // pass 1: part qq of row rr, forward; spectral operator at
        // (kr, kc) = (Q rr + q, Q (2 jj + h) + qq); y <- conj(R)
        dft32_half(h, [&](int kk) { return buf[rr * PM + qq * L + kk]; }, y);
        double acc;
        {
            float af[4] = {0.f, 0.f, 0.f, 0.f};
            mbar_wait(&bar_a, ph);
            const float* As = amp_s + rr * AP + qq * L + h * 16;
#pragma unroll
            for (int cc = 0; cc < 16; cc += 4) {
                const float4 A4 = *reinterpret_cast<const float4*>(As + cc);
                const float Av[4] = {A4.x, A4.y, A4.z, A4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float2 W = y[cc + u];
                    const float Am = Av[u];
                    float2 R;
                    if constexpr (OP == OP_INTENSITY) {
                        const float rs = (W.x * W.x + W.y * W.y) - Am;
                        af[u] = fmaf(rs, rs, af[u]);
                        R = make_float2(W.x * rs, W.y * rs);
                    } else {
                        const float m2 = fmaf(W.x, W.x, W.y * W.y);
                        const bool nz = m2 >= 1.17549435e-38f;
                        const float inv = nz ? rsqrt_ftz(m2) : 0.f;
                        const float dl = fmaf(m2, inv, -Am);
                        af[u] = fmaf(dl, dl, af[u]);
                        const float sv = fmaf(-Am, inv, 1.f);
                        R = make_float2(fmaf(W.x, sv, nz ? 0.f : -Am), W.y * sv);
                    }
                    y[cc + u] = make_float2(R.x, -R.y);
                }
            }
            acc = ((double)af[0] + (double)af[1]) + ((double)af[2] + (double)af[3]);
        }
        if (leader && next.x < r.kend) {
            const int2 pp = a.pos[next.y];
            next.z = pp.x;
            next.w = pp.y;
        }
        __syncthreads();   // the other half of this part may still be reading it
        // pass 2: DIT -- DFT_16 of this half; E (h = 0) / W32^n O (h = 1) into the part
        reg_fft<16, false>(y);
        if (h) {
            static_for<16>([&](auto nc) {
                constexpr int mm = decltype(nc)::value;
                y[mm] = twiddle_mul<32, false, mm>(y[mm]);
            });
        }
#pragma unroll
        for (int cc = 0; cc < 16; cc += 2)
            *reinterpret_cast<float4*>(&buf[rr * PM + qq * L + h * 16 + cc]) =
                make_float4(y[cc].x, y[cc].y, y[cc + 1].x, y[cc + 1].y);
        __syncthreads();
        // row DIT combine: Y_s[m] = E_s[m'] +- (W32^m' O_s)[m'], then the radix-8 combine
        {
            const int m16 = m & 15;
            const bool lo = m < 16;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                float2* row = buf + (g + 16 * i) * PM;
                float2 v[Q];
#pragma unroll
                for (int s = 0; s < Q; ++s) {
                    const float2 e = row[L * s + m16], o = row[L * s + 16 + m16];
                    v[s] = lo ? cadd(e, o) : csub(e, o);
                }
                __syncwarp();   // lanes m and m + 16 read each other's slots
#pragma unroll
                for (int s = 1; s < Q; ++s) v[s] = cmul(tw[m * s], v[s]);
                dft_q<Q>(v);
#pragma unroll
                for (int s = 0; s < Q; ++s) row[L * s + m] = v[s];
            }
        }
        __syncthreads();
        // pass 3: column c (local rows), forward; frequency 2 jj + h goes to CTA
        // (2 jj + h) / NPC, row ((2 jj + h) % NPC) Q + q
        dft32_half(h, [&](int kk) { return buf[kk * PM + c]; }, y);
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
            const int kf = 2 * jj + h;
            st_cluster_f2(mapa_u32(buf_u + (uint32_t)((((kf % NPC) * Q + q) * PM + c) * sizeof(float2)), kf / NPC),
                          y[jj]);
        }
        // epilogue probe values conj(sc P) for output rows q NPC + i + L s, i = 2h, 2h + 1
        float2 pe[2 * Q];
        if constexpr (PROBE) {
#pragma unroll
            for (int bb = 0; bb < 2; ++bb)
#pragma unroll
                for (int s = 0; s < Q; ++s)
                    pe[bb * Q + s] = __ldg(probe_epi + (size_t)(q * NPC + 2 * h + bb + L * s) * M + c);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((t & 31) == 0) red[t / 32] = acc;
        cl.sync();   // every push has landed
        if (t == 0) {
            double sm = 0.0;
#pragma unroll
            for (int i = 0; i < NT / 32; ++i) sm += red[i];
            a.misfit[(size_t)j * Q + q] = (OP == OP_DISTANCE) ? sm / (2.0 * (double)M * (double)M) : 0.5 * sm;
        }
        // (A) contributions in place, output rows i = 2h, 2h + 1 of column c
        const float sc = (OP == OP_DISTANCE) ? 1.f / (float(M) * float(M)) : 2.f;
#pragma unroll
        for (int bb = 0; bb < 2; ++bb) {
            const int i = 2 * h + bb, rw = q * NPC + i;
            float2 v[Q];
#pragma unroll
            for (int s = 0; s < Q; ++s) v[s] = buf[(i * Q + s) * PM + c];
#pragma unroll
            for (int s = 1; s < Q; ++s) v[s] = cmul(tw[rw * s], v[s]);
            dft_q<Q>(v);
#pragma unroll
            for (int s = 0; s < Q; ++s)
                buf[(i * Q + s) * PM + c] = PROBE ? epi_contrib_pre(v[s], pe[bb * Q + s]) : epi_contrib(v[s], sc);
        }
        // (B) earlier overlapping frames done
        {
            const int d0 = __ldg(r.dep_off + k), d1 = __ldg(r.dep_off + k + 1);
            for (int d = d0 + t; d < d1; d += NT) {
                const unsigned* f = r.done + __ldg(r.dep_idx + d);
                while (ld_acquire_gpu(f) < (unsigned)Q) __nanosleep(64);
            }
        }
        __syncthreads();
        // (C) read-modify-write of the CTA's 32 object rows (one batch of 8 pixel pairs / thread)
        float2* G0 = r.grad + (size_t)pj.x * n + pj.y;
        if ((pj.y & 1) == 0) {
            constexpr int HW = M / 2, PER = L * HW / NT;
            float4 gv[PER];
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int e = t + NT * u, row = e / HW, c2 = e % HW;
                const int orow = q * NPC + row / Q + L * (row % Q);
                gv[u] = __ldcg(reinterpret_cast<const float4*>(G0 + (size_t)orow * n + 2 * c2));
            }
#pragma unroll
            for (int u = 0; u < PER; ++u) {
                const int e = t + NT * u, row = e / HW, c2 = e % HW;
                const int orow = q * NPC + row / Q + L * (row % Q);
                const float4 cv = *reinterpret_cast<const float4*>(&buf[row * PM + 2 * c2]);
                __stcg(reinterpret_cast<float4*>(G0 + (size_t)orow * n + 2 * c2), f4add(gv[u], cv));
            }
        } else {
            constexpr int PER = L * M / NT, HALF = PER / 2;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                float2 gv[HALF];
#pragma unroll
                for (int u = 0; u < HALF; ++u) {
                    const int e = t + NT * (hh * HALF + u), row = e / M, cc = e % M;
                    const int orow = q * NPC + row / Q + L * (row % Q);
                    gv[u] = __ldcg(G0 + (size_t)orow * n + cc);
                }
#pragma unroll
                for (int u = 0; u < HALF; ++u) {
                    const int e = t + NT * (hh * HALF + u), row = e / M, cc = e % M;
                    const int orow = q * NPC + row / Q + L * (row % Q);
                    __stcg(G0 + (size_t)orow * n + cc, cadd(gv[u], buf[row * PM + cc]));
                }
            }
        }
        __syncthreads();
        if (t == 0) red_release_gpu_add(r.done + k, 1u);
        ph ^= 1u;
    }
}

// [j][q][r][p][h][j'] = A_j[8 r + q][8 (2 j' + h) + p]: the split order of frame_rmw2_kernel
__global__ void k_perm_amp_split(const float* __restrict__ in, float* __restrict__ out, size_t total) {
    constexpr int Q = 8, L = 32, M = 256;
    for (size_t o = blockIdx.x * (size_t)blockDim.x + threadIdx.x; o < total; o += (size_t)gridDim.x * blockDim.x) {
        const size_t jj = o / ((size_t)M * M);
        const int rem = (int)(o % ((size_t)M * M));
        const int j1 = rem % 16, hh = (rem / 16) % 2, p = (rem / L) % Q, r = (rem / M) % L, q = rem / (L * M);
        out[o] = in[jj * M * M + (size_t)(Q * r + q) * M + Q * (2 * j1 + hh) + p];
    }
}

}  // namespace ptg
