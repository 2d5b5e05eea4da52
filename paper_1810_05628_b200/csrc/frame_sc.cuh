// frame_sc.cuh — M = 128 complex64 frames, one persistent CTA per SM: the
// frame_rmw_kernel<4, 32> computation with the cluster of four 128-thread CTAs
// fused into ONE 512-thread CTA.
//
// A 128 x 128 complex64 frame is 128 KiB: unlike the 512 KiB frames of M = 256
// it fits one SM's shared memory.  The cluster kernels still split it over
// four CTAs (frame_cl.cuh), and at this size a frame's time is set by the
// fixed costs of that split, not by its arithmetic: three cluster-wide
// barriers, remote stores at the DSMEM port rate (~20 B/clk per SM against
// 128 B/clk for local shared memory) and mbarrier hand-offs per frame — a
// 128^2 frame took as long as a 256^2 one (25.6 vs 21.6 us per frame per
// cluster).  Here the four "virtual CTAs" (thread groups of 128, q = tid / 128)
// keep frame_rmw_kernel's work split, data layout and arithmetic — same
// butterflies, twiddles and summation order, so results are bit-identical to
// the cluster kernel's — but live in one CTA:
//   * every remote store is a plain shared-memory store into the owner
//     group's slice, every cluster barrier / mbarrier wait a __syncthreads();
//   * the probe rows (32 values per thread) and the NEXT frame's object window
//     sit in tensor memory (tcgen05.st / tcgen05.ld as thread-private storage,
//     no MMA; 16 warps x 64 columns x 2 blocks = the SM's 512 columns), so a
//     frame's gather touches no global memory;
//   * the gradient update is a TMA bulk reduce-add per object row in the
//     plan's dependency order (frame_rmw.cuh: done counters, one release per
//     frame worth Q arrivals, so both kernels speak the same protocol).
// Positions come from the RMW order through an atomic counter, claimed a
// frame ahead by thread 0.
//
// MEASURED AND NOT ADOPTED (PTG_SC=1 selects it; parity tests keep it green).
// Config 5's level 1 (27,556 frames of 128^2), ms per evaluation: fused 5.36,
// four-CTA cluster RMW 4.57, stash + gather 4.38 (default); with colour groups
// of two window heights (PTG_RMW_SB=256: 148 frames in flight need more
// frames per colour class) 4.33 / 4.10.  One frame per SM takes 22.8 us here
// and 21.6 us per pair of co-resident M = 256 frames: both run 16 warps per SM
// through the same ~3,650 instructions per warp and frame at ~36 % issue
// utilisation.  The frame kernels are bound by that per-warp latency chain
// (register FFT_32 passes between shared-memory exchanges at 4 warps per
// scheduler), not by the cluster barriers or the DSMEM port.
#pragma once

#include "frame_rmw.cuh"

namespace ptg {

constexpr int kScQ = 4, kScL = 32, kScM = kScQ * kScL, kScThreads = kScQ * kScM;
__host__ __device__ constexpr size_t sc_smem_bytes() {
    return sizeof(float2) * ((size_t)kScQ * kScL * cl_pitch<kScQ, kScL>() + kScM) +
           sizeof(float) * (size_t)kScQ * kScL * cl_amp_pitch<kScQ, kScL>();
}

template <int OP, bool PROBE, bool TM>
__global__ void __launch_bounds__(kScThreads, 1)
    frame_sc_kernel(FrameArgs<float> a, const float* __restrict__ amp_perm, const float2* __restrict__ tw_g,
                    const float2* __restrict__ probe_epi, RmwArgs r) {
    constexpr int Q = kScQ, L = kScL, M = kScM, NT = M, PM = cl_pitch<Q, L>(), NPC = L / Q, AP = cl_amp_pitch<Q, L>();
    constexpr int SL = L * PM;   // one group's frame slice (complex elements)
    static_assert(!TM || PROBE, "tensor-memory cache: probe frames");
    extern __shared__ __align__(16) unsigned char sc_smem[];
    float2* buf_all = reinterpret_cast<float2*>(sc_smem);      // [Q][L][PM]
    float2* tw = buf_all + Q * SL;                             // W_M^i, i < M
    float* amp_all = reinterpret_cast<float*>(tw + M);         // [Q][L][AP]
    __shared__ double red[kScThreads / 32];
    __shared__ __align__(8) unsigned long long bar_a;
    __shared__ int4 s_item[2];   // [ph] this frame, [ph ^ 1] the next one
    __shared__ uint32_t s_tmem;

    const int T = threadIdx.x;
    const int q = T >> 7;        // virtual CTA (frame_rmw_kernel's cluster rank)
    const int t = T & (NT - 1);  // its thread index
    const int n = a.n;
    float2* buf = buf_all + q * SL;
    float* amp_s = amp_all + q * L * AP;
    if (T == 0) {
        mbar_init(&bar_a, 1);
        fence_mbarrier_init();
    }
    for (int i = T; i < M; i += kScThreads) tw[i] = __ldg(tw_g + i);
    uint32_t tm = 0;
    constexpr unsigned TCOLS = 512u;   // probe block [0, 256), object-window block [256, 512)
    if constexpr (TM) {
        if (T < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                         "r"(TCOLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int wp = T >> 5;
        tm = s_tmem + ((uint32_t)((wp & 3) * 32) << 16) + (uint32_t)((wp >> 2) * 64);
#pragma unroll
        for (int b = 0; b < NPC; ++b) {
            float2 pv[Q];
#pragma unroll
            for (int s = 0; s < Q; ++s) pv[s] = __ldg(a.probe + (size_t)(q * NPC + b + L * s) * M + t);
            tmem_st_f2<Q>(tm + 2 * Q * b, pv);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    const uint32_t tmz = tm + 256u;
    // thread 0 claims frames a frame ahead: order index, position index and
    // window are three dependent L2 round trips, spread over a frame's phases
    const bool leader = T == 0;
    int4 next = make_int4(0, 0, 0, 0);
    if (leader) {
        next.x = r.kbeg + (int)atomicAdd(r.work, 1u);
        if (next.x < r.kend) {
            next.y = __ldg(r.order + next.x);
            const int2 pp = a.pos[next.y];
            next.z = pp.x;
            next.w = pp.y;
        }
        s_item[0] = next;
        next.x = r.kbeg + (int)atomicAdd(r.work, 1u);
    }
    __syncthreads();
    const int m = t % L, g = t / L;
    const int rr = t % L, qq = t / L;
    uint32_t ph = 0;
    // window (wr, wc) rows q NPC + b + L s, column t -> zv[b Q + s] (pinned loads)
    auto zpref_issue = [&](int wr, int wc, float2* zv) {
        const float2* zc = a.z + (size_t)wr * n + wc + t;
        const size_t zstep = (size_t)L * n;
#pragma unroll
        for (int b = 0; b < NPC; ++b) {
            const float2* zp = zc + (size_t)(q * NPC + b) * n;
#pragma unroll
            for (int s = 0; s < Q; ++s) {
                zv[b * Q + s] = ldg_pinned(zp);
                zp += zstep;
            }
        }
    };
    auto zpref_store = [&](const float2* zv) {
#pragma unroll
        for (int b = 0; b < NPC; ++b) tmem_st_f2<Q>(tmz + 2 * Q * b, zv + b * Q);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    };
    if constexpr (TM) {
        const int4 it0 = s_item[0];
        if (it0.x < r.kend) {
            float2 zv[L];
            zpref_issue(it0.z, it0.w, zv);
            zpref_store(zv);
        }
    }

#pragma unroll 1
    for (;;) {
        const int4 it = s_item[ph];
        const int k = it.x;
        if (k >= r.kend) break;
        const int j = it.y;
        const int2 pj = make_int2(it.z, it.w);

        if (T < 32) {   // the frame's Q L permuted amplitude rows, one bulk copy per row
            const float* src = amp_perm + (size_t)j * M * M;
            fence_proxy_async_smem();   // the previous frame's reads of these rows precede the async writes
            if (T == 0) mbar_arrive_expect_tx(&bar_a, Q * L * M * sizeof(float));
            __syncwarp();
            for (int r2 = T; r2 < Q * L; r2 += 32)
                tma_bulk_g2s(amp_all + (r2 / L) * (L * AP) + (r2 % L) * AP, src + (size_t)r2 * M, M * sizeof(float),
                             &bar_a);
        }

        // gather fused with the column DIF butterflies: group q's NPC
        // butterfly rows, outputs into the owner groups' slices
        float2 x[L];
#pragma unroll
        for (int b = 0; b < NPC; ++b) {
            const int rw = q * NPC + b;
            float2 v[Q];
            if constexpr (TM) {
                float2 pv[Q];
                tmem_ld_f2<Q>(tmz + 2 * Q * b, v);
                tmem_ld_f2<Q>(tm + 2 * Q * b, pv);
#pragma unroll
                for (int s = 0; s < Q; ++s) v[s] = cmul(pv[s], v[s]);
            } else {
                const float2* zp = a.z + (size_t)(pj.x + rw) * n + pj.y + t;
#pragma unroll
                for (int s = 0; s < Q; ++s) {
                    const float2 zz = __ldg(zp + (size_t)(L * s) * n);
                    if constexpr (PROBE) v[s] = cmul(__ldg(a.probe + (size_t)(rw + L * s) * M + t), zz);
                    else v[s] = zz;
                }
            }
            dft_q<Q>(v);
#pragma unroll
            for (int s = 1; s < Q; ++s) v[s] = cmul(tw[rw * s], v[s]);
#pragma unroll
            for (int s = 0; s < Q; ++s) buf_all[s * SL + rw * PM + t] = v[s];
        }
        if (leader && next.x < r.kend) next.y = __ldg(r.order + next.x);
        __syncthreads();   // every group's rows have landed

        double acc = 0.0;
PTG_UNROLL_N(PTG_RMW_PASS_UNROLL)
        for (int pass = 0; pass < 4; ++pass) {
            if (pass == 0 || pass == 3) {
#pragma unroll
                for (int kk = 0; kk < L; ++kk) x[kk] = buf[kk * PM + t];
                if (pass == 3) {
                    // the next frame's item for every thread, and every group's
                    // reads of its slice before the pushes below
                    if (leader) {
                        s_item[ph ^ 1u] = next;
                        next.x = r.kbeg + (int)atomicAdd(r.work, 1u);   // the frame after it, claimed ahead
                    }
                    __syncthreads();
                }
            } else if (pass == 1) {
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
                for (int kk = 0; kk < L; ++kk) buf[kk * PM + t] = x[kk];
                __syncthreads();
#pragma unroll 2
                for (int i = 0; i < NPC; ++i) {
                    float2* row = buf + (g + Q * i) * PM + m;
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
            } else if (pass == 1) {
                float af[4] = {0.f, 0.f, 0.f, 0.f};
                mbar_wait(&bar_a, ph);
#pragma unroll
                for (int c = 0; c < L; c += 4) {
                    const float4 A4 = *reinterpret_cast<const float4*>(amp_s + rr * AP + qq * L + c);
                    const float Av[4] = {A4.x, A4.y, A4.z, A4.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float2 W = x[c + u];
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
                            const float s = fmaf(-Am, inv, 1.f);
                            R = make_float2(fmaf(W.x, s, nz ? 0.f : -Am), W.y * s);
                        }
                        x[c + u] = make_float2(R.x, -R.y);
                    }
                }
                acc = ((double)af[0] + (double)af[1]) + ((double)af[2] + (double)af[3]);
                if (leader && next.x < r.kend) {
                    const int2 pp = a.pos[next.y];
                    next.z = pp.x;
                    next.w = pp.y;
                }
            } else if (pass == 2) {
#pragma unroll
                for (int c = 0; c < L; c += 2)
                    *reinterpret_cast<float4*>(&buf[rr * PM + qq * L + c]) =
                        make_float4(x[c].x, x[c].y, x[c + 1].x, x[c + 1].y);
                __syncthreads();
#pragma unroll 2
                for (int i = 0; i < NPC; ++i) {
                    float2* row = buf + (g + Q * i) * PM + m;
                    float2 v[Q];
#pragma unroll
                    for (int s = 0; s < Q; ++s) v[s] = row[L * s];
#pragma unroll
                    for (int s = 1; s < Q; ++s) v[s] = cmul(tw[m * s], v[s]);
                    dft_q<Q>(v);
#pragma unroll
                    for (int s = 0; s < Q; ++s) row[L * s] = v[s];
                }
                __syncthreads();
            } else {
#pragma unroll
                for (int kk = 0; kk < L; ++kk)   // row (kk % NPC) Q + q of group kk / NPC
                    buf_all[(kk / NPC) * SL + ((kk % NPC) * Q + q) * PM + t] = x[kk];
            }
        }
        if constexpr (TM) {
            const float scp = (OP == OP_DISTANCE) ? 1.f / (float(M) * float(M)) : 2.f;
#pragma unroll
            for (int i = 0; i < NPC; ++i) {
                float2 pv[Q];
                tmem_ld_f2<Q>(tm + 2 * Q * i, pv);
#pragma unroll
                for (int s = 0; s < Q; ++s) x[i * Q + s] = make_float2(pv[s].x * scp, -(pv[s].y * scp));
            }
        } else if constexpr (PROBE) {
#pragma unroll
            for (int i = 0; i < NPC; ++i)
#pragma unroll
                for (int s = 0; s < Q; ++s) x[i * Q + s] = __ldg(probe_epi + (size_t)(q * NPC + i + L * s) * M + t);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((T & 31) == 0) red[T >> 5] = acc;
        __syncthreads();   // every push has landed
        if (t == 0) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < NT / 32; ++i) s += red[q * (NT / 32) + i];
            constexpr int MPP = cl_mpp(Q, M);
            a.misfit[(size_t)j * MPP + q] = (OP == OP_DISTANCE) ? s / (2.0 * (double)M * (double)M) : 0.5 * s;
            if constexpr (MPP > Q) a.misfit[(size_t)j * MPP + Q + q] = 0.0;
        }

        // (A) contributions, in place: slice row i Q + s holds object row
        //     pj.x + q NPC + i + L s (columns pj.y .. pj.y + M), column t
        const float sc = (OP == OP_DISTANCE) ? 1.f / (float(M) * float(M)) : 2.f;
#pragma unroll
        for (int i = 0; i < NPC; ++i) {
            const int rw = q * NPC + i;
            float2 v[Q];
#pragma unroll
            for (int s = 0; s < Q; ++s) v[s] = buf[(i * Q + s) * PM + t];
#pragma unroll
            for (int s = 1; s < Q; ++s) v[s] = cmul(tw[rw * s], v[s]);
            dft_q<Q>(v);
#pragma unroll
            for (int s = 0; s < Q; ++s)
                buf[(i * Q + s) * PM + t] = PROBE ? epi_contrib_pre(v[s], x[i * Q + s]) : epi_contrib(v[s], sc);
        }
        // the next frame's object window, in flight across (B) and (C)
        int4 nx = make_int4(0, 0, 0, 0);
        if constexpr (TM) {
            nx = s_item[ph ^ 1u];
            if (nx.x < r.kend) zpref_issue(nx.z, nx.w, x);
        }
        // (B) every earlier overlapping frame has finished its update
        {
            const int d0 = __ldg(r.dep_off + k), d1 = __ldg(r.dep_off + k + 1);
            for (int d = d0 + T; d < d1; d += kScThreads) {
                const unsigned* f = r.done + __ldg(r.dep_idx + d);
                while (ld_acquire_gpu(f) < (unsigned)Q) __nanosleep(64);
            }
        }
        __syncthreads();
        // (C) the frame's M object rows: TMA bulk reduce-adds (16-byte aligned
        //     windows), else coalesced load + add + store
        float2* G0 = r.grad + (size_t)pj.x * n + pj.y;
        if ((pj.y & 1) == 0) {
            if (T < Q * L) {
                fence_proxy_async_smem();
                const int vq = T / L, row = T % L, orow = vq * NPC + row / Q + L * (row % Q);
                asm volatile(
                    "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                        G0 + (size_t)orow * n),
                    "r"(smem_u32(buf_all + vq * SL + row * PM)), "r"((uint32_t)(M * sizeof(float2)))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            }
        } else {
            constexpr int PER = L * M / NT, HALF = PER / 4;   // four batches of float2 per thread
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                float2 gv[HALF];
#pragma unroll
                for (int u = 0; u < HALF; ++u) {
                    const int e = t + NT * (h * HALF + u), row = e / M, c = e % M;
                    const int orow = q * NPC + row / Q + L * (row % Q);
                    gv[u] = __ldcg(G0 + (size_t)orow * n + c);
                }
#pragma unroll
                for (int u = 0; u < HALF; ++u) {
                    const int e = t + NT * (h * HALF + u), row = e / M, c = e % M;
                    const int orow = q * NPC + row / Q + L * (row % Q);
                    __stcg(G0 + (size_t)orow * n + c, cadd(gv[u], buf[row * PM + c]));
                }
            }
        }
        if constexpr (TM) {
            if (nx.x < r.kend) zpref_store(x);
        }
        // (D) publish: the frame's rows are final (Q arrivals: the cluster kernels' count)
        __syncthreads();
        if (T == 0) red_release_gpu_add(r.done + k, (unsigned)Q);
        ph ^= 1u;
    }
    if constexpr (TM) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (T < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(TCOLS) : "memory");
    }
}

}  // namespace ptg
