// frame_rmw.cuh — persistent cluster frame kernel with an in-place,
// dependency-ordered overlap-add (complex64, M = Q L = 128 / 256, w == M).
//
// The per-frame computation is frame_cl_kernel's (frame_cl.cuh: gather fused
// with the column DIF butterflies over distributed shared memory, register
// FFT_L passes, spectral operator + fp64 misfit, inverse passes, conj(P)
// epilogue; reference objectives.cpp:59-103).  What changes is where the
// contribution goes.  frame_cl_kernel stores every frame's M x M contribution
// (512 KiB at M = 256) to a per-position stash in HBM and a separate gather
// sums the stashes: 2 x 14.4 GB of HBM traffic per config-5 evaluation on top
// of the 8.3 GB the evaluation needs.  Here the frame adds its contribution
// straight into the gradient:
//
//   * the plan orders the positions (host, plan.cu build_rmw): groups of
//     consecutive window rows, inside a group greedy colour classes of
//     pairwise non-overlapping windows, class by class.  That order is the
//     summation order of every pixel -- fixed by the geometry, so results are
//     bitwise reproducible run to run (no unordered float atomics: a pixel
//     is updated by one frame at a time -- a TMA bulk reduce-add of the
//     frame's object row, or a plain load + add + store for windows that
//     start on an odd column);
//   * frame k may update the gradient only after every EARLIER overlapping
//     frame has finished its update: a per-frame completion counter (one
//     release-increment per CTA, CUTLASS GenericBarrier style) that the
//     CTAs of frame k acquire before their read-modify-write.  Overlapping
//     frames are >= one colour class apart in the order (~25 frames for
//     config 5), so the wait almost never blocks;
//   * frames are handed out by an atomic counter (persistent grid of
//     co-resident clusters; a frame is only ever waited on after a running
//     cluster claimed it, so the protocol cannot deadlock), and the gradient
//     rows being updated (window height x object width) stay L2-resident as
//     the scan advances: HBM sees the amplitudes, the object and the
//     gradient about once.
//
// The gradient is initialised (= -v for the MG/OPT shift, else 0) and the
// counters zeroed by k_rmw_init before the launch; k_finalize forms the value.
#pragma once

#include "frame_cl.cuh"

namespace ptg {

struct RmwArgs {
    const int* order;     // [N] dispatch / summation order -> position index
    const int* dep_off;   // [N + 1] CSR offsets over order indices
    const int* dep_idx;   // order indices of the earlier overlapping frames
    unsigned* done;       // [N] per order index: CTAs finished (Q = complete), zeroed per evaluation
    unsigned* work;       // dispatch counter, zeroed per evaluation
    float2* grad;         // gradient, row pitch a.n
    int kbeg, kend;       // this launch's frames: order indices [kbeg, kend) (earlier ones are complete)
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// read-only 32-bit load pinned in program order (see ldg_pinned)
__device__ __forceinline__ int ldg_pinned_i32(const int* p) {
    int v;
    asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, unsigned v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_f2(uint32_t addr, float2 v) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
    const float2 lo = cadd(make_float2(a.x, a.y), make_float2(b.x, b.y));
    const float2 hi = cadd(make_float2(a.z, a.w), make_float2(b.z, b.w));
    return make_float4(lo.x, lo.y, hi.x, hi.y);
}

// PTG_RMW_BULK: the gradient update of 16-byte-aligned windows as TMA bulk
// reduce-adds (cp.reduce.async.bulk .add.f32, one 2 KiB object row per copy,
// shared memory -> L2): the gradient rows are not read into the SM at all.
// Still one add per pixel per frame, in the dependency order, so every pixel's
// summation order is fixed.  Config 5 (ms per evaluation): 0 = load + add +
// store 22.33; 1 = bulk, completion awaited before the publish 21.64
// (default); 2 = completion awaited a gather later 22.14.
#ifndef PTG_RMW_BULK
#define PTG_RMW_BULK 1
#endif
// PTG_RMW_PUSHBAR=1: the inverse pushes as st.async completing transaction
// bytes on the owner's mbarrier (like the gather), so the owner waits for its
// own 64 KiB instead of a third cluster-wide barrier per frame
#ifndef PTG_RMW_PUSHBAR
#define PTG_RMW_PUSHBAR 0
#endif

// TM = true (M = 256 probe frames, PTG_RMW_TMEM=0 turns it off at run time):
// the probe rows of this CTA (the same 32 rows every frame, 32 values per
// thread) are kept in tensor memory -- otherwise idle on this path -- and read
// back with tcgen05.ld for the gather's probe multiply and the conj(P)
// epilogue, instead of two 512 KiB L2 reads per frame.  TMEM is used purely as
// thread-private storage (32x32b: lane = thread, 64 columns per warp, 128
// columns per CTA, two CTAs per SM), no MMA.  conj(sc P) is formed from P on
// the fly (sc a power of two: exact, the probe_epi table's bits).  Config 5:
// 21.66 -> 20.61 ms per evaluation.  cudaOccupancyMaxActiveClusters reports
// 15 instead of 33 clusters for a kernel that allocates tensor memory, so the
// grid is sized with the TM = false instantiation (same registers and shared
// memory); 33 clusters are co-resident (tools/tmem_probe.cu: two CTAs of one
// SM hold their allocations at once), and the dispatch protocol does not
// depend on co-residency anyway.

// 2 W 32-bit TMEM columns <-> W float2 registers of this thread (W = 4 | 8);
// the load includes its wait so the outputs are valid after the statement
template <int W>
__device__ __forceinline__ void tmem_st_f2(uint32_t taddr, const float2* v) {
    static_assert(W == 4 || W == 8, "tmem_st_f2: 4 or 8 values");
    if constexpr (W == 8) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16};" ::"r"(taddr),
            "f"(v[0].x), "f"(v[0].y), "f"(v[1].x), "f"(v[1].y), "f"(v[2].x), "f"(v[2].y), "f"(v[3].x), "f"(v[3].y),
            "f"(v[4].x), "f"(v[4].y), "f"(v[5].x), "f"(v[5].y), "f"(v[6].x), "f"(v[6].y), "f"(v[7].x), "f"(v[7].y)
            : "memory");
    } else {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                     "f"(v[0].x), "f"(v[0].y), "f"(v[1].x), "f"(v[1].y), "f"(v[2].x), "f"(v[2].y), "f"(v[3].x),
                     "f"(v[3].y)
                     : "memory");
    }
}
template <int W>
__device__ __forceinline__ void tmem_ld_f2(uint32_t taddr, float2* v) {
    static_assert(W == 4 || W == 8, "tmem_ld_f2: 4 or 8 values");
    if constexpr (W == 8) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15}, [%16];\n\ttcgen05.wait::ld.sync.aligned;"
            : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[1].x), "=f"(v[1].y), "=f"(v[2].x), "=f"(v[2].y), "=f"(v[3].x),
              "=f"(v[3].y), "=f"(v[4].x), "=f"(v[4].y), "=f"(v[5].x), "=f"(v[5].y), "=f"(v[6].x), "=f"(v[6].y),
              "=f"(v[7].x), "=f"(v[7].y)
            : "r"(taddr)
            : "memory");
    } else {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n\t"
            "tcgen05.wait::ld.sync.aligned;"
            : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[1].x), "=f"(v[1].y), "=f"(v[2].x), "=f"(v[2].y), "=f"(v[3].x),
              "=f"(v[3].y)
            : "r"(taddr)
            : "memory");
    }
}

// two blocks in one statement, one wait (W = 8)
__device__ __forceinline__ void tmem_ld2_f2(uint32_t ta, float2* va, uint32_t tb, float2* vb) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%32];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
        "%29, %30, %31}, [%33];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=f"(va[0].x), "=f"(va[0].y), "=f"(va[1].x), "=f"(va[1].y), "=f"(va[2].x), "=f"(va[2].y), "=f"(va[3].x),
          "=f"(va[3].y), "=f"(va[4].x), "=f"(va[4].y), "=f"(va[5].x), "=f"(va[5].y), "=f"(va[6].x), "=f"(va[6].y),
          "=f"(va[7].x), "=f"(va[7].y), "=f"(vb[0].x), "=f"(vb[0].y), "=f"(vb[1].x), "=f"(vb[1].y), "=f"(vb[2].x),
          "=f"(vb[2].y), "=f"(vb[3].x), "=f"(vb[3].y), "=f"(vb[4].x), "=f"(vb[4].y), "=f"(vb[5].x), "=f"(vb[5].y),
          "=f"(vb[6].x), "=f"(vb[6].y), "=f"(vb[7].x), "=f"(vb[7].y)
        : "r"(ta), "r"(tb)
        : "memory");
}

// PTG_RMW_ZPREF (with TM, Q = 8): the NEXT frame's object window is fetched
// during this frame's gradient update (registers are free there, the loads
// overlap the dependency wait and the bulk reduce-adds) and parked in a second
// tensor-memory block, so the gather of a frame is tensor-memory reads only:
// no L2 round trip sits on the frame's critical path.  The item of frame k + 1
// is handed to the cluster during frame k (before the inverse pushes' barrier).
#ifndef PTG_RMW_ZPREF
#define PTG_RMW_ZPREF 1
#endif
// PTG_RMW_DFTQ_UNROLL (A/B): unroll factor of the row radix-Q loops in shared memory (NPC iterations)
#ifndef PTG_RMW_DFTQ_UNROLL
#define PTG_RMW_DFTQ_UNROLL 4
#endif
// PTG_RMW_PASS_UNROLL: 4 (default) = the four FFT_L passes unrolled (each pass
// specialised, loads of the next pass scheduled across the boundary: config 5
// 19.66 -> 18.84 ms, 3,576 -> 4,416 SASS instructions); 1 = one rolled loop
#ifndef PTG_RMW_PASS_UNROLL
#define PTG_RMW_PASS_UNROLL 4
#endif
// PTG_RMW_LATE_SIGNALS=1 (default, tensor-memory path; config 5 18.78 ->
// 18.29 ms): a .release arrival first waits for every outstanding memory
// operation of its thread, so a long-latency
// operation issued just before one stalls the whole cluster.  The leader's
// claim atomic moves behind the inverse pass's arrival, and the publish of
// frame k (red.release.gpu) behind the NEXT loop-top arrival: both L2 round
// trips then overlap the barrier instead of preceding it.
#ifndef PTG_RMW_LATE_SIGNALS
#define PTG_RMW_LATE_SIGNALS 1
#endif
// PTG_RMW_LATE_BULKWAIT=1 (default, with LATE; 18.47 -> 18.33 ms): before the loop-top arrival only
// the reduce-adds' shared-memory READS are awaited (the rows are free); their
// completion is awaited by warp 0 behind the arrival, just before the publish
#ifndef PTG_RMW_LATE_BULKWAIT
#define PTG_RMW_LATE_BULKWAIT 1
#endif
// PTG_RMW_EARLY_DEPS=1 (default, tensor-memory path; 18.37 -> 18.16 ms): the dependency check's three
// dependent L2 round trips (list bounds, first entry, completion counter)
// issued in stages through the frame -- bounds at the frame start, the entry
// behind the post-gather arrival, the acquire load before the contributions --
// so that (B) usually finds its answer already in a register
// PTG_RMW_STAGGER=1 (default; 18.16 -> 17.75 ms): odd cluster ranks push to
// owners 4..7 first, even ranks to owners 0..3 first, so the Q sources do not
// all address the same owner at once.  2 = rank q starts at owner q (a branch
// per rank): 18.12, no better than unstaggered.
#ifndef PTG_RMW_STAGGER
#define PTG_RMW_STAGGER 1
#endif
#ifndef PTG_RMW_EARLY_DEPS
#define PTG_RMW_EARLY_DEPS 1
#endif
// PTG_RMW_GATHER_PLAIN=1 (default, ZP path): the gather's pushes as plain
// st.shared::cluster stores closed by a cluster barrier instead of st.async
// with a complete_tx on the owner's mbarrier per store (64 K transaction
// updates per CTA and frame): 19.78 vs 20.09 ms on config 5 (0 = st.async)
#ifndef PTG_RMW_GATHER_PLAIN
#define PTG_RMW_GATHER_PLAIN 1
#endif

// PTG_ABL_NOROWSYNC (timing ablation only, wrong results): the four CTA-wide
// barriers of the row phases replaced by __syncwarp -- an upper bound on what
// warp-local row transforms could save
#ifdef PTG_ABL_NOROWSYNC
#define ROWSYNC() __syncwarp()
#else
#define ROWSYNC() __syncthreads()
#endif

#ifdef ABL_TIMELINE   // diagnostic build: per-frame phase stamps of the first 64 CTAs (tools/rmw_timeline.py)
constexpr int kRtlCtas = 64, kRtlFrames = 128, kRtlStamps = 12;
__device__ unsigned long long g_rmw_tl[kRtlCtas * kRtlFrames * kRtlStamps];
#define RTL(k)                                                                                   \
    do {                                                                                         \
        if (threadIdx.x == 0 && blockIdx.x < kRtlCtas && rtl_f < kRtlFrames) {                   \
            unsigned long long t_;                                                               \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
            g_rmw_tl[((size_t)blockIdx.x * kRtlFrames + rtl_f) * kRtlStamps + (k)] = t_;          \
        }                                                                                        \
    } while (0)
#else
#define RTL(k)
#endif

template <int Q, int L, int OP, bool PROBE, bool TM = false>
__global__ void __launch_bounds__(Q * L, cl_min_blocks<Q, L>())
    frame_rmw_kernel(FrameArgs<float> a, const float* __restrict__ amp_perm, const float2* __restrict__ tw_g,
                     const float2* __restrict__ probe_epi, RmwArgs r) {
    namespace cg = cooperative_groups;
    constexpr int M = Q * L, NT = M, PM = cl_pitch<Q, L>(), NPC = L / Q, AP = cl_amp_pitch<Q, L>();
    static_assert(cl_amp_staged<Q, L>(), "the persistent kernel stages amplitudes");
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char cl_smem[];
    float2* buf = reinterpret_cast<float2*>(cl_smem);   // [L][PM]: this CTA's frame rows
    float2* tw = buf + L * PM;                           // W_M^i, i < M
    float* amp_s = reinterpret_cast<float*>(tw + M);     // [L][AP]
    __shared__ double red[NT / 32];
    __shared__ __align__(8) unsigned long long bar_a, bar_g;
#if PTG_RMW_PUSHBAR
    __shared__ __align__(8) unsigned long long bar_p;
#endif
    // (order index k, position j, window row, window column) of a frame; ZP:
    // [ph] this frame, [ph ^ 1] the next one (written during this frame)
    __shared__ int4 s_item[2];
    constexpr bool ZP = TM && Q == 8 && PTG_RMW_ZPREF != 0;
    constexpr unsigned TCOLS = ZP ? 256u : 128u;

    const int q = (int)cl.block_rank();
    const int t = threadIdx.x;
    const int n = a.n;
    if (t == 0) {
        mbar_init(&bar_g, 1);
        mbar_init(&bar_a, 1);
#if PTG_RMW_PUSHBAR
        mbar_init(&bar_p, 1);
#endif
        fence_mbarrier_init();
    }
    for (int i = t; i < M; i += NT) tw[i] = __ldg(tw_g + i);
    // probe rows q NPC + b + L s, column t -> this thread's TMEM lane, columns
    // 2 Q b .. 2 Q b + 2 Q - 1 of its warp's 64-column block
    static_assert(!TM || (PROBE && NT <= 256), "tensor-memory probe cache: probe frames, <= 8 warps");
    __shared__ uint32_t s_tmem;
    uint32_t tm = 0;
    if constexpr (TM) {
        if (t < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                         "r"(TCOLS)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int wp = t >> 5;
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
    // Rank 0 (thread 0) claims the next frame one frame ahead and fetches its
    // position index and window: three dependent L2 round trips, spread over
    // the current frame's phases (claim at the loop top, index after the
    // gather, window after the spectral pass) so no warp waits on them; the
    // loop top hands all four values to every CTA.
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
    const int m = t % L, g = t / L;
    const int rr = t % L, qq = t / L;
    const uint32_t bar_g_u = smem_u32(&bar_g), buf_u = smem_u32(buf);
    uint32_t ph = 0;
    // item `next` -> slot `slot` of every CTA of the cluster (leader thread)
    auto hand_item = [&](int slot) {
#pragma unroll
        for (int s = 0; s < Q; ++s) {
            const uint32_t base = mapa_u32(smem_u32(&s_item[slot]), s);
            st_cluster_u32(base, (unsigned)next.x);
            st_cluster_u32(base + 4, (unsigned)next.y);
            st_cluster_u32(base + 8, (unsigned)next.z);
            st_cluster_u32(base + 12, (unsigned)next.w);
        }
    };
    // ZP: window (wr, wc) rows q NPC + b + L s, column t -> registers zv[b Q + s]
    // (pinned loads: issued here, consumed by zpref_store)
    const uint32_t tmz = tm + 128u;
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
    if constexpr (ZP) {
        // the first item to every CTA, its window into tensor memory
        if (leader) {
            hand_item(0);
            next.x = r.kbeg + (int)atomicAdd(r.work, 1u);
        }
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        const int4 it0 = s_item[0];
        if (it0.x < r.kend) {
            float2 zv[L];
            zpref_issue(it0.z, it0.w, zv);
            zpref_store(zv);
        }
    }
#if PTG_RMW_BULK == 2
    int pend_k = -1;   // warp 0: frame whose bulk reduce-adds are in flight (published once they complete)
    auto publish_pending = [&]() {
        if (t < 32 && pend_k >= 0) {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            __syncwarp();
            if (t == 0) red_release_gpu_add(r.done + pend_k, 1u);
            pend_k = -1;
        }
    };
#endif

#ifdef ABL_TIMELINE
    int rtl_f = 0;
#endif
    constexpr bool LATE = ZP && PTG_RMW_LATE_SIGNALS != 0 && PTG_RMW_BULK != 2;
    int pub_k = -1;   // LATE: frame whose rows are final but not yet published (thread 0)
#pragma unroll 1
    for (;;) {
        RTL(0);
        // this frame's gather bytes, then the item handed to every CTA of the
        // cluster; the full cluster barrier also orders every CTA's previous
        // epilogue (reads of its own rows) before the pushes of this frame
        if (t == 0 && !(ZP && PTG_RMW_GATHER_PLAIN)) mbar_arrive_expect_tx(&bar_g, (uint32_t)(L * M * sizeof(float2)));
#if PTG_RMW_PUSHBAR
        if (t == 0) mbar_arrive_expect_tx(&bar_p, (uint32_t)(L * M * sizeof(float2)));
#endif
        if constexpr (!ZP) {
            if (leader) {
                hand_item(0);
                next.x = r.kbeg + (int)atomicAdd(r.work, 1u);   // the following frame, claimed ahead
            }
        }
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        if constexpr (LATE) {
#if PTG_RMW_LATE_BULKWAIT
            if (t < 32 && pub_k >= 0) {
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // this lane's reduce-add has been performed
                __syncwarp();
                if (t == 0) red_release_gpu_add(r.done + pub_k, 1u);
            }
#else
            if (t == 0 && pub_k >= 0) red_release_gpu_add(r.done + pub_k, 1u);
#endif
        }
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        const int4 it = s_item[ZP ? ph : 0];
        const int k = it.x;
        if (k >= r.kend) break;
        RTL(1);
        const int j = it.y;
        const int2 pj = make_int2(it.z, it.w);
        constexpr bool EDEPS = ZP && PTG_RMW_EARLY_DEPS != 0 && PTG_RMW_GATHER_PLAIN != 0;
        int ed0 = 0, ed1 = 0, edep = -1;
        unsigned edone = (unsigned)Q;
        if constexpr (EDEPS) {
            ed0 = ldg_pinned_i32(r.dep_off + k);
            ed1 = ldg_pinned_i32(r.dep_off + k + 1);
        }

        if (t < 32) {   // this CTA's L permuted amplitude rows, one bulk copy per row
            const float* src = amp_perm + (size_t)j * M * M + (size_t)q * L * M;
            if (t == 0) mbar_arrive_expect_tx(&bar_a, L * M * sizeof(float));
            __syncwarp();
            for (int r2 = t; r2 < L; r2 += 32)
                tma_bulk_g2s(amp_s + r2 * AP, src + (size_t)r2 * M, M * sizeof(float), &bar_a);
        }

        // gather fused with the column DIF butterflies (frame_cl.cuh): the NPC
        // butterfly rows of this CTA, software-pipelined two deep (the loads
        // of butterfly b + 2 are issued as soon as b's registers are consumed)
        float2 x[L];
        if constexpr (ZP) {
            // object window and probe rows from tensor memory (zpref_store of
            // the previous frame / the prologue)
#pragma unroll
            for (int b = 0; b < NPC; ++b) {
                const int rw = q * NPC + b;
                float2 v[Q], pv[Q];
                tmem_ld2_f2(tmz + 2 * Q * b, v, tm + 2 * Q * b, pv);
#pragma unroll
                for (int s = 0; s < Q; ++s) v[s] = cmul(pv[s], v[s]);
                dft_q<Q>(v);
#pragma unroll
                for (int s = 1; s < Q; ++s) v[s] = cmul(tw[rw * s], v[s]);
#if PTG_RMW_STAGGER && PTG_RMW_GATHER_PLAIN
#if PTG_RMW_STAGGER == 2
                // rank q starts at owner q: at every step the Q sources address Q different owners
#pragma unroll
                for (int R = 0; R < Q; ++R)
                    if (q == R) {
#pragma unroll
                        for (int s2 = 0; s2 < Q; ++s2) {
                            const int s = (s2 + R) % Q;
                            st_cluster_f2(mapa_u32(smem_u32(buf + rw * PM + t), s), v[s]);
                        }
                    }
#else
                if (q & 1) {
#pragma unroll
                    for (int s2 = 0; s2 < Q; ++s2) {
                        constexpr int H = Q / 2;
                        const int s = (s2 + H) % Q;
                        st_cluster_f2(mapa_u32(smem_u32(buf + rw * PM + t), s), v[s]);
                    }
                } else {
#pragma unroll
                    for (int s = 0; s < Q; ++s) st_cluster_f2(mapa_u32(smem_u32(buf + rw * PM + t), s), v[s]);
                }
#endif
#else
#pragma unroll
                for (int s = 0; s < Q; ++s) {
#if PTG_RMW_GATHER_PLAIN
                    st_cluster_f2(mapa_u32(smem_u32(buf + rw * PM + t), s), v[s]);
#else
                    st_async_f2(mapa_u32(smem_u32(buf + rw * PM + t), s), v[s], mapa_u32(bar_g_u, s));
#endif
                }
#endif
            }
        } else {
            const float2* zc = a.z + (size_t)pj.x * n + pj.y + t;
            float2 zb[2][Q], pb[TM ? 1 : 2][Q];   // TM: probe values read from tensor memory at use
            const size_t zstep = (size_t)L * n;
            auto load = [&](int b, int u) {
                // rows q NPC + b + L s through running pointers (one live
                // address per stream); volatile loads keep program order --
                // the compiler would otherwise hoist every butterfly's loads
                const float2* zp = zc + (size_t)(q * NPC + b) * n;
                const float2* pp = a.probe + (size_t)(q * NPC + b) * M + t;
#pragma unroll
                for (int s = 0; s < Q; ++s) {
                    zb[u][s] = ldg_pinned(zp);
                    zp += zstep;
                    if constexpr (PROBE && !TM) {
                        pb[u][s] = ldg_pinned(pp);
                        pp += (size_t)L * M;
                    }
                }
            };
            load(0, 0);
            if constexpr (NPC > 1) load(1, 1);
#pragma unroll
            for (int b = 0; b < NPC; ++b) {
                const int u = b & 1;
                const int rw = q * NPC + b;
                float2 v[Q];
                if constexpr (TM) tmem_ld_f2<Q>(tm + 2 * Q * b, pb[0]);
#pragma unroll
                for (int s = 0; s < Q; ++s) v[s] = PROBE ? cmul(pb[TM ? 0 : u][s], zb[u][s]) : zb[u][s];
                if (b + 2 < NPC) load(b + 2, u);
                dft_q<Q>(v);
#pragma unroll
                for (int s = 1; s < Q; ++s) v[s] = cmul(tw[rw * s], v[s]);
#pragma unroll
                for (int s = 0; s < Q; ++s)
                    st_async_f2(mapa_u32(smem_u32(buf + rw * PM + t), s), v[s], mapa_u32(bar_g_u, s));
            }
        }
        constexpr bool ORDER_LATE = LATE && PTG_RMW_GATHER_PLAIN != 0;   // the leader's load behind the arrival below
        if constexpr (!ORDER_LATE) {
            if (leader && next.x < r.kend) next.y = __ldg(r.order + next.x);
        }
        RTL(2);
#if PTG_RMW_BULK == 2
        publish_pending();   // the previous frame's reduce-adds landed during this gather
#endif
#if PTG_RMW_GATHER_PLAIN
        if constexpr (ZP) {
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            if constexpr (ORDER_LATE) {
                if (leader && next.x < r.kend) next.y = __ldg(r.order + next.x);
            }
            if constexpr (EDEPS) {
                if (ed0 + t < ed1) edep = ldg_pinned_i32(r.dep_idx + ed0 + t);
            }
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else {
            mbar_wait(&bar_g, ph);
        }
#else
        mbar_wait(&bar_g, ph);   // all Q senders' rows have landed in this CTA
#endif
        RTL(3);

        double acc = 0.0;
PTG_UNROLL_N(PTG_RMW_PASS_UNROLL)
        for (int pass = 0; pass < 4; ++pass) {
            if (pass == 0 || pass == 3) {
#pragma unroll
                for (int kk = 0; kk < L; ++kk) x[kk] = buf[kk * PM + t];
                if (pass == 3) {
                    if constexpr (ZP) {
                        // the next frame's item, visible to every CTA after this barrier
                        if (leader) {
                            hand_item((int)(ph ^ 1u));
                            if constexpr (!LATE) next.x = r.kbeg + (int)atomicAdd(r.work, 1u);   // the frame after it, claimed ahead
                        }
                    }
                    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
                    if constexpr (LATE) {
                        if (leader) next.x = r.kbeg + (int)atomicAdd(r.work, 1u);
                    }
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
#ifdef ABL_TIMELINE
            if (pass == 1) RTL(4);
#endif
            if (pass == 0) {
#pragma unroll
                for (int kk = 0; kk < L; ++kk) buf[kk * PM + t] = x[kk];
                ROWSYNC();
PTG_UNROLL_N(PTG_RMW_DFTQ_UNROLL)
                for (int i = 0; i < NPC; ++i) {
                    float2* row = buf + (g + Q * i) * PM + m;
                    float2 v[Q];
#pragma unroll
                    for (int s = 0; s < Q; ++s) v[s] = row[L * s];
                    dft_q<Q>(v);
#pragma unroll
                    for (int s = 1; s < Q; ++s) v[s] = cmul(tw[m * s], v[s]);   // W_M^{m s} from shared memory
#pragma unroll
                    for (int s = 0; s < Q; ++s) row[L * s] = v[s];
                }
                ROWSYNC();
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
                RTL(5);
            } else if (pass == 2) {
#pragma unroll
                for (int c = 0; c < L; c += 2)
                    *reinterpret_cast<float4*>(&buf[rr * PM + qq * L + c]) =
                        make_float4(x[c].x, x[c].y, x[c + 1].x, x[c + 1].y);
                ROWSYNC();
PTG_UNROLL_N(PTG_RMW_DFTQ_UNROLL)
                for (int i = 0; i < NPC; ++i) {
                    float2* row = buf + (g + Q * i) * PM + m;
                    float2 v[Q];
#pragma unroll
                    for (int s = 0; s < Q; ++s) v[s] = row[L * s];
#pragma unroll
                    for (int s = 1; s < Q; ++s) v[s] = cmul(tw[m * s], v[s]);   // W_M^{m s} from shared memory
                    dft_q<Q>(v);
#pragma unroll
                    for (int s = 0; s < Q; ++s) row[L * s] = v[s];
                }
                ROWSYNC();
                RTL(6);
            } else {
                asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
#if PTG_RMW_PUSHBAR
                const uint32_t bar_p_u = smem_u32(&bar_p);
#pragma unroll
                for (int kk = 0; kk < L; ++kk)   // remote row (kk % NPC) Q + q of CTA kk / NPC
                    st_async_f2(mapa_u32(buf_u + (uint32_t)((((kk % NPC) * Q + q) * PM + t) * sizeof(float2)),
                                         kk / NPC),
                                x[kk], mapa_u32(bar_p_u, kk / NPC));
#else
#if PTG_RMW_STAGGER == 2
                if (true) {
#pragma unroll
                    for (int R = 0; R < Q; ++R)
                        if (q == R) {
#pragma unroll
                            for (int k2 = 0; k2 < L; ++k2) {
                                const int kk = (k2 + R * NPC) % L;
                                st_cluster_f2(
                                    mapa_u32(buf_u + (uint32_t)((((kk % NPC) * Q + q) * PM + t) * sizeof(float2)),
                                             kk / NPC),
                                    x[kk]);
                            }
                        }
                } else
#elif PTG_RMW_STAGGER
                if (q & 1) {
#pragma unroll
                    for (int k2 = 0; k2 < L; ++k2) {
                        const int kk = (k2 + L / 2) % L;
                        st_cluster_f2(mapa_u32(buf_u + (uint32_t)((((kk % NPC) * Q + q) * PM + t) * sizeof(float2)),
                                               kk / NPC),
                                      x[kk]);
                    }
                } else
#endif
#pragma unroll
                for (int kk = 0; kk < L; ++kk)   // remote row (kk % NPC) Q + q of CTA kk / NPC
                    st_cluster_f2(mapa_u32(buf_u + (uint32_t)((((kk % NPC) * Q + q) * PM + t) * sizeof(float2)),
                                           kk / NPC),
                                  x[kk]);
#endif
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
        if ((t & 31) == 0) red[t / 32] = acc;
        RTL(7);
#if PTG_RMW_PUSHBAR
        mbar_wait(&bar_p, ph);   // this CTA's rows have landed (all Q senders)
        __syncthreads();         // red[] of every warp
#else
        cl.sync();   // every push has landed; no remote access to this CTA's rows until the next frame
#endif
        RTL(8);
        if (t == 0) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < NT / 32; ++i) s += red[i];
            constexpr int MPP = cl_mpp(Q, M);
            a.misfit[(size_t)j * MPP + q] = (OP == OP_DISTANCE) ? s / (2.0 * (double)M * (double)M) : 0.5 * s;
            if constexpr (MPP > Q) a.misfit[(size_t)j * MPP + Q + q] = 0.0;
        }

        if constexpr (EDEPS) {
            if (edep >= 0) edone = ld_acquire_gpu(r.done + edep);   // consumed in (B)
        }
        // (A) contributions, in place: buf row i Q + s holds object row
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
        RTL(9);
        // ZP: the next frame's object window, in flight across (B) and (C)
        int4 nx = make_int4(0, 0, 0, 0);
        if constexpr (ZP) {
            nx = s_item[ph ^ 1u];
            if (nx.x < r.kend) zpref_issue(nx.z, nx.w, x);
        }
        // (B) every earlier overlapping frame has finished its update
        if constexpr (EDEPS) {
            if (edep >= 0) {
                const unsigned* f = r.done + edep;
                while (edone < (unsigned)Q) {
                    __nanosleep(64);
                    edone = ld_acquire_gpu(f);
                }
            }
            for (int d = ed0 + t + NT; d < ed1; d += NT) {   // lists longer than the CTA (never for rasters)
                const unsigned* f = r.done + __ldg(r.dep_idx + d);
                while (ld_acquire_gpu(f) < (unsigned)Q) __nanosleep(64);
            }
        } else {
            const int d0 = __ldg(r.dep_off + k), d1 = __ldg(r.dep_off + k + 1);
            for (int d = d0 + t; d < d1; d += NT) {
                const unsigned* f = r.done + __ldg(r.dep_idx + d);
                while (ld_acquire_gpu(f) < (unsigned)Q) __nanosleep(64);
            }
        }
        __syncthreads();
        RTL(10);
        // (C) read-modify-write of this CTA's L object rows, coalesced; every
        //     load in flight at once (x[] is free again)
        float2* G0 = r.grad + (size_t)pj.x * n + pj.y;
#if PTG_RMW_BULK
        if ((pj.y & 1) == 0) {
            // the update as TMA bulk reduce-adds, one 2 KiB object row per
            // copy, smem contributions -> L2
            if (t < L) {
                fence_proxy_async_smem();
                const int row = t, orow = q * NPC + row / Q + L * (row % Q);
                asm volatile(
                    "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                        G0 + (size_t)orow * n),
                    "r"(smem_u32(buf + row * PM)), "r"((uint32_t)(M * sizeof(float2)))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
#if PTG_RMW_BULK == 2
                // only the shared-memory source must be free before the next
                // frame's pushes; completion is awaited a gather later
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                pend_k = k;
#elif PTG_RMW_LATE_BULKWAIT
                if constexpr (LATE) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                else asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#else
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#endif
            }
        } else
#endif
        if ((pj.y & 1) == 0) {
            constexpr int HW = M / 2, PER = L * HW / NT, HALF = PER / 2;   // float4 (pixel pairs) per thread
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float4 gv[HALF];
#pragma unroll
                for (int u = 0; u < HALF; ++u) {
                    const int e = t + NT * (h * HALF + u), row = e / HW, c2 = e % HW;
                    const int orow = q * NPC + row / Q + L * (row % Q);
                    gv[u] = __ldcg(reinterpret_cast<const float4*>(G0 + (size_t)orow * n + 2 * c2));
                }
#pragma unroll
                for (int u = 0; u < HALF; ++u) {
                    const int e = t + NT * (h * HALF + u), row = e / HW, c2 = e % HW;
                    const int orow = q * NPC + row / Q + L * (row % Q);
                    const float4 cv = *reinterpret_cast<const float4*>(&buf[row * PM + 2 * c2]);
                    __stcg(reinterpret_cast<float4*>(G0 + (size_t)orow * n + 2 * c2), f4add(gv[u], cv));
                }
            }
        } else {
            constexpr int PER = L * M / NT, HALF = PER / 4;   // four batches of float2 (cold path)
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
        if constexpr (ZP) {
            if (nx.x < r.kend) zpref_store(x);
        }
        // (D) publish: this CTA's rows of frame k are final
#if PTG_RMW_BULK == 2
        if ((pj.y & 1) != 0) {   // (uniform) plain-store frames publish now; bulk frames once their adds complete
            __syncthreads();
            if (t == 0) red_release_gpu_add(r.done + k, 1u);
        }
#else
        __syncthreads();
        if constexpr (LATE) pub_k = k;
        else if (t == 0) red_release_gpu_add(r.done + k, 1u);
#endif
        RTL(11);
#ifdef ABL_TIMELINE
        ++rtl_f;
#endif
        ph ^= 1u;
    }
#if PTG_RMW_BULK == 2
    publish_pending();
#endif
    if constexpr (TM) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (t < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(TCOLS) : "memory");
    }
}

// grad = -v (MG/OPT shift) or 0, <v,z> partial per block, counters zeroed
// (elements >= own: 0 and no <v,z> share -- a BANDS shard's halo rows, whose
// contributions are added on the next rank)
template <typename C>
__global__ void __launch_bounds__(256) k_rmw_init(const C* __restrict__ v, const C* __restrict__ z,
                                                  C* __restrict__ grad, size_t len, size_t own, double* dotp,
                                                  unsigned* done, int N, unsigned* work) {
    __shared__ double red[8];
    const size_t chunk = (len + gridDim.x - 1) / gridDim.x;
    const size_t lo = blockIdx.x * chunk, hi = min(lo + chunk, len);
    double d = 0.0;
    for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        C gv;
        if (v && i < own) {
            const C vv = v[i], zz = z[i];
            gv.x = -vv.x;
            gv.y = -vv.y;
            d += (double)vv.x * (double)zz.x + (double)vv.y * (double)zz.y;
        } else {
            gv.x = 0;
            gv.y = 0;
        }
        grad[i] = gv;
    }
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)N; i += (size_t)gridDim.x * blockDim.x)
        done[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) *work = 0u;
    if (!dotp) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < 8; ++i) s += red[i];
        dotp[blockIdx.x] = s;
    }
}

}  // namespace ptg
