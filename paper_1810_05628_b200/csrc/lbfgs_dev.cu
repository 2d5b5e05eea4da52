// lbfgs_dev.cu — device-resident LBFGS building blocks (see solvers.cuh).
//
// The reference's two-loop recursion (solvers.cpp:19-36) is a chain of 2k+2
// dependent inner products, each followed by an axpy.  Issued as separate
// kernels with a host read per product it costs ~2k+2 PCIe round trips per
// iteration; here it is ONE cooperative kernel: every product is reduced over
// the same fixed kReduceBlocks partition and trees as k_dot (blas.cu), the
// partials are exchanged through a double-buffered scratch with one grid
// barrier per product, and every block forms the identical total, so the
// direction is bitwise the one the kernel-per-op sequence produces.  The
// curvature-pair bookkeeping (s, y, <s,y>, |s|^2, |y|^2, |g|^2) is one more
// fused kernel whose four products are read back in a single transfer.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <new>

#include "solvers.cuh"

namespace ptg {

namespace {

constexpr int kTlThreads = 1024;                                  // 4 groups of 256 = 4 chunks per block
constexpr int kTlGroups = kTlThreads / kReduceThreads;
constexpr int kTlBlocks = kReduceBlocks / kTlGroups;              // 148

template <typename T>
struct TwoLoopArgs {
    const cplx<T>* s[kMaxPairs];
    const cplx<T>* y[kMaxPairs];
    double sy[kMaxPairs];
    int k;
    const cplx<T>* g;
    cplx<T>* q;
    double* scratch;   // 2 x kReduceBlocks
    size_t len;
};

// Register-resident two-loop for short chunks (<= 256*QE elements): every
// thread keeps its q and g elements in registers for the whole recursion,
// and the operand vectors of the next product are loaded before the barrier
// of the current one.  Same partition, trees and arithmetic as k_two_loop
// (and k_dot + k_axpy).
template <typename T, int QE>
__global__ void __launch_bounds__(kTlThreads, 1) k_two_loop_reg(const TwoLoopArgs<T> a) {
    using C = cplx<T>;
    __shared__ double red[kTlThreads / 32];
    __shared__ double total_s;
    __shared__ double alpha_s[kMaxPairs];
    const int sub = threadIdx.x / kReduceThreads, lt = threadIdx.x % kReduceThreads;
    const int lane = lt & 31, w = lt >> 5;
    const int c = blockIdx.x * kTlGroups + sub;
    const size_t chunk = (a.len + kReduceBlocks - 1) / kReduceBlocks;
    const size_t lo = min(a.len, (size_t)c * chunk), hi = min(a.len, lo + chunk);
    unsigned idx[QE];   // 32-bit element offsets (register budget: 64 per thread)
    bool ok[QE];
#pragma unroll
    for (int e = 0; e < QE; ++e) {
        const size_t i = lo + lt + (size_t)e * kReduceThreads;
        ok[e] = i < hi;
        idx[e] = ok[e] ? (unsigned)i : 0u;
    }
    const C zero = mk<T>(T(0), T(0));
    int buf = 0;

    auto load = [&](const C* v, C (&r)[QE]) {
#pragma unroll
        for (int e = 0; e < QE; ++e) r[e] = ok[e] ? v[idx[e]] : zero;
    };
    auto publish = [&](double s) {
        s = warp_tree(s);
        if (lane == 0) red[sub * 8 + w] = s;
        __syncthreads();
        if (lt == 0) {
            double t = 0.0;
            for (int i = 0; i < 8; ++i) t += red[sub * 8 + i];
            a.scratch[buf * kReduceBlocks + c] = t;
        }
        cooperative_groups::this_grid().sync();
    };
    auto total = [&]() -> double {
        if (sub == 0) {
            double t = 0.0;
            for (int i = lt; i < kReduceBlocks; i += kReduceThreads) t += __ldcg(a.scratch + buf * kReduceBlocks + i);
            t = warp_tree(t);
            if (lane == 0) red[w] = t;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double u = 0.0;
            for (int i = 0; i < 8; ++i) u += red[i];
            total_s = u;
        }
        __syncthreads();
        const double r = total_s;
        buf ^= 1;
        return r;
    };
    auto dot = [&](const C (&u)[QE], const C (&v)[QE]) {
        double p = 0.0;
#pragma unroll
        for (int e = 0; e < QE; ++e)
            if (ok[e]) p = __dadd_rn(p, dot_term(u[e], v[e]));
        return p;
    };

    const int k = a.k;
    C qv[QE], u[QE], nx[QE];   // g is re-read where needed (register budget)
    double p;
    if (k == 0) {
        load(a.g, u);
#pragma unroll
        for (int e = 0; e < QE; ++e) qv[e] = mk<T>(u[e].x * T(-1), u[e].y * T(-1));
        p = dot(qv, u);
    } else {
        load(a.g, qv);
        load(a.s[k - 1], nx);
        p = dot(nx, qv);
        load(a.y[k - 1], u);                                   // operands of the first axpy
        load(k > 1 ? a.s[k - 2] : a.y[k - 1], nx);             // and of the next product
        publish(p);
        for (int j = k - 1; j >= 0; --j) {
            const double al = total() / a.sy[j];
            if (threadIdx.x == 0) alpha_s[j] = al;
            const T coef = (T)(-al);
#pragma unroll
            for (int e = 0; e < QE; ++e) {
                qv[e].x += coef * u[e].x;
                qv[e].y += coef * u[e].y;
            }
            p = j > 0 ? dot(nx, qv) : dot(nx, nx);
            if (j > 0) {
                load(a.y[j - 1], u);
                load(j > 1 ? a.s[j - 2] : a.y[k - 1], nx);
            } else {
                load(a.y[0], nx);                              // gamma pass product
            }
            publish(p);
        }
        const T gs = (T)(a.sy[k - 1] / total());
#pragma unroll
        for (int e = 0; e < QE; ++e) qv[e] = mk<T>(qv[e].x * gs, qv[e].y * gs);
        p = dot(nx, qv);
        load(a.s[0], u);
        load(k > 1 ? a.y[1] : a.g, nx);                        // next product operand (g for the descent check)
        publish(p);
        __syncthreads();   // alpha_s visible block-wide
        for (int j = 0; j < k; ++j) {
            const double beta = total() / a.sy[j];
            const T coef = (T)(alpha_s[j] - beta);
#pragma unroll
            for (int e = 0; e < QE; ++e) {
                qv[e].x += coef * u[e].x;
                qv[e].y += coef * u[e].y;
            }
            if (j + 1 < k) {
                p = dot(nx, qv);
                load(a.s[j + 1], u);
                load(j + 2 < k ? a.y[j + 2] : a.g, nx);
                publish(p);
            } else {
#pragma unroll
                for (int e = 0; e < QE; ++e) qv[e] = mk<T>(qv[e].x * T(-1), qv[e].y * T(-1));
                p = dot(qv, nx);                               // nx = g
            }
        }
    }
    publish(p);
    if (total() >= 0.0) {
        load(a.g, u);
#pragma unroll
        for (int e = 0; e < QE; ++e) qv[e] = mk<T>(u[e].x * T(-1), u[e].y * T(-1));
    }
#pragma unroll
    for (int e = 0; e < QE; ++e)
        if (ok[e]) a.q[idx[e]] = qv[e];
}

template <typename T>
__global__ void __launch_bounds__(kTlThreads, 1) k_two_loop(const TwoLoopArgs<T> a) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    using C = cplx<T>;
    __shared__ double red[kTlThreads / 32];
    __shared__ double total_s;
    __shared__ double alpha_s[kMaxPairs];
    const int sub = threadIdx.x / kReduceThreads, lt = threadIdx.x % kReduceThreads;
    const int lane = lt & 31, w = lt >> 5;
    const int c = blockIdx.x * kTlGroups + sub;   // this group's chunk = k_dot's block c
    const size_t chunk = (a.len + kReduceBlocks - 1) / kReduceBlocks;
    const size_t lo = min(a.len, (size_t)c * chunk), hi = min(a.len, lo + chunk);
    int buf = 0;

    // group partial of chunk c (k_dot's block partial) -> scratch, then barrier
    auto publish = [&](double s) {
        s = warp_tree(s);
        if (lane == 0) red[sub * 8 + w] = s;
        __syncthreads();
        if (lt == 0) {
            double t = 0.0;
            for (int i = 0; i < 8; ++i) t += red[sub * 8 + i];
            a.scratch[buf * kReduceBlocks + c] = t;
        }
        grid.sync();
    };
    // k_dot's last-block sum over the partials, formed identically in every block
    auto total = [&]() -> double {
        if (sub == 0) {
            double t = 0.0;
            for (int i = lt; i < kReduceBlocks; i += kReduceThreads) t += __ldcg(a.scratch + buf * kReduceBlocks + i);
            t = warp_tree(t);
            if (lane == 0) red[w] = t;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double u = 0.0;
            for (int i = 0; i < 8; ++i) u += red[i];
            total_s = u;
        }
        __syncthreads();
        const double r = total_s;
        buf ^= 1;
        return r;
    };

    const int k = a.k;
    double p = 0.0;
    if (k == 0) {   // steepest descent: q = -g
        for (size_t i = lo + lt; i < hi; i += kReduceThreads) {
            const C u = a.g[i];
            const C v = mk<T>(u.x * T(-1), u.y * T(-1));
            a.q[i] = v;
            p = __dadd_rn(p, dot_term(v, u));
        }
    } else {
        // q = g ; first product <s_{k-1}, q>
        for (size_t i = lo + lt; i < hi; i += kReduceThreads) {
            const C u = a.g[i];
            a.q[i] = u;
            p = __dadd_rn(p, dot_term(a.s[k - 1][i], u));
        }
        publish(p);
        // first loop (newest to oldest): alpha_j = <s_j, q>/sy_j ; q -= alpha_j y_j
        for (int j = k - 1; j >= 0; --j) {
            const double al = total() / a.sy[j];
            if (threadIdx.x == 0) alpha_s[j] = al;
            const T coef = (T)(-al);
            p = 0.0;
            for (size_t i = lo + lt; i < hi; i += kReduceThreads) {
                C v = a.q[i];
                const C u = a.y[j][i];
                v.x += coef * u.x;
                v.y += coef * u.y;
                a.q[i] = v;
                p = __dadd_rn(p, j > 0 ? dot_term(a.s[j - 1][i], v) : dot_term(a.y[k - 1][i], a.y[k - 1][i]));
            }
            publish(p);
        }
        // H0 = gamma I, gamma = sy_new / <y_new, y_new>
        const T gs = (T)(a.sy[k - 1] / total());
        p = 0.0;
        for (size_t i = lo + lt; i < hi; i += kReduceThreads) {
            const C u = a.q[i];
            const C v = mk<T>(u.x * gs, u.y * gs);
            a.q[i] = v;
            p = __dadd_rn(p, dot_term(a.y[0][i], v));
        }
        publish(p);
        __syncthreads();   // alpha_s visible block-wide
        // second loop (oldest to newest): beta = <y_j, q>/sy_j ; q += (alpha_j - beta) s_j ; then q = -q
        for (int j = 0; j < k; ++j) {
            const double beta = total() / a.sy[j];
            const T coef = (T)(alpha_s[j] - beta);
            p = 0.0;
            for (size_t i = lo + lt; i < hi; i += kReduceThreads) {
                C v = a.q[i];
                const C u = a.s[j][i];
                v.x += coef * u.x;
                v.y += coef * u.y;
                if (j + 1 < k) {
                    a.q[i] = v;
                    p = __dadd_rn(p, dot_term(a.y[j + 1][i], v));
                } else {
                    v = mk<T>(v.x * T(-1), v.y * T(-1));
                    a.q[i] = v;
                    p = __dadd_rn(p, dot_term(v, a.g[i]));
                }
            }
            if (j + 1 < k) publish(p);
        }
    }
    // descent check (solvers.cpp:107): <d, g> >= 0 -> d = -g
    publish(p);
    if (total() >= 0.0) {
        for (size_t i = lo + lt; i < hi; i += kReduceThreads) {
            const C u = a.g[i];
            a.q[i] = mk<T>(u.x * T(-1), u.y * T(-1));
        }
    }
}

// s = nz - z, y = ng - g and <s,y>, <s,s>, <y,y>, <ng,ng> over a fixed
// partition of kPsBlocks blocks, plus the isFinite test of nz (ComplexField::isFinite)
constexpr int kPsBlocks = 296;
template <typename T>
__global__ void __launch_bounds__(kReduceThreads) k_pair_stats(const cplx<T>* nz, const cplx<T>* z,
                                                               const cplx<T>* ng, const cplx<T>* g,
                                                               cplx<T>* s_out, cplx<T>* y_out, size_t len,
                                                               double* scratch, double* out) {
    __shared__ double red[4][kReduceThreads / 32];
    __shared__ bool last;
    pdl_wait_and_trigger();
    const size_t chunk = (len + kPsBlocks - 1) / kPsBlocks;
    const size_t lo = min(len, (size_t)blockIdx.x * chunk), hi = min(len, lo + chunk);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    bool bad = false;
    for (size_t i = lo + threadIdx.x; i < hi; i += kReduceThreads) {
        const cplx<T> zn = nz[i];
        const cplx<T> s = csub(zn, z[i]), y = csub(ng[i], g[i]), gn = ng[i];
        bad |= !isfinite(zn.x) || !isfinite(zn.y);
        s_out[i] = s;
        y_out[i] = y;
        acc[0] = __dadd_rn(acc[0], dot_term(s, y));
        acc[1] = __dadd_rn(acc[1], dot_term(s, s));
        acc[2] = __dadd_rn(acc[2], dot_term(y, y));
        acc[3] = __dadd_rn(acc[3], dot_term(gn, gn));
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double t = warp_tree(acc[q]);
        if (lane == 0) red[q][w] = t;
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x < 4) {
        double t = 0.0;
        for (int i = 0; i < kReduceThreads / 32; ++i) t += red[threadIdx.x][i];
        scratch[threadIdx.x * kReduceBlocks + blockIdx.x] = t;
    }
    if (threadIdx.x == 4) scratch[4 * kReduceBlocks + blockIdx.x] = bad ? 1.0 : 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned int* ctr = reinterpret_cast<unsigned int*>(scratch + 5 * kReduceBlocks);
        last = atomicAdd(ctr, 1u) == kPsBlocks - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // all five quantities' partials in flight together (one L2 round trip), then
    // the same per-thread order and trees as a loop per quantity (same bits)
    constexpr int PER = (kPsBlocks + kReduceThreads - 1) / kReduceThreads;
    double v[5][PER];
#pragma unroll
    for (int q = 0; q < 5; ++q)
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int i = threadIdx.x + u * kReduceThreads;
            v[q][u] = i < kPsBlocks ? __ldcg(scratch + q * kReduceBlocks + i) : 0.0;
        }
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        double t = 0.0;
#pragma unroll
        for (int u = 0; u < PER; ++u)
            if (threadIdx.x + u * kReduceThreads < kPsBlocks) t += v[q][u];
        t = warp_tree(t);
        __syncthreads();
        if (lane == 0) red[0][w] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            double u = 0.0;
            for (int i = 0; i < kReduceThreads / 32; ++i) u += red[0][i];
            out[q] = u;
        }
    }
    if (threadIdx.x == 0) *reinterpret_cast<unsigned int*>(scratch + 5 * kReduceBlocks) = 0u;
}

// ------------------------------------------- compact-representation LBFGS
// For pairs a < A (pointer arrays) and two shared vectors yc, gn:
//   dot[4a + 0] = <s_a, yc>, dot[4a + 1] = <y_a, yc>, dot[4a + 2] = <s_a, gn>,
//   dot[4a + 3] = <y_a, gn>,
// each over k_dot's fixed partition (block x of row r handles pairs 4r..4r+3).
constexpr int kMdPairs = 4;
constexpr int kMdBlocks = 148;   // partition of the batched products (one tree per block and product)
template <typename T>
struct MultiDotArgs {
    const cplx<T>* s[kMaxPairs + 1];
    const cplx<T>* y[kMaxPairs + 1];
    const cplx<T>* yc;
    const cplx<T>* gn;
    int A;
    size_t len;
    double* partial;   // [4 A][kMdBlocks]
    // optional (zn != nullptr): the newest pair (a = A - 1) and yc are formed
    // in-kernel as s = zn - zo, y = yc = gn - go (k_pair_stats' arithmetic), so
    // this kernel need not wait for k_pair_stats to store them
    const cplx<T>* zn;
    const cplx<T>* zo;
    const cplx<T>* go;
};

template <typename T>
__global__ void __launch_bounds__(kReduceThreads) k_multi_dot(const MultiDotArgs<T> a) {
    using C = cplx<T>;
    __shared__ double red[kMdPairs * 4][kReduceThreads / 32];
    pdl_wait_and_trigger();
    const size_t chunk = (a.len + kMdBlocks - 1) / kMdBlocks;
    const size_t lo = min(a.len, (size_t)blockIdx.x * chunk), hi = min(a.len, lo + chunk);
    const int p0 = blockIdx.y * kMdPairs;
    double acc[kMdPairs * 4];
#pragma unroll
    for (int k = 0; k < kMdPairs * 4; ++k) acc[k] = 0.0;
    // Every load of an element is issued before any product (one HBM round
    // trip per element instead of one per pair: the history is 2 x 25 vectors,
    // far beyond L2 at the larger levels).  Rows past A read pair A - 1 again
    // (never stored); the fresh pair reads zn / gn in place of its own s / y,
    // which k_pair_stats may be writing concurrently.  Same products, same
    // order of additions as the pair-by-pair loop: same bits.
    const bool any_fresh = a.zn && p0 + kMdPairs >= a.A && p0 < a.A;
    const C* sp[kMdPairs];
    const C* yp[kMdPairs];
    bool fr[kMdPairs];
#pragma unroll
    for (int q = 0; q < kMdPairs; ++q) {
        const int pq = min(p0 + q, a.A - 1);
        fr[q] = a.zn && pq == a.A - 1;
        sp[q] = fr[q] ? a.zn : a.s[pq];
        yp[q] = fr[q] ? a.gn : a.y[pq];
    }
    const C* zop = any_fresh ? a.zo : a.gn;
#pragma unroll 2
    for (size_t i = lo + threadIdx.x; i < hi; i += kReduceThreads) {
        const C gn = a.gn[i];
        const C yo = a.zn ? a.go[i] : a.yc[i];
        const C zo = zop[i];
        C svr[kMdPairs], yvr[kMdPairs];
#pragma unroll
        for (int q = 0; q < kMdPairs; ++q) {
            svr[q] = sp[q][i];
            yvr[q] = yp[q][i];
        }
        const C yc = a.zn ? csub(gn, yo) : yo;
#pragma unroll
        for (int q = 0; q < kMdPairs; ++q) {
            const C sv = fr[q] ? csub(svr[q], zo) : svr[q];
            const C yv = fr[q] ? yc : yvr[q];
            acc[4 * q + 0] = __dadd_rn(acc[4 * q + 0], dot_term(sv, yc));
            acc[4 * q + 1] = __dadd_rn(acc[4 * q + 1], dot_term(yv, yc));
            acc[4 * q + 2] = __dadd_rn(acc[4 * q + 2], dot_term(sv, gn));
            acc[4 * q + 3] = __dadd_rn(acc[4 * q + 3], dot_term(yv, gn));
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kMdPairs * 4; ++k) {
        const double t = warp_tree(acc[k]);
        if (lane == 0) red[k][w] = t;
    }
    __syncthreads();
    if (threadIdx.x < kMdPairs * 4 && p0 + threadIdx.x / 4 < a.A) {
        double t = 0.0;
        for (int i = 0; i < kReduceThreads / 32; ++i) t += red[threadIdx.x][i];
        a.partial[(size_t)(4 * p0 + threadIdx.x) * kMdBlocks + blockIdx.x] = t;
    }
}

// out[d] = fixed tree over partial[d][*], one block per product
__global__ void __launch_bounds__(kReduceThreads) k_multi_sum(const double* partial, double* out) {
    __shared__ double red[kReduceThreads / 32];
    pdl_wait_and_trigger();
    const double* pd = partial + (size_t)blockIdx.x * kMdBlocks;
    double t = 0.0;
    for (int i = threadIdx.x; i < kMdBlocks; i += kReduceThreads) t += pd[i];
    t = warp_tree(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double u = 0.0;
        for (int i = 0; i < kReduceThreads / 32; ++i) u += red[i];
        out[blockIdx.x] = u;
    }
}

// dir = -(gamma g + sum_i u_i s_i + sum_i c_i y_i), accumulated in fp64 per entry
template <typename T>
struct CombineArgs {
    const cplx<T>* s[kMaxPairs];
    const cplx<T>* y[kMaxPairs];
    double u[kMaxPairs], c[kMaxPairs];
    double gamma;
    int k;
    const cplx<T>* g;
    cplx<T>* dir;
    size_t len;
    // optional fused first line-search trial: trial = z0 + 1 * dir (k_add_scaled's arithmetic)
    const cplx<T>* z0;
    cplx<T>* trial;
};

template <typename T>
__global__ void __launch_bounds__(256) k_combine(const CombineArgs<T> a) {
    pdl_wait_and_trigger();
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.len; i += (size_t)gridDim.x * blockDim.x) {
        const cplx<T> gv = a.g[i];
        double rx = a.gamma * (double)gv.x, ry = a.gamma * (double)gv.y;
        constexpr int U = 8;   // loads of U pairs in flight together
        for (int j0 = 0; j0 < a.k; j0 += U) {
            cplx<T> sv[U], yv[U];
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (j0 + q < a.k) {
                    sv[q] = a.s[j0 + q][i];
                    yv[q] = a.y[j0 + q][i];
                }
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (j0 + q < a.k) {
                    const int j = j0 + q;
                    rx = fma(a.u[j], (double)sv[q].x, fma(a.c[j], (double)yv[q].x, rx));
                    ry = fma(a.u[j], (double)sv[q].y, fma(a.c[j], (double)yv[q].y, ry));
                }
        }
        const cplx<T> d = mk<T>((T)-rx, (T)-ry);
        a.dir[i] = d;
        if (a.trial) {
            const T one = (T)1.0;
            const cplx<T> u = a.z0[i];
            a.trial[i] = mk<T>(u.x + one * d.x, u.y + one * d.y);
        }
    }
}

template <typename T>
void multi_dot_t(const Plan& p, const void* const* s, const void* const* y, int A, const void* yc,
                 const void* gn, double* scratch, double* out_dev) {
    MultiDotArgs<T> a{};
    for (int i = 0; i < A; ++i) {
        a.s[i] = static_cast<const cplx<T>*>(s[i]);
        a.y[i] = static_cast<const cplx<T>*>(y[i]);
    }
    a.yc = static_cast<const cplx<T>*>(yc);
    a.gn = static_cast<const cplx<T>*>(gn);
    a.A = A;
    a.len = p.nn();
    a.partial = scratch;
    a.zn = a.zo = a.go = nullptr;
    k_multi_dot<T><<<dim3(kMdBlocks, (A + kMdPairs - 1) / kMdPairs), kReduceThreads, 0, p.stream>>>(a);
    k_multi_sum<<<4 * A, kReduceThreads, 0, p.stream>>>(scratch, out_dev);
    PTG_CHECK_LAUNCH();
    count_launch(2);
}

template <typename T>
void combine_t(const Plan& p, const void* const* s, const void* const* y, const double* u, const double* c,
               double gamma, int k, const void* g, void* dir) {
    CombineArgs<T> a{};
    for (int i = 0; i < k; ++i) {
        a.s[i] = static_cast<const cplx<T>*>(s[i]);
        a.y[i] = static_cast<const cplx<T>*>(y[i]);
        a.u[i] = u[i];
        a.c[i] = c[i];
    }
    a.gamma = gamma;
    a.k = k;
    a.g = static_cast<const cplx<T>*>(g);
    a.dir = static_cast<cplx<T>*>(dir);
    a.len = p.nn();
    const int grid = (int)std::min<size_t>(148 * 8, (a.len + 255) / 256);
    k_combine<T><<<grid, 256, 0, p.stream>>>(a);
    PTG_CHECK_LAUNCH();
    count_launch();
}

template <typename K>
bool coop_fits(K kern) {
    int dev = 0, sms = 0, per_sm = 0, coop = 0;
    PTG_CUDA(cudaGetDevice(&dev));
    PTG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    PTG_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    PTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTlThreads, 0));
    return coop && per_sm * sms >= kTlBlocks;
}

template <typename T>
bool two_loop_fits() {
    static int ok = -1;
    if (ok < 0) {
        ok = coop_fits(k_two_loop<T>) && coop_fits(k_two_loop_reg<T, 1>) && coop_fits(k_two_loop_reg<T, 2>);
        if constexpr (sizeof(T) == 4) ok = ok && coop_fits(k_two_loop_reg<T, 4>);
    }
    return ok == 1;
}

template <typename T>
bool launch_two_loop(const Plan& p, const void* const* s, const void* const* y, const double* sy, int k,
                     const void* g, void* q, double* scratch) {
    if (k > kMaxPairs || !two_loop_fits<T>()) return false;
    TwoLoopArgs<T> a{};
    for (int i = 0; i < k; ++i) {
        a.s[i] = static_cast<const cplx<T>*>(s[i]);
        a.y[i] = static_cast<const cplx<T>*>(y[i]);
        a.sy[i] = sy[i];
    }
    a.k = k;
    a.g = static_cast<const cplx<T>*>(g);
    a.q = static_cast<cplx<T>*>(q);
    a.scratch = scratch;
    a.len = p.nn();
    void* args[] = {&a};
    const size_t chunk = (a.len + kReduceBlocks - 1) / kReduceBlocks;
    size_t qe = (chunk + kReduceThreads - 1) / kReduceThreads;   // elements per thread
    const void* kern = reinterpret_cast<const void*>(k_two_loop<T>);
    // PTG_TWO_LOOP=mem: memory-resident variant for any size (A/B)
    const char* tl = getenv("PTG_TWO_LOOP");
    if (tl && tl[0] == 'm') qe = ~size_t(0);
    if (qe <= 1) kern = reinterpret_cast<const void*>(k_two_loop_reg<T, 1>);
    else if (qe <= 2) kern = reinterpret_cast<const void*>(k_two_loop_reg<T, 2>);
    else if constexpr (sizeof(T) == 4) {
        if (qe <= 4) kern = reinterpret_cast<const void*>(k_two_loop_reg<T, 4>);
    }
    PTG_CUDA(cudaLaunchCooperativeKernel(kern, dim3(kTlBlocks), dim3(kTlThreads), args, 0, p.stream));
    count_launch();
    return true;
}

}  // namespace

bool dev_two_loop(const Plan& p, const void* const* s, const void* const* y, const double* sy, int k,
                  const void* g, void* q, double* scratch) {
    return p.prec == PTG_C64 ? launch_two_loop<float>(p, s, y, sy, k, g, q, scratch)
                             : launch_two_loop<double>(p, s, y, sy, k, g, q, scratch);
}

void dev_multi_dot(const Plan& p, const void* const* s, const void* const* y, int A, const void* yc,
                   const void* gn, double* scratch, double* out_dev) {
    if (A <= 0) return;
    if (A > kMaxPairs + 1) raise(PTG_ERR_INTERNAL, "multi_dot: too many pairs");
    if (p.prec == PTG_C64) multi_dot_t<float>(p, s, y, A, yc, gn, scratch, out_dev);
    else multi_dot_t<double>(p, s, y, A, yc, gn, scratch, out_dev);
}

void dev_combine(const Plan& p, const void* const* s, const void* const* y, const double* u, const double* c,
                 double gamma, int k, const void* g, void* dir) {
    if (k > kMaxPairs) raise(PTG_ERR_INTERNAL, "combine: too many pairs");
    if (p.prec == PTG_C64) combine_t<float>(p, s, y, u, c, gamma, k, g, dir);
    else combine_t<double>(p, s, y, u, c, gamma, k, g, dir);
}

void dev_pair_stats(const Plan& p, const void* nz, const void* z, const void* ng, const void* g, void* s_out,
                    void* y_out, double* scratch, double* out_dev) {
    const size_t len = p.nn();
    if (p.prec == PTG_C64)
        k_pair_stats<float><<<kPsBlocks, kReduceThreads, 0, p.stream>>>(
            (const float2*)nz, (const float2*)z, (const float2*)ng, (const float2*)g, (float2*)s_out, (float2*)y_out,
            len, scratch, out_dev);
    else
        k_pair_stats<double><<<kPsBlocks, kReduceThreads, 0, p.stream>>>(
            (const double2*)nz, (const double2*)z, (const double2*)ng, (const double2*)g, (double2*)s_out,
            (double2*)y_out, len, scratch, out_dev);
    PTG_CHECK_LAUNCH();
    count_launch();
}

// ------------------------------------------ kernel-node parameters (graphs)
// The same launches as dev_combine / dev_pair_stats / dev_multi_dot, as
// cudaKernelNodeParams: d_lbfgs replays its per-iteration sequence as a CUDA
// graph and rewrites these nodes' arguments each iteration.
namespace {
template <typename A>
A& node_store(KNode& n) {
    static_assert(sizeof(A) <= sizeof(n.store), "KNode store too small");
    return *new (n.store) A();
}
template <typename T>
void node_combine_t(const Plan& p, const void* const* s, const void* const* y, const double* u, const double* c,
                    double gamma, int k, const void* g, void* dir, KNode& n, const void* z0, void* trial) {
    CombineArgs<T>& a = node_store<CombineArgs<T>>(n);
    for (int i = 0; i < k; ++i) {
        a.s[i] = static_cast<const cplx<T>*>(s[i]);
        a.y[i] = static_cast<const cplx<T>*>(y[i]);
        a.u[i] = u[i];
        a.c[i] = c[i];
    }
    a.gamma = gamma;
    a.k = k;
    a.g = static_cast<const cplx<T>*>(g);
    a.dir = static_cast<cplx<T>*>(dir);
    a.len = p.nn();
    a.z0 = static_cast<const cplx<T>*>(z0);
    a.trial = static_cast<cplx<T>*>(trial);
    n.argp[0] = &a;
    n.prm = cudaKernelNodeParams{};
    n.prm.func = reinterpret_cast<void*>(k_combine<T>);
    n.prm.gridDim = dim3((unsigned)std::min<size_t>(148 * 8, (a.len + 255) / 256));
    n.prm.blockDim = dim3(256);
    n.prm.kernelParams = n.argp;
}
struct PairStatsArgs {
    const void *nz, *z, *ng, *g;
    void *s, *y;
    size_t len;
    double *scratch, *out;
};
template <typename T>
void node_multi_dot_t(const Plan& p, const void* const* s, const void* const* y, int A, const void* yc,
                      const void* gn, double* scratch, double* out_dev, KNode& md, KNode& ms, const void* zn,
                      const void* zo, const void* go) {
    MultiDotArgs<T>& a = node_store<MultiDotArgs<T>>(md);
    a.zn = static_cast<const cplx<T>*>(zn);
    a.zo = static_cast<const cplx<T>*>(zo);
    a.go = static_cast<const cplx<T>*>(go);
    for (int i = 0; i < A; ++i) {
        a.s[i] = static_cast<const cplx<T>*>(s[i]);
        a.y[i] = static_cast<const cplx<T>*>(y[i]);
    }
    a.yc = static_cast<const cplx<T>*>(yc);
    a.gn = static_cast<const cplx<T>*>(gn);
    a.A = A;
    a.len = p.nn();
    a.partial = scratch;
    md.argp[0] = &a;
    md.prm = cudaKernelNodeParams{};
    md.prm.func = reinterpret_cast<void*>(k_multi_dot<T>);
    md.prm.gridDim = dim3(kMdBlocks, (A + kMdPairs - 1) / kMdPairs);
    md.prm.blockDim = dim3(kReduceThreads);
    md.prm.kernelParams = md.argp;
    struct MS { const double* partial; double* out; };
    MS& b = node_store<MS>(ms);
    b.partial = scratch;
    b.out = out_dev;
    ms.argp[0] = &b.partial;
    ms.argp[1] = &b.out;
    ms.prm = cudaKernelNodeParams{};
    ms.prm.func = reinterpret_cast<void*>(k_multi_sum);
    ms.prm.gridDim = dim3(4 * A);
    ms.prm.blockDim = dim3(kReduceThreads);
    ms.prm.kernelParams = ms.argp;
}
}  // namespace

void node_combine(const Plan& p, const void* const* s, const void* const* y, const double* u, const double* c,
                  double gamma, int k, const void* g, void* dir, KNode& n, const void* z0, void* trial) {
    if (k > kMaxPairs) raise(PTG_ERR_INTERNAL, "combine: too many pairs");
    if (p.prec == PTG_C64) node_combine_t<float>(p, s, y, u, c, gamma, k, g, dir, n, z0, trial);
    else node_combine_t<double>(p, s, y, u, c, gamma, k, g, dir, n, z0, trial);
}

void node_pair_stats(const Plan& p, const void* nz, const void* z, const void* ng, const void* g, void* s_out,
                     void* y_out, double* scratch, double* out_dev, KNode& n) {
    PairStatsArgs& a = node_store<PairStatsArgs>(n);
    a = PairStatsArgs{nz, z, ng, g, s_out, y_out, p.nn(), scratch, out_dev};
    void* ptrs[9] = {&a.nz, &a.z, &a.ng, &a.g, &a.s, &a.y, &a.len, &a.scratch, &a.out};
    for (int i = 0; i < 9; ++i) n.argp[i] = ptrs[i];
    n.prm = cudaKernelNodeParams{};
    n.prm.func = p.prec == PTG_C64 ? reinterpret_cast<void*>(k_pair_stats<float>)
                                   : reinterpret_cast<void*>(k_pair_stats<double>);
    n.prm.gridDim = dim3(kPsBlocks);
    n.prm.blockDim = dim3(kReduceThreads);
    n.prm.kernelParams = n.argp;
}

void node_multi_dot(const Plan& p, const void* const* s, const void* const* y, int A, const void* yc,
                    const void* gn, double* scratch, double* out_dev, KNode& md, KNode& ms, const void* zn,
                    const void* zo, const void* go) {
    if (A <= 0 || A > kMaxPairs + 1) raise(PTG_ERR_INTERNAL, "multi_dot: pair count");
    if (p.prec == PTG_C64) node_multi_dot_t<float>(p, s, y, A, yc, gn, scratch, out_dev, md, ms, zn, zo, go);
    else node_multi_dot_t<double>(p, s, y, A, yc, gn, scratch, out_dev, md, ms, zn, zo, go);
}

void node_launch(const KNode& n, cudaStream_t s) {
    // programmatic dependent launch: the kernel's launch overlaps its
    // predecessor's tail; every one of these kernels starts with
    // griddepcontrol.wait, so nothing is read early
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = n.prm.gridDim;
    cfg.blockDim = n.prm.blockDim;
    cfg.dynamicSmemBytes = n.prm.sharedMemBytes;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PTG_CUDA(cudaLaunchKernelExC(&cfg, n.prm.func, n.prm.kernelParams));
    count_launch();
}

}  // namespace ptg
