// metrics.cu — reconstruction diagnostics on the device (metrics.cpp:67-136):
// relativeError, magnitudeRelError, canonicalPhase and phaseSSIM, so a
// solver's per-iteration callback needs no device-to-host copy of the
// iterate and no CPU SSIM.
//
// All arithmetic is fp64 whatever the field precision (complex64 entries are
// widened exactly).  Sums use a fixed partition and fixed trees (bitwise
// reproducible run to run); the 11-tap Gaussian filters keep the reference's
// per-sample order (s += g[j] * in[c + j], separately rounded), so the five
// filtered maps match the reference to the last bit given the same inputs.
#include <mutex>
#include <cmath>

#include "blas.cuh"
#include "metrics.cuh"

namespace ptg {

namespace {

constexpr int kWin = 11;            // metrics.cpp:14
constexpr double kSigma = 1.5;      // metrics.cpp:15
constexpr double kHalfPi = 1.5707963267948966192313216916398;
constexpr int kMBlocks = 296, kMThreads = 256;

__constant__ double c_gauss[kWin];

__device__ __forceinline__ double2 widen(const float2& v) { return make_double2((double)v.x, (double)v.y); }
__device__ __forceinline__ double2 widen(const double2& v) { return v; }

// fixed-partition block reduction of NV values per thread -> partial[b * NV + k]
template <int NV>
__device__ void block_partials(double (&v)[NV], double* partial) {
    __shared__ double red[NV][kMThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double t = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) red[k][w] = t;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double t = 0.0;
        for (int i = 0; i < kMThreads / 32; ++i) t += red[threadIdx.x][i];
        partial[blockIdx.x * NV + threadIdx.x] = t;
    }
}

// sum of partials in block order (one thread: kMBlocks values, fixed order)
template <int NV>
__global__ void k_sum_partials(const double* partial, double* out) {
    if (threadIdx.x < NV) {
        double t = 0.0;
        for (int b = 0; b < kMBlocks; ++b) t += partial[b * NV + threadIdx.x];
        out[threadIdx.x] = t;
    }
}

// |z - zt|^2, |zt|^2, (|z| - |zt|)^2 over a fixed partition
template <typename T>
__global__ void __launch_bounds__(kMThreads) k_error_sums(const cplx<T>* z, const cplx<T>* zt, size_t len,
                                                          double* partial) {
    const size_t chunk = (len + kMBlocks - 1) / kMBlocks;
    const size_t lo = min(len, (size_t)blockIdx.x * chunk), hi = min(len, lo + chunk);
    double v[3] = {0.0, 0.0, 0.0};
    for (size_t i = lo + threadIdx.x; i < hi; i += kMThreads) {
        const double2 a = widen(z[i]), b = widen(zt[i]);
        const double dx = a.x - b.x, dy = a.y - b.y;
        v[0] += dx * dx + dy * dy;
        v[1] += b.x * b.x + b.y * b.y;
        const double d = hypot(a.x, a.y) - hypot(b.x, b.y);   // std::abs(complex) = hypot
        v[2] += d * d;
    }
    block_partials<3>(v, partial);
}

// canonicalPhase, part 1: phase map + per-block min / max
template <typename T>
__global__ void __launch_bounds__(kMThreads) k_phase(const cplx<T>* z, size_t len, double* phase, double* partial) {
    __shared__ double smin[kMThreads / 32], smax[kMThreads / 32];
    double lo = INFINITY, hi = -INFINITY;
    for (size_t i = blockIdx.x * (size_t)kMThreads + threadIdx.x; i < len; i += (size_t)kMBlocks * kMThreads) {
        const double2 a = widen(z[i]);
        const double p = (a.x == 0.0 && a.y == 0.0) ? 0.0 : atan2(a.y, a.x);
        phase[i] = p;
        lo = fmin(lo, p);
        hi = fmax(hi, p);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        smin[threadIdx.x >> 5] = lo;
        smax[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < kMThreads / 32; ++i) {
            lo = fmin(lo, smin[i]);
            hi = fmax(hi, smax[i]);
        }
        partial[2 * blockIdx.x] = fmin(smin[0], lo);
        partial[2 * blockIdx.x + 1] = fmax(smax[0], hi);
    }
}

__global__ void k_phase_range(const double* partial, double* range) {
    if (threadIdx.x == 0) {
        double lo = INFINITY, hi = -INFINITY;
        for (int b = 0; b < kMBlocks; ++b) {
            lo = fmin(lo, partial[2 * b]);
            hi = fmax(hi, partial[2 * b + 1]);
        }
        range[0] = lo;
        range[1] = hi;
    }
}

// canonicalPhase, part 2: (p - lo) / (hi - lo) * pi/2, all zero if hi == lo
__global__ void k_phase_scale(double* phase, size_t len, const double* range) {
    const double lo = range[0], hi = range[1];
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
        phase[i] = (hi == lo) ? 0.0 : __dmul_rn(__ddiv_rn(__dsub_rn(phase[i], lo), __dsub_rn(hi, lo)), kHalfPi);
}

// phaseSSIM map over a TILE x TILE block of valid positions: rows pass of the
// five maps for the TILE + 10 input rows, then the columns pass, then the
// per-position SSIM term; block partial of the terms (fixed tree)
constexpr int kTile = 16;
__global__ void __launch_bounds__(kTile * kTile) k_ssim(const double* x, const double* y, int n, int nbx,
                                                        double* partial) {
    constexpr int R = kTile + kWin - 1;
    __shared__ double rp[5][R][kTile];   // rows-pass results (x, y, xx, yy, xy)
    __shared__ double red[kTile * kTile / 32];
    const int m = n - kWin + 1;
    const int r0 = (blockIdx.x / nbx) * kTile, c0 = (blockIdx.x % nbx) * kTile;
    const int tc = threadIdx.x % kTile, tr = threadIdx.x / kTile;
    // rows pass: rp[.][i][c] = sum_j g[j] * in(r0 + i, c0 + c + j)   (metrics.cpp:44-48)
    for (int i = tr; i < R; i += kTile) {
        const int r = r0 + i, c = c0 + tc;
        double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        if (r < n && c < m) {
            const double* xr = x + (size_t)r * n + c;
            const double* yr = y + (size_t)r * n + c;
            for (int j = 0; j < kWin; ++j) {
                const double a = xr[j], b = yr[j], g = c_gauss[j];
                s[0] = __dadd_rn(s[0], __dmul_rn(g, a));
                s[1] = __dadd_rn(s[1], __dmul_rn(g, b));
                s[2] = __dadd_rn(s[2], __dmul_rn(g, __dmul_rn(a, a)));
                s[3] = __dadd_rn(s[3], __dmul_rn(g, __dmul_rn(b, b)));
                s[4] = __dadd_rn(s[4], __dmul_rn(g, __dmul_rn(a, b)));
            }
        }
#pragma unroll
        for (int k = 0; k < 5; ++k) rp[k][i][tc] = s[k];
    }
    __syncthreads();
    // columns pass + SSIM term (metrics.cpp:50-55, :120-131)
    const int r = r0 + tr, c = c0 + tc;
    double term = 0.0;
    if (r < m && c < m) {
        double f[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < kWin; ++i) {
            const double g = c_gauss[i];
#pragma unroll
            for (int k = 0; k < 5; ++k) f[k] = __dadd_rn(f[k], __dmul_rn(g, rp[k][tr + i][tc]));
        }
        const double L = kHalfPi;
        const double c1 = __dmul_rn(__dmul_rn(0.01, L), __dmul_rn(0.01, L));
        const double c2 = __dmul_rn(__dmul_rn(0.03, L), __dmul_rn(0.03, L));
        const double mux = f[0], muy = f[1];
        const double vx = __dsub_rn(f[2], __dmul_rn(mux, mux));
        const double vy = __dsub_rn(f[3], __dmul_rn(muy, muy));
        const double cxy = __dsub_rn(f[4], __dmul_rn(mux, muy));
        const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mux), muy), c1),
                                     __dadd_rn(__dmul_rn(2.0, cxy), c2));
        const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mux, mux), __dmul_rn(muy, muy)), c1),
                                     __dadd_rn(__dadd_rn(vx, vy), c2));
        term = __ddiv_rn(num, den);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = term;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < kTile * kTile / 32; ++i) t += red[i];
        partial[blockIdx.x] = t;
    }
}

__global__ void k_sum_blocks(const double* partial, int nb, double* out) {
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int b = 0; b < nb; ++b) t += partial[b];
        out[0] = t;
    }
}

void upload_gauss() {   // __constant__ memory is per device: once per device
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    PTG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= 0 && dev < 64 && done[dev]) return;
    double g[kWin], sum = 0.0;   // metrics.cpp:22-33
    for (int i = 0; i < kWin; ++i) {
        const double x = i - kWin / 2;
        g[i] = std::exp(-x * x / (2.0 * kSigma * kSigma));
        sum += g[i];
    }
    for (double& v : g) v /= sum;
    PTG_CUDA(cudaMemcpyToSymbol(c_gauss, g, sizeof g));
    if (dev >= 0 && dev < 64) done[dev] = true;
}

template <typename T>
void metrics_t(const void* zv, const void* ztv, int n, unsigned mask, ptg_metrics* out, cudaStream_t s) {
    const size_t len = (size_t)n * n;
    const auto* z = static_cast<const cplx<T>*>(zv);
    const auto* zt = static_cast<const cplx<T>*>(ztv);
    const int nbx = n >= kWin ? (n - kWin + 1 + kTile - 1) / kTile : 0;
    const size_t nb_ssim = (size_t)nbx * nbx;
    // scratch: partials (kMBlocks * 3, 2 * kMBlocks, nb_ssim) + results + two phase maps
    const size_t nscr = 3 * (size_t)kMBlocks + 2 * (size_t)kMBlocks + nb_ssim + 8;
    double* scr = nullptr;
    double* ph = nullptr;
    PTG_CUDA(cudaMallocAsync(&scr, nscr * sizeof(double), s));
    const bool want_ssim = mask & PTG_METRIC_PHASE_SSIM;
    if (want_ssim) PTG_CUDA(cudaMallocAsync(&ph, 2 * len * sizeof(double), s));
    double* p_err = scr;
    double* p_rng = p_err + 3 * kMBlocks;
    double* p_ssim = p_rng + 2 * kMBlocks;
    double* res = p_ssim + nb_ssim;   // [0..2] error sums, [3..4] range x, [5..6] range y, [7] ssim sum
    double h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (mask & (PTG_METRIC_RELATIVE_ERROR | PTG_METRIC_MAGNITUDE_REL_ERROR)) {
        k_error_sums<T><<<kMBlocks, kMThreads, 0, s>>>(z, zt, len, p_err);
        k_sum_partials<3><<<1, 32, 0, s>>>(p_err, res);
        count_launch(2);
    }
    if (want_ssim) {
        upload_gauss();
        double* px = ph;
        double* py = ph + len;
        k_phase<T><<<kMBlocks, kMThreads, 0, s>>>(z, len, px, p_rng);
        k_phase_range<<<1, 32, 0, s>>>(p_rng, res + 3);
        k_phase_scale<<<kMBlocks, kMThreads, 0, s>>>(px, len, res + 3);
        k_phase<T><<<kMBlocks, kMThreads, 0, s>>>(zt, len, py, p_rng);
        k_phase_range<<<1, 32, 0, s>>>(p_rng, res + 5);
        k_phase_scale<<<kMBlocks, kMThreads, 0, s>>>(py, len, res + 5);
        k_ssim<<<(unsigned)nb_ssim, kTile * kTile, 0, s>>>(px, py, n, nbx, p_ssim);
        k_sum_blocks<<<1, 32, 0, s>>>(p_ssim, (int)nb_ssim, res + 7);
        count_launch(8);
    }
    PTG_CHECK_LAUNCH();
    PTG_CUDA(cudaMemcpyAsync(h, res, sizeof h, cudaMemcpyDeviceToHost, s));
    PTG_CUDA(cudaFreeAsync(scr, s));
    if (ph) PTG_CUDA(cudaFreeAsync(ph, s));
    PTG_CUDA(cudaStreamSynchronize(s));
    if (mask & PTG_METRIC_RELATIVE_ERROR) {
        if (h[1] == 0.0) raise(PTG_ERR_DOMAIN, "relativeError: zero reference field");
        out->relative_error = std::sqrt(h[0]) / std::sqrt(h[1]);   // norm2(sub) / norm2(zTrue)
    }
    if (mask & PTG_METRIC_MAGNITUDE_REL_ERROR) {
        if (h[1] == 0.0) raise(PTG_ERR_DOMAIN, "magnitudeRelError: zero reference field");
        out->magnitude_rel_error = std::sqrt(h[2]) / std::sqrt(h[1]);
    }
    if (want_ssim) {
        const double mm = (double)(n - kWin + 1) * (double)(n - kWin + 1);
        out->phase_ssim = h[7] / mm;
    }
}

template <typename T>
void canonical_phase_t(const void* zv, int n, double* out, cudaStream_t s) {
    const size_t len = (size_t)n * n;
    double* scr = nullptr;
    PTG_CUDA(cudaMallocAsync(&scr, (2 * (size_t)kMBlocks + 2) * sizeof(double), s));
    k_phase<T><<<kMBlocks, kMThreads, 0, s>>>(static_cast<const cplx<T>*>(zv), len, out, scr);
    k_phase_range<<<1, 32, 0, s>>>(scr, scr + 2 * kMBlocks);
    k_phase_scale<<<kMBlocks, kMThreads, 0, s>>>(out, len, scr + 2 * kMBlocks);
    PTG_CHECK_LAUNCH();
    count_launch(3);
    PTG_CUDA(cudaFreeAsync(scr, s));
}

}  // namespace

void dev_canonical_phase(int prec, const void* z, int n, double* out, cudaStream_t s) {
    if (n < 1) raise(PTG_ERR_DOMAIN, "metric: empty fields");
    if (prec == PTG_C64) canonical_phase_t<float>(z, n, out, s);
    else canonical_phase_t<double>(z, n, out, s);
}

void dev_metrics(int prec, const void* z, const void* z_true, int n, unsigned mask, ptg_metrics* out,
                 cudaStream_t s) {
    if (n < 1) raise(PTG_ERR_DOMAIN, "metric: empty fields");
    if ((mask & PTG_METRIC_PHASE_SSIM) && n < kWin)
        raise(PTG_ERR_METRIC, "phaseSSIM: grid side " + std::to_string(n) + " is smaller than the 11x11 window");
    if (prec == PTG_C64) metrics_t<float>(z, z_true, n, mask, out, s);
    else metrics_t<double>(z, z_true, n, mask, out, s);
}

}  // namespace ptg
