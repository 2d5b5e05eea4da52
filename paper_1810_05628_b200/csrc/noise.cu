// noise.cu — measurement noise on the device.
//
// addNoise (/root/reference/proj/src/forward.cpp:56-86,
// /root/reference/proj/include/ptycho/forward.hpp:38-48):
//   per pattern, g_i = sqrt(-2 log(1 - u1)) cos(2 pi u2) (rng::gaussian,
//   rng.hpp:18-24, one deviate per two uniforms), eps = level ||d|| / ||g|| g
//   (zero when ||g|| = 0), out = max(d + eps, 0).
// Poisson photon noise at a per-pattern photon budget (BASELINE configs 4/5;
// no reference counterpart): lambda = d * photons / sum(d), out = k / scale,
// k ~ Poisson(lambda) by inversion (lambda < 10) or Hormann's transformed
// rejection PTRS (lambda >= 10).
//
// Uniforms come from a counter-based generator, Philox4x64-10 (the bit
// generator numpy.random.Philox implements; tests pin it against numpy), so
// every sample is addressable and the kernels need no sequential state:
// counter = (pixel, pattern, tag, block), key = (seed, 0).  For bit-level
// parity with the reference's std::mt19937_64 stream, ptg_add_noise also
// accepts the uniforms themselves (the oracle test passes the reference
// engine's draws).  One CTA per pattern; fp64 sums in a fixed tree order, so
// results are run-to-run identical.
#include <cmath>

#include "plan.cuh"

namespace ptg {

namespace {

struct u64x4 { unsigned long long v[4]; };

__device__ __forceinline__ u64x4 philox4x64_10(unsigned long long c0, unsigned long long c1, unsigned long long c2,
                                               unsigned long long c3, unsigned long long k0, unsigned long long k1) {
    constexpr unsigned long long M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    constexpr unsigned long long W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const unsigned long long hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
        const unsigned long long hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
        const unsigned long long n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += W0;
        k1 += W1;
    }
    return {{c0, c1, c2, c3}};
}

// uniform01 (rng.hpp:14-16): top 53 bits of a 64-bit draw
__device__ __forceinline__ double u01(unsigned long long x) { return (double)(x >> 11) * 0x1.0p-53; }

constexpr unsigned long long kTagGauss = 1, kTagPoisson = 2;
constexpr int kNoiseThreads = 256;

// fixed-order block sum of one double per thread (warp xor tree, then warps in order)
__device__ __forceinline__ double block_sum(double x, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kNoiseThreads / 32; ++i) s += red[i];
    return s;
}

__device__ __forceinline__ double gauss_at(size_t i, int j, unsigned long long seed, const double* __restrict__ uni,
                                           size_t MM) {
    double u1, u2;
    if (uni) {
        const size_t o = 2 * ((size_t)j * MM + i);
        u1 = uni[o];
        u2 = uni[o + 1];
    } else {
        const u64x4 r = philox4x64_10(i, (unsigned long long)j, kTagGauss, 0ull, seed, 0ull);
        u1 = u01(r.v[0]);
        u2 = u01(r.v[1]);
    }
    const double rr = sqrt(-2.0 * log(1.0 - u1));
    return rr * cos(6.283185307179586476925286766559 * u2);
}

template <typename R>
__global__ void __launch_bounds__(kNoiseThreads) k_add_noise(R* __restrict__ d, size_t MM, double level,
                                                             unsigned long long seed, const double* __restrict__ uni) {
    __shared__ double red[kNoiseThreads / 32];
    const int j = blockIdx.x;
    R* dj = d + (size_t)j * MM;
    double dsq = 0.0, gsq = 0.0;
    for (size_t i = threadIdx.x; i < MM; i += kNoiseThreads) {
        const double x = (double)dj[i];
        const double g = gauss_at(i, j, seed, uni, MM);
        dsq += x * x;
        gsq += g * g;
    }
    dsq = block_sum(dsq, red);
    gsq = block_sum(gsq, red);
    const double scale = gsq > 0.0 ? level * sqrt(dsq) / sqrt(gsq) : 0.0;
    for (size_t i = threadIdx.x; i < MM; i += kNoiseThreads) {
        const double g = gauss_at(i, j, seed, uni, MM) * scale;
        dj[i] = (R)fmax((double)dj[i] + g, 0.0);
    }
}

// Poisson(lam): uniforms drawn from Philox blocks (pixel, pattern, tag, b), b = 0, 1, ...
struct UStream {
    unsigned long long i, j, seed, b = 0;
    u64x4 r;
    int k = 4;
    __device__ double next() {
        if (k == 4) {
            r = philox4x64_10(i, j, kTagPoisson, b++, seed, 0ull);
            k = 0;
        }
        return u01(r.v[k++]);
    }
};

__device__ double poisson_sample(double lam, UStream& us) {
    if (!(lam > 0.0)) return 0.0;
    if (lam < 10.0) {   // inversion
        const double u = us.next();
        double p = exp(-lam), F = p;
        int k = 0;
        while (u > F && k < 1000) {
            ++k;
            p *= lam / k;
            F += p;
        }
        return (double)k;
    }
    // PTRS (Hormann 1993, "The transformed rejection method for generating Poisson random variables")
    const double slam = sqrt(lam), loglam = log(lam);
    const double b = 0.931 + 2.53 * slam;
    const double a = -0.059 + 0.02483 * b;
    const double invalpha = 1.1239 + 1.1328 / (b - 3.4);
    const double vr = 0.9277 - 3.6224 / (b - 2.0);
    for (int it = 0; it < 10000; ++it) {
        const double U = us.next() - 0.5;
        const double V = us.next();
        const double usv = 0.5 - fabs(U);
        const double k = floor((2.0 * a / usv + b) * U + lam + 0.43);
        if (usv >= 0.07 && V <= vr) return k;
        if (k < 0.0 || (usv < 0.013 && V > usv)) continue;
        if (log(V) + log(invalpha) - log(a / (usv * usv) + b) <= -lam + k * loglam - lgamma(k + 1.0)) return k;
    }
    return floor(lam);
}

template <typename R>
__global__ void __launch_bounds__(kNoiseThreads) k_add_poisson(R* __restrict__ d, size_t MM, double photons,
                                                               unsigned long long seed) {
    __shared__ double red[kNoiseThreads / 32];
    const int j = blockIdx.x;
    R* dj = d + (size_t)j * MM;
    double tot = 0.0;
    for (size_t i = threadIdx.x; i < MM; i += kNoiseThreads) tot += (double)dj[i];
    tot = block_sum(tot, red);
    const double scale = tot > 0.0 ? photons / tot : 0.0;
    for (size_t i = threadIdx.x; i < MM; i += kNoiseThreads) {
        if (scale > 0.0) {
            UStream us{i, (unsigned long long)j, seed};
            dj[i] = (R)(poisson_sample((double)dj[i] * scale, us) / scale);
        } else {
            dj[i] = (R)0;
        }
    }
}

__global__ void k_philox_raw(unsigned long long* out, size_t nblocks, unsigned long long c1, unsigned long long c2,
                             unsigned long long c3, unsigned long long k0, unsigned long long k1,
                             unsigned long long c0) {
    for (size_t b = blockIdx.x * (size_t)blockDim.x + threadIdx.x; b < nblocks; b += (size_t)gridDim.x * blockDim.x) {
        const u64x4 r = philox4x64_10(c0 + b, c1, c2, c3, k0, k1);
#pragma unroll
        for (int k = 0; k < 4; ++k) out[4 * b + k] = r.v[k];
    }
}

}  // namespace

// the plan's intensities -> noisy intensities, amplitudes rebuilt
void plan_add_noise(Plan& p, double level, unsigned long long seed, const double* uniforms_host) {
    if (level < 0.0) raise(PTG_ERR_DOMAIN, "noise level must be non-negative");   // forward.cpp:57
    LaunchScope ls(p);
    plan_ensure(p, PTG_INTENSITY);
    const size_t len = (size_t)p.N * p.MM();
    DevMem uni;
    if (uniforms_host && len) {
        uni.alloc(2 * len * sizeof(double));
        PTG_CUDA(cudaMemcpyAsync(uni.p, uniforms_host, 2 * len * sizeof(double), cudaMemcpyHostToDevice, p.stream));
    }
    if (p.N > 0) {
        if (p.prec == PTG_C64)
            k_add_noise<float><<<p.N, kNoiseThreads, 0, p.stream>>>(p.inten.as<float>(), p.MM(), level, seed,
                                                                    uni.as<const double>());
        else
            k_add_noise<double><<<p.N, kNoiseThreads, 0, p.stream>>>(p.inten.as<double>(), p.MM(), level, seed,
                                                                     uni.as<const double>());
        PTG_CHECK_LAUNCH();
        ++p.launches;
    }
    plan_refresh_amp(p);
    PTG_CUDA(cudaStreamSynchronize(p.stream));   // `uni` is freed on return
}

void plan_add_poisson(Plan& p, double photons, unsigned long long seed) {
    if (!(photons > 0.0)) raise(PTG_ERR_DOMAIN, "photon budget must be positive");
    LaunchScope ls(p);
    plan_ensure(p, PTG_INTENSITY);
    if (p.N > 0) {
        if (p.prec == PTG_C64)
            k_add_poisson<float><<<p.N, kNoiseThreads, 0, p.stream>>>(p.inten.as<float>(), p.MM(), photons, seed);
        else
            k_add_poisson<double><<<p.N, kNoiseThreads, 0, p.stream>>>(p.inten.as<double>(), p.MM(), photons, seed);
        PTG_CHECK_LAUNCH();
        ++p.launches;
    }
    plan_refresh_amp(p);
}

void dev_philox_raw(unsigned long long* out, size_t nblocks, const unsigned long long ctr[4],
                    const unsigned long long key[2], cudaStream_t s) {
    if (!nblocks) return;
    const int blocks = (int)std::min<size_t>((nblocks + 255) / 256, 148 * 8);
    k_philox_raw<<<blocks, 256, 0, s>>>(out, nblocks, ctr[1], ctr[2], ctr[3], key[0], key[1], ctr[0]);
    PTG_CHECK_LAUNCH();
    count_launch();
}

}  // namespace ptg
