// transfer.cu — MG/OPT grid-transfer operators on the device (HBM-bound).
//
//   restrictField  multigrid.cpp:34-44  ((a+b)+(c+d)) * 1/4 on 2x2 blocks, so
//                  restrict(prolong(u)) == u bitwise (same summation order)
//   prolongField   multigrid.cpp:46-53  2x2 block copy
//   restrictData   multigrid.cpp:55-77  centred (M/2)^2 crop of the fftshifted
//                  pattern, un-shifted, x 1/16 (x 1/4 when applied to sqrt(d))
//
// One thread per coarse pixel; each thread reads/writes the two fine pixels of
// a row pair as one 16-byte vector in complex64 (float4: two float2), so warps
// touch contiguous 512 B segments; complex128 pixels are 16 B each already.
// restrictData moves four outputs per thread as one float4 whenever the
// fftshift index map keeps them contiguous (M a multiple of 16).
#include "blas.cuh"
#include "transfer.cuh"

namespace ptg {
namespace {

// complex64, n even: float4 = the two fine pixels (2c, 2c+1) of a row
__global__ void k_restrict_v4(const float4* __restrict__ fine, int n, float2* __restrict__ coarse) {
    const int nH = n / 2;
    const size_t total = (size_t)nH * nH;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / nH), c = (int)(i % nH);
        const float4 ab = fine[(size_t)(2 * r) * nH + c];
        const float4 cd = fine[(size_t)(2 * r + 1) * nH + c];
        float2 o;   // ((a + b) + (c + d)) / 4, the reference's order
        o.x = ((ab.x + ab.z) + (cd.x + cd.z)) * 0.25f;
        o.y = ((ab.y + ab.w) + (cd.y + cd.w)) * 0.25f;
        coarse[i] = o;
    }
}

__global__ void k_prolong_v4(const float2* __restrict__ coarse, int nH, float4* __restrict__ fine) {
    const size_t total = (size_t)nH * nH;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / nH), c = (int)(i % nH);
        const float2 v = coarse[i];
        const float4 vv = make_float4(v.x, v.y, v.x, v.y);
        fine[(size_t)(2 * r) * nH + c] = vv;
        fine[(size_t)(2 * r + 1) * nH + c] = vv;
    }
}

// float data, M % 16 == 0: four consecutive coarse columns map to four
// consecutive fine columns (the wrap points of the index map fall on multiples of 4)
__global__ void k_restrict_data_v4(const float* __restrict__ fine, int N, int M, float4* __restrict__ coarse,
                                   float scale) {
    const int MH = M / 2, Q4 = MH / 4;
    const size_t per4 = (size_t)MH * Q4;
    const size_t total = per4 * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t k = i / per4;
        const int rem = (int)(i % per4);
        const int u = rem / Q4, v = 4 * (rem % Q4);
        const int uf = ((u + MH / 2) % MH + 3 * M / 4) % M;
        const int vf = ((v + MH / 2) % MH + 3 * M / 4) % M;
        const float4 d = *reinterpret_cast<const float4*>(fine + k * (size_t)M * M + (size_t)uf * M + vf);
        coarse[i] = make_float4(d.x * scale, d.y * scale, d.z * scale, d.w * scale);
    }
}

template <typename T>
__global__ void k_restrict(const cplx<T>* __restrict__ fine, int n, cplx<T>* __restrict__ coarse) {
    const int nH = n / 2;
    const size_t total = (size_t)nH * nH;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / nH), c = (int)(i % nH);
        const cplx<T>* f0 = fine + (size_t)(2 * r) * n + 2 * c;
        const cplx<T>* f1 = f0 + n;
        const cplx<T> a = f0[0], b = f0[1], cc = f1[0], d = f1[1];
        cplx<T> o;
        o.x = ((a.x + b.x) + (cc.x + d.x)) * T(0.25);
        o.y = ((a.y + b.y) + (cc.y + d.y)) * T(0.25);
        coarse[i] = o;
    }
}

template <typename T>
__global__ void k_prolong(const cplx<T>* __restrict__ coarse, int nH, cplx<T>* __restrict__ fine) {
    const int n = 2 * nH;
    const size_t total = (size_t)nH * nH;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / nH), c = (int)(i % nH);
        const cplx<T> v = coarse[i];
        cplx<T>* f0 = fine + (size_t)(2 * r) * n + 2 * c;
        f0[0] = v;
        f0[1] = v;
        f0[n] = v;
        f0[n + 1] = v;
    }
}

template <typename R>
__global__ void k_restrict_data(const R* __restrict__ fine, int N, int M, R* __restrict__ coarse, R scale) {
    const int MH = M / 2;
    const size_t per = (size_t)MH * MH;
    const size_t total = per * N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t k = i / per;
        const int rem = (int)(i % per);
        const int u = rem / MH, v = rem % MH;
        const int uf = ((u + MH / 2) % MH + 3 * M / 4) % M;
        const int vf = ((v + MH / 2) % MH + 3 * M / 4) % M;
        coarse[i] = fine[k * (size_t)M * M + (size_t)uf * M + vf] * scale;
    }
}

inline int grid_for(size_t len) {
    size_t g = (len + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : (int)g;
}

}  // namespace

void dev_restrict_field(int prec, const void* fine, int n, void* coarse, cudaStream_t s) {
    if (n < 2 || n % 2 != 0)
        raise(PTG_ERR_GEOMETRY, "restrictField: grid side must be even and >= 2, got " + std::to_string(n));
    const size_t total = (size_t)(n / 2) * (n / 2);
    if (prec == PTG_C64) k_restrict_v4<<<grid_for(total), 256, 0, s>>>((const float4*)fine, n, (float2*)coarse);
    else k_restrict<double><<<grid_for(total), 256, 0, s>>>((const double2*)fine, n, (double2*)coarse);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_prolong_field(int prec, const void* coarse, int nH, void* fine, cudaStream_t s) {
    if (nH < 1) raise(PTG_ERR_GEOMETRY, "prolongField: empty grid");
    const size_t total = (size_t)nH * nH;
    if (prec == PTG_C64) k_prolong_v4<<<grid_for(total), 256, 0, s>>>((const float2*)coarse, nH, (float4*)fine);
    else k_prolong<double><<<grid_for(total), 256, 0, s>>>((const double2*)coarse, nH, (double2*)fine);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_restrict_data(int dtype, const void* fine, int N, int M, void* coarse, double scale,
                       cudaStream_t s) {
    if (M < 4 || M % 4 != 0) raise(PTG_ERR_GEOMETRY, "restrictData: grid side must be a multiple of 4");
    const size_t total = (size_t)N * (M / 2) * (M / 2);
    if (!total) return;
    if (dtype == PTG_F32 && M % 16 == 0)
        k_restrict_data_v4<<<grid_for(total / 4), 256, 0, s>>>((const float*)fine, N, M, (float4*)coarse, (float)scale);
    else if (dtype == PTG_F32) k_restrict_data<float><<<grid_for(total), 256, 0, s>>>((const float*)fine, N, M, (float*)coarse, (float)scale);
    else k_restrict_data<double><<<grid_for(total), 256, 0, s>>>((const double*)fine, N, M, (double*)coarse, scale);
    PTG_CHECK_LAUNCH();
    count_launch();
}

}  // namespace ptg
