// blas.cu — device vector algebra + deterministic fp64 reductions.
// See blas.cuh for the reference functions each entry point restates.
#include "blas.cuh"

namespace ptg {

thread_local int64_t* g_launch_counter = nullptr;

namespace {

constexpr int kThreads = 256;

inline int grid_for(size_t len) {
    size_t g = (len + kThreads - 1) / kThreads;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : (int)g;
}

template <typename T>
__global__ void k_fill_zero(cplx<T>* x, size_t len) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
        x[i] = mk<T>(T(0), T(0));
}

template <typename T>
__global__ void k_copy(cplx<T>* d, const cplx<T>* s, size_t len) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
        d[i] = s[i];
}

// y[i] += alpha * x[i] with alpha = (alpha_dev ? *alpha_dev : alpha) * coef
template <typename T>
__global__ void k_axpy(cplx<T>* y, double alpha, const double* alpha_dev, double coef,
                       const cplx<T>* x, size_t len) {
    const T a = (T)(alpha_dev ? (*alpha_dev) * coef : alpha);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
        cplx<T> v = y[i];
        const cplx<T> u = x[i];
        v.x += a * u.x;
        v.y += a * u.y;
        y[i] = v;
    }
}

template <typename T>
__global__ void k_scale(cplx<T>* out, const cplx<T>* a, double alpha, const double* alpha_dev,
                        size_t len) {
    const T s = (T)(alpha_dev ? *alpha_dev : alpha);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
        const cplx<T> u = a[i];
        out[i] = mk<T>(u.x * s, u.y * s);
    }
}

template <typename T>
__global__ void k_sub(cplx<T>* out, const cplx<T>* a, const cplx<T>* b, size_t len) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
        out[i] = csub(a[i], b[i]);
}

template <typename T>
__global__ void k_add_scaled(cplx<T>* out, const cplx<T>* a, double alpha, const cplx<T>* b, size_t len) {
    const T s = (T)alpha;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
        const cplx<T> u = a[i], v = b[i];
        out[i] = mk<T>(u.x + s * v.x, u.y + s * v.y);
    }
}

// Two-level deterministic dot: block b owns the fixed range [b*chunk, ...);
// the last block to finish sums the kReduceBlocks partials in block order.
template <typename T>
__global__ void __launch_bounds__(kReduceThreads) k_dot(const cplx<T>* a, const cplx<T>* b,
                                                        size_t len, double* scratch, double* out) {
    __shared__ double red[kReduceThreads / 32];
    __shared__ bool last;
    const size_t chunk = (len + kReduceBlocks - 1) / kReduceBlocks;
    const size_t lo = blockIdx.x * chunk;
    const size_t hi = lo + chunk < len ? lo + chunk : len;
    double s = 0.0;
    for (size_t i = lo + threadIdx.x; i < hi; i += kReduceThreads) s = __dadd_rn(s, dot_term(a[i], b[i]));
    s = warp_tree(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < kReduceThreads / 32; ++i) t += red[i];
        scratch[blockIdx.x] = t;
        __threadfence();
        unsigned int* ctr = reinterpret_cast<unsigned int*>(scratch + kReduceBlocks);
        last = (atomicAdd(ctr, 1u) == kReduceBlocks - 1);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        // fixed tree over the partials: thread t sums a fixed strided subset
        double t = 0.0;
        for (int i = threadIdx.x; i < kReduceBlocks; i += kReduceThreads)
            t += __ldcg(scratch + i);
        t = warp_tree(t);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            double u = 0.0;
            for (int i = 0; i < kReduceThreads / 32; ++i) u += red[i];
            *out = u;
            *reinterpret_cast<unsigned int*>(scratch + kReduceBlocks) = 0u;
        }
    }
}

template <typename T>
__global__ void k_nonfinite(const cplx<T>* a, size_t len, int* flag) {
    bool bad = false;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
        const cplx<T> u = a[i];
        bad |= !isfinite(u.x) || !isfinite(u.y);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <typename T>
__global__ void k_from_c128(cplx<T>* d, const double2* s, size_t len) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
        const double2 u = s[i];
        d[i] = mk<T>((T)u.x, (T)u.y);
    }
}

template <typename T>
__global__ void k_to_c128(double2* d, const cplx<T>* s, size_t len) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x) {
        const cplx<T> u = s[i];
        d[i] = make_double2((double)u.x, (double)u.y);
    }
}

template <typename D, typename S>
__global__ void k_real_convert(D* d, const S* s, size_t len) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < len; i += (size_t)gridDim.x * blockDim.x)
        d[i] = (D)s[i];
}

}  // namespace

#define DISPATCH(prec, KERNEL, ...)                                                     \
    do {                                                                                \
        if ((prec) == PTG_C64) KERNEL<float>(__VA_ARGS__); else KERNEL<double>(__VA_ARGS__); \
    } while (0)

template <typename T> using cp = cplx<T>*;
template <typename T> using ccp = const cplx<T>*;

void dev_fill_zero(int prec, void* x, size_t len, cudaStream_t s) {
    if (!len) return;
    if (prec == PTG_C64) k_fill_zero<float><<<grid_for(len), kThreads, 0, s>>>((float2*)x, len);
    else k_fill_zero<double><<<grid_for(len), kThreads, 0, s>>>((double2*)x, len);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_copy(int prec, void* dst, const void* src, size_t len, cudaStream_t s) {
    if (!len || dst == src) return;
    PTG_CUDA(cudaMemcpyAsync(dst, src, len * (prec == PTG_C64 ? 8 : 16), cudaMemcpyDeviceToDevice, s));
}

void dev_axpy(int prec, void* y, double alpha, const void* x, size_t len, cudaStream_t s) {
    if (!len) return;
    if (prec == PTG_C64) k_axpy<float><<<grid_for(len), kThreads, 0, s>>>((float2*)y, alpha, nullptr, 1.0, (const float2*)x, len);
    else k_axpy<double><<<grid_for(len), kThreads, 0, s>>>((double2*)y, alpha, nullptr, 1.0, (const double2*)x, len);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_axpy_dscalar(int prec, void* y, const double* alpha_dev, double coef, const void* x,
                      size_t len, cudaStream_t s) {
    if (!len) return;
    if (prec == PTG_C64) k_axpy<float><<<grid_for(len), kThreads, 0, s>>>((float2*)y, 0.0, alpha_dev, coef, (const float2*)x, len);
    else k_axpy<double><<<grid_for(len), kThreads, 0, s>>>((double2*)y, 0.0, alpha_dev, coef, (const double2*)x, len);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_scale(int prec, void* out, const void* a, double alpha, size_t len, cudaStream_t s) {
    if (!len) return;
    if (prec == PTG_C64) k_scale<float><<<grid_for(len), kThreads, 0, s>>>((float2*)out, (const float2*)a, alpha, nullptr, len);
    else k_scale<double><<<grid_for(len), kThreads, 0, s>>>((double2*)out, (const double2*)a, alpha, nullptr, len);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_scale_dscalar(int prec, void* out, const void* a, const double* alpha_dev, size_t len,
                       cudaStream_t s) {
    if (!len) return;
    if (prec == PTG_C64) k_scale<float><<<grid_for(len), kThreads, 0, s>>>((float2*)out, (const float2*)a, 0.0, alpha_dev, len);
    else k_scale<double><<<grid_for(len), kThreads, 0, s>>>((double2*)out, (const double2*)a, 0.0, alpha_dev, len);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_sub(int prec, void* out, const void* a, const void* b, size_t len, cudaStream_t s) {
    if (!len) return;
    if (prec == PTG_C64) k_sub<float><<<grid_for(len), kThreads, 0, s>>>((float2*)out, (const float2*)a, (const float2*)b, len);
    else k_sub<double><<<grid_for(len), kThreads, 0, s>>>((double2*)out, (const double2*)a, (const double2*)b, len);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_add_scaled(int prec, void* out, const void* a, double alpha, const void* b, size_t len,
                    cudaStream_t s) {
    if (!len) return;
    if (prec == PTG_C64) k_add_scaled<float><<<grid_for(len), kThreads, 0, s>>>((float2*)out, (const float2*)a, alpha, (const float2*)b, len);
    else k_add_scaled<double><<<grid_for(len), kThreads, 0, s>>>((double2*)out, (const double2*)a, alpha, (const double2*)b, len);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_dot(int prec, const void* a, const void* b, size_t len, double* scratch, double* out_dev,
             cudaStream_t s) {
    if (prec == PTG_C64) k_dot<float><<<kReduceBlocks, kReduceThreads, 0, s>>>((const float2*)a, (const float2*)b, len, scratch, out_dev);
    else k_dot<double><<<kReduceBlocks, kReduceThreads, 0, s>>>((const double2*)a, (const double2*)b, len, scratch, out_dev);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_nonfinite(int prec, const void* a, size_t len, int* flag_dev, cudaStream_t s) {
    PTG_CUDA(cudaMemsetAsync(flag_dev, 0, sizeof(int), s));
    if (!len) return;
    if (prec == PTG_C64) k_nonfinite<float><<<grid_for(len), kThreads, 0, s>>>((const float2*)a, len, flag_dev);
    else k_nonfinite<double><<<grid_for(len), kThreads, 0, s>>>((const double2*)a, len, flag_dev);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_from_c128(int prec, void* dst, const double* src, size_t len, cudaStream_t s) {
    if (!len) return;
    if (prec == PTG_C128) {
        if (dst != (const void*)src) PTG_CUDA(cudaMemcpyAsync(dst, src, len * 16, cudaMemcpyDeviceToDevice, s));
        return;
    }
    k_from_c128<float><<<grid_for(len), kThreads, 0, s>>>((float2*)dst, (const double2*)src, len);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_to_c128(int prec, double* dst, const void* src, size_t len, cudaStream_t s) {
    if (!len) return;
    if (prec == PTG_C128) {
        if ((const void*)dst != src) PTG_CUDA(cudaMemcpyAsync(dst, src, len * 16, cudaMemcpyDeviceToDevice, s));
        return;
    }
    k_to_c128<float><<<grid_for(len), kThreads, 0, s>>>((double2*)dst, (const float2*)src, len);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_real_convert(int dst_prec, void* dst, int src_dtype, const void* src, size_t len,
                      cudaStream_t s) {
    if (!len) return;
    const bool df = dst_prec == PTG_C64, sf = src_dtype == PTG_F32;
    if (df == sf) {
        PTG_CUDA(cudaMemcpyAsync(dst, src, len * (df ? 4 : 8), cudaMemcpyDeviceToDevice, s));
        return;
    }
    if (df) k_real_convert<float, double><<<grid_for(len), kThreads, 0, s>>>((float*)dst, (const double*)src, len);
    else k_real_convert<double, float><<<grid_for(len), kThreads, 0, s>>>((double*)dst, (const float*)src, len);
    PTG_CHECK_LAUNCH();
    count_launch();
}

}  // namespace ptg
