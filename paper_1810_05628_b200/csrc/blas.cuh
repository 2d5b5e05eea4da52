// blas.cuh — device vector algebra over complex fields (sm_100a).
//
// GPU restatement of the reference's field linear algebra
// (/root/reference/proj/src/field.cpp:87-119: norm2sq, norm2, dotReal, add,
// sub, scaled, axpy) and its deterministic blocked reductions
// (kernels.cpp:87-120).  Reductions accumulate in fp64 with a fixed
// partition (fixed grid, fixed per-thread stride, fixed shuffle tree, partials
// summed in block order), so results are bitwise reproducible run to run for
// a given length, independent of scheduling.
#pragma once

#include "common.cuh"

namespace ptg {

// precision-erased entry points (elem = PTG_C64 / PTG_C128); len = complex count
void dev_fill_zero(int prec, void* x, size_t len, cudaStream_t s);
void dev_copy(int prec, void* dst, const void* src, size_t len, cudaStream_t s);
// y += alpha * x   (field.cpp:116-119)
void dev_axpy(int prec, void* y, double alpha, const void* x, size_t len, cudaStream_t s);
// y += (*alpha_dev * coef) * x, scalar read on device (no host sync)
void dev_axpy_dscalar(int prec, void* y, const double* alpha_dev, double coef, const void* x,
                      size_t len, cudaStream_t s);
// out = a * alpha   (field.cpp:108-112)
void dev_scale(int prec, void* out, const void* a, double alpha, size_t len, cudaStream_t s);
void dev_scale_dscalar(int prec, void* out, const void* a, const double* alpha_dev, size_t len,
                       cudaStream_t s);
// out = a - b       (field.cpp:102-106)
void dev_sub(int prec, void* out, const void* a, const void* b, size_t len, cudaStream_t s);
// out = a + alpha * b
void dev_add_scaled(int prec, void* out, const void* a, double alpha, const void* b, size_t len,
                    cudaStream_t s);
// *out_dev = <a, b>_R   (kernels.cpp:104-120) ; b == a gives norm2sq
// scratch: kReduceBlocks doubles of device memory owned by the caller
void dev_dot(int prec, const void* a, const void* b, size_t len, double* scratch, double* out_dev,
             cudaStream_t s);
// *flag_dev = 1 if any entry is non-finite (ComplexField::isFinite, field.cpp:15-19)
void dev_nonfinite(int prec, const void* a, size_t len, int* flag_dev, cudaStream_t s);
// precision conversion: complex128 <-> plan precision
void dev_from_c128(int prec, void* dst, const double* src, size_t len, cudaStream_t s);
void dev_to_c128(int prec, double* dst, const void* src, size_t len, cudaStream_t s);
// real arrays: convert f64/f32 input to the precision's real type
void dev_real_convert(int dst_prec, void* dst, int src_dtype, const void* src, size_t len,
                      cudaStream_t s);

constexpr int kReduceBlocks = 592;   // 4 x 148 SMs, fixed => deterministic
constexpr int kReduceThreads = 256;

// one term of the real inner product <u, v>_R in fp64 with explicit rounding,
// so every kernel that reduces over the kReduceBlocks partition (k_dot, the
// fused LBFGS kernels) produces the same bits for the same operands
template <typename C>
__device__ __forceinline__ double dot_term(const C& u, const C& v) {
    return __fma_rn((double)u.x, (double)v.x, __dmul_rn((double)u.y, (double)v.y));
}

// fixed xor-shuffle tree over a warp (every lane gets the same sum); groups
// then add their warp sums in warp order
__device__ __forceinline__ double warp_tree(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

extern thread_local int64_t* g_launch_counter;   // per-plan counter hook
inline void count_launch(int k = 1) { if (g_launch_counter) *g_launch_counter += k; }

}  // namespace ptg
