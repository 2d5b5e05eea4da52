// halo.cu — band-decomposition exchange helpers (sharding.py).
//
// Weak scaling splits a tall object into n x n bands, consecutive bands sharing
// `ov` gradient rows.  One exchange per evaluation: every rank packs its top and
// bottom ov rows and its misfit into one buffer, one NCCL all-gather moves the
// buffers (2 ov n complex + 8 bytes per rank: ~0.4 MB at config 2), and every
// rank adds its neighbours' rows to its own (own + received; IEEE addition is
// commutative, so both copies of a shared row are bitwise equal) and sums the
// misfits in rank order (every rank forms the identical total).  Two kernel
// launches and one collective replace two point-to-point calls, two adds and a
// scalar allreduce.  Layout per rank (bytes): [top ov x n][bottom ov x n][misfit f64][pad to 16].
#include <algorithm>

#include "blas.cuh"
#include "transfer.cuh"

namespace ptg {
namespace {

template <typename T>
__global__ void k_halo_pack(const cplx<T>* __restrict__ g, int n, int ov, const double* __restrict__ val,
                            unsigned char* __restrict__ buf) {
    const size_t m = (size_t)ov * n;
    cplx<T>* top = reinterpret_cast<cplx<T>*>(buf);
    cplx<T>* bot = top + m;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
        top[i] = g[i];
        bot[i] = g[(size_t)(n - ov) * n + i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<double*>(buf + 2 * m * sizeof(cplx<T>)) = *val;
}

template <typename T>
__global__ void k_halo_unpack(cplx<T>* __restrict__ g, int n, int ov, const unsigned char* __restrict__ all,
                              size_t stride, int rank, int world, double* __restrict__ val) {
    const size_t m = (size_t)ov * n;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
        if (rank > 0) {   // my top rows += the previous band's bottom rows
            const cplx<T>* pb = reinterpret_cast<const cplx<T>*>(all + (size_t)(rank - 1) * stride) + m;
            g[i] = cadd(g[i], pb[i]);
        }
        if (rank + 1 < world) {   // my bottom rows += the next band's top rows
            const cplx<T>* nt = reinterpret_cast<const cplx<T>*>(all + (size_t)(rank + 1) * stride);
            const size_t k = (size_t)(n - ov) * n + i;
            g[k] = cadd(g[k], nt[i]);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double s = 0.0;   // rank order: the same total on every rank
        for (int r = 0; r < world; ++r) s += *reinterpret_cast<const double*>(all + (size_t)r * stride + 2 * m * sizeof(cplx<T>));
        *val = s;
    }
}

inline int halo_grid(size_t m) {
    size_t b = (m + 255) / 256;
    return (int)std::max<size_t>(1, std::min<size_t>(b, 148 * 8));
}

}  // namespace

size_t halo_bytes(int prec, int n, int ov) {
    const size_t c = prec == PTG_C64 ? 8 : 16;
    const size_t b = 2 * (size_t)ov * n * c + sizeof(double);
    return (b + 15) / 16 * 16;
}

void dev_halo_pack(int prec, const void* g, int n, int ov, const double* val, void* buf, cudaStream_t s) {
    if (n < 1 || ov < 0 || 2 * (size_t)ov > (size_t)n)   // top and bottom halo rows must not overlap
        raise(PTG_ERR_GEOMETRY, "halo: need 0 <= 2 * overlap <= n");
    const size_t m = (size_t)ov * n;
    if (prec == PTG_C64)
        k_halo_pack<float><<<halo_grid(m), 256, 0, s>>>((const float2*)g, n, ov, val, (unsigned char*)buf);
    else
        k_halo_pack<double><<<halo_grid(m), 256, 0, s>>>((const double2*)g, n, ov, val, (unsigned char*)buf);
    PTG_CHECK_LAUNCH();
    count_launch();
}

void dev_halo_unpack(int prec, void* g, int n, int ov, const void* all, int rank, int world, double* val,
                     cudaStream_t s) {
    if (n < 1 || ov < 0 || 2 * (size_t)ov > (size_t)n)   // top and bottom halo rows must not overlap
        raise(PTG_ERR_GEOMETRY, "halo: need 0 <= 2 * overlap <= n");
    if (world < 1 || rank < 0 || rank >= world) raise(PTG_ERR_CONFIG, "halo: bad rank / world size");
    const size_t m = (size_t)ov * n, stride = halo_bytes(prec, n, ov);
    if (prec == PTG_C64)
        k_halo_unpack<float><<<halo_grid(m), 256, 0, s>>>((float2*)g, n, ov, (const unsigned char*)all, stride, rank,
                                                           world, val);
    else
        k_halo_unpack<double><<<halo_grid(m), 256, 0, s>>>((double2*)g, n, ov, (const unsigned char*)all, stride, rank,
                                                            world, val);
    PTG_CHECK_LAUNCH();
    count_launch();
}

}  // namespace ptg
