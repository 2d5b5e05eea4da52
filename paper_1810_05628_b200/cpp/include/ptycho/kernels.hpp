// kernels.hpp — drop-in for /root/reference/proj/include/ptycho/kernels.hpp:
// the 2-D FFT runs on the B200 (ptg_fft2); the reductions are the blocked,
// thread-count-independent sums of kernels.cpp:87-120.
#pragma once

#include <complex>
#include <cstddef>
#include <cstring>
#include <vector>

#include "field.hpp"

namespace ptycho::kernels {

inline constexpr int kOmpMinN = 64;
inline constexpr std::size_t kReduceBlock = detail::kReduceBlock;

inline void fft2_inplace(std::complex<double>* a, int n, bool inverse) {
    std::vector<std::complex<double>> out(static_cast<std::size_t>(n) * n);
    detail::check(ptg_fft2(detail::dp(a), n, inverse ? 1 : 0, detail::dp(out.data())));
    std::memcpy(a, out.data(), out.size() * sizeof(std::complex<double>));
}
inline double norm2sq(const std::complex<double>* a, std::size_t len) {
    return detail::blocked_sum(len, [&](std::size_t i) { return std::norm(a[i]); });
}
inline double dotReal(const std::complex<double>* a, const std::complex<double>* b, std::size_t len) {
    return detail::blocked_sum(len, [&](std::size_t i) { return a[i].real() * b[i].real() + a[i].imag() * b[i].imag(); });
}

}  // namespace ptycho::kernels
