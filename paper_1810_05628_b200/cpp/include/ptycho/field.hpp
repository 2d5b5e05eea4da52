// field.hpp — drop-in for /root/reference/proj/include/ptycho/field.hpp:12-85.
//
// Value types with the reference's layout and semantics (row-major n x n,
// std::complex<double> interleaved -- what libptg's host buffers take) and
// the host-side helpers of field.cpp (windows, raster scans, the blocked
// deterministic reductions of kernels.cpp:87-120, element-wise algebra).
// fft2 / ifft2 run on the B200 (ptg_fft2: the objective kernels' own 2-D FFT).
#pragma once

#include <cmath>
#include <complex>
#include <cstddef>
#include <string>
#include <vector>

#include "detail/status.hpp"
#include "errors.hpp"

namespace ptycho {

using cdouble = std::complex<double>;

class ComplexField {
public:
    ComplexField() = default;
    explicit ComplexField(int n, cdouble fill = cdouble{0.0, 0.0}) : n_(n) {
        if (n < 0) throw GeometryError("ComplexField: negative size");
        v_.assign(static_cast<std::size_t>(n) * static_cast<std::size_t>(n), fill);
    }
    int n() const { return n_; }
    std::size_t size() const { return v_.size(); }
    cdouble& at(int row, int col) { return v_[static_cast<std::size_t>(row) * n_ + col]; }
    const cdouble& at(int row, int col) const { return v_[static_cast<std::size_t>(row) * n_ + col]; }
    cdouble& operator[](std::size_t i) { return v_[i]; }
    const cdouble& operator[](std::size_t i) const { return v_[i]; }
    cdouble* data() { return v_.data(); }
    const cdouble* data() const { return v_.data(); }
    bool isFinite() const {
        for (const cdouble& x : v_)
            if (!std::isfinite(x.real()) || !std::isfinite(x.imag())) return false;
        return true;
    }

private:
    int n_ = 0;
    std::vector<cdouble> v_;
};

class RealGrid {
public:
    RealGrid() = default;
    explicit RealGrid(int n, double fill = 0.0) : n_(n) {
        if (n < 0) throw GeometryError("RealGrid: negative size");
        v_.assign(static_cast<std::size_t>(n) * static_cast<std::size_t>(n), fill);
    }
    int n() const { return n_; }
    std::size_t size() const { return v_.size(); }
    double& at(int row, int col) { return v_[static_cast<std::size_t>(row) * n_ + col]; }
    const double& at(int row, int col) const { return v_[static_cast<std::size_t>(row) * n_ + col]; }
    double& operator[](std::size_t i) { return v_[i]; }
    const double& operator[](std::size_t i) const { return v_[i]; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    bool isFinite() const {
        for (double x : v_)
            if (!std::isfinite(x)) return false;
        return true;
    }

private:
    int n_ = 0;
    std::vector<double> v_;
};

struct ProbeWindow {
    int row0 = 0;
    int col0 = 0;
    int width = 0;
    bool contains(int row, int col) const {
        return row >= row0 && row < row0 + width && col >= col0 && col < col0 + width;
    }
};

struct ScanGeometry {
    int n = 0;
    int windowSize = 0;
    int stride = 0;
    std::vector<ProbeWindow> windows;
    int probeCount() const { return static_cast<int>(windows.size()); }
};

namespace detail {
inline ComplexField fft2_dev(const ComplexField& f, bool inverse) {
    ComplexField out(f.n());
    check(ptg_fft2(dp(f.data()), f.n(), inverse ? 1 : 0, dp(out.data())));
    return out;
}
inline void check_window(int n, const ProbeWindow& w) {
    if (w.width < 1 || w.row0 < 0 || w.col0 < 0 || w.row0 + w.width > n || w.col0 + w.width > n)
        throw GeometryError("probe window [" + std::to_string(w.row0) + "," + std::to_string(w.col0) + ")+" +
                            std::to_string(w.width) + " does not fit an n=" + std::to_string(n) + " grid");
}
// kernels.cpp:87-120: 1024-element blocks, block partials summed in order
constexpr std::size_t kReduceBlock = 1024;
template <class F>
inline double blocked_sum(std::size_t len, F term) {
    double total = 0.0;
    for (std::size_t lo = 0; lo < len; lo += kReduceBlock) {
        const std::size_t hi = lo + kReduceBlock < len ? lo + kReduceBlock : len;
        double s = 0.0;
        for (std::size_t i = lo; i < hi; ++i) s += term(i);
        total += s;
    }
    return total;
}
inline void same_size(const ComplexField& a, const ComplexField& b, const char* what) {
    if (a.n() != b.n()) throw DomainError(std::string(what) + ": size mismatch");
}
}  // namespace detail

// unnormalised forward DFT / inverse with 1/n^2, on the GPU
inline ComplexField fft2(const ComplexField& field) { return detail::fft2_dev(field, false); }
inline ComplexField ifft2(const ComplexField& field) { return detail::fft2_dev(field, true); }

// pixels inside the window copied, zero elsewhere
inline ComplexField applyProbe(const ComplexField& field, const ProbeWindow& w) {
    detail::check_window(field.n(), w);
    ComplexField out(field.n());
    for (int r = w.row0; r < w.row0 + w.width; ++r)
        for (int c = w.col0; c < w.col0 + w.width; ++c) out.at(r, c) = field.at(r, c);
    return out;
}

// serpentine raster: rows top to bottom, direction alternating per row
inline ScanGeometry generateRasterScan(int n, int windowSize, int stride) {
    if (n < 1 || windowSize < 1 || windowSize > n) throw GeometryError("raster scan: need 1 <= windowSize <= n");
    if (stride < 1) throw GeometryError("raster scan: stride must be positive");
    if ((n - windowSize) % stride != 0) throw GeometryError("raster scan: stride must divide n - windowSize");
    if (stride > windowSize) throw GeometryError("raster scan: stride > windowSize leaves coverage gaps");
    const int steps = (n - windowSize) / stride + 1;
    ScanGeometry g;
    g.n = n;
    g.windowSize = windowSize;
    g.stride = stride;
    for (int i = 0; i < steps; ++i)
        for (int j = 0; j < steps; ++j)
            g.windows.push_back(ProbeWindow{i * stride, (i % 2 ? steps - 1 - j : j) * stride, windowSize});
    return g;
}

inline double norm2sq(const ComplexField& a) {
    return detail::blocked_sum(a.size(), [&](std::size_t i) { return std::norm(a[i]); });
}
inline double norm2(const ComplexField& a) { return std::sqrt(norm2sq(a)); }
inline double dotReal(const ComplexField& a, const ComplexField& b) {
    detail::same_size(a, b, "dotReal");
    return detail::blocked_sum(a.size(), [&](std::size_t i) { return a[i].real() * b[i].real() + a[i].imag() * b[i].imag(); });
}
inline ComplexField add(const ComplexField& a, const ComplexField& b) {
    detail::same_size(a, b, "add");
    ComplexField out = a;
    for (std::size_t i = 0; i < out.size(); ++i) out[i] += b[i];
    return out;
}
inline ComplexField sub(const ComplexField& a, const ComplexField& b) {
    detail::same_size(a, b, "sub");
    ComplexField out = a;
    for (std::size_t i = 0; i < out.size(); ++i) out[i] -= b[i];
    return out;
}
inline ComplexField scaled(const ComplexField& a, double alpha) {
    ComplexField out = a;
    for (std::size_t i = 0; i < out.size(); ++i) out[i] *= alpha;
    return out;
}
inline void axpy(ComplexField& y, double alpha, const ComplexField& x) {
    detail::same_size(y, x, "axpy");
    for (std::size_t i = 0; i < y.size(); ++i) y[i] += alpha * x[i];
}

}  // namespace ptycho
