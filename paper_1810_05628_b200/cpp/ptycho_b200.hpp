// ptycho_b200.hpp — C++ drop-in mirror of the reference's public hot-path API
// (/root/reference/proj/include/ptycho/{field,forward,objectives,solvers,
// multigrid,errors}.hpp), implemented over the libptg C-ABI (include/ptg.h).
//
// Same names, argument meaning and error behaviour as the reference:
//   evaluate / phiDistance / phiIntensityGaussian / projectModulus / simulate,
//   pie, lbfgs (GPU-resident for ptychographic objectives), restrictField /
//   prolongField / restrictData, buildHierarchy / mgoptDriver, and the
//   exception hierarchy of errors.hpp.  Value types (ComplexField, RealGrid,
//   ScanGeometry, DiffractionStack, EvalCounter, SolverReport) are layout- and
//   semantics-compatible copies so existing call sites compile unchanged
//   against namespace ptycho_b200.
//
// Every objective evaluation runs on the B200; there is no CPU fallback (a
// missing device throws CudaError).  Header-only; link libptg.so.
#pragma once

#include <complex>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ptg.h"

namespace ptycho_b200 {

// ------------------------------------------------------------ errors.hpp:12-43
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : Error { using Error::Error; };
struct GeometryError : ConfigError { using ConfigError::ConfigError; };
struct DomainError : ConfigError { using ConfigError::ConfigError; };
struct MetricError : ConfigError { using ConfigError::ConfigError; };
struct IoError : Error { using Error::Error; };
struct NumericError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };   // device failure (no CPU fallback)

inline void check(int rc) {
    if (rc == PTG_OK) return;
    const std::string m = ptg_last_error();
    switch (rc) {
        case PTG_ERR_GEOMETRY: throw GeometryError(m);
        case PTG_ERR_DOMAIN: throw DomainError(m);
        case PTG_ERR_METRIC: throw MetricError(m);
        case PTG_ERR_CONFIG: throw ConfigError(m);
        case PTG_ERR_IO: throw IoError(m);
        case PTG_ERR_NUMERIC: throw NumericError(m);
        case PTG_ERR_CUDA: throw CudaError(m);
        default: throw Error(m);
    }
}

// -------------------------------------------------------------- field.hpp:12-85
using cdouble = std::complex<double>;

class ComplexField {
public:
    ComplexField() = default;
    explicit ComplexField(int n, cdouble fill = cdouble{0.0, 0.0})
        : n_(n), v_(static_cast<std::size_t>(n) * static_cast<std::size_t>(n), fill) {
        if (n < 0) throw GeometryError("ComplexField: negative size");
    }
    int n() const { return n_; }
    std::size_t size() const { return v_.size(); }
    cdouble& at(int r, int c) { return v_[static_cast<std::size_t>(r) * n_ + c]; }
    const cdouble& at(int r, int c) const { return v_[static_cast<std::size_t>(r) * n_ + c]; }
    cdouble& operator[](std::size_t i) { return v_[i]; }
    const cdouble& operator[](std::size_t i) const { return v_[i]; }
    cdouble* data() { return v_.data(); }
    const cdouble* data() const { return v_.data(); }

private:
    int n_ = 0;
    std::vector<cdouble> v_;
};

class RealGrid {
public:
    RealGrid() = default;
    explicit RealGrid(int n, double fill = 0.0)
        : n_(n), v_(static_cast<std::size_t>(n) * static_cast<std::size_t>(n), fill) {
        if (n < 0) throw GeometryError("RealGrid: negative size");
    }
    int n() const { return n_; }
    std::size_t size() const { return v_.size(); }
    double& at(int r, int c) { return v_[static_cast<std::size_t>(r) * n_ + c]; }
    const double& at(int r, int c) const { return v_[static_cast<std::size_t>(r) * n_ + c]; }
    double& operator[](std::size_t i) { return v_[i]; }
    const double& operator[](std::size_t i) const { return v_[i]; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }

private:
    int n_ = 0;
    std::vector<double> v_;
};

struct ProbeWindow {
    int row0 = 0, col0 = 0, width = 0;
};

struct ScanGeometry {
    int n = 0, windowSize = 0, stride = 0;
    std::vector<ProbeWindow> windows;
    int probeCount() const { return static_cast<int>(windows.size()); }
};

// field.cpp:62-85 serpentine raster (host-side geometry helper)
inline ScanGeometry generateRasterScan(int n, int windowSize, int stride) {
    if (n < 1 || windowSize < 1 || windowSize > n)
        throw GeometryError("raster scan: need 1 <= windowSize <= n");
    if (stride < 1) throw GeometryError("raster scan: stride must be positive");
    if ((n - windowSize) % stride != 0) throw GeometryError("raster scan: stride must divide n - windowSize");
    if (stride > windowSize) throw GeometryError("raster scan: stride > windowSize leaves coverage gaps");
    const int steps = (n - windowSize) / stride + 1;
    ScanGeometry g{n, windowSize, stride, {}};
    for (int i = 0; i < steps; ++i)
        for (int j = 0; j < steps; ++j) {
            const int jj = (i % 2 == 0) ? j : steps - 1 - j;
            g.windows.push_back(ProbeWindow{i * stride, jj * stride, windowSize});
        }
    return g;
}

struct DiffractionStack {
    int n = 0;
    std::vector<RealGrid> patterns;
    int count() const { return static_cast<int>(patterns.size()); }
};

// ------------------------------------------------------ objectives.hpp:8-44
enum class MetricKind { Distance, IntensityGaussian };

struct ObjectiveEval {
    double value = 0.0;
    ComplexField gradient;
};

// Non-owning, as the reference (objectives.hpp:18-26).  `probe` (M x M,
// optional) selects the patch model; without it the binary-window full-field
// reference model is used (frame M = n).
struct Objective {
    MetricKind kind = MetricKind::Distance;
    const ScanGeometry* geometry = nullptr;
    const DiffractionStack* data = nullptr;
    const ComplexField* shift = nullptr;
    const ComplexField* probe = nullptr;
    int precision = PTG_C128;
};

namespace detail {
struct PlanDeleter {
    void operator()(ptg_plan* p) const { ptg_plan_destroy(p); }
};
using PlanPtr = std::unique_ptr<ptg_plan, PlanDeleter>;

inline int metric_of(MetricKind k) { return k == MetricKind::Distance ? PTG_DISTANCE : PTG_INTENSITY; }

// A plan bound to the objective's CURRENT geometry/data (the reference's
// tests mutate data between calls, objectives.hpp:24, so nothing is cached
// across calls; use ptycho_b200::Plan directly for resident data).
inline PlanPtr make_plan(const Objective& o, int n) {
    if (!o.geometry || !o.data) throw ConfigError("objective is not bound to geometry/data");
    const ScanGeometry& g = *o.geometry;
    const DiffractionStack& d = *o.data;
    if (g.n != n) throw DomainError("scan geometry size mismatch");
    if (d.n != n) throw DomainError("diffraction stack size mismatch");
    if (d.count() != g.probeCount()) throw DomainError("pattern count does not match probe count");
    const int M = o.probe ? o.probe->n() : n;
    const int w = g.windows.empty() ? (o.probe ? M : 1) : g.windows[0].width;
    std::vector<int32_t> pos;
    for (const auto& win : g.windows) {
        if (win.width != w) throw GeometryError("windows of different widths");
        pos.push_back(win.row0);
        pos.push_back(win.col0);
    }
    const std::size_t MM = static_cast<std::size_t>(M) * M;
    std::vector<double> data(MM * d.count());
    for (int k = 0; k < d.count(); ++k) {
        if (d.patterns[k].n() != M) throw DomainError("diffraction pattern size mismatch");
        std::memcpy(data.data() + k * MM, d.patterns[k].data(), MM * sizeof(double));
    }
    ptg_plan_desc desc{};
    desc.n = n;
    desc.M = M;
    desc.w = w;
    desc.N = g.probeCount();
    desc.positions = pos.data();
    desc.probe = o.probe ? reinterpret_cast<const double*>(o.probe->data()) : nullptr;
    desc.data = data.data();
    desc.data_dtype = PTG_F64;
    desc.precision = o.precision;
    desc.device = 0;
    ptg_plan* p = nullptr;
    check(ptg_plan_create(&desc, &p));
    return PlanPtr(p);
}
}  // namespace detail

// objectives.cpp:106-118
inline ObjectiveEval evaluate(const Objective& o, const ComplexField& z) {
    auto plan = detail::make_plan(o, z.n());
    ObjectiveEval ev;
    ev.gradient = ComplexField(z.n());
    if (o.shift && o.shift->n() != z.n()) throw DomainError("dotReal: size mismatch");
    check(ptg_eval(plan.get(), detail::metric_of(o.kind), reinterpret_cast<const double*>(z.data()),
                   o.shift ? reinterpret_cast<const double*>(o.shift->data()) : nullptr, &ev.value,
                   reinterpret_cast<double*>(ev.gradient.data())));
    return ev;
}

inline ObjectiveEval phiDistance(const ComplexField& z, const ScanGeometry& g, const DiffractionStack& d) {
    return evaluate(Objective{MetricKind::Distance, &g, &d, nullptr}, z);
}
inline ObjectiveEval phiIntensityGaussian(const ComplexField& z, const ScanGeometry& g,
                                          const DiffractionStack& d) {
    return evaluate(Objective{MetricKind::IntensityGaussian, &g, &d, nullptr}, z);
}

// objectives.cpp:42-50 (ref model: the projection in object coordinates)
inline ComplexField projectModulus(const ComplexField& z, const ProbeWindow& w, const RealGrid& pattern) {
    ScanGeometry g{z.n(), w.width, w.width, {w}};
    DiffractionStack d{z.n(), {pattern}};
    auto plan = detail::make_plan(Objective{MetricKind::Distance, &g, &d}, z.n());
    ComplexField out(z.n());
    check(ptg_project_modulus(plan.get(), reinterpret_cast<const double*>(z.data()), 0,
                              reinterpret_cast<double*>(out.data())));
    return out;
}

// forward.cpp:40-54 on the GPU
inline DiffractionStack simulate(const ComplexField& object, const ScanGeometry& g) {
    if (object.n() != g.n) throw DomainError("simulate: object size does not match scan geometry");
    DiffractionStack d{g.n, std::vector<RealGrid>(g.probeCount(), RealGrid(g.n))};
    auto plan = detail::make_plan(Objective{MetricKind::Distance, &g, &d}, g.n);
    std::vector<double> out(static_cast<std::size_t>(g.n) * g.n * g.probeCount());
    check(ptg_simulate(plan.get(), reinterpret_cast<const double*>(object.data()), out.data()));
    const std::size_t nn = static_cast<std::size_t>(g.n) * g.n;
    for (int k = 0; k < g.probeCount(); ++k) std::memcpy(d.patterns[k].data(), out.data() + k * nn, nn * 8);
    return d;
}

// ------------------------------------------------------------ solvers.hpp
struct EvalCounter {
    double weightedEvals = 0.0;
    std::map<int, long> perLevelEvals;
    void record(int level, double weight) {
        weightedEvals += weight;
        ++perLevelEvals[level];
    }
};

enum class StopReason { Tolerance, Budget, MaxIters, Stall };

struct HistoryPoint {
    double weightedEvals = 0.0, value = 0.0, gradNorm = 0.0;
};

struct SolverReport {
    ComplexField finalIterate;
    double finalValue = 0.0;
    std::vector<HistoryPoint> history;
    StopReason reason = StopReason::MaxIters;
};

struct SolverConfig {
    int maxIters = 100;
    double gradTolRel = 0.0, gradTolAbs = 1e-13;
    int lbfgsMemory = 25, linesearchMax = 50;
    int cgMaxIters = 20;
    double cgRelTol = 0.1;
    double maxWeightedEvals = std::numeric_limits<double>::infinity();
};

namespace detail {
inline SolverReport report(const ptg_report& r, const std::vector<ptg_hist>& h, ComplexField z,
                           EvalCounter& ctr) {
    SolverReport out;
    out.finalIterate = std::move(z);
    out.finalValue = r.final_value;
    for (int i = 0; i < r.hist_len && i < (int)h.size(); ++i)
        out.history.push_back({h[i].weighted, h[i].value, h[i].gnorm});
    out.reason = static_cast<StopReason>(r.reason);
    for (int l = 0; l < 16; ++l)
        if (r.per_level[l]) ctr.perLevelEvals[l] += r.per_level[l];
    ctr.weightedEvals += r.weighted;
    return out;
}
}  // namespace detail

// solvers.cpp:229-265 (complex probes: Alg. 1 weight)
inline SolverReport pie(const ComplexField& z0, const ScanGeometry& g, const DiffractionStack& d, double gamma,
                        int sweeps, EvalCounter& ctr,
                        double maxWeighted = std::numeric_limits<double>::infinity()) {
    auto plan = detail::make_plan(Objective{MetricKind::Distance, &g, &d}, z0.n());
    ComplexField z = z0;
    std::vector<ptg_hist> h(sweeps + 2);
    int nh = 0, reason = 0;
    double fv = 0.0, wt = 0.0;
    check(ptg_pie(plan.get(), reinterpret_cast<double*>(z.data()), gamma, sweeps, maxWeighted, &fv, h.data(),
                  (int)h.size(), &nh, &wt, &reason));
    ptg_report r{};
    r.final_value = fv;
    r.weighted = wt;
    r.per_level[0] = static_cast<long>(wt);
    r.reason = reason;
    r.hist_len = nh;
    return detail::report(r, h, std::move(z), ctr);
}

namespace detail {
template <class F>
inline SolverReport solve(F fn, const Objective& o, const ComplexField& z0, const SolverConfig& cfg,
                          EvalCounter& ctr) {
    auto plan = make_plan(o, z0.n());
    ptg_solver_cfg c{cfg.maxIters,        cfg.gradTolRel,  cfg.gradTolAbs, cfg.lbfgsMemory,
                     cfg.linesearchMax,   cfg.maxWeightedEvals, cfg.cgMaxIters, cfg.cgRelTol};
    ComplexField z(z0.n()), g(z0.n());
    std::vector<ptg_hist> h(cfg.maxIters + 2);
    ptg_report r{};
    check(fn(plan.get(), metric_of(o.kind), o.shift ? reinterpret_cast<const double*>(o.shift->data()) : nullptr,
             reinterpret_cast<const double*>(z0.data()), &c, reinterpret_cast<double*>(z.data()),
             reinterpret_cast<double*>(g.data()), &r, h.data(), (int)h.size()));
    return report(r, h, std::move(z), ctr);
}
}  // namespace detail

// solvers.cpp:87-141 on the (optionally shifted) ptychographic objective, GPU-resident
inline SolverReport lbfgs(const Objective& o, const ComplexField& z0, const SolverConfig& cfg, EvalCounter& ctr) {
    return detail::solve(ptg_lbfgs, o, z0, cfg, ctr);
}

// solvers.cpp:143-227 (Newton-CG, finite-difference Hessian-vector products), GPU-resident
inline SolverReport truncatedNewton(const Objective& o, const ComplexField& z0, const SolverConfig& cfg,
                                    EvalCounter& ctr) {
    return detail::solve(ptg_truncated_newton, o, z0, cfg, ctr);
}

// ------------------------------------------------------------ multigrid.hpp
inline ComplexField restrictField(const ComplexField& fine) {
    ComplexField c(fine.n() / 2);
    check(ptg_restrict_field(reinterpret_cast<const double*>(fine.data()), fine.n(),
                             reinterpret_cast<double*>(c.data())));
    return c;
}
inline ComplexField prolongField(const ComplexField& coarse) {
    ComplexField f(coarse.n() * 2);
    check(ptg_prolong_field(reinterpret_cast<const double*>(coarse.data()), coarse.n(),
                            reinterpret_cast<double*>(f.data())));
    return f;
}
inline DiffractionStack restrictData(const DiffractionStack& fine) {
    const int n = fine.n, N = fine.count();
    if (n < 4 || n % 4 != 0) throw GeometryError("restrictData: grid side must be a multiple of 4");
    const std::size_t nn = static_cast<std::size_t>(n) * n, hh = nn / 4;
    std::vector<double> in(nn * N), out(hh * N);
    for (int k = 0; k < N; ++k) std::memcpy(in.data() + k * nn, fine.patterns[k].data(), nn * 8);
    check(ptg_restrict_data(in.data(), N, n, out.data()));
    DiffractionStack c{n / 2, std::vector<RealGrid>(N, RealGrid(n / 2))};
    for (int k = 0; k < N; ++k) std::memcpy(c.patterns[k].data(), out.data() + k * hh, hh * 8);
    return c;
}

struct MgoptConfig {
    int k1 = 1, k2 = 1, coarsestMaxIters = 0;
    double coarsestGradTolRel = 1e-4, intermediateGradTolRel = 1e-3;
    int lbfgsMemory = 25, linesearchMax = 50;
    double gradTolAbs = 1e-13;
};

struct MgoptDriverConfig {
    double budgetWeightedEvals = 100.0, gradTolRel = 0.0, gradTolAbs = 1e-13;
    int maxCycles = 1000000;
};

// buildHierarchy (multigrid.hpp:61-62): coarse levels are built on the device
class Hierarchy {
public:
    Hierarchy(const ScanGeometry& g, const DiffractionStack& d, MetricKind kind, int depth,
              const MgoptConfig& opt = {}, const ComplexField* probe = nullptr, int precision = PTG_C128)
        : plan_(detail::make_plan(Objective{kind, &g, &d, nullptr, probe, precision}, g.n)), n_(g.n) {
        ptg_mg_cfg c{opt.k1, opt.k2, opt.coarsestMaxIters, opt.coarsestGradTolRel, opt.intermediateGradTolRel,
                     opt.lbfgsMemory, opt.linesearchMax, opt.gradTolAbs};
        check(ptg_hier_create(plan_.get(), detail::metric_of(kind), depth, &c, &h_));
        depth_ = depth;
    }
    ~Hierarchy() { if (h_) ptg_hier_destroy(h_); }
    Hierarchy(const Hierarchy&) = delete;
    Hierarchy& operator=(const Hierarchy&) = delete;
    int depth() const { return depth_; }
    ptg_hier* handle() const { return h_; }
    int n() const { return n_; }

private:
    detail::PlanPtr plan_;
    ptg_hier* h_ = nullptr;
    int n_ = 0, depth_ = 0;
};

// multigrid.cpp:171-227, GPU-resident
inline SolverReport mgoptDriver(const Hierarchy& h, const ComplexField& z0, const MgoptDriverConfig& cfg,
                                EvalCounter& ctr) {
    if (z0.n() != h.n()) throw DomainError("mgoptDriver: iterate does not match the finest grid");
    ptg_driver_cfg c{cfg.budgetWeightedEvals, cfg.gradTolRel, cfg.gradTolAbs, cfg.maxCycles};
    ComplexField z(z0.n());
    std::vector<ptg_hist> hist(static_cast<std::size_t>(std::min(cfg.maxCycles, 100000)) + 2);
    ptg_report r{};
    check(ptg_mgopt_driver(h.handle(), reinterpret_cast<const double*>(z0.data()), &c,
                           reinterpret_cast<double*>(z.data()), &r, hist.data(), (int)hist.size()));
    return detail::report(r, hist, std::move(z), ctr);
}

}  // namespace ptycho_b200
