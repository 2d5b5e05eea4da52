// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" veneer over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libptycho_ref.so).  It lets the Python tests and the CPU
// baseline call the reference's own phiDistance / projectModulus / pie /
// lbfgs / mgoptDriver / transfer operators in ref mode (binary windows,
// full-field n x n FFTs).  Nothing in the product path links this.
//
// Exceptions are mapped onto the C-ABI status codes of include/ptg.h:
// ConfigError 10, GeometryError 11, DomainError 12, MetricError 13,
// IoError 2, NumericError 3, anything else 5.
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>

#include "ptycho/errors.hpp"
#include "ptycho/field.hpp"
#include "ptycho/forward.hpp"
#include "ptycho/kernels.hpp"
#include "ptycho/metrics.hpp"
#include "ptycho/multigrid.hpp"
#include "ptycho/objectives.hpp"
#include "ptycho/solvers.hpp"

using namespace ptycho;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const GeometryError& e) {
        g_err = e.what();
        return 11;
    } catch (const DomainError& e) {
        g_err = e.what();
        return 12;
    } catch (const MetricError& e) {
        g_err = e.what();
        return 13;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 10;
    } catch (const IoError& e) {
        g_err = e.what();
        return 2;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

ComplexField fieldFrom(const double* a, int n) {
    ComplexField f(n);
    if (a) std::memcpy(f.data(), a, sizeof(double) * 2 * f.size());
    return f;
}

void fieldTo(const ComplexField& f, double* out) {
    std::memcpy(out, f.data(), sizeof(double) * 2 * f.size());
}

// windows: N x 3 int32 (row0, col0, width)
ScanGeometry geometryFrom(int n, int N, const int32_t* win, int stride) {
    ScanGeometry g;
    g.n = n;
    g.windowSize = N > 0 ? win[2] : 0;
    g.stride = stride;
    for (int k = 0; k < N; ++k) g.windows.push_back(ProbeWindow{win[3 * k], win[3 * k + 1], win[3 * k + 2]});
    return g;
}

DiffractionStack stackFrom(int n, int N, const double* d) {
    DiffractionStack s;
    s.n = n;
    const std::size_t nn = static_cast<std::size_t>(n) * n;
    for (int k = 0; k < N; ++k) {
        RealGrid g(n);
        std::memcpy(g.data(), d + k * nn, sizeof(double) * nn);
        s.patterns.push_back(std::move(g));
    }
    return s;
}

void historyTo(const SolverReport& rep, double* hist, int cap, int* nhist) {
    *nhist = static_cast<int>(rep.history.size());
    for (int i = 0; i < *nhist && i < cap; ++i) {
        hist[3 * i] = rep.history[i].weightedEvals;
        hist[3 * i + 1] = rep.history[i].value;
        hist[3 * i + 2] = rep.history[i].gradNorm;
    }
}

int reasonCode(StopReason r) {
    switch (r) {
        case StopReason::Tolerance: return 0;
        case StopReason::Budget: return 1;
        case StopReason::MaxIters: return 2;
        case StopReason::Stall: return 3;
    }
    return -1;
}

}  // namespace

extern "C" {

const char* ptref_last_error() { return g_err.c_str(); }

void ptref_fft2(double* a, int n, int inverse) {
    kernels::fft2_inplace(reinterpret_cast<std::complex<double>*>(a), n, inverse != 0);
}

int ptref_fft2_checked(double* a, int n, int inverse) {
    return guard([&] { kernels::fft2_inplace(reinterpret_cast<std::complex<double>*>(a), n, inverse != 0); });
}

double ptref_norm2sq(const double* a, std::size_t len) {
    return kernels::norm2sq(reinterpret_cast<const std::complex<double>*>(a), len);
}

double ptref_dot_real(const double* a, const double* b, std::size_t len) {
    return kernels::dotReal(reinterpret_cast<const std::complex<double>*>(a),
                            reinterpret_cast<const std::complex<double>*>(b), len);
}

// field.cpp:62-85; writes N x 3 windows, returns count via *count
int ptref_raster(int n, int w, int s, int32_t* win, int cap, int* count) {
    return guard([&] {
        ScanGeometry g = generateRasterScan(n, w, s);
        *count = g.probeCount();
        for (int k = 0; k < g.probeCount() && k < cap; ++k) {
            win[3 * k] = g.windows[k].row0;
            win[3 * k + 1] = g.windows[k].col0;
            win[3 * k + 2] = g.windows[k].width;
        }
    });
}

int ptref_simulate(int n, int N, const int32_t* win, const double* z, double* data) {
    return guard([&] {
        DiffractionStack d = simulate(fieldFrom(z, n), geometryFrom(n, N, win, 1));
        const std::size_t nn = static_cast<std::size_t>(n) * n;
        for (int k = 0; k < N; ++k) std::memcpy(data + k * nn, d.patterns[k].data(), sizeof(double) * nn);
    });
}

int ptref_project_modulus(int n, const int32_t* window, const double* d, const double* z,
                          double* out) {
    return guard([&] {
        RealGrid g(n);
        std::memcpy(g.data(), d, sizeof(double) * g.size());
        ComplexField p = projectModulus(fieldFrom(z, n), ProbeWindow{window[0], window[1], window[2]}, g);
        fieldTo(p, out);
    });
}

// objectives.cpp:106-118
int ptref_evaluate(int metric, int n, int N, const int32_t* win, const double* data,
                   const double* z, const double* v, double* value, double* grad) {
    return guard([&] {
        ScanGeometry geo = geometryFrom(n, N, win, 1);
        DiffractionStack st = stackFrom(n, N, data);
        ComplexField vf;
        if (v) vf = fieldFrom(v, n);
        Objective obj{metric == 0 ? MetricKind::Distance : MetricKind::IntensityGaussian, &geo, &st,
                      v ? &vf : nullptr};
        ObjectiveEval ev = evaluate(obj, fieldFrom(z, n));
        *value = ev.value;
        fieldTo(ev.gradient, grad);
    });
}

int ptref_restrict_field(const double* fine, int n, double* coarse) {
    return guard([&] { fieldTo(restrictField(fieldFrom(fine, n)), coarse); });
}

int ptref_prolong_field(const double* coarse, int nH, double* fine) {
    return guard([&] { fieldTo(prolongField(fieldFrom(coarse, nH)), fine); });
}

int ptref_restrict_data(const double* fine, int N, int n, double* coarse) {
    return guard([&] {
        DiffractionStack s = stackFrom(n, N, fine);
        DiffractionStack c = restrictData(s);
        const std::size_t nn = static_cast<std::size_t>(c.n) * c.n;
        for (int k = 0; k < N; ++k) std::memcpy(coarse + k * nn, c.patterns[k].data(), sizeof(double) * nn);
    });
}

// solvers.cpp:229-265
int ptref_pie(int n, int N, const int32_t* win, const double* data, const double* z0,
              double gamma, int sweeps, double max_weighted, double* z_out, double* final_value,
              double* hist, int hist_cap, int* nhist, double* weighted, int* reason) {
    return guard([&] {
        ScanGeometry geo = geometryFrom(n, N, win, 1);
        DiffractionStack st = stackFrom(n, N, data);
        EvalCounter ctr;
        SolverReport rep = pie(fieldFrom(z0, n), geo, st, gamma, sweeps, ctr, {}, max_weighted);
        fieldTo(rep.finalIterate, z_out);
        *final_value = rep.finalEval.value;
        historyTo(rep, hist, hist_cap, nhist);
        *weighted = ctr.weightedEvals;
        *reason = reasonCode(rep.reason);
    });
}

// solvers.cpp:87-141 on the (optionally v-shifted) ptychographic objective
int ptref_lbfgs(int metric, int n, int N, const int32_t* win, const double* data,
                const double* v, const double* z0, int max_iters, double grad_tol_rel,
                double grad_tol_abs, int memory, int linesearch_max, double max_weighted,
                double* z_out, double* value, double* grad, double* hist, int hist_cap,
                int* nhist, double* weighted, int* reason) {
    return guard([&] {
        ScanGeometry geo = geometryFrom(n, N, win, 1);
        DiffractionStack st = stackFrom(n, N, data);
        ComplexField vf;
        if (v) vf = fieldFrom(v, n);
        Objective obj{metric == 0 ? MetricKind::Distance : MetricKind::IntensityGaussian, &geo, &st,
                      v ? &vf : nullptr};
        SolverConfig cfg;
        cfg.maxIters = max_iters;
        cfg.gradTolRel = grad_tol_rel;
        cfg.gradTolAbs = grad_tol_abs;
        cfg.lbfgsMemory = memory;
        cfg.linesearchMax = linesearch_max;
        cfg.maxWeightedEvals = max_weighted;
        EvalCounter ctr;
        SolverReport rep = lbfgs(counted(obj), fieldFrom(z0, n), cfg, ctr);
        fieldTo(rep.finalIterate, z_out);
        *value = rep.finalEval.value;
        fieldTo(rep.finalEval.gradient, grad);
        historyTo(rep, hist, hist_cap, nhist);
        *weighted = ctr.weightedEvals;
        *reason = reasonCode(rep.reason);
    });
}

// solvers.cpp:143-227 on the (optionally v-shifted) ptychographic objective
int ptref_truncated_newton(int metric, int n, int N, const int32_t* win, const double* data,
                           const double* v, const double* z0, int max_iters, double grad_tol_rel,
                           double grad_tol_abs, int linesearch_max, int cg_max_iters, double cg_rel_tol,
                           double max_weighted, double* z_out, double* value, double* grad, double* hist,
                           int hist_cap, int* nhist, double* weighted, int* reason) {
    return guard([&] {
        ScanGeometry geo = geometryFrom(n, N, win, 1);
        DiffractionStack st = stackFrom(n, N, data);
        ComplexField vf;
        if (v) vf = fieldFrom(v, n);
        Objective obj{metric == 0 ? MetricKind::Distance : MetricKind::IntensityGaussian, &geo, &st,
                      v ? &vf : nullptr};
        SolverConfig cfg;
        cfg.maxIters = max_iters;
        cfg.gradTolRel = grad_tol_rel;
        cfg.gradTolAbs = grad_tol_abs;
        cfg.linesearchMax = linesearch_max;
        cfg.cgMaxIters = cg_max_iters;
        cfg.cgRelTol = cg_rel_tol;
        cfg.maxWeightedEvals = max_weighted;
        EvalCounter ctr;
        SolverReport rep = truncatedNewton(counted(obj), fieldFrom(z0, n), cfg, ctr);
        fieldTo(rep.finalIterate, z_out);
        *value = rep.finalEval.value;
        fieldTo(rep.finalEval.gradient, grad);
        historyTo(rep, hist, hist_cap, nhist);
        *weighted = ctr.weightedEvals;
        *reason = reasonCode(rep.reason);
    });
}

// multigrid.cpp:95-227 on a raster geometry (n, w, s)
int ptref_mgopt(int metric, int n, int w, int s, const double* data, int depth, int k1, int k2,
                int coarsest_max_iters, double budget, double grad_tol_rel, double grad_tol_abs,
                int max_cycles, const double* z0, double* z_out, double* value, double* hist,
                int hist_cap, int* nhist, double* weighted, long* per_level, int* reason) {
    return guard([&] {
        ScanGeometry geo = generateRasterScan(n, w, s);
        DiffractionStack st = stackFrom(n, geo.probeCount(), data);
        MgoptConfig opt;
        opt.k1 = k1;
        opt.k2 = k2;
        opt.coarsestMaxIters = coarsest_max_iters;
        Hierarchy h = buildHierarchy(geo, st, metric == 0 ? MetricKind::Distance
                                                          : MetricKind::IntensityGaussian,
                                     depth, opt);
        MgoptDriverConfig dc;
        dc.budgetWeightedEvals = budget;
        dc.gradTolRel = grad_tol_rel;
        dc.gradTolAbs = grad_tol_abs;
        dc.maxCycles = max_cycles;
        EvalCounter ctr;
        SolverReport rep = mgoptDriver(h, fieldFrom(z0, n), dc, ctr);
        fieldTo(rep.finalIterate, z_out);
        *value = rep.finalEval.value;
        historyTo(rep, hist, hist_cap, nhist);
        *weighted = ctr.weightedEvals;
        for (int l = 0; l < depth; ++l) {
            auto it = ctr.perLevelEvals.find(l);
            per_level[l] = it == ctr.perLevelEvals.end() ? 0 : it->second;
        }
        *reason = reasonCode(rep.reason);
    });
}

// metrics.cpp:67-136 (diagnostics): out = {relativeError, magnitudeRelError, phaseSSIM}
int ptref_metrics(int n, const double* z, const double* z_true, double* out) {
    return guard([&] {
        const ComplexField a = fieldFrom(z, n), b = fieldFrom(z_true, n);
        out[0] = relativeError(a, b);
        out[1] = magnitudeRelError(a, b);
        out[2] = phaseSSIM(a, b);
    });
}

int ptref_canonical_phase(int n, const double* z, double* out) {
    return guard([&] {
        const RealGrid p = canonicalPhase(fieldFrom(z, n));
        for (std::size_t i = 0; i < p.size(); ++i) out[i] = p[i];
    });
}

}  // extern "C"

// ---- noise (forward.cpp:56-86, rng.hpp:14-24), for pinning ptg_add_noise
extern "C" {
// addNoise on N patterns of side m (RealGrid m x m): out = the reference's
// max(d + eps, 0) with a std::mt19937_64 engine seeded by `seed`
int ptref_add_noise(int N, int m, const double* data, double level, uint64_t seed, double* out) {
    return guard([&] {
        DiffractionStack d;
        d.n = m;
        const std::size_t mm = static_cast<std::size_t>(m) * m;
        for (int k = 0; k < N; ++k) {
            RealGrid g(m);
            std::memcpy(g.data(), data + k * mm, sizeof(double) * mm);
            d.patterns.push_back(std::move(g));
        }
        NoiseSpec spec;
        spec.level = level;
        spec.seed = seed;
        DiffractionStack o = addNoise(d, spec);
        for (int k = 0; k < N; ++k) std::memcpy(out + k * mm, o.patterns[k].data(), sizeof(double) * mm);
    });
}
// the first `count` rng::uniform01 draws of std::mt19937_64(seed)
int ptref_uniform_stream(uint64_t seed, std::size_t count, double* out) {
    return guard([&] {
        rng::Engine eng(seed);
        for (std::size_t i = 0; i < count; ++i) out[i] = rng::uniform01(eng);
    });
}
}
