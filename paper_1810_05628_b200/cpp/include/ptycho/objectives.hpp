// objectives.hpp — drop-in for /root/reference/proj/include/ptycho/objectives.hpp.
//
// evaluate / phiDistance / phiIntensityGaussian / projectModulus run on the
// B200 (ptg_eval / ptg_project_modulus on a resident plan, detail/plan.hpp).
// Additive extension for the patch model: Objective::probe (M x M complex
// probe; frames of side M, windows of width w <= M) and Objective::precision
// (PTG_C128 by default = the reference's arithmetic; PTG_C64 for speed).
#pragma once

#include <string>

#include "detail/plan.hpp"
#include "field.hpp"
#include "forward.hpp"

namespace ptycho {

enum class MetricKind {
    Distance,           // 1/2 sum_k || P_k(z) - Q_k z ||^2
    IntensityGaussian,  // 1/2 sum_k || |F(Q_k z)|^2 - d_k ||^2
};

struct ObjectiveEval {
    double value = 0.0;
    ComplexField gradient;
};

// non-owning (pointees must outlive the objective), as the reference
struct Objective {
    MetricKind kind = MetricKind::Distance;
    const ScanGeometry* geometry = nullptr;
    const DiffractionStack* data = nullptr;
    const ComplexField* shift = nullptr;   // v, optional
    const ComplexField* probe = nullptr;   // patch model (extension), optional
    int precision = PTG_C128;              // extension
};

namespace detail {
inline int metric_of(MetricKind k) { return k == MetricKind::Distance ? PTG_DISTANCE : PTG_INTENSITY; }

// objectives.cpp:20-26 checks, then the resident plan of (geometry, data, probe)
inline PlanPtr objective_plan(const Objective& o, int n) {
    if (!o.geometry || !o.data) throw ConfigError("objective is not bound to geometry/data");
    if (o.geometry->n != n) throw DomainError("scan geometry size mismatch");
    if (o.data->n != n) throw DomainError("diffraction stack size mismatch");
    if (o.data->count() != o.geometry->probeCount()) throw DomainError("pattern count does not match probe count");
    return cached_plan(source_of(*o.geometry, *o.data, o.probe, o.precision));
}
}  // namespace detail

// value + descent-convention gradient, shift applied if present (on the GPU)
inline ObjectiveEval evaluate(const Objective& o, const ComplexField& z) {
    auto plan = detail::objective_plan(o, z.n());
    if (o.shift && o.shift->n() != z.n()) throw DomainError("dotReal: size mismatch");
    ObjectiveEval ev;
    ev.gradient = ComplexField(z.n());
    detail::check(ptg_eval(plan.get(), detail::metric_of(o.kind), detail::dp(z.data()),
                           o.shift ? detail::dp(o.shift->data()) : nullptr, &ev.value, detail::dp(ev.gradient.data())));
    return ev;
}

inline ObjectiveEval phiDistance(const ComplexField& z, const ScanGeometry& g, const DiffractionStack& d) {
    return evaluate(Objective{MetricKind::Distance, &g, &d, nullptr}, z);
}
inline ObjectiveEval phiIntensityGaussian(const ComplexField& z, const ScanGeometry& g, const DiffractionStack& d) {
    return evaluate(Objective{MetricKind::IntensityGaussian, &g, &d, nullptr}, z);
}

// ifft2( sqrt(d) W / |W| ), W = fft2(Q z), vanishing W -> sqrt(d) (on the GPU)
inline ComplexField projectModulus(const ComplexField& z, const ProbeWindow& window, const RealGrid& pattern) {
    if (pattern.n() != z.n()) throw DomainError("diffraction pattern size mismatch");
    for (std::size_t i = 0; i < pattern.size(); ++i)
        if (pattern[i] < 0.0)
            throw DomainError("diffraction pattern has a negative intensity at index " + std::to_string(i));
    detail::check_window(z.n(), window);
    ScanGeometry g;
    g.n = z.n();
    g.windowSize = window.width;
    g.stride = window.width;
    g.windows = {window};
    DiffractionStack d;
    d.n = z.n();
    d.patterns = {pattern};
    auto plan = detail::cached_plan(detail::source_of(g, d, nullptr, PTG_C128));
    ComplexField out(z.n());
    detail::check(ptg_project_modulus(plan.get(), detail::dp(z.data()), 0, detail::dp(out.data())));
    return out;
}

}  // namespace ptycho
