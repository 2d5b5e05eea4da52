// forward.hpp — drop-in for /root/reference/proj/include/ptycho/forward.hpp.
// simulate and addNoise run on the B200 (ptg_simulate, ptg_add_noise fed the
// reference engine's own uniform stream, so results follow std::mt19937_64
// exactly); buildGroundTruth / noisePerturbation / randomInitialGuess are
// host-side set-up helpers with the reference's semantics.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "detail/plan.hpp"
#include "field.hpp"
#include "rng.hpp"

namespace ptycho {

struct GroundTruth {
    ComplexField object;
    double magnitudeMin = 0.0;
    double magnitudeMax = 1.0;
};

struct DiffractionStack {
    int n = 0;
    std::vector<RealGrid> patterns;
    int count() const { return static_cast<int>(patterns.size()); }
};

struct NoiseSpec {
    double level = 0.0;
    std::uint64_t seed = 0;
};

// magnitudes min-max mapped onto [0, 1], phases onto [0, pi/2]
inline GroundTruth buildGroundTruth(const RealGrid& magnitude, const RealGrid& phase) {
    if (magnitude.n() != phase.n()) throw DomainError("buildGroundTruth: magnitude and phase sizes differ");
    if (magnitude.n() < 1) throw DomainError("buildGroundTruth: empty source images");
    if (!magnitude.isFinite() || !phase.isFinite()) throw DomainError("buildGroundTruth: source images must be finite");
    const auto [m0, m1] = std::minmax_element(magnitude.data(), magnitude.data() + magnitude.size());
    const auto [p0, p1] = std::minmax_element(phase.data(), phase.data() + phase.size());
    GroundTruth t;
    t.object = ComplexField(magnitude.n());
    t.magnitudeMin = *m1 > *m0 ? 0.0 : 1.0;
    t.magnitudeMax = 1.0;
    for (std::size_t i = 0; i < magnitude.size(); ++i) {
        const double m = *m1 > *m0 ? (magnitude[i] - *m0) / (*m1 - *m0) : 1.0;
        const double p = *p1 > *p0 ? (phase[i] - *p0) / (*p1 - *p0) * 1.5707963267948966192313216916398 : 0.0;
        t.object[i] = std::polar(m, p);
    }
    return t;
}

namespace detail {
inline PlanSource source_of(const ScanGeometry& g, const DiffractionStack& d, const ComplexField* probe, int precision) {
    PlanSource s;
    s.n = g.n;
    s.M = probe ? probe->n() : g.n;
    s.w = g.windows.empty() ? (probe ? s.M : 1) : g.windows[0].width;
    s.probe = probe;
    s.precision = precision;
    for (const ProbeWindow& w : g.windows) {
        if (w.width != s.w) throw GeometryError("windows of different widths");
        s.pos.push_back(w.row0);
        s.pos.push_back(w.col0);
    }
    for (const RealGrid& p : d.patterns) {
        if (p.n() != s.M) throw DomainError("diffraction pattern size mismatch");
        s.patterns.push_back(&p);
    }
    return s;
}
}  // namespace detail

// d_k = |fft2(Q_k object)|^2 per window, in scan order (on the GPU)
inline DiffractionStack simulate(const ComplexField& object, const ScanGeometry& g) {
    if (object.n() != g.n) throw DomainError("simulate: object size does not match scan geometry");
    DiffractionStack d;
    d.n = g.n;
    d.patterns.assign(g.probeCount(), RealGrid(g.n));
    if (g.probeCount() == 0) return d;
    auto plan = detail::make_plan(detail::source_of(g, d, nullptr, PTG_C128));   // simulate rewrites its data
    std::vector<double> out(static_cast<std::size_t>(g.n) * g.n * g.probeCount());
    detail::check(ptg_simulate(plan.get(), detail::dp(object.data()), out.data()));
    const std::size_t nn = static_cast<std::size_t>(g.n) * g.n;
    for (int k = 0; k < g.probeCount(); ++k) std::memcpy(d.patterns[k].data(), out.data() + k * nn, nn * 8);
    return d;
}

// eps = level ||d|| / ||g|| g, g drawn row-major from eng (host helper)
inline RealGrid noisePerturbation(const RealGrid& pattern, double level, rng::Engine& eng) {
    if (level < 0.0) throw DomainError("noise level must be non-negative");
    RealGrid g(pattern.n());
    for (std::size_t i = 0; i < g.size(); ++i) g[i] = rng::gaussian(eng);
    double dd = 0.0, gg = 0.0;
    for (std::size_t i = 0; i < g.size(); ++i) {
        dd += pattern[i] * pattern[i];
        gg += g[i] * g[i];
    }
    const double sc = gg > 0.0 ? level * std::sqrt(dd) / std::sqrt(gg) : 0.0;
    for (std::size_t i = 0; i < g.size(); ++i) g[i] *= sc;
    return g;
}

// max(d + eps, 0) per pattern, one engine seeded from spec.seed (on the GPU,
// fed that engine's uniforms)
inline DiffractionStack addNoise(const DiffractionStack& data, const NoiseSpec& spec) {
    if (spec.level < 0.0) throw DomainError("noise level must be non-negative");
    DiffractionStack out;
    out.n = data.n;
    if (data.patterns.empty()) return out;
    const int m = data.patterns[0].n();
    const std::size_t mm = static_cast<std::size_t>(m) * m;
    ScanGeometry g;
    g.n = m;
    g.windowSize = m;
    g.stride = m;
    g.windows.assign(data.patterns.size(), ProbeWindow{0, 0, m});
    DiffractionStack flat;
    flat.n = m;
    flat.patterns = data.patterns;
    auto plan = detail::make_plan(detail::source_of(g, flat, nullptr, PTG_C128));   // rewritten in place
    std::vector<double> uni(2 * mm * data.patterns.size());
    rng::Engine eng(spec.seed);
    for (double& u : uni) u = rng::uniform01(eng);
    detail::check(ptg_add_noise(plan.get(), spec.level, spec.seed, uni.data()));
    std::vector<double> res(mm * data.patterns.size());
    detail::check(ptg_plan_get_data(plan.get(), PTG_INTENSITY, res.data()));
    out.patterns.assign(data.patterns.size(), RealGrid(m));
    for (std::size_t k = 0; k < data.patterns.size(); ++k) std::memcpy(out.patterns[k].data(), res.data() + k * mm, mm * 8);
    return out;
}

// real and imaginary parts i.i.d. uniform on [0, 1), row-major (re then im)
inline ComplexField randomInitialGuess(int n, std::uint64_t seed) {
    rng::Engine eng(seed);
    ComplexField z(n);
    for (std::size_t i = 0; i < z.size(); ++i) {
        const double re = rng::uniform01(eng);
        const double im = rng::uniform01(eng);
        z[i] = cdouble{re, im};
    }
    return z;
}

}  // namespace ptycho
