// test_dropin_ext.cpp — the drop-in's ADDITIVE surface on the B200, beyond
// what the reference's own unit tests (run unmodified by ref_tests_dropin)
// cover: patch-model objectives (complex probe, Objective::probe), complex64
// plans (Objective::precision), the GPU-resident solvers with callbacks and
// warm starts on ptychographic objectives, coarse-level V-cycles with a
// shift, the device FFT against a brute-force DFT.
#include <cmath>
#include <cstdio>

#include "doctest.h"
#include "ptycho_b200.hpp"

using namespace ptycho;

namespace {
ComplexField field(int n, std::uint64_t seed, double scale = 1.0) {
    rng::Engine eng(seed);
    ComplexField z(n);
    for (std::size_t i = 0; i < z.size(); ++i)
        z[i] = cdouble{scale * (2 * rng::uniform01(eng) - 1), scale * (2 * rng::uniform01(eng) - 1)};
    return z;
}
double relDiff(const ComplexField& a, const ComplexField& b) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num += std::norm(a[i] - b[i]);
        den += std::norm(b[i]);
    }
    return std::sqrt(num / (den > 0 ? den : 1));
}
}  // namespace

TEST_CASE("device fft2 matches a brute-force DFT and inverts") {
    const int n = 16;
    const ComplexField x = field(n, 1);
    ComplexField want(n);
    for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v)
            for (int r = 0; r < n; ++r)
                for (int c = 0; c < n; ++c)
                    want.at(u, v) += x.at(r, c) * std::polar(1.0, -6.283185307179586 * (double(u) * r + double(v) * c) / n);
    CHECK(relDiff(fft2(x), want) < 1e-13);
    CHECK(relDiff(ifft2(fft2(x)), x) < 1e-14);
    ComplexField y = x;
    kernels::fft2_inplace(y.data(), n, false);
    CHECK(relDiff(y, want) < 1e-13);
}

TEST_CASE("patch model: complex probe, complex64 plan close to complex128") {
    const int n = 48, M = 16;
    const ScanGeometry g = generateRasterScan(n, M, 8);
    const ComplexField truth = field(n, 2), probe = field(M, 3);
    ComplexField z = truth;
    for (std::size_t i = 0; i < z.size(); ++i) z[i] *= 0.9;
    // data of the patch model: the plan's own forward operator (c128)
    DiffractionStack d{n, std::vector<RealGrid>(g.probeCount(), RealGrid(M))};
    Objective o{MetricKind::Distance, &g, &d, nullptr, &probe, PTG_C128};
    {
        ptg_plan_desc desc{};
        std::vector<int32_t> pos;
        for (auto& w : g.windows) pos.insert(pos.end(), {w.row0, w.col0});
        desc.n = n; desc.M = M; desc.w = M; desc.N = g.probeCount(); desc.positions = pos.data();
        desc.probe = reinterpret_cast<const double*>(probe.data()); desc.precision = PTG_C128;
        ptg_plan* p = nullptr;
        REQUIRE(ptg_plan_create(&desc, &p) == PTG_OK);
        std::vector<double> out(static_cast<std::size_t>(M) * M * g.probeCount());
        REQUIRE(ptg_simulate(p, reinterpret_cast<const double*>(truth.data()), out.data()) == PTG_OK);
        for (int k = 0; k < g.probeCount(); ++k)
            std::memcpy(d.patterns[k].data(), out.data() + (std::size_t)k * M * M, M * M * 8);
        ptg_plan_destroy(p);
    }
    const ObjectiveEval e128 = evaluate(o, z);
    o.precision = PTG_C64;
    const ObjectiveEval e64 = evaluate(o, z);
    CHECK(std::fabs(e64.value - e128.value) <= 1e-5 * e128.value);
    CHECK(relDiff(e64.gradient, e128.gradient) <= 1e-4);
    o.precision = PTG_C128;
    CHECK(evaluate(o, truth).value <= 1e-20);   // the plan's forward model is consistent
}

TEST_CASE("GPU-resident lbfgs: callback, warm start, accounting at the objective's level") {
    const int n = 32;
    const ScanGeometry g = generateRasterScan(n, n / 2, n / 4);
    const DiffractionStack d = simulate(field(n, 4), g);
    const Objective o{MetricKind::Distance, &g, &d, nullptr};
    const CountedObjective obj = counted(o, 2, 0.0625);
    SolverConfig cfg;
    cfg.maxIters = 6;
    EvalCounter ctr;
    ctr.record(0, 1.0);   // a prior charge: history must continue from it
    std::vector<int> seen;
    std::vector<double> vals;
    const ComplexField z0 = field(n, 5, 0.5);
    const SolverReport rep = lbfgs(obj, z0, cfg, ctr, [&](int it, const ComplexField& z, double v, double w) {
        seen.push_back(it);
        vals.push_back(v);
        CHECK(z.n() == n);
        CHECK(w >= 1.0);
    });
    REQUIRE(seen.size() == rep.history.size());
    for (std::size_t i = 0; i < seen.size(); ++i) {
        CHECK(seen[i] == (int)i);
        CHECK(vals[i] == rep.history[i].value);
    }
    CHECK(ctr.perLevelEvals.at(2) > 0);
    CHECK(ctr.weightedEvals == 1.0 + 0.0625 * ctr.perLevelEvals.at(2));
    CHECK(rep.history.front().weightedEvals == 1.0 + 0.0625);
    // warm start: the initial evaluation is not charged again
    const ObjectiveEval ev = evaluate(o, z0);
    EvalCounter c2;
    cfg.maxIters = 0;
    lbfgs(obj, z0, cfg, c2, {}, &ev);
    CHECK(c2.weightedEvals == 0.0);
    CHECK(c2.perLevelEvals.empty());
}

TEST_CASE("pie callback per sweep and coarse V-cycle with a shift") {
    const int n = 32;
    const ScanGeometry g = generateRasterScan(n, n / 2, n / 4);
    const DiffractionStack d = simulate(field(n, 6), g);
    int calls = 0;
    EvalCounter ctr;
    const SolverReport rep = pie(field(n, 7, 0.5), g, d, 0.0, 3, ctr,
                                 [&](int, const ComplexField&, double, double) { ++calls; });
    CHECK(calls == 4);
    CHECK(ctr.weightedEvals == 3.0);
    CHECK(rep.history.back().value <= rep.history.front().value);
    const Hierarchy h = buildHierarchy(g, d, MetricKind::Distance, 2);
    const ComplexField zc = field(n / 2, 8, 0.5), vc = field(n / 2, 9, 0.01);
    EvalCounter c2;
    const CycleResult res = mgoptCycle(h, 1, zc, vc, c2);
    const Objective shifted{MetricKind::Distance, &h.levels[1].geometry, &h.levels[1].data, &vc};
    CHECK(std::fabs(evaluate(shifted, res.z).value - res.eval.value) <= 1e-10 * std::fabs(res.eval.value));
    CHECK(res.eval.value <= evaluate(shifted, zc).value);
    CHECK(c2.perLevelEvals.count(1) == 1);
    CHECK(c2.weightedEvals == 0.25 * c2.perLevelEvals.at(1));
}

int main() { return doctest::run_all(); }
