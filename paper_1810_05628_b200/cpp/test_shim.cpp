// test_shim.cpp — reference-style C++ tests of the drop-in (ptycho_b200.hpp)
// running on the B200.  Cases mirror /root/reference/proj/tests/
// test_objectives.cpp, test_solvers.cpp and test_multigrid.cpp (same names and
// assertions), with GPU floating-point tolerances where the reference checks
// bitwise equality of its own serial FFT.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "ptycho_b200.hpp"

using namespace ptycho_b200;

static int g_fail = 0, g_checks = 0;
static std::vector<std::pair<std::string, std::function<void()>>>& cases() {
    static std::vector<std::pair<std::string, std::function<void()>>> c;
    return c;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { cases().emplace_back(n, std::move(f)); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name) \
    static void CAT(tc_, __LINE__)(); \
    static Reg CAT(reg_, __LINE__)(name, CAT(tc_, __LINE__)); \
    static void CAT(tc_, __LINE__)()
#define CHECK(cond) \
    do { \
        ++g_checks; \
        if (!(cond)) { ++g_fail; std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); } \
    } while (0)
#define CHECK_THROWS_AS(expr, T) \
    do { \
        ++g_checks; \
        bool ok_ = false; \
        try { expr; } catch (const T&) { ok_ = true; } catch (...) {} \
        if (!ok_) { ++g_fail; std::printf("  FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); } \
    } while (0)

// test_support.hpp analogues
static ComplexField randomField(int n, uint64_t seed, double scale = 1.0) {
    std::mt19937_64 eng(seed);
    auto u = [&] { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
    ComplexField z(n);
    for (std::size_t i = 0; i < z.size(); ++i) z[i] = cdouble{scale * (2 * u() - 1), scale * (2 * u() - 1)};
    return z;
}
static ComplexField dftBrute(const ComplexField& x) {   // forward, unnormalised
    const int n = x.n();
    ComplexField out(n);
    for (int u = 0; u < n; ++u)
        for (int v = 0; v < n; ++v) {
            cdouble acc{0, 0};
            for (int r = 0; r < n; ++r)
                for (int c = 0; c < n; ++c)
                    acc += x.at(r, c) * std::polar(1.0, -6.283185307179586 * (double(u) * r + double(v) * c) / n);
            out.at(u, v) = acc;
        }
    return out;
}
static ComplexField applyWindow(const ComplexField& z, const ProbeWindow& w) {
    ComplexField o(z.n());
    for (int r = w.row0; r < w.row0 + w.width; ++r)
        for (int c = w.col0; c < w.col0 + w.width; ++c) o.at(r, c) = z.at(r, c);
    return o;
}
static double maxAbsDiff(const ComplexField& a, const ComplexField& b) {
    double m = 0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}
static double dotReal(const ComplexField& a, const ComplexField& b) {
    double s = 0;
    for (std::size_t i = 0; i < a.size(); ++i) s += a[i].real() * b[i].real() + a[i].imag() * b[i].imag();
    return s;
}
static double norm2(const ComplexField& a) { return std::sqrt(dotReal(a, a)); }
static bool near(double a, double b, double rel) { return std::abs(a - b) <= rel * std::max(std::abs(b), 1e-300); }

TEST_CASE("projectModulus lands on the modulus constraint set") {
    const int n = 16;
    const ComplexField z = randomField(n, 11);
    const ScanGeometry geo = generateRasterScan(n, n / 2, n / 4);
    RealGrid d(n);
    for (std::size_t i = 0; i < d.size(); ++i) d[i] = 0.5 + 0.01 * static_cast<double>(i);
    const ComplexField pf = dftBrute(projectModulus(z, geo.windows[3], d));
    for (std::size_t i = 0; i < pf.size(); ++i) CHECK(near(std::abs(pf[i]), std::sqrt(d[i]), 1e-11));
}

TEST_CASE("projectModulus fixes data-consistent iterates") {
    const int n = 16;
    const ComplexField z = randomField(n, 12);
    const ScanGeometry geo = generateRasterScan(n, n / 2, n / 4);
    const DiffractionStack data = simulate(z, geo);
    for (int k = 0; k < geo.probeCount(); ++k)
        CHECK(maxAbsDiff(projectModulus(z, geo.windows[k], data.patterns[k]), applyWindow(z, geo.windows[k])) <= 1e-12);
}

TEST_CASE("distance objective matches the frequency-space oracle per probe") {
    const int n = 16;
    const ComplexField z = randomField(n, 14);
    const ScanGeometry geo = generateRasterScan(n, n / 2, n / 4);
    const DiffractionStack data = simulate(randomField(n, 15), geo);
    for (int k = 0; k < geo.probeCount(); ++k) {
        ScanGeometry one{n, geo.windowSize, geo.windowSize, {geo.windows[k]}};
        DiffractionStack od{n, {data.patterns[k]}};
        const ComplexField W = dftBrute(applyWindow(z, geo.windows[k]));
        double want = 0;
        for (std::size_t i = 0; i < W.size(); ++i) {
            const double df = std::abs(W[i]) - std::sqrt(data.patterns[k][i]);
            want += df * df;
        }
        want /= 2.0 * n * n;
        const double got = phiDistance(z, one, od).value;
        CHECK(near(got, want, 1e-11));
        CHECK(got >= 0.0);
    }
}

TEST_CASE("objective values add over probes") {
    const int n = 16;
    const ComplexField z = randomField(n, 16);
    const ScanGeometry geo = generateRasterScan(n, n / 2, n / 4);
    const DiffractionStack data = simulate(randomField(n, 17), geo);
    for (MetricKind kind : {MetricKind::Distance, MetricKind::IntensityGaussian}) {
        const double whole = evaluate(Objective{kind, &geo, &data}, z).value;
        double sum = 0;
        for (int k = 0; k < geo.probeCount(); ++k) {
            ScanGeometry one{n, geo.windowSize, geo.windowSize, {geo.windows[k]}};
            DiffractionStack od{n, {data.patterns[k]}};
            sum += evaluate(Objective{kind, &one, &od}, z).value;
        }
        CHECK(near(whole, sum, 1e-12));
    }
}

static void fdCheck(MetricKind kind, uint64_t s0) {
    const int n = 8;
    const ComplexField z = randomField(n, s0);
    const ScanGeometry geo = generateRasterScan(n, n / 2, n / 4);
    const DiffractionStack data = simulate(randomField(n, s0 + 1), geo);
    const Objective obj{kind, &geo, &data};
    const ObjectiveEval ev = evaluate(obj, z);
    for (uint64_t s = 0; s < 4; ++s) {
        ComplexField dir = randomField(n, 300 + s);
        const double nd = norm2(dir);
        for (std::size_t i = 0; i < dir.size(); ++i) dir[i] /= nd;
        ComplexField zp = z, zm = z;
        const double h = 1e-6;
        for (std::size_t i = 0; i < z.size(); ++i) {
            zp[i] += h * dir[i];
            zm[i] -= h * dir[i];
        }
        const double fd = (evaluate(obj, zp).value - evaluate(obj, zm).value) / (2 * h);
        CHECK(std::abs(fd - dotReal(ev.gradient, dir)) <= 1e-6 * std::max(1.0, std::abs(fd)));
    }
}
TEST_CASE("finite differences confirm the distance gradient") { fdCheck(MetricKind::Distance, 18); }
TEST_CASE("finite differences confirm the intensity-Gaussian gradient") { fdCheck(MetricKind::IntensityGaussian, 20); }

TEST_CASE("distance objective is numerically zero at the true object") {
    const int n = 16;
    const ComplexField z = randomField(n, 23);
    const ScanGeometry geo = generateRasterScan(n, n / 2, n / 4);
    const DiffractionStack data = simulate(z, geo);
    const ObjectiveEval ev = phiDistance(z, geo, data);
    CHECK(ev.value >= 0.0);
    CHECK(ev.value <= 1e-24);
    CHECK(norm2(ev.gradient) <= 1e-12);
}

TEST_CASE("single-pixel analytic cases") {
    const ComplexField z1(1, cdouble{1.0, 0.0});
    ScanGeometry geo{1, 1, 1, {ProbeWindow{0, 0, 1}}};
    DiffractionStack zero{1, {RealGrid(1, 0.0)}};
    const ObjectiveEval ig = phiIntensityGaussian(z1, geo, zero);
    CHECK(near(ig.value, 0.5, 1e-15));
    CHECK(near(ig.gradient[0].real(), 2.0, 1e-15));
    DiffractionStack dist{1, {RealGrid(1, 4.0)}};
    const ObjectiveEval m = phiDistance(z1, geo, dist);
    CHECK(near(m.value, 0.5, 1e-15));
    CHECK(near(m.gradient[0].real(), -1.0, 1e-15));
}

TEST_CASE("shifted objective subtracts the linear term") {
    const int n = 8;
    const ComplexField z = randomField(n, 24), v = randomField(n, 25);
    const ScanGeometry geo = generateRasterScan(n, n / 2, n / 4);
    const DiffractionStack data = simulate(randomField(n, 26), geo);
    const ObjectiveEval a = evaluate(Objective{MetricKind::Distance, &geo, &data}, z);
    const ObjectiveEval b = evaluate(Objective{MetricKind::Distance, &geo, &data, &v}, z);
    CHECK(near(b.value, a.value - dotReal(v, z), 1e-13));
    ComplexField want = a.gradient;
    for (std::size_t i = 0; i < want.size(); ++i) want[i] -= v[i];
    CHECK(maxAbsDiff(b.gradient, want) <= 1e-15);
}

TEST_CASE("objectives validate their inputs") {
    const ComplexField z = randomField(8, 27);
    const ScanGeometry geo = generateRasterScan(8, 4, 2);
    DiffractionStack data = simulate(z, geo);
    data.patterns[0].at(1, 1) = -1.0;
    CHECK_THROWS_AS(evaluate(Objective{MetricKind::Distance, &geo, &data}, z), DomainError);
    DiffractionStack tooFew = simulate(z, geo);
    tooFew.patterns.pop_back();
    CHECK_THROWS_AS(evaluate(Objective{MetricKind::Distance, &geo, &tooFew}, z), DomainError);
    CHECK_THROWS_AS(generateRasterScan(16, 8, 3), GeometryError);
    // fft2 needs a power-of-two grid (kernels.cpp:15-19)
    const ScanGeometry g12 = generateRasterScan(12, 4, 4);
    DiffractionStack d12{12, std::vector<RealGrid>(g12.probeCount(), RealGrid(12, 1.0))};
    CHECK_THROWS_AS(evaluate(Objective{MetricKind::Distance, &g12, &d12}, randomField(12, 1)), GeometryError);
}

TEST_CASE("PIE inner update is the unit descent step") {
    const int n = 16;
    const ComplexField z = randomField(n, 30);
    const ScanGeometry full = generateRasterScan(n, n / 2, n / 4);
    ScanGeometry one{n, full.windowSize, full.windowSize, {full.windows[4]}};
    const DiffractionStack all = simulate(randomField(n, 31), full);
    DiffractionStack od{n, {all.patterns[4]}};
    EvalCounter ctr;
    const SolverReport r = pie(z, one, od, 0.0, 1, ctr);
    const ObjectiveEval ev = phiDistance(z, one, od);
    ComplexField want = z;
    for (std::size_t i = 0; i < want.size(); ++i) want[i] -= ev.gradient[i];
    CHECK(maxAbsDiff(r.finalIterate, want) <= 1e-12);
    CHECK(ctr.weightedEvals == 1.0);
}

TEST_CASE("restrict and prolong: exact identity and adjointness") {
    const ComplexField u = randomField(8, 40), w = randomField(16, 41);
    const ComplexField rp = restrictField(prolongField(u));
    bool same = true;
    for (std::size_t i = 0; i < u.size(); ++i) same &= (rp[i] == u[i]);
    CHECK(same);
    CHECK(near(dotReal(prolongField(u), w), 4.0 * dotReal(u, restrictField(w)), 1e-12));
    CHECK_THROWS_AS(restrictField(ComplexField(7)), GeometryError);
}

TEST_CASE("V-cycles decrease the objective and charge both levels") {
    const int n = 32;
    const ScanGeometry geo = generateRasterScan(n, n / 2, n / 4);
    const DiffractionStack data = simulate(randomField(n, 50, 0.5), geo);
    Hierarchy h(geo, data, MetricKind::Distance, 2);
    EvalCounter ctr;
    MgoptDriverConfig cfg;
    cfg.budgetWeightedEvals = 1e9;
    cfg.maxCycles = 4;
    ComplexField z0 = randomField(n, 51, 0.25);
    for (std::size_t i = 0; i < z0.size(); ++i) z0[i] += 1.0;
    const SolverReport r = mgoptDriver(h, z0, cfg, ctr);
    for (std::size_t i = 1; i < r.history.size(); ++i) CHECK(r.history[i].value <= r.history[i - 1].value);
    CHECK(ctr.perLevelEvals[0] > 0 && ctr.perLevelEvals[1] > 0);
    CHECK(r.history.size() == 5);
}

TEST_CASE("GPU evaluation is bitwise reproducible") {
    const int n = 32;
    const ComplexField z = randomField(n, 60);
    const ScanGeometry geo = generateRasterScan(n, n / 2, n / 8);
    const DiffractionStack data = simulate(randomField(n, 61), geo);
    const ObjectiveEval a = phiDistance(z, geo, data), b = phiDistance(z, geo, data);
    CHECK(a.value == b.value);
    CHECK(maxAbsDiff(a.gradient, b.gradient) == 0.0);
}

int main() {
    std::setvbuf(stdout, nullptr, _IONBF, 0);   // progress survives a crash
    for (auto& [name, fn] : cases()) {
        std::printf("RUN %s\n", name.c_str());
        const int before = g_fail;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("  EXCEPTION in %s: %s\n", name.c_str(), e.what());
        }
        std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name.c_str());
    }
    std::printf("[ptycho_b200] test cases: %zu, checks: %d, failed checks: %d\n", cases().size(), g_checks, g_fail);
    return g_fail ? 1 : 0;
}
