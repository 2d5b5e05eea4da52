// multigrid.hpp — drop-in for /root/reference/proj/include/ptycho/multigrid.hpp.
//
// Grid transfers run on the B200 (ptg_restrict_field / ptg_prolong_field /
// ptg_restrict_data, bit-exact).  buildHierarchy keeps the reference's host
// description (GridLevel per level: regenerated raster + restricted data) and
// lazily attaches a device hierarchy (ptg_hier_create: the same coarsening
// done in HBM) on which mgoptCycle / mgoptDriver run GPU-resident
// (ptg_mgopt_cycle / ptg_mgopt_driver_ex).  A depth-1 driver is plain lbfgs
// on the top level, as in the reference.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "solvers.hpp"

namespace ptycho {

namespace detail {
inline void check_even(int n, const char* what) {
    if (n < 2 || n % 2 != 0) throw GeometryError(std::string(what) + " must be even and >= 2, got " + std::to_string(n));
}
}  // namespace detail

// ((a + b) + (c + d)) / 4 over 2 x 2 blocks
inline ComplexField restrictField(const ComplexField& fine) {
    detail::check_even(fine.n(), "restrictField: grid side");
    ComplexField c(fine.n() / 2);
    detail::check(ptg_restrict_field(detail::dp(fine.data()), fine.n(), detail::dp(c.data())));
    return c;
}

// each coarse pixel copied into its 2 x 2 block
inline ComplexField prolongField(const ComplexField& coarse) {
    if (coarse.n() < 1) throw GeometryError("prolongField: empty grid");
    ComplexField f(coarse.n() * 2);
    detail::check(ptg_prolong_field(detail::dp(coarse.data()), coarse.n(), detail::dp(f.data())));
    return f;
}

// central (n/2)^2 block of the shifted pattern, un-shifted, x 1/16
inline DiffractionStack restrictData(const DiffractionStack& fine) {
    if (fine.n < 4 || fine.n % 4 != 0) throw GeometryError("restrictData: grid side must be a multiple of 4");
    const int n = fine.n, N = fine.count();
    const std::size_t nn = static_cast<std::size_t>(n) * n, hh = nn / 4;
    DiffractionStack c;
    c.n = n / 2;
    if (N == 0) return c;
    std::vector<double> in(nn * N), out(hh * N);
    for (int k = 0; k < N; ++k) {
        if (fine.patterns[k].n() != n) throw DomainError("diffraction pattern size mismatch");
        std::memcpy(in.data() + k * nn, fine.patterns[k].data(), nn * 8);
    }
    detail::check(ptg_restrict_data(in.data(), N, n, out.data()));
    c.patterns.assign(N, RealGrid(n / 2));
    for (int k = 0; k < N; ++k) std::memcpy(c.patterns[k].data(), out.data() + k * hh, hh * 8);
    return c;
}

struct GridLevel {
    int n = 0;
    ScanGeometry geometry;
    DiffractionStack data;
    MetricKind kind = MetricKind::Distance;
    int levelIndex = 0;
    double costWeight = 1.0;   // 4^-levelIndex
};

// geometry regenerated at n/2 (window w/2, stride s/2), data restricted
inline GridLevel buildCoarseLevel(const GridLevel& fine) {
    if (fine.n < 16) throw GeometryError("buildCoarseLevel: refuse to coarsen below n = 8");
    detail::check_even(fine.geometry.windowSize, "buildCoarseLevel: window size");
    detail::check_even(fine.geometry.stride, "buildCoarseLevel: stride");
    GridLevel c;
    c.n = fine.n / 2;
    c.geometry = generateRasterScan(fine.n / 2, fine.geometry.windowSize / 2, fine.geometry.stride / 2);
    c.data = restrictData(fine.data);
    c.kind = fine.kind;
    c.levelIndex = fine.levelIndex + 1;
    c.costWeight = fine.costWeight * 0.25;
    return c;
}

struct MgoptConfig {
    int k1 = 1;
    int k2 = 1;
    int coarsestMaxIters = 0;   // 0: 3 for depth <= 2, else 100
    double coarsestGradTolRel = 1e-4;
    double intermediateGradTolRel = 1e-3;
    int lbfgsMemory = 25;
    int linesearchMax = 50;
    double gradTolAbs = 1e-13;
};

namespace detail {
struct DeviceHier {
    PlanPtr fine;
    ptg_hier* h = nullptr;
    ~DeviceHier() {
        if (h) ptg_hier_destroy(h);
    }
};
}  // namespace detail

struct Hierarchy {
    std::vector<GridLevel> levels;   // [0] is the finest
    MgoptConfig options;
    int coarsestMaxIters = 3;
    int depth() const { return static_cast<int>(levels.size()); }

    // the device copy (built on first use; shared by copies of this value)
    mutable std::shared_ptr<detail::DeviceHier> device_;
    ptg_hier* device() const {
        if (!device_) {
            auto d = std::make_shared<detail::DeviceHier>();
            const GridLevel& top = levels.at(0);
            d->fine = detail::cached_plan(detail::source_of(top.geometry, top.data, nullptr, PTG_C128));
            ptg_mg_cfg c{options.k1, options.k2, coarsestMaxIters, options.coarsestGradTolRel,
                         options.intermediateGradTolRel, options.lbfgsMemory, options.linesearchMax,
                         options.gradTolAbs};
            detail::check(ptg_hier_create(d->fine.get(), detail::metric_of(top.kind), depth(), &c, &d->h));
            device_ = d;
        }
        return device_->h;
    }
};

inline Hierarchy buildHierarchy(const ScanGeometry& geometry, const DiffractionStack& data, MetricKind kind, int depth,
                                const MgoptConfig& options = {}) {
    if (depth < 1) throw ConfigError("hierarchy depth must be >= 1");
    if (geometry.n != data.n) throw DomainError("hierarchy: geometry and data sizes differ");
    if (data.count() != geometry.probeCount()) throw DomainError("hierarchy: pattern count does not match probe count");
    if ((geometry.n >> (depth - 1)) < 8)
        throw ConfigError("hierarchy depth " + std::to_string(depth) + " would coarsen an n = " +
                          std::to_string(geometry.n) + " grid below 8");
    Hierarchy h;
    h.options = options;
    h.coarsestMaxIters = options.coarsestMaxIters > 0 ? options.coarsestMaxIters : (depth <= 2 ? 3 : 100);
    h.levels.push_back(GridLevel{geometry.n, geometry, data, kind, 0, 1.0});
    for (int l = 1; l < depth; ++l) h.levels.push_back(buildCoarseLevel(h.levels.back()));
    return h;
}

struct CycleResult {
    ComplexField z;
    ObjectiveEval eval;   // shifted objective at the final iterate
};

namespace detail {
// per-level device evaluations at the hierarchy's cost weights
inline void charge_levels(EvalCounter& counter, const ptg_report& r, const Hierarchy& h) {
    for (int l = 0; l < h.depth() && l < 16; ++l) charge(counter, r.per_level[l], l, h.levels[l].costWeight);
}
}  // namespace detail

// one V-cycle at `level` with shift v, GPU-resident
inline CycleResult mgoptCycle(const Hierarchy& h, int level, const ComplexField& z, const ComplexField& v,
                              EvalCounter& counter, const ObjectiveEval* warmStart = nullptr) {
    if (level < 0 || level >= h.depth()) throw ConfigError("mgoptCycle: bad level");
    const int n = h.levels[level].n;
    if (z.n() != n || v.n() != n) throw DomainError("mgoptCycle: iterate / shift do not match the level's grid");
    ptg_hier* dh = h.device();
    CycleResult res;
    res.z = ComplexField(n);
    res.eval.gradient = ComplexField(n);
    ptg_report r{};
    const double wv = warmStart ? warmStart->value : 0.0;
    detail::check(ptg_mgopt_cycle(dh, level, detail::dp(z.data()), detail::dp(v.data()), warmStart ? &wv : nullptr,
                                  warmStart ? detail::dp(warmStart->gradient.data()) : nullptr, detail::dp(res.z.data()),
                                  &res.eval.value, detail::dp(res.eval.gradient.data()), &r));
    detail::charge_levels(counter, r, h);
    return res;
}

struct MgoptDriverConfig {
    double budgetWeightedEvals = 100.0;
    double gradTolRel = 0.0;
    double gradTolAbs = 1e-13;
    int maxCycles = 1000000;
};

inline SolverReport mgoptDriver(const Hierarchy& h, const ComplexField& z0, const MgoptDriverConfig& config,
                                EvalCounter& counter, const IterationCallback& callback = {}) {
    if (h.depth() < 1) throw ConfigError("mgoptDriver: empty hierarchy");
    if (z0.n() != h.levels[0].n) throw DomainError("mgoptDriver: iterate does not match the finest grid");
    const GridLevel& top = h.levels[0];
    if (h.depth() == 1) {   // degenerate hierarchy: plain LBFGS with the driver's stopping rules
        SolverConfig base;
        base.gradTolRel = config.gradTolRel;
        base.gradTolAbs = config.gradTolAbs;
        base.lbfgsMemory = h.options.lbfgsMemory;
        base.linesearchMax = h.options.linesearchMax;
        base.maxWeightedEvals = config.budgetWeightedEvals;
        base.maxIters = config.maxCycles;
        return lbfgs(counted(Objective{top.kind, &top.geometry, &top.data, nullptr}, top.levelIndex, top.costWeight),
                     z0, base, counter, callback);
    }
    ptg_hier* dh = h.device();
    const double base = counter.weightedEvals;
    ptg_driver_cfg c{config.budgetWeightedEvals - base, config.gradTolRel, config.gradTolAbs, config.maxCycles};
    SolverReport rep;
    rep.finalIterate = ComplexField(z0.n());
    rep.finalEval.gradient = ComplexField(z0.n());
    std::vector<ptg_hist> hist(static_cast<std::size_t>(std::min(config.maxCycles, 100000)) + 2);
    ptg_report r{};
    detail::CbBridge br{&callback, z0.n(), base, 1.0};
    detail::check(ptg_mgopt_driver_ex(dh, detail::dp(z0.data()), &c, detail::dp(rep.finalIterate.data()),
                                      detail::dp(rep.finalEval.gradient.data()), &r, hist.data(), (int)hist.size(),
                                      callback ? &detail::CbBridge::call : nullptr, &br));
    detail::charge_levels(counter, r, h);
    rep.finalEval.value = r.final_value;
    for (int i = 0; i < r.hist_len && i < (int)hist.size(); ++i)
        rep.history.push_back({base + hist[i].weighted, hist[i].value, hist[i].gnorm});
    rep.reason = static_cast<StopReason>(r.reason);
    return rep;
}

}  // namespace ptycho
