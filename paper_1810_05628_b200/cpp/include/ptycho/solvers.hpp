// solvers.hpp — drop-in for /root/reference/proj/include/ptycho/solvers.hpp.
//
// Same types and signatures.  A CountedObjective made by counted() carries
// the ptychographic Objective behind it (additive member `device`): lbfgs and
// truncatedNewton on such an objective run GPU-resident (ptg_lbfgs_ex /
// ptg_truncated_newton_ex: iterates, gradients and curvature pairs stay in
// HBM; the callback, if any, receives host copies).  Any other
// CountedObjective (user std::function stubs, e.g. the reference's
// quadratic test objectives) runs the same algorithms on the host below
// (solvers.cpp:19-227 restated) -- its evaluations are the user's code.
// pie runs on the GPU (ptg_pie_cb).
#pragma once

#include <algorithm>
#include <cmath>
#include <deque>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <vector>

#include "objectives.hpp"

namespace ptycho {

struct EvalCounter {
    double weightedEvals = 0.0;
    std::map<int, long> perLevelEvals;
    void record(int level, double weight) {
        weightedEvals += weight;
        ++perLevelEvals[level];
    }
};

struct CountedObjective {
    std::function<ObjectiveEval(const ComplexField&)> fn;
    int level = 0;
    double weight = 1.0;
    // extension: the ptychographic objective fn evaluates (set by counted());
    // selects the GPU-resident solver paths
    std::shared_ptr<const Objective> device;

    ObjectiveEval eval(const ComplexField& z, EvalCounter& counter) const {
        counter.record(level, weight);
        return fn(z);
    }
};

inline CountedObjective counted(Objective objective, int level = 0, double weight = 1.0) {
    CountedObjective c;
    c.fn = [objective](const ComplexField& z) { return evaluate(objective, z); };
    c.level = level;
    c.weight = weight;
    c.device = std::make_shared<const Objective>(objective);
    return c;
}

enum class StopReason { Tolerance, Budget, MaxIters, Stall };

struct HistoryPoint {
    double weightedEvals = 0.0;
    double value = 0.0;
    double gradNorm = 0.0;
};

struct SolverReport {
    ComplexField finalIterate;
    ObjectiveEval finalEval;
    std::vector<HistoryPoint> history;   // initial point + one entry per iteration
    StopReason reason = StopReason::MaxIters;
};

struct SolverConfig {
    int maxIters = 100;
    double gradTolRel = 0.0;
    double gradTolAbs = 1e-13;
    int lbfgsMemory = 25;
    int linesearchMax = 50;
    int cgMaxIters = 20;
    double cgRelTol = 0.1;
    double maxWeightedEvals = std::numeric_limits<double>::infinity();
};

using IterationCallback = std::function<void(int, const ComplexField&, double, double)>;

struct LinesearchResult {
    double alpha = 0.0;
    ComplexField z;
    ObjectiveEval eval;
    bool stalled = false;
    int trials = 0;
};

// alpha = 1, 1/2, ...: the first trial with phi(z + alpha d) <= phi(z) wins
inline LinesearchResult backtrackingLinesearch(const CountedObjective& obj, const ComplexField& z,
                                               const ComplexField& dir, EvalCounter& counter, int maxTrials,
                                               std::optional<double> phi0 = std::nullopt) {
    const double base = phi0.has_value() ? *phi0 : obj.eval(z, counter).value;
    LinesearchResult res;
    double alpha = 1.0;
    while (res.trials < maxTrials) {
        ComplexField trial = z;
        axpy(trial, alpha, dir);
        ObjectiveEval ev = obj.eval(trial, counter);
        ++res.trials;
        if (ev.value <= base) {
            res.alpha = alpha;
            res.z = std::move(trial);
            res.eval = std::move(ev);
            return res;
        }
        alpha *= 0.5;
    }
    res.z = z;
    res.stalled = true;
    return res;
}

namespace detail {

inline void require_finite(const ComplexField& z, const char* where) {
    if (!z.isFinite()) throw NumericError(std::string("non-finite iterate in ") + where);
}

// ---- host path (user std::function objectives)
struct HostRun {
    const CountedObjective& obj;
    const SolverConfig& cfg;
    EvalCounter& counter;
    const IterationCallback& cb;
    SolverReport rep;
    ComplexField z;
    ObjectiveEval cur;
    double floor = 0.0, g0 = 0.0;
    HostRun(const CountedObjective& o, const ComplexField& z0, const SolverConfig& c, EvalCounter& ctr,
            const IterationCallback& callback, const ObjectiveEval* warm, const char* name)
        : obj(o), cfg(c), counter(ctr), cb(callback), z(z0) {
        cur = warm ? *warm : obj.eval(z, counter);
        require_finite(cur.gradient, name);
        floor = cfg.gradTolAbs * (1.0 + norm2(z0));
        g0 = norm2(cur.gradient);
        note(0, g0);
    }
    void note(int iter, double gnorm) {
        rep.history.push_back({counter.weightedEvals, cur.value, gnorm});
        if (cb) cb(iter, z, cur.value, counter.weightedEvals);
    }
    bool converged(double gnorm) const { return gnorm <= std::max(cfg.gradTolRel * g0, floor); }
    // accept a line-search result; true = stop
    bool step(int iter, LinesearchResult& ls, const char* name) {
        require_finite(ls.z, name);
        z = std::move(ls.z);
        cur = std::move(ls.eval);
        const double gn = norm2(cur.gradient);
        note(iter, gn);
        if (converged(gn)) {
            rep.reason = StopReason::Tolerance;
            return true;
        }
        if (counter.weightedEvals >= cfg.maxWeightedEvals) {
            rep.reason = StopReason::Budget;
            return true;
        }
        return false;
    }
    SolverReport finish() {
        rep.finalIterate = std::move(z);
        rep.finalEval = std::move(cur);
        return std::move(rep);
    }
};

struct Pair {
    ComplexField s, y;
    double sy;
};

// -H g by the two-loop recursion, H0 = (s'y / y'y) of the newest pair
inline ComplexField two_loop(const std::deque<Pair>& mem, const ComplexField& g) {
    if (mem.empty()) return scaled(g, -1.0);
    ComplexField q = g;
    std::vector<double> a(mem.size());
    for (std::size_t i = mem.size(); i-- > 0;) {
        a[i] = dotReal(mem[i].s, q) / mem[i].sy;
        axpy(q, -a[i], mem[i].y);
    }
    q = scaled(q, mem.back().sy / dotReal(mem.back().y, mem.back().y));
    for (std::size_t i = 0; i < mem.size(); ++i) axpy(q, a[i] - dotReal(mem[i].y, q) / mem[i].sy, mem[i].s);
    return scaled(q, -1.0);
}

inline SolverReport host_lbfgs(const CountedObjective& obj, const ComplexField& z0, const SolverConfig& cfg,
                               EvalCounter& counter, const IterationCallback& cb, const ObjectiveEval* warm) {
    HostRun run(obj, z0, cfg, counter, cb, warm, "lbfgs");
    std::deque<Pair> mem;
    if (run.converged(run.g0)) {
        run.rep.reason = StopReason::Tolerance;
        return run.finish();
    }
    for (int it = 1; it <= cfg.maxIters; ++it) {
        ComplexField d = two_loop(mem, run.cur.gradient);
        if (dotReal(d, run.cur.gradient) >= 0.0) d = scaled(run.cur.gradient, -1.0);
        LinesearchResult ls = backtrackingLinesearch(obj, run.z, d, counter, cfg.linesearchMax, run.cur.value);
        if (ls.stalled) {
            run.rep.reason = StopReason::Stall;
            break;
        }
        require_finite(ls.z, "lbfgs");
        ComplexField s = sub(ls.z, run.z), y = sub(ls.eval.gradient, run.cur.gradient);
        const double sy = dotReal(s, y);
        if (sy > 1e-12 * norm2(s) * norm2(y)) {
            mem.push_back({std::move(s), std::move(y), sy});
            if ((int)mem.size() > cfg.lbfgsMemory) mem.pop_front();
        }
        if (run.step(it, ls, "lbfgs")) return run.finish();
    }
    return run.finish();
}

inline SolverReport host_truncated_newton(const CountedObjective& obj, const ComplexField& z0,
                                          const SolverConfig& cfg, EvalCounter& counter,
                                          const IterationCallback& cb, const ObjectiveEval* warm) {
    HostRun run(obj, z0, cfg, counter, cb, warm, "truncatedNewton");
    if (run.converged(run.g0)) {
        run.rep.reason = StopReason::Tolerance;
        return run.finish();
    }
    // (grad(z + delta v) - g) / delta, one counted gradient evaluation
    auto hv = [&](const ComplexField& v) {
        const double vn = norm2(v);
        if (vn == 0.0) return ComplexField(run.z.n());
        const double delta = 1e-6 * (1.0 + norm2(run.z)) / vn;
        ComplexField zp = run.z;
        axpy(zp, delta, v);
        return scaled(sub(obj.eval(zp, counter).gradient, run.cur.gradient), 1.0 / delta);
    };
    for (int it = 1; it <= cfg.maxIters; ++it) {
        ComplexField x(run.z.n());
        ComplexField r = scaled(run.cur.gradient, -1.0);
        const double rhs = norm2(r);
        ComplexField p = r;
        double rs = dotReal(r, r);
        for (int k = 0; k < cfg.cgMaxIters; ++k) {
            const ComplexField hp = hv(p);
            const double php = dotReal(p, hp);
            if (php <= 0.0) {   // negative curvature
                if (k == 0) x = r;
                break;
            }
            const double a = rs / php;
            axpy(x, a, p);
            axpy(r, -a, hp);
            const double rs2 = dotReal(r, r);
            if (std::sqrt(rs2) <= cfg.cgRelTol * rhs) break;
            ComplexField pn = r;
            axpy(pn, rs2 / rs, p);
            p = std::move(pn);
            rs = rs2;
        }
        if (norm2(x) == 0.0 || dotReal(x, run.cur.gradient) >= 0.0) x = scaled(run.cur.gradient, -1.0);
        LinesearchResult ls = backtrackingLinesearch(obj, run.z, x, counter, cfg.linesearchMax, run.cur.value);
        if (ls.stalled) {
            run.rep.reason = StopReason::Stall;
            break;
        }
        if (run.step(it, ls, "truncatedNewton")) return run.finish();
    }
    return run.finish();
}

// ---- GPU-resident path (ptychographic objectives)
struct CbBridge {
    const IterationCallback* cb;
    int n;
    double base, weight;
    static void call(void* user, int iter, const double* z, double value, double weighted) {
        auto* b = static_cast<CbBridge*>(user);
        ComplexField f(b->n);
        std::memcpy(static_cast<void*>(f.data()), z, f.size() * sizeof(cdouble));
        (*b->cb)(iter, f, value, b->base + weighted * b->weight);
    }
};

inline ptg_solver_cfg c_cfg(const SolverConfig& c, double budget) {
    return ptg_solver_cfg{c.maxIters, c.gradTolRel, c.gradTolAbs, c.lbfgsMemory, c.linesearchMax, budget, c.cgMaxIters,
                          c.cgRelTol};
}

// device evaluations are charged at weight 1 on level 0; the caller's
// counter gets them at the objective's level and weight
inline void charge(EvalCounter& counter, long evals, int level, double weight) {
    if (evals <= 0) return;
    counter.weightedEvals += static_cast<double>(evals) * weight;
    counter.perLevelEvals[level] += evals;
}

using DeviceSolver = int (*)(ptg_plan*, int, const double*, const double*, const double*, const double*,
                             const ptg_solver_cfg*, double*, double*, ptg_report*, ptg_hist*, int, ptg_iter_cb, void*);

inline SolverReport device_solve(DeviceSolver fn, const CountedObjective& obj, const ComplexField& z0,
                                 const SolverConfig& cfg, EvalCounter& counter, const IterationCallback& cb,
                                 const ObjectiveEval* warm) {
    const Objective& o = *obj.device;
    auto plan = objective_plan(o, z0.n());
    if (o.shift && o.shift->n() != z0.n()) throw DomainError("dotReal: size mismatch");
    if (warm && warm->gradient.n() != z0.n()) throw DomainError("warm start gradient size mismatch");
    const double base = counter.weightedEvals;
    // the budget test counter.weightedEvals >= maxWeightedEvals, in device units
    const double budget = std::isinf(cfg.maxWeightedEvals) ? cfg.maxWeightedEvals
                                                           : (cfg.maxWeightedEvals - base) / obj.weight;
    const ptg_solver_cfg c = c_cfg(cfg, budget);
    SolverReport rep;
    rep.finalIterate = ComplexField(z0.n());
    rep.finalEval.gradient = ComplexField(z0.n());
    std::vector<ptg_hist> h(static_cast<std::size_t>(std::max(cfg.maxIters, 0)) + 2);
    ptg_report r{};
    CbBridge br{&cb, z0.n(), base, obj.weight};
    const double wv = warm ? warm->value : 0.0;
    check(fn(plan.get(), metric_of(o.kind), o.shift ? dp(o.shift->data()) : nullptr, dp(z0.data()),
             warm ? &wv : nullptr, warm ? dp(warm->gradient.data()) : nullptr, &c, dp(rep.finalIterate.data()),
             dp(rep.finalEval.gradient.data()), &r, h.data(), (int)h.size(), cb ? &CbBridge::call : nullptr, &br));
    charge(counter, r.per_level[0], obj.level, obj.weight);
    rep.finalEval.value = r.final_value;
    for (int i = 0; i < r.hist_len && i < (int)h.size(); ++i)
        rep.history.push_back({base + h[i].weighted * obj.weight, h[i].value, h[i].gnorm});
    rep.reason = static_cast<StopReason>(r.reason);
    return rep;
}

}  // namespace detail

inline SolverReport lbfgs(const CountedObjective& obj, const ComplexField& z0, const SolverConfig& config,
                          EvalCounter& counter, const IterationCallback& callback = {},
                          const ObjectiveEval* warmStart = nullptr) {
    if (obj.device) return detail::device_solve(ptg_lbfgs_ex, obj, z0, config, counter, callback, warmStart);
    return detail::host_lbfgs(obj, z0, config, counter, callback, warmStart);
}

inline SolverReport truncatedNewton(const CountedObjective& obj, const ComplexField& z0, const SolverConfig& config,
                                    EvalCounter& counter, const IterationCallback& callback = {},
                                    const ObjectiveEval* warmStart = nullptr) {
    if (obj.device)
        return detail::device_solve(ptg_truncated_newton_ex, obj, z0, config, counter, callback, warmStart);
    return detail::host_truncated_newton(obj, z0, config, counter, callback, warmStart);
}

// sequential projection sweeps on the GPU; one sweep charged as one fine
// evaluation, history from uncounted diagnostic evaluations
inline SolverReport pie(const ComplexField& z0, const ScanGeometry& geometry, const DiffractionStack& data,
                        double gamma, int sweeps, EvalCounter& counter, const IterationCallback& callback = {},
                        double maxWeightedEvals = std::numeric_limits<double>::infinity()) {
    if (gamma < 0.0) throw ConfigError("pie: gamma must be non-negative");
    const Objective diag{MetricKind::Distance, &geometry, &data, nullptr};
    auto plan = detail::objective_plan(diag, z0.n());
    const double base = counter.weightedEvals;
    SolverReport rep;
    rep.finalIterate = z0;
    std::vector<ptg_hist> h(static_cast<std::size_t>(std::max(sweeps, 0)) + 2);
    int nh = 0, reason = 0;
    double fv = 0.0, wt = 0.0;
    detail::CbBridge br{&callback, z0.n(), base, 1.0};
    detail::check(ptg_pie_cb(plan.get(), detail::dp(rep.finalIterate.data()), gamma, sweeps, maxWeightedEvals - base,
                             &fv, h.data(), (int)h.size(), &nh, &wt, &reason,
                             callback ? &detail::CbBridge::call : nullptr, &br));
    detail::charge(counter, static_cast<long>(wt), 0, 1.0);
    for (int i = 0; i < nh && i < (int)h.size(); ++i) rep.history.push_back({base + h[i].weighted, h[i].value, h[i].gnorm});
    rep.reason = static_cast<StopReason>(reason);
    rep.finalEval = evaluate(diag, rep.finalIterate);   // uncounted diagnostic
    return rep;
}

}  // namespace ptycho
