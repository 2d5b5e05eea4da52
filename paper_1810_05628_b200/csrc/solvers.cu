// solvers.cu — GPU-resident line search / LBFGS / MG/OPT (see solvers.cuh).
#include <algorithm>
#include <cmath>

#include "solvers.cuh"
#include "transfer.cuh"

namespace ptg {

double DObj::eval(Counter& c, const void* z, void* grad) const {
    c.record(level, weight);   // charge before evaluating (solvers.hpp:33-36)
    plan_eval(*plan, metric, z, v, grad, plan->value.as<double>());
    return plan_read_scalar(*plan, plan->value.as<double>());
}

static double dnorm(Plan& p, const void* a) { return std::sqrt(plan_dot(p, a, a, p.nn())); }

LsOut d_linesearch(const DObj& obj, const void* z, const void* dir, Counter& ctr, int max_trials,
                   const double* phi0, void* z_out, void* g_out) {
    Plan& p = *obj.plan;
    LaunchScope ls(p);
    const size_t len = p.nn();
    LsOut r;
    double base;
    if (phi0) {
        base = *phi0;
    } else {
        DVec tmp(p, len);
        base = obj.eval(ctr, z, tmp.p);
    }
    DVec trial(p, len), g(p, len);
    double alpha = 1.0;
    for (int t = 0; t < max_trials; ++t) {
        dev_add_scaled(p.prec, trial.p, z, alpha, dir, len, p.stream);   // z + alpha d
        const double v = obj.eval(ctr, trial.p, g.p);
        ++r.trials;
        if (v <= base) {
            r.alpha = alpha;
            r.value = v;
            dev_copy(p.prec, z_out, trial.p, len, p.stream);
            dev_copy(p.prec, g_out, g.p, len, p.stream);
            return r;
        }
        alpha *= 0.5;
    }
    r.alpha = 0.0;
    r.stalled = true;
    if (z_out != z) dev_copy(p.prec, z_out, z, len, p.stream);
    return r;
}

namespace {
struct Pair {
    DVec s, y;
    double sy;
};

// solvers.cpp:19-36
void two_loop(Plan& p, const std::deque<Pair>& pairs, const void* g, void* q) {
    const size_t len = p.nn();
    if (pairs.empty()) {
        dev_scale(p.prec, q, g, -1.0, len, p.stream);
        return;
    }
    dev_copy(p.prec, q, g, len, p.stream);
    std::vector<double> alpha(pairs.size());
    for (size_t i = pairs.size(); i-- > 0;) {
        alpha[i] = plan_dot(p, pairs[i].s.p, q, len) / pairs[i].sy;
        dev_axpy(p.prec, q, -alpha[i], pairs[i].y.p, len, p.stream);
    }
    const Pair& newest = pairs.back();
    const double gamma = newest.sy / plan_dot(p, newest.y.p, newest.y.p, len);
    dev_scale(p.prec, q, q, gamma, len, p.stream);
    for (size_t i = 0; i < pairs.size(); ++i) {
        const double beta = plan_dot(p, pairs[i].y.p, q, len) / pairs[i].sy;
        dev_axpy(p.prec, q, alpha[i] - beta, pairs[i].s.p, len, p.stream);
    }
    dev_scale(p.prec, q, q, -1.0, len, p.stream);
}
}  // namespace

SolveOut d_lbfgs(const DObj& obj, const void* z0, const ptg_solver_cfg& cfg, Counter& ctr,
                 const double* warm_value, const void* warm_g, void* z_out, void* g_out,
                 std::vector<ptg_hist>* hist) {
    Plan& p = *obj.plan;
    LaunchScope ls(p);
    const size_t len = p.nn();
    DVec z(p, len), g(p, len), dir(p, len), nz(p, len), ng(p, len);
    dev_copy(p.prec, z.p, z0, len, p.stream);
    double cur;
    if (warm_value) {
        cur = *warm_value;
        dev_copy(p.prec, g.p, warm_g, len, p.stream);
    } else {
        cur = obj.eval(ctr, z.p, g.p);
    }
    if (plan_nonfinite(p, g.p, len)) raise(PTG_ERR_NUMERIC, "non-finite iterate in lbfgs");
    const double grad_floor = cfg.grad_tol_abs * (1.0 + dnorm(p, z0));
    const double g0 = dnorm(p, g.p);
    double gnorm = g0;
    if (hist) hist->push_back({ctr.weighted, cur, gnorm});
    auto satisfied = [&](double gn) { return gn <= std::max(cfg.grad_tol_rel * g0, grad_floor); };
    SolveOut out;
    out.reason = PTG_STOP_MAXITERS;
    std::deque<Pair> pairs;   // fresh memory per call (solvers.cpp:100)
    if (satisfied(gnorm)) {
        out.reason = PTG_STOP_TOLERANCE;
    } else {
        for (int iter = 1; iter <= cfg.max_iters; ++iter) {
            two_loop(p, pairs, g.p, dir.p);
            if (plan_dot(p, dir.p, g.p, len) >= 0.0) dev_scale(p.prec, dir.p, g.p, -1.0, len, p.stream);
            LsOut lsr = d_linesearch(obj, z.p, dir.p, ctr, cfg.linesearch_max, &cur, nz.p, ng.p);
            if (lsr.stalled) {
                out.reason = PTG_STOP_STALL;
                break;
            }
            if (plan_nonfinite(p, nz.p, len)) raise(PTG_ERR_NUMERIC, "non-finite iterate in lbfgs");
            Pair pr{DVec(p, len), DVec(p, len), 0.0};
            dev_sub(p.prec, pr.s.p, nz.p, z.p, len, p.stream);
            dev_sub(p.prec, pr.y.p, ng.p, g.p, len, p.stream);
            pr.sy = plan_dot(p, pr.s.p, pr.y.p, len);
            if (pr.sy > 1e-12 * dnorm(p, pr.s.p) * dnorm(p, pr.y.p)) {
                pairs.push_back(std::move(pr));
                if ((int)pairs.size() > cfg.lbfgs_memory) pairs.pop_front();
            }
            std::swap(z, nz);
            std::swap(g, ng);
            cur = lsr.value;
            gnorm = dnorm(p, g.p);
            if (hist) hist->push_back({ctr.weighted, cur, gnorm});
            if (satisfied(gnorm)) {
                out.reason = PTG_STOP_TOLERANCE;
                break;
            }
            if (ctr.weighted >= cfg.max_weighted) {
                out.reason = PTG_STOP_BUDGET;
                break;
            }
        }
    }
    dev_copy(p.prec, z_out, z.p, len, p.stream);
    if (g_out) dev_copy(p.prec, g_out, g.p, len, p.stream);
    out.value = cur;
    PTG_CUDA(cudaStreamSynchronize(p.stream));
    return out;
}

// ---------------------------------------------------------------- MG/OPT
std::unique_ptr<Hier> hier_build(Plan& fine, int metric, int depth, const ptg_mg_cfg& opt) {
    if (depth < 1) raise(PTG_ERR_CONFIG, "hierarchy depth must be >= 1");
    if (depth > 16) raise(PTG_ERR_CONFIG, "hierarchy depth too large");
    if ((fine.n >> (depth - 1)) < 8)
        raise(PTG_ERR_CONFIG, "hierarchy depth " + std::to_string(depth) + " would coarsen an n = " +
                                  std::to_string(fine.n) + " grid below 8");
    plan_ensure(fine, metric);
    auto h = std::make_unique<Hier>();
    h->fine = &fine;
    h->metric = metric;
    h->opt = opt;
    h->coarsest_iters = opt.coarsest_max_iters > 0 ? opt.coarsest_max_iters : (depth <= 2 ? 3 : 100);
    h->levels.push_back(&fine);
    for (int l = 1; l < depth; ++l) {
        h->owned.push_back(plan_coarsen(*h->levels.back()));
        h->owned.back()->stream = fine.stream;   // one stream orders the whole hierarchy
        h->levels.push_back(h->owned.back().get());
        plan_ensure(*h->levels.back(), metric);
    }
    return h;
}

static DObj level_obj(Hier& h, int level, const void* v) {
    DObj o;
    o.plan = h.levels[level];
    o.metric = h.metric;
    o.v = v;
    o.level = level;
    o.weight = std::ldexp(1.0, -2 * level);   // 4^-level (multigrid.cpp:91)
    return o;
}

static ptg_solver_cfg smoother_cfg(Hier& h, int level) {
    ptg_solver_cfg c;
    ptg_solver_cfg_default(&c);
    c.grad_tol_rel = (level == h.depth() - 1) ? h.opt.coarsest_grad_tol_rel : h.opt.intermediate_grad_tol_rel;
    c.grad_tol_abs = h.opt.grad_tol_abs;
    c.lbfgs_memory = h.opt.lbfgs_memory;
    c.linesearch_max = h.opt.linesearch_max;
    return c;
}

double d_mgopt_cycle(Hier& h, int level, const void* z, const void* v, Counter& ctr,
                     const double* warm_value, const void* warm_g, void* z_out, void* g_out) {
    if (level < 0 || level >= h.depth()) raise(PTG_ERR_CONFIG, "mgoptCycle: bad level");
    DObj obj = level_obj(h, level, v);
    Plan& p = *obj.plan;
    LaunchScope lsc(p);
    const size_t len = p.nn();
    if (level == h.depth() - 1) {
        ptg_solver_cfg cfg = smoother_cfg(h, level);
        cfg.max_iters = h.coarsest_iters;
        return d_lbfgs(obj, z, cfg, ctr, warm_value, warm_g, z_out, g_out, nullptr).value;
    }
    Plan& pc = *h.levels[level + 1];
    const size_t lenH = pc.nn();
    DVec zbar(p, len), gbar(p, len), gfine(p, len), corr(p, len), zplus(p, len), gplus(p, len);
    DVec zBarH(pc, lenH), vH(pc, lenH), cg(pc, lenH), tmpH(pc, lenH), zrec(pc, lenH), grec(pc, lenH),
        cgs(pc, lenH);

    ptg_solver_cfg pre = smoother_cfg(h, level);
    pre.max_iters = h.opt.k1;
    const double vbar = d_lbfgs(obj, z, pre, ctr, warm_value, warm_g, zbar.p, gbar.p, nullptr).value;

    dev_restrict_field(p.prec, zbar.p, p.n, zBarH.p, p.stream);
    // plain fine gradient = shifted gradient + v
    if (v) dev_add_scaled(p.prec, gfine.p, gbar.p, 1.0, v, len, p.stream);
    else dev_copy(p.prec, gfine.p, gbar.p, len, p.stream);
    PTG_CUDA(cudaStreamSynchronize(p.stream));
    DObj coarse_plain = level_obj(h, level + 1, nullptr);
    const double cval = coarse_plain.eval(ctr, zBarH.p, cg.p);
    // vH = R(v) + grad phi_H(zBarH) - R(grad phi_h(zBar))   (multigrid.cpp:142-147)
    if (v) {
        dev_restrict_field(p.prec, v, p.n, vH.p, pc.stream);
        dev_axpy(pc.prec, vH.p, 1.0, cg.p, lenH, pc.stream);
    } else {
        dev_copy(pc.prec, vH.p, cg.p, lenH, pc.stream);
    }
    dev_restrict_field(p.prec, gfine.p, p.n, tmpH.p, pc.stream);
    dev_axpy(pc.prec, vH.p, -1.0, tmpH.p, lenH, pc.stream);
    // coarse shifted evaluation at zBarH, free from coarseEval (:149-153)
    const double csval = cval - plan_dot(pc, vH.p, zBarH.p, lenH);
    dev_copy(pc.prec, cgs.p, cg.p, lenH, pc.stream);
    dev_axpy(pc.prec, cgs.p, -1.0, vH.p, lenH, pc.stream);

    d_mgopt_cycle(h, level + 1, zBarH.p, vH.p, ctr, &csval, cgs.p, zrec.p, grec.p);

    dev_sub(pc.prec, tmpH.p, zrec.p, zBarH.p, lenH, pc.stream);
    dev_prolong_field(pc.prec, tmpH.p, pc.n, corr.p, pc.stream);
    PTG_CUDA(cudaStreamSynchronize(pc.stream));
    LsOut lsr = d_linesearch(obj, zbar.p, corr.p, ctr, h.opt.linesearch_max, &vbar, zplus.p, gplus.p);
    double pval = lsr.value;
    if (lsr.stalled) {
        dev_copy(p.prec, zplus.p, zbar.p, len, p.stream);
        dev_copy(p.prec, gplus.p, gbar.p, len, p.stream);
        pval = vbar;
    }
    ptg_solver_cfg post = smoother_cfg(h, level);
    post.max_iters = h.opt.k2;
    return d_lbfgs(obj, zplus.p, post, ctr, &pval, gplus.p, z_out, g_out, nullptr).value;
}

SolveOut d_mgopt_driver(Hier& h, const void* z0, const ptg_driver_cfg& cfg, Counter& ctr,
                        void* z_out, std::vector<ptg_hist>* hist) {
    if (h.depth() < 1) raise(PTG_ERR_CONFIG, "mgoptDriver: empty hierarchy");
    Plan& p = *h.levels[0];
    LaunchScope lsc(p);
    const size_t len = p.nn();
    if (h.depth() == 1) {
        ptg_solver_cfg base;
        ptg_solver_cfg_default(&base);
        base.grad_tol_rel = cfg.grad_tol_rel;
        base.grad_tol_abs = cfg.grad_tol_abs;
        base.lbfgs_memory = h.opt.lbfgs_memory;
        base.linesearch_max = h.opt.linesearch_max;
        base.max_weighted = cfg.budget;
        base.max_iters = cfg.max_cycles;
        return d_lbfgs(level_obj(h, 0, nullptr), z0, base, ctr, nullptr, nullptr, z_out, nullptr, hist);
    }
    DObj top = level_obj(h, 0, nullptr);
    DVec z(p, len), g(p, len), nz(p, len), ng(p, len);
    dev_copy(p.prec, z.p, z0, len, p.stream);
    double cur = top.eval(ctr, z.p, g.p);
    if (plan_nonfinite(p, g.p, len)) raise(PTG_ERR_NUMERIC, "non-finite gradient in mgoptDriver");
    const double g0 = dnorm(p, g.p);
    const double grad_floor = cfg.grad_tol_abs * (1.0 + dnorm(p, z0));
    double gnorm = g0;
    if (hist) hist->push_back({ctr.weighted, cur, gnorm});
    SolveOut out;
    out.reason = PTG_STOP_MAXITERS;
    if (gnorm <= std::max(cfg.grad_tol_rel * g0, grad_floor)) {
        out.reason = PTG_STOP_TOLERANCE;
    } else {
        for (int cycle = 1; cycle <= cfg.max_cycles; ++cycle) {
            cur = d_mgopt_cycle(h, 0, z.p, nullptr, ctr, &cur, g.p, nz.p, ng.p);
            std::swap(z, nz);
            std::swap(g, ng);
            gnorm = dnorm(p, g.p);
            if (hist) hist->push_back({ctr.weighted, cur, gnorm});
            if (gnorm <= std::max(cfg.grad_tol_rel * g0, grad_floor)) {
                out.reason = PTG_STOP_TOLERANCE;
                break;
            }
            if (ctr.weighted >= cfg.budget) {
                out.reason = PTG_STOP_BUDGET;
                break;
            }
        }
    }
    dev_copy(p.prec, z_out, z.p, len, p.stream);
    PTG_CUDA(cudaStreamSynchronize(p.stream));
    out.value = cur;
    return out;
}

}  // namespace ptg
