// solvers.cu — GPU-resident line search / LBFGS / MG/OPT (see solvers.cuh).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "solvers.cuh"
#include "transfer.cuh"

namespace ptg {

thread_local const IterHook* g_iter_hook = nullptr;

// PTG_LBFGS_DEBUG=1: host time inside the line-search synchronisations vs the
// whole LBFGS call (dev instrumentation)
static thread_local double g_sync_us = 0.0, g_graph_us = 0.0;   // one context per host thread
static thread_local int g_graph_n = 0;
static thread_local double g_prep_us = 0.0;
static bool lbfgs_debug() {
    static const bool on = getenv("PTG_LBFGS_DEBUG") != nullptr;
    return on;
}

void DObj::eval_enqueue(Counter& c, const void* z, void* grad, double* host_value) const {
    Plan& p = *plan;
    c.record(level, weight);   // charge before evaluating (solvers.hpp:33-36)
    plan_eval(p, metric, z, v, grad, p.value.as<double>());
    PTG_CUDA(cudaMemcpyAsync(host_value, p.value.p, sizeof(double), cudaMemcpyDeviceToHost, p.stream));
}

double DObj::eval(Counter& c, const void* z, void* grad) const {
    double* h = plan->hval.as<double>();
    eval_enqueue(c, z, grad, h);
    PTG_CUDA(cudaStreamSynchronize(plan->stream));
    return h[0];
}

static double dnorm(Plan& p, const void* a) { return std::sqrt(plan_dot(p, a, a, p.nn())); }

LsOut d_linesearch(const DObj& obj, const void* z, const void* dir, Counter& ctr, int max_trials,
                   const double* phi0, void* z_out, void* g_out, const std::function<void()>& first_trial_hook) {
    Plan& p = *obj.plan;
    LaunchScope ls(p);
    const size_t len = p.nn();
    LsOut r;
    // g_out doubles as the gradient scratch of the base evaluation
    const double base = phi0 ? *phi0 : obj.eval(ctr, z, g_out);
    double* h = p.hval.as<double>();
    double alpha = 1.0;
    for (int t = 0; t < max_trials; ++t) {
        dev_add_scaled(p.prec, z_out, z, alpha, dir, len, p.stream);   // z + alpha d
        obj.eval_enqueue(ctr, z_out, g_out, h);
        if (t == 0 && first_trial_hook) first_trial_hook();
        const auto ts = std::chrono::steady_clock::now();
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        if (lbfgs_debug()) g_sync_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - ts).count();
        const double v = h[0];
        ++r.trials;
        if (v <= base) {
            r.alpha = alpha;
            r.value = v;
            return r;
        }
        alpha *= 0.5;
    }
    r.alpha = 0.0;
    r.stalled = true;
    dev_copy(p.prec, z_out, z, len, p.stream);
    return r;
}

// the rest of d_linesearch after its first trial (alpha = 1, value v1) ran
// elsewhere (the graph-replayed LBFGS iteration): same trials, same charges
LsOut d_linesearch_continue(const DObj& obj, const void* z, const void* dir, Counter& ctr, int max_trials,
                            double base, void* z_out, void* g_out, double v1) {
    Plan& p = *obj.plan;
    const size_t len = p.nn();
    double* h = p.hval.as<double>();
    LsOut r;
    r.trials = 1;
    if (v1 <= base) {
        r.alpha = 1.0;
        r.value = v1;
        return r;
    }
    double alpha = 0.5;
    for (int t = 1; t < max_trials; ++t) {
        dev_add_scaled(p.prec, z_out, z, alpha, dir, len, p.stream);
        obj.eval_enqueue(ctr, z_out, g_out, h);
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        const double v = h[0];
        ++r.trials;
        if (v <= base) {
            r.alpha = alpha;
            r.value = v;
            return r;
        }
        alpha *= 0.5;
    }
    r.alpha = 0.0;
    r.stalled = true;
    dev_copy(p.prec, z_out, z, len, p.stream);
    return r;
}

namespace {
struct Pair {
    DVec s, y;
    double sy;
};

// solvers.cpp:19-36, one kernel per operation with a host read per product
// (fallback of the fused dev_two_loop; same arithmetic, same bits)
void two_loop(Plan& p, const std::vector<const void*>& s, const std::vector<const void*>& y,
              const std::vector<double>& sy, const void* g, void* q) {
    const size_t len = p.nn(), k = s.size();
    if (k == 0) {
        dev_scale(p.prec, q, g, -1.0, len, p.stream);
        return;
    }
    dev_copy(p.prec, q, g, len, p.stream);
    std::vector<double> alpha(k);
    for (size_t i = k; i-- > 0;) {
        alpha[i] = plan_dot(p, s[i], q, len) / sy[i];
        dev_axpy(p.prec, q, -alpha[i], y[i], len, p.stream);
    }
    const double gamma = sy[k - 1] / plan_dot(p, y[k - 1], y[k - 1], len);
    dev_scale(p.prec, q, q, gamma, len, p.stream);
    for (size_t i = 0; i < k; ++i) {
        const double beta = plan_dot(p, y[i], q, len) / sy[i];
        dev_axpy(p.prec, q, alpha[i] - beta, s[i], len, p.stream);
    }
    dev_scale(p.prec, q, q, -1.0, len, p.stream);
}
}  // namespace

SolveOut d_lbfgs(const DObj& obj, const void* z0, const ptg_solver_cfg& cfg, Counter& ctr,
                 const double* warm_value, const void* warm_g, void* z_out, void* g_out,
                 std::vector<ptg_hist>* hist) {
    Plan& p = *obj.plan;
    LaunchScope ls(p);
    const auto t_call = std::chrono::steady_clock::now();
    std::string dbg_log;
    auto dbg_mark = [&](const char* what) {
        char b[64];
        snprintf(b, sizeof b, " %s@%.0f", what,
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_call).count());
        dbg_log += b;
    };
    g_sync_us = 0.0;
    g_graph_us = 0.0;
    g_graph_n = 0;
    g_prep_us = 0.0;
    int iters_done = 0;
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
    // isFinite(g), |z0|^2 and |g|^2 enqueued together, read back after one
    // synchronisation (same kernels and partitions as plan_nonfinite / dnorm)
    double z0sq = 0.0, gsq = 0.0;
    {
        static_assert(kHvalDoubles >= 8, "hval holds the solver scalars");
        double* hv = p.hval.as<double>();
        double* vd = p.value.as<double>();
        dev_nonfinite(p.prec, g.p, len, p.flag.as<int>(), p.stream);
        dev_dot(p.prec, z0, z0, len, p.scratch.as<double>(), vd + 1, p.stream);
        dev_dot(p.prec, g.p, g.p, len, p.scratch.as<double>(), vd + 2, p.stream);
        PTG_CUDA(cudaMemcpyAsync(hv + 4, vd + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, p.stream));
        PTG_CUDA(cudaMemcpyAsync(hv + 6, p.flag.p, sizeof(int), cudaMemcpyDeviceToHost, p.stream));
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        int bad = 0;
        std::memcpy(&bad, hv + 6, sizeof(int));
        if (bad) raise(PTG_ERR_NUMERIC, "non-finite iterate in lbfgs");
        z0sq = hv[4];
        gsq = hv[5];
    }
    if (lbfgs_debug()) dbg_mark("nonfinite+norms");
    const double grad_floor = cfg.grad_tol_abs * (1.0 + std::sqrt(z0sq));
    const double g0 = std::sqrt(gsq);
    double gnorm = g0;
    hist_push(hist, ctr, cur, gnorm, z0);
    auto satisfied = [&](double gn) { return gn <= std::max(cfg.grad_tol_rel * g0, grad_floor); };
    SolveOut out;
    out.reason = PTG_STOP_MAXITERS;
    // Curvature pairs live in a ring of slots allocated on first use (memory+1:
    // a candidate pair is formed before its acceptance is known); the order
    // deque holds slot ids oldest..newest.  Fresh memory per call (solvers.cpp:100).
    const int mem = std::max(0, cfg.lbfgs_memory);
    std::vector<Pair> slots;
    std::deque<int> order;
    DVec ws;   // fused-kernel scratch (two-loop partials / pair statistics / products)
    double* wsd = nullptr;
    static_assert(kHvalDoubles >= 8, "hval holds the solver scalars");
    // pinned results of an iteration: [0] first trial's value, [1..5] pair
    // statistics, [9..] compact-mode products -- one block so the graph-replayed
    // iteration reads them back with a single copy
    constexpr size_t kRes = 9 + 4 * (size_t)(kMaxPairs + 1);
    HostPinned res_h;
    res_h.ensure(kRes * sizeof(double));
    double* stats_h = res_h.as<double>() + 1;
    // Direction: "compact" (default) — the compact representation of the same
    // LBFGS matrix (Byrd, Nocedal & Schnabel 1994): the O(k) products it needs
    // are batched into one pass per iteration and ride on the line search's
    // synchronisation, the k x k algebra runs on the host, and one combine
    // pass forms d; "fused" — the reference's two-loop recursion as one
    // cooperative kernel (bitwise = "ops"); "ops" — one kernel per operation.
    const char* tl = getenv("PTG_TWO_LOOP");
    const std::string mode = tl ? std::string(tl) : std::string("compact");
    bool fused = mode != "ops";
    const bool compact = mode == "compact" && mem <= kMaxPairs;
    const int nslot_max = mem + 1;
    std::vector<double> SY, YY, Sg, Yg;   // by slot id: <s_a, y_b>, <y_a, y_b>, <s_a, g>, <y_a, g>
    if (compact) {
        SY.assign((size_t)nslot_max * nslot_max, 0.0);
        YY.assign((size_t)nslot_max * nslot_max, 0.0);
        Sg.assign(nslot_max, 0.0);
        Yg.assign(nslot_max, 0.0);
    }
    double gg = g0 * g0;   // <g, g> of the current gradient
    // per-iterate-buffer graphs of the compact iteration (PTG_LBFGS_GRAPH=0: eager)
    struct IterGraph {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t nc = nullptr, nps = nullptr, nmd = nullptr, nms = nullptr;
        const void* z = nullptr;
        int64_t launches = 0;
        ~IterGraph() {
            if (exec) cudaGraphExecDestroy(exec);
            if (graph) cudaGraphDestroy(graph);
        }
    } ig[2];
    const bool use_graph = !(getenv("PTG_LBFGS_GRAPH") && getenv("PTG_LBFGS_GRAPH")[0] == '0');
    // fork/join resources of the captured iteration (the plan's side stream)
    if (use_graph && !p.s_side) {
        PTG_CUDA(cudaStreamCreateWithFlags(&p.s_side, cudaStreamNonBlocking));
        PTG_CUDA(cudaEventCreateWithFlags(&p.ev_side[0], cudaEventDisableTiming));
        PTG_CUDA(cudaEventCreateWithFlags(&p.ev_side[1], cudaEventDisableTiming));
    }
    cudaStream_t side = p.s_side;
    cudaEvent_t* ig_ev = p.ev_side;
    if (satisfied(gnorm)) {
        out.reason = PTG_STOP_TOLERANCE;
    } else {
        ws.s = p.stream;
        ws.bytes = ((size_t)kPairScratch + kMultiDotScratch + kRes) * sizeof(double);
        PTG_CUDA(cudaMallocAsync(&ws.p, ws.bytes, p.stream));
        PTG_CUDA(cudaMemsetAsync(ws.p, 0, ws.bytes, p.stream));
        wsd = static_cast<double*>(ws.p);
        double* md_scratch = wsd + kPairScratch;
        double* res_d = md_scratch + kMultiDotScratch;   // device image of res_h
        double* stats_d = res_d + 1;
        double* md_d = res_d + 9;
        if (lbfgs_debug()) { PTG_CUDA(cudaStreamSynchronize(p.stream)); dbg_mark("ws"); }
        // per-iteration host scratch, reused (no allocations on the iteration path)
        std::vector<const void*> sp, yp, msp, myp;
        std::vector<double> syv, t, u, c, rhs;
        for (auto* vec : {&sp, &yp, &msp, &myp}) vec->reserve(mem + 2);
        for (auto* vec : {&syv, &t, &u, &c, &rhs}) vec->reserve(mem + 2);
        for (int iter = 1; iter <= cfg.max_iters; ++iter) {
            const auto t_iter = std::chrono::steady_clock::now();
            sp.clear();
            yp.clear();
            syv.clear();
            for (int id : order) {
                sp.push_back(slots[id].s.p);
                yp.push_back(slots[id].y.p);
                syv.push_back(slots[id].sy);
            }
            const int k = (int)order.size();
            const bool graph_iter = compact && use_graph && iter > 2 && cfg.linesearch_max >= 1 && !p.timing;
            // compact mode: the direction launch is a kernel node (k_combine;
            // gamma = 1, no pairs = steepest descent, bitwise -g); replayed
            // iterations also form the first trial nz = z + dir in it
            const void* tz = graph_iter ? z.p : nullptr;
            void* tn = graph_iter ? nz.p : nullptr;
            KNode nc, nps, nmd, nms;
            if (compact) {
                if (k == 0) {
                    node_combine(p, nullptr, nullptr, nullptr, nullptr, 1.0, 0, g.p, dir.p, nc, tz, tn);
                } else {
                    // H g = gamma g + [S, gamma Y] [[R^-T (D + gamma Y'Y) R^-1, -R^-T], [-R^-1, 0]] [S'g; gamma Y'g]
                    auto sy = [&](int i, int j) { return SY[(size_t)order[i] * nslot_max + order[j]]; };
                    auto yy = [&](int i, int j) { return YY[(size_t)order[i] * nslot_max + order[j]]; };
                    const double gamma = sy(k - 1, k - 1) / yy(k - 1, k - 1);
                    t.assign(k, 0.0);
                    u.assign(k, 0.0);
                    c.assign(k, 0.0);
                    rhs.assign(k, 0.0);
                    for (int i = k - 1; i >= 0; --i) {   // R t = S'g (R upper triangular)
                        double a = Sg[order[i]];
                        for (int j = i + 1; j < k; ++j) a -= sy(i, j) * t[j];
                        t[i] = a / sy(i, i);
                    }
                    for (int i = 0; i < k; ++i) {        // rhs = (D + gamma Y'Y) t - gamma Y'g
                        double a = sy(i, i) * t[i];
                        for (int j = 0; j < k; ++j) a += gamma * yy(i, j) * t[j];
                        rhs[i] = a - gamma * Yg[order[i]];
                    }
                    for (int i = 0; i < k; ++i) {        // R' u = rhs
                        double a = rhs[i];
                        for (int j = 0; j < i; ++j) a -= sy(j, i) * u[j];
                        u[i] = a / sy(i, i);
                    }
                    double dg = gamma * gg;              // <H g, g>
                    for (int i = 0; i < k; ++i) {
                        c[i] = -gamma * t[i];
                        dg += u[i] * Sg[order[i]] + c[i] * Yg[order[i]];
                    }
                    if (-dg >= 0.0) node_combine(p, nullptr, nullptr, nullptr, nullptr, 1.0, 0, g.p, dir.p, nc, tz, tn);   // descent check
                    else node_combine(p, sp.data(), yp.data(), u.data(), c.data(), gamma, k, g.p, dir.p, nc, tz, tn);
                }
            } else {
                // fused two-loop + descent check, else the kernel-per-op path
                fused = fused && dev_two_loop(p, sp.data(), yp.data(), syv.data(), k, g.p, dir.p, wsd);
                if (!fused) {
                    two_loop(p, sp, yp, syv, g.p, dir.p);
                    if (plan_dot(p, dir.p, g.p, len) >= 0.0) dev_scale(p.prec, dir.p, g.p, -1.0, len, p.stream);
                }
            }
            // candidate pair slot (not in the order deque)
            int slot = -1;
            for (int i = 0; i < (int)slots.size() && slot < 0; ++i)
                if (std::find(order.begin(), order.end(), i) == order.end()) slot = i;
            if (slot < 0) {
                slots.push_back(Pair{DVec(p, len), DVec(p, len), 0.0});
                slot = (int)slots.size() - 1;
            }
            Pair& pr = slots[slot];
            // pair statistics (+ isFinite of the new iterate) of the accepted point
            // and, in compact mode, every product the next direction needs,
            // enqueued speculatively behind the first trial's evaluation
            msp.assign(sp.begin(), sp.end());
            myp.assign(yp.begin(), yp.end());
            msp.push_back(pr.s.p);
            myp.push_back(pr.y.p);
            if (compact) {
                node_pair_stats(p, nz.p, z.p, ng.p, g.p, pr.s.p, pr.y.p, wsd, stats_d, nps);
                // the products form the new pair themselves: independent of the
                // pair statistics kernel (the graph runs the two concurrently)
                node_multi_dot(p, msp.data(), myp.data(), k + 1, pr.y.p, ng.p, md_scratch, md_d, nmd, nms, nz.p,
                               z.p, g.p);
            }
            auto stats = [&]() {
                if (compact) {
                    node_launch(nps, p.stream);
                    PTG_CUDA(cudaMemcpyAsync(stats_h, stats_d, 5 * sizeof(double), cudaMemcpyDeviceToHost, p.stream));
                    node_launch(nmd, p.stream);
                    node_launch(nms, p.stream);
                    // fixed size (graph replay: the memcpy node is not rewritten)
                    PTG_CUDA(cudaMemcpyAsync(res_h.as<double>() + 9, md_d, 4 * (size_t)(kMaxPairs + 1) * sizeof(double),
                                             cudaMemcpyDeviceToHost, p.stream));
                } else {
                    dev_pair_stats(p, nz.p, z.p, ng.p, g.p, pr.s.p, pr.y.p, wsd, stats_d);
                    PTG_CUDA(cudaMemcpyAsync(stats_h, stats_d, 5 * sizeof(double), cudaMemcpyDeviceToHost, p.stream));
                }
            };
            LsOut lsr;
            if (graph_iter) {
                // direction + first trial (alpha = 1) + its evaluation + the pair
                // statistics and products, as one graph launch per iterate
                // buffer (z / nz swap): ~10 launches' host cost -> one launch and
                // four node-argument updates
                IterGraph& G = ig[0].z == z.p ? ig[0] : ig[1].z == z.p ? ig[1] : ig[0].exec ? ig[1] : ig[0];
                if (!G.exec) {
                    const int64_t l0 = p.launches;
                    PTG_CUDA(cudaStreamBeginCapture(p.stream, cudaStreamCaptureModeThreadLocal));
                    cudaGraph_t gr = nullptr;
                    try {
                        node_launch(nc, p.stream);                              // dir and nz = z + dir
                        ctr.record(obj.level, obj.weight);                      // charge before evaluating
                        p.pdl_frames = true;
                        plan_eval(p, obj.metric, nz.p, obj.v, ng.p, res_d);     // value -> res_d[0]
                        p.pdl_frames = false;
                        // fork: products on a side stream, pair statistics here
                        PTG_CUDA(cudaEventRecord(ig_ev[0], p.stream));
                        PTG_CUDA(cudaStreamWaitEvent(side, ig_ev[0], 0));
                        node_launch(nmd, side);
                        node_launch(nms, side);                                 // -> res_d[9..]
                        PTG_CUDA(cudaEventRecord(ig_ev[1], side));
                        node_launch(nps, p.stream);                             // -> res_d[1..5]
                        PTG_CUDA(cudaStreamWaitEvent(p.stream, ig_ev[1], 0));   // join
                        PTG_CUDA(cudaMemcpyAsync(res_h.p, res_d, kRes * sizeof(double), cudaMemcpyDeviceToHost,
                                                 p.stream));
                    } catch (...) {
                        p.pdl_frames = false;
                        cudaStreamEndCapture(p.stream, &gr);
                        if (gr) cudaGraphDestroy(gr);
                        throw;
                    }
                    PTG_CUDA(cudaStreamEndCapture(p.stream, &gr));
                    G.graph = gr;
                    PTG_CUDA(cudaGraphInstantiate(&G.exec, gr, 0));
                    G.launches = p.launches - l0;
                    size_t nn_ = 0;
                    PTG_CUDA(cudaGraphGetNodes(gr, nullptr, &nn_));
                    std::vector<cudaGraphNode_t> nodes(nn_);
                    PTG_CUDA(cudaGraphGetNodes(gr, nodes.data(), &nn_));
                    for (auto nd : nodes) {
                        cudaGraphNodeType ty;
                        PTG_CUDA(cudaGraphNodeGetType(nd, &ty));
                        if (ty != cudaGraphNodeTypeKernel) continue;
                        cudaKernelNodeParams kp{};
                        PTG_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
                        if (kp.func == nc.prm.func) G.nc = nd;
                        else if (kp.func == nps.prm.func) G.nps = nd;
                        else if (kp.func == nmd.prm.func) G.nmd = nd;
                        else if (kp.func == nms.prm.func) G.nms = nd;
                    }
                    if (!G.nc || !G.nps || !G.nmd || !G.nms) raise(PTG_ERR_INTERNAL, "lbfgs graph: node lookup");
                    G.z = z.p;
                } else {
                    PTG_CUDA(cudaGraphExecKernelNodeSetParams(G.exec, G.nc, &nc.prm));
                    PTG_CUDA(cudaGraphExecKernelNodeSetParams(G.exec, G.nps, &nps.prm));
                    PTG_CUDA(cudaGraphExecKernelNodeSetParams(G.exec, G.nmd, &nmd.prm));
                    PTG_CUDA(cudaGraphExecKernelNodeSetParams(G.exec, G.nms, &nms.prm));
                    ctr.record(obj.level, obj.weight);   // charge before evaluating (solvers.hpp:33-36)
                    p.launches += G.launches;
                }
                static thread_local cudaEvent_t dbg_ev[2] = {nullptr, nullptr};
                if (lbfgs_debug()) {
                    if (!dbg_ev[0]) {
                        PTG_CUDA(cudaEventCreate(&dbg_ev[0]));
                        PTG_CUDA(cudaEventCreate(&dbg_ev[1]));
                    }
                    PTG_CUDA(cudaEventRecord(dbg_ev[0], p.stream));
                }
                if (lbfgs_debug())
                    g_prep_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_iter).count();
                PTG_CUDA(cudaGraphLaunch(G.exec, p.stream));
                if (lbfgs_debug()) PTG_CUDA(cudaEventRecord(dbg_ev[1], p.stream));
                const auto ts = std::chrono::steady_clock::now();
                PTG_CUDA(cudaStreamSynchronize(p.stream));
                if (lbfgs_debug()) {
                    g_sync_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - ts).count();
                    float ms = 0.f;
                    cudaEventElapsedTime(&ms, dbg_ev[0], dbg_ev[1]);
                    g_graph_us += ms * 1e3;
                    ++g_graph_n;
                }
                lsr = d_linesearch_continue(obj, z.p, dir.p, ctr, cfg.linesearch_max, cur, nz.p, ng.p,
                                            res_h.as<double>()[0]);
            } else {
                if (compact) node_launch(nc, p.stream);
                lsr = d_linesearch(obj, z.p, dir.p, ctr, cfg.linesearch_max, &cur, nz.p, ng.p, stats);
            }
            if (lbfgs_debug() && iter <= 2) dbg_mark("ls");
            if (lsr.stalled) {
                out.reason = PTG_STOP_STALL;
                break;
            }
            if (lsr.trials > 1) {   // the speculative statistics were for a rejected trial
                stats();
                PTG_CUDA(cudaStreamSynchronize(p.stream));
            }
            if (stats_h[4] != 0.0) raise(PTG_ERR_NUMERIC, "non-finite iterate in lbfgs");
            pr.sy = stats_h[0];
            const bool accept = pr.sy > 1e-12 * std::sqrt(stats_h[1]) * std::sqrt(stats_h[2]);
            if (compact) {
                const double* md = res_h.as<double>() + 9;
                for (int a = 0; a <= k; ++a) {
                    const int sa = a < k ? order[a] : slot;
                    if (accept) {
                        SY[(size_t)sa * nslot_max + slot] = md[4 * a];
                        YY[(size_t)sa * nslot_max + slot] = md[4 * a + 1];
                        YY[(size_t)slot * nslot_max + sa] = md[4 * a + 1];
                    }
                    Sg[sa] = md[4 * a + 2];
                    Yg[sa] = md[4 * a + 3];
                }
                gg = stats_h[3];
            }
            if (accept) {
                order.push_back(slot);
                if ((int)order.size() > mem) order.pop_front();
            }
            std::swap(z, nz);
            std::swap(g, ng);
            ++iters_done;
            cur = lsr.value;
            gnorm = std::sqrt(stats_h[3]);
            hist_push(hist, ctr, cur, gnorm, z.p);
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
    if (lbfgs_debug() && iters_done > 0) {
        const double tot = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_call).count();
        fprintf(stderr, "[lbfgs] n=%d iters %d: %.1f us/iter wall, %.1f us/iter in line-search syncs, graph %.1f us GPU, "
                "host prep %.1f us |%s\n",
                p.n, iters_done, tot / iters_done, g_sync_us / iters_done, g_graph_n ? g_graph_us / g_graph_n : 0.0,
                g_graph_n ? g_prep_us / g_graph_n : 0.0, dbg_log.c_str());
    }
    return out;
}

// ------------------------------------------------------- truncated Newton
// solvers.cpp:143-227: CG on H x = -g from x = 0, H v ~ (grad(z + d v) - g)/d
// with d = 1e-6 (1 + |z|)/|v| (one counted evaluation per product), truncated
// on negative curvature; steepest descent if CG gives nothing usable.
SolveOut d_truncated_newton(const DObj& obj, const void* z0, const ptg_solver_cfg& cfg, Counter& ctr,
                            const double* warm_value, const void* warm_g, void* z_out, void* g_out,
                            std::vector<ptg_hist>* hist) {
    Plan& p = *obj.plan;
    LaunchScope ls(p);
    const size_t len = p.nn();
    const int pr = p.prec;
    cudaStream_t st = p.stream;
    DVec z(p, len), g(p, len), x(p, len), r(p, len), pv(p, len), hp(p, len), zp(p, len), gp(p, len),
        nz(p, len), ng(p, len);
    dev_copy(pr, z.p, z0, len, st);
    double cur;
    if (warm_value) {
        cur = *warm_value;
        dev_copy(pr, g.p, warm_g, len, st);
    } else {
        cur = obj.eval(ctr, z.p, g.p);
    }
    if (plan_nonfinite(p, g.p, len)) raise(PTG_ERR_NUMERIC, "non-finite iterate in truncatedNewton");
    const double grad_floor = cfg.grad_tol_abs * (1.0 + dnorm(p, z0));
    const double g0 = dnorm(p, g.p);
    double gnorm = g0;
    hist_push(hist, ctr, cur, gnorm, z0);
    auto satisfied = [&](double gn) { return gn <= std::max(cfg.grad_tol_rel * g0, grad_floor); };
    SolveOut out;
    out.reason = PTG_STOP_MAXITERS;
    if (satisfied(gnorm)) {
        out.reason = PTG_STOP_TOLERANCE;
    } else {
        for (int iter = 1; iter <= cfg.max_iters; ++iter) {
            dev_fill_zero(pr, x.p, len, st);
            dev_scale(pr, r.p, g.p, -1.0, len, st);
            const double rhs_norm = dnorm(p, r.p);
            dev_copy(pr, pv.p, r.p, len, st);
            double rs = plan_dot(p, r.p, r.p, len);
            for (int cg = 0; cg < cfg.cg_max_iters; ++cg) {
                const double vnorm = dnorm(p, pv.p);
                if (vnorm == 0.0) {
                    dev_fill_zero(pr, hp.p, len, st);
                } else {
                    const double delta = 1e-6 * (1.0 + dnorm(p, z.p)) / vnorm;
                    dev_add_scaled(pr, zp.p, z.p, delta, pv.p, len, st);
                    obj.eval(ctr, zp.p, gp.p);
                    dev_sub(pr, hp.p, gp.p, g.p, len, st);
                    dev_scale(pr, hp.p, hp.p, 1.0 / delta, len, st);
                }
                const double php = plan_dot(p, pv.p, hp.p, len);
                if (php <= 0.0) {
                    if (cg == 0) dev_copy(pr, x.p, r.p, len, st);
                    break;
                }
                const double step = rs / php;
                dev_axpy(pr, x.p, step, pv.p, len, st);
                dev_axpy(pr, r.p, -step, hp.p, len, st);
                const double rs_new = plan_dot(p, r.p, r.p, len);
                if (std::sqrt(rs_new) <= cfg.cg_rel_tol * rhs_norm) break;
                dev_copy(pr, zp.p, r.p, len, st);   // p = r + beta p
                dev_axpy(pr, zp.p, rs_new / rs, pv.p, len, st);
                std::swap(pv, zp);
                rs = rs_new;
            }
            if (dnorm(p, x.p) == 0.0 || plan_dot(p, x.p, g.p, len) >= 0.0) dev_scale(pr, x.p, g.p, -1.0, len, st);
            LsOut lsr = d_linesearch(obj, z.p, x.p, ctr, cfg.linesearch_max, &cur, nz.p, ng.p);
            if (lsr.stalled) {
                out.reason = PTG_STOP_STALL;
                break;
            }
            if (plan_nonfinite(p, nz.p, len)) raise(PTG_ERR_NUMERIC, "non-finite iterate in truncatedNewton");
            std::swap(z, nz);
            std::swap(g, ng);
            cur = lsr.value;
            gnorm = dnorm(p, g.p);
            hist_push(hist, ctr, cur, gnorm, z.p);
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
    dev_copy(pr, z_out, z.p, len, st);
    if (g_out) dev_copy(pr, g_out, g.p, len, st);
    out.value = cur;
    PTG_CUDA(cudaStreamSynchronize(st));
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
    if (pc.stream != p.stream) PTG_CUDA(cudaStreamSynchronize(pc.stream));
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
    hist_push(hist, ctr, cur, gnorm, z.p);
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
            hist_push(hist, ctr, cur, gnorm, z.p);
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
