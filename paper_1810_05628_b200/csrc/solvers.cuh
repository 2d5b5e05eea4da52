// solvers.cuh — GPU-resident solver control flow (host C++ over device vectors).
//
// Restates /root/reference/proj/src/solvers.cpp:19-141 (two-loop LBFGS,
// backtracking line search) and multigrid.cpp:95-227 (hierarchy, V-cycle,
// driver) with every iterate, gradient, curvature pair and shift resident in
// HBM.  Only scalars (objective values, dot products) cross PCIe, one
// synchronising read each.  Accounting (EvalCounter: charge before evaluate,
// weight 4^-level) and all control decisions are identical to the reference.
#pragma once

#include <deque>
#include <functional>
#include <memory>
#include <vector>

#include "plan.cuh"

namespace ptg {

struct Counter {
    double weighted = 0.0;
    long per_level[16] = {};
    void record(int level, double w) {
        weighted += w;
        if (level >= 0 && level < 16) ++per_level[level];
    }
};

// device vector in a plan's precision, stream-ordered allocation
struct DVec {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    DVec() = default;
    DVec(Plan& pl, size_t len) { alloc(pl, len); }
    DVec(const DVec&) = delete;
    DVec& operator=(const DVec&) = delete;
    DVec(DVec&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr; o.bytes = 0; }
    DVec& operator=(DVec&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            bytes = o.bytes;
            s = o.s;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DVec() { release(); }
    void alloc(Plan& pl, size_t len) {
        release();
        s = pl.stream;
        bytes = len * pl.celem();
        if (bytes) PTG_CUDA(cudaMallocAsync(&p, bytes, s));
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        bytes = 0;
    }
};

// CountedObjective (solvers.hpp:28-37) bound to a device plan
struct DObj {
    Plan* plan = nullptr;
    int metric = PTG_DISTANCE;
    const void* v = nullptr;   // shift (device), nullptr = none
    int level = 0;
    double weight = 1.0;
    double eval(Counter& c, const void* z, void* grad) const;
    // charge + enqueue the evaluation and the value's copy into host_value
    // (pinned); the caller synchronises the plan's stream
    void eval_enqueue(Counter& c, const void* z, void* grad, double* host_value) const;
};

struct SolveOut {
    double value = 0.0;
    int reason = PTG_STOP_MAXITERS;
};

// solvers.cpp:61-85; trials are formed in z_out (gradient in g_out), so the
// accepted point needs no copy; on a stall z_out = z and g_out is scratch.
// z_out / g_out must not alias z / dir.  first_trial_hook (optional) is
// called once, after the first trial's evaluation is enqueued and before the
// stream is synchronised: work that assumes that trial is accepted (the
// common case) rides on the same synchronisation.
struct LsOut {
    double alpha = 0.0, value = 0.0;
    bool stalled = false;
    int trials = 0;
};
LsOut d_linesearch(const DObj& obj, const void* z, const void* dir, Counter& ctr, int max_trials,
                   const double* phi0, void* z_out, void* g_out,
                   const std::function<void()>& first_trial_hook = {});

// fused LBFGS kernels (lbfgs_dev.cu)
constexpr int kMaxPairs = 64;
// q = -H g by the two-loop recursion over pairs (s[i], y[i], sy[i]) oldest..newest,
// then the descent check (<q,g> >= 0 -> q = -g); one cooperative launch.
// scratch: 2 x kReduceBlocks doubles.  false = not launched (too many pairs /
// device cannot co-schedule the grid): use the kernel-per-op path.
bool dev_two_loop(const Plan& p, const void* const* s, const void* const* y, const double* sy, int k,
                  const void* g, void* q, double* scratch);
// compact representation (Byrd, Nocedal & Schnabel 1994) of the same LBFGS
// matrix: 4 products per pair a < A against two shared vectors yc, gn
// (<s_a,yc>, <y_a,yc>, <s_a,gn>, <y_a,gn> -> out_dev[4a..4a+3]); scratch:
// 4 (kMaxPairs + 1) kReduceBlocks doubles
void dev_multi_dot(const Plan& p, const void* const* s, const void* const* y, int A, const void* yc,
                   const void* gn, double* scratch, double* out_dev);
// dir = -(gamma g + sum u_i s_i + sum c_i y_i)
void dev_combine(const Plan& p, const void* const* s, const void* const* y, const double* u, const double* c,
                 double gamma, int k, const void* g, void* dir);
constexpr size_t kMultiDotScratch = 4 * (size_t)(kMaxPairs + 1) * kReduceBlocks;
// s = nz - z, y = ng - g; out_dev[0..4] = <s,y>, <s,s>, <y,y>, <ng,ng>,
// count of blocks holding a non-finite nz entry.
// scratch: kPairScratch doubles, zeroed before the first use
constexpr int kPairScratch = 5 * kReduceBlocks + 2;
void dev_pair_stats(const Plan& p, const void* nz, const void* z, const void* ng, const void* g, void* s_out,
                    void* y_out, double* scratch, double* out_dev);

// The launches of dev_combine / dev_pair_stats / dev_multi_dot (+ its sum)
// as kernel-node parameters with their argument storage, for graph replay
// (d_lbfgs rewrites them in an instantiated graph every iteration).
struct KNode {
    cudaKernelNodeParams prm{};
    void* argp[12] = {};
    alignas(16) unsigned char store[2 * (kMaxPairs + 1) * 8 + 2 * kMaxPairs * 8 + 128] = {};
};
// z0 / trial (optional): also form the first line-search trial z0 + 1 * dir
void node_combine(const Plan& p, const void* const* s, const void* const* y, const double* u, const double* c,
                  double gamma, int k, const void* g, void* dir, KNode& n, const void* z0 = nullptr,
                  void* trial = nullptr);
void node_pair_stats(const Plan& p, const void* nz, const void* z, const void* ng, const void* g, void* s_out,
                     void* y_out, double* scratch, double* out_dev, KNode& n);
// zn / zo / go (optional): form the newest pair (s = zn - zo, y = gn - go) and
// yc in-kernel instead of reading what dev_pair_stats stores (no dependency)
void node_multi_dot(const Plan& p, const void* const* s, const void* const* y, int A, const void* yc,
                    const void* gn, double* scratch, double* out_dev, KNode& md, KNode& ms,
                    const void* zn = nullptr, const void* zo = nullptr, const void* go = nullptr);
void node_launch(const KNode& n, cudaStream_t s);

// solvers.cpp:87-141.  warm_g (device) with *warm_value, or null to evaluate.
SolveOut d_lbfgs(const DObj& obj, const void* z0, const ptg_solver_cfg& cfg, Counter& ctr,
                 const double* warm_value, const void* warm_g, void* z_out, void* g_out,
                 std::vector<ptg_hist>* hist);

// solvers.cpp:143-227 (Newton-CG, finite-difference Hessian-vector products)
SolveOut d_truncated_newton(const DObj& obj, const void* z0, const ptg_solver_cfg& cfg, Counter& ctr,
                            const double* warm_value, const void* warm_g, void* z_out, void* g_out,
                            std::vector<ptg_hist>* hist);

struct Hier {
    Plan* fine = nullptr;
    std::vector<std::unique_ptr<Plan>> owned;   // levels 1..depth-1
    std::vector<Plan*> levels;
    int metric = PTG_DISTANCE;
    ptg_mg_cfg opt{};
    int coarsest_iters = 3;
    int depth() const { return (int)levels.size(); }
};

// IterationCallback (solvers.hpp:70-71) of the top-level solver call: set by
// the C-ABI for the duration of one call; fired wherever a top-level solver
// appends a history point (initial point + one per iteration / cycle) with
// the device iterate.  Nested solvers (smoothers, coarse solves) keep no
// history and so never fire it.
using IterHook = std::function<void(int iter, const void* z_dev, double value, double weighted)>;
extern thread_local const IterHook* g_iter_hook;
inline void hist_push(std::vector<ptg_hist>* hist, const Counter& ctr, double value, double gnorm, const void* z_dev) {
    if (!hist) return;
    hist->push_back({ctr.weighted, value, gnorm});
    if (g_iter_hook) (*g_iter_hook)((int)hist->size() - 1, z_dev, value, ctr.weighted);
}

std::unique_ptr<Hier> hier_build(Plan& fine, int metric, int depth, const ptg_mg_cfg& opt);
// multigrid.cpp:117-169 ; v may be null (= zero shift)
double d_mgopt_cycle(Hier& h, int level, const void* z, const void* v, Counter& ctr,
                     const double* warm_value, const void* warm_g, void* z_out, void* g_out);
// multigrid.cpp:171-227
SolveOut d_mgopt_driver(Hier& h, const void* z0, const ptg_driver_cfg& cfg, Counter& ctr,
                        void* z_out, std::vector<ptg_hist>* hist);

}  // namespace ptg
