// capi.cu — extern "C" boundary of libptg (include/ptg.h).
//
// Every entry point converts ptg::Status exceptions (and std::bad_alloc,
// CUDA errors) into an int status and a thread-local message, mirroring the
// reference's exception hierarchy (/root/reference/proj/include/ptycho/
// errors.hpp:12-43) so a C++ shim can re-throw the matching type.
#include <cmath>
#include <cstring>
#include <limits>
#include <new>
#include <random>
#include <string>

#include "plan.cuh"
#include "metrics.cuh"
#include "solvers.cuh"
#include "transfer.cuh"

struct ptg_plan {
    std::unique_ptr<ptg::Plan> p;
};
struct ptg_comm {
    ptg::Comm* c = nullptr;
};
struct ptg_hier {
    std::unique_ptr<ptg::Hier> h;
    ptg_plan* fine;
    std::vector<ptg_plan> views;   // non-owning plan handles for coarse levels
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return PTG_OK;
    } catch (const ptg::Status& s) {
        g_err = s.what();
        return s.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return PTG_ERR_INTERNAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PTG_ERR_INTERNAL;
    }
}

ptg::Plan& P(ptg_plan* p) {
    if (!p || !p->p) ptg::raise(PTG_ERR_CONFIG, "objective is not bound to geometry/data (null plan)");
    PTG_CUDA(cudaSetDevice(p->p->device));
    return *p->p;
}

// the solvers / PIE / hierarchies need whole-object vectors on every rank
ptg::Plan& P_whole(ptg_plan* p, const char* what) {
    ptg::Plan& pl = P(p);
    if (pl.shard.layout == PTG_SHARD_BANDS)
        ptg::raise(PTG_ERR_CONFIG, std::string(what) + " on an object-band shard is not supported (evaluation only); "
                                                       "use the replicated layout");
    return pl;
}

void fill_report(ptg_report* rep, const ptg::Counter& c, double value, int reason, int hist_len) {
    if (!rep) return;
    rep->final_value = value;
    rep->weighted = c.weighted;
    for (int i = 0; i < 16; ++i) rep->per_level[i] = c.per_level[i];
    rep->reason = reason;
    rep->hist_len = hist_len;
}

// IterationCallback bridge: while alive, the top-level solver's history
// points download the device iterate (complex128) and call the user's function
struct CbScope {
    ptg::IterHook fn;
    const ptg::IterHook* prev;
    CbScope(ptg::Plan& p, ptg_iter_cb cb, void* user) : prev(ptg::g_iter_hook) {
        if (!cb) return;
        fn = [&p, cb, user](int it, const void* zd, double val, double w) {
            std::vector<double> h(2 * p.nn());
            ptg::plan_download_c128(p, zd, h.data());
            PTG_CUDA(cudaStreamSynchronize(p.stream));
            cb(user, it, h.data(), val, w);
        };
        ptg::g_iter_hook = &fn;
    }
    ~CbScope() { ptg::g_iter_hook = prev; }
};

int copy_hist(const std::vector<ptg_hist>& h, ptg_hist* out, int cap) {
    const int n = (int)h.size();
    if (out)
        for (int i = 0; i < n && i < cap; ++i) out[i] = h[i];
    return n;
}
}  // namespace

namespace {
template <class F>
void with_device_buffers(size_t in_bytes, const void* in, size_t out_bytes, void* out, F&& f) {
    ptg::DevMem a, b;
    a.alloc(in_bytes);
    b.alloc(out_bytes);
    PTG_CUDA(cudaMemcpy(a.p, in, in_bytes, cudaMemcpyHostToDevice));
    f(a.p, b.p);
    PTG_CUDA(cudaDeviceSynchronize());
    PTG_CUDA(cudaMemcpy(out, b.p, out_bytes, cudaMemcpyDeviceToHost));
}
}  // namespace

static void sync_streams(ptg::Hier& h) {
    for (auto* l : h.levels) l->stream = h.fine->stream;
}

extern "C" {

const char* ptg_last_error(void) { return g_err.c_str(); }

int ptg_version(void) { return 1; }

int ptg_device_count(int* count) {
    return guard([&] {
        int c = 0;
        cudaError_t e = cudaGetDeviceCount(&c);
        if (e != cudaSuccess) c = 0;
        *count = c;
    });
}

void ptg_solver_cfg_default(ptg_solver_cfg* c) {
    c->max_iters = 100;
    c->grad_tol_rel = 0.0;
    c->grad_tol_abs = 1e-13;
    c->lbfgs_memory = 25;
    c->linesearch_max = 50;
    c->max_weighted = std::numeric_limits<double>::infinity();
    c->cg_max_iters = 20;
    c->cg_rel_tol = 0.1;
}

void ptg_mg_cfg_default(ptg_mg_cfg* c) {
    c->k1 = 1;
    c->k2 = 1;
    c->coarsest_max_iters = 0;
    c->coarsest_grad_tol_rel = 1e-4;
    c->intermediate_grad_tol_rel = 1e-3;
    c->lbfgs_memory = 25;
    c->linesearch_max = 50;
    c->grad_tol_abs = 1e-13;
}

void ptg_driver_cfg_default(ptg_driver_cfg* c) {
    c->budget = 100.0;
    c->grad_tol_rel = 0.0;
    c->grad_tol_abs = 1e-13;
    c->max_cycles = 1000000;
}

int ptg_plan_create(const ptg_plan_desc* desc, ptg_plan** out) {
    return guard([&] {
        if (!desc || !out) ptg::raise(PTG_ERR_CONFIG, "null argument");
        *out = nullptr;
        auto h = new ptg_plan;
        try {
            h->p = ptg::plan_create(*desc);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int ptg_plan_destroy(ptg_plan* plan) {
    return guard([&] {
        if (!plan) return;
        if (plan->p) {
            cudaSetDevice(plan->p->device);
            cudaStreamSynchronize(plan->p->stream);
            plan->p.reset();   // ~Plan releases the plan's own streams and events
        }
        delete plan;
    });
}

int ptg_plan_set_stream(ptg_plan* plan, void* stream) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        p.stream = stream ? static_cast<cudaStream_t>(stream) : p.own_stream;
    });
}

int ptg_plan_set_data(ptg_plan* plan, const void* host_data, int dtype) {
    return guard([&] { ptg::plan_set_data_host(P(plan), host_data, dtype); });
}

int ptg_plan_set_data_device(ptg_plan* plan, const void* dev_data, int dtype) {
    return guard([&] { ptg::plan_set_data_device(P(plan), dev_data, dtype); });
}

int ptg_plan_load_ptyf(ptg_plan* plan, const char* path) {
    return guard([&] { ptg::plan_load_ptyf(P(plan), path); });
}

int ptg_plan_get_data(ptg_plan* plan, int metric, double* out) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        ptg::LaunchScope ls(p);
        ptg::plan_ensure(p, metric);
        const size_t len = (size_t)p.N * p.MM();
        if (!len) return;
        ptg::DevMem d64;
        d64.alloc(len * 8);
        const void* src = metric == PTG_DISTANCE ? p.amp.p : p.inten.p;
        ptg::dev_real_convert(PTG_C128, d64.p, p.prec == PTG_C64 ? PTG_F32 : PTG_F64, src, len, p.stream);
        PTG_CUDA(cudaMemcpyAsync(out, d64.p, len * 8, cudaMemcpyDeviceToHost, p.stream));
        PTG_CUDA(cudaStreamSynchronize(p.stream));
    });
}

int ptg_plan_info(const ptg_plan* plan, int* n, int* M, int* w, int* N, int* precision,
                  size_t* device_bytes) {
    return guard([&] {
        if (!plan || !plan->p) ptg::raise(PTG_ERR_CONFIG, "null plan");
        const ptg::Plan& p = *plan->p;
        if (n) *n = p.n;
        if (M) *M = p.M;
        if (w) *w = p.w;
        if (N) *N = p.N;
        if (precision) *precision = p.prec;
        if (device_bytes) *device_bytes = p.device_bytes();
    });
}

int ptg_plan_launch_count(const ptg_plan* plan, int64_t* count) {
    return guard([&] {
        if (!plan || !plan->p) ptg::raise(PTG_ERR_CONFIG, "null plan");
        *count = plan->p->launches;
    });
}

int ptg_plan_set_timing(ptg_plan* plan, int enable) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        p.timing = enable != 0;
        p.ev_used = 0;
    });
}

int ptg_plan_get_timing(ptg_plan* plan, double* frame_ms, int64_t* frame_launches,
                        double* gather_ms, int64_t* gather_launches) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        double ms[3];
        int64_t cnt[3];
        p.timing_collect(ms, cnt);
        if (cnt[2]) fprintf(stderr, "[ptg] probe launches: %lld, avg %.3f us\n", (long long)cnt[2], 1e3 * ms[2] / cnt[2]);
        if (frame_ms) *frame_ms = ms[0];
        if (frame_launches) *frame_launches = cnt[0];
        if (gather_ms) *gather_ms = ms[1];
        if (gather_launches) *gather_launches = cnt[1];
    });
}

int ptg_eval(ptg_plan* plan, int metric, const double* z, const double* v, double* value,
             double* grad) {
    return guard([&] {
        ptg::plan_eval_host(P(plan), metric, z, v, value, grad);
    });
}

int ptg_eval_device(ptg_plan* plan, int metric, const void* z, const void* v, void* grad,
                    double* value_dev, double* value_host) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        double* vd = value_dev ? value_dev : p.value.as<double>();
        ptg::plan_eval(p, metric, z, v, grad, vd);
        if (value_host) *value_host = ptg::plan_read_scalar(p, vd);
    });
}

int ptg_project_modulus(ptg_plan* plan, const double* z, int k, double* frame) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        p.zbuf.ensure(p.nn() * p.celem());
        ptg::plan_upload_c128(p, z, p.zbuf.p);
        ptg::DevMem out;
        out.alloc(p.MM() * p.celem());
        ptg::plan_project(p, p.zbuf.p, k, out.p);
        ptg::DevMem out64;
        out64.alloc(p.MM() * 16);
        {
            ptg::LaunchScope ls(p);
            ptg::dev_to_c128(p.prec, out64.as<double>(), out.p, p.MM(), p.stream);
        }
        PTG_CUDA(cudaMemcpyAsync(frame, out64.p, p.MM() * 16, cudaMemcpyDeviceToHost, p.stream));
        PTG_CUDA(cudaStreamSynchronize(p.stream));
    });
}

int ptg_simulate(ptg_plan* plan, const double* z, double* data_out) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        p.zbuf.ensure(p.nn() * p.celem());
        ptg::plan_upload_c128(p, z, p.zbuf.p);
        ptg::plan_simulate(p, p.zbuf.p);
        if (data_out) {
            const size_t len = (size_t)p.N * p.MM();
            ptg::DevMem d64;
            d64.alloc(std::max<size_t>(1, len) * 8);
            {
                ptg::LaunchScope ls(p);
                ptg::dev_real_convert(PTG_C128, d64.p, p.prec == PTG_C64 ? PTG_F32 : PTG_F64, p.inten.p, len, p.stream);
            }
            PTG_CUDA(cudaMemcpyAsync(data_out, d64.p, len * 8, cudaMemcpyDeviceToHost, p.stream));
        }
        PTG_CUDA(cudaStreamSynchronize(p.stream));
    });
}

int ptg_simulate_device(ptg_plan* plan, const void* z) {
    return guard([&] { ptg::plan_simulate(P(plan), z); });
}

int ptg_add_noise(ptg_plan* plan, double level, uint64_t seed, const double* uniforms) {
    return guard([&] { ptg::plan_add_noise(P(plan), level, (unsigned long long)seed, uniforms); });
}

int ptg_add_poisson(ptg_plan* plan, double photons, uint64_t seed) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        ptg::plan_add_poisson(p, photons, (unsigned long long)seed);
        PTG_CUDA(cudaStreamSynchronize(p.stream));
    });
}

int ptg_uniform01_stream(uint64_t seed, size_t count, double* out) {
    return guard([&] {
        std::mt19937_64 eng(seed);
        for (size_t i = 0; i < count; ++i) out[i] = (double)(eng() >> 11) * 0x1.0p-53;
    });
}

int ptg_philox4x64(int device, const uint64_t ctr[4], const uint64_t key[2], size_t nblocks, uint64_t* out) {
    return guard([&] {
        ptg::check_device_public(device);
        ptg::DevMem d;
        d.alloc(std::max<size_t>(1, nblocks) * 32);
        const unsigned long long c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]}, k[2] = {key[0], key[1]};
        ptg::dev_philox_raw(d.as<unsigned long long>(), nblocks, c, k, nullptr);
        PTG_CUDA(cudaDeviceSynchronize());
        if (nblocks) PTG_CUDA(cudaMemcpy(out, d.p, nblocks * 32, cudaMemcpyDeviceToHost));
    });
}

int ptg_pie(ptg_plan* plan, double* z, double gamma, int sweeps, double max_weighted,
            double* final_value, ptg_hist* hist, int hist_cap, int* hist_len, double* weighted,
            int* reason) {
    return ptg_pie_cb(plan, z, gamma, sweeps, max_weighted, final_value, hist, hist_cap, hist_len, weighted, reason,
                      nullptr, nullptr);
}

int ptg_pie_cb(ptg_plan* plan, double* z, double gamma, int sweeps, double max_weighted,
               double* final_value, ptg_hist* hist, int hist_cap, int* hist_len, double* weighted,
               int* reason, ptg_iter_cb cb, void* user) {
    return guard([&] {
        ptg::Plan& p = P_whole(plan, "pie");
        if (gamma < 0.0) ptg::raise(PTG_ERR_CONFIG, "pie: gamma must be non-negative");
        const size_t len = p.nn();
        ptg::DVec zd(p, len), gd(p, len);
        ptg::plan_upload_c128(p, z, zd.p);
        std::vector<ptg_hist> h;
        ptg::Counter ctr;
        auto diag = [&]() {   // uncounted diagnostic evaluation (solvers.cpp:238,254,263)
            ptg::plan_eval(p, PTG_DISTANCE, zd.p, nullptr, gd.p, p.value.as<double>());
            const double val = ptg::plan_read_scalar(p, p.value.as<double>());
            return val;
        };
        CbScope cbs(p, cb, user);
        double val = diag();
        ptg::hist_push(&h, ctr, val, std::sqrt(ptg::plan_dot(p, gd.p, gd.p, len)), zd.p);
        int rsn = PTG_STOP_MAXITERS;
        for (int sweep = 1; sweep <= sweeps; ++sweep) {
            ptg::plan_pie_sweep(p, zd.p, gamma);
            if (ptg::plan_nonfinite(p, zd.p, len)) ptg::raise(PTG_ERR_NUMERIC, "non-finite iterate in pie");
            ctr.record(0, 1.0);   // one sweep = one fine-level evaluation
            val = diag();
            ptg::hist_push(&h, ctr, val, std::sqrt(ptg::plan_dot(p, gd.p, gd.p, len)), zd.p);
            if (ctr.weighted >= max_weighted) {
                rsn = PTG_STOP_BUDGET;
                break;
            }
        }
        val = diag();
        ptg::plan_download_c128(p, zd.p, z);
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        if (final_value) *final_value = val;
        const int n = copy_hist(h, hist, hist_cap);
        if (hist_len) *hist_len = n;
        if (weighted) *weighted = ctr.weighted;
        if (reason) *reason = rsn;
    });
}

int ptg_pie_sweep_device(ptg_plan* plan, void* z, double gamma) {
    return guard([&] { ptg::plan_pie_sweep(P(plan), z, gamma); });
}

// ------------------------------------------------------------- transfers

int ptg_restrict_field(const double* fine, int n, double* coarse) {
    return guard([&] {
        if (n < 2 || n % 2 != 0)
            ptg::raise(PTG_ERR_GEOMETRY, "restrictField: grid side must be even and >= 2, got " + std::to_string(n));
        const size_t fb = (size_t)n * n * 16, cb = (size_t)(n / 2) * (n / 2) * 16;
        with_device_buffers(fb, fine, cb, coarse, [&](void* a, void* b) {
            ptg::dev_restrict_field(PTG_C128, a, n, b, nullptr);
        });
    });
}

int ptg_prolong_field(const double* coarse, int nH, double* fine) {
    return guard([&] {
        if (nH < 1) ptg::raise(PTG_ERR_GEOMETRY, "prolongField: empty grid");
        const size_t cb = (size_t)nH * nH * 16, fb = (size_t)4 * nH * nH * 16;
        with_device_buffers(cb, coarse, fb, fine, [&](void* a, void* b) {
            ptg::dev_prolong_field(PTG_C128, a, nH, b, nullptr);
        });
    });
}

int ptg_restrict_data(const double* fine, int N, int M, double* coarse) {
    return guard([&] {
        if (M < 4 || M % 4 != 0) ptg::raise(PTG_ERR_GEOMETRY, "restrictData: grid side must be a multiple of 4");
        if (N <= 0) return;
        const size_t fb = (size_t)N * M * M * 8, cb = (size_t)N * (M / 2) * (M / 2) * 8;
        with_device_buffers(fb, fine, cb, coarse, [&](void* a, void* b) {
            ptg::dev_restrict_data(PTG_F64, a, N, M, b, 1.0 / 16.0, nullptr);
        });
    });
}

int ptg_restrict_field_device(int precision, const void* fine, int n, void* coarse, void* stream) {
    return guard([&] { ptg::dev_restrict_field(precision, fine, n, coarse, (cudaStream_t)stream); });
}

int ptg_prolong_field_device(int precision, const void* coarse, int nH, void* fine, void* stream) {
    return guard([&] { ptg::dev_prolong_field(precision, coarse, nH, fine, (cudaStream_t)stream); });
}

int ptg_restrict_data_device(int dtype, const void* fine, int N, int M, void* coarse, void* stream) {
    return guard([&] { ptg::dev_restrict_data(dtype, fine, N, M, coarse, 1.0 / 16.0, (cudaStream_t)stream); });
}

// ------------------------------------------------------ band exchange (halo.cu)
size_t ptg_halo_bytes(int precision, int n, int ov) { return ptg::halo_bytes(precision, n, ov); }

int ptg_halo_pack(int precision, const void* grad, int n, int ov, const double* val_dev, void* buf, void* stream) {
    return guard([&] {
        if (!grad || !val_dev || !buf) ptg::raise(PTG_ERR_CONFIG, "ptg_halo_pack: null pointer");
        ptg::dev_halo_pack(precision, grad, n, ov, val_dev, buf, (cudaStream_t)stream);
    });
}

int ptg_halo_unpack(int precision, void* grad, int n, int ov, const void* all, int rank, int world, double* val_dev,
                    void* stream) {
    return guard([&] {
        if (!grad || !val_dev || !all) ptg::raise(PTG_ERR_CONFIG, "ptg_halo_unpack: null pointer");
        ptg::dev_halo_unpack(precision, grad, n, ov, all, rank, world, val_dev, (cudaStream_t)stream);
    });
}

// ---------------------------------------------------------------- solvers
int ptg_lbfgs(ptg_plan* plan, int metric, const double* v, const double* z0,
              const ptg_solver_cfg* cfg, double* z_out, double* grad_out, ptg_report* rep,
              ptg_hist* hist, int hist_cap) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        ptg_solver_cfg c;
        if (cfg) c = *cfg;
        else ptg_solver_cfg_default(&c);
        const size_t len = p.nn();
        ptg::DVec zd(p, len), vd, zo(p, len), go(p, len);
        ptg::plan_upload_c128(p, z0, zd.p);
        if (v) {
            vd.alloc(p, len);
            ptg::plan_upload_c128(p, v, vd.p);
        }
        ptg::DObj obj;
        obj.plan = &p;
        obj.metric = metric;
        obj.v = v ? vd.p : nullptr;
        ptg::Counter ctr;
        std::vector<ptg_hist> h;
        ptg::SolveOut o = ptg::d_lbfgs(obj, zd.p, c, ctr, nullptr, nullptr, zo.p, go.p, &h);
        if (z_out) ptg::plan_download_c128(p, zo.p, z_out);
        if (grad_out) ptg::plan_download_c128(p, go.p, grad_out);
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        fill_report(rep, ctr, o.value, o.reason, copy_hist(h, hist, hist_cap));
    });
}

namespace {
int solve_ex(bool tn, ptg_plan* plan, int metric, const double* v, const double* z0, const double* warm_value,
             const double* warm_grad, const ptg_solver_cfg* cfg, double* z_out, double* grad_out, ptg_report* rep,
             ptg_hist* hist, int hist_cap, ptg_iter_cb cb, void* user) {
    return guard([&] {
        ptg::Plan& p = P_whole(plan, tn ? "truncatedNewton" : "lbfgs");
        ptg_solver_cfg c;
        if (cfg) c = *cfg;
        else ptg_solver_cfg_default(&c);
        if ((warm_value == nullptr) != (warm_grad == nullptr))
            ptg::raise(PTG_ERR_CONFIG, "warm start needs both the value and the gradient");
        const size_t len = p.nn();
        ptg::DVec zd(p, len), vd, wg, zo(p, len), go(p, len);
        ptg::plan_upload_c128(p, z0, zd.p);
        if (v) {
            vd.alloc(p, len);
            ptg::plan_upload_c128(p, v, vd.p);
        }
        if (warm_grad) {
            wg.alloc(p, len);
            ptg::plan_upload_c128(p, warm_grad, wg.p);
        }
        ptg::DObj obj;
        obj.plan = &p;
        obj.metric = metric;
        obj.v = v ? vd.p : nullptr;
        ptg::Counter ctr;
        std::vector<ptg_hist> h;
        CbScope cbs(p, cb, user);
        ptg::SolveOut o = tn ? ptg::d_truncated_newton(obj, zd.p, c, ctr, warm_value, wg.p, zo.p, go.p, &h)
                             : ptg::d_lbfgs(obj, zd.p, c, ctr, warm_value, wg.p, zo.p, go.p, &h);
        if (z_out) ptg::plan_download_c128(p, zo.p, z_out);
        if (grad_out) ptg::plan_download_c128(p, go.p, grad_out);
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        fill_report(rep, ctr, o.value, o.reason, copy_hist(h, hist, hist_cap));
    });
}
}  // namespace

int ptg_lbfgs_ex(ptg_plan* plan, int metric, const double* v, const double* z0, const double* warm_value,
                 const double* warm_grad, const ptg_solver_cfg* cfg, double* z_out, double* grad_out,
                 ptg_report* rep, ptg_hist* hist, int hist_cap, ptg_iter_cb cb, void* user) {
    return solve_ex(false, plan, metric, v, z0, warm_value, warm_grad, cfg, z_out, grad_out, rep, hist, hist_cap, cb,
                    user);
}

int ptg_truncated_newton_ex(ptg_plan* plan, int metric, const double* v, const double* z0,
                            const double* warm_value, const double* warm_grad, const ptg_solver_cfg* cfg,
                            double* z_out, double* grad_out, ptg_report* rep, ptg_hist* hist, int hist_cap,
                            ptg_iter_cb cb, void* user) {
    return solve_ex(true, plan, metric, v, z0, warm_value, warm_grad, cfg, z_out, grad_out, rep, hist, hist_cap, cb,
                    user);
}

int ptg_fft2(const double* in, int n, int inverse, double* out) {
    return guard([&] {
        if (!in || !out) ptg::raise(PTG_ERR_CONFIG, "fft2: null pointer");
        int dev = 0;
        PTG_CUDA(cudaGetDevice(&dev));
        ptg::check_device_public(dev);
        if (n < 1) ptg::raise(PTG_ERR_GEOMETRY, "fft2: grid side must be a positive power of two, got " + std::to_string(n));
        const size_t bytes = (size_t)n * n * 16;
        ptg::DevMem a, b;
        a.alloc(bytes);
        b.alloc(bytes);
        PTG_CUDA(cudaMemcpy(a.p, in, bytes, cudaMemcpyHostToDevice));
        ptg::dev_fft2(a.p, n, inverse != 0, b.p, nullptr);
        PTG_CUDA(cudaMemcpy(out, b.p, bytes, cudaMemcpyDeviceToHost));
    });
}

int ptg_comm_unique_id(unsigned char id[128]) {
    return guard([&] {
        if (!id) ptg::raise(PTG_ERR_CONFIG, "null id buffer");
        ptg::comm_unique_id(id);
    });
}

int ptg_comm_init(const unsigned char id[128], int world, int rank, int device, ptg_comm** out) {
    return guard([&] {
        if (!id || !out) ptg::raise(PTG_ERR_CONFIG, "null argument");
        auto c = std::make_unique<ptg_comm>();
        c->c = ptg::comm_init(id, world, rank, device);
        *out = c.release();
    });
}

int ptg_comm_destroy(ptg_comm* comm) {
    return guard([&] {
        if (!comm) return;
        ptg::comm_destroy(comm->c);
        delete comm;
    });
}

int ptg_shard_layout(int n, int w, int N, const int32_t* positions, int world, int rank, int layout, int out[6]) {
    return guard([&] {
        if (!out || (N > 0 && !positions)) ptg::raise(PTG_ERR_CONFIG, "null argument");
        ptg::shard_layout(n, w, N, positions, world, rank, layout, out);
    });
}

int ptg_plan_create_sharded(const ptg_plan_desc* desc, int world, int rank, int layout, ptg_plan** out) {
    return guard([&] {
        if (!desc || !out) ptg::raise(PTG_ERR_CONFIG, "null argument");
        auto h = std::make_unique<ptg_plan>();
        h->p = ptg::plan_create_sharded(*desc, world, rank, layout);
        *out = h.release();
    });
}

int ptg_plan_bind_comm(ptg_plan* plan, ptg_comm* comm) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        if (!comm || !comm->c) ptg::raise(PTG_ERR_CONFIG, "null communicator");
        if (p.shard.layout == PTG_SHARD_NONE) ptg::raise(PTG_ERR_CONFIG, "plan is not sharded (ptg_plan_create_sharded)");
        if (ptg::comm_world(comm->c) != p.shard.world || ptg::comm_rank(comm->c) != p.shard.rank)
            ptg::raise(PTG_ERR_CONFIG, "communicator rank / world size do not match the plan's shard");
        p.comm = comm->c;
    });
}

int ptg_band_sync_halo(ptg_plan* plan, void* z_dev) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        if (!z_dev) ptg::raise(PTG_ERR_CONFIG, "null iterate");
        ptg::comm_sync_halo(p, z_dev);
    });
}

int ptg_metrics_device(int precision, const void* z, const void* z_true, int n, unsigned mask,
                       ptg_metrics* out, void* stream) {
    return guard([&] {
        if (!out || !z || !z_true) ptg::raise(PTG_ERR_CONFIG, "ptg_metrics_device: null pointer");
        ptg::dev_metrics(precision, z, z_true, n, mask, out, static_cast<cudaStream_t>(stream));
    });
}

int ptg_metrics_host(const double* z, const double* z_true, int n, unsigned mask, ptg_metrics* out) {
    return guard([&] {
        if (!out || !z || !z_true) ptg::raise(PTG_ERR_CONFIG, "ptg_metrics_host: null pointer");
        if (n < 1) ptg::raise(PTG_ERR_DOMAIN, "metric: empty fields");
        const size_t bytes = (size_t)n * n * 16;
        void* d = nullptr;
        PTG_CUDA(cudaMalloc(&d, 2 * bytes));
        struct F { void* p; ~F() { cudaFree(p); } } f{d};
        PTG_CUDA(cudaMemcpy(d, z, bytes, cudaMemcpyHostToDevice));
        PTG_CUDA(cudaMemcpy(static_cast<char*>(d) + bytes, z_true, bytes, cudaMemcpyHostToDevice));
        ptg::dev_metrics(PTG_C128, d, static_cast<char*>(d) + bytes, n, mask, out, nullptr);
    });
}

int ptg_canonical_phase(const double* z, int n, double* out) {
    return guard([&] {
        if (!out || !z) ptg::raise(PTG_ERR_CONFIG, "ptg_canonical_phase: null pointer");
        if (n < 1) ptg::raise(PTG_ERR_DOMAIN, "metric: empty fields");
        const size_t len = (size_t)n * n;
        void* d = nullptr;
        PTG_CUDA(cudaMalloc(&d, len * 16 + len * 8));
        struct F { void* p; ~F() { cudaFree(p); } } f{d};
        PTG_CUDA(cudaMemcpy(d, z, len * 16, cudaMemcpyHostToDevice));
        double* ph = reinterpret_cast<double*>(static_cast<char*>(d) + len * 16);
        ptg::dev_canonical_phase(PTG_C128, d, n, ph, nullptr);
        PTG_CUDA(cudaMemcpy(out, ph, len * 8, cudaMemcpyDeviceToHost));
    });
}

int ptg_truncated_newton(ptg_plan* plan, int metric, const double* v, const double* z0,
                         const ptg_solver_cfg* cfg, double* z_out, double* grad_out, ptg_report* rep,
                         ptg_hist* hist, int hist_cap) {
    return guard([&] {
        ptg::Plan& p = P(plan);
        ptg_solver_cfg c;
        if (cfg) c = *cfg;
        else ptg_solver_cfg_default(&c);
        const size_t len = p.nn();
        ptg::DVec zd(p, len), vd, zo(p, len), go(p, len);
        ptg::plan_upload_c128(p, z0, zd.p);
        if (v) {
            vd.alloc(p, len);
            ptg::plan_upload_c128(p, v, vd.p);
        }
        ptg::DObj obj;
        obj.plan = &p;
        obj.metric = metric;
        obj.v = v ? vd.p : nullptr;
        ptg::Counter ctr;
        std::vector<ptg_hist> h;
        ptg::SolveOut o = ptg::d_truncated_newton(obj, zd.p, c, ctr, nullptr, nullptr, zo.p, go.p, &h);
        if (z_out) ptg::plan_download_c128(p, zo.p, z_out);
        if (grad_out) ptg::plan_download_c128(p, go.p, grad_out);
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        fill_report(rep, ctr, o.value, o.reason, copy_hist(h, hist, hist_cap));
    });
}

int ptg_hier_create(ptg_plan* fine, int metric, int depth, const ptg_mg_cfg* opt, ptg_hier** out) {
    return guard([&] {
        ptg::Plan& p = P(fine);
        ptg_mg_cfg o;
        if (opt) o = *opt;
        else ptg_mg_cfg_default(&o);
        auto h = new ptg_hier;
        try {
            h->h = ptg::hier_build(p, metric, depth, o);
        } catch (...) {
            delete h;
            throw;
        }
        h->fine = fine;
        *out = h;
    });
}

int ptg_hier_destroy(ptg_hier* h) {
    return guard([&] {
        if (!h) return;
        for (auto& v : h->views) v.p.release();   // non-owning
        delete h;
    });
}

int ptg_hier_level(ptg_hier* h, int level, ptg_plan** plan_out) {
    return guard([&] {
        if (!h || level < 0 || level >= h->h->depth()) ptg::raise(PTG_ERR_CONFIG, "bad hierarchy level");
        if (level == 0) {
            *plan_out = h->fine;
            return;
        }
        if (h->views.empty()) {
            h->views.resize(h->h->depth());
        }
        ptg_plan& v = h->views[level];
        if (!v.p) v.p.reset(h->h->levels[level]);
        *plan_out = &v;
    });
}


int ptg_mgopt_driver(ptg_hier* hh, const double* z0, const ptg_driver_cfg* cfg, double* z_out,
                     ptg_report* rep, ptg_hist* hist, int hist_cap) {
    return guard([&] {
        if (!hh) ptg::raise(PTG_ERR_CONFIG, "null hierarchy");
        ptg::Hier& h = *hh->h;
        ptg::Plan& p = P(hh->fine);
        sync_streams(h);
        ptg_driver_cfg c;
        if (cfg) c = *cfg;
        else ptg_driver_cfg_default(&c);
        const size_t len = p.nn();
        ptg::DVec zd(p, len), zo(p, len);
        ptg::plan_upload_c128(p, z0, zd.p);
        ptg::Counter ctr;
        std::vector<ptg_hist> hv;
        ptg::SolveOut o = ptg::d_mgopt_driver(h, zd.p, c, ctr, zo.p, &hv);
        if (z_out) ptg::plan_download_c128(p, zo.p, z_out);
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        fill_report(rep, ctr, o.value, o.reason, copy_hist(hv, hist, hist_cap));
    });
}

int ptg_mgopt_cycle(ptg_hier* hh, int level, const double* z, const double* v, const double* warm_value,
                    const double* warm_grad, double* z_out, double* value_out, double* grad_out, ptg_report* rep) {
    return guard([&] {
        if (!hh) ptg::raise(PTG_ERR_CONFIG, "null hierarchy");
        ptg::Hier& h = *hh->h;
        if (level < 0 || level >= h.depth()) ptg::raise(PTG_ERR_CONFIG, "mgoptCycle: bad level");
        if ((warm_value == nullptr) != (warm_grad == nullptr))
            ptg::raise(PTG_ERR_CONFIG, "warm start needs both the value and the gradient");
        P(hh->fine);
        sync_streams(h);
        ptg::Plan& p = *h.levels[level];
        const size_t len = p.nn();
        ptg::DVec zd(p, len), vd, wg, zo(p, len), go(p, len);
        ptg::plan_upload_c128(p, z, zd.p);
        if (v) {
            vd.alloc(p, len);
            ptg::plan_upload_c128(p, v, vd.p);
        }
        if (warm_grad) {
            wg.alloc(p, len);
            ptg::plan_upload_c128(p, warm_grad, wg.p);
        }
        ptg::Counter ctr;
        const double val = ptg::d_mgopt_cycle(h, level, zd.p, v ? vd.p : nullptr, ctr, warm_value, wg.p, zo.p, go.p);
        if (z_out) ptg::plan_download_c128(p, zo.p, z_out);
        if (grad_out) ptg::plan_download_c128(p, go.p, grad_out);
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        if (value_out) *value_out = val;
        fill_report(rep, ctr, val, PTG_STOP_MAXITERS, 0);
    });
}

int ptg_mgopt_driver_ex(ptg_hier* hh, const double* z0, const ptg_driver_cfg* cfg, double* z_out, double* grad_out,
                        ptg_report* rep, ptg_hist* hist, int hist_cap, ptg_iter_cb cb, void* user) {
    return guard([&] {
        if (!hh) ptg::raise(PTG_ERR_CONFIG, "null hierarchy");
        ptg::Hier& h = *hh->h;
        ptg::Plan& p = P(hh->fine);
        sync_streams(h);
        ptg_driver_cfg c;
        if (cfg) c = *cfg;
        else ptg_driver_cfg_default(&c);
        const size_t len = p.nn();
        ptg::DVec zd(p, len), zo(p, len);
        ptg::plan_upload_c128(p, z0, zd.p);
        ptg::Counter ctr;
        std::vector<ptg_hist> hv;
        CbScope cbs(p, cb, user);
        ptg::SolveOut o = ptg::d_mgopt_driver(h, zd.p, c, ctr, zo.p, &hv);
        if (z_out) ptg::plan_download_c128(p, zo.p, z_out);
        if (grad_out) {   // finalEval's gradient: one uncounted evaluation at the final iterate
            ptg::DVec go(p, len);
            ptg::plan_eval(p, h.metric, zo.p, nullptr, go.p, p.value.as<double>());
            ptg::plan_download_c128(p, go.p, grad_out);
        }
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        fill_report(rep, ctr, o.value, o.reason, copy_hist(hv, hist, hist_cap));
    });
}

int ptg_mgopt_cycle_device(ptg_hier* hh, void* z, double* value, void* grad, ptg_report* rep) {
    return guard([&] {
        if (!hh) ptg::raise(PTG_ERR_CONFIG, "null hierarchy");
        ptg::Hier& h = *hh->h;
        ptg::Plan& p = P(hh->fine);
        sync_streams(h);
        const size_t len = p.nn();
        ptg::DVec zo(p, len), go(p, len);
        ptg::Counter ctr;
        const double v = ptg::d_mgopt_cycle(h, 0, z, nullptr, ctr, value, grad, zo.p, go.p);
        ptg::dev_copy(p.prec, z, zo.p, len, p.stream);
        ptg::dev_copy(p.prec, grad, go.p, len, p.stream);
        PTG_CUDA(cudaStreamSynchronize(p.stream));
        *value = v;
        fill_report(rep, ctr, v, PTG_STOP_MAXITERS, 0);
    });
}

}  // extern "C"
