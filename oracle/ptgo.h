/*
 * ptgo.h — CPU ORACLE for the ptychographic objective/gradient hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a plain-C restatement of the reference
 * algorithm (/root/reference/proj/src/{kernels,field,objectives,solvers,
 * multigrid}.cpp) generalised to the patch model (complex probe P of size
 * M x M, window w <= M, free integer scan positions).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it, and only as the checker or the timed CPU baseline.  The
 * product path (paper_1810_05628_b200/, libptg.so) never links or calls it.
 *
 * Parity pinning:
 *   - ref mode (probe == NULL, M == n): bitwise against the compiled reference
 *     library oracle/_ref/libptycho_ref.so (tests/test_oracle_vs_reference.py)
 *     and against golden vectors generated from it (tests/golden/).
 *   - patch mode (complex probe, M == w): finite differences, additivity,
 *     fixed point at truth, reduction to ref mode when P == 1 and M == n.
 *
 * Conventions (all arrays row-major; complex = interleaved (re, im) doubles,
 * layout-compatible with std::complex<double>):
 *   object z         n x n complex
 *   probe P          M x M complex, or NULL for the reference's binary window
 *   positions        N x 2 int32 (row0, col0) of the window's top-left pixel
 *   data d           N x M x M intensities (>= 0)
 * Status codes follow the C-ABI (include/ptg.h): 0 ok, 10 ConfigError,
 * 11 GeometryError, 12 DomainError, 13 MetricError, 3 NumericError.
 */
#ifndef PTGO_H
#define PTGO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PTGO_OK = 0, PTGO_CONFIG = 10, PTGO_GEOMETRY = 11, PTGO_DOMAIN = 12,
       PTGO_METRIC = 13, PTGO_NUMERIC = 3, PTGO_NOMEM = 4 };
enum { PTGO_DISTANCE = 0, PTGO_INTENSITY = 1 };
enum { PTGO_STOP_TOLERANCE = 0, PTGO_STOP_BUDGET = 1, PTGO_STOP_MAXITERS = 2,
       PTGO_STOP_STALL = 3 };

const char *ptgo_last_error(void);

typedef struct {
    int n;                 /* object side */
    int M;                 /* FFT frame side (power of two) */
    int w;                 /* window side, 1 <= w <= M, w <= n */
    int N;                 /* scan positions */
    const int32_t *pos;    /* N x 2 (row0, col0) */
    const double *probe;   /* M x M complex or NULL (binary window) */
    const double *data;    /* N x M x M */
    int metric;            /* PTGO_DISTANCE / PTGO_INTENSITY */
} ptgo_problem;

/* L0 kernels (kernels.cpp:34-120) */
int ptgo_fft2(double *a, int n, int inverse);
double ptgo_norm2sq(const double *a, size_t len);
double ptgo_dot_real(const double *a, const double *b, size_t len);

/* L3 objectives (objectives.cpp:12-118) */
int ptgo_validate(const ptgo_problem *p);
int ptgo_project_modulus(const ptgo_problem *p, const double *z, int k, double *frame);
int ptgo_evaluate(const ptgo_problem *p, const double *z, const double *v,
                  double *value, double *grad);
/* forward.cpp:40-54: d_k = |fft2(P o S_k z)|^2 */
int ptgo_simulate(const ptgo_problem *p, const double *z, double *data_out);

/* L5 transfers (multigrid.cpp:34-77) */
int ptgo_restrict_field(const double *fine, int n, double *coarse);
int ptgo_prolong_field(const double *coarse, int nH, double *fine);
int ptgo_restrict_data(const double *fine, int N, int M, double *coarse);

/* accounting + reports (solvers.hpp:16-54) */
#define PTGO_MAX_LEVELS 16
typedef struct {
    double weighted;
    long per_level[PTGO_MAX_LEVELS];
} ptgo_counter;

typedef struct { double weighted, value, gnorm; } ptgo_hist;

typedef struct {
    ptgo_hist *hist;
    int len, cap;
    int reason;
} ptgo_report;

void ptgo_report_free(ptgo_report *r);

/* a counted objective over vectors of `len` complex entries */
typedef int (*ptgo_fn)(void *user, const double *z, double *value, double *grad);
typedef struct {
    ptgo_fn fn;
    void *user;
    size_t len;
    int level;
    double weight;
} ptgo_counted;

typedef struct {
    int max_iters;
    double grad_tol_rel, grad_tol_abs;
    int lbfgs_memory, linesearch_max;
    double max_weighted;   /* +inf for no budget */
    int cg_max_iters;      /* truncatedNewton inner CG */
    double cg_rel_tol;
} ptgo_solver_cfg;

void ptgo_solver_cfg_default(ptgo_solver_cfg *c);   /* solvers.hpp:56-66 */

/* solvers.cpp:61-85; z_out/value_out/grad_out receive the accepted point
 * (z_out = z when stalled; value/grad untouched then). */
int ptgo_linesearch(const ptgo_counted *obj, const double *z, const double *dir,
                    ptgo_counter *ctr, int max_trials, const double *phi0,
                    double *alpha, int *stalled, int *trials,
                    double *z_out, double *value_out, double *grad_out);

/* solvers.cpp:87-141; warm (value, grad) optional (pass NULL) */
int ptgo_lbfgs(const ptgo_counted *obj, const double *z0, const ptgo_solver_cfg *cfg,
               ptgo_counter *ctr, const double *warm_value, const double *warm_grad,
               double *z_out, double *value_out, double *grad_out, ptgo_report *rep);

/* solvers.cpp:143-227 (Newton-CG with finite-difference Hessian-vector
 * products, one counted evaluation each); warm (value, grad) optional */
int ptgo_truncated_newton(const ptgo_counted *obj, const double *z0, const ptgo_solver_cfg *cfg,
                          ptgo_counter *ctr, const double *warm_value, const double *warm_grad,
                          double *z_out, double *value_out, double *grad_out, ptgo_report *rep);

/* solvers.cpp:229-265 with Alg. 1's complex-probe weight */
int ptgo_pie(const ptgo_problem *p, const double *z0, double gamma, int sweeps,
             double max_weighted, ptgo_counter *ctr, double *z_out,
             double *final_value, ptgo_report *rep);

/* multigrid.hpp:39-49 / 82-87 */
typedef struct {
    int k1, k2, coarsest_max_iters;
    double coarsest_grad_tol_rel, intermediate_grad_tol_rel;
    int lbfgs_memory, linesearch_max;
    double grad_tol_abs;
} ptgo_mg_cfg;
typedef struct {
    double budget, grad_tol_rel, grad_tol_abs;
    int max_cycles;
} ptgo_driver_cfg;
void ptgo_mg_cfg_default(ptgo_mg_cfg *c);
void ptgo_driver_cfg_default(ptgo_driver_cfg *c);

/* hierarchy (multigrid.cpp:79-115), patch-model coarsening: n/2, M/2, w/2,
 * pos/2 (floor), probe -> restrictField(probe), data -> restrictData. */
typedef struct ptgo_hierarchy ptgo_hierarchy;
int ptgo_hierarchy_build(const ptgo_problem *fine, int depth, const ptgo_mg_cfg *opt,
                         ptgo_hierarchy **out);
void ptgo_hierarchy_free(ptgo_hierarchy *h);
const ptgo_problem *ptgo_hierarchy_level(const ptgo_hierarchy *h, int level);
int ptgo_hierarchy_depth(const ptgo_hierarchy *h);
int ptgo_hierarchy_coarsest_iters(const ptgo_hierarchy *h);

/* multigrid.cpp:117-169: one V-cycle at `level` with shift v (n_l^2 complex);
 * warm (value, grad) optional. */
int ptgo_mgopt_cycle(const ptgo_hierarchy *h, int level, const double *z,
                     const double *v, ptgo_counter *ctr, const double *warm_value,
                     const double *warm_grad, double *z_out, double *value_out,
                     double *grad_out);
/* multigrid.cpp:171-227 */
int ptgo_mgopt_driver(const ptgo_hierarchy *h, const double *z0,
                      const ptgo_driver_cfg *cfg, ptgo_counter *ctr, double *z_out,
                      double *value_out, double *grad_out, ptgo_report *rep);

/* noise (forward.cpp:56-86) and the GPU's counter-based generator / Poisson sampler */
void ptgo_philox4x64(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]);
int ptgo_add_noise(int N, size_t mm, const double *d, double level, uint64_t seed, const double *uni,
                   double *out);
int ptgo_add_poisson(int N, size_t mm, const double *d, double photons, uint64_t seed, double *out);

#ifdef __cplusplus
}
#endif
#endif
