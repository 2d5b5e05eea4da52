/*
 * ptg.h — C-ABI of libptg, the B200-native (sm_100a) ptychographic
 * objective/gradient library.  This is the drop-in boundary for the hot path
 * named in BASELINE.json (north_star): every entry point replaces one public
 * function of the reference's C++ API under /root/reference/proj/include/
 * ptycho/ (cited per function below).  Plain pointers and sizes only — no
 * torch or CUDA-runtime types appear in the signatures (streams are passed as
 * opaque void* cudaStream_t handles).
 *
 * Data model (patch generalisation of the reference):
 *   object z       n x n complex, row-major.  Host buffers are always
 *                  complex128 (interleaved doubles, layout-compatible with
 *                  std::complex<double> / ptycho::ComplexField::data()).
 *                  Device buffers (the *_device calls) are in the plan's
 *                  precision: complex64 (float2) or complex128 (double2).
 *   probe P        M x M complex, or NULL = the reference's binary window
 *                  (ProbeWindow, field.hpp:63-73).
 *   positions      N x 2 int32 (row0, col0): window top-left in the object.
 *   data d         N x M x M non-negative intensities, one pattern per position
 *                  (DiffractionStack, forward.hpp:22-27), in scan order.
 *   frame          psi_j = P o S_j x zero-padded at the origin of an M x M
 *                  frame (w <= M).  With P = NULL and M = n this is exactly
 *                  the reference's full-field model (|fft| is shift invariant).
 *
 * Status codes (every call returns one; message via ptg_last_error()):
 *   0 OK; 10 ConfigError, 11 GeometryError, 12 DomainError, 13 MetricError
 *   (errors.hpp:16-33); 2 IoError; 3 NumericError (errors.hpp:36-42);
 *   4 CUDA/NCCL failure; 5 internal.  A C++ shim re-throws the matching
 *   ptycho:: exception type.
 *
 * Threading: one plan per host thread at a time; host-pointer calls are
 * synchronous with respect to their host outputs; *_device calls are
 * asynchronous on the plan's stream unless they return a host scalar.
 * There is no CPU fallback: without a usable sm_100 device every call that
 * needs one fails with status 4.
 */
#ifndef PTG_H
#define PTG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PTG_OK 0
#define PTG_ERR_IO 2
#define PTG_ERR_NUMERIC 3
#define PTG_ERR_CUDA 4
#define PTG_ERR_INTERNAL 5
#define PTG_ERR_CONFIG 10
#define PTG_ERR_GEOMETRY 11
#define PTG_ERR_DOMAIN 12
#define PTG_ERR_METRIC 13

enum ptg_precision { PTG_C64 = 0, PTG_C128 = 1 };
enum ptg_dtype { PTG_F32 = 0, PTG_F64 = 1 };
/* objectives.hpp:8-11 MetricKind */
enum ptg_metric { PTG_DISTANCE = 0, PTG_INTENSITY = 1 };
/* solvers.hpp:41 StopReason */
enum ptg_stop { PTG_STOP_TOLERANCE = 0, PTG_STOP_BUDGET = 1, PTG_STOP_MAXITERS = 2, PTG_STOP_STALL = 3 };

const char *ptg_last_error(void);
/* library/ABI version and the device it would run on (-1 if none) */
int ptg_version(void);
int ptg_device_count(int *count);

/* ------------------------------------------------------------------ plans */
typedef struct ptg_plan ptg_plan;

typedef struct {
    int n;                    /* object side */
    int M;                    /* FFT frame side, power of two, w <= M */
    int w;                    /* window side */
    int N;                    /* scan positions */
    const int32_t *positions; /* host N x 2 (row0, col0) */
    const double *probe;      /* host M x M complex128, or NULL (binary window) */
    const void *data;         /* host N x M x M intensities, or NULL (set later) */
    int data_dtype;           /* PTG_F32 / PTG_F64 */
    int precision;            /* PTG_C64 / PTG_C128 */
    int device;               /* CUDA device ordinal */
} ptg_plan_desc;

/* Binds geometry + probe + data to one device (ScanGeometry / DiffractionStack
 * / Objective, field.hpp:75-85, forward.hpp:22-27, objectives.hpp:18-26).
 * Validates like checkStack/checkPattern/checkWindow (objectives.cpp:12-26,
 * field.cpp:45-51): GeometryError for bad windows or a non-power-of-two M,
 * DomainError for negative intensities. */
int ptg_plan_create(const ptg_plan_desc *desc, ptg_plan **out);
int ptg_plan_destroy(ptg_plan *plan);
/* run subsequent device work on this cudaStream_t (NULL = the plan's own) */
int ptg_plan_set_stream(ptg_plan *plan, void *stream);
/* re-upload / replace the diffraction data (host or device pointer) */
int ptg_plan_set_data(ptg_plan *plan, const void *host_data, int dtype);
int ptg_plan_set_data_device(ptg_plan *plan, const void *dev_data, int dtype);
/* loadRawStack (image_io.hpp:36, format :10-20) straight into the plan: the
 * PTYF float64 stack is streamed through pinned double buffers (file read
 * overlapping H2D copy + on-device conversion).  Errors: 2 (Io) for
 * open/magic/truncation, 11 (Geometry) if the stack is not N patterns of side M. */
int ptg_plan_load_ptyf(ptg_plan *plan, const char *path);
/* the resident data back to the host as N*M*M float64: the intensities d
 * (metric PTG_INTENSITY) or the amplitudes sqrt(d) (PTG_DISTANCE) */
int ptg_plan_get_data(ptg_plan *plan, int metric, double *out);
/* bytes of HBM the plan holds, and its dims (any pointer may be NULL) */
int ptg_plan_info(const ptg_plan *plan, int *n, int *M, int *w, int *N, int *precision,
                  size_t *device_bytes);
/* number of kernel launches issued by the plan since creation (for bench) */
int ptg_plan_launch_count(const ptg_plan *plan, int64_t *count);
/* Opt-in CUDA-event timing, on the stream they are launched on, of the
 * per-position frame kernel (the dominant kernel) and of the overlap-add
 * gather.  get_timing synchronises, returns totals since the last call
 * (milliseconds, launch counts) and resets them. */
int ptg_plan_set_timing(ptg_plan *plan, int enable);
int ptg_plan_get_timing(ptg_plan *plan, double *frame_ms, int64_t *frame_launches,
                        double *gather_ms, int64_t *gather_launches);

/* ------------------------------------------------------------- objectives */
/* evaluate (objectives.hpp:44, objectives.cpp:106-118) with phiDistance
 * (:38-39) or phiIntensityGaussian (:40-41): value + descent-convention
 * gradient, optional MG/OPT shift v (value -= <v,z>_R, grad -= v).
 * Host complex128 buffers; v and grad may be NULL. */
int ptg_eval(ptg_plan *plan, int metric, const double *z, const double *v, double *value,
             double *grad);
/* Device-resident variant: z, v (nullable), grad (nullable) are device buffers
 * of n*n elements in the plan precision.  *value_host (nullable) receives the
 * value (synchronises); value_dev (nullable) receives it on device. */
int ptg_eval_device(ptg_plan *plan, int metric, const void *z, const void *v, void *grad,
                    double *value_dev, double *value_host);
/* projectModulus (objectives.hpp:32-33): the M x M projected frame of
 * pattern k (host complex128 out, M*M elements). */
int ptg_project_modulus(ptg_plan *plan, const double *z, int k, double *frame);
/* simulate (forward.hpp:43): d_j = |fft2(P o S_j z)|^2 for all positions into
 * the plan's resident data (and optionally a host copy, N*M*M doubles). */
int ptg_simulate(ptg_plan *plan, const double *z, double *data_out);
int ptg_simulate_device(ptg_plan *plan, const void *z);

/* fft2 / ifft2 (field.hpp:91-93; kernels.cpp:34-85 convention: unnormalised
 * forward, inverse x 1/n^2) of a host complex128 n x n field on the current
 * device, with the objective kernels' own 2-D FFT (n a power of two <= 64) */
int ptg_fft2(const double *in, int n, int inverse, double *out);

/* ---------------------------------------------------------------- noise */
/* addNoise (forward.hpp:44-48, forward.cpp:56-86) in place on the plan's
 * resident intensities (the amplitudes are rebuilt): per pattern
 * eps = level ||d|| / ||g|| g with g_i = sqrt(-2 log(1-u1)) cos(2 pi u2)
 * (rng::gaussian, rng.hpp:18-24), d <- max(d + eps, 0).  uniforms = NULL
 * draws (u1, u2) of pixel i of pattern j from Philox4x64-10 with counter
 * (i, j, 1, 0) and key (seed, 0); otherwise `uniforms` is a host array of
 * 2 N M^2 doubles in the reference's draw order (pattern, pixel, u1/u2), so
 * the result follows the reference's std::mt19937_64 stream exactly.
 * DomainError for level < 0 (forward.cpp:57). */
int ptg_add_noise(ptg_plan *plan, double level, uint64_t seed, const double *uniforms);
/* Poisson photon noise at `photons` per pattern (BASELINE configs 4/5; no
 * reference counterpart): lambda = d photons / sum(d), d <- k / scale with
 * k ~ Poisson(lambda) (inversion below 10, PTRS transformed rejection above),
 * uniforms from Philox4x64-10 with counter (pixel, pattern, 2, block). */
int ptg_add_poisson(ptg_plan *plan, double photons, uint64_t seed);
/* the first `count` rng::uniform01 draws (rng.hpp:14-16: top 53 bits of a
 * std::mt19937_64 draw x 2^-53) of an engine seeded with `seed`, on the host
 * (no device needed): the seeded synthetic inputs of SURVEY 8(d) */
int ptg_uniform01_stream(uint64_t seed, size_t count, double *out);
/* raw Philox4x64-10 output on `device`: out[4 b + k] = word k of
 * philox(counter (ctr[0] + b, ctr[1], ctr[2], ctr[3]), key), b < nblocks
 * (host out; for pinning the generator against numpy.random.Philox) */
int ptg_philox4x64(int device, const uint64_t ctr[4], const uint64_t key[2], size_t nblocks, uint64_t *out);

/* IterationCallback (solvers.hpp:70-71): (user, iteration index, host
 * complex128 iterate n*n, objective value, weighted evaluations so far); fired
 * for the initial point (index 0) and after every iteration / sweep / cycle. */
typedef void (*ptg_iter_cb)(void *user, int iter, const double *z, double value, double weighted);

/* ----------------------------------------------------------------- PIE */
typedef struct { double weighted, value, gnorm; } ptg_hist;

/* pie (solvers.hpp:111-114, solvers.cpp:229-265) with Alg. 1's complex-probe
 * weight (|P|/max|P|) conj(P)/(|P|^2+gamma).  z is host complex128 in/out.
 * hist (cap entries) receives the initial point + one row per sweep. */
int ptg_pie(ptg_plan *plan, double *z, double gamma, int sweeps, double max_weighted,
            double *final_value, ptg_hist *hist, int hist_cap, int *hist_len,
            double *weighted, int *reason);
/* the same with an IterationCallback (cb may be NULL) */
int ptg_pie_cb(ptg_plan *plan, double *z, double gamma, int sweeps, double max_weighted,
               double *final_value, ptg_hist *hist, int hist_cap, int *hist_len, double *weighted,
               int *reason, ptg_iter_cb cb, void *user);
/* one raw sweep on a device object (no diagnostics, no accounting) */
int ptg_pie_sweep_device(ptg_plan *plan, void *z, double gamma);

/* -------------------------------------------------------------- transfers */
/* restrictField / prolongField (multigrid.hpp:15-16, multigrid.cpp:34-53) and
 * restrictData (multigrid.hpp:23, multigrid.cpp:55-77).  Host versions take
 * complex128 / float64; device versions the given precision/dtype. */
int ptg_restrict_field(const double *fine, int n, double *coarse);
int ptg_prolong_field(const double *coarse, int nH, double *fine);
int ptg_restrict_data(const double *fine, int N, int M, double *coarse);
int ptg_restrict_field_device(int precision, const void *fine, int n, void *coarse, void *stream);
int ptg_prolong_field_device(int precision, const void *coarse, int nH, void *fine, void *stream);
int ptg_restrict_data_device(int dtype, const void *fine, int N, int M, void *coarse, void *stream);

/* ------------------------------------------------------------ multi-GPU */
/* SURVEY 8(e) / north_star: one process per GPU, scan positions sharded,
 * NCCL inside libptg (bound at run time: libnccl.so.2).  No reference
 * counterpart (the reference is single-process).
 *
 * Partition (ptg_shard_layout, host-only): the global scan (positions in scan
 * order, window rows non-decreasing between rows of the scan) is cut at
 * scan-row boundaries into `world` contiguous blocks of about N / world
 * positions; rank r evaluates block r.
 *   PTG_SHARD_REPLICATED  every rank holds the whole n x n object; after its
 *                         frames one NCCL allreduce of [gradient | value] --
 *                         north_star's layout.  The solvers run replicated on
 *                         the allreduced values (identical on every rank).
 *   PTG_SHARD_BANDS       rank r holds object rows [row0, row0 + rows): its
 *                         own rows (up to the next rank's first window row)
 *                         plus the halo its windows reach below them; halo
 *                         gradient rows go to rank r + 1 (NCCL send/recv),
 *                         the value is one scalar allreduce.  Device buffers
 *                         (z, v, grad) are rows x n.  Needs own rows >= the
 *                         halo on every rank.  complex64, M = 128 / 256, w = M
 *                         (the persistent RMW path); evaluation only. */
enum ptg_shard { PTG_SHARD_NONE = 0, PTG_SHARD_REPLICATED = 1, PTG_SHARD_BANDS = 2 };
typedef struct ptg_comm ptg_comm;
/* ncclGetUniqueId on one rank; distribute the 128 bytes, then ptg_comm_init everywhere */
int ptg_comm_unique_id(unsigned char id[128]);
int ptg_comm_init(const unsigned char id[128], int world, int rank, int device, ptg_comm **out);
int ptg_comm_destroy(ptg_comm *comm);
/* out[6] = {pos_begin, pos_end, row0, rows, own_rows, halo_prev} of `rank` */
int ptg_shard_layout(int n, int w, int N, const int32_t *positions, int world, int rank, int layout, int out[6]);
/* this rank's plan of the GLOBAL problem `desc` (all N positions; desc->data
 * NULL or the rank's own patterns [pos_begin, pos_end) in scan order) */
int ptg_plan_create_sharded(const ptg_plan_desc *desc, int world, int rank, int layout, ptg_plan **out);
/* bind the communicator: every later evaluation (ptg_eval / _device) of this
 * plan returns the GLOBAL value and this rank's gradient (REPLICATED: the
 * whole gradient; BANDS: its rows, own rows final) */
int ptg_plan_bind_comm(ptg_plan *plan, ptg_comm *comm);
/* BANDS: fill the iterate's halo rows [own_rows, rows) from rank + 1 (device z) */
int ptg_band_sync_halo(ptg_plan *plan, void *z_dev);

/* ----------------------------------------------- multi-GPU band exchange */
/* No reference counterpart (the reference is single-process): helpers of the
 * band decomposition of SURVEY 8(e) (paper_1810_05628_b200/sharding.py).  A
 * rank's n x n band shares `ov` gradient rows with each neighbour.  pack:
 * [top ov rows][bottom ov rows][*val_dev (f64)] into `buf` (ptg_halo_bytes
 * bytes); after an all-gather of every rank's buffer into `all` (world x
 * ptg_halo_bytes), unpack adds the neighbours' rows to the band's own
 * (own + received) and writes the rank-ordered sum of the misfits to *val_dev.
 * Device pointers, plan precision; enqueued on `stream`. */
size_t ptg_halo_bytes(int precision, int n, int ov);
int ptg_halo_pack(int precision, const void *grad, int n, int ov, const double *val_dev, void *buf,
                  void *stream);
int ptg_halo_unpack(int precision, void *grad, int n, int ov, const void *all, int rank, int world,
                    double *val_dev, void *stream);

/* ------------------------------------------------------------- diagnostics */
/* metrics.hpp:9-24 on the device: relativeError, magnitudeRelError and
 * phaseSSIM (11x11 Gaussian window, sigma 1.5, L = pi/2), fp64 arithmetic.
 * Errors: 12 (Domain) for empty fields / zero reference, 13 (Metric) for
 * phaseSSIM with n < 11. */
#define PTG_METRIC_RELATIVE_ERROR 1u
#define PTG_METRIC_MAGNITUDE_REL_ERROR 2u
#define PTG_METRIC_PHASE_SSIM 4u
#define PTG_METRIC_ALL 7u
typedef struct {
    double relative_error, magnitude_rel_error, phase_ssim;
} ptg_metrics;
/* device fields in `precision` (n x n complex), stream may be NULL */
int ptg_metrics_device(int precision, const void *z, const void *z_true, int n, unsigned mask,
                       ptg_metrics *out, void *stream);
/* host complex128 fields */
int ptg_metrics_host(const double *z, const double *z_true, int n, unsigned mask, ptg_metrics *out);
/* canonicalPhase (metrics.hpp:15-18): host complex128 in, host fp64 n x n out */
int ptg_canonical_phase(const double *z, int n, double *out);

/* -------------------------------------------------------- solvers, MG/OPT */
/* SolverConfig (solvers.hpp:56-66) */
typedef struct {
    int max_iters;
    double grad_tol_rel, grad_tol_abs;
    int lbfgs_memory, linesearch_max;
    double max_weighted;
    int cg_max_iters;      /* truncatedNewton inner CG (cgMaxIters) */
    double cg_rel_tol;     /* cgRelTol */
} ptg_solver_cfg;
/* MgoptConfig (multigrid.hpp:39-49) */
typedef struct {
    int k1, k2, coarsest_max_iters;
    double coarsest_grad_tol_rel, intermediate_grad_tol_rel;
    int lbfgs_memory, linesearch_max;
    double grad_tol_abs;
} ptg_mg_cfg;
/* MgoptDriverConfig (multigrid.hpp:82-87) */
typedef struct {
    double budget, grad_tol_rel, grad_tol_abs;
    int max_cycles;
} ptg_driver_cfg;
/* SolverReport + EvalCounter (solvers.hpp:16-54) */
typedef struct {
    double final_value;
    double weighted;          /* EvalCounter::weightedEvals */
    long per_level[16];       /* EvalCounter::perLevelEvals */
    int reason;               /* ptg_stop */
    int hist_len;             /* entries written to the caller's hist array */
} ptg_report;

void ptg_solver_cfg_default(ptg_solver_cfg *c);
void ptg_mg_cfg_default(ptg_mg_cfg *c);
void ptg_driver_cfg_default(ptg_driver_cfg *c);

/* lbfgs (solvers.hpp:92-95) on the plan's (optionally v-shifted) objective,
 * GPU-resident: vectors never leave the device, only scalars cross PCIe. */
int ptg_lbfgs(ptg_plan *plan, int metric, const double *v, const double *z0,
              const ptg_solver_cfg *cfg, double *z_out, double *grad_out, ptg_report *rep,
              ptg_hist *hist, int hist_cap);

/* lbfgs with the reference's full signature (solvers.hpp:92-95): warmStart
 * (warm_value + host complex128 warm_grad, both or neither: the evaluation at
 * z0, not charged again) and an IterationCallback (cb may be NULL).
 * grad_out receives finalEval.gradient. */
int ptg_lbfgs_ex(ptg_plan *plan, int metric, const double *v, const double *z0, const double *warm_value,
                 const double *warm_grad, const ptg_solver_cfg *cfg, double *z_out, double *grad_out,
                 ptg_report *rep, ptg_hist *hist, int hist_cap, ptg_iter_cb cb, void *user);
/* truncatedNewton (solvers.hpp:101-104): Newton-CG with finite-difference
 * Hessian-vector products (one counted gradient evaluation each), GPU-resident. */
int ptg_truncated_newton(ptg_plan *plan, int metric, const double *v, const double *z0,
                         const ptg_solver_cfg *cfg, double *z_out, double *grad_out, ptg_report *rep,
                         ptg_hist *hist, int hist_cap);

/* truncatedNewton with warmStart and IterationCallback (solvers.hpp:101-104) */
int ptg_truncated_newton_ex(ptg_plan *plan, int metric, const double *v, const double *z0,
                            const double *warm_value, const double *warm_grad, const ptg_solver_cfg *cfg,
                            double *z_out, double *grad_out, ptg_report *rep, ptg_hist *hist, int hist_cap,
                            ptg_iter_cb cb, void *user);

typedef struct ptg_hier ptg_hier;
/* buildHierarchy (multigrid.hpp:61-62): coarse levels built ON DEVICE by
 * restrictData / restrictField(probe) / pos/2 (patch-model coarsening). */
int ptg_hier_create(ptg_plan *fine, int metric, int depth, const ptg_mg_cfg *opt,
                    ptg_hier **out);
int ptg_hier_destroy(ptg_hier *h);
int ptg_hier_level(ptg_hier *h, int level, ptg_plan **plan_out);
/* mgoptDriver (multigrid.hpp:93-95), GPU-resident */
int ptg_mgopt_driver(ptg_hier *h, const double *z0, const ptg_driver_cfg *cfg, double *z_out,
                     ptg_report *rep, ptg_hist *hist, int hist_cap);
/* mgoptDriver with an IterationCallback (one call per completed cycle) and
 * finalEval.gradient (grad_out, one uncounted evaluation; may be NULL) */
int ptg_mgopt_driver_ex(ptg_hier *h, const double *z0, const ptg_driver_cfg *cfg, double *z_out,
                        double *grad_out, ptg_report *rep, ptg_hist *hist, int hist_cap, ptg_iter_cb cb,
                        void *user);
/* mgoptCycle (multigrid.hpp:78-80) at any level with shift v (NULL = zero):
 * host complex128 buffers of that level's side; warmStart optional (both the
 * value and the gradient, or neither).  Returns the cycle's final iterate,
 * shifted value and gradient (CycleResult). ConfigError for a bad level. */
int ptg_mgopt_cycle(ptg_hier *h, int level, const double *z, const double *v, const double *warm_value,
                    const double *warm_grad, double *z_out, double *value_out, double *grad_out, ptg_report *rep);
/* one top-level V-cycle (mgoptCycle, multigrid.hpp:78-80) on device buffers:
 * z in/out (level-0 precision), warm (value, grad) in/out. */
int ptg_mgopt_cycle_device(ptg_hier *h, void *z, double *value, void *grad, ptg_report *rep);

#ifdef __cplusplus
}
#endif
#endif
