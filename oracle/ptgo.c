/*
 * ptgo.c — CPU ORACLE (test infrastructure only; see ptgo.h for the rules).
 *
 * Plain-C restatement of the reference algorithm, each function citing the
 * reference file:line it follows (paths relative to /root/reference/proj/).
 * Arithmetic is kept in the same operation order as the reference so that in
 * ref mode (binary window, M == n) results are bitwise identical to the
 * compiled reference library; build with -ffp-contract=off (oracle/Makefile).
 */
#include "ptgo.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ errors */
static _Thread_local char g_err[512];

const char *ptgo_last_error(void) { return g_err; }

static int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

#define TRY(expr)                  \
    do {                           \
        int rc_ = (expr);          \
        if (rc_ != PTGO_OK) return rc_; \
    } while (0)

static void *xcalloc(size_t n, size_t sz) { return calloc(n ? n : 1, sz); }

/* -------------------------------------------------------------- L0 kernels */

/* Optional external 2-D FFT (the reference's own OpenMP kernels::fft2_inplace,
 * installed by the CPU-baseline harness).  NULL = the restated serial FFT. */
typedef void (*ptgo_fft_fn)(double *a, int n, int inverse);
static ptgo_fft_fn g_fft_hook = NULL;
void ptgo_set_fft_hook(void *fn) { g_fft_hook = (ptgo_fft_fn)fn; }

static int g_threads = 1;
/* Pattern-parallel evaluation (results stay bitwise identical: per-pattern
 * contributions are accumulated in scan order afterwards). */
void ptgo_set_threads(int t) {
    g_threads = t < 1 ? 1 : t;
    /* also the OpenMP default of the calling thread: the reference's
       kernels::fft2_inplace parallelises its rows (kernels.cpp:126) whenever
       it runs outside the position-parallel region -- t = 1 is one thread */
    omp_set_num_threads(g_threads);
}

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

/* kernels.cpp:23-30: tw[k] = exp(-+2 pi i k / n), each from its own angle */
static void make_twiddles(double *tw, int n, int inverse) {
    const double sign = inverse ? 1.0 : -1.0;
    const double step = sign * 2.0 * 3.141592653589793238462643383279502884 / n;
    for (int k = 0; k < n / 2; ++k) {
        const double th = step * (double)k;
        tw[2 * k] = cos(th);
        tw[2 * k + 1] = sin(th);
    }
}

/* kernels.cpp:34-53: iterative radix-2 DIT on contiguous complex data */
static void fft1d(double *a, int n, const double *tw) {
    for (int i = 1, j = 0; i < n; ++i) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j |= bit;
        if (i < j) {
            double t0 = a[2 * i], t1 = a[2 * i + 1];
            a[2 * i] = a[2 * j];
            a[2 * i + 1] = a[2 * j + 1];
            a[2 * j] = t0;
            a[2 * j + 1] = t1;
        }
    }
    for (int len = 2; len <= n; len <<= 1) {
        const int half = len >> 1;
        const int step = n / len;
        for (int i = 0; i < n; i += len) {
            for (int j = 0; j < half; ++j) {
                const double *w = tw + 2 * (size_t)j * step;
                double *p = a + 2 * (size_t)(i + j);
                double *q = a + 2 * (size_t)(i + j + half);
                const double ur = p[0], ui = p[1];
                const double tr = q[0] * w[0] - q[1] * w[1];
                const double ti = q[0] * w[1] + q[1] * w[0];
                p[0] = ur + tr;
                p[1] = ui + ti;
                q[0] = ur - tr;
                q[1] = ui - ti;
            }
        }
    }
}

/* kernels.cpp:55-85: rows, gathered columns, 1/n^2 on the inverse */
static int fft2_serial(double *a, int n, int inverse) {
    if (!is_pow2(n))
        return fail(PTGO_GEOMETRY, "fft2: grid side must be a positive power of two, got %d", n);
    if (n == 1) return PTGO_OK;
    double *tw = (double *)xcalloc((size_t)n, sizeof(double));
    double *col = (double *)xcalloc((size_t)2 * n, sizeof(double));
    if (!tw || !col) { free(tw); free(col); return fail(PTGO_NOMEM, "fft2: out of memory"); }
    make_twiddles(tw, n, inverse);
    for (int r = 0; r < n; ++r) fft1d(a + 2 * (size_t)r * n, n, tw);
    for (int c = 0; c < n; ++c) {
        for (int r = 0; r < n; ++r) {
            col[2 * r] = a[2 * ((size_t)r * n + c)];
            col[2 * r + 1] = a[2 * ((size_t)r * n + c) + 1];
        }
        fft1d(col, n, tw);
        for (int r = 0; r < n; ++r) {
            a[2 * ((size_t)r * n + c)] = col[2 * r];
            a[2 * ((size_t)r * n + c) + 1] = col[2 * r + 1];
        }
    }
    if (inverse) {
        const double s = 1.0 / ((double)n * (double)n);
        const size_t total = (size_t)n * n;
        for (size_t i = 0; i < 2 * total; ++i) a[i] *= s;
    }
    free(tw);
    free(col);
    return PTGO_OK;
}

int ptgo_fft2(double *a, int n, int inverse) {
    if (!is_pow2(n))
        return fail(PTGO_GEOMETRY, "fft2: grid side must be a positive power of two, got %d", n);
    if (g_fft_hook) {
        g_fft_hook(a, n, inverse);
        return PTGO_OK;
    }
    return fft2_serial(a, n, inverse);
}

/* kernels.cpp:87-120: 1024-element blocks summed serially in block order */
#define REDUCE_BLOCK 1024
double ptgo_norm2sq(const double *a, size_t len) {
    double total = 0.0;
    for (size_t lo = 0; lo < len; lo += REDUCE_BLOCK) {
        const size_t hi = lo + REDUCE_BLOCK < len ? lo + REDUCE_BLOCK : len;
        double s = 0.0;
        for (size_t i = lo; i < hi; ++i) s += a[2 * i] * a[2 * i] + a[2 * i + 1] * a[2 * i + 1];
        total += s;
    }
    return total;
}

double ptgo_dot_real(const double *a, const double *b, size_t len) {
    double total = 0.0;
    for (size_t lo = 0; lo < len; lo += REDUCE_BLOCK) {
        const size_t hi = lo + REDUCE_BLOCK < len ? lo + REDUCE_BLOCK : len;
        double s = 0.0;
        for (size_t i = lo; i < hi; ++i) s += a[2 * i] * b[2 * i] + a[2 * i + 1] * b[2 * i + 1];
        total += s;
    }
    return total;
}

static double norm2(const double *a, size_t len) { return sqrt(ptgo_norm2sq(a, len)); }

/* field.cpp:116-119 */
static void axpy(double *y, double alpha, const double *x, size_t len) {
    for (size_t i = 0; i < len; ++i) {
        y[2 * i] += alpha * x[2 * i];
        y[2 * i + 1] += alpha * x[2 * i + 1];
    }
}
static void scale_into(double *out, const double *a, double alpha, size_t len) {
    for (size_t i = 0; i < 2 * len; ++i) out[i] = a[i] * alpha;
}
static void sub_into(double *out, const double *a, const double *b, size_t len) {
    for (size_t i = 0; i < 2 * len; ++i) out[i] = a[i] - b[i];
}
static int all_finite(const double *a, size_t len) {
    for (size_t i = 0; i < 2 * len; ++i)
        if (!isfinite(a[i])) return 0;
    return 1;
}

/* ------------------------------------------------------------- objectives */

/* ref mode: binary window and M == n -> the frame IS the reference's n x n
 * grid and the window sits in place (field.cpp:53-60); otherwise the window
 * content is placed at the frame origin (shift theorem: |fft| is invariant). */
static int ref_mode(const ptgo_problem *p) { return p->probe == NULL && p->M == p->n; }

static void frame_origin(const ptgo_problem *p, int k, int *fr, int *fc) {
    if (ref_mode(p)) {
        *fr = p->pos[2 * k];
        *fc = p->pos[2 * k + 1];
    } else {
        *fr = 0;
        *fc = 0;
    }
}

/* objectives.cpp:12-26 + field.cpp:45-51 */
int ptgo_validate(const ptgo_problem *p) {
    if (p->n < 1) return fail(PTGO_GEOMETRY, "object side must be positive");
    if (!is_pow2(p->M))
        return fail(PTGO_GEOMETRY, "fft2: grid side must be a positive power of two, got %d", p->M);
    if (p->w < 1 || p->w > p->M || p->w > p->n)
        return fail(PTGO_GEOMETRY, "window side %d must satisfy 1 <= w <= min(M, n)", p->w);
    if (p->N < 0) return fail(PTGO_DOMAIN, "negative pattern count");
    if (p->metric != PTGO_DISTANCE && p->metric != PTGO_INTENSITY)
        return fail(PTGO_CONFIG, "unknown metric kind %d", p->metric);
    for (int k = 0; k < p->N; ++k) {
        const int r = p->pos[2 * k], c = p->pos[2 * k + 1];
        if (r < 0 || c < 0 || r + p->w > p->n || c + p->w > p->n)
            return fail(PTGO_GEOMETRY, "probe window [%d,%d)+%d does not fit an n=%d grid", r, c,
                        p->w, p->n);
    }
    const size_t MM = (size_t)p->M * p->M;
    for (size_t i = 0; i < (size_t)p->N * MM; ++i)
        if (p->data[i] < 0.0)
            return fail(PTGO_DOMAIN, "diffraction pattern has a negative intensity at index %zu",
                        i % MM);
    return PTGO_OK;
}

/* psi = P o S_k z placed in the frame (applyProbe, field.cpp:53-60) */
static void gather_frame(const ptgo_problem *p, const double *z, int k, double *buf) {
    const int M = p->M, w = p->w, n = p->n;
    int fr, fc;
    frame_origin(p, k, &fr, &fc);
    memset(buf, 0, sizeof(double) * 2 * (size_t)M * M);
    const int r0 = p->pos[2 * k], c0 = p->pos[2 * k + 1];
    for (int r = 0; r < w; ++r)
        for (int c = 0; c < w; ++c) {
            const double *zz = z + 2 * ((size_t)(r0 + r) * n + (c0 + c));
            double *b = buf + 2 * ((size_t)(fr + r) * M + (fc + c));
            if (p->probe) {
                const double *P = p->probe + 2 * ((size_t)r * M + c);
                b[0] = P[0] * zz[0] - P[1] * zz[1];
                b[1] = P[0] * zz[1] + P[1] * zz[0];
            } else {
                b[0] = zz[0];
                b[1] = zz[1];
            }
        }
}

/* objectives.cpp:29-38: W -> sqrt(d) W/|W|, vanishing W -> sqrt(d) + 0i */
static void replace_modulus(double *buf, const double *d, size_t len) {
    for (size_t i = 0; i < len; ++i) {
        const double target = sqrt(d[i]);
        const double mag = hypot(buf[2 * i], buf[2 * i + 1]);
        if (mag == 0.0) {
            buf[2 * i] = target;
            buf[2 * i + 1] = 0.0;
        } else {
            const double s = target / mag;
            buf[2 * i] *= s;
            buf[2 * i + 1] *= s;
        }
    }
}

/* objectives.cpp:42-50 (validation of d happens once in ptgo_validate) */
int ptgo_project_modulus(const ptgo_problem *p, const double *z, int k, double *frame) {
    TRY(ptgo_validate(p));
    if (k < 0 || k >= p->N) return fail(PTGO_DOMAIN, "pattern index %d out of range", k);
    gather_frame(p, z, k, frame);
    TRY(ptgo_fft2(frame, p->M, 0));
    replace_modulus(frame, p->data + (size_t)k * p->M * p->M, (size_t)p->M * p->M);
    TRY(ptgo_fft2(frame, p->M, 1));
    return PTGO_OK;
}

/* Per-pattern work of phiDistance (objectives.cpp:59-72): fills contrib
 * (w x w, the term SUBTRACTED from the gradient: conj(P) o (Pi(psi) - psi))
 * and returns the pattern's value 1/2 ||Pi(psi) - psi||^2 over the frame. */
static int distance_one(const ptgo_problem *p, const double *z, int k, double *buf,
                        double *contrib, double *value) {
    const int M = p->M, w = p->w, n = p->n;
    const size_t MM = (size_t)M * M;
    int fr, fc;
    frame_origin(p, k, &fr, &fc);
    gather_frame(p, z, k, buf);
    TRY(ptgo_fft2(buf, M, 0));
    replace_modulus(buf, p->data + (size_t)k * MM, MM);
    TRY(ptgo_fft2(buf, M, 1));
    /* residual = Pi(psi) - psi over the full frame (psi vanishes off-window) */
    const int r0 = p->pos[2 * k], c0 = p->pos[2 * k + 1];
    for (int r = 0; r < w; ++r)
        for (int c = 0; c < w; ++c) {
            double *b = buf + 2 * ((size_t)(fr + r) * M + (fc + c));
            const double *zz = z + 2 * ((size_t)(r0 + r) * n + (c0 + c));
            if (p->probe) {
                const double *P = p->probe + 2 * ((size_t)r * M + c);
                b[0] -= P[0] * zz[0] - P[1] * zz[1];
                b[1] -= P[0] * zz[1] + P[1] * zz[0];
            } else {
                b[0] = b[0] - zz[0];
                b[1] = b[1] - zz[1];
            }
        }
    *value = 0.5 * ptgo_norm2sq(buf, MM);
    for (int r = 0; r < w; ++r)
        for (int c = 0; c < w; ++c) {
            const double *b = buf + 2 * ((size_t)(fr + r) * M + (fc + c));
            double *o = contrib + 2 * ((size_t)r * w + c);
            if (p->probe) {
                const double *P = p->probe + 2 * ((size_t)r * M + c);
                o[0] = P[0] * b[0] + P[1] * b[1];   /* conj(P) * b */
                o[1] = P[0] * b[1] - P[1] * b[0];
            } else {
                o[0] = b[0];
                o[1] = b[1];
            }
        }
    return PTGO_OK;
}

/* Per-pattern work of phiIntensityGaussian (objectives.cpp:83-103): contrib is
 * ADDED to the gradient: 2 M^2 conj(P) o ifft2(r o W), r = |W|^2 - d. */
static int intensity_one(const ptgo_problem *p, const double *z, int k, double *buf,
                         double *contrib, double *value) {
    const int M = p->M, w = p->w;
    const size_t MM = (size_t)M * M;
    const double n2 = (double)M * M;
    const double *d = p->data + (size_t)k * MM;
    int fr, fc;
    frame_origin(p, k, &fr, &fc);
    gather_frame(p, z, k, buf);
    TRY(ptgo_fft2(buf, M, 0));
    double sum_sq = 0.0;
    for (size_t i = 0; i < MM; ++i) {
        const double r = (buf[2 * i] * buf[2 * i] + buf[2 * i + 1] * buf[2 * i + 1]) - d[i];
        sum_sq += r * r;
        buf[2 * i] *= r;
        buf[2 * i + 1] *= r;
    }
    *value = 0.5 * sum_sq;
    TRY(ptgo_fft2(buf, M, 1));
    const double s = 2.0 * n2;
    for (int r = 0; r < w; ++r)
        for (int c = 0; c < w; ++c) {
            const double *b = buf + 2 * ((size_t)(fr + r) * M + (fc + c));
            double *o = contrib + 2 * ((size_t)r * w + c);
            if (p->probe) {
                const double *P = p->probe + 2 * ((size_t)r * M + c);
                const double br = P[0] * b[0] + P[1] * b[1];
                const double bi = P[0] * b[1] - P[1] * b[0];
                o[0] = s * br;
                o[1] = s * bi;
            } else {
                o[0] = s * b[0];
                o[1] = s * b[1];
            }
        }
    return PTGO_OK;
}

/* objectives.cpp:52-74 / 76-104 / 106-118 */
int ptgo_evaluate(const ptgo_problem *p, const double *z, const double *v, double *value,
                  double *grad) {
    TRY(ptgo_validate(p));
    const int n = p->n, M = p->M, w = p->w;
    const size_t nn = (size_t)n * n, MM = (size_t)M * M, ww = (size_t)w * w;
    memset(grad, 0, sizeof(double) * 2 * nn);
    double total = 0.0;
    const int chunk = 256;
    const int T = g_threads;
    double *bufs = (double *)xcalloc((size_t)T * 2 * MM, sizeof(double));
    double *contrib = (double *)xcalloc((size_t)chunk * 2 * ww, sizeof(double));
    double *vals = (double *)xcalloc((size_t)chunk, sizeof(double));
    int *rcs = (int *)xcalloc((size_t)chunk, sizeof(int));
    if (!bufs || !contrib || !vals || !rcs) {
        free(bufs); free(contrib); free(vals); free(rcs);
        return fail(PTGO_NOMEM, "evaluate: out of memory");
    }
    int rc = PTGO_OK;
    for (int base = 0; base < p->N && rc == PTGO_OK; base += chunk) {
        const int cnt = p->N - base < chunk ? p->N - base : chunk;
#pragma omp parallel for schedule(dynamic, 1) num_threads(T) if (T > 1)
        for (int i = 0; i < cnt; ++i) {
#ifdef _OPENMP
            const int tid = omp_get_thread_num();
#else
            const int tid = 0;
#endif
            double *buf = bufs + (size_t)tid * 2 * MM;
            rcs[i] = (p->metric == PTGO_DISTANCE)
                         ? distance_one(p, z, base + i, buf, contrib + (size_t)i * 2 * ww, &vals[i])
                         : intensity_one(p, z, base + i, buf, contrib + (size_t)i * 2 * ww, &vals[i]);
        }
        /* accumulate in scan order (objectives.cpp:59-72) */
        for (int i = 0; i < cnt; ++i) {
            if (rcs[i] != PTGO_OK) { rc = rcs[i]; break; }
            const int k = base + i;
            const int r0 = p->pos[2 * k], c0 = p->pos[2 * k + 1];
            total += vals[i];
            const double *o = contrib + (size_t)i * 2 * ww;
            for (int r = 0; r < w; ++r)
                for (int c = 0; c < w; ++c) {
                    double *g = grad + 2 * ((size_t)(r0 + r) * n + (c0 + c));
                    const double *oo = o + 2 * ((size_t)r * w + c);
                    if (p->metric == PTGO_DISTANCE) {
                        g[0] -= oo[0];
                        g[1] -= oo[1];
                    } else {
                        g[0] += oo[0];
                        g[1] += oo[1];
                    }
                }
        }
    }
    free(bufs); free(contrib); free(vals); free(rcs);
    if (rc != PTGO_OK) return rc;
    if (v) {
        total -= ptgo_dot_real(v, z, nn);
        axpy(grad, -1.0, v, nn);
    }
    *value = total;
    return PTGO_OK;
}

/* forward.cpp:40-54 */
int ptgo_simulate(const ptgo_problem *p, const double *z, double *data_out) {
    const int M = p->M;
    const size_t MM = (size_t)M * M;
    if (!is_pow2(M)) return fail(PTGO_GEOMETRY, "fft2: grid side must be a positive power of two, got %d", M);
    double *buf = (double *)xcalloc(2 * MM, sizeof(double));
    if (!buf) return fail(PTGO_NOMEM, "simulate: out of memory");
    for (int k = 0; k < p->N; ++k) {
        gather_frame(p, z, k, buf);
        int rc = ptgo_fft2(buf, M, 0);
        if (rc) { free(buf); return rc; }
        double *d = data_out + (size_t)k * MM;
        for (size_t i = 0; i < MM; ++i) d[i] = buf[2 * i] * buf[2 * i] + buf[2 * i + 1] * buf[2 * i + 1];
    }
    free(buf);
    return PTGO_OK;
}

/* -------------------------------------------------------------- transfers */

/* multigrid.cpp:34-44: ((a+b)+(c+d)) * 1/4 on disjoint 2x2 blocks */
int ptgo_restrict_field(const double *fine, int n, double *coarse) {
    if (n < 2 || n % 2 != 0)
        return fail(PTGO_GEOMETRY, "restrictField: grid side must be even and >= 2, got %d", n);
    const int nH = n / 2;
    for (int r = 0; r < nH; ++r)
        for (int c = 0; c < nH; ++c)
            for (int part = 0; part < 2; ++part) {
                const double a = fine[2 * ((size_t)(2 * r) * n + 2 * c) + part];
                const double b = fine[2 * ((size_t)(2 * r) * n + 2 * c + 1) + part];
                const double cc = fine[2 * ((size_t)(2 * r + 1) * n + 2 * c) + part];
                const double d = fine[2 * ((size_t)(2 * r + 1) * n + 2 * c + 1) + part];
                coarse[2 * ((size_t)r * nH + c) + part] = ((a + b) + (cc + d)) * 0.25;
            }
    return PTGO_OK;
}

/* multigrid.cpp:46-53: block copy */
int ptgo_prolong_field(const double *coarse, int nH, double *fine) {
    if (nH < 1) return fail(PTGO_GEOMETRY, "prolongField: empty grid");
    const int n = 2 * nH;
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) {
            fine[2 * ((size_t)r * n + c)] = coarse[2 * ((size_t)(r / 2) * nH + c / 2)];
            fine[2 * ((size_t)r * n + c) + 1] = coarse[2 * ((size_t)(r / 2) * nH + c / 2) + 1];
        }
    return PTGO_OK;
}

/* multigrid.cpp:55-77: centred low-pass crop x 1/16 */
int ptgo_restrict_data(const double *fine, int N, int M, double *coarse) {
    if (M < 4 || M % 4 != 0)
        return fail(PTGO_GEOMETRY, "restrictData: grid side must be a multiple of 4");
    const int MH = M / 2;
    for (int k = 0; k < N; ++k) {
        const double *pf = fine + (size_t)k * M * M;
        double *pc = coarse + (size_t)k * MH * MH;
        for (int u = 0; u < MH; ++u) {
            const int uf = ((u + MH / 2) % MH + 3 * M / 4) % M;
            for (int v = 0; v < MH; ++v) {
                const int vf = ((v + MH / 2) % MH + 3 * M / 4) % M;
                pc[(size_t)u * MH + v] = pf[(size_t)uf * M + vf] * (1.0 / 16.0);
            }
        }
    }
    return PTGO_OK;
}

/* ---------------------------------------------------------------- reports */

void ptgo_report_free(ptgo_report *r) {
    if (!r) return;
    free(r->hist);
    r->hist = NULL;
    r->len = r->cap = 0;
}

static int push_hist(ptgo_report *r, double weighted, double value, double gnorm) {
    if (!r) return PTGO_OK;
    if (r->len == r->cap) {
        int cap = r->cap ? 2 * r->cap : 16;
        ptgo_hist *h = (ptgo_hist *)realloc(r->hist, sizeof(ptgo_hist) * (size_t)cap);
        if (!h) return fail(PTGO_NOMEM, "history: out of memory");
        r->hist = h;
        r->cap = cap;
    }
    r->hist[r->len].weighted = weighted;
    r->hist[r->len].value = value;
    r->hist[r->len].gnorm = gnorm;
    r->len++;
    return PTGO_OK;
}

/* solvers.hpp:16-24 / 33-36: charge before evaluating */
static int counted_eval(const ptgo_counted *o, ptgo_counter *ctr, const double *z, double *value,
                        double *grad) {
    ctr->weighted += o->weight;
    if (o->level >= 0 && o->level < PTGO_MAX_LEVELS) ctr->per_level[o->level]++;
    return o->fn(o->user, z, value, grad);
}

void ptgo_solver_cfg_default(ptgo_solver_cfg *c) {
    c->max_iters = 100;
    c->grad_tol_rel = 0.0;
    c->grad_tol_abs = 1e-13;
    c->lbfgs_memory = 25;
    c->linesearch_max = 50;
    c->max_weighted = INFINITY;
    c->cg_max_iters = 20;
    c->cg_rel_tol = 0.1;
}

/* solvers.cpp:61-85 */
int ptgo_linesearch(const ptgo_counted *obj, const double *z, const double *dir,
                    ptgo_counter *ctr, int max_trials, const double *phi0, double *alpha_out,
                    int *stalled, int *trials, double *z_out, double *value_out,
                    double *grad_out) {
    const size_t len = obj->len;
    double base;
    double *tmpg = NULL;
    if (phi0) {
        base = *phi0;
    } else {
        tmpg = (double *)xcalloc(2 * len, sizeof(double));
        if (!tmpg) return fail(PTGO_NOMEM, "linesearch: out of memory");
        int rc = counted_eval(obj, ctr, z, &base, tmpg);
        free(tmpg);
        if (rc) return rc;
    }
    double *trial = (double *)xcalloc(2 * len, sizeof(double));
    double *g = (double *)xcalloc(2 * len, sizeof(double));
    if (!trial || !g) { free(trial); free(g); return fail(PTGO_NOMEM, "linesearch: out of memory"); }
    double alpha = 1.0;
    *trials = 0;
    for (int t = 0; t < max_trials; ++t) {
        memcpy(trial, z, sizeof(double) * 2 * len);
        axpy(trial, alpha, dir, len);
        double val;
        int rc = counted_eval(obj, ctr, trial, &val, g);
        if (rc) { free(trial); free(g); return rc; }
        ++*trials;
        if (val <= base) {
            *alpha_out = alpha;
            *stalled = 0;
            memcpy(z_out, trial, sizeof(double) * 2 * len);
            *value_out = val;
            memcpy(grad_out, g, sizeof(double) * 2 * len);
            free(trial); free(g);
            return PTGO_OK;
        }
        alpha *= 0.5;
    }
    *alpha_out = 0.0;
    *stalled = 1;
    if (z_out != z) memcpy(z_out, z, sizeof(double) * 2 * len);
    free(trial); free(g);
    return PTGO_OK;
}

/* solvers.cpp:19-36: two-loop recursion over the pair ring (oldest first) */
typedef struct { double *s, *y; double sy; } pair_t;

static void two_loop(const pair_t *pairs, int np, const double *g, double *q, double *alpha,
                     size_t len) {
    if (np == 0) {
        scale_into(q, g, -1.0, len);
        return;
    }
    memcpy(q, g, sizeof(double) * 2 * len);
    for (int i = np; i-- > 0;) {
        alpha[i] = ptgo_dot_real(pairs[i].s, q, len) / pairs[i].sy;
        axpy(q, -alpha[i], pairs[i].y, len);
    }
    const pair_t *newest = &pairs[np - 1];
    const double gamma = newest->sy / ptgo_dot_real(newest->y, newest->y, len);
    scale_into(q, q, gamma, len);
    for (int i = 0; i < np; ++i) {
        const double beta = ptgo_dot_real(pairs[i].y, q, len) / pairs[i].sy;
        axpy(q, alpha[i] - beta, pairs[i].s, len);
    }
    scale_into(q, q, -1.0, len);
}

/* solvers.cpp:87-141 */
int ptgo_lbfgs(const ptgo_counted *obj, const double *z0, const ptgo_solver_cfg *cfg,
               ptgo_counter *ctr, const double *warm_value, const double *warm_grad,
               double *z_out, double *value_out, double *grad_out, ptgo_report *rep) {
    const size_t len = obj->len;
    const size_t bytes = sizeof(double) * 2 * len;
    int rc = PTGO_OK;
    const int mem = cfg->lbfgs_memory > 0 ? cfg->lbfgs_memory : 1;
    double *z = (double *)malloc(bytes), *g = (double *)malloc(bytes);
    double *dir = (double *)malloc(bytes), *nz = (double *)malloc(bytes), *ng = (double *)malloc(bytes);
    double *alpha = (double *)xcalloc((size_t)mem + 1, sizeof(double));
    pair_t *pairs = (pair_t *)xcalloc((size_t)mem + 1, sizeof(pair_t));
    int np = 0;
    double cur;
    if (!z || !g || !dir || !nz || !ng || !alpha || !pairs) { rc = fail(PTGO_NOMEM, "lbfgs: out of memory"); goto done; }
    memcpy(z, z0, bytes);
    if (warm_value) {
        cur = *warm_value;
        memcpy(g, warm_grad, bytes);
    } else if ((rc = counted_eval(obj, ctr, z, &cur, g)) != PTGO_OK) {
        goto done;
    }
    if (!all_finite(g, len)) { rc = fail(PTGO_NUMERIC, "non-finite iterate in lbfgs"); goto done; }
    const double grad_floor = cfg->grad_tol_abs * (1.0 + norm2(z0, len));
    const double g0 = norm2(g, len);
    double gnorm = g0;
    if ((rc = push_hist(rep, ctr->weighted, cur, gnorm))) goto done;
    int reason = PTGO_STOP_MAXITERS;
#define SATISFIED(gn) ((gn) <= fmax(cfg->grad_tol_rel * g0, grad_floor))
    if (SATISFIED(gnorm)) {
        reason = PTGO_STOP_TOLERANCE;
    } else {
        for (int iter = 1; iter <= cfg->max_iters; ++iter) {
            two_loop(pairs, np, g, dir, alpha, len);
            if (ptgo_dot_real(dir, g, len) >= 0.0) scale_into(dir, g, -1.0, len);
            double a, val;
            int stalled, trials;
            rc = ptgo_linesearch(obj, z, dir, ctr, cfg->linesearch_max, &cur, &a, &stalled,
                                 &trials, nz, &val, ng);
            if (rc) goto done;
            if (stalled) { reason = PTGO_STOP_STALL; break; }
            if (!all_finite(nz, len)) { rc = fail(PTGO_NUMERIC, "non-finite iterate in lbfgs"); goto done; }
            double *s = (double *)malloc(bytes), *y = (double *)malloc(bytes);
            if (!s || !y) { free(s); free(y); rc = fail(PTGO_NOMEM, "lbfgs: out of memory"); goto done; }
            sub_into(s, nz, z, len);
            sub_into(y, ng, g, len);
            const double sy = ptgo_dot_real(s, y, len);
            if (sy > 1e-12 * norm2(s, len) * norm2(y, len)) {
                pairs[np].s = s;
                pairs[np].y = y;
                pairs[np].sy = sy;
                np++;
                if (np > mem) {
                    free(pairs[0].s);
                    free(pairs[0].y);
                    memmove(pairs, pairs + 1, sizeof(pair_t) * (size_t)(np - 1));
                    np--;
                }
            } else {
                free(s);
                free(y);
            }
            memcpy(z, nz, bytes);
            memcpy(g, ng, bytes);
            cur = val;
            gnorm = norm2(g, len);
            if ((rc = push_hist(rep, ctr->weighted, cur, gnorm))) goto done;
            if (SATISFIED(gnorm)) { reason = PTGO_STOP_TOLERANCE; break; }
            if (ctr->weighted >= cfg->max_weighted) { reason = PTGO_STOP_BUDGET; break; }
        }
    }
#undef SATISFIED
    if (rep) rep->reason = reason;
    memcpy(z_out, z, bytes);
    if (value_out) *value_out = cur;
    if (grad_out) memcpy(grad_out, g, bytes);
done:
    for (int i = 0; i < np; ++i) { free(pairs[i].s); free(pairs[i].y); }
    free(z); free(g); free(dir); free(nz); free(ng); free(alpha); free(pairs);
    return rc;
}

/* solvers.cpp:143-227: Newton-CG, each Hessian-vector product a counted
 * gradient evaluation at z + delta v (delta = 1e-6 (1 + |z|) / |v|) */
int ptgo_truncated_newton(const ptgo_counted *obj, const double *z0, const ptgo_solver_cfg *cfg,
                          ptgo_counter *ctr, const double *warm_value, const double *warm_grad,
                          double *z_out, double *value_out, double *grad_out, ptgo_report *rep) {
    const size_t len = obj->len;
    const size_t bytes = sizeof(double) * 2 * len;
    int rc = PTGO_OK;
    double *z = (double *)malloc(bytes), *g = (double *)malloc(bytes), *x = (double *)malloc(bytes);
    double *r = (double *)malloc(bytes), *p = (double *)malloc(bytes), *hp = (double *)malloc(bytes);
    double *zp = (double *)malloc(bytes), *gp = (double *)malloc(bytes), *nz = (double *)malloc(bytes);
    double *ng = (double *)malloc(bytes);
    double cur;
    if (!z || !g || !x || !r || !p || !hp || !zp || !gp || !nz || !ng) {
        rc = fail(PTGO_NOMEM, "truncatedNewton: out of memory");
        goto done;
    }
    memcpy(z, z0, bytes);
    if (warm_value) {
        cur = *warm_value;
        memcpy(g, warm_grad, bytes);
    } else if ((rc = counted_eval(obj, ctr, z, &cur, g)) != PTGO_OK) {
        goto done;
    }
    if (!all_finite(g, len)) { rc = fail(PTGO_NUMERIC, "non-finite iterate in truncatedNewton"); goto done; }
    const double grad_floor = cfg->grad_tol_abs * (1.0 + norm2(z0, len));
    const double g0 = norm2(g, len);
    double gnorm = g0;
    if ((rc = push_hist(rep, ctr->weighted, cur, gnorm))) goto done;
    int reason = PTGO_STOP_MAXITERS;
#define SATISFIED(gn) ((gn) <= fmax(cfg->grad_tol_rel * g0, grad_floor))
    if (SATISFIED(gnorm)) {
        reason = PTGO_STOP_TOLERANCE;
    } else {
        for (int iter = 1; iter <= cfg->max_iters; ++iter) {
            /* CG on H x = -g from x = 0 */
            memset(x, 0, bytes);
            scale_into(r, g, -1.0, len);
            const double rhs_norm = norm2(r, len);
            memcpy(p, r, bytes);
            double rs = ptgo_dot_real(r, r, len);
            for (int cg = 0; cg < cfg->cg_max_iters; ++cg) {
                /* hessVec(p) */
                const double vnorm = norm2(p, len);
                if (vnorm == 0.0) {
                    memset(hp, 0, bytes);
                } else {
                    const double delta = 1e-6 * (1.0 + norm2(z, len)) / vnorm;
                    memcpy(zp, z, bytes);
                    axpy(zp, delta, p, len);
                    double vp;
                    if ((rc = counted_eval(obj, ctr, zp, &vp, gp)) != PTGO_OK) goto done;
                    sub_into(hp, gp, g, len);
                    scale_into(hp, hp, 1.0 / delta, len);
                }
                const double php = ptgo_dot_real(p, hp, len);
                if (php <= 0.0) {
                    /* negative curvature: keep what CG built, or steepest descent at cg == 0 */
                    if (cg == 0) memcpy(x, r, bytes);
                    break;
                }
                const double step = rs / php;
                axpy(x, step, p, len);
                axpy(r, -step, hp, len);
                const double rs_new = ptgo_dot_real(r, r, len);
                if (sqrt(rs_new) <= cfg->cg_rel_tol * rhs_norm) break;
                /* p = r + beta p, formed as a copy of r then axpy */
                memcpy(zp, r, bytes);
                axpy(zp, rs_new / rs, p, len);
                memcpy(p, zp, bytes);
                rs = rs_new;
            }
            if (norm2(x, len) == 0.0 || ptgo_dot_real(x, g, len) >= 0.0) scale_into(x, g, -1.0, len);
            double a, val;
            int stalled, trials;
            rc = ptgo_linesearch(obj, z, x, ctr, cfg->linesearch_max, &cur, &a, &stalled, &trials, nz, &val, ng);
            if (rc) goto done;
            if (stalled) { reason = PTGO_STOP_STALL; break; }
            if (!all_finite(nz, len)) { rc = fail(PTGO_NUMERIC, "non-finite iterate in truncatedNewton"); goto done; }
            memcpy(z, nz, bytes);
            memcpy(g, ng, bytes);
            cur = val;
            gnorm = norm2(g, len);
            if ((rc = push_hist(rep, ctr->weighted, cur, gnorm))) goto done;
            if (SATISFIED(gnorm)) { reason = PTGO_STOP_TOLERANCE; break; }
            if (ctr->weighted >= cfg->max_weighted) { reason = PTGO_STOP_BUDGET; break; }
        }
    }
#undef SATISFIED
    if (rep) rep->reason = reason;
    memcpy(z_out, z, bytes);
    if (value_out) *value_out = cur;
    if (grad_out) memcpy(grad_out, g, bytes);
done:
    free(z); free(g); free(x); free(r); free(p); free(hp); free(zp); free(gp); free(nz); free(ng);
    return rc;
}

/* ------------------------------------------------------------------- PIE */

/* solvers.cpp:229-265.  Complex probes use Alg. 1:
 *   x_win += (|P|/max|P|) conj(P)/(|P|^2 + gamma) o (Pi(psi) - psi),
 * which reduces to (Pi(z) - z)/(1 + gamma) for the binary window. */
static int __attribute__((unused)) distance_plain(void *user, const double *z, double *value, double *grad) {
    return ptgo_evaluate((const ptgo_problem *)user, z, NULL, value, grad);
}

int ptgo_pie(const ptgo_problem *p, const double *z0, double gamma, int sweeps,
             double max_weighted, ptgo_counter *ctr, double *z_out, double *final_value,
             ptgo_report *rep) {
    if (gamma < 0.0) return fail(PTGO_CONFIG, "pie: gamma must be non-negative");
    TRY(ptgo_validate(p));
    ptgo_problem diag = *p;
    diag.metric = PTGO_DISTANCE;
    const int n = p->n, M = p->M, w = p->w;
    const size_t nn = (size_t)n * n, MM = (size_t)M * M;
    double *z = z_out;
    if (z != z0) memcpy(z, z0, sizeof(double) * 2 * nn);
    double *g = (double *)xcalloc(2 * nn, sizeof(double));
    double *buf = (double *)xcalloc(2 * MM, sizeof(double));
    double *wgt = NULL;
    int rc = PTGO_OK;
    if (!g || !buf) { rc = fail(PTGO_NOMEM, "pie: out of memory"); goto done; }
    if (p->probe) {
        wgt = (double *)xcalloc(2 * (size_t)w * w, sizeof(double));
        if (!wgt) { rc = fail(PTGO_NOMEM, "pie: out of memory"); goto done; }
        double pmax = 0.0;
        for (size_t i = 0; i < MM; ++i) pmax = fmax(pmax, hypot(p->probe[2 * i], p->probe[2 * i + 1]));
        for (int r = 0; r < w; ++r)
            for (int c = 0; c < w; ++c) {
                const double *P = p->probe + 2 * ((size_t)r * M + c);
                const double a = hypot(P[0], P[1]);
                const double s = (pmax > 0.0 ? a / pmax : 0.0) / (a * a + gamma);
                wgt[2 * ((size_t)r * w + c)] = s * P[0];
                wgt[2 * ((size_t)r * w + c) + 1] = -s * P[1];
            }
    }
    double val;
    if ((rc = ptgo_evaluate(&diag, z, NULL, &val, g))) goto done;   /* uncounted diagnostic */
    if ((rc = push_hist(rep, ctr->weighted, val, norm2(g, nn)))) goto done;
    int reason = PTGO_STOP_MAXITERS;
    const double damping = 1.0 / (1.0 + gamma);
    for (int sweep = 1; sweep <= sweeps; ++sweep) {
        for (int k = 0; k < p->N; ++k) {
            int fr, fc;
            frame_origin(p, k, &fr, &fc);
            gather_frame(p, z, k, buf);
            if ((rc = ptgo_fft2(buf, M, 0))) goto done;
            replace_modulus(buf, p->data + (size_t)k * MM, MM);
            if ((rc = ptgo_fft2(buf, M, 1))) goto done;
            const int r0 = p->pos[2 * k], c0 = p->pos[2 * k + 1];
            for (int r = 0; r < w; ++r)
                for (int c = 0; c < w; ++c) {
                    double *zz = z + 2 * ((size_t)(r0 + r) * n + (c0 + c));
                    const double *b = buf + 2 * ((size_t)(fr + r) * M + (fc + c));
                    if (p->probe) {
                        const double *P = p->probe + 2 * ((size_t)r * M + c);
                        const double dr = b[0] - (P[0] * zz[0] - P[1] * zz[1]);
                        const double di = b[1] - (P[0] * zz[1] + P[1] * zz[0]);
                        const double *W = wgt + 2 * ((size_t)r * w + c);
                        zz[0] += W[0] * dr - W[1] * di;
                        zz[1] += W[0] * di + W[1] * dr;
                    } else {
                        const double dr = b[0] - zz[0];
                        const double di = b[1] - zz[1];
                        zz[0] += damping * dr;
                        zz[1] += damping * di;
                    }
                }
        }
        if (!all_finite(z, nn)) { rc = fail(PTGO_NUMERIC, "non-finite iterate in pie"); goto done; }
        ctr->weighted += 1.0;   /* one sweep = one fine-level evaluation */
        ctr->per_level[0]++;
        if ((rc = ptgo_evaluate(&diag, z, NULL, &val, g))) goto done;
        if ((rc = push_hist(rep, ctr->weighted, val, norm2(g, nn)))) goto done;
        if (ctr->weighted >= max_weighted) { reason = PTGO_STOP_BUDGET; break; }
    }
    if (rep) rep->reason = reason;
    if ((rc = ptgo_evaluate(&diag, z, NULL, &val, g))) goto done;    /* final diagnostic */
    if (final_value) *final_value = val;
done:
    free(g); free(buf); free(wgt);
    return rc;
}

/* ------------------------------------------------------------- multigrid */

void ptgo_mg_cfg_default(ptgo_mg_cfg *c) {
    c->k1 = 1;
    c->k2 = 1;
    c->coarsest_max_iters = 0;
    c->coarsest_grad_tol_rel = 1e-4;
    c->intermediate_grad_tol_rel = 1e-3;
    c->lbfgs_memory = 25;
    c->linesearch_max = 50;
    c->grad_tol_abs = 1e-13;
}

void ptgo_driver_cfg_default(ptgo_driver_cfg *c) {
    c->budget = 100.0;
    c->grad_tol_rel = 0.0;
    c->grad_tol_abs = 1e-13;
    c->max_cycles = 1000000;
}

typedef struct {
    ptgo_problem prob;
    int32_t *pos;
    double *probe;
    double *data;
    int level;
    double weight;
} level_t;

struct ptgo_hierarchy {
    level_t levels[PTGO_MAX_LEVELS];
    int depth;
    ptgo_mg_cfg opt;
    int coarsest_iters;
};

void ptgo_hierarchy_free(ptgo_hierarchy *h) {
    if (!h) return;
    for (int l = 0; l < h->depth; ++l) {
        free(h->levels[l].pos);
        free(h->levels[l].probe);
        free(h->levels[l].data);
    }
    free(h);
}

/* multigrid.cpp:79-93 restated for the patch model */
static int coarsen(const level_t *f, level_t *c) {
    const ptgo_problem *fp = &f->prob;
    if (fp->n < 16) return fail(PTGO_GEOMETRY, "buildCoarseLevel: refuse to coarsen below n = 8");
    if (fp->w < 2 || fp->w % 2 != 0)
        return fail(PTGO_GEOMETRY, "buildCoarseLevel: window size must be even and >= 2, got %d", fp->w);
    if (fp->M < 4 || fp->M % 4 != 0)
        return fail(PTGO_GEOMETRY, "restrictData: grid side must be a multiple of 4");
    const int N = fp->N, MH = fp->M / 2;
    c->pos = (int32_t *)xcalloc((size_t)2 * N, sizeof(int32_t));
    c->data = (double *)xcalloc((size_t)N * MH * MH, sizeof(double));
    c->probe = NULL;
    if (!c->pos || !c->data) return fail(PTGO_NOMEM, "hierarchy: out of memory");
    for (int i = 0; i < 2 * N; ++i) c->pos[i] = fp->pos[i] / 2;
    TRY(ptgo_restrict_data(fp->data, N, fp->M, c->data));
    if (fp->probe) {
        c->probe = (double *)xcalloc(2 * (size_t)MH * MH, sizeof(double));
        if (!c->probe) return fail(PTGO_NOMEM, "hierarchy: out of memory");
        TRY(ptgo_restrict_field(fp->probe, fp->M, c->probe));
    }
    c->prob.n = fp->n / 2;
    c->prob.M = MH;
    c->prob.w = fp->w / 2;
    c->prob.N = N;
    c->prob.pos = c->pos;
    c->prob.probe = c->probe;
    c->prob.data = c->data;
    c->prob.metric = fp->metric;
    c->level = f->level + 1;
    c->weight = f->weight * 0.25;
    return PTGO_OK;
}

/* multigrid.cpp:95-115 */
int ptgo_hierarchy_build(const ptgo_problem *fine, int depth, const ptgo_mg_cfg *opt,
                         ptgo_hierarchy **out) {
    if (depth < 1) return fail(PTGO_CONFIG, "hierarchy depth must be >= 1");
    if (depth > PTGO_MAX_LEVELS) return fail(PTGO_CONFIG, "hierarchy depth too large");
    if ((fine->n >> (depth - 1)) < 8)
        return fail(PTGO_CONFIG, "hierarchy depth %d would coarsen an n = %d grid below 8", depth,
                    fine->n);
    TRY(ptgo_validate(fine));
    ptgo_hierarchy *h = (ptgo_hierarchy *)xcalloc(1, sizeof(ptgo_hierarchy));
    if (!h) return fail(PTGO_NOMEM, "hierarchy: out of memory");
    h->opt = *opt;
    h->coarsest_iters = opt->coarsest_max_iters > 0 ? opt->coarsest_max_iters : (depth <= 2 ? 3 : 100);
    level_t *l0 = &h->levels[0];
    const size_t MM = (size_t)fine->M * fine->M;
    l0->pos = (int32_t *)xcalloc((size_t)2 * fine->N, sizeof(int32_t));
    l0->data = (double *)xcalloc((size_t)fine->N * MM, sizeof(double));
    h->depth = 1;
    if (!l0->pos || !l0->data) { ptgo_hierarchy_free(h); return fail(PTGO_NOMEM, "hierarchy: out of memory"); }
    memcpy(l0->pos, fine->pos, sizeof(int32_t) * 2 * (size_t)fine->N);
    memcpy(l0->data, fine->data, sizeof(double) * (size_t)fine->N * MM);
    if (fine->probe) {
        l0->probe = (double *)xcalloc(2 * MM, sizeof(double));
        if (!l0->probe) { ptgo_hierarchy_free(h); return fail(PTGO_NOMEM, "hierarchy: out of memory"); }
        memcpy(l0->probe, fine->probe, sizeof(double) * 2 * MM);
    }
    l0->prob = *fine;
    l0->prob.pos = l0->pos;
    l0->prob.data = l0->data;
    l0->prob.probe = l0->probe;
    l0->level = 0;
    l0->weight = 1.0;
    for (int l = 1; l < depth; ++l) {
        int rc = coarsen(&h->levels[l - 1], &h->levels[l]);
        h->depth = l + 1;
        if (rc) { ptgo_hierarchy_free(h); return rc; }
    }
    *out = h;
    return PTGO_OK;
}

const ptgo_problem *ptgo_hierarchy_level(const ptgo_hierarchy *h, int level) {
    return (level >= 0 && level < h->depth) ? &h->levels[level].prob : NULL;
}
int ptgo_hierarchy_depth(const ptgo_hierarchy *h) { return h->depth; }
int ptgo_hierarchy_coarsest_iters(const ptgo_hierarchy *h) { return h->coarsest_iters; }

/* levelObjective (multigrid.cpp:16-20): the shifted objective of one level */
typedef struct { const ptgo_problem *p; const double *v; } shifted_t;

static int shifted_fn(void *user, const double *z, double *value, double *grad) {
    const shifted_t *s = (const shifted_t *)user;
    return ptgo_evaluate(s->p, z, s->v, value, grad);
}

static ptgo_counted level_objective(const ptgo_hierarchy *h, int level, shifted_t *st,
                                    const double *v) {
    st->p = &h->levels[level].prob;
    st->v = v;
    ptgo_counted o;
    o.fn = shifted_fn;
    o.user = st;
    o.len = (size_t)st->p->n * st->p->n;
    o.level = h->levels[level].level;
    o.weight = h->levels[level].weight;
    return o;
}

/* multigrid.cpp:22-31 */
static ptgo_solver_cfg smoother_cfg(const ptgo_hierarchy *h, int level) {
    ptgo_solver_cfg c;
    ptgo_solver_cfg_default(&c);
    c.grad_tol_rel = (level == h->depth - 1) ? h->opt.coarsest_grad_tol_rel
                                             : h->opt.intermediate_grad_tol_rel;
    c.grad_tol_abs = h->opt.grad_tol_abs;
    c.lbfgs_memory = h->opt.lbfgs_memory;
    c.linesearch_max = h->opt.linesearch_max;
    return c;
}

/* multigrid.cpp:117-169 */
int ptgo_mgopt_cycle(const ptgo_hierarchy *h, int level, const double *z, const double *v,
                     ptgo_counter *ctr, const double *warm_value, const double *warm_grad,
                     double *z_out, double *value_out, double *grad_out) {
    if (level < 0 || level >= h->depth) return fail(PTGO_CONFIG, "mgoptCycle: bad level");
    shifted_t st;
    ptgo_counted obj = level_objective(h, level, &st, v);
    const size_t len = obj.len;
    if (level == h->depth - 1) {
        ptgo_solver_cfg cfg = smoother_cfg(h, level);
        cfg.max_iters = h->coarsest_iters;
        return ptgo_lbfgs(&obj, z, &cfg, ctr, warm_value, warm_grad, z_out, value_out, grad_out, NULL);
    }
    const int nH = h->levels[level + 1].prob.n;
    const size_t lenH = (size_t)nH * nH;
    const size_t b = sizeof(double) * 2 * len, bH = sizeof(double) * 2 * lenH;
    double *zbar = malloc(b), *gbar = malloc(b), *gfine = malloc(b), *corr = malloc(b);
    double *zplus = malloc(b), *gplus = malloc(b);
    double *zBarH = malloc(bH), *vH = malloc(bH), *cg = malloc(bH), *tmpH = malloc(bH);
    double *zrec = malloc(bH), *grec = malloc(bH), *cgs = malloc(bH);
    int rc = PTGO_OK;
    if (!zbar || !gbar || !gfine || !corr || !zplus || !gplus || !zBarH || !vH || !cg || !tmpH ||
        !zrec || !grec || !cgs) { rc = fail(PTGO_NOMEM, "mgoptCycle: out of memory"); goto done; }

    ptgo_solver_cfg pre = smoother_cfg(h, level);
    pre.max_iters = h->opt.k1;
    double vbar;
    if ((rc = ptgo_lbfgs(&obj, z, &pre, ctr, warm_value, warm_grad, zbar, &vbar, gbar, NULL))) goto done;

    if ((rc = ptgo_restrict_field(zbar, st.p->n, zBarH))) goto done;
    memcpy(gfine, gbar, b);
    axpy(gfine, 1.0, v, len);   /* plain gradient = shifted + v */
    shifted_t stc;
    ptgo_counted coarse_plain = level_objective(h, level + 1, &stc, NULL);
    double cval;
    if ((rc = counted_eval(&coarse_plain, ctr, zBarH, &cval, cg))) goto done;
    if ((rc = ptgo_restrict_field(v, st.p->n, vH))) goto done;
    axpy(vH, 1.0, cg, lenH);
    if ((rc = ptgo_restrict_field(gfine, st.p->n, tmpH))) goto done;
    axpy(vH, -1.0, tmpH, lenH);

    const double cs_val = cval - ptgo_dot_real(vH, zBarH, lenH);
    memcpy(cgs, cg, bH);
    axpy(cgs, -1.0, vH, lenH);

    double rval;
    if ((rc = ptgo_mgopt_cycle(h, level + 1, zBarH, vH, ctr, &cs_val, cgs, zrec, &rval, grec))) goto done;

    sub_into(tmpH, zrec, zBarH, lenH);
    if ((rc = ptgo_prolong_field(tmpH, nH, corr))) goto done;
    double alpha, pval;
    int stalled, trials;
    if ((rc = ptgo_linesearch(&obj, zbar, corr, ctr, h->opt.linesearch_max, &vbar, &alpha, &stalled,
                              &trials, zplus, &pval, gplus))) goto done;
    if (stalled) {
        memcpy(zplus, zbar, b);
        memcpy(gplus, gbar, b);
        pval = vbar;
    }
    ptgo_solver_cfg post = smoother_cfg(h, level);
    post.max_iters = h->opt.k2;
    rc = ptgo_lbfgs(&obj, zplus, &post, ctr, &pval, gplus, z_out, value_out, grad_out, NULL);
done:
    free(zbar); free(gbar); free(gfine); free(corr); free(zplus); free(gplus);
    free(zBarH); free(vH); free(cg); free(tmpH); free(zrec); free(grec); free(cgs);
    return rc;
}

/* multigrid.cpp:171-227 */
int ptgo_mgopt_driver(const ptgo_hierarchy *h, const double *z0, const ptgo_driver_cfg *cfg,
                      ptgo_counter *ctr, double *z_out, double *value_out, double *grad_out,
                      ptgo_report *rep) {
    if (h->depth < 1) return fail(PTGO_CONFIG, "mgoptDriver: empty hierarchy");
    const size_t len = (size_t)h->levels[0].prob.n * h->levels[0].prob.n;
    const size_t b = sizeof(double) * 2 * len;
    shifted_t st;
    if (h->depth == 1) {
        ptgo_solver_cfg base;
        ptgo_solver_cfg_default(&base);
        base.grad_tol_rel = cfg->grad_tol_rel;
        base.grad_tol_abs = cfg->grad_tol_abs;
        base.lbfgs_memory = h->opt.lbfgs_memory;
        base.linesearch_max = h->opt.linesearch_max;
        base.max_weighted = cfg->budget;
        base.max_iters = cfg->max_cycles;
        ptgo_counted top = level_objective(h, 0, &st, NULL);
        return ptgo_lbfgs(&top, z0, &base, ctr, NULL, NULL, z_out, value_out, grad_out, rep);
    }
    ptgo_counted top = level_objective(h, 0, &st, NULL);
    double *z = malloc(b), *g = malloc(b), *nz = malloc(b), *ng = malloc(b), *vzero = xcalloc(2 * len, sizeof(double));
    int rc = PTGO_OK;
    if (!z || !g || !nz || !ng || !vzero) { rc = fail(PTGO_NOMEM, "mgoptDriver: out of memory"); goto done; }
    memcpy(z, z0, b);
    double cur;
    if ((rc = counted_eval(&top, ctr, z, &cur, g))) goto done;
    if (!all_finite(g, len)) { rc = fail(PTGO_NUMERIC, "non-finite gradient in mgoptDriver"); goto done; }
    const double g0 = norm2(g, len);
    const double grad_floor = cfg->grad_tol_abs * (1.0 + norm2(z0, len));
    double gnorm = g0;
    if ((rc = push_hist(rep, ctr->weighted, cur, gnorm))) goto done;
    int reason = PTGO_STOP_MAXITERS;
    if (gnorm <= fmax(cfg->grad_tol_rel * g0, grad_floor)) {
        reason = PTGO_STOP_TOLERANCE;
    } else {
        for (int cycle = 1; cycle <= cfg->max_cycles; ++cycle) {
            double nval;
            if ((rc = ptgo_mgopt_cycle(h, 0, z, vzero, ctr, &cur, g, nz, &nval, ng))) goto done;
            memcpy(z, nz, b);
            memcpy(g, ng, b);
            cur = nval;
            gnorm = norm2(g, len);
            if ((rc = push_hist(rep, ctr->weighted, cur, gnorm))) goto done;
            if (gnorm <= fmax(cfg->grad_tol_rel * g0, grad_floor)) { reason = PTGO_STOP_TOLERANCE; break; }
            if (ctr->weighted >= cfg->budget) { reason = PTGO_STOP_BUDGET; break; }
        }
    }
    if (rep) rep->reason = reason;
    memcpy(z_out, z, b);
    if (value_out) *value_out = cur;
    if (grad_out) memcpy(grad_out, g, b);
done:
    free(z); free(g); free(nz); free(ng); free(vzero);
    return rc;
}

/* ------------------------------------------------------------------ noise */
/* Philox4x64-10 (Salmon et al., SC'11; the bit generator of
 * numpy.random.Philox): counter c, key k -> 4 x 64-bit words. */
void ptgo_philox4x64(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
    uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3], k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        const unsigned __int128 p0 = (unsigned __int128)M0 * c0, p1 = (unsigned __int128)M1 * c2;
        const uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
        const uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += W0;
        k1 += W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static double u01(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }   /* rng.hpp:14-16 */

static double gauss_at(size_t i, int j, uint64_t seed, const double *uni, size_t mm) {
    double u1, u2;
    if (uni) {
        u1 = uni[2 * ((size_t)j * mm + i)];
        u2 = uni[2 * ((size_t)j * mm + i) + 1];
    } else {
        const uint64_t c[4] = {(uint64_t)i, (uint64_t)j, 1, 0}, k[2] = {seed, 0};
        uint64_t r[4];
        ptgo_philox4x64(c, k, r);
        u1 = u01(r[0]);
        u2 = u01(r[1]);
    }
    const double rr = sqrt(-2.0 * log(1.0 - u1));   /* rng::gaussian, rng.hpp:18-24 */
    return rr * cos(6.283185307179586476925286766559 * u2);
}

/* addNoise (forward.cpp:56-86): per pattern eps = level ||d|| / ||g|| g,
 * out = max(d + eps, 0).  uni = NULL: Philox uniforms (the GPU's stream);
 * otherwise 2 N mm uniforms in the reference's draw order. */
int ptgo_add_noise(int N, size_t mm, const double *d, double level, uint64_t seed, const double *uni,
                   double *out) {
    if (level < 0.0) return fail(PTGO_DOMAIN, "noise level must be non-negative");
    for (int j = 0; j < N; ++j) {
        const double *dj = d + (size_t)j * mm;
        double dsq = 0.0, gsq = 0.0;
        for (size_t i = 0; i < mm; ++i) {
            const double g = gauss_at(i, j, seed, uni, mm);
            dsq += dj[i] * dj[i];
            gsq += g * g;
        }
        const double scale = gsq > 0.0 ? level * sqrt(dsq) / sqrt(gsq) : 0.0;
        for (size_t i = 0; i < mm; ++i) {
            const double v = dj[i] + gauss_at(i, j, seed, uni, mm) * scale;
            out[(size_t)j * mm + i] = v > 0.0 ? v : 0.0;
        }
    }
    return PTGO_OK;
}

typedef struct { uint64_t i, j, seed, b; uint64_t r[4]; int k; } ustream;
static double us_next(ustream *s) {
    if (s->k == 4) {
        const uint64_t c[4] = {s->i, s->j, 2, s->b++}, key[2] = {s->seed, 0};
        ptgo_philox4x64(c, key, s->r);
        s->k = 0;
    }
    return u01(s->r[s->k++]);
}

/* Poisson(lam): inversion below 10, Hormann's PTRS above (the GPU's sampler) */
static double poisson_sample(double lam, ustream *us) {
    if (!(lam > 0.0)) return 0.0;
    if (lam < 10.0) {
        const double u = us_next(us);
        double p = exp(-lam), F = p;
        int k = 0;
        while (u > F && k < 1000) { ++k; p *= lam / k; F += p; }
        return (double)k;
    }
    const double slam = sqrt(lam), loglam = log(lam);
    const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
    const double invalpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2.0);
    for (int it = 0; it < 10000; ++it) {
        const double U = us_next(us) - 0.5, V = us_next(us);
        const double usv = 0.5 - fabs(U);
        const double k = floor((2.0 * a / usv + b) * U + lam + 0.43);
        if (usv >= 0.07 && V <= vr) return k;
        if (k < 0.0 || (usv < 0.013 && V > usv)) continue;
        if (log(V) + log(invalpha) - log(a / (usv * usv) + b) <= -lam + k * loglam - lgamma(k + 1.0)) return k;
    }
    return floor(lam);
}

/* Poisson photon noise at `photons` per pattern: out = k / scale */
int ptgo_add_poisson(int N, size_t mm, const double *d, double photons, uint64_t seed, double *out) {
    if (!(photons > 0.0)) return fail(PTGO_DOMAIN, "photon budget must be positive");
    for (int j = 0; j < N; ++j) {
        const double *dj = d + (size_t)j * mm;
        double tot = 0.0;
        for (size_t i = 0; i < mm; ++i) tot += dj[i];
        const double scale = tot > 0.0 ? photons / tot : 0.0;
        for (size_t i = 0; i < mm; ++i) {
            double v = 0.0;
            if (scale > 0.0) {
                ustream us = {(uint64_t)i, (uint64_t)j, seed, 0, {0, 0, 0, 0}, 4};
                v = poisson_sample(dj[i] * scale, &us) / scale;
            }
            out[(size_t)j * mm + i] = v;
        }
    }
    return PTGO_OK;
}
