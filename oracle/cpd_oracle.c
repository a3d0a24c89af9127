/* C restatement of the reference CP-ALS-QR hot path -- the CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY (see cpd_oracle.h).  Each routine restates the
 * reference algorithm with the same floating-point operation order, so that
 * with -ffp-contract=off it is bit-identical to the reference compiled from
 * /root/reference (oracle/_ref).  Citations: file:line under
 * /root/reference/proj/include/cpd.
 */
#define _POSIX_C_SOURCE 200809L
#include "cpd_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <pthread.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

static char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* cpdo_last_error(void) { return g_err; }

static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz);
    if (!p) {
        fprintf(stderr, "cpd_oracle: out of memory (%zu x %zu)\n", n, sz);
        abort();
    }
    return p;
}

static double* dupd(const double* src, size_t n) {
    double* p = (double*)xcalloc(n, sizeof(double));
    memcpy(p, src, n * sizeof(double));
    return p;
}

/* ---------------------------------------------------------------- rng.hpp:15-70
 * splitmix64 expands the seed into the xoshiro256++ state; normals come from
 * the Marsaglia polar method with the second variate cached. */
static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void cpdo_rng_seed(cpdo_rng* g, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) {
        x += 0x9E3779B97F4A7C15ULL;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        g->s[i] = z ^ (z >> 31);
    }
    g->spare = 0.0;
    g->has_spare = 0;
}

uint64_t cpdo_rng_u64(cpdo_rng* g) {
    uint64_t* s = g->s;
    const uint64_t out = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
}

double cpdo_rng_uniform(cpdo_rng* g) { return (double)(cpdo_rng_u64(g) >> 11) * 0x1.0p-53; }

double cpdo_rng_normal(cpdo_rng* g) {
    if (g->has_spare) {
        g->has_spare = 0;
        return g->spare;
    }
    double u, v, s;
    do {
        u = 2.0 * cpdo_rng_uniform(g) - 1.0;
        v = 2.0 * cpdo_rng_uniform(g) - 1.0;
        s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    const double m = sqrt(-2.0 * log(s) / s);
    g->spare = v * m;
    g->has_spare = 1;
    return u * m;
}

int cpdo_rng_normals(uint64_t seed, uint64_t n, double* out) {
    cpdo_rng g;
    cpdo_rng_seed(&g, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = cpdo_rng_normal(&g);
    return CPDO_OK;
}

/* ------------------------------------------------------- dense tensor kernels */

static uint64_t prod(const uint64_t* d, uint32_t from, uint32_t to) {
    uint64_t p = 1;
    for (uint32_t k = from; k < to; ++k) p *= d[k];
    return p;
}

/* Static parallel-for over [0, n) on host threads (CPDO_THREADS, default: the
 * online cores).  The oracle splits OUTPUT elements between threads only:
 * every element keeps the reference's operation order, so the result is
 * bit-identical to the serial loops (tests/test_oracle.py checks it against
 * oracle/_ref). */
typedef void (*range_fn)(void* ctx, uint64_t begin, uint64_t end);
typedef struct {
    range_fn fn;
    void* ctx;
    uint64_t begin, end;
} range_job;

static void* range_run(void* p) {
    range_job* j = (range_job*)p;
    j->fn(j->ctx, j->begin, j->end);
    return NULL;
}

static int oracle_threads(void) {
    static int n = 0;
    if (n == 0) {
        const char* e = getenv("CPDO_THREADS");
        n = e ? atoi(e) : (int)sysconf(_SC_NPROCESSORS_ONLN);
        if (n < 1) n = 1;
        if (n > 64) n = 64;
    }
    return n;
}

static void par_for(uint64_t n, uint64_t min_per_thread, range_fn fn, void* ctx) {
    int nt = oracle_threads();
    if ((uint64_t)nt > n / (min_per_thread ? min_per_thread : 1)) nt = (int)(n / (min_per_thread ? min_per_thread : 1));
    if (nt <= 1) {
        fn(ctx, 0, n);
        return;
    }
    pthread_t th[64];
    range_job jobs[64];
    for (int t = 0; t < nt; ++t) {
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].begin = n * (uint64_t)t / (uint64_t)nt;
        jobs[t].end = n * (uint64_t)(t + 1) / (uint64_t)nt;
    }
    for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, range_run, &jobs[t]);
    range_run(&jobs[0]);
    for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
}

/* tensor.hpp:288-315 with the loops of detail::gemm (:137-149) and
 * detail::gemm_bt (:153-165): every output element accumulates its K products
 * in ascending contraction index, starting from +0. */
typedef struct {
    const double *t, *b;
    double* out;
    uint64_t outer, inner, ext, rows, jc, nj;
} ttm_ctx;

static void ttm_rows_range(void* p, uint64_t i0, uint64_t i1) { /* gemm_bt, tensor.hpp:153-165 */
    const ttm_ctx* c = (const ttm_ctx*)p;
    for (uint64_t i = i0; i < i1; ++i) {
        const double* xrow = c->t + i * c->ext;
        for (uint64_t r = 0; r < c->rows; ++r) {
            const double* brow = c->b + r * c->ext;
            double acc = 0.0;
            for (uint64_t k = 0; k < c->ext; ++k) acc += xrow[k] * brow[k];
            c->out[i * c->rows + r] = acc;
        }
    }
}

static void ttm_items_range(void* p, uint64_t a, uint64_t z) { /* gemm, tensor.hpp:137-149 */
    const ttm_ctx* c = (const ttm_ctx*)p;
    /* item = (o, j-chunk): the rows x chunk block of Y stays in cache while
     * the slab X[o][:][chunk] streams once (the reference's r-outer loop
     * would re-read it per r); each Y element still sums over k ascending */
    for (uint64_t it = a; it < z; ++it) {
        const uint64_t o = it / c->nj;
        const uint64_t j0 = (it % c->nj) * c->jc;
        const uint64_t j1 = j0 + c->jc < c->inner ? j0 + c->jc : c->inner;
        const double* xs = c->t + o * c->ext * c->inner;
        double* ys = c->out + o * c->rows * c->inner;
        for (uint64_t r = 0; r < c->rows; ++r)
            for (uint64_t j = j0; j < j1; ++j) ys[r * c->inner + j] = 0.0;
        for (uint64_t k = 0; k < c->ext; ++k) {
            const double* xrow = xs + k * c->inner;
            for (uint64_t r = 0; r < c->rows; ++r) {
                const double w = c->b[r * c->ext + k];
                double* yrow = ys + r * c->inner;
                for (uint64_t j = j0; j < j1; ++j) yrow[j] += w * xrow[j];
            }
        }
    }
}

/* Every output element accumulates its ext products in ascending contraction
 * index from +0 (the reference's order); work items are (o, j-chunk) so a
 * contraction of the leading mode (outer == 1) still spreads. */
static void ttm_raw(const double* t, const uint64_t* dims, uint32_t order, const double* b,
                    uint64_t rows, uint32_t mode, double* out) {
    ttm_ctx c;
    c.t = t;
    c.b = b;
    c.out = out;
    c.outer = prod(dims, 0, mode);
    c.inner = prod(dims, mode + 1, order);
    c.ext = dims[mode];
    c.rows = rows;
    c.jc = 256;
    c.nj = (c.inner + c.jc - 1) / c.jc;
    if (c.inner == 1) {
        par_for(c.outer, 256, ttm_rows_range, &c);
        return;
    }
    par_for(c.outer * c.nj, 4, ttm_items_range, &c);
}

int cpdo_ttm(const double* t, const uint64_t* dims, uint32_t order, const double* b,
             uint64_t b_rows, uint32_t mode, double* out) {
    if (mode >= order) return fail(CPDO_INVALID_ARGUMENT, "ttm: mode out of range");
    ttm_raw(t, dims, order, b, b_rows, mode, out);
    return CPDO_OK;
}

/* tensor.hpp:217-250: row = index of `mode`; column runs over the other modes
 * with the EARLIEST mode fastest.  (A permutation: threads take ranges of
 * the input, the column index is updated incrementally.) */
typedef struct {
    const double* t;
    double* out;
    const uint64_t* dims;
    uint64_t weight[CPDO_MAX_ORDER];
    uint64_t cols;
    uint32_t order, mode;
} unfold_ctx;

static void unfold_range(void* p, uint64_t lin0, uint64_t lin1) {
    const unfold_ctx* c = (const unfold_ctx*)p;
    uint64_t idx[CPDO_MAX_ORDER] = {0}, rem = lin0, col = 0;
    for (uint32_t k = c->order; k-- > 0;) {
        idx[k] = rem % c->dims[k];
        rem /= c->dims[k];
        if (k != c->mode) col += idx[k] * c->weight[k];
    }
    for (uint64_t lin = lin0; lin < lin1; ++lin) {
        c->out[idx[c->mode] * c->cols + col] = c->t[lin];
        for (uint32_t k = c->order; k-- > 0;) {
            const uint64_t w = k == c->mode ? 0 : c->weight[k];
            if (++idx[k] < c->dims[k]) {
                col += w;
                break;
            }
            col -= (c->dims[k] - 1) * w;
            idx[k] = 0;
        }
    }
}

int cpdo_unfold(const double* t, const uint64_t* dims, uint32_t order, uint32_t mode,
                double* out) {
    if (mode >= order) return fail(CPDO_INVALID_ARGUMENT, "unfold: mode out of range");
    unfold_ctx c;
    memset(&c, 0, sizeof c);
    c.t = t;
    c.out = out;
    c.dims = dims;
    c.order = order;
    c.mode = mode;
    const uint64_t total = prod(dims, 0, order);
    c.cols = total / dims[mode];
    uint64_t w = 1;
    for (uint32_t k = 0; k < order; ++k)
        if (k != mode) {
            c.weight[k] = w;
            w *= dims[k];
        }
    par_for(total, 1u << 16, unfold_range, &c);
    return CPDO_OK;
}

/* tensor.hpp:343-368: fold left to right, out(i*K + r, j) = acc(i, j) * m(r, j) */
int cpdo_khatri_rao(const double* const* mats, const uint64_t* rows, uint32_t count, uint64_t cols,
                    double* out) {
    if (count == 0) return fail(CPDO_INVALID_ARGUMENT, "khatri_rao: empty list");
    uint64_t cur_rows = rows[0], total = 1;
    for (uint32_t i = 0; i < count; ++i) total *= rows[i];
    double* cur = dupd(mats[0], rows[0] * cols);
    for (uint32_t li = 1; li < count; ++li) {
        const double* m = mats[li];
        const uint64_t mr = rows[li];
        double* next = (double*)xcalloc(cur_rows * mr * cols, sizeof(double));
        for (uint64_t i = 0; i < cur_rows; ++i)
            for (uint64_t r = 0; r < mr; ++r)
                for (uint64_t j = 0; j < cols; ++j)
                    next[(i * mr + r) * cols + j] = cur[i * cols + j] * m[r * cols + j];
        free(cur);
        cur = next;
        cur_rows *= mr;
    }
    memcpy(out, cur, total * cols * sizeof(double));
    free(cur);
    return CPDO_OK;
}

/* linalg.hpp:39-99: Householder with alpha = -sign(x_k) ||x||, Q accumulated
 * backwards from the first n columns of I, then rows of R / columns of Q
 * flipped so diag(R) >= 0.  A zero column leaves its reflector empty. */
/* out (cols x rows) = in (rows x cols)^T, tiled, threads over row tiles */
typedef struct {
    const double* in;
    double* out;
    uint64_t rows, cols;
} tp_ctx;

static void tp_range(void* p, uint64_t t0, uint64_t t1) {
    const tp_ctx* c = (const tp_ctx*)p;
    for (uint64_t t = t0; t < t1; ++t) {
        const uint64_t i0 = t * 64, i1 = i0 + 64 < c->rows ? i0 + 64 : c->rows;
        for (uint64_t j0 = 0; j0 < c->cols; j0 += 64) {
            const uint64_t j1 = j0 + 64 < c->cols ? j0 + 64 : c->cols;
            for (uint64_t i = i0; i < i1; ++i)
                for (uint64_t j = j0; j < j1; ++j) c->out[j * c->rows + i] = c->in[i * c->cols + j];
        }
    }
}

static void transpose_par(const double* in, uint64_t rows, uint64_t cols, double* out) {
    tp_ctx c = {in, out, rows, cols};
    par_for((rows + 63) / 64, 64, tp_range, &c);
}

/* The QR works on a COLUMN-MAJOR copy: each column is contiguous, so the
 * column loop of linalg.hpp:62-67 (s_j = beta * sum_i v_i w_ij ascending in
 * i, then w_ij -= s_j v_i) streams one contiguous column per j, and threads
 * take disjoint columns.  Same operations in the same order per column ->
 * bit-identical to the reference (tests/test_oracle.py checks it). */
typedef struct {
    double* wt; /* n columns of length m */
    const double* v;
    uint64_t m, k, j_lo;
    double beta;
} refl_ctx;

static void refl_range(void* p, uint64_t c0, uint64_t c1) {
    const refl_ctx* c = (const refl_ctx*)p;
    for (uint64_t jj = c0; jj < c1; ++jj) {
        double* col = c->wt + (c->j_lo + jj) * c->m;
        const double* v = c->v - c->k;  /* v[i] for i >= k */
        double s = 0.0;
        for (uint64_t i = c->k; i < c->m; ++i) s += v[i] * col[i];
        s *= c->beta;
        for (uint64_t i = c->k; i < c->m; ++i) col[i] -= s * v[i];
    }
}

static void apply_reflector(double* wt, uint64_t m, uint64_t n, uint64_t k, uint64_t j_lo,
                            const double* v, double beta) {
    refl_ctx c = {wt, v, m, k, j_lo, beta};
    par_for(n - j_lo, (m - k) > (1u << 14) ? 1 : (uint64_t)-1, refl_range, &c);
}

/* linalg.hpp:39-99: Householder with alpha = -sign(x_k) ||x||, Q accumulated
 * backwards from the first n columns of I, then rows of R / columns of Q
 * flipped so diag(R) >= 0.  A zero column leaves its reflector empty. */
int cpdo_thin_qr(const double* a, uint64_t m, uint64_t n, double* q, double* r) {
    if (m < n) return fail(CPDO_INVALID_ARGUMENT, "thin_qr: requires rows >= cols");
    double* wt = (double*)xcalloc(m * n, sizeof(double)); /* column-major work */
    transpose_par(a, m, n, wt);
    double* refl = (double*)xcalloc(m * n, sizeof(double)); /* column k: v in rows k.. */
    double* beta = (double*)xcalloc(n, sizeof(double));
    char* has = (char*)xcalloc(n, 1);
    for (uint64_t k = 0; k < n; ++k) {
        const double* ck = wt + k * m;
        double nsq = 0.0;
        for (uint64_t i = k; i < m; ++i) nsq += ck[i] * ck[i];
        const double nrm = sqrt(nsq);
        if (nrm == 0.0) continue;
        const double alpha = ck[k] >= 0.0 ? -nrm : nrm;
        double* v = refl + k * m; /* v[0..m-k) */
        v[0] = ck[k] - alpha;
        for (uint64_t i = k + 1; i < m; ++i) v[i - k] = ck[i];
        double vsq = 0.0;
        for (uint64_t i = 0; i < m - k; ++i) vsq += v[i] * v[i];
        const double bt = 2.0 / vsq;
        apply_reflector(wt, m, n, k, k, v, bt);
        wt[k * m + k] = alpha;
        beta[k] = bt;
        has[k] = 1;
    }
    memset(r, 0, n * n * sizeof(double));
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = i; j < n; ++j) r[i * n + j] = wt[j * m + i];
    double* qt = wt; /* reuse: Q column-major */
    memset(qt, 0, m * n * sizeof(double));
    for (uint64_t j = 0; j < n; ++j) qt[j * m + j] = 1.0;
    for (uint64_t k = n; k-- > 0;) {
        if (!has[k]) continue;
        apply_reflector(qt, m, n, k, 0, refl + k * m, beta[k]);
    }
    for (uint64_t k = 0; k < n; ++k)
        if (r[k * n + k] < 0.0) {
            for (uint64_t j = k; j < n; ++j) r[k * n + j] = -r[k * n + j];
            for (uint64_t i = 0; i < m; ++i) qt[k * m + i] = -qt[k * m + i];
        }
    transpose_par(qt, n, m, q);
    free(wt);
    free(refl);
    free(beta);
    free(has);
    return CPDO_OK;
}

/* linalg.hpp:192-216 */
int cpdo_solve_rows_lower(const double* l, uint64_t n, const double* rhs, uint64_t rows,
                          double* out, int64_t* bad_column) {
    if (bad_column) *bad_column = -1;
    double maxd = 0.0;
    for (uint64_t i = 0; i < n; ++i) maxd = fmax(maxd, fabs(l[i * n + i]));
    const double tau = 1e-14 * maxd;
    for (uint64_t i = 0; i < n; ++i)
        if (fabs(l[i * n + i]) <= tau) {
            if (bad_column) *bad_column = (int64_t)i;
            return fail(CPDO_SINGULAR_TRIANGULAR,
                        "triangular solve: diagonal entry of column %llu is %g",
                        (unsigned long long)i, l[i * n + i]);
        }
    memcpy(out, rhs, rows * n * sizeof(double));
    for (uint64_t row = 0; row < rows; ++row) {
        double* x = out + row * n;
        for (uint64_t c = n; c-- > 0;) {
            double s = x[c];
            for (uint64_t j = c + 1; j < n; ++j) s -= x[j] * l[j * n + c];
            x[c] = s / l[c * n + c];
        }
    }
    return CPDO_OK;
}

/* linalg.hpp:225-242 */
int cpdo_normalize_columns(const double* a, uint64_t m, uint64_t n, double* out, double* weights) {
    if (out != a) memcpy(out, a, m * n * sizeof(double));
    for (uint64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (uint64_t i = 0; i < m; ++i) s += out[i * n + j] * out[i * n + j];
        const double nrm = sqrt(s);
        if (nrm < 1e-300) {
            for (uint64_t i = 0; i < m; ++i) out[i * n + j] = 0.0;
            out[j] = 1.0;
            weights[j] = 0.0;
        } else {
            for (uint64_t i = 0; i < m; ++i) out[i * n + j] /= nrm;
            weights[j] = nrm;
        }
    }
    return CPDO_OK;
}

/* solvers.hpp:75-86 */
int cpdo_extrapolate_q0(const double* now, const double* prev, uint64_t rows, uint64_t cols,
                        double beta, double alpha, double* out) {
    const uint64_t n = rows * cols;
    if (beta == 0.0) {
        memcpy(out, now, n * sizeof(double));
        return CPDO_OK;
    }
    for (uint64_t i = 0; i < n; ++i) out[i] = now[i] + beta * (now[i] - alpha * prev[i]);
    return CPDO_OK;
}

/* solvers.hpp:92-101 */
int cpdo_select_beta(double prev, double now, double gap, double* beta) {
    const double p = prev < 0.0 ? 0.0 : (prev > 1.0 ? 1.0 : prev);
    const double c = now < 0.0 ? 0.0 : (now > 1.0 ? 1.0 : now);
    *beta = 0.0;
    if (fabs(c - p) >= gap) return 0;
    *beta = c > 0.90 ? 1.0 / 2000.0 : (c >= 0.70 ? 1.0 / 500.0 : 1.0 / 250.0);
    return 1;
}

/* kruskal.hpp:109-128, with matmul/gram/dot in the loop orders of
 * tensor.hpp:137-211. */
int cpdo_fitness_fast_qr(double nx2, const double* v, const double* ah, uint64_t rows,
                         const double* r0, const double* rn, const double* lam, uint64_t r,
                         double* fitness, double* raw) {
    if (!(nx2 > 0.0)) return fail(CPDO_INVALID_ARGUMENT, "fitness_fast_qr: zero-norm tensor");
    double* c = (double*)xcalloc(rows * r, sizeof(double));
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t p = 0; p < r; ++p) {
            const double av = ah[i * r + p];
            for (uint64_t j = 0; j < r; ++j) c[i * r + j] += av * r0[j * r + p];
        }
    double xk = 0.0;
    for (uint64_t i = 0; i < rows * r; ++i) xk += v[i] * c[i];
    free(c);
    double* g0 = (double*)xcalloc(r * r, sizeof(double));
    double* gn = (double*)xcalloc(r * r, sizeof(double));
    for (uint64_t p = 0; p < r; ++p)
        for (uint64_t i = 0; i < r; ++i) {
            const double a0 = r0[p * r + i], an = rn[p * r + i];
            for (uint64_t j = 0; j < r; ++j) {
                g0[i * r + j] += a0 * r0[p * r + j];
                gn[i * r + j] += an * rn[p * r + j];
            }
        }
    double kk = 0.0;
    for (uint64_t i = 0; i < r; ++i)
        for (uint64_t j = 0; j < r; ++j) kk += g0[i * r + j] * lam[i] * gn[i * r + j] * lam[j];
    free(g0);
    free(gn);
    const double rw = nx2 - 2.0 * xk + kk;
    const double rad = rw < 0.0 ? 0.0 : rw;
    *fitness = 1.0 - sqrt(rad) / sqrt(nx2);
    *raw = rw;
    return CPDO_OK;
}

/* ------------------------------------------------------------ schedules
 * dim_tree.hpp:191-426.  A plan is a list of updates; an update is a mode and
 * a chain of (source set, contracted mode) steps.  The fixed plans are written
 * as tables: per update {mode, nsteps, (source, contract)...}, source == 0xFF
 * meaning the root (full set). */

#define MAXSTEPS 8
typedef struct {
    uint32_t source, contract, produces;
} step_t;
typedef struct {
    uint32_t mode, nsteps;
    step_t steps[MAXSTEPS];
} update_t;
typedef struct {
    update_t u[CPDO_MAX_ORDER];
} iter_t;
typedef struct {
    uint32_t order;
    int32_t strategy;
    uint64_t n;
    uint64_t cycle_start, cycle_length;
    iter_t* it;
} sched_t;

#define ROOT 0xFFu

static uint32_t full_set(uint32_t order) { return (1u << order) - 1u; }

/* table rows: mode, nsteps, then nsteps pairs (source bitmask or ROOT, contract) */
static const int kDimTree3[] = {0, 2, ROOT, 2, 0x3, 1, 1, 1, 0x3, 0, 2, 2, ROOT, 1, 0x5, 0};
static const int kDimTree4[] = {0, 3, ROOT, 3, 0x7, 2, 0x3, 1, 1, 1, 0x3, 0,
                                2, 2, 0x7, 1, 0x5, 0, 3, 3, ROOT, 0, 0xE, 1, 0xC, 2};
static const int kReuse3b[] = {0, 1, 0x5, 2, 2, 1, 0x5, 0, 1, 2, ROOT, 0, 0x6, 2};
static const int kReuse3c[] = {1, 1, 0x6, 2, 2, 1, 0x6, 1, 0, 2, ROOT, 1, 0x5, 2};
static const int kReuse4b[] = {2, 1, 0xC, 3, 3, 1, 0xC, 2, 1, 2, 0xE, 2, 0xA, 3,
                               0, 3, ROOT, 1, 0xD, 2, 0x9, 3};
static const int kReuse4c[] = {0, 1, 0x9, 3, 2, 2, 0xD, 3, 0x5, 0, 3, 2, 0xD, 2, 0x9, 0,
                               1, 3, ROOT, 2, 0xB, 0, 0xA, 3};

static void iter_from_table(iter_t* it, uint32_t order, const int* t) {
    const uint32_t root = full_set(order);
    size_t p = 0;
    for (uint32_t b = 0; b < order; ++b) {
        update_t* u = &it->u[b];
        u->mode = (uint32_t)t[p++];
        u->nsteps = (uint32_t)t[p++];
        for (uint32_t s = 0; s < u->nsteps; ++s) {
            const uint32_t src = t[p] == (int)ROOT ? root : (uint32_t)t[p];
            const uint32_t c = (uint32_t)t[p + 1];
            p += 2;
            u->steps[s] = (step_t){src, c, src & ~(1u << c)};
        }
    }
}

/* dim_tree.hpp:210-238 */
static void naive_iter(iter_t* it, uint32_t order) {
    static const uint32_t t3[3][2] = {{2, 1}, {0, 2}, {1, 0}};
    static const uint32_t t4[4][3] = {{3, 2, 1}, {3, 2, 0}, {0, 1, 3}, {0, 1, 2}};
    for (uint32_t mode = 0; mode < order; ++mode) {
        uint32_t seq[CPDO_MAX_ORDER], ns = 0;
        if (order == 3)
            for (int i = 0; i < 2; ++i) seq[ns++] = t3[mode][i];
        else if (order == 4)
            for (int i = 0; i < 3; ++i) seq[ns++] = t4[mode][i];
        else
            for (uint32_t k = order; k-- > 0;)
                if (k != mode) seq[ns++] = k;
        update_t* u = &it->u[mode];
        u->mode = mode;
        u->nsteps = ns;
        uint32_t cur = full_set(order);
        for (uint32_t s = 0; s < ns; ++s) {
            u->steps[s] = (step_t){cur, seq[s], cur & ~(1u << seq[s])};
            cur = u->steps[s].produces;
        }
    }
}

static uint32_t permute_set(uint32_t set, const uint32_t* perm, uint32_t order) {
    uint32_t out = 0;
    for (uint32_t m = 0; m < order; ++m)
        if (set & (1u << m)) out |= 1u << perm[m];
    return out;
}

/* dim_tree.hpp:312-331 */
static void permute_iter(iter_t* dst, const iter_t* src, const uint32_t* perm, uint32_t order) {
    for (uint32_t b = 0; b < order; ++b) {
        const update_t* u = &src->u[b];
        update_t* v = &dst->u[b];
        v->mode = perm[u->mode];
        v->nsteps = u->nsteps;
        for (uint32_t s = 0; s < u->nsteps; ++s)
            v->steps[s] = (step_t){permute_set(u->steps[s].source, perm, order),
                                   perm[u->steps[s].contract],
                                   permute_set(u->steps[s].produces, perm, order)};
    }
}

/* dim_tree.hpp:335-379: structure + version simulation */
static int validate(const sched_t* s) {
    const uint32_t order = s->order, root = full_set(order);
    uint64_t version[CPDO_MAX_ORDER];
    for (uint32_t k = 0; k < order; ++k) version[k] = 1;
    /* stamps per produced set: stamp[set][mode], 0 = mode not absorbed */
    uint64_t (*stamp)[CPDO_MAX_ORDER] = xcalloc((size_t)1 << order, sizeof *stamp);
    char* avail = (char*)xcalloc((size_t)1 << order, 1);
    int rc = CPDO_OK;
    for (uint64_t i = 0; i < s->n && rc == CPDO_OK; ++i) {
        uint32_t seen = 0;
        for (uint32_t b = 0; b < order && rc == CPDO_OK; ++b) {
            const update_t* u = &s->it[i].u[b];
            if (u->mode >= order || (seen & (1u << u->mode))) {
                rc = fail(CPDO_LOGIC, "schedule: duplicate or out-of-range update mode");
                break;
            }
            seen |= 1u << u->mode;
            if (u->nsteps == 0 || u->steps[u->nsteps - 1].produces != (1u << u->mode)) {
                rc = fail(CPDO_LOGIC, "schedule: update must end in its final tensor");
                break;
            }
            for (uint32_t k = 0; k < u->nsteps; ++k) {
                const step_t* st = &u->steps[k];
                if (!(st->source & (1u << st->contract))) {
                    rc = fail(CPDO_LOGIC, "schedule: contract mode not free in source");
                    break;
                }
                if (st->produces != (st->source & ~(1u << st->contract))) {
                    rc = fail(CPDO_LOGIC, "schedule: produced set must drop the contracted mode");
                    break;
                }
                uint64_t cur[CPDO_MAX_ORDER] = {0};
                if (st->source != root) {
                    if (!avail[st->source]) {
                        rc = fail(CPDO_LOGIC, "schedule: source not available at iteration %llu",
                                  (unsigned long long)(i + 1));
                        break;
                    }
                    for (uint32_t m = 0; m < order; ++m)
                        if (stamp[st->source][m] && stamp[st->source][m] != version[m]) {
                            rc = fail(CPDO_STALE, "schedule: stale source at iteration %llu",
                                      (unsigned long long)(i + 1));
                            break;
                        }
                    if (rc) break;
                    memcpy(cur, stamp[st->source], sizeof cur);
                }
                cur[st->contract] = version[st->contract];
                if (st->produces != (1u << u->mode)) {
                    memcpy(stamp[st->produces], cur, sizeof cur);
                    avail[st->produces] = 1;
                }
            }
            ++version[u->mode];
        }
        if (rc == CPDO_OK && seen != full_set(order))
            rc = fail(CPDO_LOGIC, "schedule: iteration must update every mode exactly once");
    }
    free(stamp);
    free(avail);
    return rc;
}

/* dim_tree.hpp:386-426 */
static int build(sched_t* s, uint32_t order, int32_t strategy, uint64_t n) {
    memset(s, 0, sizeof *s);
    if (n == 0) return fail(CPDO_INVALID_ARGUMENT, "build_schedule: need at least one iteration");
    if (order < 2) return fail(CPDO_INVALID_ARGUMENT, "build_schedule: order must be >= 2");
    if (strategy < 0 || strategy > 2) return fail(CPDO_INVALID_ARGUMENT, "unknown strategy");
    if (strategy != 0 && order != 3 && order != 4)
        return fail(CPDO_INVALID_ARGUMENT,
                    "build_schedule: tree strategies are defined for orders 3 and 4 only");
    if (order > CPDO_MAX_ORDER) return fail(CPDO_INVALID_ARGUMENT, "build_schedule: order too large");
    s->order = order;
    s->strategy = strategy;
    s->n = n;
    s->cycle_start = 0;
    s->cycle_length = 1;
    s->it = (iter_t*)xcalloc(n, sizeof(iter_t));
    if (strategy == 0) {
        for (uint64_t i = 0; i < n; ++i) naive_iter(&s->it[i], order);
    } else if (strategy == 1) {
        for (uint64_t i = 0; i < n; ++i)
            iter_from_table(&s->it[i], order, order == 3 ? kDimTree3 : kDimTree4);
    } else if (order == 3) {
        s->cycle_start = 1;
        s->cycle_length = 2;
        iter_from_table(&s->it[0], 3, kDimTree3);
        if (n > 1) iter_from_table(&s->it[1], 3, kReuse3b);
        if (n > 2) iter_from_table(&s->it[2], 3, kReuse3c);
        for (uint64_t i = 3; i < n; ++i) s->it[i] = s->it[i - 2];
    } else {
        static const uint32_t sigma[4] = {1, 2, 0, 3};
        s->cycle_start = 2;
        s->cycle_length = 3;
        iter_from_table(&s->it[0], 4, kDimTree4);
        if (n > 1) iter_from_table(&s->it[1], 4, kReuse4b);
        if (n > 2) iter_from_table(&s->it[2], 4, kReuse4c);
        for (uint64_t i = 3; i < n; ++i) permute_iter(&s->it[i], &s->it[i - 1], sigma, 4);
    }
    return validate(s);
}

static void sched_free(sched_t* s) {
    free(s->it);
    s->it = NULL;
}

/* dim_tree.hpp:433-465 */
static uint32_t retained(const sched_t* s, uint64_t iter, uint32_t block, uint32_t* keys) {
    uint64_t next = iter + 1;
    if (next >= s->n) {
        if (next > s->cycle_start)
            next = s->cycle_start + (next - s->cycle_start) % s->cycle_length;
        if (next >= s->n) next = s->n - 1;
    }
    const iter_t* horizon[2] = {&s->it[iter], &s->it[next]};
    const uint32_t root = full_set(s->order);
    uint32_t nk = 0, over[2 * CPDO_MAX_ORDER * MAXSTEPS], no = 0;
    for (int h = 0; h < 2; ++h)
        for (uint32_t b = 0; b < s->order; ++b) {
            if (h == 0 && b <= block) continue;
            const update_t* u = &horizon[h]->u[b];
            for (uint32_t k = 0; k < u->nsteps; ++k) {
                const step_t* st = &u->steps[k];
                int was = 0;
                for (uint32_t o = 0; o < no; ++o) was |= over[o] == st->source;
                if (st->source != root && !was) keys[nk++] = st->source;
                over[no++] = st->produces;
            }
        }
    return nk;
}

int cpdo_schedule(uint32_t order, int32_t strategy, uint64_t iterations, int64_t* out,
                  uint64_t cap, uint64_t* n_steps, uint64_t* cycle) {
    sched_t s;
    int rc = build(&s, order, strategy, iterations);
    if (rc) {
        sched_free(&s);
        return rc;
    }
    uint64_t n = 0;
    for (uint64_t i = 0; i < s.n; ++i)
        for (uint32_t b = 0; b < order; ++b) {
            const update_t* u = &s.it[i].u[b];
            for (uint32_t k = 0; k < u->nsteps; ++k, ++n)
                if (n < cap) {
                    int64_t* row = out + 6 * n;
                    row[0] = (int64_t)i;
                    row[1] = b;
                    row[2] = u->mode;
                    row[3] = u->steps[k].source;
                    row[4] = u->steps[k].contract;
                    row[5] = u->steps[k].produces;
                }
        }
    *n_steps = n;
    cycle[0] = s.cycle_start;
    cycle[1] = s.cycle_length;
    sched_free(&s);
    return CPDO_OK;
}

int cpdo_retained_keys(uint32_t order, int32_t strategy, uint64_t iterations, uint64_t iter,
                       uint64_t block, uint32_t* out, uint64_t cap, uint64_t* n) {
    sched_t s;
    int rc = build(&s, order, strategy, iterations);
    if (rc) {
        sched_free(&s);
        return rc;
    }
    uint32_t keys[2 * CPDO_MAX_ORDER * MAXSTEPS];
    const uint32_t nk = retained(&s, iter, (uint32_t)block, keys);
    *n = nk;
    for (uint32_t i = 0; i < nk && i < cap; ++i) out[i] = keys[i];
    sched_free(&s);
    return CPDO_OK;
}

static void cost_of(const sched_t* s, const uint64_t* dims, uint64_t rank, uint64_t iters,
                    uint64_t* flops, uint64_t* roots) {
    const uint32_t root = full_set(s->order);
    *flops = 0;
    *roots = 0;
    for (uint64_t i = 0; i < iters && i < s->n; ++i)
        for (uint32_t b = 0; b < s->order; ++b) {
            const update_t* u = &s->it[i].u[b];
            for (uint32_t k = 0; k < u->nsteps; ++k) {
                const uint32_t src = u->steps[k].source;
                uint64_t f = 2;
                uint32_t pc = 0;
                for (uint32_t m = 0; m < s->order; ++m)
                    if (src & (1u << m)) {
                        f *= dims[m];
                        ++pc;
                    }
                for (uint32_t p = 0; p < s->order - pc + 1; ++p) f *= rank;
                *flops += f;
                if (src == root) ++*roots;
            }
        }
}

int cpdo_measured_cost(uint32_t order, int32_t strategy, const uint64_t* dims, uint64_t rank,
                       uint64_t iterations, uint64_t* total_flops, uint64_t* roots) {
    sched_t s;
    int rc = build(&s, order, strategy, iterations);
    if (rc == CPDO_OK) cost_of(&s, dims, rank, iterations, total_flops, roots);
    sched_free(&s);
    return rc;
}

/* ------------------------------------------------------- factor state + cache */

typedef struct {
    uint32_t order;
    uint64_t rank;
    uint64_t dims[CPDO_MAX_ORDER];
    double* a[CPDO_MAX_ORDER]; /* I_k x R factor */
    double* q[CPDO_MAX_ORDER]; /* I_k x R */
    double* r[CPDO_MAX_ORDER]; /* R x R */
    uint64_t version[CPDO_MAX_ORDER];
    double* lambda;
} fstate_t;

/* factor_state.hpp:42-47: re-QR and bump the version */
static void fs_update(fstate_t* f, uint32_t mode, const double* factor) {
    const uint64_t I = f->dims[mode], R = f->rank;
    memcpy(f->a[mode], factor, I * R * sizeof(double));
    cpdo_thin_qr(f->a[mode], I, R, f->q[mode], f->r[mode]);
    ++f->version[mode];
}

static void fs_init(fstate_t* f, uint32_t order, const uint64_t* dims, uint64_t R,
                    const double* factors) {
    memset(f, 0, sizeof *f);
    f->order = order;
    f->rank = R;
    const double* p = factors;
    for (uint32_t k = 0; k < order; ++k) {
        f->dims[k] = dims[k];
        f->a[k] = (double*)xcalloc(dims[k] * R, sizeof(double));
        f->q[k] = (double*)xcalloc(dims[k] * R, sizeof(double));
        f->r[k] = (double*)xcalloc(R * R, sizeof(double));
        f->version[k] = 0;
        fs_update(f, k, p); /* from_factors: version 1 (factor_state.hpp:28-34) */
        p += dims[k] * R;
    }
    f->lambda = (double*)xcalloc(R, sizeof(double));
    for (uint64_t j = 0; j < R; ++j) f->lambda[j] = 1.0;
}

static void fs_free(fstate_t* f) {
    for (uint32_t k = 0; k < f->order; ++k) {
        free(f->a[k]);
        free(f->q[k]);
        free(f->r[k]);
    }
    free(f->lambda);
}

typedef struct {
    int used;
    uint32_t key;
    uint64_t dims[CPDO_MAX_ORDER];
    uint64_t stamp[CPDO_MAX_ORDER]; /* 0 = mode not absorbed */
    double* data;
} centry_t;

typedef struct {
    centry_t e[64];
} cache_t;

static centry_t* cache_find(cache_t* c, uint32_t key) {
    for (int i = 0; i < 64; ++i)
        if (c->e[i].used && c->e[i].key == key) return &c->e[i];
    return NULL;
}

static void cache_put(cache_t* c, uint32_t key, double* data, const uint64_t* dims,
                      const uint64_t* stamp, uint32_t order) {
    centry_t* e = cache_find(c, key);
    if (!e)
        for (int i = 0; i < 64 && !e; ++i)
            if (!c->e[i].used) e = &c->e[i];
    if (!e) abort();
    if (e->used) free(e->data);
    e->used = 1;
    e->key = key;
    e->data = data;
    memcpy(e->dims, dims, order * sizeof(uint64_t));
    memcpy(e->stamp, stamp, CPDO_MAX_ORDER * sizeof(uint64_t));
}

static void cache_clear(cache_t* c) {
    for (int i = 0; i < 64; ++i)
        if (c->e[i].used) {
            free(c->e[i].data);
            c->e[i].used = 0;
        }
}

static void transpose(const double* a, uint64_t rows, uint64_t cols, double* t) {
    for (uint64_t i = 0; i < rows; ++i)
        for (uint64_t j = 0; j < cols; ++j) t[j * rows + i] = a[i * cols + j];
}

/* dim_tree.hpp:473-544.  Returns the final Y (malloc'd, dims in ydims) and
 * adds the TTM cost of the steps to *flops / *roots. */
static int execute(const sched_t* s, const double* x, const uint64_t* xdims, const fstate_t* st,
                   cache_t* cache, uint64_t iteration, uint32_t mode, double** y,
                   uint64_t* ydims, uint64_t* flops, uint64_t* roots) {
    const uint32_t order = s->order, root = full_set(order);
    const iter_t* it = &s->it[iteration];
    uint32_t block = order;
    for (uint32_t b = 0; b < order; ++b)
        if (it->u[b].mode == mode) {
            block = b;
            break;
        }
    if (block == order) return fail(CPDO_INVALID_ARGUMENT, "execute: mode not in iteration");
    const update_t* u = &it->u[block];
    *y = NULL;
    for (uint32_t k = 0; k < u->nsteps; ++k) {
        const step_t* sp = &u->steps[k];
        const double* src;
        uint64_t sd[CPDO_MAX_ORDER], stamp[CPDO_MAX_ORDER] = {0};
        if (sp->source == root) {
            src = x;
            memcpy(sd, xdims, order * sizeof(uint64_t));
        } else {
            centry_t* e = cache_find(cache, sp->source);
            if (!e)
                return fail(CPDO_LOGIC, "execute: scheduled source missing from cache");
            for (uint32_t m = 0; m < order; ++m)
                if (e->stamp[m] && e->stamp[m] != st->version[m])
                    return fail(CPDO_STALE,
                                "execute: stale intermediate (mode %u stamped v%llu, current "
                                "v%llu) at iteration %llu, update of mode %u",
                                m + 1, (unsigned long long)e->stamp[m],
                                (unsigned long long)st->version[m],
                                (unsigned long long)(iteration + 1), mode + 1);
            src = e->data;
            memcpy(sd, e->dims, order * sizeof(uint64_t));
            memcpy(stamp, e->stamp, sizeof stamp);
        }
        const uint32_t c = sp->contract;
        const uint64_t R = st->rank, ext = sd[c];
        double* qt = (double*)xcalloc(R * ext, sizeof(double));
        transpose(st->q[c], ext, R, qt);
        uint64_t od[CPDO_MAX_ORDER];
        memcpy(od, sd, order * sizeof(uint64_t));
        od[c] = R;
        const uint64_t n_out = prod(od, 0, order);
        double* out = (double*)xcalloc(n_out, sizeof(double));
        ttm_raw(src, sd, order, qt, R, c, out);
        free(qt);
        *flops += 2ull * n_out * ext;
        if (sp->source == root) ++*roots;
        stamp[c] = st->version[c];
        if (sp->produces == (1u << mode)) {
            free(*y);
            *y = out;
            memcpy(ydims, od, order * sizeof(uint64_t));
        } else {
            cache_put(cache, sp->produces, out, od, stamp, order);
        }
    }
    uint32_t keep[2 * CPDO_MAX_ORDER * MAXSTEPS];
    const uint32_t nk = retained(s, iteration, block, keep);
    for (int i = 0; i < 64; ++i) {
        centry_t* e = &cache->e[i];
        if (!e->used) continue;
        int needed = 0;
        for (uint32_t j = 0; j < nk; ++j) needed |= keep[j] == e->key;
        if (!needed) {
            free(e->data);
            e->used = 0;
        }
    }
    return CPDO_OK;
}

int cpdo_execute_run(const double* x, const uint64_t* dims, uint32_t order, uint64_t rank,
                     int32_t strategy, uint64_t iterations, uint64_t seed,
                     const double* init_factors, double* y_out, uint64_t* flops_out) {
    sched_t s;
    int rc = build(&s, order, strategy, iterations);
    if (rc) {
        sched_free(&s);
        return rc;
    }
    fstate_t st;
    fs_init(&st, order, dims, rank, init_factors);
    cache_t cache;
    memset(&cache, 0, sizeof cache);
    cpdo_rng g;
    cpdo_rng_seed(&g, seed);
    double* out = y_out;
    uint64_t nu = 0;
    for (uint64_t it = 0; it < iterations && rc == CPDO_OK; ++it)
        for (uint32_t b = 0; b < order && rc == CPDO_OK; ++b) {
            const uint32_t mode = s.it[it].u[b].mode;
            double* y = NULL;
            uint64_t yd[CPDO_MAX_ORDER], fl = 0, ro = 0;
            rc = execute(&s, x, dims, &st, &cache, it, mode, &y, yd, &fl, &ro);
            if (rc) break;
            const uint64_t ny = prod(yd, 0, order);
            memcpy(out, y, ny * sizeof(double));
            out += ny;
            free(y);
            if (flops_out) flops_out[nu] = fl;
            ++nu;
            const uint64_t I = dims[mode];
            double* m = (double*)xcalloc(I * rank, sizeof(double));
            double* w = (double*)xcalloc(rank, sizeof(double));
            for (uint64_t i = 0; i < I * rank; ++i) m[i] = cpdo_rng_normal(&g);
            cpdo_normalize_columns(m, I, rank, m, w);
            fs_update(&st, mode, m);
            free(m);
            free(w);
        }
    cache_clear(&cache);
    fs_free(&st);
    sched_free(&s);
    return rc;
}

/* ------------------------------------------------------------ the solver */

static double now_seconds(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* solvers.hpp:105-124: N(0,1) factors from Rng(seed), mode by mode, then
 * column normalisation */
static void initial_factors(uint32_t order, const uint64_t* dims, uint64_t R, uint64_t seed,
                            double* out) {
    cpdo_rng g;
    cpdo_rng_seed(&g, seed);
    double* p = out;
    double* w = (double*)xcalloc(R, sizeof(double));
    for (uint32_t k = 0; k < order; ++k) {
        for (uint64_t i = 0; i < dims[k] * R; ++i) p[i] = cpdo_rng_normal(&g);
        cpdo_normalize_columns(p, dims[k], R, p, w);
        p += dims[k] * R;
    }
    free(w);
}

/* X contracted with Q_k^T for every mode outside `key`, descending mode
 * order (cache warm-up on resume; freshness invariant dim_tree.hpp:109-111). */
static double* rebuild_entry(const double* x, const uint64_t* xdims, const fstate_t* st,
                             uint32_t key, uint64_t* odims) {
    const uint32_t order = st->order;
    uint64_t d[CPDO_MAX_ORDER];
    memcpy(d, xdims, order * sizeof(uint64_t));
    double* cur = dupd(x, prod(d, 0, order));
    for (uint32_t k = order; k-- > 0;) {
        if (key & (1u << k)) continue;
        double* qt = (double*)xcalloc(st->rank * d[k], sizeof(double));
        transpose(st->q[k], d[k], st->rank, qt);
        uint64_t nd[CPDO_MAX_ORDER];
        memcpy(nd, d, sizeof nd);
        nd[k] = st->rank;
        double* next = (double*)xcalloc(prod(nd, 0, order), sizeof(double));
        ttm_raw(cur, d, order, qt, st->rank, k, next);
        free(qt);
        free(cur);
        cur = next;
        memcpy(d, nd, sizeof d);
    }
    memcpy(odims, d, order * sizeof(uint64_t));
    return cur;
}

/* V = unfold(Y, n) * Q (tensor.hpp:184-189 matmul, ikj loop); threads take
 * disjoint rows of V */
typedef struct {
    const double *yn, *q;
    double* v;
    uint64_t K, R;
} vg_ctx;

static void v_gemm_range(void* p, uint64_t i0, uint64_t i1) {
    const vg_ctx* c = (const vg_ctx*)p;
    /* blocks of 512 rows of Q stay in cache across this thread's rows of V;
     * each V element still sums over pp ascending */
    const uint64_t pb = 512;
    for (uint64_t p0 = 0; p0 < c->K; p0 += pb) {
        const uint64_t p1 = p0 + pb < c->K ? p0 + pb : c->K;
        for (uint64_t i = i0; i < i1; ++i)
            for (uint64_t pp = p0; pp < p1; ++pp) {
                const double a = c->yn[i * c->K + pp];
                for (uint64_t j = 0; j < c->R; ++j) c->v[i * c->R + j] += a * c->q[pp * c->R + j];
            }
    }
}

static void v_gemm(const double* yn, uint64_t rows, uint64_t K, const double* q, uint64_t R,
                   double* v) {
    memset(v, 0, rows * R * sizeof(double));
    vg_ctx c = {yn, q, v, K, R};
    par_for(rows, K * R > (1u << 16) ? 1 : rows, v_gemm_range, &c);
}

int cpdo_solve(const double* x, const uint64_t* dims, uint32_t order, const cpdo_config* cfg,
               cpdo_state* stin, cpdo_trace_row* trace, uint64_t* trace_len, double* out_lambda,
               double* out_factors, double* factors_per_sweep, double* lambda_per_sweep,
               cpdo_q0_observer observer, void* observer_user) {
    /* SolverConfig::validate (solvers.hpp:41-49) */
    const uint64_t R = cfg->rank;
    if (R == 0) return fail(CPDO_INVALID_ARGUMENT, "SolverConfig: rank must be >= 1");
    if (cfg->max_iterations == 0)
        return fail(CPDO_INVALID_ARGUMENT, "SolverConfig: need at least one iteration");
    if (!(cfg->fitness_threshold >= 0.0 && cfg->fitness_threshold <= 1.0))
        return fail(CPDO_INVALID_ARGUMENT, "SolverConfig: fitness threshold must be in [0,1]");
    if (!isfinite(cfg->alpha) || !isfinite(cfg->activation_gap))
        return fail(CPDO_INVALID_ARGUMENT, "SolverConfig: alpha and activation gap must be finite");
    if (order < 2) return fail(CPDO_INVALID_ARGUMENT, "cp_als_qr: tensor order must be >= 2");
    if (order > CPDO_MAX_ORDER) return fail(CPDO_INVALID_ARGUMENT, "order too large");
    const uint64_t total = prod(dims, 0, order);
    double nx2 = 0.0;
    for (uint64_t i = 0; i < total; ++i) nx2 += x[i] * x[i]; /* inner(x,x) tensor.hpp:394 */
    if (nx2 == 0.0) return fail(CPDO_INVALID_ARGUMENT, "cp_als_qr: zero-norm tensor");
    for (uint32_t k = 0; k < order; ++k)
        if (R > dims[k])
            return fail(CPDO_INVALID_ARGUMENT,
                        "cp_als_qr: rank must not exceed any mode extent (compact QR)");

    const int extrap = cfg->extrapolate != 0;
    const uint64_t done = stin ? stin->sweeps_done : 0;
    uint64_t nfac = 0;
    for (uint32_t k = 0; k < order; ++k) nfac += dims[k] * R;
    double* init = (double*)xcalloc(nfac, sizeof(double));
    if (stin && stin->factors)
        memcpy(init, stin->factors, nfac * sizeof(double));
    else
        initial_factors(order, dims, R, cfg->seed, init);
    fstate_t st;
    fs_init(&st, order, dims, R, init);
    free(init);
    if (stin && stin->lambda) memcpy(st.lambda, stin->lambda, R * sizeof(double));

    const int32_t strategy = extrap ? 2 : cfg->strategy;
    sched_t s;
    int rc = build(&s, order, strategy, done + cfg->max_iterations);
    if (rc) {
        sched_free(&s);
        fs_free(&st);
        return rc;
    }
    cache_t cache;
    memset(&cache, 0, sizeof cache);
    if (done > 0) {
        uint32_t keys[2 * CPDO_MAX_ORDER * MAXSTEPS];
        const uint32_t nk = retained(&s, done - 1, order - 1, keys);
        for (uint32_t i = 0; i < nk; ++i) {
            if (cache_find(&cache, keys[i])) continue;
            uint64_t od[CPDO_MAX_ORDER], stamp[CPDO_MAX_ORDER] = {0};
            double* data = rebuild_entry(x, dims, &st, keys[i], od);
            for (uint32_t k = 0; k < order; ++k)
                if (!(keys[i] & (1u << k))) stamp[k] = st.version[k];
            cache_put(&cache, keys[i], data, od, stamp, order);
        }
    }

    uint64_t zrows = 1;
    for (uint32_t k = 1; k < order; ++k) zrows *= R;
    double* hist[CPDO_MAX_ORDER] = {0};
    if (stin && stin->q0_history)
        for (uint32_t n = 0; n < order; ++n)
            if (stin->history_mask & (1u << n)) hist[n] = dupd(stin->q0_history + n * zrows * R, zrows * R);
    int has_beta = 0;
    double beta = 0.0;
    if (extrap && cfg->has_beta_override) {
        has_beta = 1;
        beta = cfg->beta_override;
    }
    if (extrap && stin && stin->has_active_beta && !has_beta) {
        has_beta = 1;
        beta = stin->active_beta;
    }
    int has_prev = stin && stin->has_prev_fitness;
    double prev_fit = has_prev ? stin->prev_fitness : 0.0;

    uint64_t tot_flops = 0, tot_roots = 0;
    if (done > 0) cost_of(&s, dims, R, done, &tot_flops, &tot_roots);

    /* scratch */
    double* z = (double*)xcalloc(zrows * R, sizeof(double));
    double* q0 = (double*)xcalloc(zrows * R, sizeof(double));
    double* r0 = (double*)xcalloc(R * R, sizeof(double));
    double* qx = (double*)xcalloc(zrows * R, sizeof(double));
    double* r0t = (double*)xcalloc(R * R, sizeof(double));
    uint64_t maxI = 0;
    for (uint32_t k = 0; k < order; ++k) maxI = dims[k] > maxI ? dims[k] : maxI;
    double* yn = (double*)xcalloc(maxI * zrows, sizeof(double));
    double* v = (double*)xcalloc(maxI * R, sizeof(double));
    double* ah = (double*)xcalloc(maxI * R, sizeof(double));
    double* an = (double*)xcalloc(maxI * R, sizeof(double));
    double* lam = (double*)xcalloc(R, sizeof(double));
    double* v_last = (double*)xcalloc(maxI * R, sizeof(double));
    double* ah_last = (double*)xcalloc(maxI * R, sizeof(double));
    double* r0_last = (double*)xcalloc(R * R, sizeof(double));

    const double t0 = now_seconds();
    uint64_t rows_out = 0;
    for (uint64_t sweep = done + 1; sweep <= done + cfg->max_iterations && rc == CPDO_OK; ++sweep) {
        const iter_t* it = &s.it[sweep - 1];
        uint32_t last_mode = 0;
        uint64_t last_rows = 0;
        double beta_used = 0.0;
        for (uint32_t b = 0; b < order; ++b) {
            const uint32_t n = it->u[b].mode;
            /* solvers.hpp:250-255: Khatri-Rao of R_k, k != n, descending */
            const double* mats[CPDO_MAX_ORDER];
            uint64_t mrows[CPDO_MAX_ORDER];
            uint32_t cnt = 0;
            for (uint32_t k = order; k-- > 0;)
                if (k != n) {
                    mats[cnt] = st.r[k];
                    mrows[cnt++] = R;
                }
            double tp0 = now_seconds();
            cpdo_khatri_rao(mats, mrows, cnt, R, z);
            double tp1 = now_seconds();
            cpdo_thin_qr(z, zrows, R, q0, r0);
            double tp2 = now_seconds();
            if (observer) observer(observer_user, sweep, n, q0, zrows, R);
            const double* qused = q0;
            if (extrap && has_beta && beta != 0.0 && hist[n]) {
                cpdo_extrapolate_q0(q0, hist[n], zrows, R, beta, cfg->alpha, qx);
                qused = qx;
                beta_used = beta;
            }
            if (extrap) {
                if (!hist[n]) hist[n] = (double*)xcalloc(zrows * R, sizeof(double));
                memcpy(hist[n], q0, zrows * R * sizeof(double));
            }
            double* y = NULL;
            uint64_t yd[CPDO_MAX_ORDER];
            double tp3 = now_seconds();
            rc = execute(&s, x, dims, &st, &cache, sweep - 1, n, &y, yd, &tot_flops, &tot_roots);
            if (rc) break;
            const uint64_t I = dims[n];
            double tp4 = now_seconds();
            cpdo_unfold(y, yd, order, n, yn);
            free(y);
            double tp5 = now_seconds();
            v_gemm(yn, I, zrows, qused, R, v);
            double tp6 = now_seconds();
            if (getenv("CPDO_PROFILE"))
                fprintf(stderr, "mode %u: kr %.3f qr %.3f ex %.3f ttm %.3f unfold %.3f vgemm %.3f\n", n,
                        tp1 - tp0, tp2 - tp1, tp3 - tp2, tp4 - tp3, tp5 - tp4, tp6 - tp5);
            transpose(r0, R, R, r0t);
            rc = cpdo_solve_rows_lower(r0t, R, v, I, ah, NULL);
            if (rc) break;
            cpdo_normalize_columns(ah, I, R, an, lam);
            memcpy(st.lambda, lam, R * sizeof(double));
            fs_update(&st, n, an);
            if (b == order - 1 && qused != q0) v_gemm(yn, I, zrows, q0, R, v);
            memcpy(v_last, v, I * R * sizeof(double));
            memcpy(ah_last, ah, I * R * sizeof(double));
            memcpy(r0_last, r0, R * R * sizeof(double));
            last_mode = n;
            last_rows = I;
        }
        if (rc) break;
        double fit = 0.0, raw = 0.0;
        cpdo_fitness_fast_qr(nx2, v_last, ah_last, last_rows, r0_last, st.r[last_mode], st.lambda,
                             R, &fit, &raw);
        if (trace) {
            cpdo_trace_row* row = trace + rows_out;
            memset(row, 0, sizeof *row);
            row->iteration = sweep;
            row->order = order;
            for (uint32_t b = 0; b < order; ++b) row->update_order[b] = it->u[b].mode;
            row->fitness = fit;
            row->raw_radicand = raw;
            row->wall_seconds = now_seconds() - t0;
            row->root_ttm_count = tot_roots;
            row->flops = tot_flops;
            row->beta_used = beta_used;
        }
        if (factors_per_sweep) {
            double* p = factors_per_sweep + rows_out * nfac;
            for (uint32_t k = 0; k < order; ++k) {
                memcpy(p, st.a[k], dims[k] * R * sizeof(double));
                p += dims[k] * R;
            }
        }
        if (lambda_per_sweep) memcpy(lambda_per_sweep + rows_out * R, st.lambda, R * sizeof(double));
        ++rows_out;
        if (extrap && !has_beta && !cfg->has_beta_override && sweep >= 2 && has_prev)
            has_beta = cpdo_select_beta(prev_fit, fit, cfg->activation_gap, &beta);
        prev_fit = fit;
        has_prev = 1;
        if (fit >= cfg->fitness_threshold) break;
    }
    if (trace_len) *trace_len = rows_out;
    if (rc == CPDO_OK) {
        if (out_lambda) memcpy(out_lambda, st.lambda, R * sizeof(double));
        if (out_factors) {
            double* p = out_factors;
            for (uint32_t k = 0; k < order; ++k) {
                memcpy(p, st.a[k], dims[k] * R * sizeof(double));
                p += dims[k] * R;
            }
        }
        if (stin) {
            stin->sweeps_done = done + rows_out;
            if (stin->lambda) memcpy(stin->lambda, st.lambda, R * sizeof(double));
            if (stin->factors) {
                double* p = stin->factors;
                for (uint32_t k = 0; k < order; ++k) {
                    memcpy(p, st.a[k], dims[k] * R * sizeof(double));
                    p += dims[k] * R;
                }
            }
            if (stin->q0_history) {
                stin->history_mask = 0;
                for (uint32_t n = 0; n < order; ++n)
                    if (hist[n]) {
                        memcpy(stin->q0_history + n * zrows * R, hist[n], zrows * R * sizeof(double));
                        stin->history_mask |= 1u << n;
                    }
            }
            stin->has_active_beta = has_beta;
            stin->active_beta = has_beta ? beta : 0.0;
            stin->has_prev_fitness = has_prev;
            stin->prev_fitness = prev_fit;
        }
    }
    for (uint32_t n = 0; n < order; ++n) free(hist[n]);
    free(z);
    free(q0);
    free(r0);
    free(qx);
    free(r0t);
    free(yn);
    free(v);
    free(ah);
    free(an);
    free(lam);
    free(v_last);
    free(ah_last);
    free(r0_last);
    cache_clear(&cache);
    fs_free(&st);
    sched_free(&s);
    return rc;
}

/* kruskal.hpp:54-67 reconstruct: A_0 diag(lambda) times the ascending
 * Khatri-Rao of the other factors (gemm_bt loop order, detail::scale_columns
 * applied to A_0 first). */
int cpdo_reconstruct(const uint64_t* dims, uint32_t order, uint64_t R, const double* lambda,
                     const double* factors, double* out) {
    if (order < 1 || order > CPDO_MAX_ORDER) return fail(CPDO_INVALID_ARGUMENT, "reconstruct: order");
    const double* f[CPDO_MAX_ORDER];
    const double* p = factors;
    for (uint32_t k = 0; k < order; ++k) {
        f[k] = p;
        p += dims[k] * R;
    }
    uint64_t krows = 1;
    const double* mats[CPDO_MAX_ORDER];
    uint64_t mrows[CPDO_MAX_ORDER];
    for (uint32_t k = 1; k < order; ++k) {
        mats[k - 1] = f[k];
        mrows[k - 1] = dims[k];
        krows *= dims[k];
    }
    double* kr = (double*)xcalloc(krows * R, sizeof(double));
    if (order > 1)
        cpdo_khatri_rao(mats, mrows, order - 1, R, kr);
    else
        for (uint64_t j = 0; j < R; ++j) kr[j] = 1.0;
    double* a0 = (double*)xcalloc(dims[0] * R, sizeof(double));
    for (uint64_t i = 0; i < dims[0]; ++i)
        for (uint64_t j = 0; j < R; ++j) a0[i * R + j] = f[0][i * R + j] * lambda[j];
    for (uint64_t i = 0; i < dims[0]; ++i)
        for (uint64_t j = 0; j < krows; ++j) {
            double acc = 0.0;
            for (uint64_t q = 0; q < R; ++q) acc += a0[i * R + q] * kr[j * R + q];
            out[i * krows + j] = acc;
        }
    free(a0);
    free(kr);
    return CPDO_OK;
}

/* BASELINE synthetic construction (definition in oracle/ref_runner.cpp,
 * cpdref_synth_baseline); reconstruct per kruskal.hpp:54-67 (A_0 times the
 * ascending Khatri-Rao of the other factors, gemm_bt loop order). */
int cpdo_synth_baseline(int32_t kind, const uint64_t* dims, uint32_t order, uint64_t R, double rho,
                        uint64_t seed, double* out, double* truth_factors) {
    if (kind != 0 && kind != 1) return fail(CPDO_INVALID_ARGUMENT, "synth: unknown kind");
    cpdo_rng g;
    cpdo_rng_seed(&g, seed);
    double* f[CPDO_MAX_ORDER];
    for (uint32_t k = 0; k < order; ++k) {
        const uint64_t I = dims[k];
        f[k] = (double*)xcalloc(I * R, sizeof(double));
        if (kind == 0) {
            for (uint64_t i = 0; i < I * R; ++i) f[k][i] = cpdo_rng_normal(&g);
        } else {
            double* gv = (double*)xcalloc(I, sizeof(double));
            for (uint64_t i = 0; i < I; ++i) gv[i] = cpdo_rng_normal(&g);
            for (uint64_t j = 0; j < R; ++j) {
                const double sc = pow(10.0, -3.0 * cpdo_rng_uniform(&g));
                for (uint64_t i = 0; i < I; ++i)
                    f[k][i * R + j] = sc * (sqrt(0.9) * gv[i] + sqrt(0.1) * cpdo_rng_normal(&g));
            }
            free(gv);
        }
    }
    /* kr = khatri_rao(f[1], ..., f[N-1]) */
    uint64_t krows = 1;
    const double* mats[CPDO_MAX_ORDER];
    uint64_t mrows[CPDO_MAX_ORDER];
    for (uint32_t k = 1; k < order; ++k) {
        mats[k - 1] = f[k];
        mrows[k - 1] = dims[k];
        krows *= dims[k];
    }
    double* kr = (double*)xcalloc(krows * R, sizeof(double));
    if (order > 1)
        cpdo_khatri_rao(mats, mrows, order - 1, R, kr);
    else
        for (uint64_t j = 0; j < R; ++j) kr[j] = 1.0;
    const uint64_t I0 = dims[0];
    for (uint64_t i = 0; i < I0; ++i)
        for (uint64_t j = 0; j < krows; ++j) {
            double acc = 0.0;
            for (uint64_t p = 0; p < R; ++p) acc += (f[0][i * R + p] * 1.0) * kr[j * R + p];
            out[i * krows + j] = acc;
        }
    free(kr);
    const uint64_t total = I0 * krows;
    if (rho > 0.0) {
        double* e = (double*)xcalloc(total, sizeof(double));
        for (uint64_t i = 0; i < total; ++i) e[i] = cpdo_rng_normal(&g);
        double sx = 0.0, se = 0.0;
        for (uint64_t i = 0; i < total; ++i) sx += out[i] * out[i];
        for (uint64_t i = 0; i < total; ++i) se += e[i] * e[i];
        const double scale = rho * sqrt(sx) / sqrt(se);
        for (uint64_t i = 0; i < total; ++i) out[i] += scale * e[i];
        free(e);
    }
    if (truth_factors) {
        double* p = truth_factors;
        for (uint32_t k = 0; k < order; ++k) {
            memcpy(p, f[k], dims[k] * R * sizeof(double));
            p += dims[k] * R;
        }
    }
    for (uint32_t k = 0; k < order; ++k) free(f[k]);
    return CPDO_OK;
}
