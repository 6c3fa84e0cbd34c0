/* bto_oracle.c -- CPU restatement of the reference's fused loops.  TEST INFRASTRUCTURE.
 *
 * This file is the parity oracle for the B200 kernels.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may call it; the product path (paper_1205_1098_b200/) never does.
 *
 * What it restates.  The reference (matfuse, /root/reference/pkg/src/matfuse)
 * has no checked-in kernel source: its code generator prints C99 + OpenMP at
 * run time.  Each function below is the loop nest that generator prints for
 * the organism `search.max_fuse(graph, t)` picks,
 * written by hand from the emission rules, with the thread count `t` turned
 * into a run-time argument (the reference bakes it into the pragma,
 * cemit.py:190-193):
 *
 *   - parallel region protocol ........ cemit.py:180-202  (emit_region)
 *       block p of t owns  lo = (ext*p)/t .. hi = (ext*(p+1))/t
 *       `#pragma omp parallel for num_threads(t) schedule(static)` over p
 *   - partitioned reductions ........... lower.py:123-135, cemit.py:204-222
 *       per-block partial buffer [t x extent], zeroed inside the worker
 *       (lower.py:220-240), joined serially in ASCENDING block order
 *   - statement forms .................. cemit.py:112-136 (`=` / `+=`, one
 *       rounded binary op per statement, contracted temporaries are scalars)
 *   - flat row-major indexing i*N + j .. cemit.py:54-72
 *   - which temporaries are scalars .... fuse.py:660-688 (contracted_temporaries)
 *   - op order per kernel .............. graph.py:285-315 (canonical ops)
 *
 * Compile with the reference's own flags (runtime.py:26, `cc -O3 -fopenmp`,
 * no -ffast-math, no -march): then results are BIT-IDENTICAL to the
 * reference's generated C at the same t (tests/test_oracle.py checks this
 * against oracle/_ref, the generated C compiled from /root/reference).
 *
 * Pinning: tests/golden/ holds outputs of the reference itself
 * (reference_evaluate = O1, generated C via run_kernel = O2) produced by
 * tests/golden/make_golden.py in the build container.
 */
#include <stdlib.h>
#include <stddef.h>

#if defined(_OPENMP)
#include <omp.h>
#endif

#define BTO_ORACLE_VERSION 1

int bto_oracle_version(void) { return BTO_ORACLE_VERSION; }

int bto_oracle_max_threads(void)
{
#if defined(_OPENMP)
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Serial ascending-block join of a [t x ext] partial buffer (cemit.py:204-222). */
static void join_blocks(const double *part, double *out, long ext, int t)
{
    for (long e = 0; e < ext; ++e) {
        double acc = part[e];
        for (long b = 1; b < t; ++b) {
            acc += part[b * ext + e];
        }
        out[e] = acc;
    }
}

/* ---- AXPYDOT: z = w - alpha*v ; beta = z'u ------------------------------
 * kernels/axpydot.bto:1-10; organism {_{p(k)}{_k 1 2 3}}; t0 contracted.
 * ops (tests/test_graph.py:63-69): t0 = v*alpha; z = w - t0; beta += z*u. */
void oracle_axpydot(const double *restrict w, const double *restrict v,
                    const double *restrict u, double alpha,
                    double *restrict z, double *beta, long M, int t)
{
    double *beta_part = (double *)malloc(sizeof(double) * (size_t)t);
    #pragma omp parallel for num_threads(t) schedule(static)
    for (long p = 0; p < t; ++p) {
        long lo = (M * p) / t;
        long hi = (M * (p + 1)) / t;
        double acc = 0.0;
        for (long k = lo; k < hi; ++k) {
            double t0 = v[k] * alpha;
            z[k] = w[k] - t0;
            acc += z[k] * u[k];
        }
        beta_part[p] = acc;
    }
    double total = beta_part[0];
    for (long b = 1; b < t; ++b) {
        total += beta_part[b];
    }
    *beta = total;
    free(beta_part);
}

/* ---- BiCGK: q = A p ; s = A' r ------------------------------------------
 * kernels/bicgk.bto:1-9; organism {_{p(i)}{_i{_j 1 2}}}; nothing contracted.
 * Row blocks; q[i] is block-local, s needs [t x N] partials + join. */
void oracle_bicgk(const double *restrict A, const double *restrict p,
                  const double *restrict r, double *restrict q,
                  double *restrict s, long M, long N, int t)
{
    double *s_part = (double *)malloc(sizeof(double) * (size_t)t * (size_t)N);
    #pragma omp parallel for num_threads(t) schedule(static)
    for (long b = 0; b < t; ++b) {
        long lo = (M * b) / t;
        long hi = (M * (b + 1)) / t;
        double *sp = s_part + b * N;
        for (long j = 0; j < N; ++j) {
            sp[j] = 0.0;
        }
        for (long i = lo; i < hi; ++i) {
            const double *row = A + i * N;
            double ri = r[i];
            double qi = 0.0;
            for (long j = 0; j < N; ++j) {
                qi += row[j] * p[j];
                sp[j] += row[j] * ri;
            }
            q[i] = qi;
        }
    }
    join_blocks(s_part, s, N, t);
    free(s_part);
}

/* ---- ATAX: y = A'(A x) ----------------------------------------------------
 * kernels/atax.bto:1-8; organism {_{p(i)}{_i{_j 1}{_j 2}}}; t0 contracted to
 * a per-row scalar; the two j loops stay sequential (reduction barrier). */
void oracle_atax(const double *restrict A, const double *restrict x,
                 double *restrict y, long M, long N, int t)
{
    double *y_part = (double *)malloc(sizeof(double) * (size_t)t * (size_t)N);
    #pragma omp parallel for num_threads(t) schedule(static)
    for (long b = 0; b < t; ++b) {
        long lo = (M * b) / t;
        long hi = (M * (b + 1)) / t;
        double *yp = y_part + b * N;
        for (long j = 0; j < N; ++j) {
            yp[j] = 0.0;
        }
        for (long i = lo; i < hi; ++i) {
            const double *row = A + i * N;
            double t0 = 0.0;
            for (long j = 0; j < N; ++j) {
                t0 += row[j] * x[j];
            }
            for (long j = 0; j < N; ++j) {
                yp[j] += row[j] * t0;
            }
        }
    }
    join_blocks(y_part, y, N, t);
    free(y_part);
}

/* ---- BATAX: y = beta * A'(A x) -------------------------------------------
 * kernels/batax.bto; organism {_{p(i)}{_i{_j 1}{_j 2}}}{_{p(j)}{_j 3}}:
 * ATAX into temporary t1, then a second region scales it. */
void oracle_batax(const double *restrict x, double beta,
                  const double *restrict A, double *restrict y,
                  long M, long N, int t)
{
    double *t1 = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    oracle_atax(A, x, t1, M, N, t);
    #pragma omp parallel for num_threads(t) schedule(static)
    for (long b = 0; b < t; ++b) {
        long lo = (N * b) / t;
        long hi = (N * (b + 1)) / t;
        for (long j = lo; j < hi; ++j) {
            y[j] = t1[j] * beta;
        }
    }
    free(t1);
}

/* ---- GESUMMV: y = alpha A x + beta B x -----------------------------------
 * kernels/gesummv.bto:1-9; organism {_{p(i)}{_i{_j 1 3} 2 4 5}}; t0..t3 all
 * contracted; both dot products share ONE j loop; no partials, no join. */
void oracle_gesummv(double alpha, double beta, const double *restrict A,
                    const double *restrict B, const double *restrict x,
                    double *restrict y, long M, long N, int t)
{
    #pragma omp parallel for num_threads(t) schedule(static)
    for (long b = 0; b < t; ++b) {
        long lo = (M * b) / t;
        long hi = (M * (b + 1)) / t;
        for (long i = lo; i < hi; ++i) {
            const double *ra = A + i * N;
            const double *rb = B + i * N;
            double t0 = 0.0;
            double t2 = 0.0;
            for (long j = 0; j < N; ++j) {
                t0 += ra[j] * x[j];
                t2 += rb[j] * x[j];
            }
            double t1 = t0 * alpha;
            double t3 = t2 * beta;
            y[i] = t1 + t3;
        }
    }
}

/* ---- DGEMV: z = alpha A x + beta y ---------------------------------------
 * kernels/dgemv.bto; organism {_{p(i)}{_i{_j 1} 2 3 4}}. */
void oracle_dgemv(double alpha, const double *restrict A,
                  const double *restrict x, double beta,
                  const double *restrict y, double *restrict z,
                  long M, long N, int t)
{
    #pragma omp parallel for num_threads(t) schedule(static)
    for (long b = 0; b < t; ++b) {
        long lo = (M * b) / t;
        long hi = (M * (b + 1)) / t;
        for (long i = lo; i < hi; ++i) {
            const double *row = A + i * N;
            double t0 = 0.0;
            for (long j = 0; j < N; ++j) {
                t0 += row[j] * x[j];
            }
            double t1 = t0 * alpha;
            double t2 = y[i] * beta;
            z[i] = t1 + t2;
        }
    }
}

/* Shared tail of GEMVER / DGEMVT (column-partitioned second half):
 *   x[j] = t[j]*beta + z[j]  for the block's columns, then
 *   part[b][i] = sum_{j in block} Mx[i,j] * x[j], joined ascending, then
 *   a second region scales w[i] = acc[i] * alpha.
 * The caller runs the block's first loop nest through `first`. */
typedef void (*colblock_fn)(long j_lo, long j_hi, double *t, void *ctx);

static void colblock_pipeline(const double *Mx, double alpha,
                              double beta, const double *restrict z,
                              double *restrict x, double *restrict w,
                              long M, long N, int t,
                              colblock_fn first, void *ctx)
{
    double *tcol = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    double *acc = (double *)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1));
    double *part = (double *)malloc(sizeof(double) * (size_t)t
                                    * (size_t)(M > 0 ? M : 1));
    #pragma omp parallel for num_threads(t) schedule(static)
    for (long b = 0; b < t; ++b) {
        long j_lo = (N * b) / t;
        long j_hi = (N * (b + 1)) / t;
        for (long j = j_lo; j < j_hi; ++j) {
            tcol[j] = 0.0;
        }
        first(j_lo, j_hi, tcol, ctx);
        for (long j = j_lo; j < j_hi; ++j) {
            double scaled = tcol[j] * beta;
            x[j] = scaled + z[j];
        }
        for (long i = 0; i < M; ++i) {
            double rowsum = 0.0;
            for (long j = j_lo; j < j_hi; ++j) {
                rowsum += Mx[i * N + j] * x[j];
            }
            part[b * M + i] = rowsum;
        }
    }
    join_blocks(part, acc, M, t);
    free(part);
    #pragma omp parallel for num_threads(t) schedule(static)
    for (long b = 0; b < t; ++b) {
        long lo = (M * b) / t;
        long hi = (M * (b + 1)) / t;
        for (long i = lo; i < hi; ++i) {
            w[i] = acc[i] * alpha;
        }
    }
    free(tcol);
    free(acc);
}

/* ---- GEMVER: B = A + u1 v1' + u2 v2' ; x = beta B' y + z ; w = alpha B x --
 * kernels/gemver.bto:1-13 (9 ops, tests/test_graph.py:163-166); organism
 * {_{p(j)}{_i{_j 1 2 3 4 5}}{_j 6 7}{_i{_j 8}}}{_{p(i)}{_i 9}}: COLUMN
 * blocks.  Per element: t0 = u1[i]*v1[j]; t1 = A + t0; t2 = u2[i]*v2[j];
 * B = t1 + t2 (each rounded, no FMA); t3[j] += B*y[i]. */
struct gemver_ctx {
    const double *A, *u1, *v1, *u2, *v2, *y;
    double *B;
    long M, N;
};

static void gemver_first(long j_lo, long j_hi, double *t3, void *vctx)
{
    struct gemver_ctx *c = (struct gemver_ctx *)vctx;
    const long N = c->N;
    for (long i = 0; i < c->M; ++i) {
        for (long j = j_lo; j < j_hi; ++j) {
            double t0 = c->u1[i] * c->v1[j];
            double t1 = c->A[i * N + j] + t0;
            double t2 = c->u2[i] * c->v2[j];
            c->B[i * N + j] = t1 + t2;
            t3[j] += c->B[i * N + j] * c->y[i];
        }
    }
}

void oracle_gemver(const double *restrict A, const double *restrict u1,
                   const double *restrict v1, const double *restrict u2,
                   const double *restrict v2, double alpha, double beta,
                   const double *restrict y, const double *restrict z,
                   double *restrict B, double *restrict x,
                   double *restrict w, long M, long N, int t)
{
    struct gemver_ctx c = {A, u1, v1, u2, v2, y, B, M, N};
    colblock_pipeline(B, alpha, beta, z, x, w, M, N, t, gemver_first, &c);
}

/* ---- DGEMVT: x = beta A' y + z ; w = alpha A x ---------------------------
 * kernels/dgemvt.bto; organism
 * {_{p(j)}{_i{_j 1}}{_j 2 3}{_i{_j 4}}}{_{p(i)}{_i 5}} (GEMVER minus rank-2). */
struct dgemvt_ctx {
    const double *A, *y;
    long M, N;
};

static void dgemvt_first(long j_lo, long j_hi, double *t0, void *vctx)
{
    struct dgemvt_ctx *c = (struct dgemvt_ctx *)vctx;
    const long N = c->N;
    for (long i = 0; i < c->M; ++i) {
        for (long j = j_lo; j < j_hi; ++j) {
            t0[j] += c->A[i * N + j] * c->y[i];
        }
    }
}

void oracle_dgemvt(double alpha, double beta, const double *restrict A,
                   const double *restrict y, const double *restrict z,
                   double *restrict x, double *restrict w,
                   long M, long N, int t)
{
    struct dgemvt_ctx c = {A, y, M, N};
    colblock_pipeline(A, alpha, beta, z, x, w, M, N, t, dgemvt_first, &c);
}

/* ---- VADD: x = w + y + z -------------------------------------------------
 * kernels/vadd.bto; organism {_{p(k)}{_k 1 2}}: t0 = w + y; x = t0 + z. */
void oracle_vadd(const double *restrict w, const double *restrict y,
                 const double *restrict z, double *restrict x, long M, int t)
{
    #pragma omp parallel for num_threads(t) schedule(static)
    for (long b = 0; b < t; ++b) {
        long lo = (M * b) / t;
        long hi = (M * (b + 1)) / t;
        for (long k = lo; k < hi; ++k) {
            double t0 = w[k] + y[k];
            x[k] = t0 + z[k];
        }
    }
}

/* ---- WAXPBY: w = alpha x + beta y ----------------------------------------
 * kernels/waxpby.bto; organism {_{p(k)}{_k 1 2 3}}. */
void oracle_waxpby(double alpha, const double *restrict x, double beta,
                   const double *restrict y, double *restrict w,
                   long M, int t)
{
    #pragma omp parallel for num_threads(t) schedule(static)
    for (long b = 0; b < t; ++b) {
        long lo = (M * b) / t;
        long hi = (M * (b + 1)) / t;
        for (long k = lo; k < hi; ++k) {
            double t0 = x[k] * alpha;
            double t1 = y[k] * beta;
            w[k] = t0 + t1;
        }
    }
}
