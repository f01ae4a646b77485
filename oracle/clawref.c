/* oracle/clawref.c -- TEST INFRASTRUCTURE ONLY (the parity checker / CPU
 * baseline).  Never linked or loaded by the product package.
 *
 * C restatement of clawtile's directional sweep (reference
 * pkg/src/clawtile/sweep.py:183-263 kernel, :307-377 driver, :275-291
 * pencil bases) for the monolithic tile plan.  Pencils are split across
 * POSIX threads in contiguous blocks; every pencil's arithmetic is the
 * serial one, so results are bitwise identical for any thread count
 * (the same guarantee as the reference's tile pool,
 * pkg/tests/test_sweep.py:191-226).
 *
 * Build: oracle/Makefile  (gcc -O2 -ffp-contract=off -fno-fast-math).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CR_ADVECTION 0
#define CR_ACOUSTICS 1
#define CR_SHALLOW_WATER 2
#define CR_VC_ACOUSTICS 3
#define CR_MAXM 8
#define CR_MAXW 3

#define T double
#define SUF _f64
#define CR_SQRT(x) sqrt(x)
#define CR_ABS(x) fabs(x)
#include "clawref_impl.h"
#undef T
#undef SUF
#undef CR_SQRT
#undef CR_ABS

#define T float
#define SUF _f32
#define CR_SQRT(x) sqrtf(x)
#define CR_ABS(x) fabsf(x)
#include "clawref_impl.h"
#undef T
#undef SUF
#undef CR_SQRT
#undef CR_ABS

typedef struct {
    const void *qin;
    void *qout;
    int64_t sstride;
    int m;
    const int64_t *bases;
    int64_t nbases;
    int64_t stride, lo, hi;
    double dtdx;
    int normal;
    const void *params;
    int limiter_id, nw, solver, itemsize;
    double smax;
} cr_job;

static void *cr_run(void *arg)
{
    cr_job *j = (cr_job *)arg;
    if (j->nbases <= 0) { j->smax = 0.0; return NULL; }
    if (j->itemsize == 8) {
        j->smax = sweep_tile_f64((const double *)j->qin, (double *)j->qout, j->sstride, j->m,
                                 j->bases, j->nbases, j->stride, j->lo, j->hi, j->dtdx,
                                 j->normal, (const double *)j->params, j->limiter_id, j->nw,
                                 j->solver);
    } else {
        j->smax = (double)sweep_tile_f32((const float *)j->qin, (float *)j->qout, j->sstride,
                                         j->m, j->bases, j->nbases, j->stride, j->lo, j->hi,
                                         (float)j->dtdx, j->normal, (const float *)j->params,
                                         j->limiter_id, j->nw, j->solver);
    }
    return NULL;
}

/* Full monolithic sweep (sweep.py:380-391 sweep_axis) over padded SoA
 * arrays shaped (m, [nz+4,] [ny+4,] nx+4).  `params` is packed in the run
 * dtype exactly as RiemannSolver.pack_params (riemann.py:235-253); `dtdx`
 * is T(dt/dx) widened to double.  Writes interior cells of qout only.
 * Returns max |s| over every interface solved (widened to double), or -1
 * on a bad argument. */
double clawref_sweep(int ndim, const int64_t *cells, int m, int itemsize,
                     const void *qin, void *qout, int axis, double dtdx,
                     int solver, int normal, const void *params, int limiter_id,
                     int nw, int nthreads)
{
    if (ndim < 1 || ndim > 3 || axis < 0 || axis >= ndim || m < 1 || m > CR_MAXM ||
        nw < 1 || nw > CR_MAXW || (itemsize != 4 && itemsize != 8))
        return -1.0;
    const int g = 2;
    int64_t padded[3] = {1, 1, 1}, strides[3] = {0, 0, 0};
    int64_t acc = 1;
    for (int ax = 0; ax < ndim; ++ax) {
        padded[ax] = cells[ax] + 2 * g;
        strides[ax] = acc;
        acc *= padded[ax];
    }
    const int64_t sstride = acc;
    /* sweep.py:275-291: outermost transverse axis slowest */
    int trans[2] = {-1, -1};
    int nt = 0;
    for (int ax = 0; ax < ndim; ++ax)
        if (ax != axis) trans[nt++] = ax;
    int64_t nbases = 1;
    for (int t = 0; t < nt; ++t) nbases *= cells[trans[t]];
    int64_t *bases = (int64_t *)malloc(sizeof(int64_t) * (size_t)nbases);
    if (!bases) return -1.0;
    int64_t idx = 0;
    if (nt == 0) {
        bases[idx++] = 0;
    } else if (nt == 1) {
        for (int64_t a = 0; a < cells[trans[0]]; ++a)
            bases[idx++] = (g + a) * strides[trans[0]];
    } else {
        for (int64_t b = 0; b < cells[trans[1]]; ++b)
            for (int64_t a = 0; a < cells[trans[0]]; ++a)
                bases[idx++] = (g + a) * strides[trans[0]] + (g + b) * strides[trans[1]];
    }
    if (nthreads < 1) nthreads = 1;
    if (nthreads > nbases) nthreads = (int)nbases;
    cr_job *jobs = (cr_job *)calloc((size_t)nthreads, sizeof(cr_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(bases); free(jobs); free(th); return -1.0; }
    int64_t per = nbases / nthreads, rem = nbases % nthreads, start = 0;
    for (int t = 0; t < nthreads; ++t) {
        int64_t cnt = per + (t < rem ? 1 : 0);
        cr_job *j = &jobs[t];
        j->qin = qin; j->qout = qout; j->sstride = sstride; j->m = m;
        j->bases = bases + start; j->nbases = cnt;
        j->stride = strides[axis]; j->lo = g; j->hi = g + cells[axis];
        j->dtdx = dtdx; j->normal = normal; j->params = params;
        j->limiter_id = limiter_id; j->nw = nw; j->solver = solver; j->itemsize = itemsize;
        start += cnt;
    }
    if (nthreads == 1) {
        cr_run(&jobs[0]);
    } else {
        for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, cr_run, &jobs[t]);
        for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    }
    double smax = 0.0;
    for (int t = 0; t < nthreads; ++t)
        if (jobs[t].smax > smax) smax = jobs[t].smax;
    free(bases); free(jobs); free(th);
    return smax;
}

/* Single-interface solve, for solver identity tests. */
void clawref_solve(int solver, int itemsize, const void *ql, const void *qr, int m,
                   int normal, const void *params, void *W, void *s)
{
    if (itemsize == 8)
        solve_f64(solver, (const double *)ql, (const double *)qr, m, normal,
                  (const double *)params, (double *)W, (double *)s);
    else
        solve_f32(solver, (const float *)ql, (const float *)qr, m, normal,
                  (const float *)params, (float *)W, (float *)s);
}

double clawref_limiter(double theta, int kind) { return limiter_value_f64(theta, kind); }
