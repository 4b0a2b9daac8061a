/*
 * tweed_oracle.c -- CPU ORACLE (test infrastructure only; never the product path).
 *
 * A plain-C restatement of the reference `tweedmg` hot path
 * (/root/reference/pkg/src/tweedmg), used ONLY by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
 * `--impl reference` legs.  The product (paper_2110_08389_b200) never links,
 * imports or calls anything in this directory.
 *
 * Every routine follows the reference's arithmetic order operation by
 * operation so that results are bit-identical to the reference's Cython
 * backend (compile with -O2 -ffp-contract=off, no -march flags):
 *
 *   orc_relax_points   <- _ckernels.pyx:42-51   (_frozen_rhs 34-39)
 *   orc_relax_chain    <- _ckernels.pyx:91-103  (_chain_system 54-71,
 *                                                _thomas_inplace 74-88)
 *   orc_relax_ring     <- _ckernels.pyx:106-141 (circulant Thomas)
 *   orc_relax_legged   <- _ckernels.pyx:144-185 (m-legged Thomas)
 *   layouts            <- layout.py:61-168, smoothers.py:42-104
 *   orc_sweep          <- smoothers.py:121-150
 *   orc_apply/defect   <- stencil.py:76-96
 *   orc_restrict       <- transfer.py:21-39
 *   orc_prolong_add    <- transfer.py:42-56 + mgcycle.py:102
 *   orc_dense_solve    <- stencil.py:129-155 (SuperLU replaced by dense LU
 *                         with partial pivoting; equal to rounding)
 *
 * Fields are (nx+1) x (ny+1) row-major, u[i*(ny+1)+j] (stencil.py:12-15).
 * Pivot checks |p| < 1e-300 return ORC_SINGULAR (tridiag.py:17-27).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_SINGULAR 1
#define ORC_BADARG 2

#define U(i, j) u[(size_t)(i) * ld + (j)]
#define F(i, j) f[(size_t)(i) * ld + (j)]

static inline int piv_bad(double v) { return (-1e-300 < v && v < 1e-300); }

/* _ckernels.pyx:21-31 */
static inline double coupling(const double *W, const double *E, const double *S,
                              const double *N, long i, long j, long pi, long pj) {
    if (pi == i - 1) return W[i];
    if (pi == i + 1) return E[i];
    if (pj == j - 1) return S[j];
    return N[j];
}

/* _ckernels.pyx:34-39 */
static inline double frozen_rhs(const double *W, const double *E, const double *S,
                                const double *N, const double *u, const double *f,
                                size_t ld, long i, long j) {
    return (F(i, j) - W[i] * U(i - 1, j) - E[i] * U(i + 1, j) - S[j] * U(i, j - 1) -
            N[j] * U(i, j + 1));
}

/* _ckernels.pyx:42-51 */
int orc_relax_points(long n, const long *ii, const long *jj, const double *W,
                     const double *E, const double *S, const double *N, double *u,
                     const double *f, long ld) {
    for (long k = 0; k < n; k++) {
        long i = ii[k], j = jj[k];
        double b = -(W[i] + E[i] + S[j] + N[j]);
        U(i, j) = frozen_rhs(W, E, S, N, u, f, ld, i, j) / b;
    }
    return ORC_OK;
}

/* _ckernels.pyx:54-71 */
static void chain_system(long m, const long *ii, const long *jj, const double *W,
                         const double *E, const double *S, const double *N,
                         const double *u, const double *f, size_t ld, double *a,
                         double *b, double *c, double *r) {
    for (long k = 0; k < m; k++) {
        b[k] = -(W[ii[k]] + E[ii[k]] + S[jj[k]] + N[jj[k]]);
        r[k] = frozen_rhs(W, E, S, N, u, f, ld, ii[k], jj[k]);
    }
    a[0] = 0.0;
    c[m - 1] = 0.0;
    for (long k = 1; k < m; k++) {
        a[k] = coupling(W, E, S, N, ii[k], jj[k], ii[k - 1], jj[k - 1]);
        r[k] += a[k] * U(ii[k - 1], jj[k - 1]);
        c[k - 1] = coupling(W, E, S, N, ii[k - 1], jj[k - 1], ii[k], jj[k]);
        r[k - 1] += c[k - 1] * U(ii[k], jj[k]);
    }
}

/* _ckernels.pyx:74-88 */
static int thomas_inplace(long m, const double *a, double *b, const double *c, double *r) {
    for (long k = 1; k < m; k++) {
        if (piv_bad(b[k - 1])) return ORC_SINGULAR;
        double w = a[k] / b[k - 1];
        b[k] -= w * c[k - 1];
        r[k] -= w * r[k - 1];
    }
    if (piv_bad(b[m - 1])) return ORC_SINGULAR;
    r[m - 1] /= b[m - 1];
    for (long k = m - 2; k >= 0; k--) r[k] = (r[k] - c[k] * r[k + 1]) / b[k];
    return ORC_OK;
}

/* _ckernels.pyx:91-103 */
int orc_relax_chain(long m, const long *ii, const long *jj, const double *W,
                    const double *E, const double *S, const double *N, double *u,
                    const double *f, long ld) {
    if (m == 1) return orc_relax_points(1, ii, jj, W, E, S, N, u, f, ld);
    double *s = (double *)malloc(sizeof(double) * 4 * (size_t)m);
    double *a = s, *b = s + m, *c = s + 2 * m, *r = s + 3 * m;
    chain_system(m, ii, jj, W, E, S, N, u, f, ld, a, b, c, r);
    int st = thomas_inplace(m, a, b, c, r);
    if (st == ORC_OK)
        for (long k = 0; k < m; k++) U(ii[k], jj[k]) = r[k];
    free(s);
    return st;
}

/* _ckernels.pyx:106-141 */
int orc_relax_ring(long m, const long *ii, const long *jj, const double *W,
                   const double *E, const double *S, const double *N, double *u,
                   const double *f, long ld) {
    long mm = m - 1;
    if (m < 3) return ORC_BADARG;
    double *s = (double *)malloc(sizeof(double) * 7 * (size_t)m);
    double *a = s, *b = s + m, *c = s + 2 * m, *r = s + 3 * m;
    double *g = s + 4 * m, *y = s + 5 * m, *z = s + 6 * m;
    int st = ORC_OK;
    chain_system(m, ii, jj, W, E, S, N, u, f, ld, a, b, c, r);
    a[0] = coupling(W, E, S, N, ii[0], jj[0], ii[mm], jj[mm]);
    c[mm] = coupling(W, E, S, N, ii[mm], jj[mm], ii[0], jj[0]);
    r[0] += a[0] * U(ii[mm], jj[mm]);
    r[mm] += c[mm] * U(ii[0], jj[0]);
    for (long k = 0; k < mm; k++) g[k] = 0.0;
    g[0] = a[0];
    g[mm - 1] += c[mm - 1];
    for (long k = 1; k < mm; k++) {
        if (piv_bad(b[k - 1])) { st = ORC_SINGULAR; goto out; }
        double w = a[k] / b[k - 1];
        b[k] -= w * c[k - 1];
        r[k] -= w * r[k - 1];
        g[k] -= w * g[k - 1];
    }
    if (piv_bad(b[mm - 1])) { st = ORC_SINGULAR; goto out; }
    y[mm - 1] = r[mm - 1] / b[mm - 1];
    z[mm - 1] = g[mm - 1] / b[mm - 1];
    for (long k = mm - 2; k >= 0; k--) {
        y[k] = (r[k] - c[k] * y[k + 1]) / b[k];
        z[k] = (g[k] - c[k] * z[k + 1]) / b[k];
    }
    {
        double den = b[mm] - c[mm] * z[0] - a[mm] * z[mm - 1];
        if (piv_bad(den)) { st = ORC_SINGULAR; goto out; }
        double xm = (r[mm] - c[mm] * y[0] - a[mm] * y[mm - 1]) / den;
        for (long k = 0; k < mm; k++) U(ii[k], jj[k]) = y[k] - z[k] * xm;
        U(ii[mm], jj[mm]) = xm;
    }
out:
    free(s);
    return st;
}

/* _ckernels.pyx:144-185 */
int orc_relax_legged(long n, const long *ii, const long *jj, long m, const long *offs,
                     long bi, long bj, const double *W, const double *E, const double *S,
                     const double *N, double *u, const double *f, long ld) {
    double *s = (double *)malloc(sizeof(double) * (4 * (size_t)n + (size_t)m));
    double *a = s, *b = s + n, *c = s + 2 * n, *r = s + 3 * n, *d = s + 4 * n;
    int st = ORC_OK;
    double num = frozen_rhs(W, E, S, N, u, f, ld, bi, bj);
    double den = -(W[bi] + E[bi] + S[bj] + N[bj]);
    for (long k = 0; k < m; k++) {
        long lo = offs[k], hi = offs[k + 1];
        chain_system(hi - lo, ii + lo, jj + lo, W, E, S, N, u, f, ld, a + lo, b + lo,
                     c + lo, r + lo);
        c[hi - 1] = coupling(W, E, S, N, ii[hi - 1], jj[hi - 1], bi, bj);
        r[hi - 1] += c[hi - 1] * U(bi, bj);
        d[k] = coupling(W, E, S, N, bi, bj, ii[hi - 1], jj[hi - 1]);
        num += d[k] * U(ii[hi - 1], jj[hi - 1]);
        for (long t = lo + 1; t < hi; t++) {
            if (piv_bad(b[t - 1])) { st = ORC_SINGULAR; goto out; }
            double w = a[t] / b[t - 1];
            b[t] -= w * c[t - 1];
            r[t] -= w * r[t - 1];
        }
        if (piv_bad(b[hi - 1])) { st = ORC_SINGULAR; goto out; }
        num -= d[k] * r[hi - 1] / b[hi - 1];
        den -= d[k] * c[hi - 1] / b[hi - 1];
    }
    if (piv_bad(den)) { st = ORC_SINGULAR; goto out; }
    {
        double xb = num / den;
        U(bi, bj) = xb;
        for (long k = 0; k < m; k++) {
            long lo = offs[k], hi = offs[k + 1];
            double xk = (r[hi - 1] - c[hi - 1] * xb) / b[hi - 1];
            U(ii[hi - 1], jj[hi - 1]) = xk;
            for (long t = hi - 2; t >= lo; t--) {
                xk = (r[t] - c[t] * xk) / b[t];
                U(ii[t], jj[t]) = xk;
            }
        }
    }
out:
    free(s);
    return st;
}

/* ------------------------------------------------------------------------ */
/* Block layouts (layout.py:61-168, smoothers.py:65-104), built as flat lists */

enum { BK_POINT = 0, BK_LINE = 1, BK_LEGGED = 2, BK_RING = 3 };

typedef struct {
    int kind, red;
    long npts; /* members incl. branch for legged */
    long *ii, *jj;
    long nlegs;
    long offs[5];
    long bi, bj;
} OBlock;

typedef struct {
    OBlock *b;
    long n, cap;
} OLayout;

static OBlock *lay_new(OLayout *L, int kind, int red, long npts) {
    if (L->n == L->cap) {
        L->cap = L->cap ? 2 * L->cap : 64;
        L->b = (OBlock *)realloc(L->b, sizeof(OBlock) * (size_t)L->cap);
    }
    OBlock *B = &L->b[L->n++];
    memset(B, 0, sizeof(*B));
    B->kind = kind;
    B->red = red;
    B->npts = npts;
    B->ii = (long *)malloc(sizeof(long) * (size_t)(npts > 0 ? npts : 1));
    B->jj = (long *)malloc(sizeof(long) * (size_t)(npts > 0 ? npts : 1));
    return B;
}

static void lay_free(OLayout *L) {
    for (long k = 0; k < L->n; k++) { free(L->b[k].ii); free(L->b[k].jj); }
    free(L->b);
}

static int parity_red(long k) { return (int)(k % 2 != 0); } /* layout.py:22-23 */

/* legged block: legs given as (start i, start j, di, dj, len) tip -> branch */
static void add_legged(OLayout *L, int red, int nl, const long (*leg)[5], long bi, long bj) {
    long tot = 0;
    for (int k = 0; k < nl; k++) tot += leg[k][4];
    OBlock *B = lay_new(L, BK_LEGGED, red, tot); /* branch kept separately */
    B->nlegs = nl;
    B->bi = bi;
    B->bj = bj;
    long p = 0;
    B->offs[0] = 0;
    for (int k = 0; k < nl; k++) {
        for (long t = 0; t < leg[k][4]; t++) {
            B->ii[p] = leg[k][0] + t * leg[k][2];
            B->jj[p] = leg[k][1] + t * leg[k][3];
            p++;
        }
        B->offs[k + 1] = p;
    }
}

/* layout.py:61-133 */
static void tweed_layout(long nx, long ny, OLayout *L) {
    long mx = nx - 1, my = ny - 1, s = mx < my ? mx : my, c = (s + 1) / 2;
    long corners[4][4] = {{1, 1, 1, 1}, {mx, 1, -1, 1}, {1, my, 1, -1}, {mx, my, -1, -1}};
    for (int q = 0; q < 4; q++) {
        OBlock *B = lay_new(L, BK_POINT, 1, 1);
        B->ii[0] = corners[q][0];
        B->jj[0] = corners[q][1];
    }
    for (long k = 2; k < c; k++) {
        int red = parity_red(k);
        for (int q = 0; q < 4; q++) {
            long x0 = corners[q][0], y0 = corners[q][1], sx = corners[q][2], sy = corners[q][3];
            long bi = x0 + sx * (k - 1), bj = y0 + sy * (k - 1);
            long legs[2][5] = {{x0, bj, sx, 0, k - 1}, {bi, y0, 0, sy, k - 1}};
            add_legged(L, red, 2, (const long (*)[5])legs, bi, bj);
        }
    }
    int redc = parity_red(c);
    if (mx == my) {
        long legs[4][5] = {{1, c, 1, 0, c - 1}, {mx, c, -1, 0, mx - c},
                           {c, 1, 0, 1, c - 1}, {c, my, 0, -1, my - c}};
        add_legged(L, redc, 4, (const long (*)[5])legs, c, c);
    } else if (mx > my) {
        long legs_l[3][5] = {{1, c, 1, 0, c - 1}, {c, 1, 0, 1, c - 1}, {c, my, 0, -1, my - c}};
        add_legged(L, redc, 3, (const long (*)[5])legs_l, c, c);
        long br = mx + 1 - c;
        long legs_r[3][5] = {{mx, c, -1, 0, mx - br}, {br, 1, 0, 1, c - 1}, {br, my, 0, -1, my - c}};
        add_legged(L, redc, 3, (const long (*)[5])legs_r, br, c);
        for (long i = c + 1; i < mx - c + 1; i++) {
            OBlock *B = lay_new(L, BK_LINE, parity_red(i), my);
            for (long j = 1; j <= my; j++) { B->ii[j - 1] = i; B->jj[j - 1] = j; }
        }
    } else {
        long legs_b[3][5] = {{c, 1, 0, 1, c - 1}, {1, c, 1, 0, c - 1}, {mx, c, -1, 0, mx - c}};
        add_legged(L, redc, 3, (const long (*)[5])legs_b, c, c);
        long br = my + 1 - c;
        long legs_t[3][5] = {{c, my, 0, -1, my - br}, {1, br, 1, 0, c - 1}, {mx, br, -1, 0, mx - c}};
        add_legged(L, redc, 3, (const long (*)[5])legs_t, c, br);
        for (long j = c + 1; j < my - c + 1; j++) {
            OBlock *B = lay_new(L, BK_LINE, parity_red(j), mx);
            for (long i = 1; i <= mx; i++) { B->ii[i - 1] = i; B->jj[i - 1] = j; }
        }
    }
}

/* layout.py:136-168 */
static void wireframe_layout(long nx, long ny, OLayout *L) {
    long mx = nx - 1, my = ny - 1, s = mx < my ? mx : my, q = (s - 1) / 2;
    for (long r = 1; r <= q; r++) {
        long lo_i = r, hi_i = mx + 1 - r, lo_j = r, hi_j = my + 1 - r;
        long m = 2 * (hi_i - lo_i) + 2 * (hi_j - lo_j);
        OBlock *B = lay_new(L, BK_RING, parity_red(r), m);
        long p = 0;
        for (long i = lo_i; i <= hi_i; i++) { B->ii[p] = i; B->jj[p] = lo_j; p++; }
        for (long j = lo_j + 1; j <= hi_j; j++) { B->ii[p] = hi_i; B->jj[p] = j; p++; }
        for (long i = hi_i - 1; i >= lo_i; i--) { B->ii[p] = i; B->jj[p] = hi_j; p++; }
        for (long j = hi_j - 1; j > lo_j; j--) { B->ii[p] = lo_i; B->jj[p] = j; p++; }
    }
    int tred = parity_red(q + 1);
    if (mx == my) {
        OBlock *B = lay_new(L, BK_POINT, tred, 1);
        B->ii[0] = q + 1;
        B->jj[0] = q + 1;
    } else if (mx > my) {
        long j0 = q + 1, n = mx - 2 * q;
        OBlock *B = lay_new(L, BK_LINE, tred, n);
        for (long t = 0; t < n; t++) { B->ii[t] = q + 1 + t; B->jj[t] = j0; }
    } else {
        long i0 = q + 1, n = my - 2 * q;
        OBlock *B = lay_new(L, BK_LINE, tred, n);
        for (long t = 0; t < n; t++) { B->ii[t] = i0; B->jj[t] = q + 1 + t; }
    }
}

/* smoothers.py:65-89 */
static void zebra_layout(long nx, long ny, int axis_x, OLayout *L) {
    if (axis_x) {
        for (long j = 1; j < ny; j++) {
            OBlock *B = lay_new(L, BK_LINE, (int)(j % 2), nx - 1);
            for (long i = 1; i < nx; i++) { B->ii[i - 1] = i; B->jj[i - 1] = j; }
        }
    } else {
        for (long i = 1; i < nx; i++) {
            OBlock *B = lay_new(L, BK_LINE, (int)(i % 2), ny - 1);
            for (long j = 1; j < ny; j++) { B->ii[j - 1] = i; B->jj[j - 1] = j; }
        }
    }
}

/* scheme ids shared with oracle.py */
enum { SK_CHECKER = 0, SK_ZEBRA_X = 1, SK_ZEBRA_Y = 2, SK_TWEED = 4, SK_WIRE = 5 };

static int build_layout(int scheme, long nx, long ny, OLayout *L) {
    memset(L, 0, sizeof(*L));
    switch (scheme) {
    case SK_ZEBRA_X: zebra_layout(nx, ny, 1, L); return ORC_OK;
    case SK_ZEBRA_Y: zebra_layout(nx, ny, 0, L); return ORC_OK;
    case SK_TWEED:
        if (nx < 4 || ny < 4 || nx % 2 || ny % 2) return ORC_BADARG;
        tweed_layout(nx, ny, L);
        return ORC_OK;
    case SK_WIRE:
        if (nx < 4 || ny < 4 || nx % 2 || ny % 2) return ORC_BADARG;
        wireframe_layout(nx, ny, L);
        return ORC_OK;
    default: return ORC_BADARG;
    }
}

/* One colour stage, blocks in construction order (smoothers.py:139-150).
 * Same-colour blocks are independent, so the OpenMP split over
 * blocks gives bit-identical results to the serial loop. */
/* Sharding group of an interior point for the multi-GPU partition (test
 * oracle for DESIGN.md §6 / SURVEY.md §8(e)): tweed L-shells by
 * max(i', j') and wireframe rings by min(i', j') with the mirrored indices
 * of SURVEY.md §8(a'); zebra_x lines by j; zebra_y lines and checkerboard
 * points by i.  Every block lies in one group. */
long orc_group(int scheme, long nx, long ny, long i, long j) {
    long ip = i < nx - i ? i : nx - i, jp = j < ny - j ? j : ny - j;
    if (scheme == SK_TWEED) return ip > jp ? ip : jp;
    if (scheme == SK_WIRE) return ip < jp ? ip : jp;
    if (scheme == SK_ZEBRA_X) return j;
    return i;
}

static long block_group(int scheme, long nx, long ny, const OBlock *B) {
    if (B->kind == BK_LEGGED) return orc_group(scheme, nx, ny, B->bi, B->bj);
    return orc_group(scheme, nx, ny, B->ii[0], B->jj[0]);
}

static int run_stage_part(const OLayout *L, int red, const double *W, const double *E,
                          const double *S, const double *N, double *u, const double *f,
                          long ld, int nthreads, int scheme, long nx, long g0, long g1);

static int run_stage(const OLayout *L, int red, const double *W, const double *E,
                     const double *S, const double *N, double *u, const double *f,
                     long ld, int nthreads) {
    return run_stage_part(L, red, W, E, S, N, u, f, ld, nthreads, -1, 0, 0, 0);
}

/* one colour stage over the blocks of groups [g0, g1) (scheme < 0: all) */
static int run_stage_part(const OLayout *L, int red, const double *W, const double *E,
                          const double *S, const double *N, double *u, const double *f,
                          long ld, int nthreads, int scheme, long nx, long g0, long g1) {
    int status = ORC_OK;
    /* points first (merged), then legged, lines, rings: order is irrelevant
     * for the result but kept for fidelity */
    for (int pass = 0; pass < 4; pass++) {
        int kind = pass == 0 ? BK_POINT : pass == 1 ? BK_LEGGED : pass == 2 ? BK_LINE : BK_RING;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) if (nthreads > 1)
        for (long k = 0; k < L->n; k++) {
            const OBlock *B = &L->b[k];
            if (B->kind != kind || B->red != red) continue;
            if (scheme >= 0) {
                long grp = block_group(scheme, nx, ld - 1, B);
                if (grp < g0 || grp >= g1) continue;
            }
            int st = ORC_OK;
            if (kind == BK_POINT)
                st = orc_relax_points(B->npts, B->ii, B->jj, W, E, S, N, u, f, ld);
            else if (kind == BK_LEGGED)
                st = orc_relax_legged(B->npts, B->ii, B->jj, B->nlegs, B->offs, B->bi, B->bj,
                                      W, E, S, N, u, f, ld);
            else if (kind == BK_LINE)
                st = orc_relax_chain(B->npts, B->ii, B->jj, W, E, S, N, u, f, ld);
            else
                st = orc_relax_ring(B->npts, B->ii, B->jj, W, E, S, N, u, f, ld);
            if (st != ORC_OK) {
#pragma omp critical
                status = st;
            }
        }
    }
    return status;
}

/* smoothers.py:121-150 for one non-alternating scheme */
int orc_sweep(int scheme, long nx, long ny, const double *W, const double *E,
              const double *S, const double *N, double *u, const double *f,
              int nthreads) {
    long ld = ny + 1;
    if (scheme == SK_CHECKER) { /* smoothers.py:65-75: red = (i+j) even */
        for (int red = 1; red >= 0; red--) {
#pragma omp parallel for schedule(static) num_threads(nthreads) if (nthreads > 1)
            for (long i = 1; i < nx; i++)
                for (long j = 1; j < ny; j++) {
                    if ((((i + j) % 2) == 0) != red) continue;
                    long ii = i, jj = j;
                    orc_relax_points(1, &ii, &jj, W, E, S, N, u, f, ld);
                }
        }
        return ORC_OK;
    }
    OLayout L;
    int st = build_layout(scheme, nx, ny, &L);
    if (st != ORC_OK) return st;
    st = run_stage(&L, 1, W, E, S, N, u, f, ld, nthreads);
    if (st == ORC_OK) st = run_stage(&L, 0, W, E, S, N, u, f, ld, nthreads);
    lay_free(&L);
    return st;
}

/* One colour stage (red = 1 / black = 0) of one rank's share, the blocks of
 * sharding groups [g0, g1) -- the CPU restatement of a sharded sweep. */
int orc_sweep_part(int scheme, long nx, long ny, const double *W, const double *E,
                   const double *S, const double *N, double *u, const double *f,
                   int red, long g0, long g1, int nthreads) {
    long ld = ny + 1;
    if (scheme == SK_CHECKER) {
#pragma omp parallel for schedule(static) num_threads(nthreads) if (nthreads > 1)
        for (long i = (g0 > 1 ? g0 : 1); i < (g1 < nx ? g1 : nx); i++)
            for (long j = 1; j < ny; j++) {
                if ((((i + j) % 2) == 0) != red) continue;
                long ii = i, jj = j;
                orc_relax_points(1, &ii, &jj, W, E, S, N, u, f, ld);
            }
        return ORC_OK;
    }
    OLayout L;
    int st = build_layout(scheme, nx, ny, &L);
    if (st != ORC_OK) return st;
    st = run_stage_part(&L, red, W, E, S, N, u, f, ld, nthreads, scheme, nx, g0, g1);
    lay_free(&L);
    return st;
}

/* Layout export for tests: fills per-point (i, j, block id, red) in block
 * member order (legged: legs then branch, as layout.py:55-58).  Returns the
 * number of points written (or needed if cap is too small). */
long orc_layout_dump(int scheme, long nx, long ny, long *out_i, long *out_j,
                     long *out_blk, long *out_red, long cap) {
    OLayout L;
    if (build_layout(scheme, nx, ny, &L) != ORC_OK) return -1;
    long p = 0;
    for (long k = 0; k < L.n; k++) {
        const OBlock *B = &L.b[k];
        long np = B->npts + (B->kind == BK_LEGGED ? 1 : 0);
        for (long t = 0; t < np; t++) {
            if (p < cap) {
                int br = (B->kind == BK_LEGGED && t == B->npts);
                out_i[p] = br ? B->bi : B->ii[t];
                out_j[p] = br ? B->bj : B->jj[t];
                out_blk[p] = k;
                out_red[p] = B->red;
            }
            p++;
        }
    }
    lay_free(&L);
    return p;
}

/* ------------------------------------------------------------------------ */
/* stencil.py:76-96: (L u) then d = f - L u, numpy evaluation order.         */
int orc_defect(long nx, long ny, const double *W, const double *E, const double *S,
               const double *N, const double *u, const double *f, double *d,
               int nthreads) {
    long ld = ny + 1;
#pragma omp parallel for schedule(static) num_threads(nthreads) if (nthreads > 1)
    for (long i = 0; i <= nx; i++) {
        for (long j = 0; j <= ny; j++) {
            if (i == 0 || i == nx || j == 0 || j == ny) { d[i * ld + j] = 0.0; continue; }
            double C = -(W[i] + E[i] + S[j] + N[j]);
            double Lu = W[i] * U(i - 1, j) + E[i] * U(i + 1, j) + S[j] * U(i, j - 1) +
                        N[j] * U(i, j + 1) + C * U(i, j);
            d[i * ld + j] = -Lu + F(i, j);
        }
    }
    return ORC_OK;
}

/* max |f - L u| over the interior (mgcycle.py:122,130); NaN propagates */
double orc_defect_max(long nx, long ny, const double *W, const double *E, const double *S,
                      const double *N, const double *u, const double *f, int nthreads) {
    long ld = ny + 1;
    double mx = 0.0;
    int nan = 0;
#pragma omp parallel for schedule(static) num_threads(nthreads) reduction(max : mx) reduction(| : nan) if (nthreads > 1)
    for (long i = 1; i < nx; i++) {
        for (long j = 1; j < ny; j++) {
            double C = -(W[i] + E[i] + S[j] + N[j]);
            double Lu = W[i] * U(i - 1, j) + E[i] * U(i + 1, j) + S[j] * U(i, j - 1) +
                        N[j] * U(i, j + 1) + C * U(i, j);
            double v = fabs(-Lu + F(i, j));
            if (v != v) nan = 1;
            if (v > mx) mx = v;
        }
    }
    return nan ? NAN : mx;
}

/* transfer.py:21-39 (kind 0 = half, 1 = full) */
int orc_restrict(int full, long nxf, long nyf, const double *d, double *out) {
    if (nxf % 2 || nyf % 2) return ORC_BADARG;
    long nxc = nxf / 2, nyc = nyf / 2, ldf = nyf + 1, ldc = nyc + 1;
    for (long I = 0; I <= nxc; I++)
        for (long J = 0; J <= nyc; J++) {
            double v = 0.0;
            if (I > 0 && I < nxc && J > 0 && J < nyc) {
                long i = 2 * I, j = 2 * J;
#define D(a, b) d[(a) * ldf + (b)]
                double ctr = D(i, j);
                double edges = D(i - 1, j) + D(i + 1, j) + D(i, j - 1) + D(i, j + 1);
                if (full) {
                    double diags = D(i - 1, j - 1) + D(i + 1, j - 1) + D(i - 1, j + 1) + D(i + 1, j + 1);
                    v = 0.25 * ctr + 0.125 * edges + 0.0625 * diags;
                } else {
                    v = 0.5 * ctr + 0.125 * edges;
                }
#undef D
            }
            out[I * ldc + J] = v;
        }
    return ORC_OK;
}

/* transfer.py:42-56 then u += v (mgcycle.py:102) */
int orc_prolong_add(long nxc, long nyc, const double *uc, double *u) {
    long nxf = 2 * nxc, nyf = 2 * nyc, ldf = nyf + 1, ldc = nyc + 1;
#define C_(a, b) uc[(a) * ldc + (b)]
    for (long i = 1; i < nxf; i++)
        for (long j = 1; j < nyf; j++) {
            long I = i / 2, J = j / 2;
            double v;
            if (i % 2 == 0 && j % 2 == 0) v = C_(I, J);
            else if (i % 2 == 0) v = 0.5 * (C_(I, J) + C_(I, J + 1));
            else if (j % 2 == 0) v = 0.5 * (C_(I, J) + C_(I + 1, J));
            else v = 0.25 * (C_(I, J) + C_(I + 1, J) + C_(I, J + 1) + C_(I + 1, J + 1));
            u[i * ldf + j] += v;
        }
#undef C_
    return ORC_OK;
}

/* stencil.py:129-155: u = L^-1 (f - boundary couplings) on the interior, with
 * the boundary ring of u kept.  Dense LU with partial pivoting over the
 * j-outer / i-inner interior ordering (stencil.py:111). */
int orc_dense_solve(long nx, long ny, const double *W, const double *E, const double *S,
                    const double *N, double *u, const double *f) {
    long ld = ny + 1, mi = nx - 1, mj = ny - 1, n = mi * mj;
    double *A = (double *)calloc((size_t)n * (size_t)n, sizeof(double));
    double *x = (double *)malloc(sizeof(double) * (size_t)n);
    long *perm = (long *)malloc(sizeof(long) * (size_t)n);
    int st = ORC_OK;
    for (long i = 1; i < nx; i++)
        for (long j = 1; j < ny; j++) {
            long k = (j - 1) * mi + (i - 1);
            A[k * n + k] = -(W[i] + E[i] + S[j] + N[j]);
            if (i > 1) A[k * n + k - 1] = W[i];
            if (i < nx - 1) A[k * n + k + 1] = E[i];
            if (j > 1) A[k * n + k - mi] = S[j];
            if (j < ny - 1) A[k * n + k + mi] = N[j];
            /* boundary couplings folded into the rhs, interior taken as 0 */
            double C = -(W[i] + E[i] + S[j] + N[j]);
            double bu = (i == 1 ? U(0, j) : 0.0), be = (i == nx - 1 ? U(nx, j) : 0.0);
            double bs = (j == 1 ? U(i, 0) : 0.0), bn = (j == ny - 1 ? U(i, ny) : 0.0);
            double Lu = W[i] * bu + E[i] * be + S[j] * bs + N[j] * bn + C * 0.0;
            x[k] = F(i, j) - Lu;
        }
    for (long k = 0; k < n; k++) perm[k] = k;
    for (long k = 0; k < n; k++) {
        long p = k;
        for (long r = k + 1; r < n; r++)
            if (fabs(A[r * n + k]) > fabs(A[p * n + k])) p = r;
        if (piv_bad(A[p * n + k])) { st = ORC_SINGULAR; goto out; }
        if (p != k) {
            for (long c = 0; c < n; c++) {
                double t = A[k * n + c]; A[k * n + c] = A[p * n + c]; A[p * n + c] = t;
            }
            double t = x[k]; x[k] = x[p]; x[p] = t;
        }
        for (long r = k + 1; r < n; r++) {
            double l = A[r * n + k] / A[k * n + k];
            if (l == 0.0) continue;
            for (long c = k; c < n; c++) A[r * n + c] -= l * A[k * n + c];
            x[r] -= l * x[k];
        }
    }
    for (long k = n - 1; k >= 0; k--) {
        double s = x[k];
        for (long c = k + 1; c < n; c++) s -= A[k * n + c] * x[c];
        x[k] = s / A[k * n + k];
    }
    for (long i = 1; i < nx; i++)
        for (long j = 1; j < ny; j++) U(i, j) = x[(j - 1) * mi + (i - 1)];
out:
    free(A); free(x); free(perm);
    return st;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
