/*
 * tweed3d_oracle.c -- CPU ORACLE for the 3D tweed path (test infrastructure
 * only; never the product path).
 *
 * The reference is 2D only ("3D: no oracle, parity
 * unpinned"); this file restates the 2D semantics in 3D so that the device
 * version has a checker:
 *   - operator: stencil.py:43-96 with a third axis (7-point, coefficients
 *     B, T along k); fields u[i][j][k], k fastest;
 *   - tweed blocks: the survey's cube layout (SURVEY.md §8(c) "Candidate 3D
 *     layouts"): a point lies on the line along the axis of its unique
 *     smallest mirrored coordinate, running from the wall to the first tie
 *     point (the branch); branches with s1 = s2 < s3 carry 2 legs, s1 = s2 =
 *     s3 < c carry 3, the centre (c, c, c) 6; colour = parity(s1 + s3) of the
 *     branch's sorted mirrored coordinates, red = even (the corners);
 *   - block solve: the m-legged Thomas of _ckernels.pyx:144-185 /
 *     tridiag.py:84-125, legs tip -> branch, frozen out-of-block neighbours;
 *   - transfers: full weighting as the tensor product of [1/4, 1/2, 1/4]
 *     (transfer.py:21-39 in 3D) and trilinear prolongation (transfer.py:42-56).
 * Cubes only (nx = ny = nz = n, n even).  The parity of this oracle with the
 * device is checked by tests; its own soundness by property tests (partition,
 * same-colour independence, exactness by colour, dense block Gauss-Seidel).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define O3_OK 0
#define O3_SINGULAR 1
#define O3_BADARG 2

static inline long mir(long x, long n) { return x < n - x ? x : n - x; }
static inline int piv_bad3(double v) { return (-1e-300 < v && v < 1e-300); }

/* a block: branch + up to 6 legs (axis, step, start point, length) */
typedef struct {
    long bi, bj, bk;
    int red, nleg;
    int axis[6], step[6];
    long len[6];
    long si[6], sj[6], sk[6]; /* tip point of each leg */
} O3Block;

static void sorted3(long a, long b, long c, long *s1, long *s2, long *s3) {
    long x = a, y = b, z = c, t;
    if (x > y) { t = x; x = y; y = t; }
    if (y > z) { t = y; y = z; z = t; }
    if (x > y) { t = x; x = y; y = t; }
    *s1 = x; *s2 = y; *s3 = z;
}

/* Enumerate the blocks of the n^3 cube; returns the count (writes up to cap). */
long orc3_blocks(long n, O3Block *out, long cap) {
    const long c = n / 2;
    long nb = 0;
    for (long i = 1; i < n; i++)
        for (long j = 1; j < n; j++)
            for (long k = 1; k < n; k++) {
                const long m[3] = {mir(i, n), mir(j, n), mir(k, n)};
                long s1, s2, s3;
                sorted3(m[0], m[1], m[2], &s1, &s2, &s3);
                if (s1 != s2) continue; /* a leg point */
                if (nb < cap) {
                    O3Block *B = &out[nb];
                    memset(B, 0, sizeof(*B));
                    B->bi = i; B->bj = j; B->bk = k;
                    B->red = ((s1 + s3) % 2) == 0;
                    const long x[3] = {i, j, k};
                    for (int a = 0; a < 3; a++) {
                        if (m[a] != s1 || s1 < 2) continue;
                        /* leg(s) along axis a toward the branch */
                        for (int side = 0; side < 2; side++) {
                            long tip;
                            int step;
                            if (side == 0) {
                                if (x[a] > c) continue;
                                tip = 1; step = +1;
                            } else {
                                if (x[a] < c) continue;
                                tip = n - 1; step = -1;
                            }
                            int L = B->nleg++;
                            B->axis[L] = a;
                            B->step[L] = step;
                            B->len[L] = s1 - 1;
                            B->si[L] = a == 0 ? tip : i;
                            B->sj[L] = a == 1 ? tip : j;
                            B->sk[L] = a == 2 ? tip : k;
                        }
                    }
                }
                nb++;
            }
    return nb;
}

typedef struct {
    long n;
    const double *W, *E, *S, *N, *Bc, *Tc;
} Grid3;

#define IDX(i, j, k) (((size_t)(i) * (size_t)(n + 1) + (size_t)(j)) * (size_t)(n + 1) + (size_t)(k))

/* coupling of (i,j,k) toward its neighbour one step along axis a, direction s */
static inline double cpl(const Grid3 *g, int a, int s, long i, long j, long k) {
    if (a == 0) return s < 0 ? g->W[i] : g->E[i];
    if (a == 1) return s < 0 ? g->S[j] : g->N[j];
    return s < 0 ? g->Bc[k] : g->Tc[k];
}

static inline double diag3(const Grid3 *g, long i, long j, long k) {
    return -(g->W[i] + g->E[i] + g->S[j] + g->N[j] + g->Bc[k] + g->Tc[k]);
}

/* f - sum of the neighbours not excluded by mask (bit 2a + (s>0)) */
static inline double rhs3(const Grid3 *g, const double *u, const double *f, long i, long j,
                          long k, unsigned skip) {
    const long n = g->n;
    double r = f[IDX(i, j, k)];
    if (!(skip & 1u)) r -= g->W[i] * u[IDX(i - 1, j, k)];
    if (!(skip & 2u)) r -= g->E[i] * u[IDX(i + 1, j, k)];
    if (!(skip & 4u)) r -= g->S[j] * u[IDX(i, j - 1, k)];
    if (!(skip & 8u)) r -= g->N[j] * u[IDX(i, j + 1, k)];
    if (!(skip & 16u)) r -= g->Bc[k] * u[IDX(i, j, k - 1)];
    if (!(skip & 32u)) r -= g->Tc[k] * u[IDX(i, j, k + 1)];
    return r;
}

static inline unsigned dirbit(int a, int s) { return 1u << (2 * a + (s > 0 ? 1 : 0)); }

/* m-legged Thomas for one block (tridiag.py:84-125 in 3D) */
static int solve_block(const Grid3 *g, const O3Block *B, double *u, const double *f,
                       double *wk) {
    const long n = g->n;
    unsigned bskip = 0;
    for (int l = 0; l < B->nleg; l++) bskip |= dirbit(B->axis[l], -B->step[l]);
    double num = rhs3(g, u, f, B->bi, B->bj, B->bk, bskip);
    double den = diag3(g, B->bi, B->bj, B->bk);
    /* per leg: b', r' of every point, c of every point (wk: 3 * len) */
    long off = 0;
    for (int l = 0; l < B->nleg; l++) {
        const int a = B->axis[l], s = B->step[l];
        const long L = B->len[l];
        double *bp = wk + off, *rp = wk + off + L, *cp = wk + off + 2 * L;
        for (long t = 0; t < L; t++) {
            const long i = B->si[l] + (a == 0 ? s * t : 0);
            const long j = B->sj[l] + (a == 1 ? s * t : 0);
            const long k = B->sk[l] + (a == 2 ? s * t : 0);
            unsigned skip = dirbit(a, s); /* next point (or the branch) */
            if (t > 0) skip |= dirbit(a, -s);
            const double r = rhs3(g, u, f, i, j, k, skip);
            const double b = diag3(g, i, j, k);
            const double cn = cpl(g, a, s, i, j, k); /* toward t+1 / the branch */
            if (t == 0) {
                bp[t] = b;
                rp[t] = r;
            } else {
                const double am = cpl(g, a, -s, i, j, k); /* toward t-1 */
                if (piv_bad3(bp[t - 1])) return O3_SINGULAR;
                const double w = am / bp[t - 1];
                bp[t] = b - w * cp[t - 1];
                rp[t] = r - w * rp[t - 1];
            }
            cp[t] = cn;
        }
        if (L > 0) {
            const long i = B->si[l] + (a == 0 ? s * (L - 1) : 0);
            const long j = B->sj[l] + (a == 1 ? s * (L - 1) : 0);
            const long k = B->sk[l] + (a == 2 ? s * (L - 1) : 0);
            /* coupling of the branch toward the leg's last point */
            const double d = cpl(g, a, -s, B->bi, B->bj, B->bk);
            (void)i; (void)j; (void)k;
            if (piv_bad3(bp[L - 1])) return O3_SINGULAR;
            num -= d * rp[L - 1] / bp[L - 1];
            den -= d * cp[L - 1] / bp[L - 1];
        }
        off += 3 * L;
    }
    if (piv_bad3(den)) return O3_SINGULAR;
    const double xb = num / den;
    u[IDX(B->bi, B->bj, B->bk)] = xb;
    off = 0;
    for (int l = 0; l < B->nleg; l++) {
        const int a = B->axis[l], s = B->step[l];
        const long L = B->len[l];
        const double *bp = wk + off, *rp = wk + off + L, *cp = wk + off + 2 * L;
        double x = xb;
        for (long t = L - 1; t >= 0; t--) {
            x = (rp[t] - cp[t] * x) / bp[t];
            const long i = B->si[l] + (a == 0 ? s * t : 0);
            const long j = B->sj[l] + (a == 1 ? s * t : 0);
            const long k = B->sk[l] + (a == 2 ? s * t : 0);
            u[IDX(i, j, k)] = x;
        }
        off += 3 * L;
    }
    return O3_OK;
}

/* One 3D tweed sweep (red blocks, then black) */
int orc3_sweep(long n, const double *W, const double *E, const double *S, const double *N,
               const double *Bc, const double *Tc, double *u, const double *f, int nthreads) {
    if (n < 2 || n % 2) return O3_BADARG;
    const Grid3 g = {n, W, E, S, N, Bc, Tc};
    long nb = orc3_blocks(n, NULL, 0);
    O3Block *blocks = (O3Block *)malloc(sizeof(O3Block) * (size_t)(nb > 0 ? nb : 1));
    orc3_blocks(n, blocks, nb);
    int status = O3_OK;
    for (int red = 1; red >= 0; red--) {
#pragma omp parallel num_threads(nthreads) if (nthreads > 1)
        {
            double *wk = (double *)malloc(sizeof(double) * 3 * 6 * (size_t)n);
#pragma omp for schedule(dynamic, 64)
            for (long b = 0; b < nb; b++) {
                if (blocks[b].red != red) continue;
                int st = solve_block(&g, &blocks[b], u, f, wk);
                if (st != O3_OK) {
#pragma omp critical
                    status = st;
                }
            }
            free(wk);
        }
    }
    free(blocks);
    return status;
}

/* Block export for tests: per member point (i, j, k, block, red); legs tip ->
 * branch, then the branch.  Returns the member count. */
long orc3_layout_dump(long n, long *oi, long *oj, long *ok, long *oblk, long *ored, long cap) {
    long nb = orc3_blocks(n, NULL, 0);
    O3Block *blocks = (O3Block *)malloc(sizeof(O3Block) * (size_t)(nb > 0 ? nb : 1));
    orc3_blocks(n, blocks, nb);
    long p = 0;
    for (long b = 0; b < nb; b++) {
        const O3Block *B = &blocks[b];
        for (int l = 0; l <= B->nleg; l++) {
            const long L = l < B->nleg ? B->len[l] : 1;
            for (long t = 0; t < L; t++) {
                long i = B->bi, j = B->bj, k = B->bk;
                if (l < B->nleg) {
                    i = B->si[l] + (B->axis[l] == 0 ? B->step[l] * t : 0);
                    j = B->sj[l] + (B->axis[l] == 1 ? B->step[l] * t : 0);
                    k = B->sk[l] + (B->axis[l] == 2 ? B->step[l] * t : 0);
                }
                if (p < cap) {
                    oi[p] = i; oj[p] = j; ok[p] = k; oblk[p] = b; ored[p] = B->red;
                }
                p++;
            }
        }
    }
    free(blocks);
    return p;
}

/* d = f - L u on the interior, 0 on the boundary */
int orc3_defect(long n, const double *W, const double *E, const double *S, const double *N,
                const double *Bc, const double *Tc, const double *u, const double *f, double *d,
                int nthreads) {
    const size_t tot = (size_t)(n + 1) * (n + 1) * (n + 1);
    memset(d, 0, sizeof(double) * tot);
#pragma omp parallel for num_threads(nthreads) if (nthreads > 1)
    for (long i = 1; i < n; i++)
        for (long j = 1; j < n; j++)
            for (long k = 1; k < n; k++) {
                const double cc = -(W[i] + E[i] + S[j] + N[j] + Bc[k] + Tc[k]);
                double acc = W[i] * u[IDX(i - 1, j, k)];
                acc += E[i] * u[IDX(i + 1, j, k)];
                acc += S[j] * u[IDX(i, j - 1, k)];
                acc += N[j] * u[IDX(i, j + 1, k)];
                acc += Bc[k] * u[IDX(i, j, k - 1)];
                acc += Tc[k] * u[IDX(i, j, k + 1)];
                acc += cc * u[IDX(i, j, k)];
                d[IDX(i, j, k)] = f[IDX(i, j, k)] - acc;
            }
    return O3_OK;
}

/* full weighting: tensor product of [1/4, 1/2, 1/4]; coarse boundary 0 */
int orc3_restrict(long nf, const double *d, double *out) {
    const long nc = nf / 2;
    const size_t totc = (size_t)(nc + 1) * (nc + 1) * (nc + 1);
    memset(out, 0, sizeof(double) * totc);
    const double w[3] = {0.25, 0.5, 0.25};
    for (long I = 1; I < nc; I++)
        for (long J = 1; J < nc; J++)
            for (long K = 1; K < nc; K++) {
                double acc = 0.0;
                for (int a = 0; a < 3; a++)
                    for (int b = 0; b < 3; b++)
                        for (int c = 0; c < 3; c++) {
                            const long n = nf;
                            acc += w[a] * w[b] * w[c] *
                                   d[IDX(2 * I - 1 + a, 2 * J - 1 + b, 2 * K - 1 + c)];
                        }
                const long n = nc;
                out[IDX(I, J, K)] = acc;
            }
    return O3_OK;
}

/* u += P uc on the fine interior (trilinear) */
int orc3_prolong_add(long nc, const double *uc, double *u) {
    const long nf = 2 * nc;
    for (long i = 1; i < nf; i++)
        for (long j = 1; j < nf; j++)
            for (long k = 1; k < nf; k++) {
                const long I = i / 2, J = j / 2, K = k / 2;
                const int oi = i & 1, oj = j & 1, ok = k & 1;
                double acc = 0.0;
                for (int a = 0; a <= oi; a++)
                    for (int b = 0; b <= oj; b++)
                        for (int c = 0; c <= ok; c++) {
                            const long n = nc;
                            acc += uc[IDX(I + a, J + b, K + c)];
                        }
                const double wgt = 1.0 / (double)((1 + oi) * (1 + oj) * (1 + ok));
                const long n = nf;
                u[IDX(i, j, k)] += acc * wgt;
            }
    return O3_OK;
}

/* coarsest level n = 2: one interior unknown */
int orc3_coarse_solve(const double *W, const double *E, const double *S, const double *N,
                      const double *Bc, const double *Tc, double *u, const double *f) {
    const long n = 2;
    const double cc = -(W[1] + E[1] + S[1] + N[1] + Bc[1] + Tc[1]);
    double r = f[IDX(1, 1, 1)] - W[1] * u[IDX(0, 1, 1)] - E[1] * u[IDX(2, 1, 1)] -
               S[1] * u[IDX(1, 0, 1)] - N[1] * u[IDX(1, 2, 1)] - Bc[1] * u[IDX(1, 1, 0)] -
               Tc[1] * u[IDX(1, 1, 2)];
    if (piv_bad3(cc)) return O3_SINGULAR;
    u[IDX(1, 1, 1)] = r / cc;
    return O3_OK;
}
