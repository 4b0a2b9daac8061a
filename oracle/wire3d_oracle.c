/*
 * wire3d_oracle.c -- CPU ORACLE for the 3D wireframe path (BASELINE config 5;
 * test infrastructure only, never the product path).
 *
 * The reference is 2D only ("3D: no oracle, parity
 * unpinned"); this file carries its wireframe semantics to cubes so the
 * device version has a checker:
 *   - operator: the 7-point restatement of stencil.py:43-96 shared with
 *     tweed3d_oracle.c (coefficients B, T along k; u[i][j][k], k fastest);
 *   - blocks: the survey's 3D wireframe layout (SURVEY.md §8(c) "Candidate 3D
 *     layouts"), with s1 <= s2 <= s3 the sorted mirrored coordinates:
 *       s1 == s2      -> the edge frame of shell r = s1: the 12 cube edges of
 *                        the shell [r, n-r]^3 and its 8 corners (degree-3
 *                        vertices); r = c (= n/2) is the centre point;
 *       s1 <  s2      -> ring level t = s2 of the shell-s1 face normal to the
 *                        axis of s1: a closed square ring in that face, or the
 *                        face-centre point when t = c;
 *     colour = parity(s1 + s2), red = even (every frame, the corners);
 *   - ring order: the 2D ring order of layout.py:136-143 in the face's two
 *     in-plane axes (first axis increasing first), solved by the circulant
 *     Thomas of tridiag.py:46-81 / _ckernels.pyx:106-141;
 *   - frame solve (the survey's "reduce to the 8 corner unknowns"): each edge
 *     is eliminated by Thomas with the two corner values kept as columns,
 *     x = alpha + beta * x_start + gamma * x_end; the 8 corner rows form a
 *     dense system (Gaussian elimination, partial pivoting); back
 *     substitution along the edges;
 *   - in-block neighbours are excluded from the frozen right-hand side (the
 *     algebraically identical form SURVEY.md §8(a') allows).
 * Soundness is pinned by property tests (tests/test_3d_wire.py: partition,
 * same-colour independence, one sweep equal to a dense block Gauss-Seidel).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define W3_OK 0
#define W3_SINGULAR 1
#define W3_BADARG 2

static inline long wmir(long x, long n) { return x < n - x ? x : n - x; }
static inline int wbad(double v) { return (-1e-300 < v && v < 1e-300); }

typedef struct {
    long n;
    const double *lo[3], *hi[3]; /* W/S/B and E/N/T */
} WG;

#define WIDX(p) (((size_t)(p)[0] * (size_t)(g->n + 1) + (size_t)(p)[1]) * (size_t)(g->n + 1) + (size_t)(p)[2])

static inline double wcpl(const WG *g, int a, int s, const long *p) {
    return s < 0 ? g->lo[a][p[a]] : g->hi[a][p[a]];
}

static inline double wdiag(const WG *g, const long *p) {
    return -(g->lo[0][p[0]] + g->hi[0][p[0]] + g->lo[1][p[1]] + g->hi[1][p[1]] +
             g->lo[2][p[2]] + g->hi[2][p[2]]);
}

static inline unsigned wbit(int a, int s) { return 1u << (2 * a + (s > 0 ? 1 : 0)); }

/* f - sum of the neighbours not in `skip` (bit 2a + (s > 0)), in the order
 * W E S N B T of tweed3d_oracle.c */
static double wrhs(const WG *g, const double *u, const double *f, const long *p, unsigned skip) {
    double r = f[WIDX(p)];
    for (int a = 0; a < 3; a++)
        for (int s = -1; s <= 1; s += 2) {
            if (skip & wbit(a, s)) continue;
            long q[3] = {p[0], p[1], p[2]};
            q[a] += s;
            r -= wcpl(g, a, s, p) * u[WIDX(q)];
        }
    return r;
}

/* the in-face axes (b, c) of a face normal to axis a, in increasing order */
static inline void face_axes(int a, int *b, int *c) {
    *b = a == 0 ? 1 : 0;
    *c = a == 2 ? 1 : 2;
}

/* Point p of the ring (a, xa, t) at ring position q (0 <= q < 4m, m = n - 2t):
 * layout.py:136-143 in the (b, c) plane: start (t, t), b increasing, then c
 * increasing, b decreasing, c decreasing, ending at (t, t + 1). */
static void ring_point(long n, int a, long xa, long t, long q, long *p) {
    int b, c;
    face_axes(a, &b, &c);
    const long m = n - 2 * t, s = q / m, o = q - s * m;
    long pb, pc;
    if (s == 0) { pb = t + o; pc = t; }
    else if (s == 1) { pb = n - t; pc = t + o; }
    else if (s == 2) { pb = n - t - o; pc = n - t; }
    else { pb = t; pc = n - t - o; }
    p[a] = xa;
    p[b] = pb;
    p[c] = pc;
}

/* direction (axis, step) from point q of a ring to point q2 (a neighbour) */
static void step_dir(const long *p, const long *p2, int *ax, int *st) {
    for (int a = 0; a < 3; a++)
        if (p[a] != p2[a]) {
            *ax = a;
            *st = p2[a] > p[a] ? 1 : -1;
            return;
        }
    *ax = 0;
    *st = 0;
}

/* circulant Thomas on the ring (_ckernels.pyx:106-141, tridiag.py:46-81) */
static int solve_ring(const WG *g, int a, long xa, long t, double *u, const double *f,
                      double *wk) {
    const long n = g->n, m = 4 * (n - 2 * t), mm = m - 1;
    double *A = wk, *Bd = wk + m, *C = wk + 2 * m, *R = wk + 3 * m;
    double *G = wk + 4 * m, *Y = wk + 5 * m, *Z = wk + 6 * m;
    for (long q = 0; q < m; q++) {
        long p[3], pp[3], pn[3];
        ring_point(n, a, xa, t, q, p);
        ring_point(n, a, xa, t, (q + m - 1) % m, pp);
        ring_point(n, a, xa, t, (q + 1) % m, pn);
        int ap, sp, an, sn;
        step_dir(p, pp, &ap, &sp);
        step_dir(p, pn, &an, &sn);
        A[q] = wcpl(g, ap, sp, p);
        C[q] = wcpl(g, an, sn, p);
        Bd[q] = wdiag(g, p);
        R[q] = wrhs(g, u, f, p, wbit(ap, sp) | wbit(an, sn));
    }
    for (long k = 0; k < mm; k++) G[k] = 0.0;
    G[0] = A[0];
    G[mm - 1] += C[mm - 1];
    for (long k = 1; k < mm; k++) {
        if (wbad(Bd[k - 1])) return W3_SINGULAR;
        const double w = A[k] / Bd[k - 1];
        Bd[k] -= w * C[k - 1];
        R[k] -= w * R[k - 1];
        G[k] -= w * G[k - 1];
    }
    if (wbad(Bd[mm - 1])) return W3_SINGULAR;
    Y[mm - 1] = R[mm - 1] / Bd[mm - 1];
    Z[mm - 1] = G[mm - 1] / Bd[mm - 1];
    for (long k = mm - 2; k >= 0; k--) {
        Y[k] = (R[k] - C[k] * Y[k + 1]) / Bd[k];
        Z[k] = (G[k] - C[k] * Z[k + 1]) / Bd[k];
    }
    const double den = Bd[mm] - C[mm] * Z[0] - A[mm] * Z[mm - 1];
    if (wbad(den)) return W3_SINGULAR;
    const double xm = (R[mm] - C[mm] * Y[0] - A[mm] * Y[mm - 1]) / den;
    for (long k = 0; k < m; k++) {
        long p[3];
        ring_point(n, a, xa, t, k, p);
        u[WIDX(p)] = k < mm ? Y[k] - Z[k] * xm : xm;
    }
    return W3_OK;
}

static int solve_point(const WG *g, const long *p, double *u, const double *f) {
    const double d = wdiag(g, p);
    if (wbad(d)) return W3_SINGULAR;
    u[WIDX(p)] = wrhs(g, u, f, p, 0u) / d;
    return W3_OK;
}

/* corner K (bit a set: coordinate n - r on axis a, else r) */
static inline void corner_point(long n, long r, int K, long *p) {
    for (int a = 0; a < 3; a++) p[a] = (K >> a) & 1 ? n - r : r;
}

/* edge e = 4 x + h: along axis x, the other two axes (in increasing order) at
 * bit 0 / bit 1 of h; from the corner with bit x clear to the one with it set */
static inline void edge_corners(int e, int *x, int *K0, int *K1) {
    const int ax = e / 4, h = e % 4;
    int o1, o2;
    face_axes(ax, &o1, &o2);
    const int base = ((h & 1) << o1) | (((h >> 1) & 1) << o2);
    *x = ax;
    *K0 = base;
    *K1 = base | (1 << ax);
}

/* The edge frame of shell r (1 <= r < c): 12 edges of e = n - 2r - 1 points. */
static int solve_frame(const WG *g, long r, double *u, const double *f, double *wk) {
    const long n = g->n, e = n - 2 * r - 1;
    /* per edge: alpha, beta, gamma, pivots (4 e) */
    double M[8][9];
    memset(M, 0, sizeof(M));
    for (int K = 0; K < 8; K++) {
        long p[3];
        corner_point(n, r, K, p);
        unsigned skip = 0;
        for (int a = 0; a < 3; a++) skip |= wbit(a, (K >> a) & 1 ? -1 : 1);
        M[K][K] = wdiag(g, p);
        M[K][8] = wrhs(g, u, f, p, skip);
    }
    for (int ed = 0; ed < 12; ed++) {
        int x, K0, K1;
        edge_corners(ed, &x, &K0, &K1);
        double *al = wk + (size_t)ed * 4 * e, *be = al + e, *ga = be + e, *bp = ga + e;
        long p0[3];
        corner_point(n, r, K0, p0);
        /* forward: rho in al, lambda (x_start column) in be */
        double cprev = 0.0;
        for (long k = 0; k < e; k++) {
            long p[3] = {p0[0], p0[1], p0[2]};
            p[x] = r + 1 + k;
            const double am = wcpl(g, x, -1, p), cn = wcpl(g, x, 1, p);
            const double b = wdiag(g, p);
            const double rr = wrhs(g, u, f, p, wbit(x, -1) | wbit(x, 1));
            if (k == 0) {
                bp[k] = b;
                al[k] = rr;
                be[k] = -am;
            } else {
                if (wbad(bp[k - 1])) return W3_SINGULAR;
                const double w = am / bp[k - 1];
                bp[k] = b - w * cprev;
                al[k] = rr - w * al[k - 1];
                be[k] = -w * be[k - 1];
            }
            cprev = cn;
            ga[k] = cn; /* c_k, replaced by gamma in the back pass */
        }
        /* back: x_k = alpha_k + beta_k x_start + gamma_k x_end */
        for (long k = e - 1; k >= 0; k--) {
            if (wbad(bp[k])) return W3_SINGULAR;
            const double ck = ga[k];
            if (k == e - 1) {
                al[k] = al[k] / bp[k];
                be[k] = be[k] / bp[k];
                ga[k] = -ck / bp[k];
            } else {
                al[k] = (al[k] - ck * al[k + 1]) / bp[k];
                be[k] = (be[k] - ck * be[k + 1]) / bp[k];
                ga[k] = -ck * ga[k + 1] / bp[k];
            }
        }
        /* corner rows: K0's neighbour is the first edge point, K1's the last */
        long q0[3], q1[3];
        corner_point(n, r, K0, q0);
        corner_point(n, r, K1, q1);
        const double c0 = wcpl(g, x, 1, q0), c1 = wcpl(g, x, -1, q1);
        M[K0][K0] += c0 * be[0];
        M[K0][K1] += c0 * ga[0];
        M[K0][8] -= c0 * al[0];
        M[K1][K0] += c1 * be[e - 1];
        M[K1][K1] += c1 * ga[e - 1];
        M[K1][8] -= c1 * al[e - 1];
    }
    /* Gaussian elimination with partial pivoting on the 8 corner rows */
    for (int col = 0; col < 8; col++) {
        int piv = col;
        for (int rr = col + 1; rr < 8; rr++)
            if (fabs(M[rr][col]) > fabs(M[piv][col])) piv = rr;
        if (wbad(M[piv][col])) return W3_SINGULAR;
        if (piv != col)
            for (int q = 0; q < 9; q++) {
                const double tmp = M[col][q];
                M[col][q] = M[piv][q];
                M[piv][q] = tmp;
            }
        for (int rr = col + 1; rr < 8; rr++) {
            const double w = M[rr][col] / M[col][col];
            for (int q = col; q < 9; q++) M[rr][q] -= w * M[col][q];
        }
    }
    double xc[8];
    for (int rr = 7; rr >= 0; rr--) {
        double s = M[rr][8];
        for (int q = rr + 1; q < 8; q++) s -= M[rr][q] * xc[q];
        xc[rr] = s / M[rr][rr];
    }
    for (int K = 0; K < 8; K++) {
        long p[3];
        corner_point(n, r, K, p);
        u[WIDX(p)] = xc[K];
    }
    for (int ed = 0; ed < 12; ed++) {
        int x, K0, K1;
        edge_corners(ed, &x, &K0, &K1);
        const double *al = wk + (size_t)ed * 4 * e, *be = al + e, *ga = be + e;
        long p0[3];
        corner_point(n, r, K0, p0);
        for (long k = 0; k < e; k++) {
            long p[3] = {p0[0], p0[1], p0[2]};
            p[x] = r + 1 + k;
            u[WIDX(p)] = al[k] + be[k] * xc[K0] + ga[k] * xc[K1];
        }
    }
    return W3_OK;
}

/* Block list: kind 0 = frame (r), 1 = ring (a, xa, t), 2 = point (i, j, k). */
typedef struct {
    int kind, red, a;
    long x0, x1, x2;
} WBlock;

long orcw3_blocks(long n, WBlock *out, long cap) {
    const long c = n / 2;
    long nb = 0;
#define PUSH(K, RED, A, X0, X1, X2)                                   \
    do {                                                              \
        if (nb < cap) {                                               \
            WBlock *B_ = &out[nb];                                    \
            B_->kind = (K); B_->red = (RED); B_->a = (A);             \
            B_->x0 = (X0); B_->x1 = (X1); B_->x2 = (X2);              \
        }                                                             \
        nb++;                                                         \
    } while (0)
    for (long r = 1; r < c; r++) PUSH(0, 1, 0, r, 0, 0);
    PUSH(2, 1, 0, c, c, c); /* the centre: frame of shell c */
    for (int a = 0; a < 3; a++)
        for (int side = 0; side < 2; side++)
            for (long s1 = 1; s1 < c; s1++) {
                const long xa = side ? n - s1 : s1;
                for (long t = s1 + 1; t <= c; t++) {
                    const int red = ((s1 + t) % 2) == 0;
                    if (t < c) {
                        PUSH(1, red, a, xa, t, s1);
                    } else {
                        long p[3];
                        p[a] = xa;
                        int b, cc;
                        face_axes(a, &b, &cc);
                        p[b] = c;
                        p[cc] = c;
                        PUSH(2, red, 0, p[0], p[1], p[2]);
                    }
                }
            }
#undef PUSH
    return nb;
}

static int solve_wblock(const WG *g, const WBlock *B, double *u, const double *f, double *wk) {
    if (B->kind == 0) return solve_frame(g, B->x0, u, f, wk);
    if (B->kind == 1) return solve_ring(g, B->a, B->x0, B->x1, u, f, wk);
    const long p[3] = {B->x0, B->x1, B->x2};
    return solve_point(g, p, u, f);
}

/* One 3D wireframe sweep (red blocks, then black) */
int orcw3_sweep(long n, const double *W, const double *E, const double *S, const double *N,
                const double *Bc, const double *Tc, double *u, const double *f, int nthreads) {
    if (n < 2 || n % 2) return W3_BADARG;
    const WG g = {n, {W, S, Bc}, {E, N, Tc}};
    const long nb = orcw3_blocks(n, NULL, 0);
    WBlock *blocks = (WBlock *)malloc(sizeof(WBlock) * (size_t)(nb > 0 ? nb : 1));
    orcw3_blocks(n, blocks, nb);
    int status = W3_OK;
    for (int red = 1; red >= 0; red--) {
#pragma omp parallel num_threads(nthreads) if (nthreads > 1)
        {
            double *wk = (double *)malloc(sizeof(double) * 48 * (size_t)(n + 1));
#pragma omp for schedule(dynamic, 16)
            for (long b = 0; b < nb; b++) {
                if (blocks[b].red != red) continue;
                const int st = solve_wblock(&g, &blocks[b], u, f, wk);
                if (st != W3_OK) {
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

/* One colour stage (red = 1 / black = 0) of the blocks whose sharding group
 * lies in [g0, g1): group = min(i', j', k') of the block's points (the
 * shell: frame r, the rings and face centres of shell s1, the centre c).
 * The rank-local sweep of the sharded V-cycle. */
int orcw3_sweep_part(long n, const double *W, const double *E, const double *S, const double *N,
                     const double *Bc, const double *Tc, double *u, const double *f, int red,
                     long g0, long g1) {
    if (n < 2 || n % 2) return W3_BADARG;
    const WG g = {n, {W, S, Bc}, {E, N, Tc}};
    const long nb = orcw3_blocks(n, NULL, 0);
    WBlock *blocks = (WBlock *)malloc(sizeof(WBlock) * (size_t)(nb > 0 ? nb : 1));
    orcw3_blocks(n, blocks, nb);
    double *wk = (double *)malloc(sizeof(double) * 48 * (size_t)(n + 1));
    int status = W3_OK;
    for (long b = 0; b < nb; b++) {
        const WBlock *B = &blocks[b];
        if (B->red != red) continue;
        long grp;
        if (B->kind == 0) grp = B->x0;                 /* frame r */
        else if (B->kind == 1) grp = B->x2;            /* ring of shell s1 */
        else {                                         /* point: min mirrored coordinate */
            const long m0 = wmir(B->x0, n), m1 = wmir(B->x1, n), m2 = wmir(B->x2, n);
            grp = m0 < m1 ? (m0 < m2 ? m0 : m2) : (m1 < m2 ? m1 : m2);
        }
        if (grp < g0 || grp >= g1) continue;
        const int st = solve_wblock(&g, B, u, f, wk);
        if (st != W3_OK) status = st;
    }
    free(wk);
    free(blocks);
    return status;
}

/* Block export for tests: per member point (i, j, k, block, red); frames list
 * their corners then edges, rings in ring order.  Returns the member count. */
long orcw3_layout_dump(long n, long *oi, long *oj, long *ok, long *oblk, long *ored, long cap) {
    const long nb = orcw3_blocks(n, NULL, 0);
    WBlock *blocks = (WBlock *)malloc(sizeof(WBlock) * (size_t)(nb > 0 ? nb : 1));
    orcw3_blocks(n, blocks, nb);
    long q = 0;
#define EMIT(P)                                                      \
    do {                                                             \
        if (q < cap) {                                               \
            oi[q] = (P)[0]; oj[q] = (P)[1]; ok[q] = (P)[2];          \
            oblk[q] = b; ored[q] = B->red;                           \
        }                                                            \
        q++;                                                         \
    } while (0)
    for (long b = 0; b < nb; b++) {
        const WBlock *B = &blocks[b];
        if (B->kind == 0) {
            const long r = B->x0, e = n - 2 * r - 1;
            for (int K = 0; K < 8; K++) {
                long p[3];
                corner_point(n, r, K, p);
                EMIT(p);
            }
            for (int ed = 0; ed < 12; ed++) {
                int x, K0, K1;
                edge_corners(ed, &x, &K0, &K1);
                long p[3];
                corner_point(n, r, K0, p);
                for (long k = 0; k < e; k++) {
                    p[x] = r + 1 + k;
                    EMIT(p);
                }
            }
        } else if (B->kind == 1) {
            const long m = 4 * (n - 2 * B->x1);
            for (long k = 0; k < m; k++) {
                long p[3];
                ring_point(n, B->a, B->x0, B->x1, k, p);
                EMIT(p);
            }
        } else {
            const long p[3] = {B->x0, B->x1, B->x2};
            EMIT(p);
        }
    }
#undef EMIT
    free(blocks);
    return q;
}
