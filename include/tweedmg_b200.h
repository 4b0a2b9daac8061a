/*
 * tweedmg_b200.h -- C ABI of the B200-native multigrid V-cycle hot path.
 *
 * Drop-in boundary for the reference `tweedmg` package (arXiv 2110.08389).
 * Every entry point is extern "C", takes plain pointers and sizes (device
 * pointers for fields, a cudaStream_t passed as void*), is stream-ordered
 * unless it says "synchronizes", and returns an int status:
 *
 *   TMG_OK        0
 *   TMG_SINGULAR  1  vanishing pivot |p| < 1e-300; the reference raises
 *                    SingularSystemError(ValueError)  (tridiag.py:17-27,
 *                    _ckernels.pyx:11-18)
 *   TMG_BADARG    2  shape / kind / size error; the reference raises
 *                    ValueError (smoothers.py:134-137, stencil.py:70-73,
 *                    transfer.py:13-17, layout.py:50-52)
 *   TMG_CUDA      3  CUDA runtime error
 *
 * tmg_last_error() returns the message of the last failure on the calling
 * thread.  Fields are fp64, C-order (nx+1) x (ny+1), u[i*(ny+1)+j]
 * (stencil.py:12-15).  Coefficients W, E (length nx+1) and S, N (ny+1) are
 * the stencil.assemble arrays (stencil.py:48-67).  Handles are bound to the
 * device current at creation and must not be shared across host threads.
 */
#ifndef TWEEDMG_B200_H
#define TWEEDMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMG_OK 0
#define TMG_SINGULAR 1
#define TMG_BADARG 2
#define TMG_CUDA 3

/* smoother kinds, smoothers.py:18-22 order */
#define TMG_CHECKERBOARD 0
#define TMG_ZEBRA_X 1
#define TMG_ZEBRA_Y 2
#define TMG_ZEBRA_ALT 3
#define TMG_TWEED 4
#define TMG_WIREFRAME 5
#define TMG_TWEED_WIRE_ALT 6

typedef struct tmg_level tmg_level; /* grid level: coefficients, plans, workspace */
typedef struct tmg_hier tmg_hier;   /* V-cycle hierarchy over levels */

const char* tmg_last_error(void);
int tmg_version(void);

/* ---- levels: grid.Level + stencil.StencilCoeffs (grid.py:105-135,
 *      stencil.py:25-67).  W, E, S, N are HOST arrays, copied to the device. */
int tmg_level_create(int nx, int ny, const double* W, const double* E, const double* S,
                     const double* N, tmg_level** out);
int tmg_level_destroy(tmg_level* lv);
/* bytes of device memory held by the level (coefficients + plans) */
long long tmg_level_device_bytes(tmg_level* lv);
/* read and clear the level's device error flags; synchronizes `stream` */
int tmg_level_check(tmg_level* lv, void* stream);

/* ---- smoother: smoothers.sweep (smoothers.py:121-150), in place on u */
int tmg_sweep(tmg_level* lv, int kind, double* u, const double* f, void* stream);
/* one colour stage (red = 1 first, black = 0), test_smoothers.py:27-39 */
int tmg_sweep_colour(tmg_level* lv, int kind, int red, double* u, const double* f,
                     void* stream);

/* ---- stencil.apply / stencil.defect (stencil.py:76-96) */
int tmg_apply(tmg_level* lv, const double* u, double* out, void* stream);
int tmg_defect(tmg_level* lv, const double* u, const double* f, double* d, void* stream);
/* max over the interior of |f - L u| (mgcycle.py:122,130); synchronizes */
int tmg_defect_norm(tmg_level* lv, const double* u, const double* f, double* out_host,
                    void* stream);

/* ---- transfers (transfer.py:21-56); full = 1 full weighting, 0 half */
int tmg_restrict(int nxf, int nyf, int full, const double* d, double* out, void* stream);
int tmg_prolong(int nxc, int nyc, const double* uc, double* v, void* stream);
/* fused: fc = R (f - L u)  (mgcycle.py:98-99) */
int tmg_defect_restrict(tmg_level* fine, int full, const double* u, const double* f,
                        double* fc, void* stream);
/* fused: u += P uc  (mgcycle.py:102) */
int tmg_prolong_correct(int nxc, int nyc, const double* uc, double* u, void* stream);

/* ---- vector helpers of the two-grid analyser (spectral.py:92-120):
 *      out_host = sqrt(sum x^2) in a fixed summation order (work: DEVICE
 *      scratch of >= 1024 doubles; synchronizes); x *= alpha */
int tmg_vec_norm2(const double* x, long n, double* work, double* out_host, void* stream);
int tmg_vec_scale(double* x, long n, double alpha, void* stream);
/* the next n uniform [0, 1) values of the Lcg64 stream (rng.py:20-40) whose
 * current state is `state`, into DEVICE out (per-element jump-ahead; the
 * caller advances its host state by n) */
int tmg_lcg_fill(unsigned long long state, long n, double* out, void* stream);

/* ---- DirectSolver (stencil.py:129-155): factor once, then u_int = L^-1 (f -
 *      boundary couplings of u's ring); u's boundary ring is kept */
int tmg_direct_solve(tmg_level* lv, double* u, const double* f, void* stream);

/* ---- V-cycle hierarchy (mgcycle.py:64-139).  levels[0] is the finest. */
int tmg_hier_create(int nlevels, tmg_level* const* levels, tmg_hier** out);
int tmg_hier_destroy(tmg_hier* h);
/* one V-cycle in place on u (mgcycle.py:80-104) */
int tmg_vcycle(tmg_hier* h, int kind, int full, int nu1, int nu2, double* u, const double* f,
               void* stream);
/* the solve loop from the given u (mgcycle.py:107-139); norms_out (host) gets
 * max_cycles + 1 entries at most; synchronizes once per cycle */
int tmg_solve(tmg_hier* h, int kind, int full, int nu1, int nu2, double tol, int max_cycles,
              double* u, const double* f, double* norms_out, int* cycles_out,
              int* converged_out, void* stream);
/* capture one V-cycle for (u, f) into a CUDA graph and replay it `reps` times */
int tmg_vcycle_graph(tmg_hier* h, int kind, int full, int nu1, int nu2, double* u,
                     const double* f, int reps, void* stream);
/* kernel nodes in the most recently replayed V-cycle graph (launches/cycle) */
int tmg_hier_graph_kernels(tmg_hier* h);
/* bytes of device work fields held by the hierarchy */
long long tmg_hier_device_bytes(tmg_hier* h);

/* ---- solver sessions: the hierarchy keeps u and f of the finest level in
 *      its working layout (the smoother's preferred hybrid N/T layout, see
 *      DESIGN.md) across calls.  tmg_vcycle / tmg_solve are load + cycles +
 *      store on the caller's C-order arrays. */
int tmg_session_load(tmg_hier* h, int kind, const double* u, const double* f, void* stream);
int tmg_session_cycles(tmg_hier* h, int kind, int full, int nu1, int nu2, int reps,
                       void* stream);
/* finest-level max |f - L u| of the session, plus the pivot flags; synchronizes */
int tmg_session_norm(tmg_hier* h, double* out_host, void* stream);
int tmg_session_store(tmg_hier* h, double* u, void* stream);
/* `reps` finest-level sweeps on the session's fields (smoothers.sweep on the
 * solver state; used to time the smoother alone) */
int tmg_session_sweeps(tmg_hier* h, int kind, int reps, void* stream);

/* ---- sharded V-cycle (one process per GPU).
 *      The grid's blocks fall into a chain of sharding groups (tweed L-shells
 *      max(i',j'), wireframe rings min(i',j'), zebra_x rows j, zebra_y and
 *      checkerboard columns i; coarse group G = fine group 2G).  A rank owns a
 *      contiguous group range, sweeps only its blocks and exchanges halo
 *      groups with its neighbours; the replaced reference loop is
 *      mgcycle.py:89-104 with smoothers.py:139-150 split by rank.
 *      Pair kinds (zebra_alt, tweed_wire_alt) do not shard. */
/* number of groups (numbered 1..G), 0 if the kind does not shard; host only */
int tmg_group_count(int kind, int nx, int ny);
/* sizes[g] = interior points of group g, g = 0..G; returns G + 1 (-1: bad kind) */
long tmg_group_sizes(int kind, int nx, int ny, long long* sizes, long cap);
/* encoded work-field positions (2 * element offset + 1 if in the transposed
 * buffer) of the interior points of groups [g0, g1) in C order, in the
 * session layout of `kind`; returns the count (entries beyond cap are not
 * written).  Host only. */
long tmg_group_offsets(int kind, int nx, int ny, int g0, int g1, long long* enc, long cap);
/* one colour stage (red = 1 / black = 0) of the blocks in groups [g0, g1) */
int tmg_session_sweep_part(tmg_hier* h, int level, int kind, int red, int g0, int g1,
                           void* stream);
/* f[level+1] = R (f - L u)[level] and u[level+1] = 0 (mgcycle.py:98-100) */
int tmg_session_restrict(tmg_hier* h, int level, int full, void* stream);
/* one rank's share of the two transfers (sharded V-cycle): the coarse points
 * of sharding groups [cg0, cg1) of `kind` get f = R (f - L u) and u = 0; the
 * fine points of groups [fg0, fg1) get u += P u[level+1] */
int tmg_session_restrict_part(tmg_hier* h, int level, int full, int kind, int cg0, int cg1,
                              void* stream);
int tmg_session_prolong_part(tmg_hier* h, int level, int kind, int fg0, int fg1, void* stream);
/* copy one level's u (which = 0) or f (1) out of the session's layout into a
 * C-order (nx+1) x (ny+1) device array (tests, diagnostics) */
int tmg_session_read(tmg_hier* h, int level, int which, double* out, void* stream);
/* u[level] += P u[level+1] (mgcycle.py:101-102) */
int tmg_session_prolong(tmg_hier* h, int level, void* stream);
/* the V-cycle from `level` down to the coarsest and back (replicated tail) */
int tmg_session_tail(tmg_hier* h, int level, int kind, int full, int nu1, int nu2,
                     void* stream);
/* out[k] = field at enc[k] / field at enc[k] = in[k]; which: 0 u, 1 f;
 * enc, out, in: DEVICE arrays */
int tmg_session_gather(tmg_hier* h, int level, int which, const long long* enc, long n,
                       double* out, void* stream);
int tmg_session_scatter(tmg_hier* h, int level, int which, const long long* enc, long n,
                        const double* in, void* stream);
/* finest-level max |f - L u| over groups [g0, g1) plus the pivot flags of
 * every level; synchronizes */
int tmg_session_norm_part(tmg_hier* h, int kind, int g0, int g1, double* out_host,
                          void* stream);
/* pivot flags of every level; synchronizes */
int tmg_session_check(tmg_hier* h, void* stream);

/* ---- block geometry (layout.py:61-168): per-member (i, j, block, flags) in
 *      the reference's member order (legs tip -> branch then the branch; rings
 *      counter-clockwise from the lower-left point).  flags: bit 0 red,
 *      bits 1-3 leg index (7 = hub / branch / closing point), bits 4-5 block
 *      kind (0 point, 1 line, 2 legged, 3 ring).  Returns the member count, or
 *      -1 on bad dimensions.  Host only; no GPU needed. */
long tmg_layout_dump(int kind, int nx, int ny, int* oi, int* oj, int* oblk, int* oflags,
                     long cap);

/* ---- per-block plugin shims (kernels.active().relax_*, _ckernels.pyx:42-185)
 *      ii, jj, offs: DEVICE int64 arrays; W, E, S, N, u, f: DEVICE arrays */
int tmg_relax_points(long n, const int64_t* ii, const int64_t* jj, int nx, int ny,
                     const double* W, const double* E, const double* S, const double* N,
                     double* u, const double* f, void* stream);
int tmg_relax_chain(long n, const int64_t* ii, const int64_t* jj, int nx, int ny,
                    const double* W, const double* E, const double* S, const double* N,
                    double* u, const double* f, void* stream);
int tmg_relax_ring(long n, const int64_t* ii, const int64_t* jj, int nx, int ny,
                   const double* W, const double* E, const double* S, const double* N,
                   double* u, const double* f, void* stream);
int tmg_relax_legged(long n, const int64_t* ii, const int64_t* jj, long m, const int64_t* offs,
                     long bi, long bj, int nx, int ny, const double* W, const double* E,
                     const double* S, const double* N, double* u, const double* f,
                     void* stream);

/* ---- 3D tweed on cubes (BASELINE config 4; no reference counterpart: the
 *      2D semantics of stencil.py / transfer.py / tridiag.py:84-125 extended
 *      to a third axis on the survey's cube layout).  Fields
 *      are DEVICE (n+1)^3 C-order arrays, k fastest.  x: HOST coordinates
 *      (n+1), used on all three axes. */
typedef struct tmg_cube tmg_cube;
const char* tmg_cube_last_error(void);
int tmg_cube_create(int n, const double* x, tmg_cube** out); /* = scheme 0 */
/* scheme 0: 3D tweed (config 4); 1: 3D wireframe (config 5: shell frames of
 * 12 edges / 8 corners and closed face rings, SURVEY.md §8(c) "Candidate 3D
 * layouts"; the ring solve restates _ckernels.pyx:106-141 per face) */
int tmg_cube_create_scheme(int n, const double* x, int scheme, tmg_cube** out);
int tmg_cube_destroy(tmg_cube* h);
int tmg_cube_levels(tmg_cube* h);
long tmg_cube_blocks(tmg_cube* h, int level, int red);
/* one 3D sweep (red blocks, then black) of the finest level */
int tmg_cube_sweep(tmg_cube* h, double* u, const double* f, void* stream);
int tmg_cube_defect(tmg_cube* h, const double* u, const double* f, double* d, void* stream);
/* session: load u, f; replay V(nu1, nu2) cycles (CUDA graph); norm + pivot
 * flag (synchronizes); store u */
int tmg_cube_load(tmg_cube* h, const double* u, const double* f, void* stream);
int tmg_cube_cycles(tmg_cube* h, int nu1, int nu2, int reps, void* stream);
int tmg_cube_norm(tmg_cube* h, double* out_host, void* stream);
/* mgcycle.py:128-138 in 3D on the device: V(nu1, nu2) cycles of the loaded
 * session until max|f - Lu| <= tol * d0 (d0 from tmg_cube_norm), a non-finite
 * defect, a vanishing pivot (TMG_SINGULAR) or max_cycles; one while-node
 * graph launch, no host round trip per cycle.  norms_out[1..*cycles_out]. */
int tmg_cube_solve_loop(tmg_cube* h, int nu1, int nu2, double d0, double tol, int max_cycles,
                        double* norms_out, int* cycles_out, int* converged_out, void* stream);
int tmg_cube_store(tmg_cube* h, double* u, void* stream);
/* `reps` finest-level sweeps on the session (the smoother alone, on the
 * layout the V-cycle uses: i- / j-contiguous views for the 3D wireframe) */
int tmg_cube_sweeps(tmg_cube* h, int reps, void* stream);

/* ---- sharded cube V-cycle (BASELINE config 5 across GPUs).
 *      Sharding groups 1 .. n/2: 3D wireframe min(i',j',k') (a shell: its
 *      frame, face rings and face centres), 3D tweed max(i',j',k'); a block
 *      never spans two groups, a point's neighbours lie in groups g-1 .. g+1,
 *      coarse group G is fine group 2G.  Same protocol as the 2D
 *      tmg_session_* entry points above (mgcycle.py:89-104 split by rank). */
/* number of groups, 0 for a bad scheme / n; host only */
int tmg_cube_group_count(int scheme, int n);
/* sizes[g] = interior points of group g, g = 0..G; returns G + 1 (-1: bad args) */
long tmg_cube_group_sizes(int scheme, int n, long long* sizes, long cap);
/* element offsets (C order, (n+1)^3 field) of the interior points of groups
 * [g0, g1), increasing; returns the count (entries beyond cap not written) */
long tmg_cube_group_offsets(int scheme, int n, int g0, int g1, long long* off, long cap);
/* one colour stage (red = 1 / black = 0) of the session's level blocks in
 * groups [g0, g1) (3D wireframe only) */
int tmg_cube_sweep_part(tmg_cube* h, int level, int red, int g0, int g1, void* stream);
/* F[level+1] = R (f - L u)[level], U[level+1] = 0 */
int tmg_cube_restrict(tmg_cube* h, int level, void* stream);
/* U[level] += P U[level+1] */
int tmg_cube_prolong(tmg_cube* h, int level, void* stream);
/* the V(nu1, nu2) cycle from `level` down and back (replicated tail) */
int tmg_cube_tail(tmg_cube* h, int level, int nu1, int nu2, void* stream);
/* out[q] = field[off[q]] / field[off[q]] = in[q]; which: 0 u, 1 f;
 * off, out, in: DEVICE arrays */
int tmg_cube_gather(tmg_cube* h, int level, int which, const long long* off, long m, double* out,
                    void* stream);
int tmg_cube_scatter(tmg_cube* h, int level, int which, const long long* off, long m,
                     const double* in, void* stream);
/* finest-level max |f - L u| over groups [g0, g1) + pivot flag; synchronizes */
int tmg_cube_norm_part(tmg_cube* h, int g0, int g1, double* out_host, void* stream);

/* ---- line-solver API (tweedmg.tridiag.thomas / circulant_thomas /
 *      m_legged_thomas, tridiag.py:30-125): HOST arrays, one system per call,
 *      solved on the device in the reference's operation order (results
 *      bit-identical to the reference's numpy code); synchronizes.
 *      TMG_SINGULAR on a vanishing pivot (tridiag.py:23-27), TMG_BADARG on
 *      m < 3 (circulant) / fewer than 2 legs (tridiag.py:56-57, 100-101).
 *      a, b, c, r, x: length m (thomas, circulant; wraparound entries a[0],
 *      c[m-1] as in the reference).  legged: nleg legs packed back to back,
 *      leg k at [offs[k], offs[k+1]) ordered tip -> branch, c at a leg's last
 *      entry couples it to the branch, d[k] the branch row's coupling. */
int tmg_thomas(long m, const double* a, const double* b, const double* c, const double* r,
               double* x, void* stream);
int tmg_circulant_thomas(long m, const double* a, const double* b, const double* c,
                         const double* r, double* x, void* stream);
int tmg_legged_thomas(long nleg, const long* offs, const double* a, const double* b,
                      const double* c, const double* r, const double* d, double d_centre,
                      double r_centre, double* x, double* x_branch, void* stream);

/* ---- profiling aid: average per-CTA cycles between the phase marks of the
 *      block-solver kernel (gather, elimination, reduced solve, hub, finalize,
 *      scatter) over the last launch; non-zero only in builds made with
 *      EXTRA=-DTMG_PHASE_TIMING.  Returns the number of CTAs sampled. */
int tmg_debug_phase_cycles(double* out6);
/* kernels this library has put on streams so far (host-side count; a graph
 * replay adds its kernel nodes) */
long long tmg_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* TWEEDMG_B200_H */
