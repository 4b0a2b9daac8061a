// Tweed L-shell colour stage on sm_100a: a persistent, TMA-fed block solver
// for the two-legged blocks of square tweed grids in the hybrid layout
// (tmg_layout.h, LM_TWEED).  Same exact block Gauss-Seidel as
// relax_legged (_ckernels.pyx:144-185) / m_legged_thomas (tridiag.py:84-125)
// on the L-shell blocks of tweed_layout (layout.py:75-84): every leg of a
// shell is one contiguous run of its owner buffer (x-legs in T, y-legs in N),
// and its two cross-neighbour runs are the adjacent rows of the same buffer.
//
// Work split (host, build_leg_plan): blocks of shells k in [kLegK0, c) are
// packed into items of <= 256 chunks of 17 points (a chunk per thread, legs
// never split across CTAs); a block whose legs exceed 128 chunks each is
// split over the two CTAs of a cluster (one leg each, the branch row
// exchanged through DSMEM).  Clusters walk a static item schedule.
//
// Per item (one CTA):
//   TMA     one thread issues cp.async.bulk copies of every leg's f run and
//           its two u cross-neighbour runs into a shared stage (two stages:
//           the next item streams in while this one is solved);
//   chunk   per thread, in registers: frozen RHS r = f - cross couplings
//           (_ckernels.pyx:34-39), Thomas down sweep and an affine back pass
//           leaving x_k = alpha_k + beta_k X_left + gamma_k X (X = the chunk's
//           last point); along couplings from a chunk-permuted coefficient
//           copy (one coalesced 16-byte load per point, no staging);
//   reduced the chunk ends of each leg form a tridiagonal system with the
//           branch as a second right-hand side, solved by parallel cyclic
//           reduction in shared memory;
//   branch  one scalar row per block (m_legged_thomas's branch equation);
//   store   finalize in registers, stage through shared memory, coalesced
//           stores.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tmg_kernels.h"
#include "tmg_tweedleg.h"

namespace cg = cooperative_groups;

// -DTMG_CHECK (make check): device-side bounds checks on every shared-memory
// slot a chunk, a bulk copy or the reduced system touches, and on the global
// offsets of the branch and boundary loads.  A failed check prints and traps
// (the launch fails loudly).  compute-sanitizer is not available on the GPU
// pool; this build is its stand-in (profiles/r02_boundscheck.txt).
#ifdef TMG_CHECK
#define LEGK_CHECK(cond, what)                                                             \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("leg kernel check failed: %s (block %d thread %d)\n", what, (int)blockIdx.x, \
             (int)threadIdx.x);                                                            \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define LEGK_CHECK(cond, what) \
  do {                         \
  } while (0)
#endif

#ifndef TMG_LEGK_SPLITISSUE
#define TMG_LEGK_SPLITISSUE 1  // 0: warp 0 alone issues an item's stores and the next item's loads
#endif

namespace tmg {

namespace {

constexpr int LQ = kLegQ;         // points per thread chunk (odd: conflict-free
                                  // per-thread shared-memory rows)
constexpr int LT = kLegThreads;   // threads per CTA
constexpr int LCAP = LT * LQ;     // points per item

__device__ __forceinline__ bool bad_pivot(double v) { return v > -1e-300 && v < 1e-300; }

// the ~20-bit hardware reciprocal refined by two Newton steps (== 1.0 / x,
// tmg_sweep.cu)
__device__ __forceinline__ double drcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ unsigned mapa_u32(const void* p, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_v2(unsigned addr, double x, double y) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(unsigned addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Geometry of one leg of the L-shell block (k, quad) of an n x n grid
// (layout.py:75-84; quad bit 0: the block's corner is at i = n-1, bit 1: at
// j = n-1).  Leg 0 (x-leg) lives in T row bj, leg 1 (y-leg) in N row bi; both
// run tip -> branch with point e at position p0 + dir * e of their row.
struct LegGeo {
  int m, dir, p0, row, orient, sx, sy, bi, bj;
  __device__ __forceinline__ void set(int k, int quad, int leg, int n) {
    sx = (quad & 1) ? -1 : 1;
    sy = (quad & 2) ? -1 : 1;
    const int x0 = sx > 0 ? 1 : n - 1, y0 = sy > 0 ? 1 : n - 1;
    bi = x0 + sx * (k - 1);
    bj = y0 + sy * (k - 1);
    m = k - 1;
    if (leg == 0) {
      dir = sx;
      p0 = x0;
      row = bj;
      orient = sx > 0 ? 0 : 1;
    } else {
      dir = sy;
      p0 = y0;
      row = bi;
      orient = sy > 0 ? 2 : 3;
    }
  }
};

// issue an item's bulk loads from its descriptor blob in shared memory (one
// warp).  part -1: everything; 0: the u rows; 1: the f runs.  The stage
// barrier counts one arrival per part (-1 arrives for both).
__device__ __forceinline__ void issue_loads_blob(const LegArgs& a, const unsigned char* blob,
                                                 double* stage, uint64_t* bar, int part = -1) {
  const int lane = threadIdx.x & 31;
  const LegBlobHead* hd = reinterpret_cast<const LegBlobHead*>(blob);
  const LegCopy* cps = reinterpret_cast<const LegCopy*>(blob + sizeof(LegBlobHead));
  const int ncopy = hd->ncopy;
  if (lane == 0) {
#if TMG_LEGK_SPLITISSUE
    if (part != 1) mbar_expect_tx(bar, (unsigned)(hd->bytes - hd->bytes_f));
    if (part != 0) mbar_expect_tx(bar, (unsigned)hd->bytes_f);
#else
    mbar_expect_tx(bar, (unsigned)hd->bytes);
#endif
  }
  __syncwarp();
  for (int c = lane; c < ncopy; c += 32) {
    const LegCopy cp = cps[c];
    if (part >= 0 && (cp.s < kLegArrF) != (part == 1)) continue;
    const double* src = cp.src == 0 ? a.fn : cp.src == 1 ? a.ft : cp.src == 2 ? a.un : a.ut;
    LEGK_CHECK(cp.s >= 0 && cp.n > 0 && cp.g >= 0 && (cp.s & 1) == 0 && (cp.g & 1) == 0 &&
                   (cp.s < kLegArrF ? cp.s + cp.n <= kLegArrF
                                    : cp.s + cp.n <= kLegArrF + 2 * kLegArrU &&
                                          (cp.s >= kLegArrF + kLegArrU ||
                                           cp.s + cp.n <= kLegArrF + kLegArrU)) &&
                   cp.g + cp.n <= (long)a.ld * a.ld,
               "bulk load range");
    bulk_g2s(stage + cp.s, src + cp.g, (unsigned)cp.n * 8u, bar);
  }
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

#ifndef TMG_LEGK_L2PF
#define TMG_LEGK_L2PF 1  // 1: warp 0 prefetches the next item's runs into L2 while this one is solved
#endif
#ifndef TMG_LEGK_BLOBPF
#define TMG_LEGK_BLOBPF 0  // 1: L2 prefetch of the CTA's descriptor blobs at kernel start (measured: no gain)
#endif
#ifndef TMG_LEGK_STAGGER
#define TMG_LEGK_STAGGER 0  // > 0: odd clusters start late by this many units of 1024 ns
#endif
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// warp 0: the bulk loads an item's blob lists, as L2 prefetches
__device__ __forceinline__ void prefetch_loads_blob(const LegArgs& a, const unsigned char* blob) {
  const int lane = threadIdx.x & 31;
  const LegBlobHead* hd = reinterpret_cast<const LegBlobHead*>(blob);
  const LegCopy* cps = reinterpret_cast<const LegCopy*>(blob + sizeof(LegBlobHead));
  const int ncopy = hd->ncopy;
  for (int c = lane; c < ncopy; c += 32) {
    const LegCopy cp = cps[c];
    const double* src = cp.src == 0 ? a.fn : cp.src == 1 ? a.ft : cp.src == 2 ? a.un : a.ut;
    bulk_prefetch_l2(src + cp.g, (unsigned)cp.n * 8u);
  }
}

// One thread's chunk of 17 consecutive leg points: point k's f slot is
// pF[DIR * k] (also the chunk's scratch: rho / p, then alpha, then the
// solution), its u neighbours pL / pH[DIR * k] and its couplings
// pc[32 * k] = (a, c) toward the previous / next point (the diagonal is
// -(a + c + cross couplings)).  The tip chunk holds `pad` dummy points in
// front of the tip with couplings (1e300, 0): their reciprocal pivots vanish,
// so the tip is decoupled from them (its Dirichlet neighbour is folded into
// f) and they only touch the private gap the plan leaves before the tip's f
// slot.  Every chunk is therefore full and the leg's last chunk ends on the
// leg's last point.
//
// The forward pass keeps, per interior point k, the pivot-scaled data
// rho_k / p_k (f slot), lam_k / p_k and c_k / p_k (registers), so the back
// pass needs no coefficient reload: x_k = alpha_k + be_k * Xleft + ga_k * X
// (k < 16, X = point 16) with alpha in the f slots.
struct ChunkOut {
  double ad, bd, gd;  // form of point 15
  double au, bu, gu;  // form of point 0
  double a_end, c_end, r_end;
  int phi;            // smallest high word of |pivot| (vanishing-pivot check)
};

struct CoefSrc {
  const double2* __restrict__ p;  // chunk-permuted table, point k at p[32 k]
};
__device__ __forceinline__ double2 coef_at(const CoefSrc& c, int k) { return __ldg(c.p + 32 * k); }

template <int DIR>
__device__ __forceinline__ void chunk_forward(double* __restrict__ pF,
                                              const double* __restrict__ pL,
                                              const double* __restrict__ pH,
                                              const CoefSrc& pc, double clo,
                                              double chi, bool first, int wallfix, double uwall,
                                              double uwall2,
                                              double (&lam)[LQ - 1], double (&cg_)[LQ - 1],
                                              ChunkOut& o) {
  const double csum = clo + chi;
  double ivp = 0.0, rho = 0.0, lm = 0.0, cprev = 0.0;
  int phi = 0x7fffffff;
#pragma unroll
  for (int k = 0; k < LQ - 1; k++) {
    const double r = fma(-chi, pH[DIR * k], fma(-clo, pL[DIR * k], pF[DIR * k]));
    const double2 ac = coef_at(pc, k);
    const double bb = -(ac.x + ac.y + csum);
    double bp;
    if (k == 0) {
      bp = bb;
      rho = r;
      lm = first ? 0.0 : -ac.x;
    } else {
      const double w = ac.x * ivp;
      bp = fma(-w, cprev, bb);
      rho = fma(-w, rho, r);
      lm = -w * lm;
    }
    phi = min(phi, __double2hiint(bp) & 0x7fffffff);
    ivp = drcp(bp);
    pF[DIR * k] = rho * ivp;
    lam[k] = lm * ivp;
    cg_[k] = ac.y * ivp;
    cprev = ac.y;
  }
  constexpr int k = LQ - 1;  // the chunk-end row
  double r;
  if (!wallfix) {
    r = fma(-chi, pH[DIR * k], fma(-clo, pL[DIR * k], pF[DIR * k]));
  } else {  // x-leg's last point: its wall-side cross neighbour is an N-owned branch
    // 1: the u-1 side, 2: the u+1 side, 3: both (the cross's x-legs)
    const double ul = wallfix == 2 ? pL[DIR * k] : uwall;
    const double uh = wallfix == 1 ? pH[DIR * k] : wallfix == 2 ? uwall : uwall2;
    r = pF[DIR * k] - clo * ul - chi * uh;
  }
  const double2 ac = coef_at(pc, k);
  o.a_end = ac.x;
  o.c_end = ac.y;
  o.r_end = r;
  o.phi = phi;
}

// affine back pass: alpha into the f slots, beta into the thread's row of
// the scratch (stride 17: conflict-free), gamma in place of c / p
template <int DIR>
__device__ __forceinline__ void chunk_back(double* __restrict__ pF, double* __restrict__ sb,
                                           const double (&lam)[LQ - 1], double (&ga)[LQ - 1],
                                           ChunkOut& o) {
  double A_ = pF[DIR * (LQ - 2)];
  double B_ = lam[LQ - 2];
  double G_ = -ga[LQ - 2];
  o.ad = A_;
  o.bd = B_;
  o.gd = G_;
  sb[LQ - 2] = B_;
  ga[LQ - 2] = G_;
#pragma unroll
  for (int k = LQ - 3; k >= 0; k--) {
    const double g = ga[k];
    A_ = fma(-g, A_, pF[DIR * k]);
    B_ = fma(-g, B_, lam[k]);
    G_ = -g * G_;
    pF[DIR * k] = A_;
    sb[k] = B_;
    ga[k] = G_;
  }
  o.au = A_;
  o.bu = B_;
  o.gu = G_;
}

// Twisted (two-ended) chunk elimination, TMG_LEGK_TWIST: the same exact
// solve of the chunk's 16 interior rows as chunk_forward / chunk_back, but
// eliminated from both ends at once so every thread runs two independent
// 8-step chains (twice the ILP of the one-ended sweep, the forward / back
// phases being latency-bound).  Top rows k = 0..7 go down as above
// (f slot rho_k / p_k, lam_k = coefficient of X_left / p_k, ga_k = c_k / p_k);
// bottom rows k = 15..8 go up (f slot sig_k / q_k, lam_k = coefficient of X
// / q_k, ga_k = a_k / q_k).  Rows 7 and 8 meet in a 2 x 2 step scaled by
// s = 1 / (1 - (a_8 / q_8)(c_7 / p_7)) (no determinant: the tip dummies'
// 1e300 pivots cannot overflow it), then both halves back-substitute outward.
template <int DIR>
__device__ __forceinline__ void chunk_forward_tw(double* __restrict__ pF,
                                                 const double* __restrict__ pL,
                                                 const double* __restrict__ pH,
                                                 const CoefSrc& pc, double clo, double chi,
                                                 bool first, int wallfix, double uwall,
                                                 double uwall2, double (&lam)[LQ - 1],
                                                 double (&cg_)[LQ - 1], ChunkOut& o) {
  constexpr int H = (LQ - 1) / 2;  // rows per half
  const double csum = clo + chi;
  double ivp = 0.0, rho = 0.0, lm = 0.0, cprev = 0.0;
  double ivq = 0.0, sig = 0.0, mu = 0.0, anext = 0.0;
  int phi = 0x7fffffff;
#pragma unroll
  for (int j = 0; j < H; j++) {
    const int kt = j, kb = LQ - 2 - j;
    const double2 act = coef_at(pc, kt);
    const double2 acb = coef_at(pc, kb);
    const double rt = fma(-chi, pH[DIR * kt], fma(-clo, pL[DIR * kt], pF[DIR * kt]));
    const double rb = fma(-chi, pH[DIR * kb], fma(-clo, pL[DIR * kb], pF[DIR * kb]));
    const double bbt = -(act.x + act.y + csum);
    const double bbb = -(acb.x + acb.y + csum);
    double bp, bq;
    if (j == 0) {
      bp = bbt;
      rho = rt;
      lm = first ? 0.0 : -act.x;
      bq = bbb;
      sig = rb;
      mu = -acb.y;
    } else {
      const double w = act.x * ivp;
      bp = fma(-w, cprev, bbt);
      rho = fma(-w, rho, rt);
      lm = -w * lm;
      const double v = acb.y * ivq;
      bq = fma(-v, anext, bbb);
      sig = fma(-v, sig, rb);
      mu = -v * mu;
    }
    phi = min(phi, min(__double2hiint(bp) & 0x7fffffff, __double2hiint(bq) & 0x7fffffff));
    ivp = drcp(bp);
    ivq = drcp(bq);
    pF[DIR * kt] = rho * ivp;
    lam[kt] = lm * ivp;
    cg_[kt] = act.y * ivp;
    cprev = act.y;
    pF[DIR * kb] = sig * ivq;
    lam[kb] = mu * ivq;
    cg_[kb] = acb.x * ivq;
    anext = acb.x;
  }
  constexpr int k = LQ - 1;  // the chunk-end row
  double r;
  if (!wallfix) {
    r = fma(-chi, pH[DIR * k], fma(-clo, pL[DIR * k], pF[DIR * k]));
  } else {
    const double ul = wallfix == 2 ? pL[DIR * k] : uwall;
    const double uh = wallfix == 1 ? pH[DIR * k] : wallfix == 2 ? uwall : uwall2;
    r = pF[DIR * k] - clo * ul - chi * uh;
  }
  const double2 ac = coef_at(pc, k);
  o.a_end = ac.x;
  o.c_end = ac.y;
  o.r_end = r;
  o.phi = phi;
}

template <int DIR>
__device__ __forceinline__ void chunk_back_tw(double* __restrict__ pF, double* __restrict__ sb,
                                              const double (&lam)[LQ - 1], double (&ga)[LQ - 1],
                                              ChunkOut& o) {
  constexpr int H = (LQ - 1) / 2;
  // rows H-1 and H: x_H = sig_H + mu_H X - ag_H x_{H-1},
  //                 x_{H-1} = rho_{H-1} + lam_{H-1} XL - cg_{H-1} x_H
  const double agm = ga[H], cgm = ga[H - 1];
  const double den = fma(-agm, cgm, 1.0);
  const double s = drcp(den);
  o.phi = min(o.phi, __double2hiint(den) & 0x7fffffff);
  const double rt = pF[DIR * (H - 1)];
  const double Am = s * fma(-agm, rt, pF[DIR * H]);
  const double Bm = -s * agm * lam[H - 1];
  const double Gm = s * lam[H];
  // top half (k = H-1 .. 0) and bottom half (k = H+1 .. LQ-2), interleaved
  double At = Am, Bt = Bm, Gt = Gm, Ab = Am, Bb = Bm, Gb = Gm;
#pragma unroll
  for (int j = 0; j < H; j++) {
    const int kt = H - 1 - j;
    const double g = ga[kt];
    At = fma(-g, At, pF[DIR * kt]);
    Bt = fma(-g, Bt, lam[kt]);
    Gt = -g * Gt;
    pF[DIR * kt] = At;
    sb[kt] = Bt;
    ga[kt] = Gt;
    if (j < H - 1) {
      const int kb = H + 1 + j;
      const double gb = ga[kb];
      Ab = fma(-gb, Ab, pF[DIR * kb]);
      Bb = -gb * Bb;
      Gb = fma(-gb, Gb, lam[kb]);
      pF[DIR * kb] = Ab;
      sb[kb] = Bb;
      ga[kb] = Gb;
    }
  }
  pF[DIR * H] = Am;
  sb[H] = Bm;
  ga[H] = Gm;
  o.au = At;
  o.bu = Bt;
  o.gu = Gt;
  o.ad = Ab;
  o.bd = Bb;
  o.gd = Gb;
}

template <int DIR>
__device__ __forceinline__ void chunk_store(double* __restrict__ pF, const double* __restrict__ sb,
                                            const double (&ga)[LQ - 1], double XL, double X) {
#pragma unroll
  for (int k = 0; k < LQ - 1; k++) pF[DIR * k] = fma(ga[k], X, fma(sb[k], XL, pF[DIR * k]));
  pF[DIR * (LQ - 1)] = X;
}

#ifndef TMG_LEGK_RED2
#define TMG_LEGK_RED2 0  // 1: the reduced system solved by one warp in two levels (measured slower: 0.66 -> 0.77 ms)
#endif
// padded index of reduced row t: groups of eight rows start 9 slots apart, so
// a lane walking its group and a warp walking consecutive rows are both free
// of bank conflicts
__device__ __forceinline__ int ridx(int t) { return t + (t >> 3); }

// Two-level solve of an item's reduced system by one warp (TMG_LEGK_RED2).
// The 256 chunk-end rows  A X[t-1] + B X[t] + C X[t+1] = D - H x_branch  form
// one tridiagonal system (A = 0 / C = 0 at leg ends, idle rows are identity
// rows), kept at padded slots.  Lane j eliminates rows 8j .. 8j+6 (Thomas
// down sweep, then an affine back pass: X[r] = al + be X[8j-1] + ga X[8j+7],
// two right-hand sides D and H), the 32 group-end rows are solved by cyclic
// reduction on warp shuffles, and every lane back-substitutes its group.
// Out: sP / sQ (padded), X[t] = sP[t] - sQ[t] x_branch.
__device__ __forceinline__ void red2_solve(double2* __restrict__ rAC, double2* __restrict__ rDH,
                                           const double* __restrict__ rB, double* __restrict__ sP,
                                           double* __restrict__ sQ, int& phi) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int q0 = 9 * lane;
  double cp, dp, hp, lp;
  {
    const double2 ac = rAC[q0], dh = rDH[q0];
    const double b = rB[q0];
    phi = min(phi, __double2hiint(b) & 0x7fffffff);
    const double iv = drcp(b);
    cp = ac.y * iv;
    dp = dh.x * iv;
    hp = dh.y * iv;
    lp = -ac.x * iv;
    rAC[q0] = make_double2(lp, cp);
    rDH[q0] = make_double2(dp, hp);
  }
#pragma unroll 1
  for (int r = 1; r < 7; r++) {
    const double2 ac = rAC[q0 + r], dh = rDH[q0 + r];
    const double w = ac.x;
    const double pv = fma(-w, cp, rB[q0 + r]);
    phi = min(phi, __double2hiint(pv) & 0x7fffffff);
    const double iv = drcp(pv);
    cp = ac.y * iv;
    dp = fma(-w, dp, dh.x) * iv;
    hp = fma(-w, hp, dh.y) * iv;
    lp = (-w * lp) * iv;
    if (r < 6) {
      rAC[q0 + r] = make_double2(lp, cp);
      rDH[q0 + r] = make_double2(dp, hp);
    }
  }
  // X[8j+6] = ad + bd XL + gd X - hd x_branch; back pass to the group's first row
  const double ad = dp, hd = hp, bd = lp, gd = -cp;
  rAC[q0 + 6] = make_double2(bd, gd);
  rDH[q0 + 6] = make_double2(ad, hd);
  double al = ad, et = hd, be = bd, ga = gd;
#pragma unroll 1
  for (int r = 5; r >= 0; r--) {
    const double2 lc = rAC[q0 + r], dh = rDH[q0 + r];
    al = fma(-lc.y, al, dh.x);
    et = fma(-lc.y, et, dh.y);
    be = fma(-lc.y, be, lc.x);
    ga = -lc.y * ga;
    rAC[q0 + r] = make_double2(be, ga);
    rDH[q0 + r] = make_double2(al, et);
  }
  // the group-end row, with the next group's first-row form
  double A, Bv, C, D, H;
  {
    const double2 ac = rAC[q0 + 7], dh = rDH[q0 + 7];
    const double aun = __shfl_down_sync(FULL, al, 1), etn = __shfl_down_sync(FULL, et, 1);
    const double bun = __shfl_down_sync(FULL, be, 1), gun = __shfl_down_sync(FULL, ga, 1);
    A = ac.x * bd;
    Bv = fma(ac.y, bun, fma(ac.x, gd, rB[q0 + 7]));
    C = ac.y * gun;  // row 255 ends a leg or is idle: C = 0 there
    D = fma(-ac.y, aun, fma(-ac.x, ad, dh.x));
    H = fma(-ac.y, etn, fma(-ac.x, hd, dh.y));
  }
  double iB = drcp(Bv);
#pragma unroll 1
  for (int d = 1; d < 32; d <<= 1) {
    const double Am = __shfl_up_sync(FULL, A, d), Cm = __shfl_up_sync(FULL, C, d);
    const double Dm = __shfl_up_sync(FULL, D, d), Hm = __shfl_up_sync(FULL, H, d);
    const double im = __shfl_up_sync(FULL, iB, d);
    const double Ap = __shfl_down_sync(FULL, A, d), Cq = __shfl_down_sync(FULL, C, d);
    const double Dq = __shfl_down_sync(FULL, D, d), Hq = __shfl_down_sync(FULL, H, d);
    const double ip = __shfl_down_sync(FULL, iB, d);
    // rows closer than d to an end have no coupling that far (A or C is 0)
    const double k1 = lane >= d ? A * im : 0.0, k2 = lane + d < 32 ? C * ip : 0.0;
    A = -k1 * Am;
    C = -k2 * Cq;
    Bv = fma(-k2, Ap, fma(-k1, Cm, Bv));
    D = fma(-k2, Dq, fma(-k1, Dm, D));
    H = fma(-k2, Hq, fma(-k1, Hm, H));
    iB = drcp(Bv);
  }
  phi = min(phi, __double2hiint(Bv) & 0x7fffffff);
  const double P2 = D * iB, Q2 = H * iB;
  double PL = __shfl_up_sync(FULL, P2, 1), QL = __shfl_up_sync(FULL, Q2, 1);
  if (lane == 0) PL = QL = 0.0;  // row 0 starts a leg: its be is 0
#pragma unroll 1
  for (int r = 0; r < 7; r++) {
    const double2 lc = rAC[q0 + r], dh = rDH[q0 + r];
    sP[q0 + r] = fma(lc.y, P2, fma(lc.x, PL, dh.x));
    sQ[q0 + r] = fma(lc.y, Q2, fma(lc.x, QL, dh.y));
  }
  sP[q0 + 7] = P2;
  sQ[q0 + 7] = Q2;
}

#ifndef TMG_LEGK_XMB
#define TMG_LEGK_XMB 1  // 0: split pairs exchange through a full cluster barrier
#endif
#ifndef TMG_LEGK_TWIST
#define TMG_LEGK_TWIST 1  // 0: the one-ended chunk sweep
#endif
#if TMG_LEGK_TWIST
#define LEGK_FWD chunk_forward_tw
#define LEGK_BACK chunk_back_tw
#else
#define LEGK_FWD chunk_forward
#define LEGK_BACK chunk_back
#endif

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(LT, 2)
    leg_sweep_kernel(LegArgs a) {
  extern __shared__ __align__(128) double smem[];
  double* F = smem;            // f, then the chunk scratch, then the new u
  double* Ls = F + kLegArrF;   // u row on the low side
  double* Hs = Ls + kLegArrU;  // u row on the high side
  uint64_t* bar = reinterpret_cast<uint64_t*>(Hs + kLegArrU);
  uint64_t* xbar = bar + 1;  // split pairs: the peer's leg end has arrived
  double* xch = reinterpret_cast<double*>(bar + 2);  // [2 parities][P, Qh]
  uint64_t* bbar = reinterpret_cast<uint64_t*>(xch + 4);  // descriptor blob buffers 0, 1
  unsigned char* blobs = reinterpret_cast<unsigned char*>(bbar + 2);
  const int tid = threadIdx.x;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int n = a.n, ld = a.ld;

  // every staged value a dummy point may read must be finite
  for (int i = tid; i < kLegStage / 2; i += LT)
    reinterpret_cast<double2*>(smem)[i] = make_double2(0, 0);
  if (tid == 0) {
#if TMG_LEGK_SPLITISSUE
    mbar_init(bar, 2);  // the u rows and the f runs arrive separately
#else
    mbar_init(bar, 1);
#endif
    mbar_init(bbar, 1);
    mbar_init(bbar + 1, 1);
#if TMG_LEGK_XMB
    mbar_init(xbar, 1);
#endif
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
#if TMG_LEGK_XMB
  cluster_arrive();  // the peer's exchange barrier is initialised before any remote arrive
  cluster_wait();
#else
  __syncthreads();
#endif
#if TMG_LEGK_BLOBPF
  // this CTA's descriptor blobs (static plan data) start toward L2 while the
  // previous kernel drains: the per-item blob fetches then hit L2
  if (tid < 32) {
    for (int s2 = tid;; s2 += 32) {
      const int ci = cid + s2 * ncl;
      if (ci >= a.nsched) break;
      const int4 e = a.bsched[ci];
      const int off = rank ? e.z : e.x, nb = rank ? e.w : e.y;
      if (nb > 0) bulk_prefetch_l2(a.blob + (size_t)off * 16, (unsigned)nb);
    }
  }
#endif
  pdl_wait();  // the fields of the previous kernel are complete from here on
#if TMG_LEGK_STAGGER
  if ((blockIdx.x >> 1) & 1)
    for (int i = 0; i < TMG_LEGK_STAGGER; i++) __nanosleep(1024);
#endif
  if (a.corners && blockIdx.x == 0 && tid < 4) {
    // the four interior corner points: point blocks of the red stage
    // (layout.py:72-74, relax_points _ckernels.pyx:42-51); their
    // neighbours are boundary or black-shell points, frozen in this stage
    const int i = (tid & 1) ? n - 1 : 1, j = (tid & 2) ? n - 1 : 1;
    auto uat = [&](int ii, int jj) {
      return owns_t(LM_TWEED, n, n, ii, jj) ? a.ut[(size_t)jj * ld + ii] : a.un[(size_t)ii * ld + jj];
    };
    const double Wi = __ldg(a.W + i), Ei = __ldg(a.E + i), Sj = __ldg(a.S + j),
                 Nj = __ldg(a.N + j);
    const double b = -(Wi + Ei + Sj + Nj);
    const double r = a.fn[(size_t)i * ld + j] - Wi * uat(i - 1, j) - Ei * uat(i + 1, j) -
                     Sj * uat(i, j - 1) - Nj * uat(i, j + 1);
    if (bad_pivot(b)) atomicOr(a.err, 1);
    a.un[(size_t)i * ld + j] = r / b;
  }

  auto sched_at = [&](int s) -> int4 {
    const int ci = cid + s * ncl;
    return ci < a.nsched ? a.sched[ci] : make_int4(-2, -2, 0, 0);
  };
  // this rank's descriptor blob of cluster iteration s: (offset / 16, bytes)
  auto blob_at = [&](int s) -> int2 {
    const int ci = cid + s * ncl;
    if (ci >= a.nsched) return make_int2(0, 0);
    const int4 e = a.bsched[ci];
    return rank ? make_int2(e.z, e.w) : make_int2(e.x, e.y);
  };
  // warp 0, lane 0: blob of iteration s into buffer s & 1
  auto fetch_blob = [&](int2 bl, int s) {
    if (bl.y > 0) {
      uint64_t* bb = bbar + (s & 1);
      mbar_expect_tx(bb, (unsigned)bl.y);
      bulk_g2s(blobs + (s & 1) * kLegBlob, a.blob + (size_t)bl.x * 16, (unsigned)bl.y, bb);
    }
  };
  int4 sc = sched_at(0);
  unsigned bph = 0;  // parity of each blob buffer's next fill
  if (tid < 32) {
    if (tid == 0) {
      fetch_blob(blob_at(0), 0);
      fetch_blob(blob_at(1), 1);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int it = rank ? sc.y : sc.x;
    if (it >= 0) {
      mbar_wait(bbar, 0);
      issue_loads_blob(a, blobs, smem, bar);
    }
  }
  int nsplit = 0, phi = 0x7fffffff, ph = 0;
  bool bad = false;
  // phase clocks of a -DTMG_LEGK_TIMING build (make timing): setup, stage
  // wait, forward, back, reduced system, branch, finalize, stores
#ifdef TMG_LEGK_TIMING
  long long tacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tlast = clock64();
  const bool timing = a.timing != nullptr && (tid == 0 || tid == 96);
#define LEGK_MARK(i)                     \
  do {                                   \
    if (timing) {                        \
      const long long tn = clock64();    \
      tacc[i] += tn - tlast;             \
      tlast = tn;                        \
    }                                    \
  } while (0)
#else
#define LEGK_MARK(i) \
  do {               \
  } while (0)
#endif

  for (int s = 0; sc.x != -2; s++) {
    const int item = rank ? sc.y : sc.x;
    const bool split = (sc.z & 1) != 0;
    const int steps = (sc.z >> (rank ? 16 : 8)) & 0xff;
    const int4 scn = sched_at(s + 1);
    const unsigned char* blob = blobs + (s & 1) * kLegBlob;

    // ---- per-thread chunk setup (overlaps the wait for the staged rows) ----
    uint16_t tm = 0xFFFF;
    LegBlock B{};
    if (item >= 0) {
      mbar_wait(bbar + (s & 1), (bph >> (s & 1)) & 1u);
      bph ^= 1u << (s & 1);
      const LegBlobHead* hd = reinterpret_cast<const LegBlobHead*>(blob);
      tm = reinterpret_cast<const uint16_t*>(blob + hd->off_tmap)[tid];
      if (tm != 0xFFFF) B = reinterpret_cast<const LegBlock*>(blob + hd->off_blocks)[tm >> 1];
    }
    const bool act = tm != 0xFFFF;
    const int slot = tm >> 1, leg = tm & 1;
    LegGeo g;
    g.set(act ? B.k : 2, B.quad, leg, n);
    const int m = g.m;
    const int nch = (m + LQ - 1) / LQ;
    const int pad = nch * LQ - m;
    const int ch = act ? tid - (leg ? B.t0[1] : B.t0[0]) : 0;
    const bool first = act && ch == 0, lastc = act && ch == nch - 1;
    const int e0 = ch * LQ - pad;  // leg point of chunk point 0
    double clo = 0.0, chi = 0.0;
    if (act) {
      clo = leg == 0 ? __ldg(a.S + g.bj) : __ldg(a.W + g.bi);
      chi = leg == 0 ? __ldg(a.N + g.bj) : __ldg(a.E + g.bi);
    }
    const size_t cofs =
        (size_t)(g.orient * LQ + pad) * a.cstride + (ch >> 5) * (32 * LQ) + (ch & 31);
    const int bF = leg ? B.sb[1][0] : B.sb[0][0];
    const int bL = leg ? B.sb[1][1] : B.sb[0][1];
    const int bH = leg ? B.sb[1][2] : B.sb[0][2];
    // branch row: frozen terms (the hub thread is the last chunk of leg 0, or
    // of the CTA's own leg in a split block)
    const bool hubthr = lastc && (leg == 0 || B.split >= 2);
    const bool crossb = B.split >= 3;
    double hub_num = 0.0, den0 = 1.0, cx = 0.0, cy = 0.0;
    if (hubthr) {
      const int bi = g.bi, bj = g.bj;
      const double Wi = __ldg(a.W + bi), Ei = __ldg(a.E + bi), Sj = __ldg(a.S + bj),
                   Nj = __ldg(a.N + bj);
      den0 = -(Wi + Ei + Sj + Nj);
      cx = g.sx > 0 ? Wi : Ei;  // toward the x-leg end
      cy = g.sy > 0 ? Sj : Nj;  // toward the y-leg end
      const double ex = g.sx > 0 ? Ei : Wi, ey = g.sy > 0 ? Nj : Sj;
      hub_num = a.fn[(size_t)bi * ld + bj];
      if (!crossb)  // the cross's branch has no frozen neighbour
        hub_num = hub_num - ex * a.un[(size_t)(bi + g.sx) * ld + bj] -
                  ey * a.ut[(size_t)(bj + g.sy) * ld + bi];
    }
    double tip_u = 0.0, tip_a = 0.0, uwall = 0.0;
    if (first) {  // Dirichlet neighbour of the tip (N buffer ring) and its coupling
      tip_u = leg == 0 ? a.un[(size_t)(g.p0 - g.sx) * ld + g.bj]
                       : a.un[(size_t)g.bi * ld + (g.p0 - g.sy)];
      const int tp = g.p0;
      tip_a = leg == 0 ? (g.sx > 0 ? __ldg(a.W + tp) : __ldg(a.E + tp))
                       : (g.sy > 0 ? __ldg(a.S + tp) : __ldg(a.N + tp));
    }
    // x-leg's last point: true wall-side neighbour (1: the u-1 row, 2: the u+1 row)
    // (the cross's x-legs end between two N-owned branches: both sides)
    const int wallfix = (lastc && leg == 0) ? (crossb ? 3 : g.sy > 0 ? 1 : 2) : 0;
    double uwall2 = 0.0;
    if (wallfix == 3) {
      const size_t xl = (size_t)(g.p0 + g.sx * (m - 1)) * ld;
      uwall = a.un[xl + g.bj - 1];
      uwall2 = a.un[xl + g.bj + 1];
    } else if (wallfix) {
      uwall = a.un[(size_t)(g.p0 + g.sx * (m - 1)) * ld + (g.bj - g.sy)];
    }

    CoefSrc cpre;
    cpre.p = a.coef + cofs;
    LEGK_MARK(0);
    if (item >= 0) {
      mbar_wait(bar, (unsigned)ph);
      ph ^= 1;
    }
    LEGK_MARK(1);
    double lam[LQ - 1], ga[LQ - 1];
    ChunkOut co{0, 1, 0, 0, 0, 1, 0, 0, 0, 0x7fffffff};
    double* pF = F + bF + g.dir * e0;
#ifdef TMG_CHECK
    if (act) {  // every slot of the chunk (dummies included) inside its array
      const int f0 = bF + g.dir * e0, f1 = f0 + g.dir * (LQ - 1);
      const int l0 = bL + g.dir * e0, l1 = l0 + g.dir * (LQ - 1);
      const int h0 = bH + g.dir * e0, h1 = h0 + g.dir * (LQ - 1);
      LEGK_CHECK(min(f0, f1) >= 0 && max(f0, f1) < kLegArrF, "f slots");
      LEGK_CHECK(min(l0, l1) >= 0 && max(l0, l1) < kLegArrU, "u-1 slots");
      LEGK_CHECK(min(h0, h1) >= 0 && max(h0, h1) < kLegArrU, "u+1 slots");
      LEGK_CHECK(pad >= 0 && pad < LQ && (!first || e0 == -pad), "tip padding");
      LEGK_CHECK(ch >= 0 && ch < nch && tid - ch + nch <= LT, "chunk range");
      LEGK_CHECK(cofs + 32 * (LQ - 1) < (size_t)4 * LQ * a.cstride, "coefficient index");
      if (hubthr) {
        LEGK_CHECK(B.split || tid + nch < LT, "branch partner");
        LEGK_CHECK(g.bi > 0 && g.bi < n && g.bj > 0 && g.bj < n, "branch inside");
      }
    }
#endif
    if (act) {
      if (first) pF[g.dir * pad] -= tip_a * tip_u;  // only this thread reads the tip's f
      if (g.dir > 0)
        LEGK_FWD<1>(pF, Ls + bL + e0, Hs + bH + e0, cpre, clo, chi,
                    first, wallfix, uwall, uwall2, lam, ga, co);
      else
        LEGK_FWD<-1>(pF, Ls + bL - e0, Hs + bH - e0, cpre, clo,
                     chi, first, wallfix, uwall, uwall2, lam, ga, co);
    }
    __syncthreads();  // every thread is done with the staged u rows
    LEGK_MARK(2);
#if TMG_LEGK_L2PF
    // the next item's runs start toward L2 now (its blob, requested at the end of
    // the previous item, has arrived by the time the forward pass is done); the
    // stage loads issued after this item's stores then hit L2
    if (tid < 32 && (rank ? scn.y : scn.x) >= 0) {
      const int b1 = (s + 1) & 1;
      mbar_wait(bbar + b1, (bph >> b1) & 1u);
      prefetch_loads_blob(a, blobs + b1 * kLegBlob);
    }
#endif
    double* sb = Hs + tid * LQ;  // this thread's beta row
    if (act) {
      if (g.dir > 0)
        LEGK_BACK<1>(pF, sb, lam, ga, co);
      else
        LEGK_BACK<-1>(pF, sb, lam, ga, co);
    }

    phi = min(phi, co.phi);

    // ---- reduced system over the chunk ends (shared memory in Ls) ----------
    double2* sFU = reinterpret_cast<double2*>(Ls);  // first-point forms (au, bu)
    double* sGU = Ls + 2 * LT;                      // ... gu
    // PCR rows, two buffers of 5 LT doubles: (A, C) pairs, (D, H) pairs, 1/B
    auto rAC = [&](int b) { return reinterpret_cast<double2*>(Ls + (3 + 5 * b) * LT); };
    auto rDH = [&](int b) { return reinterpret_cast<double2*>(Ls + (5 + 5 * b) * LT); };
    auto rIB = [&](int b) { return Ls + (7 + 5 * b) * LT; };
    double* sP = Ls + 13 * LT;  // X = P - Qh * x_branch
    double* sQ = Ls + 14 * LT;
    double* sX = Ls + 15 * LT;  // branch value per block slot
    sFU[tid] = make_double2(co.au, co.bu);
    sGU[tid] = co.gu;
    __syncthreads();
    LEGK_MARK(3);
    double A = 0.0, Bv = 1.0, C = 0.0, D = 0.0, H = 0.0;
    if (act) {
      const double ae = co.a_end, ce = co.c_end;
      const double bbe = -(ae + ce + clo + chi);
      A = first ? 0.0 : ae * co.bd;
      Bv = fma(ae, co.gd, bbe);
      D = fma(-ae, co.ad, co.r_end);
      if (lastc) {
        H = ce;  // the branch
      } else {
        const double2 fu = sFU[tid + 1];
        Bv = fma(ce, fu.y, Bv);
        C = ce * sGU[tid + 1];
        D = fma(-ce, fu.x, D);
      }
    }
#if TMG_LEGK_RED2
#define LEGK_SP(t) sP2[ridx(t)]
#define LEGK_SQ(t) sQ2[ridx(t)]
    constexpr int LTP = LT + LT / 8;  // padded rows
    double2* r2AC = reinterpret_cast<double2*>(Ls + 3 * LT);
    double2* r2DH = r2AC + LTP;
    double* r2B = reinterpret_cast<double*>(r2DH + LTP);
    double* sP2 = r2B + LTP;
    double* sQ2 = sP2 + LTP;
    static_assert(3 * LT + 7 * LTP + LT <= kLegArrU, "reduced-system scratch");
    const int rq = ridx(tid);
    r2AC[rq] = make_double2(A, C);
    r2DH[rq] = make_double2(D, H);
    r2B[rq] = Bv;
    __syncthreads();
    if ((tid >> 5) == 2) red2_solve(r2AC, r2DH, r2B, sP2, sQ2, phi);
    __syncthreads();
    LEGK_MARK(4);
    const double P = sP2[rq], Qh = sQ2[rq];
#else
#define LEGK_SP(t) sP[t]
#define LEGK_SQ(t) sQ[t]
    double iB = drcp(Bv);
    // parallel cyclic reduction, double-buffered (one barrier per step).  A row
    // whose partner at distance d lies outside the CTA has no coupling that far
    // (legs never cross items), so the clamped partner only needs to be finite.
    rAC(0)[tid] = make_double2(A, C);
    rDH(0)[tid] = make_double2(D, H);
    rIB(0)[tid] = iB;
    __syncthreads();
    for (int stp = 0; stp < steps; stp++) {
      const int d = 1 << stp, src = stp & 1;
      const int im = max(tid - d, 0), ip = min(tid + d, LT - 1);
      const double2 acm = rAC(src)[im], dhm = rDH(src)[im];
      const double2 acp = rAC(src)[ip], dhp = rDH(src)[ip];
      const double k1 = A * rIB(src)[im], k2 = C * rIB(src)[ip];
      A = -k1 * acm.x;
      C = -k2 * acp.y;
      Bv = fma(-k2, acp.x, fma(-k1, acm.y, Bv));
      D = fma(-k2, dhp.x, fma(-k1, dhm.x, D));
      H = fma(-k2, dhp.y, fma(-k1, dhm.y, H));
      iB = drcp(Bv);
      rAC(src ^ 1)[tid] = make_double2(A, C);
      rDH(src ^ 1)[tid] = make_double2(D, H);
      rIB(src ^ 1)[tid] = iB;
      __syncthreads();
    }
    LEGK_MARK(4);
    if (act) phi = min(phi, __double2hiint(Bv) & 0x7fffffff);
    const double P = D * iB, Qh = H * iB;
    sP[tid] = P;
    sQ[tid] = Qh;
#endif
#if TMG_LEGK_XMB
    if (split && hubthr) {
      // the leg end of this CTA's half of a split block goes straight into the
      // peer's exchange slot; the remote arrive (release, cluster scope)
      // completes the peer's exchange-barrier phase
      const int par = nsplit & 1;
      st_cluster_v2(mapa_u32(xch + 2 * par, rank ^ 1), P, Qh);
      mbar_arrive_remote(mapa_u32(xbar, rank ^ 1));
    }
#if !TMG_LEGK_RED2
    __syncthreads();
#endif
#else
    if (split) {
      // the leg end of each CTA's half of a split block goes to the peer
      const int par = nsplit & 1;
      if (hubthr) {
        xch[2 * par] = P;
        xch[2 * par + 1] = Qh;
      }
      cluster_arrive();
      cluster_wait();
    } else {
      __syncthreads();
    }
#endif

    // ---- branch rows ----------------------------------------------------------
    if (hubthr && crossb) {
      // central cross: the four leg ends meet through the global mailbox
      // (every leg CTA runs in the first two cluster iterations, all resident)
      const int sl = B.split - 3;
      volatile double* mb = a.mail;
      int* cnt = reinterpret_cast<int*>(a.mail + 8);
      mb[2 * sl] = P;
      mb[2 * sl + 1] = Qh;
      __threadfence();
      atomicAdd(cnt, 1);
      while (atomicAdd(cnt, 0) < 4) __nanosleep(64);
      __threadfence();
      const int c = n / 2;
      const double cf[4] = {__ldg(a.W + c), __ldg(a.E + c), __ldg(a.S + c), __ldg(a.N + c)};
      double num = hub_num, den = den0;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        num -= cf[q] * mb[2 * q];
        den -= cf[q] * mb[2 * q + 1];
      }
      bad |= bad_pivot(den);
      const double xb = num / den;
      sX[slot] = xb;
      if (sl == 0) a.un[(size_t)c * ld + c] = xb;
      if (atomicAdd(cnt + 1, 1) == 3) {  // the last reader rearms the mailbox
        cnt[0] = 0;
        cnt[1] = 0;
        __threadfence();
      }
    } else if (hubthr) {
      double px, qx, py, qy;
      if (B.split) {
        const int par = nsplit & 1;
#if TMG_LEGK_XMB
        mbar_wait_cluster(xbar, (unsigned)par);
        const double pp = xch[2 * par], qp = xch[2 * par + 1];
#else
        const double* peer = cluster.map_shared_rank(xch, rank ^ 1);
        const double pp = peer[2 * par], qp = peer[2 * par + 1];
#endif
        if (leg == 0) { px = P; qx = Qh; py = pp; qy = qp; }
        else { px = pp; qx = qp; py = P; qy = Qh; }
      } else {
        const int ty = B.t0[1] + nch - 1;
        px = P;
        qx = Qh;
        py = LEGK_SP(ty);
        qy = LEGK_SQ(ty);
      }
      const double den = den0 - cx * qx - cy * qy;
      bad |= bad_pivot(den);
      const double xb = (hub_num - cx * px - cy * py) / den;
      sX[slot] = xb;
      if (B.split != 2) a.un[(size_t)g.bi * ld + g.bj] = xb;
    }
    if (split) nsplit++;
    __syncthreads();
    LEGK_MARK(5);

    // ---- finalize into the f slots ------------------------------------------
    if (act) {
      const double xb = sX[slot];
      const double X = fma(-Qh, xb, P);
      const double XL = first ? 0.0 : fma(-LEGK_SQ(tid - 1), xb, LEGK_SP(tid - 1));
      if (g.dir > 0)
        chunk_store<1>(pF, sb, ga, XL, X);
      else
        chunk_store<-1>(pF, sb, ga, XL, X);
    }
    __syncthreads();
    LEGK_MARK(6);

    // ---- stores and the next item's loads: warp 0 bulk-copies the aligned
    // leg interiors (single elements at unaligned ends), waits until they have
    // left shared memory, issues the next item's loads from its blob (fetched
    // an item ago) and refills this item's blob buffer two items ahead.
    const int nx = rank ? scn.y : scn.x;
#if TMG_LEGK_SPLITISSUE
    // warp 1: the next item's u rows go out at once (Ls / Hs are free after
    // the finalize barrier); warp 0: bulk stores first, the edge elements
    // while they drain, then the next item's f runs into the freed f array
    if (tid >= 32 && tid < 64 && nx >= 0) {
      const int b1 = (s + 1) & 1;
      mbar_wait(bbar + b1, (bph >> b1) & 1u);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_loads_blob(a, blobs + b1 * kLegBlob, smem, bar, 0);
    }
    if (tid < 32) {
      if (item >= 0) {
        const LegBlobHead* hd = reinterpret_cast<const LegBlobHead*>(blob);
        const LegCopy* cps = reinterpret_cast<const LegCopy*>(blob + sizeof(LegBlobHead));
        const int ncopy = hd->ncopy, nstore = hd->nstore, nedge = hd->nedge;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int c = tid; c < nstore; c += 32) {
          const LegCopy cp = cps[ncopy + c];
          bulk_s2g((cp.src == 3 ? a.ut : a.un) + cp.g, F + cp.s, (unsigned)cp.n * 8u);
        }
        bulk_commit();
        for (int c = tid; c < nedge; c += 32) {
          const LegCopy cp = cps[ncopy + nstore + c];
          (cp.src == 3 ? a.ut : a.un)[cp.g] = F[cp.s];
        }
      }
      LEGK_MARK(8);
      if (nx >= 0) {
        const int b1 = (s + 1) & 1;
        mbar_wait(bbar + b1, (bph >> b1) & 1u);
        LEGK_MARK(9);
        bulk_wait_read();  // the stores have left shared memory
        LEGK_MARK(10);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_loads_blob(a, blobs + b1 * kLegBlob, smem, bar, 1);
      }
      __syncwarp();  // every lane is done with this item's blob
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        fetch_blob(blob_at(s + 2), s + 2);  // its latency hides under the stage loads
      }
    }
#else
    if (tid < 32) {
      if (item >= 0) {
        const LegBlobHead* hd = reinterpret_cast<const LegBlobHead*>(blob);
        const LegCopy* cps = reinterpret_cast<const LegCopy*>(blob + sizeof(LegBlobHead));
        const int ncopy = hd->ncopy, nstore = hd->nstore, nedge = hd->nedge;
        for (int c = tid; c < nedge; c += 32) {
          const LegCopy cp = cps[ncopy + nstore + c];
          (cp.src == 3 ? a.ut : a.un)[cp.g] = F[cp.s];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int c = tid; c < nstore; c += 32) {
          const LegCopy cp = cps[ncopy + c];
          bulk_s2g((cp.src == 3 ? a.ut : a.un) + cp.g, F + cp.s, (unsigned)cp.n * 8u);
        }
        bulk_commit();
      }
      LEGK_MARK(8);
      if (nx >= 0) {
        const int b1 = (s + 1) & 1;
        mbar_wait(bbar + b1, (bph >> b1) & 1u);
        LEGK_MARK(9);
        bulk_wait_read();  // the stores have left shared memory
        LEGK_MARK(10);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_loads_blob(a, blobs + b1 * kLegBlob, smem, bar);
      }
      __syncwarp();  // every lane is done with this item's blob
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        fetch_blob(blob_at(s + 2), s + 2);  // its latency hides under the stage loads
      }
    }
#endif
    LEGK_MARK(7);
    sc = scn;
  }
#undef LEGK_MARK
#ifdef TMG_LEGK_TIMING
  if (timing)
    for (int i = 0; i < 12; i++) a.timing[(blockIdx.x + (tid ? gridDim.x : 0)) * 12 + i] = tacc[i];
#ifdef TMG_LEGK_TIMING
  if (a.timing && tid == 0) {  // SM of every CTA (cluster placement)
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    a.timing[24 * 1024 + blockIdx.x] = sm;
  }
#endif
#endif
  if (tid < 32) bulk_wait_all();
  bad |= phi < 0x01A56E1F;  // |pivot| < 1e-300 (high word of 1e-300)
  if (bad) atomicOr(a.err, 1);
  pdl_trigger();
  // no CTA may exit while its peer can still read its exchange slots
  cluster_arrive();
  cluster_wait();
}

// ============================ host side =====================================

namespace {

struct HostBlock {
  int k, quad, chunks;  // chunks per leg
};

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
// thread slots a leg of `chunks` chunks takes in an item (TMG_LEGK_WALIGN:
// legs of a warp or more are padded to whole warps)
inline int leg_slots(int chunks) {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("TMG_LEGK_WALIGN");
    on = e ? std::atoi(e) != 0 : 0;  // measured: 0.660 -> 0.670 ms (the padding costs more items)
  }
  return on && chunks >= 32 ? (chunks + 31) & ~31 : chunks;
}

}  // namespace

bool leg_plan_applies(int scheme, int nx, int ny, int mode) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* s = std::getenv("TMG_LEGK");
    enabled = s ? std::atoi(s) != 0 : 1;
  }
  static int nmin = 0;
  if (!nmin) {
    const char* s = std::getenv("TMG_LEGK_NMIN");
    nmin = s && std::atoi(s) > 0 ? std::atoi(s) : kLegNmin;
  }
  return enabled && scheme == SCHEME_TWEED && mode == LM_TWEED && nx == ny && nx >= nmin &&
         nx % 2 == 0;
}

int leg_k0() {
  static int k0 = 0;
  if (!k0) {
    const char* s = std::getenv("TMG_LEGK_K0");
    k0 = s && std::atoi(s) >= 2 ? std::atoi(s) : kLegK0;
  }
  return k0;
}

// Blocks of one colour on an n x n grid handled by the leg kernel: shells
// k in [k0, c) of that colour, the four quadrants (layout.py:75-84).
static void colour_blocks(int n, int red, int kmin, int kmax, std::vector<HostBlock>& out) {
  const int c = n / 2;  // (s + 1) / 2 with s = n - 1
  for (int k = std::min(c - 1, kmax); k >= std::max(leg_k0(), kmin); k--) {
    if (((k % 2) != 0) != (red != 0)) continue;  // layout.py:22-23
    for (int q = 0; q < 4; q++) out.push_back(HostBlock{k, q, ceil_div(k - 1, LQ)});
  }
}

std::string build_leg_plan(int n, LegPlan& P, int kmin, int kmax) {
  P = LegPlan();
  P.n = n;
  const int ld = n + 1;
  for (int red = 1; red >= 0; red--) {
    LegColour& C = P.col[red];
    std::vector<HostBlock> blocks;
    colour_blocks(n, red, kmin, kmax, blocks);
    std::vector<LegItem> items;
    std::vector<LegBlock> iblocks;
    std::vector<uint16_t> tmap;
    std::vector<LegCopy> copies;
    std::vector<int> item_chunks;
    std::vector<unsigned char> blob;   // descriptor blobs, 16-byte aligned
    std::vector<int2> item_blob;       // (offset / 16, bytes) per item

    struct Open {
      std::vector<std::pair<HostBlock, int>> members;  // block, split (0/1/2)
      int chunks = 0;
    };
    auto emit = [&](const Open& o) -> int {
      LegItem it{};
      it.blk0 = (int32_t)iblocks.size();
      it.nblk = (int16_t)o.members.size();
      std::vector<uint16_t> map(LT, 0xFFFF);
      std::vector<LegCopy> loads, stores, edges;
      int t = 0, soff[3] = {kLegHead, kLegHead, kLegHead}, maxch = 1;
      long bytes = 0;
      for (size_t bi = 0; bi < o.members.size(); bi++) {
        const HostBlock& hb = o.members[bi].first;
        const int split = o.members[bi].second;
        LegBlock lb{};
        lb.k = (int16_t)hb.k;
        lb.quad = (uint8_t)hb.quad;
        lb.split = (uint8_t)split;
        lb.t0[0] = lb.t0[1] = -1;
        const int sx = (hb.quad & 1) ? -1 : 1, sy = (hb.quad & 2) ? -1 : 1;
        const int x0 = sx > 0 ? 1 : n - 1, y0 = sy > 0 ? 1 : n - 1;
        const int bi_ = x0 + sx * (hb.k - 1), bj_ = y0 + sy * (hb.k - 1), m = hb.k - 1;
        for (int leg = 0; leg < 2; leg++) {
          // split 1 / 2: the leg 0 / 1 half of a split block; 3..6: one leg of
          // the central cross (W, E as x-legs of the LL / LR shell c, S, N as
          // y-legs of the LL / UL shell c)
          const int only = split == 1 ? 0 : split == 2 ? 1 : split >= 3 ? (split >= 5 ? 1 : 0) : -1;
          if (only >= 0 && leg != only) continue;
          // a leg of a warp or more starts on a warp boundary: no warp then
          // holds chunks of two legs running in opposite directions (each
          // direction is its own instantiation of the chunk passes)
          if (leg_slots(33) == 64 && hb.chunks >= 32) t = (t + 31) & ~31;
          lb.t0[leg] = (int16_t)t;
          for (int c = 0; c < hb.chunks; c++) map[t + c] = (uint16_t)((bi << 1) | leg);
          t += hb.chunks;
          maxch = std::max(maxch, hb.chunks);
          const int dir = leg == 0 ? sx : sy, p0 = leg == 0 ? x0 : y0;
          const int row = leg == 0 ? bj_ : bi_;
          const int lo = std::min(p0, p0 + dir * (m - 1)), hi = std::max(p0, p0 + dir * (m - 1));
          long gsF = 0;
          int soffF = 0;
          const int nchl = hb.chunks, padl = nchl * LQ - m;
          for (int arr = 0; arr < 3; arr++) {
            const long r = arr == 0 ? row : arr == 1 ? row - 1 : row + 1;
            const long g0 = r * ld + lo, g1 = r * ld + hi + 1;  // [g0, g1)
            const long gs = g0 & ~1L, ge = (g1 + 1) & ~1L;
            const long gtip = r * ld + p0;
            // the tip chunk's dummies write a private gap in front of the tip
            // (before the run for ascending legs, after it for descending ones)
            const int gap_lo = arr == 0 && dir > 0 ? std::max(0, padl - (int)(gtip - gs)) : 0;
            const int gap_hi = arr == 0 && dir < 0 ? std::max(0, padl - (int)(ge - 1 - gtip)) : 0;
            soff[arr] += (gap_lo + 1) & ~1;
            LegCopy cp{};
            cp.g = gs;
            cp.s = (arr == 0 ? 0 : arr == 1 ? kLegArrF : kLegArrF + kLegArrU) + soff[arr];
            cp.n = (int32_t)(ge - gs);
            // sources: 0 f N, 1 f T, 2 u N, 3 u T
            cp.src = (uint8_t)(arr == 0 ? (leg == 0 ? 1 : 0) : (leg == 0 ? 3 : 2));
            loads.push_back(cp);
            bytes += 8L * cp.n;
            lb.sb[leg][arr] = (int16_t)(soff[arr] + (gtip - gs));
            if (arr == 0) {
              gsF = gs;
              soffF = soff[arr];
            }
            soff[arr] += (int)(ge - gs) + ((gap_hi + 1) & ~1);
            if (soff[arr] + kLegHead > (arr == 0 ? kLegArrF : kLegArrU)) return -1;
          }
          // the new values: bulk stores of the 16-byte aligned interior of the
          // leg's run, single elements at unaligned ends
          const long glo = (long)row * ld + lo, ghi = (long)row * ld + hi;
          const long is = (glo + 1) & ~1L, ie = (ghi + 1) & ~1L;
          const uint8_t dst = (uint8_t)(leg == 0 ? 3 : 2);
          if (ie > is) {
            LegCopy cp{};
            cp.g = is;
            cp.s = soffF + (int)(is - gsF);
            cp.n = (int32_t)(ie - is);
            cp.src = dst;
            stores.push_back(cp);
          }
          for (int side = 0; side < 2; side++) {
            const long ge_ = side ? ghi : glo;
            if (ge_ >= is && ge_ < ie) continue;
            if (side == 1 && ghi == glo) continue;  // a one-point leg has one edge
            LegCopy cp{};
            cp.g = ge_;
            cp.s = soffF + (int)(ge_ - gsF);
            cp.n = 1;
            cp.src = dst;
            edges.push_back(cp);
          }
        }
        iblocks.push_back(lb);
      }
      it.copy0 = (int32_t)copies.size();
      it.ncopy = (int32_t)loads.size();
      copies.insert(copies.end(), loads.begin(), loads.end());
      it.store0 = (int32_t)copies.size();
      it.nstore = (int32_t)stores.size();
      copies.insert(copies.end(), stores.begin(), stores.end());
      it.edge0 = (int32_t)copies.size();
      it.nedge = (int32_t)edges.size();
      copies.insert(copies.end(), edges.begin(), edges.end());
      it.bytes = (int32_t)bytes;
      {  // the item's descriptor blob: header, copies, blocks, thread map
        LegBlobHead hd{};
        hd.nblk = it.nblk;
        hd.ncopy = it.ncopy;
        hd.nstore = it.nstore;
        hd.nedge = it.nedge;
        hd.bytes = it.bytes;
        hd.bytes_f = 0;
        for (const LegCopy& cp : loads)
          if (cp.s < kLegArrF) hd.bytes_f += 8 * cp.n;
        const int ncp = it.ncopy + it.nstore + it.nedge;
        hd.off_blocks = (int32_t)(sizeof(LegBlobHead) + ncp * sizeof(LegCopy));
        hd.off_tmap = hd.off_blocks + (int32_t)(o.members.size() * sizeof(LegBlock));
        hd.off_tmap = (hd.off_tmap + 1) & ~1;
        const int size = ((hd.off_tmap + LT * 2) + 15) & ~15;
        if (size > kLegBlob) return -1;
        std::vector<unsigned char> b(size, 0);
        std::memcpy(b.data(), &hd, sizeof hd);
        std::memcpy(b.data() + sizeof hd, copies.data() + it.copy0, ncp * sizeof(LegCopy));
        std::memcpy(b.data() + hd.off_blocks, iblocks.data() + it.blk0,
                    o.members.size() * sizeof(LegBlock));
        std::memcpy(b.data() + hd.off_tmap, map.data(), LT * 2);
        item_blob.push_back(make_int2((int)(blob.size() / 16), size));
        blob.insert(blob.end(), b.begin(), b.end());
      }
      int steps = 0;
      while ((1 << steps) < maxch) steps++;
      it.steps = (int16_t)steps;
      items.push_back(it);
      tmap.insert(tmap.end(), map.begin(), map.end());
      item_chunks.push_back(t);
      return (int)items.size() - 1;
    };

    // the central cross (square grids, colour of shell c): four one-leg items
    // run in the first two cluster iterations (all four CTAs co-resident;
    // the branch row goes through a global mailbox)
    std::vector<int4> sched_split;
    const int c = n / 2;
    if (((c % 2) != 0) == (red != 0) && kmin <= c && c <= kmax) {
      const int quads[4] = {0, 1, 0, 2};  // W: LL x-leg, E: LR x-leg, S: LL y-leg, N: UL y-leg
      int ids[4];
      for (int q = 0; q < 4; q++) {
        Open o;
        o.members.push_back({HostBlock{c, quads[q], ceil_div(c - 1, LQ)}, 3 + q});
        o.chunks = ceil_div(c - 1, LQ);
        ids[q] = emit(o);
        if (ids[q] < 0) return "leg plan: staging overflow";
      }
      sched_split.push_back(make_int4(ids[0], ids[1], (items[ids[0]].steps << 8) |
                                                          (items[ids[1]].steps << 16), 0));
      sched_split.push_back(make_int4(ids[2], ids[3], (items[ids[2]].steps << 8) |
                                                          (items[ids[3]].steps << 16), 0));
      C.cross = 1;
    }
    // split blocks: one item per leg, scheduled on the two CTAs of a cluster
    std::vector<Open> open;
    for (const HostBlock& hb : blocks) {
      if (hb.chunks > LT / 2) {
        Open a_, b_;
        a_.members.push_back({hb, 1});
        a_.chunks = hb.chunks;
        b_.members.push_back({hb, 2});
        b_.chunks = hb.chunks;
        const int ia = emit(a_), ib = emit(b_);
        if (ia < 0 || ib < 0) return "leg plan: staging overflow";
        sched_split.push_back(
            make_int4(ia, ib, 1 | (items[ia].steps << 8) | (items[ib].steps << 16), hb.chunks));
        continue;
      }
      // first fit (blocks arrive in decreasing size)
      bool placed = false;
      for (Open& o : open) {
        if (o.chunks + 2 * leg_slots(hb.chunks) <= LT && (int)o.members.size() < kLegMaxBlocks) {
          o.members.push_back({hb, 0});
          o.chunks += 2 * leg_slots(hb.chunks);
          placed = true;
          break;
        }
      }
      if (!placed) {
        Open o;
        o.members.push_back({hb, 0});
        o.chunks = 2 * leg_slots(hb.chunks);
        open.push_back(o);
      }
    }
    std::vector<std::pair<int, int>> whole;  // (chunks, item)
    for (const Open& o : open) {
      const int id = emit(o);
      if (id < 0) return "leg plan: staging overflow";
      whole.push_back({o.chunks, id});
    }
    std::sort(whole.begin(), whole.end(), [](auto& x, auto& y) { return x.first > y.first; });
    std::vector<int4> sched = sched_split;
    for (size_t i = 0; i < whole.size(); i += 2) {
      const int ia = whole[i].second;
      const int ib = i + 1 < whole.size() ? whole[i + 1].second : -1;
      const int sb = ib >= 0 ? items[ib].steps : 0;
      sched.push_back(make_int4(ia, ib, (items[ia].steps << 8) | (sb << 16), whole[i].first));
    }
    std::vector<int4> bsched;
    for (const int4& e : sched) {
      const int2 b0 = e.x >= 0 ? item_blob[e.x] : make_int2(0, 0);
      const int2 b1 = e.y >= 0 ? item_blob[e.y] : make_int2(0, 0);
      bsched.push_back(make_int4(b0.x, b0.y, b1.x, b1.y));
    }
    C.corners = red && kmin <= 1;  // the four corner points (k = 1, red)
    C.nsched = (int)sched.size();
    C.nitems = (int)items.size();
    C.points = 0;
    for (const HostBlock& hb : blocks) C.points += 2L * (hb.k - 1) + 1;
    std::string err;
    auto up = [&](auto& v, auto*& d) {
      using T = typename std::remove_reference<decltype(v)>::type::value_type;
      if (v.empty()) return;
      if (cudaMalloc(&d, v.size() * sizeof(T)) != cudaSuccess ||
          cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
        err = "leg plan upload failed";
      P.device_bytes += v.size() * sizeof(T);
    };
    up(items, C.items);
    up(iblocks, C.blocks);
    up(tmap, C.tmap);
    if (C.cross) {  // cross mailbox: 4 x (P, Qh), then two counters
      if (cudaMalloc(&C.mail, 8 * sizeof(double) + 2 * sizeof(int)) != cudaSuccess ||
          cudaMemset(C.mail, 0, 8 * sizeof(double) + 2 * sizeof(int)) != cudaSuccess)
        err = "leg plan mailbox";
    }
    up(copies, C.copies);
    up(sched, C.sched);
    up(blob, C.blob);
    up(bsched, C.bsched);
    if (!err.empty()) return err;
  }
  return "";
}

std::string leg_plan_set_coefs(LegPlan& P, const double* W, const double* E, const double* S,
                               const double* N) {
  const int n = P.n;
  const int mmax = n / 2 - 1;  // longest leg (a leg of the central cross)
  const int nch = ceil_div(std::max(mmax, 1), LQ);
  const int cstride = ceil_div(nch, 32) * 32 * LQ;
  std::vector<double2> h((size_t)4 * LQ * cstride, make_double2(0.0, 0.0));
  for (int o = 0; o < 4; o++) {
    for (int pad = 0; pad < LQ; pad++) {
      const size_t base = (size_t)(o * LQ + pad) * cstride;
      for (int ch = 0; ch < nch; ch++) {
        for (int k = 0; k < LQ; k++) {
          const int e = ch * LQ + k - pad;  // leg point (tip = 0)
          // dummies: a huge diagonal (1e300, so a vanishing reciprocal) and
          // no coupling toward the next point decouple them from the tip
          if (e < 0) {
            h[base + (ch >> 5) * (32 * LQ) + k * 32 + (ch & 31)] = make_double2(1e300, 0.0);
            continue;
          }
          if (e < 0 || e > n - 2) continue;  // dummies: no coupling
          const int pos = (o % 2 == 0) ? 1 + e : n - 1 - e;
          double av, cv;
          switch (o) {
            case 0: av = W[pos]; cv = E[pos]; break;
            case 1: av = E[pos]; cv = W[pos]; break;
            case 2: av = S[pos]; cv = N[pos]; break;
            default: av = N[pos]; cv = S[pos]; break;
          }
          const size_t ix = base + (ch >> 5) * (32 * LQ) + k * 32 + (ch & 31);
          // the tip's coupling toward the wall is folded into f (not eliminated)
          h[ix] = make_double2(av, cv);
        }
      }
    }
  }
  P.cstride = cstride;
  if (cudaMalloc(&P.coef, h.size() * sizeof(double2)) != cudaSuccess ||
      cudaMemcpy(P.coef, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice) !=
          cudaSuccess)
    return "leg plan coefficient upload failed";
  P.device_bytes += h.size() * sizeof(double2);
  return "";
}

void free_leg_plan(LegPlan& P) {
  for (LegColour& C : P.col) {
    cudaFree(C.items);
    cudaFree(C.blocks);
    cudaFree(C.tmap);
    cudaFree(C.copies);
    cudaFree(C.mail);
    cudaFree(C.sched);
    cudaFree(C.blob);
    cudaFree(C.bsched);
    C = LegColour();
  }
  cudaFree(P.coef);
  P.coef = nullptr;
}

size_t leg_smem_bytes() {
  // stage, bar + xbar, xch (4 doubles), two blob barriers, two blob buffers
  return sizeof(double) * kLegStage + 2 * sizeof(uint64_t) + 4 * sizeof(double) +
         2 * sizeof(uint64_t) + 2 * kLegBlob;
}

cudaError_t init_leg_kernel() {
  static cudaError_t done = cudaErrorNotReady;
  if (done == cudaErrorNotReady)
    done = cudaFuncSetAttribute(leg_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)leg_smem_bytes());
  return done;
}

namespace {
long long* g_leg_timing = nullptr;
int g_leg_timing_ctas = 0;
bool leg_timing_on() {
  static int on = -1;
  if (on < 0) {
    const char* s = std::getenv("TMG_LEGK_TIMING");
    on = s && std::atoi(s) != 0;
  }
  return on != 0;
}
}  // namespace

cudaError_t launch_leg_colour(const LegPlan& P, int red, const SweepArgs& s, cudaStream_t stream) {
  const LegColour& C = P.col[red ? 1 : 0];
  if (C.nsched == 0 && !C.corners) return cudaSuccess;
  cudaError_t e = init_leg_kernel();
  if (e != cudaSuccess) return e;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
  }
  LegArgs a{};
  a.un = s.u;
  a.ut = s.ut;
  a.fn = s.f;
  a.ft = s.ft;
  a.W = s.W;
  a.E = s.E;
  a.S = s.S;
  a.N = s.N;
  a.coef = P.coef;
  a.cstride = P.cstride;
  a.n = P.n;
  a.ld = P.n + 1;
  a.items = C.items;
  a.blocks = C.blocks;
  a.tmap = C.tmap;
  a.copies = C.copies;
  a.mail = C.mail;
  a.corners = C.corners;
  a.sched = C.sched;
  a.blob = C.blob;
  a.bsched = C.bsched;
  a.nsched = C.nsched;
  a.err = s.err;
  const int ncl = std::max(1, std::min(sms, C.nsched));  // two CTAs per SM (>= 1 for the corners)
  a.timing = nullptr;
  if (leg_timing_on()) {
    if (!g_leg_timing) cudaMalloc(&g_leg_timing, sizeof(long long) * 26 * 1024);
    a.timing = g_leg_timing;
    g_leg_timing_ctas = 2 * ncl;
  }
  TMG_COUNT(1);
  return launch_pdl(leg_sweep_kernel, dim3(2 * ncl), dim3(LT), leg_smem_bytes(), stream, a);
}

}  // namespace tmg

// Average per-CTA clock cycles of the leg kernel's phases in its last launch
// (TMG_LEGK_TIMING=1 only): setup, stage wait, forward, back, reduced system,
// branch, finalize, stores.  Returns the number of CTAs averaged.
// SM ids of the last timed launch's CTAs (TMG_LEGK_TIMING builds): returns the count
extern "C" int tmg_debug_leg_smids(int* out, int cap) {
  if (!tmg::g_leg_timing) return 0;
  const int n = std::min(cap, tmg::g_leg_timing_ctas);
  std::vector<long long> h(n);
  cudaMemcpy(h.data(), tmg::g_leg_timing + 24 * 1024, n * sizeof(long long), cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; i++) out[i] = (int)h[i];
  return n;
}

extern "C" int tmg_debug_leg_phases(double* out /* [24] */) {
  for (int i = 0; i < 24; i++) out[i] = 0.0;
  if (!tmg::g_leg_timing || tmg::g_leg_timing_ctas == 0) return 0;
  const size_t nc = (size_t)tmg::g_leg_timing_ctas;
  // out[0..11]: thread 0 (warp 0, which also issues the bulk copies);
  // out[12..23]: thread 96.  Slots 0-7 as in the kernel's phase list, 8-10
  // split warp 0's store phase: store issue, blob wait, wait for the stores'
  // shared-memory reads (slot 7 keeps the load issue)
  std::vector<long long> h(24 * nc);
  if (cudaMemcpy(h.data(), tmg::g_leg_timing, h.size() * sizeof(long long),
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  for (size_t c = 0; c < nc; c++)
    for (int i = 0; i < 12; i++) {
      out[i] += (double)h[c * 12 + i];
      out[12 + i] += (double)h[(nc + c) * 12 + i];
    }
  for (int i = 0; i < 24; i++) out[i] /= (double)nc;
  return tmg::g_leg_timing_ctas;
}
