// Shared-memory coarse tail: the smallest levels of a V-cycle
// (mgcycle.py:89-104 from the first tail level down to the direct solve and
// back up) as ONE launch of one CTA.  u and f of every tail level, the 1D
// coefficient arrays and the block plan live in shared memory; colour stages
// and transfers are separated by __syncthreads instead of graph nodes (a
// per-stage launch costs ~4 us at these sizes, a stage here 1-2 us of
// dependent shared-memory and fp64 latency).
//
// Smoothing is the reference's per-block algorithm (relax_points / relax_chain /
// relax_ring / relax_legged, _ckernels.pyx:42-185) in two phases per colour
// stage: a thread per member builds its row (diagonal, along couplings, f
// minus the couplings to neighbours outside its block), then a thread per
// chain / ring / leg eliminates serially with register-carried reciprocal
// pivots; the legs of a block sit in adjacent lanes and close their branch row
// through warp shuffles, so a stage needs two barriers.  Results agree with
// the reference within rounding (gated at 1e-12 per sweep like the block
// kernels).  Residual, full / half weighting, bilinear prolongation +
// correction and the coarsest-level solve use the arithmetic of
// tmg_transfer_dev.cuh (stencil.py:82-87, transfer.py:33-38, 51-53,
// stencil.py:129-155) and are bit-identical to the per-stage kernels.
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "tmg_minitail.h"
#include "tmg_plan.h"

// -DTMG_CHECK (make check): device-side bounds checks of every member, unit
// and scratch index of the tail (the sanitizer stand-in)
#ifdef TMG_CHECK
#define MINI_CHECK(cond, what)                                                  \
  do {                                                                          \
    if (!(cond)) {                                                              \
      printf("mini tail check failed: %s (thread %d)\n", what, (int)threadIdx.x); \
      __trap();                                                                 \
    }                                                                           \
  } while (0)
#else
#define MINI_CHECK(cond, what) \
  do {                         \
  } while (0)
#endif

namespace tmg {

namespace {

#ifndef TMG_MINI_THREADS
#define TMG_MINI_THREADS 640  // 512: +1.8 %, 384 / 768: +1 / +2.5 % (config 1 V-cycle)
#endif
constexpr int MT = TMG_MINI_THREADS;  // threads of the tail CTA

struct MiniUnit {   // a chain, a ring, or one leg of a legged block
  uint16_t m0, cnt;  // members [m0, m0 + cnt) of the stage's member arrays
  uint8_t kind;      // 1 chain, 2 leg, 3 ring, 255 padding (a block's legs share a warp)
  uint8_t leg;       // legs: leg index (low nibble), legs of the block (high nibble)
  uint16_t mb;       // legs: the block's branch member
};
struct MiniStage {  // one colour of one sub-scheme on one level
  int unit0, nunits, mem0, nmem;
};
struct MiniMem {  // one member: its point, i * (ny + 1) + j and its flags
  uint8_t i, j;
  uint16_t p, fl, pad;
};
// Per-member flags (the build phase runs a thread per member).  Directions:
// 0 none, 1 W (i-1), 2 E (i+1), 3 S (j-1), 4 N (j+1).
enum : uint16_t {
  MF_ADIR = 7,           // bits 0-2: toward the previous member of the unit (a ring's
                         //           first member: toward its last one)
  MF_CDIR = 7 << 3,      // bits 3-5: toward the next member (ring last -> first, a
                         //           leg's innermost point -> the branch)
  MF_POINT = 1 << 6,     // a point block / a one-point chain: relax_points
  MF_RING_FIRST = 1 << 7,
  MF_LEG_LAST = 1 << 8,
  MF_BRANCH = 1 << 9     // the branch of a legged block (member of no unit)
};
struct MiniLevel {
  int nx, ny;
  int off_u, off_f, off_w;  // shared-memory offsets (doubles)
  int stage0, nstage;
  int pad;
  const double *W, *E, *S, *N;
};

struct MiniArgs {
  const unsigned char* blob;
  int blob_bytes;
  int o_lev, o_stage, o_unit, o_mem;  // byte offsets in the blob
  int nlev;
  int off_scratch, maxmem;  // doubles, after the blob copy
  FieldView U0, F0;
  const double* ainv;
  int full, nu1, nu2;
  int* err;
};

struct Lv {
  int nx, ny, ld, cap;  // cap: scratch entries per member array (TMG_CHECK)
  double *u, *f;
  const double *W, *E, *S, *N;
};

__device__ __forceinline__ bool badp(double v) { return v > -1e-300 && v < 1e-300; }

// _frozen_rhs (_ckernels.pyx:34-39)
__device__ __forceinline__ double frozen(const Lv& L, int i, int j) {
  const double* u = L.u + i * L.ld + j;
  double r = __dsub_rn(L.f[i * L.ld + j], __dmul_rn(L.W[i], u[-L.ld]));
  r = __dsub_rn(r, __dmul_rn(L.E[i], u[L.ld]));
  r = __dsub_rn(r, __dmul_rn(L.S[j], u[-1]));
  return __dsub_rn(r, __dmul_rn(L.N[j], u[1]));
}
__device__ __forceinline__ double diag(const Lv& L, int i, int j) {
  return -__dadd_rn(__dadd_rn(__dadd_rn(L.W[i], L.E[i]), L.S[j]), L.N[j]);
}
// _coupling (_ckernels.pyx:21-31)
__device__ __forceinline__ double coupling(const Lv& L, int i, int j, int pi, int pj) {
  if (pi == i - 1) return L.W[i];
  if (pi == i + 1) return L.E[i];
  if (pj == j - 1) return L.S[j];
  return L.N[j];
}

// the ~20-bit hardware reciprocal refined by two Newton steps (tmg_sweep.cu)
__device__ __forceinline__ double drcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Forward elimination rows 1 .. m-1 (with an optional carried column g).  The
// serial chain carries the pivot and its reciprocal in registers and
// multiplies by the reciprocal where the reference divides (the divisions of
// a dependent chain cost ~10x a multiply here); b[] is left holding the
// RECIPROCAL pivots for the back substitution.
__device__ __forceinline__ bool eliminate(int m, const double* __restrict__ a,
                                          double* __restrict__ b, const double* __restrict__ c,
                                          double* __restrict__ r, double* __restrict__ g) {
  double bp = b[0], rp = r[0], gp = g ? g[0] : 0.0;
  bool ok = !badp(bp);
  double ib = drcp(bp);
  b[0] = ib;
  // the next row's entries are loaded while this row's chain runs
  double an = 0.0, cn = c[0], bn = 0.0, rn = 0.0, gn = 0.0;
  if (m > 1) {
    an = a[1];
    bn = b[1];
    rn = r[1];
    if (g) gn = g[1];
  }
  for (int k = 1; k < m; k++) {
    const double ak = an, ck = cn, bk = bn, rk = rn, gk = gn;
    if (k + 1 < m) {
      an = a[k + 1];
      cn = c[k];
      bn = b[k + 1];
      rn = r[k + 1];
      if (g) gn = g[k + 1];
    }
    const double w = ak * ib;
    bp = fma(-w, ck, bk);
    rp = fma(-w, rp, rk);
    r[k] = rp;
    if (g) {
      gp = fma(-w, gp, gk);
      g[k] = gp;
    }
    ok &= !badp(bp);
    ib = drcp(bp);
    b[k] = ib;
  }
  return ok;
}

struct Scratch {
  double *a, *b, *c, *r, *g, *y, *z;
};

// Phase 1, a thread per member: its row of _chain_system (_ckernels.pyx:54-71)
// with the ring closure (:114-117) or the branch coupling (:158-161) — the
// diagonal, the two along couplings and the frozen right-hand side, i.e. f
// minus the couplings to the neighbours OUTSIDE the unit (the reference
// subtracts all four and adds the in-block ones back; here they are left out,
// a difference of rounding only).  Every in-block neighbour is a grid
// neighbour, so a direction code replaces the index lookups.  Points finish
// here (relax_points); branches leave their frozen row for the legs' warp.
// Reads the old u only; writes u only at points.
__device__ __forceinline__ void member_build(const Lv& L, int k, const MiniMem* mem,
                                             const Scratch& S) {
  const MiniMem M = mem[k];
  const int i = M.i, j = M.j, p = M.p;
  const unsigned fl = M.fl;
  MINI_CHECK(k >= 0 && k < L.cap, "member scratch slot");
  MINI_CHECK(i > 0 && j > 0 && i < L.nx && j < L.ny && p == i * L.ld + j, "member point");
  const double Wi = L.W[i], Ei = L.E[i], Sj = L.S[j], Nj = L.N[j];
  const double uw = L.u[p - L.ld], ue = L.u[p + L.ld], us = L.u[p - 1], un = L.u[p + 1];
  const double fv = L.f[p], uc = L.u[p];
  const int ad = fl & 7, cd = (fl >> 3) & 7;
  // couplings that stay on the right-hand side: every direction but ad / cd
  const double mW = (ad == 1 || cd == 1) ? 0.0 : Wi, mE = (ad == 2 || cd == 2) ? 0.0 : Ei;
  const double mS = (ad == 3 || cd == 3) ? 0.0 : Sj, mN = (ad == 4 || cd == 4) ? 0.0 : Nj;
  const double r = (fv - fma(mE, ue, mW * uw)) - fma(mN, un, mS * us);
  const double b = -((Wi + Ei) + (Sj + Nj));
  if (fl & MF_POINT) {  // relax_points (_ckernels.pyx:42-51)
    L.u[p] = r * drcp(b);
    return;
  }
  if (fl & MF_BRANCH) {
    S.r[k] = r;
    S.b[k] = b;
    return;
  }
  const double av = ad == 0 ? 0.0 : ad == 1 ? Wi : ad == 2 ? Ei : ad == 3 ? Sj : Nj;
  const double cv = cd == 0 ? 0.0 : cd == 1 ? Wi : cd == 2 ? Ei : cd == 3 ? Sj : Nj;
  if (fl & MF_LEG_LAST) {  // d[k]: the branch row's coupling toward this point
    const double d = cd == 1 ? L.E[i - 1] : cd == 2 ? L.W[i + 1] : cd == 3 ? L.N[j - 1] : L.S[j + 1];
    S.g[k] = d;
    S.y[k] = d * uc;  // the branch's frozen row subtracted this (old) value: added back
  }
  S.a[k] = av;
  S.b[k] = b;
  S.c[k] = cv;
  S.r[k] = r;
}

// Phase 2, a thread per unit (every thread of a warp calls it: the legs of a
// block sit in adjacent lanes and meet through shuffles): the serial
// elimination, the branch row, the back substitution, new values into u.
__device__ __forceinline__ void unit_run(const Lv& L, bool active, const MiniUnit& un,
                                         const MiniMem* smem_, const Scratch& S, int* bad) {
  const unsigned FULL = 0xffffffffu;
  const int kind = active ? un.kind : 255;
  const int m = un.cnt;
  const MiniMem* mm_ = smem_ + un.m0;
  MINI_CHECK(!active || un.kind == 255 || (un.cnt >= 1 && un.m0 + un.cnt <= L.cap), "unit range");
  MINI_CHECK(!active || un.kind != 2 ||
                 (un.mb < L.cap && (smem_[un.mb].fl & MF_BRANCH) &&
                  (int)(threadIdx.x & 31) - (un.leg & 15) >= 0 &&
                  (int)(threadIdx.x & 31) - (un.leg & 15) + (un.leg >> 4) <= 32),
             "leg block in one warp");
  double *a = S.a + un.m0, *b = S.b + un.m0, *c = S.c + un.m0, *r = S.r + un.m0;
  double cn = 0.0, cdn = 0.0;
  if (kind == 1) {  // relax_chain: _thomas_inplace (_ckernels.pyx:74-103)
    if (!eliminate(m, a, b, c, r, nullptr)) *bad = 1;
    double x = r[m - 1] * b[m - 1];
    L.u[mm_[m - 1].p] = x;
    for (int k = m - 2; k >= 0; k--) {
      x = fma(-c[k], x, r[k]) * b[k];
      L.u[mm_[k].p] = x;
    }
  } else if (kind == 3) {  // relax_ring (_ckernels.pyx:118-141)
    double *g = S.g + un.m0, *y = S.y + un.m0, *z = S.z + un.m0;
    const int mm = m - 1;
    const double bmm = b[mm];
    for (int k = 0; k < mm; k++) g[k] = 0.0;
    g[0] = a[0];
    g[mm - 1] = g[mm - 1] + c[mm - 1];
    if (!eliminate(mm, a, b, c, r, g)) *bad = 1;
    double yv = r[mm - 1] * b[mm - 1], zv = g[mm - 1] * b[mm - 1];
    y[mm - 1] = yv;
    z[mm - 1] = zv;
    for (int k = mm - 2; k >= 0; k--) {
      yv = fma(-c[k], yv, r[k]) * b[k];
      zv = fma(-c[k], zv, g[k]) * b[k];
      y[k] = yv;
      z[k] = zv;
    }
    const double den = bmm - c[mm] * z[0] - a[mm] * z[mm - 1];
    if (badp(den)) *bad = 1;
    const double xm = (r[mm] - c[mm] * y[0] - a[mm] * y[mm - 1]) * drcp(den);
    for (int k = 0; k < mm; k++) L.u[mm_[k].p] = fma(-z[k], xm, y[k]);
    L.u[mm_[mm].p] = xm;
  } else if (kind == 2) {  // one leg of relax_legged (_ckernels.pyx:163-170)
    if (!eliminate(m, a, b, c, r, nullptr)) *bad = 1;
    const int e = m - 1;
    const double dib = S.g[un.m0 + e] * b[e];  // b holds the reciprocal pivots
    cn = fma(-dib, r[e], S.y[un.m0 + e]);
    cdn = -dib * c[e];
  }
  // the branch row (_ckernels.pyx:171-175): leg 0 gathers its block's legs
  const int leg = un.leg & 15, nleg = un.leg >> 4;
  double num = cn, den = cdn;
#pragma unroll
  for (int sft = 1; sft < 4; sft++) {
    const double vn = __shfl_down_sync(FULL, cn, sft), vd = __shfl_down_sync(FULL, cdn, sft);
    if (kind == 2 && leg == 0 && sft < nleg) {
      num += vn;
      den += vd;
    }
  }
  double xb = 0.0;
  if (kind == 2 && leg == 0) {
    num += S.r[un.mb];
    den += S.b[un.mb];
    if (badp(den)) *bad = 1;
    xb = num * drcp(den);
    L.u[smem_[un.mb].p] = xb;
  }
  const int src = (threadIdx.x & 31) - (kind == 2 ? leg : 0);
  xb = __shfl_sync(FULL, xb, src);
  if (kind == 2) {  // back substitution (_ckernels.pyx:176-185)
    double xk = fma(-c[m - 1], xb, r[m - 1]) * b[m - 1];
    L.u[mm_[m - 1].p] = xk;
    double cn = 0.0, rn = 0.0, bn = 0.0;
    int pn = 0;
    if (m > 1) {
      cn = c[m - 2];
      rn = r[m - 2];
      bn = b[m - 2];
      pn = mm_[m - 2].p;
    }
    for (int t = m - 2; t >= 0; t--) {
      const double ct = cn, rt = rn, bt = bn;
      const int pt = pn;
      if (t > 0) {
        cn = c[t - 1];
        rn = r[t - 1];
        bn = b[t - 1];
        pn = mm_[t - 1].p;
      }
      xk = fma(-ct, xk, rt) * bt;
      L.u[pt] = xk;
    }
  }
}

#ifdef TMG_MINI_TIMING
#define MINI_MARK(i)                  \
  do {                                \
    if (tid == 0) {                   \
      const long long tn = clock64(); \
      tacc[i] += tn - tlast;          \
      tlast = tn;                     \
    }                                 \
  } while (0)
#else
#define MINI_MARK(i) \
  do {               \
  } while (0)
#endif

__global__ void __launch_bounds__(MT) mini_tail_kernel(MiniArgs a) {
  extern __shared__ __align__(16) unsigned char msm[];
  const int tid = threadIdx.x;
#ifdef TMG_MINI_TIMING
  // thread 0's clocks: prologue, entry load, build, solve (slots 4, 5 unused),
  // residual + restriction, coarse solve, prolongation, exit store
  long long tacc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tlast = clock64();
#endif
  // the plan blob (static) into shared memory while the predecessor drains
#pragma unroll 4
  for (int i = tid; i < a.blob_bytes / 16; i += MT)
    reinterpret_cast<int4*>(msm)[i] = __ldg(reinterpret_cast<const int4*>(a.blob) + i);
  __syncthreads();
  const MiniLevel* lev = reinterpret_cast<const MiniLevel*>(msm + a.o_lev);
  const MiniStage* stages = reinterpret_cast<const MiniStage*>(msm + a.o_stage);
  const MiniUnit* units = reinterpret_cast<const MiniUnit*>(msm + a.o_unit);
  const MiniMem* smem_all = reinterpret_cast<const MiniMem*>(msm + a.o_mem);
  double* dsm = reinterpret_cast<double*>(msm + a.blob_bytes);
  Scratch S;
  S.a = dsm + a.off_scratch;
  S.b = S.a + a.maxmem;
  S.c = S.b + a.maxmem;
  S.r = S.c + a.maxmem;
  S.g = S.r + a.maxmem;
  S.y = S.g + a.maxmem;
  S.z = S.y + a.maxmem;
  __shared__ int s_bad;
  if (tid == 0) s_bad = 0;
  auto level = [&](int l) {
    const MiniLevel& M = lev[l];
    Lv L;
    L.nx = M.nx;
    L.ny = M.ny;
    L.ld = M.ny + 1;
    L.cap = a.maxmem;
    L.u = dsm + M.off_u;
    L.f = dsm + M.off_f;
    L.W = dsm + M.off_w;
    L.E = L.W + M.nx + 1;
    L.S = L.E + M.nx + 1;
    L.N = L.S + M.ny + 1;
    return L;
  };
  // zero fields below the first level; the coefficients, a warp per level so
  // that the levels' global-memory latencies overlap
  for (int l = 1; l < a.nlev; l++) {
    const MiniLevel& M = lev[l];
    const int np = (M.nx + 1) * (M.ny + 1);
    for (int p = tid; p < np; p += MT) {
      dsm[M.off_u + p] = 0.0;
      dsm[M.off_f + p] = 0.0;
    }
  }
  for (int l = tid >> 5; l < a.nlev; l += MT / 32) {
    const MiniLevel& M = lev[l];
    double* w = dsm + M.off_w;
    const int lane = tid & 31;
    for (int i = lane; i <= M.nx; i += 32) {
      const double wv = __ldg(M.W + i), ev = __ldg(M.E + i);
      w[i] = wv;
      w[M.nx + 1 + i] = ev;
    }
    for (int j = lane; j <= M.ny; j += 32) {
      const double sv = __ldg(M.S + j), nv = __ldg(M.N + j);
      w[2 * (M.nx + 1) + j] = sv;
      w[2 * (M.nx + 1) + M.ny + 1 + j] = nv;
    }
  }
  MINI_MARK(0);
  pdl_wait();  // the restriction above (or the caller's fields) is complete
  pdl_trigger();
  {  // the first tail level's u and f: three rounds of loads in flight at once
    const Lv L = level(0);
    const int np = (L.nx + 1) * (L.ny + 1);
    for (int p0 = 0; p0 < np; p0 += 3 * MT) {
      double uv[3], fv[3];
#pragma unroll
      for (int q = 0; q < 3; q++) {
        const int p = p0 + q * MT + tid;
        uv[q] = fv[q] = 0.0;
        if (p < np) {
          const int i = p / L.ld, j = p - i * L.ld;
          uv[q] = *a.U0.at(i, j);
          if (i > 0 && j > 0 && i < L.nx && j < L.ny) fv[q] = *a.F0.at(i, j);
        }
      }
#pragma unroll
      for (int q = 0; q < 3; q++) {
        const int p = p0 + q * MT + tid;
        if (p < np) {
          L.u[p] = uv[q];
          L.f[p] = fv[q];
        }
      }
    }
  }
  __syncthreads();
  MINI_MARK(1);

  auto sweep = [&](const Lv& L, const MiniLevel& M) {
    for (int sidx = 0; sidx < M.nstage; sidx++) {
      const MiniStage st = stages[M.stage0 + sidx];
      const MiniUnit* un = units + st.unit0;
      const MiniMem* mem = smem_all + st.mem0;
      for (int k = tid; k < st.nmem; k += MT) member_build(L, k, mem, S);
      __syncthreads();
      MINI_MARK(2);
      for (int q0 = 0; q0 < st.nunits; q0 += MT) {  // whole warps: the legs meet by shuffles
        const bool active = q0 + tid < st.nunits;
        unit_run(L, active, un[active ? q0 + tid : 0], mem, S, &s_bad);
      }
      __syncthreads();
      MINI_MARK(3);
    }
  };

  // ---- down: smooth, residual + restriction, zero guess (mgcycle.py:96-100) --
  for (int l = 0; l + 1 < a.nlev; l++) {
    const Lv L = level(l);
    const MiniLevel& M = lev[l];
    for (int k = 0; k < a.nu1; k++) sweep(L, M);
    const Lv C = level(l + 1);
    double* dfc = S.a;  // defect of the fine level (stencil.py:82-87), ring 0
    const int np = (L.nx + 1) * (L.ny + 1);
    for (int p = tid; p < np; p += MT) {
      const int i = p / L.ld, j = p - i * L.ld;
      double dv = 0.0;
      if (i > 0 && j > 0 && i < L.nx && j < L.ny) {
        const double Wi = L.W[i], Ei = L.E[i], Sj = L.S[j], Nj = L.N[j];
        const double Cc = -__dadd_rn(__dadd_rn(__dadd_rn(Wi, Ei), Sj), Nj);
        double acc = __dmul_rn(Wi, L.u[p - L.ld]);
        acc = __dadd_rn(acc, __dmul_rn(Ei, L.u[p + L.ld]));
        acc = __dadd_rn(acc, __dmul_rn(Sj, L.u[p - 1]));
        acc = __dadd_rn(acc, __dmul_rn(Nj, L.u[p + 1]));
        dv = __dadd_rn(-__dadd_rn(acc, __dmul_rn(Cc, L.u[p])), L.f[p]);
      }
      dfc[p] = dv;
    }
    __syncthreads();
    const int npc = (C.nx + 1) * (C.ny + 1);
    for (int p = tid; p < npc; p += MT) {
      const int I = p / C.ld, J = p - I * C.ld;
      C.u[p] = 0.0;
      if (I > 0 && J > 0 && I < C.nx && J < C.ny) {  // transfer.py:33-38
        const int o = 2 * I * L.ld + 2 * J, di = L.ld, dj = 1;
        const double ctr = dfc[o];
        const double edges =
            __dadd_rn(__dadd_rn(__dadd_rn(dfc[o - di], dfc[o + di]), dfc[o - dj]), dfc[o + dj]);
        double v;
        if (!a.full) {
          v = __dadd_rn(__dmul_rn(0.5, ctr), __dmul_rn(0.125, edges));
        } else {
          const double diags =
              __dadd_rn(__dadd_rn(__dadd_rn(dfc[o - di - dj], dfc[o + di - dj]), dfc[o - di + dj]),
                        dfc[o + di + dj]);
          v = __dadd_rn(__dadd_rn(__dmul_rn(0.25, ctr), __dmul_rn(0.125, edges)),
                        __dmul_rn(0.0625, diags));
        }
        C.f[p] = v;
      }
    }
    __syncthreads();
    MINI_MARK(6);
  }

  // ---- coarsest level: direct solve (mgcycle.py:93-95, tmg_transfer_dev.cuh) --
  {
    const Lv L = level(a.nlev - 1);
    const int mi_ = L.nx - 1, n = mi_ * (L.ny - 1);
    double* rhs = S.a;
    for (int k = tid; k < n; k += MT) {
      const int i = k % mi_ + 1, j = k / mi_ + 1;
      const double* u = L.u + i * L.ld + j;
      const double bw = i == 1 ? u[-L.ld] : 0.0, be = i == L.nx - 1 ? u[L.ld] : 0.0;
      const double bs = j == 1 ? u[-1] : 0.0, bn = j == L.ny - 1 ? u[1] : 0.0;
      double acc = __dmul_rn(L.W[i], bw);
      acc = __dadd_rn(acc, __dmul_rn(L.E[i], be));
      acc = __dadd_rn(acc, __dmul_rn(L.S[j], bs));
      acc = __dadd_rn(acc, __dmul_rn(L.N[j], bn));
      rhs[k] = __dadd_rn(L.f[i * L.ld + j], -acc);
    }
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    if (n == 1) {
      if (tid == 0) L.u[L.ld + 1] = rhs[0] / __ldg(a.ainv);
    } else {
      for (int row = warp; row < n; row += MT / 32) {
        double acc = 0.0;
        for (int c = lane; c < n; c += 32) acc += __ldg(a.ainv + (size_t)row * n + c) * rhs[c];
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
        if (lane == 0) L.u[(row % mi_ + 1) * L.ld + row / mi_ + 1] = acc;
      }
    }
    __syncthreads();
    MINI_MARK(7);
  }

  // ---- up: prolongation + correction, smooth (mgcycle.py:101-103) ------------
  for (int l = a.nlev - 2; l >= 0; l--) {
    const Lv L = level(l);
    const Lv C = level(l + 1);
    const int np = (L.nx + 1) * (L.ny + 1);
    for (int p = tid; p < np; p += MT) {
      const int i = p / L.ld, j = p - i * L.ld;
      if (i <= 0 || j <= 0 || i >= L.nx || j >= L.ny) continue;
      const int o = (i >> 1) * C.ld + (j >> 1), cI = C.ld, cJ = 1;
      const double* sc = C.u;
      double pv;  // transfer.py:51-53
      if (!(i & 1) && !(j & 1)) pv = sc[o];
      else if (!(i & 1)) pv = __dmul_rn(0.5, __dadd_rn(sc[o], sc[o + cJ]));
      else if (!(j & 1)) pv = __dmul_rn(0.5, __dadd_rn(sc[o], sc[o + cI]));
      else
        pv = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(sc[o], sc[o + cI]), sc[o + cJ]),
                                       sc[o + cI + cJ]));
      L.u[p] = __dadd_rn(L.u[p], pv);
    }
    __syncthreads();
    MINI_MARK(8);
    for (int k = 0; k < a.nu2; k++) sweep(L, lev[l]);
  }

  // ---- the first tail level's iterate back to the hierarchy's work field ------
  {
    const Lv L = level(0);
    const int np = (L.nx + 1) * (L.ny + 1);
    for (int p = tid; p < np; p += MT) {
      const int i = p / L.ld, j = p - i * L.ld;
      if (i > 0 && j > 0 && i < L.nx && j < L.ny) *a.U0.at(i, j) = L.u[p];
    }
  }
  if (tid == 0 && s_bad) atomicOr(a.err, 1);
#ifdef TMG_MINI_TIMING
  MINI_MARK(9);
  if (tid == 0)
    printf("mini tail cycles: prologue %lld entry %lld build %lld solve %lld branch %lld store %lld "
           "restrict %lld coarse %lld prolong %lld exit %lld\n",
           tacc[0], tacc[1], tacc[2], tacc[3], tacc[4], tacc[5], tacc[6], tacc[7], tacc[8], tacc[9]);
#endif
}

}  // namespace

int mini_max_unit(const std::vector<int>& schemes, int nx, int ny) {
  int mx = 1;
  for (int sc : schemes) {
    Geometry g;
    if (!build_geometry(sc, nx, ny, g).empty()) return -1;
    for (const LegD& L : g.legs) mx = std::max(mx, (int)L.npts);
    for (const BlockD& B : g.blocks) {
      if (B.nleg && B.hi >= 0 && (g.legs[B.leg0].flags & 1)) {  // ring: one thread walks it
        int tot = 1;
        for (int l = 0; l < B.nleg; l++) tot += g.legs[B.leg0 + l].npts;
        mx = std::max(mx, tot);
      }
    }
  }
  return mx;
}

std::string build_mini_tail(const std::vector<MiniLevelIn>& lv, const std::vector<int>& schemes,
                            MiniTail& out) {
  out = MiniTail();
  const int nlev = (int)lv.size();
  if (nlev < 2) return "mini tail needs two levels";
  std::vector<MiniLevel> levs(nlev);
  std::vector<MiniStage> stages;
  std::vector<MiniUnit> units;
  std::vector<uint8_t> mi, mj;
  std::vector<uint16_t> mf;
  std::vector<MiniMem> mems;  // (i, j, flags) of mi / mj / mf with the level's row stride
  int maxmem = 1, maxfield = 1, off = 0;
  // direction of (pi, pj) seen from (i, j), _coupling's precedence (_ckernels.pyx:21-31)
  auto dir = [](int i, int j, int pi, int pj) {
    return pi == i - 1 ? 1 : pi == i + 1 ? 2 : pj == j - 1 ? 3 : 4;
  };
  for (int l = 0; l < nlev; l++) {
    MiniLevel& M = levs[l];
    std::memset(&M, 0, sizeof M);
    M.nx = lv[l].nx;
    M.ny = lv[l].ny;
    if (M.nx > 255 || M.ny > 255) return "mini tail level too large";
    M.W = lv[l].W;
    M.E = lv[l].E;
    M.S = lv[l].S;
    M.N = lv[l].N;
    const int np = (M.nx + 1) * (M.ny + 1);
    maxfield = std::max(maxfield, np);
    M.off_w = off;
    off += 2 * (M.nx + 1) + 2 * (M.ny + 1);
    off = (off + 1) & ~1;
    M.off_u = off;
    off += np + (np & 1);
    M.off_f = off;
    off += np + (np & 1);
    M.stage0 = (int)stages.size();
    if (l == nlev - 1) continue;  // the coarsest level is solved directly
    for (int sc : schemes) {
      Geometry g;
      std::string err = build_geometry(sc, M.nx, M.ny, g);
      if (!err.empty()) return err;
      const long n = dump_members(g, nullptr, nullptr, nullptr, nullptr, 0);
      std::vector<int> oi(n), oj(n), ob(n), of(n);
      dump_members(g, oi.data(), oj.data(), ob.data(), of.data(), n);
      for (int red = 1; red >= 0; red--) {
        MiniStage st{};
        st.unit0 = (int)units.size();
        st.mem0 = (int)mi.size();
        // members [s, e) of one unit; `to` = the point its last member couples
        // to beyond the unit (ring: its first member, leg: the branch), or -1
        auto push_members = [&](long s, long e, int ukind, long to) {
          for (long t = s; t < e; t++) {
            mi.push_back((uint8_t)oi[t]);
            mj.push_back((uint8_t)oj[t]);
            unsigned fl = 0;
            if (ukind == 0 || (ukind == 1 && e - s == 1)) {
              fl = MF_POINT;
            } else {
              if (t > s) fl |= dir(oi[t], oj[t], oi[t - 1], oj[t - 1]);
              if (t + 1 < e) fl |= dir(oi[t], oj[t], oi[t + 1], oj[t + 1]) << 3;
              if (ukind == 3 && t == s)
                fl |= MF_RING_FIRST | dir(oi[t], oj[t], oi[e - 1], oj[e - 1]);
              if (t + 1 == e && to >= 0) fl |= dir(oi[t], oj[t], oi[to], oj[to]) << 3;
              if (ukind == 2 && t + 1 == e) fl |= MF_LEG_LAST;
            }
            mf.push_back((uint16_t)fl);
          }
        };
        long p = 0;
        while (p < n) {
          long q = p;
          while (q < n && ob[q] == ob[p]) q++;  // members [p, q) of one block
          if ((of[p] & 1) == red) {
            const int kind = (of[p] >> 4) & 3;
            const int m0 = (int)mi.size() - st.mem0;
            if (kind == 0 || (kind == 1 && q - p == 1)) {
              push_members(p, q, 0, -1);  // a point: finished by the build phase
            } else if (kind == 1 || kind == 3) {
              // line: the chain; ring: the traversal, closing point last
              MiniUnit u{};
              u.m0 = (uint16_t)m0;
              u.cnt = (uint16_t)(q - p);
              u.kind = (uint8_t)kind;
              push_members(p, q, kind, kind == 3 ? p : -1);
              units.push_back(u);
            } else {  // legged: legs tip -> branch, the branch last
              std::vector<std::pair<long, long>> legs;
              for (long s = p; s < q - 1;) {
                long e = s;
                while (e < q - 1 && ((of[e] >> 1) & 7) == ((of[s] >> 1) & 7)) e++;
                legs.push_back({s, e});
                s = e;
              }
              const int nleg = (int)legs.size();
              if (nleg < 1 || nleg > 4) return "mini tail: unsupported leg count";
              // a block's legs sit in adjacent lanes of one warp
              while (((int)units.size() - st.unit0) % 32 + nleg > 32) {
                MiniUnit pad{};
                pad.kind = 255;
                units.push_back(pad);
              }
              int total = 0;
              for (auto& le : legs) total += (int)(le.second - le.first);
              const int mb = m0 + total;  // the branch follows the legs' members
              for (int k = 0; k < nleg; k++) {
                MiniUnit u{};
                u.m0 = (uint16_t)((int)mi.size() - st.mem0);
                u.cnt = (uint16_t)(legs[k].second - legs[k].first);
                u.kind = 2;
                u.leg = (uint8_t)(k | (nleg << 4));
                u.mb = (uint16_t)mb;
                push_members(legs[k].first, legs[k].second, 2, q - 1);
                units.push_back(u);
              }
              mi.push_back((uint8_t)oi[q - 1]);
              mj.push_back((uint8_t)oj[q - 1]);
              mf.push_back((uint16_t)MF_BRANCH);
            }
          }
          p = q;
        }
        st.nunits = (int)units.size() - st.unit0;
        st.nmem = (int)mi.size() - st.mem0;
        for (size_t t = mems.size(); t < mi.size(); t++) {
          MiniMem mm{};
          mm.i = mi[t];
          mm.j = mj[t];
          mm.p = (uint16_t)(mi[t] * (M.ny + 1) + mj[t]);
          mm.fl = mf[t];
          mems.push_back(mm);
        }
        if (st.nmem > 65535) return "mini tail stage too large";
        maxmem = std::max(maxmem, st.nmem);
        stages.push_back(st);
      }
    }
    M.nstage = (int)stages.size() - M.stage0;
  }
  // scratch: seven member arrays (also the defect of a whole field and the
  // coarse right-hand side)
  maxmem = std::max(maxmem, (maxfield + 6) / 7 + 1);
  maxmem = (maxmem + 1) & ~1;
  out.off_scratch = off;
  out.maxmem = maxmem;
  off += 7 * maxmem + 2;
  auto align16 = [](size_t v) { return (v + 15) & ~(size_t)15; };
  std::vector<unsigned char> blob;
  auto put = [&](const void* p, size_t nb) {
    const size_t o = blob.size();
    blob.resize(align16(o + nb), 0);
    if (nb) std::memcpy(blob.data() + o, p, nb);
    return (int)o;
  };
  out.o_lev = put(levs.data(), levs.size() * sizeof(MiniLevel));
  out.o_stage = put(stages.data(), stages.size() * sizeof(MiniStage));
  out.o_unit = put(units.data(), units.size() * sizeof(MiniUnit));
  out.o_mem = put(mems.data(), mems.size() * sizeof(MiniMem));
  out.blob_bytes = (int)blob.size();
  out.smem = blob.size() + (size_t)off * sizeof(double);
  if (out.smem > 200 * 1024) return "mini tail does not fit shared memory";
  if (cudaMalloc(&out.d_blob, blob.size()) != cudaSuccess ||
      cudaMemcpy(out.d_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return "mini tail upload failed";
  out.nlev = nlev;
  return "";
}

void free_mini_tail(MiniTail& t) {
  cudaFree(t.d_blob);
  t = MiniTail();
}

cudaError_t launch_mini_tail(const MiniTail& t, const FieldView& U0, const FieldView& F0,
                             const double* ainv, int full, int nu1, int nu2, int* err,
                             cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(mini_tail_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  MiniArgs a{};
  a.blob = static_cast<const unsigned char*>(t.d_blob);
  a.blob_bytes = t.blob_bytes;
  a.o_lev = t.o_lev;
  a.o_stage = t.o_stage;
  a.o_unit = t.o_unit;
  a.o_mem = t.o_mem;
  a.nlev = t.nlev;
  a.off_scratch = t.off_scratch;
  a.maxmem = t.maxmem;
  a.U0 = U0;
  a.F0 = F0;
  a.ainv = ainv;
  a.full = full;
  a.nu1 = nu1;
  a.nu2 = nu2;
  a.err = err;
  TMG_COUNT(1);
  return launch_pdl(mini_tail_kernel, dim3(1), dim3(MT), t.smem, s, a);
}

}  // namespace tmg
