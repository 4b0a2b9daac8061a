// Shared-memory coarse tail: the smallest levels of a V-cycle
// (mgcycle.py:89-104 from the first tail level down to the direct solve and
// back up) as ONE launch of one CTA.  u and f of every tail level, the 1D
// coefficient arrays and the block plan live in shared memory; colour stages
// and transfers are separated by __syncthreads instead of graph nodes (a
// per-stage launch costs ~4 us at these sizes, a stage here well under 1 us
// of shared-memory latency).
//
// Smoothing follows the reference's per-block kernels statement by statement
// (relax_points / relax_chain / relax_ring / relax_legged,
// _ckernels.pyx:42-185: frozen right-hand side, in-block couplings added
// back in the reference's order by a thread per member; Thomas / circulant /
// m-legged elimination by a thread per chain, ring or leg, multiplying by
// reciprocal pivots where the reference divides: same algorithm, results
// within rounding, gated at 1e-12 per sweep like the block kernels).
// Residual, full / half weighting, bilinear prolongation + correction and the
// coarsest-level solve use the arithmetic of tmg_transfer_dev.cuh
// (stencil.py:82-87, transfer.py:33-38, 51-53, stencil.py:129-155).
#include <cstdint>
#include <cstring>

#include "tmg_minitail.h"
#include "tmg_plan.h"

namespace tmg {

namespace {

constexpr int MT = 256;  // threads of the tail CTA

struct MiniUnit {   // a chain, a ring, a point or one leg of a legged block
  uint16_t m0, cnt;  // members [m0, m0 + cnt) of the stage's member arrays
  uint8_t kind;      // 0 point, 1 chain, 2 leg, 3 ring
  uint8_t leg;       // leg index in its block
  uint16_t blk;      // legged block of the stage (kind 2)
};
struct MiniBlk {  // a legged block: branch point and its leg units
  uint8_t bi, bj, nleg, pad;
  uint16_t unit0, pad2;
};
struct MiniStage {  // one colour of one sub-scheme on one level
  int unit0, nunits, blk0, nblk, mem0, nmem;
};
// per-member flags (the build phase runs a thread per member)
enum : uint8_t {
  MF_PREV = 1,       // couples to the previous member of its unit
  MF_NEXT = 2,       // ... to the next one
  MF_RING_FIRST = 4, // first member of a ring: previous = the ring's last member
  MF_RING_LAST = 8,  // last member of a ring: next = the ring's first member
  MF_LEG_LAST = 16,  // innermost point of a leg: next = the block's branch
  MF_POINT = 32      // a point block / a one-point chain: relax_points
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
  int o_lev, o_stage, o_unit, o_blk, o_mi, o_mj, o_mu, o_mf;  // byte offsets in the blob
  int nlev;
  int off_scratch, maxmem, maxblk;  // doubles, after the blob copy
  FieldView U0, F0;
  const double* ainv;
  int full, nu1, nu2;
  int* err;
};

struct Lv {
  int nx, ny, ld;
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
__device__ bool eliminate(int m, const double* a, double* b, const double* c, double* r,
                          double* g) {
  double bp = b[0], rp = r[0], gp = g ? g[0] : 0.0;
  bool ok = !badp(bp);
  double ib = drcp(bp);
  b[0] = ib;
  for (int k = 1; k < m; k++) {
    const double w = a[k] * ib;
    bp = fma(-w, c[k - 1], b[k]);
    rp = fma(-w, rp, r[k]);
    r[k] = rp;
    if (g) {
      gp = fma(-w, gp, g[k]);
      g[k] = gp;
    }
    ok &= !badp(bp);
    ib = drcp(bp);
    b[k] = ib;
  }
  return ok;
}

struct Scratch {
  double *a, *b, *c, *r, *g, *y, *z, *bx;
};

// phase A1, a thread per member: its row of _chain_system (_ckernels.pyx:54-71)
// with the ring closure (:114-117) or the branch coupling (:158-161) — the
// diagonal, the frozen right-hand side with the in-block couplings added back
// in the reference's order, the two along couplings
__device__ void member_build(const Lv& L, int k, const MiniUnit* units, const MiniBlk* blks,
                             const uint8_t* mi, const uint8_t* mj, const uint16_t* mu,
                             const uint8_t* mf, const Scratch& S) {
  const int i = mi[k], j = mj[k];
  const uint8_t fl = mf[k];
  double r = frozen(L, i, j);
  const double b = diag(L, i, j);
  if (fl & MF_POINT) {  // relax_points (_ckernels.pyx:42-51)
    S.r[k] = __ddiv_rn(r, b);
    return;
  }
  const MiniUnit un = units[mu[k]];
  double av = 0.0, cv = 0.0;
  if (fl & MF_RING_FIRST) {  // the chain's c term first, the closure's a term after
    cv = coupling(L, i, j, mi[k + 1], mj[k + 1]);
    r = __dadd_rn(r, __dmul_rn(cv, L.u[mi[k + 1] * L.ld + mj[k + 1]]));
    const int e = un.m0 + un.cnt - 1;
    av = coupling(L, i, j, mi[e], mj[e]);
    r = __dadd_rn(r, __dmul_rn(av, L.u[mi[e] * L.ld + mj[e]]));
  } else {
    if (fl & MF_PREV) {
      av = coupling(L, i, j, mi[k - 1], mj[k - 1]);
      r = __dadd_rn(r, __dmul_rn(av, L.u[mi[k - 1] * L.ld + mj[k - 1]]));
    }
    if (fl & MF_NEXT) {
      cv = coupling(L, i, j, mi[k + 1], mj[k + 1]);
      r = __dadd_rn(r, __dmul_rn(cv, L.u[mi[k + 1] * L.ld + mj[k + 1]]));
    } else if (fl & MF_RING_LAST) {
      cv = coupling(L, i, j, mi[un.m0], mj[un.m0]);
      r = __dadd_rn(r, __dmul_rn(cv, L.u[mi[un.m0] * L.ld + mj[un.m0]]));
    } else if (fl & MF_LEG_LAST) {
      const MiniBlk B = blks[un.blk];
      cv = coupling(L, i, j, B.bi, B.bj);
      r = __dadd_rn(r, __dmul_rn(cv, L.u[B.bi * L.ld + B.bj]));
      S.g[un.m0] = coupling(L, B.bi, B.bj, i, j);  // d[k] of the branch row
    }
  }
  S.a[k] = av;
  S.b[k] = b;
  S.c[k] = cv;
  S.r[k] = r;
}

// phase A2, a thread per unit: the serial eliminations
__device__ void unit_solve(const MiniUnit& un, const Scratch& S, int* bad) {
  const int m = un.cnt;
  double *a = S.a + un.m0, *b = S.b + un.m0, *c = S.c + un.m0, *r = S.r + un.m0;
  if (un.kind == 0 || (un.kind == 1 && m == 1)) return;
  if (un.kind == 1) {  // relax_chain: _thomas_inplace (_ckernels.pyx:74-103)
    if (!eliminate(m, a, b, c, r, nullptr)) *bad = 1;
    double x = r[m - 1] * b[m - 1];
    r[m - 1] = x;
    for (int k = m - 2; k >= 0; k--) {
      x = fma(-c[k], x, r[k]) * b[k];
      r[k] = x;
    }
    return;
  }
  if (un.kind == 2) {  // one leg of relax_legged (_ckernels.pyx:163-168)
    if (!eliminate(m, a, b, c, r, nullptr)) *bad = 1;
    return;
  }
  // relax_ring (_ckernels.pyx:118-141)
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
  if (badp(den)) {
    *bad = 1;
    return;
  }
  const double xm = (r[mm] - c[mm] * y[0] - a[mm] * y[mm - 1]) * drcp(den);
  for (int k = 0; k < mm; k++) r[k] = fma(-z[k], xm, y[k]);
  r[mm] = xm;
}

// phase B: the branch row of a legged block, legs in order (_ckernels.pyx:156-173)
__device__ void block_branch(const Lv& L, const MiniBlk& B, const MiniUnit* units,
                             const uint8_t* smi, const uint8_t* smj, const Scratch& S, int blk,
                             int* bad) {
  double num = frozen(L, B.bi, B.bj);
  double den = diag(L, B.bi, B.bj);
  for (int k = 0; k < B.nleg; k++) {
    const MiniUnit un = units[B.unit0 + k];
    const int e = un.m0 + un.cnt - 1;
    const double d = S.g[un.m0];
    num = __dadd_rn(num, __dmul_rn(d, L.u[smi[e] * L.ld + smj[e]]));
    const double dib = d * S.b[e];  // b holds the reciprocal pivots
    num = fma(-dib, S.r[e], num);
    den = fma(-dib, S.c[e], den);
  }
  if (badp(den)) {
    *bad = 1;
    den = 1.0;
  }
  S.bx[blk] = num * drcp(den);
}

// phase C: back substitution of a leg, new values into u (_ckernels.pyx:176-185)
__device__ void leg_store(const Lv& L, const MiniUnit& un, const MiniBlk* blks,
                          const uint8_t* smi, const uint8_t* smj, const Scratch& S) {
  const int m = un.cnt;
  const uint8_t *mi = smi + un.m0, *mj = smj + un.m0;
  const double *b = S.b + un.m0, *c = S.c + un.m0, *r = S.r + un.m0;
  const MiniBlk B = blks[un.blk];
  const double xb = S.bx[un.blk];
  if (un.leg == 0) L.u[B.bi * L.ld + B.bj] = xb;
  double xk = fma(-c[m - 1], xb, r[m - 1]) * b[m - 1];
  L.u[mi[m - 1] * L.ld + mj[m - 1]] = xk;
  for (int t = m - 2; t >= 0; t--) {
    xk = fma(-c[t], xk, r[t]) * b[t];
    L.u[mi[t] * L.ld + mj[t]] = xk;
  }
}

__global__ void __launch_bounds__(MT) mini_tail_kernel(MiniArgs a) {
  extern __shared__ __align__(16) unsigned char msm[];
  const int tid = threadIdx.x;
  // the plan blob (static) into shared memory while the predecessor drains
  for (int i = tid; i < a.blob_bytes / 16; i += MT)
    reinterpret_cast<int4*>(msm)[i] = __ldg(reinterpret_cast<const int4*>(a.blob) + i);
  __syncthreads();
  const MiniLevel* lev = reinterpret_cast<const MiniLevel*>(msm + a.o_lev);
  const MiniStage* stages = reinterpret_cast<const MiniStage*>(msm + a.o_stage);
  const MiniUnit* units = reinterpret_cast<const MiniUnit*>(msm + a.o_unit);
  const MiniBlk* blks = reinterpret_cast<const MiniBlk*>(msm + a.o_blk);
  const uint8_t* smi = msm + a.o_mi;
  const uint8_t* smj = msm + a.o_mj;
  const uint16_t* smu = reinterpret_cast<const uint16_t*>(msm + a.o_mu);
  const uint8_t* smf = msm + a.o_mf;
  double* dsm = reinterpret_cast<double*>(msm + a.blob_bytes);
  Scratch S;
  S.a = dsm + a.off_scratch;
  S.b = S.a + a.maxmem;
  S.c = S.b + a.maxmem;
  S.r = S.c + a.maxmem;
  S.g = S.r + a.maxmem;
  S.y = S.g + a.maxmem;
  S.z = S.y + a.maxmem;
  S.bx = S.z + a.maxmem;
  __shared__ int s_bad;
  if (tid == 0) s_bad = 0;
  auto level = [&](int l) {
    const MiniLevel& M = lev[l];
    Lv L;
    L.nx = M.nx;
    L.ny = M.ny;
    L.ld = M.ny + 1;
    L.u = dsm + M.off_u;
    L.f = dsm + M.off_f;
    L.W = dsm + M.off_w;
    L.E = L.W + M.nx + 1;
    L.S = L.E + M.nx + 1;
    L.N = L.S + M.ny + 1;
    return L;
  };
  // coefficients of every level; zero fields below the first level
  for (int l = 0; l < a.nlev; l++) {
    const MiniLevel& M = lev[l];
    double* w = dsm + M.off_w;
    for (int i = tid; i <= M.nx; i += MT) {
      w[i] = __ldg(M.W + i);
      w[M.nx + 1 + i] = __ldg(M.E + i);
    }
    for (int j = tid; j <= M.ny; j += MT) {
      w[2 * (M.nx + 1) + j] = __ldg(M.S + j);
      w[2 * (M.nx + 1) + M.ny + 1 + j] = __ldg(M.N + j);
    }
    if (l > 0) {
      const int np = (M.nx + 1) * (M.ny + 1);
      for (int p = tid; p < np; p += MT) {
        dsm[M.off_u + p] = 0.0;
        dsm[M.off_f + p] = 0.0;
      }
    }
  }
  pdl_wait();  // the restriction above (or the caller's fields) is complete
  pdl_trigger();
  {
    const Lv L = level(0);
    const int np = (L.nx + 1) * (L.ny + 1);
    for (int p = tid; p < np; p += MT) {
      const int i = p / L.ld, j = p - i * L.ld;
      L.u[p] = *a.U0.at(i, j);
      const bool interior = i > 0 && j > 0 && i < L.nx && j < L.ny;
      L.f[p] = interior ? *a.F0.at(i, j) : 0.0;
    }
  }
  __syncthreads();

  auto sweep = [&](const Lv& L, const MiniLevel& M) {
    for (int sidx = 0; sidx < M.nstage; sidx++) {
      const MiniStage st = stages[M.stage0 + sidx];
      const MiniUnit* un = units + st.unit0;
      const MiniBlk* bl = blks + st.blk0;
      const uint8_t *mi = smi + st.mem0, *mj = smj + st.mem0, *mf = smf + st.mem0;
      const uint16_t* mu = smu + st.mem0;
      for (int k = tid; k < st.nmem; k += MT) member_build(L, k, un, bl, mi, mj, mu, mf, S);
      __syncthreads();
      for (int q = tid; q < st.nunits; q += MT) unit_solve(un[q], S, &s_bad);
      if (st.nblk) {
        __syncthreads();
        for (int q = tid; q < st.nblk; q += MT) block_branch(L, bl[q], un, mi, mj, S, q, &s_bad);
      }
      __syncthreads();
      for (int k = tid; k < st.nmem; k += MT)
        if (un[mu[k]].kind != 2) L.u[mi[k] * L.ld + mj[k]] = S.r[k];
      for (int q = tid; q < st.nunits; q += MT)
        if (un[q].kind == 2) leg_store(L, un[q], bl, mi, mj, S);
      __syncthreads();
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
  std::vector<MiniBlk> blks;
  std::vector<uint8_t> mi, mj, mf;
  std::vector<uint16_t> mu;
  int maxmem = 1, maxblk = 1, maxfield = 1, off = 0;
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
        st.blk0 = (int)blks.size();
        st.mem0 = (int)mi.size();
        long p = 0;
        while (p < n) {
          long q = p;
          while (q < n && ob[q] == ob[p]) q++;  // members [p, q) of one block
          if ((of[p] & 1) == red) {
            const int kind = (of[p] >> 4) & 3;
            // members [s, e) of the unit about to be pushed, with their flags
            auto push_members = [&](long s, long e, int ukind) {
              const int uidx = (int)units.size() - st.unit0;
              for (long t = s; t < e; t++) {
                mi.push_back((uint8_t)oi[t]);
                mj.push_back((uint8_t)oj[t]);
                mu.push_back((uint16_t)uidx);
                uint8_t fl = 0;
                if (ukind == 0 || (ukind == 1 && e - s == 1)) {
                  fl = MF_POINT;
                } else {
                  if (t > s) fl |= MF_PREV;
                  if (t + 1 < e) fl |= MF_NEXT;
                  if (ukind == 3 && t == s) fl |= MF_RING_FIRST;
                  if (ukind == 3 && t + 1 == e) fl |= MF_RING_LAST;
                  if (ukind == 2 && t + 1 == e) fl |= MF_LEG_LAST;
                }
                mf.push_back(fl);
              }
            };
            const int m0 = (int)mi.size() - st.mem0;
            if (kind == 0 || kind == 1 || kind == 3) {
              // point: its one member; line: the chain; ring: the traversal
              // (closing point last, as the reference's member order)
              MiniUnit u{};
              u.m0 = (uint16_t)m0;
              u.cnt = (uint16_t)(q - p);
              u.kind = (uint8_t)(kind == 3 ? 3 : kind);
              push_members(p, q, u.kind);
              units.push_back(u);
            } else {  // legged: legs tip -> branch, the branch last
              MiniBlk B{};
              B.bi = (uint8_t)oi[q - 1];
              B.bj = (uint8_t)oj[q - 1];
              B.unit0 = (uint16_t)((int)units.size() - st.unit0);
              const int blk = (int)blks.size() - st.blk0;
              long s = p;
              int nleg = 0;
              while (s < q - 1) {
                long e = s;
                while (e < q - 1 && ((of[e] >> 1) & 7) == ((of[s] >> 1) & 7)) e++;
                MiniUnit u{};
                u.m0 = (uint16_t)((int)mi.size() - st.mem0);
                u.cnt = (uint16_t)(e - s);
                u.kind = 2;
                u.leg = (uint8_t)nleg++;
                u.blk = (uint16_t)blk;
                push_members(s, e, 2);
                units.push_back(u);
                s = e;
              }
              B.nleg = (uint8_t)nleg;
              blks.push_back(B);
            }
          }
          p = q;
        }
        st.nunits = (int)units.size() - st.unit0;
        st.nblk = (int)blks.size() - st.blk0;
        st.nmem = (int)mi.size() - st.mem0;
        if (st.nmem > 65535) return "mini tail stage too large";
        maxmem = std::max(maxmem, st.nmem);
        maxblk = std::max(maxblk, st.nblk);
        stages.push_back(st);
      }
    }
    M.nstage = (int)stages.size() - M.stage0;
  }
  // scratch: seven member arrays (also the defect of a whole field and the
  // coarse right-hand side) and the branch values
  maxmem = std::max(maxmem, (maxfield + 6) / 7 + 1);
  maxmem = (maxmem + 1) & ~1;
  out.off_scratch = off;
  out.maxmem = maxmem;
  out.maxblk = maxblk;
  off += 7 * maxmem + maxblk + 2;
  // the blob
  auto align16 = [](size_t v) { return (v + 15) & ~(size_t)15; };
  std::vector<unsigned char> blob;
  auto put = [&](const void* p, size_t nb) {
    const size_t o = blob.size();
    blob.resize(align16(o + nb), 0);
    if (nb) std::memcpy(blob.data() + o, p, nb);
    return o;
  };
  const size_t o_lev = put(levs.data(), levs.size() * sizeof(MiniLevel));
  const size_t o_stage = put(stages.data(), stages.size() * sizeof(MiniStage));
  const size_t o_unit = put(units.data(), units.size() * sizeof(MiniUnit));
  const size_t o_blk = put(blks.data(), blks.size() * sizeof(MiniBlk));
  const size_t o_mi = put(mi.data(), mi.size());
  const size_t o_mj = put(mj.data(), mj.size());
  const size_t o_mu = put(mu.data(), mu.size() * sizeof(uint16_t));
  const size_t o_mf = put(mf.data(), mf.size());
  out.o_mu = (int)o_mu;
  out.o_mf = (int)o_mf;
  out.smem = blob.size() + (size_t)off * sizeof(double);
  if (out.smem > 200 * 1024) return "mini tail does not fit shared memory";
  if (cudaMalloc(&out.d_blob, blob.size()) != cudaSuccess ||
      cudaMemcpy(out.d_blob, blob.data(), blob.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    return "mini tail upload failed";
  out.nlev = nlev;
  // offsets are kept as fake pointers relative to the blob
  out.d_lev = reinterpret_cast<const void*>(o_lev);
  out.d_stage = reinterpret_cast<const void*>(o_stage);
  out.d_unit = reinterpret_cast<const void*>(o_unit);
  out.d_blk = reinterpret_cast<const void*>(o_blk);
  out.d_mi = reinterpret_cast<const unsigned char*>(o_mi);
  out.d_mj = reinterpret_cast<const unsigned char*>(o_mj);
  // blob size rides in maxblk's neighbour: store it in smem - scratch layout
  out.maxblk = maxblk;
  out.smem = blob.size() + (size_t)off * sizeof(double);
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
  a.o_lev = (int)reinterpret_cast<size_t>(t.d_lev);
  a.o_stage = (int)reinterpret_cast<size_t>(t.d_stage);
  a.o_unit = (int)reinterpret_cast<size_t>(t.d_unit);
  a.o_blk = (int)reinterpret_cast<size_t>(t.d_blk);
  a.o_mi = (int)reinterpret_cast<size_t>(t.d_mi);
  a.o_mj = (int)reinterpret_cast<size_t>(t.d_mj);
  a.o_mu = t.o_mu;
  a.o_mf = t.o_mf;
  a.nlev = t.nlev;
  a.off_scratch = t.off_scratch;
  a.maxmem = t.maxmem;
  a.maxblk = t.maxblk;
  const size_t doubles = (size_t)t.off_scratch + 7 * (size_t)t.maxmem + t.maxblk + 2;
  a.blob_bytes = (int)(t.smem - doubles * sizeof(double));
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
