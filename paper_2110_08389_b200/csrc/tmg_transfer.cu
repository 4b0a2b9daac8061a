// Grid-transfer and residual kernels on the hybrid N/T field layout, second
// generation: every CTA first issues all of its global loads at once (the
// u tile with its halo through registers into shared memory, plus the f
// values of its own points), then computes from shared memory.  Tiles whose
// points (halo included) all live in one buffer are read with lanes along
// that buffer's contiguous axis and kept in shared memory in that
// orientation; the stencil then runs with per-tile strides.  Arithmetic is
// the reference's order with explicit round-to-nearest intrinsics
// (stencil.py:82-87, transfer.py:33-38, 51-53), bit-identical to the
// natural-layout kernels of tmg_grid.cu.
#include <cstdlib>
#include <string>

#include "tmg_kernels.h"
#include "tmg_transfer_dev.cuh"

namespace tmg {

namespace {

// (L u) at smem offset o with element steps si (i) and sj (j), reference order
__device__ __forceinline__ double lu_s(const double* s, int o, int si, int sj, double Wi,
                                      double Ei, double Sj, double Nj) {
  const double Cc = -__dadd_rn(__dadd_rn(__dadd_rn(Wi, Ei), Sj), Nj);
  double acc = __dmul_rn(Wi, s[o - si]);
  acc = __dadd_rn(acc, __dmul_rn(Ei, s[o + si]));
  acc = __dadd_rn(acc, __dmul_rn(Sj, s[o - sj]));
  acc = __dadd_rn(acc, __dmul_rn(Nj, s[o + sj]));
  return __dadd_rn(acc, __dmul_rn(Cc, s[o]));
}

// W, E at i0 .. i0+E-1 and S, N at j0 .. j0+E-1 into shared memory (0
// outside the grid), so that the stencil reads them with LDS
template <int E>
__device__ __forceinline__ void load_coefs(const GridArgs& g, int i0, int j0, double* cW,
                                           double* cE, double* cS, double* cN) {
  for (int t = threadIdx.x; t < 4 * E; t += blockDim.x) {
    const int which = t / E, k = t - which * E;
    if (which < 2) {
      const int i = i0 + k;
      const double v = (i >= 0 && i <= g.nx) ? __ldg((which ? g.E : g.W) + i) : 0.0;
      (which ? cE : cW)[k] = v;
    } else {
      const int j = j0 + k;
      const double v = (j >= 0 && j <= g.ny) ? __ldg((which == 3 ? g.N : g.S) + j) : 0.0;
      (which == 3 ? cN : cS)[k] = v;
    }
  }
}

// ---- residual max-norm: 32 x 32 points per CTA, 4 per thread ----------------

__global__ void __launch_bounds__(256) norm2_kernel(GridArgs g, FieldView U, FieldView F,
                                                    unsigned long long* dmax, GroupSel2 gsel) {
  __shared__ double su[NE * NLD];
  pdl_trigger();
  const int i0 = 1 + blockIdx.y * NT, j0 = 1 + blockIdx.x * NT;
  const int own = box_owner(U, i0 - 1, j0 - 1, NE, NE);
  pdl_wait();
  double fv[4];
  int pi[4], pj[4];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int t = threadIdx.x + k * 256, y = t >> 5, x = t & 31;
    pi[k] = own == 1 ? i0 + x : i0 + y;
    pj[k] = own == 1 ? j0 + y : j0 + x;
    fv[k] = (pi[k] < g.nx && pj[k] < g.ny) ? ld_view(F, own, pi[k], pj[k]) : 0.0;
  }
  __shared__ double cW[NT], cE[NT], cS[NT], cN[NT];
  load_box<NE, NLD>(U, own, i0 - 1, j0 - 1, su);
  load_coefs<NT>(g, i0, j0, cW, cE, cS, cN);
  __syncthreads();
  const int si = own == 1 ? 1 : NLD, sj = own == 1 ? NLD : 1;
  unsigned long long m = 0ull;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int i = pi[k], j = pj[k];
    if (i >= g.nx || j >= g.ny) continue;
    if (gsel.g0 > 0) {
      const int grp = point_group(gsel.scheme, g.nx, g.ny, i, j);
      if (grp < gsel.g0 || grp >= gsel.g1) continue;
    }
    const int t = threadIdx.x + k * 256, y = t >> 5, x = t & 31;
    const double lu = lu_s(su, (y + 1) * NLD + (x + 1), si, sj, cW[i - i0], cE[i - i0],
                           cS[j - j0], cN[j - j0]);
    const double d = fabs(__dadd_rn(-lu, fv[k]));
    const unsigned long long bits = (unsigned long long)__double_as_longlong(d);
    m = bits > m ? bits : m;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, m, s);
    m = o2 > m ? o2 : m;
  }
  // one atomic per CTA (per-warp atomics on one address serialise in L2)
  __shared__ unsigned long long wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 1; k < 8; k++) m = wm[k] > m ? wm[k] : m;
    if (m) atomicMax(dmax, m);
  }
}

// ---- fused residual + restriction: 16 x 16 coarse points per CTA ----------
#ifndef TMG_RC
#define TMG_RC 16
#endif
constexpr int RC = TMG_RC, RD = 2 * RC + 1, RU = 2 * RC + 3, RLU = RU + 1, RLD = RD + 1;
constexpr size_t kRestrictSmem = sizeof(double) * (size_t)(RU * RLU + RD * RLD);
constexpr int RPER = (RD * RD + 255) / 256;

// zero_uc: also write the coarse level's zero initial guess (UC, same layout
// as FC) at every coarse interior point (mgcycle.py:100, fused so that the
// V-cycle needs no separate zeroing launch; the rings stay 0)
__global__ void __launch_bounds__(256) restrict2_kernel(GridArgs g, int full, FieldView U,
                                                        FieldView F, FieldView FC, FieldView UC,
                                                        int zero_uc, GroupSel2 csel) {
  extern __shared__ double rsm[];
  double* su = rsm;
  double* sd = rsm + RU * RLU;
  const int nxc = g.nx / 2, nyc = g.ny / 2;
  const int I0 = 1 + blockIdx.y * RC, J0 = 1 + blockIdx.x * RC;
  const int ui0 = 2 * I0 - 2, uj0 = 2 * J0 - 2;
  pdl_trigger();
  // a partial restriction (one rank's coarse groups) skips tiles outside them
  if (!box_in_groups(csel, nxc, nyc, I0, J0, RC, RC)) {
    pdl_wait();
    return;
  }
  const int own = box_owner(U, ui0, uj0, RU, RU);
  pdl_wait();
  double fv[RPER];
  const bool inner = own >= 0 && ui0 + RD < g.nx && uj0 + RD < g.ny;  // every defect point interior
  if (inner) {
    const double* base = own == 1 ? F.t + F.off_t(ui0 + 1, uj0 + 1) : F.n + F.off_n(ui0 + 1, uj0 + 1);
    const int ldr = own == 1 ? g.nx + 1 : g.ny + 1;
#pragma unroll
    for (int k = 0; k < RPER; k++) {
      const int t = threadIdx.x + k * 256, y = t / RD, x = t - y * RD;
      fv[k] = t < RD * RD ? __ldg(base + (size_t)y * ldr + x) : 0.0;
    }
  } else {
#pragma unroll
    for (int k = 0; k < RPER; k++) {
      const int t = threadIdx.x + k * 256, y = t / RD, x = t - y * RD;
      const int i = ui0 + 1 + (own == 1 ? x : y), j = uj0 + 1 + (own == 1 ? y : x);
      fv[k] = (t < RD * RD && i < g.nx && j < g.ny) ? ld_view(F, own, i, j) : 0.0;
    }
  }
  __shared__ double cW[RD], cE[RD], cS[RD], cN[RD];
  load_box<RU, RLU>(U, own, ui0, uj0, su);
  load_coefs<RD>(g, ui0 + 1, uj0 + 1, cW, cE, cS, cN);
  __syncthreads();
  const int si = own == 1 ? 1 : RLU, sj = own == 1 ? RLU : 1;
#pragma unroll
  for (int k = 0; k < RPER; k++) {
    const int t = threadIdx.x + k * 256, y = t / RD, x = t - y * RD;
    if (t >= RD * RD) continue;
    const int i = ui0 + 1 + (own == 1 ? x : y), j = uj0 + 1 + (own == 1 ? y : x);
    double dv = 0.0;
    if (i < g.nx && j < g.ny) {
      const double lu = lu_s(su, (y + 1) * RLU + (x + 1), si, sj, cW[i - ui0 - 1],
                             cE[i - ui0 - 1], cS[j - uj0 - 1], cN[j - uj0 - 1]);
      dv = __dadd_rn(-lu, fv[k]);
    }
    sd[y * RLD + x] = dv;
  }
  __syncthreads();
  // coarse point, lanes along the coarse owner's contiguous axis
  const int cown = box_owner(FC, I0, J0, RC, RC);
  for (int cpt = threadIdx.x; cpt < RC * RC; cpt += 256) {
  const int p = cpt / RC, q = cpt - p * RC;
  const int ca = cown == 1 ? q : p, cb = cown == 1 ? p : q;  // I offset, J offset
  const int I = I0 + ca, J = J0 + cb;
  if (I < nxc && J < nyc && in_groups(csel, nxc, nyc, I, J)) {
    const int a = 2 * ca + 1, b = 2 * cb + 1;  // fine (i, j) offsets in the defect tile
    const int o = own == 1 ? b * RLD + a : a * RLD + b;
    const int di = own == 1 ? 1 : RLD, dj = own == 1 ? RLD : 1;
    const double ctr = sd[o];
    const double edges = __dadd_rn(__dadd_rn(__dadd_rn(sd[o - di], sd[o + di]), sd[o - dj]),
                                   sd[o + dj]);
    double v;
    if (!full) {
      v = __dadd_rn(__dmul_rn(0.5, ctr), __dmul_rn(0.125, edges));
    } else {
      const double diags = __dadd_rn(
          __dadd_rn(__dadd_rn(sd[o - di - dj], sd[o + di - dj]), sd[o - di + dj]), sd[o + di + dj]);
      v = __dadd_rn(__dadd_rn(__dmul_rn(0.25, ctr), __dmul_rn(0.125, edges)),
                    __dmul_rn(0.0625, diags));
    }
    if (cown == 1) FC.t[FC.off_t(I, J)] = v;
    else if (cown == 0) FC.n[FC.off_n(I, J)] = v;
    else *FC.at(I, J) = v;
    if (zero_uc) {
      if (cown == 1) UC.t[UC.off_t(I, J)] = 0.0;
      else if (cown == 0) UC.n[UC.off_n(I, J)] = 0.0;
      else *UC.at(I, J) = 0.0;
    }
  }
  }
}

// ---- fused residual + restriction, second layout: 15 x 15 coarse points per
// CTA (31 x 31 fine defects, a 33 x 33 u box), warps along the tile's rows and
// lanes along its columns in the owner buffer's orientation, so that every
// index is a compile-time offset (restrict2_kernel spends most of its issue
// slots on per-element index division).  Same arithmetic, bit for bit.
// ---- fused residual + restriction, second layout: 15 x 15 coarse points per
// CTA (31 x 31 fine defects, a 33 x 33 u box), warps along the tile's rows and
// lanes along its columns in the owner buffer's orientation, every index a
// compile-time offset from one per-thread base (restrict2_kernel spends most
// of its issue slots on per-element index division).  Same arithmetic, bit
// for bit.
#ifndef TMG_RESTRICT_MINB
#define TMG_RESTRICT_MINB 4
#endif
__global__ void __launch_bounds__(256, TMG_RESTRICT_MINB) restrict3_kernel(GridArgs g, int full, FieldView U,
                                                           FieldView F, FieldView FC,
                                                           FieldView UC, int zero_uc,
                                                           GroupSel2 csel) {
  __shared__ double su[R3U * R3LU];
  __shared__ double sd[R3D * R3LD];
  pdl_trigger();
  restrict3_tile(g, full, U, F, FC, UC, zero_uc, csel, 1 + blockIdx.y * R3C,
                 1 + blockIdx.x * R3C, su, sd);
}

// ---- fused prolongation + correction: 32 x 32 fine points per CTA --------
#ifndef TMG_PROLONG_MINB
#define TMG_PROLONG_MINB 6  // resident CTAs per SM the register allocation aims at (40 registers:
                            // 326 -> 254 us at 8193^2, the kernel is bound by loads in flight)
#endif
__global__ void __launch_bounds__(256, TMG_PROLONG_MINB) prolong2_kernel(int nx, int ny, FieldView C, FieldView U,
                                                       GroupSel2 fsel, int skip_red) {
  __shared__ double sc[PC_E * PC_LD];
  prolong2_tile(nx, ny, C, U, fsel, 1 + blockIdx.y * NT, 1 + blockIdx.x * NT, sc, skip_red);
}

// ---- black-only prolongation + correction of square tweed levels (hybrid
// layout): 64 x 64 fine points per CTA.  In a single-owner tile the rows of
// the owner buffer are shell rows, the black ones are the even rows, and a
// thread takes four of them in two column blocks: eight loads in flight per
// thread where the 32 x 32 kernel with half of its warps idle has four.
// Black rows have an even index across the rows, so only the two interpolation
// classes of transfer.py:51-53 with that index even occur.  Same expressions
// as prolong2_tile (bit-identical); other tiles go through it, 32 x 32 at a
// time.
constexpr int PB_E = 33, PB_LD = 34;
__global__ void __launch_bounds__(256, 4) prolong_black_kernel(int nx, int ny, FieldView C,
                                                             FieldView U) {
  __shared__ double sc[PB_E * PB_LD];
  const int i0 = 1 + blockIdx.y * 64, j0 = 1 + blockIdx.x * 64;
  const int own = box_owner(U, i0, j0, 64, 64);
  const int Ic0 = i0 >> 1, Jc0 = j0 >> 1;
  pdl_trigger();
  const int cown = box_owner(C, Ic0, Jc0, PB_E, PB_E);
  if (!(own >= 0 && cown >= 0 && i0 + 64 <= nx && j0 + 64 <= ny)) {
    for (int q = 0; q < 4; q++) {  // prolong2_tile waits for the predecessor itself
      prolong2_tile(nx, ny, C, U, GroupSel2{0, 0, 0}, i0 + 32 * (q >> 1), j0 + 32 * (q & 1), sc, 1);
      __syncthreads();
    }
    return;
  }
  pdl_wait();
  const bool T = own == 1;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t ldr = T ? nx + 1 : ny + 1, l16 = 16 * ldr;
  // black rows of the tile: offsets 1, 3, ..., 63 from its (odd) first row
  double* up = (T ? U.t : U.n) + ((T ? j0 : i0) + 1 + 2 * w) * ldr + (T ? i0 : j0) + lane;
  double uv[4][2];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uv[q][0] = up[q * l16];
    uv[q][1] = up[q * l16 + 32];
  }
  load_box<PB_E, PB_LD>(C, cown, Ic0, Jc0, sc);
  __syncthreads();
  const int cI = cown == 1 ? 1 : PB_LD, cJ = cown == 1 ? PB_LD : 1;
  const int cR = T ? cJ : cI, cA = T ? cI : cJ;  // coarse strides across / along the rows
  const bool a_even = lane & 1;                   // the column index (i0, j0 are odd)
#pragma unroll
  for (int q = 0; q < 4; q++) {
#pragma unroll
    for (int hb = 0; hb < 2; hb++) {
      const int o = (1 + w + 8 * q) * cR + (((1 + lane) >> 1) + 16 * hb) * cA;
      const double pv = a_even ? sc[o] : __dmul_rn(0.5, __dadd_rn(sc[o], sc[o + cA]));
      up[q * l16 + 32 * hb] = __dadd_rn(uv[q][hb], pv);
    }
  }
}

// ---- marching residual kernels (large levels) -----------------------------
// A warp owns 64 consecutive points along its buffer's contiguous ("lane")
// axis, two per lane, and marches along the other ("march") axis keeping a
// three-row window of u in registers: every u and f value is loaded once per
// warp (coalesced, 512 B per row), the lane-axis neighbours come from the
// adjacent lanes by shuffles and the window's edge columns from three extra
// loads (lanes 0, 1 and 31).  No shared memory, no per-point index division:
// the residual work is a handful of instructions per point, so the kernel
// runs at the HBM rate where the tiled kernels above are issue-bound.
// Mode 0: the warp's box lives in N (lanes along j), 1: in T (lanes along i),
// 2: mixed ownership (lanes along j, every load through FieldView::at).

template <int MODE>
struct RowLoader {
  const double* base;  // owner buffer (modes 0, 1)
  FieldView v;         // mode 2
  int ldr, nA, nM;     // row stride, last lane-axis / march-axis index (the ring)
  __device__ __forceinline__ double ld(int m, int a) const {
    if (a < 0 || a > nA || m < 0 || m > nM) return 0.0;
    if constexpr (MODE == 2) return __ldg(v.at(m, a));
    else return __ldg(base + (size_t)m * ldr + a);
  }
};

template <int MODE>
__device__ __forceinline__ RowLoader<MODE> row_loader(const FieldView& v) {
  RowLoader<MODE> r;
  r.v = v;
  if constexpr (MODE == 1) {
    r.base = v.t; r.ldr = v.nx + 1; r.nA = v.nx; r.nM = v.ny;
  } else {
    r.base = v.n; r.ldr = v.ny + 1; r.nA = v.ny; r.nM = v.nx;
  }
  return r;
}

// one row of a lane's window: lane-axis points a0, a0 + 1 and the lane's
// extra column (lane 0: first - 1, lane 1: first - 2, lane 31: first + 64)
struct Row3 {
  double c0, c1, x;
};

template <int MODE>
__device__ __forceinline__ Row3 load_row(const RowLoader<MODE>& L, int m, int a0, int ax) {
  Row3 r;
  r.c0 = L.ld(m, a0);
  r.c1 = L.ld(m, a0 + 1);
  r.x = ax >= -1 ? L.ld(m, ax) : 0.0;
  return r;
}

// defect f - L u at one point in the reference's order (stencil.py:82-87):
// (mm, mp) the march-axis neighbours, (am, ap) the lane-axis ones, (lm_lo,
// lm_hi) the march-axis coefficients toward them, (la_lo, la_hi) the lane-axis
// ones.  Mode 1 has i along the lane axis.
template <int MODE>
__device__ __forceinline__ double defect_pt(double c, double mm, double mp, double am, double ap,
                                            double cm_lo, double cm_hi, double ca_lo, double ca_hi,
                                            double fv) {
  double Wi, Ei, Sj, Nj, im, ip, jm, jp;
  if constexpr (MODE == 1) {
    Wi = ca_lo; Ei = ca_hi; Sj = cm_lo; Nj = cm_hi; im = am; ip = ap; jm = mm; jp = mp;
  } else {
    Wi = cm_lo; Ei = cm_hi; Sj = ca_lo; Nj = ca_hi; im = mm; ip = mp; jm = am; jp = ap;
  }
  const double Cc = -__dadd_rn(__dadd_rn(__dadd_rn(Wi, Ei), Sj), Nj);
  double acc = __dmul_rn(Wi, im);
  acc = __dadd_rn(acc, __dmul_rn(Ei, ip));
  acc = __dadd_rn(acc, __dmul_rn(Sj, jm));
  acc = __dadd_rn(acc, __dmul_rn(Nj, jp));
  return __dadd_rn(-__dadd_rn(acc, __dmul_rn(Cc, c)), fv);
}

// Defects of fine row m at the lane's points a0, a0 + 1 (d0, d1) and, on lane
// 0, at a0 - 1 (dx).  (p, r, n) = u rows m - 1, m, m + 1.
template <int MODE>
__device__ __forceinline__ void defect_row(const Row3& p, const Row3& r, const Row3& n,
                                           const Row3& f, double cm_lo, double cm_hi,
                                           const double (&ca_lo)[3], const double (&ca_hi)[3],
                                           int lane, double& d0, double& d1, double& dx) {
  constexpr unsigned FULL = 0xffffffffu;
  const double up1 = __shfl_up_sync(FULL, r.c1, 1);   // u at a0 - 1 (lanes > 0)
  const double dn0 = __shfl_down_sync(FULL, r.c0, 1); // u at a0 + 2 (lanes < 31)
  const double x1 = __shfl_down_sync(FULL, r.x, 1);   // lane 0: u at a0 - 2 (lane 1's extra)
  const double am0 = lane == 0 ? r.x : up1;
  const double ap1 = lane == 31 ? r.x : dn0;
  d0 = defect_pt<MODE>(r.c0, p.c0, n.c0, am0, r.c1, cm_lo, cm_hi, ca_lo[0], ca_hi[0], f.c0);
  d1 = defect_pt<MODE>(r.c1, p.c1, n.c1, r.c0, ap1, cm_lo, cm_hi, ca_lo[1], ca_hi[1], f.c1);
  dx = defect_pt<MODE>(r.x, p.x, n.x, x1, r.c0, cm_lo, cm_hi, ca_lo[2], ca_hi[2], f.x);
}

// Residual max-norm over a 128 x 128 fine box per CTA (warp: 64 lane-axis
// points x 32 march steps).
template <int MODE>
__device__ __forceinline__ unsigned long long norm_march_warp(const GridArgs& g, const FieldView& U,
                                                              const FieldView& F, int i0, int j0) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int A0 = (MODE == 1 ? i0 : j0) + 64 * (w & 1);
  const int R0 = (MODE == 1 ? j0 : i0) + 32 * (w >> 1);
  const int nA = MODE == 1 ? g.nx : g.ny, nM = MODE == 1 ? g.ny : g.nx;
  const int Rend = min(R0 + 32, nM);
  unsigned long long mx = 0ull;
  if (R0 >= Rend || A0 >= nA) return mx;
  const RowLoader<MODE> LU = row_loader<MODE>(U), LF = row_loader<MODE>(F);
  const int a0 = A0 + 2 * lane;
  const int ax = lane == 0 ? A0 - 1 : lane == 31 ? A0 + 64 : -2;
  const double* alo = MODE == 1 ? g.W : g.S;
  const double* ahi = MODE == 1 ? g.E : g.N;
  const double* mlo = MODE == 1 ? g.S : g.W;
  const double* mhi = MODE == 1 ? g.N : g.E;
  double ca_lo[3], ca_hi[3];
  {
    const int cols[3] = {a0, a0 + 1, a0};
#pragma unroll
    for (int k = 0; k < 3; k++) {
      const int c = min(cols[k], nA);
      ca_lo[k] = __ldg(alo + c);
      ca_hi[k] = __ldg(ahi + c);
    }
  }
  const bool v0 = a0 < nA, v1 = a0 + 1 < nA;  // interior lane-axis points
  Row3 rp = load_row(LU, R0 - 1, a0, ax), rc = load_row(LU, R0, a0, ax);
  Row3 rn = load_row(LU, R0 + 1, a0, ax), fr = load_row(LF, R0, a0, -2);
  for (int m = R0; m < Rend; m++) {
    Row3 nn, nf;
    const bool more = m + 1 < Rend;
    if (more) {
      nn = load_row(LU, m + 2, a0, ax);
      nf = load_row(LF, m + 1, a0, -2);
    }
    double d0, d1, dx;
    defect_row<MODE>(rp, rc, rn, fr, __ldg(mlo + m), __ldg(mhi + m), ca_lo, ca_hi, lane, d0, d1,
                     dx);
    if (v0) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(d0));
      mx = b > mx ? b : mx;
    }
    if (v1) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(d1));
      mx = b > mx ? b : mx;
    }
    rp = rc; rc = rn;
    if (more) { rn = nn; fr = nf; }
  }
  return mx;
}

__global__ void __launch_bounds__(256, 4) norm_march_kernel(GridArgs g, FieldView U, FieldView F,
                                                         unsigned long long* dmax) {
  const int i0 = 1 + 128 * blockIdx.y, j0 = 1 + 128 * blockIdx.x;
  pdl_trigger();
  const int own = box_owner(U, i0 - 1, j0 - 1, 130, 130);
  pdl_wait();
  unsigned long long m;
  if (own == 1) m = norm_march_warp<1>(g, U, F, i0, j0);
  else if (own == 0) m = norm_march_warp<0>(g, U, F, i0, j0);
  else m = norm_march_warp<2>(g, U, F, i0, j0);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, m, s);
    m = o2 > m ? o2 : m;
  }
  __shared__ unsigned long long wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 1; k < 8; k++) m = wm[k] > m ? wm[k] : m;
    if (m) atomicMax(dmax, m);
  }
}

// Residual max-norm, strip variant: a thread owns SR consecutive points
// along the march axis of one lane-axis column and issues every load of the
// strip at once (SR + 2 centre-column values, 2 SR side values -- L1 hits of
// the neighbouring lanes' lines -- and SR f values), then evaluates the SR
// defects from registers.  A warp covers 32 lane-axis columns x SR steps;
// a CTA 64 x (4 SR) points (same box for both orientations).
#ifndef TMG_NORM_SR
#define TMG_NORM_SR 8
#endif
template <int MODE>
__device__ __forceinline__ unsigned long long norm_strip_warp(const GridArgs& g, const FieldView& U,
                                                              const FieldView& F, int i0, int j0) {
  constexpr int SR = TMG_NORM_SR;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int a = (MODE == 1 ? i0 : j0) + 32 * (w & 1) + lane;
  const int R0 = (MODE == 1 ? j0 : i0) + SR * (w >> 1);
  const int nA = MODE == 1 ? g.nx : g.ny, nM = MODE == 1 ? g.ny : g.nx;
  const RowLoader<MODE> LU = row_loader<MODE>(U), LF = row_loader<MODE>(F);
  double uc[SR + 2], ul[SR], uh[SR], fv[SR];
#pragma unroll
  for (int k = 0; k < SR + 2; k++) uc[k] = LU.ld(R0 - 1 + k, a);
#pragma unroll
  for (int k = 0; k < SR; k++) {
    ul[k] = LU.ld(R0 + k, a - 1);
    uh[k] = LU.ld(R0 + k, a + 1);
    fv[k] = LF.ld(R0 + k, a);
  }
  const double* alo = MODE == 1 ? g.W : g.S;
  const double* ahi = MODE == 1 ? g.E : g.N;
  const double* mlo = MODE == 1 ? g.S : g.W;
  const double* mhi = MODE == 1 ? g.N : g.E;
  const int ac = min(a, nA);
  const double ca_lo = __ldg(alo + ac), ca_hi = __ldg(ahi + ac);
  unsigned long long mx = 0ull;
  if (a >= nA) return mx;
#pragma unroll
  for (int k = 0; k < SR; k++) {
    const int m = R0 + k;
    if (m < nM) {
      const double d = defect_pt<MODE>(uc[k + 1], uc[k], uc[k + 2], ul[k], uh[k], __ldg(mlo + m),
                                       __ldg(mhi + m), ca_lo, ca_hi, fv[k]);
      const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(d));
      mx = b > mx ? b : mx;
    }
  }
  return mx;
}

__global__ void __launch_bounds__(256) norm_strip_kernel(GridArgs g, FieldView U, FieldView F,
                                                         unsigned long long* dmax) {
  constexpr int BM = 4 * TMG_NORM_SR;  // march-axis extent of the CTA box (lane axis: 64)
  // CTA box: 64 x 64 points, 64 / BM passes of the eight warps
  const int i0 = 1 + 64 * blockIdx.y, j0 = 1 + 64 * blockIdx.x;
  pdl_trigger();
  const int own = box_owner(U, i0 - 1, j0 - 1, 66, 66);
  pdl_wait();
  unsigned long long m = 0ull;
#pragma unroll 1
  for (int pass = 0; pass < 64 / BM; pass++) {
    unsigned long long p;
    const int di = own == 1 ? 0 : pass * BM, dj = own == 1 ? pass * BM : 0;
    if (own == 1) p = norm_strip_warp<1>(g, U, F, i0 + di, j0 + dj);
    else if (own == 0) p = norm_strip_warp<0>(g, U, F, i0 + di, j0 + dj);
    else p = norm_strip_warp<2>(g, U, F, i0 + di, j0 + dj);
    m = p > m ? p : m;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, m, s);
    m = o2 > m ? o2 : m;
  }
  __shared__ unsigned long long wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 1; k < 8; k++) m = wm[k] > m ? wm[k] : m;
    if (m) atomicMax(dmax, m);
  }
}

// levels at least this large (fine points per axis) take the strip / marching norm kernels
int march_min() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("TMG_MARCH_MIN");  // A/B knob: a huge value disables
    v = e ? std::atoi(e) : 4096;
  }
  return v;
}

int norm_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("TMG_NORM");  // A/B knob: 1 marching warps, else strips
    v = e ? std::atoi(e) : 0;
  }
  return v;
}

}  // namespace

cudaError_t launch_norm2(const GridArgs& g, const FieldView& U, const FieldView& F,
                         unsigned long long* dmax, cudaStream_t s, int scheme, int g0, int g1) {
  if (g.nx < 2 || g.ny < 2) return cudaSuccess;
  if (g0 <= 0 && g.nx >= march_min() && g.ny >= march_min()) {
    TMG_COUNT(1);
    if (norm_variant() == 1) {
      dim3 grid((g.ny - 1 + 127) / 128, (g.nx - 1 + 127) / 128);
      return launch_pdl(norm_march_kernel, grid, dim3(256), 0, s, g, U, F, dmax);
    }
    dim3 grid((g.ny - 1 + 63) / 64, (g.nx - 1 + 63) / 64);
    return launch_pdl(norm_strip_kernel, grid, dim3(256), 0, s, g, U, F, dmax);
  }
  dim3 grid((g.ny - 1 + NT - 1) / NT, (g.nx - 1 + NT - 1) / NT);
  TMG_COUNT(1);
  return launch_pdl(norm2_kernel, grid, dim3(256), 0, s, g, U, F, dmax,
                    GroupSel2{scheme, g0, g1});
}

cudaError_t launch_restrict2(const GridArgs& g, int full, const FieldView& U, const FieldView& F,
                             const FieldView& FC, cudaStream_t s, const FieldView* UC, int scheme,
                             int cg0, int cg1) {
  const int nxc = g.nx / 2, nyc = g.ny / 2;
  if (nxc < 2 || nyc < 2) return cudaSuccess;
  static int v2 = -1;
  if (v2 < 0) {
    const char* e = std::getenv("TMG_RESTRICT");
    v2 = e && std::string(e) == "v2";
  }
  if (!v2) {  // restrict3_kernel (same arithmetic, 2D thread mapping)
    dim3 grid3((nyc - 1 + R3C - 1) / R3C, (nxc - 1 + R3C - 1) / R3C);
    TMG_COUNT(1);
    return launch_pdl(restrict3_kernel, grid3, dim3(256), 0, s, g, full, U, F, FC,
                      UC ? *UC : FC, UC ? 1 : 0, GroupSel2{scheme, cg0, cg1});
  }
  dim3 grid((nyc - 1 + RC - 1) / RC, (nxc - 1 + RC - 1) / RC);
  TMG_COUNT(1);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(restrict2_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kRestrictSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  return launch_pdl(restrict2_kernel, grid, dim3(256), kRestrictSmem, s, g, full, U, F, FC,
                    UC ? *UC : FC, UC ? 1 : 0, GroupSel2{scheme, cg0, cg1});
}

cudaError_t launch_prolong2(int nx, int ny, const FieldView& C, const FieldView& U,
                            cudaStream_t s, int scheme, int fg0, int fg1, int skip_red) {
  if (nx < 2 || ny < 2) return cudaSuccess;
  static const int black64 = [] {
    const char* e = std::getenv("TMG_PROLONG_BLACK64");
    return e ? std::atoi(e) : 1;
  }();
  // small levels keep the 32 x 32 kernel: most of their tiles straddle the
  // owner diagonals and would take the four-sub-tile path (config 1: +5 %)
  if (skip_red && fg0 <= 0 && black64 && U.mode == LM_TWEED && nx >= 512) {
    dim3 grid64((ny - 1 + 63) / 64, (nx - 1 + 63) / 64);
    TMG_COUNT(1);
    return launch_pdl(prolong_black_kernel, grid64, dim3(256), 0, s, nx, ny, C, U);
  }
  dim3 grid((ny - 1 + NT - 1) / NT, (nx - 1 + NT - 1) / NT);
  TMG_COUNT(1);
  return launch_pdl(prolong2_kernel, grid, dim3(256), 0, s, nx, ny, C, U,
                    GroupSel2{scheme, fg0, fg1}, skip_red);
}

}  // namespace tmg
