// Device bodies shared by the transfer kernels (tmg_transfer.cu) and the
// persistent coarse-tail kernel (tmg_sweep.cu): owner-buffer helpers of the
// hybrid N/T layout, the tiled residual + restriction (15 x 15 coarse points)
// and prolongation + correction (32 x 32 fine points), the coarsest-level
// direct solve.  Arithmetic in the reference's order with explicit
// round-to-nearest intrinsics (stencil.py:82-87, transfer.py:33-38, 51-53).
#pragma once

#include "tmg_kernels.h"

namespace tmg {
namespace {

__device__ __forceinline__ void mirror_range2(int a, int b, int n, int& lo, int& hi) {
  const int ma = min(a, n - a), mb = min(b, n - b);
  lo = min(ma, mb);
  hi = (a <= n / 2 && n / 2 <= b) ? n / 2 : max(ma, mb);
}

// 1: every interior point of the box is T-owned, 0: every one N-owned,
// -1: mixed (tmg_hybrid.cu tile_owner_exact; ring points count as both)
__device__ __forceinline__ int box_owner(const FieldView& v, int i0, int j0, int ni, int nj) {
  if (v.mode == LM_NATURAL) return 0;
  const int ia = max(i0, 1), ib = min(i0 + ni - 1, v.nx - 1);
  const int ja = max(j0, 1), jb = min(j0 + nj - 1, v.ny - 1);
  if (ia > ib || ja > jb) return 0;
  if (v.mode == LM_XLINES) return 1;
  int ilo, ihi, jlo, jhi;
  mirror_range2(ia, ib, v.nx, ilo, ihi);
  mirror_range2(ja, jb, v.ny, jlo, jhi);
  if (v.mode == LM_TWEED) {
    if (ihi < jlo) return 1;
    if (ilo >= jhi) return 0;
    return -1;
  }
  if (jhi < ilo) return 1;
  if (jlo >= ihi) return 0;
  return -1;
}

__device__ __forceinline__ double ld_view(const FieldView& v, int own, int i, int j) {
  return own == 1 ? __ldg(v.t + v.off_t(i, j)) : own == 0 ? __ldg(v.n + v.off_n(i, j))
                                                          : __ldg(v.at(i, j));
}

// Box of E x E points at (i0, j0) -> s[y * LDS + x]; (x, y) = (j - j0, i - i0)
// unless own == 1, then (i - i0, j - j0).  Points outside the grid read 0.
template <int E, int LDS>
__device__ __forceinline__ void load_box(const FieldView& v, int own, int i0, int j0, double* s) {
  constexpr int N = E * E, PER = (N + 255) / 256;
  double val[PER];
  if (own >= 0 && i0 >= 0 && j0 >= 0 && i0 + E - 1 <= v.nx && j0 + E - 1 <= v.ny) {
    // uniform box inside the grid: one base pointer, row stride of the buffer
    const double* base = own == 1 ? v.t + v.off_t(i0, j0) : v.n + v.off_n(i0, j0);
    const int ldr = own == 1 ? v.nx + 1 : v.ny + 1;
#pragma unroll
    for (int k = 0; k < PER; k++) {
      const int t = threadIdx.x + k * 256;
      const int y = t / E, x = t - y * E;
      val[k] = t < N ? __ldg(base + (size_t)y * ldr + x) : 0.0;
    }
  } else {
#pragma unroll
    for (int k = 0; k < PER; k++) {
      const int t = threadIdx.x + k * 256;
      val[k] = 0.0;
      if (t < N) {
        const int y = t / E, x = t - y * E;
        const int i = own == 1 ? i0 + x : i0 + y, j = own == 1 ? j0 + y : j0 + x;
        if (i >= 0 && j >= 0 && i <= v.nx && j <= v.ny) val[k] = ld_view(v, own, i, j);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const int t = threadIdx.x + k * 256;
    if (t < N) {
      const int y = t / E, x = t - y * E;
      s[y * LDS + x] = val[k];
    }
  }
}

struct GroupSel2 {
  int scheme, g0, g1;
};

// (lo, hi) = the smallest / largest sharding group (tmg_layout.h point_group)
// of the interior points of a box; a CTA whose box misses [g0, g1) skips
__device__ __forceinline__ bool box_in_groups(const GroupSel2& s, int nx, int ny, int i0, int j0,
                                              int ni, int nj) {
  if (s.g0 <= 0) return true;
  const int ia = max(i0, 1), ib = min(i0 + ni - 1, nx - 1);
  const int ja = max(j0, 1), jb = min(j0 + nj - 1, ny - 1);
  if (ia > ib || ja > jb) return false;
  int lo, hi;
  if (s.scheme == 1) {  // zebra_x: row j
    lo = ja;
    hi = jb;
  } else if (s.scheme == 4 || s.scheme == 5) {
    int ilo, ihi, jlo, jhi;
    mirror_range2(ia, ib, nx, ilo, ihi);
    mirror_range2(ja, jb, ny, jlo, jhi);
    lo = s.scheme == 4 ? max(ilo, jlo) : min(ilo, jlo);
    hi = s.scheme == 4 ? max(ihi, jhi) : min(ihi, jhi);
  } else {  // zebra_y, checkerboard: column i
    lo = ia;
    hi = ib;
  }
  return hi >= s.g0 && lo < s.g1;
}
__device__ __forceinline__ bool in_groups(const GroupSel2& s, int nx, int ny, int i, int j) {
  if (s.g0 <= 0) return true;
  const int gp = point_group(s.scheme, nx, ny, i, j);
  return gp >= s.g0 && gp < s.g1;
}

constexpr int NT = 32, NE = NT + 2, NLD = NE + 1;

constexpr int R3C = 15, R3D = 31, R3U = 33, R3LU = 34, R3LD = 32;

// MODE 0: box inside the grid in the natural buffer (rows = i), 1: inside the
// grid in the transposed buffer (rows = j), 2: anything else (rows = i, each
// point read through its owner: grid edges, mixed-ownership boxes)
template <int MODE>
__device__ __forceinline__ void restrict3_body(const GridArgs& g, int full, const FieldView& U,
                                               const FieldView& F, const FieldView& FC,
                                               const FieldView& UC, int zero_uc,
                                               const GroupSel2& csel, int own, int I0, int J0,
                                               double* su, double* sd) {
  constexpr bool T = MODE == 1, GEN = MODE == 2;
  const int nxc = g.nx / 2, nyc = g.ny / 2;
  const int ui0 = 2 * I0 - 2, uj0 = 2 * J0 - 2;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nA = T ? g.nx : g.ny, nM = T ? g.ny : g.nx;  // column / row axis extents
  const int a0 = T ? ui0 : uj0, m0 = T ? uj0 : ui0;       // tile origin (column, row)
  const double* colLo = T ? g.W : g.S;  // couplings along the column axis
  const double* colHi = T ? g.E : g.N;
  const double* rowLo = T ? g.S : g.W;  // along the row axis
  const double* rowHi = T ? g.N : g.E;
  // per-thread couplings: the defect column x = lane and rows y = w + 8q
  const int xc = a0 + 1 + lane;
  const bool colok = lane < R3D && (!GEN || xc < nA);
  const double cLo = colok ? __ldg(colLo + xc) : 0.0;
  const double cHi = colok ? __ldg(colHi + xc) : 0.0;
  double rLo[4], rHi[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int y = w + 8 * q, mr = m0 + 1 + y;
    const bool ok = (q < 3 || y < R3D) && (!GEN || mr < nM);
    rLo[q] = ok ? __ldg(rowLo + mr) : 0.0;
    rHi[q] = ok ? __ldg(rowHi + mr) : 0.0;
  }
  pdl_wait();
  double fv[4], uv[5], ux[5];
  if (!GEN) {
    // the whole 33 x 33 box lies in [0, n] and every defect point is interior
    const size_t ldr = (size_t)nA + 1, l8 = 8 * ldr;
    const double* fp = (T ? F.t : F.n) + (m0 + 1 + w) * ldr + a0 + 1 + lane;
    const double* up = (T ? U.t : U.n) + (m0 + w) * ldr + a0 + lane;
#pragma unroll
    for (int q = 0; q < 4; q++)
      fv[q] = ((q < 3 || w < 7) && lane < R3D) ? __ldg(fp + q * l8) : 0.0;
#pragma unroll
    for (int q = 0; q < 5; q++) {
      const bool ok = q < 4 || w == 0;
      uv[q] = ok ? __ldg(up + q * l8) : 0.0;
      ux[q] = (ok && lane == 0) ? __ldg(up + q * l8 + 32) : 0.0;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int y = w + 8 * q, mr = m0 + 1 + y, ac = a0 + 1 + lane;
      const bool in = y < R3D && lane < R3D && mr < nM && ac < nA;
      fv[q] = in ? ld_view(F, own, mr, ac) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 5; q++) {
      const int mr = m0 + w + 8 * q, ac = a0 + lane;
      const bool y_in = w + 8 * q < R3U && mr <= nM;
      uv[q] = (y_in && ac <= nA) ? ld_view(U, own, mr, ac) : 0.0;
      ux[q] = (y_in && lane == 0 && a0 + 32 <= nA) ? ld_view(U, own, mr, a0 + 32) : 0.0;
    }
  }
#pragma unroll
  for (int q = 0; q < 5; q++) {
    if (q < 4 || w == 0) {
      const int y = w + 8 * q;
      su[y * R3LU + lane] = uv[q];
      if (lane == 0) su[y * R3LU + 32] = ux[q];
    }
  }
  __syncthreads();
  // defects: (i, j) order of stencil.py:82-87 whatever the orientation
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int y = w + 8 * q;
    if ((q == 3 && y >= R3D) || lane >= R3D) continue;
    double dv = 0.0;
    if (!GEN || (m0 + 1 + y < nM && a0 + 1 + lane < nA)) {
      const int o = (y + 1) * R3LU + (lane + 1);
      const double c = su[o], uu = su[o - R3LU], dd = su[o + R3LU], ll = su[o - 1], rr = su[o + 1];
      // i neighbours: rows in N, columns in T
      const double im = T ? ll : uu, ip = T ? rr : dd, jm = T ? uu : ll, jp = T ? dd : rr;
      const double Wi = T ? cLo : rLo[q], Ei = T ? cHi : rHi[q];
      const double Sj = T ? rLo[q] : cLo, Nj = T ? rHi[q] : cHi;
      const double Cc = -__dadd_rn(__dadd_rn(__dadd_rn(Wi, Ei), Sj), Nj);
      double acc = __dmul_rn(Wi, im);
      acc = __dadd_rn(acc, __dmul_rn(Ei, ip));
      acc = __dadd_rn(acc, __dmul_rn(Sj, jm));
      acc = __dadd_rn(acc, __dmul_rn(Nj, jp));
      dv = __dadd_rn(-__dadd_rn(acc, __dmul_rn(Cc, c)), fv[q]);
    }
    sd[y * R3LD + lane] = dv;
  }
  __syncthreads();
  // coarse points, lanes along the coarse owner's contiguous axis
  const int cown = box_owner(FC, I0, J0, R3C, R3C);
  const int cpt = threadIdx.x;
  if (cpt >= R3C * R3C) return;
  const int p = cpt / R3C, qq = cpt - p * R3C;
  const int ca = cown == 1 ? qq : p, cb = cown == 1 ? p : qq;  // I offset, J offset
  const int I = I0 + ca, J = J0 + cb;
  if ((GEN && (I >= nxc || J >= nyc)) || !in_groups(csel, nxc, nyc, I, J)) return;
  const int a = 2 * ca + 1, b = 2 * cb + 1;  // fine (i, j) offsets in the defect tile
  const int o = T ? b * R3LD + a : a * R3LD + b;
  constexpr int di = T ? 1 : R3LD, dj = T ? R3LD : 1;
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

// One 15 x 15 coarse tile at (I0, J0): the CTA body of restrict3_kernel (and
// of the coarse-tail kernel's restriction op, tmg_sweep.cu)
__device__ __forceinline__ void restrict3_tile(const GridArgs& g, int full, const FieldView& U,
                                               const FieldView& F, const FieldView& FC,
                                               const FieldView& UC, int zero_uc,
                                               const GroupSel2& csel, int I0, int J0, double* su,
                                               double* sd) {
  const int nxc = g.nx / 2, nyc = g.ny / 2;
  if (!box_in_groups(csel, nxc, nyc, I0, J0, R3C, R3C)) {
    pdl_wait();
    return;
  }
  const int ui0 = 2 * I0 - 2, uj0 = 2 * J0 - 2;
  const int own = box_owner(U, ui0, uj0, R3U, R3U);
  const bool inner = own >= 0 && ui0 + R3U - 1 <= g.nx && uj0 + R3U - 1 <= g.ny;
  if (inner && own == 0)
    restrict3_body<0>(g, full, U, F, FC, UC, zero_uc, csel, own, I0, J0, su, sd);
  else if (inner)
    restrict3_body<1>(g, full, U, F, FC, UC, zero_uc, csel, own, I0, J0, su, sd);
  else
    restrict3_body<2>(g, full, U, F, FC, UC, zero_uc, csel, own, I0, J0, su, sd);
}

constexpr int PC_E = NT / 2 + 1, PC_LD = PC_E + 1;

// One 32 x 32 fine tile at (i0, j0) of the fused prolongation + correction
// skip_red: the caller smooths next with the square tweed scheme, whose red
// stage overwrites every red point (shell index max(i', j') odd,
// layout.py:22-23, 75-84) without reading its old value — block Gauss-Seidel
// solves all unknowns of a block from their out-of-block neighbours
// (_ckernels.pyx:34-39) and same-colour blocks never touch —
// so only the black points need the correction: half the fine traffic.
__device__ __forceinline__ void prolong2_tile(int nx, int ny, const FieldView& C,
                                              const FieldView& U, const GroupSel2& fsel, int i0,
                                              int j0, double* sc, int skip_red = 0) {
  if (!box_in_groups(fsel, nx, ny, i0, j0, NT, NT)) {  // outside a rank's groups
    pdl_trigger();
    pdl_wait();
    return;
  }
  const int own = box_owner(U, i0, j0, NT, NT);
  const int Ic0 = i0 >> 1, Jc0 = j0 >> 1;
  pdl_trigger();
  const int cown = box_owner(C, Ic0, Jc0, PC_E, PC_E);
  pdl_wait();
#ifndef TMG_PROLONG_FAST
#define TMG_PROLONG_FAST 1  // 0: every tile takes the generic per-point path
#endif
  if (TMG_PROLONG_FAST && fsel.g0 <= 0 && own >= 0 && cown >= 0 && i0 + NT <= nx &&
      j0 + NT <= ny && (!skip_red || U.mode == LM_TWEED)) {
    // Interior tile owned by one buffer, coarse box by one buffer (nearly every
    // tile of a large level): one base pointer and a row stride, and — the tile
    // origin being odd — a thread's four points (rows w, w + 8, ...) share
    // their parity class and walk the coarse tile with a fixed step.  Same
    // expressions as the generic path below (transfer.py:51-53, bit-identical).
    const bool T = own == 1;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t ldr = T ? nx + 1 : ny + 1, l8 = 8 * ldr;
    double* up = (T ? U.t : U.n) + ((T ? j0 : i0) + w) * ldr + (T ? i0 : j0) + lane;
    // the rows of a single-owner tile of the tweed layout are shell rows (T owns
    // i' < j', N the rest): row m of the owner buffer is shell min(m, n - m),
    // and a thread's rows w, w + 8, ... share its parity (n is even)
    const int mrow = (T ? j0 : i0) + w;
    const bool skip = skip_red && (min(mrow, (T ? ny : nx) - mrow) & 1);
    double uv[4] = {0.0, 0.0, 0.0, 0.0};
    if (!skip) {
#pragma unroll
      for (int q = 0; q < 4; q++) uv[q] = up[q * l8];
    }
    load_box<PC_E, PC_LD>(C, cown, Ic0, Jc0, sc);
    __syncthreads();
    if (skip) return;
    const int cI = cown == 1 ? 1 : PC_LD, cJ = cown == 1 ? PC_LD : 1;
    const int di = T ? lane : w, dj = T ? w : lane;  // i - i0, j - j0 of the first point
    const bool i_even = di & 1, j_even = dj & 1;      // i0, j0 are odd
    int o = ((1 + di) >> 1) * cI + ((1 + dj) >> 1) * cJ;
    const int step = 4 * (T ? cJ : cI);  // eight fine rows = four coarse rows
#pragma unroll
    for (int q = 0; q < 4; q++, o += step) {
      double pv;
      if (i_even && j_even) pv = sc[o];
      else if (i_even) pv = __dmul_rn(0.5, __dadd_rn(sc[o], sc[o + cJ]));
      else if (j_even) pv = __dmul_rn(0.5, __dadd_rn(sc[o], sc[o + cI]));
      else
        pv = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(sc[o], sc[o + cI]), sc[o + cJ]),
                                       sc[o + cI + cJ]));
      up[q * l8] = __dadd_rn(uv[q], pv);
    }
    return;
  }
  double uv[4];
  int pi[4], pj[4];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int t = threadIdx.x + k * 256, y = t >> 5, x = t & 31;
    pi[k] = own == 1 ? i0 + x : i0 + y;
    pj[k] = own == 1 ? j0 + y : j0 + x;
    uv[k] = (pi[k] < nx && pj[k] < ny) ? ld_view(U, own, pi[k], pj[k]) : 0.0;
  }
  load_box<PC_E, PC_LD>(C, cown, Ic0, Jc0, sc);
  __syncthreads();
  const int cI = cown == 1 ? 1 : PC_LD, cJ = cown == 1 ? PC_LD : 1;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int i = pi[k], j = pj[k];
    if (i >= nx || j >= ny || !in_groups(fsel, nx, ny, i, j)) continue;
    if (skip_red && (point_group(4, nx, ny, i, j) & 1)) continue;
    const int I = i >> 1, J = j >> 1;
    const int o = (I - Ic0) * cI + (J - Jc0) * cJ;
    double pv;
    if (!(i & 1) && !(j & 1)) pv = sc[o];
    else if (!(i & 1)) pv = __dmul_rn(0.5, __dadd_rn(sc[o], sc[o + cJ]));
    else if (!(j & 1)) pv = __dmul_rn(0.5, __dadd_rn(sc[o], sc[o + cI]));
    else
      pv = __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(sc[o], sc[o + cI]), sc[o + cJ]),
                                     sc[o + cI + cJ]));
    const double r = __dadd_rn(uv[k], pv);
    if (own == 1) U.t[U.off_t(i, j)] = r;
    else if (own == 0) U.n[U.off_n(i, j)] = r;
    else *U.at(i, j) = r;
  }
}

// Coarsest level (mgcycle.py:93-95): rhs = f - (boundary couplings) over the
// interior in j-outer order, then u = Ainv rhs one warp per row
__device__ __forceinline__ void dense_rhs(const GridArgs& g, const FieldView& U,
                                          const FieldView& F, double* rhs, int t0, int nt) {
  const int mi = g.nx - 1, n = mi * (g.ny - 1);
  for (int k = t0; k < n; k += nt) {
    const int i = k % mi + 1, j = k / mi + 1;
    const double bw = i == 1 ? *U.at(i - 1, j) : 0.0, be = i == g.nx - 1 ? *U.at(i + 1, j) : 0.0;
    const double bs = j == 1 ? *U.at(i, j - 1) : 0.0, bn = j == g.ny - 1 ? *U.at(i, j + 1) : 0.0;
    double acc = __dmul_rn(g.W[i], bw);
    acc = __dadd_rn(acc, __dmul_rn(g.E[i], be));
    acc = __dadd_rn(acc, __dmul_rn(g.S[j], bs));
    acc = __dadd_rn(acc, __dmul_rn(g.N[j], bn));
    rhs[k] = __dadd_rn(*F.at(i, j), -acc);
  }
}

__device__ __forceinline__ void dense_apply(const GridArgs& g, const double* Ainv,
                                            const double* rhs, const FieldView& U, int warp,
                                            int lane) {
  const int mi = g.nx - 1, n = mi * (g.ny - 1);
  if (warp >= n) return;
  if (n == 1) {
    if (lane == 0) *U.at(1, 1) = rhs[0] / Ainv[0];
    return;
  }
  double acc = 0.0;
  for (int c = lane; c < n; c += 32) acc += Ainv[(size_t)warp * n + c] * rhs[c];
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) *U.at(warp % mi + 1, warp / mi + 1) = acc;
}

}  // namespace
}  // namespace tmg
