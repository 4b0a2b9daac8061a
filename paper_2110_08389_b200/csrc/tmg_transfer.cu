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

struct GroupSel2 {
  int scheme, g0, g1;
};

// ---- residual max-norm: 32 x 32 points per CTA, 4 per thread ----------------
constexpr int NT = 32, NE = NT + 2, NLD = NE + 1;

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

__global__ void __launch_bounds__(256) restrict2_kernel(GridArgs g, int full, FieldView U,
                                                        FieldView F, FieldView FC) {
  extern __shared__ double rsm[];
  double* su = rsm;
  double* sd = rsm + RU * RLU;
  const int nxc = g.nx / 2, nyc = g.ny / 2;
  const int I0 = 1 + blockIdx.y * RC, J0 = 1 + blockIdx.x * RC;
  const int ui0 = 2 * I0 - 2, uj0 = 2 * J0 - 2;
  pdl_trigger();
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
  if (I < nxc && J < nyc) {
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
  }
  }
}

// ---- fused prolongation + correction: 32 x 32 fine points per CTA --------
constexpr int PC_E = NT / 2 + 1, PC_LD = PC_E + 1;

__global__ void __launch_bounds__(256) prolong2_kernel(int nx, int ny, FieldView C, FieldView U) {
  __shared__ double sc[PC_E * PC_LD];
  const int i0 = 1 + blockIdx.y * NT, j0 = 1 + blockIdx.x * NT;
  const int own = box_owner(U, i0, j0, NT, NT);
  const int Ic0 = i0 >> 1, Jc0 = j0 >> 1;
  pdl_trigger();
  const int cown = box_owner(C, Ic0, Jc0, PC_E, PC_E);
  pdl_wait();
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
    if (i >= nx || j >= ny) continue;
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

}  // namespace

cudaError_t launch_norm2(const GridArgs& g, const FieldView& U, const FieldView& F,
                         unsigned long long* dmax, cudaStream_t s, int scheme, int g0, int g1) {
  if (g.nx < 2 || g.ny < 2) return cudaSuccess;
  dim3 grid((g.ny - 1 + NT - 1) / NT, (g.nx - 1 + NT - 1) / NT);
  TMG_COUNT(1);
  return launch_pdl(norm2_kernel, grid, dim3(256), 0, s, g, U, F, dmax,
                    GroupSel2{scheme, g0, g1});
}

cudaError_t launch_restrict2(const GridArgs& g, int full, const FieldView& U, const FieldView& F,
                             const FieldView& FC, cudaStream_t s) {
  const int nxc = g.nx / 2, nyc = g.ny / 2;
  if (nxc < 2 || nyc < 2) return cudaSuccess;
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
  return launch_pdl(restrict2_kernel, grid, dim3(256), kRestrictSmem, s, g, full, U, F, FC);
}

cudaError_t launch_prolong2(int nx, int ny, const FieldView& C, const FieldView& U,
                            cudaStream_t s) {
  if (nx < 2 || ny < 2) return cudaSuccess;
  dim3 grid((ny - 1 + NT - 1) / NT, (nx - 1 + NT - 1) / NT);
  TMG_COUNT(1);
  return launch_pdl(prolong2_kernel, grid, dim3(256), 0, s, nx, ny, C, U);
}

}  // namespace tmg
