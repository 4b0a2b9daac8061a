// 3D tweed V-cycle on cubes (BASELINE config 4).
//
// The reference is 2D only; this path extends its semantics to a third axis
// (stencil.py:43-96 with coefficients B, T along k; transfer.py:21-56 as
// tensor products; the m-legged Thomas of tridiag.py:84-125 for blocks of up
// to 6 legs) on the survey's cube layout: a point lies on the line along the
// axis of its unique smallest mirrored coordinate, from the wall to the first
// tie point (the branch); colour = parity(s1 + s3) of the branch's sorted
// mirrored coordinates, red = even.  Its checker is the CPU restatement in
// oracle/tweed3d_oracle.c.
//
// Fields are C-order (n+1)^3 with k fastest.  A colour stage runs the block
// kernel of tmg3dw.cu on hub blocks (a branch with 2, 3 or 6 legs from the
// walls): per leg a coalesced gather, chunked elimination and PCR with the
// branch and the wall as end columns, then the branch row, then finalise;
// blocks are enumerated with k fastest, so neighbouring blocks are
// neighbouring lines.  This file holds the block enumeration, the 7-point
// residual, the transfers, the V-cycle (one CUDA graph) and the C ABI.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <map>
#include <tuple>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tweedmg_b200.h"
#include "tmg3d.h"
#include "tmg_kernels.h"

using namespace tmg;
using tmg3::Coef3;
using tmg3::idx3;
using tmg3::mirror;

namespace {

using Block3 = tmg3::HubB;  // branch, legs (s1 - 1 points each), colour

// sharding group of an interior point: 3D tweed blocks lie in
// one max(i', j', k') shell, 3D wireframe blocks in one min(i', j', k') shell
__device__ __forceinline__ int cube_group(int scheme, int n, int i, int j, int k) {
  const int a = (int)mirror(i, n), b = (int)mirror(j, n), c = (int)mirror(k, n);
  return scheme == 1 ? min(a, min(b, c)) : max(a, max(b, c));
}

// d = f - L u (interior), 0 on the boundary; or the max |f - L u| over the
// points of groups [g0, g1) into dmax
__global__ void __launch_bounds__(256) defect3_kernel(int n, Coef3 c, const double* __restrict__ u,
                                                      const double* __restrict__ f,
                                                      double* __restrict__ d,
                                                      unsigned long long* dmax, int gscheme = 0,
                                                      int g0 = 0, int g1 = 1 << 30) {
  pdl_trigger();
  pdl_wait();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y, i = blockIdx.z;
  const size_t o = idx3(n, i, j, k < n ? k : n);
  double v = 0.0;
  if (i > 0 && j > 0 && k > 0 && i < n && j < n && k < n) {
    const double cc = -(__ldg(c.W + i) + __ldg(c.E + i) + __ldg(c.S + j) + __ldg(c.N + j) +
                        __ldg(c.B + k) + __ldg(c.T + k));
    double acc = __dmul_rn(__ldg(c.W + i), u[idx3(n, i - 1, j, k)]);
    acc = __dadd_rn(acc, __dmul_rn(__ldg(c.E + i), u[idx3(n, i + 1, j, k)]));
    acc = __dadd_rn(acc, __dmul_rn(__ldg(c.S + j), u[idx3(n, i, j - 1, k)]));
    acc = __dadd_rn(acc, __dmul_rn(__ldg(c.N + j), u[idx3(n, i, j + 1, k)]));
    acc = __dadd_rn(acc, __dmul_rn(__ldg(c.B + k), u[o - 1]));
    acc = __dadd_rn(acc, __dmul_rn(__ldg(c.T + k), u[o + 1]));
    acc = __dadd_rn(acc, __dmul_rn(cc, u[o]));
    v = __dadd_rn(f[o], -acc);
  }
  if (d && k <= n) d[o] = v;
  if (dmax) {  // every lane takes part (lanes past the row carry v = 0)
    if (g0 > 0 || g1 < (1 << 30)) {
      const int grp = v != 0.0 ? cube_group(gscheme, n, i, j, k) : g0;
      if (grp < g0 || grp >= g1) v = 0.0;
    }
    unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(v));
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, bits, s);
      bits = o2 > bits ? o2 : bits;
    }
    // one atomic per CTA (per-warp atomics on one address serialise in L2)
    __shared__ unsigned long long wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = bits;
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int w = 1; w < 8; w++) bits = wm[w] > bits ? wm[w] : bits;
      if (bits) atomicMax(dmax, bits);
    }
  }
}

// Fused residual + full weighting (mgcycle.py:98-99 in 3D), marching along
// i: a CTA owns a coarse (J, K) tile of 8 x 32 points and a run of coarse
// planes; per fine plane it stages the u plane in a three-plane shared ring
// buffer (rows along k, coalesced), computes the fine defects of its tile
// (defect3_kernel's arithmetic) into shared memory and folds them into the
// coarse points in the oracle's order (orc3_restrict: a, b, e nested), while
// u and f are read once (16 B per fine point, no defect field in HBM).
constexpr int kRTJ = 8, kRTK = 31;                          // coarse tile (63 fine columns: 4 x 63 threads)
constexpr int kRDJ = 2 * kRTJ + 1, kRDK = 2 * kRTK + 1;     // fine defects
constexpr int kRUJ = kRDJ + 2, kRUK = kRDK + 2;             // u with halo

// 8-byte asynchronous global -> shared copy; src_bytes = 0 zero-fills
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

constexpr int kRU = kRUJ * kRUK, kRD = kRDJ * kRDK;
constexpr size_t kRestrictSmem3 = (4 * kRU + 3 * kRD + 2 * kRDJ + 2 * kRDK) * sizeof(double);

// Coarse planes [I0, I0 + ti) per CTA.  u planes stream through a 4-slot
// shared ring and f planes through 2 slots by cp.async, two fine planes
// ahead of the defect computation, so HBM latency overlaps the stencil.
__global__ void __launch_bounds__(256, 3) defect_restrict3_kernel(int nf, Coef3 c,
                                                                  const double* __restrict__ u,
                                                                  const double* __restrict__ f,
                                                                  double* __restrict__ out,
                                                                  int ti) {
  extern __shared__ double rsm[];
  double* su = rsm;              // 4 x kRU
  double* sf = su + 4 * kRU;     // 2 x kRD
  double* sd = sf + 2 * kRD;     // kRD defects
  double* cS = sd + kRD;         // S, N along the tile's rows; B, T along its columns
  double* cN = cS + kRDJ;
  double* cB = cN + kRDJ;
  double* cT = cB + kRDK;
  pdl_trigger();
  const int nc = nf / 2;
  const int J0 = 1 + blockIdx.y * kRTJ, K0 = 1 + blockIdx.x * kRTK;
  const int I0 = 1 + blockIdx.z * ti, I1 = min(I0 + ti, nc);
  const int jd0 = 2 * J0 - 1, kd0 = 2 * K0 - 1;  // fine origin of the defect tile
  const int tid = threadIdx.x;
  const size_t n1 = (size_t)nf + 1;
  for (int t = tid; t < kRDJ; t += 256) {
    const int j = min(jd0 + t, nf);
    cS[t] = __ldg(c.S + j);
    cN[t] = __ldg(c.N + j);
  }
  for (int t = tid; t < kRDK; t += 256) {
    const int k = min(kd0 + t, nf);
    cB[t] = __ldg(c.B + k);
    cT[t] = __ldg(c.T + k);
  }
  // per-thread element offsets within a plane (fixed for every plane): u
  // tile elements t = tid + 256 m, f / defect elements likewise; -1 = outside
  constexpr int PU = (kRU + 255) / 256, PD = (kRD + 255) / 256;
  int uo[PU], fo[PD];
#pragma unroll
  for (int m = 0; m < PU; m++) {
    const int t = tid + 256 * m, r = t / kRUK, q = t - r * kRUK;
    const int j = jd0 - 1 + r, k = kd0 - 1 + q;
    uo[m] = (t < kRU && j <= nf && k <= nf) ? j * (nf + 1) + k : -1;
  }
#pragma unroll
  for (int m = 0; m < PD; m++) {
    const int t = tid + 256 * m, r = t / kRDK, q = t - r * kRDK;
    const int j = jd0 + r, k = kd0 + q;
    fo[m] = (t < kRD && j < nf && k < nf) ? j * (nf + 1) + k : -1;
  }
  // defect mapping: a thread per fine column q and a run of rows (a sliding
  // window down the column: one new u load per row)
  static_assert(4 * kRDK <= 256 && kRDJ == 17, "defect mapping");
  const int dq = tid % kRDK, dg = tid / kRDK;
  const int dr0 = dg == 0 ? 0 : 1 + 4 * dg, dr1 = dg == 0 ? 5 : 5 + 4 * dg;  // rows [dr0, dr1)
  const bool dlive = dg < 4 && kd0 + dq < nf;
  const size_t plane = n1 * n1;
  auto issue_u = [&](int i) {  // plane i (0 .. nf) into slot i % 4
    double* dst = su + (i & 3) * kRU;
    const double* base = u + (size_t)i * plane;
    const bool pin = i <= nf;
#pragma unroll
    for (int m = 0; m < PU; m++) {
      const int t = tid + 256 * m;
      if (t < kRU) {
        const bool ok = pin && uo[m] >= 0;
        cp_async8(dst + t, ok ? base + uo[m] : u, ok);
      }
    }
  };
  auto issue_f = [&](int i) {  // plane i into slot i % 2
    double* dst = sf + (i & 1) * kRD;
    const double* base = f + (size_t)i * plane;
    const bool pin = i < nf;
#pragma unroll
    for (int m = 0; m < PD; m++) {
      const int t = tid + 256 * m;
      if (t < kRD) {
        const bool ok = pin && fo[m] >= 0;
        cp_async8(dst + t, ok ? base + fo[m] : f, ok);
      }
    }
  };
  pdl_wait();
  issue_u(2 * I0 - 2);
  issue_u(2 * I0 - 1);
  issue_u(2 * I0);
  issue_f(2 * I0 - 1);
  cp_async_commit();
  issue_u(2 * I0 + 1);
  issue_f(2 * I0);
  cp_async_commit();
  const int tj = tid / kRTK, tk = tid % kRTK, J = J0 + tj, K = K0 + tk;
  const bool own = tid < kRTJ * kRTK && J < nc && K < nc;
  double acc = 0.0;
  for (int i = 2 * I0 - 1; i <= 2 * I1 - 1; i++) {
    cp_async_wait1();  // u planes up to i + 1 and f plane i have landed
    __syncthreads();
    const double* um = su + ((i - 1) & 3) * kRU;
    const double* uc = su + (i & 3) * kRU;
    const double* up = su + ((i + 1) & 3) * kRU;
    const double* fc = sf + (i & 1) * kRD;
    const double Wi = __ldg(c.W + i), Ei = __ldg(c.E + i);
    if (dlive) {
      const double Bk = cB[dq], Tk = cT[dq];
      int o = (dr0 + 1) * kRUK + (dq + 1);
      double up_c = uc[o - kRUK], cur = uc[o];
#pragma unroll
      for (int r = 0; r < 5; r++) {
        const int rr = dr0 + r;
        if (rr >= dr1) break;
        const double nxt = uc[o + kRUK];
        double v = 0.0;
        if (jd0 + rr < nf) {
          const double Sj = cS[rr], Nj = cN[rr];
          const double cc = -(Wi + Ei + Sj + Nj + Bk + Tk);
          double a = __dmul_rn(Wi, um[o]);
          a = __dadd_rn(a, __dmul_rn(Ei, up[o]));
          a = __dadd_rn(a, __dmul_rn(Sj, up_c));
          a = __dadd_rn(a, __dmul_rn(Nj, nxt));
          a = __dadd_rn(a, __dmul_rn(Bk, uc[o - 1]));
          a = __dadd_rn(a, __dmul_rn(Tk, uc[o + 1]));
          a = __dadd_rn(a, __dmul_rn(cc, cur));
          v = __dadd_rn(fc[rr * kRDK + dq], -a);
        }
        sd[rr * kRDK + dq] = v;
        up_c = cur;
        cur = nxt;
        o += kRUK;
      }
    } else if (dg < 4) {
      for (int rr = dr0; rr < dr1; rr++) sd[rr * kRDK + dq] = 0.0;
    }
    __syncthreads();  // defects complete; u plane i-1 and f plane i are free
    if (i + 3 <= 2 * I1) issue_u(i + 3);
    if (i + 2 <= 2 * I1 - 1) issue_f(i + 2);
    cp_async_commit();  // (possibly empty) keeps the group count per plane fixed
    // plane i is a = 2 of coarse plane (i - 1) / 2 and a = 0 of (i + 1) / 2
    // (odd i), or a = 1 of i / 2 (even i)
    const int a_lo = (i & 1) ? 2 : 1, I_lo = (i & 1) ? (i - 1) / 2 : i / 2;
    for (int pass = 0; pass < ((i & 1) ? 2 : 1); pass++) {
      const int a = pass == 0 ? a_lo : 0, I = pass == 0 ? I_lo : (i + 1) / 2;
      if (I < I0 || I >= I1) continue;
      if (a == 0) acc = 0.0;
      if (own) {
        const double wa = a == 1 ? 0.5 : 0.25;
#pragma unroll
        for (int b = 0; b < 3; b++)
#pragma unroll
          for (int e = 0; e < 3; e++)
            acc += wa * (b == 1 ? 0.5 : 0.25) * (e == 1 ? 0.5 : 0.25) *
                   sd[(2 * tj + b) * kRDK + 2 * tk + e];
      }
      if (a == 2 && own) out[((size_t)I * (nc + 1) + J) * (nc + 1) + K] = acc;
    }
  }
}

// u += trilinear P uc on the fine interior: a thread per fine i, coarse row
// Jc and coarse column K, writing the 2 x 2 fine points j = 2Jc-1, 2Jc and
// k = 2K-1, 2K from the 2 x 2 (x 2 in i) coarse values they share; sums in
// orc3_prolong_add's order (a, b, e nested), lanes along K
__global__ void __launch_bounds__(256) prolong3v2_kernel(int nc, const double* __restrict__ uc,
                                                         double* __restrict__ u) {
  pdl_trigger();
  pdl_wait();
  const int nf = 2 * nc;
  const int K = 1 + blockIdx.x * blockDim.x + threadIdx.x;
  const int Jc = 1 + blockIdx.y, i = 1 + blockIdx.z;
  if (K > nc) return;
  const int I = i / 2, oi = i & 1;
  const size_t c1 = (size_t)nc + 1;
  double oo = 0.0, oe = 0.0, eo = 0.0, ee = 0.0;  // (j odd / even, k odd / even)
  for (int a = 0; a <= oi; a++) {
    const size_t r0 = ((size_t)(I + a) * c1 + (Jc - 1)) * c1, r1 = r0 + c1;
    const double v00 = __ldg(uc + r0 + K - 1), v01 = __ldg(uc + r0 + K);
    const double v10 = __ldg(uc + r1 + K - 1), v11 = __ldg(uc + r1 + K);
    oo += v00;
    oo += v01;
    oo += v10;
    oo += v11;
    oe += v01;
    oe += v11;
    eo += v10;
    eo += v11;
    ee += v11;
  }
  const double w1 = 1.0 / (double)(1 + oi);
  const size_t n1 = (size_t)nf + 1;
  const size_t ro = ((size_t)i * n1 + (2 * Jc - 1)) * n1, re = ro + n1;
  u[ro + 2 * K - 1] += oo * (w1 / 4.0);
  if (2 * K < nf) u[ro + 2 * K] += oe * (w1 / 2.0);
  if (2 * Jc < nf) {
    u[re + 2 * K - 1] += eo * (w1 / 2.0);
    if (2 * K < nf) u[re + 2 * K] += ee * w1;
  }
}

// ---- hybrid layout of the 3D wireframe V-cycle ------------
// View V (0: i-contiguous [j][k][i], 1: j-contiguous [i][k][j]) owns the
// points whose strictly largest mirrored coordinate is on axis V; ties and
// the boundary live in every view; the natural array is view 2.  A tile of
// 32 (axis V) x 32 (k) points at a fixed third index moves through shared
// memory so that both sides are read and written along a contiguous axis;
// CTAs walk (k tile, fixed index) fastest and the axis-V tile slowest, so a
// wave touches 32 planes of the natural array (TLB reach, DRAM rows).
__device__ __forceinline__ int owner_h(int n, int i, int j, int k, bool smallest) {
  if (i <= 0 || j <= 0 || k <= 0 || i >= n || j >= n || k >= n) return -1;
  int a = (int)mirror(i, n), b = (int)mirror(j, n), c = (int)mirror(k, n);
  if (smallest) { a = -a; b = -b; c = -c; }
  return (a > b && a > c) ? 0 : ((b > a && b > c) ? 1 : ((c > a && c > b) ? 2 : -1));
}

// TO_VIEW: natural -> view V for the points `mask` selects (1, u: every
// point whose mirrored axis-V coordinate is not below the other two -- the
// owned points, the ties and boundary points next to them, all a view-V edge
// reads; 2, f: the owned points); else view V -> natural for the owned
// points.  Tiles without such points are skipped (a view covers ~1/3 of the
// cube).
template <int V, bool TO_VIEW, bool SMALL>
__global__ void __launch_bounds__(256) hybrid_kernel(int n, double* __restrict__ nat,
                                                     double* __restrict__ view, int mask) {
  constexpr int NF = 4;  // fixed-index planes per CTA: their tile loads are in flight together
  __shared__ double t[NF][32][33];
  pdl_trigger();
  const int kt = blockIdx.x * 32, at = blockIdx.z * 32;
  const size_t n1 = (size_t)n + 1;
  const int lane = threadIdx.x & 31, row = threadIdx.x >> 5;
  // tile test on the mirrored coordinates (negated for SMALL, the 3D tweed):
  // the tile's best axis-V value against the fixed index's and the k range's
  const int a1 = min(at + 31, n), k1 = min(kt + 31, n);
  const int sg = SMALL ? -1 : 1;
  const int ma = SMALL ? -min((int)mirror(at, n), (int)mirror(a1, n))
                       : ((at <= n / 2 && n / 2 <= a1) ? n / 2
                                                        : max((int)mirror(at, n), (int)mirror(a1, n)));
  const int mk = SMALL ? -((kt <= n / 2 && n / 2 <= k1) ? n / 2
                                                        : max((int)mirror(kt, n), (int)mirror(k1, n)))
                       : min((int)mirror(kt, n), (int)mirror(k1, n));
  const bool strict = !(TO_VIEW && mask == 1);
  bool any = false;
  bool use[NF];
#pragma unroll
  for (int q = 0; q < NF; q++) {
    const int fx = blockIdx.y * NF + q;
    const int mf = sg * (int)mirror(min(fx, n), n);
    use[q] = fx <= n && (strict ? (ma > mf && ma > mk) : (ma >= mf && ma >= mk));
    any |= use[q];
  }
  if (!any) return;
  pdl_wait();
  auto nat_off = [&](int fx, int a, int k) {
    return V == 0 ? ((size_t)a * n1 + fx) * n1 + k : ((size_t)fx * n1 + a) * n1 + k;
  };
  auto view_off = [&](int fx, int a, int k) { return ((size_t)fx * n1 + k) * n1 + a; };
  auto sel = [&](int fx, int a, int k) {
    const int i = V == 0 ? a : fx, j = V == 0 ? fx : a;
    if (!strict) {
      const int mv = sg * (int)mirror(a, n), mo = max(sg * (int)mirror(fx, n), sg * (int)mirror(k, n));
      return mv >= mo;
    }
    return owner_h(n, i, j, k, SMALL) == V;
  };
  double r[NF][4];
#pragma unroll
  for (int q = 0; q < NF; q++) {
    const int fx = blockIdx.y * NF + q;
#pragma unroll
    for (int m = 0; m < 4; m++) {
      const int rr = row + 8 * m;
      if (TO_VIEW) {
        const int a = at + rr, k = kt + lane;
        r[q][m] = (use[q] && a <= n && k <= n) ? nat[nat_off(fx, a, k)] : 0.0;
      } else {
        const int k = kt + rr, a = at + lane;
        r[q][m] = (use[q] && a <= n && k <= n) ? view[view_off(fx, a, k)] : 0.0;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NF; q++)
#pragma unroll
    for (int m = 0; m < 4; m++) {
      const int rr = row + 8 * m;
      if (TO_VIEW) t[q][rr][lane] = r[q][m];
      else t[q][lane][rr] = r[q][m];
    }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NF; q++) {
    if (!use[q]) continue;
    const int fx = blockIdx.y * NF + q;
#pragma unroll
    for (int m = 0; m < 4; m++) {
      const int rr = row + 8 * m;
      if (TO_VIEW) {
        const int k = kt + rr, a = at + lane;
        if (a <= n && k <= n && sel(fx, a, k)) view[view_off(fx, a, k)] = t[q][lane][rr];
      } else {
        const int a = at + rr, k = kt + lane;
        if (a <= n && k <= n && sel(fx, a, k)) nat[nat_off(fx, a, k)] = t[q][rr][lane];
      }
    }
  }
}

__global__ void coarse3_kernel(Coef3 c, double* u, const double* f) {
  pdl_trigger();
  pdl_wait();
  const int n = 2;
  const double cc = -(c.W[1] + c.E[1] + c.S[1] + c.N[1] + c.B[1] + c.T[1]);
  const double r = f[idx3(n, 1, 1, 1)] - c.W[1] * u[idx3(n, 0, 1, 1)] - c.E[1] * u[idx3(n, 2, 1, 1)] -
                   c.S[1] * u[idx3(n, 1, 0, 1)] - c.N[1] * u[idx3(n, 1, 2, 1)] -
                   c.B[1] * u[idx3(n, 1, 1, 0)] - c.T[1] * u[idx3(n, 1, 1, 2)];
  u[idx3(n, 1, 1, 1)] = r / cc;
}

__global__ void __launch_bounds__(256) zero3_kernel(double* __restrict__ p, size_t m) {
  pdl_trigger();
  pdl_wait();
  for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (size_t)gridDim.x * blockDim.x)
    p[q] = 0.0;
}

__global__ void cube_gather_kernel(const double* __restrict__ fld, const long long* __restrict__ off,
                                   long m, double* __restrict__ out) {
  const long q = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < m) out[q] = fld[off[q]];
}

__global__ void cube_scatter_kernel(double* __restrict__ fld, const long long* __restrict__ off,
                                    long m, const double* __restrict__ in) {
  const long q = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < m) fld[off[q]] = in[q];
}

std::string g_err3;
int fail3(int code, const std::string& m) {
  g_err3 = m;
  return code;
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

struct tmg_cube {
  int scheme = 0;                     // 0 tweed, 1 wireframe
  std::vector<tmg3::WLevel> wl;       // wireframe blocks per level
  std::vector<tmg3::HubLevel> hl;     // 3D tweed blocks per level (the block kernel)
  std::map<std::tuple<int, int, int>, tmg3::WLevel> wparts;  // (level, g0, g1): a rank's blocks
  std::vector<int> n;                 // per level
  std::vector<double*> coef;          // per level: W E S N B T (6 (n+1))
  std::vector<int> nblocks[2];        // per level: black, red 3D tweed block counts
  std::vector<double*> U, F;          // per level work fields (level 0: session)
  // 3D wireframe hybrid views (i- and j-contiguous copies) of the levels with
  // n >= hyb_min; null elsewhere
  std::vector<double*> UI, UJ, FI, FJ;
  int hyb_min = 256;                  // levels with n >= hyb_min get the views
  bool nat_stale = false;             // level-0 natural u behind its views (lazy cycles)
  int* err = nullptr;
  unsigned long long* dmax = nullptr;
  int* h_err = nullptr;
  unsigned long long* h_dmax = nullptr;
  cudaGraphExec_t graph = nullptr;
  int gnu1 = -1, gnu2 = -1;
  int graph_kernels = 0;
  // device-driven solve loop (tmg_cube_solve_loop): state and while-node graph
  tmg::SolveDev* d_solve = nullptr;
  int solve_cap = 0;
  cudaGraphExec_t solve_graph = nullptr;
  int snu1 = -1, snu2 = -1, solve_kernels = 0;
};

namespace {

int cuda3(cudaError_t e, const char* w) {
  return e == cudaSuccess ? TMG_OK : fail3(TMG_CUDA, std::string(w) + ": " + cudaGetErrorString(e));
}
#define T3(x)                                   \
  do {                                          \
    int _s = cuda3((x), #x);                    \
    if (_s) return _s;                          \
  } while (0)

void build_blocks(int n, std::vector<Block3> out[2]) {
  const int c = n / 2;
  for (int i = 1; i < n; i++)
    for (int j = 1; j < n; j++)
      for (int k = 1; k < n; k++) {
        const long m[3] = {mirror(i, n), mirror(j, n), mirror(k, n)};
        long s1 = m[0], s2 = m[1], s3 = m[2], t;
        if (s1 > s2) { t = s1; s1 = s2; s2 = t; }
        if (s2 > s3) { t = s2; s2 = s3; s3 = t; }
        if (s1 > s2) { t = s1; s1 = s2; s2 = t; }
        if (s1 != s2) continue;
        Block3 B;
        std::memset(&B, 0, sizeof(B));
        B.bi = i; B.bj = j; B.bk = k;
        B.red = ((s1 + s3) % 2) == 0;
        B.len = (int16_t)(s1 >= 2 ? s1 - 1 : 0);
        const int x[3] = {i, j, k};
        if (s1 >= 2)
          for (int a = 0; a < 3; a++) {
            if (m[a] != s1) continue;
            if (x[a] <= c) B.leg[B.nleg++] = (uint8_t)a;        // tip at 1
            if (x[a] >= c) B.leg[B.nleg++] = (uint8_t)(a | 4);  // tip at n-1
          }
        out[B.red].push_back(B);
      }
}

Coef3 coefs(const tmg_cube* h, int l) {
  const int n1 = h->n[l] + 1;
  double* p = h->coef[l];
  return Coef3{p, p + n1, p + 2 * n1, p + 3 * n1, p + 4 * n1, p + 5 * n1};
}

bool hyb(const tmg_cube* h, int l) { return l < (int)h->UI.size() && h->UI[l]; }

// hybrid <-> natural for level l: which = 0 u, 1 f
int convert3(tmg_cube* h, int l, int which, bool to_view, cudaStream_t s) {
  const int n = h->n[l];
  const dim3 grid((n + 32) / 32, (n + 4) / 4, (n + 32) / 32);  // 4 fixed-index planes per CTA
  double* nat = which ? h->F[l] : h->U[l];
  double* v0 = which ? h->FI[l] : h->UI[l];
  double* v1 = which ? h->FJ[l] : h->UJ[l];
  const int mask = which ? 2 : 1;
  TMG_COUNT(2);
  if (h->scheme == 1) {
    if (to_view) {
      T3(launch_pdl(hybrid_kernel<0, true, false>, grid, dim3(256), 0, s, n, nat, v0, mask));
      T3(launch_pdl(hybrid_kernel<1, true, false>, grid, dim3(256), 0, s, n, nat, v1, mask));
    } else {
      T3(launch_pdl(hybrid_kernel<0, false, false>, grid, dim3(256), 0, s, n, nat, v0, mask));
      T3(launch_pdl(hybrid_kernel<1, false, false>, grid, dim3(256), 0, s, n, nat, v1, mask));
    }
  } else if (to_view) {
    T3(launch_pdl(hybrid_kernel<0, true, true>, grid, dim3(256), 0, s, n, nat, v0, mask));
    T3(launch_pdl(hybrid_kernel<1, true, true>, grid, dim3(256), 0, s, n, nat, v1, mask));
  } else {
    T3(launch_pdl(hybrid_kernel<0, false, true>, grid, dim3(256), 0, s, n, nat, v0, mask));
    T3(launch_pdl(hybrid_kernel<1, false, true>, grid, dim3(256), 0, s, n, nat, v1, mask));
  }
  return TMG_OK;
}

// the natural level-0 u of the session, current (after lazy cycles)
int ensure_natural(tmg_cube* h, cudaStream_t s) {
  if (!h->nat_stale) return TMG_OK;
  h->nat_stale = false;
  return convert3(h, 0, 0, false, s);
}

// one sweep of level l: on the caller's natural arrays (u, f), or on the
// session's hybrid views when use_views
int sweep3(tmg_cube* h, int l, double* u, const double* f, cudaStream_t s, bool use_views = false) {
  const int n = h->n[l];
  if (h->scheme == 1) {
    const tmg3::Fields3 F = use_views && hyb(h, l)
                                ? tmg3::Fields3{{h->UI[l], h->UJ[l], u}, {h->FI[l], h->FJ[l], f}, 1}
                                : tmg3::Fields3{{u, u, u}, {f, f, f}, 0};
    for (int red = 1; red >= 0; red--)
      if (tmg3::wire_stage(h->wl[l], n, coefs(h, l), red, F, h->err, s))
        return cuda3(cudaGetLastError(), "wireframe stage");
    return TMG_OK;
  }
  const tmg3::Fields3 F = use_views && hyb(h, l)
                              ? tmg3::Fields3{{h->UI[l], h->UJ[l], u}, {h->FI[l], h->FJ[l], f}, 2}
                              : tmg3::Fields3{{u, u, u}, {f, f, f}, 0};
  for (int red = 1; red >= 0; red--)
    if (tmg3::hub_stage(h->hl[l], n, coefs(h, l), red, F, h->err, s))
      return cuda3(cudaGetLastError(), "tweed stage");
  return TMG_OK;
}

dim3 grid3(int n) { return dim3((n + 1 + 255) / 256, n + 1, n + 1); }
// coarse planes per CTA: enough CTAs for ~4 waves of 148 SMs x 4
int restrict_ti(int nf) {
  const int m = nf / 2 - 1;
  const long tiles = (long)((m + kRTK - 1) / kRTK) * ((m + kRTJ - 1) / kRTJ);
  int ti = 16;
  while (ti > 1 && tiles * ((m + ti - 1) / ti) < 4L * 148 * 4) ti /= 2;
  return ti;
}
dim3 grid_restrict(int nf) {
  const int m = nf / 2 - 1, ti = restrict_ti(nf);  // interior coarse points per axis
  return dim3((m + kRTK - 1) / kRTK, (m + kRTJ - 1) / kRTJ, (m + ti - 1) / ti);
}
dim3 grid_prolong(int nc) { return dim3((nc + 255) / 256, nc, 2 * nc - 1); }

// The V-cycle from level l0.  Hybrid levels keep u in the views during the
// sweeps and in the natural array for the transfers; on return both forms of
// u[l0] are current.  entry: the views of l0 are to be filled first (the
// replicated tail of the sharded cycle; a session keeps them current).
// lazy: leave the natural u[l0] stale at the end (the session's graph; the
// next cycle converts after its pre-smoothing, readers call ensure_natural)
int cycle3(tmg_cube* h, int nu1, int nu2, cudaStream_t s, int l0 = 0, bool entry = false,
           bool lazy = false) {
  const int L = (int)h->n.size();
  if (entry && l0 < L - 1 && hyb(h, l0)) {
    int st = convert3(h, l0, 0, true, s);
    if (!st) st = convert3(h, l0, 1, true, s);
    if (st) return st;
  }
  for (int l = l0; l < L - 1; l++) {
    for (int k = 0; k < nu1; k++) {
      int st = sweep3(h, l, h->U[l], h->F[l], s, true);
      if (st) return st;
    }
    if (hyb(h, l) && (nu1 > 0 || (lazy && l == l0))) {
      int st = convert3(h, l, 0, false, s);
      if (st) return st;
    }
    TMG_COUNT(1);
    T3(launch_pdl(defect_restrict3_kernel, grid_restrict(h->n[l]), dim3(256), kRestrictSmem3, s,
                  h->n[l], coefs(h, l), h->U[l], h->F[l], h->F[l + 1], restrict_ti(h->n[l])));
    const size_t nc = (size_t)(h->n[l + 1] + 1) * (h->n[l + 1] + 1) * (h->n[l + 1] + 1);
    const dim3 zg((unsigned)std::min<size_t>((nc + 255) / 256, 148 * 16));
    TMG_COUNT(1);
    T3(launch_pdl(zero3_kernel, zg, dim3(256), 0, s, h->U[l + 1], nc));
    if (hyb(h, l + 1)) {
      TMG_COUNT(2);
      T3(launch_pdl(zero3_kernel, zg, dim3(256), 0, s, h->UI[l + 1], nc));
      T3(launch_pdl(zero3_kernel, zg, dim3(256), 0, s, h->UJ[l + 1], nc));
      int st = convert3(h, l + 1, 1, true, s);
      if (st) return st;
    }
  }
  TMG_COUNT(1);
  T3(launch_pdl(coarse3_kernel, dim3(1), dim3(1), 0, s, coefs(h, L - 1), h->U[L - 1], h->F[L - 1]));
  for (int l = L - 2; l >= l0; l--) {
    TMG_COUNT(1);
    T3(launch_pdl(prolong3v2_kernel, grid_prolong(h->n[l + 1]), dim3(256), 0, s, h->n[l + 1],
                  h->U[l + 1], h->U[l]));
    if (hyb(h, l)) {
      int st = convert3(h, l, 0, true, s);
      if (st) return st;
    }
    for (int k = 0; k < nu2; k++) {
      int st = sweep3(h, l, h->U[l], h->F[l], s, true);
      if (st) return st;
    }
    if (hyb(h, l) && nu2 > 0 && !(lazy && l == l0)) {  // natural u for the transfers / the caller
      int st = convert3(h, l, 0, false, s);
      if (st) return st;
    }
  }
  return cuda3(cudaGetLastError(), "cycle3");
}

}  // namespace

extern "C" {

const char* tmg_cube_last_error(void) { return g_err3.c_str(); }

// Hierarchy of cube levels from the finest 1D coordinates (n+1 values);
// coefficients W/E, S/N, B/T from the same coordinates on every axis
int tmg_cube_create(int n, const double* x, tmg_cube** out) {
  return tmg_cube_create_scheme(n, x, 0, out);
}

// scheme 0: 3D tweed (config 4), 1: 3D wireframe (config 5)
int tmg_cube_create_scheme(int n, const double* x, int scheme, tmg_cube** out) {
  if (!out || !x || n < 2 || n % 2) return fail3(TMG_BADARG, "cube needs even n >= 2");
  if (scheme != 0 && scheme != 1) return fail3(TMG_BADARG, "cube scheme must be 0 (tweed) or 1 (wireframe)");
  T3(cudaFuncSetAttribute(defect_restrict3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)kRestrictSmem3));
  tmg_cube* h = new tmg_cube();
  h->scheme = scheme;
  // hybrid views from 257^3 (wireframe) / 513^3 (tweed) up: measured break-even
  // against the conversions
  h->hyb_min = scheme == 1 ? 256 : 512;
  if (const char* e = getenv("TMG_HYB_MIN")) h->hyb_min = atoi(e);  // A/B: a large value disables
  std::vector<double> xs(x, x + n + 1);
  while (true) {
    const int m = (int)xs.size() - 1;
    h->n.push_back(m);
    // stencil.py:48-67 per axis
    std::vector<double> lo(m + 1, 0.0), hi(m + 1, 0.0);
    for (int i = 1; i < m; i++) {
      const double dc = (xs[i + 1] - xs[i - 1]) / 2.0;
      lo[i] = 1.0 / (dc * (xs[i] - xs[i - 1]));
      hi[i] = 1.0 / (dc * (xs[i + 1] - xs[i]));
    }
    std::vector<double> all;
    for (int rep = 0; rep < 3; rep++) {
      all.insert(all.end(), lo.begin(), lo.end());
      all.insert(all.end(), hi.begin(), hi.end());
    }
    double* dc = nullptr;
    T3(cudaMalloc(&dc, all.size() * sizeof(double)));
    T3(cudaMemcpy(dc, all.data(), all.size() * sizeof(double), cudaMemcpyHostToDevice));
    h->coef.push_back(dc);
    if (scheme == 1) {
      h->wl.emplace_back();
      std::string err;
      const int st = tmg3::wire_build_level(m, h->wl.back(), err);
      if (st) {
        tmg_cube_destroy(h);
        return fail3(st == 2 ? TMG_BADARG : TMG_CUDA, err);
      }
    }
    std::vector<Block3> bl[2];
    if (scheme == 0) {
      build_blocks(m, bl);
      h->hl.emplace_back();
      std::string err;
      const int st = tmg3::hub_build_level(m, bl, h->hl.back(), err);
      if (st) {
        tmg_cube_destroy(h);
        return fail3(st == 2 ? TMG_BADARG : TMG_CUDA, err);
      }
    }
    for (int r = 0; r < 2; r++) h->nblocks[r].push_back((int)bl[r].size());
    const size_t tot = (size_t)(m + 1) * (m + 1) * (m + 1);
    double *pu = nullptr, *pf = nullptr;
    T3(cudaMalloc(&pu, tot * sizeof(double)));
    T3(cudaMalloc(&pf, tot * sizeof(double)));
    T3(cudaMemset(pu, 0, tot * sizeof(double)));
    T3(cudaMemset(pf, 0, tot * sizeof(double)));
    h->U.push_back(pu);
    h->F.push_back(pf);
    double* views[4] = {nullptr, nullptr, nullptr, nullptr};
    if (m >= h->hyb_min)
      for (double*& v : views) {
        T3(cudaMalloc(&v, tot * sizeof(double)));
        T3(cudaMemset(v, 0, tot * sizeof(double)));
      }
    h->UI.push_back(views[0]);
    h->UJ.push_back(views[1]);
    h->FI.push_back(views[2]);
    h->FJ.push_back(views[3]);
    if (m % 2 || m / 2 < 2) break;
    std::vector<double> c;
    for (int i = 0; i <= m; i += 2) c.push_back(xs[i]);
    xs.swap(c);
  }
  const size_t tot = (size_t)(n + 1) * (n + 1) * (n + 1);
  T3(cudaMalloc(&h->err, sizeof(int) + sizeof(unsigned long long) * 2));
  h->dmax = reinterpret_cast<unsigned long long*>(h->err + 2);
  T3(cudaMemset(h->err, 0, sizeof(int)));
  T3(cudaMallocHost(&h->h_err, sizeof(int) * 2 + sizeof(unsigned long long) * 2));
  h->h_dmax = reinterpret_cast<unsigned long long*>(h->h_err + 2);
  *out = h;
  return TMG_OK;
}

int tmg_cube_destroy(tmg_cube* h) {
  if (!h) return TMG_OK;
  if (h->graph) cudaGraphExecDestroy(h->graph);
  if (h->solve_graph) cudaGraphExecDestroy(h->solve_graph);
  cudaFree(h->d_solve);
  for (double* p : h->coef) cudaFree(p);
  for (auto& w : h->wl) tmg3::wire_free_level(w);
  for (auto& kv : h->wparts) tmg3::wire_free_level(kv.second);
  for (auto& w : h->hl) tmg3::hub_free_level(w);
  for (double* p : h->U) cudaFree(p);
  for (double* p : h->F) cudaFree(p);
  for (auto* vv : {&h->UI, &h->UJ, &h->FI, &h->FJ})
    for (double* p : *vv) cudaFree(p);
  cudaFree(h->err);
  cudaFreeHost(h->h_err);
  delete h;
  return TMG_OK;
}

int tmg_cube_levels(tmg_cube* h) { return h ? (int)h->n.size() : 0; }

long tmg_cube_blocks(tmg_cube* h, int level, int red) {
  if (!h || level < 0 || level >= (int)h->n.size()) return -1;
  if (h->scheme == 1) return tmg3::wire_blocks(h->wl[level], red ? 1 : 0);
  return h->nblocks[red ? 1 : 0][level];
}

// one sweep of the finest level on caller arrays u, f (device, (n+1)^3)
int tmg_cube_sweep(tmg_cube* h, double* u, const double* f, void* stream) {
  if (!h) return fail3(TMG_BADARG, "null cube");
  return sweep3(h, 0, u, f, (cudaStream_t)stream);
}

// d = f - L u on the finest level (device arrays)
int tmg_cube_defect(tmg_cube* h, const double* u, const double* f, double* d, void* stream) {
  if (!h) return fail3(TMG_BADARG, "null cube");
  TMG_COUNT(1);
  defect3_kernel<<<grid3(h->n[0]), 256, 0, (cudaStream_t)stream>>>(h->n[0], coefs(h, 0), u, f, d,
                                                                   nullptr);
  return cuda3(cudaGetLastError(), "defect3");
}

// session: copy u, f (device, finest) in; cycles; norm; copy u out
int tmg_cube_load(tmg_cube* h, const double* u, const double* f, void* stream) {
  if (!h) return fail3(TMG_BADARG, "null cube");
  const size_t tot = (size_t)(h->n[0] + 1) * (h->n[0] + 1) * (h->n[0] + 1);
  cudaStream_t s = (cudaStream_t)stream;
  T3(cudaMemcpyAsync(h->U[0], u, tot * sizeof(double), cudaMemcpyDeviceToDevice, s));
  T3(cudaMemcpyAsync(h->F[0], f, tot * sizeof(double), cudaMemcpyDeviceToDevice, s));
  h->nat_stale = false;
  if (hyb(h, 0)) {
    int st = convert3(h, 0, 0, true, s);
    if (!st) st = convert3(h, 0, 1, true, s);
    if (st) return st;
  }
  return TMG_OK;
}

int tmg_cube_store(tmg_cube* h, double* u, void* stream) {
  if (!h) return fail3(TMG_BADARG, "null cube");
  if (int st = ensure_natural(h, (cudaStream_t)stream)) return st;
  const size_t tot = (size_t)(h->n[0] + 1) * (h->n[0] + 1) * (h->n[0] + 1);
  T3(cudaMemcpyAsync(u, h->U[0], tot * sizeof(double), cudaMemcpyDeviceToDevice,
                     (cudaStream_t)stream));
  return TMG_OK;
}

// `reps` V(nu1, nu2) cycles on the session (CUDA graph replay)
int tmg_cube_cycles(tmg_cube* h, int nu1, int nu2, int reps, void* stream) {
  if (!h) return fail3(TMG_BADARG, "null cube");
  if (nu1 < 0 || nu2 < 0 || nu1 + nu2 < 1) return fail3(TMG_BADARG, "need nu1 + nu2 >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->graph || h->gnu1 != nu1 || h->gnu2 != nu2) {
    if (h->graph) cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
    cudaStream_t cs;
    T3(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g;
    const long long counted = launch_counter();
    T3(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int st = cycle3(h, nu1, nu2, cs, 0, false, true);
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    launch_counter() = counted;
    cudaStreamDestroy(cs);
    if (st) return st;
    T3(e);
    size_t nn = 0;
    T3(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    T3(cudaGraphGetNodes(g, nodes.data(), &nn));
    h->graph_kernels = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      T3(cudaGraphNodeGetType(nd, &t));
      h->graph_kernels += t == cudaGraphNodeTypeKernel;
    }
    T3(cudaGraphInstantiate(&h->graph, g, 0));
    cudaGraphDestroy(g);
    h->gnu1 = nu1;
    h->gnu2 = nu2;
  }
  for (int r = 0; r < reps; r++) {
    T3(cudaGraphLaunch(h->graph, s));
    TMG_COUNT(h->graph_kernels);
  }
  if (reps > 0 && hyb(h, 0)) h->nat_stale = true;
  return TMG_OK;
}

// `reps` finest-level sweeps on the session's fields (the hybrid views when
// the level has them; both forms of u current on return): the smoother
// alone, as the V-cycle runs it
int tmg_cube_sweeps(tmg_cube* h, int reps, void* stream) {
  if (!h) return fail3(TMG_BADARG, "null cube");
  cudaStream_t s = (cudaStream_t)stream;
  h->nat_stale = false;  // the views are current; natural follows below
  for (int r = 0; r < reps; r++) {
    int st = sweep3(h, 0, h->U[0], h->F[0], s, true);
    if (st) return st;
  }
  if (hyb(h, 0)) return convert3(h, 0, 0, false, s);
  return TMG_OK;
}

// finest-level max |f - L u| of the session plus the pivot flag; synchronizes
int tmg_cube_norm(tmg_cube* h, double* out_host, void* stream) {
  if (!h) return fail3(TMG_BADARG, "null cube");
  cudaStream_t s = (cudaStream_t)stream;
  if (int st = ensure_natural(h, s)) return st;
  T3(cudaMemsetAsync(h->dmax, 0, sizeof(unsigned long long), s));
  TMG_COUNT(1);
  defect3_kernel<<<grid3(h->n[0]), 256, 0, s>>>(h->n[0], coefs(h, 0), h->U[0], h->F[0], nullptr,
                                                h->dmax);
  T3(cudaGetLastError());
  T3(cudaMemcpyAsync(h->h_dmax, h->dmax, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  T3(cudaMemcpyAsync(h->h_err, h->err, sizeof(int), cudaMemcpyDeviceToHost, s));
  T3(cudaMemsetAsync(h->err, 0, sizeof(int), s));
  T3(cudaStreamSynchronize(s));
  double v;
  std::memcpy(&v, h->h_dmax, sizeof(v));
  *out_host = v;
  if (*h->h_err & 1) return fail3(TMG_SINGULAR, "zero pivot during 3D block elimination");
  return TMG_OK;
}

// V(nu1, nu2) cycles on the loaded session until max |f - L u| <= tol * d0, a
// non-finite defect, a vanishing pivot or max_cycles (mgcycle.py:128-138 in
// 3D), run on the device as one while-node graph launch (V-cycle, defect
// norm, check kernel per iteration).  norms_out[1 .. cycles] receive the
// per-cycle defect norms; d0 is the caller's initial norm (tmg_cube_norm).
int tmg_cube_solve_loop(tmg_cube* h, int nu1, int nu2, double d0, double tol, int max_cycles,
                        double* norms_out, int* cycles_out, int* converged_out, void* stream) {
  if (!h) return fail3(TMG_BADARG, "null cube");
  if (nu1 < 0 || nu2 < 0 || nu1 + nu2 < 1) return fail3(TMG_BADARG, "need nu1 + nu2 >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  *cycles_out = 0;
  *converged_out = 0;
  if (max_cycles < 1) return TMG_OK;
  if (!h->d_solve || h->solve_cap < max_cycles) {
    if (h->solve_graph) cudaGraphExecDestroy(h->solve_graph);  // it bakes the state's address
    h->solve_graph = nullptr;
    cudaFree(h->d_solve);
    h->d_solve = nullptr;
    const int cap = max_cycles > 64 ? max_cycles : 64;
    T3(cudaMalloc(&h->d_solve, sizeof(tmg::SolveDev) + sizeof(double) * (size_t)cap));
    h->solve_cap = cap;
  }
  if (int st = ensure_natural(h, s)) return st;
  if (!h->solve_graph || h->snu1 != nu1 || h->snu2 != nu2) {
    if (h->solve_graph) cudaGraphExecDestroy(h->solve_graph);
    h->solve_graph = nullptr;
    tmg::ErrPtrs ep{};
    ep.n = 1;
    ep.p[0] = h->err;
    int st = tmg::build_while_graph(
        [&](cudaStream_t cs, cudaGraphConditionalHandle hdl) -> int {
          int st3 = cycle3(h, nu1, nu2, cs, 0, false, false);
          if (st3) return st3;
          TMG_COUNT(1);
          defect3_kernel<<<grid3(h->n[0]), 256, 0, cs>>>(h->n[0], coefs(h, 0), h->U[0], h->F[0],
                                                         nullptr, h->dmax);
          cudaError_t e = cudaGetLastError();
          if (e == cudaSuccess) e = tmg::launch_solve_check(cs, hdl, h->d_solve, h->dmax, ep);
          return cuda3(e, "cube solve graph body");
        },
        &h->solve_graph, &h->solve_kernels);
    if (st) return st;
    h->snu1 = nu1;
    h->snu2 = nu2;
  }
  tmg::SolveDev hs = {};
  hs.d0 = d0;
  hs.tol = tol;
  hs.max_cycles = max_cycles;
  T3(cudaMemcpyAsync(h->d_solve, &hs, offsetof(tmg::SolveDev, norms), cudaMemcpyHostToDevice, s));
  T3(cudaMemsetAsync(h->dmax, 0, sizeof(unsigned long long), s));
  T3(cudaGraphLaunch(h->solve_graph, s));
  T3(cudaMemcpyAsync(&hs, h->d_solve, offsetof(tmg::SolveDev, norms), cudaMemcpyDeviceToHost, s));
  T3(cudaMemcpyAsync(h->h_err, h->err, sizeof(int), cudaMemcpyDeviceToHost, s));
  T3(cudaMemsetAsync(h->err, 0, sizeof(int), s));
  T3(cudaStreamSynchronize(s));
  TMG_COUNT((long long)h->solve_kernels * hs.cycle);
  if (*h->h_err & 1) return fail3(TMG_SINGULAR, "zero pivot during 3D block elimination");
  if (hs.cycle > 0)
    T3(cudaMemcpy(norms_out + 1, h->d_solve->norms + 1, sizeof(double) * (size_t)hs.cycle,
                  cudaMemcpyDeviceToHost));
  *cycles_out = hs.cycle;
  *converged_out = hs.converged;
  return TMG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// sharded cube V-cycle (one rank's share, DESIGN.md §7/§11).
// Groups: 3D wireframe min(i', j', k') (the shell: its frame, the rings of its
// faces, its face centres), 3D tweed max(i', j', k') (the blocks whose branch
// has that largest mirrored coordinate); groups 1 .. n/2, neighbours of a
// point lie in groups g-1 .. g+1 and coarse group G is fine group 2G.

namespace {

// k' in [a, b] (inclusive, 1 <= a): k in [a, b] or [n-b, n-a], merged when
// they touch; visits the interior k in increasing order
template <class F>
void for_k_mirror_range(int n, int a, int b, F&& fn) {
  if (a > b) return;
  const int lo1 = a, hi1 = std::min(b, n - 1), lo2 = std::max(n - b, 1), hi2 = n - a;
  if (lo2 <= hi1 + 1) {
    for (int k = lo1; k <= std::max(hi1, hi2); k++) fn(k);
  } else {
    for (int k = lo1; k <= hi1; k++) fn(k);
    for (int k = lo2; k <= hi2; k++) fn(k);
  }
}

int cube_session_level(tmg_cube* h, int level, int need_coarser) {
  if (!h) return fail3(TMG_BADARG, "null cube");
  if (level < 0 || level >= (int)h->n.size() - need_coarser)
    return fail3(TMG_BADARG, "level " + std::to_string(level) + " out of range");
  return TMG_OK;
}

}  // namespace

extern "C" {

int tmg_cube_group_count(int scheme, int n) {
  if ((scheme != 0 && scheme != 1) || n < 2 || n % 2) return 0;
  return n / 2;
}

long tmg_cube_group_sizes(int scheme, int n, long long* sizes, long cap) {
  const int G = tmg_cube_group_count(scheme, n);
  if (G < 1) {
    g_err3 = "cube groups need scheme 0/1 and an even n >= 2";
    return -1;
  }
  if (cap < G + 1) return G + 1;
  // per axis: interior indices with mirrored coordinate >= g (n - 2g + 1) or <= g
  auto ge = [n](long g) -> long long { return g > n / 2 ? 0 : (long long)(n - 2 * g + 1); };
  auto le = [n](long g) -> long long { return g >= n / 2 ? (long long)(n - 1) : 2 * g; };
  sizes[0] = 0;
  for (int g = 1; g <= G; g++) {
    if (scheme == 1)
      sizes[g] = ge(g) * ge(g) * ge(g) - ge(g + 1) * ge(g + 1) * ge(g + 1);
    else
      sizes[g] = le(g) * le(g) * le(g) - le(g - 1) * le(g - 1) * le(g - 1);
  }
  return G + 1;
}

long tmg_cube_group_offsets(int scheme, int n, int g0, int g1, long long* off, long cap) {
  const int G = tmg_cube_group_count(scheme, n);
  if (G < 1) {
    g_err3 = "cube groups need scheme 0/1 and an even n >= 2";
    return -1;
  }
  g0 = std::max(g0, 1);
  g1 = std::min(g1, G + 1);
  long m = 0;
  const long long n1 = n + 1;
  for (int i = 1; i < n; i++)
    for (int j = 1; j < n; j++) {
      const int a = (int)mirror(i, n), b = (int)mirror(j, n);
      int lo, hi;  // allowed k' range
      if (scheme == 1) {  // min(a, b, k') in [g0, g1)
        const int m2 = std::min(a, b);
        if (m2 < g0) continue;
        lo = g0;
        hi = m2 >= g1 ? g1 - 1 : G;
      } else {  // max(a, b, k') in [g0, g1)
        const int m2 = std::max(a, b);
        if (m2 >= g1) continue;
        lo = m2 < g0 ? g0 : 1;
        hi = g1 - 1;
      }
      for_k_mirror_range(n, lo, std::min(hi, G), [&](int k) {
        if (m < cap) off[m] = (i * n1 + j) * n1 + k;
        m++;
      });
    }
  return m;
}

// one colour stage (red = 1 / black = 0) of the session's level-`level`
// blocks in groups [g0, g1)
int tmg_cube_sweep_part(tmg_cube* h, int level, int red, int g0, int g1, void* stream) {
  int st = cube_session_level(h, level, 0);
  if (st) return st;
  if ((st = ensure_natural(h, (cudaStream_t)stream))) return st;
  if (h->scheme != 1)
    return fail3(TMG_BADARG, "only the 3D wireframe shards (config 5); 3D tweed runs on one GPU");
  const auto key = std::make_tuple(level, g0, g1);
  auto it = h->wparts.find(key);
  if (it == h->wparts.end()) {
    std::string err;
    tmg3::WLevel w;
    const int b = tmg3::wire_build_level(h->n[level], w, err, g0, g1);
    if (b) return fail3(b == 2 ? TMG_BADARG : TMG_CUDA, err);
    it = h->wparts.emplace(key, w).first;
  }
  if (tmg3::wire_stage(it->second, h->n[level], coefs(h, level), red ? 1 : 0, h->U[level],
                       h->F[level], h->err, (cudaStream_t)stream))
    return cuda3(cudaGetLastError(), "wireframe part stage");
  return TMG_OK;
}

// F[level+1] = R (f - L u)[level], U[level+1] = 0 (mgcycle.py:98-100)
int tmg_cube_restrict(tmg_cube* h, int level, void* stream) {
  int st = cube_session_level(h, level, 1);
  if (st) return st;
  if ((st = ensure_natural(h, (cudaStream_t)stream))) return st;
  cudaStream_t s = (cudaStream_t)stream;
  TMG_COUNT(1);
  defect_restrict3_kernel<<<grid_restrict(h->n[level]), 256, kRestrictSmem3, s>>>(
      h->n[level], coefs(h, level), h->U[level], h->F[level], h->F[level + 1],
      restrict_ti(h->n[level]));
  const size_t nc = (size_t)(h->n[level + 1] + 1) * (h->n[level + 1] + 1) * (h->n[level + 1] + 1);
  T3(cudaMemsetAsync(h->U[level + 1], 0, nc * sizeof(double), s));
  return cuda3(cudaGetLastError(), "cube restrict");
}

// U[level] += P U[level+1] (mgcycle.py:101-102)
int tmg_cube_prolong(tmg_cube* h, int level, void* stream) {
  int st = cube_session_level(h, level, 1);
  if (st) return st;
  if ((st = ensure_natural(h, (cudaStream_t)stream))) return st;
  TMG_COUNT(1);
  prolong3v2_kernel<<<grid_prolong(h->n[level + 1]), 256, 0, (cudaStream_t)stream>>>(
      h->n[level + 1], h->U[level + 1], h->U[level]);
  return cuda3(cudaGetLastError(), "cube prolong");
}

// the V-cycle from `level` down to the coarsest and back (replicated tail)
int tmg_cube_tail(tmg_cube* h, int level, int nu1, int nu2, void* stream) {
  int st = cube_session_level(h, level, 0);
  if (st) return st;
  if ((st = ensure_natural(h, (cudaStream_t)stream))) return st;
  if (nu1 < 0 || nu2 < 0 || nu1 + nu2 < 1) return fail3(TMG_BADARG, "need nu1 + nu2 >= 1");
  return cycle3(h, nu1, nu2, (cudaStream_t)stream, level, true);
}

// out[q] = field[off[q]] / field[off[q]] = in[q]; which: 0 u, 1 f; off, out,
// in: DEVICE arrays (element offsets in the (n+1)^3 C-order level field)
int tmg_cube_gather(tmg_cube* h, int level, int which, const long long* off, long m, double* out,
                    void* stream) {
  int st = cube_session_level(h, level, 0);
  if (st || m <= 0) return st;
  if ((st = ensure_natural(h, (cudaStream_t)stream))) return st;
  TMG_COUNT(1);
  cube_gather_kernel<<<(unsigned)((m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      which ? h->F[level] : h->U[level], off, m, out);
  return cuda3(cudaGetLastError(), "cube gather");
}

int tmg_cube_scatter(tmg_cube* h, int level, int which, const long long* off, long m,
                     const double* in, void* stream) {
  int st = cube_session_level(h, level, 0);
  if (st || m <= 0) return st;
  if ((st = ensure_natural(h, (cudaStream_t)stream))) return st;
  TMG_COUNT(1);
  cube_scatter_kernel<<<(unsigned)((m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      which ? h->F[level] : h->U[level], off, m, in);
  return cuda3(cudaGetLastError(), "cube scatter");
}

// finest-level max |f - L u| over groups [g0, g1) plus the pivot flag;
// synchronizes
int tmg_cube_norm_part(tmg_cube* h, int g0, int g1, double* out_host, void* stream) {
  int st = cube_session_level(h, 0, 0);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = ensure_natural(h, s))) return st;
  T3(cudaMemsetAsync(h->dmax, 0, sizeof(unsigned long long), s));
  TMG_COUNT(1);
  defect3_kernel<<<grid3(h->n[0]), 256, 0, s>>>(h->n[0], coefs(h, 0), h->U[0], h->F[0], nullptr,
                                                h->dmax, h->scheme, g0, g1);
  T3(cudaGetLastError());
  T3(cudaMemcpyAsync(h->h_dmax, h->dmax, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  T3(cudaMemcpyAsync(h->h_err, h->err, sizeof(int), cudaMemcpyDeviceToHost, s));
  T3(cudaMemsetAsync(h->err, 0, sizeof(int), s));
  T3(cudaStreamSynchronize(s));
  double v;
  std::memcpy(&v, h->h_dmax, sizeof(v));
  *out_host = v;
  if (*h->h_err & 1) return fail3(TMG_SINGULAR, "zero pivot during 3D block elimination");
  return TMG_OK;
}

}  // extern "C"
