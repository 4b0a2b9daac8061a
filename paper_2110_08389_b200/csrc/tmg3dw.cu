// 3D wireframe colour stages on cubes (BASELINE config 5; SURVEY.md §8(c)
// "Candidate 3D layouts", the 3D wireframe).  The reference is 2D only; this
// carries its wireframe semantics (rings solved exactly as closed chains,
// _ckernels.pyx:106-141 / tridiag.py:46-81) to the survey's cube layout:
// with s1 <= s2 <= s3 the sorted mirrored coordinates of a point,
//   s1 == s2  the edge frame of shell r = s1 (12 edges, 8 degree-3 corners;
//             the cube centre for r = c), red;
//   s1 <  s2  ring level t = s2 in the shell-s1 face normal to the axis of
//             s1 (the face-centre point for t = c), colour parity(s1 + t),
//             red = even.
// The checker is oracle/wire3d_oracle.c (same layout, same ring order).
//
// Rings hold ~all the points.  One slice of TR threads per ring (TR = 32 ..
// 512 by ring length, several rings per 256-thread CTA for the short ones):
// the ring minus its closing point (the hub, the last point of the 2D ring
// order) is cut into chunks of <= 8 points, one per thread; each thread
// eliminates its chunk in registers to x = alpha + beta * X_left + gamma *
// X_end, the chunk ends form a tridiagonal system with a hub column (PCR in
// shared memory), one thread per ring solves the hub row, every thread
// finalises its chunk.  The 2D analogue is tmg_sweep.cu phases B-C.
// Frames (0.3 % of the points at 1025^3) are eliminated per edge with the two
// corner values as columns, the 8 corner rows are solved densely, and the
// edges are back-substituted.
#include <algorithm>
#include <cstring>
#include <vector>

#include "tmg3d.h"
#include "tmg_kernels.h"

namespace tmg3 {
namespace {

constexpr int kQW = 8;  // ring points per thread

__device__ __forceinline__ bool wbad(double v) { return v > -1e-300 && v < 1e-300; }

__device__ __forceinline__ const double* lo_of(const Coef3& c, int a) {
  return a == 0 ? c.W : (a == 1 ? c.S : c.B);
}
__device__ __forceinline__ const double* hi_of(const Coef3& c, int a) {
  return a == 0 ? c.E : (a == 1 ? c.N : c.T);
}

// hoisted geometry of one ring: face normal a at xa, in-face axes b < c
struct RingG {
  const double *lob, *hib, *loc, *hic;
  double kal, kah;  // couplings across the face (constant on the ring)
  long sa, sb, sc;
  size_t base;
  int t, m;
};

__device__ __forceinline__ RingG ring_geom(const Coef3& c, int n, const Ring3& R) {
  RingG G;
  const int a = R.a, b = a == 0 ? 1 : 0, cc = a == 2 ? 1 : 2;
  const long n1 = n + 1;
  auto str = [n1](int x) { return x == 0 ? n1 * n1 : (x == 1 ? n1 : 1L); };
  G.lob = lo_of(c, b);
  G.hib = hi_of(c, b);
  G.loc = lo_of(c, cc);
  G.hic = hi_of(c, cc);
  G.kal = __ldg(lo_of(c, a) + R.xa);
  G.kah = __ldg(hi_of(c, a) + R.xa);
  G.sa = str(a);
  G.sb = str(b);
  G.sc = str(cc);
  G.base = (size_t)R.xa * G.sa;
  G.t = R.t;
  G.m = n - 2 * R.t;
  return G;
}

// in-face coordinates of ring position p (layout.py:136-143 in the face)
__device__ __forceinline__ void ring_pos(const RingG& G, int n, int p, int& s, int& off, int& pb,
                                         int& pc) {
  s = p / G.m;
  off = p - s * G.m;
  const int t = G.t;
  if (s == 0) { pb = t + off; pc = t; }
  else if (s == 1) { pb = n - t; pc = t + off; }
  else if (s == 2) { pb = n - t - off; pc = n - t; }
  else { pb = t; pc = n - t - off; }
}

// A position on the ring: side s, offset off along it, in-face coordinates.
struct RingW {
  int s, off, pb, pc;
  __device__ __forceinline__ void init(const RingG& G, int n, int p) { ring_pos(G, n, p, s, off, pb, pc); }
  // one step toward p + 1
  __device__ __forceinline__ void next(const RingG& G) {
    if (++off == G.m) {
      off = 0;
      ++s;
    }
    // the corner that opens side s has the previous side's direction applied
    const int ds = off == 0 ? s - 1 : s;
    pb += ds == 0 ? 1 : (ds == 2 ? -1 : 0);
    pc += ds == 1 ? 1 : (ds == 3 ? -1 : 0);
  }
};

// Row of the ring point at walker W: frozen right-hand side r (all
// neighbours off the ring), diagonal d, couplings toward p-1 (am) and p+1
// (cn), element offset o.  In-face directions: 0 = b-, 1 = b+, 2 = c-, 3 =
// c+; side s runs toward fwd(s) = {1, 3, 0, 2}[s].
__device__ __forceinline__ void ring_row(const RingG& G, const double* __restrict__ u,
                                         const double* __restrict__ f, const RingW& W, double& r,
                                         double& d, double& am, double& cn, size_t& o) {
  const int s = W.s, off = W.off, pb = W.pb, pc = W.pc;
  o = G.base + (size_t)pb * G.sb + (size_t)pc * G.sc;
  const double c0 = __ldg(G.lob + pb), c1 = __ldg(G.hib + pb), c2 = __ldg(G.loc + pc),
               c3 = __ldg(G.hic + pc);
  const int fwd_s = s == 0 ? 1 : (s == 1 ? 3 : (s == 2 ? 0 : 2));
  const int sp = off > 0 ? s : (s + 3) & 3;
  const int fwd_p = sp == 0 ? 1 : (sp == 1 ? 3 : (sp == 2 ? 0 : 2));
  const int dnext = fwd_s, dprev = fwd_p ^ 1;
  const unsigned in = (1u << dnext) | (1u << dprev);  // the two ring directions
  d = -(c0 + c1 + c2 + c3 + G.kal + G.kah);
  double rr = f[o] - G.kal * u[o - G.sa] - G.kah * u[o + G.sa];
  if (!(in & 1u)) rr -= c0 * u[o - G.sb];
  if (!(in & 2u)) rr -= c1 * u[o + G.sb];
  if (!(in & 4u)) rr -= c2 * u[o - G.sc];
  if (!(in & 8u)) rr -= c3 * u[o + G.sc];
  r = rr;
  am = dprev == 0 ? c0 : (dprev == 1 ? c1 : (dprev == 2 ? c2 : c3));
  cn = dnext == 0 ? c0 : (dnext == 1 ? c1 : (dnext == 2 ? c2 : c3));
}


template <int TR>
__global__ void __launch_bounds__(TR > 256 ? TR : 256)
    ring3_kernel(int n, Coef3 c, const Ring3* __restrict__ rings, int nr, double* __restrict__ u,
                 const double* __restrict__ f, int* err) {
  constexpr int BD = TR > 256 ? TR : 256;
  __shared__ double sA[BD], sB[BD], sC[BD], sD[BD], sH[BD];
  __shared__ double sX[BD / TR];
  const int tid = threadIdx.x, lt = tid % TR;
  const int rid = blockIdx.x * (BD / TR) + tid / TR;
  const bool live = rid < nr;
  Ring3 R;
  if (live) R = rings[rid];
  else { R.a = 0; R.t = 1; R.xa = 1; }
  const RingG G = ring_geom(c, n, R);
  const int Lg = 4 * G.m - 1;  // open chain: every ring point but the hub
  const int q = (Lg + TR - 1) / TR;
  const int p0 = lt * q;
  const int cnt = live ? max(0, min(q, Lg - p0)) : 0;
  const int nI = cnt - 1;
  double rho[kQW], lam[kQW], ivr[kQW], cc[kQW];
  bool bad = false;
  double bp = 0.0, rp = 0.0, lm = 0.0, cprev = 0.0, a_first = 0.0;
  double r_end = 0.0, b_end = 1.0, a_end = 0.0, c_end = 0.0, ivp = 0.0;
  RingW W0;
  W0.init(G, n, min(p0, Lg));
  RingW W = W0;
#pragma unroll
  for (int k = 0; k < kQW; k++) {
    if (k > nI) continue;
    double r, d, am, cn;
    size_t o;
    if (k > 0) W.next(G);
    ring_row(G, u, f, W, r, d, am, cn, o);
    cc[k] = cn;
    if (k == 0) a_first = am;
    if (k == nI) {  // the chunk end keeps its raw row for the reduced system
      r_end = r;
      b_end = d;
      a_end = am;
      c_end = cn;
      continue;
    }
    if (k == 0) {
      bp = d;
      rp = r;
      lm = -am;
    } else {
      const double w = am * ivp;
      bp = d - w * cprev;
      rp = r - w * rp;
      lm = -w * lm;
    }
    bad |= wbad(bp);
    ivp = rcp3(bp);
    rho[k] = rp;
    lam[k] = lm;
    ivr[k] = ivp;
    cprev = cn;
  }
  // affine back pass: x_k = alpha + beta X_left + gamma X_end
  double ad = 0.0, bd = 1.0, gd = 0.0, au = 0.0, bu = 0.0, gu = 1.0;
  if (nI > 0) {
    double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
    for (int k = kQW - 1; k >= 0; k--) {
      if (k >= nI) continue;
      if (k == nI - 1) {
        al = rho[k] * ivr[k];
        be = lam[k] * ivr[k];
        ga = -cc[k] * ivr[k];
        ad = al; bd = be; gd = ga;
      } else {
        al = (rho[k] - cc[k] * al) * ivr[k];
        be = (lam[k] - cc[k] * be) * ivr[k];
        ga = -cc[k] * ga * ivr[k];
      }
      rho[k] = al;
      lam[k] = be;
      ivr[k] = ga;
    }
    au = al; bu = be; gu = ga;
  }
  sA[tid] = au;
  sB[tid] = bu;
  sC[tid] = gu;
  __syncthreads();
  // reduced row of the chunk end: A X_prev + B X + C X_next + H x_hub = D
  double A = 0.0, B = 1.0, Cc = 0.0, D = 0.0, H = 0.0;
  if (cnt > 0) {
    const double ae = nI > 0 ? a_end : a_first;
    if (nI > 0) {
      A = ae * bd;
      B = b_end + ae * gd;
      D = r_end - ae * ad;
    } else {
      A = ae;
      B = b_end;
      D = r_end;
    }
    if (p0 + cnt < Lg) {  // the next chunk's first point: an + bn X + gn X_next
      B += c_end * sB[tid + 1];
      Cc = c_end * sC[tid + 1];
      D -= c_end * sA[tid + 1];
    } else {
      H += c_end;  // the last leg point's successor is the hub
    }
    if (lt == 0) {  // the first point's predecessor is the hub
      H += A;
      A = 0.0;
    }
  }
  __syncthreads();
  sA[tid] = A; sB[tid] = B; sC[tid] = Cc; sD[tid] = D; sH[tid] = H;
  __syncthreads();
  for (int dd = 1; dd < TR; dd <<= 1) {
    double Am = 0, Bm = 1, Cm = 0, Dm = 0, Hm = 0, Ap = 0, Bp = 1, Cp = 0, Dp = 0, Hp = 0;
    if (lt - dd >= 0) {
      Am = sA[tid - dd]; Bm = sB[tid - dd]; Cm = sC[tid - dd]; Dm = sD[tid - dd]; Hm = sH[tid - dd];
    }
    if (lt + dd < TR) {
      Ap = sA[tid + dd]; Bp = sB[tid + dd]; Cp = sC[tid + dd]; Dp = sD[tid + dd]; Hp = sH[tid + dd];
    }
    __syncthreads();
    const double k1 = A * rcp3(Bm), k2 = Cc * rcp3(Bp);
    A = -k1 * Am;
    Cc = -k2 * Cp;
    B = B - k1 * Cm - k2 * Ap;
    D = D - k1 * Dm - k2 * Dp;
    H = H - k1 * Hm - k2 * Hp;
    sA[tid] = A; sB[tid] = B; sC[tid] = Cc; sD[tid] = D; sH[tid] = H;
    __syncthreads();
  }
  bad |= cnt > 0 && wbad(B);
  const double iB = rcp3(B);
  const double P = D * iB, Qh = H * iB;  // X_end = P - Qh x_hub
  sD[tid] = P;
  sH[tid] = Qh;
  __syncthreads();
  if (live && lt == 0) {  // the hub row
    double r, d, am, cn;
    size_t o;
    RingW Wh;
    Wh.init(G, n, Lg);
    ring_row(G, u, f, Wh, r, d, am, cn, o);
    const int last = tid + (Lg - 1) / q;
    const double Pl = sD[last], Ql = sH[last];
    const double num = r - am * Pl - cn * (au + gu * P);
    const double den = d - am * Ql + cn * (bu - gu * Qh);
    bad |= wbad(den);
    const double xh = num / den;
    u[o] = xh;
    sX[tid / TR] = xh;
  }
  __syncthreads();
  if (cnt > 0) {
    const double xh = sX[tid / TR];
    const double X = P - Qh * xh;
    const double Xl = lt == 0 ? xh : sD[tid - 1] - sH[tid - 1] * xh;
    RingW Wf = W0;
#pragma unroll
    for (int k = 0; k < kQW; k++) {
      if (k > nI) continue;
      if (k > 0) Wf.next(G);
      const size_t o = G.base + (size_t)Wf.pb * G.sb + (size_t)Wf.pc * G.sc;
      u[o] = k == nI ? X : rho[k] + lam[k] * Xl + ivr[k] * X;
    }
  }
  if (bad) atomicOr(err, 1);
}

// corner K of shell r: bit a set -> coordinate n - r on axis a
__device__ __forceinline__ size_t corner_off(int n, int r, int K) {
  const int i = K & 1 ? n - r : r, j = K & 2 ? n - r : r, k = K & 4 ? n - r : r;
  return idx3(n, i, j, k);
}

// Per frame edge: Thomas from the start corner with the two corner values as
// columns; scratch (4 per point) ends as alpha, beta, gamma; the first and
// last point forms go to ends.
__global__ void __launch_bounds__(128) frame_edge_kernel(int n, Coef3 c, const WEdge* __restrict__ edges,
                                                         int ne, const double* __restrict__ u,
                                                         const double* __restrict__ f,
                                                         double* __restrict__ scr,
                                                         double* __restrict__ ends, int* err) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= ne) return;
  const WEdge E = edges[id];
  const int r = E.r, x = E.ax, e = n - 2 * r - 1;
  const int o1 = x == 0 ? 1 : 0, o2 = x == 2 ? 1 : 2;
  const long n1 = n + 1, str[3] = {n1 * n1, n1, 1};
  int p[3];
  for (int a = 0; a < 3; a++) p[a] = (E.k0 >> a) & 1 ? n - r : r;
  const double t0 = __ldg(lo_of(c, o1) + p[o1]), t1 = __ldg(hi_of(c, o1) + p[o1]);
  const double t2 = __ldg(lo_of(c, o2) + p[o2]), t3 = __ldg(hi_of(c, o2) + p[o2]);
  const double tsum = t0 + t1 + t2 + t3;
  const double *lox = lo_of(c, x), *hix = hi_of(c, x);
  p[x] = 0;
  const size_t base = ((size_t)p[0] * n1 + p[1]) * (size_t)n1 + p[2];
  double* s = scr + 4 * (size_t)E.off;
  bool bad = false;
  double bp = 0.0, rp = 0.0, lm = 0.0, cprev = 0.0, ivp = 0.0;
#pragma unroll 4
  for (int k = 0; k < e; k++) {
    const int xx = r + 1 + k;
    const size_t o = base + (size_t)xx * str[x];
    const double am = __ldg(lox + xx), cn = __ldg(hix + xx);
    const double d = -(am + cn + tsum);
    const double rr = f[o] - t0 * u[o - str[o1]] - t1 * u[o + str[o1]] - t2 * u[o - str[o2]] -
                      t3 * u[o + str[o2]];
    if (k == 0) {
      bp = d;
      rp = rr;
      lm = -am;
    } else {
      const double w = am * ivp;
      bp = d - w * cprev;
      rp = rr - w * rp;
      lm = -w * lm;
    }
    bad |= wbad(bp);
    ivp = rcp3(bp);
    cprev = cn;
    s[4 * k + 0] = rp;
    s[4 * k + 1] = lm;
    s[4 * k + 2] = cn;
    s[4 * k + 3] = ivp;
  }
  double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll 4
  for (int k = e - 1; k >= 0; k--) {
    const double rk = s[4 * k + 0], lk = s[4 * k + 1], ck = s[4 * k + 2], ik = s[4 * k + 3];
    if (k == e - 1) {
      al = rk * ik;
      be = lk * ik;
      ga = -ck * ik;
    } else {
      al = (rk - ck * al) * ik;
      be = (lk - ck * be) * ik;
      ga = -ck * ga * ik;
    }
    s[4 * k + 0] = al;
    s[4 * k + 1] = be;
    s[4 * k + 2] = ga;
    if (k == e - 1) {
      ends[6 * (size_t)id + 3] = al;
      ends[6 * (size_t)id + 4] = be;
      ends[6 * (size_t)id + 5] = ga;
    }
  }
  ends[6 * (size_t)id + 0] = al;
  ends[6 * (size_t)id + 1] = be;
  ends[6 * (size_t)id + 2] = ga;
  if (bad) atomicOr(err, 1);
}

// Per frame: the 8 corner rows with the edge end forms substituted, solved by
// Gaussian elimination with partial pivoting (as the oracle).
__global__ void __launch_bounds__(64) frame_corner_kernel(int n, Coef3 c, const int* __restrict__ frames,
                                                          int nf, const WEdge* __restrict__ edges,
                                                          const double* __restrict__ ends,
                                                          double* __restrict__ u,
                                                          const double* __restrict__ f, int* err) {
  const int fi = blockIdx.x * blockDim.x + threadIdx.x;
  if (fi >= nf) return;
  const int r = frames[fi];
  double M[8][9];
  for (int K = 0; K < 8; K++) {
    const int p[3] = {K & 1 ? n - r : r, K & 2 ? n - r : r, K & 4 ? n - r : r};
    const size_t o = idx3(n, p[0], p[1], p[2]);
    const long n1 = n + 1, str[3] = {n1 * n1, n1, 1};
    double d = 0.0, rr = f[o];
    for (int a = 0; a < 3; a++) {
      const double lo = __ldg(lo_of(c, a) + p[a]), hi = __ldg(hi_of(c, a) + p[a]);
      d -= lo + hi;
      // the in-frame neighbour lies toward the shell's inside
      if (K >> a & 1) rr -= hi * u[o + str[a]];
      else rr -= lo * u[o - str[a]];
    }
    for (int q = 0; q < 8; q++) M[K][q] = 0.0;
    M[K][K] = d;
    M[K][8] = rr;
  }
  for (int ed = 0; ed < 12; ed++) {
    const WEdge E = edges[12 * fi + ed];
    const double* en = ends + 6 * (size_t)(12 * fi + ed);
    const int x = E.ax, K0 = E.k0, K1 = E.k1;
    const double c0 = __ldg(hi_of(c, x) + r), c1 = __ldg(lo_of(c, x) + (n - r));
    M[K0][K0] += c0 * en[1];
    M[K0][K1] += c0 * en[2];
    M[K0][8] -= c0 * en[0];
    M[K1][K0] += c1 * en[4];
    M[K1][K1] += c1 * en[5];
    M[K1][8] -= c1 * en[3];
  }
  bool bad = false;
  for (int col = 0; col < 8; col++) {
    int piv = col;
    for (int rr = col + 1; rr < 8; rr++)
      if (fabs(M[rr][col]) > fabs(M[piv][col])) piv = rr;
    bad |= wbad(M[piv][col]);
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
  for (int K = 0; K < 8; K++) u[corner_off(n, r, K)] = xc[K];
  if (bad) atomicOr(err, 1);
}

__global__ void __launch_bounds__(128) frame_back_kernel(int n, const WEdge* __restrict__ edges, int ne,
                                                         const double* __restrict__ scr,
                                                         double* __restrict__ u) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= ne) return;
  const WEdge E = edges[id];
  const int r = E.r, x = E.ax, e = n - 2 * r - 1;
  const double x0 = u[corner_off(n, r, E.k0)], x1 = u[corner_off(n, r, E.k1)];
  const long n1 = n + 1, str[3] = {n1 * n1, n1, 1};
  int p[3];
  for (int a = 0; a < 3; a++) p[a] = (E.k0 >> a) & 1 ? n - r : r;
  p[x] = 0;
  const size_t base = ((size_t)p[0] * n1 + p[1]) * (size_t)n1 + p[2];
  const double* s = scr + 4 * (size_t)E.off;
#pragma unroll 4
  for (int k = 0; k < e; k++)
    u[base + (size_t)(r + 1 + k) * str[x]] = s[4 * k] + s[4 * k + 1] * x0 + s[4 * k + 2] * x1;
}

__global__ void __launch_bounds__(128) wpoint_kernel(int n, Coef3 c, const int4* __restrict__ pts,
                                                     int np, double* __restrict__ u,
                                                     const double* __restrict__ f, int* err) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= np) return;
  const int4 P = pts[id];
  const int i = P.x, j = P.y, k = P.z;
  const size_t o = idx3(n, i, j, k);
  const double d = -(__ldg(c.W + i) + __ldg(c.E + i) + __ldg(c.S + j) + __ldg(c.N + j) +
                     __ldg(c.B + k) + __ldg(c.T + k));
  const double r = f[o] - __ldg(c.W + i) * u[idx3(n, i - 1, j, k)] -
                   __ldg(c.E + i) * u[idx3(n, i + 1, j, k)] -
                   __ldg(c.S + j) * u[idx3(n, i, j - 1, k)] -
                   __ldg(c.N + j) * u[idx3(n, i, j + 1, k)] - __ldg(c.B + k) * u[o - 1] -
                   __ldg(c.T + k) * u[o + 1];
  if (wbad(d)) atomicOr(err, 1);
  u[o] = r / d;
}

constexpr int kTR[kRingClasses] = {32, 64, 128, 256, 512};

template <typename T>
int upload(const std::vector<T>& v, T** out, std::string& err) {
  *out = nullptr;
  if (v.empty()) return 0;
  cudaError_t e = cudaMalloc(out, v.size() * sizeof(T));
  if (e == cudaSuccess) e = cudaMemcpy(*out, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    err = std::string("wireframe level upload: ") + cudaGetErrorString(e);
    return 3;
  }
  return 0;
}

}  // namespace

int wire_build_level(int n, WLevel& L, std::string& err) {
  const int c = n / 2;
  // Rings in launch order so that same-colour rings sharing 32-byte sectors
  // run together: a sector holds four consecutive k.  On faces normal to i or
  // j the k-neighbours of a strided side point are rings t +- 1, t +- 2 of
  // the same face: order (a, xa, t).  On faces normal to k they are the
  // faces of shells s1 +- 1, s1 +- 2: order (a, t, xa).
  std::vector<Ring3> rg[2][kRingClasses];
  for (int a = 0; a < 3; a++)
    for (int outer = 1; outer < n; outer++)
      for (int inner = 1; inner < n; inner++) {
        const int t = a == 2 ? outer : inner, xa = a == 2 ? inner : outer;
        if (t < 2 || t >= c) continue;
        const long s1 = mirror(xa, n);
        if (s1 >= t) continue;
        const int Lg = 4 * (n - 2 * t) - 1;
        int cls = 0;
        while (cls < kRingClasses && kTR[cls] * kQW < Lg) cls++;
        if (cls == kRingClasses) {
          err = "3D wireframe rings longer than " + std::to_string(kTR[kRingClasses - 1] * kQW + 1) +
                " points (n > 1026) are not supported";
          return 2;
        }
        const int red = ((s1 + t) % 2) == 0;
        rg[red][cls].push_back(Ring3{(int16_t)a, (int16_t)t, xa});
      }
  // frames (red) and their edges; scratch slots per edge point
  std::vector<int> fr;
  std::vector<WEdge> eg;
  int off = 0;
  for (int r = 1; r < c; r++) {
    const int e = n - 2 * r - 1;
    for (int ed = 0; ed < 12; ed++) {
      const int x = ed / 4, h = ed % 4;
      const int o1 = x == 0 ? 1 : 0, o2 = x == 2 ? 1 : 2;
      const int base = ((h & 1) << o1) | (((h >> 1) & 1) << o2);
      eg.push_back(WEdge{r, off, (int)fr.size(), (uint8_t)x, (uint8_t)base,
                         (uint8_t)(base | (1 << x)), (uint8_t)ed});
      off += e;
    }
    fr.push_back(r);
  }
  // points: the centre (red) and the face centres
  std::vector<int4> pt[2];
  pt[1].push_back(make_int4(c, c, c, 0));
  for (int a = 0; a < 3; a++)
    for (int side = 0; side < 2; side++)
      for (int s1 = 1; s1 < c; s1++) {
        int p[3] = {c, c, c};
        p[a] = side ? n - s1 : s1;
        pt[((s1 + c) % 2) == 0].push_back(make_int4(p[0], p[1], p[2], 0));
      }
  for (int red = 0; red < 2; red++) {
    for (int k = 0; k < kRingClasses; k++) {
      if (upload(rg[red][k], &L.rings[red][k], err)) return 3;
      L.nrings[red][k] = (int)rg[red][k].size();
    }
    if (upload(pt[red], &L.points[red], err)) return 3;
    L.npoints[red] = (int)pt[red].size();
  }
  if (upload(eg, &L.edges, err) || upload(fr, &L.frames, err)) return 3;
  L.nedges = (int)eg.size();
  L.nframes = (int)fr.size();
  if (off > 0) {
    cudaError_t e = cudaMalloc(&L.scratch, 4 * (size_t)off * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&L.ends, 6 * (size_t)L.nedges * sizeof(double));
    if (e != cudaSuccess) {
      err = std::string("wireframe scratch: ") + cudaGetErrorString(e);
      return 3;
    }
  }
  return 0;
}

void wire_free_level(WLevel& L) {
  for (int red = 0; red < 2; red++) {
    for (int k = 0; k < kRingClasses; k++) cudaFree(L.rings[red][k]);
    cudaFree(L.points[red]);
  }
  cudaFree(L.edges);
  cudaFree(L.frames);
  cudaFree(L.scratch);
  cudaFree(L.ends);
  L = WLevel();
}

long wire_blocks(const WLevel& L, int red) {
  long nb = L.npoints[red] + (red ? L.nframes : 0);
  for (int k = 0; k < kRingClasses; k++) nb += L.nrings[red][k];
  return nb;
}

template <int TR>
static void launch_rings(const WLevel& L, int n, const Coef3& c, int red, int k, double* u,
                         const double* f, int* err, cudaStream_t s) {
  constexpr int BD = TR > 256 ? TR : 256;
  const int nr = L.nrings[red][k];
  if (!nr) return;
  TMG_COUNT(1);
  ring3_kernel<TR><<<(nr + BD / TR - 1) / (BD / TR), BD, 0, s>>>(n, c, L.rings[red][k], nr, u, f,
                                                                  err);
}

int wire_stage(const WLevel& L, int n, const Coef3& c, int red, double* u, const double* f,
               int* err, cudaStream_t s) {
  launch_rings<32>(L, n, c, red, 0, u, f, err, s);
  launch_rings<64>(L, n, c, red, 1, u, f, err, s);
  launch_rings<128>(L, n, c, red, 2, u, f, err, s);
  launch_rings<256>(L, n, c, red, 3, u, f, err, s);
  launch_rings<512>(L, n, c, red, 4, u, f, err, s);
  if (red && L.nedges) {
    TMG_COUNT(3);
    frame_edge_kernel<<<(L.nedges + 127) / 128, 128, 0, s>>>(n, c, L.edges, L.nedges, u, f,
                                                             L.scratch, L.ends, err);
    frame_corner_kernel<<<(L.nframes + 63) / 64, 64, 0, s>>>(n, c, L.frames, L.nframes, L.edges,
                                                             L.ends, u, f, err);
    frame_back_kernel<<<(L.nedges + 127) / 128, 128, 0, s>>>(n, L.edges, L.nedges, L.scratch, u);
  }
  if (L.npoints[red]) {
    TMG_COUNT(1);
    wpoint_kernel<<<(L.npoints[red] + 127) / 128, 128, 0, s>>>(n, c, L.points[red],
                                                               L.npoints[red], u, f, err);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 3;
}

}  // namespace tmg3
