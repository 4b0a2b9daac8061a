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
// Device design: rings and frames are the same kind of block, straight
// edges between corners — a ring is 4 edges and 4 corners, a frame 12 edges
// and 8 corners — so every edge point is addressed as corner + q * stride
// and its row needs two 1D couplings and a per-edge constant.  One slice of
// TE threads per edge, <= kQW points per thread:
//  1. gather (one point per lane, coalesced along k): the frozen right-hand
//     side of every edge point into shared memory, and the corner rows;
//  2. per thread, backward elimination of its chunk and the affine forms of
//     its first and last interior points (chunk_eliminate);
//  3. per edge, the chunk ends' tridiagonal system with the two corner
//     values as columns, PCR in shared memory: every chunk end is
//     X = P - Q0 x_K0 - Q1 x_K1;
//  4. the corner rows with the edges' end points substituted: a dense 4 x 4
//     (ring) or 8 x 8 (frame, the survey's reduction to the corner unknowns)
//     system, one thread per block, partial pivoting;
//  5. every chunk finalised with both ends known (chunk_finalise), and a
//     coalesced scatter.
// The solve is exact for the block (the reference's block Gauss-Seidel
// step); only the elimination order differs from the circulant Thomas.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tmg3d.h"
#include "tmg_kernels.h"

namespace tmg3 {
namespace {

#ifndef TMG_WMINB
#define TMG_WMINB 2
#endif
#ifndef TMG_SKEL
#define TMG_SKEL 0
#endif
#ifndef TMG_WNB
#define TMG_WNB 4
#endif
#ifndef TMG_WQ
#define TMG_WQ 16
#endif
constexpr int kQW = 16;      // frame edge points per thread (one chunk)
constexpr int kRQ = TMG_WQ;  // ring side points per thread
constexpr int kRBD = 256;    // threads per ring CTA (at least)
constexpr int kMaxN = 1028;  // edges of <= 64 * 16 points

__device__ __forceinline__ bool wbad(double v) { return v > -1e-300 && v < 1e-300; }

// padded index into the shared-memory coupling tables: chunk-per-thread
// accesses (lane stride kQW points) land in distinct banks
template <int Q>
__device__ __forceinline__ int tix(int x) { return x + x / Q; }
__host__ __device__ constexpr int tab_len(int n) { return n + 1 + (n + 1) / 8 + 2; }

// shared-memory slot of edge point q: chunk rows of kQW, XOR swizzled so
// that both the chunk-per-thread and the point-per-lane accesses are
// conflict free
template <int Q>
__device__ __forceinline__ int rsw(int p) { return (p & ~(Q - 1)) | ((p ^ (p / Q)) & (Q - 1)); }

// Field views of a colour stage.  Natural mode: the three
// views alias the C-order arrays.  Hybrid mode (3D wireframe V-cycle): view
// 0 is an i-contiguous copy ([j][k][i]) owning the points whose largest
// mirrored coordinate is strictly i' (the i-edges), view 1 a j-contiguous
// copy ([i][k][j]) owning the j-edges, view 2 the natural array owning the
// k-edges; ties (ring and frame corners, face and cube centres) and the
// boundary are valid in all three.
__device__ __forceinline__ size_t off3(int lay, int n, int i, int j, int k) {
  const size_t n1 = (size_t)n + 1;
  return lay == 0 ? ((size_t)j * n1 + k) * n1 + i
                  : (lay == 1 ? ((size_t)i * n1 + k) * n1 + j : ((size_t)i * n1 + j) * n1 + k);
}
__device__ __forceinline__ long str3(int lay, int n, int axis) {
  const long n1 = n + 1;
  if (lay == 0) return axis == 0 ? 1 : (axis == 1 ? n1 * n1 : n1);
  if (lay == 1) return axis == 1 ? 1 : (axis == 0 ? n1 * n1 : n1);
  return axis == 0 ? n1 * n1 : (axis == 1 ? n1 : 1);
}
// owner view of a point in hybrid mode: the axis of the strictly largest
// mirrored coordinate (3D wireframe edges, HYB = 1) or of the strictly
// smallest (3D tweed legs, HYB = 2); -1 for ties and the boundary (valid in
// every view)
__device__ __forceinline__ int owner3(int n, int i, int j, int k, bool smallest) {
  if (i <= 0 || j <= 0 || k <= 0 || i >= n || j >= n || k >= n) return -1;
  int a = (int)mirror(i, n), b = (int)mirror(j, n), c = (int)mirror(k, n);
  if (smallest) { a = -a; b = -b; c = -c; }
  return (a > b && a > c) ? 0 : ((b > a && b > c) ? 1 : ((c > a && c > b) ? 2 : -1));
}
template <int HYB>
__device__ __forceinline__ double u_at(const Fields3& F, int n, int i, int j, int k) {
  if (!HYB) return F.u[2][off3(2, n, i, j, k)];
  const int o = owner3(n, i, j, k, HYB == 2), v = o < 0 ? 2 : o;
  return F.u[v][off3(v, n, i, j, k)];
}
// a tie (or any point in natural mode): every view
template <int HYB>
__device__ __forceinline__ void u_put_all(const Fields3& F, int n, int i, int j, int k, double x) {
  F.u[2][off3(2, n, i, j, k)] = x;
  if (HYB) {
    F.u[0][off3(0, n, i, j, k)] = x;
    F.u[1][off3(1, n, i, j, k)] = x;
  }
}

// Block kinds.  A ring (NE = 4 edges: face normal a at xa, level t), a frame
// (NE = 12: shell t) or a 3D tweed hub block (NE = 2, 3 or 6 legs meeting at
// a branch; tmg3d.cu).  Corners: ring K = 0..3 at in-face (b, c) = (t, t),
// (n-t, t), (n-t, n-t), (t, n-t) (layout.py:136-143's ring order: side 0
// runs K0 -> K1, side 1 K1 -> K2, side 2 K2 -> K3, side 3 K3 -> K0); frame K
// = 0..7 with bit a set for coordinate n - t on axis a; hub K = 0 the branch
// (the only unknown corner), K = 1 + e the wall point at the tip end of leg
// e (a Dirichlet value).
constexpr int kRing = 0, kFrame = 1, kHub = 2;

template <int KIND, int NE>
constexpr int ncorners() { return KIND == kRing ? 4 : (KIND == kFrame ? 8 : 1 + NE); }

struct WBlk {
  int a, xa, t;    // ring / frame
  int p[3];        // hub: the branch
  unsigned codes;  // hub: leg e in bits 3e .. 3e+2 (axis; bit 2: tip at n-1)
  int nleg;        // hub: legs in use (NE = 6 kernels also take 3-leg blocks)
};

template <int KIND, int NE>
__device__ __forceinline__ void corner_pos(const WBlk& B, int n, int K, int P[3]) {
  if (KIND == kFrame) {
    P[0] = K & 1 ? n - B.t : B.t;
    P[1] = K & 2 ? n - B.t : B.t;
    P[2] = K & 4 ? n - B.t : B.t;
  } else if (KIND == kRing) {
    const int pb = (K == 1 || K == 2) ? n - B.t : B.t, pc = K >= 2 ? n - B.t : B.t;
    P[0] = B.a == 0 ? B.xa : pb;
    P[1] = B.a == 1 ? B.xa : (B.a == 0 ? pb : pc);
    P[2] = B.a == 2 ? B.xa : pc;
  } else {
    P[0] = B.p[0];
    P[1] = B.p[1];
    P[2] = B.p[2];
    if (K > 0) {
      const unsigned code = (B.codes >> (3 * (K - 1))) & 7u;
      const int a = code & 3, w = (code & 4) ? n : 0;
      P[0] = a == 0 ? w : P[0];
      P[1] = a == 1 ? w : P[1];
      P[2] = a == 2 ? w : P[2];
    }
  }
}

// edge e: axis x, from corner K0 (lower coordinate) to K1
template <int KIND, int NE>
__device__ __forceinline__ void edge_def(const WBlk& B, int e, int& x, int& K0, int& K1) {
  if (KIND == kFrame) {
    x = e >> 2;
    const int h = e & 3, o1 = x == 0 ? 1 : 0, o2 = x == 2 ? 1 : 2;
    K0 = ((h & 1) << o1) | (((h >> 1) & 1) << o2);
    K1 = K0 | (1 << x);
  } else if (KIND == kRing) {
    const int b = B.a == 0 ? 1 : 0, c = B.a == 2 ? 1 : 2;
    x = (e & 1) ? c : b;
    K0 = e == 0 ? 0 : (e == 1 ? 1 : (e == 2 ? 3 : 0));
    K1 = e == 0 ? 1 : (e == 1 ? 2 : (e == 2 ? 2 : 3));
  } else {
    const unsigned code = (B.codes >> (3 * e)) & 7u;
    x = code & 3;
    K0 = (code & 4) ? 0 : 1 + e;  // tip at n-1: the branch is the lower end
    K1 = (code & 4) ? 1 + e : 0;
  }
}

// One edge's hoisted geometry: point q (0 .. L-1) at offset o0 + (q+1) sx,
// coordinate x0 + 1 + q along the axis; the four transverse couplings are
// constant along the edge.
struct EdgeG {
  double t0, t1, t2, t3, tsum;
  long sx, so1, so2;
  size_t o0;
  int x0, L;
  double* u;        // the view owning the edge (natural mode: the C-order array)
  const double* f;
};

// The cube API builds every axis from one coordinate array
// (tmg_cube_create), so W = S = B and E = N = T: c.W / c.E serve every axis.
template <int KIND, int NE, int HYB>
__device__ __forceinline__ EdgeG edge_geom(const Coef3& c, int n, const WBlk& B, int e,
                                           const Fields3& F) {
  int x, K0, K1, P0[3], P1[3];
  edge_def<KIND, NE>(B, e, x, K0, K1);
  corner_pos<KIND, NE>(B, n, K0, P0);
  corner_pos<KIND, NE>(B, n, K1, P1);
  const int o1 = x == 0 ? 1 : 0, o2 = x == 2 ? 1 : 2;
  EdgeG G;
  const int p1 = o1 == 0 ? P0[0] : P0[1], p2 = o2 == 1 ? P0[1] : P0[2];
  G.t0 = __ldg(c.W + p1);
  G.t1 = __ldg(c.E + p1);
  G.t2 = __ldg(c.W + p2);
  G.t3 = __ldg(c.E + p2);
  G.tsum = G.t0 + G.t1 + G.t2 + G.t3;
  const int lay = HYB ? x : 2;
  G.sx = str3(lay, n, x);
  G.so1 = str3(lay, n, o1);
  G.so2 = str3(lay, n, o2);
  G.o0 = off3(lay, n, P0[0], P0[1], P0[2]);
  G.u = F.u[lay];
  G.f = F.f[lay];
  G.x0 = x == 0 ? P0[0] : (x == 1 ? P0[1] : P0[2]);
  const int x1 = x == 0 ? P1[0] : (x == 1 ? P1[1] : P1[2]);
  G.L = x1 - G.x0 - 1;
  return G;
}

// Row of edge point q from the shared-memory coupling tables: the along
// couplings toward q-1 (am) and q+1 (cn), the diagonal d.
template <int Q>
struct EdgeCpl {
  const EdgeG& G;
  const double *tlo, *thi;
  __device__ __forceinline__ void operator()(int q, double& am, double& d, double& cn) const {
    const int xx = tix<Q>(G.x0 + 1 + q);
    am = tlo[xx];
    cn = thi[xx];
    d = -(am + cn + G.tsum);
  }
};

// Chunk passes.  A thread owns the chunk points p0 .. p0+e (e <= kQW-1); the
// interior 0 .. e-1 couples to X_left (the previous chunk's end, or a
// corner) and X_end (point e).  Backward elimination from e-1 down to 0
// leaves every interior row as
//   x_k = Rq_k + Mu_k X_end - Am_k x_{k-1}        (x_{-1} = X_left),
// Rq in shared memory (over r), Mu / Am in registers; a forward pass over
// those gives the affine forms of the first and last interior points, and the
// same recurrence finalises the chunk once X_left / X_end are known.
struct ChunkForms {
  double au = 0.0, bu = 0.0, gu = 1.0;  // x_0     = au + bu X_left + gu X_end
  double ad = 0.0, bd = 0.0, gd = 0.0;  // x_{e-1} = ad + bd X_left + gd X_end
};

template <int Q, class CPL>
__device__ __forceinline__ ChunkForms chunk_eliminate(const CPL& cpl, double* rr, int p0, int e,
                                                      double (&mu)[Q - 1], double (&amq)[Q - 1],
                                                      bool& bad) {
  ChunkForms F;
  if (e <= 0) return F;
  double bq = 0.0, rq = 0.0, m = 0.0, anext = 0.0, ivq = 0.0;
#pragma unroll
  for (int k = Q - 2; k >= 0; k--) {
    if (k < e) {
      double am, d, cn;
      cpl(p0 + k, am, d, cn);
      const int sl = rsw<Q>(p0 + k);
      const double r = rr[sl];
      if (k == e - 1) {
        bq = d;
        rq = r;
        m = -cn;
      } else {
        const double w = cn * ivq;
        bq = d - w * anext;
        rq = r - w * rq;
        m = -w * m;
      }
      bad |= wbad(bq);
      ivq = rcp3(bq);
      anext = am;
      rr[sl] = rq * ivq;
      mu[k] = m * ivq;
      amq[k] = am * ivq;
    }
  }
  double al = 0.0, be = 1.0, ga = 0.0;
#pragma unroll
  for (int k = 0; k < Q - 1; k++) {
    if (k < e) {
      const double rq_k = rr[rsw<Q>(p0 + k)];
      al = rq_k - amq[k] * al;
      be = -amq[k] * be;
      ga = mu[k] - amq[k] * ga;
      if (k == 0) {
        F.au = al;
        F.bu = be;
        F.gu = ga;
      }
    }
  }
  F.ad = al;
  F.bd = be;
  F.gd = ga;
  return F;
}

template <int Q>
__device__ __forceinline__ void chunk_finalise(double* rr, int p0, int e, double XL, double XE,
                                               const double (&mu)[Q - 1],
                                               const double (&amq)[Q - 1]) {
  double x = XL;
#pragma unroll
  for (int k = 0; k < Q - 1; k++) {
    if (k < e) {
      const int sl = rsw<Q>(p0 + k);
      x = rr[sl] + mu[k] * XE - amq[k] * x;
      rr[sl] = x;
    }
  }
  rr[rsw<Q>(p0 + e)] = XE;
}

// blocks of NE * TE threads per CTA (at most BDMAX threads), and the CTA
// size rounded up to whole warps (the extra threads idle: the PCR shuffles
// need full warps)
template <int NE, int TE, int BDMAX>
constexpr int wblock_bpc() { return BDMAX / (NE * TE); }
template <int NE, int TE, int BDMAX>
constexpr int wblock_bd() { return (wblock_bpc<NE, TE, BDMAX>() * NE * TE + 31) / 32 * 32; }

template <int NE, int TE, int BDMAX, int Q>
constexpr size_t wblock_smem() {
  return ((size_t)wblock_bd<NE, TE, BDMAX>() * (Q + 6) + 2 * (size_t)tab_len(kMaxN)) * sizeof(double);
}

// Blocks of one kind and class: whole blocks of NE * TE threads per CTA, TE
// threads per edge.  `blocks`: Ring3 (rings), int shell (frames) or HubB
// (3D tweed hub blocks).
template <int KIND, int NE, int TE, int BDMAX, int Q, int HYB>
__global__ void __launch_bounds__(wblock_bd<NE, TE, BDMAX>(), KIND == kFrame ? 1 : TMG_WMINB)
    wblock_kernel(int n, Coef3 c, const void* __restrict__ blocks, int nb, Fields3 F, int* err) {
  constexpr int NK = ncorners<KIND, NE>();
  constexpr int SL = NE * TE;  // threads per block
  constexpr int BD = wblock_bd<NE, TE, BDMAX>();
  constexpr int BPC = wblock_bpc<NE, TE, BDMAX>();
  static_assert(BPC >= 1 && (SL >= NK || KIND == kHub), "block slice");
  extern __shared__ double wsm[];
  double* sR = wsm;  // BD * Q
  double *sA = sR + BD * Q, *sB = sA + BD, *sC = sB + BD, *sD = sC + BD, *sH0 = sD + BD,
         *sH1 = sH0 + BD;
  double *tlo = sH1 + BD, *thi = tlo + tab_len(n);
  __shared__ double sEnd[BPC][NE][6];  // per edge: first / last point as al + be x_K0 + ga x_K1
  __shared__ double sKr[BPC][NK], sKd[BPC][NK], sXc[BPC][NK];
  const int tid = threadIdx.x, g = tid / SL, ed = (tid % SL) / TE, lt = tid % TE;
  const int bid = blockIdx.x * BPC + g;
  const bool live = g < BPC && bid < nb;  // threads past BPC blocks only fill the last warp
  WBlk B;
  B.a = 0; B.xa = 0; B.t = 1; B.p[0] = B.p[1] = B.p[2] = 1; B.codes = 0; B.nleg = NE;
  if (KIND == kRing) {
    if (live) {
      const Ring3 R = static_cast<const Ring3*>(blocks)[bid];
      B.a = R.a; B.xa = R.xa; B.t = R.t;
    }
  } else if (KIND == kFrame) {
    if (live) B.t = static_cast<const int*>(blocks)[bid];
  } else if (live) {
    const HubB H = static_cast<const HubB*>(blocks)[bid];
    B.p[0] = H.bi; B.p[1] = H.bj; B.p[2] = H.bk;
    B.nleg = H.nleg;
    for (int e = 0; e < NE; e++) B.codes |= (unsigned)(e < H.nleg ? H.leg[e] : 0) << (3 * e);
  }
  for (int x = tid; x <= n; x += BD) {
    tlo[tix<Q>(x)] = __ldg(c.W + x);
    thi[tix<Q>(x)] = __ldg(c.E + x);
  }
  const EdgeG G = edge_geom<KIND, NE, HYB>(c, n, B, ed, F);
  const int L = live && (KIND != kHub || ed < B.nleg) ? G.L : 0;  // unused hub legs: empty
  double* rr = sR + (g * NE + ed) * TE * Q;
  tmg::pdl_wait();  // the previous kernel's fields are complete from here on
  // 1. gather: edge points (four transverse neighbours), and the corner rows
  {
    constexpr int NB = TMG_WNB;  // points whose loads are in flight together
#pragma unroll 1
    for (int i0 = 0; i0 < Q; i0 += NB) {
      if (lt + i0 * TE >= L) break;
      double f0[NB], v0[NB], v1[NB], v2[NB], v3[NB];
#pragma unroll
      for (int b = 0; b < NB; b++) {
        const int q = min(lt + (i0 + b) * TE, L - 1);  // clamped: loads stay unconditional
        const size_t o = G.o0 + (size_t)(q + 1) * G.sx;
        f0[b] = G.f[o];
        v0[b] = G.u[o - G.so1];
        v1[b] = G.u[o + G.so1];
        v2[b] = G.u[o - G.so2];
        v3[b] = G.u[o + G.so2];
      }
#pragma unroll
      for (int b = 0; b < NB; b++) {
        const int q = lt + (i0 + b) * TE;
        if (q < L)
          rr[rsw<Q>(q)] = f0[b] - G.t0 * v0[b] - G.t1 * v1[b] - G.t2 * v2[b] - G.t3 * v3[b];
      }
    }
  }
  for (int K = tid % SL; live && K < NK; K += SL) {
    int P[3];
    corner_pos<KIND, NE>(B, n, K, P);
    if (KIND == kHub && K > 0) {
      sXc[g][K] = u_at<HYB>(F, n, P[0], P[1], P[2]);  // a wall point: its Dirichlet value
    } else {
      unsigned in = 0;  // in-block directions: bit 2a (toward -), 2a+1 (toward +)
      for (int e = 0; e < (KIND == kHub ? B.nleg : NE); e++) {
        int x, K0, K1;
        edge_def<KIND, NE>(B, e, x, K0, K1);
        if (K0 == K) in |= 2u << (2 * x);
        if (K1 == K) in |= 1u << (2 * x);
      }
      double d = 0.0, rk = F.f[2][off3(2, n, P[0], P[1], P[2])];
      for (int a = 0; a < 3; a++) {
        const double lo = __ldg(c.W + P[a]), hi = __ldg(c.E + P[a]);
        d -= lo + hi;
        const int i0 = P[0] - (a == 0), j0 = P[1] - (a == 1), k0 = P[2] - (a == 2);
        const int i1 = P[0] + (a == 0), j1 = P[1] + (a == 1), k1 = P[2] + (a == 2);
        if (!(in & (1u << (2 * a)))) rk -= lo * u_at<HYB>(F, n, i0, j0, k0);
        if (!(in & (2u << (2 * a)))) rk -= hi * u_at<HYB>(F, n, i1, j1, k1);
      }
      sKr[g][K] = rk;
      sKd[g][K] = d;
    }
  }
  __syncthreads();
#if TMG_SKEL
  bool bad = false;
#if TMG_SKEL == 2  // + three factor streams of 8 B per point (the factorised-solve estimate)
  if (KIND == kRing && L > 0) {
    double acc = 0.0;
    const int p0s = lt * Q;
    const double* src = G.f + G.o0 + 1;
#pragma unroll
    for (int k = 0; k < Q; k++)
      if (p0s + k < L) acc += __ldg(src + p0s + k) + __ldg(src + ((p0s + k + 7) % L)) * 0.5 +
                              __ldg(src + ((p0s + k + 13) % L)) * 0.25;
    if (p0s < L) rr[rsw<Q>(p0s)] += acc * 1e-300;
  }
#endif
  if (KIND != kRing) {
#endif
  // 2. chunk eliminations
  const EdgeCpl<Q> cpl{G, tlo, thi};
  const int p0 = lt * Q;
  const int cnt = max(0, min(Q, L - p0));
  const int e = cnt - 1;
  bool bad = false;
  double mu[Q - 1], amq[Q - 1];
  const ChunkForms Fm = chunk_eliminate<Q>(cpl, rr, p0, e, mu, amq, bad);
  sA[tid] = Fm.au;
  sB[tid] = Fm.bu;
  sC[tid] = Fm.gu;
  __syncthreads();
  // 3. reduced row of the chunk end: A X_prev + B X + C X_next + H0 x_K0 + H1 x_K1 = D
  double A = 0.0, Bv = 1.0, Cc = 0.0, D = 0.0, H0 = 0.0, H1 = 0.0;
  if (cnt > 0) {
    double ae, be, ce;
    cpl(p0 + e, ae, be, ce);
    const double re = rr[rsw<Q>(p0 + e)];
    if (e > 0) {
      A = ae * Fm.bd;
      Bv = be + ae * Fm.gd;
      D = re - ae * Fm.ad;
    } else {
      A = ae;
      Bv = be;
      D = re;
    }
    if (p0 + cnt < L) {  // the next chunk's first point: an + bn X + gn X_next
      Bv += ce * sB[tid + 1];
      Cc = ce * sC[tid + 1];
      D -= ce * sA[tid + 1];
    } else {
      H1 = ce;  // the last edge point's successor is the end corner
    }
    if (lt == 0) {  // the first edge point's predecessor is the start corner
      H0 = A;
      A = 0.0;
    }
  }
  // PCR over the edge's TE chunk ends: by shuffles when the edge is one
  // aligned lane segment of a warp (TE <= 32), through shared memory when it
  // spans two warps (TE = 64: a lane's partner at distance dd may sit in the
  // other warp for every dd)
  constexpr int WS = TE < 32 ? TE : 32;
  constexpr unsigned FULL = 0xffffffffu;
#pragma unroll
  for (int dd = 1; dd < TE; dd <<= 1) {
    double Am = 0, Bm = 1, Cm = 0, Dm = 0, Gm = 0, Hm = 0, Ap = 0, Bp = 1, Cp = 0, Dp = 0, Gp = 0,
           Hp = 0;
    if (TE <= 32) {  // the edge is one lane segment of a warp
      const double a1 = __shfl_up_sync(FULL, A, dd, WS), b1 = __shfl_up_sync(FULL, Bv, dd, WS);
      const double c1 = __shfl_up_sync(FULL, Cc, dd, WS), d1 = __shfl_up_sync(FULL, D, dd, WS);
      const double g1 = __shfl_up_sync(FULL, H0, dd, WS), h1 = __shfl_up_sync(FULL, H1, dd, WS);
      const double a2 = __shfl_down_sync(FULL, A, dd, WS), b2 = __shfl_down_sync(FULL, Bv, dd, WS);
      const double c2 = __shfl_down_sync(FULL, Cc, dd, WS), d2 = __shfl_down_sync(FULL, D, dd, WS);
      const double g2 = __shfl_down_sync(FULL, H0, dd, WS), h2 = __shfl_down_sync(FULL, H1, dd, WS);
      if (lt - dd >= 0) { Am = a1; Bm = b1; Cm = c1; Dm = d1; Gm = g1; Hm = h1; }
      if (lt + dd < TE) { Ap = a2; Bp = b2; Cp = c2; Dp = d2; Gp = g2; Hp = h2; }
    } else {
      __syncthreads();  // the previous phase's readers of the row arrays are done
      sA[tid] = A; sB[tid] = Bv; sC[tid] = Cc; sD[tid] = D; sH0[tid] = H0; sH1[tid] = H1;
      __syncthreads();
      if (lt - dd >= 0) {
        Am = sA[tid - dd]; Bm = sB[tid - dd]; Cm = sC[tid - dd]; Dm = sD[tid - dd];
        Gm = sH0[tid - dd]; Hm = sH1[tid - dd];
      }
      if (lt + dd < TE) {
        Ap = sA[tid + dd]; Bp = sB[tid + dd]; Cp = sC[tid + dd]; Dp = sD[tid + dd];
        Gp = sH0[tid + dd]; Hp = sH1[tid + dd];
      }
    }
    const double k1 = A * rcp3(Bm), k2 = Cc * rcp3(Bp);
    A = -k1 * Am;
    Cc = -k2 * Cp;
    Bv = Bv - k1 * Cm - k2 * Ap;
    D = D - k1 * Dm - k2 * Dp;
    H0 = H0 - k1 * Gm - k2 * Gp;
    H1 = H1 - k1 * Hm - k2 * Hp;
  }
  __syncthreads();  // every read of the row arrays is done before they are reused
  bad |= cnt > 0 && wbad(Bv);
  const double iB = rcp3(Bv);
  const double P = D * iB, Q0 = H0 * iB, Q1 = H1 * iB;  // X_end = P - Q0 x_K0 - Q1 x_K1
  sD[tid] = P;
  sH0[tid] = Q0;
  sH1[tid] = Q1;
  if (cnt > 0 && lt == 0) {  // the first edge point
    if (e > 0) {
      sEnd[g][ed][0] = Fm.au + Fm.gu * P;
      sEnd[g][ed][1] = Fm.bu - Fm.gu * Q0;
      sEnd[g][ed][2] = -Fm.gu * Q1;
    } else {
      sEnd[g][ed][0] = P;
      sEnd[g][ed][1] = -Q0;
      sEnd[g][ed][2] = -Q1;
    }
  }
  if (cnt > 0 && p0 + cnt == L) {  // the last edge point
    sEnd[g][ed][3] = P;
    sEnd[g][ed][4] = -Q0;
    sEnd[g][ed][5] = -Q1;
  }
  __syncthreads();
  // 4. the corner rows with the edge end points substituted.  Rings and hubs:
  // every thread solves the small system itself (no serial section, no
  // barrier); frames: one thread per frame, 8 x 8 with partial pivoting.
  double xc[4] = {0.0, 0.0, 0.0, 0.0};  // ring corners / the hub (xc[0])
  if (KIND == kHub && live) {
    // the branch row (m_legged_thomas's closing row, tridiag.py:84-125) with
    // every leg's end point next to it substituted; the walls are known
    double m = sKd[g][0], rhs = sKr[g][0];
    for (int eg = 0; eg < B.nleg; eg++) {
      int x, K0, K1, P0[3];
      edge_def<KIND, NE>(B, eg, x, K0, K1);
      corner_pos<KIND, NE>(B, n, 0, P0);
      const int xb = x == 0 ? P0[0] : (x == 1 ? P0[1] : P0[2]);
      if (K1 == 0) {  // tip at the low wall: the branch follows the leg's last point
        const double cw = __ldg(c.W + xb);
        m += cw * sEnd[g][eg][5];
        rhs -= cw * (sEnd[g][eg][3] + sEnd[g][eg][4] * sXc[g][K0]);
      } else {
        const double ce = __ldg(c.E + xb);
        m += ce * sEnd[g][eg][1];
        rhs -= ce * (sEnd[g][eg][0] + sEnd[g][eg][2] * sXc[g][K1]);
      }
    }
    bad |= wbad(m);
    xc[0] = rhs / m;
  }
  if (KIND == kRing && live) {
    // 4 x 4 corner system in registers (static indices): the Schur
    // complement of the diagonally dominant ring, eliminated without pivoting
    double M[4][5];
#pragma unroll
    for (int K = 0; K < 4; K++) {
#pragma unroll
      for (int q = 0; q < 4; q++) M[K][q] = 0.0;
      M[K][K] = sKd[g][K];
      M[K][4] = sKr[g][K];
    }
#pragma unroll
    for (int eg = 0; eg < 4; eg++) {
      const int K0 = eg == 0 ? 0 : (eg == 1 ? 1 : (eg == 2 ? 3 : 0));
      const int K1 = eg == 0 ? 1 : (eg == 1 ? 2 : (eg == 2 ? 2 : 3));
      // the corners' coordinates along the edge (b for even edges, c for odd)
      const int y0 = (eg & 1) ? ((K0 >= 2) ? n - B.t : B.t) : ((K0 == 1 || K0 == 2) ? n - B.t : B.t);
      const int y1 = (eg & 1) ? ((K1 >= 2) ? n - B.t : B.t) : ((K1 == 1 || K1 == 2) ? n - B.t : B.t);
      const double c0 = __ldg(c.E + y0), c1 = __ldg(c.W + y1);
      M[K0][K0] += c0 * sEnd[g][eg][1];
      M[K0][K1] += c0 * sEnd[g][eg][2];
      M[K0][4] -= c0 * sEnd[g][eg][0];
      M[K1][K0] += c1 * sEnd[g][eg][4];
      M[K1][K1] += c1 * sEnd[g][eg][5];
      M[K1][4] -= c1 * sEnd[g][eg][3];
    }
#pragma unroll
    for (int col = 0; col < 4; col++) {
      bad |= wbad(M[col][col]);
      const double iv = 1.0 / M[col][col];
#pragma unroll
      for (int q = col + 1; q < 4; q++) {
        const double w = M[q][col] * iv;
#pragma unroll
        for (int v = col; v <= 4; v++) M[q][v] -= w * M[col][v];
      }
    }
#pragma unroll
    for (int q = 3; q >= 0; q--) {
      double sum = M[q][4];
#pragma unroll
      for (int v = q + 1; v < 4; v++) sum -= M[q][v] * xc[v];
      xc[q] = sum / M[q][q];
    }
  }
  if (KIND == kFrame && live && tid % SL == 0) {
    double M[NK][NK + 1];
    for (int K = 0; K < NK; K++) {
      for (int q = 0; q < NK; q++) M[K][q] = 0.0;
      M[K][K] = sKd[g][K];
      M[K][NK] = sKr[g][K];
    }
    for (int eg = 0; eg < NE; eg++) {
      int x, K0, K1, P0[3], P1[3];
      edge_def<KIND, NE>(B, eg, x, K0, K1);
      corner_pos<KIND, NE>(B, n, K0, P0);
      corner_pos<KIND, NE>(B, n, K1, P1);
      const int x0 = x == 0 ? P0[0] : (x == 1 ? P0[1] : P0[2]);
      const int x1 = x == 0 ? P1[0] : (x == 1 ? P1[1] : P1[2]);
      const double c0 = __ldg(c.E + x0), c1 = __ldg(c.W + x1);
      M[K0][K0] += c0 * sEnd[g][eg][1];
      M[K0][K1] += c0 * sEnd[g][eg][2];
      M[K0][NK] -= c0 * sEnd[g][eg][0];
      M[K1][K0] += c1 * sEnd[g][eg][4];
      M[K1][K1] += c1 * sEnd[g][eg][5];
      M[K1][NK] -= c1 * sEnd[g][eg][3];
    }
    for (int col = 0; col < NK; col++) {
      int piv = col;
      for (int q = col + 1; q < NK; q++)
        if (fabs(M[q][col]) > fabs(M[piv][col])) piv = q;
      bad |= wbad(M[piv][col]);
      if (piv != col)
        for (int q = 0; q <= NK; q++) {
          const double tmp = M[col][q];
          M[col][q] = M[piv][q];
          M[piv][q] = tmp;
        }
      for (int q = col + 1; q < NK; q++) {
        const double w = M[q][col] / M[col][col];
        for (int v = col; v <= NK; v++) M[q][v] -= w * M[col][v];
      }
    }
    for (int q = NK - 1; q >= 0; q--) {
      double sum = M[q][NK];
      for (int v = q + 1; v < NK; v++) sum -= M[q][v] * sXc[g][v];
      sXc[g][q] = sum / M[q][q];
    }
  }
  if (KIND == kFrame) __syncthreads();  // the frame's corners from its solver thread
  auto corner_val = [&](int K) {
    if (KIND == kFrame) return sXc[g][K];
    if (KIND == kHub) return K == 0 ? xc[0] : sXc[g][K];
    return K == 0 ? xc[0] : (K == 1 ? xc[1] : (K == 2 ? xc[2] : xc[3]));
  };
  if (live && tid % SL < (KIND == kHub ? 1 : NK)) {  // hubs: the walls stay
    int P3[3];
    corner_pos<KIND, NE>(B, n, tid % SL, P3);
    u_put_all<HYB>(F, n, P3[0], P3[1], P3[2], corner_val(tid % SL));
  }
  // 5. finalise every chunk with both ends known, then scatter
  if (cnt > 0) {
    int x, K0, K1;
    edge_def<KIND, NE>(B, ed, x, K0, K1);
    const double xa = corner_val(K0), xb = corner_val(K1);
    const double XE = P - Q0 * xa - Q1 * xb;
    const double XL = lt == 0 ? xa : sD[tid - 1] - sH0[tid - 1] * xa - sH1[tid - 1] * xb;
    chunk_finalise<Q>(rr, p0, e, XL, XE, mu, amq);
  }
#if TMG_SKEL
  }
#endif
  __syncthreads();
  tmg::pdl_trigger();  // the successor may launch while this CTA scatters
#pragma unroll 4
  for (int it = 0; it < Q; it++) {
    const int q = lt + it * TE;
    if (q < L) G.u[G.o0 + (size_t)(q + 1) * G.sx] = rr[rsw<Q>(q)];
  }
  if (bad) atomicOr(err, 1);
}

template <int HYB>
__global__ void __launch_bounds__(128) wpoint_kernel(int n, Coef3 c, const int4* __restrict__ pts,
                                                     int np, Fields3 F, int* err) {
  tmg::pdl_trigger();
  tmg::pdl_wait();
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= np) return;
  const int4 P = pts[id];
  const int i = P.x, j = P.y, k = P.z;
  const double d = -(__ldg(c.W + i) + __ldg(c.E + i) + __ldg(c.S + j) + __ldg(c.N + j) +
                     __ldg(c.B + k) + __ldg(c.T + k));
  const double r = F.f[2][off3(2, n, i, j, k)] - __ldg(c.W + i) * u_at<HYB>(F, n, i - 1, j, k) -
                   __ldg(c.E + i) * u_at<HYB>(F, n, i + 1, j, k) -
                   __ldg(c.S + j) * u_at<HYB>(F, n, i, j - 1, k) -
                   __ldg(c.N + j) * u_at<HYB>(F, n, i, j + 1, k) - __ldg(c.B + k) * u_at<HYB>(F, n, i, j, k - 1) -
                   __ldg(c.T + k) * u_at<HYB>(F, n, i, j, k + 1);
  if (wbad(d)) atomicOr(err, 1);
  u_put_all<HYB>(F, n, i, j, k, r / d);
}

// test knob: TMG_FORCE_TE=t runs rings and frames with at least t threads
// per edge (small grids then exercise the wide classes, e.g. the two-warp
// PCR of TE = 64)
int force_te() {
  const char* e = getenv("TMG_FORCE_TE");
  return e ? atoi(e) : 0;
}

// ring classes: TE = 1 .. 64 threads per side (edges of m - 1 <= TE kQW points)
constexpr int kTE[kRingClasses] = {1, 2, 4, 8, 16, 32, 64, 128};
constexpr int ring_bd(int te) { return 4 * te > kRBD ? 4 * te : kRBD; }

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

template <int KIND, int NE, int TE, int BDMAX, int Q, int HYB = 0>
cudaError_t allow_smem() {
  if (HYB == 0 && KIND != kHub) {
    const cudaError_t e = allow_smem<KIND, NE, TE, BDMAX, Q, 1>();
    if (e != cudaSuccess) return e;
  }
  if (HYB == 0 && KIND == kHub) {
    const cudaError_t e = allow_smem<KIND, NE, TE, BDMAX, Q, 2>();
    if (e != cudaSuccess) return e;
  }
  return cudaFuncSetAttribute(wblock_kernel<KIND, NE, TE, BDMAX, Q, HYB>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)wblock_smem<NE, TE, BDMAX, Q>());
}

template <int KIND, int NE, int TE, int BDMAX, int Q, int HYB>
void launch_blocks(const void* blocks, int nb, int n, const Coef3& c, const Fields3& F, int* err,
                   cudaStream_t s) {
  if (!nb) return;
  constexpr int BD = wblock_bd<NE, TE, BDMAX>(), BPC = wblock_bpc<NE, TE, BDMAX>();
  TMG_COUNT(1);
  tmg::launch_pdl(wblock_kernel<KIND, NE, TE, BDMAX, Q, HYB>, dim3((nb + BPC - 1) / BPC), dim3(BD),
                  wblock_smem<NE, TE, BDMAX, Q>(), s, n, c, blocks, nb, F, err);
}

template <int TE, int HYB>
void launch_rings(const WLevel& L, int n, const Coef3& c, int red, int k, const Fields3& F, int* err,
                  cudaStream_t s) {
  launch_blocks<kRing, 4, TE, ring_bd(TE), kRQ, HYB>(L.rings[red][k], L.nrings[red][k], n, c, F, err, s);
}

template <int TE, int HYB>
void launch_frames(const WLevel& L, int n, const Coef3& c, const Fields3& F, int* err,
                   cudaStream_t s) {
  launch_blocks<kFrame, 12, TE, 12 * TE, kQW, HYB>(L.frames, L.nframes, n, c, F, err, s);
}

// 3D tweed hub blocks: classes by legs (2, 3, 6) and threads per leg
constexpr int kHubLegs[kHubKinds] = {2, 6};  // 3-leg blocks run in the 6-leg kernels
constexpr int kHubTE[kHubClasses] = {1, 2, 4, 8, 16, 32};

// A launch class with less than two waves of CTAs is folded into the next
// larger class (its blocks then run with idle threads): the small classes of
// the coarse levels cost a launch latency each and little work.
template <class T>
void merge_small_classes(std::vector<T>* cls, int nc, int ne, const int* te) {
  for (int q = 0; q + 1 < nc; q++) {
    const size_t per_cta = std::max(1, kRBD / (ne * te[q]));
    static const int waves = [] {
      const char* e = getenv("TMG_MERGE_WAVES");  // A/B knob: launch waves below which a class folds
      return e ? atoi(e) : 2;
    }();
    if (cls[q].empty() || cls[q].size() >= (size_t)waves * 148 * per_cta) continue;
    int nxt = q + 1;
    while (nxt + 1 < nc && cls[nxt].empty()) nxt++;
    if (cls[nxt].empty()) continue;  // the largest non-empty class stays
    cls[nxt].insert(cls[nxt].begin(), cls[q].begin(), cls[q].end());
    cls[q].clear();
  }
}

template <int NL, int HYB>
void launch_hubs(const HubLevel& L, int kind, int n, const Coef3& c, int red, const Fields3& F,
                 int* err, cudaStream_t s) {
  const HubB* const* b = L.blocks[red][kind];
  const int* nb = L.nblocks[red][kind];
  launch_blocks<kHub, NL, 1, kRBD, kQW, HYB>(b[0], nb[0], n, c, F, err, s);
  launch_blocks<kHub, NL, 2, kRBD, kQW, HYB>(b[1], nb[1], n, c, F, err, s);
  launch_blocks<kHub, NL, 4, kRBD, kQW, HYB>(b[2], nb[2], n, c, F, err, s);
  launch_blocks<kHub, NL, 8, kRBD, kQW, HYB>(b[3], nb[3], n, c, F, err, s);
  launch_blocks<kHub, NL, 16, kRBD, kQW, HYB>(b[4], nb[4], n, c, F, err, s);
  launch_blocks<kHub, NL, 32, kRBD, kQW, HYB>(b[5], nb[5], n, c, F, err, s);
}

template <int NL>
cudaError_t allow_hub_smem() {
  cudaError_t e = allow_smem<kHub, NL, 1, kRBD, kQW>();
  if (e == cudaSuccess) e = allow_smem<kHub, NL, 2, kRBD, kQW>();
  if (e == cudaSuccess) e = allow_smem<kHub, NL, 4, kRBD, kQW>();
  if (e == cudaSuccess) e = allow_smem<kHub, NL, 8, kRBD, kQW>();
  if (e == cudaSuccess) e = allow_smem<kHub, NL, 16, kRBD, kQW>();
  if (e == cudaSuccess) e = allow_smem<kHub, NL, 32, kRBD, kQW>();
  return e;
}

}  // namespace

int wire_build_level(int n, WLevel& L, std::string& err, int g0, int g1) {
  if (n > kMaxN) {
    err = "3D wireframe cubes above " + std::to_string(kMaxN) + " intervals are not supported";
    return 2;
  }
  const int c = n / 2;
  // Rings in launch order so that same-colour rings sharing 32-byte sectors
  // run together: a sector holds four consecutive k.  On faces normal to i or
  // j the k-neighbours of a strided side point are rings t +- 1, t +- 2 of
  // the same face: order (a, xa, t).  On faces normal to k they are the
  // faces of shells s1 +- 1, s1 +- 2: order (a, t, xa).
  std::vector<Ring3> rg[2][kRingClasses];
  const int fte = force_te();
  for (int a = 0; a < 3; a++)
    for (int outer = 1; outer < n; outer++)
      for (int inner = 1; inner < n; inner++) {
        const int t = a == 2 ? outer : inner, xa = a == 2 ? inner : outer;
        if (t < 2 || t >= c) continue;
        const long s1 = mirror(xa, n);
        if (s1 >= t || s1 < g0 || s1 >= g1) continue;  // the ring's sharding group is s1
        const int side = n - 2 * t - 1;  // points between two corners
        int cls = 0;
        while (cls < kRingClasses - 1 && (kTE[cls] * kRQ < side || kTE[cls] < fte)) cls++;
        const int red = ((s1 + t) % 2) == 0;
        rg[red][cls].push_back(Ring3{(int16_t)a, (int16_t)t, xa});
      }
  for (int red = 0; red < 2; red++) merge_small_classes(rg[red], kRingClasses, 4, kTE);
  std::vector<int> fr;  // frames (red): shells 1 .. c-1
  for (int r = std::max(1, g0); r < std::min(c, g1); r++) fr.push_back(r);
  // points: the centre (red, group c) and the face centres (group s1)
  std::vector<int4> pt[2];
  if (c >= g0 && c < g1) pt[1].push_back(make_int4(c, c, c, 0));
  for (int a = 0; a < 3; a++)
    for (int side = 0; side < 2; side++)
      for (int s1 = std::max(1, g0); s1 < std::min(c, g1); s1++) {
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
  if (upload(fr, &L.frames, err)) return 3;
  L.nframes = (int)fr.size();
  // dynamic shared memory above 48 KB (per function: sized for the largest n)
  cudaError_t e = allow_smem<kRing, 4, 1, ring_bd(1), kRQ>();
  if (e == cudaSuccess) e = allow_smem<kRing, 4, 2, ring_bd(2), kRQ>();
  if (e == cudaSuccess) e = allow_smem<kRing, 4, 4, ring_bd(4), kRQ>();
  if (e == cudaSuccess) e = allow_smem<kRing, 4, 8, ring_bd(8), kRQ>();
  if (e == cudaSuccess) e = allow_smem<kRing, 4, 16, ring_bd(16), kRQ>();
  if (e == cudaSuccess) e = allow_smem<kRing, 4, 32, ring_bd(32), kRQ>();
  if (e == cudaSuccess) e = allow_smem<kRing, 4, 64, ring_bd(64), kRQ>();
  if (kRQ < 16 && e == cudaSuccess) e = allow_smem<kRing, 4, 128, ring_bd(128), kRQ>();
  if (e == cudaSuccess) e = allow_smem<kFrame, 12, 4, 48, kQW>();
  if (e == cudaSuccess) e = allow_smem<kFrame, 12, 16, 192, kQW>();
  if (e == cudaSuccess) e = allow_smem<kFrame, 12, 64, 768, kQW>();
  if (e != cudaSuccess) {
    err = std::string("wireframe kernel shared memory: ") + cudaGetErrorString(e);
    return 3;
  }
  return 0;
}

void wire_free_level(WLevel& L) {
  for (int red = 0; red < 2; red++) {
    for (int k = 0; k < kRingClasses; k++) cudaFree(L.rings[red][k]);
    cudaFree(L.points[red]);
  }
  cudaFree(L.frames);
  L = WLevel();
}

long wire_blocks(const WLevel& L, int red) {
  long nb = L.npoints[red] + (red ? L.nframes : 0);
  for (int k = 0; k < kRingClasses; k++) nb += L.nrings[red][k];
  return nb;
}

template <int HYB>
void wire_stage_t(const WLevel& L, int n, const Coef3& c, int red, const Fields3& F, int* err,
                  cudaStream_t s) {
  launch_rings<1, HYB>(L, n, c, red, 0, F, err, s);
  launch_rings<2, HYB>(L, n, c, red, 1, F, err, s);
  launch_rings<4, HYB>(L, n, c, red, 2, F, err, s);
  launch_rings<8, HYB>(L, n, c, red, 3, F, err, s);
  launch_rings<16, HYB>(L, n, c, red, 4, F, err, s);
  launch_rings<32, HYB>(L, n, c, red, 5, F, err, s);
  launch_rings<64, HYB>(L, n, c, red, 6, F, err, s);
  if (kRQ < 16) launch_rings<128, HYB>(L, n, c, red, 7, F, err, s);
  if (red && L.nframes) {
    const int emax = std::max(n - 3, force_te() * kQW);  // the outermost frame's edges
    if (emax <= 4 * kQW) launch_frames<4, HYB>(L, n, c, F, err, s);
    else if (emax <= 16 * kQW) launch_frames<16, HYB>(L, n, c, F, err, s);
    else launch_frames<64, HYB>(L, n, c, F, err, s);
  }
  if (L.npoints[red]) {
    TMG_COUNT(1);
    tmg::launch_pdl(wpoint_kernel<HYB>, dim3((L.npoints[red] + 127) / 128), dim3(128), 0, s, n, c,
                    L.points[red], L.npoints[red], F, err);
  }
}

int wire_stage(const WLevel& L, int n, const Coef3& c, int red, const Fields3& F, int* err,
               cudaStream_t s) {
  if (F.hybrid) wire_stage_t<1>(L, n, c, red, F, err, s);
  else wire_stage_t<0>(L, n, c, red, F, err, s);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 3;
}

int wire_stage(const WLevel& L, int n, const Coef3& c, int red, double* u, const double* f,
               int* err, cudaStream_t s) {
  return wire_stage(L, n, c, red, Fields3{{u, u, u}, {f, f, f}, 0}, err, s);
}

int hub_build_level(int n, const std::vector<HubB> blocks[2], HubLevel& L, std::string& err) {
  if (n > kMaxN) {
    err = "3D tweed cubes above " + std::to_string(kMaxN) + " intervals are not supported";
    return 2;
  }
  const int fte = force_te();
  for (int red = 0; red < 2; red++) {
    std::vector<HubB> cls[kHubKinds][kHubClasses];
    std::vector<int4> pts;
    for (const HubB& B : blocks[red]) {
      if (B.len == 0) {  // a branch without legs: a point block, run as a hub with no legs
        HubB P = B;        // in the 6-leg kernels (its row alone: one launch less per stage)
        P.nleg = 0;
        cls[1][0].push_back(P);
        continue;
      }
      if (B.nleg != 2 && B.nleg != 3 && B.nleg != 6) {
        err = "3D tweed block with " + std::to_string(B.nleg) + " legs";
        return 2;
      }
      const int kind = B.nleg == 2 ? 0 : 1;
      int q = 0;
      while (q < kHubClasses - 1 && (kHubTE[q] * kQW < B.len || kHubTE[q] < fte)) q++;
      cls[kind][q].push_back(B);
    }
    for (int k = 0; k < kHubKinds; k++) merge_small_classes(cls[k], kHubClasses, kHubLegs[k], kHubTE);
    for (int k = 0; k < kHubKinds; k++)
      for (int q = 0; q < kHubClasses; q++) {
        if (upload(cls[k][q], &L.blocks[red][k][q], err)) return 3;
        L.nblocks[red][k][q] = (int)cls[k][q].size();
      }
    if (upload(pts, &L.points[red], err)) return 3;
    L.npoints[red] = (int)pts.size();
  }
  cudaError_t e = allow_hub_smem<2>();
  if (e == cudaSuccess) e = allow_hub_smem<6>();
  if (e != cudaSuccess) {
    err = std::string("tweed kernel shared memory: ") + cudaGetErrorString(e);
    return 3;
  }
  return 0;
}

void hub_free_level(HubLevel& L) {
  for (int red = 0; red < 2; red++) {
    for (int k = 0; k < kHubKinds; k++)
      for (int q = 0; q < kHubClasses; q++) cudaFree(L.blocks[red][k][q]);
    cudaFree(L.points[red]);
  }
  L = HubLevel();
}

template <int HYB>
void hub_stage_t(const HubLevel& L, int n, const Coef3& c, int red, const Fields3& F, int* err,
                 cudaStream_t s) {
  launch_hubs<2, HYB>(L, 0, n, c, red, F, err, s);
  launch_hubs<6, HYB>(L, 1, n, c, red, F, err, s);
  if (L.npoints[red]) {
    TMG_COUNT(1);
    tmg::launch_pdl(wpoint_kernel<HYB>, dim3((L.npoints[red] + 127) / 128), dim3(128), 0, s, n, c,
                    L.points[red], L.npoints[red], F, err);
  }
}

int hub_stage(const HubLevel& L, int n, const Coef3& c, int red, const Fields3& F, int* err,
              cudaStream_t s) {
  if (F.hybrid) hub_stage_t<2>(L, n, c, red, F, err, s);
  else hub_stage_t<0>(L, n, c, red, F, err, s);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 3;
}

int hub_stage(const HubLevel& L, int n, const Coef3& c, int red, double* u, const double* f,
              int* err, cudaStream_t s) {
  return hub_stage(L, n, c, red, Fields3{{u, u, u}, {f, f, f}, 0}, err, s);
}

}  // namespace tmg3
