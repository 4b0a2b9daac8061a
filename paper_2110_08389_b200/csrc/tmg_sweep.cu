// Block Gauss-Seidel colour stage on sm_100a: every same-colour block of a
// launch class is solved exactly, one bin (cluster of CTAs) per group of
// blocks.  Replaces relax_points / relax_chain / relax_ring / relax_legged
// (_ckernels.pyx:42-185) driven by smoothers.sweep (smoothers.py:121-150).
//
// Algorithm per bin (all fp64):
//  A  coalesced gather: each block point p gets r_p = f_p - sum of its
//     out-of-block neighbours (the frozen-RHS of _ckernels.pyx:34-39 without
//     the subtract/add-back of in-block neighbours, algebraically equal),
//     staged in shared memory in a chunk-major padded layout.
//  B  each thread owns a chunk of <= q consecutive leg points.  A down sweep
//     (Thomas forward elimination) and an affine back pass express every
//     chunk point as x = alpha + beta*x_{s-1} + gamma*x_e, leaving one reduced
//     unknown per chunk (its last point).  The reduced system is tridiagonal
//     per leg and is solved by parallel cyclic reduction across the CTA with
//     two right-hand sides: the data and the hub-coupling column.  The hub
//     (branch point / ring closing point) row then reduces to a scalar solve,
//     exactly as m_legged_thomas / circulant_thomas do (tridiag.py:46-125).
//  C  coalesced scatter of the new values.
#include <cooperative_groups.h>

#include "tmg_kernels.h"

namespace cg = cooperative_groups;

namespace tmg {

namespace {

struct PInfo {
  int i, j, dprev, dnext;
};

__device__ __forceinline__ PInfo leg_point(const LegD& L, int p) {
  PInfo r;
  r.i = L.i0;
  r.j = L.j0;
  r.dprev = (p == 0) ? ((L.flags & 1) ? (int)L.hub_dir_first : (int)DNONE) : (int)DNONE;
  r.dnext = (p == L.npts - 1) ? ((L.flags & 2) ? (int)L.hub_dir_last : (int)DNONE) : (int)DNONE;
  int cum = 0;
#pragma unroll
  for (int s = 0; s < 4; s++) {
    if (s < L.nseg) {
      int len = L.seg_len[s], d = L.seg_dir[s];
      int st = min(max(p - cum, 0), len);
      r.i += st * dir_di(d);
      r.j += st * dir_dj(d);
      if (p >= 1 && p > cum && p <= cum + len) r.dprev = dir_opp(d);
      if (p < L.npts - 1 && p + 1 > cum && p + 1 <= cum + len) r.dnext = d;
      cum += len;
    }
  }
  return r;
}

__device__ __forceinline__ void chunk_range(const LegD& L, int c, int q, int& s, int& e) {
  if (L.flags & 1) {
    if (c == 0) {
      s = 0;
      e = 0;
      return;
    }
    s = 1 + (c - 1) * q;
  } else {
    s = c * q;
  }
  e = min(s + q - 1, L.npts - 1);
}

__device__ __forceinline__ bool bad_pivot(double v) { return v > -1e-300 && v < 1e-300; }

template <bool CLUSTER>
__device__ __forceinline__ double* remote(double* p, int rank) {
  if constexpr (CLUSTER) {
    return cg::this_cluster().map_shared_rank(p, rank);
  } else {
    return p;
  }
}

template <bool CLUSTER>
__device__ __forceinline__ void bin_sync() {
  if constexpr (CLUSTER) {
    cg::this_cluster().sync();
  } else {
    __syncthreads();
  }
}

}  // namespace

// Shared-memory carve-up (doubles):
//   R   [T * QSMAX]   chunk-major point values (rhs -> rho -> alpha -> x)
//   E5  [5 * T]       reduced equations (A, B, C, D, H); also UP triples
//   XH  [T]           hub values of blocks whose hub thread lives here
constexpr int QSMAX = kQmax | 1;
constexpr size_t kSweepSmem = sizeof(double) * (size_t)(kThreads * QSMAX + 6 * kThreads);

template <bool CLUSTER>
__global__ void __launch_bounds__(kThreads, 2)
block_sweep_kernel(SweepArgs a, const ThreadD* __restrict__ threads,
                   const BinD* __restrict__ bins, int q, int cs) {
  extern __shared__ double smem[];
  constexpr int T = kThreads;
  double* R = smem;
  double* sA = R + T * QSMAX;
  double* sB = sA + T;
  double* sC = sB + T;
  double* sD = sC + T;
  double* sH = sD + T;
  double* XH = sH + T;

  const int tid = threadIdx.x;
  const int rank = CLUSTER ? (int)cg::this_cluster().block_rank() : 0;
  const int bin = blockIdx.x / cs;
  const int tv = rank * T + tid;  // virtual thread within the bin
  const ThreadD* th = threads + (size_t)blockIdx.x * T;
  const int QS = q | 1;
  const double* __restrict__ W = a.W;
  const double* __restrict__ E = a.E;
  const double* __restrict__ S = a.S;
  const double* __restrict__ N = a.N;
  const size_t ld = (size_t)a.ld;
  double* __restrict__ u = a.u;
  const double* __restrict__ f = a.f;

  auto coef = [&](int d, int i, int j) -> double {
    switch (d) {
      case DW: return __ldg(W + i);
      case DE: return __ldg(E + i);
      case DS: return __ldg(S + j);
      case DN: return __ldg(N + j);
      default: return 0.0;
    }
  };
  auto diag = [&](int i, int j) -> double {
    return -(__ldg(W + i) + __ldg(E + i) + __ldg(S + j) + __ldg(N + j));
  };
  // f - sum of neighbours not in `skip` (bit d set: neighbour d is in-block)
  auto frozen_rhs = [&](int i, int j, unsigned skip) -> double {
    const size_t o = (size_t)i * ld + j;
    double r = f[o];
    if (!(skip & 1u)) r -= __ldg(W + i) * u[o - ld];
    if (!(skip & 2u)) r -= __ldg(E + i) * u[o + ld];
    if (!(skip & 4u)) r -= __ldg(S + j) * u[o - 1];
    if (!(skip & 8u)) r -= __ldg(N + j) * u[o + 1];
    return r;
  };
  auto skipmask = [](int dp, int dn) -> unsigned {
    return (dp < 4 ? (1u << dp) : 0u) | (dn < 4 ? (1u << dn) : 0u);
  };

  // ---------------- phase A: coalesced gather of frozen right-hand sides ----
  for (int L = tid; L < T * q; L += T) {
    const int t = L / q, k = L - t * q;
    const int code = th[t];
    if (code < 0) continue;
    const LegD lg = a.legs[code];
    int s, e;
    chunk_range(lg, rank * T + t - lg.tbase, q, s, e);
    const int p = s + k;
    if (p > e) continue;
    const PInfo pi = leg_point(lg, p);
    R[t * QS + k] = frozen_rhs(pi.i, pi.j, skipmask(pi.dprev, pi.dnext));
  }
  __syncthreads();

  // ---------------- phase B: chunk elimination -------------------------------
  const int code = th[tid];
  LegD lg;
  int s = 0, e = -1, nI = 0, c = 0;
  if (code >= 0) {
    lg = a.legs[code];
    c = tv - lg.tbase;
    chunk_range(lg, c, q, s, e);
    nI = e - s;
  }
  double lam[kQmax], ivr[kQmax];
  double ad = 0.0, bd = 1.0, gd = 0.0;  // x_{e-1} = ad + bd*L + gd*X
  double au = 0.0, bu = 0.0, gu = 1.0;  // x_s     = au + bu*L + gu*X
  bool bad = false;
  double* Rt = R + tid * QS;
  if (nI > 0) {
    double bp = 0.0, rho = 0.0, lm = 0.0, cprev = 0.0, ivp = 0.0;
#pragma unroll
    for (int k = 0; k < kQmax; k++) {
      if (k < nI) {
        const PInfo pi = leg_point(lg, s + k);
        const double ap = coef(pi.dprev, pi.i, pi.j);
        const double bb = diag(pi.i, pi.j);
        const double rp = Rt[k];
        if (k == 0) {
          bp = bb;
          rho = rp;
          lm = -ap;
        } else {
          const double w = ap * ivp;
          bp = bb - w * cprev;
          rho = rp - w * rho;
          lm = -w * lm;
        }
        bad |= bad_pivot(bp);
        ivp = 1.0 / bp;
        Rt[k] = rho;
        lam[k] = lm;
        ivr[k] = ivp;
        cprev = coef(pi.dnext, pi.i, pi.j);
      }
    }
    // affine back substitution; cprev now holds c_{e-1}
    double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
    for (int k = kQmax - 1; k >= 0; k--) {
      if (k < nI) {
        if (k == nI - 1) {
          al = Rt[k] * ivr[k];
          be = lam[k] * ivr[k];
          ga = -cprev * ivr[k];
          ad = al;
          bd = be;
          gd = ga;
        } else {
          const PInfo pi = leg_point(lg, s + k);
          const double cp = coef(pi.dnext, pi.i, pi.j);
          al = (Rt[k] - cp * al) * ivr[k];
          be = (lam[k] - cp * be) * ivr[k];
          ga = -cp * ga * ivr[k];
        }
        Rt[k] = al;
        lam[k] = be;
        ivr[k] = ga;
      }
    }
    au = al;
    bu = be;
    gu = ga;
  }
  // publish the first-point affine form for the left neighbour chunk
  sA[tid] = au;
  sB[tid] = bu;
  sC[tid] = gu;
  __syncthreads();

  // reduced row of the chunk end e
  double A = 0.0, B = 1.0, C = 0.0, D = 0.0, H = 0.0;
  if (code >= 0) {
    const PInfo pe = leg_point(lg, e);
    const double ae = coef(pe.dprev, pe.i, pe.j);
    const double ce = coef(pe.dnext, pe.i, pe.j);
    A = ae * bd;
    B = diag(pe.i, pe.j) + ae * gd;
    D = Rt[nI] - ae * ad;
    if (c == lg.nchunk - 1) {
      if (lg.flags & 2) H += ce;
    } else {
      const double au1 = sA[tid + 1], bu1 = sB[tid + 1], gu1 = sC[tid + 1];
      B += ce * bu1;
      C = ce * gu1;
      D -= ce * au1;
    }
    if (c == 0) {
      if (lg.flags & 1) H += A;
      A = 0.0;
    }
  }
  __syncthreads();
  sA[tid] = A;
  sB[tid] = B;
  sC[tid] = C;
  sD[tid] = D;
  sH[tid] = H;
  __syncthreads();

  // parallel cyclic reduction of the per-leg reduced systems (legs never
  // straddle CTAs, so the exchange stays inside this CTA)
  const int steps = bins[bin].pcr_steps;
  for (int st = 0; st < steps; st++) {
    const int d = 1 << st;
    double Am = 0, Bm = 1, Cm = 0, Dm = 0, Hm = 0, Ap = 0, Bp = 1, Cp = 0, Dp = 0, Hp = 0;
    if (tid - d >= 0) {
      Am = sA[tid - d]; Bm = sB[tid - d]; Cm = sC[tid - d]; Dm = sD[tid - d]; Hm = sH[tid - d];
    }
    if (tid + d < T) {
      Ap = sA[tid + d]; Bp = sB[tid + d]; Cp = sC[tid + d]; Dp = sD[tid + d]; Hp = sH[tid + d];
    }
    __syncthreads();
    const double k1 = A / Bm, k2 = C / Bp;
    A = -k1 * Am;
    C = -k2 * Cp;
    B = B - k1 * Cm - k2 * Ap;
    D = D - k1 * Dm - k2 * Dp;
    H = H - k1 * Hm - k2 * Hp;
    sA[tid] = A; sB[tid] = B; sC[tid] = C; sD[tid] = D; sH[tid] = H;
    __syncthreads();
  }
  bad |= (code >= 0) && bad_pivot(B);
  const double P = D / B, Q = H / B;  // X_t = P - Q * x_hub
  sD[tid] = P;
  sH[tid] = Q;
  bin_sync<CLUSTER>();

  // hub rows: chunk 0 of a block's first leg, or the dedicated point thread
  int hub_blk = -1;
  if (code <= -2) hub_blk = -(code + 2);
  else if (code >= 0 && c == 0 && code == a.blocks[lg.block].leg0) hub_blk = lg.block;
  if (hub_blk >= 0) {
    const BlockD bk = a.blocks[hub_blk];
    if (bk.hi >= 0) {
      const int hi = bk.hi, hj = bk.hj;
      double num = frozen_rhs(hi, hj, bk.hub_mask);
      double den = diag(hi, hj);
      for (int l = 0; l < bk.nleg; l++) {
        const LegD L2 = a.legs[bk.leg0 + l];
        if (L2.flags & 2) {
          const int ta = L2.tbase + L2.nchunk - 1;
          const double cf = coef(dir_opp(L2.hub_dir_last), hi, hj);
          num -= cf * remote<CLUSTER>(sD, ta / T)[ta % T];
          den -= cf * remote<CLUSTER>(sH, ta / T)[ta % T];
        }
        if (L2.flags & 1) {
          const int ta = L2.tbase;
          const double cf = coef(dir_opp(L2.hub_dir_first), hi, hj);
          num -= cf * remote<CLUSTER>(sD, ta / T)[ta % T];
          den -= cf * remote<CLUSTER>(sH, ta / T)[ta % T];
        }
      }
      bad |= bad_pivot(den);
      const double xh = num / den;
      XH[tid] = xh;
      u[(size_t)hi * ld + hj] = xh;
    }
  }
  bin_sync<CLUSTER>();

  // final values of the chunk
  if (code >= 0) {
    const BlockD bk = a.blocks[lg.block];
    double xh = 0.0;
    if (bk.hi >= 0) xh = remote<CLUSTER>(XH, bk.hub_thread / T)[bk.hub_thread % T];
    const double X = P - Q * xh;
    double Lv;
    if (c == 0) Lv = (lg.flags & 1) ? xh : 0.0;
    else Lv = sD[tid - 1] - sH[tid - 1] * xh;
#pragma unroll
    for (int k = 0; k < kQmax; k++)
      if (k < nI) Rt[k] = Rt[k] + lam[k] * Lv + ivr[k] * X;
    Rt[nI] = X;
  }
  if (bad) atomicOr(a.err, 1);
  bin_sync<CLUSTER>();

  // ---------------- phase C: coalesced scatter ------------------------------
  for (int L = tid; L < T * q; L += T) {
    const int t = L / q, k = L - t * q;
    const int cd = th[t];
    if (cd < 0) continue;
    const LegD l2 = a.legs[cd];
    int s2, e2;
    chunk_range(l2, rank * T + t - l2.tbase, q, s2, e2);
    const int p = s2 + k;
    if (p > e2) continue;
    const PInfo pi = leg_point(l2, p);
    u[(size_t)pi.i * ld + pi.j] = R[t * QS + k];
  }
}

// Point Gauss-Seidel colour stage for checkerboard (smoothers.py:65-75,
// _ckernels.pyx:42-51): red = (i + j) even.
__global__ void __launch_bounds__(256) point_sweep_kernel(SweepArgs a, int nx, int ny, int red) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int i = blockIdx.y + 1;
  if (j >= ny || i >= nx) return;
  if ((((i + j) & 1) == 0) != (red != 0)) return;
  const size_t ld = (size_t)a.ld, o = (size_t)i * ld + j;
  const double Wi = __ldg(a.W + i), Ei = __ldg(a.E + i), Sj = __ldg(a.S + j), Nj = __ldg(a.N + j);
  const double b = -(Wi + Ei + Sj + Nj);
  const double r = a.f[o] - Wi * a.u[o - ld] - Ei * a.u[o + ld] - Sj * a.u[o - 1] - Nj * a.u[o + 1];
  a.u[o] = r / b;
}

cudaError_t init_sweep_kernels() {
  static cudaError_t done = cudaErrorNotReady;
  if (done == cudaErrorNotReady) {
    done = cudaFuncSetAttribute(block_sweep_kernel<false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
    if (done == cudaSuccess)
      done = cudaFuncSetAttribute(block_sweep_kernel<true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepSmem);
  }
  return done;
}

cudaError_t launch_colour(const Plan& P, int red, const SweepArgs& a, cudaStream_t stream) {
  if (P.point_scheme) {
    dim3 grid((P.geo.ny - 1 + 255) / 256, P.geo.nx - 1);
    point_sweep_kernel<<<grid, 256, 0, stream>>>(a, P.geo.nx, P.geo.ny, red);
    return cudaGetLastError();
  }
  for (const LaunchClass& lc : P.classes) {
    if (lc.red != red || lc.nbins == 0) continue;
    if (lc.cs == 1) {
      block_sweep_kernel<false><<<lc.nbins, kThreads, kSweepSmem, stream>>>(a, lc.threads, lc.bins,
                                                                            lc.q, 1);
    } else {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(lc.nbins * lc.cs);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = kSweepSmem;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = lc.cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&cfg, block_sweep_kernel<true>, a,
                                         (const ThreadD*)lc.threads, (const BinD*)lc.bins, lc.q,
                                         lc.cs);
      if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace tmg
