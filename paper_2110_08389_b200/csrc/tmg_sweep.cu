// Block Gauss-Seidel colour stage on sm_100a: every same-colour block of a
// launch class is solved exactly, one bin (cluster of CTAs) per group of
// blocks.  Replaces relax_points / relax_chain / relax_ring / relax_legged
// (_ckernels.pyx:42-185) driven by smoothers.sweep (smoothers.py:121-150).
//
// Work decomposition (host side, tmg_plan.cu): every leg of a block is cut
// into straight chunks of <= q points, one chunk per thread, described by a
// 16-byte ChunkD (element offset, stride, along/cross indices, the couplings
// of its two ends).  Per bin, all fp64:
//  A  coalesced gather: lane-consecutive points of the bin's chunks read f and
//     the out-of-block neighbours of u and stage the frozen right-hand side
//     r_p = f_p - sum(out-of-block couplings) in shared memory (the frozen RHS
//     of _ckernels.pyx:34-39 without the subtract / add-back of in-block
//     neighbours, which is algebraically equal).
//  B  per thread: a Thomas down sweep and an affine back pass over the chunk
//     interior express every chunk point as x = alpha + beta*x_left + gamma*X,
//     X being the chunk's last point; the chunk ends form a tridiagonal reduced
//     system per leg, solved by parallel cyclic reduction (warp shuffles, then
//     shared memory) with two right-hand sides: the data and the hub coupling.
//     The hub row (branch point / ring closing point) is then a scalar solve,
//     as in m_legged_thomas / circulant_thomas (tridiag.py:46-125).
//  C  coalesced scatter of the new values.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "tmg_kernels.h"
#include "tmg_transfer_dev.cuh"

namespace cg = cooperative_groups;

// -DTMG_CHECK (make check): device bounds checks on the gathered / scattered
// global offsets, the hub couplings and the DSMEM ranks (stand-in for
// compute-sanitizer, which the GPU pool does not offer; profiles/r02_boundscheck.txt)
#ifdef TMG_CHECK
#define SWEEP_CHECK(cond, what)                                                              \
  do {                                                                                       \
    if (!(cond)) {                                                                           \
      printf("block kernel check failed: %s (block %d thread %d)\n", what, (int)blockIdx.x, \
             (int)threadIdx.x);                                                              \
      __trap();                                                                              \
    }                                                                                        \
  } while (0)
#else
#define SWEEP_CHECK(cond, what) \
  do {                          \
  } while (0)
#endif



#ifndef TMG_SKIP
#define TMG_SKIP 0  // profiling only: 1 skip elimination, 2 skip PCR, 4 skip hubs, 8 skip finalize, 16 skip chunk-end pass
#endif


#ifndef TMG_BATCH
#define TMG_BATCH 8  // gather items in flight per lane
#endif
#ifndef TMG_PDL_LATE
#define TMG_PDL_LATE 1  // 0: signal the dependent launch at entry instead of after the solve
#endif

#ifndef TMG_STAGE_ALONG
#define TMG_STAGE_ALONG 1  // 0: read the along couplings per thread through L1 (measured slower)
#endif

#ifndef TMG_MINB8
#define TMG_MINB8 TMG_MINB  // resident CTAs per SM targeted by the q <= 8 kernels
#endif

#ifndef TMG_MINB
#define TMG_MINB (TMG_THREADS >= 512 ? 1 : 2)  // resident CTAs per SM the register budget is sized for
#endif

namespace tmg {

namespace {

__device__ __forceinline__ bool bad_pivot(double v) { return v > -1e-300 && v < 1e-300; }

// reciprocal: the ~20-bit hardware approximation refined by two Newton steps
// (measured on B200 over 4M values in [1e-8, 1e14]: equal to 1.0/x;
// tools/micro/rcp_test.cu)
__device__ __forceinline__ double drcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#ifdef TMG_FAKE_RCP
  return r;  // timing experiment only: wrong results
#endif
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

template <bool CLUSTER>
__device__ __forceinline__ double* remote(double* p, int rank) {
  if constexpr (CLUSTER) {
    return cg::this_cluster().map_shared_rank(p, rank);
  } else {
    return p;
  }
}

// split cluster barrier: arrive once this CTA's DSMEM reads are done, wait
// before exiting (no CTA may exit while a peer can still read its memory)
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <bool CLUSTER>
__device__ __forceinline__ void bin_sync() {
  if constexpr (CLUSTER) {
    cg::this_cluster().sync();
  } else {
    __syncthreads();
  }
}

struct Coefs {
  const double* __restrict__ W;
  const double* __restrict__ E;
  const double* __restrict__ S;
  const double* __restrict__ N;
  __device__ __forceinline__ double dir(int d, int i, int j) const {
    switch (d) {
      case DW: return __ldg(W + i);
      case DE: return __ldg(E + i);
      case DS: return __ldg(S + j);
      case DN: return __ldg(N + j);
      default: return 0.0;
    }
  }
};

// Geometry of one chunk, unpacked into registers.
struct Chunk {
  int off, stride, a0, da, cidx, cs, n, dfirst, dlast, link, hub, own, axis, tb;
  const double* __restrict__ pa;  // along coupling toward the previous point
  const double* __restrict__ pc;  // along coupling toward the next point
  const double* __restrict__ xl;  // cross coefficients (low / high side)
  const double* __restrict__ xh;

  __device__ __forceinline__ void unpack(const ChunkD& c, const Coefs& C, int ld, int ldt) {
    n = c.n;
    off = c.off;
    a0 = c.a0;
    cidx = c.cidx;
    axis = c.geo & 1;
    const int neg = (c.geo >> 1) & 1;
    tb = (c.geo >> 2) & 1;
    da = neg ? -1 : 1;
    // along / cross strides inside the owning buffer (tmg_layout.h)
    const int si = tb ? 1 : ld, sj = tb ? ldt : 1;
    stride = (axis ? sj : si) * da;
    cs = axis ? si : sj;
    dfirst = c.link & 7;
    dlast = (c.link >> 3) & 7;
    link = c.link;
    hub = c.hub;
    own = c.own;
    const double* lo = axis ? C.S : C.W;
    const double* hi = axis ? C.N : C.E;
    pa = neg ? hi : lo;
    pc = neg ? lo : hi;
    xl = axis ? C.W : C.S;
    xh = axis ? C.E : C.N;
  }
  __device__ __forceinline__ void ij(int k, int& i, int& j) const {
    const int a = a0 + k * da;
    i = axis ? cidx : a;
    j = axis ? a : cidx;
  }
};

}  // namespace

#ifdef TMG_PHASE_TIMING
__device__ long long g_phase_t[12][1 << 16];
__device__ int g_phase_n;
#define TMG_T(slot)                                                        \
  do {                                                                     \
    if (threadIdx.x == 0 && blockIdx.x < (1 << 16)) {                      \
      g_phase_t[slot][blockIdx.x] = clock64();                             \
      if (slot == 0) atomicMax(&g_phase_n, (int)blockIdx.x + 1);           \
    }                                                                      \
  } while (0)
#else
#define TMG_T(slot) \
  do {              \
  } while (0)
#endif

// Shared memory (doubles):
//   R [, PA, PC] [T * Q] chunk-major point values: the right-hand side
//                     (later rho, alpha, x) and, when TMG_STAGE_ALONG, the
//                     along couplings toward the previous / next point
//                     (otherwise each thread reads them from the 1D
//                     coefficient arrays through L1); row t slot k lives at
//                     t*Q + (k ^ (t & (Q-1))) (XOR swizzle: conflict-free
//                     for both the lane-along-chunk gather and the
//                     lane-per-chunk elimination, no padding)
//   E5        [5 * T] reduced rows (A, B, C, D, H); first-point triples
//   XH        [T]     hub values, slot = owner thread
template <int Q>
constexpr size_t sweep_smem() {
  return sizeof(double) * (size_t)((TMG_STAGE_ALONG ? 3 : 1) * kThreads * Q + 6 * kThreads);
}

template <int Q>
__device__ __forceinline__ int sw(int t, int k) {
  return t * Q + (k ^ (t & (Q - 1)));
}

// Along couplings of a thread's chunk point k: toward the previous (a) and
// the next (c) point.  Staged rows in shared memory, or the 1D coefficient
// arrays (the same values: a chunk is one straight run, so point k's
// couplings sit at a fixed element step from the first point's).
template <int Q>
struct AlongStaged {
  const double* PA;
  const double* PC;
  int tid;
  __device__ __forceinline__ double a(int k) const { return PA[sw<Q>(tid, k)]; }
  __device__ __forceinline__ double c(int k) const { return PC[sw<Q>(tid, k)]; }
};
struct AlongL1 {
  const double* __restrict__ pa;
  const double* __restrict__ pc;
  int da;
  __device__ __forceinline__ double a(int k) const { return __ldg(pa + k * da); }
  __device__ __forceinline__ double c(int k) const { return __ldg(pc + k * da); }
};
#if TMG_STAGE_ALONG
template <int Q>
using Along = AlongStaged<Q>;
#else
template <int Q>
using Along = AlongL1;
#endif

// Phase B of one chunk: Thomas down sweep over the chunk interior (the
// coupling to the previous chunk's end kept as the column lam) and an affine
// back pass leaving x_k = alpha_k + beta_k * Xleft + gamma_k * X in (R, lam,
// ivr).  NI > 0: compile-time interior count (full chunks, no predicates);
// NI == 0: runtime count nI.  (ad, bd, gd) = the form of the last interior
// point, (au, bu, gu) = that of the first.
template <int Q, int NI, class AL>
__device__ __forceinline__ void chunk_eliminate(int tid, int nI, double* R, const AL& cpl,
                                                double csum, double a_first,
                                                double (&lam)[Q], double (&ivr)[Q], bool& bad,
                                                double& ad, double& bd, double& gd, double& au,
                                                double& bu, double& gu) {
  const int n = NI > 0 ? NI : nI;
  double bp = 0.0, rho = 0.0, lm = 0.0, ivp = 0.0, cprev = 0.0;
#pragma unroll
  for (int k = 0; k < Q; k++) {
    if (k < n) {
      const int sl = sw<Q>(tid, k);
      const double pav = cpl.a(k), pcv = cpl.c(k), rp = R[sl];
      const double bb = -(pav + pcv + csum);
      if (k == 0) {
        bp = bb;
        rho = rp;
        lm = -a_first;
      } else {
        const double w = pav * ivp;
        bp = fma(-w, cprev, bb);
        rho = fma(-w, rho, rp);
        lm = -w * lm;
      }
      bad |= bad_pivot(bp);
      ivp = drcp(bp);
      R[sl] = rho;
      lam[k] = lm;
      ivr[k] = ivp;
      cprev = pcv;
    }
  }
  // affine back substitution; cprev = c_{e-1}
  double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
  for (int k = Q - 1; k >= 0; k--) {
    if (k < n) {
      const int sl = sw<Q>(tid, k);
      if (k == n - 1) {
        al = R[sl] * ivr[k];
        be = lam[k] * ivr[k];
        ga = -cprev * ivr[k];
        ad = al;
        bd = be;
        gd = ga;
      } else {
        const double cp = cpl.c(k);
        al = fma(-cp, al, R[sl]) * ivr[k];
        be = fma(-cp, be, lam[k]) * ivr[k];
        ga = -cp * ga * ivr[k];
      }
      R[sl] = al;
      lam[k] = be;
      ivr[k] = ga;
    }
  }
  au = al;
  bu = be;
  gu = ga;
}

// One bin (a cluster's worth of chunks) of a colour stage.
template <bool CLUSTER, bool XCTA, int Q>
__device__ __forceinline__ void sweep_bin(const SweepArgs& a, const ChunkD* __restrict__ chunks,
                                          const BinD* __restrict__ bins,
                                          const HubD* __restrict__ hubs, int cs_size, int bin,
                                          int rank, double* smem) {
  constexpr int T = kThreads;
  double* R = smem;
  double* PA = R + T * Q;  // staged along couplings (TMG_STAGE_ALONG only)
  double* PC = PA + T * Q;
  double* sA = TMG_STAGE_ALONG ? PC + T * Q : R + T * Q;
  double* sB = sA + T;
  double* sC = sB + T;
  double* sD = sC + T;
  double* sH = sD + T;
  double* XH = sH + T;

  const int tid = threadIdx.x;
  const int ld = a.ld;
  const Coefs C{a.W, a.E, a.S, a.N};
  double* __restrict__ u = a.u;
  const double* __restrict__ f = a.f;

  TMG_T(0);
  if (!TMG_PDL_LATE) pdl_trigger();
  // static plan data and couplings first: under PDL these loads overlap the
  // previous kernel, and none of them waits on another after the wait
  const ChunkD mine = chunks[((size_t)bin * cs_size + rank) * T + tid];
  const BinD bd_ = bins[bin];
  Chunk c;
  c.unpack(mine, C, ld, a.ldt);
  const bool has_hub = !(TMG_SKIP & 4) && c.own >= 0;
  HubD hb0{};
  double hW = 0.0, hE = 0.0, hS = 0.0, hN = 0.0;
  if (has_hub) {
    const HubD& hb = hb0;
    hb0 = hubs[bd_.hub0 + c.own];
    hW = __ldg(a.W + hb.i);
    hE = __ldg(a.E + hb.i);
    hS = __ldg(a.S + hb.j);
    hN = __ldg(a.N + hb.j);
  }

  const double xlv = c.n > 0 ? __ldg(c.xl + c.cidx) : 0.0;
  const double xhv = c.n > 0 ? __ldg(c.xh + c.cidx) : 0.0;
  pdl_wait();  // the field data of the previous kernel are complete from here on
  TMG_T(7);
  const FieldView U{u, a.ut, a.nx, a.ny, a.mode};
  const FieldView F{const_cast<double*>(f), const_cast<double*>(a.ft), a.nx, a.ny, a.mode};
  // frozen part of this thread's hub row (its out-of-block neighbours are
  // never written during this colour stage), loaded now so that the loads
  // overlap the gather instead of sitting on the hub step's critical path
  // Every load below is unconditional (clamped to a valid point when unused)
  // and masked through its coupling, so that all of them are in flight at
  // once: under per-load branches they issued one round trip at a time.
  double hub_num = 0.0, hub_den = 1.0;
  {
    const HubD& hb = hb0;
    const int hi = has_hub ? hb.i : 1, hj = has_hub ? hb.j : 1;
    const double* pf = has_hub ? (hb.tbuf ? a.ft : f) + hb.off : f;
    const double h0 = *pf, h1 = *U.at(hi - 1, hj), h2 = *U.at(hi + 1, hj);
    const double h3 = *U.at(hi, hj - 1), h4 = *U.at(hi, hj + 1);
    if (has_hub) {
      hub_num = h0;
      hub_num -= ((hb.mask & 1u) ? 0.0 : hW) * h1;
      hub_num -= ((hb.mask & 2u) ? 0.0 : hE) * h2;
      hub_num -= ((hb.mask & 4u) ? 0.0 : hS) * h3;
      hub_num -= ((hb.mask & 8u) ? 0.0 : hN) * h4;
      hub_den = -(hW + hE + hS + hN);
    }
  }
  // chunk ends: neighbours outside the block from the link directions.  The
  // gather's value is already exact for an end whose in-block neighbours are
  // the two along neighbours and whose cross neighbours live in the chunk's
  // buffer (most chunk ends); the others (leg tips, corners, points next to
  // an ownership boundary) are recomputed here, their loads in flight with
  // the gather's, and written over the gathered value after it.
  // (small chunks, latency-bound levels: issued before the gather; q >= 8,
  // throughput-bound levels: after it, keeping the gather's registers free)
  double rend[2] = {0.0, 0.0};
  bool fixe[2] = {false, false};
  auto chunk_ends = [&]() {
    const int alo = c.da > 0 ? (c.axis ? DS : DW) : (c.axis ? DN : DE);  // toward k-1
    const int ahi = alo ^ 1;                                             // toward k+1
    int ei[2], ej[2];
    unsigned skip[2];
#pragma unroll
    for (int e = 0; e < 2; e++) {
      const int k = e ? max(c.n - 1, 0) : 0;
      const int dp = k == 0 ? c.dfirst : alo;
      const int dn = k == c.n - 1 ? c.dlast : ahi;
      int i, j;
      c.ij(k, i, j);
      const bool live = !(TMG_SKIP & 16) && c.n > 0 && (e == 0 || c.n > 1);
      i = live ? i : 1;
      j = live ? j : 1;
      bool fix = dp != alo || dn != ahi;
      if (a.mode != LM_NATURAL) {
        const int i1 = c.axis ? i - 1 : i, j1 = c.axis ? j : j - 1;
        const int i2 = c.axis ? i + 1 : i, j2 = c.axis ? j : j + 1;
        fix |= (owns_t(a.mode, a.nx, a.ny, i1, j1) != (c.tb != 0)) & (i1 > 0) & (j1 > 0) |
               (owns_t(a.mode, a.nx, a.ny, i2, j2) != (c.tb != 0)) & (i2 < a.nx) & (j2 < a.ny);
      }
      ei[e] = i;
      ej[e] = j;
      skip[e] = (dp < 4 ? 1u << dp : 0u) | (dn < 4 ? 1u << dn : 0u);
      fixe[e] = live && fix;
    }
    // all loads of both ends first, then the arithmetic
    double v[2][9];
#pragma unroll
    for (int e = 0; e < 2; e++) {
      const int i = ei[e], j = ej[e];
      v[e][0] = *F.at(i, j);
      v[e][1] = *U.at(i - 1, j);
      v[e][2] = *U.at(i + 1, j);
      v[e][3] = *U.at(i, j - 1);
      v[e][4] = *U.at(i, j + 1);
      v[e][5] = __ldg(a.W + i);
      v[e][6] = __ldg(a.E + i);
      v[e][7] = __ldg(a.S + j);
      v[e][8] = __ldg(a.N + j);
    }
#pragma unroll
    for (int e = 0; e < 2; e++) {
      double r = v[e][0];
      r -= ((skip[e] & 1u) ? 0.0 : v[e][5]) * v[e][1];
      r -= ((skip[e] & 2u) ? 0.0 : v[e][6]) * v[e][2];
      r -= ((skip[e] & 4u) ? 0.0 : v[e][7]) * v[e][3];
      r -= ((skip[e] & 8u) ? 0.0 : v[e][8]) * v[e][4];
      rend[e] = r;
    }
  };
  if constexpr (Q <= 4) chunk_ends();
  TMG_T(8);
  const int lane = tid & 31, wbase = tid & ~31;
  constexpr int PER = 32 / Q;  // chunks covered by one warp-wide pass
  constexpr int BATCH = Q < TMG_BATCH ? Q : TMG_BATCH;
  const int ksub = lane % Q, csub = lane / Q;
  constexpr unsigned FULL = 0xffffffffu;

  // ---------------- phase A: coalesced gather --------------------------------
  // Warp-local: the warp streams the points of its own 32 chunks, lanes
  // consecutive along each chunk, all loads of a batch in flight together.
  // Each point stages its frozen right-hand side (interior points subtract
  // the two cross neighbours; chunk ends are redone below with their exact
  // in-block neighbour sets) and its two along couplings.
  // Per-chunk gather records, read with broadcast LDS by the 32/Q lanes that
  // stream the chunk; they live in the reduced-row region (free until the
  // elimination is done) and are only read inside the owning warp.  The
  // coefficient arrays W, E, S, N are one allocation, so a chunk's along
  // couplings are addressed by element offsets from W.
  // A warp whose chunks are one straight run of full chunks (the bulk of
  // every long leg) addresses its points arithmetically: lane l of pass m
  // takes point p = 32 m + l of the run, which is point l % Q of chunk
  // m * 32/Q + l / Q -- the same slots as the record-driven path below.
  const int pa_rel = (int)(c.pa - a.W) + c.a0, pc_rel = (int)(c.pc - a.W) + c.a0;
  bool uniform;
  {
    const int off_p = __shfl_up_sync(FULL, c.off, 1), str_p = __shfl_up_sync(FULL, c.stride, 1);
    const int tb_p = __shfl_up_sync(FULL, c.tb, 1), cid_p = __shfl_up_sync(FULL, c.cidx, 1);
    const bool contig = c.n == Q && (lane == 0 || (str_p == c.stride && off_p + Q * str_p == c.off &&
                                                   tb_p == c.tb && cid_p == c.cidx));
    uniform = __all_sync(FULL, contig);
  }
  if (uniform) {
    const int off0 = __shfl_sync(FULL, c.off, 0), str0 = __shfl_sync(FULL, c.stride, 0);
    const int cs0 = __shfl_sync(FULL, c.cs, 0), tb0 = __shfl_sync(FULL, c.tb, 0);
    const int pa0 = __shfl_sync(FULL, pa_rel, 0), pc0 = __shfl_sync(FULL, pc_rel, 0);
    const int da0 = __shfl_sync(FULL, c.da, 0);
    const double xl0 = __shfl_sync(FULL, xlv, 0), xh0 = __shfl_sync(FULL, xhv, 0);
    const double* ub = tb0 ? a.ut : u;
    const double* fb = tb0 ? a.ft : f;
#pragma unroll
    for (int m0 = 0; m0 < Q; m0 += BATCH) {
      double vf[BATCH], vl[BATCH], vh[BATCH], va[BATCH], vc[BATCH];
#pragma unroll
      for (int b = 0; b < BATCH; b++) {
        const int p = 32 * (m0 + b) + lane;
        const int o = off0 + p * str0;
        SWEEP_CHECK(o - cs0 >= 0 && o + cs0 < (a.nx + 1) * (a.ny + 1), "uniform gather offset");
        vf[b] = fb[o];
        vl[b] = ub[o - cs0];
        vh[b] = ub[o + cs0];
        if (TMG_STAGE_ALONG) {
          va[b] = __ldg(a.W + pa0 + p * da0);
          vc[b] = __ldg(a.W + pc0 + p * da0);
        }
      }
#pragma unroll
      for (int b = 0; b < BATCH; b++) {
        const int sl = sw<Q>(wbase + (m0 + b) * PER + csub, ksub);
        R[sl] = fma(-xh0, vh[b], fma(-xl0, vl[b], vf[b]));
        if (TMG_STAGE_ALONG) {
          PA[sl] = va[b];
          PC[sl] = vc[b];
        }
      }
    }
  } else {
    int4* recI = reinterpret_cast<int4*>(sA);
    int4* recJ = recI + T;
    double2* recX = reinterpret_cast<double2*>(recJ + T);
    recI[tid] = make_int4(c.off, c.stride, c.cs, c.n | (c.tb << 8));
    recJ[tid] = make_int4(pa_rel, pc_rel, c.da, 0);
    recX[tid] = make_double2(xlv, xhv);
  __syncwarp();
  {
    const int4* recI = reinterpret_cast<const int4*>(sA);
    const int4* recJ = recI + T;
    const double2* recX = reinterpret_cast<const double2*>(recJ + T);
#pragma unroll
    for (int m0 = 0; m0 < Q; m0 += BATCH) {
      double vf[BATCH], vl[BATCH], vh[BATCH], va[BATCH], vc[BATCH];
      int slot[BATCH];
#pragma unroll
      for (int b = 0; b < BATCH; b++) {
        const int src = wbase + (m0 + b) * PER + csub;
        const int4 ri = recI[src];
        const int4 rj = recJ[src];
        const bool tb_s = (ri.w >> 8) & 1;
        const double* ub = tb_s ? a.ut : u;
        const double* fb = tb_s ? a.ft : f;
        const int o = ri.x + ksub * ri.y;
        SWEEP_CHECK(ksub >= (ri.w & 255) || (o - ri.z >= 0 && o + ri.z < (a.nx + 1) * (a.ny + 1)),
                    "record gather offset");
        const int ai = ksub * rj.z;
        slot[b] = ksub < (ri.w & 255) ? sw<Q>(src, ksub) : -1;
        if (slot[b] >= 0) {
          vf[b] = fb[o];
          vl[b] = ub[o - ri.z];
          vh[b] = ub[o + ri.z];
          if (TMG_STAGE_ALONG) {
            va[b] = __ldg(a.W + rj.x + ai);
            vc[b] = __ldg(a.W + rj.y + ai);
          }
        }
      }
#pragma unroll
      for (int b = 0; b < BATCH; b++) {
        const double2 rx = recX[wbase + (m0 + b) * PER + csub];
        if (slot[b] >= 0) {
          R[slot[b]] = fma(-rx.y, vh[b], fma(-rx.x, vl[b], vf[b]));
          if (TMG_STAGE_ALONG) {
            PA[slot[b]] = va[b];
            PC[slot[b]] = vc[b];
          }
        }
      }
    }
  }
  }  // record-driven gather
  __syncwarp();
  TMG_T(9);
  if constexpr (Q > 4) chunk_ends();
  if (fixe[0]) R[sw<Q>(tid, 0)] = rend[0];
  if (fixe[1]) R[sw<Q>(tid, c.n - 1)] = rend[1];
  __syncwarp();
  TMG_T(1);

  // ---------------- phase B: chunk elimination -------------------------------
  // Down sweep (Thomas forward elimination over the chunk interior, the
  // coupling to the previous chunk's end kept as a column) and an affine back
  // pass: x_k = alpha_k + beta_k * Xleft + gamma_k * X.
  const int nI = c.n - 1;  // interior points (all but the chunk end)
  double lam[Q], ivr[Q];
  double ad = 0.0, bd = 1.0, gd = 0.0;  // x_{e-1} = ad + bd*Xleft + gd*X
  double au = 0.0, bu = 0.0, gu = 1.0;  // x_s     = au + bu*Xleft + gu*X
  bool bad = false;
  const double csum = xlv + xhv;
#if TMG_STAGE_ALONG
  const Along<Q> cpl{PA, PC, tid};
#else
  const Along<Q> cpl{a.W + pa_rel, a.W + pc_rel, c.da};
#endif
  double a_first = 0.0;
  if (c.n > 0) {
    int i0, j0;
    c.ij(0, i0, j0);
    a_first = C.dir(c.dfirst, i0, j0);
  }
  if constexpr (Q > 1 && !(TMG_SKIP & 1)) {
    // full chunks (all but the last chunk of a leg) take the predicate-free path
    if (nI > 0)
      chunk_eliminate<Q, 0>(tid, nI, R, cpl, csum, a_first, lam, ivr, bad, ad, bd, gd, au, bu, gu);
  }
  TMG_T(2);
  // publish the first-point affine form for the left neighbour chunk
  constexpr bool xcta = XCTA;  // some leg of every bin of this launch crosses a CTA boundary
  __syncthreads();  // every warp is done with its gather records (same region)
  sA[tid] = au;
  sB[tid] = bu;
  sC[tid] = gu;
  if (CLUSTER && xcta) bin_sync<CLUSTER>();
  else __syncthreads();

  // reduced row of the chunk end
  double A = 0.0, B = 1.0, Cc = 0.0, D = 0.0, H = 0.0;
  if (c.n > 0) {
    int ie, je;
    c.ij(nI, ie, je);
    const int sl = sw<Q>(tid, nI);
    const double pav = cpl.a(nI), pcv = cpl.c(nI);
    const double ae = nI > 0 ? pav : a_first;
    const double ce = C.dir(c.dlast, ie, je);
    A = ae * bd;
    B = -(pav + pcv + csum) + ae * gd;
    D = R[sl] - ae * ad;
    if (c.link & kLinkRightNext) {
      double an, bn, gn;
      if (CLUSTER && tid == T - 1) {  // the next chunk opens the next CTA
        SWEEP_CHECK(rank + 1 < cs_size, "DSMEM rank");
        an = remote<CLUSTER>(sA, rank + 1)[0];
        bn = remote<CLUSTER>(sB, rank + 1)[0];
        gn = remote<CLUSTER>(sC, rank + 1)[0];
      } else {
        an = sA[tid + 1];
        bn = sB[tid + 1];
        gn = sC[tid + 1];
      }
      B = fma(ce, bn, B);
      Cc = ce * gn;
      D = fma(-ce, an, D);
    } else if (c.link & kLinkRightHub) {
      H += ce;
    }
    if (c.link & kLinkLeftHub) H += A;
    if (!(c.link & kLinkLeftPrev)) A = 0.0;
  }

  // parallel cyclic reduction of the per-leg reduced systems.  Legs never
  // straddle CTAs; when no leg of the bin straddles a warp either, the
  // exchange runs on warp shuffles without block barriers.
  const int steps = (TMG_SKIP & 2) ? 0 : bd_.pcr_steps;
  if (bd_.warp_local == 1) {
    for (int st = 0; st < steps; st++) {
      const int d = 1 << st;
      double Am = __shfl_up_sync(FULL, A, d), Bm = __shfl_up_sync(FULL, B, d);
      double Cm = __shfl_up_sync(FULL, Cc, d), Dm = __shfl_up_sync(FULL, D, d);
      double Hm = __shfl_up_sync(FULL, H, d);
      double Ap = __shfl_down_sync(FULL, A, d), Bp = __shfl_down_sync(FULL, B, d);
      double Cp = __shfl_down_sync(FULL, Cc, d), Dp = __shfl_down_sync(FULL, D, d);
      double Hp = __shfl_down_sync(FULL, H, d);
      if (lane < d) { Am = 0.0; Bm = 1.0; Cm = 0.0; Dm = 0.0; Hm = 0.0; }
      if (lane + d > 31) { Ap = 0.0; Bp = 1.0; Cp = 0.0; Dp = 0.0; Hp = 0.0; }
      const double k1 = A * drcp(Bm), k2 = Cc * drcp(Bp);
      A = -k1 * Am;
      B = B - k1 * Cm - k2 * Ap;
      D = D - k1 * Dm - k2 * Dp;
      H = H - k1 * Hm - k2 * Hp;
      Cc = -k2 * Cp;
    }
  } else if (CLUSTER && xcta && steps > 0) {
    // some leg runs across CTAs of the cluster: the same reduction over the
    // cluster's virtual thread index, neighbours read through DSMEM
    const int vt = rank * T + tid, vtot = cs_size * T;
    bin_sync<CLUSTER>();
    sA[tid] = A; sB[tid] = B; sC[tid] = Cc; sD[tid] = D; sH[tid] = H;
    bin_sync<CLUSTER>();
    for (int st = 0; st < steps; st++) {
      const int d = 1 << st;
      double Am = 0, Bm = 1, Cm = 0, Dm = 0, Hm = 0, Ap = 0, Bp = 1, Cp = 0, Dp = 0, Hp = 0;
      if (vt - d >= 0) {
        const int r = (vt - d) / T, l = (vt - d) % T;
        Am = remote<CLUSTER>(sA, r)[l]; Bm = remote<CLUSTER>(sB, r)[l];
        Cm = remote<CLUSTER>(sC, r)[l]; Dm = remote<CLUSTER>(sD, r)[l];
        Hm = remote<CLUSTER>(sH, r)[l];
      }
      if (vt + d < vtot) {
        const int r = (vt + d) / T, l = (vt + d) % T;
        Ap = remote<CLUSTER>(sA, r)[l]; Bp = remote<CLUSTER>(sB, r)[l];
        Cp = remote<CLUSTER>(sC, r)[l]; Dp = remote<CLUSTER>(sD, r)[l];
        Hp = remote<CLUSTER>(sH, r)[l];
      }
      bin_sync<CLUSTER>();
      const double k1 = A * drcp(Bm), k2 = Cc * drcp(Bp);
      A = -k1 * Am;
      Cc = -k2 * Cp;
      B = B - k1 * Cm - k2 * Ap;
      D = D - k1 * Dm - k2 * Dp;
      H = H - k1 * Hm - k2 * Hp;
      sA[tid] = A; sB[tid] = B; sC[tid] = Cc; sD[tid] = D; sH[tid] = H;
      bin_sync<CLUSTER>();
    }
  } else if (steps > 0) {
    __syncthreads();  // sA..sC held the first-point triples
    sA[tid] = A; sB[tid] = B; sC[tid] = Cc; sD[tid] = D; sH[tid] = H;
    __syncthreads();
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
      const double k1 = A * drcp(Bm), k2 = Cc * drcp(Bp);
      A = -k1 * Am;
      Cc = -k2 * Cp;
      B = B - k1 * Cm - k2 * Ap;
      D = D - k1 * Dm - k2 * Dp;
      H = H - k1 * Hm - k2 * Hp;
      sA[tid] = A; sB[tid] = B; sC[tid] = Cc; sD[tid] = D; sH[tid] = H;
      __syncthreads();
    }
  }
  bad |= (c.n > 0) && bad_pivot(B);
  const double iB = drcp(B);
  const double P = D * iB, Qh = H * iB;  // X_t = P - Qh * x_hub
  sD[tid] = P;
  sH[tid] = Qh;
  TMG_T(3);
  bin_sync<CLUSTER>();

  // hub rows
  if (has_hub) {
    // q >= 8: the descriptor again (L1) rather than 6 registers held throughout
    const HubD hb = Q <= 4 ? hb0 : hubs[bd_.hub0 + c.own];
    const int o = hb.off;
    double num = hub_num, den = hub_den;
    // couplings to the adjacent chunk ends, all four loads in flight at once
    double hcf[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int d = hb.adj_d[q];
      const double* p = d == DW ? a.W + hb.i : d == DE ? a.E + hb.i : d == DS ? a.S + hb.j
                                                                              : a.N + hb.j;
      hcf[q] = __ldg(p);
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      if (q >= hb.nadj) break;
      const int ta = hb.adj_t[q];
      SWEEP_CHECK(ta >= 0 && ta < T * cs_size && hb.off >= 0 &&
                      hb.off < (a.nx + 1) * (a.ny + 1),
                  "hub coupling");
      const double cf = hcf[q];
      num -= cf * remote<CLUSTER>(sD, ta / T)[ta % T];
      den -= cf * remote<CLUSTER>(sH, ta / T)[ta % T];
    }
    bad |= bad_pivot(den);
    const double xh = num / den;
    XH[tid] = xh;
    if (!(hb.pad & 1)) (hb.tbuf ? a.ut : u)[o] = xh;  // one copy stores the hub
  }
  __syncthreads();  // every CTA holding chunks of a block solves its own hub copy

  TMG_T(4);
  // final values of the chunk
  if (!(TMG_SKIP & 8) && c.n > 0) {
    const double xh = c.hub >= 0 ? XH[c.hub % T] : 0.0;
    const double X = fma(-Qh, xh, P);
    double Lv = 0.0;
    if (c.link & kLinkLeftPrev) {
      if (CLUSTER && tid == 0) {  // the previous chunk ends the previous CTA
        Lv = fma(-remote<CLUSTER>(sH, rank - 1)[T - 1], xh, remote<CLUSTER>(sD, rank - 1)[T - 1]);
      } else {
        Lv = fma(-sH[tid - 1], xh, sD[tid - 1]);
      }
    } else if (c.link & kLinkLeftHub) {
      Lv = xh;
    }
#pragma unroll
    for (int k = 0; k < Q; k++)
      if (k < nI) {
        const int sl = sw<Q>(tid, k);
        R[sl] = fma(ivr[k], X, fma(lam[k], Lv, R[sl]));
      }
    R[sw<Q>(tid, nI)] = X;
  }
  if (bad) atomicOr(a.err, 1);
  TMG_T(5);
  if (TMG_PDL_LATE) pdl_trigger();  // the successor may launch while this CTA scatters
  if constexpr (CLUSTER) cluster_arrive();  // this CTA's DSMEM reads are done
  // scatter records (sA/sB are free after the reduced solve; the finalize of
  // other warps reads only sD, sH and XH)
  reinterpret_cast<int2*>(sA)[tid] = make_int2(c.off, c.stride);
  reinterpret_cast<int*>(sC)[tid] = c.n | (c.tb << 8);
  __syncwarp();

  // ---------------- phase C: coalesced scatter (warp-local) ----------------
  if (uniform) {
    const int off0 = __shfl_sync(FULL, c.off, 0), str0 = __shfl_sync(FULL, c.stride, 0);
    double* ub = __shfl_sync(FULL, c.tb, 0) ? a.ut : u;
#pragma unroll
    for (int m = 0; m < Q; m++)
      ub[off0 + (32 * m + lane) * str0] = R[sw<Q>(wbase + m * PER + csub, ksub)];
  } else {
    const int2* recO = reinterpret_cast<const int2*>(sA);
    const int* recN = reinterpret_cast<const int*>(sC);
#pragma unroll
    for (int m = 0; m < Q; m++) {
      const int src = wbase + m * PER + csub;
      const int nt = recN[src];
      if (ksub < (nt & 255)) {
        const int2 ro = recO[src];
        ((nt >> 8) ? a.ut : u)[ro.x + ksub * ro.y] = R[sw<Q>(src, ksub)];
      }
    }
  }
  TMG_T(6);
}

// One CTA (cluster) per bin.
template <bool CLUSTER, bool XCTA, int Q>
__global__ void __launch_bounds__(kThreads, Q <= 8 ? TMG_MINB8 : TMG_MINB)
block_sweep_kernel(SweepArgs a, const ChunkD* __restrict__ chunks, const BinD* __restrict__ bins,
                   const HubD* __restrict__ hubs, int cs_size) {
  extern __shared__ double smem[];
  const int rank = CLUSTER ? (int)cg::this_cluster().block_rank() : 0;
  sweep_bin<CLUSTER, XCTA, Q>(a, chunks, bins, hubs, cs_size, blockIdx.x / cs_size, rank, smem);
  if constexpr (CLUSTER) cluster_wait();
}

// ---- persistent coarse tail ------------------------------------------------
// Grid barrier of the cooperative tail launch: bar[0] counts arrivals,
// bar[1] is the generation the last arrival bumps (both return to their
// start state's form after every barrier, so graph replays reuse them).
__device__ __forceinline__ void tail_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen;
    asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    if (old == nblocks - 1) {
      asm volatile("st.relaxed.gpu.u32 [%0], 0;" ::"l"(bar) : "memory");
      asm volatile("red.release.gpu.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
    } else {
      unsigned g2;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g2) : "l"(bar + 1) : "memory");
      } while (g2 == gen);
    }
  }
  __syncthreads();
}

// (not inlined: each op body keeps its own register allocation)
template <int Q>
__device__ __noinline__ void tail_bins(const TailOp* __restrict__ opp, int b0, double* smem) {
  const TailOp& op = *opp;
  const SweepArgs sa = op.sa;
  for (int b = b0; b < op.nitems; b += gridDim.x) {
    sweep_bin<false, false, Q>(sa, op.chunks, op.bins, op.hubs, 1, b, 0, smem);
    __syncthreads();  // the next bin's gather overwrites the staged rows
  }
}

__device__ __noinline__ void tail_restrict(const TailOp* __restrict__ opp, int b0, double* smem) {
  const TailOp& op = *opp;
  for (int t = b0; t < op.nitems; t += gridDim.x) {
    const int by = t / op.gx, bx = t - by * op.gx;
    restrict3_tile(op.g, op.full, op.U, op.F, op.CF, op.CU, 1, GroupSel2{0, 0, 0}, 1 + by * R3C,
                   1 + bx * R3C, smem, smem + R3U * R3LU);
    __syncthreads();
  }
}

__device__ __noinline__ void tail_prolong(const TailOp* __restrict__ opp, int b0, double* smem) {
  const TailOp& op = *opp;
  for (int t = b0; t < op.nitems; t += gridDim.x) {
    const int by = t / op.gx, bx = t - by * op.gx;
    prolong2_tile(op.g.nx, op.g.ny, op.CU, op.U, GroupSel2{0, 0, 0}, 1 + by * NT, 1 + bx * NT,
                  smem);
    __syncthreads();
  }
}

#ifdef TMG_TAIL_TIMING
__device__ unsigned long long g_tail_t[2][4096];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

// One CTA per SM at most; every CTA walks the whole op list.
__global__ void __launch_bounds__(kThreads, 1)
tail_kernel(const TailOp* __restrict__ ops, int nops, unsigned* bar) {
  extern __shared__ double smem[];
  const int G = gridDim.x;
  for (int k = 0; k < nops; k++) {
    const TailOp& op = ops[k];
    int b0 = ((int)blockIdx.x - op.base) % G;
    if (b0 < 0) b0 += G;
#ifdef TMG_TAIL_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0 && k < 4096) g_tail_t[0][k] = gtimer();
#endif
    switch (op.type) {
      case TAIL_SWEEP:
        switch (op.q) {
          case 16: tail_bins<16>(ops + k, b0, smem); break;
          case 8: tail_bins<8>(ops + k, b0, smem); break;
          case 4: tail_bins<4>(ops + k, b0, smem); break;
          case 2: tail_bins<2>(ops + k, b0, smem); break;
          default: tail_bins<1>(ops + k, b0, smem); break;
        }
        break;
      case TAIL_RESTRICT: tail_restrict(ops + k, b0, smem); break;
      case TAIL_PROLONG: tail_prolong(ops + k, b0, smem); break;
      case TAIL_DENSE_RHS:
        dense_rhs(op.g, op.U, op.F, op.work, b0 * kThreads + threadIdx.x, G * kThreads);
        break;
      case TAIL_DENSE_APPLY:
        for (int w = b0 * (kThreads / 32) + (threadIdx.x >> 5); w < op.nitems;
             w += G * (kThreads / 32))
          dense_apply(op.g, op.ainv, op.work, op.U, w, threadIdx.x & 31);
        break;
      default: break;
    }
#ifdef TMG_TAIL_TIMING
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0 && k < 4096) g_tail_t[1][k] = gtimer();
#endif
    if (op.barrier) tail_barrier(bar, G);
  }
}

extern "C" int tmg_debug_tail_times(unsigned long long* out, int n) {
#ifdef TMG_TAIL_TIMING
  if (n > 4096) n = 4096;
  cudaMemcpyFromSymbol(out, g_tail_t, sizeof(unsigned long long) * 2 * 4096);
  return n;
#else
  (void)out;
  (void)n;
  return 0;
#endif
}

// Point Gauss-Seidel colour stage for checkerboard (smoothers.py:65-75,
// _ckernels.pyx:42-51): red = (i + j) even.
// Rows i in [i0, i0 + gridDim.y) (a partial plan covers its sharding groups).
__global__ void __launch_bounds__(256) point_sweep_kernel(SweepArgs a, int nx, int ny, int red,
                                                          int i0) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int i = blockIdx.y + i0;
  pdl_trigger();
  pdl_wait();
  if (j >= ny || i >= nx) return;
  if ((((i + j) & 1) == 0) != (red != 0)) return;
  const size_t ld = (size_t)a.ld, o = (size_t)i * ld + j;
  const double Wi = __ldg(a.W + i), Ei = __ldg(a.E + i), Sj = __ldg(a.S + j), Nj = __ldg(a.N + j);
  const double b = -(Wi + Ei + Sj + Nj);
  const double r = a.f[o] - Wi * a.u[o - ld] - Ei * a.u[o + ld] - Sj * a.u[o - 1] - Nj * a.u[o + 1];
  a.u[o] = r / b;
}

namespace {
// TMG_SMEM_PAD (bytes, profiling only) inflates the dynamic shared memory
// per CTA to study the kernel at lower residency
size_t smem_pad() {
  static long pad = -1;
  if (pad < 0) {
    const char* s = std::getenv("TMG_SMEM_PAD");
    pad = s ? std::atol(s) : 0;
    if (pad < 0) pad = 0;
  }
  return (size_t)pad;
}

template <int Q>
size_t smem_bytes() {
  return sweep_smem<Q>() + smem_pad();
}

template <int Q>
cudaError_t set_attrs() {
  const int sm = (int)smem_bytes<Q>();
  cudaError_t e = cudaFuncSetAttribute(block_sweep_kernel<false, false, Q>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(block_sweep_kernel<true, false, Q>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(block_sweep_kernel<true, true, Q>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  if (e == cudaSuccess)  // clusters of 16 CTAs (rings of wireframe grids >= 8193^2)
    e = cudaFuncSetAttribute(block_sweep_kernel<true, false, Q>,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(block_sweep_kernel<true, true, Q>,
                             cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}

template <int Q>
cudaError_t launch_class(const LaunchClass& lc, const SweepArgs& a, cudaStream_t stream) {
  const int grid = lc.nbins;
  if (lc.cs == 1) {
    TMG_COUNT(1);
    return launch_pdl(block_sweep_kernel<false, false, Q>, dim3(grid), dim3(kThreads),
                      smem_bytes<Q>(), stream, a, (const ChunkD*)lc.chunks, (const BinD*)lc.bins,
                      (const HubD*)lc.hubs, 1);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid * lc.cs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes<Q>();
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = lc.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  TMG_COUNT(1);
  if (lc.xcta)
    return cudaLaunchKernelEx(&cfg, block_sweep_kernel<true, true, Q>, a,
                              (const ChunkD*)lc.chunks, (const BinD*)lc.bins,
                              (const HubD*)lc.hubs, lc.cs);
  return cudaLaunchKernelEx(&cfg, block_sweep_kernel<true, false, Q>, a, (const ChunkD*)lc.chunks,
                            (const BinD*)lc.bins, (const HubD*)lc.hubs, lc.cs);
}
}  // namespace

// Average per-CTA cycles between the phase marks of the last launches
// (debug builds with -DTMG_PHASE_TIMING; zeros otherwise).
// gather sub-phases: descriptor load + unpack + PDL wait, hub preload, main
// gather, chunk-end fix (same builds)
extern "C" int tmg_debug_gather_cycles(double* out4) {
  for (int k = 0; k < 4; k++) out4[k] = 0.0;
#ifdef TMG_PHASE_TIMING
  int n = 0;
  cudaMemcpyFromSymbol(&n, g_phase_n, sizeof(int));
  if (n <= 0) return 0;
  std::vector<long long> t(12 * (size_t)(1 << 16));
  cudaMemcpyFromSymbol(t.data(), g_phase_t, t.size() * sizeof(long long));
  const int from[4] = {0, 7, 8, 9}, to[4] = {7, 8, 9, 1};
  for (int b = 0; b < n; b++)
    for (int k = 0; k < 4; k++)
      out4[k] += (double)(t[(size_t)to[k] * (1 << 16) + b] - t[(size_t)from[k] * (1 << 16) + b]);
  for (int k = 0; k < 4; k++) out4[k] /= n;
  return n;
#else
  return 0;
#endif
}

extern "C" int tmg_debug_phase_cycles(double* out6) {
  for (int k = 0; k < 6; k++) out6[k] = 0.0;
#ifdef TMG_PHASE_TIMING
  int n = 0;
  cudaMemcpyFromSymbol(&n, g_phase_n, sizeof(int));
  if (n <= 0) return 0;
  std::vector<long long> t(8 * (size_t)(1 << 16));
  cudaMemcpyFromSymbol(t.data(), g_phase_t, t.size() * sizeof(long long));
  for (int b = 0; b < n; b++)
    for (int k = 0; k < 6; k++) out6[k] += (double)(t[(size_t)(k + 1) * (1 << 16) + b] - t[(size_t)k * (1 << 16) + b]);
  for (int k = 0; k < 6; k++) out6[k] /= n;
  int z = 0;
  cudaMemcpyToSymbol(g_phase_n, &z, sizeof(int));
  return n;
#else
  return 0;
#endif
}

cudaError_t init_sweep_kernels() {
  static cudaError_t done = cudaErrorNotReady;
  if (done == cudaErrorNotReady) {
    done = set_attrs<16>();
    if (done == cudaSuccess) done = set_attrs<8>();
    if (done == cudaSuccess) done = set_attrs<4>();
    if (done == cudaSuccess) done = set_attrs<2>();
    if (done == cudaSuccess) done = set_attrs<1>();
  }
  return done;
}

cudaError_t tail_prepare(int qmax, size_t* smem, int* max_ctas) {
  size_t sm = sizeof(double) * (size_t)(R3U * R3LU + R3D * R3LD);
  const size_t sw = qmax >= 16 ? sweep_smem<16>() : qmax >= 8 ? sweep_smem<8>()
                  : qmax >= 4 ? sweep_smem<4>() : qmax >= 2 ? sweep_smem<2>() : sweep_smem<1>();
  sm = std::max(sm, sw);
  *smem = sm;
  *max_ctas = 0;
  cudaError_t e = cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sm);
  if (e != cudaSuccess) return e;
  int per_sm = 0, dev = 0, sms = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tail_kernel, kThreads, sm);
  if (e == cudaSuccess) e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  *max_ctas = per_sm * sms;
  return cudaSuccess;
}

cudaError_t launch_tail(const TailOp* ops, int nops, int ctas, size_t smem, unsigned* bar,
                        cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barriers)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TMG_COUNT(1);
  return cudaLaunchKernelEx(&cfg, tail_kernel, ops, nops, bar);
}

cudaError_t launch_colour(const Plan& P, int red, const SweepArgs& a, cudaStream_t stream) {
  if (P.point_scheme) {
    const int i0 = P.g0 > 0 ? P.g0 : 1, i1 = P.g0 > 0 ? P.g1 : P.geo.nx;
    dim3 grid((P.geo.ny - 1 + 255) / 256, i1 - i0);
    TMG_COUNT(1);
    return launch_pdl(point_sweep_kernel, grid, dim3(256), 0, stream, a, P.geo.nx, P.geo.ny, red,
                      i0);
  }
  for (const LaunchClass& lc : P.classes) {
    if (lc.red != red || lc.nbins == 0) continue;
    cudaError_t e;
    switch (lc.q) {
      case 16: e = launch_class<16>(lc, a, stream); break;
      case 8: e = launch_class<8>(lc, a, stream); break;
      case 4: e = launch_class<4>(lc, a, stream); break;
      case 2: e = launch_class<2>(lc, a, stream); break;
      default: e = launch_class<1>(lc, a, stream); break;
    }
    if (e != cudaSuccess) return e;
  }
  if (P.lp) return launch_leg_colour(*P.lp, red, a, stream);
  return cudaSuccess;
}

}  // namespace tmg
