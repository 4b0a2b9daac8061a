// Grid kernels on the hybrid N/T field layout (tmg_layout.h) used inside the
// V-cycle: residual max-norm, fused residual + restriction, fused bilinear
// prolongation + correction, coarse dense solve, and the conversions between
// the reference's C-order arrays and the hybrid layout.
//
// Every kernel walks 32 x 32 tiles.  A tile whose points all live in one
// buffer is walked with lanes along that buffer's contiguous axis (coalesced
// in both the N and the T regions); the few tiles straddling an ownership
// boundary address point by point.  Arithmetic is the reference's order
// (stencil.py:82-87, transfer.py:33-38, 51-53) with explicit round-to-nearest
// intrinsics, so results are bit-identical to the natural-layout kernels.
#include <cstdlib>
#include <cstring>

#include "tmg_kernels.h"
#include "tmg_transfer_dev.cuh"

namespace tmg {

namespace {

constexpr int TILE = 32;

// range of the mirrored index m(i) = min(i, n - i) over [a, b] (concave:
// the minimum sits at an end, the maximum at n/2 when the range covers it)
__device__ __forceinline__ void mirror_range(int a, int b, int n, int& lo, int& hi) {
  const int ma = min(a, n - a), mb = min(b, n - b);
  lo = min(ma, mb);
  hi = (a <= n / 2 && n / 2 <= b) ? n / 2 : max(ma, mb);
}

// Owner of the tile [i0, i0+ni) x [j0, j0+nj): 1 if every interior point is
// T-owned, 0 if every one is N-owned, -1 if mixed.  Ownership compares i'
// with j' (tmg_layout.h), and max over the tile of (i' - j') separates into
// max i' - min j', so the test is exact.  Ring points are readable through
// both buffers and do not count.
__device__ __forceinline__ int tile_owner_exact(const FieldView& v, int i0, int j0, int ni, int nj) {
  if (v.mode == LM_NATURAL) return 0;
  const int ia = max(i0, 1), ib = min(i0 + ni - 1, v.nx - 1);
  const int ja = max(j0, 1), jb = min(j0 + nj - 1, v.ny - 1);
  if (ia > ib || ja > jb) return 0;
  if (v.mode == LM_XLINES) return 1;
  int ilo, ihi, jlo, jhi;
  mirror_range(ia, ib, v.nx, ilo, ihi);
  mirror_range(ja, jb, v.ny, jlo, jhi);
  if (v.mode == LM_TWEED) {  // T iff i' < j'
    if (ihi < jlo) return 1;
    if (ilo >= jhi) return 0;
    return -1;
  }
  // LM_WIRE: T iff j' < i'
  if (jhi < ilo) return 1;
  if (jlo >= ihi) return 0;
  return -1;
}

// (L u)(i, j) in the reference's order with per-point addressing
__device__ __forceinline__ double lu_view(const FieldView& U, int i, int j, double Wi, double Ei,
                                          double Sj, double Nj) {
  const double Cc = -__dadd_rn(__dadd_rn(__dadd_rn(Wi, Ei), Sj), Nj);
  double acc = __dmul_rn(Wi, *U.at(i - 1, j));
  acc = __dadd_rn(acc, __dmul_rn(Ei, *U.at(i + 1, j)));
  acc = __dadd_rn(acc, __dmul_rn(Sj, *U.at(i, j - 1)));
  acc = __dadd_rn(acc, __dmul_rn(Nj, *U.at(i, j + 1)));
  return __dadd_rn(acc, __dmul_rn(Cc, *U.at(i, j)));
}

// same with fixed strides inside one buffer (uniform tiles): o = offset of
// (i, j) in `b`, si / sj = element steps of i / j in that buffer
__device__ __forceinline__ double lu_strided(const double* __restrict__ b, size_t o, int si, int sj,
                                             double Wi, double Ei, double Sj, double Nj) {
  const double Cc = -__dadd_rn(__dadd_rn(__dadd_rn(Wi, Ei), Sj), Nj);
  double acc = __dmul_rn(Wi, b[o - si]);
  acc = __dadd_rn(acc, __dmul_rn(Ei, b[o + si]));
  acc = __dadd_rn(acc, __dmul_rn(Sj, b[o - sj]));
  acc = __dadd_rn(acc, __dmul_rn(Nj, b[o + sj]));
  return __dadd_rn(acc, __dmul_rn(Cc, b[o]));
}

// Residual max-norm over the interior; one 32x32 tile per CTA (256 threads,
// 4 points per thread), lanes along the owning buffer's contiguous axis.
// With gsel.g0 > 0 only points of sharding groups [g0, g1) count (one rank's
// share in a sharded solve; the ranks then all-reduce the maximum).
struct GroupSel {
  int scheme, g0, g1;
};

__global__ void __launch_bounds__(256) hdefect_norm_kernel(GridArgs g, FieldView U, FieldView F,
                                                           unsigned long long* dmax, GroupSel gsel) {
  const int i0 = 1 + blockIdx.y * TILE, j0 = 1 + blockIdx.x * TILE;
  const int ni = min(TILE, g.nx - i0), nj = min(TILE, g.ny - j0);
  const int own = tile_owner_exact(U, i0 - 1, j0 - 1, ni + 2, nj + 2);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long m = 0ull;
  for (int r = w; r < TILE; r += 8) {
    // along = contiguous axis of the owner, cross = the other one
    const int a = lane, b = r;
    const int i = own == 1 ? i0 + a : i0 + b;
    const int j = own == 1 ? j0 + b : j0 + a;
    if (i >= g.nx || j >= g.ny) continue;
    if (gsel.g0 > 0) {
      const int grp = point_group(gsel.scheme, g.nx, g.ny, i, j);
      if (grp < gsel.g0 || grp >= gsel.g1) continue;
    }
    const double Wi = __ldg(g.W + i), Ei = __ldg(g.E + i), Sj = __ldg(g.S + j), Nj = __ldg(g.N + j);
    double lu, fv;
    if (own == 1) {
      const size_t o = U.off_t(i, j);
      lu = lu_strided(U.t, o, 1, g.nx + 1, Wi, Ei, Sj, Nj);
      fv = F.t[o];
    } else if (own == 0) {
      const size_t o = U.off_n(i, j);
      lu = lu_strided(U.n, o, g.ny + 1, 1, Wi, Ei, Sj, Nj);
      fv = F.n[o];
    } else {
      lu = lu_view(U, i, j, Wi, Ei, Sj, Nj);
      fv = *F.at(i, j);
    }
    const double d = fabs(__dadd_rn(-lu, fv));
    const unsigned long long bits = (unsigned long long)__double_as_longlong(d);
    m = bits > m ? bits : m;
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, m, s);
    m = o2 > m ? o2 : m;
  }
  if (lane == 0 && m) atomicMax(dmax, m);
}

__device__ __forceinline__ double restrict_smem(const double* d, int o, int ld, int full) {
  const double ctr = d[o];
  const double edges = __dadd_rn(__dadd_rn(__dadd_rn(d[o - ld], d[o + ld]), d[o - 1]), d[o + 1]);
  if (!full) return __dadd_rn(__dmul_rn(0.5, ctr), __dmul_rn(0.125, edges));
  const double diags = __dadd_rn(__dadd_rn(__dadd_rn(d[o - ld - 1], d[o + ld - 1]), d[o - ld + 1]),
                                 d[o + ld + 1]);
  return __dadd_rn(__dadd_rn(__dmul_rn(0.25, ctr), __dmul_rn(0.125, edges)),
                   __dmul_rn(0.0625, diags));
}

// Fused residual + restriction: coarse tile 16 x 16 (I x J) per CTA; the fine
// defect on (2*16+1)^2 points is computed into shared memory from a u tile
// with a one-point halo, then restricted.  Shared arrays are indexed
// [i][j]; loads walk the owner's contiguous axis.
constexpr int CT = 16;
constexpr int FD = 2 * CT + 1;  // fine defect tile edge
constexpr int FU = 2 * CT + 3;  // fine u tile edge (with halo)

__global__ void __launch_bounds__(256) hdefect_restrict_kernel(GridArgs g, int full, FieldView U,
                                                               FieldView F, FieldView FC) {
  __shared__ double su[FU * FU];
  __shared__ double sd[FD * FD];
  const int nxc = g.nx / 2, nyc = g.ny / 2;
  const int I0 = 1 + blockIdx.y * CT, J0 = 1 + blockIdx.x * CT;
  const int ui0 = 2 * I0 - 2, uj0 = 2 * J0 - 2;
  const int own = tile_owner_exact(U, ui0, uj0, min(FU, g.nx + 1 - ui0), min(FU, g.ny + 1 - uj0));
  // u tile
  for (int t = threadIdx.x; t < FU * FU; t += blockDim.x) {
    const int p = t / FU, q = t - p * FU;  // q is the fast (lane) index
    const int a = own == 1 ? q : p, b = own == 1 ? p : q;  // a: i offset, b: j offset
    const int i = ui0 + a, j = uj0 + b;
    double v = 0.0;
    if (i <= g.nx && j <= g.ny)
      v = own == 1 ? U.t[U.off_t(i, j)] : own == 0 ? U.n[U.off_n(i, j)] : *U.at(i, j);
    su[a * FU + b] = v;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < FD * FD; t += blockDim.x) {
    const int p = t / FD, q = t - p * FD;
    const int a = own == 1 ? q : p, b = own == 1 ? p : q;
    const int i = ui0 + 1 + a, j = uj0 + 1 + b;
    double dv = 0.0;
    if (i < g.nx && j < g.ny) {
      const double lu = lu_strided(su, (size_t)(a + 1) * FU + (b + 1), FU, 1, __ldg(g.W + i),
                                   __ldg(g.E + i), __ldg(g.S + j), __ldg(g.N + j));
      const double fv = own == 1 ? F.t[F.off_t(i, j)] : own == 0 ? F.n[F.off_n(i, j)] : *F.at(i, j);
      dv = __dadd_rn(-lu, fv);
    }
    sd[a * FD + b] = dv;
  }
  __syncthreads();
  const int cown = tile_owner_exact(FC, I0, J0, min(CT, nxc - I0), min(CT, nyc - J0));
  const int p = threadIdx.x / CT, q = threadIdx.x - p * CT;
  const int a = cown == 1 ? q : p, b = cown == 1 ? p : q;
  const int I = I0 + a, J = J0 + b;
  if (I < nxc && J < nyc) {
    const double v = restrict_smem(sd, (2 * a + 1) * FD + (2 * b + 1), FD, full);
    if (cown == 1) FC.t[FC.off_t(I, J)] = v;
    else if (cown == 0) FC.n[FC.off_n(I, J)] = v;
    else *FC.at(I, J) = v;
  }
}

__device__ __forceinline__ double prolong_view(const FieldView& C, int i, int j) {
  const int I = i >> 1, J = j >> 1;
  if (!(i & 1) && !(j & 1)) return *C.at(I, J);
  if (!(i & 1)) return __dmul_rn(0.5, __dadd_rn(*C.at(I, J), *C.at(I, J + 1)));
  if (!(j & 1)) return __dmul_rn(0.5, __dadd_rn(*C.at(I, J), *C.at(I + 1, J)));
  return __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(*C.at(I, J), *C.at(I + 1, J)), *C.at(I, J + 1)),
                                   *C.at(I + 1, J + 1)));
}

// Fused prolongation + correction on a 32x32 fine tile per CTA; the coarse
// values come through L1 (each coarse point feeds up to 9 fine points).
__global__ void __launch_bounds__(256) hprolong_correct_kernel(int nx, int ny, FieldView C,
                                                               FieldView U) {
  const int i0 = 1 + blockIdx.y * TILE, j0 = 1 + blockIdx.x * TILE;
  const int ni = min(TILE, nx - i0), nj = min(TILE, ny - j0);
  const int own = tile_owner_exact(U, i0, j0, ni, nj);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int r = w; r < TILE; r += 8) {
    const int i = own == 1 ? i0 + lane : i0 + r;
    const int j = own == 1 ? j0 + r : j0 + lane;
    if (i >= nx || j >= ny) continue;
    double* p = own == 1 ? U.t + U.off_t(i, j) : own == 0 ? U.n + U.off_n(i, j) : U.at(i, j);
    *p = __dadd_rn(*p, prolong_view(C, i, j));
  }
}

// natural -> hybrid: the N buffer is a plain copy (done with cudaMemcpy by
// the caller); this writes the T buffer as the transpose of the natural array
// (all points, so T also carries the Dirichlet ring).
__global__ void __launch_bounds__(256) to_t_kernel(int nx, int ny, const double* __restrict__ nat,
                                                   double* __restrict__ t) {
  __shared__ double tile[TILE][TILE + 1];
  const int i0 = blockIdx.y * TILE, j0 = blockIdx.x * TILE;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int r = w; r < TILE; r += 8) {
    const int i = i0 + r, j = j0 + lane;
    if (i <= nx && j <= ny) tile[r][lane] = nat[(size_t)i * (ny + 1) + j];
  }
  __syncthreads();
  for (int r = w; r < TILE; r += 8) {
    const int j = j0 + r, i = i0 + lane;
    if (i <= nx && j <= ny) t[(size_t)j * (nx + 1) + i] = tile[lane][r];
  }
}

// hybrid -> natural
__global__ void __launch_bounds__(256) from_hybrid_kernel(FieldView V, double* __restrict__ nat) {
  __shared__ double tile[TILE][TILE + 1];
  const int nx = V.nx, ny = V.ny;
  const int i0 = blockIdx.y * TILE, j0 = blockIdx.x * TILE;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int r = w; r < TILE; r += 8) {  // T values, lanes along i
    const int j = j0 + r, i = i0 + lane;
    if (i <= nx && j <= ny && owns_t(V.mode, nx, ny, i, j)) tile[lane][r] = V.t[V.off_t(i, j)];
  }
  __syncthreads();
  for (int r = w; r < TILE; r += 8) {  // N values and the write, lanes along j
    const int i = i0 + r, j = j0 + lane;
    if (i <= nx && j <= ny) {
      const size_t o = (size_t)i * (ny + 1) + j;
      nat[o] = owns_t(V.mode, nx, ny, i, j) ? tile[r][lane] : V.n[o];
    }
  }
}

__global__ void hdense_rhs_kernel(GridArgs g, FieldView U, FieldView F, double* __restrict__ rhs) {
  pdl_trigger();
  pdl_wait();
  dense_rhs(g, U, F, rhs, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

__global__ void hdense_apply_kernel(GridArgs g, const double* __restrict__ Ainv,
                                    const double* __restrict__ rhs, FieldView U) {
  pdl_trigger();
  pdl_wait();
  dense_apply(g, Ainv, rhs, U, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, threadIdx.x & 31);
}

}  // namespace

bool transfer_v1() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("TMG_TRANSFER");
    v = (e && std::strcmp(e, "v1") == 0) ? 1 : 0;
  }
  return v == 1;
}

cudaError_t launch_hdefect_norm(const GridArgs& g, const FieldView& U, const FieldView& F,
                                unsigned long long* dmax, cudaStream_t s, int scheme, int g0,
                                int g1) {
  if (g.nx < 2 || g.ny < 2) return cudaSuccess;
  if (!transfer_v1()) return launch_norm2(g, U, F, dmax, s, scheme, g0, g1);
  dim3 grid((g.ny - 1 + TILE - 1) / TILE, (g.nx - 1 + TILE - 1) / TILE);
  TMG_COUNT(1);
  hdefect_norm_kernel<<<grid, 256, 0, s>>>(g, U, F, dmax, GroupSel{scheme, g0, g1});
  return cudaGetLastError();
}

namespace {
// enc = 2 * element offset + (1 if the point lives in the T buffer)
__global__ void gather_points_kernel(FieldView V, const long long* __restrict__ enc, long n,
                                     double* __restrict__ out) {
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const long long e = enc[k];
    out[k] = ((e & 1) ? V.t : V.n)[e >> 1];
  }
}
__global__ void scatter_points_kernel(FieldView V, const long long* __restrict__ enc, long n,
                                      const double* __restrict__ in) {
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
    const long long e = enc[k];
    ((e & 1) ? V.t : V.n)[e >> 1] = in[k];
  }
}
int point_blocks(long n) {
  const long b = (n + 255) / 256;
  return (int)(b < 148 * 8 ? (b > 0 ? b : 1) : 148 * 8);
}
}  // namespace

cudaError_t launch_gather_points(const FieldView& V, const long long* enc, long n, double* out,
                                 cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  TMG_COUNT(1);
  gather_points_kernel<<<point_blocks(n), 256, 0, s>>>(V, enc, n, out);
  return cudaGetLastError();
}

cudaError_t launch_scatter_points(const FieldView& V, const long long* enc, long n,
                                  const double* in, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  TMG_COUNT(1);
  scatter_points_kernel<<<point_blocks(n), 256, 0, s>>>(V, enc, n, in);
  return cudaGetLastError();
}

cudaError_t launch_hdefect_restrict(const GridArgs& g, int full, const FieldView& U,
                                    const FieldView& F, const FieldView& FC, cudaStream_t s,
                                    const FieldView* UC, bool* uc_zeroed) {
  if (uc_zeroed) *uc_zeroed = false;
  const int nxc = g.nx / 2, nyc = g.ny / 2;
  if (nxc < 2 || nyc < 2) return cudaSuccess;
  if (!transfer_v1()) {
    if (uc_zeroed) *uc_zeroed = UC != nullptr;
    return launch_restrict2(g, full, U, F, FC, s, UC);
  }
  dim3 grid((nyc - 1 + CT - 1) / CT, (nxc - 1 + CT - 1) / CT);
  TMG_COUNT(1);
  hdefect_restrict_kernel<<<grid, 256, 0, s>>>(g, full, U, F, FC);
  return cudaGetLastError();
}

cudaError_t launch_hprolong_correct(int nx, int ny, const FieldView& C, const FieldView& U,
                                    cudaStream_t s, int skip_red) {
  if (nx < 2 || ny < 2) return cudaSuccess;
  if (!transfer_v1()) return launch_prolong2(nx, ny, C, U, s, 0, 0, 0, skip_red);
  dim3 grid((ny - 1 + TILE - 1) / TILE, (nx - 1 + TILE - 1) / TILE);
  TMG_COUNT(1);
  hprolong_correct_kernel<<<grid, 256, 0, s>>>(nx, ny, C, U);
  return cudaGetLastError();
}

cudaError_t launch_to_hybrid(const FieldView& V, const double* nat, cudaStream_t s) {
  const size_t n = (size_t)(V.nx + 1) * (V.ny + 1);
  cudaError_t e = cudaMemcpyAsync(V.n, nat, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess || V.mode == LM_NATURAL) return e;
  dim3 grid((V.ny + 1 + TILE - 1) / TILE, (V.nx + 1 + TILE - 1) / TILE);
  TMG_COUNT(1);
  to_t_kernel<<<grid, 256, 0, s>>>(V.nx, V.ny, nat, V.t);
  return cudaGetLastError();
}

cudaError_t launch_from_hybrid(const FieldView& V, double* nat, cudaStream_t s) {
  if (V.mode == LM_NATURAL) {
    const size_t n = (size_t)(V.nx + 1) * (V.ny + 1);
    if (V.n == nat) return cudaSuccess;
    return cudaMemcpyAsync(nat, V.n, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
  }
  dim3 grid((V.ny + 1 + TILE - 1) / TILE, (V.nx + 1 + TILE - 1) / TILE);
  TMG_COUNT(1);
  from_hybrid_kernel<<<grid, 256, 0, s>>>(V, nat);
  return cudaGetLastError();
}

cudaError_t launch_hdense_solve(const GridArgs& g, const double* Ainv, const FieldView& U,
                                const FieldView& F, double* work, cudaStream_t s) {
  const int n = (g.nx - 1) * (g.ny - 1);
  if (n <= 0) return cudaSuccess;
  TMG_COUNT(1);
  cudaError_t e = launch_pdl(hdense_rhs_kernel, dim3((n + 255) / 256), dim3(256), 0, s, g, U, F,
                             work);
  if (e != cudaSuccess) return e;
  TMG_COUNT(1);
  e = launch_pdl(hdense_apply_kernel, dim3((n * 32 + 255) / 256), dim3(256), 0, s, g, Ainv,
                 (const double*)work, U);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace tmg
