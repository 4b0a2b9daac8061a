// Grid kernels: residual, residual max-norm, fused residual + restriction,
// restriction, prolongation (+ correction), coarse dense solve.
//
// The residual and transfers use explicit round-to-nearest intrinsics in the
// reference's numpy evaluation order (stencil.py:82-87, transfer.py:33-38,
// 51-53), so they are bit-identical to the reference (no FMA contraction).
// All are HBM-streaming kernels: rows of the C-order field map to warps along
// the contiguous j axis.
#include "tmg_kernels.h"

namespace tmg {

namespace {

// (L u)(i, j): ((((W uw + E ue) + S us) + N un) + C uc), C = -(((W+E)+S)+N)
__device__ __forceinline__ double lu_at(const double* __restrict__ u, size_t o, size_t ld,
                                        double Wi, double Ei, double Sj, double Nj) {
  const double Cc = -__dadd_rn(__dadd_rn(__dadd_rn(Wi, Ei), Sj), Nj);
  double acc = __dmul_rn(Wi, u[o - ld]);
  acc = __dadd_rn(acc, __dmul_rn(Ei, u[o + ld]));
  acc = __dadd_rn(acc, __dmul_rn(Sj, u[o - 1]));
  acc = __dadd_rn(acc, __dmul_rn(Nj, u[o + 1]));
  return __dadd_rn(acc, __dmul_rn(Cc, u[o]));
}

__global__ void __launch_bounds__(256) apply_kernel(GridArgs g, const double* __restrict__ u,
                                                    const double* __restrict__ f,
                                                    double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j > g.ny) return;
  const size_t ld = (size_t)g.ny + 1, o = (size_t)i * ld + j;
  if (i == 0 || i == g.nx || j == 0 || j == g.ny) {
    out[o] = 0.0;
    return;
  }
  const double lu = lu_at(u, o, ld, __ldg(g.W + i), __ldg(g.E + i), __ldg(g.S + j), __ldg(g.N + j));
  out[o] = f ? __dadd_rn(-lu, f[o]) : lu;
}

__global__ void __launch_bounds__(256) defect_norm_kernel(GridArgs g, const double* __restrict__ u,
                                                          const double* __restrict__ f,
                                                          unsigned long long* dmax) {
  const size_t ld = (size_t)g.ny + 1;
  unsigned long long m = 0ull;
  for (int i = blockIdx.y + 1; i < g.nx; i += gridDim.y) {
    const double Wi = __ldg(g.W + i), Ei = __ldg(g.E + i);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x + 1; j < g.ny; j += gridDim.x * blockDim.x) {
      const size_t o = (size_t)i * ld + j;
      const double lu = lu_at(u, o, ld, Wi, Ei, __ldg(g.S + j), __ldg(g.N + j));
      const double d = fabs(__dadd_rn(-lu, f[o]));
      const unsigned long long b = (unsigned long long)__double_as_longlong(d);
      m = b > m ? b : m;  // bit order == value order for |d|; NaN sorts on top
    }
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
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) m = wm[w] > m ? wm[w] : m;
    if (m) atomicMax(dmax, m);
  }
}

__device__ __forceinline__ double restrict_at(const double* d, size_t o, size_t ld, int full) {
  // transfer.py:33-38: edges = ((d[i-1,j] + d[i+1,j]) + d[i,j-1]) + d[i,j+1]
  const double ctr = d[o];
  double edges = __dadd_rn(__dadd_rn(__dadd_rn(d[o - ld], d[o + ld]), d[o - 1]), d[o + 1]);
  if (!full) return __dadd_rn(__dmul_rn(0.5, ctr), __dmul_rn(0.125, edges));
  double diags = __dadd_rn(__dadd_rn(__dadd_rn(d[o - ld - 1], d[o + ld - 1]), d[o - ld + 1]),
                           d[o + ld + 1]);
  return __dadd_rn(__dadd_rn(__dmul_rn(0.25, ctr), __dmul_rn(0.125, edges)),
                   __dmul_rn(0.0625, diags));
}

constexpr int RTI = 8, RTJ = 32;  // coarse tile of the fused residual+restriction
constexpr int RUI = 2 * RTI + 3, RUJ = 2 * RTJ + 3;  // fine u tile incl. halo
constexpr int RDI = 2 * RTI + 1, RDJ = 2 * RTJ + 1;  // fine defect tile

__global__ void __launch_bounds__(256) defect_restrict_kernel(GridArgs g, int full,
                                                              const double* __restrict__ u,
                                                              const double* __restrict__ f,
                                                              double* __restrict__ fc) {
  __shared__ double su[RUI * RUJ];
  __shared__ double sd[RDI * RDJ];
  const int nxc = g.nx / 2, nyc = g.ny / 2;
  const int I0 = blockIdx.y * RTI + 1, J0 = blockIdx.x * RTJ + 1;
  const int ui0 = 2 * I0 - 2, uj0 = 2 * J0 - 2;  // fine origin of the u tile
  const size_t ld = (size_t)g.ny + 1;
  for (int t = threadIdx.x; t < RUI * RUJ; t += blockDim.x) {
    const int a = t / RUJ, b = t - a * RUJ;
    const int i = ui0 + a, j = uj0 + b;
    su[t] = (i <= g.nx && j <= g.ny) ? u[(size_t)i * ld + j] : 0.0;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < RDI * RDJ; t += blockDim.x) {
    const int a = t / RDJ, b = t - a * RDJ;
    const int i = ui0 + 1 + a, j = uj0 + 1 + b;
    double dv = 0.0;
    if (i < g.nx && j < g.ny) {
      const double lu = lu_at(su, (size_t)(a + 1) * RUJ + (b + 1), RUJ, __ldg(g.W + i),
                              __ldg(g.E + i), __ldg(g.S + j), __ldg(g.N + j));
      dv = __dadd_rn(-lu, f[(size_t)i * ld + j]);
    }
    sd[t] = dv;
  }
  __syncthreads();
  const int ti = threadIdx.x / RTJ, tj = threadIdx.x - ti * RTJ;
  const int I = I0 + ti, J = J0 + tj;
  if (I < nxc && J < nyc)
    fc[(size_t)I * (nyc + 1) + J] = restrict_at(sd, (size_t)(2 * ti + 1) * RDJ + (2 * tj + 1), RDJ, full);
}

__global__ void __launch_bounds__(256) restrict_kernel(int nxf, int nyf, int full,
                                                       const double* __restrict__ d,
                                                       double* __restrict__ out) {
  const int nxc = nxf / 2, nyc = nyf / 2;
  const int J = blockIdx.x * blockDim.x + threadIdx.x, I = blockIdx.y;
  if (J > nyc) return;
  const size_t o = (size_t)I * (nyc + 1) + J;
  if (I == 0 || I == nxc || J == 0 || J == nyc) {
    out[o] = 0.0;
    return;
  }
  out[o] = restrict_at(d, (size_t)(2 * I) * (nyf + 1) + 2 * J, (size_t)nyf + 1, full);
}

// transfer.py:45-53 value at fine (i, j) from coarse uc
__device__ __forceinline__ double prolong_at(const double* __restrict__ uc, size_t ldc, int i, int j) {
  const int I = i >> 1, J = j >> 1;
  const size_t o = (size_t)I * ldc + J;
  if (!(i & 1) && !(j & 1)) return uc[o];
  if (!(i & 1)) return __dmul_rn(0.5, __dadd_rn(uc[o], uc[o + 1]));
  if (!(j & 1)) return __dmul_rn(0.5, __dadd_rn(uc[o], uc[o + ldc]));
  return __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(uc[o], uc[o + ldc]), uc[o + 1]),
                                   uc[o + ldc + 1]));
}

__global__ void __launch_bounds__(256) prolong_kernel(int nxc, int nyc, const double* __restrict__ uc,
                                                      double* __restrict__ v) {
  const int nxf = 2 * nxc, nyf = 2 * nyc;
  const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (j > nyf) return;
  const size_t o = (size_t)i * (nyf + 1) + j;
  if (i == 0 || i == nxf || j == 0 || j == nyf) {
    v[o] = 0.0;
    return;
  }
  v[o] = prolong_at(uc, (size_t)nyc + 1, i, j);
}

__global__ void __launch_bounds__(256) prolong_correct_kernel(int nxc, int nyc,
                                                              const double* __restrict__ uc,
                                                              double* __restrict__ u) {
  const int nxf = 2 * nxc, nyf = 2 * nyc;
  const int j = blockIdx.x * blockDim.x + threadIdx.x + 1, i = blockIdx.y + 1;
  if (j >= nyf || i >= nxf) return;
  const size_t o = (size_t)i * (nyf + 1) + j;
  u[o] = __dadd_rn(u[o], prolong_at(uc, (size_t)nyc + 1, i, j));
}

// rhs over the interior in j-outer order (stencil.py:150-153)
__global__ void dense_rhs_kernel(GridArgs g, const double* __restrict__ u,
                                 const double* __restrict__ f, double* __restrict__ rhs) {
  const int mi = g.nx - 1, n = mi * (g.ny - 1);
  const size_t ld = (size_t)g.ny + 1;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int i = k % mi + 1, j = k / mi + 1;
    const size_t o = (size_t)i * ld + j;
    const double Wi = g.W[i], Ei = g.E[i], Sj = g.S[j], Nj = g.N[j];
    const double bw = i == 1 ? u[o - ld] : 0.0, be = i == g.nx - 1 ? u[o + ld] : 0.0;
    const double bs = j == 1 ? u[o - 1] : 0.0, bn = j == g.ny - 1 ? u[o + 1] : 0.0;
    double acc = __dmul_rn(Wi, bw);
    acc = __dadd_rn(acc, __dmul_rn(Ei, be));
    acc = __dadd_rn(acc, __dmul_rn(Sj, bs));
    acc = __dadd_rn(acc, __dmul_rn(Nj, bn));
    rhs[k] = __dadd_rn(f[o], -acc);
  }
}

// one warp per interior unknown: x_k = sum_c Ainv[k, c] rhs[c].  A single
// unknown is divided instead (Ainv then holds the 1x1 operator itself), which
// is what SuperLU does for the 1x1 coarsest level of every BASELINE config.
__global__ void dense_apply_kernel(GridArgs g, const double* __restrict__ Ainv,
                                   const double* __restrict__ rhs, double* __restrict__ u) {
  const int mi = g.nx - 1, n = mi * (g.ny - 1);
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  if (n == 1) {
    if (lane == 0) u[(size_t)1 * (g.ny + 1) + 1] = rhs[0] / Ainv[0];
    return;
  }
  double acc = 0.0;
  for (int c = lane; c < n; c += 32) acc += Ainv[(size_t)warp * n + c] * rhs[c];
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) {
    const int i = warp % mi + 1, j = warp / mi + 1;
    u[(size_t)i * (g.ny + 1) + j] = acc;
  }
}

}  // namespace

cudaError_t launch_apply(const GridArgs& g, const double* u, const double* f, double* out,
                         cudaStream_t s) {
  dim3 grid((g.ny + 1 + 255) / 256, g.nx + 1);
  TMG_COUNT(1);
  apply_kernel<<<grid, 256, 0, s>>>(g, u, f, out);
  return cudaGetLastError();
}

cudaError_t launch_defect_norm(const GridArgs& g, const double* u, const double* f,
                               unsigned long long* dmax_bits, cudaStream_t s) {
  if (g.nx < 2 || g.ny < 2) return cudaSuccess;
  const int bx = (g.ny - 1 + 255) / 256;
  int by = g.nx - 1;
  const int cap = 148 * 16 / (bx > 0 ? bx : 1);
  if (by > cap) by = cap > 0 ? cap : 1;
  TMG_COUNT(1);
  defect_norm_kernel<<<dim3(bx, by), 256, 0, s>>>(g, u, f, dmax_bits);
  return cudaGetLastError();
}

cudaError_t launch_defect_restrict(const GridArgs& g, int full, const double* u, const double* f,
                                   double* fc, cudaStream_t s) {
  const int nxc = g.nx / 2, nyc = g.ny / 2;
  if (nxc < 2 || nyc < 2) return cudaSuccess;
  dim3 grid((nyc - 1 + RTJ - 1) / RTJ, (nxc - 1 + RTI - 1) / RTI);
  TMG_COUNT(1);
  defect_restrict_kernel<<<grid, 256, 0, s>>>(g, full, u, f, fc);
  return cudaGetLastError();
}

cudaError_t launch_restrict(int nxf, int nyf, int full, const double* d, double* out,
                            cudaStream_t s) {
  const int nxc = nxf / 2, nyc = nyf / 2;
  dim3 grid((nyc + 1 + 255) / 256, nxc + 1);
  TMG_COUNT(1);
  restrict_kernel<<<grid, 256, 0, s>>>(nxf, nyf, full, d, out);
  return cudaGetLastError();
}

cudaError_t launch_prolong(int nxc, int nyc, const double* uc, double* v, cudaStream_t s) {
  dim3 grid((2 * nyc + 1 + 255) / 256, 2 * nxc + 1);
  TMG_COUNT(1);
  prolong_kernel<<<grid, 256, 0, s>>>(nxc, nyc, uc, v);
  return cudaGetLastError();
}

cudaError_t launch_prolong_correct(int nxc, int nyc, const double* uc, double* u, cudaStream_t s) {
  if (nxc < 1 || nyc < 1) return cudaSuccess;
  dim3 grid((2 * nyc - 1 + 255) / 256, 2 * nxc - 1);
  TMG_COUNT(1);
  prolong_correct_kernel<<<grid, 256, 0, s>>>(nxc, nyc, uc, u);
  return cudaGetLastError();
}

cudaError_t launch_dense_solve(const GridArgs& g, const double* Ainv, double* u, const double* f,
                               double* work, cudaStream_t s) {
  const int n = (g.nx - 1) * (g.ny - 1);
  if (n <= 0) return cudaSuccess;
  TMG_COUNT(1);
  dense_rhs_kernel<<<(n + 255) / 256, 256, 0, s>>>(g, u, f, work);
  TMG_COUNT(1);
  dense_apply_kernel<<<(n * 32 + 255) / 256, 256, 0, s>>>(g, Ainv, work, u);
  return cudaGetLastError();
}

namespace {
// deterministic sum of squares: fixed per-block partial sums, then one block
// adds the partials in index order (the power iteration must be reproducible)
constexpr int kNormBlocks = 1024;

__global__ void __launch_bounds__(256) sumsq_partial_kernel(const double* __restrict__ x, long n,
                                                            double* __restrict__ part) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (long k = blockIdx.x * 256L + threadIdx.x; k < n; k += (long)gridDim.x * 256)
    acc = fma(x[k], x[k], acc);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(256) sumsq_final_kernel(double* __restrict__ part, int m) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int k = threadIdx.x; k < m; k += 256) acc += part[k];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[0] = sqrt(sh[0]);
}

__global__ void scale_kernel(double* __restrict__ x, long n, double alpha) {
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x)
    x[k] *= alpha;
}
}  // namespace

cudaError_t launch_vec_norm2(const double* x, long n, double* work, cudaStream_t s) {
  const long nb = (n + 255) / 256;
  const int blocks = (int)(nb < kNormBlocks ? (nb > 0 ? nb : 1) : kNormBlocks);
  TMG_COUNT(2);
  sumsq_partial_kernel<<<blocks, 256, 0, s>>>(x, n, work);
  sumsq_final_kernel<<<1, 256, 0, s>>>(work, blocks);
  return cudaGetLastError();
}

cudaError_t launch_vec_scale(double* x, long n, double alpha, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long nb = (n + 255) / 256;
  TMG_COUNT(1);
  scale_kernel<<<(int)(nb < 148 * 16 ? nb : 148 * 16), 256, 0, s>>>(x, n, alpha);
  return cudaGetLastError();
}

namespace {
// Lcg64 stream on the device (rng.py:20-40): value k (0-based) comes from
// state_{k+1} = A^{k+1} s + C_{k+1}; thread-wise jump-ahead by squaring of
// the affine map x -> M x + I (mod 2^64), identical to the scalar recurrence.
__global__ void lcg_fill_kernel(unsigned long long s0, long n, double* __restrict__ out) {
  const unsigned long long M = 6364136223846793005ull, I = 1442695040888963407ull;
  for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n;
       k += (long)gridDim.x * blockDim.x) {
    unsigned long long e = (unsigned long long)k + 1ull;  // steps to take
    unsigned long long a = 1ull, c = 0ull;                // accumulated map
    unsigned long long pa = M, pc = I;                    // map^(2^bit)
    while (e) {
      if (e & 1ull) {  // acc = p o acc
        a = pa * a;
        c = pa * c + pc;
      }
      pc = pa * pc + pc;  // p = p o p
      pa = pa * pa;
      e >>= 1;
    }
    const unsigned long long st = a * s0 + c;
    out[k] = (double)(st >> 11) * (1.0 / 9007199254740992.0);
  }
}
}  // namespace

cudaError_t launch_lcg_fill(unsigned long long state, long n, double* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long nb = (n + 255) / 256;
  TMG_COUNT(1);
  lcg_fill_kernel<<<(int)(nb < 148 * 32 ? nb : 148 * 32), 256, 0, s>>>(state, n, out);
  return cudaGetLastError();
}

namespace {
__global__ void zero_kernel(double* __restrict__ p, size_t n) {
  pdl_trigger();
  pdl_wait();
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n;
       k += (size_t)gridDim.x * blockDim.x)
    p[k] = 0.0;
}
}  // namespace

cudaError_t launch_zero(double* p, size_t n, cudaStream_t s) {
  if (!n) return cudaSuccess;
  const size_t nb = (n + 255) / 256;
  TMG_COUNT(1);
  return launch_pdl(zero_kernel, dim3((unsigned)(nb < 148 * 16 ? nb : 148 * 16)), dim3(256), 0, s,
                    p, n);
}

}  // namespace tmg
