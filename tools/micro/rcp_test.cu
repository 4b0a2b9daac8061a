// accuracy of rcp.approx.ftz.f64 refined by k Newton steps vs 1.0/x
#include <cstdio>
#include <cmath>
#include <cstdint>
__global__ void k(const double* x, double* e0, double* e1, double* e2, int n) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double v = x[t], r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
  double ex = 1.0 / v;
  e0[t] = fabs(r - ex) / fabs(ex);
  double e = fma(-v, r, 1.0); double r1 = fma(r, e, r);
  e1[t] = fabs(r1 - ex) / fabs(ex);
  e = fma(-v, r1, 1.0); double r2 = fma(r1, e, r1);
  e2[t] = fabs(r2 - ex) / fabs(ex);
}
int main() {
  const int n = 1 << 22;
  double *x, *a, *b, *c;
  cudaMallocManaged(&x, n * 8); cudaMallocManaged(&a, n * 8); cudaMallocManaged(&b, n * 8); cudaMallocManaged(&c, n * 8);
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < n; i++) { s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    double u = (s >> 11) * (1.0 / 9007199254740992.0); x[i] = (i & 1 ? -1 : 1) * pow(10.0, -8 + 22 * u); }
  k<<<(n + 255) / 256, 256>>>(x, a, b, c, n);
  cudaDeviceSynchronize();
  double m0 = 0, m1 = 0, m2 = 0;
  for (int i = 0; i < n; i++) { m0 = fmax(m0, a[i]); m1 = fmax(m1, b[i]); m2 = fmax(m2, c[i]); }
  printf("max rel err: approx %.3e  1 newton %.3e  2 newton %.3e  (ulp %.3e)\n", m0, m1, m2, 1.1e-16);
}
