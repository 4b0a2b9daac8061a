// Line-gather bandwidth on an (n+1)^3 fp64 cube, n = 1024: one CTA per line
// of n-1 points along axis x, one point per lane, f plus four transverse u
// neighbours loaded, u written (the 3D wireframe edge gather/scatter access
// pattern).  Prints GB/s (24 B per point) per axis and CTA order.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256) line(int n, int x, int order, const double* __restrict__ f,
                                            double* __restrict__ u) {
  const long n1 = n + 1, str[3] = {n1 * n1, n1, 1};
  const int o1 = x == 0 ? 1 : 0, o2 = x == 2 ? 1 : 2;
  const int b = blockIdx.x, m = n - 1;
  // order 0: consecutive CTAs step the fastest transverse axis; 1: the slowest
  const int c1 = order ? 1 + b % m : 1 + b / m, c2 = order ? 1 + b / m : 1 + b % m;
  const size_t base = (size_t)c1 * str[o1] + (size_t)c2 * str[o2];
  for (int p = threadIdx.x; p < m; p += 256) {
    const size_t o = base + (size_t)(p + 1) * str[x];
    const double r = f[o] - 0.1 * u[o - str[o1]] - 0.2 * u[o + str[o1]] - 0.3 * u[o - str[o2]] -
                     0.4 * u[o + str[o2]];
    u[o] = r;  // same-colour lines do not touch: here every line writes its own points
  }
}
int main() {
  const int n = 1024;
  const size_t N = (size_t)(n + 1) * (n + 1) * (n + 1);
  double *f, *u;
  cudaMalloc(&f, N * 8);
  cudaMalloc(&u, N * 8);
  cudaMemset(f, 0, N * 8);
  cudaMemset(u, 0, N * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int lines = (n - 1) * (n - 1);
  for (int x = 0; x < 3; x++)
    for (int order = 0; order < 2; order++) {
      line<<<lines, 256>>>(n, x, order, f, u);
      cudaEventRecord(a);
      line<<<lines, 256>>>(n, x, order, f, u);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double pts = (double)lines * (n - 1);
      printf("axis %d order %d: %.2f ms, %.0f GB/s (24 B/pt)\n", x, order, ms, 24.0 * pts / ms / 1e6);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
