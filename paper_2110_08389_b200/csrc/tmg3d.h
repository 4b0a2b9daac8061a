// Shared pieces of the 3D cube paths (tmg3d.cu: tweed and the V-cycle;
// tmg3dw.cu: wireframe blocks).  Fields are C-order (n+1)^3, k fastest.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace tmg3 {

struct Coef3 {
  const double *W, *E, *S, *N, *B, *T;
};

// Field views of the 3D block kernels (tmg3dw.cu): natural mode (hybrid = 0)
// aliases the C-order arrays; hybrid mode adds i- and j-contiguous copies
// (views 0, 1) next to the natural array (view 2); hybrid = 1:
// a point belongs to the axis of its largest mirrored coordinate (3D
// wireframe edges), 2: of its smallest (3D tweed legs).
struct Fields3 {
  double* u[3];
  const double* f[3];
  int hybrid;
};

__host__ __device__ inline long mirror(long x, long n) { return x < n - x ? x : n - x; }

// reciprocal: the hardware approximation refined by two Newton steps (the
// 2D solver's drcp, tmg_sweep.cu)
__device__ __forceinline__ double rcp3(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ size_t idx3(int n, int i, int j, int k) {
  return ((size_t)i * (n + 1) + j) * (size_t)(n + 1) + k;
}

// ---------------------------------------------------------------------------
// 3D wireframe (tmg3dw.cu).  Blocks of one level and colour:
//   rings  closed square rings of a shell face: 4 edges between 4 corners,
//          grouped in classes by the threads per edge (kRingClasses);
//   frames the 12-edge / 8-corner frame of a shell (red only);
//   points face centres and the cube centre.
constexpr int kRingClasses = 8;  // TE = 1 .. 128 threads per ring side

struct Ring3 {
  int16_t a;   // axis normal to the face
  int16_t t;   // ring level in the face
  int32_t xa;  // coordinate of the face along a
};

struct WLevel {
  Ring3* rings[2][kRingClasses] = {};
  int nrings[2][kRingClasses] = {};
  int* frames = nullptr;   // shell r of each frame
  int nframes = 0;
  int4* points[2] = {};
  int npoints[2] = {};
};

// blocks of sharding groups [g0, g1) only (group = min(i', j', k'): the shell)
// ---------------------------------------------------------------------------
// 3D tweed hub blocks (tmg3dw.cu, the same block kernel): a branch with 2, 3
// or 6 legs running from the walls (tmg3d.cu build_blocks)
struct HubB {
  int32_t bi, bj, bk;  // the branch
  int16_t len;         // points per leg (s1 - 1)
  uint8_t nleg;
  uint8_t red;
  uint8_t leg[6];      // bits 0-1 axis, bit 2: step -1 (tip at n-1)
  uint8_t pad[2];
};
static_assert(sizeof(HubB) == 24, "HubB layout");

constexpr int kHubKinds = 2;    // 2 legs; 3 or 6 legs
constexpr int kHubClasses = 6;  // TE = 1 .. 32 threads per leg

struct HubLevel {
  HubB* blocks[2][kHubKinds][kHubClasses] = {};
  int nblocks[2][kHubKinds][kHubClasses] = {};
  int4* points[2] = {};  // legless branches
  int npoints[2] = {};
};

int hub_build_level(int n, const std::vector<HubB> blocks[2], HubLevel& L, std::string& err);
void hub_free_level(HubLevel& L);
int hub_stage(const HubLevel& L, int n, const Coef3& c, int red, double* u, const double* f,
              int* err, cudaStream_t s);
int hub_stage(const HubLevel& L, int n, const Coef3& c, int red, const Fields3& F, int* err,
              cudaStream_t s);

int wire_build_level(int n, WLevel& L, std::string& err, int g0 = 0, int g1 = 1 << 30);
void wire_free_level(WLevel& L);
// one colour stage (red = 1 / black = 0) of the wireframe sweep
int wire_stage(const WLevel& L, int n, const Coef3& c, int red, double* u, const double* f,
               int* err, cudaStream_t s);
int wire_stage(const WLevel& L, int n, const Coef3& c, int red, const Fields3& F, int* err,
               cudaStream_t s);
// blocks of a colour (for tmg_cube_blocks)
long wire_blocks(const WLevel& L, int red);

}  // namespace tmg3
