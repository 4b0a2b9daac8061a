// Hybrid HBM layout of the V-cycle fields.
//
// A field is held in two buffers: N, C-order (i, j) with j contiguous (the
// reference's layout, stencil.py:12-15), and T, its transpose with i
// contiguous.  Every interior point is owned by exactly one buffer, chosen so
// that every smoother line runs along the contiguous axis of its owner:
//   LM_NATURAL  all points in N (plain C order; used for API-level calls)
//   LM_TWEED    x-legs (i' < j', mirrored indices) in T, y-legs / branches /
//               corners in N (layout.py:61-133 geometry)
//   LM_WIRE     ring x-edges (j' < i') in T, y-edges / corners in N
//               (layout.py:136-168)
//   LM_XLINES   every interior point in T (zebra_x)
// The Dirichlet ring is owned by N and mirrored into T, so it can be read
// through either buffer.  Kernels address a point through field_at().
#pragma once
#include <cstddef>

namespace tmg {

enum LayoutMode : int { LM_NATURAL = 0, LM_TWEED = 1, LM_WIRE = 2, LM_XLINES = 3 };

// Branch-free (bitwise & / |, no short circuit): the device code computes a
// buffer address per point without control flow, so independent loads
// through FieldView::at issue back to back.
__host__ __device__ inline bool owns_t(int mode, int nx, int ny, int i, int j) {
  const int ip = i < nx - i ? i : nx - i;
  const int jp = j < ny - j ? j : ny - j;
  const bool interior = (i > 0) & (j > 0) & (i < nx) & (j < ny);
  return interior & (((mode == LM_TWEED) & (ip < jp)) | ((mode == LM_WIRE) & (jp < ip)) |
                     (mode == LM_XLINES));
}

// layout a smoother kind runs fastest on
__host__ __device__ inline int layout_for_kind(int kind) {
  switch (kind) {
    case 1: return LM_XLINES;   // zebra_x
    case 4: return LM_TWEED;    // tweed
    case 5: return LM_WIRE;     // wireframe
    default: return LM_NATURAL; // checkerboard, zebra_y, alternating kinds
  }
}

// Sharding group of an interior point (multi-GPU unit): every
// block of a scheme lies in one group, groups form a chain (a point's stencil
// neighbours are in groups g-1..g+1), and coarse group G is fine group 2G.
//   tweed        L-shell / cross / strip index max(i', j')   (layout.py:61-133)
//   wireframe    ring index min(i', j'), the centre is q+1   (layout.py:136-168)
//   zebra_x      row j;  zebra_y, checkerboard: column i     (smoothers.py:65-89)
// Scheme codes as tmg_internal.h / include/tweedmg_b200.h.
__host__ __device__ inline int point_group(int scheme, int nx, int ny, int i, int j) {
  const int ip = i < nx - i ? i : nx - i;
  const int jp = j < ny - j ? j : ny - j;
  switch (scheme) {
    case 4: return ip > jp ? ip : jp;
    case 5: return ip < jp ? ip : jp;
    case 1: return j;
    default: return i;
  }
}
// groups are numbered 1..group_count (0 if the scheme does not shard)
__host__ __device__ inline int group_count(int scheme, int nx, int ny) {
  switch (scheme) {
    case 4: return (nx > ny ? nx : ny) / 2;
    case 5: return (nx < ny ? nx : ny) / 2;
    case 1: return ny - 1;
    case 0:
    case 2: return nx - 1;
    default: return 0;
  }
}

struct FieldView {
  double* n;
  double* t;
  int nx, ny, mode;
  __host__ __device__ inline size_t off_n(int i, int j) const { return (size_t)i * (ny + 1) + j; }
  __host__ __device__ inline size_t off_t(int i, int j) const { return (size_t)j * (nx + 1) + i; }
  __host__ __device__ inline double* at(int i, int j) const {
    return owns_t(mode, nx, ny, i, j) ? t + off_t(i, j) : n + off_n(i, j);
  }
};

}  // namespace tmg
