// Internal types shared by the host plan builder, the runtime and the kernels.
// Not part of the C ABI (include/tweedmg_b200.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tmg {

// Direction codes: the neighbour of (i, j) in direction d.
// Coupling coefficient toward d (stencil.py:12-15): W[i], E[i], S[j], N[j].
enum Dir : int { DW = 0, DE = 1, DS = 2, DN = 3, DNONE = 7 };
__host__ __device__ inline int dir_di(int d) { return d == DW ? -1 : d == DE ? 1 : 0; }
__host__ __device__ inline int dir_dj(int d) { return d == DS ? -1 : d == DN ? 1 : 0; }
__host__ __device__ inline int dir_opp(int d) { return d ^ 1; }

enum Scheme : int {
  SCHEME_CHECKERBOARD = 0,
  SCHEME_ZEBRA_X = 1,
  SCHEME_ZEBRA_Y = 2,
  SCHEME_ZEBRA_ALT = 3,
  SCHEME_TWEED = 4,
  SCHEME_WIREFRAME = 5,
  SCHEME_TWEED_WIRE_ALT = 6,
};

// One leg: a chain of grid points walked from (i0, j0) through up to four
// straight segments.  Legs of tweed blocks run tip -> branch (layout.py:81-82);
// a wireframe ring is one leg (the ring minus its closing point) whose two
// ends couple to the closing point, which plays the hub (_ckernels.pyx:114-141).
struct LegD {
  int32_t i0, j0;
  int32_t npts;
  int32_t tbase;       // first virtual thread (chunk) of this leg within its bin
  int32_t nchunk;      // chunks == threads
  int32_t block;       // owning block (global index)
  int32_t seg_len[4];  // steps per segment
  uint8_t seg_dir[4];
  uint8_t nseg;
  uint8_t flags;       // 1: first point couples to the hub, 2: last point does
  uint8_t hub_dir_first, hub_dir_last;  // direction from the end point to the hub
};

// One block: an optional hub (branch point / ring closing point / single
// point) and 0..4 legs.  Same-colour blocks never touch.
struct BlockD {
  int32_t hi, hj;      // hub point; hi < 0 if the block has no hub
  int32_t leg0, nleg;  // global leg indices
  int32_t hub_thread;  // virtual thread (within bin) that solves the hub row
  int32_t bin;
  uint8_t hub_mask;    // bit d: hub neighbour in direction d is a block member
  uint8_t red;
  uint8_t pad[2];
};

// One thread's chunk: <= q consecutive points of a leg lying on one straight
// run (chunks never turn a corner), so point k of the chunk is at element
// offset off + k*stride and along-axis index a0 + k*da.
struct ChunkD {
  int32_t off;    // element offset of the first point
  int16_t a0;     // along-axis index of the first point (i if axis 0, else j)
  int16_t cidx;   // cross-axis index (j if axis 0, else i)
  int16_t hub;    // virtual thread that owns the block's hub value, -1 if none
  int16_t own;    // index of the hub this thread solves (within the bin), -1
  uint8_t n;      // points in the chunk (0: no chunk)
  uint8_t geo;    // bit 0: axis (0: i varies, 1: j varies); bit 1: decreasing;
                  // bit 2: the chunk lives in the transposed buffer (tmg_layout.h)
  uint16_t link;  // bits 0-2 dfirst, 3-5 dlast (direction from the first /
                  // last point to its in-block neighbour outside the chunk,
                  // 7 = none); bit 6 left = previous thread, bit 7 left = hub,
                  // bit 8 right = next thread, bit 9 right = hub
};
static_assert(sizeof(ChunkD) == 16, "ChunkD must stay 16 bytes");

constexpr int kLinkLeftPrev = 1 << 6, kLinkLeftHub = 1 << 7;
constexpr int kLinkRightNext = 1 << 8, kLinkRightHub = 1 << 9;

// Hub row of one block (branch point, ring closing point or a point block).
struct HubD {
  int32_t off;
  int16_t i, j;
  uint8_t mask;       // bit d: the hub's neighbour in direction d is in-block
  uint8_t nadj;       // adjacent chunk ends (0..4)
  int16_t adj_t[4];   // virtual thread whose reduced unknown is that point
  uint8_t adj_d[4];   // direction from the hub to that point
  uint8_t tbuf;       // 1: the hub point lives in the transposed buffer
  uint8_t pad;        // bit 0: a CTA-local copy that does not store the hub
};
static_assert(sizeof(HubD) == 24, "HubD layout");

struct BinD {
  int32_t pcr_steps;  // ceil(log2(max chunks of any leg in the bin))
  int32_t hub0;       // first hub of the bin in the class hub array
  int32_t nhub;
  int32_t warp_local;  // 1: every leg lies inside one warp; 2: some leg spans CTAs
};

// One kernel launch worth of bins sharing (q, cluster size).
struct LaunchClass {
  int q;
  int cs;          // CTAs per cluster (1, 2, 4, 8, 16)
  int nbins;
  int red;
  int xcta;        // 1: every bin has a leg crossing a CTA boundary of its cluster
  ChunkD* chunks;  // nbins * cs * kThreads
  BinD* bins;
  HubD* hubs;
};

#ifndef TMG_THREADS
#define TMG_THREADS 256
#endif
constexpr int kThreads = TMG_THREADS;  // threads per CTA of the block-solver kernel
constexpr int kMaxCluster = 16;  // CTAs per cluster (16 is a non-portable size on B200)
constexpr int kQmax = 16;       // max points per thread chunk

}  // namespace tmg
