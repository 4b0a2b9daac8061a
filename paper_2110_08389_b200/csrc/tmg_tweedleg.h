// Tweed L-shell kernel (tmg_tweedleg.cu): plan types and entry points.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace tmg {

struct SweepArgs;

constexpr int kLegQ = 17;          // points per thread chunk
constexpr int kLegThreads = 256;   // threads per CTA
#ifndef TMG_LEGK_MAXB
#define TMG_LEGK_MAXB 8
#endif
constexpr int kLegMaxBlocks = TMG_LEGK_MAXB;  // blocks per item
// Staged arrays (doubles): 18 slots of headroom (dummy points in front of a
// leg's tip read finite values there), the runs of the item's legs (<= 256
// chunks of 17 points, <= 2 alignment elements per leg run), 18 slots of
// tail room.  The f array also holds, per leg, the private gap (<= 16 slots)
// its tip chunk's dummies write.
constexpr int kLegHead = 18;
constexpr int kLegArrU = kLegHead + kLegThreads * kLegQ + 4 * kLegMaxBlocks + 18;
constexpr int kLegArrF = kLegArrU + 2 * 16 * kLegMaxBlocks;
constexpr int kLegStage = kLegArrF + 2 * kLegArrU;
constexpr int kLegK0 = 2;      // smallest shell the kernel takes (at 2 it takes the corners too)
constexpr int kLegNmin = 1024;  // smallest grid (n) the kernel runs on (512: V-cycle +0.8 %)

struct LegItem {  // one CTA's work of one cluster iteration
  int32_t blk0;   // first LegBlock
  int16_t nblk;
  int16_t steps;  // PCR steps (ceil(log2(max chunks of a leg)))
  int32_t copy0, ncopy;    // bulk loads (LegCopy)
  int32_t bytes;           // staged bytes (mbarrier transaction count)
  int32_t store0, nstore;  // bulk stores of the aligned leg interiors (LegCopy)
  int32_t edge0, nedge;    // single-element stores at unaligned leg ends (LegCopy, n = 1)
};
struct LegBlock {
  int16_t k;       // shell (layout.py:75-84)
  uint8_t quad;    // bit 0: corner at i = n-1, bit 1: at j = n-1
  uint8_t split;   // 0 whole block, 1 this CTA holds leg 0 only, 2 leg 1 only,
                   // 3..6 one leg (W, E, S, N) of the central cross
  int16_t t0[2];   // thread of each leg's tip chunk (-1: on the peer CTA)
  int16_t sb[2][3];  // shared slot of each leg's tip element in the f / u-1 / u+1 arrays
};
struct LegCopy {  // one bulk copy between a field buffer and the shared stage
  int64_t g;      // element offset in the field buffer (even for bulk copies)
  int32_t s;      // element offset in the stage (even for bulk copies)
  int32_t n;      // elements (even for bulk copies)
  uint8_t src;    // buffer: 0 f N, 1 f T, 2 u N, 3 u T
  uint8_t pad[7];
};
// Per-item descriptor blob (16-byte aligned, <= kLegBlob bytes): the header,
// the item's LegCopy records (loads, stores, edge stores), its LegBlocks and
// its thread map, bulk-copied into shared memory one item ahead so neither
// the per-thread setup nor warp 0's store / load issue waits on L2.
constexpr int kLegBlob = 3072;
struct LegBlobHead {
  int32_t nblk, ncopy, nstore, nedge;
  int32_t bytes;       // staged bytes (mbarrier transaction count)
  int32_t off_blocks;  // byte offsets in the blob
  int32_t off_tmap;
  int32_t bytes_f;     // the f runs' share of `bytes`
};
struct LegColour {
  LegItem* items = nullptr;
  LegBlock* blocks = nullptr;
  uint16_t* tmap = nullptr;  // [item][thread]: (block slot << 1 | leg), 0xFFFF idle
  LegCopy* copies = nullptr;  // loads, stores and edge stores of every item
  int4* sched = nullptr;     // cluster iteration: (item rank 0, item rank 1, split, load)
  unsigned char* blob = nullptr;  // descriptor blobs of every item
  int4* bsched = nullptr;    // per cluster iteration: (blob offset / 16, bytes) of rank 0, rank 1
  int nsched = 0, nitems = 0;
  int cross = 0;              // this colour holds the central cross
  int corners = 0;            // this colour (red) relaxes the four corner points
  double* mail = nullptr;     // cross mailbox: 4 x (P, Qh), two counters
  long points = 0;
};
struct LegPlan {
  int n = 0;
  // (a, c) along couplings, chunk-permuted: [orientation][tip pad 0..16][cstride]
  double2* coef = nullptr;
  int cstride = 0;
  LegColour col[2];         // [black, red]
  size_t device_bytes = 0;
};

struct LegArgs {
  double* un;
  double* ut;
  const double* fn;
  const double* ft;
  const double* W;
  const double* E;
  const double* S;
  const double* N;
  const double2* coef;
  int cstride;
  int n, ld;
  const LegItem* items;
  const LegBlock* blocks;
  const uint16_t* tmap;
  const LegCopy* copies;
  const int4* sched;
  const unsigned char* blob;
  const int4* bsched;
  int nsched;
  int* err;
  long long* timing;  // per-CTA phase clocks (TMG_LEGK_TIMING), or null
  double* mail;       // cross mailbox (colour with the central cross), or null
  int corners;        // CTA 0 relaxes the four corner points first
};

// true if the L-shell kernel takes part of this plan's colour stages
bool leg_plan_applies(int scheme, int nx, int ny, int mode);
int leg_k0();
// shells k in [kmin, kmax] (k = n/2: the central cross); default: all
std::string build_leg_plan(int n, LegPlan& P, int kmin = 0, int kmax = 1 << 30);
std::string leg_plan_set_coefs(LegPlan& P, const double* W, const double* E, const double* S,
                               const double* N);
void free_leg_plan(LegPlan& P);
cudaError_t launch_leg_colour(const LegPlan& P, int red, const SweepArgs& a, cudaStream_t s);

}  // namespace tmg
