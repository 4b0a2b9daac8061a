// Host-side block geometry and launch planning (native runtime).
#pragma once
#include <string>
#include <vector>

#include "tmg_internal.h"
#include "tmg_layout.h"
#include "tmg_tweedleg.h"

namespace tmg {

// Closed-form block decomposition of one smoothing scheme on an nx x ny grid.
// Blocks are emitted in the reference's construction order (layout.py:61-168,
// smoothers.py:65-89) so that member dumps can be compared one to one.
struct Geometry {
  int scheme = 0, nx = 0, ny = 0;
  std::vector<BlockD> blocks;
  std::vector<LegD> legs;
};

// Returns "" on success, else an error message (bad dims / scheme).
std::string build_geometry(int scheme, int nx, int ny, Geometry& g);

// Per-point member dump in layout.py order (legs tip->branch, then branch;
// rings in traversal order).  Returns the number of members.
long dump_members(const Geometry& g, int* oi, int* oj, int* oblk, int* oflags, long cap);

// Device-resident launch plan for one (scheme, grid): geometry + bins.
struct Plan {
  Geometry geo;
  int q = kQmax;
  int mode = LM_NATURAL;  // field layout the chunk offsets address
  LegD* d_legs = nullptr;
  BlockD* d_blocks = nullptr;
  std::vector<LaunchClass> classes;  // red classes first, then black
  bool point_scheme = false;         // checkerboard: dedicated point kernel
  int g0 = 0, g1 = 0;                // group range of a partial plan (0, 0: all)
  size_t device_bytes = 0;
  // tweed L-shells of square hybrid grids run on the TMA-fed leg kernel
  // (tmg_tweedleg.cu); the generic classes then hold the remaining blocks
  LegPlan* lp = nullptr;
  bool arena = false;  // device arrays live in an UploadArena
};

// Grow-only device buffer the shims pack their one-block plans into.
struct UploadArena {
  char* base = nullptr;
  size_t cap = 0, used = 0;
  cudaStream_t stream = nullptr;
};
// Route pack_plan's uploads into `a` (nullptr: cudaMalloc per array).
void set_upload_arena(UploadArena* a);

std::string build_plan(int scheme, int nx, int ny, int q, int mode, Plan& p);
// Plan restricted to the blocks of sharding groups [g0, g1) (point_group in
// tmg_layout.h): one rank's share of a colour stage in a sharded V-cycle.
std::string build_plan_part(int scheme, int nx, int ny, int q, int mode, int g0, int g1, Plan& p);
// Keep only the blocks whose group lies in [g0, g1).
void filter_groups(Geometry& g, int g0, int g1);
// Pack an explicit geometry (e.g. one block from the per-block shims).
std::string pack_plan(Geometry&& g, int q, int mode, Plan& p);
// Append a block made of explicit member paths (host index arrays).
// kind: 0 points (each a hub-only block), 1 chain, 2 ring, 3 legged.
std::string add_explicit_block(Geometry& g, int kind, long n, const long long* ii,
                               const long long* jj, long m, const long long* offs, long bi,
                               long bj);
void free_plan(Plan& p);

}  // namespace tmg
