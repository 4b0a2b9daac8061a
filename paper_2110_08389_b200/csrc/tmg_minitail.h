// Shared-memory coarse tail (tmg_minitail.cu): the smallest levels of a
// V-cycle as ONE single-CTA launch with every field resident in shared memory.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "tmg_kernels.h"
#include "tmg_layout.h"

namespace tmg {

// One tail level as the host hands it over (fine -> coarse order).
struct MiniLevelIn {
  int nx, ny;
  const double *W, *E, *S, *N;  // device 1D coefficient arrays
};

struct MiniTail {
  void* d_blob = nullptr;  // every plan array, one allocation
  size_t smem = 0;         // dynamic shared memory of the launch
  int nlev = 0;
  int blob_bytes = 0;
  // byte offsets of the plan tables in the blob
  int o_lev = 0, o_stage = 0, o_unit = 0, o_mem = 0;
  int off_scratch = 0, maxmem = 0;  // doubles, after the blob's copy in shared memory
};

// largest smoothing block (members solved by one thread: a leg, a chain, a
// ring) of `schemes` on an nx x ny grid; < 0 on error
int mini_max_unit(const std::vector<int>& schemes, int nx, int ny);

// Build the plan of the levels `lv` (fine -> coarse; the last one is solved
// directly) for one sweep = the sub-schemes `schemes` in order, red then black.
std::string build_mini_tail(const std::vector<MiniLevelIn>& lv, const std::vector<int>& schemes,
                            MiniTail& out);
void free_mini_tail(MiniTail& t);

// U0 / F0: the hierarchy's work fields of the first tail level; ainv: the
// coarsest level's dense factor (tmg_runtime.cu factor_coarse); err: pivot flag
cudaError_t launch_mini_tail(const MiniTail& t, const FieldView& U0, const FieldView& F0,
                             const double* ainv, int full, int nu1, int nu2, int* err,
                             cudaStream_t s);

}  // namespace tmg
