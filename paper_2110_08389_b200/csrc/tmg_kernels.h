// Kernel launch entry points (internal).
#pragma once
#include <cuda_runtime.h>

#include <functional>

#include "tmg_internal.h"
#include "tmg_layout.h"
#include "tmg_plan.h"

namespace tmg {

// Programmatic dependent launch inside the V-cycle: a kernel launched with
// launch_pdl() may start while its predecessor finishes; it calls
// pdl_trigger() early (its own successor may then launch) and pdl_wait()
// before it touches field data (the predecessor has completed and its
// writes are visible).  Every kernel launched this way waits exactly once.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
bool pdl_enabled();  // TMG_PDL=0 launches without the attribute

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Device-driven solve loops (mgcycle.py:128-138 on the GPU, tmg_runtime.cu):
// a while-node graph whose body is one V-cycle, the defect norm and a check
// kernel that appends the norm and decides whether another cycle runs.
struct SolveDev {
  double d0, tol;
  int max_cycles, cycle, converged, err;
  double norms[1];  // [capacity + 1]
};
struct ErrPtrs {  // pivot flags the check kernel ORs together
  int* p[32];
  int n;
};
cudaError_t launch_solve_check(cudaStream_t s, cudaGraphConditionalHandle hdl, SolveDev* sd,
                               unsigned long long* d_norm, const ErrPtrs& e);
// body(stream, handle) captures one iteration (ending with launch_solve_check)
int build_while_graph(const std::function<int(cudaStream_t, cudaGraphConditionalHandle)>& body,
                      cudaGraphExec_t* out, int* kernels_per_cycle);

// Host-side count of the kernels this library has put on streams (graph
// replays add their kernel nodes); tmg_kernel_launches() reads it.
long long& launch_counter();
#define TMG_COUNT(n) (::tmg::launch_counter() += (n))

struct SweepArgs {
  const LegD* legs;
  const BlockD* blocks;
  // one allocation [W | E | S | N] (lengths nx+1, nx+1, ny+1, ny+1): the
  // block solver addresses a chunk's couplings by element offsets from W
  const double* W;
  const double* E;
  const double* S;
  const double* N;
  double* u;         // N buffer (C order)
  const double* f;
  int ld;            // N row length ny + 1
  int* err;          // device error flags (bit 0: vanishing pivot)
  double* ut;        // T buffer (== u in LM_NATURAL)
  const double* ft;
  int ldt;           // T row length nx + 1
  int mode;          // LayoutMode of u / f
  int nx, ny;
};

// Set kernel attributes once (host only, never inside stream capture).
cudaError_t init_sweep_kernels();
// One colour stage (red = 1 / black = 0) of a compiled plan.
cudaError_t launch_colour(const Plan& P, int red, const SweepArgs& a, cudaStream_t stream);

struct GridArgs {
  int nx, ny;
  const double* W;
  const double* E;
  const double* S;
  const double* N;
};

// Persistent coarse tail (tmg_sweep.cu tail_kernel): the levels of a V-cycle
// below a size bound (mgcycle.py:89-104 from that level down and back up)
// run as ONE cooperative launch executing a list of ops; a grid barrier
// separates ops whose outputs feed the next (colour stages, transfers, the
// direct solve), instead of one graph node per stage.
enum TailOpType {
  TAIL_SWEEP = 0,        // the bins of one launch class of a colour stage
  TAIL_RESTRICT = 1,     // residual + restriction (+ zero coarse guess), 15 x 15 coarse tiles
  TAIL_PROLONG = 2,      // prolongation + correction, 32 x 32 fine tiles
  TAIL_DENSE_RHS = 3,    // coarsest level: right-hand side of the direct solve
  TAIL_DENSE_APPLY = 4,  // coarsest level: u = Ainv rhs, one warp per row
};
struct TailOp {
  int type;
  int barrier;  // 1: grid barrier after this op
  int q;        // sweep: points per thread chunk
  int nitems;   // bins / tiles / rows
  int gx;       // tiles along the fast grid axis (transfers)
  int base;     // CTA rotation (ops sharing one barrier interval spread over the grid)
  int full;     // restriction weighting
  const ChunkD* chunks;
  const BinD* bins;
  const HubD* hubs;
  SweepArgs sa;
  GridArgs g;           // the (fine) level's grid
  FieldView U, F;       // the level's u, f
  FieldView CF, CU;     // restriction: coarse f, u; prolongation: CU = coarse u
  const double* ainv;   // dense solve
  double* work;
};
// Dynamic shared memory and kernel attributes of the tail kernel for chunk
// sizes up to qmax; *max_ctas = co-resident CTAs (0: cannot run).
cudaError_t tail_prepare(int qmax, size_t* smem, int* max_ctas);
cudaError_t launch_tail(const TailOp* ops, int nops, int ctas, size_t smem, unsigned* bar,
                        cudaStream_t s);

// out = L u on the interior (0 on the boundary) if negate == 0, or
// out = f - L u (defect) if f != nullptr.  stencil.py:76-96.
cudaError_t launch_apply(const GridArgs& g, const double* u, const double* f, double* out,
                         cudaStream_t s);
// *dmax_bits = max over the interior of |f - L u| as IEEE bits (atomicMax on
// non-negative doubles); caller zeroes it.  mgcycle.py:122,130.
cudaError_t launch_defect_norm(const GridArgs& g, const double* u, const double* f,
                               unsigned long long* dmax_bits, cudaStream_t s);
// fc = R (f - L u), fused residual + restriction (full = 1 / half = 0).
// stencil.py:91-96 + transfer.py:21-39 + mgcycle.py:98-99.
cudaError_t launch_defect_restrict(const GridArgs& g, int full, const double* u,
                                   const double* f, double* fc, cudaStream_t s);
// out = R d (transfer.py:21-39)
cudaError_t launch_restrict(int nxf, int nyf, int full, const double* d, double* out,
                            cudaStream_t s);
// v = P uc (transfer.py:42-56), fine shape (2 ncx - 1, 2 ncy - 1)
cudaError_t launch_prolong(int nxc, int nyc, const double* uc, double* v, cudaStream_t s);
// u += P uc on the fine interior (transfer.py:42-56 + mgcycle.py:102)
cudaError_t launch_prolong_correct(int nxc, int nyc, const double* uc, double* u,
                                   cudaStream_t s);
// Coarse direct solve with a precomputed dense inverse of the interior
// operator (j-outer ordering, stencil.py:111): u_int = Ainv (f - B u_bdry).
cudaError_t launch_dense_solve(const GridArgs& g, const double* Ainv, double* u,
                               const double* f, double* work, cudaStream_t s);

// p[0 .. n) = 0 (a PDL-aware kernel, so the V-cycle graph stays a kernel chain)
cudaError_t launch_zero(double* p, size_t n, cudaStream_t s);
// sqrt(sum x^2) into work[0] (work: >= 1024 doubles), deterministic order
cudaError_t launch_vec_norm2(const double* x, long n, double* work, cudaStream_t s);
// out[k] = uniform [0, 1) value k of the Lcg64 stream after `state`
cudaError_t launch_lcg_fill(unsigned long long state, long n, double* out, cudaStream_t s);
// x *= alpha
cudaError_t launch_vec_scale(double* x, long n, double alpha, cudaStream_t s);

// ---- hybrid-layout (tmg_layout.h) versions used inside the V-cycle ----
// scheme / [g0, g1): only points of those sharding groups count (g0 = 0: all)
cudaError_t launch_hdefect_norm(const GridArgs& g, const FieldView& U, const FieldView& F,
                                unsigned long long* dmax, cudaStream_t s, int scheme = 0,
                                int g0 = 0, int g1 = 0);
// out[k] = V at enc[k] / V at enc[k] = in[k]; enc = 2 * offset + (T buffer)
cudaError_t launch_gather_points(const FieldView& V, const long long* enc, long n, double* out,
                                 cudaStream_t s);
cudaError_t launch_scatter_points(const FieldView& V, const long long* enc, long n,
                                  const double* in, cudaStream_t s);
cudaError_t launch_hdefect_restrict(const GridArgs& g, int full, const FieldView& U,
                                    const FieldView& F, const FieldView& FC, cudaStream_t s,
                                    const FieldView* UC = nullptr, bool* uc_zeroed = nullptr);
// u += P uc on the fine interior; (nx, ny) are the FINE dimensions
// skip_red: only the black points of the square tweed scheme (the caller's next
// red stage overwrites the red ones without reading them; tmg_transfer_dev.cuh)
cudaError_t launch_hprolong_correct(int nx, int ny, const FieldView& C, const FieldView& U,
                                    cudaStream_t s, int skip_red = 0);
// second-generation versions (tmg_transfer.cu), used unless TMG_TRANSFER=v1
cudaError_t launch_norm2(const GridArgs& g, const FieldView& U, const FieldView& F,
                         unsigned long long* dmax, cudaStream_t s, int scheme, int g0, int g1);
// [cg0, cg1) / [fg0, fg1): only the coarse / fine points of those sharding
// groups of `scheme` (one rank's share; g0 = 0: every point)
cudaError_t launch_restrict2(const GridArgs& g, int full, const FieldView& U, const FieldView& F,
                             const FieldView& FC, cudaStream_t s, const FieldView* UC = nullptr,
                             int scheme = 0, int cg0 = 0, int cg1 = 0);
cudaError_t launch_prolong2(int nx, int ny, const FieldView& C, const FieldView& U,
                            cudaStream_t s, int scheme = 0, int fg0 = 0, int fg1 = 0,
                            int skip_red = 0);
bool transfer_v1();
cudaError_t launch_to_hybrid(const FieldView& V, const double* nat, cudaStream_t s);
cudaError_t launch_from_hybrid(const FieldView& V, double* nat, cudaStream_t s);
cudaError_t launch_hdense_solve(const GridArgs& g, const double* Ainv, const FieldView& U,
                                const FieldView& F, double* work, cudaStream_t s);

}  // namespace tmg
