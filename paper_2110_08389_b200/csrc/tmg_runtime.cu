// Native runtime behind the C ABI (include/tweedmg_b200.h): level handles
// with lazily compiled device plans, the coarse direct solver, the V-cycle
// driver (mgcycle.py:80-139) on the hybrid field layout, solver sessions and
// CUDA-graph replay of whole cycles.
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/tweedmg_b200.h"
#include "tmg_kernels.h"
#include "tmg_minitail.h"
#include "tmg_plan.h"

using namespace tmg;

namespace {
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(TMG_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define TMG_CUDA_TRY(expr)                              \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

// Points per thread chunk.  TMG_CHUNK forces a value; otherwise a level
// keeps q = 16 while one colour stage still fills about one wave of
// resident CTAs (2 per SM), and smaller levels halve q (down to 2) so that
// their launches spread over the GPU with shorter per-thread chains.
int default_q(int nx = 0, int ny = 0) {
  const char* s = std::getenv("TMG_CHUNK");
  if (s) {
    int q = std::atoi(s);
    if (q >= 1 && q <= kQmax && !(q & (q - 1))) return q;
  }
  static int wave = 0;
  if (!wave) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      sms = 148;
    wave = sms / 2;  // a quarter of the resident CTAs (2 per SM): measured best
    const char* w = std::getenv("TMG_QWAVES");  // tuning: waves a q = 16 launch must fill
    if (w && std::atof(w) > 0) wave = (int)(wave * std::atof(w));
  }
  const double per_colour = 0.5 * (double)(nx - 1) * (double)(ny - 1);
  static int qmin = 0;
  if (!qmin) {
    const char* m = std::getenv("TMG_QMIN");  // tuning: smallest adaptive q
    qmin = m && std::atoi(m) >= 1 ? std::atoi(m) : 2;
  }
  int q = kQmax;
  while (q > qmin && per_colour < (double)wave * kThreads * q) q /= 2;
  return q;
}

bool valid_kind(int k) { return k >= TMG_CHECKERBOARD && k <= TMG_TWEED_WIRE_ALT; }

// the hierarchy's working layout: the preferred one of the smoother unless
// TMG_LAYOUT=natural forces plain C order (for A/B measurements)
int session_mode(int kind) {
  const char* s = std::getenv("TMG_LAYOUT");
  if (s && std::strcmp(s, "natural") == 0) return LM_NATURAL;
  return layout_for_kind(kind);
}
}  // namespace

struct tmg_level {
  int nx = 0, ny = 0, device = 0;
  double *W = nullptr, *E = nullptr, *S = nullptr, *N = nullptr;
  std::vector<double> hW, hE, hS, hN;
  Plan* plans[7][4] = {};  // [scheme][layout mode]
  std::map<std::tuple<int, int, int, int>, Plan*> part_plans;  // (scheme, mode, g0, g1)
  int* d_err = nullptr;
  unsigned long long* d_norm = nullptr;
  int* h_err = nullptr;                  // pinned
  unsigned long long* h_norm = nullptr;  // pinned
  double* d_ainv = nullptr;              // coarse dense inverse (or the 1x1 operator)
  double* d_work = nullptr;
  long long bytes = 0;

  GridArgs grid() const { return GridArgs{nx, ny, W, E, S, N}; }
};

struct tmg_hier {
  std::vector<tmg_level*> lv;
  int mode = -1;                // layout of the work fields (-1: not allocated)
  std::vector<FieldView> U, F;  // work fields of every level (level 0 included)
  std::vector<double*> blocks;  // allocations
  bool loaded = false;          // level 0 holds a session's u and f
  std::map<std::tuple<int, int, int, int>, std::pair<cudaGraphExec_t, int>> graphs;
  int last_kernels = 0;
  long long bytes = 0;
  SolveDev* d_solve = nullptr;  // device-driven solve loop state (solve_graph)
  int solve_cap = 0;            // cycles d_solve has room for
  std::map<std::tuple<int, int, int, int>, std::pair<cudaGraphExec_t, int>> solve_graphs;
  // persistent coarse-tail programs per (kind, full, nu1, nu2, first level)
  struct TailProg {
    TailOp* d_ops = nullptr;
    int nops = 0, ctas = 0, level = 0;
    size_t smem = 0;
    MiniTail* mini = nullptr;  // the shared-memory tail (tmg_minitail.cu) instead of an op list
  };
  std::map<std::tuple<int, int, int, int, int>, TailProg> tails;
  unsigned* d_tail_bar = nullptr;  // grid barrier state of the tail kernel
};

namespace {

int get_plan(tmg_level* lv, int scheme, int mode, Plan** out) {
  if (!lv->plans[scheme][mode]) {
    cudaError_t e = init_sweep_kernels();
    if (e != cudaSuccess) return cuda_fail(e, "kernel attributes");
    Plan* p = new Plan();
    std::string err = build_plan(scheme, lv->nx, lv->ny, default_q(lv->nx, lv->ny), mode, *p);
    if (err.empty() && p->lp)
      err = leg_plan_set_coefs(*p->lp, lv->hW.data(), lv->hE.data(), lv->hS.data(),
                               lv->hN.data());
    if (!err.empty()) {
      free_plan(*p);
      delete p;
      return fail(TMG_BADARG, err);
    }
    lv->plans[scheme][mode] = p;
    lv->bytes += (long long)p->device_bytes;
  }
  *out = lv->plans[scheme][mode];
  return TMG_OK;
}

// plan of one rank's sharding groups [g0, g1) (sharded V-cycle)
int get_part_plan(tmg_level* lv, int scheme, int mode, int g0, int g1, Plan** out) {
  auto key = std::make_tuple(scheme, mode, g0, g1);
  auto it = lv->part_plans.find(key);
  if (it == lv->part_plans.end()) {
    cudaError_t e = init_sweep_kernels();
    if (e != cudaSuccess) return cuda_fail(e, "kernel attributes");
    Plan* p = new Plan();
    std::string err =
        build_plan_part(scheme, lv->nx, lv->ny, default_q(lv->nx, lv->ny), mode, g0, g1, *p);
    if (err.empty() && p->lp)
      err = leg_plan_set_coefs(*p->lp, lv->hW.data(), lv->hE.data(), lv->hS.data(),
                               lv->hN.data());
    if (!err.empty()) {
      free_plan(*p);
      delete p;
      return fail(TMG_BADARG, err);
    }
    lv->bytes += (long long)p->device_bytes;
    it = lv->part_plans.emplace(key, p).first;
  }
  *out = it->second;
  return TMG_OK;
}

SweepArgs sweep_args(tmg_level* lv, const Plan* p, const FieldView& U, const FieldView& F) {
  SweepArgs a{};
  a.legs = p->d_legs;
  a.blocks = p->d_blocks;
  a.W = lv->W;
  a.E = lv->E;
  a.S = lv->S;
  a.N = lv->N;
  a.u = U.n;
  a.f = F.n;
  a.ld = lv->ny + 1;
  a.err = lv->d_err;
  a.ut = U.t;
  a.ft = F.t;
  a.ldt = lv->nx + 1;
  a.mode = U.mode;
  a.nx = lv->nx;
  a.ny = lv->ny;
  return a;
}

FieldView natural_view(tmg_level* lv, double* p) {
  return FieldView{p, p, lv->nx, lv->ny, LM_NATURAL};
}

int sweep_one(tmg_level* lv, int scheme, int colour_mask, const FieldView& U, const FieldView& F,
              cudaStream_t s) {
  Plan* p = nullptr;
  int st = get_plan(lv, scheme, U.mode, &p);
  if (st) return st;
  SweepArgs a = sweep_args(lv, p, U, F);
  for (int red = 1; red >= 0; red--) {
    if (!(colour_mask & (red ? 1 : 2))) continue;
    cudaError_t e = launch_colour(*p, red, a, s);
    if (e != cudaSuccess) return cuda_fail(e, "sweep launch");
  }
  return TMG_OK;
}

int sweep_kind(tmg_level* lv, int kind, int colour_mask, const FieldView& U, const FieldView& F,
               cudaStream_t s) {
  if (!valid_kind(kind)) return fail(TMG_BADARG, "unknown smoother kind " + std::to_string(kind));
  if (kind == TMG_ZEBRA_ALT) {  // smoothers.py:126-129
    int st = sweep_one(lv, TMG_ZEBRA_X, colour_mask, U, F, s);
    return st ? st : sweep_one(lv, TMG_ZEBRA_Y, colour_mask, U, F, s);
  }
  if (kind == TMG_TWEED_WIRE_ALT) {  // smoothers.py:130-133
    int st = sweep_one(lv, TMG_TWEED, colour_mask, U, F, s);
    return st ? st : sweep_one(lv, TMG_WIREFRAME, colour_mask, U, F, s);
  }
  return sweep_one(lv, kind, colour_mask, U, F, s);
}

// Dense inverse of the interior operator in j-outer ordering (stencil.py:99-126),
// Gauss-Jordan with partial pivoting, computed once per level on the host.
int factor_coarse(tmg_level* lv) {
  if (lv->d_ainv) return TMG_OK;
  const int mi = lv->nx - 1, mj = lv->ny - 1;
  const long n = (long)mi * mj;
  if (n < 1) return fail(TMG_BADARG, "grid has no interior");
  if (n > 4096)
    return fail(TMG_BADARG, "direct solve supports at most 4096 interior unknowns, got " +
                                std::to_string(n));
  std::vector<double> A((size_t)n * n, 0.0), X((size_t)n * n, 0.0);
  for (int i = 1; i <= mi; i++)
    for (int j = 1; j <= mj; j++) {
      const long k = (long)(j - 1) * mi + (i - 1);
      A[k * n + k] = -(lv->hW[i] + lv->hE[i] + lv->hS[j] + lv->hN[j]);
      if (i > 1) A[k * n + k - 1] = lv->hW[i];
      if (i < mi) A[k * n + k + 1] = lv->hE[i];
      if (j > 1) A[k * n + k - mi] = lv->hS[j];
      if (j < mj) A[k * n + k + mi] = lv->hN[j];
      X[k * n + k] = 1.0;
    }
  if (n == 1) {
    X[0] = A[0];  // divided on the device, as SuperLU does for a 1x1 system
    if (std::fabs(A[0]) < 1e-300) return fail(TMG_SINGULAR, "zero pivot in direct solve");
  } else if (n > 256) {
    // banded LU (bandwidth mi, no pivoting: the five-point operator is a
    // diagonally dominant M-matrix), then the inverse column by column:
    // O(n mi^2 + n^2 mi) instead of Gauss-Jordan's O(n^3)
    const long bw = mi;
    std::vector<double> B((size_t)n * (2 * bw + 1), 0.0);  // B[r][c - r + bw]
    auto at = [&](long r, long c) -> double& { return B[(size_t)r * (2 * bw + 1) + (c - r + bw)]; };
    for (long r = 0; r < n; r++)
      for (long c = std::max(0L, r - bw); c <= std::min(n - 1, r + bw); c++) at(r, c) = A[r * n + c];
    for (long k = 0; k < n; k++) {
      const double p = at(k, k);
      if (std::fabs(p) < 1e-300) return fail(TMG_SINGULAR, "zero pivot in direct solve");
      for (long r = k + 1; r <= std::min(n - 1, k + bw); r++) {
        const double l = at(r, k) / p;
        at(r, k) = l;
        for (long c = k + 1; c <= std::min(n - 1, k + bw); c++) at(r, c) -= l * at(k, c);
      }
    }
    std::vector<double> col((size_t)n);
    for (long c = 0; c < n; c++) {
      std::fill(col.begin(), col.end(), 0.0);
      col[c] = 1.0;
      for (long r = c + 1; r < n; r++) {  // L y = e_c (unit lower, y_r = 0 for r < c)
        double acc = col[r];
        for (long k = std::max(c, r - bw); k < r; k++) acc -= at(r, k) * col[k];
        col[r] = acc;
      }
      for (long r = n - 1; r >= 0; r--) {  // U x = y
        double acc = col[r];
        for (long k = r + 1; k <= std::min(n - 1, r + bw); k++) acc -= at(r, k) * col[k];
        col[r] = acc / at(r, r);
      }
      for (long r = 0; r < n; r++) X[r * n + c] = col[r];
    }
  } else {
    for (long c = 0; c < n; c++) {
      long p = c;
      for (long r = c + 1; r < n; r++)
        if (std::fabs(A[r * n + c]) > std::fabs(A[p * n + c])) p = r;
      if (std::fabs(A[p * n + c]) < 1e-300) return fail(TMG_SINGULAR, "zero pivot in direct solve");
      if (p != c)
        for (long k = 0; k < n; k++) {
          std::swap(A[c * n + k], A[p * n + k]);
          std::swap(X[c * n + k], X[p * n + k]);
        }
      const double inv = 1.0 / A[c * n + c];
      for (long k = 0; k < n; k++) {
        A[c * n + k] *= inv;
        X[c * n + k] *= inv;
      }
      for (long r = 0; r < n; r++) {
        if (r == c) continue;
        const double l = A[r * n + c];
        if (l == 0.0) continue;
        for (long k = 0; k < n; k++) {
          A[r * n + k] -= l * A[c * n + k];
          X[r * n + k] -= l * X[c * n + k];
        }
      }
    }
  }
  TMG_CUDA_TRY(cudaMalloc(&lv->d_ainv, sizeof(double) * (size_t)n * n));
  TMG_CUDA_TRY(cudaMalloc(&lv->d_work, sizeof(double) * (size_t)n));
  TMG_CUDA_TRY(cudaMemcpy(lv->d_ainv, X.data(), sizeof(double) * (size_t)n * n,
                          cudaMemcpyHostToDevice));
  lv->bytes += (long long)(sizeof(double) * (size_t)n * (n + 1));
  return TMG_OK;
}

int fetch_flags_async(tmg_level* lv, cudaStream_t s) {
  TMG_CUDA_TRY(cudaMemcpyAsync(lv->h_err, lv->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  TMG_CUDA_TRY(cudaMemsetAsync(lv->d_err, 0, sizeof(int), s));
  return TMG_OK;
}

int check_fetched(tmg_level* lv) {
  if (*lv->h_err & 1) return fail(TMG_SINGULAR, "zero pivot during block elimination");
  return TMG_OK;
}

int read_flags(tmg_level* lv, cudaStream_t s) {
  int st = fetch_flags_async(lv, s);
  if (st) return st;
  TMG_CUDA_TRY(cudaStreamSynchronize(s));
  return check_fetched(lv);
}

double bits_to_double(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, sizeof(d));
  return d;
}

// work fields of every level in layout `mode` (re-allocated on a mode change)
int ensure_fields(tmg_hier* h, int mode) {
  if (h->mode == mode) return TMG_OK;
  for (double* p : h->blocks) cudaFree(p);
  h->blocks.clear();
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second.first);
  h->graphs.clear();
  for (auto& kv : h->solve_graphs) cudaGraphExecDestroy(kv.second.first);
  h->solve_graphs.clear();
  for (auto& kv : h->tails) {
    cudaFree(kv.second.d_ops);
    if (kv.second.mini) {
      free_mini_tail(*kv.second.mini);
      delete kv.second.mini;
    }
  }
  h->tails.clear();
  h->bytes = 0;
  const int L = (int)h->lv.size();
  h->U.assign(L, FieldView{});
  h->F.assign(L, FieldView{});
  for (int l = 0; l < L; l++) {
    const int nx = h->lv[l]->nx, ny = h->lv[l]->ny;
    // buffers start on 256-byte boundaries (bulk copies need 16-byte alignment)
    const size_t n = ((size_t)(nx + 1) * (ny + 1) + 31) & ~(size_t)31;
    const int nbuf = mode == LM_NATURAL ? 2 : 4;
    double* p = nullptr;
    TMG_CUDA_TRY(cudaMalloc(&p, nbuf * n * sizeof(double)));
    TMG_CUDA_TRY(cudaMemset(p, 0, nbuf * n * sizeof(double)));
    h->blocks.push_back(p);
    h->bytes += (long long)(nbuf * n * sizeof(double));
    double* un = p;
    double* fn = p + n;
    double* ut = mode == LM_NATURAL ? un : p + 2 * n;
    double* ft = mode == LM_NATURAL ? fn : p + 3 * n;
    h->U[l] = FieldView{un, ut, nx, ny, mode};
    h->F[l] = FieldView{fn, ft, nx, ny, mode};
  }
  h->mode = mode;
  h->loaded = false;
  return TMG_OK;
}

size_t field_elems(const FieldView& v) { return (size_t)(v.nx + 1) * (v.ny + 1); }

int zero_field(const FieldView& v, cudaStream_t s) {
  TMG_CUDA_TRY(launch_zero(v.n, field_elems(v), s));
  if (v.t != v.n) TMG_CUDA_TRY(launch_zero(v.t, field_elems(v), s));
  return TMG_OK;
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// smoothing schemes one sweep of `kind` runs (sweep_kind)
std::vector<int> sub_schemes(int kind) {
  if (kind == TMG_ZEBRA_ALT) return {TMG_ZEBRA_X, TMG_ZEBRA_Y};
  if (kind == TMG_TWEED_WIRE_ALT) return {TMG_TWEED, TMG_WIREFRAME};
  return {kind};
}

// First level of the persistent coarse tail (lv.size(): none): the levels
// from there down are at most TMG_TAIL_NMAX (default 1024) points per axis,
// their colour stages are single-CTA block classes (no leg kernel, no
// clusters, no point scheme), and each restricts onto a grid with interior.
// Opt-in (TMG_TAIL=1): measured slower than one PDL graph node per stage
// (coarse tail), kept as a bit-identical alternative.
int tail_start(tmg_hier* h, int kind, int l0) {
  const int L = (int)h->lv.size();
  if (env_int("TMG_TAIL", 0) == 0 || transfer_v1() || L < 2) return L;
  const int nmax = env_int("TMG_TAIL_NMAX", 1024);
  int lt = L;
  for (int l = L - 2; l >= l0; l--) {
    tmg_level* lv = h->lv[l];
    if (std::max(lv->nx, lv->ny) > nmax || lv->nx / 2 < 2 || lv->ny / 2 < 2) break;
    bool ok = true;
    for (int sc : sub_schemes(kind)) {
      Plan* p = nullptr;
      if (get_plan(lv, sc, h->mode, &p)) return L;
      if (p->lp || p->point_scheme) ok = false;
      for (const LaunchClass& c : p->classes)
        if (c.nbins && (c.cs != 1 || c.xcta)) ok = false;
    }
    if (!ok) break;
    lt = l;
  }
  return lt;
}

// Build (once, outside any stream capture) the op list of the tail entered
// at level >= l0; vcycle_launches uses it when present.
// Shared-memory tail (tmg_minitail.cu, default on; TMG_MINI=0 turns it off):
// the levels from the coarsest up whose axes have at most TMG_MINI_NMAX
// (default 32) intervals and whose longest chain / ring / leg has at most
// TMG_MINI_UNIT (default 32) points run as one single-CTA launch.
int prepare_mini_tail(tmg_hier* h, int kind, int full, int nu1, int nu2, int l0) {
  const int L = (int)h->lv.size();
  auto key = std::make_tuple(kind, full, nu1, nu2, l0);
  if (h->tails.count(key) || L < 2 || env_int("TMG_MINI", 1) == 0 || transfer_v1()) return TMG_OK;
  const int nmax = env_int("TMG_MINI_NMAX", 32), umax = env_int("TMG_MINI_UNIT", 32);
  const std::vector<int> schemes = sub_schemes(kind);
  int lt = L;
  for (int l = L - 1; l >= l0; l--) {
    tmg_level* lv = h->lv[l];
    if (std::max(lv->nx, lv->ny) > nmax) break;
    if (l < L - 1) {
      const int mu = mini_max_unit(schemes, lv->nx, lv->ny);
      if (mu < 0 || mu > umax) break;
    }
    lt = l;
  }
  if (lt > L - 2) return TMG_OK;
  int st = factor_coarse(h->lv[L - 1]);
  if (st) return st;
  std::vector<MiniLevelIn> in;
  for (int l = lt; l < L; l++) {
    tmg_level* lv = h->lv[l];
    in.push_back(MiniLevelIn{lv->nx, lv->ny, lv->W, lv->E, lv->S, lv->N});
  }
  MiniTail* mt = new MiniTail();
  const std::string err = build_mini_tail(in, schemes, *mt);
  if (!err.empty()) {  // the per-stage path stays
    delete mt;
    return TMG_OK;
  }
  tmg_hier::TailProg tp;
  tp.level = lt;
  tp.mini = mt;
  h->tails.emplace(key, tp);
  return TMG_OK;
}

int prepare_tail(tmg_hier* h, int kind, int full, int nu1, int nu2, int l0) {
  {
    int st = prepare_mini_tail(h, kind, full, nu1, nu2, l0);
    if (st) return st;
  }
  const int L = (int)h->lv.size();
  const int lt = tail_start(h, kind, l0);
  auto key = std::make_tuple(kind, full, nu1, nu2, l0);
  if (lt >= L - 1 || h->tails.count(key)) return TMG_OK;
  std::vector<TailOp> ops;
  int maxitems = 1, qmax = 1;
  auto sweeps = [&](int l) -> int {
    tmg_level* lv = h->lv[l];
    for (int sc : sub_schemes(kind)) {
      Plan* p = nullptr;
      int st = get_plan(lv, sc, h->mode, &p);
      if (st) return st;
      const SweepArgs a = sweep_args(lv, p, h->U[l], h->F[l]);
      for (int red = 1; red >= 0; red--) {
        int base = 0;
        for (const LaunchClass& c : p->classes) {
          if (c.red != red || c.nbins == 0) continue;
          TailOp o{};
          o.type = TAIL_SWEEP;
          o.q = c.q;
          o.nitems = c.nbins;
          o.base = base;
          o.chunks = c.chunks;
          o.bins = c.bins;
          o.hubs = c.hubs;
          o.sa = a;
          base += c.nbins;
          qmax = std::max(qmax, c.q);
          ops.push_back(o);
        }
        if (base) ops.back().barrier = 1;
        maxitems = std::max(maxitems, base);
      }
    }
    return TMG_OK;
  };
  for (int l = lt; l < L - 1; l++) {
    for (int k = 0; k < nu1; k++) {
      int st = sweeps(l);
      if (st) return st;
    }
    tmg_level* lv = h->lv[l];
    const int nxc = lv->nx / 2, nyc = lv->ny / 2;
    TailOp o{};
    o.type = TAIL_RESTRICT;
    o.barrier = 1;
    o.gx = (nyc - 1 + 14) / 15;
    o.nitems = o.gx * ((nxc - 1 + 14) / 15);
    o.full = full;
    o.g = lv->grid();
    o.U = h->U[l];
    o.F = h->F[l];
    o.CF = h->F[l + 1];
    o.CU = h->U[l + 1];
    ops.push_back(o);
    maxitems = std::max(maxitems, o.nitems);
  }
  {
    tmg_level* lc = h->lv[L - 1];
    int st = factor_coarse(lc);
    if (st) return st;
    const int n = (lc->nx - 1) * (lc->ny - 1);
    if (n > 0) {
      TailOp o{};
      o.type = TAIL_DENSE_RHS;
      o.barrier = 1;
      o.nitems = n;
      o.g = lc->grid();
      o.U = h->U[L - 1];
      o.F = h->F[L - 1];
      o.ainv = lc->d_ainv;
      o.work = lc->d_work;
      ops.push_back(o);
      o.type = TAIL_DENSE_APPLY;
      ops.push_back(o);
      maxitems = std::max(maxitems, (n + kThreads / 32 - 1) / (kThreads / 32));
    }
  }
  for (int l = L - 2; l >= lt; l--) {
    tmg_level* lv = h->lv[l];
    TailOp o{};
    o.type = TAIL_PROLONG;
    o.barrier = 1;
    o.gx = (lv->ny - 1 + 31) / 32;
    o.nitems = o.gx * ((lv->nx - 1 + 31) / 32);
    o.g = lv->grid();
    o.U = h->U[l];
    o.CU = h->U[l + 1];
    ops.push_back(o);
    maxitems = std::max(maxitems, o.nitems);
    for (int k = 0; k < nu2; k++) {
      int st = sweeps(l);
      if (st) return st;
    }
  }
  ops.back().barrier = 0;  // the kernel's end orders the last op
  tmg_hier::TailProg tp;
  int max_ctas = 0;
  TMG_CUDA_TRY(tail_prepare(qmax, &tp.smem, &max_ctas));
  if (max_ctas < 1) return TMG_OK;  // cannot run: the per-stage path stays
  tp.ctas = std::min(std::min(max_ctas, maxitems), std::max(1, env_int("TMG_TAIL_CTAS", 1 << 20)));
  tp.nops = (int)ops.size();
  tp.level = lt;
  if (!h->d_tail_bar) {
    TMG_CUDA_TRY(cudaMalloc(&h->d_tail_bar, 2 * sizeof(unsigned)));
    TMG_CUDA_TRY(cudaMemset(h->d_tail_bar, 0, 2 * sizeof(unsigned)));
  }
  TMG_CUDA_TRY(cudaMalloc(&tp.d_ops, ops.size() * sizeof(TailOp)));
  TMG_CUDA_TRY(cudaMemcpy(tp.d_ops, ops.data(), ops.size() * sizeof(TailOp),
                          cudaMemcpyHostToDevice));
  h->tails.emplace(key, tp);
  return TMG_OK;
}

// one V-cycle on the hierarchy's work fields (mgcycle.py:89-104), entered at
// level l0 (0: the whole cycle; > 0: the replicated tail of a sharded cycle)
int vcycle_launches(tmg_hier* h, int kind, int full, int nu1, int nu2, cudaStream_t s,
                    int l0 = 0) {
  const int L = (int)h->lv.size();
  // levels >= lt run inside one persistent tail launch (prepare_tail)
  auto tit = h->tails.find(std::make_tuple(kind, full, nu1, nu2, l0));
  const tmg_hier::TailProg* tp = tit == h->tails.end() ? nullptr : &tit->second;
  const int lt = tp ? tp->level : L - 1;
  for (int l = l0; l < lt; l++) {  // down: smooth, residual + restriction, zero guess
    tmg_level* lv = h->lv[l];
    for (int k = 0; k < nu1; k++) {
      int st = sweep_kind(lv, kind, 3, h->U[l], h->F[l], s);
      if (st) return st;
    }
    bool zeroed = false;  // the restriction wrote the coarse zero guess itself
    cudaError_t e = launch_hdefect_restrict(lv->grid(), full, h->U[l], h->F[l], h->F[l + 1], s,
                                            &h->U[l + 1], &zeroed);
    if (e != cudaSuccess) return cuda_fail(e, "defect_restrict");
    if (!zeroed) {
      int st = zero_field(h->U[l + 1], s);
      if (st) return st;
    }
  }
  if (tp && tp->mini) {
    cudaError_t e = launch_mini_tail(*tp->mini, h->U[lt], h->F[lt], h->lv[L - 1]->d_ainv, full & 1,
                                     nu1, nu2, h->lv[lt]->d_err, s);
    if (e != cudaSuccess) return cuda_fail(e, "shared-memory coarse tail");
  } else if (tp) {
    cudaError_t e = launch_tail(tp->d_ops, tp->nops, tp->ctas, tp->smem, h->d_tail_bar, s);
    if (e != cudaSuccess) return cuda_fail(e, "coarse tail");
  } else {  // coarsest level: direct solve (mgcycle.py:93-95)
    tmg_level* lc = h->lv[L - 1];
    int st = factor_coarse(lc);
    if (st) return st;
    cudaError_t e = launch_hdense_solve(lc->grid(), lc->d_ainv, h->U[L - 1], h->F[L - 1],
                                        lc->d_work, s);
    if (e != cudaSuccess) return cuda_fail(e, "coarse solve");
  }
  for (int l = lt - 1; l >= l0; l--) {  // up: prolongation + correction, smooth
    tmg_level* lv = h->lv[l];
    // the post-smoothing's first red stage overwrites the red points of a square
    // tweed level unread: the correction goes to the black ones only
    // (TMG_PROLONG_BLACK=0: everywhere).  Hybrid layout only: its sweeps are
    // bit-identical with and without (tools/dbg_black.py); the natural-layout
    // gather reads in-block values it cancels later, so it keeps the full
    // correction.
    static const int black_only = env_int("TMG_PROLONG_BLACK", 1);
    const int skip_red = black_only && nu2 > 0 && kind == TMG_TWEED && h->mode == LM_TWEED &&
                         lv->nx == lv->ny && lv->nx % 2 == 0 && lv->nx >= 4;
    cudaError_t e = launch_hprolong_correct(lv->nx, lv->ny, h->U[l + 1], h->U[l], s, skip_red);
    if (e != cudaSuccess) return cuda_fail(e, "prolong_correct");
    for (int k = 0; k < nu2; k++) {
      int st = sweep_kind(lv, kind, 3, h->U[l], h->F[l], s);
      if (st) return st;
    }
  }
  return TMG_OK;
}

int check_hier_args(tmg_hier* h, int kind, int nu1, int nu2) {
  if (!h || h->lv.empty()) return fail(TMG_BADARG, "null hierarchy");
  if (!valid_kind(kind)) return fail(TMG_BADARG, "unknown smoother " + std::to_string(kind));
  if (nu1 < 0 || nu2 < 0 || nu1 + nu2 < 1)
    return fail(TMG_BADARG, "need nu1, nu2 >= 0 with nu1 + nu2 >= 1");
  return TMG_OK;
}

// plans and coarse factors allocate: build them before any stream capture
int prepare(tmg_hier* h, int kind) {
  int sub[2] = {kind, -1};
  if (kind == TMG_ZEBRA_ALT) {
    sub[0] = TMG_ZEBRA_X;
    sub[1] = TMG_ZEBRA_Y;
  }
  if (kind == TMG_TWEED_WIRE_ALT) {
    sub[0] = TMG_TWEED;
    sub[1] = TMG_WIREFRAME;
  }
  for (size_t l = 0; l + 1 < h->lv.size(); l++)
    for (int k : sub) {
      if (k < 0) continue;
      Plan* p;
      int st = get_plan(h->lv[l], k, h->mode, &p);
      if (st) return st;
    }
  return factor_coarse(h->lv.back());
}

int session_load(tmg_hier* h, int kind, const double* u, const double* f, cudaStream_t s) {
  int st = ensure_fields(h, session_mode(kind));
  if (st) return st;
  cudaError_t e = launch_to_hybrid(h->U[0], u, s);
  if (e == cudaSuccess) e = launch_to_hybrid(h->F[0], f, s);
  if (e != cudaSuccess) return cuda_fail(e, "layout conversion");
  h->loaded = true;
  return TMG_OK;
}

int session_store(tmg_hier* h, double* u, cudaStream_t s) {
  if (!h->loaded) return fail(TMG_BADARG, "no solver session loaded");
  cudaError_t e = launch_from_hybrid(h->U[0], u, s);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "layout conversion");
}

int session_norm_async(tmg_hier* h, cudaStream_t s);

int session_cycles(tmg_hier* h, int kind, int full, int nu1, int nu2, int reps, cudaStream_t s) {
  if (!h->loaded) return fail(TMG_BADARG, "no solver session loaded");
  if (session_mode(kind) != h->mode)
    return fail(TMG_BADARG, "smoother kind does not match the loaded session's layout");
  auto key = std::make_tuple(kind, full, nu1, nu2);
  auto it = h->graphs.find(key);
  if (it == h->graphs.end()) {
    int st = prepare(h, kind);
    if (!st) st = prepare_tail(h, kind, full & 1, nu1, nu2, 0);
    if (st) return st;
    cudaStream_t cs;
    TMG_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g;
    const long long counted = launch_counter();  // captured launches do not run
    TMG_CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    // full & 2: the host solve loop's check (defect norm, pivot flags of
    // every level) rides in the same graph, one launch and one sync per cycle
    // (tmg_solve's fallback when the while-node graph is unavailable)
    int st3 = vcycle_launches(h, kind, full & 1, nu1, nu2, cs);
    if (!st3 && (full & 2)) {
      st3 = session_norm_async(h, cs);
      for (auto* lv : h->lv)
        if (!st3) st3 = fetch_flags_async(lv, cs);
    }
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    launch_counter() = counted;
    cudaStreamDestroy(cs);
    if (st3) return st3;
    if (e != cudaSuccess) return cuda_fail(e, "graph capture");
    size_t nn = 0;
    TMG_CUDA_TRY(cudaGraphGetNodes(g, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    TMG_CUDA_TRY(cudaGraphGetNodes(g, nodes.data(), &nn));
    int kernels = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      TMG_CUDA_TRY(cudaGraphNodeGetType(nd, &t));
      kernels += (t == cudaGraphNodeTypeKernel);
    }
    cudaGraphExec_t ge;
    TMG_CUDA_TRY(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    it = h->graphs.emplace(key, std::make_pair(ge, kernels)).first;
  }
  h->last_kernels = it->second.second;
  for (int r = 0; r < reps; r++) {
    TMG_CUDA_TRY(cudaGraphLaunch(it->second.first, s));
    TMG_COUNT(it->second.second);
  }
  return TMG_OK;
}

int session_norm_async(tmg_hier* h, cudaStream_t s) {
  tmg_level* fine = h->lv[0];
  TMG_CUDA_TRY(cudaMemsetAsync(fine->d_norm, 0, sizeof(unsigned long long), s));
  cudaError_t e = launch_hdefect_norm(fine->grid(), h->U[0], h->F[0], fine->d_norm, s);
  if (e != cudaSuccess) return cuda_fail(e, "defect_norm");
  TMG_CUDA_TRY(cudaMemcpyAsync(fine->h_norm, fine->d_norm, sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s));
  return TMG_OK;
}

int flags_all(tmg_hier* h, cudaStream_t s) {
  for (auto* lv : h->lv) {
    int st = fetch_flags_async(lv, s);
    if (st) return st;
  }
  TMG_CUDA_TRY(cudaStreamSynchronize(s));
  for (auto* lv : h->lv) {
    int st = check_fetched(lv);
    if (st) return st;
  }
  return TMG_OK;
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const std::exception& ex) {
    return fail(TMG_CUDA, ex.what());
  }
}

}  // namespace

namespace tmg {
thread_local bool g_pdl_off = false;  // set while capturing a body that may not use PDL

bool pdl_enabled() {
  if (g_pdl_off) return false;
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("TMG_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

long long& launch_counter() {
  static long long n = 0;
  return n;
}
}  // namespace tmg

extern "C" {

const char* tmg_last_error(void) { return g_last_error.c_str(); }
long long tmg_kernel_launches(void) { return launch_counter(); }
int tmg_version(void) { return 110; }

int tmg_level_create(int nx, int ny, const double* W, const double* E, const double* S,
                     const double* N, tmg_level** out) {
  return guarded([&]() -> int {
    if (!out) return fail(TMG_BADARG, "null output handle");
    if (nx < 2 || ny < 2) return fail(TMG_BADARG, "grid needs nx, ny >= 2");
    tmg_level* lv = new tmg_level();
    lv->nx = nx;
    lv->ny = ny;
    cudaGetDevice(&lv->device);
    lv->hW.assign(W, W + nx + 1);
    lv->hE.assign(E, E + nx + 1);
    lv->hS.assign(S, S + ny + 1);
    lv->hN.assign(N, N + ny + 1);
    size_t bx = sizeof(double) * (nx + 1), by = sizeof(double) * (ny + 1);
    TMG_CUDA_TRY(cudaMalloc(&lv->W, 2 * bx + 2 * by));
    lv->E = lv->W + (nx + 1);
    lv->S = lv->E + (nx + 1);
    lv->N = lv->S + (ny + 1);
    TMG_CUDA_TRY(cudaMemcpy(lv->W, W, bx, cudaMemcpyHostToDevice));
    TMG_CUDA_TRY(cudaMemcpy(lv->E, E, bx, cudaMemcpyHostToDevice));
    TMG_CUDA_TRY(cudaMemcpy(lv->S, S, by, cudaMemcpyHostToDevice));
    TMG_CUDA_TRY(cudaMemcpy(lv->N, N, by, cudaMemcpyHostToDevice));
    TMG_CUDA_TRY(cudaMalloc(&lv->d_err, sizeof(int) * 2 + sizeof(unsigned long long) * 2));
    lv->d_norm = reinterpret_cast<unsigned long long*>(lv->d_err + 2);
    TMG_CUDA_TRY(cudaMemset(lv->d_err, 0, sizeof(int)));
    TMG_CUDA_TRY(cudaMallocHost(&lv->h_err, sizeof(int) * 2 + sizeof(unsigned long long) * 2));
    lv->h_norm = reinterpret_cast<unsigned long long*>(lv->h_err + 2);
    lv->bytes = (long long)(2 * bx + 2 * by);
    *out = lv;
    return TMG_OK;
  });
}

int tmg_level_destroy(tmg_level* lv) {
  if (!lv) return TMG_OK;
  for (auto& row : lv->plans)
    for (auto& p : row)
      if (p) {
        free_plan(*p);
        delete p;
      }
  for (auto& kv : lv->part_plans) {
    free_plan(*kv.second);
    delete kv.second;
  }
  cudaFree(lv->W);
  cudaFree(lv->d_err);
  cudaFreeHost(lv->h_err);
  cudaFree(lv->d_ainv);
  cudaFree(lv->d_work);
  delete lv;
  return TMG_OK;
}

long long tmg_level_device_bytes(tmg_level* lv) { return lv ? lv->bytes : 0; }

int tmg_level_check(tmg_level* lv, void* stream) {
  if (!lv) return fail(TMG_BADARG, "null level");
  return read_flags(lv, (cudaStream_t)stream);
}

int tmg_sweep(tmg_level* lv, int kind, double* u, const double* f, void* stream) {
  if (!lv) return fail(TMG_BADARG, "null level");
  return guarded([&] {
    return sweep_kind(lv, kind, 3, natural_view(lv, u), natural_view(lv, const_cast<double*>(f)),
                      (cudaStream_t)stream);
  });
}

int tmg_sweep_colour(tmg_level* lv, int kind, int red, double* u, const double* f, void* stream) {
  if (!lv) return fail(TMG_BADARG, "null level");
  return guarded([&] {
    return sweep_kind(lv, kind, red ? 1 : 2, natural_view(lv, u),
                      natural_view(lv, const_cast<double*>(f)), (cudaStream_t)stream);
  });
}

int tmg_apply(tmg_level* lv, const double* u, double* out, void* stream) {
  if (!lv) return fail(TMG_BADARG, "null level");
  cudaError_t e = launch_apply(lv->grid(), u, nullptr, out, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "apply");
}

int tmg_defect(tmg_level* lv, const double* u, const double* f, double* d, void* stream) {
  if (!lv) return fail(TMG_BADARG, "null level");
  cudaError_t e = launch_apply(lv->grid(), u, f, d, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "defect");
}

int tmg_defect_norm(tmg_level* lv, const double* u, const double* f, double* out_host,
                    void* stream) {
  if (!lv) return fail(TMG_BADARG, "null level");
  cudaStream_t s = (cudaStream_t)stream;
  TMG_CUDA_TRY(cudaMemsetAsync(lv->d_norm, 0, sizeof(unsigned long long), s));
  cudaError_t e = launch_defect_norm(lv->grid(), u, f, lv->d_norm, s);
  if (e != cudaSuccess) return cuda_fail(e, "defect_norm");
  TMG_CUDA_TRY(cudaMemcpyAsync(lv->h_norm, lv->d_norm, sizeof(unsigned long long),
                               cudaMemcpyDeviceToHost, s));
  TMG_CUDA_TRY(cudaStreamSynchronize(s));
  *out_host = bits_to_double(*lv->h_norm);
  return TMG_OK;
}

int tmg_vec_norm2(const double* x, long n, double* work, double* out_host, void* stream) {
  if (n < 0 || (!x && n)) return fail(TMG_BADARG, "bad vector");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_vec_norm2(x, n, work, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out_host, work, sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "vec_norm2");
}

int tmg_lcg_fill(unsigned long long state, long n, double* out, void* stream) {
  cudaError_t e = launch_lcg_fill(state, n, out, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "lcg_fill");
}

int tmg_vec_scale(double* x, long n, double alpha, void* stream) {
  cudaError_t e = launch_vec_scale(x, n, alpha, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "vec_scale");
}

int tmg_restrict(int nxf, int nyf, int full, const double* d, double* out, void* stream) {
  if (nxf % 2 || nyf % 2 || nxf < 2 || nyf < 2)
    return fail(TMG_BADARG, "fine grid cannot be halved");
  cudaError_t e = launch_restrict(nxf, nyf, full, d, out, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "restrict");
}

int tmg_prolong(int nxc, int nyc, const double* uc, double* v, void* stream) {
  if (nxc < 2 || nyc < 2) return fail(TMG_BADARG, "coarse grid has no interior to interpolate");
  cudaError_t e = launch_prolong(nxc, nyc, uc, v, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "prolong");
}

int tmg_defect_restrict(tmg_level* fine, int full, const double* u, const double* f, double* fc,
                        void* stream) {
  if (!fine) return fail(TMG_BADARG, "null level");
  if (fine->nx % 2 || fine->ny % 2) return fail(TMG_BADARG, "fine grid cannot be halved");
  cudaError_t e = launch_defect_restrict(fine->grid(), full, u, f, fc, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "defect_restrict");
}

int tmg_prolong_correct(int nxc, int nyc, const double* uc, double* u, void* stream) {
  cudaError_t e = launch_prolong_correct(nxc, nyc, uc, u, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "prolong_correct");
}

int tmg_direct_solve(tmg_level* lv, double* u, const double* f, void* stream) {
  if (!lv) return fail(TMG_BADARG, "null level");
  return guarded([&]() -> int {
    int st = factor_coarse(lv);
    if (st) return st;
    cudaError_t e =
        launch_dense_solve(lv->grid(), lv->d_ainv, u, f, lv->d_work, (cudaStream_t)stream);
    return e == cudaSuccess ? TMG_OK : cuda_fail(e, "direct solve");
  });
}

int tmg_hier_create(int nlevels, tmg_level* const* levels, tmg_hier** out) {
  return guarded([&]() -> int {
    if (nlevels < 1 || !levels || !out) return fail(TMG_BADARG, "bad hierarchy arguments");
    for (int l = 1; l < nlevels; l++)
      if (levels[l]->nx * 2 != levels[l - 1]->nx || levels[l]->ny * 2 != levels[l - 1]->ny)
        return fail(TMG_BADARG, "each level must halve the previous one");
    tmg_hier* h = new tmg_hier();
    h->lv.assign(levels, levels + nlevels);
    *out = h;
    return TMG_OK;
  });
}

int tmg_hier_destroy(tmg_hier* h) {
  if (!h) return TMG_OK;
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second.first);
  for (auto& kv : h->solve_graphs) cudaGraphExecDestroy(kv.second.first);
  cudaFree(h->d_solve);
  for (auto& kv : h->tails) {
    cudaFree(kv.second.d_ops);
    if (kv.second.mini) {
      free_mini_tail(*kv.second.mini);
      delete kv.second.mini;
    }
  }
  cudaFree(h->d_tail_bar);
  for (double* p : h->blocks) cudaFree(p);
  delete h;
  return TMG_OK;
}

int tmg_hier_graph_kernels(tmg_hier* h) { return h ? h->last_kernels : 0; }

long long tmg_hier_device_bytes(tmg_hier* h) { return h ? h->bytes : 0; }

int tmg_session_load(tmg_hier* h, int kind, const double* u, const double* f, void* stream) {
  if (!h || h->lv.empty()) return fail(TMG_BADARG, "null hierarchy");
  if (!valid_kind(kind)) return fail(TMG_BADARG, "unknown smoother " + std::to_string(kind));
  return guarded([&] { return session_load(h, kind, u, f, (cudaStream_t)stream); });
}

int tmg_session_cycles(tmg_hier* h, int kind, int full, int nu1, int nu2, int reps,
                       void* stream) {
  int st = check_hier_args(h, kind, nu1, nu2);
  if (st) return st;
  return guarded(
      [&] { return session_cycles(h, kind, full ? 1 : 0, nu1, nu2, reps, (cudaStream_t)stream); });
}

int tmg_session_norm(tmg_hier* h, double* out_host, void* stream) {
  if (!h || !h->loaded) return fail(TMG_BADARG, "no solver session loaded");
  return guarded([&]() -> int {
    cudaStream_t s = (cudaStream_t)stream;
    int st = session_norm_async(h, s);
    if (st) return st;
    st = flags_all(h, s);
    if (st) return st;
    *out_host = bits_to_double(*h->lv[0]->h_norm);
    return TMG_OK;
  });
}

int tmg_session_store(tmg_hier* h, double* u, void* stream) {
  if (!h) return fail(TMG_BADARG, "null hierarchy");
  return guarded([&] { return session_store(h, u, (cudaStream_t)stream); });
}

int tmg_session_sweeps(tmg_hier* h, int kind, int reps, void* stream) {
  if (!h || !h->loaded) return fail(TMG_BADARG, "no solver session loaded");
  if (!valid_kind(kind) || session_mode(kind) != h->mode)
    return fail(TMG_BADARG, "smoother kind does not match the loaded session's layout");
  return guarded([&]() -> int {
    for (int r = 0; r < reps; r++) {
      int st = sweep_kind(h->lv[0], kind, 3, h->U[0], h->F[0], (cudaStream_t)stream);
      if (st) return st;
    }
    return TMG_OK;
  });
}

int tmg_vcycle_graph(tmg_hier* h, int kind, int full, int nu1, int nu2, double* u,
                     const double* f, int reps, void* stream) {
  int st = check_hier_args(h, kind, nu1, nu2);
  if (st) return st;
  return guarded([&]() -> int {
    cudaStream_t s = (cudaStream_t)stream;
    int st2 = session_load(h, kind, u, f, s);
    if (!st2) st2 = session_cycles(h, kind, full ? 1 : 0, nu1, nu2, reps, s);
    if (!st2) st2 = session_store(h, u, s);
    return st2;
  });
}

int tmg_vcycle(tmg_hier* h, int kind, int full, int nu1, int nu2, double* u, const double* f,
               void* stream) {
  return tmg_vcycle_graph(h, kind, full, nu1, nu2, u, f, 1, stream);
}

}  // extern "C"

namespace {
// after a cycle: record its defect norm, stop on convergence, a non-finite
// norm, a vanishing pivot or max_cycles (the host loop's rule, same order)
__global__ void solve_check_kernel(cudaGraphConditionalHandle hdl, SolveDev* sd,
                                   unsigned long long* d_norm, ErrPtrs e) {
  unsigned long long b = *d_norm;
  *d_norm = 0ull;  // the next cycle's norm accumulates from zero
  double dn;
  memcpy(&dn, &b, sizeof(dn));
  const int c = sd->cycle + 1;
  sd->cycle = c;
  sd->norms[c] = dn;
  int err = 0;
  for (int k = 0; k < e.n; k++) err |= *e.p[k];
  sd->err = err;
  bool stop = (err & 1) || c >= sd->max_cycles || !isfinite(dn);
  if (!(err & 1) && isfinite(dn) && dn <= sd->tol * sd->d0) {
    sd->converged = 1;
    stop = true;
  }
  cudaGraphSetConditional(hdl, stop ? 0u : 1u);
}
}  // namespace

cudaError_t tmg::launch_solve_check(cudaStream_t s, cudaGraphConditionalHandle hdl, SolveDev* sd,
                               unsigned long long* d_norm, const ErrPtrs& e) {
  solve_check_kernel<<<1, 1, 0, s>>>(hdl, sd, d_norm, e);
  return cudaGetLastError();
}

int tmg::build_while_graph(const std::function<int(cudaStream_t, cudaGraphConditionalHandle)>& body,
                      cudaGraphExec_t* out, int* kernels_per_cycle) {
  cudaError_t last = cudaSuccess;
  for (int attempt = 0; attempt < 2; attempt++) {
    cudaGraph_t g = nullptr;
    TMG_CUDA_TRY(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hdl;
    cudaGraphExec_t ge = nullptr;
    int kernels = 0;
    cudaError_t e = cudaGraphConditionalHandleCreate(&hdl, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hdl;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    if (e == cudaSuccess) e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
    if (e == cudaSuccess) {
      cudaGraph_t bg = cp.conditional.phGraph_out[0];
      cudaStream_t cs;
      TMG_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      const long long counted = launch_counter();
      g_pdl_off = attempt == 1;
      e = cudaStreamBeginCaptureToGraph(cs, bg, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeThreadLocal);
      int st3 = TMG_OK;
      if (e == cudaSuccess) {
        st3 = body(cs, hdl);
        cudaGraph_t captured = nullptr;
        cudaError_t e3 = cudaStreamEndCapture(cs, &captured);
        if (e == cudaSuccess) e = e3;
      }
      g_pdl_off = false;
      launch_counter() = counted;
      cudaStreamDestroy(cs);
      if (st3) {
        cudaGraphDestroy(g);
        // a launch refused inside the capture (e.g. PDL in a conditional
        // body): clear it and retry once without PDL
        if (attempt == 0 && st3 == TMG_CUDA) {
          cudaGetLastError();
          last = cudaErrorNotSupported;
          continue;
        }
        return st3;
      }
      if (e == cudaSuccess) {
        size_t nn = 0;
        e = cudaGraphGetNodes(bg, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        if (e == cudaSuccess) e = cudaGraphGetNodes(bg, nodes.data(), &nn);
        for (size_t k = 0; e == cudaSuccess && k < nn; k++) {
          cudaGraphNodeType t;
          e = cudaGraphNodeGetType(nodes[k], &t);
          kernels += (t == cudaGraphNodeTypeKernel);
        }
      }
      if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
    }
    cudaGraphDestroy(g);
    if (e == cudaSuccess) {
      *out = ge;
      *kernels_per_cycle = kernels;
      return TMG_OK;
    }
    cudaGetLastError();  // clear a refused capture before the retry without PDL
    last = e;
  }
  return cuda_fail(last, "solve graph");
}

extern "C" {

namespace {
// one graph per (kind, full, nu1, nu2): a while-node whose body is the
// V-cycle, the defect norm and the check kernel -- no host round trip per
// cycle.
int solve_graph(tmg_hier* h, int kind, int full, int nu1, int nu2, cudaGraphExec_t* out,
                int* kernels_per_cycle) {
  auto key = std::make_tuple(kind, full, nu1, nu2);
  auto it = h->solve_graphs.find(key);
  if (it != h->solve_graphs.end()) {
    *out = it->second.first;
    *kernels_per_cycle = it->second.second;
    return TMG_OK;
  }
  int st = prepare(h, kind);
  if (!st) st = prepare_tail(h, kind, full, nu1, nu2, 0);
  if (st) return st;
  if (h->lv.size() > 32) return fail(TMG_BADARG, "too many levels for the solve graph");
  ErrPtrs ep{};
  ep.n = (int)h->lv.size();
  for (int k = 0; k < ep.n; k++) ep.p[k] = h->lv[k]->d_err;
  st = build_while_graph(
      [&](cudaStream_t cs, cudaGraphConditionalHandle hdl) -> int {
        int st3 = vcycle_launches(h, kind, full, nu1, nu2, cs);
        if (st3) return st3;
        tmg_level* fine = h->lv[0];
        cudaError_t e2 = launch_hdefect_norm(fine->grid(), h->U[0], h->F[0], fine->d_norm, cs);
        if (e2 == cudaSuccess) e2 = launch_solve_check(cs, hdl, h->d_solve, fine->d_norm, ep);
        return e2 == cudaSuccess ? TMG_OK : cuda_fail(e2, "solve graph body");
      },
      out, kernels_per_cycle);
  if (st) return st;
  h->solve_graphs.emplace(key, std::make_pair(*out, *kernels_per_cycle));
  return TMG_OK;
}

int ensure_solve_state(tmg_hier* h, int max_cycles) {
  if (h->d_solve && h->solve_cap >= max_cycles) return TMG_OK;
  for (auto& kv : h->solve_graphs) cudaGraphExecDestroy(kv.second.first);
  h->solve_graphs.clear();  // the graphs bake the state's address
  cudaFree(h->d_solve);
  h->d_solve = nullptr;
  const int cap = max_cycles > 64 ? max_cycles : 64;
  TMG_CUDA_TRY(cudaMalloc(&h->d_solve, sizeof(SolveDev) + sizeof(double) * (size_t)cap));
  h->solve_cap = cap;
  return TMG_OK;
}
}  // namespace

int tmg_solve(tmg_hier* h, int kind, int full, int nu1, int nu2, double tol, int max_cycles,
              double* u, const double* f, double* norms_out, int* cycles_out, int* converged_out,
              void* stream) {
  int st = check_hier_args(h, kind, nu1, nu2);
  if (st) return st;
  if (!(tol > 0)) return fail(TMG_BADARG, "tol must be positive");
  return guarded([&]() -> int {
    cudaStream_t s = (cudaStream_t)stream;
    *cycles_out = 0;
    *converged_out = 0;
    int st2 = session_load(h, kind, u, f, s);
    if (!st2) st2 = session_norm_async(h, s);
    if (st2) return st2;
    TMG_CUDA_TRY(cudaStreamSynchronize(s));
    const double d0 = bits_to_double(*h->lv[0]->h_norm);
    norms_out[0] = d0;
    if (d0 == 0.0) {  // mgcycle.py:124-126
      *converged_out = 1;
      return session_store(h, u, s);
    }
    if (max_cycles < 1) return session_store(h, u, s);
    // mgcycle.py:128-138 on the device: one launch of the while-node graph
    st2 = ensure_solve_state(h, max_cycles);
    cudaGraphExec_t ge;
    int per_cycle = 0;
    const char* force_host = std::getenv("TMG_SOLVE_HOST");
    if (!st2 && force_host && force_host[0] == '1') st2 = TMG_CUDA;
    else if (!st2) st2 = solve_graph(h, kind, full ? 1 : 0, nu1, nu2, &ge, &per_cycle);
    if (st2 == TMG_CUDA) {
      // no conditional-node support (driver / capture refused): the same
      // loop driven from the host, one graph launch and one sync per cycle
      cudaGetLastError();
      for (int c = 1; c <= max_cycles; c++) {
        st2 = session_cycles(h, kind, (full ? 1 : 0) | 2, nu1, nu2, 1, s);
        if (st2) return st2;
        TMG_CUDA_TRY(cudaStreamSynchronize(s));
        for (auto* lv : h->lv) {
          st2 = check_fetched(lv);
          if (st2) return st2;
        }
        const double dn = bits_to_double(*h->lv[0]->h_norm);
        norms_out[c] = dn;
        *cycles_out = c;
        if (!std::isfinite(dn)) break;
        if (dn <= tol * d0) {
          *converged_out = 1;
          break;
        }
      }
      return session_store(h, u, s);
    }
    if (st2) return st2;
    SolveDev hs = {};
    hs.d0 = d0;
    hs.tol = tol;
    hs.max_cycles = max_cycles;
    TMG_CUDA_TRY(cudaMemcpyAsync(h->d_solve, &hs, offsetof(SolveDev, norms), cudaMemcpyHostToDevice, s));
    TMG_CUDA_TRY(cudaMemsetAsync(h->lv[0]->d_norm, 0, sizeof(unsigned long long), s));
    TMG_CUDA_TRY(cudaGraphLaunch(ge, s));
    TMG_CUDA_TRY(cudaMemcpyAsync(&hs, h->d_solve, offsetof(SolveDev, norms), cudaMemcpyDeviceToHost, s));
    TMG_CUDA_TRY(cudaStreamSynchronize(s));
    TMG_COUNT((long long)per_cycle * hs.cycle);
    std::vector<double> nv((size_t)hs.cycle + 1);
    TMG_CUDA_TRY(cudaMemcpy(nv.data(), h->d_solve->norms, sizeof(double) * nv.size(),
                            cudaMemcpyDeviceToHost));
    st2 = flags_all(h, s);  // raises on a vanishing pivot (and clears the flags)
    if (st2) return st2;
    for (int c = 1; c <= hs.cycle; c++) norms_out[c] = nv[(size_t)c];
    *cycles_out = hs.cycle;
    *converged_out = hs.converged;
    return session_store(h, u, s);
  });
}

// ---- sharded V-cycle support (one rank's share) ----

int tmg_group_count(int kind, int nx, int ny) {
  if (!valid_kind(kind) || nx < 2 || ny < 2) return 0;
  return group_count(kind, nx, ny);
}

long tmg_group_sizes(int kind, int nx, int ny, long long* sizes, long cap) {
  const int G = tmg_group_count(kind, nx, ny);
  if (G < 1) {
    g_last_error = "smoother kind " + std::to_string(kind) + " does not shard";
    return -1;
  }
  if (cap < G + 1) return G + 1;
  for (int g = 0; g <= G; g++) sizes[g] = 0;
  for (int i = 1; i < nx; i++)
    for (int j = 1; j < ny; j++) sizes[point_group(kind, nx, ny, i, j)]++;
  return G + 1;
}

long tmg_group_offsets(int kind, int nx, int ny, int g0, int g1, long long* enc, long cap) {
  const int G = tmg_group_count(kind, nx, ny);
  if (G < 1) {
    g_last_error = "smoother kind " + std::to_string(kind) + " does not shard";
    return -1;
  }
  const FieldView v{nullptr, nullptr, nx, ny, session_mode(kind)};
  long n = 0;
  for (int i = 1; i < nx; i++)
    for (int j = 1; j < ny; j++) {
      const int grp = point_group(kind, nx, ny, i, j);
      if (grp < g0 || grp >= g1) continue;
      if (n < cap) {
        const bool t = owns_t(v.mode, nx, ny, i, j);
        enc[n] = 2 * (long long)(t ? v.off_t(i, j) : v.off_n(i, j)) + (t ? 1 : 0);
      }
      n++;
    }
  return n;
}

}  // extern "C"

namespace {
int session_level(tmg_hier* h, int level, int need_coarser) {
  if (!h || !h->loaded) return fail(TMG_BADARG, "no solver session loaded");
  if (level < 0 || level >= (int)h->lv.size() - need_coarser)
    return fail(TMG_BADARG, "level " + std::to_string(level) + " out of range");
  return TMG_OK;
}
}  // namespace

extern "C" {

int tmg_session_sweep_part(tmg_hier* h, int level, int kind, int red, int g0, int g1,
                           void* stream) {
  int st = session_level(h, level, 0);
  if (st) return st;
  if (!valid_kind(kind) || session_mode(kind) != h->mode)
    return fail(TMG_BADARG, "smoother kind does not match the loaded session's layout");
  return guarded([&]() -> int {
    tmg_level* lv = h->lv[level];
    Plan* p = nullptr;
    int st2 = get_part_plan(lv, kind, h->mode, g0, g1, &p);
    if (st2) return st2;
    cudaError_t e = launch_colour(*p, red ? 1 : 0, sweep_args(lv, p, h->U[level], h->F[level]),
                                  (cudaStream_t)stream);
    return e == cudaSuccess ? TMG_OK : cuda_fail(e, "sweep launch");
  });
}

int tmg_session_restrict(tmg_hier* h, int level, int full, void* stream) {
  int st = session_level(h, level, 1);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_hdefect_restrict(h->lv[level]->grid(), full, h->U[level], h->F[level],
                                          h->F[level + 1], s);
  if (e != cudaSuccess) return cuda_fail(e, "defect_restrict");
  return zero_field(h->U[level + 1], s);
}

int tmg_session_restrict_part(tmg_hier* h, int level, int full, int kind, int cg0, int cg1,
                              void* stream) {
  int st = session_level(h, level, 1);
  if (st) return st;
  if (!valid_kind(kind) || cg0 < 1 || cg1 <= cg0)
    return fail(TMG_BADARG, "bad kind or coarse group range");
  cudaError_t e = launch_restrict2(h->lv[level]->grid(), full, h->U[level], h->F[level],
                                   h->F[level + 1], (cudaStream_t)stream, &h->U[level + 1], kind,
                                   cg0, cg1);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "defect_restrict part");
}

int tmg_session_prolong_part(tmg_hier* h, int level, int kind, int fg0, int fg1, void* stream) {
  int st = session_level(h, level, 1);
  if (st) return st;
  if (!valid_kind(kind) || fg0 < 1 || fg1 <= fg0)
    return fail(TMG_BADARG, "bad kind or fine group range");
  tmg_level* lv = h->lv[level];
  cudaError_t e = launch_prolong2(lv->nx, lv->ny, h->U[level + 1], h->U[level],
                                  (cudaStream_t)stream, kind, fg0, fg1);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "prolong_correct part");
}

int tmg_session_read(tmg_hier* h, int level, int which, double* out, void* stream) {
  if (!h || !h->loaded) return fail(TMG_BADARG, "no solver session loaded");
  if (level < 0 || level >= (int)h->lv.size() || (which != 0 && which != 1))
    return fail(TMG_BADARG, "bad level or field");
  const FieldView& v = which ? h->F[level] : h->U[level];
  cudaError_t e = launch_from_hybrid(v, out, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "session read");
}

int tmg_session_prolong(tmg_hier* h, int level, void* stream) {
  int st = session_level(h, level, 1);
  if (st) return st;
  tmg_level* lv = h->lv[level];
  cudaError_t e = launch_hprolong_correct(lv->nx, lv->ny, h->U[level + 1], h->U[level],
                                          (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "prolong_correct");
}

int tmg_session_tail(tmg_hier* h, int level, int kind, int full, int nu1, int nu2, void* stream) {
  int st = check_hier_args(h, kind, nu1, nu2);
  if (!st) st = session_level(h, level, 0);
  if (st) return st;
  if (session_mode(kind) != h->mode)
    return fail(TMG_BADARG, "smoother kind does not match the loaded session's layout");
  return guarded([&]() -> int {
    int st2 = prepare(h, kind);
    if (!st2) st2 = prepare_tail(h, kind, full, nu1, nu2, level);
    return st2 ? st2 : vcycle_launches(h, kind, full, nu1, nu2, (cudaStream_t)stream, level);
  });
}

int tmg_session_gather(tmg_hier* h, int level, int which, const long long* enc, long n,
                       double* out, void* stream) {
  int st = session_level(h, level, 0);
  if (st) return st;
  const FieldView& v = which ? h->F[level] : h->U[level];
  cudaError_t e = launch_gather_points(v, enc, n, out, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "gather");
}

int tmg_session_scatter(tmg_hier* h, int level, int which, const long long* enc, long n,
                        const double* in, void* stream) {
  int st = session_level(h, level, 0);
  if (st) return st;
  const FieldView& v = which ? h->F[level] : h->U[level];
  cudaError_t e = launch_scatter_points(v, enc, n, in, (cudaStream_t)stream);
  return e == cudaSuccess ? TMG_OK : cuda_fail(e, "scatter");
}

int tmg_session_norm_part(tmg_hier* h, int kind, int g0, int g1, double* out_host, void* stream) {
  int st = session_level(h, 0, 0);
  if (st) return st;
  if (tmg_group_count(kind, h->lv[0]->nx, h->lv[0]->ny) < 1)
    return fail(TMG_BADARG, "smoother kind does not shard");
  return guarded([&]() -> int {
    cudaStream_t s = (cudaStream_t)stream;
    tmg_level* fine = h->lv[0];
    TMG_CUDA_TRY(cudaMemsetAsync(fine->d_norm, 0, sizeof(unsigned long long), s));
    cudaError_t e = launch_hdefect_norm(fine->grid(), h->U[0], h->F[0], fine->d_norm, s, kind,
                                        g0, g1);
    if (e != cudaSuccess) return cuda_fail(e, "defect_norm");
    TMG_CUDA_TRY(cudaMemcpyAsync(fine->h_norm, fine->d_norm, sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, s));
    int st2 = flags_all(h, s);
    if (st2) return st2;
    *out_host = bits_to_double(*fine->h_norm);
    return TMG_OK;
  });
}

int tmg_session_check(tmg_hier* h, void* stream) {
  if (!h) return fail(TMG_BADARG, "null hierarchy");
  return guarded([&] { return flags_all(h, (cudaStream_t)stream); });
}

long tmg_layout_dump(int kind, int nx, int ny, int* oi, int* oj, int* oblk, int* oflags,
                     long cap) {
  Geometry g;
  std::string err = build_geometry(kind, nx, ny, g);
  if (!err.empty()) {
    g_last_error = err;
    return -1;
  }
  return dump_members(g, oi, oj, oblk, oflags, cap);
}

}  // extern "C"

// ---------------- per-block shims (test / plugin surface) -------------------
namespace {

// Index arrays may live in host or device memory: host indices (the
// reference's numpy plans) are used in place, device ones are read back.
bool host_pointer(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

// Per-thread shim workspace: the plan arena, the merged coefficient array
// and the pivot flag, grown on demand and reused by every later call.
struct ShimWork {
  UploadArena arena;
  double* cw = nullptr;
  size_t cw_cap = 0;
  int* d_err = nullptr;
  int* h_err = nullptr;
};
thread_local ShimWork g_shim;

int relax_explicit(int kind, long n, const int64_t* ii, const int64_t* jj, long m,
                   const int64_t* offs, long bi, long bj, int nx, int ny, const double* W,
                   const double* E, const double* S, const double* N, double* u, const double* f,
                   cudaStream_t s) {
  if (n < 1) return TMG_OK;
  std::vector<long long> hi, hj, ho;
  const long long* pi = reinterpret_cast<const long long*>(ii);
  const long long* pj = reinterpret_cast<const long long*>(jj);
  const long long* po = reinterpret_cast<const long long*>(offs);
  if (!host_pointer(ii) || !host_pointer(jj) || (kind == 3 && !host_pointer(offs))) {
    hi.resize(n);
    hj.resize(n);
    ho.resize(m > 0 ? m + 1 : 1);
    TMG_CUDA_TRY(cudaMemcpyAsync(hi.data(), ii, sizeof(int64_t) * n, cudaMemcpyDefault, s));
    TMG_CUDA_TRY(cudaMemcpyAsync(hj.data(), jj, sizeof(int64_t) * n, cudaMemcpyDefault, s));
    if (kind == 3)
      TMG_CUDA_TRY(cudaMemcpyAsync(ho.data(), offs, sizeof(int64_t) * (m + 1), cudaMemcpyDefault,
                                   s));
    TMG_CUDA_TRY(cudaStreamSynchronize(s));
    pi = hi.data();
    pj = hj.data();
    po = ho.data();
  }
  for (long k = 0; k < n; k++)
    if (pi[k] < 1 || pi[k] >= nx || pj[k] < 1 || pj[k] >= ny)
      return fail(TMG_BADARG, "block member outside the grid interior");
  Geometry g;
  g.nx = nx;
  g.ny = ny;
  g.scheme = -1;
  std::string err = add_explicit_block(g, kind, n, pi, pj, m, po, bi, bj);
  if (!err.empty()) return fail(TMG_BADARG, err);
  cudaError_t e = init_sweep_kernels();
  if (e != cudaSuccess) return cuda_fail(e, "kernel attributes");
  ShimWork& w = g_shim;
  // arena: room for this block's plan (chunk records of 16 bytes, bins,
  // hubs, legs) with slack; grown (the only allocation) when too small
  const size_t need = (size_t)4096 + (size_t)(n / 2 + 64) * 64 * 4;
  if (w.arena.cap < need) {
    if (w.arena.base) {
      TMG_CUDA_TRY(cudaStreamSynchronize(s));
      cudaFree(w.arena.base);
    }
    w.arena.cap = std::max(need, (size_t)1 << 20);
    TMG_CUDA_TRY(cudaMalloc(&w.arena.base, w.arena.cap));
  }
  const size_t bx = (size_t)nx + 1, by = (size_t)ny + 1;
  if (w.cw_cap < 2 * bx + 2 * by) {
    if (w.cw) {
      TMG_CUDA_TRY(cudaStreamSynchronize(s));
      cudaFree(w.cw);
    }
    w.cw_cap = std::max(2 * bx + 2 * by, (size_t)4096);
    TMG_CUDA_TRY(cudaMalloc(&w.cw, sizeof(double) * w.cw_cap));
  }
  if (!w.d_err) {
    TMG_CUDA_TRY(cudaMalloc(&w.d_err, sizeof(int)));
    TMG_CUDA_TRY(cudaMallocHost(&w.h_err, sizeof(int)));
  }
  w.arena.used = 0;
  w.arena.stream = s;
  Plan p;
  set_upload_arena(&w.arena);
  err = pack_plan(std::move(g), kQmax, LM_NATURAL, p);
  set_upload_arena(nullptr);
  p.arena = true;
  if (!err.empty()) {
    free_plan(p);
    return fail(TMG_BADARG, err);
  }
  // the kernel addresses W, E, S, N as one allocation (tmg_kernels.h)
  double* cw = w.cw;
  TMG_CUDA_TRY(cudaMemsetAsync(w.d_err, 0, sizeof(int), s));
  TMG_CUDA_TRY(cudaMemcpyAsync(cw, W, sizeof(double) * bx, cudaMemcpyDefault, s));
  TMG_CUDA_TRY(cudaMemcpyAsync(cw + bx, E, sizeof(double) * bx, cudaMemcpyDefault, s));
  TMG_CUDA_TRY(cudaMemcpyAsync(cw + 2 * bx, S, sizeof(double) * by, cudaMemcpyDefault, s));
  TMG_CUDA_TRY(cudaMemcpyAsync(cw + 2 * bx + by, N, sizeof(double) * by, cudaMemcpyDefault, s));
  SweepArgs a{};
  a.legs = p.d_legs;
  a.blocks = p.d_blocks;
  a.W = cw;
  a.E = cw + bx;
  a.S = cw + 2 * bx;
  a.N = cw + 2 * bx + by;
  a.u = u;
  a.f = f;
  a.ld = ny + 1;
  a.err = w.d_err;
  a.ut = u;
  a.ft = f;
  a.ldt = nx + 1;
  a.mode = LM_NATURAL;
  a.nx = nx;
  a.ny = ny;
  e = launch_colour(p, 1, a, s);
  // the reference raises SingularSystemError at once: one flag readback
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(w.h_err, w.d_err, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  free_plan(p);
  if (e != cudaSuccess) return cuda_fail(e, "relax shim");
  if (*w.h_err & 1) return fail(TMG_SINGULAR, "zero pivot");
  return TMG_OK;
}

}  // namespace

extern "C" {

int tmg_relax_points(long n, const int64_t* ii, const int64_t* jj, int nx, int ny, const double* W,
                     const double* E, const double* S, const double* N, double* u, const double* f,
                     void* stream) {
  return guarded([&] {
    return relax_explicit(0, n, ii, jj, 0, nullptr, 0, 0, nx, ny, W, E, S, N, u, f,
                          (cudaStream_t)stream);
  });
}

int tmg_relax_chain(long n, const int64_t* ii, const int64_t* jj, int nx, int ny, const double* W,
                    const double* E, const double* S, const double* N, double* u, const double* f,
                    void* stream) {
  return guarded([&] {
    return relax_explicit(1, n, ii, jj, 0, nullptr, 0, 0, nx, ny, W, E, S, N, u, f,
                          (cudaStream_t)stream);
  });
}

int tmg_relax_ring(long n, const int64_t* ii, const int64_t* jj, int nx, int ny, const double* W,
                   const double* E, const double* S, const double* N, double* u, const double* f,
                   void* stream) {
  return guarded([&] {
    return relax_explicit(2, n, ii, jj, 0, nullptr, 0, 0, nx, ny, W, E, S, N, u, f,
                          (cudaStream_t)stream);
  });
}

int tmg_relax_legged(long n, const int64_t* ii, const int64_t* jj, long m, const int64_t* offs,
                     long bi, long bj, int nx, int ny, const double* W, const double* E,
                     const double* S, const double* N, double* u, const double* f, void* stream) {
  return guarded([&] {
    return relax_explicit(3, n, ii, jj, m, offs, bi, bj, nx, ny, W, E, S, N, u, f,
                          (cudaStream_t)stream);
  });
}


// ---- line-solver API (tridiag.py:30-125) ------------------------------------
// The reference's three direct solvers on host arrays, executed on the device
// in the reference's operation order (separate multiply / subtract / divide,
// round to nearest: bit-identical to numpy).  One system per call: these are
// the reference's specification functions, not a hot path.
}  // extern "C"

namespace {

__device__ __forceinline__ bool tri_bad(double p) { return fabs(p) < 1e-300; }

// forward elimination of one leg / chain (tridiag.py:35-38); returns false at
// the first vanishing pivot among bb[0 .. m-2]
__device__ bool tri_forward(long m, const double* a, const double* c, double* bb, double* rr,
                            double* gg) {
  for (long k = 1; k < m; k++) {
    if (tri_bad(bb[k - 1])) return false;
    const double w = __ddiv_rn(a[k], bb[k - 1]);
    bb[k] = __dsub_rn(bb[k], __dmul_rn(w, c[k - 1]));
    rr[k] = __dsub_rn(rr[k], __dmul_rn(w, rr[k - 1]));
    if (gg) gg[k] = __dsub_rn(gg[k], __dmul_rn(w, gg[k - 1]));
  }
  return true;
}

__global__ void thomas_kernel(long m, const double* a, double* bb, const double* c, double* rr,
                              double* x, int* err) {
  if (!tri_forward(m, a, c, bb, rr, nullptr) || tri_bad(bb[m - 1])) {
    *err = 1;
    return;
  }
  x[m - 1] = __ddiv_rn(rr[m - 1], bb[m - 1]);
  for (long k = m - 2; k >= 0; k--)
    x[k] = __ddiv_rn(__dsub_rn(rr[k], __dmul_rn(c[k], x[k + 1])), bb[k]);
}

// tridiag.py:46-81; bb, rr hold copies of b, r (length m), gg / y / z scratch
__global__ void circulant_kernel(long m, const double* a, const double* b, double* bb,
                                 const double* c, const double* r, double* rr, double* gg,
                                 double* y, double* z, double* x, int* err) {
  const long mm = m - 1;
  for (long k = 0; k < mm; k++) gg[k] = 0.0;
  gg[0] = a[0];
  gg[mm - 1] = __dadd_rn(gg[mm - 1], c[mm - 1]);
  if (!tri_forward(mm, a, c, bb, rr, gg) || tri_bad(bb[mm - 1])) {
    *err = 1;
    return;
  }
  y[mm - 1] = __ddiv_rn(rr[mm - 1], bb[mm - 1]);
  z[mm - 1] = __ddiv_rn(gg[mm - 1], bb[mm - 1]);
  for (long k = mm - 2; k >= 0; k--) {
    y[k] = __ddiv_rn(__dsub_rn(rr[k], __dmul_rn(c[k], y[k + 1])), bb[k]);
    z[k] = __ddiv_rn(__dsub_rn(gg[k], __dmul_rn(c[k], z[k + 1])), bb[k]);
  }
  const double den = __dsub_rn(__dsub_rn(b[m - 1], __dmul_rn(c[m - 1], z[0])),
                               __dmul_rn(a[m - 1], z[mm - 1]));
  if (tri_bad(den)) {
    *err = 1;
    return;
  }
  const double xm = __ddiv_rn(__dsub_rn(__dsub_rn(r[m - 1], __dmul_rn(c[m - 1], y[0])),
                                        __dmul_rn(a[m - 1], y[mm - 1])),
                              den);
  for (long k = 0; k < mm; k++) x[k] = __dsub_rn(y[k], __dmul_rn(z[k], xm));
  x[m - 1] = xm;
}

// tridiag.py:84-125: a thread per leg eliminates tip -> branch, thread 0
// closes the branch row in leg order, every thread substitutes back
__global__ void legged_kernel(int nleg, const long* offs, const double* a, double* bb,
                              const double* c, double* rr, const double* d, double d_centre,
                              double r_centre, double* x, double* xb_out, int* err) {
  __shared__ double xb;
  __shared__ int bad;
  const int t = threadIdx.x;
  if (t == 0) bad = 0;
  __syncthreads();
  const long o = t < nleg ? offs[t] : 0, p = t < nleg ? offs[t + 1] - o : 0;
  if (t < nleg && (!tri_forward(p, a + o, c + o, bb + o, rr + o, nullptr) || tri_bad(bb[o + p - 1])))
    atomicExch(&bad, 1);
  __syncthreads();
  if (bad) {
    if (t == 0) *err = 1;
    return;
  }
  if (t == 0) {
    double num = r_centre, den = d_centre;
    for (int k = 0; k < nleg; k++) {
      const long e = offs[k + 1] - 1;
      num = __dsub_rn(num, __ddiv_rn(__dmul_rn(d[k], rr[e]), bb[e]));
      den = __dsub_rn(den, __ddiv_rn(__dmul_rn(d[k], c[e]), bb[e]));
    }
    if (tri_bad(den)) {
      *err = 1;
      bad = 1;
    } else {
      xb = __ddiv_rn(num, den);
      *xb_out = xb;
    }
  }
  __syncthreads();
  if (bad || t >= nleg) return;
  x[o + p - 1] = __ddiv_rn(__dsub_rn(rr[o + p - 1], __dmul_rn(c[o + p - 1], xb)), bb[o + p - 1]);
  for (long k = p - 2; k >= 0; k--)
    x[o + k] = __ddiv_rn(__dsub_rn(rr[o + k], __dmul_rn(c[o + k], x[o + k + 1])), bb[o + k]);
}

// device scratch of one line-solver call: `nd` doubles, the flag after them
struct TriScratch {
  double* d = nullptr;
  int* err = nullptr;
  ~TriScratch() { cudaFree(d); }
  cudaError_t init(size_t nd) {
    cudaError_t e = cudaMalloc(&d, nd * sizeof(double) + sizeof(int));
    if (e != cudaSuccess) return e;
    err = reinterpret_cast<int*>(d + nd);
    return cudaMemset(err, 0, sizeof(int));
  }
};

int tri_finish(TriScratch& w, cudaStream_t st, double* x_host, const double* x_dev, long n,
               double* extra_host, const double* extra_dev) {
  int flag = 0;
  TMG_CUDA_TRY(cudaGetLastError());
  TMG_CUDA_TRY(cudaMemcpyAsync(&flag, w.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  TMG_CUDA_TRY(cudaMemcpyAsync(x_host, x_dev, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (extra_host)
    TMG_CUDA_TRY(cudaMemcpyAsync(extra_host, extra_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  TMG_CUDA_TRY(cudaStreamSynchronize(st));
  if (flag) return fail(TMG_SINGULAR, "zero pivot during tridiagonal elimination");
  return TMG_OK;
}

}  // namespace

extern "C" {

int tmg_thomas(long m, const double* a, const double* b, const double* c, const double* r,
               double* x, void* stream) {
  return guarded([&]() -> int {
    if (m < 1 || !a || !b || !c || !r || !x) return fail(TMG_BADARG, "thomas: need m >= 1 and arrays");
    cudaStream_t st = (cudaStream_t)stream;
    TriScratch w;
    TMG_CUDA_TRY(w.init(5 * (size_t)m));
    const double* src[4] = {a, b, c, r};
    for (int q = 0; q < 4; q++)
      TMG_CUDA_TRY(cudaMemcpyAsync(w.d + q * m, src[q], m * sizeof(double), cudaMemcpyHostToDevice, st));
    TMG_COUNT(1);
    thomas_kernel<<<1, 1, 0, st>>>(m, w.d, w.d + m, w.d + 2 * m, w.d + 3 * m, w.d + 4 * m, w.err);
    return tri_finish(w, st, x, w.d + 4 * m, m, nullptr, nullptr);
  });
}

int tmg_circulant_thomas(long m, const double* a, const double* b, const double* c,
                         const double* r, double* x, void* stream) {
  return guarded([&]() -> int {
    if (m < 3) return fail(TMG_BADARG, "circulant system needs m >= 3, got " + std::to_string(m));
    if (!a || !b || !c || !r || !x) return fail(TMG_BADARG, "circulant_thomas: null array");
    cudaStream_t st = (cudaStream_t)stream;
    TriScratch w;
    TMG_CUDA_TRY(w.init(10 * (size_t)m));
    double* D = w.d;  // a, b, c, r, bb, rr, gg, y, z, x
    const double* src[6] = {a, b, c, r, b, r};
    for (int q = 0; q < 6; q++)
      TMG_CUDA_TRY(cudaMemcpyAsync(D + q * m, src[q], m * sizeof(double), cudaMemcpyHostToDevice, st));
    TMG_COUNT(1);
    circulant_kernel<<<1, 1, 0, st>>>(m, D, D + m, D + 4 * m, D + 2 * m, D + 3 * m, D + 5 * m,
                                      D + 6 * m, D + 7 * m, D + 8 * m, D + 9 * m, w.err);
    return tri_finish(w, st, x, D + 9 * m, m, nullptr, nullptr);
  });
}

int tmg_legged_thomas(long nleg, const long* offs, const double* a, const double* b,
                      const double* c, const double* r, const double* d, double d_centre,
                      double r_centre, double* x, double* x_branch, void* stream) {
  return guarded([&]() -> int {
    if (nleg < 2) return fail(TMG_BADARG, "need m >= 2 legs, got " + std::to_string(nleg));
    if (nleg > 1024) return fail(TMG_BADARG, "legged_thomas: at most 1024 legs");
    if (!offs || !a || !b || !c || !r || !d || !x || !x_branch)
      return fail(TMG_BADARG, "legged_thomas: null array");
    for (long k = 0; k < nleg; k++)
      if (offs[k + 1] <= offs[k]) return fail(TMG_BADARG, "legged_thomas: empty leg");
    const long n = offs[nleg] - offs[0];
    if (offs[0] != 0) return fail(TMG_BADARG, "legged_thomas: offs[0] must be 0");
    cudaStream_t st = (cudaStream_t)stream;
    TriScratch w;
    // a, bb, c, rr, x (n each), d (nleg), x_branch, offs (as longs, 8-byte slots)
    const size_t nd = 5 * (size_t)n + nleg + 1 + (nleg + 1);
    TMG_CUDA_TRY(w.init(nd));
    double* D = w.d;
    const double* src[4] = {a, b, c, r};
    for (int q = 0; q < 4; q++)
      TMG_CUDA_TRY(cudaMemcpyAsync(D + q * n, src[q], n * sizeof(double), cudaMemcpyHostToDevice, st));
    double* dd = D + 5 * n;
    double* xb = dd + nleg;
    long* doffs = reinterpret_cast<long*>(xb + 1);
    static_assert(sizeof(long) == sizeof(double), "offsets share the scratch");
    TMG_CUDA_TRY(cudaMemcpyAsync(dd, d, nleg * sizeof(double), cudaMemcpyHostToDevice, st));
    TMG_CUDA_TRY(cudaMemcpyAsync(doffs, offs, (nleg + 1) * sizeof(long), cudaMemcpyHostToDevice, st));
    TMG_COUNT(1);
    const int threads = (int)((nleg + 31) / 32 * 32);
    legged_kernel<<<1, threads, 0, st>>>((int)nleg, doffs, D, D + n, D + 2 * n, D + 3 * n, dd,
                                         d_centre, r_centre, D + 4 * n, xb, w.err);
    return tri_finish(w, st, x, D + 4 * n, n, x_branch, xb);
  });
}

}  // extern "C"
