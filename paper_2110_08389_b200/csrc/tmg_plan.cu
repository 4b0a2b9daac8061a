// Host-side block geometry (closed form) and bin packing for the block-solver
// kernel.  Replaces the reference's Python-tuple plans (layout.py:61-168,
// smoothers.py:42-118): a block here is a hub plus up to four legs described
// by straight segments, O(#blocks) to build instead of O(#points) tuples.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "tmg_plan.h"

namespace tmg {

namespace {

int parity_red(int k) { return (k % 2) != 0; }  // layout.py:22-23

void leg_point_host(const LegD& L, int p, int& i, int& j) {
  i = L.i0;
  j = L.j0;
  int rem = p;
  for (int s = 0; s < L.nseg && rem > 0; s++) {
    int st = std::min(rem, L.seg_len[s]);
    i += st * dir_di(L.seg_dir[s]);
    j += st * dir_dj(L.seg_dir[s]);
    rem -= st;
  }
}



struct Builder {
  Geometry& g;
  explicit Builder(Geometry& gg) : g(gg) {}

  int new_block(int red, int hi, int hj) {
    BlockD b;
    std::memset(&b, 0, sizeof(b));
    b.hi = hi;
    b.hj = hj;
    b.leg0 = (int)g.legs.size();
    b.nleg = 0;
    b.hub_thread = -1;
    b.bin = -1;
    b.red = (uint8_t)red;
    g.blocks.push_back(b);
    return (int)g.blocks.size() - 1;
  }

  // Straight leg of npts points starting at (i0, j0) stepping in direction d.
  // If to_hub, the point after the last one (same direction) is the hub.
  void straight_leg(int blk, int i0, int j0, int d, int npts, bool to_hub) {
    LegD L;
    std::memset(&L, 0, sizeof(L));
    L.i0 = i0;
    L.j0 = j0;
    L.npts = npts;
    L.block = blk;
    L.nseg = 1;
    L.seg_dir[0] = (uint8_t)d;
    L.seg_len[0] = npts - 1;
    L.flags = to_hub ? 2 : 0;
    L.hub_dir_first = DNONE;
    L.hub_dir_last = to_hub ? (uint8_t)d : (uint8_t)DNONE;
    g.legs.push_back(L);
    BlockD& b = g.blocks[blk];
    b.nleg++;
    if (to_hub) b.hub_mask |= (uint8_t)(1u << dir_opp(d));
  }
};

// layout.py:61-133
void tweed(Builder& B, int nx, int ny) {
  int mx = nx - 1, my = ny - 1, s = std::min(mx, my), c = (s + 1) / 2;
  int corners[4][4] = {{1, 1, 1, 1}, {mx, 1, -1, 1}, {1, my, 1, -1}, {mx, my, -1, -1}};
  for (auto& cr : corners) B.new_block(1, cr[0], cr[1]);
  for (int k = 2; k < c; k++) {
    int red = parity_red(k);
    for (auto& cr : corners) {
      int x0 = cr[0], y0 = cr[1], sx = cr[2], sy = cr[3];
      int bi = x0 + sx * (k - 1), bj = y0 + sy * (k - 1);
      int b = B.new_block(red, bi, bj);
      B.straight_leg(b, x0, bj, sx > 0 ? DE : DW, k - 1, true);  // leg_x
      B.straight_leg(b, bi, y0, sy > 0 ? DN : DS, k - 1, true);  // leg_y
    }
  }
  int redc = parity_red(c);
  if (mx == my) {
    int b = B.new_block(redc, c, c);
    B.straight_leg(b, 1, c, DE, c - 1, true);
    B.straight_leg(b, mx, c, DW, mx - c, true);
    B.straight_leg(b, c, 1, DN, c - 1, true);
    B.straight_leg(b, c, my, DS, my - c, true);
  } else if (mx > my) {
    int b = B.new_block(redc, c, c);
    B.straight_leg(b, 1, c, DE, c - 1, true);
    B.straight_leg(b, c, 1, DN, c - 1, true);
    B.straight_leg(b, c, my, DS, my - c, true);
    int br = mx + 1 - c;
    b = B.new_block(redc, br, c);
    B.straight_leg(b, mx, c, DW, mx - br, true);
    B.straight_leg(b, br, 1, DN, c - 1, true);
    B.straight_leg(b, br, my, DS, my - c, true);
    for (int i = c + 1; i < mx - c + 1; i++) {
      int l = B.new_block(parity_red(i), -1, -1);
      B.straight_leg(l, i, 1, DN, my, false);
    }
  } else {
    int b = B.new_block(redc, c, c);
    B.straight_leg(b, c, 1, DN, c - 1, true);
    B.straight_leg(b, 1, c, DE, c - 1, true);
    B.straight_leg(b, mx, c, DW, mx - c, true);
    int br = my + 1 - c;
    b = B.new_block(redc, c, br);
    B.straight_leg(b, c, my, DS, my - br, true);
    B.straight_leg(b, 1, br, DE, c - 1, true);
    B.straight_leg(b, mx, br, DW, mx - c, true);
    for (int j = c + 1; j < my - c + 1; j++) {
      int l = B.new_block(parity_red(j), -1, -1);
      B.straight_leg(l, 1, j, DE, mx, false);
    }
  }
}

// layout.py:136-168.  Ring r is the chain p_0..p_{m-2} (counter-clockwise
// from (r, r), x increasing first) plus the closing point p_{m-1} = (r, r+1)
// as the hub, coupled to both chain ends (_ckernels.pyx:114-118).
void wireframe(Builder& B, int nx, int ny) {
  int mx = nx - 1, my = ny - 1, s = std::min(mx, my), q = (s - 1) / 2;
  for (int r = 1; r <= q; r++) {
    int hi_i = mx + 1 - r, hi_j = my + 1 - r;
    int b = B.new_block(parity_red(r), r, r + 1);
    LegD L;
    std::memset(&L, 0, sizeof(L));
    L.i0 = r;
    L.j0 = r;
    L.block = b;
    L.nseg = 4;
    L.seg_dir[0] = DE; L.seg_len[0] = hi_i - r;
    L.seg_dir[1] = DN; L.seg_len[1] = hi_j - r;
    L.seg_dir[2] = DW; L.seg_len[2] = hi_i - r;
    L.seg_dir[3] = DS; L.seg_len[3] = hi_j - r - 2;
    L.npts = 1 + L.seg_len[0] + L.seg_len[1] + L.seg_len[2] + L.seg_len[3];
    L.flags = 3;
    L.hub_dir_first = DN;  // (r, r) -> (r, r+1)
    L.hub_dir_last = DS;   // (r, r+2) -> (r, r+1)
    B.g.legs.push_back(L);
    BlockD& bb = B.g.blocks[b];
    bb.nleg = 1;
    bb.hub_mask = (uint8_t)((1u << DS) | (1u << DN));
  }
  int tred = parity_red(q + 1);
  if (mx == my) {
    B.new_block(tred, q + 1, q + 1);
  } else if (mx > my) {
    int l = B.new_block(tred, -1, -1);
    B.straight_leg(l, q + 1, q + 1, DE, mx - 2 * q, false);
  } else {
    int l = B.new_block(tred, -1, -1);
    B.straight_leg(l, q + 1, q + 1, DN, my - 2 * q, false);
  }
}

// smoothers.py:77-89.  A line longer than one CTA holds at q = 16 (kThreads
// * kQmax points) is solved as a two-legged block around its middle point
// (legs from both walls toward it): the same exact line solve, eliminated
// from both ends, so its two halves sit in different CTAs of a cluster
// without a reduced system spanning them.
void zebra(Builder& B, int nx, int ny, bool axis_x) {
  const int len = axis_x ? nx - 1 : ny - 1;
  const bool split = len > kThreads * kQmax;
  const int h = (len + 1) / 2;  // hub: point h of the line (1-based)
  for (int t = 1; t < (axis_x ? ny : nx); t++) {
    const int red = t % 2;
    if (!split) {
      int l = B.new_block(red, -1, -1);
      if (axis_x) B.straight_leg(l, 1, t, DE, len, false);
      else B.straight_leg(l, t, 1, DN, len, false);
      continue;
    }
    if (axis_x) {
      int b = B.new_block(red, h, t);
      B.straight_leg(b, 1, t, DE, h - 1, true);
      B.straight_leg(b, len, t, DW, len - h, true);
    } else {
      int b = B.new_block(red, t, h);
      B.straight_leg(b, t, 1, DN, h - 1, true);
      B.straight_leg(b, t, len, DS, len - h, true);
    }
  }
}

// Direction of step p (the step arriving at point p >= 1) of a leg.
int step_direction(const LegD& L, int p) {
  int cum = 0;
  for (int s = 0; s < L.nseg; s++) {
    if (p > cum && p <= cum + L.seg_len[s]) return L.seg_dir[s];
    cum += L.seg_len[s];
  }
  return L.seg_dir[L.nseg - 1];
}

// Split a leg into straight runs (pieces) and the pieces into chunks of at
// most q points.  A leg whose first point couples to the hub starts with a
// one-point chunk, so that every hub neighbour is a chunk end (a reduced
// unknown).  With a hybrid field layout a run is further cut wherever the
// owning buffer changes, and a point whose cross neighbour lives in the other
// buffer becomes a one-point chunk, so that inside every chunk the point and
// its two cross neighbours are addressed through one buffer with fixed
// strides.  Returns [first, last] point ranges.
std::vector<std::pair<int, int>> leg_chunks(const LegD& L, int q, int mode, int nx, int ny) {
  std::vector<std::pair<int, int>> pieces, runs, out;
  int start = 0;
  if (L.flags & 1) {
    pieces.push_back({0, 0});
    start = 1;
  }
  int cum = 0;
  for (int s = 0; s < L.nseg; s++) {
    const int endp = cum + L.seg_len[s];
    if (endp >= start) {
      pieces.push_back({start, endp});
      start = endp + 1;
    }
    cum = endp;
  }
  if (start <= L.npts - 1) pieces.push_back({start, L.npts - 1});
  auto interior = [&](int i, int j) { return i > 0 && j > 0 && i < nx && j < ny; };
  // A chunk's end points are addressed one by one (tmg_sweep.cu); only its
  // inner points need their cross neighbours in the chunk's own buffer.
  std::vector<char> bad;
  for (auto& pc : pieces) {
    if (mode == LM_NATURAL || pc.first == pc.second) {
      for (int a = pc.first; a <= pc.second; a += q)
        out.push_back({a, std::min(a + q - 1, pc.second)});
      continue;
    }
    const int d = step_direction(L, pc.first + 1);
    const bool axis_i = (d == DW || d == DE);
    bad.assign(pc.second - pc.first + 1, 0);
    runs.clear();
    int rs = pc.first, rown = -1;
    for (int p = pc.first; p <= pc.second; p++) {
      int i, j;
      leg_point_host(L, p, i, j);
      const int o = owns_t(mode, nx, ny, i, j);
      const int i1 = axis_i ? i : i - 1, j1 = axis_i ? j - 1 : j;
      const int i2 = axis_i ? i : i + 1, j2 = axis_i ? j + 1 : j;
      bad[p - pc.first] = (interior(i1, j1) && owns_t(mode, nx, ny, i1, j1) != (bool)o) ||
                          (interior(i2, j2) && owns_t(mode, nx, ny, i2, j2) != (bool)o);
      if (p > pc.first && o != rown) {  // the owning buffer changes
        runs.push_back({rs, p - 1});
        rs = p;
      }
      rown = o;
    }
    runs.push_back({rs, pc.second});
    for (auto& r : runs) {
      int a = r.first;
      while (a <= r.second) {
        int e = std::min(a + q - 1, r.second);
        for (int p = a + 1; p < e; p++)  // a mismatching point may only be a chunk end
          if (bad[p - pc.first]) {
            e = p;
            break;
          }
        out.push_back({a, e});
        a = e + 1;
      }
    }
  }
  return out;
}

}  // namespace

std::string build_geometry(int scheme, int nx, int ny, Geometry& g) {
  g = Geometry();
  g.scheme = scheme;
  g.nx = nx;
  g.ny = ny;
  Builder B(g);
  switch (scheme) {
    case SCHEME_ZEBRA_X:
    case SCHEME_ZEBRA_Y:
      if (nx < 2 || ny < 2) return "zebra needs nx, ny >= 2";
      zebra(B, nx, ny, scheme == SCHEME_ZEBRA_X);
      return "";
    case SCHEME_TWEED:
    case SCHEME_WIREFRAME:
      if (nx < 4 || ny < 4 || nx % 2 || ny % 2)
        return "block layouts need even nx, ny >= 4, got (" + std::to_string(nx) + ", " +
               std::to_string(ny) + ")";
      if (scheme == SCHEME_TWEED) tweed(B, nx, ny);
      else wireframe(B, nx, ny);
      return "";
    default:
      return "no block geometry for scheme " + std::to_string(scheme);
  }
}

long dump_members(const Geometry& g, int* oi, int* oj, int* oblk, int* oflags, long cap) {
  long p = 0;
  auto put = [&](int i, int j, int b, int flags) {
    if (p < cap) { oi[p] = i; oj[p] = j; oblk[p] = b; oflags[p] = flags; }
    p++;
  };
  for (size_t b = 0; b < g.blocks.size(); b++) {
    const BlockD& B = g.blocks[b];
    // kind: 0 point, 1 line, 2 legged, 3 ring (layout.py:30)
    int kind = B.nleg == 0 ? 0 : B.hi < 0 ? 1 : (g.legs[B.leg0].flags & 1) ? 3 : 2;
    for (int l = 0; l < B.nleg; l++) {
      const LegD& L = g.legs[B.leg0 + l];
      for (int t = 0; t < L.npts; t++) {
        int i, j;
        leg_point_host(L, t, i, j);
        put(i, j, (int)b, B.red | (l << 1) | (kind << 4));
      }
    }
    if (B.hi >= 0) put(B.hi, B.hj, (int)b, B.red | (7 << 1) | (kind << 4));
  }
  return p;
}

// plan statistics without a device (tmg_plan_stats): uploads are skipped
static thread_local bool g_dry_run = false;
static thread_local long long g_stats[10];

// Upload arena of the per-block shims (tmg_relax_*): while set, plan arrays
// are carved from one grow-only device buffer and copied asynchronously on
// its stream, so a shim call allocates nothing once the arena is warm.
static thread_local UploadArena* g_arena = nullptr;
void set_upload_arena(UploadArena* a) { g_arena = a; }

template <class T>
static T* upload(const std::vector<T>& v, size_t& bytes, std::string& err) {
  if (v.empty() || g_dry_run) return nullptr;
  if (g_arena) {
    const size_t nb = (v.size() * sizeof(T) + 255) & ~(size_t)255;
    if (g_arena->used + nb > g_arena->cap) {
      err = "shim arena too small";
      return nullptr;
    }
    T* d = reinterpret_cast<T*>(g_arena->base + g_arena->used);
    g_arena->used += nb;
    cudaError_t e = cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice,
                                    g_arena->stream);
    if (e != cudaSuccess) err = cudaGetErrorString(e);
    return d;
  }
  T* d = nullptr;
  cudaError_t e = cudaMalloc(&d, v.size() * sizeof(T));
  if (e != cudaSuccess) { err = cudaGetErrorString(e); return nullptr; }
  e = cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { err = cudaGetErrorString(e); return nullptr; }
  bytes += v.size() * sizeof(T);
  return d;
}

std::string build_plan(int scheme, int nx, int ny, int q, int mode, Plan& P) {
  P = Plan();
  if (q < 1 || q > kQmax) return "chunk size q out of range";
  P.q = q;
  if (scheme == SCHEME_CHECKERBOARD) {
    if (nx < 2 || ny < 2) return "checkerboard needs nx, ny >= 2";
    P.geo.scheme = scheme;
    P.geo.nx = nx;
    P.geo.ny = ny;
    P.mode = mode;
    P.point_scheme = true;
    return "";
  }
  Geometry g;
  std::string err = build_geometry(scheme, nx, ny, g);
  if (!err.empty()) return err;
  const bool legk = leg_plan_applies(scheme, nx, ny, mode) && !g_dry_run;
  if (legk) {  // L-shells k in [k0, c) and the cross go to the leg kernel
    // (with the default k0 = 2 the corner points go to it as well)
    const int k0 = leg_k0() <= 2 ? 1 : leg_k0(), c = nx / 2;
    Geometry out;
    out.scheme = g.scheme;
    out.nx = g.nx;
    out.ny = g.ny;
    for (const BlockD& B : g.blocks) {
      int i = B.hi, j = B.hj;
      if (i < 0) {
        i = g.legs[B.leg0].i0;
        j = g.legs[B.leg0].j0;
      }
      const int grp = point_group(g.scheme, g.nx, g.ny, i, j);
      if (grp >= k0 && grp <= c) continue;  // L-shells and the central cross
      BlockD nb = B;
      nb.leg0 = (int32_t)out.legs.size();
      for (int l = 0; l < B.nleg; l++) {
        LegD L = g.legs[B.leg0 + l];
        L.block = (int32_t)out.blocks.size();
        out.legs.push_back(L);
      }
      out.blocks.push_back(nb);
    }
    g = std::move(out);
  }
  err = pack_plan(std::move(g), q, mode, P);
  if (!err.empty() || !legk) return err;
  P.lp = new LegPlan();
  err = build_leg_plan(nx, *P.lp);
  P.device_bytes += P.lp->device_bytes;
  return err;
}

void filter_groups(Geometry& g, int g0, int g1) {
  Geometry out;
  out.scheme = g.scheme;
  out.nx = g.nx;
  out.ny = g.ny;
  for (const BlockD& B : g.blocks) {
    int i = B.hi, j = B.hj;
    if (i < 0) {
      i = g.legs[B.leg0].i0;
      j = g.legs[B.leg0].j0;
    }
    const int grp = point_group(g.scheme, g.nx, g.ny, i, j);
    if (grp < g0 || grp >= g1) continue;
    BlockD nb = B;
    nb.leg0 = (int32_t)out.legs.size();
    for (int l = 0; l < B.nleg; l++) {
      LegD L = g.legs[B.leg0 + l];
      L.block = (int32_t)out.blocks.size();
      out.legs.push_back(L);
    }
    out.blocks.push_back(nb);
  }
  g = std::move(out);
}

std::string build_plan_part(int scheme, int nx, int ny, int q, int mode, int g0, int g1,
                            Plan& P) {
  const int G = group_count(scheme, nx, ny);
  if (G < 1) return "smoother kind " + std::to_string(scheme) + " has no sharding groups";
  if (g0 < 1 || g1 > G + 1 || g0 >= g1)
    return "group range [" + std::to_string(g0) + ", " + std::to_string(g1) +
           ") outside 1.." + std::to_string(G);
  if (scheme == SCHEME_CHECKERBOARD) {
    std::string err = build_plan(scheme, nx, ny, q, mode, P);
    P.g0 = g0;  // rows i in [g0, g1)
    P.g1 = g1;
    return err;
  }
  Geometry g;
  std::string err = build_geometry(scheme, nx, ny, g);
  if (!err.empty()) return err;
  filter_groups(g, g0, g1);
  // a rank's L-shells and (if it owns group c) the cross on the leg kernel
  const bool legk = leg_plan_applies(scheme, nx, ny, mode) && !g_dry_run;
  const int k0 = leg_k0() <= 2 ? 1 : leg_k0(), c = nx / 2;  // 1: the corner points too
  const int ka = std::max(g0, k0), kb = std::min(g1 - 1, c);
  if (legk && ka <= kb) {
    Geometry out;
    out.scheme = g.scheme;
    out.nx = g.nx;
    out.ny = g.ny;
    for (const BlockD& B : g.blocks) {
      int i = B.hi, j = B.hj;
      if (i < 0) {
        i = g.legs[B.leg0].i0;
        j = g.legs[B.leg0].j0;
      }
      const int grp = point_group(g.scheme, g.nx, g.ny, i, j);
      if (grp >= ka && grp <= kb) continue;
      BlockD nb = B;
      nb.leg0 = (int32_t)out.legs.size();
      for (int l = 0; l < B.nleg; l++) {
        LegD L = g.legs[B.leg0 + l];
        L.block = (int32_t)out.blocks.size();
        out.legs.push_back(L);
      }
      out.blocks.push_back(nb);
    }
    g = std::move(out);
  }
  err = pack_plan(std::move(g), q, mode, P);
  P.g0 = g0;
  P.g1 = g1;
  if (!err.empty() || !legk || ka > kb) return err;
  P.lp = new LegPlan();
  err = build_leg_plan(nx, *P.lp, ka, kb);
  P.device_bytes += P.lp->device_bytes;
  return err;
}

std::string pack_plan(Geometry&& geo, int q, int mode, Plan& P) {
  P = Plan();
  if (q < 1 || q > kQmax || (q & (q - 1))) return "chunk size q must be a power of two <= 16";
  P.q = q;
  P.mode = mode;
  P.geo = std::move(geo);
  Geometry& g = P.geo;
  std::string err;
  const int T = kThreads;
  const FieldView fv{nullptr, nullptr, g.nx, g.ny, mode};

  std::vector<std::vector<std::pair<int, int>>> lchunks(g.legs.size());
  for (size_t l = 0; l < g.legs.size(); l++) {
    lchunks[l] = leg_chunks(g.legs[l], q, mode, g.nx, g.ny);
    g.legs[l].nchunk = (int)lchunks[l].size();
    if (g.legs[l].nchunk > kMaxCluster * T)
      return "leg of " + std::to_string(g.legs[l].npts) +
             " points exceeds the cluster solver capacity (" + std::to_string(kMaxCluster * T * q) + ")";
  }
  // Virtual-thread placement of a leg of nch chunks at position v (rank * T
  // + offset): a leg of <= 32 chunks stays inside one warp (shuffle-only
  // reduction), a leg of <= T chunks inside one CTA; a longer leg runs on
  // across CTA boundaries of its cluster (cross-CTA reduction via DSMEM).
  auto place = [&](int v, int nch) {
    const int o = v % T;
    if (nch <= 32 && (o / 32) != ((o + nch - 1) / 32)) v += 32 - o % 32;
    if (nch <= T && (v % T) + nch > T) v += T - v % T;
    return v;
  };
  // minimal cluster size per block
  std::vector<int> need(g.blocks.size());
  for (size_t b = 0; b < g.blocks.size(); b++) {
    const BlockD& B = g.blocks[b];
    int v = B.nleg == 0 ? 1 : 0;
    for (int l = 0; l < B.nleg; l++) {
      const int nch = g.legs[B.leg0 + l].nchunk;
      v = place(v, nch) + nch;
    }
    const int ctas = (v + T - 1) / T;
    int cs = 1;
    while (cs < ctas) cs *= 2;
    if (cs > kMaxCluster) return "block needs more than " + std::to_string(kMaxCluster) + " CTAs";
    need[b] = cs;
  }

  // Chunk descriptors, hub rows and bin records of one launch class whose
  // blocks have been assigned to bins (B.bin, L.tbase, B.hub_thread).
  auto emit = [&](int red, int cs, const std::vector<int>& blks, std::vector<BinD>& bins,
                  const std::vector<int>& maxch, const std::vector<int>& xcta,
                  bool warp_aligned) -> std::string {
    LaunchClass lc;
    lc.q = q;
    lc.cs = cs;
    lc.red = red;
    lc.xcta = 0;
    lc.nbins = (int)bins.size();
    ChunkD idle;
    std::memset(&idle, 0, sizeof(idle));
    idle.hub = -1;
    idle.own = -1;
    idle.link = (uint16_t)(DNONE | (DNONE << 3));
    std::vector<ChunkD> ch((size_t)lc.nbins * cs * T, idle);
    std::vector<std::vector<HubD>> bhubs(lc.nbins);
    for (int b : blks) {
      BlockD& B = g.blocks[b];
      const size_t base = (size_t)B.bin * cs * T;
      // hub: one copy per CTA holding chunks of the block (so that the hub
      // value is read locally in the finalize step); owner = the first
      // adjacent chunk thread in that CTA, else its first chunk thread, or
      // the reserved thread of a point block.  Copies after the first only
      // solve, they do not store the hub point (HubD.pad bit 0).
      int owner_cta[kMaxCluster];
      std::fill(owner_cta, owner_cta + kMaxCluster, -1);
      if (B.hi >= 0) {
        HubD H;
        std::memset(&H, 0, sizeof(H));
        H.tbuf = owns_t(mode, g.nx, g.ny, B.hi, B.hj) ? 1 : 0;
        H.off = (int32_t)(H.tbuf ? fv.off_t(B.hi, B.hj) : fv.off_n(B.hi, B.hj));
        H.i = (int16_t)B.hi;
        H.j = (int16_t)B.hj;
        H.mask = B.hub_mask;
        for (int l = 0; l < B.nleg; l++) {
          const LegD& L = g.legs[B.leg0 + l];
          if (L.flags & 2) {
            H.adj_t[H.nadj] = (int16_t)(L.tbase + L.nchunk - 1);
            H.adj_d[H.nadj++] = (uint8_t)dir_opp(L.hub_dir_last);
          }
          if (L.flags & 1) {
            H.adj_t[H.nadj] = (int16_t)L.tbase;
            H.adj_d[H.nadj++] = (uint8_t)dir_opp(L.hub_dir_first);
          }
        }
        if (B.nleg == 0) {
          owner_cta[B.hub_thread / T] = B.hub_thread;
        } else {
          for (int q = 0; q < H.nadj; q++)
            if (owner_cta[H.adj_t[q] / T] < 0) owner_cta[H.adj_t[q] / T] = H.adj_t[q];
          for (int l = 0; l < B.nleg; l++) {
            const LegD& L = g.legs[B.leg0 + l];
            for (int c = 0; c < L.nchunk; c++)
              if (owner_cta[(L.tbase + c) / T] < 0) owner_cta[(L.tbase + c) / T] = L.tbase + c;
          }
        }
        bool primary = true;
        for (int r = 0; r < cs; r++) {
          const int ow = owner_cta[r];
          if (ow < 0) continue;
          HubD Hc = H;
          Hc.pad = primary ? 0 : 1;
          if (primary) B.hub_thread = ow;
          primary = false;
          ch[base + ow].own = (int16_t)bhubs[B.bin].size();
          ch[base + ow].hub = (int16_t)ow;
          bhubs[B.bin].push_back(Hc);
        }
      }
      for (int l = 0; l < B.nleg; l++) {
        const LegD& L = g.legs[B.leg0 + l];
        const auto& cks = lchunks[B.leg0 + l];
        for (int c = 0; c < (int)cks.size(); c++) {
          const int s = cks[c].first, e = cks[c].second;
          int i, j;
          leg_point_host(L, s, i, j);
          // direction of the run containing the chunk
          const int d = (e > s) ? step_direction(L, s + 1)
                                : (s > 0 ? step_direction(L, s) : L.seg_dir[0]);
          const int axis = (d == DS || d == DN) ? 1 : 0;
          const int neg = (d == DW || d == DS) ? 1 : 0;
          int dfirst = DNONE, dlast = DNONE, link = 0;
          if (s == 0) {
            if (L.flags & 1) { dfirst = L.hub_dir_first; link |= kLinkLeftHub; }
          } else {
            dfirst = dir_opp(step_direction(L, s));
            link |= kLinkLeftPrev;
          }
          if (e == L.npts - 1) {
            if (L.flags & 2) { dlast = L.hub_dir_last; link |= kLinkRightHub; }
          } else {
            dlast = step_direction(L, e + 1);
            link |= kLinkRightNext;
          }
          ChunkD& C = ch[base + L.tbase + c];
          const bool tb = owns_t(mode, g.nx, g.ny, i, j);
          C.off = (int32_t)(tb ? fv.off_t(i, j) : fv.off_n(i, j));
          C.a0 = (int16_t)(axis ? j : i);
          C.cidx = (int16_t)(axis ? i : j);
          C.n = (uint8_t)(e - s + 1);
          C.geo = (uint8_t)(axis | (neg << 1) | (tb ? 4 : 0));
          C.link = (uint16_t)(dfirst | (dlast << 3) | link);
          C.hub = (int16_t)owner_cta[(L.tbase + c) / T];
        }
      }
    }
    std::vector<HubD> hubs;
    for (int k = 0; k < lc.nbins; k++) {
      int st = 0;
      while ((1 << st) < maxch[k]) st++;
      bins[k].pcr_steps = st;
      bins[k].warp_local = xcta[k] ? 2 : (warp_aligned && maxch[k] <= 32 ? 1 : 0);
      bins[k].hub0 = (int)hubs.size();
      bins[k].nhub = (int)bhubs[k].size();
      hubs.insert(hubs.end(), bhubs[k].begin(), bhubs[k].end());
    }
    if (g_dry_run) {  // [red|black] x (CTAs, threads with a chunk, points, hubs)
      long long* st = g_stats + (red ? 0 : 4);
      st[0] += (long long)lc.nbins * cs;
      for (const ChunkD& c : ch) {
        st[1] += c.n > 0;
        st[2] += c.n;
      }
      for (const auto& bh : bhubs) st[3] += (long long)bh.size();
      // warps whose 32 chunks are one straight run of full chunks (the
      // kernel's arithmetic gather path): g_stats[8]; all warps: [9]
      for (size_t w = 0; w + 32 <= ch.size(); w += 32) {
        bool uni = true;
        for (int l = 0; l < 32 && uni; l++) {
          const ChunkD& c = ch[w + l];
          uni = c.n == q;
          if (uni && l > 0) {
            const ChunkD& p = ch[w + l - 1];
            const int tb = (c.geo >> 2) & 1, axis = c.geo & 1, neg = (c.geo >> 1) & 1;
            const int si = tb ? 1 : g.ny + 1, sj = tb ? g.nx + 1 : 1;
            const int str = (axis ? sj : si) * (neg ? -1 : 1);
            uni = p.geo == c.geo && p.cidx == c.cidx && p.off + q * str == c.off;
          }
        }
        g_stats[8] += uni;
        g_stats[9] += 1;
      }
    }
    // bins with a leg across a CTA boundary run on their own kernel
    // instantiation (the cross-CTA reduced solve), the others keep theirs
    for (int want = 0; want <= 1; want++) {
      std::vector<ChunkD> ch2;
      std::vector<BinD> bins2;
      std::vector<HubD> hubs2;
      for (int k = 0; k < lc.nbins; k++) {
        if ((xcta[k] != 0) != (want != 0)) continue;
        const size_t per = (size_t)cs * T;
        ch2.insert(ch2.end(), ch.begin() + (size_t)k * per, ch.begin() + (size_t)(k + 1) * per);
        BinD b2 = bins[k];
        b2.hub0 = (int)hubs2.size();
        hubs2.insert(hubs2.end(), hubs.begin() + bins[k].hub0,
                     hubs.begin() + bins[k].hub0 + bins[k].nhub);
        bins2.push_back(b2);
      }
      if (bins2.empty()) continue;
      LaunchClass l2 = lc;
      l2.xcta = want;
      l2.nbins = (int)bins2.size();
      l2.chunks = upload(ch2, P.device_bytes, err);
      l2.bins = upload(bins2, P.device_bytes, err);
      l2.hubs = upload(hubs2, P.device_bytes, err);
      if (!err.empty()) return err;
      P.classes.push_back(l2);
    }
    return std::string();
  };

  const char* pk = std::getenv("TMG_PACK");
  const bool dense = !(pk && std::strcmp(pk, "sequential") == 0);
  std::vector<char> taken(g.blocks.size(), 0);
  auto block_size = [&](int b) {
    const BlockD& B = g.blocks[b];
    int n = B.nleg == 0 ? 1 : 0;
    for (int l = 0; l < B.nleg; l++) n += g.legs[B.leg0 + l].nchunk;
    return n;
  };
  for (int red = 1; red >= 0; red--) {
    // Dense packing (first-fit decreasing over blocks sorted by size): legs
    // of <= 32 chunks go into any warp with room (never straddling a warp,
    // so bins of short legs keep the shuffle-only reduction); longer legs
    // start at the first free slot of a warp and run on through empty warps
    // of one CTA (of the cluster if longer than a CTA); the legs of a block
    // may sit in different CTAs of a cluster (hubs through DSMEM).  Clusters
    // are opened by the blocks that need them and their spare warps filled
    // with the colour's smaller blocks; the rest go to single-CTA bins packed
    // the same way.  The sequential placement below (TMG_PACK=sequential)
    // leaves 25-35 % of the thread slots idle on tweed and wireframe grids.
    int csmax = 1;
    std::vector<int> order;
    for (size_t b = 0; b < g.blocks.size(); b++) {
      if (g.blocks[b].red != red) continue;
      order.push_back((int)b);
      csmax = std::max(csmax, need[b]);
    }
    if (dense) {
      std::stable_sort(order.begin(), order.end(),
                       [&](int x, int y) { return block_size(x) > block_size(y); });
      constexpr int NW = T / 32;
      for (int pass_cs : {csmax, 1}) {
        std::vector<BinD> bins;
        std::vector<int> maxch, xcta, blks;
        std::vector<std::vector<int>> fill;  // per bin: per warp (cta * NW + w) slots used
        size_t first_open = 0;
        for (int b : order) {
          if (taken[b]) continue;
          if (pass_cs == 1 && need[b] > 1) continue;
          BlockD& B = g.blocks[b];
          std::vector<int> items;
          for (int l = 0; l < B.nleg; l++) items.push_back(l);
          std::stable_sort(items.begin(), items.end(), [&](int x, int y) {
            return g.legs[B.leg0 + x].nchunk > g.legs[B.leg0 + y].nchunk;
          });
          auto try_bin = [&](size_t k, bool commit) {
            std::vector<int> f = fill[k];
            std::vector<int> tb(B.nleg, -1);
            int hub_t = -1;
            auto small = [&](int nch) {  // first warp with room
              for (int w = 0; w < pass_cs * NW; w++)
                if (f[w] + nch <= 32) {
                  const int t = w * 32 + f[w];
                  f[w] += nch;
                  return t;
                }
              return -1;
            };
            if (B.nleg == 0 && (hub_t = small(1)) < 0) return false;
            for (int l : items) {
              const int nch = g.legs[B.leg0 + l].nchunk;
              if (nch <= 32) {
                if ((tb[l] = small(nch)) < 0) return false;
                continue;
              }
              // a long leg starts at the first free slot of a warp and runs
              // on through empty warps of the same CTA (of the whole cluster
              // for a leg longer than a CTA: cross-CTA reduction)
              const bool cross = nch > T;
              for (int c = 0; c < (cross ? 1 : pass_cs) && tb[l] < 0; c++)
                for (int w = c * NW; w < (cross ? pass_cs : c + 1) * NW && tb[l] < 0; w++) {
                  if (f[w] >= 32) continue;
                  const int start = w * 32 + f[w], end = start + nch - 1, we = end / 32;
                  if (we >= (cross ? pass_cs : c + 1) * NW) break;
                  bool empty = true;
                  for (int x = w + 1; x <= we; x++) empty &= f[x] == 0;
                  if (!empty) continue;
                  tb[l] = start;
                  for (int x = w; x < we; x++) f[x] = 32;
                  f[we] = end % 32 + 1;
                }
              if (tb[l] < 0) return false;
            }
            if (!commit) return true;
            fill[k] = f;
            B.bin = (int)k;
            for (int l = 0; l < B.nleg; l++) {
              LegD& L = g.legs[B.leg0 + l];
              L.tbase = tb[l];
              maxch[k] = std::max(maxch[k], L.nchunk);
              if (tb[l] / T != (tb[l] + L.nchunk - 1) / T) xcta[k] = 1;
            }
            B.hub_thread = B.nleg ? -1 : hub_t;
            return true;
          };
          bool ok = false;
          for (size_t k = first_open; k < bins.size() && !ok; k++)
            if (try_bin(k, false)) ok = try_bin(k, true);
          if (!ok && (pass_cs == 1 || need[b] > 1)) {
            bins.push_back(BinD{0, 0, 0, 0});
            maxch.push_back(1);
            xcta.push_back(0);
            fill.push_back(std::vector<int>(pass_cs * NW, 0));
            ok = try_bin(bins.size() - 1, true);
            if (!ok) return "internal: block does not fit an empty bin";
          }
          if (!ok) continue;
          taken[b] = 1;
          blks.push_back(b);
          while (first_open < bins.size() &&
                 *std::min_element(fill[first_open].begin(), fill[first_open].end()) >= 32)
            first_open++;
        }
        if (!blks.empty()) {
          err = emit(red, pass_cs, blks, bins, maxch, xcta, true);
          if (!err.empty()) return err;
        }
        if (pass_cs == 1) break;
      }
    }
    for (int cs = 1; cs <= kMaxCluster; cs *= 2) {
      std::vector<int> blks;
      for (size_t b = 0; b < g.blocks.size(); b++)
        if (g.blocks[b].red == red && need[b] == cs && !taken[b]) blks.push_back((int)b);
      if (blks.empty()) continue;
      std::vector<BinD> bins;
      std::vector<int> maxch, xcta;
      int bin = -1, vpos = 0;
      for (int b : blks) {
        BlockD& B = g.blocks[b];
        for (int attempt = 0; attempt < 2; attempt++) {
          int v = vpos;
          bool ok = bin >= 0;
          std::vector<int> tb(B.nleg);
          int hub_t = -1;
          if (ok && B.nleg == 0) {
            hub_t = v;
            v += 1;
          }
          for (int l = 0; ok && l < B.nleg; l++) {
            const int nch = g.legs[B.leg0 + l].nchunk;
            tb[l] = place(v, nch);
            v = tb[l] + nch;
          }
          if (ok && v > cs * T) ok = false;
          if (!ok) {
            if (attempt == 1) return "internal: block does not fit an empty bin";
            bin++;
            vpos = 0;
            bins.push_back(BinD{0, 0, 0, 0});
            maxch.push_back(1);
            xcta.push_back(0);
            continue;
          }
          vpos = v;
          B.bin = bin;
          for (int l = 0; l < B.nleg; l++) {
            LegD& L = g.legs[B.leg0 + l];
            L.tbase = tb[l];
            maxch[bin] = std::max(maxch[bin], L.nchunk);
            if (tb[l] / T != (tb[l] + L.nchunk - 1) / T) xcta[bin] = 1;
          }
          B.hub_thread = B.nleg ? -1 : hub_t;
          break;
        }
      }
      err = emit(red, cs, blks, bins, maxch, xcta, true);
      if (!err.empty()) return err;
    }
  }
  P.d_legs = upload(g.legs, P.device_bytes, err);
  P.d_blocks = upload(g.blocks, P.device_bytes, err);
  return err;
}

static int step_dir(long di, long dj) {
  if (di == -1 && dj == 0) return DW;
  if (di == 1 && dj == 0) return DE;
  if (di == 0 && dj == -1) return DS;
  if (di == 0 && dj == 1) return DN;
  return -1;
}

// Path p_0..p_{n-1} of 4-neighbour steps -> leg with <= 4 straight segments.
static std::string path_leg(int blk, const long long* ii, const long long* jj, long n, LegD& L) {
  std::memset(&L, 0, sizeof(L));
  if (n < 1) return "empty leg";
  L.i0 = (int)ii[0];
  L.j0 = (int)jj[0];
  L.npts = (int)n;
  L.block = blk;
  L.hub_dir_first = DNONE;
  L.hub_dir_last = DNONE;
  L.nseg = 1;
  L.seg_dir[0] = DE;
  L.seg_len[0] = 0;
  int ns = 0;
  for (long k = 1; k < n; k++) {
    int d = step_dir(ii[k] - ii[k - 1], jj[k] - jj[k - 1]);
    if (d < 0) return "block members are not 4-neighbour adjacent";
    if (ns > 0 && L.seg_dir[ns - 1] == d) {
      L.seg_len[ns - 1]++;
    } else {
      if (ns == 4) return "block path has more than 4 straight segments";
      L.seg_dir[ns] = (uint8_t)d;
      L.seg_len[ns] = 1;
      ns++;
    }
  }
  L.nseg = (uint8_t)(ns > 0 ? ns : 1);
  return "";
}

std::string add_explicit_block(Geometry& g, int kind, long n, const long long* ii,
                               const long long* jj, long m, const long long* offs, long bi,
                               long bj) {
  auto new_block = [&](int hi, int hj) {
    BlockD b;
    std::memset(&b, 0, sizeof(b));
    b.hi = hi;
    b.hj = hj;
    b.leg0 = (int)g.legs.size();
    b.hub_thread = -1;
    b.bin = -1;
    b.red = 1;
    g.blocks.push_back(b);
    return (int)g.blocks.size() - 1;
  };
  std::string err;
  if (kind == 0) {  // merged point blocks
    for (long k = 0; k < n; k++) new_block((int)ii[k], (int)jj[k]);
    return "";
  }
  if (kind == 1) {  // open chain (_ckernels.pyx:91-103); m == 1 is a point
    if (n == 1) { new_block((int)ii[0], (int)jj[0]); return ""; }
    int b = new_block(-1, -1);
    LegD L;
    err = path_leg(b, ii, jj, n, L);
    if (!err.empty()) return err;
    g.legs.push_back(L);
    g.blocks[b].nleg = 1;
    return "";
  }
  if (kind == 2) {  // ring: chain p_0..p_{n-2}, hub p_{n-1} (_ckernels.pyx:106-141)
    if (n < 3) return "circulant system needs m >= 3";
    int b = new_block((int)ii[n - 1], (int)jj[n - 1]);
    LegD L;
    err = path_leg(b, ii, jj, n - 1, L);
    if (!err.empty()) return err;
    int df = step_dir(ii[n - 1] - ii[0], jj[n - 1] - jj[0]);
    int dl = step_dir(ii[n - 1] - ii[n - 2], jj[n - 1] - jj[n - 2]);
    if (df < 0 || dl < 0) return "ring is not closed by 4-neighbour steps";
    L.flags = 3;
    L.hub_dir_first = (uint8_t)df;
    L.hub_dir_last = (uint8_t)dl;
    g.legs.push_back(L);
    g.blocks[b].nleg = 1;
    g.blocks[b].hub_mask = (uint8_t)((1u << dir_opp(df)) | (1u << dir_opp(dl)));
    return "";
  }
  if (kind == 3) {  // legged (_ckernels.pyx:144-185)
    if (m < 1) return "legged block needs legs";
    int b = new_block((int)bi, (int)bj);
    for (long k = 0; k < m; k++) {
      long lo = (long)offs[k], hi = (long)offs[k + 1];
      LegD L;
      err = path_leg(b, ii + lo, jj + lo, hi - lo, L);
      if (!err.empty()) return err;
      int dl = step_dir(bi - ii[hi - 1], bj - jj[hi - 1]);
      if (dl < 0) return "leg does not end next to the branch point";
      L.flags = 2;
      L.hub_dir_last = (uint8_t)dl;
      g.legs.push_back(L);
      g.blocks[b].nleg++;
      g.blocks[b].hub_mask |= (uint8_t)(1u << dir_opp(dl));
    }
    return "";
  }
  return "bad block kind";
}

void free_plan(Plan& p) {
  if (p.arena) {  // arena-backed arrays are owned by the arena
    p.classes.clear();
    p.d_legs = nullptr;
    p.d_blocks = nullptr;
    return;
  }
  for (auto& c : p.classes) {
    cudaFree(c.chunks);
    cudaFree(c.bins);
    cudaFree(c.hubs);
  }
  p.classes.clear();
  cudaFree(p.d_legs);
  cudaFree(p.d_blocks);
  p.d_legs = nullptr;
  p.d_blocks = nullptr;
  if (p.lp) {
    free_leg_plan(*p.lp);
    delete p.lp;
    p.lp = nullptr;
  }
}

}  // namespace tmg

// Packing statistics of a full plan, computed on the host without a device:
// out[0..3] red (CTAs, threads holding a chunk, points in chunks, hubs),
// out[4..7] the same for black.  Returns 0, or -1 with the error in stderr.
extern "C" int tmg_plan_stats(int scheme, int nx, int ny, int q, int mode, long long* out) {
  tmg::g_dry_run = true;
  for (auto& v : tmg::g_stats) v = 0;
  tmg::Plan P;
  std::string err = tmg::build_plan(scheme, nx, ny, q, mode, P);
  tmg::g_dry_run = false;
  for (int k = 0; k < 8; k++) out[k] = tmg::g_stats[k];
  std::fprintf(stderr, "uniform warps %lld of %lld\n", tmg::g_stats[8], tmg::g_stats[9]);
  if (!err.empty()) {
    std::fprintf(stderr, "tmg_plan_stats: %s\n", err.c_str());
    return -1;
  }
  return 0;
}
