// Two-sided hierarchical proximity search between surface vertices and
// surface triangles of different bodies, for per-object search radii that
// vary over orders of magnitude within one sweep (the exact collect can move
// whole bodies while most of the surface barely moves).
//
// Each object carries a radius rho = b * s + pad, s = its step length |dx|
// (a triangle: max over its corners). A (v, t) pair with
//     dist(x_v, T(x)) < rho_v + rho_t
// has overlapping boxes (v's box of half-size rho_v, t's AABB inflated by
// rho_t), and every such pair meets in one hierarchical grid:
//   * objects are binned by level l = ceil(log2(rho / cell)) (cell * 2^l is
//     the cell size of grid l, so a box covers at most 4^3 cells of its own
//     grid);
//   * triangles of level <= L are inserted into triangle grid L; a vertex of
//     level L queries triangle grid L;
//   * vertices of level <= L are inserted into vertex grid L; a triangle of
//     level L queries vertex grid L.
// A pair is seen by the query of its higher-level object (both queries when
// the levels tie). Objects whose own-level box would still cover more than
// kHierMaxCells cells ("big", only for steps of kilometres) scan all
// opposing objects instead.
//
// Two uses:
//   * feasibility_step_cap (assembly.py:279-290), MIN mode: 0.9 min over
//     cross pairs of dist / (s_v + s_t). Given an upper bound cap_ub, only
//     pairs with dist < (cap_ub / 0.9)(s_v + s_t) can lower it: b = cap_ub /
//     0.9, pad = 0. Repeats are harmless for a min.
//   * the candidate superset of the batched backtracking trials
//     (trials.cuh), LIST mode: every pair that can be within dhat at any
//     x + gamma dx, gamma <= gamma_max, has dist(x) < dhat + gamma_max (s_v +
//     s_t): b = gamma_max, pad = dhat / 2, and the exact distance at x
//     filters the boxes. Each pair is emitted exactly once: the triangle
//     side drops level ties, and within a query a pair is only reported in
//     the grid cell holding the min corner of the intersection of the two
//     boxes (a cell both objects cover).
// Cell entries are in ascending object order and objects are numbered body
// by body, so own-body runs are skipped without being read (own_run).
//
// Cells are indexed densely: every level's grid covers the bounding box of
// the surface (cell coordinates are clamped to it, which keeps every
// overlapping pair of boxes meeting: an overlap of two boxes around objects
// inside the bounding box always reaches into it), a 32-bit key is the
// level's offset plus the row-major cell index, and a per-cell [start, end)
// directory built after the radix sort replaces a binary search per lookup.
// The level-0 cell is at least 1/255 of the largest extent.
#pragma once
#include <chrono>
#include "broadphase.cuh"
#include "contact.cuh"

namespace jgs2 {

constexpr int kHierLevels = 14;
constexpr long long kHierMaxCells = 4096;
constexpr int kHierBig = 0x100;  // level flag: object scans all opposing objects

enum HierMode { HIER_MIN = 0, HIER_COUNT = 1, HIER_WRITE = 2 };

struct HierGeom {
  double org[3];              // bounding-box origin (lower corner)
  int n[kHierLevels][3];      // cells per axis at each level
  unsigned off[kHierLevels];  // first cell index of each level
  unsigned ncells;            // all levels
};

struct HierArgs {
  ContactDev cd;
  const double* x;
  const double* dx;
  double b;      // radius per unit step
  double pad;    // radius added to every object
  double cell;   // level-0 cell size
  double dlim;   // LIST mode: keep pairs with dist < 2 pad + b (s_v + s_t) (slack included in b, pad)
  HierGeom g;
  unsigned long long* stats = nullptr;  // diagnostics (JGS2_DEBUG_HIER): cells, cross entries, pairs
};

__device__ __forceinline__ int hier_level(double rho, double cell) {
  if (!(rho > cell)) return 0;
  double q = ceil(log2(rho / cell));
  if (!(q < kHierLevels - 1)) return kHierLevels - 1;  // also catches NaN
  return q < 0 ? 0 : (int)q;
}
// clamped cell coordinate along axis k at level L (monotone in v)
__device__ __forceinline__ int hier_coord(const HierArgs& a, int L, int k, double v, double inv) {
  double c = floor((v - a.g.org[k]) * inv);
  int hi = a.g.n[L][k] - 1;
  return c < 0.0 ? 0 : (c > (double)hi ? hi : (int)c);  // NaN -> hi
}
__device__ __forceinline__ unsigned hier_cell(const HierArgs& a, int L, int i, int j, int k) {
  return a.g.off[L] + ((unsigned)k * a.g.n[L][1] + j) * a.g.n[L][0] + i;
}

__device__ __forceinline__ double tri_step(const double* dx, const int* st, int t) {
  return fmax(fmax(norm3_np(dx + 3 * st[3 * t]), norm3_np(dx + 3 * st[3 * t + 1])),
              norm3_np(dx + 3 * st[3 * t + 2]));
}
__device__ __forceinline__ void tri_box(const HierArgs& a, int t, double r, double* lo, double* hi) {
  const int* st = a.cd.st;
  for (int k = 0; k < 3; ++k) {
    double p0 = a.x[3 * st[3 * t] + k], p1 = a.x[3 * st[3 * t + 1] + k], p2 = a.x[3 * st[3 * t + 2] + k];
    lo[k] = fmin(p0, fmin(p1, p2)) - r;
    hi[k] = fmax(p0, fmax(p1, p2)) + r;
  }
}
__device__ __forceinline__ void vtx_box(const HierArgs& a, int v, double r, double* lo, double* hi) {
  for (int k = 0; k < 3; ++k) { lo[k] = a.x[3 * v + k] - r; hi[k] = a.x[3 * v + k] + r; }
}
__device__ __forceinline__ double vtx_rho(const HierArgs& a, int v) { return a.b * norm3_np(a.dx + 3 * v) + a.pad; }
__device__ __forceinline__ double tri_rho(const HierArgs& a, int t) { return a.b * tri_step(a.dx, a.cd.st, t) + a.pad; }

__device__ __forceinline__ double level_inv(const HierArgs& a, int L) { return 1.0 / (a.cell * (double)(1LL << L)); }

// clamped cell range of a box at level L; returns the number of cells
__device__ __forceinline__ long long box_cells(const HierArgs& a, int L, const double* lo, const double* hi,
                                               int* c0, int* c1) {
  double inv = level_inv(a, L);
  long long n = 1;
  for (int k = 0; k < 3; ++k) {
    c0[k] = hier_coord(a, L, k, lo[k], inv);
    c1[k] = hier_coord(a, L, k, hi[k], inv);
    n *= (long long)(c1[k] - c0[k] + 1);
  }
  return n;
}

// Objects are indexed o in [0, nsv + nst): surface vertices (sv index) first,
// then surface triangles. Both grids share one sorted entry list: a vertex
// entry's key is ncells + cell (vertex grid), a triangle entry's key is the
// cell (triangle grid).

// per-object levels (+ kHierBig) and level occupancy masks [vertices, triangles]
__global__ void k_hier_levels(HierArgs a, int* lev, unsigned* masks) {
  int o = blockIdx.x * blockDim.x + threadIdx.x;
  int nsv = a.cd.nsv;
  unsigned vbit = 0, tbit = 0;
  if (o < nsv + a.cd.nst) {
    double lo[3], hi[3];
    int c0[3], c1[3];
    double r;
    if (o < nsv) {
      int v = a.cd.sv[o];
      r = vtx_rho(a, v);
      vtx_box(a, v, r, lo, hi);
    } else {
      r = tri_rho(a, o - nsv);
      tri_box(a, o - nsv, r, lo, hi);
    }
    int l = hier_level(r, a.cell);
    bool big = box_cells(a, l, lo, hi, c0, c1) > kHierMaxCells;
    lev[o] = l | (big ? kHierBig : 0);
    (o < nsv ? vbit : tbit) = 1u << l;
  }
  // one atomic per warp and side (a same-address atomic per thread serialises)
  vbit = __reduce_or_sync(0xffffffffu, vbit);
  tbit = __reduce_or_sync(0xffffffffu, tbit);
  if ((threadIdx.x & 31) == 0) {
    if (vbit) atomicOr(masks, vbit);
    if (tbit) atomicOr(masks + 1, tbit);
  }
}

// grid entries of one object: the cells of its box in every grid L >= its
// level that the opposing side occupies (big objects: none)
template <bool WRITE>
__global__ void k_hier_entries(HierArgs a, const int* lev, const unsigned* masks, const long long* off,
                               long long* cnt, unsigned* keys, int* ids) {
  int o = blockIdx.x * blockDim.x + threadIdx.x;
  int nsv = a.cd.nsv;
  if (o >= nsv + a.cd.nst) return;
  bool vert = o < nsv;
  double lo[3], hi[3];
  if (vert) vtx_box(a, a.cd.sv[o], vtx_rho(a, a.cd.sv[o]), lo, hi);
  else tri_box(a, o - nsv, tri_rho(a, o - nsv), lo, hi);
  int lv = lev[o];
  long long n = 0;
  if (!(lv & kHierBig)) {
    unsigned mask = masks[vert ? 1 : 0];  // levels the opposing side occupies
    unsigned base = vert ? a.g.ncells : 0u;
    int id = vert ? o : o - nsv;
    long long q = WRITE ? off[o] : 0;
    for (int L = lv; L < kHierLevels; ++L) {
      if (!((mask >> L) & 1u)) continue;
      int c0[3], c1[3];
      long long nc = box_cells(a, L, lo, hi, c0, c1);
      if (WRITE)
        for (int k = c0[2]; k <= c1[2]; ++k)
          for (int j = c0[1]; j <= c1[1]; ++j)
            for (int i = c0[0]; i <= c1[0]; ++i) {
              keys[q] = base + hier_cell(a, L, i, j, k);
              ids[q] = id;
              ++q;
            }
      n += nc;
    }
  }
  if (!WRITE) cnt[o] = n;
}

// Body runs of the sorted entries: a run is a maximal stretch of one cell
// and one body (entries of a cell are in ascending object order, objects
// numbered body by body). flag[i] = 1 where a run starts.
__device__ __forceinline__ int entry_body(const ContactDev& cd, unsigned key, int id, unsigned ncells) {
  return key >= ncells ? cd.vbody[cd.sv[id]] : cd.tbody[id];
}
__global__ void k_hier_run_flags(ContactDev cd, const unsigned* keys, const int* ids, long long n, unsigned ncells,
                                 int* flag) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned k = keys[i];
  flag[i] = (i == 0 || keys[i - 1] != k ||
             entry_body(cd, k, ids[i], ncells) != entry_body(cd, keys[i - 1], ids[i - 1], ncells)) ? 1 : 0;
}
// runs (begin entry, body; run_begin[R] = n) and the per-cell run range
// [cstart, cend) (cells without entries keep 0, 0)
__global__ void k_hier_runs(ContactDev cd, const unsigned* keys, const int* ids, long long n, unsigned ncells,
                            const int* flag, const int* rix, int* run_begin, int* run_body, int* cstart, int* cend) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned k = keys[i];
  int r = rix[i] + flag[i] - 1;  // run of entry i (rix = exclusive scan of the starts)
  if (flag[i]) {
    run_begin[r] = (int)i;
    run_body[r] = entry_body(cd, k, ids[i], ncells);
  }
  if (i == 0 || keys[i - 1] != k) cstart[k] = r;
  if (i == n - 1 || keys[i + 1] != k) cend[k] = r + 1;
  if (i == n - 1) run_begin[r + 1] = (int)n;
}

// visit(e) for the entries of cell runs [r0, r1) whose body is not `own`, in order
template <class Visit>
__device__ __forceinline__ void visit_cross_runs(int r0, int r1, int own, const int* run_begin, const int* run_body,
                                                 Visit visit) {
  for (int r = r0; r < r1; ++r) {
    if (run_body[r] == own) continue;
    for (int e = run_begin[r], e1 = run_begin[r + 1]; e < e1; ++e) visit(e);
  }
}

// dist(x_v, T(x)) and the pair's step rate s_v + s_t (cross-body pairs only)
__device__ __forceinline__ double pair_dist(const HierArgs& a, int v, int t, double* rate) {
  const int* st = a.cd.st;
  int a0 = st[3 * t], a1 = st[3 * t + 1], a2 = st[3 * t + 2];
  *rate = norm3_np(a.dx + 3 * v) + tri_step(a.dx, st, t);
  double bary[3];
  return closest_point_tri(a.x + 3 * v, a.x + 3 * a0, a.x + 3 * a1, a.x + 3 * a2, bary);
}

// the min-corner cell rule: is (p, q, s) the (clamped) cell of max(lo_a, lo_b)?
__device__ __forceinline__ bool owns_pair(const HierArgs& a, int L, const double* la, const double* lb, double inv,
                                          int p, int q, int s) {
  return hier_coord(a, L, 0, fmax(la[0], lb[0]), inv) == p && hier_coord(a, L, 1, fmax(la[1], lb[1]), inv) == q &&
         hier_coord(a, L, 2, fmax(la[2], lb[2]), inv) == s;
}

struct HierOut {
  double mn = INFINITY;   // MIN
  long long n = 0;        // COUNT / WRITE
  long long o = 0;        // WRITE cursor
  int* cv = nullptr;
  int* ct = nullptr;
  unsigned long long ncell = 0, nent = 0, npair = 0;
  __device__ __forceinline__ void flush(const HierArgs& a) {
    if (a.stats) { atomicAdd(a.stats, ncell); atomicAdd(a.stats + 1, nent); atomicAdd(a.stats + 2, npair); }
  }
  template <int MODE>
  __device__ __forceinline__ void take(const HierArgs& a, int v, int t) {
    ++npair;
    double rate;
    double d = pair_dist(a, v, t, &rate);
    if (MODE == HIER_MIN) {
      if (rate > 1e-30) mn = fmin(mn, d / rate);
    } else if (d < a.dlim + a.b * rate) {
      if (MODE == HIER_WRITE) { cv[o] = v; ct[o] = t; ++o; }
      ++n;
    }
  }
};

// Grouped form of the MIN and COUNT queries: kHierGroup lanes per object,
// the object's cells (or, for big objects, the opposing objects) strided
// over the lanes. Per-object work varies by orders of magnitude (box sizes
// follow the step rates), and one thread per object left the launch a
// long tail (ncu: 6-7% achieved occupancy of 25% theoretical, IPC 0.4).
// MIN is a min and COUNT an integer sum, so both results are identical to
// a sequential per-object scan; WRITE (k_hier_write_grp) keeps that scan's
// candidate order.
constexpr int kHierGroup = 8;
template <int MODE>
__global__ void k_hier_query_grp(HierArgs a, const int* lev, const int* cstart, const int* cend, const int* ids,
                                 const int* run_begin, const int* run_body, long long* cnt, double* partials,
                                 unsigned* counter, double* out) {
  static_assert(MODE != HIER_WRITE, "WRITE is k_hier_write_grp");
  HierOut R;
  const int nsv = a.cd.nsv, nobj = nsv + a.cd.nst;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int sub = gt % kHierGroup;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = ((1u << kHierGroup) - 1u) << (lane & ~(kHierGroup - 1));
  const int ng = (gridDim.x * blockDim.x) / kHierGroup;
  for (int o = gt / kHierGroup; o < nobj; o += ng) {
    int lv = lev[o];
    if (o < nsv) {  // ---- vertex side
      int v = a.cd.sv[o];
      int bv = a.cd.vbody[v];
      if (lv & kHierBig) {
        for (int t = sub; t < a.cd.nst; t += kHierGroup)
          if (a.cd.tbody[t] != bv && !(lev[nsv + t] & kHierBig)) R.take<MODE>(a, v, t);
      } else {
        double lo[3], hi[3], tl[3], th[3];
        vtx_box(a, v, vtx_rho(a, v), lo, hi);
        double inv = level_inv(a, lv);
        int c0[3], c1[3];
        box_cells(a, lv, lo, hi, c0, c1);
        int nx = c1[0] - c0[0] + 1, nxy = nx * (c1[1] - c0[1] + 1);
        int ncl = nxy * (c1[2] - c0[2] + 1);
        for (int k = sub; k < ncl; k += kHierGroup) {
          int s = c0[2] + k / nxy, q = c0[1] + (k % nxy) / nx, p = c0[0] + k % nx;
          unsigned cell = hier_cell(a, lv, p, q, s);
          ++R.ncell;
          visit_cross_runs(cstart[cell], cend[cell], bv, run_begin, run_body, [&](int e) {
            ++R.nent;
            int t = ids[e];
            if (MODE != HIER_MIN) {
              tri_box(a, t, tri_rho(a, t), tl, th);
              if (!owns_pair(a, lv, lo, tl, inv, p, q, s)) return;
            }
            R.take<MODE>(a, v, t);
          });
        }
      }
    } else {  // ---- triangle side
      int t = o - nsv;
      int bt = a.cd.tbody[t];
      if (lv & kHierBig) {
        for (int i = sub; i < nsv; i += kHierGroup) {
          int v = a.cd.sv[i];
          if (a.cd.vbody[v] != bt) R.take<MODE>(a, v, t);
        }
      } else {
        double lo[3], hi[3], vl[3], vh[3];
        tri_box(a, t, tri_rho(a, t), lo, hi);
        double inv = level_inv(a, lv);
        int c0[3], c1[3];
        box_cells(a, lv, lo, hi, c0, c1);
        int nx = c1[0] - c0[0] + 1, nxy = nx * (c1[1] - c0[1] + 1);
        int ncl = nxy * (c1[2] - c0[2] + 1);
        for (int k = sub; k < ncl; k += kHierGroup) {
          int s = c0[2] + k / nxy, q = c0[1] + (k % nxy) / nx, p = c0[0] + k % nx;
          unsigned cell = a.g.ncells + hier_cell(a, lv, p, q, s);
          ++R.ncell;
          visit_cross_runs(cstart[cell], cend[cell], bt, run_begin, run_body, [&](int e) {
            ++R.nent;
            int i = ids[e];
            int v = a.cd.sv[i];
            if (MODE != HIER_MIN) {
              if ((lev[i] & ~kHierBig) >= lv) return;  // level tie: the vertex side has it
              vtx_box(a, v, vtx_rho(a, v), vl, vh);
              if (!owns_pair(a, lv, lo, vl, inv, p, q, s)) return;
            }
            R.take<MODE>(a, v, t);
          });
        }
      }
    }
    if (MODE == HIER_COUNT) {
      long long n = R.n;
#pragma unroll
      for (int off = kHierGroup / 2; off; off >>= 1) n += __shfl_xor_sync(gmask, n, off, kHierGroup);
      if (sub == 0) cnt[o] = n;
      R.n = 0;
    }
  }
  R.flush(a);
  if (MODE == HIER_MIN) grid_reduce<OP_MIN>(R.mn, partials, counter, out);
}

// Item k of object o's query (a cell of its box, or an opposing object for
// big ones), feeding R.take<MODE>.
struct HierObj {
  int lv, own, id;   // level, own body, vertex (vertex side) or triangle id
  bool vert, big;
  int c0[3], nx, nxy, nitems;
  double lo[3], inv;
};
__device__ __forceinline__ HierObj hier_obj(const HierArgs& a, const int* lev, int o) {
  HierObj h;
  const int nsv = a.cd.nsv;
  h.lv = lev[o];
  h.vert = o < nsv;
  h.big = (h.lv & kHierBig) != 0;
  double hi[3];
  if (h.vert) {
    h.id = a.cd.sv[o];
    h.own = a.cd.vbody[h.id];
    if (!h.big) vtx_box(a, h.id, vtx_rho(a, h.id), h.lo, hi);
  } else {
    h.id = o - nsv;
    h.own = a.cd.tbody[h.id];
    if (!h.big) tri_box(a, h.id, tri_rho(a, h.id), h.lo, hi);
  }
  if (h.big) {
    h.nitems = h.vert ? a.cd.nst : nsv;
  } else {
    h.inv = level_inv(a, h.lv);
    int c1[3];
    box_cells(a, h.lv, h.lo, hi, h.c0, c1);
    h.nx = c1[0] - h.c0[0] + 1;
    h.nxy = h.nx * (c1[1] - h.c0[1] + 1);
    h.nitems = h.nxy * (c1[2] - h.c0[2] + 1);
  }
  return h;
}
template <int MODE>
__device__ __forceinline__ void hier_item(const HierArgs& a, const HierObj& h, int k, const int* lev,
                                          const int* cstart, const int* cend, const int* ids, const int* run_begin,
                                          const int* run_body, HierOut& R) {
  const int nsv = a.cd.nsv;
  if (h.big) {
    if (h.vert) {
      if (a.cd.tbody[k] != h.own && !(lev[nsv + k] & kHierBig)) R.take<MODE>(a, h.id, k);
    } else {
      int v = a.cd.sv[k];
      if (a.cd.vbody[v] != h.own) R.take<MODE>(a, v, h.id);
    }
    return;
  }
  int s = h.c0[2] + k / h.nxy, q = h.c0[1] + (k % h.nxy) / h.nx, p = h.c0[0] + k % h.nx;
  double bl[3], bh[3];
  if (h.vert) {
    unsigned cell = hier_cell(a, h.lv, p, q, s);
    visit_cross_runs(cstart[cell], cend[cell], h.own, run_begin, run_body, [&](int e) {
      int t = ids[e];
      tri_box(a, t, tri_rho(a, t), bl, bh);
      if (!owns_pair(a, h.lv, h.lo, bl, h.inv, p, q, s)) return;
      R.take<MODE>(a, h.id, t);
    });
  } else {
    unsigned cell = a.g.ncells + hier_cell(a, h.lv, p, q, s);
    visit_cross_runs(cstart[cell], cend[cell], h.own, run_begin, run_body, [&](int e) {
      int i = ids[e];
      int v = a.cd.sv[i];
      if ((lev[i] & ~kHierBig) >= h.lv) return;  // level tie: the vertex side has it
      vtx_box(a, v, vtx_rho(a, v), bl, bh);
      if (!owns_pair(a, h.lv, h.lo, bl, h.inv, p, q, s)) return;
      R.take<MODE>(a, v, h.id);
    });
  }
}

// Grouped WRITE: the object's items go to the group in chunks of
// kHierGroup consecutive items; each lane counts its item's pairs, an
// in-group scan places them, and the lane writes them. Items, and pairs
// within an item, land in sequential scan order, so the candidate
// list is bit-identical to a sequential per-object scan's.
__global__ void k_hier_write_grp(HierArgs a, const int* lev, const int* cstart, const int* cend, const int* ids,
                                 const int* run_begin, const int* run_body, const long long* off, int* cv,
                                 int* ct) {
  const int nobj = a.cd.nsv + a.cd.nst;
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int sub = gt % kHierGroup;
  const int lane = threadIdx.x & 31;
  const unsigned gmask = ((1u << kHierGroup) - 1u) << (lane & ~(kHierGroup - 1));
  const int ng = (gridDim.x * blockDim.x) / kHierGroup;
  for (int o = gt / kHierGroup; o < nobj; o += ng) {
    HierObj h = hier_obj(a, lev, o);
    long long base = off[o];
    for (int k0 = 0; k0 < h.nitems; k0 += kHierGroup) {
      int k = k0 + sub;
      HierOut C;
      if (k < h.nitems) hier_item<HIER_COUNT>(a, h, k, lev, cstart, cend, ids, run_begin, run_body, C);
      int c = (int)C.n, incl = c;
#pragma unroll
      for (int d = 1; d < kHierGroup; d <<= 1) {
        int y = __shfl_up_sync(gmask, incl, d, kHierGroup);
        if (sub >= d) incl += y;
      }
      int total = __shfl_sync(gmask, incl, kHierGroup - 1, kHierGroup);
      if (c) {
        HierOut W;
        W.cv = cv; W.ct = ct; W.o = base + incl - c;
        hier_item<HIER_WRITE>(a, h, k, lev, cstart, cend, ids, run_begin, run_body, W);
      }
      base += total;
    }
  }
}

// bounding box of the surface vertices: per-block (min xyz, -max xyz), then one block
__global__ void k_sv_bbox(ContactDev cd, const double* x, double* part) {
  double m[6] = {INFINITY, INFINITY, INFINITY, INFINITY, INFINITY, INFINITY};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cd.nsv; i += gridDim.x * blockDim.x) {
    const double* p = x + 3 * cd.sv[i];
    for (int k = 0; k < 3; ++k) { m[k] = fmin(m[k], p[k]); m[3 + k] = fmin(m[3 + k], -p[k]); }
  }
  for (int k = 0; k < 6; ++k) {
    double r = block_reduce<OP_MIN>(m[k]);
    if (threadIdx.x == 0) part[k * kMaxPartials + blockIdx.x] = r;
    __syncthreads();
  }
}
__global__ void k_bbox_final(const double* part, int nb, double* out) {
  for (int k = 0; k < 6; ++k) {
    double m = INFINITY;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) m = fmin(m, part[k * kMaxPartials + i]);
    m = block_reduce<OP_MIN>(m);
    if (threadIdx.x == 0) out[k] = m;
    __syncthreads();
  }
}

// bounding box of the surface at x, reduced on the device into out[6]
// (min xyz, -max xyz); no host sync
inline void hier_bbox_launch(Ctx& C, const double* x, double* out) {
  if (!C.bbox_part) C.bbox_part = C.alloc<double>(6 * kMaxPartials);
  int nb = std::min(red_grid(C.nsv), kMaxPartials);
  k_sv_bbox<<<nb, kBlock, 0, C.stream>>>(contactdev(C), x, C.bbox_part);
  C.check_launch();
  k_bbox_final<<<1, kBlock, 0, C.stream>>>(C.bbox_part, nb, out);
  C.check_launch();
}

// bounding box on the host: bb[6] = (min xyz, -max xyz)
inline void hier_bbox(Ctx& C, const double* x, double* bb) {
  if (!C.bbox_res) C.bbox_res = C.alloc<double>(6);
  hier_bbox_launch(C, x, C.bbox_res);
  JGS2_CUDA(cudaMemcpyAsync(bb, C.bbox_res, 6 * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
}

// level-0 cell and the dense per-level grids over the bounding box bb
// (any box is correct: cell coordinates are clamped; it only sets the
// resolution)
inline void hier_geometry(Ctx& C, const double* bb, HierArgs& a) {
  double ext[3], emax = 0.0;
  for (int k = 0; k < 3; ++k) {
    double lo = bb[k], hi = -bb[3 + k];
    if (!std::isfinite(lo) || !std::isfinite(hi) || hi < lo) lo = hi = 0.0;
    a.g.org[k] = lo;
    ext[k] = hi - lo;
    emax = std::max(emax, ext[k]);
  }
  a.cell = std::max(C.grid_cell, emax / 255.0);
  unsigned off = 0;
  for (int L = 0; L < kHierLevels; ++L) {
    double cl = a.cell * (double)(1LL << L);
    long long cells = 1;
    for (int k = 0; k < 3; ++k) {
      a.g.n[L][k] = (int)std::min(256.0, std::floor(ext[k] / cl) + 1.0);
      cells *= a.g.n[L][k];
    }
    a.g.off[L] = off;
    off += (unsigned)cells;
  }
  a.g.ncells = off;
}

// exclusive scan of n+1 counts (last one zeroed) -> off; returns the total
inline long long scan_counts(Ctx& C, long long* cnt, long long* off, long long n) {
  JGS2_CUDA(cudaMemsetAsync(cnt + n, 0, sizeof(long long), C.stream));
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, n + 1, C.stream);
  if (tb > C.scan_temp_bytes) { C.scan_temp = C.alloc<char>(tb + tb / 2); C.scan_temp_bytes = tb + tb / 2; }
  JGS2_CUDA(cub::DeviceScan::ExclusiveSum(C.scan_temp, tb, cnt, off, n + 1, C.stream));
  ++C.launches;
  long long total = 0;
  JGS2_CUDA(cudaMemcpyAsync(&total, off + n, sizeof(long long), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  return total;
}

// geometry, levels, both grids (one sorted list) and the cell directory for
// radii b * s + pad. One host sync (the entry count).
inline void hier_prepare(Ctx& C, HierArgs& a, const double* bb) {
  hier_geometry(C, bb, a);
  HierList& h = C.hier;
  int nobj = C.nsv + C.nst;
  if (!C.hier_lev) {
    C.hier_lev = C.alloc<int>(nobj + 1);
    C.hier_masks = C.alloc<unsigned>(2);
    h.cnt = C.alloc<long long>(nobj + 1);
    h.off = C.alloc<long long>(nobj + 1);
  }
  unsigned ndir = 2 * a.g.ncells;
  if ((long long)ndir > h.ncells_cap) {
    h.cstart = C.alloc<int>(ndir);
    h.cend = C.alloc<int>(ndir);
    h.ncells_cap = ndir;
  }
  JGS2_CUDA(cudaMemsetAsync(C.hier_masks, 0, 2 * sizeof(unsigned), C.stream));
  JGS2_CUDA(cudaMemsetAsync(h.cstart, 0, ndir * sizeof(int), C.stream));
  JGS2_CUDA(cudaMemsetAsync(h.cend, 0, ndir * sizeof(int), C.stream));
  k_hier_levels<<<grid_for(nobj), kBlock, 0, C.stream>>>(a, C.hier_lev, C.hier_masks);
  C.check_launch();
  k_hier_entries<false><<<grid_for(nobj), kBlock, 0, C.stream>>>(a, C.hier_lev, C.hier_masks, nullptr, h.cnt,
                                                                nullptr, nullptr);
  C.check_launch();
  long long total = scan_counts(C, h.cnt, h.off, nobj);
  if (total < 0 || total > (long long)INT32_MAX)
    throw Error(-2, "hierarchical grid: entry count " + std::to_string(total) + " out of range");
  if (total > h.cap) {
    long long cap = std::max<long long>(total + total / 2, 4096);
    h.ka = C.alloc<unsigned>(cap); h.kb = C.alloc<unsigned>(cap);
    h.ia = C.alloc<int>(cap); h.ib = C.alloc<int>(cap);
    h.flag = C.alloc<int>(cap); h.rix = C.alloc<int>(cap);
    h.run_begin = C.alloc<int>(cap + 1); h.run_body = C.alloc<int>(cap);
    h.cap = cap;
  }
  h.n = total;
  if (total == 0) return;
  k_hier_entries<true><<<grid_for(nobj), kBlock, 0, C.stream>>>(a, C.hier_lev, C.hier_masks, h.off, nullptr,
                                                               h.ka, h.ia);
  C.check_launch();
  int bits = 1;
  while (bits < 32 && (1ull << bits) < (unsigned long long)ndir) ++bits;
  size_t sb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sb, h.ka, h.kb, h.ia, h.ib, (int)total, 0, bits, C.stream);
  if (sb > C.scan_temp_bytes) { C.scan_temp = C.alloc<char>(sb + sb / 2); C.scan_temp_bytes = sb + sb / 2; }
  JGS2_CUDA(cub::DeviceRadixSort::SortPairs(C.scan_temp, sb, h.ka, h.kb, h.ia, h.ib, (int)total, 0, bits,
                                            C.stream));
  ++C.launches;
  ContactDev cd = contactdev(C);
  k_hier_run_flags<<<grid_for(total), kBlock, 0, C.stream>>>(cd, h.kb, h.ib, total, a.g.ncells, h.flag);
  C.check_launch();
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, h.flag, h.rix, (int)total, C.stream);
  if (tb > C.scan_temp_bytes) { C.scan_temp = C.alloc<char>(tb + tb / 2); C.scan_temp_bytes = tb + tb / 2; }
  JGS2_CUDA(cub::DeviceScan::ExclusiveSum(C.scan_temp, tb, h.flag, h.rix, (int)total, C.stream));
  ++C.launches;
  k_hier_runs<<<grid_for(total), kBlock, 0, C.stream>>>(cd, h.kb, h.ib, total, a.g.ncells, h.flag, h.rix,
                                                        h.run_begin, h.run_body, h.cstart, h.cend);
  C.check_launch();
}

// min over cross-body pairs of dist / rate among the pairs with rate < b
// (those whose boxes of radius b s overlap); INFINITY if there are none
inline double hier_min_ratio(Ctx& C, const double* x, const double* dx, double b, const double* bb) {
  HierArgs a;
  a.cd = contactdev(C);
  a.x = x;
  a.dx = dx;
  a.b = b;
  a.pad = 0.0;
  a.dlim = 0.0;
  bool dbg = getenv("JGS2_DEBUG_HIER") != nullptr;
  auto now = [&]() { if (dbg) C.sync(); return std::chrono::steady_clock::now(); };
  unsigned long long* st = nullptr;
  if (dbg) {
    JGS2_CUDA(cudaMalloc(&st, 6 * sizeof(unsigned long long)));
    JGS2_CUDA(cudaMemset(st, 0, 6 * sizeof(unsigned long long)));
    a.stats = st;
  }
  auto t0 = now();
  hier_prepare(C, a, bb);
  auto t1 = now();
  const HierList& h = C.hier;
  double m = INFINITY;
  int nobj = C.nsv + C.nst;
  k_hier_query_grp<HIER_MIN><<<red_grid((int64_t)nobj * kHierGroup), kBlock, 0, C.stream>>>(
      a, C.hier_lev, h.cstart, h.cend, h.ib, h.run_begin, h.run_body, nullptr, C.partials + R_CAP * kMaxPartials,
      C.counters + R_CAP, C.res + R_CAP);
  C.check_launch();
  JGS2_CUDA(cudaMemcpyAsync(&m, C.res + R_CAP, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  if (dbg) {
    auto t2 = now();
    unsigned mk[2];
    JGS2_CUDA(cudaMemcpy(mk, C.hier_masks, sizeof(mk), cudaMemcpyDeviceToHost));
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    unsigned long long hs[3];
    JGS2_CUDA(cudaMemcpy(hs, st, sizeof(hs), cudaMemcpyDeviceToHost));
    cudaFree(st);
    fprintf(stderr, "hier_min_ratio b=%.3e cell=%.3e ncells=%u entries=%lld masks v=%x t=%x m=%.3e "
            "ms prep %.2f q %.2f | cells %llu cross %llu pairs %llu\n",
            a.b, a.cell, a.g.ncells, h.n, mk[0], mk[1], m, ms(t0, t1), ms(t1, t2), hs[0], hs[1], hs[2]);
  }
  return m;
}

// min over cross-body pairs of dist / rate among pairs that can lower
// cap_ub (ratio < cap_ub / 0.9). The search radius grows geometrically from
// one that keeps every box within 2 level-0 cells: a round with radius
// factor b examines every pair of ratio < b, so the first round that finds
// one has the exact minimum. Steps can be huge (the exact collect spreads
// barrier forces over whole bodies), and the limiting pair is then found
// with small boxes instead of body-sized ones.
inline double hier_cap_min(Ctx& C, const double* x, const double* dx, double cap_ub, double smax,
                           const double* bb) {
  double bmax = cap_ub / 0.9 * (1.0 + 1e-6);
  if (!(smax > 0.0)) return INFINITY;  // nothing moves: no pair lowers the cap
  double b = std::isfinite(smax) ? std::min(bmax, 2.0 * C.grid_cell / smax) : bmax;
  for (;;) {
    double m = hier_min_ratio(C, x, dx, b, bb);
    if (m < b || b >= bmax) return m;
    b = std::min(bmax, 4.0 * b);
  }
}

// Cross-body (vertex, triangle) pairs that can be within dhat at some
// x + gamma dx, gamma <= gmax, each exactly once, into (cv, ct). Returns the
// count, or -1 (nothing written) when it exceeds `budget`.
inline long long hier_candidates(Ctx& C, const double* x, const double* dx, double gmax, long long budget,
                                 const double* bb_in = nullptr) {
  HierArgs a;
  a.cd = contactdev(C);
  a.x = x;
  a.dx = dx;
  a.b = gmax * (1.0 + 1e-6);
  a.pad = 0.5 * C.dhat * (1.0 + 1e-6);
  a.dlim = 2.0 * a.pad;
  double bb[6];
  if (bb_in) memcpy(bb, bb_in, sizeof(bb));
  else hier_bbox(C, x, bb);
  hier_prepare(C, a, bb);
  const HierList& h = C.hier;
  int nobj = C.nsv + C.nst;
  if (!C.cand_cnt) {
    C.cand_cnt = C.alloc<long long>(nobj + 1);
    C.cand_off = C.alloc<long long>(nobj + 1);
  }
  k_hier_query_grp<HIER_COUNT><<<grid_for((int64_t)nobj * kHierGroup), kBlock, 0, C.stream>>>(
      a, C.hier_lev, h.cstart, h.cend, h.ib, h.run_begin, h.run_body, C.cand_cnt, nullptr, nullptr, nullptr);
  C.check_launch();
  long long total = scan_counts(C, C.cand_cnt, C.cand_off, nobj);
  if (total > budget) return -1;
  if (total > C.cand_cap) {
    int64_t cap = std::max<int64_t>(2 * (int64_t)total, 4096);
    C.cand_v = C.alloc<int>(cap);
    C.cand_t = C.alloc<int>(cap);
    C.cand_cap = cap;
  }
  if (total == 0) return 0;
  k_hier_write_grp<<<grid_for((int64_t)nobj * kHierGroup), kBlock, 0, C.stream>>>(
      a, C.hier_lev, h.cstart, h.cend, h.ib, h.run_begin, h.run_body, C.cand_off, C.cand_v, C.cand_t);
  C.check_launch();
  return total;
}

}  // namespace jgs2
