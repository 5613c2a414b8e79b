// Exact multi-body feasibility cap with widely varying step sizes.
//
// feasibility_step_cap (assembly.py:279-290) is 0.9 min over cross-body
// (surface vertex v, surface triangle t) of dist / (s_v + s_t), s = step
// length (max over the triangle's corners). Given an upper bound cap_ub
// (planes, active pairs), only pairs with dist < b (s_v + s_t), b =
// cap_ub / 0.9, can lower it. With rho_v = b s_v, rho_t = b s_t that is the
// overlap of a box of half-size rho_v around v with t's AABB inflated by
// rho_t. Radii vary over orders of magnitude within one sweep (the exact
// collect can move whole bodies), so objects are binned by level
// l = ceil(log2(rho / cell)) and two hierarchical grids are used:
//   * triangles of level <= L are inserted into triangle grid L (cell
//     cell * 2^L, inflated by rho_t); a vertex of level L queries grid L;
//   * vertices of level <= L are inserted into vertex grid L; a triangle of
//     level L queries it.
// Every relevant pair meets in the grid of the larger level; repeats are
// harmless for the min. Objects whose box would cover more than
// kHierMaxCells cells are checked by brute force (rare).
#pragma once
#include "broadphase.cuh"
#include "contact.cuh"

namespace jgs2 {

constexpr int kHierLevels = 14;
constexpr long long kHierMaxCells = 4096;

__device__ __forceinline__ int hier_level(double rho, double cell) {
  if (!(rho > cell)) return 0;
  int l = (int)ceil(log2(rho / cell));
  return l < 0 ? 0 : (l >= kHierLevels ? kHierLevels - 1 : l);
}
__device__ __forceinline__ unsigned long long hier_key(int level, long long ix, long long iy, long long iz) {
  const long long off = 1LL << 19;
  auto cl = [&](long long c) { return c < -off + 1 ? -off + 1 : (c > off - 2 ? off - 2 : c); };
  return ((unsigned long long)level << 60) | ((unsigned long long)(cl(ix) + off) << 40) |
         ((unsigned long long)(cl(iy) + off) << 20) | (unsigned long long)(cl(iz) + off);
}

struct HierArgs {
  ContactDev cd;
  const double* x;
  const double* dx;
  double b;      // cap_ub / 0.9 (with slack)
  double cell;   // level-0 cell size
};

__device__ __forceinline__ double tri_step(const HierArgs& a, int t) {
  const int* st = a.cd.st;
  return fmax(fmax(norm3_np(a.dx + 3 * st[3 * t]), norm3_np(a.dx + 3 * st[3 * t + 1])),
              norm3_np(a.dx + 3 * st[3 * t + 2]));
}
__device__ __forceinline__ void tri_box(const HierArgs& a, int t, double r, double* lo, double* hi) {
  const int* st = a.cd.st;
  for (int k = 0; k < 3; ++k) {
    double p0 = a.x[3 * st[3 * t] + k], p1 = a.x[3 * st[3 * t + 1] + k], p2 = a.x[3 * st[3 * t + 2] + k];
    lo[k] = fmin(p0, fmin(p1, p2)) - r;
    hi[k] = fmax(p0, fmax(p1, p2)) + r;
  }
}
__device__ __forceinline__ long long box_cells(const double* lo, const double* hi, double inv, long long* c0,
                                               long long* c1) {
  long long n = 1;
  for (int k = 0; k < 3; ++k) {
    c0[k] = (long long)floor(lo[k] * inv);
    c1[k] = (long long)floor(hi[k] * inv);
    long long w = c1[k] - c0[k] + 1;
    if (!(w > 0) || w > kHierMaxCells) return kHierMaxCells + 1;
    n *= w;
    if (n > kHierMaxCells) return kHierMaxCells + 1;
  }
  return n;
}

// level occupancy masks and per-object levels
__global__ void k_hier_levels(HierArgs a, int* vlev, int* tlev, unsigned* vmask, unsigned* tmask) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.cd.nsv) {
    int l = hier_level(a.b * norm3_np(a.dx + 3 * a.cd.sv[i]), a.cell);
    vlev[i] = l;
    atomicOr(vmask, 1u << l);
  }
  if (i < a.cd.nst) {
    int l = hier_level(a.b * tri_step(a, i), a.cell);
    tlev[i] = l;
    atomicOr(tmask, 1u << l);
  }
}

// triangle entries: t into grids L >= level(t) that some vertex occupies
template <bool WRITE>
__global__ void k_hier_tri_entries(HierArgs a, const int* tlev, const unsigned* vmask, const long long* off,
                                   long long* cnt, unsigned long long* keys, int* ids, int* over_n, int* over) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.cd.nst) return;
  double r = a.b * tri_step(a, t);
  double lo[3], hi[3];
  tri_box(a, t, r, lo, hi);
  long long n = 0, o = WRITE ? off[t] : 0;
  bool big = false;
  for (int L = tlev[t]; L < kHierLevels; ++L) {
    if (!((*vmask >> L) & 1u)) continue;
    double inv = 1.0 / (a.cell * (double)(1LL << L));
    long long c0[3], c1[3];
    long long nc = box_cells(lo, hi, inv, c0, c1);
    if (nc > kHierMaxCells) { big = true; break; }
    if (WRITE) {
      for (long long i = c0[0]; i <= c1[0]; ++i)
        for (long long j = c0[1]; j <= c1[1]; ++j)
          for (long long k = c0[2]; k <= c1[2]; ++k) {
            keys[o] = hier_key(L, i, j, k);
            ids[o] = t;
            ++o;
          }
    }
    n += nc;
  }
  if (!WRITE) {
    cnt[t] = big ? 0 : n;
    if (big) over[atomicAdd(over_n, 1)] = t;
  }
}

// vertex entries: v into grids L >= level(v) that some triangle occupies
template <bool WRITE>
__global__ void k_hier_vtx_entries(HierArgs a, const int* vlev, const unsigned* tmask, const long long* off,
                                   long long* cnt, unsigned long long* keys, int* ids, int* over_n, int* over) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.cd.nsv) return;
  int v = a.cd.sv[i];
  double r = a.b * norm3_np(a.dx + 3 * v);
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) { lo[k] = a.x[3 * v + k] - r; hi[k] = a.x[3 * v + k] + r; }
  long long n = 0, o = WRITE ? off[i] : 0;
  bool big = false;
  for (int L = vlev[i]; L < kHierLevels; ++L) {
    if (!((*tmask >> L) & 1u)) continue;
    double inv = 1.0 / (a.cell * (double)(1LL << L));
    long long c0[3], c1[3];
    long long nc = box_cells(lo, hi, inv, c0, c1);
    if (nc > kHierMaxCells) { big = true; break; }
    if (WRITE) {
      for (long long p = c0[0]; p <= c1[0]; ++p)
        for (long long q = c0[1]; q <= c1[1]; ++q)
          for (long long s = c0[2]; s <= c1[2]; ++s) {
            keys[o] = hier_key(L, p, q, s);
            ids[o] = i;
            ++o;
          }
    }
    n += nc;
  }
  if (!WRITE) {
    cnt[i] = big ? 0 : n;
    if (big) over[atomicAdd(over_n, 1)] = i;
  }
}

__device__ __forceinline__ void key_range(const unsigned long long* keys, long long n, unsigned long long key,
                                          long long* first, long long* last) {
  long long lo = 0, hi = n;
  while (lo < hi) { long long m = (lo + hi) >> 1; if (keys[m] < key) lo = m + 1; else hi = m; }
  *first = lo;
  hi = n;
  while (lo < hi) { long long m = (lo + hi) >> 1; if (keys[m] <= key) lo = m + 1; else hi = m; }
  *last = lo;
}

__device__ __forceinline__ double pair_ratio(const HierArgs& a, int v, int t) {
  const ContactDev& cd = a.cd;
  if (cd.tbody[t] == cd.vbody[v]) return INFINITY;
  int a0 = cd.st[3 * t], a1 = cd.st[3 * t + 1], a2 = cd.st[3 * t + 2];
  double stt = fmax(fmax(norm3_np(a.dx + 3 * a0), norm3_np(a.dx + 3 * a1)), norm3_np(a.dx + 3 * a2));
  double rate = norm3_np(a.dx + 3 * v) + stt;
  if (!(rate > 1e-30)) return INFINITY;
  double bary[3];
  return closest_point_tri(a.x + 3 * v, a.x + 3 * a0, a.x + 3 * a1, a.x + 3 * a2, bary) / rate;
}

// vertex-side queries (triangle grid) + brute force for oversized vertices
__global__ void k_hier_query_v(HierArgs a, const int* vlev, const unsigned long long* tkeys, const int* tids,
                               long long ntk, const int* over_t, const int* n_over_t, double* partials,
                               unsigned* counter, double* out) {
  double mn = INFINITY;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.cd.nsv; i += gridDim.x * blockDim.x) {
    int v = a.cd.sv[i];
    int no = *n_over_t;
    for (int q = 0; q < no; ++q) mn = fmin(mn, pair_ratio(a, v, over_t[q]));
    double r = a.b * norm3_np(a.dx + 3 * v);
    double lo[3], hi[3];
    for (int k = 0; k < 3; ++k) { lo[k] = a.x[3 * v + k] - r; hi[k] = a.x[3 * v + k] + r; }
    int L = vlev[i];
    double inv = 1.0 / (a.cell * (double)(1LL << L));
    long long c0[3], c1[3];
    if (box_cells(lo, hi, inv, c0, c1) > kHierMaxCells) {
      for (int t = 0; t < a.cd.nst; ++t) mn = fmin(mn, pair_ratio(a, v, t));
      continue;
    }
    for (long long p = c0[0]; p <= c1[0]; ++p)
      for (long long q = c0[1]; q <= c1[1]; ++q)
        for (long long s = c0[2]; s <= c1[2]; ++s) {
          long long f, l;
          key_range(tkeys, ntk, hier_key(L, p, q, s), &f, &l);
          for (long long e = f; e < l; ++e) mn = fmin(mn, pair_ratio(a, v, tids[e]));
        }
  }
  grid_reduce<OP_MIN>(mn, partials, counter, out);
}

// triangle-side queries (vertex grid) + brute force for oversized triangles
__global__ void k_hier_query_t(HierArgs a, const int* tlev, const unsigned long long* vkeys, const int* vids,
                               long long nvk, const int* over_v, const int* n_over_v, double* partials,
                               unsigned* counter, double* out) {
  double mn = INFINITY;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < a.cd.nst; t += gridDim.x * blockDim.x) {
    int no = *n_over_v;
    for (int q = 0; q < no; ++q) mn = fmin(mn, pair_ratio(a, a.cd.sv[over_v[q]], t));
    double r = a.b * tri_step(a, t);
    double lo[3], hi[3];
    tri_box(a, t, r, lo, hi);
    int L = tlev[t];
    double inv = 1.0 / (a.cell * (double)(1LL << L));
    long long c0[3], c1[3];
    if (box_cells(lo, hi, inv, c0, c1) > kHierMaxCells) {
      for (int i = 0; i < a.cd.nsv; ++i) mn = fmin(mn, pair_ratio(a, a.cd.sv[i], t));
      continue;
    }
    for (long long p = c0[0]; p <= c1[0]; ++p)
      for (long long q = c0[1]; q <= c1[1]; ++q)
        for (long long s = c0[2]; s <= c1[2]; ++s) {
          long long f, l;
          key_range(vkeys, nvk, hier_key(L, p, q, s), &f, &l);
          for (long long e = f; e < l; ++e) mn = fmin(mn, pair_ratio(a, a.cd.sv[vids[e]], t));
        }
  }
  grid_reduce<OP_MIN>(mn, partials, counter, out);
}

inline void hier_alloc(Ctx& C, HierList& h, int nobj) {
  if (h.cnt) return;
  h.cnt = C.alloc<long long>(nobj + 1);
  h.off = C.alloc<long long>(nobj + 1);
  h.over = C.alloc<int>(nobj + 1);
  h.n_over = C.alloc<int>(1);
}

template <class CountK, class WriteK>
inline void hier_build(Ctx& C, HierList& h, int nobj, CountK count, WriteK write) {
  hier_alloc(C, h, nobj);
  JGS2_CUDA(cudaMemsetAsync(h.n_over, 0, sizeof(int), C.stream));
  JGS2_CUDA(cudaMemsetAsync(h.cnt + nobj, 0, sizeof(long long), C.stream));
  count(h);
  C.check_launch();
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, h.cnt, h.off, nobj + 1, C.stream);
  if (tb > C.scan_temp_bytes) { C.scan_temp = C.alloc<char>(tb); C.scan_temp_bytes = tb; }
  JGS2_CUDA(cub::DeviceScan::ExclusiveSum(C.scan_temp, tb, h.cnt, h.off, nobj + 1, C.stream));
  ++C.launches;
  long long total = 0;
  JGS2_CUDA(cudaMemcpyAsync(&total, h.off + nobj, sizeof(long long), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  if (total > h.cap) {
    long long cap = std::max<long long>(total + total / 2, 4096);
    h.ka = C.alloc<unsigned long long>(cap); h.kb = C.alloc<unsigned long long>(cap);
    h.ia = C.alloc<int>(cap); h.ib = C.alloc<int>(cap);
    h.cap = cap;
  }
  h.n = total;
  write(h);
  C.check_launch();
  size_t sb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sb, h.ka, h.kb, h.ia, h.ib, (int)total, 0, 64, C.stream);
  if (sb > C.scan_temp_bytes) { C.scan_temp = C.alloc<char>(sb); C.scan_temp_bytes = sb; }
  JGS2_CUDA(cub::DeviceRadixSort::SortPairs(C.scan_temp, sb, h.ka, h.kb, h.ia, h.ib, (int)total, 0, 64,
                                            C.stream));
  ++C.launches;
}

// min over cross-body pairs of dist / rate among pairs that can lower cap_ub
inline double hier_cap_min(Ctx& C, const double* x, const double* dx, double cap_ub) {
  HierArgs a;
  a.cd = contactdev(C);
  a.x = x;
  a.dx = dx;
  a.b = cap_ub / 0.9 * (1.0 + 1e-6);
  a.cell = C.grid_cell;
  if (!C.hier_vlev) {
    C.hier_vlev = C.alloc<int>(C.nsv + 1);
    C.hier_tlev = C.alloc<int>(C.nst + 1);
    C.hier_masks = C.alloc<unsigned>(2);
  }
  JGS2_CUDA(cudaMemsetAsync(C.hier_masks, 0, 2 * sizeof(unsigned), C.stream));
  int nmax = std::max(C.nsv, C.nst);
  k_hier_levels<<<grid_for(nmax), kBlock, 0, C.stream>>>(a, C.hier_vlev, C.hier_tlev, C.hier_masks,
                                                         C.hier_masks + 1);
  C.check_launch();
  HierList& T = C.hier_tri;
  HierList& V = C.hier_vtx;
  hier_build(C, T, C.nst,
             [&](HierList& h) {
               k_hier_tri_entries<false><<<grid_for(C.nst), kBlock, 0, C.stream>>>(
                   a, C.hier_tlev, C.hier_masks, nullptr, h.cnt, nullptr, nullptr, h.n_over, h.over);
             },
             [&](HierList& h) {
               k_hier_tri_entries<true><<<grid_for(C.nst), kBlock, 0, C.stream>>>(
                   a, C.hier_tlev, C.hier_masks, h.off, nullptr, h.ka, h.ia, nullptr, nullptr);
             });
  hier_build(C, V, C.nsv,
             [&](HierList& h) {
               k_hier_vtx_entries<false><<<grid_for(C.nsv), kBlock, 0, C.stream>>>(
                   a, C.hier_vlev, C.hier_masks + 1, nullptr, h.cnt, nullptr, nullptr, h.n_over, h.over);
             },
             [&](HierList& h) {
               k_hier_vtx_entries<true><<<grid_for(C.nsv), kBlock, 0, C.stream>>>(
                   a, C.hier_vlev, C.hier_masks + 1, h.off, nullptr, h.ka, h.ia, nullptr, nullptr);
             });
  k_hier_query_v<<<red_grid(C.nsv), kBlock, 0, C.stream>>>(a, C.hier_vlev, T.kb, T.ib, T.n, T.over, T.n_over,
                                                           C.partials + R_CAP * kMaxPartials,
                                                           C.counters + R_CAP, C.res + R_CAP);
  C.check_launch();
  double m1 = INFINITY, m2 = INFINITY;
  JGS2_CUDA(cudaMemcpyAsync(&m1, C.res + R_CAP, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  k_hier_query_t<<<red_grid(C.nst), kBlock, 0, C.stream>>>(a, C.hier_tlev, V.kb, V.ib, V.n, V.over, V.n_over,
                                                           C.partials + R_CAP * kMaxPartials,
                                                           C.counters + R_CAP, C.res + R_CAP);
  C.check_launch();
  JGS2_CUDA(cudaMemcpyAsync(&m2, C.res + R_CAP, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  return std::fmin(m1, m2);
}

}  // namespace jgs2
