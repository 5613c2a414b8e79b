// GPU uniform-grid broadphase for vertex-triangle proximity.
//
// Reference: contact.point_distances / feasibility_step_cap test ALL
// (surface vertex, surface triangle) pairs of distinct bodies by brute force
// (contact.py:229-239, assembly.py:279-290). Here every surface triangle is
// inserted into each grid cell its AABB, inflated by the query radius r,
// overlaps; a vertex only visits the triangles of its own cell. Any
// triangle within distance < r of the vertex contains the vertex in its
// inflated AABB, so the candidate set is a superset of the exact set and
// the (unchanged, reference-rounding) narrowphase yields the identical pair
// set. Entries are radix-sorted by cell key (stable, so the triangles of a
// cell stay in ascending id order): candidates arrive in the reference's
// row-major (vertex, triangle) order without a per-vertex sort.
#pragma once
#include <chrono>
#include <cstdio>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "context.cuh"
#include "geometry.cuh"

namespace jgs2 {

constexpr long long kCellOff = 1LL << 20;

__device__ __forceinline__ long long cell_coord(double v, double inv_cell) {
  long long c = (long long)floor(v * inv_cell);
  c = c < -kCellOff + 1 ? -kCellOff + 1 : (c > kCellOff - 2 ? kCellOff - 2 : c);
  return c;
}
__device__ __forceinline__ unsigned long long cell_key(long long ix, long long iy, long long iz) {
  return ((unsigned long long)(ix + kCellOff) << 42) | ((unsigned long long)(iy + kCellOff) << 21) |
         (unsigned long long)(iz + kCellOff);
}

struct TriGridDev {
  const unsigned long long* keys;  // sorted cell keys
  const int* tris;                 // triangle ids, ascending within a key
  long long n;
  double inv_cell;
};

__device__ __forceinline__ void tri_bounds(const int* st, int t, const double* x, const double* dx,
                                           double gamma, double r, double inv_cell, long long* lo,
                                           long long* hi) {
  double a[3], b[3], c[3];
  load_pos(x, dx, gamma, st[3 * t], a);
  load_pos(x, dx, gamma, st[3 * t + 1], b);
  load_pos(x, dx, gamma, st[3 * t + 2], c);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double mn = fmin(a[k], fmin(b[k], c[k])) - r;
    double mx = fmax(a[k], fmax(b[k], c[k])) + r;
    lo[k] = cell_coord(mn, inv_cell);
    hi[k] = cell_coord(mx, inv_cell);
  }
}

__global__ void k_grid_count(int nst, const int* st, const double* x, const double* dx, double gamma,
                             double r, double inv_cell, long long* counts) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > nst) return;
  if (t == nst) { counts[t] = 0; return; }
  long long lo[3], hi[3];
  tri_bounds(st, t, x, dx, gamma, r, inv_cell, lo, hi);
  long long c = (hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1);
  counts[t] = (c > 0 && c < (1LL << 20)) ? c : (1LL << 40);  // flags garbage (NaN) bounds
}

__global__ void k_grid_write(int nst, const int* st, const double* x, const double* dx, double gamma,
                             double r, double inv_cell, const long long* off, unsigned long long* keys,
                             int* tris) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nst) return;
  long long lo[3], hi[3];
  tri_bounds(st, t, x, dx, gamma, r, inv_cell, lo, hi);
  long long o = off[t];
  if (off[t + 1] == o) return;
  for (long long i = lo[0]; i <= hi[0]; ++i)
    for (long long j = lo[1]; j <= hi[1]; ++j)
      for (long long k = lo[2]; k <= hi[2]; ++k) {
        keys[o] = cell_key(i, j, k);
        tris[o] = t;
        ++o;
      }
}

// [first, last) of entries with this key
__device__ __forceinline__ void grid_range(const TriGridDev& g, unsigned long long key, long long* first,
                                           long long* last) {
  long long lo = 0, hi = g.n;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (g.keys[mid] < key) lo = mid + 1; else hi = mid;
  }
  *first = lo;
  hi = g.n;
  while (lo < hi) {
    long long mid = (lo + hi) >> 1;
    if (g.keys[mid] <= key) lo = mid + 1; else hi = mid;
  }
  *last = lo;
}

// Entries of one cell are in ascending object id order and objects are
// numbered body by body, so the entries of body `bv` form one contiguous
// run [o0, o1) of [q0, q1). Cross-body queries visit [q0, o0) and [o1, q1)
// (still ascending) and never touch the own-body bulk of a cell, which is
// nearly all of it for a surface vertex. body(q) = body of entry q.
template <class BodyOf>
__device__ __forceinline__ void own_run(long long q0, long long q1, int bv, BodyOf body, long long* o0,
                                        long long* o1) {
  if (q0 >= q1 || body(q0) > bv || body(q1 - 1) < bv) { *o0 = *o1 = q1; return; }
  long long lo = q0, hi = q1;
  while (lo < hi) { long long m = (lo + hi) >> 1; if (body(m) < bv) lo = m + 1; else hi = m; }
  *o0 = lo;
  hi = q1;
  while (lo < hi) { long long m = (lo + hi) >> 1; if (body(m) <= bv) lo = m + 1; else hi = m; }
  *o1 = lo;
}

// visit(entry) for the entries of [q0, q1) not of body bv, in order
template <class BodyOf, class Visit>
__device__ __forceinline__ void visit_cross(long long q0, long long q1, int bv, BodyOf body, Visit visit) {
  long long o0, o1;
  own_run(q0, q1, bv, body, &o0, &o1);
  for (long long q = q0; q < o0; ++q) visit(q);
  for (long long q = o1; q < q1; ++q) visit(q);
}

__device__ __forceinline__ unsigned long long point_key(const double* p, double inv_cell) {
  return cell_key(cell_coord(p[0], inv_cell), cell_coord(p[1], inv_cell), cell_coord(p[2], inv_cell));
}

inline TriGridDev grid_dev(const TriGrid& g) {
  return TriGridDev{g.keys_b, g.tris_b, g.n, 1.0 / g.cell};
}

inline void tri_grid_free(TriGrid& g) {
  cudaFree(g.counts); cudaFree(g.off); cudaFree(g.keys_a); cudaFree(g.keys_b);
  cudaFree(g.tris_a); cudaFree(g.tris_b); cudaFree(g.temp);
  g = TriGrid();
}

// Build the grid of surface triangles at x + gamma*dx inflated by r.
// One host sync (the entry count).
inline void tri_grid_build(Ctx& C, TriGrid& g, const double* x, const double* dx, double gamma, double r,
                           double cell) {
  int nst = C.nst;
  g.cell = cell;
  if (!g.counts) {
    JGS2_CUDA(cudaMalloc(&g.counts, (nst + 1) * sizeof(long long)));
    JGS2_CUDA(cudaMalloc(&g.off, (nst + 1) * sizeof(long long)));
  }
  k_grid_count<<<grid_for(nst + 1), kBlock, 0, C.stream>>>(nst, C.st, x, dx, gamma, r, 1.0 / cell, g.counts);
  C.check_launch();
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, g.counts, g.off, nst + 1, C.stream);
  if (tb > g.temp_bytes) {  // grow with slack: cudaFree/cudaMalloc stall the device
    cudaFree(g.temp);
    JGS2_CUDA(cudaMalloc(&g.temp, 2 * tb));
    g.temp_bytes = 2 * tb;
  }
  JGS2_CUDA(cub::DeviceScan::ExclusiveSum(g.temp, tb, g.counts, g.off, nst + 1, C.stream));
  ++C.launches;
  long long total = 0;
  static const bool dbg = getenv("JGS2_DEBUG_PAIRS") != nullptr;
  auto tq = std::chrono::steady_clock::now();
  JGS2_CUDA(cudaMemcpyAsync(&total, g.off + nst, sizeof(long long), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  if (dbg) {
    double w = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq).count();
    if (w > 20.0) fprintf(stderr, "grid: count+scan sync waited %.2f ms\n", w);
  }
  if (total < 0 || total > 64LL * (nst + 1) + (1LL << 24))
    throw Error(-2, "broadphase: grid entry count " + std::to_string(total) +
                        " out of range (non-finite positions or oversized query radius)");
  if (total > g.cap) {
    cudaFree(g.keys_a); cudaFree(g.keys_b); cudaFree(g.tris_a); cudaFree(g.tris_b);
    long long cap = std::max<long long>(total + total / 2, 1024);
    JGS2_CUDA(cudaMalloc(&g.keys_a, cap * sizeof(unsigned long long)));
    JGS2_CUDA(cudaMalloc(&g.keys_b, cap * sizeof(unsigned long long)));
    JGS2_CUDA(cudaMalloc(&g.tris_a, cap * sizeof(int)));
    JGS2_CUDA(cudaMalloc(&g.tris_b, cap * sizeof(int)));
    g.cap = cap;
  }
  g.n = total;
  k_grid_write<<<grid_for(nst), kBlock, 0, C.stream>>>(nst, C.st, x, dx, gamma, r, 1.0 / cell, g.off, g.keys_a,
                                                       g.tris_a);
  C.check_launch();
  size_t sb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sb, g.keys_a, g.keys_b, g.tris_a, g.tris_b, (int)total, 0, 63,
                                  C.stream);
  if (sb > g.temp_bytes) {  // the sort's scratch grows with the entry count: 1.5x slack
    cudaFree(g.temp);
    JGS2_CUDA(cudaMalloc(&g.temp, sb + sb / 2));
    g.temp_bytes = sb + sb / 2;
  }
  JGS2_CUDA(cub::DeviceRadixSort::SortPairs(g.temp, sb, g.keys_a, g.keys_b, g.tris_a, g.tris_b, (int)total,
                                            0, 63, C.stream));
  ++C.launches;
  if (dbg) {
    auto ts = std::chrono::steady_clock::now();
    C.sync();
    double w = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts).count();
    if (w > 20.0) fprintf(stderr, "grid: write+sort took %.2f ms (entries %lld)\n", w, total);
  }
}

}  // namespace jgs2
