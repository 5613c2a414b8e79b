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

// Cell keys are packed relative to the bounding box of all triangle cells
// (k_grid_count reduces it): key = (ix-X0) << (by+bz) | (iy-Y0) << bz | (iz-Z0),
// so the radix sort covers bx+by+bz bits (about 24-30 at C4) instead of 63.
// The key order across cells is irrelevant to the lookups; within a cell the
// stable sort keeps the entries in ascending triangle id.
struct TriGridDev {
  const unsigned long long* keys;  // sorted cell keys
  const int* tris;                 // triangle ids, ascending within a key
  long long n;
  double inv_cell;
  long long x0, y0, z0, x1, y1, z1;  // cell bounding box (inclusive)
  int sy, sz;                        // shifts of the x and y fields
};

__device__ __forceinline__ unsigned long long box_key(const TriGridDev& g, long long i, long long j, long long k) {
  return ((unsigned long long)(i - g.x0) << g.sy) | ((unsigned long long)(j - g.y0) << g.sz) |
         (unsigned long long)(k - g.z0);
}

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

__global__ void k_box_init(long long* box) {
  if (threadIdx.x < 3) box[threadIdx.x] = LLONG_MAX;
  else if (threadIdx.x < 6) box[threadIdx.x] = LLONG_MIN;
}

// entries per triangle, and the cell bounding box of all triangles (box:
// min x y z, max x y z; block-reduced, then one atomic per block and bound)
__global__ void k_grid_count(int nst, const int* st, const double* x, const double* dx, double gamma,
                             double r, double inv_cell, long long* counts, long long* box) {
  __shared__ long long sb[6][kBlock / 32];
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  long long lo[3] = {LLONG_MAX, LLONG_MAX, LLONG_MAX}, hi[3] = {LLONG_MIN, LLONG_MIN, LLONG_MIN};
  if (t < nst) {
    tri_bounds(st, t, x, dx, gamma, r, inv_cell, lo, hi);
    long long c = (hi[0] - lo[0] + 1) * (hi[1] - lo[1] + 1) * (hi[2] - lo[2] + 1);
    counts[t] = (c > 0 && c < (1LL << 20)) ? c : (1LL << 40);  // flags garbage (NaN) bounds
  } else if (t == nst) {
    counts[t] = 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = min(lo[a], __shfl_down_sync(0xffffffffu, lo[a], o));
      hi[a] = max(hi[a], __shfl_down_sync(0xffffffffu, hi[a], o));
    }
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0)
    for (int a = 0; a < 3; ++a) { sb[a][w] = lo[a]; sb[3 + a][w] = hi[a]; }
  __syncthreads();
  if (threadIdx.x < 6) {
    long long v = sb[threadIdx.x][0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      v = threadIdx.x < 3 ? min(v, sb[threadIdx.x][k]) : max(v, sb[threadIdx.x][k]);
    if (threadIdx.x < 3) { if (v != LLONG_MAX) atomicMin(box + threadIdx.x, v); }
    else if (v != LLONG_MIN) atomicMax(box + threadIdx.x, v);
  }
}

__global__ void k_grid_write(int nst, const int* st, const double* x, const double* dx, double gamma,
                             double r, TriGridDev g, const long long* off, unsigned long long* keys,
                             int* tris) {
  const double inv_cell = g.inv_cell;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nst) return;
  long long lo[3], hi[3];
  tri_bounds(st, t, x, dx, gamma, r, inv_cell, lo, hi);
  long long o = off[t];
  if (off[t + 1] == o) return;
  for (long long i = lo[0]; i <= hi[0]; ++i)
    for (long long j = lo[1]; j <= hi[1]; ++j)
      for (long long k = lo[2]; k <= hi[2]; ++k) {
        keys[o] = box_key(g, i, j, k);
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

// the key of p's cell, or ~0 (matches no entry) outside the triangles' box
__device__ __forceinline__ unsigned long long point_key(const TriGridDev& g, const double* p) {
  long long i = cell_coord(p[0], g.inv_cell), j = cell_coord(p[1], g.inv_cell), k = cell_coord(p[2], g.inv_cell);
  if (i < g.x0 || i > g.x1 || j < g.y0 || j > g.y1 || k < g.z0 || k > g.z1) return ~0ULL;
  return box_key(g, i, j, k);
}

inline TriGridDev grid_dev(const TriGrid& g) {
  TriGridDev d{g.keys_b, g.tris_b, g.n, 1.0 / g.cell};
  d.x0 = g.box[0]; d.y0 = g.box[1]; d.z0 = g.box[2];
  d.x1 = g.box[3]; d.y1 = g.box[4]; d.z1 = g.box[5];
  d.sy = g.sy; d.sz = g.sz;
  return d;
}

inline void tri_grid_free(TriGrid& g) {
  cudaFree(g.counts); cudaFree(g.off); cudaFree(g.keys_a); cudaFree(g.keys_b);
  cudaFree(g.tris_a); cudaFree(g.tris_b); cudaFree(g.temp); cudaFree(g.dbox);
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
  if (!g.dbox) JGS2_CUDA(cudaMalloc(&g.dbox, 6 * sizeof(long long)));
  k_box_init<<<1, 32, 0, C.stream>>>(g.dbox);
  C.check_launch();
  k_grid_count<<<grid_for(nst + 1), kBlock, 0, C.stream>>>(nst, C.st, x, dx, gamma, r, 1.0 / cell, g.counts,
                                                           g.dbox);
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
  JGS2_CUDA(cudaMemcpyAsync(g.box, g.dbox, 6 * sizeof(long long), cudaMemcpyDeviceToHost, C.stream));
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
  auto bits_for = [](long long n) { int b = 0; while (b < 62 && (1LL << b) < n) ++b; return b; };
  int bx = 1, by = 1, bz = 1;
  if (total > 0) {
    bx = std::max(1, bits_for(g.box[3] - g.box[0] + 1));
    by = std::max(1, bits_for(g.box[4] - g.box[1] + 1));
    bz = std::max(1, bits_for(g.box[5] - g.box[2] + 1));
  } else {
    for (int a = 0; a < 3; ++a) { g.box[a] = 0; g.box[3 + a] = -1; }  // empty box: no query matches
  }
  if (bx + by + bz > 63) throw Error(-2, "broadphase: cell box too large for 63-bit keys");
  g.sz = bz;
  g.sy = by + bz;
  const int end_bit = bx + by + bz;
  k_grid_write<<<grid_for(nst), kBlock, 0, C.stream>>>(nst, C.st, x, dx, gamma, r, grid_dev(g), g.off, g.keys_a,
                                                       g.tris_a);
  C.check_launch();
  size_t sb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sb, g.keys_a, g.keys_b, g.tris_a, g.tris_b, (int)total, 0, end_bit,
                                  C.stream);
  if (sb > g.temp_bytes) {  // the sort's scratch grows with the entry count: 1.5x slack
    cudaFree(g.temp);
    JGS2_CUDA(cudaMalloc(&g.temp, sb + sb / 2));
    g.temp_bytes = sb + sb / 2;
  }
  JGS2_CUDA(cub::DeviceRadixSort::SortPairs(g.temp, sb, g.keys_a, g.keys_b, g.tris_a, g.tris_b, (int)total,
                                            0, end_bit, C.stream));
  ++C.launches;
  if (dbg) {
    auto ts = std::chrono::steady_clock::now();
    C.sync();
    double w = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts).count();
    if (w > 20.0) fprintf(stderr, "grid: write+sort took %.2f ms (entries %lld)\n", w, total);
  }
}

}  // namespace jgs2
