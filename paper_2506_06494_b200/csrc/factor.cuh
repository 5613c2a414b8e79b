// Rest-Hessian factor: assembly, multifrontal Cholesky and the per-sweep
// supernodal forward/backward substitution of the exact reduced collect
// (reference: local_solver.py:115-126 -> SciPy SuperLU.solve).
//
// Layout in HBM: all front panels live in one FP64 array L; front f owns a
// column-major (nf x ns) panel at f_loff[f] with leading dimension
// nf = ns + nr: rows [0, ns) are the dense diagonal block (lower triangle
// used), rows [ns, nf) the off-diagonal rows (its row structure).
#pragma once
#include "context.cuh"
#include "element_hessian.cuh"

#include <algorithm>
#include <chrono>
#include <map>

namespace jgs2 {

// ---------------------------------------------------------------- element Hessians
// Hbar BSR block (i, j) of free vertices: sum over elements containing both
// (ascending element id) of the projected rest element block + mass term.
__global__ void k_bsr_blocks(int nblocks, const int* brow, const int* bcol, const int* inc_ptr,
                             const int* inc, const int4* tets, const double* mplus_all,
                             const double* mass, double inv_h2, double* bval) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nblocks) return;
  int i = brow[k], j = bcol[k];
  double acc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = 0.0;
  for (int p = inc_ptr[i]; p < inc_ptr[i + 1]; ++p) {
    int code = inc[p], e = code >> 2, si = code & 3;
    int4 t = tets[e];
    int sj = (t.x == j) ? 0 : (t.y == j) ? 1 : (t.z == j) ? 2 : (t.w == j) ? 3 : -1;
    if (sj < 0) continue;
    const double* M = mplus_all + 45 * (size_t)e;
    // H12 block (si, sj) = sum_{p,q} U[si][p] M[(p r),(q s)] U[sj][q]
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        double v = 0.0;
#pragma unroll
        for (int pp = 0; pp < 3; ++pp)
#pragma unroll
          for (int qq = 0; qq < 3; ++qq)
            v += kHad(si, pp) * M[tri9(3 * pp + r, 3 * qq + s)] * kHad(sj, qq);
        acc[3 * r + s] += v;
      }
  }
  if (i == j) {
    double m = mass[i] * inv_h2;
    acc[0] += m; acc[4] += m; acc[8] += m;
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) bval[9 * (size_t)k + q] = acc[q];
}

__global__ void k_scatter_orig(int nblocks, const int64_t* dst, const int* ld, const double* bval,
                               double* L) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nblocks) return;
  int64_t d = dst[k];
  if (d < 0) return;
  int l = ld[k];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) L[d + (int64_t)c * l + a] = bval[9 * (size_t)k + 3 * a + c];
}

// Extend-add of a child's update matrix (nr_c x nr_c, lower) into its parent.
__global__ void k_extend_add(int nrc, const double* Uc, const int* rmap, int nsp, int nfp,
                             double* Lp, int nrp, double* Up) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t tot = (int64_t)nrc * nrc;
  if (idx >= tot) return;
  int a = (int)(idx % nrc), bcol = (int)(idx / nrc);
  if (a < bcol) return;
  double v = Uc[idx];
  int ra = rmap[a], rb = rmap[bcol];
  if (rb < nsp) Lp[(int64_t)rb * nfp + ra] += v;
  else Up[(int64_t)(rb - nsp) * nrp + (ra - nsp)] += v;
}

// ------------------------------------------------------------------ solve kernels
// Partitioned-inverse storage (Alvarado-Pothen style): every front keeps
//   P = [ L11^-1 ; W ],  W = L21 L11^-1   (nf x ns, column major, ld nf)
// so the forward step of a front is one matvec  t = P v_s
//   z_s = t[0:ns],  u = v_r - t[ns:nf]
// and the backward step one transposed matvec  x_s = P^T [z_s ; -x_r].
// There is no dependency chain inside a front: a front's rows (forward) or
// columns (backward) are split over many CTAs; fronts depend only on their
// children (forward) / ancestors (backward), one launch per tree level.
constexpr int kSolveThreads = 256;
// Panel leading dimension, in doubles. The apply kernels read 64-row chunks
// of a column; with columns aligned to 128 B (the L2 line) a chunk covers
// whole lines. At 16-B alignment (ld even) ncu counted 10% more DRAM bytes
// than the panels hold (profiles/r2_traffic_c4.json). Override with
// JGS2_LD_ALIGN (2 = round-1 layout) for A/B measurements.
constexpr int kLdAlignDefault = 16;
inline int ld_align() {
  static const int a = [] {
    const char* e = getenv("JGS2_LD_ALIGN");
    int v = e ? atoi(e) : kLdAlignDefault;
    return (v >= 2 && (v & 1) == 0) ? v : kLdAlignDefault;
  }();
  return a;
}
constexpr int kSmemCapDoubles = 16384;  // 128 KB vector cache

__global__ void k_zero_upper(int ns, int nf, double* P) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t tot = (int64_t)ns * ns;
  if (idx >= tot) return;
  int r = (int)(idx % ns), c = (int)(idx / ns);
  if (r < c) P[(int64_t)c * nf + r] = 0.0;
}

// forward assembly: v_f = [y_cols ; 0] + extend-add of the children's
// update vectors (children in ascending order: deterministic)
__global__ void __launch_bounds__(kSolveThreads)
k_fwd_assemble(const int* fronts, const int* colbeg, const int* f_ns, const int* f_nr,
               const int64_t* uoff, const int64_t* woff, const int* cptr, const int* clist,
               const int64_t* sptr, const int* rmap, const double* b, const double* u, double* w) {
  int f = fronts[blockIdx.x];
  int ns = f_ns[f], nf = ns + f_nr[f];
  double* v = w + woff[f];
  int cb = colbeg[f];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) v[i] = (i < ns) ? b[cb + i] : 0.0;
  __syncthreads();
  for (int k = cptr[f]; k < cptr[f + 1]; ++k) {
    int c = clist[k];
    int nrc = f_nr[c];
    const int* rm = rmap + sptr[c];
    const double* uc = u + uoff[c];
    for (int i = threadIdx.x; i < nrc; i += blockDim.x) v[rm[i]] += uc[i];
    __syncthreads();
  }
}

// forward apply, task = (front, row_begin, row_end): rows of t = P v_s.
// Persistent CTAs stride over the level's tasks. Lanes own row pairs
// (double2 loads: 512 B per warp-load, columns are 16-B aligned since ld is
// even), warps split the columns (w, w+8, ...), 8 loads in flight per warp;
// partial sums are combined across warps in a fixed order (deterministic).
constexpr int kVecCache = 4096;  // doubles of the vector cached in smem (32 KB)
constexpr int kApplyCtasPerSm = 4;
// persistent grid of the block apply kernels, CTAs per SM (JGS2_SOLVE_CTAS)
inline int solve_ctas() {
  static const int v = [] {
    const char* e = getenv("JGS2_SOLVE_CTAS");
    int c = e ? atoi(e) : kApplyCtasPerSm;
    return (c >= 1 && c <= kApplyCtasPerSm) ? c : kApplyCtasPerSm;
  }();
  return v;
}

__global__ void __launch_bounds__(kSolveThreads, kApplyCtasPerSm)
k_fwd_apply(const int4* tasks, int ntasks, const int* colbeg, const int* f_ns, const int* f_nr,
            const int* f_ld, const int64_t* loff, const int64_t* uoff, const int64_t* woff,
            const double* __restrict__ L, const double* __restrict__ w, double* b, double* u) {
  __shared__ double sv[kVecCache];
  __shared__ double red[8][65];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    int4 tk = tasks[t];
    int f = tk.x, r0 = tk.y, r1 = tk.z;
    int ns = f_ns[f], nf = ns + f_nr[f], ld = f_ld[f];
    const double* P = L + loff[f];
    const double* v = w + woff[f];
    int cmax = min(ns, r1);
    const double* vs = v;
    __syncthreads();  // previous task done with sv
    if (cmax <= kVecCache) {
      for (int i = threadIdx.x; i < cmax; i += blockDim.x) sv[i] = v[i];
      vs = sv;
    }
    __syncthreads();
    int cb = colbeg[f];
    for (int i0 = r0; i0 < r1; i0 += 64) {
      int row = i0 + 2 * lane;  // rows row, row + 1 (row + 1 may be the zero pad row)
      int cend = min(ns, i0 + 64);
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
      if (row < r1) {
        const double2* Pr = reinterpret_cast<const double2*>(P + row);
        const int64_t s = (int64_t)ld / 2;  // column stride in double2
        int j = warp;
        for (; j + 24 < cend; j += 32) {
          double2 p0 = __ldg(Pr + (int64_t)j * s);
          double2 p1 = __ldg(Pr + (int64_t)(j + 8) * s);
          double2 p2 = __ldg(Pr + (int64_t)(j + 16) * s);
          double2 p3 = __ldg(Pr + (int64_t)(j + 24) * s);
          double v0 = vs[j], v1 = vs[j + 8], v2 = vs[j + 16], v3 = vs[j + 24];
          a0 += p0.x * v0; b0 += p0.y * v0;
          a1 += p1.x * v1; b1 += p1.y * v1;
          a2 += p2.x * v2; b2 += p2.y * v2;
          a3 += p3.x * v3; b3 += p3.y * v3;
        }
        for (; j < cend; j += 8) {
          double2 p0 = __ldg(Pr + (int64_t)j * s);
          double v0 = vs[j];
          a0 += p0.x * v0; b0 += p0.y * v0;
        }
      }
      red[warp][2 * lane] = (a0 + a1) + (a2 + a3);
      red[warp][2 * lane + 1] = (b0 + b1) + (b2 + b3);
      __syncthreads();
      if (warp < 2) {
        int r = i0 + 32 * warp + lane;
        int c = 32 * warp + lane;
        if (r < r1) {
          double tt = ((red[0][c] + red[1][c]) + (red[2][c] + red[3][c])) +
                      ((red[4][c] + red[5][c]) + (red[6][c] + red[7][c]));
          if (r < ns) b[cb + r] = tt;
          else u[uoff[f] + (r - ns)] = v[r] - tt;
        }
      }
      __syncthreads();
    }
  }
}

// forward apply on the top levels, where a few wide fronts give too few row
// tasks to fill the GPU (65-189 CTAs measured on C4: 0.8-2.6 TB/s). A task is
// (64-row block, column chunk); every chunk writes its partial rows to
// scratch, and the last chunk of a row block to finish (atomic ticket) sums
// the partials in chunk order (deterministic) and writes z / u. The ticket
// is reset by that last chunk, so the captured graph replays.
struct SplitTask {
  int f, r0, c0, c1;      // rows [r0, r0 + 64), columns [c0, c1)
  int slot, nk, k, blk;   // partials at part[(slot + k) * 64], nk chunks, ticket blk
};
constexpr int kSplitMaxCols = 2048;
__global__ void __launch_bounds__(kSolveThreads, kApplyCtasPerSm)
k_fwd_apply_split(const SplitTask* tasks, int ntasks, const int* colbeg, const int* f_ns, const int* f_nr,
                  const int* f_ld, const int64_t* loff, const int64_t* uoff, const int64_t* woff,
                  const double* __restrict__ L, const double* __restrict__ w, double* b, double* u,
                  double* part, unsigned* ticket) {
  __shared__ double sv[kSplitMaxCols];
  __shared__ double red[8][65];
  __shared__ int last;
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    SplitTask tk = tasks[t];
    int f = tk.f, r0 = tk.r0, c0 = tk.c0;
    int ns = f_ns[f], nf = ns + f_nr[f], ld = f_ld[f];
    int r1 = min(nf, r0 + 64);
    int c1 = min(tk.c1, min(ns, r1));
    const double* P = L + loff[f];
    const double* v = w + woff[f];
    __syncthreads();  // previous task done with sv / red
    for (int i = threadIdx.x; i < c1 - c0; i += blockDim.x) sv[i] = v[c0 + i];
    __syncthreads();
    int row = r0 + 2 * lane;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, b0 = 0, b1 = 0, b2 = 0, b3 = 0;
    if (row < r1) {
      const double2* Pr = reinterpret_cast<const double2*>(P + row);
      const int64_t s = (int64_t)ld / 2;
      int j = c0 + warp;
      for (; j + 24 < c1; j += 32) {
        double2 p0 = __ldg(Pr + (int64_t)j * s);
        double2 p1 = __ldg(Pr + (int64_t)(j + 8) * s);
        double2 p2 = __ldg(Pr + (int64_t)(j + 16) * s);
        double2 p3 = __ldg(Pr + (int64_t)(j + 24) * s);
        double v0 = sv[j - c0], v1 = sv[j + 8 - c0], v2 = sv[j + 16 - c0], v3 = sv[j + 24 - c0];
        a0 += p0.x * v0; b0 += p0.y * v0;
        a1 += p1.x * v1; b1 += p1.y * v1;
        a2 += p2.x * v2; b2 += p2.y * v2;
        a3 += p3.x * v3; b3 += p3.y * v3;
      }
      for (; j < c1; j += 8) {
        double2 p0 = __ldg(Pr + (int64_t)j * s);
        double v0 = sv[j - c0];
        a0 += p0.x * v0; b0 += p0.y * v0;
      }
    }
    red[warp][2 * lane] = (a0 + a1) + (a2 + a3);
    red[warp][2 * lane + 1] = (b0 + b1) + (b2 + b3);
    __syncthreads();
    int r = r0 + threadIdx.x;  // threads 0-63 own one row each
    double tt = 0.0;
    if (threadIdx.x < 64) {
      int c = threadIdx.x;
      tt = ((red[0][c] + red[1][c]) + (red[2][c] + red[3][c])) +
           ((red[4][c] + red[5][c]) + (red[6][c] + red[7][c]));
    }
    if (tk.nk == 1) {
      if (threadIdx.x < 64 && r < r1) {
        if (r < ns) b[colbeg[f] + r] = tt;
        else u[uoff[f] + (r - ns)] = v[r] - tt;
      }
      continue;
    }
    if (threadIdx.x < 64) part[(int64_t)(tk.slot + tk.k) * 64 + threadIdx.x] = tt;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(ticket + tk.blk, 1u) == (unsigned)tk.nk - 1);
    __syncthreads();
    if (!last) continue;
    __threadfence();
    if (threadIdx.x < 64 && r < r1) {
      double acc = 0.0;
      for (int k = 0; k < tk.nk; ++k) acc += __ldcg(part + (int64_t)(tk.slot + k) * 64 + threadIdx.x);
      if (r < ns) b[colbeg[f] + r] = acc;
      else u[uoff[f] + (r - ns)] = v[r] - acc;
    }
    if (threadIdx.x == 0) ticket[tk.blk] = 0u;
  }
}

// forward apply for narrow fronts (ns <= kNarrowCols: the leaves and the
// small separators of the lower levels), task = (front, 64-row chunk): one
// warp per task, lanes own row pairs across all columns, v broadcast from
// L1. No shared memory and no block barriers (the block-level kernel's
// per-64-row cross-warp reduction dominates on narrow panels).
constexpr int kNarrowCols = 128;
// A/B switches for the solve schedule (measurements in DESIGN.md §4):
// JGS2_BWD_NARROW=0 runs narrow fronts' backward step in the block kernel,
// JGS2_SOLVE_FORK=0 serialises a level's narrow and wide launches.
inline bool env_on(const char* name) {
  const char* e = getenv(name);
  return !(e && e[0] == '0');
}
// narrow backward tasks only for short fronts: a tall narrow front (a small
// separator high in the tree) streams each column from one warp, where the
// block kernel puts 8 warps on it. JGS2_BWD_NARROW=<rows> (0 = off).
inline int narrow_bwd_rows() {
  static const int v = [] {
    const char* e = getenv("JGS2_BWD_NARROW");
    return e ? atoi(e) : 512;
  }();
  return v;
}
inline bool split_fwd() {
  static const bool v = env_on("JGS2_SPLIT_FWD");
  return v;
}
inline bool solve_fork() {
  static const bool v = env_on("JGS2_SOLVE_FORK");
  return v;
}
__global__ void __launch_bounds__(kSolveThreads)
k_fwd_apply_narrow(const int4* tasks, int ntasks, const int* colbeg, const int* f_ns, const int* f_nr,
                   const int* f_ld, const int64_t* loff, const int64_t* uoff, const int64_t* woff,
                   const double* __restrict__ L, const double* __restrict__ w, double* b, double* u) {
  int lane = threadIdx.x & 31;
  int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = w0; t < ntasks; t += nw) {
    int4 tk = tasks[t];
    int f = tk.x, r0 = tk.y, r1 = tk.z;
    int ns = f_ns[f], ld = f_ld[f];
    const double* P = L + loff[f];
    const double* v = w + woff[f];
    int row = r0 + 2 * lane;
    if (row >= r1) continue;
    int cend = min(ns, r1);
    const double2* Pr = reinterpret_cast<const double2*>(P + row);
    const int64_t s2 = (int64_t)ld / 2;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0, c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    int j = 0;
    for (; j + 7 < cend; j += 8) {  // 8 column loads in flight per lane
      double2 p0 = __ldg(Pr + (int64_t)j * s2);
      double2 p1 = __ldg(Pr + (int64_t)(j + 1) * s2);
      double2 p2 = __ldg(Pr + (int64_t)(j + 2) * s2);
      double2 p3 = __ldg(Pr + (int64_t)(j + 3) * s2);
      double2 p4 = __ldg(Pr + (int64_t)(j + 4) * s2);
      double2 p5 = __ldg(Pr + (int64_t)(j + 5) * s2);
      double2 p6 = __ldg(Pr + (int64_t)(j + 6) * s2);
      double2 p7 = __ldg(Pr + (int64_t)(j + 7) * s2);
      double v0 = __ldg(v + j), v1 = __ldg(v + j + 1), v2 = __ldg(v + j + 2), v3 = __ldg(v + j + 3);
      double v4 = __ldg(v + j + 4), v5 = __ldg(v + j + 5), v6 = __ldg(v + j + 6), v7 = __ldg(v + j + 7);
      a0 += p0.x * v0; c0 += p0.y * v0;
      a1 += p1.x * v1; c1 += p1.y * v1;
      a2 += p2.x * v2; c2 += p2.y * v2;
      a3 += p3.x * v3; c3 += p3.y * v3;
      a0 += p4.x * v4; c0 += p4.y * v4;
      a1 += p5.x * v5; c1 += p5.y * v5;
      a2 += p6.x * v6; c2 += p6.y * v6;
      a3 += p7.x * v7; c3 += p7.y * v7;
    }
    for (; j + 3 < cend; j += 4) {
      double2 p0 = __ldg(Pr + (int64_t)j * s2);
      double2 p1 = __ldg(Pr + (int64_t)(j + 1) * s2);
      double2 p2 = __ldg(Pr + (int64_t)(j + 2) * s2);
      double2 p3 = __ldg(Pr + (int64_t)(j + 3) * s2);
      double v0 = __ldg(v + j), v1 = __ldg(v + j + 1), v2 = __ldg(v + j + 2), v3 = __ldg(v + j + 3);
      a0 += p0.x * v0; c0 += p0.y * v0;
      a1 += p1.x * v1; c1 += p1.y * v1;
      a2 += p2.x * v2; c2 += p2.y * v2;
      a3 += p3.x * v3; c3 += p3.y * v3;
    }
    for (; j < cend; ++j) {
      double2 p0 = __ldg(Pr + (int64_t)j * s2);
      double v0 = __ldg(v + j);
      a0 += p0.x * v0; c0 += p0.y * v0;
    }
    double t0 = (a0 + a1) + (a2 + a3), t1 = (c0 + c1) + (c2 + c3);
    int cb = colbeg[f];
    int64_t uo = uoff[f];
    if (row < ns) b[cb + row] = t0;
    else u[uo + (row - ns)] = v[row] - t0;
    if (row + 1 < r1) {
      if (row + 1 < ns) b[cb + row + 1] = t1;
      else u[uo + (row + 1 - ns)] = v[row + 1] - t1;
    }
  }
}

// flat forward assembly: w[dst] = b[bsrc] (or 0) + sum of the children's
// update entries mapped to this position (child order, deterministic)
__global__ void k_fwd_assemble_flat(int64_t n, const int64_t* dst, const int* bsrc, const int64_t* cp,
                                    const int64_t* src, const double* b, const double* u, double* w) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int bs = bsrc[k];
  double acc = bs >= 0 ? b[bs] : 0.0;
  for (int64_t q = cp[k]; q < cp[k + 1]; ++q) acc += u[src[q]];
  w[dst[k]] = acc;
}

// flat backward gather: w[dst] = z (src >= 0, from b) or -x (src < 0, from q)
__global__ void k_bwd_gather_flat(int64_t n, const int64_t* dst, const int* src, const double* b,
                                  const double* q, double* w) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  int s = src[k];
  w[dst[k]] = s >= 0 ? b[s] : -q[-1 - s];
}

// backward gather: w_f = [z_s ; -x_r] (contiguous, per front of the level)
__global__ void __launch_bounds__(kSolveThreads)
k_bwd_gather(const int* fronts, const int* colbeg, const int* f_ns, const int* f_nr,
             const int64_t* woff, const int64_t* sptr, const int* sdof, const double* b,
             const double* q, double* w) {
  int f = fronts[blockIdx.x];
  int ns = f_ns[f], nf = ns + f_nr[f];
  if (ns == 0) return;
  double* wf = w + woff[f];
  int cb = colbeg[f];
  const int* sd = sdof + sptr[f];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) wf[i] = (i < ns) ? b[cb + i] : -q[sd[i - ns]];
}

// backward apply, task = (front, col_begin, col_end): x_j = P[:, j] . w_f.
// Persistent CTAs; one warp per column, lanes own row pairs (double2) from the
// even row at or above the diagonal (the entry above it is an explicit zero).
__global__ void __launch_bounds__(kSolveThreads, kApplyCtasPerSm)
k_bwd_apply(const int4* tasks, int ntasks, const int* colbeg, const int* f_ns, const int* f_nr,
            const int* f_ld, const int64_t* loff, const int64_t* woff, const double* __restrict__ L,
            const double* __restrict__ w, double* q) {
  __shared__ double sw[kVecCache];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    int4 tk = tasks[t];
    int f = tk.x, c0 = tk.y, c1 = tk.z;
    int ns = f_ns[f], nf = ns + f_nr[f], ld = f_ld[f];
    const double* P = L + loff[f];
    const double* wf = w + woff[f];
    int e0 = c0 & ~1;        // even start
    int len = ld - e0;       // includes the zero pad row
    const double* ws = wf;
    __syncthreads();
    if (len <= kVecCache) {
      for (int i = threadIdx.x; i < len; i += blockDim.x) sw[i] = wf[e0 + i];
      ws = sw - e0;
    }
    __syncthreads();
    int cb = colbeg[f];
    for (int j = c0 + warp; j < c1; j += 8) {
      const double2* col = reinterpret_cast<const double2*>(P + (int64_t)j * ld);
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
      int i = (j & ~1) + 2 * lane;
      for (; i + 192 < ld; i += 256) {
        double2 p0 = __ldg(col + (i >> 1));
        double2 p1 = __ldg(col + ((i + 64) >> 1));
        double2 p2 = __ldg(col + ((i + 128) >> 1));
        double2 p3 = __ldg(col + ((i + 192) >> 1));
        a0 += p0.x * ws[i] + p0.y * ws[i + 1];
        a1 += p1.x * ws[i + 64] + p1.y * ws[i + 65];
        a2 += p2.x * ws[i + 128] + p2.y * ws[i + 129];
        a3 += p3.x * ws[i + 192] + p3.y * ws[i + 193];
      }
      for (; i < ld; i += 64) {
        double2 p0 = __ldg(col + (i >> 1));
        a0 += p0.x * ws[i] + p0.y * ws[i + 1];
      }
      double acc = warp_sum((a0 + a1) + (a2 + a3));
      if (lane == 0) q[cb + j] = acc;
    }
    (void)nf;
  }
}

// backward apply for narrow fronts (ns <= kNarrowCols), task = (front, group of
// <= 8 columns): one warp per task, no shared memory and no block barriers
// (the block kernel's per-task vector staging and 8-warp split left most warps
// idle on these short columns: 0.9-2.5 TB/s on the lower levels). Lanes own
// row pairs and keep the group's 8 column loads in flight; column j starts at
// its even row at or above the diagonal. The 8 sums are reduced by a
// transposing butterfly (9 shuffles, fixed order: deterministic).
__global__ void __launch_bounds__(kSolveThreads)
k_bwd_apply_narrow(const int4* tasks, int ntasks, const int* colbeg, const int* f_ns, const int* f_nr,
                   const int* f_ld, const int64_t* loff, const int64_t* woff, const double* __restrict__ L,
                   const double* __restrict__ w, double* q) {
  const unsigned full = 0xffffffffu;
  int lane = threadIdx.x & 31;
  int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int t = w0; t < ntasks; t += nw) {
    int4 tk = tasks[t];
    int f = tk.x, c0 = tk.y, c1 = tk.z;
    int nf = f_ns[f] + f_nr[f], ld = f_ld[f];
    const double* P = L + loff[f] + (int64_t)c0 * ld;
    const double2* wf = reinterpret_cast<const double2*>(w + woff[f]);
    int nc = c1 - c0;
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = 0.0;
    for (int i = (c0 & ~1) + 2 * lane; i < nf; i += 64) {
      // all 8 loads issued before any use (a guarded load-use pair per
      // column compiled to one load in flight per warp)
      double2 p[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        p[k] = (k < nc && i + 1 >= c0 + k) ? __ldg(reinterpret_cast<const double2*>(P + (int64_t)k * ld + i))
                                           : make_double2(0.0, 0.0);
      double2 wv = __ldg(wf + (i >> 1));
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] += p[k].x * wv.x + p[k].y * wv.y;
    }
    // lane bit 4 selects columns 0-3 / 4-7, bit 3 pairs, bit 2 the column
    bool h = lane & 16;
    double b4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double send = h ? a[k] : a[k + 4], keep = h ? a[k + 4] : a[k];
      b4[k] = keep + __shfl_xor_sync(full, send, 16);
    }
    h = lane & 8;
    double b2[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      double send = h ? b4[k] : b4[k + 2], keep = h ? b4[k + 2] : b4[k];
      b2[k] = keep + __shfl_xor_sync(full, send, 8);
    }
    h = lane & 4;
    double s = (h ? b2[1] : b2[0]) + __shfl_xor_sync(full, h ? b2[0] : b2[1], 4);
    s += __shfl_xor_sync(full, s, 2);
    s += __shfl_xor_sync(full, s, 1);
    int k = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    if ((lane & 3) == 0 && k < nc) q[colbeg[f] + c0 + k] = s;
  }
}

// ------------------------------------------------------------------ host side
inline void factor_release(Ctx& C) { C.fac = Factor(); }

struct BlockInput {
  int64_t nblocks;
  const int64_t* brow;
  const int64_t* bcol;
  const double* bval;
};

void metis_nd(int n, const int64_t* ptr, const int32_t* adj, int32_t* p);  // fill.cpp
void metis_nd_components(int n, const int64_t* ptr, const int32_t* adj, int32_t* p);
constexpr bool kDefaultMetis = true;

// Build the factor of the free-vertex rest Hessian on the device: either
// assembled from the model at h_ref (blocks == nullptr) or from caller blocks.
void factor_build(Ctx& C, double h_ref, int leaf, const BlockInput* blocks = nullptr) {
  auto t0 = std::chrono::steady_clock::now();
  Factor& F = C.fac;
  F = Factor();
  const int nv = C.nv, ne = C.ne;
  // ---- free-vertex graph (vertex adjacency through elements, incl. self)
  std::vector<int> loc(nv, -1), glob;
  for (int v = 0; v < nv; ++v)
    if (!C.h_fixed[v] && C.owns(v)) { loc[v] = (int)glob.size(); glob.push_back(v); }  // this rank's bodies
  int n = (int)glob.size();
  F.nfree = n;
  std::vector<std::vector<int>> nb(n);
  if (blocks) {
    for (int64_t k = 0; k < blocks->nblocks; ++k) {
      int64_t r = blocks->brow[k], c = blocks->bcol[k];
      if (r < 0 || r >= nv || c < 0 || c >= nv) throw Error(-1, "block index out of range");
      int lr = loc[r], lc = loc[c];
      if (lr >= 0 && lc >= 0) { nb[lr].push_back(lc); nb[lc].push_back(lr); }
    }
  }
  for (int e = 0; e < (blocks ? 0 : ne); ++e) {
    const int64_t* t = &C.h_tets[4 * (size_t)e];
    for (int a = 0; a < 4; ++a) {
      int la = loc[t[a]];
      if (la < 0) continue;
      for (int c = 0; c < 4; ++c) {
        int lc = loc[t[c]];
        if (lc >= 0) nb[la].push_back(lc);
      }
    }
  }
  std::vector<int64_t> aptr(n + 1, 0);
  std::vector<int32_t> adj;
  for (int i = 0; i < n; ++i) {
    auto& s = nb[i];
    s.push_back(i);
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    aptr[i + 1] = aptr[i] + (int64_t)s.size();
    adj.insert(adj.end(), s.begin(), s.end());
  }
  std::vector<double> coords(3 * (size_t)n);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) coords[3 * (size_t)i + c] = C.h_rest[3 * (size_t)glob[i] + c];
  // ordering: METIS nested dissection (cusolverSpXcsrmetisndHost, fill.cpp)
  // with an etree-based front tree, or geometric nested dissection
  // (symbolic.cpp); JGS2_ORDERING=metis|geometric, JGS2_RELAX = amalgamation
  // limit in vertices
  static const char* ord_env = getenv("JGS2_ORDERING");
  const bool use_metis = ord_env ? std::string(ord_env) == "metis"
                                 : (C.ordering >= 0 ? C.ordering == 1 : kDefaultMetis);
  F.ordering_metis = use_metis;
  if (use_metis && n > 0) {
    std::vector<int32_t> pm(n);
    metis_nd_components(n, aptr.data(), adj.data(), pm.data());
    static const char* rx = getenv("JGS2_RELAX");
    build_symbolic_perm(n, aptr.data(), adj.data(), pm.data(), rx ? atoi(rx) : leaf, F.sym);
  } else {
    build_symbolic(n, aptr.data(), adj.data(), coords.data(), leaf, F.sym);
  }
  Symbolic& S = F.sym;
  F.nfronts = S.nfronts;
  F.nlevels = S.nlevels;
  const int NF = S.nfronts;
  // ---- per-front metadata (DOF units)
  std::vector<int> colbeg(NF), fns(NF), fnr(NF), fld(NF), cptr(S.child_ptr), clist(S.child_list);
  std::vector<int64_t> loff(NF + 1, 0), uoff(NF + 1, 0), woff(NF + 1, 0), sptr(NF + 1, 0);
  for (int f = 0; f < NF; ++f) {
    colbeg[f] = 3 * S.col_begin[f];
    fns[f] = 3 * (S.col_end[f] - S.col_begin[f]);
    fnr[f] = 3 * (int)(S.struct_ptr[f + 1] - S.struct_ptr[f]);
    int nf = fns[f] + fnr[f];
    fld[f] = (nf + ld_align() - 1) / ld_align() * ld_align();  // aligned columns (ld_align)
    loff[f + 1] = loff[f] + (int64_t)fld[f] * fns[f];
    uoff[f + 1] = uoff[f] + fnr[f];
    woff[f + 1] = woff[f] + fld[f];
    sptr[f + 1] = sptr[f] + fnr[f];
    F.max_nf = std::max(F.max_nf, nf);
  }
  F.nnz_alloc = loff[NF];
  std::vector<int> sdof(sptr[NF]), rmap(sptr[NF], -1);
  for (int f = 0; f < NF; ++f) {
    int64_t o = sptr[f];
    for (int64_t k = S.struct_ptr[f]; k < S.struct_ptr[f + 1]; ++k)
      for (int c = 0; c < 3; ++c) sdof[o++] = 3 * S.struct_pos[k] + c;
  }
  for (int f = 0; f < NF; ++f) {
    int p = S.parent[f];
    if (p < 0) continue;
    int pcb = S.col_begin[p], pce = S.col_end[p];
    const int* ps = S.struct_pos.data() + S.struct_ptr[p];
    int pn = (int)(S.struct_ptr[p + 1] - S.struct_ptr[p]);
    int pns = 3 * (pce - pcb);
    int64_t o = sptr[f];
    for (int64_t k = S.struct_ptr[f]; k < S.struct_ptr[f + 1]; ++k) {
      int q = S.struct_pos[k];
      int locq;
      if (q >= pcb && q < pce) locq = 3 * (q - pcb);
      else {
        const int* it = std::lower_bound(ps, ps + pn, q);
        if (it == ps + pn || *it != q) throw Error(-1, "symbolic: child row missing from parent");
        locq = pns + 3 * (int)(it - ps);
      }
      for (int c = 0; c < 3; ++c) rmap[o++] = locq + c;
    }
  }
  // levels
  F.level_ptr.assign(F.nlevels + 1, 0);
  for (int f = 0; f < NF; ++f) F.level_ptr[S.level[f] + 1]++;
  for (int l = 0; l < F.nlevels; ++l) F.level_ptr[l + 1] += F.level_ptr[l];
  std::vector<int> lf(NF), fill(F.level_ptr.begin(), F.level_ptr.end() - 1);
  for (int f = 0; f < NF; ++f) lf[fill[S.level[f]]++] = f;
  F.level_maxnf.assign(F.nlevels, 0);
  for (int f = 0; f < NF; ++f)
    F.level_maxnf[S.level[f]] = std::max(F.level_maxnf[S.level[f]], fns[f] + fnr[f]);
  // ---- solve task lists: per level, split fronts into row blocks (forward,
  // multiples of 32 rows) / column blocks (backward, multiples of 8
  // columns) of roughly equal entry counts; enough tasks to fill 2 waves.
  {
    std::vector<int4> ft, bt, fn, bn;
    std::vector<SplitTask> st;
    std::vector<int> wide;
    int split_blocks = 0, split_slots = 0;
    F.split_level_ptr.assign(F.nlevels + 1, 0);
    F.fwd_level_ptr.assign(F.nlevels + 1, 0);
    F.fwdn_level_ptr.assign(F.nlevels + 1, 0);
    F.bwd_level_ptr.assign(F.nlevels + 1, 0);
    F.bwdn_level_ptr.assign(F.nlevels + 1, 0);
    F.fwd_level_smem.assign(F.nlevels, 0);
    F.bwd_level_smem.assign(F.nlevels, 0);
    for (int l = 0; l < F.nlevels; ++l) {
      double work = 0;
      for (int k = F.level_ptr[l]; k < F.level_ptr[l + 1]; ++k) {
        int f = lf[k];
        double ns = fns[f], nr = fnr[f];
        work += ns * (ns + 1) / 2 + nr * ns + nr;
      }
      double T = std::max(work / (16.0 * 148), 4096.0);
      for (int k = F.level_ptr[l]; k < F.level_ptr[l + 1]; ++k) {
        int f = lf[k];
        int ns = fns[f], nf = fns[f] + fnr[f];
        // forward rows
        int r0 = 0;
        double acc = 0;
        if (ns <= kNarrowCols) {  // narrow front: one warp task per 64-row chunk
          for (int i0 = 0; i0 < nf; i0 += 64) fn.push_back(make_int4(f, i0, std::min(nf, i0 + 64), 0));
          r0 = nf;
        }
        if (r0 < nf) wide.push_back(f);
        for (int i0 = r0; i0 < nf; i0 += 64) {
          int rows = std::min(64, nf - i0);
          int cols = std::min(ns, i0 + 64);
          acc += (double)rows * std::max(cols, 1);
          if (acc >= T || i0 + 64 >= nf) {
            int r1 = std::min(nf, i0 + 64);
            ft.push_back(make_int4(f, r0, r1, 0));
            F.fwd_level_smem[l] = std::max(F.fwd_level_smem[l], std::min(ns, r1));
            r0 = r1;
            acc = 0;
          }
        }
        // backward columns
        int c0 = 0;
        acc = 0;
        if (ns <= kNarrowCols && nf <= narrow_bwd_rows()) {  // narrow front: one warp task per 8 columns
          for (int j = 0; j < ns; j += 8) bn.push_back(make_int4(f, j, std::min(ns, j + 8), 0));
          continue;
        }
        for (int j = 0; j < ns; j += 8) {
          int cols = std::min(8, ns - j);
          acc += (double)cols * (nf - j);
          if (acc >= T || j + 8 >= ns) {
            int c1 = std::min(ns, j + 8);
            bt.push_back(make_int4(f, c0, c1, 0));
            F.bwd_level_smem[l] = std::max(F.bwd_level_smem[l], nf - c0);
            c0 = c1;
            acc = 0;
          }
        }
      }
      // too few row tasks to fill the GPU: (64-row block, column chunk) tasks
      int nrow = (int)ft.size() - F.fwd_level_ptr[l];
      if (split_fwd() && nrow > 0 && nrow < 148 * kApplyCtasPerSm / 2) {
        ft.resize(F.fwd_level_ptr[l]);
        double ent = 0;
        for (int f : wide) {
          double ns = fns[f], nf = fns[f] + fnr[f];
          ent += ns * (ns + 1) / 2 + (nf - ns) * ns;
        }
        int W = (int)(ent / (64.0 * 2 * 148 * kApplyCtasPerSm)) / 64 * 64;
        W = std::min(std::max(W, 256), kSplitMaxCols);
        for (int f : wide) {
          int ns = fns[f], nf = fns[f] + fnr[f];
          for (int i0 = 0; i0 < nf; i0 += 64) {
            int cmax = std::min(ns, i0 + 64);
            int nk = std::max(1, (cmax + W - 1) / W);
            int blk = nk > 1 ? split_blocks++ : -1;
            int slot = nk > 1 ? split_slots : -1;
            if (nk > 1) split_slots += nk;
            for (int k = 0; k < nk; ++k)
              st.push_back(SplitTask{f, i0, k * W, std::min(cmax, (k + 1) * W), slot, nk, k, blk});
          }
        }
      }
      F.split_level_ptr[l + 1] = (int)st.size();
      wide.clear();
      F.fwd_level_ptr[l + 1] = (int)ft.size();
      F.fwdn_level_ptr[l + 1] = (int)fn.size();
      F.bwd_level_ptr[l + 1] = (int)bt.size();
      F.bwdn_level_ptr[l + 1] = (int)bn.size();
    }
    F.fwd_tasks = C.upload(ft.data(), ft.size());
    F.fwdn_tasks = C.upload(fn.data(), fn.size());
    F.split_tasks = C.upload(st.data(), st.size());
    F.split_part = C.alloc<double>((size_t)split_slots * 64 + 1);
    F.split_ticket = C.alloc<unsigned>((size_t)split_blocks + 1);
    JGS2_CUDA(cudaMemset(F.split_ticket, 0, ((size_t)split_blocks + 1) * sizeof(unsigned)));
    // flat per-level assemble map (forward) and gather map (backward):
    // one entry per front position; contributions in child order.
    std::vector<int64_t> adst, acp(1, 0), asrc, gdst;
    std::vector<int> ab, gsrc;
    F.asm_level_ptr.assign(F.nlevels + 1, 0);
    F.gat_level_ptr.assign(F.nlevels + 1, 0);
    for (int l = 0; l < F.nlevels; ++l) {
      for (int k = F.level_ptr[l]; k < F.level_ptr[l + 1]; ++k) {
        int f = lf[k];
        int ns = fns[f], nf = fns[f] + fnr[f];
        std::vector<int> cnt(nf + 1, 0);
        for (int q = cptr[f]; q < cptr[f + 1]; ++q) {
          int c = clist[q];
          for (int64_t t = sptr[c]; t < sptr[c + 1]; ++t) cnt[rmap[t] + 1]++;
        }
        for (int i = 0; i < nf; ++i) cnt[i + 1] += cnt[i];
        std::vector<int64_t> src(cnt[nf]);
        std::vector<int> fill(cnt.begin(), cnt.end() - 1);
        for (int q = cptr[f]; q < cptr[f + 1]; ++q) {
          int c = clist[q];
          for (int64_t t = sptr[c]; t < sptr[c + 1]; ++t)
            src[fill[rmap[t]]++] = uoff[c] + (t - sptr[c]);
        }
        for (int i = 0; i < nf; ++i) {
          adst.push_back(woff[f] + i);
          ab.push_back(i < ns ? colbeg[f] + i : -1);
          for (int c = cnt[i]; c < cnt[i + 1]; ++c) asrc.push_back(src[c]);
          acp.push_back((int64_t)asrc.size());
          if (ns > 0) {
            gdst.push_back(woff[f] + i);
            gsrc.push_back(i < ns ? colbeg[f] + i : -1 - sdof[sptr[f] + (i - ns)]);
          }
        }
      }
      F.asm_level_ptr[l + 1] = (int64_t)adst.size();
      F.gat_level_ptr[l + 1] = (int64_t)gdst.size();
    }
    F.asm_dst = C.upload(adst.data(), adst.size());
    F.asm_b = C.upload(ab.data(), ab.size());
    F.asm_cp = C.upload(acp.data(), acp.size());
    F.asm_src = C.upload(asrc.data(), asrc.size());
    F.gat_dst = C.upload(gdst.data(), gdst.size());
    F.gat_src = C.upload(gsrc.data(), gsrc.size());
    F.bwd_tasks = C.upload(bt.data(), bt.size());
    F.bwdn_tasks = C.upload(bn.data(), bn.size());
  }
  // ---- device metadata
  F.f_colbeg = C.upload(colbeg.data(), NF);
  F.f_ns = C.upload(fns.data(), NF);
  F.f_nr = C.upload(fnr.data(), NF);
  F.f_ld = C.upload(fld.data(), NF);
  F.f_loff = C.upload(loff.data(), NF + 1);
  F.f_uoff = C.upload(uoff.data(), NF + 1);
  F.f_woff = C.upload(woff.data(), NF + 1);
  F.f_cptr = C.upload(cptr.data(), NF + 1);
  F.f_clist = C.upload(clist.data(), clist.size());
  F.f_sptr = C.upload(sptr.data(), NF + 1);
  F.f_sdof = C.upload(sdof.data(), sdof.size());
  F.f_rmap = C.upload(rmap.data(), rmap.size());
  F.level_fronts = C.upload(lf.data(), NF);
  F.u = C.alloc<double>(uoff[NF]);
  F.w = C.alloc<double>(woff[NF]);
  JGS2_CUDA(cudaMemsetAsync(F.w, 0, woff[NF] * sizeof(double), C.stream));
  F.L = C.alloc<double>(F.nnz_alloc);
  JGS2_CUDA(cudaMemsetAsync(F.L, 0, F.nnz_alloc * sizeof(double), C.stream));
  // vertex -> position map for the sweep kernels
  std::vector<int> pos(nv, -1), freel(n);
  for (int i = 0; i < n; ++i) { pos[glob[i]] = S.iperm[i]; freel[i] = glob[i]; }
  C.pos = C.upload(pos.data(), nv);
  F.h_ns = fns; F.h_nr = fnr; F.h_fld = fld; F.h_pos = pos;
  F.h_loff.assign(loff.begin(), loff.end());
  F.h_sptr.assign(sptr.begin(), sptr.end());

  // ---- Hbar blocks (projected rest element Hessians, subspace.py:48-57)
  double* mp_all = nullptr;
  if (!blocks) {
    JGS2_CUDA(cudaMallocAsync(&mp_all, 45 * (size_t)std::max(ne, 1) * sizeof(double), C.stream));
    int* tmp_list = nullptr;
    JGS2_CUDA(cudaMallocAsync(&tmp_list, 2 * (size_t)std::max(ne, 1) * sizeof(int), C.stream));
    launch_element_mplus(ne, nullptr, C.rest, C.tets, C.dminv, C.eprops, mp_all, C.hess_count, tmp_list,
                         C.stream);
    C.launches += 1;
    JGS2_CUDA(cudaFreeAsync(tmp_list, C.stream));
    C.check_launch();
  }
  int64_t nblocks = aptr[n];
  std::vector<int> pfront(n, -1);
  for (int f = 0; f < NF; ++f)
    for (int p = S.col_begin[f]; p < S.col_end[f]; ++p) pfront[p] = f;
  std::vector<int> brow(nblocks), bcol(nblocks), bld(nblocks);
  std::vector<int64_t> bdst(nblocks, -1);
  for (int i = 0; i < n; ++i) {
    int pi = S.iperm[i];
    for (int64_t k = aptr[i]; k < aptr[i + 1]; ++k) {
      int j = adj[k];
      brow[k] = glob[i];
      bcol[k] = glob[j];
      int pj = S.iperm[j];
      if (pi < pj) continue;  // strictly upper in ND order
      int f = pfront[pj];
      int nf = fns[f] + fnr[f];
      int lj = 3 * (pj - S.col_begin[f]);
      int li;
      if (pi < S.col_end[f]) li = 3 * (pi - S.col_begin[f]);
      else {
        const int* ps = S.struct_pos.data() + S.struct_ptr[f];
        int pn = (int)(S.struct_ptr[f + 1] - S.struct_ptr[f]);
        const int* it = std::lower_bound(ps, ps + pn, pi);
        if (it == ps + pn || *it != pi) throw Error(-1, "symbolic: entry outside front structure");
        li = fns[f] + 3 * (int)(it - ps);
      }
      bdst[k] = loff[f] + (int64_t)lj * fld[f] + li;
      bld[k] = fld[f];
    }
  }
  int* d_brow = C.upload(brow.data(), nblocks);
  int* d_bcol = C.upload(bcol.data(), nblocks);
  int* d_bld = C.upload(bld.data(), nblocks);
  int64_t* d_bdst = C.upload(bdst.data(), nblocks);
  double* d_bval = C.alloc<double>(9 * (size_t)nblocks);
  if (blocks) {
    // caller values: sum duplicates per (row, col) in input order
    std::map<std::pair<int, int>, int64_t> where;
    for (int64_t k = 0; k < nblocks; ++k) where[{brow[k], bcol[k]}] = k;
    std::vector<double> hv(9 * (size_t)nblocks, 0.0);
    for (int64_t q = 0; q < blocks->nblocks; ++q) {
      auto it = where.find({(int)blocks->brow[q], (int)blocks->bcol[q]});
      if (it == where.end()) continue;  // touches a fixed vertex
      for (int i = 0; i < 9; ++i) hv[9 * it->second + i] += blocks->bval[9 * q + i];
    }
    JGS2_CUDA(cudaMemcpyAsync(d_bval, hv.data(), hv.size() * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    C.sync();
  } else {
    k_bsr_blocks<<<grid_for(nblocks), kBlock, 0, C.stream>>>((int)nblocks, d_brow, d_bcol,
                                                              C.inc_ptr, C.inc, C.tets, mp_all,
                                                              C.mass, 1.0 / (h_ref * h_ref), d_bval);
    C.check_launch();
  }
  k_scatter_orig<<<grid_for(nblocks), kBlock, 0, C.stream>>>((int)nblocks, d_bdst, d_bld, d_bval, F.L);
  C.check_launch();
  if (mp_all) JGS2_CUDA(cudaFreeAsync(mp_all, C.stream));

  // ---- multifrontal numeric factorization in postorder
  if (!C.cublas) {
    if (cublasCreate(&C.cublas) != CUBLAS_STATUS_SUCCESS) throw Error(-2, "cublasCreate failed");
    if (cusolverDnCreate(&C.cusolver) != CUSOLVER_STATUS_SUCCESS) throw Error(-2, "cusolverDnCreate failed");
  }
  cublasSetStream(C.cublas, C.stream);
  cusolverDnSetStream(C.cusolver, C.stream);
  int max_ns = 0;
  for (int f = 0; f < NF; ++f) max_ns = std::max(max_ns, fns[f]);
  int lwork = 0;
  if (max_ns > 0 &&
      cusolverDnDpotrf_bufferSize(C.cusolver, CUBLAS_FILL_MODE_LOWER, max_ns, F.L, max_ns + 1,
                                  &lwork) != CUSOLVER_STATUS_SUCCESS)
    throw Error(-2, "potrf buffer size");
  double* work = C.alloc<double>(std::max(lwork, 1));
  int* infos = C.alloc<int>(2 * NF);
  int* infos2 = infos + NF;
  JGS2_CUDA(cudaMemsetAsync(infos, 0, 2 * NF * sizeof(int), C.stream));
  size_t tri_dbytes = 0, tri_hbytes = 0;
  if (max_ns > 0 &&
      cusolverDnXtrtri_bufferSize(C.cusolver, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, max_ns,
                                  CUDA_R_64F, F.L, max_ns + 1, &tri_dbytes, &tri_hbytes) !=
          CUSOLVER_STATUS_SUCCESS)
    throw Error(-2, "trtri buffer size");
  void* tri_d = C.alloc<char>(std::max<size_t>(tri_dbytes, 16));
  std::vector<char> tri_h(std::max<size_t>(tri_hbytes, 16));
  std::vector<double*> Ubuf(NF, nullptr);
  const double one = 1.0, mone = -1.0;
  for (int f = 0; f < NF; ++f) {
    int ns = fns[f], nr = fnr[f], nf = fld[f];  // nf: leading dimension below
    double* Pf = F.L + loff[f];
    if (nr > 0) {
      JGS2_CUDA(cudaMallocAsync(&Ubuf[f], (size_t)nr * nr * sizeof(double), C.stream));
      JGS2_CUDA(cudaMemsetAsync(Ubuf[f], 0, (size_t)nr * nr * sizeof(double), C.stream));
    }
    for (int k = cptr[f]; k < cptr[f + 1]; ++k) {
      int c = clist[k];
      int nrc = fnr[c];
      if (nrc > 0) {
        int64_t tot = (int64_t)nrc * nrc;
        k_extend_add<<<grid_for(tot), kBlock, 0, C.stream>>>(nrc, Ubuf[c], F.f_rmap + sptr[c], ns,
                                                             nf, Pf, nr, Ubuf[f]);
        C.check_launch();
        JGS2_CUDA(cudaFreeAsync(Ubuf[c], C.stream));
        Ubuf[c] = nullptr;
      }
    }
    if (ns > 0) {
      if (cusolverDnDpotrf(C.cusolver, CUBLAS_FILL_MODE_LOWER, ns, Pf, nf, work, lwork, infos + f) !=
          CUSOLVER_STATUS_SUCCESS)
        throw Error(-2, "cusolverDnDpotrf failed");
      if (nr > 0) {
        if (cublasDtrsm(C.cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T,
                        CUBLAS_DIAG_NON_UNIT, nr, ns, &one, Pf, nf, Pf + ns, nf) != CUBLAS_STATUS_SUCCESS)
          throw Error(-2, "cublasDtrsm failed");
        if (cublasDsyrk(C.cublas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, nr, ns, &mone, Pf + ns, nf,
                        &one, Ubuf[f], nr) != CUBLAS_STATUS_SUCCESS)
          throw Error(-2, "cublasDsyrk failed");
      }
      // partitioned inverse: L11 -> L11^-1 (strict upper zeroed), L21 -> L21 L11^-1
      if (cusolverDnXtrtri(C.cusolver, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, ns, CUDA_R_64F,
                           Pf, nf, tri_d, tri_dbytes, tri_h.data(), tri_hbytes, infos2 + f) !=
          CUSOLVER_STATUS_SUCCESS)
        throw Error(-2, "cusolverDnXtrtri failed");
      k_zero_upper<<<grid_for((int64_t)ns * ns), kBlock, 0, C.stream>>>(ns, nf, Pf);
      C.check_launch();
      if (nr > 0 &&
          cublasDtrmm(C.cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N,
                      CUBLAS_DIAG_NON_UNIT, nr, ns, &one, Pf, nf, Pf + ns, nf, Pf + ns, nf) !=
              CUBLAS_STATUS_SUCCESS)
        throw Error(-2, "cublasDtrmm failed");
    }
  }
  for (int f = 0; f < NF; ++f)
    if (Ubuf[f]) JGS2_CUDA(cudaFreeAsync(Ubuf[f], C.stream));
  std::vector<int> hinfo(2 * NF);
  JGS2_CUDA(cudaMemcpyAsync(hinfo.data(), infos, 2 * NF * sizeof(int), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  for (int f = 0; f < 2 * NF; ++f)
    if (hinfo[f] != 0)
      throw Error(-3, std::string("rest Hessian factorization failed: front ") + std::to_string(f % NF) +
                          (f < NF ? " not positive definite" : " singular diagonal block") +
                          " (info " + std::to_string(hinfo[f]) + ")");
  F.ready = true;
  F.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// q <- Hbar_ff^{-1} b (ND-ordered DOFs): forward level sweeps (assemble +
// apply) leave z in b; backward level sweeps (gather + apply) write x into q.
void factor_solve_launches(Ctx& C) {
  Factor& F = C.fac;
  // A level's narrow-front launch runs on the side stream beside its wide
  // launch (disjoint fronts); both join before the next level (captured as
  // parallel graph branches). The narrow grid fills the wide kernel's tail.
  const bool fork = solve_fork() && C.solve_side;
  auto side_begin = [&](bool wide_too) -> cudaStream_t {
    if (!fork || !wide_too) return C.stream;
    JGS2_CUDA(cudaEventRecord(C.ev_sfork, C.stream));
    JGS2_CUDA(cudaStreamWaitEvent(C.solve_side, C.ev_sfork, 0));
    return C.solve_side;
  };
  auto side_end = [&](cudaStream_t s) {
    if (s == C.stream) return;
    JGS2_CUDA(cudaEventRecord(C.ev_sjoin, s));
    JGS2_CUDA(cudaStreamWaitEvent(C.stream, C.ev_sjoin, 0));
  };
  for (int l = 0; l < F.nlevels; ++l) {
    int64_t na = F.asm_level_ptr[l + 1] - F.asm_level_ptr[l];
    int64_t o = F.asm_level_ptr[l];
    int nt = F.fwd_level_ptr[l + 1] - F.fwd_level_ptr[l];
    int nn = F.fwdn_level_ptr[l + 1] - F.fwdn_level_ptr[l];
    int nsp = F.split_level_ptr[l + 1] - F.split_level_ptr[l];
    if (na == 0 && nt == 0 && nn == 0 && nsp == 0) continue;  // level of zero-size joining fronts
    if (na > 0)
    k_fwd_assemble_flat<<<grid_for(na), kBlock, 0, C.stream>>>(na, F.asm_dst + o, F.asm_b + o,
                                                               F.asm_cp + o, F.asm_src, C.b, F.u, F.w);
    C.check_launch();
    cudaStream_t sn = C.stream;
    if (nn > 0) {
      sn = side_begin(nt > 0 || nsp > 0);
      int gn = std::min((nn + 7) / 8, 148 * 8);
      k_fwd_apply_narrow<<<gn, kSolveThreads, 0, sn>>>(F.fwdn_tasks + F.fwdn_level_ptr[l], nn,
                                                       F.f_colbeg, F.f_ns, F.f_nr, F.f_ld, F.f_loff,
                                                       F.f_uoff, F.f_woff, F.L, F.w, C.b, F.u);
      C.check_launch();
    }
    int ns_ = F.split_level_ptr[l + 1] - F.split_level_ptr[l];
    if (ns_ > 0) {
      int g = std::min(ns_, 148 * solve_ctas());
      k_fwd_apply_split<<<g, kSolveThreads, 0, C.stream>>>(F.split_tasks + F.split_level_ptr[l], ns_,
                                                           F.f_colbeg, F.f_ns, F.f_nr, F.f_ld, F.f_loff,
                                                           F.f_uoff, F.f_woff, F.L, F.w, C.b, F.u,
                                                           F.split_part, F.split_ticket);
      C.check_launch();
    }
    if (nt > 0) {
      int g = std::min(nt, 148 * solve_ctas());
      k_fwd_apply<<<g, kSolveThreads, 0, C.stream>>>(F.fwd_tasks + F.fwd_level_ptr[l], nt, F.f_colbeg,
                                                     F.f_ns, F.f_nr, F.f_ld, F.f_loff, F.f_uoff,
                                                     F.f_woff, F.L, F.w, C.b, F.u);
      C.check_launch();
    }
    side_end(sn);
  }
  for (int l = F.nlevels - 1; l >= 0; --l) {
    int nt = F.bwd_level_ptr[l + 1] - F.bwd_level_ptr[l];
    int nn = F.bwdn_level_ptr[l + 1] - F.bwdn_level_ptr[l];
    if (nt == 0 && nn == 0) continue;
    int64_t ng = F.gat_level_ptr[l + 1] - F.gat_level_ptr[l];
    int64_t o = F.gat_level_ptr[l];
    if (ng > 0)
    k_bwd_gather_flat<<<grid_for(ng), kBlock, 0, C.stream>>>(ng, F.gat_dst + o, F.gat_src + o, C.b,
                                                             C.q, F.w);
    C.check_launch();
    cudaStream_t sn = C.stream;
    if (nn > 0) {
      sn = side_begin(nt > 0);
      int gn = std::min((nn + 7) / 8, 148 * 8);
      k_bwd_apply_narrow<<<gn, kSolveThreads, 0, sn>>>(F.bwdn_tasks + F.bwdn_level_ptr[l], nn, F.f_colbeg,
                                                       F.f_ns, F.f_nr, F.f_ld, F.f_loff, F.f_woff, F.L,
                                                       F.w, C.q);
      C.check_launch();
    }
    if (nt > 0) {
      int gb = std::min(nt, 148 * solve_ctas());
      k_bwd_apply<<<gb, kSolveThreads, 0, C.stream>>>(F.bwd_tasks + F.bwd_level_ptr[l], nt, F.f_colbeg,
                                                      F.f_ns, F.f_nr, F.f_ld, F.f_loff, F.f_woff, F.L,
                                                      F.w, C.q);
      C.check_launch();
    }
    side_end(sn);
  }
}

// The solve is replayed from a CUDA graph captured once (all pointers are
// fixed for the life of the factor): ~4 launches per tree level.
void factor_solve(Ctx& C) {
  Factor& F = C.fac;
  if (!F.graph_exec) {
    int64_t l0 = C.launches;
    JGS2_CUDA(cudaStreamBeginCapture(C.stream, cudaStreamCaptureModeThreadLocal));
    cudaGraph_t g = nullptr;
    try {
      factor_solve_launches(C);
    } catch (...) {
      cudaStreamEndCapture(C.stream, &g);  // leave capture mode before reporting
      if (g) cudaGraphDestroy(g);
      cudaGetLastError();
      throw;
    }
    JGS2_CUDA(cudaStreamEndCapture(C.stream, &g));
    JGS2_CUDA(cudaGraphInstantiate(&F.graph_exec, g, 0));
    JGS2_CUDA(cudaGraphDestroy(g));
    F.graph_launches = C.launches - l0;
    C.launches = l0;
  }
  JGS2_CUDA(cudaGraphLaunch(F.graph_exec, C.stream));
  C.launches += F.graph_launches;
}

}  // namespace jgs2
