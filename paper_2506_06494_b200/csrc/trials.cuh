// Batched trial energies of the sweep-level backtracking guard
// (local_solver.py:555-577; total_energy assembly.py:183-192 with
// find_pairs(x_try) per trial).
//
// The reference evaluates E(x + gamma_j dx) for gamma_j = cap 2^-j one trial
// at a time, re-detecting the active pairs at every trial. Here up to
// kTrialBatch trials are evaluated in one pass over the mesh: elastic +
// inertia terms per element/vertex chunk for every gamma (k_energy_chunks,
// partition.cuh), and the barrier over
//   * all (surface vertex, plane) pairs, and
//   * a candidate list of cross-body (vertex, triangle) pairs built once per
//     sweep (hier_grid.cuh): a pair at distance < dhat at any trial
//     position has dist(x) < dhat + gamma_max (s_v + s_t), so the candidates
//     contain every trial's exact pair set; each trial keeps the candidates
//     whose distance (reference rounding) is < dhat.
// A trial with any active distance <= 0 is infeasible (E = inf).
#pragma once
#include "contact.cuh"
#include "sweep.cuh"

namespace jgs2 {

constexpr int kTrialBatch = 8;
struct Gammas {
  double g[kTrialBatch];
  int n;
};

// per-block partials for each trial: partials[k * kMaxPartials + block]
template <int OP>
__device__ void block_reduce_multi(double* acc, int n, double* partials) {
  for (int k = 0; k < kTrialBatch; ++k) {
    if (k >= n) break;
    double s = block_reduce<OP>(acc[k]);
    if (threadIdx.x == 0) partials[k * kMaxPartials + blockIdx.x] = s;
    __syncthreads();
  }
}

// Elastic + inertia trial energies: k_energy_chunks (partition.cuh).

// barrier energies: planes over all surface vertices + candidate tri pairs
__global__ void __launch_bounds__(kBlock)
k_barrier_batch(ContactDev cd, int ncand, const int* cand_v, const int* cand_t, const double* x0,
                const double* dx, Gammas G, double* partials, int* flags) {
  double acc[kTrialBatch];
  int bad[kTrialBatch];
#pragma unroll
  for (int k = 0; k < kTrialBatch; ++k) { acc[k] = 0.0; bad[k] = 0; }
  int np = cd.nsv * cd.nplanes;
  int n = np + ncand;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i < np) {
      int pl = i / cd.nsv, v = cd.sv[i % cd.nsv];
      const double* P = cd.planes + 6 * pl;
#pragma unroll
      for (int k = 0; k < kTrialBatch; ++k) {
        if (k >= G.n) break;
        double p[3];
        load_pos(x0, dx, G.g[k], v, p);
        double d = plane_dist(p, P);
        if (d < cd.dhat) {
          if (d <= 0.0) bad[k] = 1;
          acc[k] += barrier_fn(d, cd.dhat, cd.kappa).b;
        }
      }
    } else {
      int j = i - np;
      int v = cand_v[j], t = cand_t[j];
      int a0 = cd.st[3 * t], a1 = cd.st[3 * t + 1], a2 = cd.st[3 * t + 2];
#pragma unroll
      for (int k = 0; k < kTrialBatch; ++k) {
        if (k >= G.n) break;
        double p[3], a[3], b[3], c[3], bary[3];
        load_pos(x0, dx, G.g[k], v, p);
        load_pos(x0, dx, G.g[k], a0, a);
        load_pos(x0, dx, G.g[k], a1, b);
        load_pos(x0, dx, G.g[k], a2, c);
        double d = closest_point_tri(p, a, b, c, bary);
        if (d < cd.dhat) {
          if (d <= 0.0) bad[k] = 1;
          acc[k] += barrier_fn(d, cd.dhat, cd.kappa).b;
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kTrialBatch; ++k)
    if (k < G.n && bad[k]) atomicOr(flags + k, 1);
  block_reduce_multi<OP_SUM>(acc, G.n, partials);
}

// final deterministic reduction of per-block partials for n trials (1 block)
__global__ void k_reduce_batch(const double* partials, int nblocks, int n, double* out) {
  for (int k = 0; k < n; ++k) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += blockDim.x) acc += partials[k * kMaxPartials + i];
    acc = block_reduce<OP_SUM>(acc);
    if (threadIdx.x == 0) out[k] = acc;
    __syncthreads();
  }
}

}  // namespace jgs2
