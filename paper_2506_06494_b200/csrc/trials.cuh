// Batched trial energies of the sweep-level backtracking guard
// (local_solver.py:555-577; total_energy assembly.py:183-192 with
// find_pairs(x_try) per trial).
//
// The reference evaluates E(x + gamma_j dx) for gamma_j = cap 2^-j one trial
// at a time, re-detecting the active pairs at every trial. Here up to
// kTrialBatch trials are evaluated in one pass over the mesh: elastic +
// inertia terms per element/vertex for every gamma, and the barrier over
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

// 2 blocks per SM (<= 128 registers): at 155 registers one 256-thread block
// per SM left the FP64 pipes latency-bound (ncu: 12.5% occupancy)
__global__ void __launch_bounds__(kBlock, 2)
k_energy_batch(DevModel m, const double* __restrict__ x0, const double* __restrict__ dx, Gammas G,
               const double* __restrict__ z, double h, double* partials) {
  double acc[kTrialBatch];
#pragma unroll
  for (int k = 0; k < kTrialBatch; ++k) acc[k] = 0.0;
  int n = max(m.ne, m.nv);
  double inv2h2 = 0.5 / (h * h);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i < m.ne) {
      int4 t = __ldg(m.tets + i);
      int cs[4] = {t.x, t.y, t.z, t.w};
      double xb[4][3], db[4][3];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          xb[a][c] = __ldg(x0 + 3 * cs[a] + c);
          db[a][c] = __ldg(dx + 3 * cs[a] + c);
        }
      double D[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) D[q] = __ldg(m.dminv + 9 * (size_t)i + q);
      double4 ep = m.eprops[i];
      SnhConst kc = snh_const(ep.y, ep.z);
      // Each trial forms the rounded positions x_try = fl(x + fl(gamma dx))
      // and F = Ds(x_try) Dm^-1, exactly as the reference evaluates
      // total_energy(x_before + gamma * dx) (local_solver.py:564-567). Near
      // the halving floor E(x_try) - E(x) is at the 1e-12 acceptance slack
      // and dominated by that rounding of x_try, so an F affine in gamma
      // (exact arithmetic) would flip accept/reject decisions there.
#pragma unroll 1
      for (int k = 0; k < kTrialBatch; ++k) {
        if (k >= G.n) break;
        const double g = G.g[k];
        double xt[4][3];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 3; ++c) xt[a][c] = __dadd_rn(xb[a][c], __dmul_rn(g, db[a][c]));
        double F[9];
        deformation_gradient(xt[0], xt[1], xt[2], xt[3], D, F);
        acc[k] += ep.x * snh_psi(F, kc);
      }
    }
    if (i < m.nv) {
      double xb[3], db[3], zz[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        xb[c] = __ldg(x0 + 3 * i + c);
        db[c] = __ldg(dx + 3 * i + c);
        zz[c] = z[3 * i + c];
      }
      double mi = m.mass[i];
#pragma unroll
      for (int k = 0; k < kTrialBatch; ++k) {
        if (k >= G.n) break;
        double dd = 0.0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double df = __dadd_rn(xb[c], __dmul_rn(G.g[k], db[c])) - zz[c];
          dd += df * df;
        }
        acc[k] += mi * dd * inv2h2;
      }
    }
  }
  block_reduce_multi<OP_SUM>(acc, G.n, partials);
}

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
