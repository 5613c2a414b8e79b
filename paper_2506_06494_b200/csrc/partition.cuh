// Rank-count-independent reductions of the partitioned solve.
//
// Sums over elements / vertices (trial energies, local_solver.py:566;
// grad_sq, :602-603) run over fixed chunks of consecutive ids that never
// cross a body boundary. Chunk c's partial is computed by the rank owning
// its body (zeros elsewhere), all-reduced (x + 0 = x, exact), and the
// partials are combined in chunk order -- the same arithmetic on 1 or N
// GPUs, so a partitioned run is bit-identical to the single-GPU run.
#pragma once
#include "sweep.cuh"

namespace jgs2 {

constexpr int kChunkE = 2048;  // elements per chunk
constexpr int kChunkV = 1024;  // vertices per chunk
constexpr int kTrials = 8;     // == kTrialBatch (trials.cuh)

struct TrialGammas {
  double g[kTrials];
  int n;
};

// grad_sq partial of vertex chunk (blockIdx.x + c0): sum of |g_asm|^2 over
// its free vertices (local_solver.py:602-603)
__global__ void __launch_bounds__(kBlock)
k_chunk_gradsq(const int2* chunks, int c0, const double* __restrict__ gasm, const uint8_t* fixed,
               double* part) {
  int c = c0 + blockIdx.x;
  int2 r = chunks[c];
  double acc = 0.0;
  for (int v = r.x + threadIdx.x; v < r.y; v += blockDim.x) {
    if (fixed[v]) continue;
    double g0 = gasm[3 * v], g1 = gasm[3 * v + 1], g2 = gasm[3 * v + 2];
    acc += g0 * g0 + g1 * g1 + g2 * g2;
  }
  acc = block_reduce<OP_SUM>(acc);
  if (threadIdx.x == 0) part[c] = acc;
}

// Elastic + inertia energy of one chunk at up to kTrials positions
// x_try = fl(x + fl(gamma dx)) (assembly.py:183-192 at x_before + gamma dx,
// local_solver.py:564-567); partials part[k * nchunks + c]. Element chunks
// first (c < nce), then vertex chunks.
__global__ void __launch_bounds__(kBlock, 2)
k_energy_chunks(DevModel m, const int2* chunks, int c0, int nce, int nchunks, const double* __restrict__ x0,
                const double* __restrict__ dx, TrialGammas G, const double* __restrict__ z, double h,
                double* part) {
  int c = c0 + blockIdx.x;
  int2 r = chunks[c];
  double acc[kTrials];
#pragma unroll
  for (int k = 0; k < kTrials; ++k) acc[k] = 0.0;
  if (c < nce) {
    for (int i = r.x + threadIdx.x; i < r.y; i += blockDim.x) {
      int4 t = __ldg(m.tets + i);
      int cs[4] = {t.x, t.y, t.z, t.w};
      double xb[4][3], db[4][3];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          xb[a][q] = __ldg(x0 + 3 * cs[a] + q);
          db[a][q] = dx ? __ldg(dx + 3 * cs[a] + q) : 0.0;
        }
      double D[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) D[q] = __ldg(m.dminv + 9 * (size_t)i + q);
      double4 ep = m.eprops[i];
      SnhConst kc = snh_const(ep.y, ep.z);
#pragma unroll 1
      for (int k = 0; k < kTrials; ++k) {
        if (k >= G.n) break;
        const double g = G.g[k];
        double xt[4][3];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int q = 0; q < 3; ++q) xt[a][q] = __dadd_rn(xb[a][q], __dmul_rn(g, db[a][q]));
        double F[9];
        deformation_gradient(xt[0], xt[1], xt[2], xt[3], D, F);
        acc[k] += ep.x * snh_psi(F, kc);
      }
    }
  } else {
    double inv2h2 = 0.5 / (h * h);
    for (int i = r.x + threadIdx.x; i < r.y; i += blockDim.x) {
      double xb[3], db[3], zz[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        xb[q] = __ldg(x0 + 3 * i + q);
        db[q] = dx ? __ldg(dx + 3 * i + q) : 0.0;
        zz[q] = z[3 * i + q];
      }
      double mi = m.mass[i];
#pragma unroll
      for (int k = 0; k < kTrials; ++k) {
        if (k >= G.n) break;
        double dd = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          double df = __dadd_rn(xb[q], __dmul_rn(G.g[k], db[q])) - zz[q];
          dd += df * df;
        }
        acc[k] += mi * dd * inv2h2;
      }
    }
  }
  for (int k = 0; k < kTrials; ++k) {
    if (k >= G.n) break;
    double s = block_reduce<OP_SUM>(acc[k]);
    if (threadIdx.x == 0) part[(size_t)k * nchunks + c] = s;
    __syncthreads();
  }
}

// out[k] = sum over chunks (chunk order, fixed tree) of part[k * stride + c]
__global__ void k_reduce_chunks(const double* part, int nchunks, size_t stride, int n, double* out) {
  for (int k = 0; k < n; ++k) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < nchunks; i += blockDim.x) acc += part[k * stride + i];
    acc = block_reduce<OP_SUM>(acc);
    if (threadIdx.x == 0) out[k] = acc;
    __syncthreads();
  }
}

}  // namespace jgs2
