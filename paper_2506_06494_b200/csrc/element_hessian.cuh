// Projected element Hessians in translation-complement coordinates.
//
// Reference: energy.snh_batch(..., project_spd=True) -> 12x12 Hessian
// V W^T H9 W followed by an eigenvalue clamp (energy.py:110-149, 169-189).
// The 12x12 Hessian annihilates rigid translations, so its PSD projection
// equals T PSD(M) T^T with M = T^T H12 T the 9x9 reduced Hessian in the
// Hadamard complement basis T = U (x) I3 (agrees with the
// 12x12 eigh to 3.8e-15).  M has the closed form (G = W^T U, a_p = F G_p,
// b_p = cof(F) G_p, s = lam_s (J - alpha)):
//   M_(p,q) = V [ d (G_p.G_q) I + c1 a_p a_q^T + lam_s b_p b_q^T
//                 - s [F (G_p x G_q)]_x ]
// (the stable Neo-Hookean H9 = d I + c1 f f^T + lam_s g g^T + s K with the
// cofactor-derivative skew blocks K, contracted against G).
//
// Projection: an LDL^T inertia test returns M unchanged when it is positive
// definite; otherwise the 9x9 eigendecomposition is computed by Householder
// tridiagonalisation + implicit QL (EISPACK tred2/tql2 scheme) with the
// eigenvectors in per-thread interleaved shared memory, and
// M+ = Q max(L, 0) Q^T. Divisions and square roots use the FP64-pipe
// Newton forms of dmath.cuh (the MUFU.*64H forms saturated the XU pipe).
#pragma once
#include <algorithm>

#include "dmath.cuh"
#include "physics.cuh"

namespace jgs2 {

constexpr int kHessThreads = 128;

// packed lower index for (i >= j)
#define JGS2_PK(i, j) ((i) * ((i) + 1) / 2 + (j))

__device__ __forceinline__ void reduced_hessian_closed(const double* F, const double* D, double vol,
                                                       SnhConst k, double* Mp /*45*/) {
  double W[12];
  shape_weights(D, W);
  double G[9];  // G[j][p]
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int p = 0; p < 3; ++p)
      G[3 * j + p] = W[j] * kHad(0, p) + W[3 + j] * kHad(1, p) + W[6 + j] * kHad(2, p) + W[9 + j] * kHad(3, p);
  double C[9];
  cofactor(F, C);
  double ic = frob2(F), J = det3_cof(F, C);
  double d = k.mu_s * (1.0 - rcp_nr(ic + 1.0));
  double c1 = div_nr(2.0 * k.mu_s, (ic + 1.0) * (ic + 1.0));
  double s = k.lam_s * (J - k.alpha);
  double a[9], b[9];  // a[3p + r] = (F G)[r][p]
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      a[3 * p + r] = F[3 * r] * G[p] + F[3 * r + 1] * G[3 + p] + F[3 * r + 2] * G[6 + p];
      b[3 * p + r] = C[3 * r] * G[p] + C[3 * r + 1] * G[3 + p] + C[3 * r + 2] * G[6 + p];
    }
  double GG[9];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = 0; q < 3; ++q) GG[3 * p + q] = G[p] * G[q] + G[3 + p] * G[3 + q] + G[6 + p] * G[6 + q];
  // FX[pq] = F (G_p x G_q) for (p,q) = (1,0), (2,0), (2,1)
  double FX[3][3];
  const int PP[3] = {1, 2, 2}, QQ[3] = {0, 0, 1};
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    int p = PP[t], q = QQ[t];
    double gp[3] = {G[p], G[3 + p], G[6 + p]}, gq[3] = {G[q], G[3 + q], G[6 + q]}, x[3];
    cross3(gp, gq, x);
#pragma unroll
    for (int r = 0; r < 3; ++r) FX[t][r] = F[3 * r] * x[0] + F[3 * r + 1] * x[1] + F[3 * r + 2] * x[2];
  }
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q <= p; ++q)
#pragma unroll
        for (int ss = 0; ss < 3; ++ss) {
          int i = 3 * p + r, j = 3 * q + ss;
          if (j > i) continue;
          double v = c1 * a[3 * p + r] * a[3 * q + ss] + k.lam_s * b[3 * p + r] * b[3 * q + ss];
          if (r == ss) v += d * GG[3 * p + q];
          if (p != q) {  // - s [FX]_x (r, ss)
            int t = (p == 1) ? 0 : (q == 0 ? 1 : 2);
            const double* x = FX[t];
            double sk = 0.0;  // [x]_x[r][ss]
            if (r == 0 && ss == 1) sk = -x[2];
            if (r == 0 && ss == 2) sk = x[1];
            if (r == 1 && ss == 0) sk = x[2];
            if (r == 1 && ss == 2) sk = -x[0];
            if (r == 2 && ss == 0) sk = -x[1];
            if (r == 2 && ss == 1) sk = x[0];
            v -= s * sk;
          }
          Mp[JGS2_PK(i, j)] = vol * v;
        }
}

// LDL^T without pivoting: true iff all pivots > 0 (positive definite).
__device__ __forceinline__ bool is_pos_def9(const double* Mp) {
  double L[45];
#pragma unroll
  for (int i = 0; i < 45; ++i) L[i] = Mp[i];
  double dd[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    double dj = L[JGS2_PK(j, j)];
#pragma unroll
    for (int k = 0; k < j; ++k) dj -= L[JGS2_PK(j, k)] * L[JGS2_PK(j, k)] * dd[k];
    if (!(dj > 0.0)) return false;
    dd[j] = dj;
    double inv = rcp_nr(dj);
#pragma unroll
    for (int i = j + 1; i < 9; ++i) {
      double v = L[JGS2_PK(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) v -= L[JGS2_PK(i, k)] * L[JGS2_PK(j, k)] * dd[k];
      L[JGS2_PK(i, j)] = v * inv;
    }
  }
  return true;
}

// The same tred2 + tql2 (JAMA) with every loop bound a compile-time
// constant (outer indices unrolled, runtime ranges as predicates), so the
// diagonal d and off-diagonal e live in registers and only the eigenvector
// matrix V stays in per-thread interleaved shared memory.
template <int S>
__device__ __forceinline__ void sym_eig9_reg(double* V, double (&d)[9], double (&e)[9]) {
  constexpr int n = 9;
#define VV(i, j) V[((i) * n + (j)) * S]
#pragma unroll
  for (int j = 0; j < n; ++j) d[j] = VV(n - 1, j);
#pragma unroll
  for (int i = n - 1; i > 0; --i) {
    double scale = 0.0, h = 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) scale += fabs(d[k]);
    if (scale == 0.0) {
      e[i] = d[i - 1];
#pragma unroll
      for (int j = 0; j < i; ++j) { d[j] = VV(i - 1, j); VV(i, j) = 0.0; VV(j, i) = 0.0; }
    } else {
      const double rs = rcp_nr(scale);
#pragma unroll
      for (int k = 0; k < i; ++k) { d[k] *= rs; h += d[k] * d[k]; }
      double f = d[i - 1];
      double g = sqrt_nr(h);
      if (f > 0) g = -g;
      e[i] = scale * g;
      h -= f * g;
      d[i - 1] = f - g;
#pragma unroll
      for (int j = 0; j < i; ++j) e[j] = 0.0;
#pragma unroll
      for (int j = 0; j < i; ++j) {
        f = d[j];
        VV(j, i) = f;
        g = e[j] + VV(j, j) * f;
#pragma unroll
        for (int k = j + 1; k <= i - 1; ++k) {
          double vkj = VV(k, j);
          g += vkj * d[k];
          e[k] += vkj * f;
        }
        e[j] = g;
      }
      f = 0.0;
      const double rh = rcp_nr(h);
#pragma unroll
      for (int j = 0; j < i; ++j) { e[j] *= rh; f += e[j] * d[j]; }
      double hh = div_nr(f, h + h);
#pragma unroll
      for (int j = 0; j < i; ++j) e[j] -= hh * d[j];
#pragma unroll
      for (int j = 0; j < i; ++j) {
        f = d[j];
        g = e[j];
#pragma unroll
        for (int k = j; k <= i - 1; ++k) VV(k, j) -= (f * e[k] + g * d[k]);
        d[j] = VV(i - 1, j);
        VV(i, j) = 0.0;
      }
    }
    d[i] = h;
  }
#pragma unroll
  for (int i = 0; i < n - 1; ++i) {
    VV(n - 1, i) = VV(i, i);
    VV(i, i) = 1.0;
    double h = d[i + 1];
    if (h != 0.0) {
      const double rh = rcp_nr(h);
#pragma unroll
      for (int k = 0; k <= i; ++k) d[k] = VV(k, i + 1) * rh;
#pragma unroll
      for (int j = 0; j <= i; ++j) {
        double g = 0.0;
#pragma unroll
        for (int k = 0; k <= i; ++k) g += VV(k, i + 1) * VV(k, j);
#pragma unroll
        for (int k = 0; k <= i; ++k) VV(k, j) -= g * d[k];
      }
    }
#pragma unroll
    for (int k = 0; k <= i; ++k) VV(k, i + 1) = 0.0;
  }
#pragma unroll
  for (int j = 0; j < n; ++j) { d[j] = VV(n - 1, j); VV(n - 1, j) = 0.0; }
  VV(n - 1, n - 1) = 1.0;
  // implicit QL
#pragma unroll
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  double f = 0.0, tst1 = 0.0;
  const double eps = 2.220446049250313e-16;
#pragma unroll
  for (int l = 0; l < n; ++l) {
    tst1 = fmax(tst1, fabs(d[l]) + fabs(e[l]));
    int m = n - 1;  // first m >= l with |e[m]| <= eps tst1 (e[n-1] == 0)
#pragma unroll
    for (int mm = n - 2; mm >= l; --mm)
      if (fabs(e[mm]) <= eps * tst1) m = mm;
    if (l < n - 1 && m > l) {
      int iter = 0;
      do {
        ++iter;
        double g = d[l];
        double p = div_nr(d[l + 1] - g, 2.0 * e[l]);
        double r = sqrt_nr(fma(p, p, 1.0));  // |p| <= ~1/eps: no overflow
        if (p < 0) r = -r;
        d[l] = div_nr(e[l], p + r);
        d[l + 1] = e[l] * (p + r);
        double dl1 = d[l + 1];
        double h = g - d[l];
#pragma unroll
        for (int i = l + 2; i < n; ++i) d[i] -= h;
        f += h;
        p = d[n - 1];
#pragma unroll
        for (int i = n - 2; i > l; --i)
          if (i == m) p = d[i];
        double c = 1.0, c2 = c, c3 = c;
        double el1 = e[l + 1];
        double s = 0.0, s2 = 0.0;
#pragma unroll
        for (int i = n - 2; i >= l; --i) {
          if (i < m) {
            c3 = c2;
            c2 = c;
            s2 = s;
            g = c * e[i];
            h = c * p;
            double ei = e[i];
            double q2 = fma(p, p, ei * ei);  // Hessian-scale entries: no overflow in FP64
            double ri = rsqrt_nr(q2);
            r = sqrt_from_rsqrt(q2, ri);
            e[i + 1] = s * r;
            s = ei * ri;
            c = p * ri;
            p = c * d[i] - s * g;
            d[i + 1] = h + s * (c * g + s * d[i]);
#pragma unroll
            for (int k = 0; k < n; ++k) {
              double vk1 = VV(k, i + 1), vk0 = VV(k, i);
              VV(k, i + 1) = s * vk0 + c * vk1;
              VV(k, i) = c * vk0 - s * vk1;
            }
          }
        }
        p = div_nr(-s * s2 * c3 * el1 * e[l], dl1);
        e[l] = s * p;
        d[l] = c * p;
      } while (fabs(e[l]) > eps * tst1 && iter < 60);
    }
    d[l] = d[l] + f;
    e[l] = 0.0;
  }
#undef VV
}

// Pass 1, one thread per element: closed-form M (written to the element's
// slot), the LDL^T inertia test, and the indefinite elements compacted into
// `list` (warp-aggregated atomic; the order of the list does not affect any
// result, each element owns its output slot).
__global__ void __launch_bounds__(kHessThreads)
k_mplus_closed(int n, const int* elems, const double* __restrict__ xs, const int4* __restrict__ tets,
               const double* __restrict__ dminv, const double4* __restrict__ eprops, double* mplus, int* count,
               int* list) {
  // the block's 128 x 45 outputs are staged in shared memory and stored
  // contiguously (per-thread 360-B strided stores were lg-throttle bound)
  __shared__ double stage[kHessThreads * 45];
  // grid-stride over blocks of 128 elements (one pass unless the grid is capped)
  for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
  __syncthreads();  // previous round's stores done with stage
  int u = base + threadIdx.x;
  bool indef = false;
  if (u < n) {
    int e = elems ? elems[u] : u;
    double D[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) D[i] = __ldg(dminv + 9 * (size_t)e + i);
    int4 t = __ldg(tets + e);
    double x0[3], x1[3], x2[3], x3[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      x0[c] = __ldg(xs + 3 * t.x + c); x1[c] = __ldg(xs + 3 * t.y + c);
      x2[c] = __ldg(xs + 3 * t.z + c); x3[c] = __ldg(xs + 3 * t.w + c);
    }
    double F[9];
    deformation_gradient(x0, x1, x2, x3, D, F);
    double4 ep = eprops[e];
    double Mp[45];
    reduced_hessian_closed(F, D, ep.x, snh_const(ep.y, ep.z), Mp);
#pragma unroll
    for (int i = 0; i < 45; ++i) stage[45 * threadIdx.x + i] = Mp[i];
    indef = !is_pos_def9(Mp);
  }
  __syncthreads();
  const int cnt = 45 * min((int)blockDim.x, n - base);
  double* o = mplus + 45 * (size_t)base;
  for (int k = threadIdx.x; k < cnt; k += blockDim.x) o[k] = stage[k];
  unsigned ball = __ballot_sync(0xffffffffu, indef);
  int lane = threadIdx.x & 31, b0 = 0;
  if (lane == 0 && ball) b0 = atomicAdd(count, __popc(ball));
  b0 = __shfl_sync(0xffffffffu, b0, 0);
  if (indef) list[b0 + __popc(ball & ((1u << lane) - 1u))] = u;
  }
}

// ---- negative-eigenspace projection (pass 2)
//
// M+ = Q max(L, 0) Q^T = M - sum_{l_j < 0} l_j q_j q_j^T: only the negative
// eigenpairs are needed (typically 1-3 of 9). Householder reduction
// M = Q T Q^T (Numerical Recipes tred2 order, reflectors kept in the packed
// lower triangle), eigenvalues of T by implicit QL without vectors, then per
// negative eigenvalue inverse iteration on T (guarded LDL^T), Gram-Schmidt
// against the previous ones (clustered spectra), and the back-transform
// q = H_{n-1} ... H_1 y. More than kNegMax negative eigenvalues fall back to
// the full tred2/tql2 eigendecomposition.
constexpr int kNegMax = 4;
#ifndef JGS2_PROJ_MINBLOCKS
#define JGS2_PROJ_MINBLOCKS 2
#endif
#ifndef JGS2_HESS_MINBLOCKS
#define JGS2_HESS_MINBLOCKS 2
#endif
#define JGS2_A(i, j) A[JGS2_PK(i, j) * S]

template <int S>
__device__ __forceinline__ void tred9_packed(double* A, double (&d)[9], double (&e)[9], double (&hv)[9]) {
  constexpr int n = 9;
#pragma unroll
  for (int i = n - 1; i > 0; --i) {
    const int l = i - 1;
    double h = 0.0;
    if (l > 0) {
      double scale = 0.0;
#pragma unroll
      for (int k = 0; k <= l; ++k) scale += fabs(JGS2_A(i, k));
      if (scale == 0.0) {
        e[i] = JGS2_A(i, l);
      } else {
        const double rs = rcp_nr(scale);
#pragma unroll
        for (int k = 0; k <= l; ++k) {
          double v = JGS2_A(i, k) * rs;
          JGS2_A(i, k) = v;
          h += v * v;
        }
        double f = JGS2_A(i, l);
        double g = sqrt_nr(h);
        if (f >= 0.0) g = -g;
        e[i] = scale * g;
        h -= f * g;
        JGS2_A(i, l) = f - g;
        const double rh = rcp_nr(h);
        f = 0.0;
#pragma unroll
        for (int j = 0; j <= l; ++j) {
          double gg = 0.0;
#pragma unroll
          for (int k = 0; k <= j; ++k) gg += JGS2_A(j, k) * JGS2_A(i, k);
#pragma unroll
          for (int k = j + 1; k <= l; ++k) gg += JGS2_A(k, j) * JGS2_A(i, k);
          e[j] = gg * rh;
          f += e[j] * JGS2_A(i, j);
        }
        const double hh = f * 0.5 * rh;
#pragma unroll
        for (int j = 0; j <= l; ++j) {
          f = JGS2_A(i, j);
          const double gg = e[j] - hh * f;
          e[j] = gg;
#pragma unroll
          for (int k = 0; k <= j; ++k) JGS2_A(j, k) -= (f * e[k] + gg * JGS2_A(i, k));
        }
      }
    } else {
      e[i] = JGS2_A(i, l);
    }
    hv[i] = h;
  }
  hv[0] = 0.0;
  e[0] = 0.0;
#pragma unroll
  for (int i = 0; i < n; ++i) d[i] = JGS2_A(i, i);
}

// eigenvalues of the symmetric tridiagonal T (diagonal d, T(i, i-1) = e[i])
// in place in d (implicit QL, JAMA tql2 without the vector updates)
__device__ __forceinline__ void tql1_9(double (&d)[9], double (&e)[9]) {
  constexpr int n = 9;
#pragma unroll
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  double f = 0.0, tst1 = 0.0;
  const double eps = 2.220446049250313e-16;
#pragma unroll
  for (int l = 0; l < n; ++l) {
    tst1 = fmax(tst1, fabs(d[l]) + fabs(e[l]));
    int m = n - 1;
#pragma unroll
    for (int mm = n - 2; mm >= l; --mm)
      if (fabs(e[mm]) <= eps * tst1) m = mm;
    if (l < n - 1 && m > l) {
      int iter = 0;
      do {
        ++iter;
        double g = d[l];
        double p = div_nr(d[l + 1] - g, 2.0 * e[l]);
        double r = sqrt_nr(fma(p, p, 1.0));
        if (p < 0) r = -r;
        d[l] = div_nr(e[l], p + r);
        d[l + 1] = e[l] * (p + r);
        double dl1 = d[l + 1];
        double h = g - d[l];
#pragma unroll
        for (int i = l + 2; i < n; ++i) d[i] -= h;
        f += h;
        p = d[n - 1];
#pragma unroll
        for (int i = n - 2; i > l; --i)
          if (i == m) p = d[i];
        double c = 1.0, c2 = c, c3 = c;
        double el1 = e[l + 1];
        double s = 0.0, s2 = 0.0;
#pragma unroll
        for (int i = n - 2; i >= l; --i) {
          if (i < m) {
            c3 = c2;
            c2 = c;
            s2 = s;
            g = c * e[i];
            h = c * p;
            double ei = e[i];
            double q2 = fma(p, p, ei * ei);
            double ri = rsqrt_nr(q2);
            r = sqrt_from_rsqrt(q2, ri);
            e[i + 1] = s * r;
            s = ei * ri;
            c = p * ri;
            p = c * d[i] - s * g;
            d[i + 1] = h + s * (c * g + s * d[i]);
          }
        }
        p = div_nr(-s * s2 * c3 * el1 * e[l], dl1);
        e[l] = s * p;
        d[l] = c * p;
      } while (fabs(e[l]) > eps * tst1 && iter < 60);
    }
    d[l] = d[l] + f;
    e[l] = 0.0;
  }
}

// y <- normalized solution of (T - lam I) y = y (3 steps), T = (d, e), guarded
// LDL^T without pivoting (near-singular by construction)
__device__ __forceinline__ void inverse_iteration9(const double (&d)[9], const double (&e)[9], double lam,
                                                   double tnorm, double (&y)[9]) {
  constexpr int n = 9;
  const double tiny = 2.220446049250313e-16 * tnorm + 1e-300;
  double Lo[9], Di[9];
  double Dk = d[0] - lam;
  if (fabs(Dk) < tiny) Dk = tiny;
  Lo[0] = 0.0;
  Di[0] = rcp_nr(Dk);
#pragma unroll
  for (int k = 1; k < n; ++k) {
    Lo[k] = e[k] * Di[k - 1];
    Dk = (d[k] - lam) - Lo[k] * e[k];
    if (fabs(Dk) < tiny) Dk = tiny;
    Di[k] = rcp_nr(Dk);
  }
#pragma unroll 1
  for (int it = 0; it < 3; ++it) {
#pragma unroll
    for (int k = 1; k < n; ++k) y[k] -= Lo[k] * y[k - 1];
#pragma unroll
    for (int k = 0; k < n; ++k) y[k] *= Di[k];
#pragma unroll
    for (int k = n - 2; k >= 0; --k) y[k] -= Lo[k + 1] * y[k + 1];
    double nn = 0.0;
#pragma unroll
    for (int k = 0; k < n; ++k) nn += y[k] * y[k];
    const double rn = rsqrt_nr(nn);
#pragma unroll
    for (int k = 0; k < n; ++k) y[k] *= rn;
  }
}

// Pass 2 over the compacted indefinite elements (grid-stride up to *count):
// M+ written over M in place.
__global__ void __launch_bounds__(kHessThreads, JGS2_PROJ_MINBLOCKS)
k_mplus_project(int* count, const int* list, int* list2, double* mplus) {
  extern __shared__ double hsm[];
  constexpr int S = kHessThreads;
  const int n = *count;
  for (int i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x) {
    int idx = i0 + threadIdx.x;
    if (idx >= n) break;
    double* o = mplus + 45 * (size_t)list[idx];
    double* A = hsm + threadIdx.x;              // packed lower 45 (reflectors after tred)
    double* Y = hsm + 45 * S + threadIdx.x;     // kNegMax - 1 tridiagonal-space vectors
    double* Tm = hsm + (45 + 9 * (kNegMax - 1)) * S + threadIdx.x;  // T: diagonal, subdiagonal
    double tnorm = 0.0;
#pragma unroll
    for (int q = 0; q < 45; ++q) {
      double m = o[q];
      A[q * S] = m;
      tnorm = fmax(tnorm, fabs(m));
    }
    double lam[9], ee[9];
    {
      double hv[9];
      tred9_packed<S>(A, lam, ee, hv);
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        JGS2_A(i, i) = hv[i];  // reflector norms h_i in the (now unused) diagonal slots
        Tm[i * S] = lam[i];
        Tm[(9 + i) * S] = ee[i];
      }
    }
    tql1_9(lam, ee);
    // negative eigenvalues, ascending (at most 9; selection into neg[])
    int k = 0;
#pragma unroll
    for (int q = 0; q < 9; ++q) k += lam[q] < 0.0;
    if (k == 0) continue;  // PSD already (LDL^T failed on a zero pivot)
    if (k > kNegMax) {  // many negative modes: the full eigendecomposition (k_mplus_full)
      int slot = atomicAdd(count + 1, 1);
      list2[slot] = list[idx];
      continue;
    }
#pragma unroll 1
    for (int j = 0; j < k; ++j) {
      double l = 0.0;  // j-th smallest eigenvalue (negative), removed from lam
#pragma unroll
      for (int q = 0; q < 9; ++q) l = fmin(l, lam[q]);
      bool done = false;
#pragma unroll
      for (int q = 0; q < 9; ++q)
        if (!done && lam[q] == l) { lam[q] = 0.0; done = true; }
      double y[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) y[q] = 1.0 + 0.1 * q + 0.01 * j * q * q;
      {
        double d[9], e[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) { d[q] = Tm[q * S]; e[q] = Tm[(9 + q) * S]; }
        inverse_iteration9(d, e, l, tnorm, y);
      }
#pragma unroll 1
      for (int t = 0; t < j; ++t) {  // Gram-Schmidt against earlier negative vectors
        const double* Yt = Y + 9 * t * S;
        double dp = 0.0;
#pragma unroll
        for (int q = 0; q < 9; ++q) dp += Yt[q * S] * y[q];
#pragma unroll
        for (int q = 0; q < 9; ++q) y[q] -= dp * Yt[q * S];
      }
      double nn = 0.0;
#pragma unroll
      for (int q = 0; q < 9; ++q) nn += y[q] * y[q];
      const double rn = rsqrt_nr(nn);
#pragma unroll
      for (int q = 0; q < 9; ++q) y[q] *= rn;
      if (j < kNegMax - 1) {
#pragma unroll
        for (int q = 0; q < 9; ++q) Y[(9 * j + q) * S] = y[q];
      }
      // back-transform q = H_8 ... H_1 y, H_i = I - u_i u_i^T / h_i, u_i = A(i, 0..i-1)
#pragma unroll
      for (int i = 1; i < 9; ++i) {
        const double hi = JGS2_A(i, i);
        if (hi != 0.0) {
          double dp = 0.0;
#pragma unroll
          for (int c = 0; c < i; ++c) dp += JGS2_A(i, c) * y[c];
          dp *= rcp_nr(hi);
#pragma unroll
          for (int c = 0; c < i; ++c) y[c] -= dp * JGS2_A(i, c);
        }
      }
#pragma unroll
      for (int a = 0; a < 9; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) o[JGS2_PK(a, b)] -= l * y[a] * y[b];
    }
  }
}
#undef JGS2_A

// One-pass form (JGS2_HESS_ONEPASS=1, for A/B measurements): the full
// eigendecomposition for every indefinite element of a warp.
// One thread per element: closed-form M, LDL^T inertia test, and (when
// indefinite) the tred2/tql2 projection on per-thread interleaved shared
// memory. The number of indefinite elements is accumulated with one
// warp-aggregated atomic per warp (diagnostic only; results do not depend
// on it).
__global__ void __launch_bounds__(kHessThreads, JGS2_HESS_MINBLOCKS)
k_element_mplus(int n, const int* elems, const double* __restrict__ xs, const int4* __restrict__ tets,
                const double* __restrict__ dminv, const double4* __restrict__ eprops, double* mplus,
                int* count) {
  extern __shared__ double hsm[];
  int u = blockIdx.x * blockDim.x + threadIdx.x;
  bool active = u < n;
  bool indef = false;
  if (active) {
    int e = elems ? elems[u] : u;
    double D[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) D[i] = __ldg(dminv + 9 * (size_t)e + i);
    int4 t = __ldg(tets + e);
    double x0[3], x1[3], x2[3], x3[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      x0[c] = __ldg(xs + 3 * t.x + c); x1[c] = __ldg(xs + 3 * t.y + c);
      x2[c] = __ldg(xs + 3 * t.z + c); x3[c] = __ldg(xs + 3 * t.w + c);
    }
    double F[9];
    deformation_gradient(x0, x1, x2, x3, D, F);
    double4 ep = eprops[e];
    double Mp[45];
    reduced_hessian_closed(F, D, ep.x, snh_const(ep.y, ep.z), Mp);
    double* o = mplus + 45 * (size_t)u;
    if (is_pos_def9(Mp)) {
#pragma unroll
      for (int i = 0; i < 45; ++i) o[i] = Mp[i];
    } else {
      indef = true;
      double* Vs = hsm + threadIdx.x;
#pragma unroll
      for (int i = 0; i < 9; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
          Vs[(9 * i + j) * kHessThreads] = Mp[JGS2_PK(i, j)];
          Vs[(9 * j + i) * kHessThreads] = Mp[JGS2_PK(i, j)];
        }
      double dg[9], od[9];
      sym_eig9_reg<kHessThreads>(Vs, dg, od);
      double lam[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) lam[q] = fmax(dg[q], 0.0);
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        double vi[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) vi[q] = Vs[(9 * i + q) * kHessThreads] * lam[q];
#pragma unroll
        for (int j = 0; j <= i; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < 9; ++q) acc += vi[q] * Vs[(9 * j + q) * kHessThreads];
          o[JGS2_PK(i, j)] = acc;
        }
      }
    }
  }
  unsigned ball = __ballot_sync(0xffffffffu, indef);
  if ((threadIdx.x & 31) == 0 && ball) atomicAdd(count, __popc(ball));
}
constexpr size_t kHessSmemBytes = 81 * kHessThreads * sizeof(double);
constexpr size_t kProjSmemBytes = (45 + 9 * (kNegMax - 1) + 18) * kHessThreads * sizeof(double);

// Pass 3: the rare elements with more than kNegMax negative modes, full
// tred2/tql2 eigendecomposition (grid-stride up to count[1]).
__global__ void __launch_bounds__(kHessThreads, 2)
k_mplus_full(const int* count, const int* list2, double* mplus) {
  extern __shared__ double hsm[];
  constexpr int S = kHessThreads;
  const int n = count[1];
  for (int i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x) {
    int idx = i0 + threadIdx.x;
    if (idx >= n) break;
    double* o = mplus + 45 * (size_t)list2[idx];
    double* V = hsm + threadIdx.x;
#pragma unroll
    for (int a = 0; a < 9; ++a)
#pragma unroll
      for (int b = 0; b <= a; ++b) {
        double m = o[JGS2_PK(a, b)];
        V[(9 * a + b) * S] = m;
        V[(9 * b + a) * S] = m;
      }
    double dg[9], od[9];
    sym_eig9_reg<S>(V, dg, od);
#pragma unroll
    for (int q = 0; q < 9; ++q) dg[q] = fmax(dg[q], 0.0);
#pragma unroll
    for (int a = 0; a < 9; ++a) {
      double vi[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) vi[q] = V[(9 * a + q) * S] * dg[q];
#pragma unroll
      for (int b = 0; b <= a; ++b) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 9; ++q) acc += vi[q] * V[(9 * b + q) * S];
        o[JGS2_PK(a, b)] = acc;
      }
    }
  }
}

// Projected reduced Hessians of n elements (elems[u], or u when null) into
// out[45 u]: pass 1 for all, pass 2 for the indefinite ones only (about half
// of the cubature elements in a deforming scene; a warp of the one-pass form
// paid the eigen solve whenever any of its 32 elements needed it).
// count: 2 device ints (zeroed here; count[0] = indefinite elements,
// count[1] = those with more than kNegMax negative modes);
// list: device scratch of 2n ints.
// blocks_per_sm > 0 caps every pass at that many resident blocks per SM
// (grid-stride), leaving the rest of each SM to a concurrent memory-bound
// kernel (JGS2_HESS_OVERLAP: the passes under the factor solve).
inline void launch_element_mplus(int n, const int* elems, const double* xs, const int4* tets,
                                 const double* dminv, const double4* eprops, double* out, int* count,
                                 int* list, cudaStream_t stream, int blocks_per_sm = 0) {
  if (n <= 0) return;
  int grid = (n + kHessThreads - 1) / kHessThreads;
  cudaMemsetAsync(count, 0, 2 * sizeof(int), stream);
  static const bool onepass = getenv("JGS2_HESS_ONEPASS") != nullptr;
  if (onepass) {
    k_element_mplus<<<grid, kHessThreads, kHessSmemBytes, stream>>>(n, elems, xs, tets, dminv, eprops, out,
                                                                    count);
    return;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid1 = blocks_per_sm > 0 ? std::min(grid, sms * blocks_per_sm) : grid;
  k_mplus_closed<<<grid1, kHessThreads, 0, stream>>>(n, elems, xs, tets, dminv, eprops, out, count, list);
  int grid2 = std::min(grid, sms * (blocks_per_sm > 0 ? blocks_per_sm : JGS2_HESS_MINBLOCKS * 4));
  k_mplus_project<<<std::min(grid, sms * (blocks_per_sm > 0 ? blocks_per_sm : 3 * 4)), kHessThreads,
                    kProjSmemBytes, stream>>>(count, list, list + n, out);
  k_mplus_full<<<grid2, kHessThreads, kHessSmemBytes, stream>>>(count, list + n, out);
}

}  // namespace jgs2
