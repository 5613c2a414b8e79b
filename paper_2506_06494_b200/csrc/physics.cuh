// Device math for the JGS2 runtime path (sm_100a, FP64 throughout).
//
// Conventions follow the reference (pkg/src/tetsolve/energy.py:1-7):
//   * 3x3 matrices are row-major double[9], m[3*r + c];
//   * vec(F)[3*j + r] = F[r][j] (column stacked); element DOFs vertex-major;
//   * W[m][j] = dF[:, j]/dx_m  (energy.py:152-157).
// Where a threshold decision downstream depends on the rounding of a
// product, the reference's numpy rounding order is reproduced explicitly
// (SURVEY App. B / C5): batched 3x3 matmul = fma(x2,y2,fma(x1,y1,x0*y0)).
#pragma once
#include <cstdint>
#include <cmath>
#include "dmath.cuh"

#define JGS2_HD __host__ __device__ __forceinline__

namespace jgs2 {

// ---------------------------------------------------------------- 3x3 algebra
JGS2_HD void mat3_zero(double* a) {
#pragma unroll
  for (int i = 0; i < 9; ++i) a[i] = 0.0;
}
JGS2_HD void mat3_eye(double* a) {
#pragma unroll
  for (int i = 0; i < 9; ++i) a[i] = (i % 4 == 0) ? 1.0 : 0.0;
}
// c = a * b (numpy batched-matmul FMA chain order)
JGS2_HD void mat3_mul(const double* a, const double* b, double* c) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      c[3 * r + k] = fma(a[3 * r + 2], b[6 + k], fma(a[3 * r + 1], b[3 + k], a[3 * r] * b[k]));
}
// c = a * b^T
JGS2_HD void mat3_mul_bt(const double* a, const double* b, double* c) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      c[3 * r + k] = a[3 * r] * b[3 * k] + a[3 * r + 1] * b[3 * k + 1] + a[3 * r + 2] * b[3 * k + 2];
}
// c = a^T * b
JGS2_HD void mat3_mul_at(const double* a, const double* b, double* c) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      c[3 * r + k] = a[r] * b[k] + a[3 + r] * b[3 + k] + a[6 + r] * b[6 + k];
}
// R a R^T
JGS2_HD void mat3_conj(const double* R, const double* a, double* out) {
  double t[9];
  mat3_mul(R, a, t);
  mat3_mul_bt(t, R, out);
}
JGS2_HD void mat3_vec(const double* a, const double* v, double* o) {
#pragma unroll
  for (int r = 0; r < 3; ++r) o[r] = a[3 * r] * v[0] + a[3 * r + 1] * v[1] + a[3 * r + 2] * v[2];
}
JGS2_HD void mat3_tvec(const double* a, const double* v, double* o) {
#pragma unroll
  for (int r = 0; r < 3; ++r) o[r] = a[r] * v[0] + a[3 + r] * v[1] + a[6 + r] * v[2];
}
JGS2_HD double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
JGS2_HD void cross3(const double* a, const double* b, double* c) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}
// numpy norm rounding order: sqrt((x^2 + y^2) + z^2)
__device__ __forceinline__ double norm3_np(const double* a) {
  return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(a[0], a[0]), __dmul_rn(a[1], a[1])), __dmul_rn(a[2], a[2])));
}

// ------------------------------------------------------- symmetric eigen (Jacobi)
// Cyclic Jacobi on a symmetric N x N matrix a (row-major, full storage).
// On exit the diagonal holds eigenvalues; if V != nullptr its columns are the
// eigenvectors (V[i*N + k] = component i of eigenvector k).
template <int N>
JGS2_HD void jacobi_eig(double* a, double* V, int max_sweeps = 20) {
  if (V) {
    for (int i = 0; i < N * N; ++i) V[i] = 0.0;
    for (int i = 0; i < N; ++i) V[i * N + i] = 1.0;
  }
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int p = 0; p < N; ++p) {
      diag += a[p * N + p] * a[p * N + p];
      for (int q = p + 1; q < N; ++q) off += a[p * N + q] * a[p * N + q];
    }
    if (off <= 1e-34 * diag || off == 0.0) break;
    for (int p = 0; p < N - 1; ++p) {
      for (int q = p + 1; q < N; ++q) {
        double apq = a[p * N + q];
        if (apq == 0.0) continue;
        double app = a[p * N + p], aqq = a[q * N + q];
        double num = aqq - app, den = 2.0 * apq;
        double t = 0.0;  // |theta| >= 1e150: apq negligible, t ~ 1/(2 theta) -> 0
        if (fabs(num) < 1e150 * fabs(den)) {
          double theta = hd_div(num, den);
          t = hd_div(theta >= 0.0 ? 1.0 : -1.0, fabs(theta) + hd_sqrt(theta * theta + 1.0));
        }
        double c = hd_rsqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < N; ++k) {
          double akp = a[k * N + p], akq = a[k * N + q];
          a[k * N + p] = c * akp - s * akq;
          a[k * N + q] = s * akp + c * akq;
        }
        for (int k = 0; k < N; ++k) {
          double apk = a[p * N + k], aqk = a[q * N + k];
          a[p * N + k] = c * apk - s * aqk;
          a[q * N + k] = s * apk + c * aqk;
        }
        a[p * N + q] = a[q * N + p] = 0.0;
        if (V) {
          for (int k = 0; k < N; ++k) {
            double vkp = V[k * N + p], vkq = V[k * N + q];
            V[k * N + p] = c * vkp - s * vkq;
            V[k * N + q] = s * vkp + c * vkq;
          }
        }
      }
    }
  }
}

// Smallest eigenvalue of a symmetric 3x3 (for the SPD floor,
// local_solver.py:409-414).
JGS2_HD double sym3_min_eig(const double* a_in) {
  double a[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) a[i] = a_in[i];
  jacobi_eig<3>(a, nullptr);
  return fmin(a[0], fmin(a[4], a[8]));
}

// Rotation of the polar decomposition of A with the reference's handling of
// reflections and degenerate input (subspace.py:206-231):
//   R = U diag(1, 1, sign det(U V^T)) V^T,  identity if |A|_F <= 1e-12 or
//   sigma_max <= 1e-12 * max(|A|_F, 1).
JGS2_HD void polar_rotation(const double* A, double* R) {
  double nrm2 = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) nrm2 += A[i] * A[i];
  double nrm = sqrt(nrm2);
  if (!(nrm > 1e-12)) { mat3_eye(R); return; }
  double B[9], V[9];
  mat3_mul_at(A, A, B);  // A^T A
  jacobi_eig<3>(B, V, 30);
  double lam[3] = {B[0], B[4], B[8]};
  int o[3] = {0, 1, 2};
  // sort descending
  if (lam[o[0]] < lam[o[1]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
  if (lam[o[1]] < lam[o[2]]) { int t = o[1]; o[1] = o[2]; o[2] = t; }
  if (lam[o[0]] < lam[o[1]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
  double v1[3], v2[3], v3[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) { v1[i] = V[i * 3 + o[0]]; v2[i] = V[i * 3 + o[1]]; v3[i] = V[i * 3 + o[2]]; }
  double s1 = sqrt(fmax(lam[o[0]], 0.0));
  if (s1 <= 1e-12 * fmax(nrm, 1.0)) { mat3_eye(R); return; }
  // right-handed V
  double c12[3];
  cross3(v1, v2, c12);
  if (dot3(c12, v3) < 0.0) { v3[0] = -v3[0]; v3[1] = -v3[1]; v3[2] = -v3[2]; }
  double u1[3], u2[3], u3[3];
  mat3_vec(A, v1, u1);
  double r1 = hd_rsqrt(dot3(u1, u1));
  u1[0] *= r1; u1[1] *= r1; u1[2] *= r1;
  mat3_vec(A, v2, u2);
  double p = dot3(u1, u2);
  u2[0] -= p * u1[0]; u2[1] -= p * u1[1]; u2[2] -= p * u1[2];
  double n2 = sqrt(dot3(u2, u2));
  if (!(n2 > 0.0)) {  // rank-1: any completion (reference: LAPACK's)
    double e[3] = {fabs(u1[0]) < 0.9 ? 1.0 : 0.0, fabs(u1[0]) < 0.9 ? 0.0 : 1.0, 0.0};
    double pe = dot3(u1, e);
    u2[0] = e[0] - pe * u1[0]; u2[1] = e[1] - pe * u1[1]; u2[2] = e[2] - pe * u1[2];
    n2 = sqrt(dot3(u2, u2));
  }
  double r2 = hd_rcp(n2);
  u2[0] *= r2; u2[1] *= r2; u2[2] *= r2;
  cross3(u1, u2, u3);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) R[3 * r + c] = u1[r] * v1[c] + u2[r] * v2[c] + u3[r] * v3[c];
}

// LU with partial pivoting 3x3 solve (LAPACK gesv semantics,
// local_solver.py:580-588). Returns false if singular / non-finite.
JGS2_HD bool solve3_lu(const double* a_in, const double* b_in, double* x) {
  double a[9], b[3];
#pragma unroll
  for (int i = 0; i < 9; ++i) a[i] = a_in[i];
  b[0] = b_in[0]; b[1] = b_in[1]; b[2] = b_in[2];
  for (int k = 0; k < 3; ++k) {
    int piv = k;
    double best = fabs(a[3 * k + k]);
    for (int r = k + 1; r < 3; ++r)
      if (fabs(a[3 * r + k]) > best) { best = fabs(a[3 * r + k]); piv = r; }
    if (best == 0.0) return false;
    if (piv != k) {
      for (int c = 0; c < 3; ++c) { double t = a[3 * k + c]; a[3 * k + c] = a[3 * piv + c]; a[3 * piv + c] = t; }
      double t = b[k]; b[k] = b[piv]; b[piv] = t;
    }
    for (int r = k + 1; r < 3; ++r) {
      double l = a[3 * r + k] / a[3 * k + k];
      for (int c = k + 1; c < 3; ++c) a[3 * r + c] -= l * a[3 * k + c];
      b[r] -= l * b[k];
    }
  }
  for (int k = 2; k >= 0; --k) {
    double s = b[k];
    for (int c = k + 1; c < 3; ++c) s -= a[3 * k + c] * x[c];
    x[k] = s / a[3 * k + k];
  }
  return isfinite(x[0]) && isfinite(x[1]) && isfinite(x[2]);
}

// ------------------------------------------------------------ stable Neo-Hookean
struct SnhConst { double mu_s, lam_s, alpha; };
// energy.py:62-68
JGS2_HD SnhConst snh_const(double mu, double lam) {
  SnhConst c;
  c.mu_s = 4.0 * mu / 3.0;
  c.lam_s = lam + 5.0 * mu / 6.0;
  c.alpha = 1.0 + 0.75 * c.mu_s / c.lam_s;
  return c;
}

// F = Ds * Dm^-1 (energy.py:53-59); x0..x3 corner positions, D row-major.
JGS2_HD void deformation_gradient(const double* x0, const double* x1, const double* x2,
                                  const double* x3, const double* D, double* F) {
  double ds[9];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    ds[3 * r + 0] = x1[r] - x0[r];
    ds[3 * r + 1] = x2[r] - x0[r];
    ds[3 * r + 2] = x3[r] - x0[r];
  }
  mat3_mul(ds, D, F);
}

// cofactor columns (energy.py:71-76): cof[:,0]=F1xF2, cof[:,1]=F2xF0, cof[:,2]=F0xF1
JGS2_HD void cofactor(const double* F, double* C) {
  double f0[3] = {F[0], F[3], F[6]}, f1[3] = {F[1], F[4], F[7]}, f2[3] = {F[2], F[5], F[8]};
  double c0[3], c1[3], c2[3];
  cross3(f1, f2, c0);
  cross3(f2, f0, c1);
  cross3(f0, f1, c2);
#pragma unroll
  for (int r = 0; r < 3; ++r) { C[3 * r] = c0[r]; C[3 * r + 1] = c1[r]; C[3 * r + 2] = c2[r]; }
}

JGS2_HD double frob2(const double* F) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) s += F[i] * F[i];
  return s;
}

JGS2_HD double det3_cof(const double* F, const double* C) {
  return F[0] * C[0] + F[3] * C[3] + F[6] * C[6];
}

// psi(F) (energy.py:79-86)
JGS2_HD double snh_psi(const double* F, SnhConst k) {
  double C[9];
  cofactor(F, C);
  double ic = frob2(F), J = det3_cof(F, C);
  double psi0 = -0.5 * k.mu_s * log(4.0) + 0.5 * k.lam_s * (1.0 - k.alpha) * (1.0 - k.alpha);
  return 0.5 * k.mu_s * (ic - 3.0) - 0.5 * k.mu_s * log(ic + 1.0)
       + 0.5 * k.lam_s * (J - k.alpha) * (J - k.alpha) - psi0;
}

// First Piola-Kirchhoff P (energy.py:89-97)
JGS2_HD void snh_piola(const double* F, SnhConst k, double* P) {
  double C[9];
  cofactor(F, C);
  double ic = frob2(F), J = det3_cof(F, C);
  double t1 = k.mu_s * (1.0 - 1.0 / (ic + 1.0));
  double t2 = k.lam_s * (J - k.alpha);
#pragma unroll
  for (int i = 0; i < 9; ++i) P[i] = t1 * F[i] + t2 * C[i];
}

// W = [-1^T Dm^-1; Dm^-1] (energy.py:152-157); W[m*3 + j]
JGS2_HD void shape_weights(const double* D, double* W) {
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    W[j] = -(D[j] + D[3 + j] + D[6 + j]);
    W[3 + j] = D[j];
    W[6 + j] = D[3 + j];
    W[9 + j] = D[6 + j];
  }
}

// d2psi/dF2 (9x9, vec order 3j+r) (energy.py:110-141)
JGS2_HD void snh_hessian9(const double* F, SnhConst k, double* H) {
  double C[9];
  cofactor(F, C);
  double ic = frob2(F), J = det3_cof(F, C);
  double d = k.mu_s * (1.0 - 1.0 / (ic + 1.0));
  double c1 = 2.0 * k.mu_s / ((ic + 1.0) * (ic + 1.0));
  double s = k.lam_s * (J - k.alpha);
  double f[9], g[9];
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int r = 0; r < 3; ++r) { f[3 * j + r] = F[3 * r + j]; g[3 * j + r] = C[3 * r + j]; }
#pragma unroll
  for (int a = 0; a < 9; ++a)
#pragma unroll
    for (int b = 0; b < 9; ++b)
      H[9 * a + b] = (a == b ? d : 0.0) + c1 * f[a] * f[b] + k.lam_s * g[a] * g[b];
  // skew blocks: H[blk(bi,bj)] += s * (+/-)[F_c]x
  auto addskew = [&](int bi, int bj, int col, double sign) {
    double v0 = F[col], v1 = F[3 + col], v2 = F[6 + col];
    double S[9] = {0.0, -v2, v1, v2, 0.0, -v0, -v1, v0, 0.0};
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) H[9 * (3 * bi + r) + 3 * bj + c] += s * sign * S[3 * r + c];
  };
  addskew(0, 1, 2, -1.0);
  addskew(0, 2, 1, +1.0);
  addskew(1, 0, 2, +1.0);
  addskew(1, 2, 0, -1.0);
  addskew(2, 0, 1, -1.0);
  addskew(2, 1, 0, +1.0);
}

// Translation-complement basis U (4x3, Hadamard columns, exact in binary):
// the 12x12 element Hessian annihilates rigid translations, so
// PSD(H12) = T PSD(T^T H12 T) T^T with T = U (x) I3.
__host__ __device__ constexpr double kHad(int m, int p) {
  // columns: (1,1,-1,-1)/2, (1,-1,1,-1)/2, (1,-1,-1,1)/2
  return (m == 0) ? 0.5
       : (p == 0) ? ((m == 1) ? 0.5 : -0.5)
       : (p == 1) ? ((m == 2) ? 0.5 : -0.5)
                  : ((m == 3) ? 0.5 : -0.5);
}

// Reduced 9x9 element Hessian M = V (G(x)I)^T H9 (G(x)I), G = W^T U (3x3).
// Index convention: M[(3p + r)*9 + (3q + s)] in complement coordinates.
JGS2_HD void reduced_hessian9(const double* F, const double* D, double vol, SnhConst k,
                              double* M) {
  double H9[81];
  snh_hessian9(F, k, H9);
  double W[12];
  shape_weights(D, W);
  double G[9];  // G[j][p]
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int p = 0; p < 3; ++p)
      G[3 * j + p] = W[j] * kHad(0, p) + W[3 + j] * kHad(1, p) + W[6 + j] * kHad(2, p) +
                     W[9 + j] * kHad(3, p);
  // T1[(j r), (q s)] = sum_k H9[(j r),(k s)] G[k][q]
  double T1[81];
#pragma unroll
  for (int a = 0; a < 9; ++a)
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int s = 0; s < 3; ++s)
        T1[9 * a + 3 * q + s] = H9[9 * a + s] * G[q] + H9[9 * a + 3 + s] * G[3 + q] +
                                H9[9 * a + 6 + s] * G[6 + q];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int b = 0; b < 9; ++b)
        M[9 * (3 * p + r) + b] = vol * (G[p] * T1[9 * r + b] + G[3 + p] * T1[9 * (3 + r) + b] +
                                        G[6 + p] * T1[9 * (6 + r) + b]);
}

// In-place PSD projection of a symmetric 9x9 (energy.py:144-149 on the
// reduced coordinates); out = Q max(L,0) Q^T.
JGS2_HD void psd_project9(double* M) {
  double a[81], Q[81];
#pragma unroll 1
  for (int i = 0; i < 81; ++i) a[i] = M[i];
  // symmetrize like the reference (0.5*(h + h^T))
#pragma unroll 1
  for (int i = 0; i < 9; ++i)
    for (int j = i + 1; j < 9; ++j) {
      double s = 0.5 * (a[9 * i + j] + a[9 * j + i]);
      a[9 * i + j] = a[9 * j + i] = s;
    }
  jacobi_eig<9>(a, Q, 30);
  double lam[9];
#pragma unroll 1
  for (int i = 0; i < 9; ++i) lam[i] = fmax(a[9 * i + i], 0.0);
#pragma unroll 1
  for (int i = 0; i < 9; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0.0;
      for (int k = 0; k < 9; ++k) s += Q[9 * i + k] * lam[k] * Q[9 * j + k];
      M[9 * i + j] = M[9 * j + i] = s;
    }
}

// Packed lower-triangle index for symmetric 9x9 (45 entries).
JGS2_HD int tri9(int i, int j) { return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i; }

// Expand the 12x12 Hessian from the reduced 9x9: H12[(m r),(n s)] =
// sum_{p,q} U[m][p] M[(p r),(q s)] U[n][q].
JGS2_HD void expand_hessian12(const double* M, double* H12) {
  for (int m = 0; m < 4; ++m)
    for (int r = 0; r < 3; ++r)
      for (int n = 0; n < 4; ++n)
        for (int s = 0; s < 3; ++s) {
          double acc = 0.0;
          for (int p = 0; p < 3; ++p)
            for (int q = 0; q < 3; ++q)
              acc += kHad(m, p) * M[9 * (3 * p + r) + 3 * q + s] * kHad(n, q);
          H12[12 * (3 * m + r) + 3 * n + s] = acc;
        }
}

}  // namespace jgs2
