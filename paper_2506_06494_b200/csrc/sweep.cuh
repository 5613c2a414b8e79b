// Per-sweep kernels of the JGS2 Jacobi iteration (corotated_cubature).
// Reference: local_solver.py:306-323 (assembled field), 355-416 (sampled
// corrections + reduced systems), 530-553 (local line search), 555-577
// (global backtrack), 580-588 (3x3 solves), 606-655 (sweep);
// subspace.py:206-231 (rotations); assembly.py:183-192 (energy).
#pragma once
#include "context.cuh"
#include "geometry.cuh"

namespace jgs2 {

struct DevModel {
  int nv, ne, smax, gmax, nfree;
  const int4* tets;
  const double* dminv;
  const double4* eprops;
  const int* inc_ptr;
  const int* inc;
  const double* mass;
  const uint8_t* fixed;
  const int* pos;
  const int* free_list;
  int v0, v1;  // this rank's vertex range (vertex pass)
};

// ---------------------------------------------------------------- vertex pass
// Per vertex, over its incident elements in ascending element order:
//   g_asm[v] = sum_e (V_e P_e W_e[slot] + qm_e (x_v - z_v)/h^2)   (cubature.py:37-60, 83-90)
//   acc[v]   = sum_e V_e F_e -> R[v] = polar(acc)               (subspace.py:206-231)
// Elements are re-evaluated per incident vertex (4x) instead of staging
// per-element results through HBM; the element record (120 B) is
// L2-resident across the 4 visits for a locality-ordered mesh.
template <bool ROT>
__global__ void __launch_bounds__(kBlock)
k_vertex_pass(DevModel m, const double* __restrict__ x, const double* __restrict__ z, double h,
              double* __restrict__ R, double* __restrict__ gasm) {
  int v = m.v0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= m.v1) return;
  double h2 = h * h;
  double xv[3] = {x[3 * v], x[3 * v + 1], x[3 * v + 2]};
  double dv[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) dv[c] = (xv[c] - z[3 * v + c]) / h2;
  double acc[9], g[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 9; ++i) acc[i] = 0.0;
  int p0 = m.inc_ptr[v], p1 = m.inc_ptr[v + 1];
  for (int p = p0; p < p1; ++p) {
    int code = __ldg(m.inc + p), e = code >> 2, slot = code & 3;
    int4 t = __ldg(m.tets + e);
    double D[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) D[i] = __ldg(m.dminv + 9 * (size_t)e + i);
    double4 ep = m.eprops[e];
    double x0[3], x1[3], x2[3], x3[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      x0[c] = __ldg(x + 3 * t.x + c); x1[c] = __ldg(x + 3 * t.y + c);
      x2[c] = __ldg(x + 3 * t.z + c); x3[c] = __ldg(x + 3 * t.w + c);
    }
    double F[9];
    deformation_gradient(x0, x1, x2, x3, D, F);
    if (ROT) {
#pragma unroll
      for (int i = 0; i < 9; ++i) acc[i] += F[i] * ep.x;
    }
    double P[9];
    snh_piola(F, snh_const(ep.y, ep.z), P);
    double Wm[3];
    if (slot == 0) {
#pragma unroll
      for (int j = 0; j < 3; ++j) Wm[j] = -(D[j] + D[3 + j] + D[6 + j]);
    } else {
#pragma unroll
      for (int j = 0; j < 3; ++j) Wm[j] = D[3 * (slot - 1) + j];
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double s = Wm[0] * P[3 * r] + Wm[1] * P[3 * r + 1] + Wm[2] * P[3 * r + 2];
      g[r] += ep.x * s + ep.w * dv[r];
    }
  }
  if (p1 == p0) {  // isolated vertex: inertia directly (local_solver.py:315-318)
    double c = m.mass[v] / h2;
#pragma unroll
    for (int r = 0; r < 3; ++r) g[r] += c * (xv[r] - z[3 * v + r]);
  }
  gasm[3 * v] = g[0]; gasm[3 * v + 1] = g[1]; gasm[3 * v + 2] = g[2];
  if (ROT) {
    double Rv[9];
    polar_rotation(acc, Rv);
#pragma unroll
    for (int i = 0; i < 9; ++i) R[9 * (size_t)v + i] = Rv[i];
  }
}

// Element stencil gradients (cubature.stencil_gradients, cubature.py:37-60):
// V P W^T per corner plus the element's quarter-mass inertia share,
// out[12 e + 3 a + r] (vertex-major element DOFs).
__global__ void __launch_bounds__(kBlock)
k_stencil_grads(DevModel m, const double* __restrict__ x, const double* __restrict__ z, double h, double* out) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m.ne) return;
  int4 t = __ldg(m.tets + e);
  int cs[4] = {t.x, t.y, t.z, t.w};
  double D[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) D[i] = __ldg(m.dminv + 9 * (size_t)e + i);
  double xa[4][3];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) xa[a][c] = x[3 * cs[a] + c];
  double F[9], P[9];
  deformation_gradient(xa[0], xa[1], xa[2], xa[3], D, F);
  double4 ep = m.eprops[e];
  snh_piola(F, snh_const(ep.y, ep.z), P);
  double h2 = h * h;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double Wm[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) Wm[j] = a == 0 ? -(D[j] + D[3 + j] + D[6 + j]) : D[3 * (a - 1) + j];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double s = Wm[0] * P[3 * r] + Wm[1] * P[3 * r + 1] + Wm[2] * P[3 * r + 2];
      out[12 * (size_t)e + 3 * a + r] = ep.x * s + ep.w * ((xa[a][r] - z[3 * cs[a] + r]) / h2);
    }
  }
}

// y = R^T g into the ND-ordered rhs for free vertices (local_solver.py:124-125);
// grad_sq is reduced in vertex chunks (partition.cuh)
__global__ void __launch_bounds__(kBlock)
k_rhs(DevModel m, const double* __restrict__ R, const double* __restrict__ gasm, double* b) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.nfree) return;
  int v = m.free_list[i];
  double g[3] = {gasm[3 * v], gasm[3 * v + 1], gasm[3 * v + 2]};
  double y[3];
  mat3_tvec(R + 9 * (size_t)v, g, y);
  int p = m.pos[v];
  b[3 * p] = y[0]; b[3 * p + 1] = y[1]; b[3 * p + 2] = y[2];
}

// q lookup in the ND-ordered solution (fixed vertices: q = 0)
__device__ __forceinline__ void q_of(const DevModel& m, const double* b, int w, double* q) {
  int p = m.pos[w];
  if (p < 0) { q[0] = q[1] = q[2] = 0.0; return; }
  q[0] = b[3 * p]; q[1] = b[3 * p + 1]; q[2] = b[3 * p + 2];
}

struct LocalArgs {
  const double* R;
  const double* gasm;       // assembled field (plain mode)
  const double* b;          // collect solution q (ND order)
  const double* gbar;       // nv*9
  const int* group;         // nv*gmax
  const double* grows;      // nv*9*gmax  (3 x 3gmax row-major)
  // cubature slots, slot-major SoA (coalesced across the vertices of a warp):
  // cub_u/w/verts[s * nv + v], cub_rows[(s * 36 + q) * nv + v]
  const int* cub_u;
  const double* cub_w;
  const double* cub_rows;
  const int4* cub_verts;
  int nv;
  const double* crest;
  const double* mplus;
  double h;
  // outputs
  double* A_out;            // optional nv*9 (reduced systems, debug)
  double* g_out;            // optional nv*3
  double* corr_out;         // optional nv*9 (sampled corrections, debug)
  double* delta;            // nv*3
  double* alpha0;           // nv
  int* kacc;                // nv
  // line search
  int line_search;
  int max_halvings;
  unsigned long long* ls_max;
  int* ls_cnt;
  // contact (pair table at the sweep-start x)
  int npairs;
  const double* x;
  const double* pairs;      // rows of kPairRow
  const double* pair_g;     // 12 per pair
  const double* pair_h;     // 144 per pair (PSD projected)
  const int* vp_ptr;        // vertex -> (pair*4 + member slot), ascending pair
  const int* vp_list;
  const double* planes;     // (point, normal) per plane
  const int* vr_ptr;        // retained rows CSR (keys ascending)
  const int* vr_keys;
  const double* vr_rows;
};

// Coupling rows of a triangle pair for sub-problem v at member slot s
// (local_solver.py:85-112; corotated_cubature mode, rows (12 x 3) as 4
// blocks). blk[c] = 3x3 block of DOF slot c.
__device__ void pair_rows_tri(const LocalArgs& a, int v, const double* row, int s, double blk[4][9]) {
  for (int c = 0; c < 4; ++c)
    for (int i = 0; i < 9; ++i) blk[c][i] = 0.0;
  const double* bary = row + 7;
  if (s == 0) {
    for (int i = 0; i < 3; ++i) blk[0][4 * i] = 1.0;
    for (int c = 0; c < 3; ++c)
      for (int i = 0; i < 3; ++i) blk[1 + c][4 * i] = bary[c];
    return;
  }
  int j = s - 1;
  for (int i = 0; i < 3; ++i) { blk[1 + j][4 * i] = 1.0; blk[0][4 * i] = bary[j]; }
  const double* Ri = a.R + 9 * (size_t)v;
  int k0 = a.vr_ptr[v], k1 = a.vr_ptr[v + 1];
  for (int c = 0; c < 3; ++c) {
    if (c == j) continue;
    int w = (int)row[2 + c];
    int lo = k0, hi = k1;  // binary search in ascending keys
    while (lo < hi) { int mid = (lo + hi) >> 1; if (a.vr_keys[mid] < w) lo = mid + 1; else hi = mid; }
    if (lo < k1 && a.vr_keys[lo] == w) {
      double t[9];
      mat3_mul(a.R + 9 * (size_t)w, a.vr_rows + 9 * (size_t)lo, t);
      mat3_mul_bt(t, Ri, blk[1 + c]);
    }
  }
}

// A += rows^T hp rows; g += rows^T gp - own gp for every pair touching v
// (local_solver.py:418-447, own_in_field=False).
__device__ void add_pair_terms(const LocalArgs& a, int v, double* A, double* g) {
  for (int q = a.vp_ptr[v]; q < a.vp_ptr[v + 1]; ++q) {
    int k = a.vp_list[q] >> 2, s = a.vp_list[q] & 3;
    const double* row = a.pairs + (size_t)kPairRow * k;
    const double* gp = a.pair_g + 12 * (size_t)k;
    const double* H = a.pair_h + 144 * (size_t)k;
    if (row[0] == 0.0) {  // plane: rows = I; projected force equals own force
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) A[3 * i + j] += H[12 * i + j];
      continue;
    }
    double blk[4][9];
    pair_rows_tri(a, v, row, s, blk);
    // HR = H rows (12 x 3)
    double HR[36];
    for (int i = 0; i < 12; ++i)
      for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int m = 0; m < 4; ++m)
          for (int r = 0; r < 3; ++r) acc += H[12 * i + 3 * m + r] * blk[m][3 * r + c];
        HR[3 * i + c] = acc;
      }
    for (int c = 0; c < 3; ++c) {
      for (int d = 0; d < 3; ++d) {
        double acc = 0.0;
        for (int m = 0; m < 4; ++m)
          for (int r = 0; r < 3; ++r) acc += blk[m][3 * r + c] * HR[3 * (3 * m + r) + d];
        A[3 * c + d] += acc;
      }
      double pr = 0.0;
      for (int m = 0; m < 4; ++m)
        for (int r = 0; r < 3; ++r) pr += blk[m][3 * r + c] * gp[3 * m + r];
      g[c] += pr - gp[3 * s + c];
    }
  }
}

// Per-vertex step cap over its pairs (local_solver.py:450-470).
__device__ double alpha_cap(const LocalArgs& a, int v, const double* d) {
  double alpha = 1.0;
  double dn = norm3_np(d);
  for (int q = a.vp_ptr[v]; q < a.vp_ptr[v + 1]; ++q) {
    int k = a.vp_list[q] >> 2;
    const double* row = a.pairs + (size_t)kPairRow * k;
    double dist, rate;
    if (row[0] == 0.0) {
      const double* pl = a.planes + 6 * (int)row[5];
      dist = plane_dist(a.x + 3 * (int)row[1], pl);
      double dn_ = __dadd_rn(__dadd_rn(__dmul_rn(d[0], pl[3]), __dmul_rn(d[1], pl[4])), __dmul_rn(d[2], pl[5]));
      rate = fmax(-dn_, 0.0);
    } else {
      double bary[3];
      dist = closest_point_tri(a.x + 3 * (int)row[1], a.x + 3 * (int)row[2], a.x + 3 * (int)row[3],
                               a.x + 3 * (int)row[4], bary);
      rate = 2.0 * dn;
    }
    if (rate > 0) alpha = fmin(alpha, 0.9 * dist / rate);
  }
  return fmin(alpha, 1.0);
}

// Sum_s w_s B_s^T Hcur_s B_s with B_s = blockdiag(R_w) V_s (rows before the
// R_i conjugation).  rows^T (R_blk H_rest R_blk^T) rows = R_i V^T H_rest V R_i^T
// because R_w^T R_w = I, so the rest part is the precomputed C_v.
// One cubature slot: E = sum_k Had(k,:) (x) R_{w_k} rows_k, X += w E^T M+ E.
__device__ __forceinline__ void sampled_slot(const LocalArgs& a, int v, int s, int u, double w, int4 cv,
                                             double* X) {
  const double* rows = a.cub_rows + (size_t)s * 36 * a.nv + v;  // rows[q * nv]
  const double* M = a.mplus + 45 * (size_t)u;
  double E[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) E[i] = 0.0;
  int corner[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double Bk[9], rk[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) rk[q] = __ldg(rows + (size_t)(9 * k + q) * a.nv);
    mat3_mul(a.R + 9 * (size_t)corner[k], rk, Bk);
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      double hw = kHad(k, p);
#pragma unroll
      for (int i = 0; i < 9; ++i) E[9 * p + i] += hw * Bk[i];  // E[(p r), c] = E[9p + 3r + c]
    }
  }
  double T1[27];  // M E
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      double mij = __ldg(M + tri9(i, j));
      t0 += mij * E[3 * j]; t1 += mij * E[3 * j + 1]; t2 += mij * E[3 * j + 2];
    }
    T1[3 * i] = t0; T1[3 * i + 1] = t1; T1[3 * i + 2] = t2;
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      double k = 0.0;
#pragma unroll
      for (int i = 0; i < 9; ++i) k += E[3 * i + c] * T1[3 * i + d];
      X[3 * c + d] += w * k;
    }
}

// The per-slot indices (unique element, corners) of every slot are
// loaded up front, so the dependent M+/R gathers of all slots start after
// one memory round trip instead of one per slot (ncu: k_local was
// long-scoreboard bound). Slot order and arithmetic are unchanged.
constexpr int kSlotsHoisted = 8;
__device__ void sampled_inner(const DevModel& m, const LocalArgs& a, int v, double* X) {
#pragma unroll
  for (int i = 0; i < 9; ++i) X[i] = 0.0;
  if (m.smax <= kSlotsHoisted) {
    int us[kSlotsHoisted];
    int4 cvs[kSlotsHoisted];
#pragma unroll
    for (int s = 0; s < kSlotsHoisted; ++s) {
      us[s] = -1;
      if (s < m.smax) {
        size_t vs = (size_t)s * a.nv + v;
        us[s] = __ldg(a.cub_u + vs);
        cvs[s] = __ldg(a.cub_verts + vs);
      }
    }
#pragma unroll 1
    for (int s = 0; s < m.smax; ++s)
      if (us[s] >= 0) sampled_slot(a, v, s, us[s], __ldg(a.cub_w + (size_t)s * a.nv + v), cvs[s], X);
    return;
  }
  for (int s = 0; s < m.smax; ++s) {
    size_t vs = (size_t)s * a.nv + v;
    int u = a.cub_u[vs];
    if (u < 0) continue;
    sampled_slot(a, v, s, u, a.cub_w[vs], a.cub_verts[vs], X);
  }
}

// Everything after the sampled sum S of one vertex (local_solver.py:392-553).
__device__ __forceinline__ void local_tail(const DevModel& m, const LocalArgs& a, int v, const double* S) {
  const double* Ri = a.R + 9 * (size_t)v;
  double X[9], A[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) X[k] = S[k] - a.crest[9 * (size_t)v + k];
  if (a.corr_out) {
    double Cc[9];
    mat3_conj(Ri, X, Cc);
#pragma unroll
    for (int k = 0; k < 9; ++k) a.corr_out[9 * (size_t)v + k] = Cc[k];
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) X[k] -= a.gbar[9 * (size_t)v + k];
  mat3_conj(Ri, X, A);
  // symmetrize (local_solver.py:408)
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = r + 1; c < 3; ++c) {
      double s = 0.5 * (A[3 * r + c] + A[3 * c + r]);
      A[3 * r + c] = A[3 * c + r] = s;
    }
  double wmin = sym3_min_eig(A);
  if (wmin <= 0.0) {  // SPD floor (local_solver.py:409-414)
    double sh = 1e-9 * (m.mass[v] / (a.h * a.h)) - wmin;
    A[0] += sh; A[4] += sh; A[8] += sh;
  }
  // g = -R_i sum_k gbar_rows[:, 3k:3k+3] q[group_k] (local_solver.py:402-403)
  double gr[3] = {0.0, 0.0, 0.0};
  const double* GR = a.grows + 9 * (size_t)m.gmax * v;
  for (int k = 0; k < m.gmax; ++k) {
    int w = a.group[(size_t)m.gmax * v + k];
    if (w < 0) continue;
    double q[3];
    q_of(m, a.b, w, q);
#pragma unroll
    for (int r = 0; r < 3; ++r)
      gr[r] += GR[3 * m.gmax * r + 3 * k] * q[0] + GR[3 * m.gmax * r + 3 * k + 1] * q[1] +
               GR[3 * m.gmax * r + 3 * k + 2] * q[2];
  }
  double g[3];
  mat3_vec(Ri, gr, g);
  g[0] = -g[0]; g[1] = -g[1]; g[2] = -g[2];
  if (a.npairs > 0) add_pair_terms(a, v, A, g);
  if (a.A_out) {
#pragma unroll
    for (int k = 0; k < 9; ++k) a.A_out[9 * (size_t)v + k] = A[k];
  }
  if (a.g_out) {
#pragma unroll
    for (int k = 0; k < 3; ++k) a.g_out[3 * (size_t)v + k] = g[k];
  }
  // delta = A^-1 (-g) (local_solver.py:580-588 / 72-82)
  double rhs[3] = {-g[0], -g[1], -g[2]}, d[3];
  if (!solve3_lu(A, rhs, d)) {
    double tr = A[0] + A[4] + A[8];
    if (tr > 0) { d[0] = rhs[0] * (3.0 / tr); d[1] = rhs[1] * (3.0 / tr); d[2] = rhs[2] * (3.0 / tr); }
    else d[0] = d[1] = d[2] = 0.0;
  }
  a.delta[3 * v] = d[0]; a.delta[3 * v + 1] = d[1]; a.delta[3 * v + 2] = d[2];
  // local line search on the quadratic model (local_solver.py:523-553)
  double al0 = 1.0;
  int kv = 0;
  if (a.line_search) {
    if (a.npairs > 0) al0 = alpha_cap(a, v, d);
    double Ad[3];
    int acc_it = a.max_halvings + 1;
    double al = al0;
    for (int it = 0; it <= a.max_halvings; ++it) {
      double st[3] = {al * d[0], al * d[1], al * d[2]};
      mat3_vec(A, st, Ad);
      double mq = (st[0] * g[0] + st[1] * g[1] + st[2] * g[2]) +
                  0.5 * (st[0] * Ad[0] + st[1] * Ad[1] + st[2] * Ad[2]);
      if (mq <= 0.0) { acc_it = it; break; }
      al *= 0.5;
    }
    kv = acc_it;
    if (kv > 0) {
      int lim = min(kv, a.max_halvings + 1);
      for (int it = 0; it < lim; ++it) {
        atomicAdd(a.ls_cnt + it, 1);
        atomicMax(a.ls_max + it, (unsigned long long)__double_as_longlong(al0));
      }
    }
  }
  a.alpha0[v] = al0;
  a.kacc[v] = kv;
}

// One thread per free vertex (any number of cubature slots).
__global__ void __launch_bounds__(128, 4)
k_local(DevModel m, LocalArgs a) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.nfree) return;
  int v = m.free_list[i];
  double S[9];
  sampled_inner(m, a, v, S);
  local_tail(m, a, v, S);
}

// Global part of the local line search: loop exit iteration and floor flag
// (local_solver.py:539-552). Single thread.
__global__ void k_ls_final(int max_halvings, double alpha_floor, const int* cnt,
                           const unsigned long long* mx, int* out) {
  int T = -1, fl = 0;
  double scale = 1.0;
  for (int it = 0; it <= max_halvings; ++it) {
    if (cnt[it] == 0) { T = it; break; }
    scale *= 0.5;
    double m = __longlong_as_double((long long)mx[it]) * scale;
    if (m < alpha_floor) { T = it; fl = 1; break; }
  }
  if (T < 0) T = max_halvings;
  out[0] = T;
  out[1] = fl;
  out[2] = cnt[0];
}

// Final local step fraction of one vertex (local_solver.py:539-553): the
// vertex accepted at halving kv <= T keeps alpha0 2^-kv; vertices still
// unaccepted after the last halving T take the floor (or 2^-(max+1)).
__device__ __forceinline__ double final_alpha(double alpha0, int kv, const int* lsf, int max_halvings,
                                              double alpha_floor) {
  int T = lsf[0], fl = lsf[1];
  double al = alpha0;
  if (kv <= T) {
    for (int it = 0; it < kv; ++it) al *= 0.5;
  } else if (fl) {
    al = alpha_floor;
  } else {
    for (int it = 0; it <= max_halvings; ++it) al *= 0.5;
  }
  return al;
}

// dx = alpha * delta for free vertices (local_solver.py:604, 622-624).
__global__ void __launch_bounds__(kBlock)
k_apply_alpha(DevModel m, const double* delta, const double* alpha0, const int* kacc,
              const int* lsf, int line_search, int max_halvings, double alpha_floor, double* dx) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= m.nv) return;
  if (m.fixed[v] || m.pos[v] < 0) {
    dx[3 * v] = dx[3 * v + 1] = dx[3 * v + 2] = 0.0;
    return;
  }
  double al = line_search ? final_alpha(alpha0[v], kacc[v], lsf, max_halvings, alpha_floor) : 1.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) dx[3 * v + c] = al * delta[3 * v + c];
}

// Per-vertex step fractions of the local search (parity entry point):
// alpha[v] for free vertices, 1 elsewhere.
__global__ void __launch_bounds__(kBlock)
k_alpha_out(DevModel m, const double* alpha0, const int* kacc, const int* lsf, int line_search,
            int max_halvings, double alpha_floor, double* alpha) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= m.nv) return;
  alpha[v] = (m.fixed[v] || m.pos[v] < 0 || !line_search)
                 ? 1.0 : final_alpha(alpha0[v], kacc[v], lsf, max_halvings, alpha_floor);
}

// Incremental potential at x0 + gamma*dx (assembly.py:183-192). Elastic
// per element and inertia per vertex in one grid-stride pass; barrier
// energies of the active pairs are added by the contact path.
__global__ void __launch_bounds__(kBlock)
k_energy(DevModel m, const double* __restrict__ x0, const double* __restrict__ dx, double gamma,
         const double* __restrict__ z, double h, double* partials, unsigned* counter, double* out) {
  double acc = 0.0;
  int n = max(m.ne, m.nv);
  double inv2h2 = 0.5 / (h * h);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (i < m.ne) {
      int4 t = __ldg(m.tets + i);
      int cs[4] = {t.x, t.y, t.z, t.w};
      double xs[4][3];
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double xv = __ldg(x0 + 3 * cs[k] + c);
          xs[k][c] = dx ? __dadd_rn(xv, __dmul_rn(gamma, __ldg(dx + 3 * cs[k] + c))) : xv;
        }
      double D[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) D[q] = __ldg(m.dminv + 9 * (size_t)i + q);
      double4 ep = m.eprops[i];
      double F[9];
      deformation_gradient(xs[0], xs[1], xs[2], xs[3], D, F);
      acc += ep.x * snh_psi(F, snh_const(ep.y, ep.z));
    }
    if (i < m.nv) {
      double dd = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double xv = __ldg(x0 + 3 * i + c);
        if (dx) xv = __dadd_rn(xv, __dmul_rn(gamma, __ldg(dx + 3 * i + c)));
        double df = xv - z[3 * i + c];
        dd += df * df;
      }
      acc += m.mass[i] * dd * inv2h2;
    }
  }
  grid_reduce<OP_SUM>(acc, partials, counter, out);
}

// x <- x + gamma*dx, dx <- gamma*dx; |dx|^2 and max_v |dx_v| reductions
// (local_solver.py:576-577, 654; assembly.py:118-120).
__global__ void __launch_bounds__(kBlock)
k_finalize(int nv, double* x, double* dx, double gamma, int scale_dx, double* partials,
           unsigned* counters, double* res) {
  double s2 = 0.0, mx = 0.0;
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    double d[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      d[c] = scale_dx ? __dmul_rn(gamma, dx[3 * v + c]) : dx[3 * v + c];
      x[3 * v + c] = __dadd_rn(x[3 * v + c], d[c]);
      dx[3 * v + c] = d[c];
    }
    s2 += d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    mx = fmax(mx, norm3_np(d));
  }
  grid_reduce<OP_SUM>(s2, partials, counters, res + R_DX2);
  grid_reduce<OP_MAX>(mx, partials + kMaxPartials, counters + 1, res + R_DXMAX);
}

// C_v = sum_s w_s V_s^T H_rest V_s (rest constant of the correction).
__global__ void __launch_bounds__(kBlock)
k_rest_constant(DevModel m, LocalArgs a, double* crest) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.nfree) return;
  int v = m.free_list[i];
  double X[9];
  sampled_inner(m, a, v, X);  // with R = identity rotations and rest mplus
#pragma unroll
  for (int k = 0; k < 9; ++k) crest[9 * (size_t)v + k] = X[k];
}

__global__ void k_fill_identity(int nv, double* R) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
#pragma unroll
  for (int i = 0; i < 9; ++i) R[9 * (size_t)v + i] = (i % 4 == 0) ? 1.0 : 0.0;
}

}  // namespace jgs2
