// IPC barrier path of the JGS2 sweep.
// Reference: contact.py:142-284 (distances, derivatives, pair energies),
// contact.py:162-240 (closest points + active-set detection),
// assembly.py:263-291 (feasibility cap), local_solver.py:85-112, 418-470
// (pair coupling rows, pair terms, alpha caps), energy.py:205-221 (barrier).
//
// Pair detection reproduces the reference's rounding order so the active
// set is bit-exact: 3-term dots as (p0+p2)+p1 without FMA,
// norms as sqrt((x^2+y^2)+z^2), region tests in the reference's order.
#pragma once
#include <chrono>
#include <cstdio>
#include "context.cuh"
#include "sweep.cuh"
#include "geometry.cuh"
#include "broadphase.cuh"
#include "element_hessian.cuh"

namespace jgs2 {

struct ContactDev {
  int nsv, nst, nplanes;
  double dhat, kappa;
  const int* sv;
  const int* st;
  const int* vbody;
  const int* tbody;
  const double* planes;  // (point, normal) x nplanes
};

// Pass 1: per surface vertex, counts of plane hits (per plane) and
// cross-body triangle hits (grid candidates, ascending triangle id).
__global__ void k_pair_count(ContactDev cd, TriGridDev g, int use_grid, const double* x, const double* dx,
                             double gamma, int* cnt /* (nplanes+1) x nsv */) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cd.nsv) return;
  int v = cd.sv[i];
  double p[3];
  load_pos(x, dx, gamma, v, p);
  for (int pl = 0; pl < cd.nplanes; ++pl)
    cnt[pl * cd.nsv + i] = (plane_dist(p, cd.planes + 6 * pl) < cd.dhat) ? 1 : 0;
  int hits = 0;
  int bv = cd.vbody[v];
  auto test = [&](int t) {
    double a[3], b[3], c[3], bary[3];
    load_pos(x, dx, gamma, cd.st[3 * t], a);
    load_pos(x, dx, gamma, cd.st[3 * t + 1], b);
    load_pos(x, dx, gamma, cd.st[3 * t + 2], c);
    if (closest_point_tri(p, a, b, c, bary) < cd.dhat) ++hits;
  };
  if (use_grid) {
    long long q0, q1;
    grid_range(g, point_key(g, p), &q0, &q1);
    visit_cross(q0, q1, bv, [&](long long q) { return cd.tbody[g.tris[q]]; },
                [&](long long q) { test(g.tris[q]); });
  } else {
    for (int t = 0; t < cd.nst; ++t)
      if (cd.tbody[t] != bv) test(t);
  }
  cnt[cd.nplanes * cd.nsv + i] = hits;
}

// Pass 2: write pair rows in the reference order (contact.py:224-239).
__global__ void k_pair_write(ContactDev cd, TriGridDev g, int use_grid, const double* x, const double* dx,
                             double gamma, const int* off, int cap, double* rows, int* flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cd.nsv) return;
  int v = cd.sv[i];
  double p[3];
  load_pos(x, dx, gamma, v, p);
  for (int pl = 0; pl < cd.nplanes; ++pl) {
    double d = plane_dist(p, cd.planes + 6 * pl);
    if (d < cd.dhat) {
      int o = off[pl * cd.nsv + i];
      if (o < cap) {
        double* r = rows + (size_t)kPairRow * o;
        r[0] = 0; r[1] = v; r[2] = r[3] = r[4] = 0; r[5] = pl; r[6] = d; r[7] = r[8] = r[9] = 0.0;
      }
      if (d <= 0.0) atomicOr(flag, 1);
    }
  }
  int o = off[cd.nplanes * cd.nsv + i];
  int bv = cd.vbody[v];
  auto emit = [&](int t) {
    double a[3], b[3], c[3], bary[3];
    load_pos(x, dx, gamma, cd.st[3 * t], a);
    load_pos(x, dx, gamma, cd.st[3 * t + 1], b);
    load_pos(x, dx, gamma, cd.st[3 * t + 2], c);
    double d = closest_point_tri(p, a, b, c, bary);
    if (d < cd.dhat) {
      if (o < cap) {
        double* r = rows + (size_t)kPairRow * o;
        r[0] = 1; r[1] = v; r[2] = cd.st[3 * t]; r[3] = cd.st[3 * t + 1]; r[4] = cd.st[3 * t + 2];
        r[5] = -1; r[6] = d; r[7] = bary[0]; r[8] = bary[1]; r[9] = bary[2];
      }
      if (d <= 0.0) atomicOr(flag, 1);
      ++o;
    }
  };
  if (use_grid) {
    long long q0, q1;
    grid_range(g, point_key(g, p), &q0, &q1);
    visit_cross(q0, q1, bv, [&](long long q) { return cd.tbody[g.tris[q]]; },
                [&](long long q) { emit(g.tris[q]); });
  } else {
    for (int t = 0; t < cd.nst; ++t)
      if (cd.tbody[t] != bv) emit(t);
  }
}

// ------------------------------------------------ barrier + distance derivatives
struct Barrier { double b, db, ddb; };
// energy.py:205-221 (d <= 0 handled by the caller's feasibility flag)
__device__ __forceinline__ Barrier barrier_fn(double d, double dhat, double kappa) {
  Barrier r{0.0, 0.0, 0.0};
  if (!(d > 0.0) || d >= dhat) return r;
  double gap = d - dhat;
  double ln = log(d / dhat);
  r.b = -kappa * gap * gap * ln;
  r.db = -kappa * (2.0 * gap * ln + gap * gap / d);
  r.ddb = -kappa * (2.0 * ln + 4.0 * gap / d - gap * gap / (d * d));
  return r;
}

__device__ __forceinline__ void skew3(const double* v, double* S) {
  S[0] = 0.0; S[1] = -v[2]; S[2] = v[1];
  S[3] = v[2]; S[4] = 0.0; S[5] = -v[0];
  S[6] = -v[1]; S[7] = v[0]; S[8] = 0.0;
}

// Distance derivatives w.r.t. the 12 stencil DOFs (x, a, b, c) for a
// triangle pair with frozen region (contact.py:51-159). g[12], H[144].
__device__ double tri_pair_derivs(const double* X, const double* bary, double* g, double* H) {
  for (int i = 0; i < 12; ++i) g[i] = 0.0;
  for (int i = 0; i < 144; ++i) H[i] = 0.0;
  int nz[3], cntnz = 0;
  for (int k = 0; k < 3; ++k)
    if (bary[k] != 0.0) nz[cntnz++] = k;
  const double* x = X;
  if (cntnz == 1) {  // point-point (contact.py:51-59)
    int s = 1 + nz[0];
    const double* y = X + 3 * s;
    double r[3] = {x[0] - y[0], x[1] - y[1], x[2] - y[2]};
    double d = norm3_np(r);
    double u[3] = {r[0] / d, r[1] / d, r[2] / d};
    for (int i = 0; i < 3; ++i) { g[i] = u[i]; g[3 * s + i] = -u[i]; }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double k = ((i == j ? 1.0 : 0.0) - u[i] * u[j]) / d;
        H[12 * i + j] = k;
        H[12 * i + 3 * s + j] = -k;
        H[12 * (3 * s + i) + j] = -k;
        H[12 * (3 * s + i) + 3 * s + j] = k;
      }
    return d;
  }
  if (cntnz == 2) {  // point-edge (contact.py:62-92), slots (0, 1+nz0, 1+nz1)
    int sa = 1 + nz[0], sb = 1 + nz[1];
    const double* a = X + 3 * sa;
    const double* b = X + 3 * sb;
    double w[3] = {x[0] - a[0], x[1] - a[1], x[2] - a[2]};
    double e[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
    double m[3];
    cross3(w, e, m);
    double r = norm3_np(m), el = norm3_np(e);
    double d = r / el;
    double mh[3] = {m[0] / r, m[1] / r, m[2] / r};
    // sub-stencil DOFs (9): [x(0..2), a(3..5), b(6..8)]
    double jw[27] = {0}, je[27] = {0}, jm[27];
    for (int i = 0; i < 3; ++i) {
      jw[9 * i + i] = 1.0; jw[9 * i + 3 + i] = -1.0;
      je[9 * i + 3 + i] = -1.0; je[9 * i + 6 + i] = 1.0;
    }
    double Se[9], Sw[9];
    skew3(e, Se); skew3(w, Sw);
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 9; ++k) {
        double s = 0.0;
        for (int j = 0; j < 3; ++j) s += -Se[3 * i + j] * jw[9 * j + k] + Sw[3 * i + j] * je[9 * j + k];
        jm[9 * i + k] = s;
      }
    double gm[3] = {mh[0] / el, mh[1] / el, mh[2] / el};
    double el3 = el * el * el;
    double ge[3] = {-(r / el3) * e[0], -(r / el3) * e[1], -(r / el3) * e[2]};
    double gs[9];
    for (int k = 0; k < 9; ++k) {
      double s = 0.0;
      for (int i = 0; i < 3; ++i) s += jm[9 * i + k] * gm[i] + je[9 * i + k] * ge[i];
      gs[k] = s;
    }
    double bmm[9], bme[9], bee[9];
    double el5 = el3 * el * el;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double I = (i == j) ? 1.0 : 0.0;
        bmm[3 * i + j] = (I - mh[i] * mh[j]) / (r * el);
        bme[3 * i + j] = -mh[i] * e[j] / el3;
        bee[3 * i + j] = r * (3.0 * e[i] * e[j] / el5 - I / el3);
      }
    double Sg[9];
    skew3(gm, Sg);
    double hs[81];
    for (int k = 0; k < 9; ++k)
      for (int l = 0; l < 9; ++l) {
        double s = 0.0;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            s += jm[9 * i + k] * bmm[3 * i + j] * jm[9 * j + l];
            s += jm[9 * i + k] * bme[3 * i + j] * je[9 * j + l];
            s += je[9 * i + k] * bme[3 * j + i] * jm[9 * j + l];
            s += je[9 * i + k] * bee[3 * i + j] * je[9 * j + l];
            s += jw[9 * i + k] * (-Sg[3 * i + j]) * je[9 * j + l];
            s += je[9 * i + k] * Sg[3 * i + j] * jw[9 * j + l];
          }
        hs[9 * k + l] = s;
      }
    int slots[3] = {0, sa, sb};
    for (int bi = 0; bi < 3; ++bi)
      for (int r2 = 0; r2 < 3; ++r2) {
        g[3 * slots[bi] + r2] = gs[3 * bi + r2];
        for (int bj = 0; bj < 3; ++bj)
          for (int c2 = 0; c2 < 3; ++c2)
            H[12 * (3 * slots[bi] + r2) + 3 * slots[bj] + c2] = hs[9 * (3 * bi + r2) + 3 * bj + c2];
      }
    return d;
  }
  // point-face (contact.py:95-127)
  const double* a = X + 3;
  const double* b = X + 6;
  const double* c = X + 9;
  double w[3] = {x[0] - a[0], x[1] - a[1], x[2] - a[2]};
  double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  double n[3];
  cross3(u, v, n);
  double ln = norm3_np(n);
  double nh[3] = {n[0] / ln, n[1] / ln, n[2] / ln};
  double s = w[0] * nh[0] + w[1] * nh[1] + w[2] * nh[2];
  double jw[36] = {0}, ju[36] = {0}, jv[36] = {0}, jn[36];
  for (int i = 0; i < 3; ++i) {
    jw[12 * i + i] = 1.0; jw[12 * i + 3 + i] = -1.0;
    ju[12 * i + 3 + i] = -1.0; ju[12 * i + 6 + i] = 1.0;
    jv[12 * i + 3 + i] = -1.0; jv[12 * i + 9 + i] = 1.0;
  }
  double Sv[9], Su[9];
  skew3(v, Sv); skew3(u, Su);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 12; ++k) {
      double t = 0.0;
      for (int j = 0; j < 3; ++j) t += -Sv[3 * i + j] * ju[12 * j + k] + Su[3 * i + j] * jv[12 * j + k];
      jn[12 * i + k] = t;
    }
  double gn[3] = {(w[0] - s * nh[0]) / ln, (w[1] - s * nh[1]) / ln, (w[2] - s * nh[2]) / ln};
  for (int k = 0; k < 12; ++k) {
    double t = 0.0;
    for (int i = 0; i < 3; ++i) t += jw[12 * i + k] * nh[i] + jn[12 * i + k] * gn[i];
    g[k] = t;
  }
  double pn[9], bnn[9];
  double ln2 = ln * ln;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double I = (i == j) ? 1.0 : 0.0;
      pn[3 * i + j] = (I - nh[i] * nh[j]) / ln;
      bnn[3 * i + j] = (-w[i] * nh[j] - nh[i] * w[j] - s * I + 3.0 * s * nh[i] * nh[j]) / ln2;
    }
  double Sg[9];
  skew3(gn, Sg);
  for (int k = 0; k < 12; ++k)
    for (int l = 0; l < 12; ++l) {
      double t = 0.0;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          t += jw[12 * i + k] * pn[3 * i + j] * jn[12 * j + l];
          t += jn[12 * i + k] * pn[3 * i + j] * jw[12 * j + l];
          t += jn[12 * i + k] * bnn[3 * i + j] * jn[12 * j + l];
          t += ju[12 * i + k] * (-Sg[3 * i + j]) * jv[12 * j + l];
          t += jv[12 * i + k] * Sg[3 * i + j] * ju[12 * j + l];
        }
      H[12 * k + l] = t;
    }
  double sign = (s >= 0.0) ? 1.0 : -1.0;
  for (int k = 0; k < 12; ++k) g[k] *= sign;
  for (int k = 0; k < 144; ++k) H[k] *= sign;
  return fabs(s);
}

// Per pair: barrier energy, stencil gradient and PSD-projected Hessian
// (contact.py:254-263 with project_spd=True). A vertex-triangle distance is
// translation invariant, so its 12x12 barrier Hessian lives in the 9-dim
// complement of the 3 translations: with the orthonormal basis
// U = [h_m (x) e_c], h = (1,1,-1,-1)/2, (1,-1,1,-1)/2, (1,-1,-1,1)/2 over the
// stencil (x, a, b, c), M = U^T H U (9x9) is projected (same tred2/tql2 as the
// element Hessians) and H+ = U M+ U^T; the translation eigenvalues are 0 and
// stay 0 under the reference's 12x12 eigh clamp.
constexpr int kPairThreads = 64;
__device__ __forceinline__ double hsign(int m, int p) {  // h_m[p] * 2
  // m = 0: (1,1,-1,-1), 1: (1,-1,1,-1), 2: (1,-1,-1,1)
  int b = m == 0 ? (p >> 1) : (m == 1 ? (p & 1) : ((p >> 1) ^ (p & 1)));
  return b ? -1.0 : 1.0;
}

__global__ void __launch_bounds__(kPairThreads)
k_pair_terms(int npairs, const double* rows, const double* x, const double* planes, double dhat, double kappa,
             double* pg, double* ph, double* pe) {
  extern __shared__ double psm[];
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= npairs) return;
  const double* r = rows + (size_t)kPairRow * k;
  double* g = pg + 12 * (size_t)k;
  double* H = ph + 144 * (size_t)k;
  if (r[0] == 0.0) {  // plane: d = (x - p).n, grad n, hess 0
    const double* pl = planes + 6 * (int)r[5];
    int v = (int)r[1];
    double d = plane_dist(x + 3 * v, pl);
    Barrier B = barrier_fn(d, dhat, kappa);
    for (int i = 0; i < 12; ++i) g[i] = 0.0;
    for (int i = 0; i < 144; ++i) H[i] = 0.0;
    double h3[9];
    for (int i = 0; i < 3; ++i) {
      g[i] = B.db * pl[3 + i];
      for (int j = 0; j < 3; ++j) h3[3 * i + j] = B.ddb * pl[3 + i] * pl[3 + j];
    }
    double V[9];
    double a[9];
    for (int i = 0; i < 9; ++i) a[i] = h3[i];
    jacobi_eig<3>(a, V, 30);
    double lam[3] = {fmax(a[0], 0.0), fmax(a[4], 0.0), fmax(a[8], 0.0)};
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;
        for (int q = 0; q < 3; ++q) s += V[3 * i + q] * lam[q] * V[3 * j + q];
        H[12 * i + j] = s;
      }
    pe[k] = B.b;
    return;
  }
  double X[12];
  for (int s = 0; s < 4; ++s) {
    int w = (int)r[1 + s];
    for (int c = 0; c < 3; ++c) X[3 * s + c] = x[3 * w + c];
  }
  double gd[12], Hd[144];
  double d = tri_pair_derivs(X, r + 7, gd, Hd);
  Barrier B = barrier_fn(d, dhat, kappa);
  for (int i = 0; i < 12; ++i) g[i] = B.db * gd[i];
  // complement coordinates: index q = 3 m + c
  double G[9];
  for (int m = 0; m < 3; ++m)
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int p = 0; p < 4; ++p) s += hsign(m, p) * gd[3 * p + c];
      G[3 * m + c] = 0.5 * s;
    }
  double* Vs = psm + threadIdx.x;
  for (int qi = 0; qi < 9; ++qi) {
    int mi = qi / 3, ci = qi % 3;
    for (int qj = 0; qj <= qi; ++qj) {
      int mj = qj / 3, cj = qj % 3;
      double s = 0.0;
      for (int p = 0; p < 4; ++p) {
        double hp = hsign(mi, p);
        for (int q = 0; q < 4; ++q)
          s += hp * hsign(mj, q) * 0.5 * (Hd[12 * (3 * p + ci) + 3 * q + cj] + Hd[12 * (3 * q + cj) + 3 * p + ci]);
      }
      double mij = B.ddb * G[qi] * G[qj] + B.db * (0.25 * s);
      Vs[(9 * qi + qj) * kPairThreads] = mij;
      Vs[(9 * qj + qi) * kPairThreads] = mij;
    }
  }
  double dg[9], od[9];
  sym_eig9_reg<kPairThreads>(Vs, dg, od);
  double lam[9];
  for (int q = 0; q < 9; ++q) lam[q] = fmax(dg[q], 0.0);
  // M+ = V lam V^T, then H+ = U M+ U^T
  double Mp[45];
  for (int i = 0; i < 9; ++i)
    for (int j = 0; j <= i; ++j) {
      double acc = 0.0;
      for (int q = 0; q < 9; ++q) acc += Vs[(9 * i + q) * kPairThreads] * lam[q] * Vs[(9 * j + q) * kPairThreads];
      Mp[JGS2_PK(i, j)] = acc;
    }
  for (int p = 0; p < 4; ++p)
    for (int ci = 0; ci < 3; ++ci)
      for (int q = 0; q < 4; ++q)
        for (int cj = 0; cj < 3; ++cj) {
          double s = 0.0;
          for (int mi = 0; mi < 3; ++mi)
            for (int mj = 0; mj < 3; ++mj) {
              int a = 3 * mi + ci, b = 3 * mj + cj;
              double mab = a >= b ? Mp[JGS2_PK(a, b)] : Mp[JGS2_PK(b, a)];
              s += hsign(mi, p) * hsign(mj, q) * mab;
            }
          H[12 * (3 * p + ci) + 3 * q + cj] = 0.25 * s;
        }
  pe[k] = B.b;
}

// Vertex -> pair incidence: counts (pass 1) and ordered fill (pass 2, one
// thread per vertex scanning the pair list: deterministic, pair order).
__global__ void k_vp_count(int npairs, const double* rows, int* cnt) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= npairs) return;
  const double* r = rows + (size_t)kPairRow * k;
  int nm = (r[0] == 0.0) ? 1 : 4;
  for (int s = 0; s < nm; ++s) atomicAdd(cnt + (int)r[1 + s], 1);
}
__global__ void k_vp_fill(int npairs, const double* rows, const int* ptr, int* fillpos, int* list) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= npairs) return;
  const double* r = rows + (size_t)kPairRow * k;
  int nm = (r[0] == 0.0) ? 1 : 4;
  for (int s = 0; s < nm; ++s) {
    int v = (int)r[1 + s];
    int slot = atomicAdd(fillpos + v, 1);
    list[ptr[v] + slot] = 4 * k + s;
  }
}
// sort each vertex's short list by pair id (deterministic order)
__global__ void k_vp_sort(int nv, const int* ptr, int* list) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  int a = ptr[v], b = ptr[v + 1];
  for (int i = a + 1; i < b; ++i) {
    int key = list[i], j = i - 1;
    while (j >= a && list[j] > key) { list[j + 1] = list[j]; --j; }
    list[j + 1] = key;
  }
}

// g_asm[v] += pair gradient blocks (ascending pair order) (local_solver.py:319-322)
__global__ void k_pair_grad_add(int nv, const int* ptr, const int* list, const double* pg, double* gasm) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  for (int q = ptr[v]; q < ptr[v + 1]; ++q) {
    int k = list[q] >> 2, s = list[q] & 3;
    for (int c = 0; c < 3; ++c) gasm[3 * v + c] += pg[12 * (size_t)k + 3 * s + c];
  }
}

// barrier energy sum over the pair table (deterministic tree) into res[slot] += ...
__global__ void k_pair_energy_sum(int npairs, const double* rows, double dhat, double kappa,
                                  double* partials, unsigned* counter, double* out) {
  double acc = 0.0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < npairs; k += gridDim.x * blockDim.x) {
    double d = rows[(size_t)kPairRow * k + 6];
    acc += barrier_fn(d, dhat, kappa).b;
  }
  grid_reduce<OP_SUM>(acc, partials, counter, out);
}
__global__ void k_add_scalar(double* dst, const double* src) { *dst += *src; }

// feasibility_step_cap (assembly.py:263-291): min over planes of d/rate
// (moving surface vertices) and over all cross-body (sv, tri) of
// dist / (|dx_v| + max |dx_tri|); returns 0.9 * min, capped at 1.
__global__ void k_cap_planes(ContactDev cd, const double* x, const double* dx, double* partials,
                             unsigned* counter, double* out) {
  double mn = INFINITY;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cd.nsv * max(cd.nplanes, 1);
       i += gridDim.x * blockDim.x) {
    if (cd.nplanes == 0) break;
    int pl = i / cd.nsv, j = i % cd.nsv;
    int v = cd.sv[j];
    const double* P = cd.planes + 6 * pl;
    double d = plane_dist(x + 3 * v, P);
    double rate = -__dadd_rn(__dadd_rn(__dmul_rn(dx[3 * v], P[3]), __dmul_rn(dx[3 * v + 1], P[4])),
                             __dmul_rn(dx[3 * v + 2], P[5]));
    if (rate > 0) mn = fmin(mn, d / rate);
  }
  grid_reduce<OP_MIN>(mn, partials, counter, out);
}
// max_v |dx_v| over surface vertices (query radius of the cap grid)
__global__ void k_sv_maxstep(ContactDev cd, const double* dx, double* partials, unsigned* counter,
                             double* out) {
  double mx = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cd.nsv; i += gridDim.x * blockDim.x)
    mx = fmax(mx, norm3_np(dx + 3 * cd.sv[i]));
  grid_reduce<OP_MAX>(mx, partials, counter, out);
}

// min over the active triangle pairs of the current pair table of d / rate
// (an upper bound source for the cap: these pairs are among all pairs)
__global__ void k_cap_pairtable(int npairs, const double* rows, const double* dx, double* partials,
                                unsigned* counter, double* out) {
  double mn = INFINITY;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < npairs; k += gridDim.x * blockDim.x) {
    const double* r = rows + (size_t)kPairRow * k;
    if (r[0] == 0.0) continue;
    double sp = norm3_np(dx + 3 * (int)r[1]);
    double stt = fmax(fmax(norm3_np(dx + 3 * (int)r[2]), norm3_np(dx + 3 * (int)r[3])),
                      norm3_np(dx + 3 * (int)r[4]));
    double rate = sp + stt;
    if (rate > 1e-30) mn = fmin(mn, r[6] / rate);
  }
  grid_reduce<OP_MIN>(mn, partials, counter, out);
}

// ------------------------------------------------------------------ host glue

inline ContactDev contactdev(const Ctx& C) {
  ContactDev cd;
  cd.nsv = C.nsv; cd.nst = C.nst; cd.nplanes = C.nplanes; cd.dhat = C.dhat; cd.kappa = C.kappa;
  cd.sv = C.sv; cd.st = C.st; cd.vbody = C.vbody; cd.tbody = C.tbody; cd.planes = C.planes;
  return cd;
}

void contact_setup(Ctx& C, const jgs2_model* md) {
  C.has_barrier = md->has_barrier != 0;
  if (!C.has_barrier) return;
  C.dhat = md->dhat;
  C.kappa = md->kappa;
  C.nplanes = (int)md->n_planes;
  C.nbodies = (int)std::max<int64_t>(md->n_bodies, 1);
  C.nsv = (int)md->n_surface_vertices;
  C.nst = (int)md->n_surface_tris;
  C.h_planes.assign(6 * (size_t)std::max(C.nplanes, 1), 0.0);
  for (int p = 0; p < C.nplanes; ++p)
    for (int c = 0; c < 3; ++c) {
      C.h_planes[6 * p + c] = md->plane_points[3 * p + c];
      C.h_planes[6 * p + 3 + c] = md->plane_normals[3 * p + c];
    }
  C.planes = C.upload(C.h_planes.data(), C.h_planes.size());
  std::vector<int> sv(C.nsv), st(3 * (size_t)C.nst), vb(C.nv), tb(C.nst);
  C.h_surface.assign(C.nv, 0);
  for (int i = 0; i < C.nsv; ++i) {
    sv[i] = (int)md->surface_vertices[i];
    if (sv[i] < 0 || sv[i] >= C.nv) throw Error(-1, "surface vertex out of range");
    C.h_surface[sv[i]] = 1;
  }
  for (size_t i = 0; i < st.size(); ++i) st[i] = (int)md->surface_tris[i];
  for (int i = 0; i < C.nv; ++i) vb[i] = md->vertex_body ? (int)md->vertex_body[i] : 0;
  for (int i = 0; i < C.nst; ++i) tb[i] = md->surface_tri_body ? (int)md->surface_tri_body[i] : 0;
  C.sv = C.upload(sv.data(), sv.size());
  C.st = C.upload(st.data(), st.size());
  C.vbody = C.upload(vb.data(), vb.size());
  C.tbody = C.upload(tb.data(), tb.size());
  C.pair_count_sv = C.alloc<int>((size_t)(C.nplanes + 1) * C.nsv + 1);
  C.vp_cnt = C.alloc<int>(C.nv + 1);
  C.pair_off_sv = C.alloc<int>((size_t)(C.nplanes + 1) * C.nsv + 1);
  C.vp_ptr = C.alloc<int>(C.nv + 1);
  C.flag_d = C.alloc<int>(2);
  C.npairs_d = C.alloc<int>(2);
  // grid cell: 2x the mean surface-triangle edge at rest, at least 2 dhat
  double el = 0.0;
  for (int t = 0; t < C.nst; ++t)
    for (int k = 0; k < 3; ++k) {
      int a = st[3 * t + k], b = st[3 * t + (k + 1) % 3];
      double d2 = 0.0;
      for (int c = 0; c < 3; ++c) {
        double dd = C.h_rest[3 * (size_t)a + c] - C.h_rest[3 * (size_t)b + c];
        d2 += dd * dd;
      }
      el += std::sqrt(d2);
    }
  el = C.nst > 0 ? el / (3.0 * C.nst) : 1.0;
  C.grid_cell = std::max(2.0 * el, 2.0 * C.dhat);
}

void ensure_pair_capacity(Ctx& C, int64_t need) {
  if (need <= C.cap_pairs) return;
  int64_t cap = std::max<int64_t>(need * 2, 1024);
  C.pairs = C.alloc<double>((size_t)cap * kPairRow);
  C.pair_g = C.alloc<double>((size_t)cap * 12);
  C.pair_h = C.alloc<double>((size_t)cap * 144);
  C.pair_e = C.alloc<double>((size_t)cap);
  C.vp_list = C.alloc<int>((size_t)cap * 4);
  C.cap_pairs = cap;
}

// exclusive scan of n ints into out[0..n] (out[n] = total), CUB device scan
void scan_ints(Ctx& C, int* in, int* out, int n) {
  JGS2_CUDA(cudaMemsetAsync(in + n, 0, sizeof(int), C.stream));
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n + 1, C.stream);
  if (tb > C.scan_temp_bytes) {
    C.scan_temp = C.alloc<char>(tb + tb / 2);
    C.scan_temp_bytes = tb + tb / 2;
  }
  JGS2_CUDA(cub::DeviceScan::ExclusiveSum(C.scan_temp, tb, in, out, n + 1, C.stream));
  ++C.launches;
}

bool use_tri_grid(const Ctx& C) { return C.nbodies > 1 && C.nst > 0; }

// Detect active pairs at x + gamma*dx into the pair table; sets C.npairs
// (host sync) and the infeasibility flag.
void contact_find_pairs(Ctx& C, const double* x, const double* dx, double gamma) {
  ContactDev cd = contactdev(C);
  int n = (C.nplanes + 1) * C.nsv;
  JGS2_CUDA(cudaMemsetAsync(C.flag_d, 0, sizeof(int), C.stream));
  int ug = use_tri_grid(C) ? 1 : 0;
  TriGridDev gd{nullptr, nullptr, 0, 1.0, 0, 0, 0, -1, -1, -1, 0, 0};
  static const bool dbg = getenv("JGS2_DEBUG_PAIRS") != nullptr;
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  auto t0 = clk::now();
  if (ug) {
    tri_grid_build(C, C.pair_grid, x, dx, gamma, C.dhat * (1.0 + 1e-6) + 1e-300, C.grid_cell);
    gd = grid_dev(C.pair_grid);
  } else {
    cd.nst = 0;  // single body: no cross-body triangle pairs
  }
  auto t1 = clk::now();
  k_pair_count<<<grid_for(C.nsv, 128), 128, 0, C.stream>>>(cd, gd, ug, x, dx, gamma, C.pair_count_sv);
  C.check_launch();
  scan_ints(C, C.pair_count_sv, C.pair_off_sv, n);
  int total = 0;
  JGS2_CUDA(cudaMemcpyAsync(&total, C.pair_off_sv + n, sizeof(int), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  auto t2 = clk::now();
  ensure_pair_capacity(C, total);
  auto t3 = clk::now();
  k_pair_write<<<grid_for(C.nsv, 128), 128, 0, C.stream>>>(cd, gd, ug, x, dx, gamma, C.pair_off_sv,
                                                           (int)C.cap_pairs, C.pairs, C.flag_d);
  C.check_launch();
  C.npairs = total;
  if (dbg && ms(t0, t3) > 20.0)
    fprintf(stderr, "find_pairs slow: grid %.2f ms (entries %lld) count+scan+sync %.2f ms alloc %.2f ms pairs %d\n",
            ms(t0, t1), C.pair_grid.n, ms(t1, t2), ms(t2, t3), total);
}

bool contact_infeasible(Ctx& C) {
  int f = 0;
  JGS2_CUDA(cudaMemcpyAsync(&f, C.flag_d, sizeof(int), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  return f != 0;
}

// barrier energy of the current pair table added to res[slot]
void contact_energy_at(Ctx& C, const double* dx, double gamma, int slot) {
  contact_find_pairs(C, C.x, dx, gamma);
  if (C.npairs == 0) return;
  int s2 = R_AUX;
  k_pair_energy_sum<<<std::min(grid_for(C.npairs), 64), kBlock, 0, C.stream>>>(
      C.npairs, C.pairs, C.dhat, C.kappa, C.partials + s2 * kMaxPartials, C.counters + s2, C.res + s2);
  C.check_launch();
  k_add_scalar<<<1, 1, 0, C.stream>>>(C.res + slot, C.res + s2);
  C.check_launch();
}

// Pair terms at the current x and vertex->pair incidence; adds pair
// gradients into g_asm.
void contact_add_gradients(Ctx& C) {
  if (C.npairs == 0) return;
  k_pair_terms<<<grid_for(C.npairs, kPairThreads), kPairThreads, 81 * kPairThreads * sizeof(double), C.stream>>>(
      C.npairs, C.pairs, C.x, C.planes, C.dhat, C.kappa, C.pair_g, C.pair_h, C.pair_e);
  C.check_launch();
  JGS2_CUDA(cudaMemsetAsync(C.vp_cnt, 0, (C.nv + 1) * sizeof(int), C.stream));
  k_vp_count<<<grid_for(C.npairs), kBlock, 0, C.stream>>>(C.npairs, C.pairs, C.vp_cnt);
  C.check_launch();
  scan_ints(C, C.vp_cnt, C.vp_ptr, C.nv);
  JGS2_CUDA(cudaMemsetAsync(C.vp_cnt, 0, (C.nv + 1) * sizeof(int), C.stream));
  k_vp_fill<<<grid_for(C.npairs), kBlock, 0, C.stream>>>(C.npairs, C.pairs, C.vp_ptr, C.vp_cnt, C.vp_list);
  C.check_launch();
  k_vp_sort<<<grid_for(C.nv), kBlock, 0, C.stream>>>(C.nv, C.vp_ptr, C.vp_list);
  C.check_launch();
  k_pair_grad_add<<<grid_for(C.nv), kBlock, 0, C.stream>>>(C.nv, C.vp_ptr, C.vp_list, C.pair_g, C.gasm);
  C.check_launch();
}

inline double hier_cap_min(Ctx& C, const double* x, const double* dx, double cap_ub, double smax,
                           const double* bb);
inline void hier_bbox_launch(Ctx& C, const double* x, double* out);

// feasibility_step_cap (assembly.py:263-291). pairs_at_x: the pair table
// holds the pairs detected at this x (their d equal the reference's
// closest-point distances bitwise) and gives an upper bound cap_ub; only
// pairs with dist < cap_ub (s_v + s_t) / 0.9 can lower it further, so the
// grid radii scale with cap_ub (exact). The plane, pair-table, max-step and
// bounding-box reductions share one host sync; bb_out (6 doubles, may be
// null) receives the surface bounding box at x for later grids.
double contact_step_cap(Ctx& C, const double* x, const double* dx, bool pairs_at_x = false,
                        double* bb_out = nullptr) {
  ContactDev cd = contactdev(C);
  bool tri = use_tri_grid(C);
  bool pt = tri && pairs_at_x && C.npairs > 0;
  if (!C.bbox_res) C.bbox_res = C.alloc<double>(6);
  if (C.nplanes > 0) {
    k_cap_planes<<<red_grid(C.nsv * C.nplanes), kBlock, 0, C.stream>>>(
        cd, x, dx, C.partials + R_CAP * kMaxPartials, C.counters + R_CAP, C.res + R_CAP);
    C.check_launch();
  }
  if (pt) {
    k_cap_pairtable<<<std::min(grid_for(C.npairs), 256), kBlock, 0, C.stream>>>(
        C.npairs, C.pairs, dx, C.partials + R_CAP2 * kMaxPartials, C.counters + R_CAP2, C.res + R_CAP2);
    C.check_launch();
  }
  if (tri) {
    k_sv_maxstep<<<red_grid(C.nsv), kBlock, 0, C.stream>>>(cd, dx, C.partials + R_AUX * kMaxPartials,
                                                           C.counters + R_AUX, C.res + R_AUX);
    C.check_launch();
    hier_bbox_launch(C, x, C.bbox_res);
  }
  double* h = C.h_res + 40;  // pinned scratch: res slots + bounding box
  JGS2_CUDA(cudaMemcpyAsync(h, C.res, R_NSLOTS * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  if (tri) JGS2_CUDA(cudaMemcpyAsync(h + R_NSLOTS, C.bbox_res, 6 * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  double cap = 1.0;
  if (C.nplanes > 0 && std::isfinite(h[R_CAP])) cap = std::min(cap, 0.9 * h[R_CAP]);
  if (pt && std::isfinite(h[R_CAP2])) cap = std::min(cap, 0.9 * h[R_CAP2]);
  if (tri) {
    if (bb_out) memcpy(bb_out, h + R_NSLOTS, 6 * sizeof(double));
    if (!(cap > 0)) return std::max(cap, 0.0);
    double m = hier_cap_min(C, x, dx, cap, h[R_AUX], h + R_NSLOTS);
    if (std::isfinite(m)) cap = std::min(cap, 0.9 * m);
  }
  return std::max(cap, 0.0);
}

}  // namespace jgs2
