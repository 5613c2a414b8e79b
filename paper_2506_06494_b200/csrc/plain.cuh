// Plain vertex block descent (subspace="none"): the reference's baseline
// mode, local_solver.py:325-353 (_plain_systems) and 472-522
// (_local_estimates, plain branch).
//
// Per free vertex: A = sum over incident elements of the own 3x3 block of the
// PSD-projected element Hessian (+ the element's quarter-mass inertia),
// g = g_asm[v] (+ each touching pair's own gradient: own_in_field=True,
// local_solver.py:352, 418-447 -- the assembled field already holds the pair
// force, which the reference adds a second time), delta = A^-1 (-g), the
// alpha caps, then the local search on the exact own-stencil energy: the
// incident elements' elastic + inertia energies with the vertex moved, plus
// the barrier energy of every pair touching it (FeasibilityError -> inf).
#pragma once
#include "contact.cuh"
#include "sweep.cuh"

namespace jgs2 {

struct PlainArgs {
  const double* mplus_all;  // 45 per element: projected reduced Hessian at x (element_hessian.cuh)
  const double* z;
  double dhat, kappa;
};

// own-stencil energy of vertex v with x_v <- x_v + step (rounded like the
// reference: pos[own] += step, step = alpha * delta)
__device__ double plain_energy(const DevModel& m, const LocalArgs& a, const PlainArgs& p, int v,
                               const double* step) {
  const double* x = a.x;
  double pv[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) pv[c] = __dadd_rn(x[3 * v + c], step[c]);
  const double ih2 = 1.0 / (a.h * a.h);
  double e = 0.0;
  int p0 = m.inc_ptr[v], p1 = m.inc_ptr[v + 1];
  for (int q = p0; q < p1; ++q) {
    int code = __ldg(m.inc + q), el = code >> 2, slot = code & 3;
    int4 t = __ldg(m.tets + el);
    int cs[4] = {t.x, t.y, t.z, t.w};
    double xs[4][3];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) xs[k][c] = (k == slot) ? pv[c] : x[3 * cs[k] + c];
    double D[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) D[i] = __ldg(m.dminv + 9 * (size_t)el + i);
    double F[9];
    deformation_gradient(xs[0], xs[1], xs[2], xs[3], D, F);
    double4 ep = m.eprops[el];
    double ee = ep.x * snh_psi(F, snh_const(ep.y, ep.z));
    double dd = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double df = xs[k][c] - p.z[3 * cs[k] + c];
        dd += df * df;
      }
    e += ee + 0.5 * ep.w * ih2 * dd;
  }
  if (p1 == p0) {  // isolated vertex: inertia only
    double dd = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double df = pv[c] - p.z[3 * v + c];
      dd += df * df;
    }
    e += 0.5 * m.mass[v] * ih2 * dd;
  }
  const int qb = a.npairs > 0 ? a.vp_ptr[v] : 0, qe = a.npairs > 0 ? a.vp_ptr[v + 1] : 0;
  for (int q = qb; q < qe; ++q) {  // barrier of the pairs touching v
    int k = a.vp_list[q] >> 2;
    const double* row = a.pairs + (size_t)kPairRow * k;
    auto posn = [&](int w, double* o) {
#pragma unroll
      for (int c = 0; c < 3; ++c) o[c] = (w == v) ? pv[c] : x[3 * w + c];
    };
    double d;
    if (row[0] == 0.0) {
      double pp[3];
      posn((int)row[1], pp);
      d = plane_dist(pp, a.planes + 6 * (int)row[5]);
    } else {
      double pp[3], pa[3], pb[3], pc[3], bary[3];
      posn((int)row[1], pp);
      posn((int)row[2], pa);
      posn((int)row[3], pb);
      posn((int)row[4], pc);
      d = closest_point_tri(pp, pa, pb, pc, bary);
    }
    if (!(d > 0.0)) return INFINITY;
    e += barrier_fn(d, p.dhat, p.kappa).b;
  }
  return e;
}

__global__ void __launch_bounds__(128)
k_plain_local(DevModel m, LocalArgs a, PlainArgs p) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.nfree) return;
  int v = m.free_list[i];
  // A: own blocks of the incident projected element Hessians + inertia
  double A[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) A[k] = 0.0;
  const double ih2 = 1.0 / (a.h * a.h);
  int p0 = m.inc_ptr[v], p1 = m.inc_ptr[v + 1];
  for (int q = p0; q < p1; ++q) {
    int code = __ldg(m.inc + q), el = code >> 2, s = code & 3;
    const double* M = p.mplus_all + 45 * (size_t)el;
    double qm = m.eprops[el].w * ih2;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int pp = 0; pp < 3; ++pp)
#pragma unroll
          for (int qq = 0; qq < 3; ++qq) acc += kHad(s, pp) * M[tri9(3 * pp + r, 3 * qq + c)] * kHad(s, qq);
        A[3 * r + c] += acc + (r == c ? qm : 0.0);
      }
  }
  if (p1 == p0) {
    double mm = m.mass[v] * ih2;
    A[0] += mm; A[4] += mm; A[8] += mm;
  }
  double g[3] = {a.gasm[3 * v], a.gasm[3 * v + 1], a.gasm[3 * v + 2]};
  const int qb = a.npairs > 0 ? a.vp_ptr[v] : 0, qe = a.npairs > 0 ? a.vp_ptr[v + 1] : 0;
  for (int q = qb; q < qe; ++q) {  // own rows only (coupled = False)
    int k = a.vp_list[q] >> 2, s = a.vp_list[q] & 3;
    const double* row = a.pairs + (size_t)kPairRow * k;
    const double* gp = a.pair_g + 12 * (size_t)k;
    const double* H = a.pair_h + 144 * (size_t)k;
    int o = (row[0] == 0.0) ? 0 : 3 * s;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
      for (int c = 0; c < 3; ++c) A[3 * r + c] += H[12 * (o + r) + o + c];
      g[r] += gp[o + r];
    }
  }
  if (a.A_out) {
#pragma unroll
    for (int k = 0; k < 9; ++k) a.A_out[9 * (size_t)v + k] = A[k];
  }
  if (a.g_out) {
#pragma unroll
    for (int k = 0; k < 3; ++k) a.g_out[3 * (size_t)v + k] = g[k];
  }
  double rhs[3] = {-g[0], -g[1], -g[2]}, d[3];
  if (!solve3_lu(A, rhs, d)) {
    double tr = A[0] + A[4] + A[8];
    if (tr > 0) { d[0] = rhs[0] * (3.0 / tr); d[1] = rhs[1] * (3.0 / tr); d[2] = rhs[2] * (3.0 / tr); }
    else d[0] = d[1] = d[2] = 0.0;
  }
  a.delta[3 * v] = d[0]; a.delta[3 * v + 1] = d[1]; a.delta[3 * v + 2] = d[2];
  double al0 = 1.0;
  int kv = 0;
  if (a.line_search) {
    if (a.npairs > 0) al0 = alpha_cap(a, v, d);
    const double zero[3] = {0.0, 0.0, 0.0};
    double base = plain_energy(m, a, p, v, zero);
    int acc_it = a.max_halvings + 1;
    double al = al0;
    for (int it = 0; it <= a.max_halvings; ++it) {
      double st[3] = {__dmul_rn(al, d[0]), __dmul_rn(al, d[1]), __dmul_rn(al, d[2])};
      double cand = plain_energy(m, a, p, v, st);
      if (cand <= base + 1e-12 * fabs(base)) { acc_it = it; break; }
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

}  // namespace jgs2
