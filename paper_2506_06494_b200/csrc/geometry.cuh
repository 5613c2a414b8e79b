// Contact geometry with the reference's rounding order (contact.py:162-213,
// 216-240). Shared by the pair detection, the live distances of the
// alpha caps and the feasibility cap.
#pragma once
#include "physics.cuh"

namespace jgs2 {

__device__ __forceinline__ double dot3_np(const double* a, const double* b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[2], b[2])), __dmul_rn(a[1], b[1]));
}
// plane distance (x - p) @ n   (BLAS gemv order: sequential)
__device__ __forceinline__ double plane_dist(const double* x, const double* pl) {
  double d0 = x[0] - pl[0], d1 = x[1] - pl[1], d2 = x[2] - pl[2];
  return __dadd_rn(__dadd_rn(__dmul_rn(d0, pl[3]), __dmul_rn(d1, pl[4])), __dmul_rn(d2, pl[5]));
}

// Closest point of p to triangle (a, b, c): distance and barycentrics with
// exact zeros in clamped regions (contact.py:162-213).
__device__ double closest_point_tri(const double* p, const double* a, const double* b, const double* c,
                                    double* bary) {
  double ab[3], ac[3], ap[3], bp[3], cp[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ab[k] = b[k] - a[k]; ac[k] = c[k] - a[k];
    ap[k] = p[k] - a[k]; bp[k] = p[k] - b[k]; cp[k] = p[k] - c[k];
  }
  double d1 = dot3_np(ab, ap), d2 = dot3_np(ac, ap);
  double d3 = dot3_np(ab, bp), d4 = dot3_np(ac, bp);
  double d5 = dot3_np(ab, cp), d6 = dot3_np(ac, cp);
  double vc = __dsub_rn(__dmul_rn(d1, d4), __dmul_rn(d3, d2));
  double vb = __dsub_rn(__dmul_rn(d5, d2), __dmul_rn(d1, d6));
  double va = __dsub_rn(__dmul_rn(d3, d6), __dmul_rn(d5, d4));
  double b0, b1, b2;
  if (d1 <= 0 && d2 <= 0) { b0 = 1.0; b1 = 0.0; b2 = 0.0; }
  else if (d3 >= 0 && d4 <= d3) { b0 = 0.0; b1 = 1.0; b2 = 0.0; }
  else if (d6 >= 0 && d5 <= d6) { b0 = 0.0; b1 = 0.0; b2 = 1.0; }
  else if (vc <= 0 && d1 >= 0 && d3 <= 0) {
    double v = __ddiv_rn(d1, __dsub_rn(d1, d3));
    b0 = __dsub_rn(1.0, v); b1 = v; b2 = 0.0;
  } else if (vb <= 0 && d2 >= 0 && d6 <= 0) {
    double w = __ddiv_rn(d2, __dsub_rn(d2, d6));
    b0 = __dsub_rn(1.0, w); b1 = 0.0; b2 = w;
  } else if (va <= 0 && __dsub_rn(d4, d3) >= 0 && __dsub_rn(d5, d6) >= 0) {
    double w = __ddiv_rn(__dsub_rn(d4, d3), __dadd_rn(__dsub_rn(d4, d3), __dsub_rn(d5, d6)));
    b0 = 0.0; b1 = __dsub_rn(1.0, w); b2 = w;
  } else {
    double den = __dadd_rn(__dadd_rn(va, vb), vc);
    b0 = __ddiv_rn(va, den); b1 = __ddiv_rn(vb, den); b2 = __ddiv_rn(vc, den);
  }
  bary[0] = b0; bary[1] = b1; bary[2] = b2;
  double q[3], r[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    q[k] = __dadd_rn(__dadd_rn(__dmul_rn(b0, a[k]), __dmul_rn(b1, b[k])), __dmul_rn(b2, c[k]));
    r[k] = __dsub_rn(p[k], q[k]);
  }
  return norm3_np(r);
}

__device__ __forceinline__ void load_pos(const double* x, const double* dx, double gamma, int v, double* o) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double xv = x[3 * v + c];
    o[c] = dx ? __dadd_rn(xv, __dmul_rn(gamma, dx[3 * v + c])) : xv;
  }
}


}  // namespace jgs2
