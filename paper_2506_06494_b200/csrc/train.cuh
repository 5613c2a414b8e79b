// Scalable precompute, host side: per-vertex bases from the
// selected inverse and cubature training per vertex.
//
// Reference: subspace.precompute_bases / retain_rows (subspace.py:133-203),
// cubature._labels / train_cubature / nnls / train_all (cubature.py:113-291).
// The reference solves Hbar Y = S^T for the dense N x 3 column of every
// vertex. Here every block it needs comes from Z = Hbar^-1 on the factor's
// pattern (selinv.cuh):
//   Gbar_v = -[(Hbar^-1)_vv]^-1,  U_v[w] = -(Hbar^-1)_wv Gbar_v,
//   labels  U_v^T (g_t - g_t|inc(v)) = -Gbar_v^T [(Hbar^-1 g_t)_v
//             - sum_{w in inc(v)} (Hbar^-1)_vw g_t|inc(v)[w]]     (one solve
//             per pose, shared by all vertices: the adjoint form),
//   candidate columns stencil_grads[:, e] @ U_v[tets[e]].
// The greedy selection + NNLS refit is the reference's algorithm (same
// target, round limit, size cap, zero-weight eviction, Lawson-Hanson NNLS);
// the candidate pool is the non-incident elements whose corners lie in the
// vertex's front (the rows the selected inverse provides: the vertex's
// nested-dissection cell and its separators), drawn with a counter-based
// RNG seeded per vertex, instead of all elements with numpy's Generator.
#pragma once
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "context.cuh"

namespace jgs2 {

struct TrainOut {
  std::vector<int64_t> vertices, vr_ptr, vr_keys, cub_ptr, cub_elems;
  std::vector<double> gbar, vrows, cub_w, residual;
  std::vector<uint8_t> converged;
};

struct HostInverse {
  const Symbolic* S;
  const std::vector<int>* pos;
  const std::vector<int>* pfront;
  const std::vector<int64_t>* loff;
  const std::vector<int>* fld;
  const double* Z;
  // (Hbar^-1)_{wv}, row-major 3x3; false if not on the filled pattern
  bool block(int v, int w, double* o) const {
    int pv = (*pos)[v], pw = (*pos)[w];
    if (pv < 0 || pw < 0) {
      for (int q = 0; q < 9; ++q) o[q] = 0.0;
      return true;
    }
    int fv = (*pfront)[pv];
    int cb = S->col_begin[fv], ce = S->col_end[fv];
    int ns = 3 * (ce - cb), c = 3 * (pv - cb), r = -1;
    if (pw >= cb && pw < ce) {
      r = 3 * (pw - cb);
    } else {
      const int* a = S->struct_pos.data() + S->struct_ptr[fv];
      const int* b = S->struct_pos.data() + S->struct_ptr[fv + 1];
      const int* it = std::lower_bound(a, b, pw);
      if (it != b && *it == pw) r = ns + 3 * (int)(it - a);
    }
    if (r >= 0) {
      const double* Zf = Z + (*loff)[fv];
      int ld = (*fld)[fv];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          int rr = r + i, cc = c + j;
          o[3 * i + j] = rr >= cc ? Zf[(int64_t)cc * ld + rr] : Zf[(int64_t)rr * ld + cc];
        }
      return true;
    }
    int fw = (*pfront)[pw];
    int cbw = S->col_begin[fw];
    int nsw = 3 * (S->col_end[fw] - cbw);
    const int* a = S->struct_pos.data() + S->struct_ptr[fw];
    const int* b = S->struct_pos.data() + S->struct_ptr[fw + 1];
    const int* it = std::lower_bound(a, b, pv);
    if (it != b && *it == pv) {
      const double* Zf = Z + (*loff)[fw];
      int ld = (*fld)[fw];
      int cw = 3 * (pw - cbw), rv = nsw + 3 * (int)(it - a);
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o[3 * i + j] = Zf[(int64_t)(cw + i) * ld + rv + j];
      return true;
    }
    for (int q = 0; q < 9; ++q) o[q] = 0.0;
    return false;
  }
};

// splitmix64 stream per (seed, vertex)
struct Rng {
  uint64_t s;
  Rng(uint64_t seed, uint64_t v) : s(seed * 0x9E3779B97F4A7C15ull ^ (v + 0x632BE59BD9B4E019ull)) { next(); }
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  size_t below(size_t n) { return (size_t)(next() % n); }
};

// least squares min |A x - b| (m x k column-major, k <= 8) by Householder QR;
// columns with a negligible pivot get x = 0
inline void lstsq_small(const std::vector<double>& A, int m, int k, const std::vector<double>& b, double* x) {
  std::vector<double> R(A), y(b);
  std::vector<double> diag(k, 0.0);
  double rmax = 0.0;
  for (int j = 0; j < k; ++j) {
    double nrm = 0.0;
    for (int i = j; i < m; ++i) nrm += R[(size_t)j * m + i] * R[(size_t)j * m + i];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) { diag[j] = 0.0; continue; }
    double a0 = R[(size_t)j * m + j];
    double alpha = a0 > 0 ? -nrm : nrm;
    double v0 = a0 - alpha;
    // v = [v0, R[j+1..m)], H = I - 2 v v^T / (v^T v)
    double vtv = v0 * v0;
    for (int i = j + 1; i < m; ++i) vtv += R[(size_t)j * m + i] * R[(size_t)j * m + i];
    auto apply = [&](double* col) {
      double d = v0 * col[j];
      for (int i = j + 1; i < m; ++i) d += R[(size_t)j * m + i] * col[i];
      double t = 2.0 * d / vtv;
      col[j] -= t * v0;
      for (int i = j + 1; i < m; ++i) col[i] -= t * R[(size_t)j * m + i];
    };
    for (int c = j + 1; c < k; ++c) apply(&R[(size_t)c * m]);
    apply(y.data());
    diag[j] = alpha;
    rmax = std::max(rmax, std::fabs(alpha));
  }
  for (int j = k - 1; j >= 0; --j) {
    if (std::fabs(diag[j]) <= 1e-14 * rmax || diag[j] == 0.0) { x[j] = 0.0; continue; }
    double s = y[j];
    for (int c = j + 1; c < k; ++c) s -= R[(size_t)c * m + j] * x[c];
    x[j] = s / diag[j];
  }
}

// Lawson-Hanson NNLS (cubature.py:113-167); returns false past the iteration cap
inline bool nnls_small(const std::vector<double>& A, int m, int n, const std::vector<double>& b, std::vector<double>& w) {
  int maxiter = std::max(10 * n, 50);
  auto atv = [&](const std::vector<double>& r, std::vector<double>& out) {
    out.assign(n, 0.0);
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int i = 0; i < m; ++i) s += A[(size_t)j * m + i] * r[i];
      out[j] = s;
    }
  };
  std::vector<double> dual;
  atv(b, dual);
  double amax = 0.0;
  for (double d : dual) amax = std::max(amax, std::fabs(d));
  double tol = 1e-10 * std::max(amax, 1.0);
  w.assign(n, 0.0);
  std::vector<char> passive(n, 0), barred(n, 0);
  std::vector<double> resid(b), s(n);
  int iters = 0;
  auto solve_passive = [&](std::vector<double>& out) {
    out.assign(n, 0.0);
    std::vector<int> cols;
    for (int j = 0; j < n; ++j)
      if (passive[j]) cols.push_back(j);
    if (cols.empty()) return;
    std::vector<double> As((size_t)m * cols.size());
    for (size_t q = 0; q < cols.size(); ++q)
      for (int i = 0; i < m; ++i) As[q * m + i] = A[(size_t)cols[q] * m + i];
    std::vector<double> x(cols.size());
    lstsq_small(As, m, (int)cols.size(), b, x.data());
    for (size_t q = 0; q < cols.size(); ++q) out[cols[q]] = x[q];
  };
  while (true) {
    bool any = false;
    int jbest = -1;
    double dbest = -INFINITY;
    for (int j = 0; j < n; ++j) {
      if (passive[j] || barred[j]) continue;
      if (dual[j] > tol) any = true;
      if (dual[j] > dbest) { dbest = dual[j]; jbest = j; }
    }
    if (!any || jbest < 0) break;
    int j = jbest;
    passive[j] = 1;
    while (true) {
      if (++iters > maxiter) return false;
      solve_passive(s);
      double smin = INFINITY;
      for (int q = 0; q < n; ++q)
        if (passive[q]) smin = std::min(smin, s[q]);
      if (smin > 0.0) { w = s; break; }
      if (s[j] <= 0.0 && w[j] == 0.0) {
        passive[j] = 0;
        barred[j] = 1;
        solve_passive(s);
        for (int q = 0; q < n; ++q) w[q] = passive[q] ? s[q] : 0.0;
        break;
      }
      double alpha = INFINITY;
      for (int q = 0; q < n; ++q)
        if (passive[q] && s[q] <= 0.0) alpha = std::min(alpha, w[q] / (w[q] - s[q]));
      for (int q = 0; q < n; ++q) w[q] = w[q] + alpha * (s[q] - w[q]);
      for (int q = 0; q < n; ++q) {
        if (passive[q] && !(w[q] > tol)) passive[q] = 0;
        if (!passive[q]) w[q] = 0.0;
      }
    }
    for (int i = 0; i < m; ++i) {
      double r = b[i];
      for (int q = 0; q < n; ++q) r -= A[(size_t)q * m + i] * w[q];
      resid[i] = r;
    }
    atv(resid, dual);
  }
  return true;
}

inline void inv3(const double* a, double* o) {
  double c00 = a[4] * a[8] - a[5] * a[7], c01 = a[5] * a[6] - a[3] * a[8], c02 = a[3] * a[7] - a[4] * a[6];
  double det = a[0] * c00 + a[1] * c01 + a[2] * c02;
  double id = 1.0 / det;
  o[0] = c00 * id; o[1] = (a[2] * a[7] - a[1] * a[8]) * id; o[2] = (a[1] * a[5] - a[2] * a[4]) * id;
  o[3] = c01 * id; o[4] = (a[0] * a[8] - a[2] * a[6]) * id; o[5] = (a[2] * a[3] - a[0] * a[5]) * id;
  o[6] = c02 * id; o[7] = (a[1] * a[6] - a[0] * a[7]) * id; o[8] = (a[0] * a[4] - a[1] * a[3]) * id;
}

struct TrainParams {
  int T, cand, max_size;
  double target;
  uint64_t seed;
  const double* grads;  // T x ne x 12
  const double* solves; // T x nv x 3   (Hbar^-1 g_t)
};

// per-vertex result (then flattened in ascending vertex order)
struct VertexResult {
  double gbar[9];
  std::vector<int> keys;
  std::vector<double> rows;
  std::vector<int> elems;
  std::vector<double> weights;
  double residual = 0.0;
  bool converged = true;
  bool ok = true;
};

}  // namespace jgs2

namespace jgs2 {

inline void train_vertex(int v, const std::vector<int>& pool, const HostInverse& H, const TrainParams& P,
                         const std::vector<int64_t>& tets, const std::vector<int>& inc_ptr,
                         const std::vector<int>& inc, int nv, std::vector<int>& ustamp, std::vector<int>& uslot,
                         std::vector<double>& ublk, VertexResult& R) {
  const int T = P.T;
  double Y[9], G[9];
  H.block(v, v, Y);
  inv3(Y, G);
  for (int q = 0; q < 9; ++q) R.gbar[q] = -G[q];  // Gbar = -[(Hbar^-1)_vv]^-1
  const double* Gb = R.gbar;
  ublk.clear();
  auto getU = [&](int w) -> const double* {
    if (ustamp[w] == v) return &ublk[9 * (size_t)uslot[w]];
    double Yw[9];
    if (!H.block(v, w, Yw)) return nullptr;
    size_t s = ublk.size() / 9;
    ublk.resize(ublk.size() + 9);
    double* U = &ublk[9 * s];
    for (int i = 0; i < 3; ++i)  // U = -Y Gbar
      for (int j = 0; j < 3; ++j)
        U[3 * i + j] = -(Yw[3 * i] * Gb[j] + Yw[3 * i + 1] * Gb[3 + j] + Yw[3 * i + 2] * Gb[6 + j]);
    ustamp[w] = v;
    uslot[w] = (int)s;
    return &ublk[9 * s];
  };
  // labels (cubature.py:170-183), adjoint form
  std::vector<double> lab(3 * T, 0.0);
  {
    std::vector<double> acc(3 * T, 0.0);
    for (int p = inc_ptr[v]; p < inc_ptr[v + 1]; ++p) {
      int e = inc[p];
      for (int a = 0; a < 4; ++a) {
        int w = (int)tets[4 * (size_t)e + a];
        double Yw[9];
        H.block(v, w, Yw);  // ring vertices are adjacent: always on the pattern
        for (int t = 0; t < T; ++t) {
          const double* ge = P.grads + ((size_t)t * (size_t)(tets.size() / 4) + e) * 12 + 3 * a;
          for (int j = 0; j < 3; ++j)  // (Hbar^-1)_vw = Y_wv^T
            acc[3 * t + j] += Yw[j] * ge[0] + Yw[3 + j] * ge[1] + Yw[6 + j] * ge[2];
        }
      }
    }
    for (int t = 0; t < T; ++t) {
      const double* zt = P.solves + ((size_t)t * nv + v) * 3;
      double r[3] = {zt[0] - acc[3 * t], zt[1] - acc[3 * t + 1], zt[2] - acc[3 * t + 2]};
      for (int j = 0; j < 3; ++j)  // -Gbar^T r
        lab[3 * t + j] = -(Gb[j] * r[0] + Gb[3 + j] * r[1] + Gb[6 + j] * r[2]);
    }
  }
  // retained rows: own + incident-element vertices (+ cubature corners below)
  std::vector<int> keys;
  keys.push_back(v);
  for (int p = inc_ptr[v]; p < inc_ptr[v + 1]; ++p)
    for (int a = 0; a < 4; ++a) keys.push_back((int)tets[4 * (size_t)inc[p] + a]);
  // cubature training (cubature.py:192-276)
  std::vector<double> norms(T);
  double nmax = 0.0;
  for (int t = 0; t < T; ++t) {
    norms[t] = std::sqrt(lab[3 * t] * lab[3 * t] + lab[3 * t + 1] * lab[3 * t + 1] + lab[3 * t + 2] * lab[3 * t + 2]);
    nmax = std::max(nmax, norms[t]);
  }
  std::vector<int> usable;
  for (int t = 0; t < T; ++t)
    if (norms[t] > 1e-8 * nmax) usable.push_back(t);
  std::vector<int> selected;
  std::vector<double> weights;
  R.residual = 0.0;
  R.converged = true;
  if (!usable.empty()) {
    const int m = 3 * (int)usable.size();
    std::vector<double> b(m);
    for (size_t q = 0; q < usable.size(); ++q)
      for (int j = 0; j < 3; ++j) b[3 * q + j] = lab[3 * usable[q] + j] / norms[usable[q]];
    double bn = 0.0;
    for (double x : b) bn += x * x;
    bn = std::sqrt(bn);
    // pool minus the incident elements (ascending)
    std::vector<int> incv(inc.begin() + inc_ptr[v], inc.begin() + inc_ptr[v + 1]);
    std::sort(incv.begin(), incv.end());
    std::vector<int> remaining;
    remaining.reserve(pool.size());
    std::set_difference(pool.begin(), pool.end(), incv.begin(), incv.end(), std::back_inserter(remaining));
    const int ne = (int)(tets.size() / 4);
    auto col_for = [&](int e, std::vector<double>& col) -> bool {
      const double* U[4];
      for (int a = 0; a < 4; ++a) {
        U[a] = getU((int)tets[4 * (size_t)e + a]);
        if (!U[a]) return false;
      }
      col.assign(m, 0.0);
      for (size_t q = 0; q < usable.size(); ++q) {
        int t = usable[q];
        const double* ge = P.grads + ((size_t)t * ne + e) * 12;
        for (int j = 0; j < 3; ++j) {
          double s = 0.0;
          for (int a = 0; a < 4; ++a)
            for (int i = 0; i < 3; ++i) s += U[a][3 * i + j] * ge[3 * a + i];
          col[3 * q + j] = s / norms[t];
        }
      }
      return true;
    };
    Rng rng(P.seed, (uint64_t)v);
    std::vector<std::vector<double>> columns;
    std::vector<double> resid(b), col, bestcol, A;
    double rel = 1.0;
    for (int round = 0; round < 6 * P.max_size; ++round) {
      if (rel <= P.target) break;
      if ((int)selected.size() >= P.max_size) {
        bool all = weights.size() == selected.size();
        for (size_t q = 0; q < std::min(weights.size(), selected.size()); ++q) all = all && weights[q] > 0.0;
        if (all) break;
        std::vector<int> s2;
        std::vector<std::vector<double>> c2;
        for (size_t q = 0; q < selected.size() && q < weights.size(); ++q)
          if (weights[q] > 0.0) { s2.push_back(selected[q]); c2.push_back(columns[q]); }
        selected.swap(s2);
        columns.swap(c2);
      }
      if (remaining.empty()) break;
      size_t k = std::min<size_t>((size_t)P.cand, remaining.size());
      // k distinct candidates (partial Fisher-Yates on a copy)
      std::vector<int> rem(remaining);
      int best = -1;
      double best_score = -INFINITY;
      for (size_t i = 0; i < k; ++i) {
        size_t jdx = i + rng.below(rem.size() - i);
        std::swap(rem[i], rem[jdx]);
        int e = rem[i];
        if (!col_for(e, col)) continue;
        double cn = 0.0, dp = 0.0;
        for (int q = 0; q < m; ++q) { cn += col[q] * col[q]; dp += col[q] * resid[q]; }
        cn = std::sqrt(cn);
        if (cn <= 0.0) continue;
        double score = dp / cn;
        if (score > best_score) { best = e; best_score = score; bestcol = col; }
      }
      if (best < 0) break;
      selected.push_back(best);
      columns.push_back(bestcol);
      remaining.erase(std::lower_bound(remaining.begin(), remaining.end(), best));
      int n = (int)columns.size();
      A.assign((size_t)m * n, 0.0);
      for (int q = 0; q < n; ++q) std::copy(columns[q].begin(), columns[q].end(), A.begin() + (size_t)q * m);
      if (!nnls_small(A, m, n, b, weights)) { R.ok = false; break; }
      double rn = 0.0;
      for (int i = 0; i < m; ++i) {
        double r = b[i];
        for (int q = 0; q < n; ++q) r -= A[(size_t)q * m + i] * weights[q];
        resid[i] = r;
        rn += r * r;
      }
      rel = std::sqrt(rn) / bn;
    }
    std::vector<int> s3;
    std::vector<double> w3;
    for (size_t q = 0; q < selected.size() && q < weights.size(); ++q)
      if (weights[q] > 0.0) { s3.push_back(selected[q]); w3.push_back(weights[q]); }
    selected.swap(s3);
    weights.swap(w3);
    R.residual = rel;
    R.converged = rel <= P.target;
  }
  // cubature elements in selection order (CubatureSet.elements), their corners retained
  for (int e : selected)
    for (int a = 0; a < 4; ++a) keys.push_back((int)tets[4 * (size_t)e + a]);
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  R.keys = keys;
  R.rows.resize(9 * keys.size());
  for (size_t q = 0; q < keys.size(); ++q) {
    const double* U = getU(keys[q]);
    if (!U) { R.ok = false; continue; }
    std::copy(U, U + 9, R.rows.begin() + 9 * q);
  }
  R.elems = selected;
  R.weights = weights;
}

inline void train_all_host(Ctx& C, const TrainParams& P, TrainOut& out) {
  Factor& F = C.fac;
  const Symbolic& S = F.sym;
  const int nv = C.nv, ne = C.ne, NF = S.nfronts;
  std::vector<double> Zh((size_t)F.nnz_alloc);
  JGS2_CUDA(cudaMemcpy(Zh.data(), F.Z, Zh.size() * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<int> pfront(S.n, -1), pos2v(S.n, -1);
  for (int f = 0; f < NF; ++f)
    for (int q = S.col_begin[f]; q < S.col_end[f]; ++q) pfront[q] = f;
  for (int v = 0; v < nv; ++v)
    if (F.h_pos[v] >= 0) pos2v[F.h_pos[v]] = v;
  HostInverse H{&S, &F.h_pos, &pfront, &F.h_loff, &F.h_fld, Zh.data()};
  std::vector<int> inc_ptr(nv + 1, 0), inc(4 * (size_t)ne);
  for (size_t k = 0; k < 4 * (size_t)ne; ++k) inc_ptr[C.h_tets[k] + 1]++;
  for (int v = 0; v < nv; ++v) inc_ptr[v + 1] += inc_ptr[v];
  {
    std::vector<int> fill(inc_ptr.begin(), inc_ptr.end() - 1);
    for (int e = 0; e < ne; ++e)
      for (int a = 0; a < 4; ++a) inc[fill[C.h_tets[4 * (size_t)e + a]]++] = e;
  }
  std::vector<VertexResult> res(nv);
#pragma omp parallel
  {
    std::vector<int> vmark(nv, -1), emark(ne, -1), ustamp(nv, -1), uslot(nv, 0);
    std::vector<double> ublk;
#pragma omp for schedule(dynamic, 1)
    for (int f = 0; f < NF; ++f) {
      if (S.col_end[f] == S.col_begin[f]) continue;
      std::vector<int> fverts;
      for (int q = S.col_begin[f]; q < S.col_end[f]; ++q) fverts.push_back(pos2v[q]);
      for (int64_t k = S.struct_ptr[f]; k < S.struct_ptr[f + 1]; ++k) fverts.push_back(pos2v[S.struct_pos[k]]);
      for (int w : fverts) vmark[w] = f;
      std::vector<int> pool;
      for (int w : fverts)
        for (int p = inc_ptr[w]; p < inc_ptr[w + 1]; ++p) {
          int e = inc[p];
          if (emark[e] == f) continue;
          emark[e] = f;
          bool in = true;
          for (int a = 0; a < 4 && in; ++a) {
            int c = (int)C.h_tets[4 * (size_t)e + a];
            in = vmark[c] == f || C.h_fixed[c];
          }
          if (in) pool.push_back(e);
        }
      std::sort(pool.begin(), pool.end());
      for (int q = S.col_begin[f]; q < S.col_end[f]; ++q) {
        int v = pos2v[q];
        train_vertex(v, pool, H, P, C.h_tets, inc_ptr, inc, nv, ustamp, uslot, ublk, res[v]);
      }
    }
  }
  out = TrainOut();
  out.vr_ptr.push_back(0);
  out.cub_ptr.push_back(0);
  for (int v = 0; v < nv; ++v) {
    if (F.h_pos[v] < 0) continue;  // fixed (or another rank's) vertex
    VertexResult& R = res[v];
    if (!R.ok) throw Error(JGS2_E_FACTOR, "precompute: basis rows off the factor pattern at vertex " +
                                              std::to_string(v));
    out.vertices.push_back(v);
    out.gbar.insert(out.gbar.end(), R.gbar, R.gbar + 9);
    for (size_t q = 0; q < R.keys.size(); ++q) out.vr_keys.push_back(R.keys[q]);
    out.vrows.insert(out.vrows.end(), R.rows.begin(), R.rows.end());
    out.vr_ptr.push_back((int64_t)out.vr_keys.size());
    for (size_t q = 0; q < R.elems.size(); ++q) {
      out.cub_elems.push_back(R.elems[q]);
      out.cub_w.push_back(R.weights[q]);
    }
    out.cub_ptr.push_back((int64_t)out.cub_elems.size());
    out.residual.push_back(R.residual);
    out.converged.push_back(R.converged ? 1 : 0);
  }
}

}  // namespace jgs2
