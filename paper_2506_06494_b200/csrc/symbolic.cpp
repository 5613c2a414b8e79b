// Geometric nested dissection + supernodal front tree (host C++).
// See symbolic.h for the contract.
#include "symbolic.h"

#include <algorithm>
#include <numeric>
#include <stdexcept>

namespace jgs2 {

namespace {

struct NdBuilder {
  int n;
  const int64_t* ap;
  const int32_t* aj;
  const double* xyz;
  int leaf;
  std::vector<int> side;   // -1 = not in current subset, 0 = A, 1 = B
  std::vector<int> order;  // positions assigned in postorder
  Symbolic* S;
  std::vector<std::vector<int>> kids;

  int new_front(const int* verts, int count) {
    int id = S->nfronts++;
    S->col_begin.push_back((int)order.size());
    for (int k = 0; k < count; ++k) order.push_back(verts[k]);
    S->col_end.push_back((int)order.size());
    S->parent.push_back(-1);
    kids.emplace_back();
    return id;
  }

  // Dissect verts[lo, hi); returns the front id of the subtree root.
  int dissect(std::vector<int>& v, int lo, int hi, int depth) {
    int cnt = hi - lo;
    if (cnt <= leaf || depth > 60) {
      std::sort(v.begin() + lo, v.begin() + hi);
      return new_front(v.data() + lo, cnt);
    }
    double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
    for (int k = lo; k < hi; ++k)
      for (int d = 0; d < 3; ++d) {
        double c = xyz[3 * (size_t)v[k] + d];
        mn[d] = std::min(mn[d], c);
        mx[d] = std::max(mx[d], c);
      }
    int axis = 0;
    for (int d = 1; d < 3; ++d)
      if (mx[d] - mn[d] > mx[axis] - mn[axis]) axis = d;
    int mid = lo + cnt / 2;
    std::nth_element(v.begin() + lo, v.begin() + mid, v.begin() + hi, [&](int a, int b) {
      double ca = xyz[3 * (size_t)a + axis], cb = xyz[3 * (size_t)b + axis];
      return ca < cb || (ca == cb && a < b);
    });
    for (int k = lo; k < hi; ++k) side[v[k]] = (k < mid) ? 0 : 1;
    // one-sided vertex separators; keep the smaller
    std::vector<char> bnd(cnt, 0);
    int na = 0, nb = 0;
    for (int k = lo; k < hi; ++k) {
      int u = v[k], su = side[u];
      for (int64_t e = ap[u]; e < ap[u + 1]; ++e) {
        int w = aj[e];
        if (w != u && side[w] >= 0 && side[w] != su) { bnd[k - lo] = 1; break; }
      }
      if (bnd[k - lo]) (su == 0 ? na : nb)++;
    }
    int sep_side = (na <= nb) ? 0 : 1;
    std::vector<int> A, B, Sep;
    A.reserve(cnt); B.reserve(cnt);
    for (int k = lo; k < hi; ++k) {
      int u = v[k];
      if (bnd[k - lo] && side[u] == sep_side) Sep.push_back(u);
      else if (side[u] == 0) A.push_back(u);
      else B.push_back(u);
    }
    for (int k = lo; k < hi; ++k) side[v[k]] = -1;
    if (Sep.empty() && (A.empty() || B.empty())) {  // no progress: make a leaf
      std::sort(v.begin() + lo, v.begin() + hi);
      return new_front(v.data() + lo, cnt);
    }
    int p = lo;
    for (int u : A) v[p++] = u;
    int bl = p;
    for (int u : B) v[p++] = u;
    int sl = p;
    for (int u : Sep) v[p++] = u;
    int ca = -1, cb = -1;
    if (bl > lo) {
      for (int k = lo; k < bl; ++k) side[v[k]] = -1;
      ca = dissect(v, lo, bl, depth + 1);
    }
    if (sl > bl) cb = dissect(v, bl, sl, depth + 1);
    if (Sep.empty()) {
      // disconnected halves: the two subtrees become siblings under a
      // zero-column virtual front is unnecessary; chain them instead
      if (ca >= 0 && cb >= 0) {
        int id = new_front(nullptr, 0);
        S->parent[ca] = id; kids[id].push_back(ca);
        S->parent[cb] = id; kids[id].push_back(cb);
        return id;
      }
      return ca >= 0 ? ca : cb;
    }
    std::sort(v.begin() + sl, v.begin() + hi);
    int id = new_front(v.data() + sl, hi - sl);
    if (ca >= 0) { S->parent[ca] = id; kids[id].push_back(ca); }
    if (cb >= 0) { S->parent[cb] = id; kids[id].push_back(cb); }
    return id;
  }
};

}  // namespace

void build_symbolic(int n, const int64_t* adj_ptr, const int32_t* adj, const double* coords,
                    int leaf_size, Symbolic& S) {
  S = Symbolic();
  S.n = n;
  if (n == 0) return;
  NdBuilder b{n, adj_ptr, adj, coords, std::max(1, leaf_size)};
  b.side.assign(n, -1);
  b.order.reserve(n);
  b.S = &S;
  // Connected components first: each is dissected on its own coordinates
  // (bodies of a multi-body scene share overlapping rest frames, so a
  // geometric split across components would be meaningless), and the
  // component roots are joined pairwise by zero-column fronts.
  std::vector<int> comp(n, -1), v;
  v.reserve(n);
  std::vector<int> cstart;
  for (int s = 0; s < n; ++s) {
    if (comp[s] >= 0) continue;
    int c = (int)cstart.size();
    cstart.push_back((int)v.size());
    comp[s] = c;
    size_t head = v.size();
    v.push_back(s);
    while (head < v.size()) {
      int u = v[head++];
      for (int64_t e = adj_ptr[u]; e < adj_ptr[u + 1]; ++e) {
        int w = adj[e];
        if (comp[w] < 0) { comp[w] = c; v.push_back(w); }
      }
    }
  }
  cstart.push_back(n);
  std::vector<int> roots;
  for (size_t c = 0; c + 1 < cstart.size(); ++c) roots.push_back(b.dissect(v, cstart[c], cstart[c + 1], 0));
  while (roots.size() > 1) {
    std::vector<int> next;
    for (size_t k = 0; k + 1 < roots.size(); k += 2) {
      int id = b.new_front(nullptr, 0);
      S.parent[roots[k]] = id; b.kids[id].push_back(roots[k]);
      S.parent[roots[k + 1]] = id; b.kids[id].push_back(roots[k + 1]);
      next.push_back(id);
    }
    if (roots.size() % 2) next.push_back(roots.back());
    roots.swap(next);
  }
  if ((int)b.order.size() != n) throw std::runtime_error("nested dissection lost vertices");
  S.perm = b.order;
  S.iperm.assign(n, -1);
  for (int p = 0; p < n; ++p) S.iperm[S.perm[p]] = p;
  int F = S.nfronts;
  S.child_ptr.assign(F + 1, 0);
  for (int f = 0; f < F; ++f) S.child_ptr[f + 1] = S.child_ptr[f] + (int)b.kids[f].size();
  S.child_list.reserve(S.child_ptr[F]);
  for (int f = 0; f < F; ++f) {
    auto k = b.kids[f];
    std::sort(k.begin(), k.end());
    for (int c : k) S.child_list.push_back(c);
  }
  // row structures bottom-up (fronts are in postorder: children before parent)
  S.struct_ptr.assign(F + 1, 0);
  std::vector<std::vector<int>> st(F);
  std::vector<int> mark(n, -1);
  S.level.assign(F, 0);
  for (int f = 0; f < F; ++f) {
    int cb = S.col_begin[f], ce = S.col_end[f];
    std::vector<int>& s = st[f];
    for (int p = cb; p < ce; ++p) {
      int u = S.perm[p];
      for (int64_t e = adj_ptr[u]; e < adj_ptr[u + 1]; ++e) {
        int q = S.iperm[adj[e]];
        if (q >= ce && mark[q] != f) { mark[q] = f; s.push_back(q); }
      }
    }
    int lev = 0;
    for (int k = S.child_ptr[f]; k < S.child_ptr[f + 1]; ++k) {
      int c = S.child_list[k];
      lev = std::max(lev, S.level[c] + 1);
      for (int q : st[c])
        if (q >= ce && mark[q] != f) { mark[q] = f; s.push_back(q); }
      std::vector<int>().swap(st[c]);  // consumed by the (unique) parent
    }
    S.level[f] = lev;
    std::sort(s.begin(), s.end());
    S.struct_ptr[f + 1] = S.struct_ptr[f] + (int64_t)s.size();
    S.struct_pos.insert(S.struct_pos.end(), s.begin(), s.end());
  }
  S.nlevels = 0;
  for (int f = 0; f < F; ++f) S.nlevels = std::max(S.nlevels, S.level[f] + 1);
  // a parent's level must exceed all children's (guaranteed above); fronts
  // at one level are independent.
  int64_t nnz = 0;
  for (int f = 0; f < F; ++f) {
    int64_t ns = 3LL * (S.col_end[f] - S.col_begin[f]);
    int64_t nr = 3LL * (S.struct_ptr[f + 1] - S.struct_ptr[f]);
    nnz += ns * (ns + 1) / 2 + nr * ns;
  }
  S.nnz_dof = nnz;
}

}  // namespace jgs2
