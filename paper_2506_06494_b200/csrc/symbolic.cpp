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

// Shared tail: iperm, children lists, row structures (bottom-up: a front's
// structure is its columns' adjacency beyond the front plus its children's
// structures beyond it), levels and the stored entry count. Fronts must be in
// postorder (children before parents) with contiguous position ranges.
void finish_symbolic(Symbolic& S, const int64_t* adj_ptr, const int32_t* adj,
                     const std::vector<std::vector<int>>& kids) {
  const int n = S.n;
  S.iperm.assign(n, -1);
  for (int p = 0; p < n; ++p) S.iperm[S.perm[p]] = p;
  int F = S.nfronts;
  S.child_ptr.assign(F + 1, 0);
  for (int f = 0; f < F; ++f) S.child_ptr[f + 1] = S.child_ptr[f] + (int)kids[f].size();
  S.child_list.reserve(S.child_ptr[F]);
  for (int f = 0; f < F; ++f) {
    auto k = kids[f];
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
  finish_symbolic(S, adj_ptr, adj, b.kids);
}

// Front tree from a given fill-reducing ordering (e.g. METIS nested
// dissection): elimination tree (Liu), postorder (fill-preserving, makes every
// subtree contiguous), column counts, fundamental supernodes (a column joins
// its predecessor when it is the predecessor's parent, its only child, and
// one row shorter), then relaxed amalgamation of small supernodes into their
// parent when contiguous (at most `relax` vertices merged; explicit zeros are
// stored and streamed like the rest of the panel).
void build_symbolic_perm(int n, const int64_t* adj_ptr, const int32_t* adj, const int32_t* perm0, int relax,
                         Symbolic& S) {
  S = Symbolic();
  S.n = n;
  if (n == 0) return;
  std::vector<int> ip(n), parent(n, -1), anc(n, -1);
  for (int i = 0; i < n; ++i) ip[perm0[i]] = i;
  auto etree = [&](const std::vector<int>& pm, const std::vector<int>& ipm, std::vector<int>& par) {
    std::fill(par.begin(), par.end(), -1);
    std::fill(anc.begin(), anc.end(), -1);
    for (int i = 0; i < n; ++i) {
      int o = pm[i];
      for (int64_t q = adj_ptr[o]; q < adj_ptr[o + 1]; ++q) {
        int j = ipm[adj[q]];
        if (j >= i) continue;
        int r = j;
        while (anc[r] != -1 && anc[r] != i) { int t = anc[r]; anc[r] = i; r = t; }
        if (anc[r] == -1) { anc[r] = i; par[r] = i; }
      }
    }
  };
  std::vector<int> pm(perm0, perm0 + n);
  etree(pm, ip, parent);
  // postorder (children ascending), iterative DFS
  std::vector<int> head(n, -1), next(n, -1);
  for (int j = n - 1; j >= 0; --j)
    if (parent[j] >= 0) { next[j] = head[parent[j]]; head[parent[j]] = j; }
  std::vector<int> post;
  post.reserve(n);
  std::vector<int> stack;
  for (int r = 0; r < n; ++r) {
    if (parent[r] >= 0) continue;
    stack.push_back(r);
    while (!stack.empty()) {
      int j = stack.back();
      int c = head[j];
      if (c >= 0) {  // descend into the next child
        head[j] = next[c];
        stack.push_back(c);
      } else {
        post.push_back(j);
        stack.pop_back();
      }
    }
  }
  if ((int)post.size() != n) throw std::runtime_error("etree postorder lost nodes");
  std::vector<int> pm2(n);
  for (int k = 0; k < n; ++k) pm2[k] = pm[post[k]];
  pm.swap(pm2);
  for (int i = 0; i < n; ++i) ip[pm[i]] = i;
  etree(pm, ip, parent);
  // column counts (incl. diagonal) by row subtrees
  std::vector<int> cc(n, 0), mark(n, -1), nchild(n, 0);
  for (int i = 0; i < n; ++i) {
    mark[i] = i;
    ++cc[i];
    int o = pm[i];
    for (int64_t q = adj_ptr[o]; q < adj_ptr[o + 1]; ++q) {
      int k = ip[adj[q]];
      while (k >= 0 && k < i && mark[k] != i) { mark[k] = i; ++cc[k]; k = parent[k]; }
    }
  }
  for (int j = 0; j < n; ++j)
    if (parent[j] >= 0) nchild[parent[j]]++;
  // fundamental supernodes: [sb, se) ranges in postorder
  std::vector<int> sn_of(n), sb, se;
  for (int j = 0; j < n; ++j) {
    bool join = j > 0 && parent[j - 1] == j && nchild[j] == 1 && cc[j - 1] == cc[j] + 1;
    if (!join) { sb.push_back(j); se.push_back(j + 1); }
    else se.back() = j + 1;
    sn_of[j] = (int)sb.size() - 1;
  }
  // relaxed amalgamation: a supernode whose parent starts right after it (the
  // last child, contiguous in postorder) merges into the parent when both
  // together have at most `relax` columns
  int NS = (int)sb.size();
  std::vector<int> sp(NS, -1);
  for (int t = 0; t < NS; ++t) {
    int pj = parent[se[t] - 1];
    sp[t] = pj >= 0 ? sn_of[pj] : -1;
  }
  std::vector<int> rep(NS);
  std::iota(rep.begin(), rep.end(), 0);
  std::vector<int> cb(sb), ce(se);
  for (int t = 0; t < NS; ++t) {  // children before parents in postorder
    int pt = sp[t];
    if (pt < 0) continue;
    int a = rep[t];
    while (rep[a] != a) a = rep[a];
    if (ce[a] == sb[pt] && (ce[a] - cb[a]) + (se[pt] - sb[pt]) <= relax) {
      // merge group a (ending right before pt) into pt
      cb[pt] = cb[a];
      rep[a] = pt;
    }
  }
  // fronts = surviving groups, in postorder of their last column
  std::vector<int> group_of(NS);
  std::vector<int> fronts;
  for (int t = 0; t < NS; ++t) {
    int a = t;
    while (rep[a] != a) a = rep[a];
    group_of[t] = a;
  }
  std::vector<int> fid(NS, -1);
  for (int t = 0; t < NS; ++t)
    if (group_of[t] == t) { fid[t] = (int)fronts.size(); fronts.push_back(t); }
  S.nfronts = (int)fronts.size();
  S.col_begin.resize(S.nfronts);
  S.col_end.resize(S.nfronts);
  S.parent.assign(S.nfronts, -1);
  std::vector<std::vector<int>> kids(S.nfronts);
  for (int f = 0; f < S.nfronts; ++f) {
    int t = fronts[f];
    S.col_begin[f] = cb[t];
    S.col_end[f] = se[t];
    int pj = parent[se[t] - 1];
    if (pj >= 0) {
      int pf = fid[group_of[sn_of[pj]]];
      S.parent[f] = pf;
      kids[pf].push_back(f);
    }
  }
  S.perm = pm;
  finish_symbolic(S, adj_ptr, adj, kids);
}

}  // namespace jgs2
