// Fill of the rest-Hessian Cholesky factor under two orderings (SURVEY
// §8(d): the judge compares nnz(L) of the solve's ordering with METIS nested
// dissection). Exact column counts from the elimination tree, O(nnz(L)).
#include <cusolverSp.h>
#include <cusparse.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace jgs2 {

// nnz of the lower Cholesky factor (incl. diagonal) of the n-node symmetric
// pattern (ptr/adj, any self loops ignored) under the ordering p
// (p[new] = old): elimination tree (Liu, path compression), then each row's
// structure is the union of the etree paths from its lower neighbours.
int64_t chol_nnz(int n, const int64_t* ptr, const int32_t* adj, const int32_t* p) {
  std::vector<int> ip(n), parent(n, -1), anc(n, -1), mark(n, -1);
  for (int i = 0; i < n; ++i) ip[p[i]] = i;
  for (int i = 0; i < n; ++i) {
    int o = p[i];
    for (int64_t q = ptr[o]; q < ptr[o + 1]; ++q) {
      int j = ip[adj[q]];
      if (j >= i) continue;
      int r = j;
      while (anc[r] != -1 && anc[r] != i) {
        int t = anc[r];
        anc[r] = i;
        r = t;
      }
      if (anc[r] == -1) {
        anc[r] = i;
        parent[r] = i;
      }
    }
  }
  int64_t nnz = 0;
  for (int i = 0; i < n; ++i) {
    mark[i] = i;
    ++nnz;
    int o = p[i];
    for (int64_t q = ptr[o]; q < ptr[o + 1]; ++q) {
      int k = ip[adj[q]];
      while (k < i && mark[k] != i) {
        mark[k] = i;
        ++nnz;
        k = parent[k];
        if (k < 0) break;
      }
    }
  }
  return nnz;
}

// METIS nested-dissection ordering of the pattern (cuSOLVER's
// cusolverSpXcsrmetisndHost), p[new] = old
void metis_nd(int n, const int64_t* ptr, const int32_t* adj, int32_t* p) {
  // symmetric CSR without self loops, int32 offsets
  std::vector<int> rp(n + 1, 0), ci;
  ci.reserve(ptr[n]);
  for (int i = 0; i < n; ++i) {
    for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q)
      if (adj[q] != i) ci.push_back(adj[q]);
    rp[i + 1] = (int)ci.size();
  }
  cusolverSpHandle_t h = nullptr;
  cusparseMatDescr_t d = nullptr;
  if (cusolverSpCreate(&h) != CUSOLVER_STATUS_SUCCESS) throw std::runtime_error("cusolverSpCreate failed");
  cusparseCreateMatDescr(&d);
  cusparseSetMatType(d, CUSPARSE_MATRIX_TYPE_GENERAL);
  cusparseSetMatIndexBase(d, CUSPARSE_INDEX_BASE_ZERO);
  cusolverStatus_t st = cusolverSpXcsrmetisndHost(h, n, (int)ci.size(), d, rp.data(), ci.data(), nullptr, p);
  cusparseDestroyMatDescr(d);
  cusolverSpDestroy(h);
  if (st != CUSOLVER_STATUS_SUCCESS) throw std::runtime_error("cusolverSpXcsrmetisndHost failed");
}

// METIS nested dissection of each connected component on its own,
// components concatenated in order of their smallest node. A body's ordering
// (and so its factor, bit for bit) does not depend on the other bodies in
// the graph: a partitioned solve factoring a subset of the bodies
// reproduces the single-GPU factor of each.
void metis_nd_components(int n, const int64_t* ptr, const int32_t* adj, int32_t* p) {
  std::vector<int> comp(n, -1), order;
  order.reserve(n);
  int out = 0;
  std::vector<int64_t> cptr;
  std::vector<int32_t> cadj;
  std::vector<int> loc(n, -1);
  for (int s = 0; s < n; ++s) {
    if (comp[s] >= 0) continue;
    order.clear();
    order.push_back(s);
    comp[s] = s;
    for (size_t h = 0; h < order.size(); ++h) {
      int u = order[h];
      for (int64_t q = ptr[u]; q < ptr[u + 1]; ++q) {
        int w = adj[q];
        if (comp[w] < 0) { comp[w] = s; order.push_back(w); }
      }
    }
    std::sort(order.begin(), order.end());  // component nodes ascending
    const int m = (int)order.size();
    for (int k = 0; k < m; ++k) loc[order[k]] = k;
    cptr.assign(m + 1, 0);
    cadj.clear();
    for (int k = 0; k < m; ++k) {
      int u = order[k];
      for (int64_t q = ptr[u]; q < ptr[u + 1]; ++q) cadj.push_back(loc[adj[q]]);
      cptr[k + 1] = (int64_t)cadj.size();
    }
    std::vector<int32_t> cp(m);
    if (m <= 2) {
      for (int k = 0; k < m; ++k) cp[k] = k;
    } else {
      metis_nd(m, cptr.data(), cadj.data(), cp.data());
    }
    for (int k = 0; k < m; ++k) p[out++] = order[cp[k]];
  }
}

}  // namespace jgs2
