// Symbolic analysis for the rest-Hessian factor used by the exact reduced
// collect (reference: SciPy SuperLU on Hbar, subspace.py:126-130 /
// local_solver.py:115-126).  The CUDA path replaces SuperLU-COLAMD with a
// supernodal Cholesky on a geometric nested-dissection ordering of the free
// vertices (3x3 blocks); every ND node is one front (supernode):
//   leaves = dense fronts of <= leaf_size vertices, separators = one front.
// Fronts are numbered in postorder; positions (the permuted vertex order)
// are assigned so that each front's columns are contiguous.
#pragma once
#include <cstdint>
#include <vector>

namespace jgs2 {

struct Symbolic {
  int n = 0;                        // free vertices (graph nodes)
  std::vector<int> perm;            // perm[pos] = node
  std::vector<int> iperm;           // iperm[node] = pos
  int nfronts = 0;
  std::vector<int> parent;          // front -> parent front (-1 = root)
  std::vector<int> col_begin;       // front columns = positions [col_begin, col_end)
  std::vector<int> col_end;
  std::vector<int64_t> struct_ptr;  // row structure beyond the columns (positions, ascending)
  std::vector<int> struct_pos;
  std::vector<int> level;           // 0 = leaf; parent level > child level
  int nlevels = 0;
  std::vector<int> child_ptr, child_list;  // children per front (ascending front id)
  // node counts of the factor in 3x3-block (vertex) units and in DOFs
  int64_t nnz_dof = 0;              // sum over fronts of ns(ns+1)/2 + nr*ns (DOF units)
};

// Build the ND ordering + front tree.
//   adj_ptr/adj : symmetric adjacency of the free-vertex graph (no self loops
//                 required; they are ignored)
//   coords      : n x 3 coordinates (rest positions) for geometric bisection
void build_symbolic(int n, const int64_t* adj_ptr, const int32_t* adj, const double* coords,
                    int leaf_size, Symbolic& out);

// Front tree from a given ordering perm (perm[pos] = node), e.g. METIS
// nested dissection: etree postorder, fundamental supernodes, relaxed
// amalgamation up to `relax` vertices per merged front.
void build_symbolic_perm(int n, const int64_t* adj_ptr, const int32_t* adj, const int32_t* perm, int relax,
                         Symbolic& out);

}  // namespace jgs2
