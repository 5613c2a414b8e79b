// Selected inversion of the rest-Hessian factor (scalable precompute,
// SURVEY §8(f)#1): Z = Hbar^-1 on the sparsity pattern of the supernodal
// factor, from the partitioned-inverse panels P = [L11^-1; L21 L11^-1].
//
// Takahashi's equations per front, parents before children:
//   Z_SJ = -Z_SS P21,   Z_JJ = P11^T P11 - P21^T Z_SJ
// where Z_SS (the front's structure rows, a clique of the filled graph) is
// gathered from the parent's dense front matrix. Every entry of Hbar^-1
// between adjacent vertices of the filled graph -- the vertex's own block,
// its 1-ring, and every vertex of its front -- is then available. Those are
// exactly the blocks the reference's per-vertex bases read
// (subspace.py:133-203: Gbar_v = -[(Hbar^-1)_vv]^-1, rows U_v[w] =
// -(Hbar^-1)_wv Gbar_v), without the dense N x 3 column per vertex.
// Z is stored with the layout of L (front f: column-major fld x ns panel).
#pragma once
#include "context.cuh"

namespace jgs2 {

// lower entries (a >= b) of a child's Z_SS from the parent's dense front
// matrix (column major, ld nfp), via the child's struct-row -> parent map
__global__ void k_gather_zss(int nr, const int* rmap, const double* Zp, int nfp, double* Zc, int ldc) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nr * nr) return;
  int a = (int)(idx % nr), b = (int)(idx / nr);
  if (a < b) return;
  int ra = rmap[a], rb = rmap[b];  // ra >= rb (monotone map)
  Zc[(int64_t)b * ldc + a] = Zp[(int64_t)rb * nfp + ra];
}

// (Hbar^-1)_{w v} 3x3 blocks (row-major) for vertex pairs; found[k] = 0 when
// the pair is not adjacent in the filled graph. Fixed vertices: zero block.
struct SelinvDev {
  const int* pos;        // nv: factor position of a free vertex, -1 fixed
  const int* pfront;     // position -> front
  const int* cbeg;       // front -> first column position (vertex units)
  const int* cend;
  const int64_t* sptr;   // front -> struct positions (vertex units)
  const int* spos;
  const int64_t* loff;   // front panel offset
  const int* fld;        // leading dimension
  const double* Z;
};

__device__ __forceinline__ int find_pos(const int* a, int64_t lo, int64_t hi, int key) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return (int)lo;
}

__global__ void k_inverse_blocks(SelinvDev S, int n, const int64_t* pv_, const int64_t* pw_, double* out,
                                 int* found) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int v = (int)pv_[k], w = (int)pw_[k];
  double* o = out + 9 * (size_t)k;
  int pv = S.pos[v], pw = S.pos[w];
  if (pv < 0 || pw < 0) {
#pragma unroll
    for (int q = 0; q < 9; ++q) o[q] = 0.0;
    found[k] = 1;
    return;
  }
  int fv = S.pfront[pv];
  int ns = 3 * (S.cend[fv] - S.cbeg[fv]);
  int c = 3 * (pv - S.cbeg[fv]);
  int r = -1;
  if (pw >= S.cbeg[fv] && pw < S.cend[fv]) {
    r = 3 * (pw - S.cbeg[fv]);
  } else {
    int64_t a = S.sptr[fv], b = S.sptr[fv + 1];
    int i = find_pos(S.spos, a, b, pw);
    if (i < b && S.spos[i] == pw) r = ns + 3 * (int)(i - a);
  }
  if (r >= 0) {  // column v of front fv holds (row w, col v)
    const double* Z = S.Z + S.loff[fv];
    int ld = S.fld[fv];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        int rr = r + i, cc = c + j;
        o[3 * i + j] = rr >= cc ? Z[(int64_t)cc * ld + rr] : Z[(int64_t)rr * ld + cc];
      }
    found[k] = 1;
    return;
  }
  // v in the structure of w's front: (Hbar^-1)_{wv} = [(Hbar^-1)_{vw}]^T
  int fw = S.pfront[pw];
  int nsw = 3 * (S.cend[fw] - S.cbeg[fw]);
  int64_t a = S.sptr[fw], b = S.sptr[fw + 1];
  int i0 = find_pos(S.spos, a, b, pv);
  if (i0 < b && S.spos[i0] == pv) {
    const double* Z = S.Z + S.loff[fw];
    int ld = S.fld[fw];
    int cw = 3 * (pw - S.cbeg[fw]), rv = nsw + 3 * (int)(i0 - a);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) o[3 * i + j] = Z[(int64_t)(cw + i) * ld + rv + j];
    found[k] = 1;
    return;
  }
#pragma unroll
  for (int q = 0; q < 9; ++q) o[q] = 0.0;
  found[k] = 0;
}

// Z on the factor's pattern (device, layout of L). Fronts in reverse
// postorder (parents first); each keeps a dense nf x nf front matrix (lower
// triangle) until its children have gathered their Z_SS from it.
inline void selected_inverse(Ctx& C) {
  Factor& F = C.fac;
  Symbolic& S = F.sym;
  const int NF = S.nfronts;
  if (!F.Z) F.Z = C.alloc<double>(std::max<int64_t>(F.nnz_alloc, 1));
  std::vector<int> pending(NF, 0);
  for (int f = 0; f < NF; ++f)
    if (S.parent[f] >= 0) pending[S.parent[f]]++;
  std::vector<double*> Zf(NF, nullptr);
  const double one = 1.0, zero = 0.0, mone = -1.0;
  cublasSetStream(C.cublas, C.stream);
  for (int f = NF - 1; f >= 0; --f) {
    const int ns = F.h_ns[f], nr = F.h_nr[f], nf = ns + nr, ld = F.h_fld[f];
    const double* P = F.L + F.h_loff[f];
    JGS2_CUDA(cudaMallocAsync(&Zf[f], std::max<size_t>((size_t)nf * nf, 1) * sizeof(double), C.stream));
    double* Zd = Zf[f];
    const int p = S.parent[f];
    if (nr > 0) {
      if (p < 0 || !Zf[p]) throw Error(-2, "selected inverse: missing parent front");
      const int nfp = F.h_ns[p] + F.h_nr[p];
      int64_t tot = (int64_t)nr * nr;
      k_gather_zss<<<grid_for(tot), kBlock, 0, C.stream>>>(nr, F.f_rmap + F.h_sptr[f], Zf[p], nfp,
                                                           Zd + (int64_t)ns * nf + ns, nf);
      C.check_launch();
      if (ns > 0 &&
          cublasDsymm(C.cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, nr, ns, &mone,
                      Zd + (int64_t)ns * nf + ns, nf, P + ns, ld, &zero, Zd + ns, nf) != CUBLAS_STATUS_SUCCESS)
        throw Error(-2, "cublasDsymm failed");
    }
    if (ns > 0) {
      if (cublasDsyrk(C.cublas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, ns, ns, &one, P, ld, &zero, Zd, nf) !=
          CUBLAS_STATUS_SUCCESS)
        throw Error(-2, "cublasDsyrk failed");
      if (nr > 0 &&
          cublasDgemm(C.cublas, CUBLAS_OP_T, CUBLAS_OP_N, ns, ns, nr, &mone, P + ns, ld, Zd + ns, nf, &one, Zd,
                      nf) != CUBLAS_STATUS_SUCCESS)
        throw Error(-2, "cublasDgemm failed");
      JGS2_CUDA(cudaMemcpy2DAsync(F.Z + F.h_loff[f], (size_t)ld * sizeof(double), Zd, (size_t)nf * sizeof(double),
                                  (size_t)nf * sizeof(double), ns, cudaMemcpyDeviceToDevice, C.stream));
    }
    if (p >= 0 && --pending[p] == 0) {
      JGS2_CUDA(cudaFreeAsync(Zf[p], C.stream));
      Zf[p] = nullptr;
    }
    if (pending[f] == 0) {
      JGS2_CUDA(cudaFreeAsync(Zf[f], C.stream));
      Zf[f] = nullptr;
    }
  }
  for (int f = 0; f < NF; ++f)
    if (Zf[f]) JGS2_CUDA(cudaFreeAsync(Zf[f], C.stream));
  // lookup metadata
  std::vector<int> pfront(S.n, -1), cb(NF), ce(NF);
  for (int f = 0; f < NF; ++f) {
    cb[f] = S.col_begin[f];
    ce[f] = S.col_end[f];
    for (int q = S.col_begin[f]; q < S.col_end[f]; ++q) pfront[q] = f;
  }
  F.d_pfront = C.upload(pfront.data(), pfront.size());
  F.d_cbeg = C.upload(cb.data(), NF);
  F.d_cend = C.upload(ce.data(), NF);
  F.d_spptr = C.upload(S.struct_ptr.data(), S.struct_ptr.size());
  F.d_spos = C.upload(S.struct_pos.data(), S.struct_pos.size());
  C.sync();
}

inline SelinvDev selinv_dev(const Ctx& C) {
  SelinvDev d;
  d.pos = C.pos;
  d.pfront = C.fac.d_pfront;
  d.cbeg = C.fac.d_cbeg;
  d.cend = C.fac.d_cend;
  d.sptr = C.fac.d_spptr;
  d.spos = C.fac.d_spos;
  d.loff = C.fac.f_loff;
  d.fld = C.fac.f_ld;
  d.Z = C.fac.Z;
  return d;
}

}  // namespace jgs2
