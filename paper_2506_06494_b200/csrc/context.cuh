// Device context of one JGS2 solver instance (one GPU, one stream).
#pragma once
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "physics.cuh"
#include "symbolic.h"

namespace jgs2 {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define JGS2_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::jgs2::Error(-2, std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

constexpr int kBlock = 256;
constexpr int kMaxPartials = 4096;  // grid-reduction partial slots per reduction
constexpr int kPairRow = 10;

// Reduction result slots (device doubles), see Ctx::res.
enum ResSlot {
  R_ENERGY = 0,   // total energy of the last energy launch
  R_GRADSQ,       // sum of g_asm^2 over free vertices
  R_DX2,          // |dx|^2
  R_DXMAX,        // max_v |dx_v|
  R_CAP,          // feasibility cap (min)
  R_EBEFORE,      // energy at the sweep start
  R_AUX,          // scratch (barrier sum, max step)
  R_CAP2,         // feasibility cap: active pair-table bound
  R_NSLOTS = 8
};

// Broadphase grid buffers (see broadphase.cuh; grow on demand).
struct TriGrid {
  long long cap = 0, n = 0;
  long long* counts = nullptr;  // nst + 1
  long long* off = nullptr;
  unsigned long long *keys_a = nullptr, *keys_b = nullptr;
  int *tris_a = nullptr, *tris_b = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  double cell = 0.0;
  long long* dbox = nullptr;  // device cell bounding box (min xyz, max xyz)
  long long box[6] = {0, 0, 0, -1, -1, -1};
  int sy = 0, sz = 0;         // key shifts (broadphase.cuh)
};

// Sorted (key, id) entry list of the hierarchical cap grids (hier_grid.cuh).
struct HierList {
  long long cap = 0, n = 0;
  long long *cnt = nullptr, *off = nullptr;
  unsigned *ka = nullptr, *kb = nullptr;  // dense cell index (all levels)
  int *ia = nullptr, *ib = nullptr;
  int *flag = nullptr, *rix = nullptr;    // run starts and their exclusive scan
  int *run_begin = nullptr, *run_body = nullptr;  // body runs of the sorted entries
  int *cstart = nullptr, *cend = nullptr; // per-cell run range [cstart, cend)
  long long ncells_cap = 0;
};

// Collective layer of a partitioned solve (one rank per GPU):
// in-place all-reduce of device buffers on the context stream. NCCL in
// production; a host callback (torch.distributed/gloo) for multi-process
// tests that share one GPU.
enum CommType { CT_F64 = 0, CT_I32 = 1, CT_U64 = 2 };
enum CommOp { CO_SUM = 0, CO_MAX = 1 };
struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() {}
  virtual void allreduce(void* buf, size_t count, int type, int op, cudaStream_t s) = 0;
};

// Device-side factor of the free-vertex rest Hessian (supernodal, ND order).
struct Factor {
  bool ready = false;
  bool ordering_metis = false;
  Symbolic sym;
  int nfree = 0;
  int nfronts = 0, nlevels = 0;
  int64_t nnz_alloc = 0;  // doubles in L storage
  double* L = nullptr;
  // per-front (device)
  int* f_colbeg = nullptr;     // first DOF position
  int* f_ns = nullptr;         // columns (DOF)
  int* f_nr = nullptr;         // struct rows (DOF)
  int* f_ld = nullptr;         // panel leading dimension (nf rounded up to even)
  int64_t* f_loff = nullptr;   // panel offset in L (ld = ns + nr)
  int64_t* f_uoff = nullptr;   // update-vector offset (nr entries)
  int64_t* f_woff = nullptr;   // work-vector offset (nf entries)
  int* f_cptr = nullptr;       // children CSR
  int* f_clist = nullptr;
  int64_t* f_sptr = nullptr;   // struct DOF list CSR (DOF units)
  int* f_sdof = nullptr;       // global DOF positions of struct rows
  int* f_rmap = nullptr;       // per front: struct row -> local index in parent (DOF)
  int* level_fronts = nullptr; // fronts grouped by level
  std::vector<int> level_ptr;  // host
  std::vector<int> level_maxnf;
  int4* fwd_tasks = nullptr;   // (front, row_begin, row_end)
  int4* fwdn_tasks = nullptr;  // narrow fronts: (front, 64-row chunk)
  std::vector<int> fwdn_level_ptr;
  int4* bwd_tasks = nullptr;   // (front, col_begin, col_end)
  int4* bwdn_tasks = nullptr;  // narrow fronts: (front, <= 8 columns)
  std::vector<int> bwdn_level_ptr;
  struct SplitTask* split_tasks = nullptr;  // top levels: (64-row block, column chunk)
  std::vector<int> split_level_ptr;
  double* split_part = nullptr;
  unsigned* split_ticket = nullptr;
  std::vector<int> fwd_level_ptr, bwd_level_ptr, fwd_level_smem, bwd_level_smem;
  std::vector<int64_t> asm_level_ptr, gat_level_ptr;
  int64_t* asm_dst = nullptr;  // flat forward assembly map
  int* asm_b = nullptr;
  int64_t* asm_cp = nullptr;
  int64_t* asm_src = nullptr;
  int64_t* gat_dst = nullptr;  // flat backward gather map
  int* gat_src = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  int64_t graph_launches = 0;
  // host copies of the front metadata (selected inversion, selinv.cuh)
  std::vector<int> h_ns, h_nr, h_fld, h_pfront, h_pos;
  std::vector<int64_t> h_loff, h_sptr;
  double* Z = nullptr;         // selected inverse, layout of L (after jgs2_selected_inverse)
  int* d_pfront = nullptr;
  int* d_cbeg = nullptr;
  int* d_cend = nullptr;
  int64_t* d_spptr = nullptr;
  int* d_spos = nullptr;
  double* u = nullptr;         // update vectors
  double* w = nullptr;         // work vectors (global fallback)
  int max_nf = 0;
  double seconds = 0.0;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;

  // sizes
  int nv = 0, ne = 0, nfree = 0, smax = 0, gmax = 1, nuniq = 0;
  int64_t nslots = 0;
  bool have_model = false, have_pre = false;
  double norm_scale = 1.0;
  // config
  double tol_dx = 1e-3, alpha_floor = 1e-6;
  int max_outer = 500, max_halvings = 30;
  bool local_line_search = true, track_energy = true;
  int last_halvings = 0;  // previous sweep's backtracking halvings (sizes the first trial batch)
  int mode = 0;                // 0 jacobi, 1 gauss_seidel
  bool plain = false;          // subspace="none" (plain.cuh): no precompute, no factor
  double* mplus_all = nullptr; // plain mode: projected reduced Hessian of every element (45 each)
  int* hess_list_all = nullptr;
  // Gauss-Seidel colour groups: free vertices by colour (ascending id)
  std::vector<int> color_ptr;
  int* color_verts = nullptr;
  double* x0 = nullptr;        // sweep-start positions (GS)
  double* gs_gsq = nullptr;    // per-colour grad_sq (device)
  double* cap_x = nullptr;     // jgs2_step_cap scratch (host x, dx in)
  double* cap_dx = nullptr;

  // partition (jgs2_set_partition): this rank owns vertices [own_v0, own_v1)
  // and elements [own_e0, own_e1) -- whole bodies, so the rest Hessian is
  // block diagonal across ranks. Reductions run over fixed chunks aligned to
  // body boundaries, so the result is the same for every rank count.
  int own_v0 = 0, own_v1 = 0, own_e0 = 0, own_e1 = 0;
  bool partitioned = false;
  Comm* comm = nullptr;
  std::vector<int> body_v, body_e;  // body boundaries (vertex / element ids), size nbodies+1
  int2* chunks = nullptr;           // element chunks, then vertex chunks: [begin, end)
  int nchunk_e = 0, nchunk_v = 0;
  int chunk_own0 = 0, chunk_own1 = 0;      // owned element chunks [c0, c1)
  int vchunk_own0 = 0, vchunk_own1 = 0;    // owned vertex chunks (global chunk ids)
  double* cpart = nullptr;          // (kTrialBatch + 1) * nchunks partial sums
  std::vector<int> chunk_first_e, chunk_first_v;  // first chunk of each body (+ end)
  bool own_stream = true;
  bool owns(int v) const { return v >= own_v0 && v < own_v1; }

  // static device data
  int4* tets = nullptr;
  double* dminv = nullptr;     // ne*9
  double4* eprops = nullptr;   // (vol, mu, lam, qmass)
  int* inc_ptr = nullptr;      // nv+1
  int* inc = nullptr;          // 4ne: e*4+slot, ascending e per vertex
  double* mass = nullptr;
  uint8_t* fixed = nullptr;
  int* pos = nullptr;          // nv: factor position of a free vertex, -1 fixed
  int* free_list = nullptr;    // nfree
  double* rest = nullptr;      // nv*3
  std::vector<double> h_rest;  // host copy for ND coordinates
  std::vector<int64_t> h_tets;
  std::vector<uint8_t> h_fixed;

  // precompute (per vertex rows, zero for vertices without a basis)
  double* gbar = nullptr;      // nv*9
  int* group = nullptr;        // nv*gmax (vertex ids, -1 pad)
  double* grows = nullptr;     // nv*3*3*gmax
  int* cub_u = nullptr;        // nv*smax unique-element index, -1 invalid
  double* cub_w = nullptr;     // nv*smax
  double* cub_rows = nullptr;  // nv*smax*36
  int4* cub_verts = nullptr;   // nv*smax
  double* crest = nullptr;     // nv*9 rest constant C_v
  int* uniq = nullptr;         // nuniq element ids
  double* mplus = nullptr;     // nuniq*45 per-sweep projected reduced Hessians
  int* hess_count = nullptr;   // indefinite-element count (pass 1 -> pass 2)
  int* hess_list = nullptr;    // compacted indefinite elements
  cudaStream_t stream2 = nullptr;  // side stream for the element-Hessian passes
  cudaStream_t solve_side = nullptr;  // factor solve: a level's narrow launches beside the wide ones
  cudaEvent_t ev_sfork = nullptr, ev_sjoin = nullptr;
  cudaStream_t vp_stream = nullptr;  // vertex pass under the pair detection
  cudaEvent_t ev_vfork = nullptr, ev_vjoin = nullptr;
  bool vp_overlap = [] {
    const char* e = getenv("JGS2_VP_OVERLAP");
    return !(e && e[0] == '0');
  }();
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool hess_pending = false;
  // retained rows CSR for contact coupling rows (local_solver.py:85-112)
  int* vr_ptr = nullptr;       // nv+1
  int* vr_keys = nullptr;
  double* vr_rows = nullptr;

  // state
  double h = 0.01;
  double* x = nullptr;         // nv*3
  double* z = nullptr;
  double* R = nullptr;         // nv*9
  double* gasm = nullptr;      // nv*3
  double* b = nullptr;         // 3*nfree (rhs, then forward result; ND order)
  double* q = nullptr;         // 3*nfree collect solution q (ND order)
  double* delta = nullptr;     // nv*3
  double* alpha0 = nullptr;    // nv
  int* kacc = nullptr;         // nv accept iteration of the local search
  double* dx = nullptr;        // nv*3
  double* xprev = nullptr;     // frame state (device frame driver)
  double* vel = nullptr;
  double* dz = nullptr;
  double* xprev0 = nullptr;    // frame state saved by jgs2_set_frame_state
  double* vel0 = nullptr;
  double gravity[3] = {0.0, 0.0, 0.0};
  bool rot_valid = false;

  // reductions
  double* partials = nullptr;  // R_NSLOTS * kMaxPartials
  unsigned* counters = nullptr;
  double* res = nullptr;       // R_NSLOTS results (device)
  double* h_res = nullptr;     // pinned mirror
  // local line search bookkeeping
  unsigned long long* ls_max = nullptr;  // (max_halvings+2) maxima of alpha0 over unaccepted (bits)
  int* ls_cnt = nullptr;                  // (max_halvings+2) counts of unaccepted
  int* ls_final = nullptr;                // [T, floor_flag]

  // contact
  bool has_barrier = false;
  double dhat = 0, kappa = 0;
  int nplanes = 0, nbodies = 1, nsv = 0, nst = 0;
  double* planes = nullptr;    // nplanes*6 (point, normal)
  std::vector<double> h_planes;
  int* sv = nullptr;           // surface vertices
  std::vector<uint8_t> h_surface;  // host surface-vertex mask
  int* st = nullptr;           // surface tris *3
  int* vbody = nullptr;        // nv
  int* tbody = nullptr;        // nst
  // pair table (device, capacity cap_pairs)
  int64_t cap_pairs = 0;
  double* pairs = nullptr;     // rows of kPairRow
  int* npairs_d = nullptr;
  int* pair_count_sv = nullptr;  // per surface vertex counts (plane+tri)
  int* pair_off_sv = nullptr;
  int npairs = 0;              // host copy for the current pair table
  int* vp_cnt = nullptr;       // per-vertex pair counts (nv+1)
  int* vp_ptr = nullptr;       // vertex -> pair incidence CSR (nv+1)
  int* vp_list = nullptr;      // pair*4 + member slot
  double* pair_g = nullptr;    // per pair 12 gradient
  double* pair_h = nullptr;    // per pair 144 projected Hessian
  double* pair_e = nullptr;    // per pair barrier energy
  int* flag_d = nullptr;       // infeasibility flag
  double grid_cell = 1.0;      // broadphase cell size
  TriGrid pair_grid;
  HierList hier;               // both hierarchical grids (hier_grid.cuh)
  int* hier_lev = nullptr;     // per object (surface vertices, then triangles)
  unsigned* hier_masks = nullptr;
  double* bbox_part = nullptr;  // surface bounding-box reduction (hier_grid.cuh)
  double* bbox_res = nullptr;
  int* cand_v = nullptr;       // trial candidate pairs (vertex, triangle)
  int* cand_t = nullptr;
  int64_t cand_cap = 0;
  int ncand = 0;               // -1: too many candidates, exact per-trial detection
  long long* cand_cnt = nullptr;
  long long* cand_off = nullptr;
  double* tpart = nullptr;     // trial-batch partial sums
  double* tres = nullptr;      // trial-batch results (elastic+inertia | barrier)
  int* tflags = nullptr;       // trial-batch infeasibility flags
  void* scan_temp = nullptr;   // CUB scan workspace
  size_t scan_temp_bytes = 0;

  // measurement: per-phase CUDA-event intervals (accumulated at sync points)
  bool profiling = false;
  static constexpr int kPhases = 11;
  double phase_ms[kPhases] = {0};
  int64_t phase_launch[kPhases] = {0};
  double phase_bytes[kPhases] = {0};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> event_pool;
  int cur_phase = -1;
  int64_t launch_mark = 0;
  cudaEvent_t cur_start = nullptr;
  cudaEvent_t tstart = nullptr, tstop = nullptr;
  cudaEvent_t take_event() {
    if (event_pool.empty()) {
      cudaEvent_t e;
      JGS2_CUDA(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  void phase_begin(int p, double bytes) {
    phase_bytes[p] += bytes;
    if (!profiling) return;
    cur_phase = p;
    launch_mark = launches;
    cur_start = take_event();
    JGS2_CUDA(cudaEventRecord(cur_start, stream));
  }
  void phase_end() {
    if (!profiling || cur_phase < 0) return;
    cudaEvent_t stop = take_event();
    JGS2_CUDA(cudaEventRecord(stop, stream));
    phase_launch[cur_phase] += launches - launch_mark;
    pending.push_back({cur_phase, {cur_start, stop}});
    cur_phase = -1;
  }
  void collect_phases() {  // call after a stream sync; side-stream intervals may still be running
    size_t keep = 0;
    for (auto& p : pending) {
      if (cudaEventQuery(p.second.second) == cudaErrorNotReady) {
        pending[keep++] = p;
        continue;
      }
      float ms = 0.f;
      JGS2_CUDA(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
      phase_ms[p.first] += ms;
      event_pool.push_back(p.second.first);
      event_pool.push_back(p.second.second);
    }
    pending.resize(keep);
    cudaGetLastError();  // clear the not-ready status
  }

  Factor fac;
  // element Hessians under the factor solve, blocks per SM (0 = before k_local)
  int hess_overlap = [] {
    const char* e = getenv("JGS2_HESS_OVERLAP");
    return e ? atoi(e) : 1;
  }();
  int ordering = -1;           // jgs2_set_ordering: 1 METIS ND, 0 geometric ND, -1 default (METIS)
  std::shared_ptr<struct TrainOut> train;  // scalable precompute output (train.cuh)
  cublasHandle_t cublas = nullptr;
  cusolverDnHandle_t cusolver = nullptr;

  std::vector<void*> allocs;
  template <class T>
  T* alloc(size_t count) {
    if (count == 0) count = 1;
    void* p = nullptr;
    JGS2_CUDA(cudaMalloc(&p, count * sizeof(T)));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const T* host, size_t count) {
    T* d = alloc<T>(count);
    if (count) JGS2_CUDA(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, stream));
    return d;
  }
  void sync() {
    JGS2_CUDA(cudaStreamSynchronize(stream));
    if (!pending.empty()) collect_phases();
  }
  void check_launch() {
    ++launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(-2, std::string("kernel launch: ") + cudaGetErrorString(e));
  }
  // all-reduce of a device buffer across ranks (no-op on one rank)
  void allreduce(void* buf, size_t count, int type, int op) {
    if (comm && comm->world > 1) comm->allreduce(buf, count, type, op, stream);
  }
  ~Ctx();
};

inline int grid_for(int64_t n, int block = kBlock) {
  int64_t g = (n + block - 1) / block;
  return (int)(g < 1 ? 1 : g);
}
// grid for grid-stride reductions (<= kMaxPartials blocks)
inline int red_grid(int64_t n) { int g = grid_for(n); return g < 148 * 8 ? g : 148 * 8; }
inline bool contact_active(const Ctx& C) { return C.has_barrier && C.nsv > 0; }

// ------------------------------------------------------ deterministic reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

enum RedOp { OP_SUM = 0, OP_MAX = 1, OP_MIN = 2 };

template <int OP>
__device__ __forceinline__ double red_combine(double a, double b) {
  return OP == OP_SUM ? a + b : (OP == OP_MAX ? fmax(a, b) : fmin(a, b));
}
template <int OP>
__device__ __forceinline__ double red_warp(double v) {
  return OP == OP_SUM ? warp_sum(v) : (OP == OP_MAX ? warp_max(v) : warp_min(v));
}

// Block reduction (fixed tree), result valid in thread 0.
template <int OP>
__device__ double block_reduce(double v) {
  __shared__ double sh[32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = red_warp<OP>(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  int nw = (blockDim.x + 31) >> 5;
  double ident = OP == OP_SUM ? 0.0 : (OP == OP_MAX ? -INFINITY : INFINITY);
  v = (threadIdx.x < nw) ? sh[threadIdx.x] : ident;
  if (wid == 0) v = red_warp<OP>(v);
  return v;
}

// Single-pass grid reduction: every block deposits its partial; the last
// block to finish combines all partials in block order (deterministic) and
// writes res[slot]. gridDim.x must be <= kMaxPartials.
template <int OP>
__device__ void grid_reduce(double v, double* partials, unsigned* counter, double* out) {
  double bsum = block_reduce<OP>(v);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bsum;
    __threadfence();
    unsigned t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double ident = OP == OP_SUM ? 0.0 : (OP == OP_MAX ? -INFINITY : INFINITY);
  double acc = ident;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
    acc = red_combine<OP>(acc, ((volatile double*)partials)[i]);
  acc = block_reduce<OP>(acc);
  if (threadIdx.x == 0) {
    *out = acc;
    *counter = 0u;
  }
}

}  // namespace jgs2
