// C-ABI implementation of the B200-native JGS2 runtime iteration.
// See include/jgs2.h for the contract and DESIGN.md for the data layout.
#include <cuda_profiler_api.h>
#include "../../include/jgs2.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>

#include "context.cuh"
#include "factor.cuh"
#include "sweep.cuh"
#include "contact.cuh"
#include "trials.cuh"
#include "hier_grid.cuh"
#include "partition.cuh"
#include "comm.cuh"
#include "selinv.cuh"
#include "train.cuh"
#include "plain.cuh"

namespace jgs2 {  // fill.cpp
int64_t chol_nnz(int n, const int64_t* ptr, const int32_t* adj, const int32_t* p);
}  // namespace jgs2

using namespace jgs2;

jgs2::Ctx::~Ctx() {
  if (stream) cudaStreamSynchronize(stream);
  for (void* p : allocs) cudaFree(p);
  if (h_res) cudaFreeHost(h_res);
  for (auto& p : pending) { cudaEventDestroy(p.second.first); cudaEventDestroy(p.second.second); }
  for (auto e : event_pool) cudaEventDestroy(e);
  if (tstart) cudaEventDestroy(tstart);
  if (tstop) cudaEventDestroy(tstop);
  if (cublas) cublasDestroy(cublas);
  if (cusolver) cusolverDnDestroy(cusolver);
  if (stream2) cudaStreamSynchronize(stream2);
  tri_grid_free(pair_grid);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (stream2) cudaStreamDestroy(stream2);
  if (ev_sfork) cudaEventDestroy(ev_sfork);
  if (ev_sjoin) cudaEventDestroy(ev_sjoin);
  if (solve_side) cudaStreamDestroy(solve_side);
  if (vp_stream) cudaStreamSynchronize(vp_stream);
  if (ev_vfork) cudaEventDestroy(ev_vfork);
  if (ev_vjoin) cudaEventDestroy(ev_vjoin);
  if (vp_stream) cudaStreamDestroy(vp_stream);
  if (fac.graph_exec) cudaGraphExecDestroy(fac.graph_exec);
  delete comm;
  if (stream && own_stream) cudaStreamDestroy(stream);
}

struct jgs2_ctx {
  Ctx c;
};
struct jgs2_sym {
  Symbolic s;
};

namespace {

template <class F>
int32_t guarded(jgs2_ctx* ctx, F&& fn) {
  if (!ctx) return JGS2_E_ARG;
  // a call that threw between a side-stream fork and its join (element
  // Hessians under the solve, vertex pass under the pair detection) leaves
  // that work in flight: order it before anything later on the main stream,
  // and never let a later sweep join the stale Hessians as its own
  auto settle = [](Ctx& C) {
    if (C.hess_pending) {
      if (C.ev_join) cudaStreamWaitEvent(C.stream, C.ev_join, 0);
      C.hess_pending = false;
    }
    if (C.ev_vjoin) cudaStreamWaitEvent(C.stream, C.ev_vjoin, 0);
    cudaGetLastError();
  };
  try {
    ctx->c.err.clear();
    JGS2_CUDA(cudaSetDevice(ctx->c.device));
    fn(ctx->c);
    return JGS2_OK;
  } catch (const Error& e) {
    ctx->c.err = e.what();
    settle(ctx->c);
    return e.code;
  } catch (const std::exception& e) {
    ctx->c.err = e.what();
    settle(ctx->c);
    return JGS2_E_ARG;
  }
}

DevModel devmodel(const Ctx& C) {
  DevModel m;
  m.nv = C.nv; m.ne = C.ne; m.smax = C.smax; m.gmax = C.gmax; m.nfree = C.nfree;
  m.tets = C.tets; m.dminv = C.dminv; m.eprops = C.eprops; m.inc_ptr = C.inc_ptr; m.inc = C.inc;
  m.mass = C.mass; m.fixed = C.fixed; m.pos = C.pos; m.free_list = C.free_list;
  m.v0 = C.own_v0; m.v1 = C.own_v1;
  return m;
}

LocalArgs localargs(Ctx& C) {
  LocalArgs a;
  memset(&a, 0, sizeof(a));
  a.R = C.R; a.gasm = C.gasm; a.b = C.q; a.gbar = C.gbar; a.group = C.group; a.grows = C.grows;
  a.cub_u = C.cub_u; a.cub_w = C.cub_w; a.cub_rows = C.cub_rows; a.cub_verts = C.cub_verts;
  a.nv = C.nv;
  a.crest = C.crest; a.mplus = C.mplus; a.h = C.h;
  a.delta = C.delta; a.alpha0 = C.alpha0; a.kacc = C.kacc;
  a.line_search = C.local_line_search ? 1 : 0;
  a.max_halvings = C.max_halvings;
  a.ls_max = C.ls_max; a.ls_cnt = C.ls_cnt;
  return a;
}


void require_ready(Ctx& C) {
  if (!C.have_model) throw Error(JGS2_E_ARG, "model not set");
  if (!C.have_pre) throw Error(JGS2_E_ARG, "precompute not set");
  if (!C.plain && !C.fac.ready) throw Error(JGS2_E_ARG, "rest factor not built (jgs2_factor_rest)");
}

// ---- algorithmic bytes per phase: unique bytes a
// phase must move at least once; re-reads served by L2 are not counted.
double bytes_vertex(const Ctx& C) { return C.ne * (16.0 + 72 + 32 + 16) + C.nv * (24.0 + 24 + 8 + 72 + 24); }
double bytes_rhs(const Ctx& C) { return C.nfree * (4.0 + 4 + 72 + 24 + 24); }
double bytes_solve(const Ctx& C) { return 16.0 * (double)C.fac.sym.nnz_dof + 4.0 * 8 * 3 * C.nfree; }
double bytes_cub(const Ctx& C) { return C.nuniq * (4.0 + 16 + 72 + 32 + 96 + 360); }
double bytes_local(const Ctx& C) {
  return C.nfree * (4.0 + 72 * 4 + 24 + 4 + 36 + 8 + 24) + C.nslots * (4.0 + 8 + 288 + 16) +
         C.nuniq * 360.0 + C.nv * 72.0;
}
double bytes_energy(const Ctx& C, bool dx) { return C.ne * (16.0 + 72 + 32) + C.nv * (24.0 + 24 + 8 + (dx ? 24 : 0)); }
double bytes_final(const Ctx& C) { return C.nv * (24.0 * 4) + C.nv * (24.0 + 8 + 4 + 24); }

// Energy at x + gamma*dx (dx may be null) into res[slot]; includes the
// barrier energies of the pairs active at that position.
void launch_energy(Ctx& C, const double* dx, double gamma, int slot) {
  DevModel m = devmodel(C);
  int n = std::max(C.ne, C.nv);
  C.phase_begin(5, bytes_energy(C, dx != nullptr));
  k_energy<<<red_grid(n), kBlock, 0, C.stream>>>(m, C.x, dx, gamma, C.z, C.h,
                                                  C.partials + slot * kMaxPartials,
                                                  C.counters + slot, C.res + slot);
  C.check_launch();
  C.phase_end();
  if (contact_active(C)) {
    C.phase_begin(9, 0.0);
    contact_energy_at(C, dx, gamma, slot);
    C.phase_end();
  }
}

void vertex_pass(Ctx& C, bool rot) {
  DevModel m = devmodel(C);
  C.phase_begin(0, bytes_vertex(C));
  int nown = C.own_v1 - C.own_v0;  // this rank's vertices (all of them on one GPU)
  if (rot) k_vertex_pass<true><<<grid_for(nown), kBlock, 0, C.stream>>>(m, C.x, C.z, C.h, C.R, C.gasm);
  else k_vertex_pass<false><<<grid_for(nown), kBlock, 0, C.stream>>>(m, C.x, C.z, C.h, C.R, C.gasm);
  C.check_launch();
  C.phase_end();
  if (rot) C.rot_valid = true;
}

// The vertex pass on a side stream under the pair detection (both read x
// only; the detection is latency bound with host syncs for its counts):
// joined before the pair gradients are added to g_asm.
void vertex_pass_async(Ctx& C, bool rot) {
  DevModel m = devmodel(C);
  JGS2_CUDA(cudaEventRecord(C.ev_vfork, C.stream));
  JGS2_CUDA(cudaStreamWaitEvent(C.vp_stream, C.ev_vfork, 0));
  C.phase_bytes[0] += bytes_vertex(C);
  cudaEvent_t a = nullptr;
  if (C.profiling) {
    a = C.take_event();
    JGS2_CUDA(cudaEventRecord(a, C.vp_stream));
  }
  int nown = C.own_v1 - C.own_v0;
  if (rot) k_vertex_pass<true><<<grid_for(nown), kBlock, 0, C.vp_stream>>>(m, C.x, C.z, C.h, C.R, C.gasm);
  else k_vertex_pass<false><<<grid_for(nown), kBlock, 0, C.vp_stream>>>(m, C.x, C.z, C.h, C.R, C.gasm);
  C.check_launch();
  if (C.profiling) {
    cudaEvent_t b = C.take_event();
    JGS2_CUDA(cudaEventRecord(b, C.vp_stream));
    C.phase_launch[0] += 1;
    C.pending.push_back({0, {a, b}});
  }
  JGS2_CUDA(cudaEventRecord(C.ev_vjoin, C.vp_stream));
  if (rot) C.rot_valid = true;
}

void vertex_pass_join(Ctx& C) { JGS2_CUDA(cudaStreamWaitEvent(C.stream, C.ev_vjoin, 0)); }

// grad_sq over the free vertices (local_solver.py:602-603) in vertex chunks:
// this rank's chunks, all-reduced, combined in chunk order into res[R_GRADSQ]
void gradsq_chunks(Ctx& C) {
  double* row = C.cpart + (size_t)kTrials * (C.nchunk_e + C.nchunk_v);
  if (C.partitioned)
    JGS2_CUDA(cudaMemsetAsync(row, 0, (size_t)(C.nchunk_e + C.nchunk_v) * sizeof(double), C.stream));
  int n = C.vchunk_own1 - C.vchunk_own0;
  if (n > 0) {
    k_chunk_gradsq<<<n, kBlock, 0, C.stream>>>(C.chunks, C.vchunk_own0, C.gasm, C.fixed, row);
    C.check_launch();
  }
  C.allreduce(row + C.nchunk_e, C.nchunk_v, CT_F64, CO_SUM);
  k_reduce_chunks<<<1, kBlock, 0, C.stream>>>(row + C.nchunk_e, C.nchunk_v, 0, 1, C.res + R_GRADSQ);
  C.check_launch();
}

void collect(Ctx& C) {
  if (C.plain) {  // no reduced collect in plain mode (local_solver.py:597): grad_sq only
    gradsq_chunks(C);
    return;
  }
  DevModel m = devmodel(C);
  C.phase_begin(1, bytes_rhs(C));
  k_rhs<<<grid_for(C.nfree), kBlock, 0, C.stream>>>(m, C.R, C.gasm, C.b);
  C.check_launch();
  gradsq_chunks(C);
  C.phase_end();
  C.phase_begin(2, bytes_solve(C));
  factor_solve(C);
  C.phase_end();
}

// Element Hessians at x on the side stream: compute-bound FP64 work that
// overlaps the memory-bound vertex pass + collect on the main stream
// (independent: H_cur depends on x only); joined before k_local.
void hessians_async(Ctx& C, int blocks_per_sm = 0) {
  if (C.nuniq == 0 || C.hess_pending) return;
  JGS2_CUDA(cudaEventRecord(C.ev_fork, C.stream));
  JGS2_CUDA(cudaStreamWaitEvent(C.stream2, C.ev_fork, 0));
  C.phase_bytes[3] += bytes_cub(C);
  cudaEvent_t a = nullptr;
  if (C.profiling) {
    a = C.take_event();
    JGS2_CUDA(cudaEventRecord(a, C.stream2));
  }
  launch_element_mplus(C.nuniq, C.uniq, C.x, C.tets, C.dminv, C.eprops, C.mplus, C.hess_count,
                       C.hess_list, C.stream2, blocks_per_sm);
  C.launches += 3;
  C.check_launch();
  if (C.profiling) {
    cudaEvent_t b = C.take_event();
    JGS2_CUDA(cudaEventRecord(b, C.stream2));
    C.phase_launch[3] += 1;
    C.pending.push_back({3, {a, b}});
  }
  JGS2_CUDA(cudaEventRecord(C.ev_join, C.stream2));
  C.hess_pending = true;
}

void hessians_join(Ctx& C) {
  if (!C.hess_pending) return;
  JGS2_CUDA(cudaStreamWaitEvent(C.stream, C.ev_join, 0));
  C.hess_pending = false;
}

// Local systems of the free vertices, or of the vertices in `list` (a
// Gauss-Seidel colour; the element Hessians are then already in place).
void local_systems(Ctx& C, double* A_out, double* g_out, double* corr_out, const int* list = nullptr,
                   int nlist = 0, bool hess_ready = false) {
  DevModel m = devmodel(C);
  if (list) {
    m.nfree = nlist;
    m.free_list = list;
  } else if (!hess_ready) {
    hessians_async(C);  // no-op if already in flight
    hessians_join(C);
  }
  C.phase_begin(4, bytes_local(C));
  JGS2_CUDA(cudaMemsetAsync(C.ls_cnt, 0, (C.max_halvings + 2) * sizeof(int), C.stream));
  JGS2_CUDA(cudaMemsetAsync(C.ls_max, 0, (C.max_halvings + 2) * sizeof(unsigned long long), C.stream));
  LocalArgs a = localargs(C);
  a.A_out = A_out; a.g_out = g_out; a.corr_out = corr_out;
  a.npairs = contact_active(C) ? C.npairs : 0;
  a.x = C.x; a.pairs = C.pairs; a.pair_g = C.pair_g; a.pair_h = C.pair_h;
  a.vp_ptr = C.vp_ptr; a.vp_list = C.vp_list; a.planes = C.planes;
  a.vr_ptr = C.vr_ptr; a.vr_keys = C.vr_keys; a.vr_rows = C.vr_rows;
  if (C.plain) {  // own-stencil systems: projected Hessians of every element at the current x
    C.phase_end();
    C.phase_begin(3, C.ne * 580.0);
    launch_element_mplus(C.ne, nullptr, C.x, C.tets, C.dminv, C.eprops, C.mplus_all, C.hess_count,
                         C.hess_list_all, C.stream);
    C.launches += 3;
    C.phase_end();
    C.phase_begin(4, 0.0);
    PlainArgs pa{C.mplus_all, C.z, C.dhat, C.kappa};
    if (m.nfree > 0) k_plain_local<<<grid_for(m.nfree, 128), 128, 0, C.stream>>>(m, a, pa);
  } else if (m.nfree > 0) {
    k_local<<<grid_for(m.nfree, 128), 128, 0, C.stream>>>(m, a);
  }
  C.check_launch();
  // the local search's halving rounds are global (local_solver.py:539-553):
  // counts of unaccepted vertices and the max alpha0 among them per round
  C.allreduce(C.ls_cnt, C.max_halvings + 2, CT_I32, CO_SUM);
  C.allreduce(C.ls_max, C.max_halvings + 2, CT_U64, CO_MAX);
  C.phase_end();
}

// Candidate cross-body (vertex, triangle) pairs for every trial position
// x + gamma dx, gamma <= gmax (see trials.cuh).
constexpr long long kCandBudget = 1LL << 26;

void trial_candidates(Ctx& C, double gmax, const double* bb = nullptr) {
  C.ncand = 0;
  if (!contact_active(C) || !use_tri_grid(C)) return;
  long long n = hier_candidates(C, C.x, C.dx, gmax, kCandBudget, bb);
  C.ncand = n < 0 ? -1 : (int)n;  // -1: a huge step, exact per-trial detection
}

// E(x + gamma_k dx) for n <= kTrialBatch gammas (host results), with
// infeasibility flags (a barrier distance <= 0).
void trial_energies(Ctx& C, const double* gam, int n, double* E, bool* infeasible) {
  DevModel m = devmodel(C);
  Gammas G;
  G.n = n;
  for (int k = 0; k < kTrialBatch; ++k) G.g[k] = k < n ? gam[k] : 0.0;
  int grid = red_grid(std::max(C.ne, C.nv));
  C.phase_begin(5, bytes_energy(C, true));
  {  // elastic + inertia per chunk (this rank's chunks), all-reduced, chunk order
    const int nch = C.nchunk_e + C.nchunk_v;
    TrialGammas TG;
    TG.n = n;
    for (int k = 0; k < kTrials; ++k) TG.g[k] = G.g[k];
    if (C.partitioned) JGS2_CUDA(cudaMemsetAsync(C.cpart, 0, (size_t)n * nch * sizeof(double), C.stream));
    int ne_own = C.chunk_own1 - C.chunk_own0, nv_own = C.vchunk_own1 - C.vchunk_own0;
    if (ne_own > 0) {
      k_energy_chunks<<<ne_own, kBlock, 0, C.stream>>>(m, C.chunks, C.chunk_own0, C.nchunk_e, nch, C.x, C.dx,
                                                        TG, C.z, C.h, C.cpart);
      C.check_launch();
    }
    if (nv_own > 0) {
      k_energy_chunks<<<nv_own, kBlock, 0, C.stream>>>(m, C.chunks, C.vchunk_own0, C.nchunk_e, nch, C.x, C.dx,
                                                        TG, C.z, C.h, C.cpart);
      C.check_launch();
    }
    C.allreduce(C.cpart, (size_t)n * nch, CT_F64, CO_SUM);
    k_reduce_chunks<<<1, kBlock, 0, C.stream>>>(C.cpart, nch, (size_t)nch, n, C.tres);
    C.check_launch();
  }
  C.phase_end();
  bool contact = contact_active(C);
  if (contact && C.ncand < 0) {
    // fallback: exact pair detection at every trial position (reference
    // find_pairs(x_try)), one trial at a time
    double* h = C.h_res;
    JGS2_CUDA(cudaMemcpyAsync(h, C.tres, n * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    C.sync();
    std::vector<double> el(h, h + n);
    for (int k = 0; k < n; ++k) {
      C.phase_begin(9, 0.0);
      contact_find_pairs(C, C.x, C.dx, gam[k]);
      bool inf = contact_infeasible(C);
      double bar = 0.0;
      if (C.npairs > 0) {
        k_pair_energy_sum<<<std::min(grid_for(C.npairs), 64), kBlock, 0, C.stream>>>(
            C.npairs, C.pairs, C.dhat, C.kappa, C.partials + R_AUX * kMaxPartials, C.counters + R_AUX,
            C.res + R_AUX);
        C.check_launch();
        JGS2_CUDA(cudaMemcpyAsync(&bar, C.res + R_AUX, sizeof(double), cudaMemcpyDeviceToHost, C.stream));
        C.sync();
      }
      C.phase_end();
      E[k] = el[k] + bar;
      infeasible[k] = inf;
    }
    return;
  }
  if (contact) {
    C.phase_begin(9, 0.0);
    ContactDev cd = contactdev(C);
    int nb = std::max(1, std::min(red_grid((int64_t)C.nsv * C.nplanes + C.ncand), 1024));
    JGS2_CUDA(cudaMemsetAsync(C.tflags, 0, kTrialBatch * sizeof(int), C.stream));
    k_barrier_batch<<<nb, kBlock, 0, C.stream>>>(cd, C.ncand, C.cand_v, C.cand_t, C.x, C.dx, G,
                                                 C.tpart + kTrialBatch * kMaxPartials, C.tflags);
    C.check_launch();
    k_reduce_batch<<<1, kBlock, 0, C.stream>>>(C.tpart + kTrialBatch * kMaxPartials, nb, n,
                                               C.tres + kTrialBatch);
    C.check_launch();
    C.phase_end();
  }
  double* h = C.h_res;  // pinned scratch (>= 3 * kTrialBatch doubles)
  JGS2_CUDA(cudaMemcpyAsync(h, C.tres, 2 * kTrialBatch * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  JGS2_CUDA(cudaMemcpyAsync(h + 2 * kTrialBatch, C.tflags, kTrialBatch * sizeof(int), cudaMemcpyDeviceToHost,
                            C.stream));
  C.sync();
  const int* fl = reinterpret_cast<const int*>(h + 2 * kTrialBatch);
  for (int k = 0; k < n; ++k) {
    E[k] = contact ? h[k] + h[kTrialBatch + k] : h[k];
    infeasible[k] = contact && fl[k] != 0;
  }
}

// ---- Gauss-Seidel colour updates (local_solver.py:627-649)
// sum of g_asm^2 over a colour's vertices (deterministic two-level reduction)
__global__ void k_sumsq_list(const int* list, int n, const double* g, double* partials, unsigned* counter,
                             double* out) {
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int v = list[i];
    acc += g[3 * v] * g[3 * v] + g[3 * v + 1] * g[3 * v + 1] + g[3 * v + 2] * g[3 * v + 2];
  }
  grid_reduce<OP_SUM>(acc, partials, counter, out);
}

// step = alpha delta for a colour's vertices (k_apply_alpha's rule); x += step, dx += step
__global__ void k_apply_list(const int* list, int n, const double* delta, const double* alpha0, const int* kacc,
                             const int* lsf, int line_search, int max_halvings, double alpha_floor, double* x,
                             double* dx) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int v = list[i];
  double al = line_search ? final_alpha(alpha0[v], kacc[v], lsf, max_halvings, alpha_floor) : 1.0;
  for (int c = 0; c < 3; ++c) {
    double st = al * delta[3 * v + c];
    x[3 * v + c] += st;
    dx[3 * v + c] += st;
  }
}

// Colour sweeps: q0 (collect) and the element Hessians (corrections) at the
// sweep start; per colour ascending, pairs + assembled field at the current
// positions, local systems with q0 / corrections, the colour's local search,
// x += step. Leaves C.x = x0 (sweep start) and C.dx = the summed steps for
// the global backtracking. Returns sum of grad_sq; acts += activations.
double gauss_seidel_colours(Ctx& C, int* acts, bool hess_ready) {
  bool guard = C.local_line_search;
  size_t bytes = 3 * (size_t)C.nv * sizeof(double);
  if (!hess_ready) {
    hessians_async(C);
    hessians_join(C);
  }
  if (!C.x0) {
    C.x0 = C.alloc<double>(3 * (size_t)C.nv);
    C.gs_gsq = C.alloc<double>(std::max<size_t>(C.color_ptr.size(), 1));
  }
  JGS2_CUDA(cudaMemcpyAsync(C.x0, C.x, bytes, cudaMemcpyDeviceToDevice, C.stream));
  JGS2_CUDA(cudaMemsetAsync(C.dx, 0, bytes, C.stream));
  int nc = (int)C.color_ptr.size() - 1;
  std::vector<int> act(std::max(nc, 1), 0);
  int* hacts = reinterpret_cast<int*>(C.h_res + 32);  // pinned scratch (<= 32 colours per chunk)
  for (int c = 0; c < nc; ++c) {
    const int* list = C.color_verts + C.color_ptr[c];
    int n = C.color_ptr[c + 1] - C.color_ptr[c];
    if (n == 0) continue;
    if (c > 0) {  // positions moved: pairs and assembled field at the current x
      if (contact_active(C)) {
        C.phase_begin(7, 0.0);
        contact_find_pairs(C, C.x, nullptr, 0.0);
        C.phase_end();
        if (contact_infeasible(C)) throw Error(JGS2_E_INFEASIBLE, "barrier distance <= 0 during a colour sweep");
      }
      vertex_pass(C, false);
      if (contact_active(C)) {
        C.phase_begin(7, 0.0);
        contact_add_gradients(C);
        C.phase_end();
      }
    }
    k_sumsq_list<<<std::min(red_grid(n), 256), kBlock, 0, C.stream>>>(
        list, n, C.gasm, C.partials + R_AUX * kMaxPartials, C.counters + R_AUX, C.gs_gsq + c);
    C.check_launch();
    local_systems(C, nullptr, nullptr, nullptr, list, n);
    if (guard) {
      k_ls_final<<<1, 1, 0, C.stream>>>(C.max_halvings, C.alpha_floor, C.ls_cnt, C.ls_max, C.ls_final);
      C.check_launch();
      JGS2_CUDA(cudaMemcpyAsync(hacts + (c % 32), C.ls_final + 2, sizeof(int), cudaMemcpyDeviceToHost, C.stream));
    }
    k_apply_list<<<grid_for(n), kBlock, 0, C.stream>>>(list, n, C.delta, C.alpha0, C.kacc, C.ls_final,
                                                       guard ? 1 : 0, C.max_halvings, C.alpha_floor, C.x,
                                                       C.dx);
    C.check_launch();
    if (guard && (c % 32 == 31 || c == nc - 1)) {
      C.sync();
      for (int k = c - (c % 32); k <= c; ++k) act[k] = hacts[k % 32];
    }
  }
  std::vector<double> gsq(std::max(nc, 1), 0.0);
  if (nc > 0)
    JGS2_CUDA(cudaMemcpyAsync(gsq.data(), C.gs_gsq, nc * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  JGS2_CUDA(cudaMemcpyAsync(C.x, C.x0, bytes, cudaMemcpyDeviceToDevice, C.stream));
  C.sync();
  double tot = 0.0;
  for (int c = 0; c < nc; ++c) {
    tot += gsq[c];
    if (C.color_ptr[c + 1] > C.color_ptr[c]) *acts += act[c];
  }
  return tot;
}

// One sweep on the device state. rot: compute rotations at x (outer_solve);
// otherwise use the context's current rotations.
void sweep_core(Ctx& C, bool rot, jgs2_sweep_info* info) {
  require_ready(C);
  if (!rot && !C.rot_valid && !C.plain) throw Error(JGS2_E_ARG, "rotations not set");
  DevModel m = devmodel(C);
  bool guard = C.local_line_search;
  // Optional (JGS2_HESS_EARLY=1): element Hessians at x (compute-bound FP64,
  // x only) on the low-priority side stream under the latency-bound pair
  // detection and vertex pass, joined before the collect. Measured neutral on
  // B200 (C4 49.2-51.1 vs 50.6 sweeps/s): the Hessian grid saturates the SMs,
  // so there is little idle time to fill. Overlapping them uncapped with the
  // solve is slower (the persistent solve CTAs lose residency: 31.9 vs 26.4
  // ms/sweep in round 1); the default below caps them at one block per SM.
  static const bool early_env = getenv("JGS2_HESS_EARLY") != nullptr;
  const bool early = early_env && contact_active(C);
  if (early) hessians_async(C);
  const bool vp_async = C.vp_overlap && contact_active(C);
  if (vp_async) vertex_pass_async(C, rot);
  if (contact_active(C)) {  // pairs at x (local_solver.py:612)
    C.phase_begin(7, 0.0);
    contact_find_pairs(C, C.x, nullptr, 0.0);
    C.phase_end();
    if (vp_async) vertex_pass_join(C);
    if (contact_infeasible(C)) throw Error(JGS2_E_INFEASIBLE, "barrier distance <= 0 at the sweep start");
  }
  if (!vp_async) vertex_pass(C, rot);
  if (contact_active(C)) {
    C.phase_begin(7, 0.0);
    contact_add_gradients(C);
    C.phase_end();
  }
  hessians_join(C);  // no-op unless launched above
  // The element Hessians (FP64 ALU, x only) run on the side stream under the
  // factor solve (HBM), capped at one resident block per SM so the solve's
  // CTAs keep the rest of each SM; joined before k_local. C4: 81.8 -> 86.5
  // sweeps/s (solve 6.9 -> 8.1 ms, the 1.8 ms Hessian phase hidden; 2 blocks
  // per SM: 82.2). JGS2_HESS_OVERLAP=<blocks per SM>, 0 = before k_local.
  if (C.hess_overlap > 0 && !early && !C.plain) hessians_async(C, C.hess_overlap);
  collect(C);
  const int npairs_x = C.npairs;  // pairs at the sweep-start x
  const bool gs = C.mode == 1 && C.color_ptr.size() > 1;
  if (gs && C.partitioned) throw Error(JGS2_E_ARG, "the partitioned solve runs Jacobi sweeps only");
  int gs_acts = 0;
  double gs_gradsq = 0.0;
  if (gs) {
    gs_gradsq = gauss_seidel_colours(C, &gs_acts, early);
  } else {
    local_systems(C, nullptr, nullptr, nullptr, nullptr, 0, early);
    C.phase_begin(6, bytes_final(C));
    if (guard) {
      k_ls_final<<<1, 1, 0, C.stream>>>(C.max_halvings, C.alpha_floor, C.ls_cnt, C.ls_max, C.ls_final);
      C.check_launch();
    }
    k_apply_alpha<<<grid_for(C.nv), kBlock, 0, C.stream>>>(m, C.delta, C.alpha0, C.kacc, C.ls_final,
                                                            guard ? 1 : 0, C.max_halvings,
                                                            C.alpha_floor, C.dx);
    C.check_launch();
    // dx: each rank holds its own vertices' rows (zeros elsewhere)
    C.allreduce(C.dx, 3 * (size_t)C.nv, CT_F64, CO_SUM);
    C.phase_end();
  }
  double gamma = 1.0, energy = 0.0, cap_used = 1.0;
  int halvings = 0;
  bool have_energy = false;
  int pairs_at_start = npairs_x;
  int acts_ls = gs_acts;
  if (guard) {
    // global backtracking (local_solver.py:555-577), trials in batches
    bool cap_needed = contact_active(C) && (npairs_x > 0 || C.nplanes > 0);
    double cap = 1.0;
    double bb[6];
    bool have_bb = false;
    if (cap_needed) {
      C.phase_begin(8, 0.0);
      // the pair table bounds the cap only when it holds the pairs at x
      // (after colour sweeps it holds the last colour's pairs)
      cap = contact_step_cap(C, C.x, C.dx, !gs, bb);
      have_bb = use_tri_grid(C);
      C.phase_end();
    }
    if (!gs)
      JGS2_CUDA(cudaMemcpyAsync(&acts_ls, C.ls_final + 2, sizeof(int), cudaMemcpyDeviceToHost, C.stream));
    if (contact_active(C)) {
      C.phase_begin(9, 0.0);
      trial_candidates(C, cap, have_bb ? bb : nullptr);
      C.phase_end();
    }
    cap_used = cap;
    const int MH = C.max_halvings;
    std::vector<double> gam(MH + 2);
    gam[0] = cap;
    for (int j = 1; j <= MH + 1; ++j) gam[j] = gam[j - 1] * 0.5;
    double e0 = 0.0;
    int accepted = -1, next = 0;
    double Eb[kTrialBatch];
    bool bad[kTrialBatch];
    double gb[kTrialBatch];
    bool first = true;
    while (accepted < 0 && next <= MH) {
      int n = 0, base = next;
      if (first) gb[n++] = 0.0;  // e_before rides in the first batch
      // the first batch carries e_before plus one trial, or a full batch when
      // the previous sweep needed halvings (results do not depend on batching)
      // the first batch is sized to the previous sweep's halvings + 3 trials
      // (C4: 87.3 -> 87.9 sweeps/s, energy phase 0.46 -> 0.38 ms; a larger
      // need takes a second, full batch). JGS2_TRIAL_SLACK=k (-1: full batch).
      static const int slack = [] {
        const char* e = getenv("JGS2_TRIAL_SLACK");
        return e ? atoi(e) : 3;
      }();
      int want = first ? (C.last_halvings > 0 ? (slack >= 0 ? std::min(kTrialBatch - 1, C.last_halvings + slack)
                                                            : kTrialBatch - 1)
                                              : 1)
                       : kTrialBatch;
      for (int q = 0; q < want && next <= MH; ++q) gb[n++] = gam[next++];
      if (next > MH && n < kTrialBatch) gb[n++] = gam[MH + 1];  // floor energy (track_energy)
      trial_energies(C, gb, n, Eb, bad);
      int k0 = 0;
      if (first) {
        if (bad[0]) throw Error(JGS2_E_INFEASIBLE, "barrier distance <= 0 at the sweep start");
        e0 = Eb[0];
        k0 = 1;
        first = false;
      }
      for (int k = k0; k < n; ++k) {
        int j = base + (k - k0);
        if (j > MH) {  // the floor position (only its energy is used)
          energy = Eb[k];
          have_energy = true;
          break;
        }
        double et = bad[k] ? INFINITY : Eb[k];
        if (et <= e0 + 1e-12 * std::fabs(e0)) {
          accepted = j;
          energy = Eb[k];
          have_energy = true;
          break;
        }
      }
    }
    if (accepted >= 0) {
      halvings = accepted;
      gamma = gam[accepted];
    } else {
      halvings = MH + 1;
      gamma = gam[MH + 1];
    }
    C.last_halvings = halvings;
  }
  C.phase_begin(6, C.nv * 96.0);
  k_finalize<<<red_grid(C.nv), kBlock, 0, C.stream>>>(C.nv, C.x, C.dx, gamma, guard ? 1 : 0,
                                                       C.partials + R_DX2 * kMaxPartials,
                                                       C.counters + R_DX2, C.res);
  C.check_launch();
  C.phase_end();
  if (C.track_energy && !have_energy) {  // energy at the new x (gamma = 0 on the updated state)
    double g0 = 0.0, E1;
    bool b1;
    if (contact_active(C)) {
      C.phase_begin(9, 0.0);
      trial_candidates(C, 0.0);
      C.phase_end();
    }
    trial_energies(C, &g0, 1, &E1, &b1);
    energy = b1 ? INFINITY : E1;
  }
  JGS2_CUDA(cudaMemcpyAsync(C.h_res, C.res, R_NSLOTS * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  int n_indef = 0;
  if (C.partitioned) {
    if (C.nuniq == 0) JGS2_CUDA(cudaMemsetAsync(C.hess_count, 0, sizeof(int), C.stream));
    C.allreduce(C.hess_count, 1, CT_I32, CO_SUM);
  }
  if (C.nuniq > 0 || C.partitioned)
    JGS2_CUDA(cudaMemcpyAsync(C.h_res + R_NSLOTS + 1, C.hess_count, sizeof(int), cudaMemcpyDeviceToHost, C.stream));
  C.sync();
  if (C.nuniq > 0 || C.partitioned) memcpy(&n_indef, C.h_res + R_NSLOTS + 1, sizeof(int));
  if (info) {
    info->line_search_activations = guard ? acts_ls + halvings : 0;
    info->n_indefinite = n_indef;
    double gsq = gs ? gs_gradsq : C.h_res[R_GRADSQ];
    info->grad_sq = gsq;
    info->grad_norm = std::sqrt(gsq);
    info->max_local_step = C.h_res[R_DXMAX];
    info->dx_norm = C.norm_scale * std::sqrt(C.h_res[R_DX2]);
    info->energy = energy;
    info->halvings = halvings;
    info->n_pairs = pairs_at_start;
    info->gamma = gamma;
    info->cap = cap_used;
  }
}

}  // namespace

// ============================================================= lifecycle
extern "C" {

int32_t jgs2_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

jgs2_ctx* jgs2_create(int32_t device) {
  int n = jgs2_device_count();
  if (n <= 0 || device < 0 || device >= n) return nullptr;
  jgs2_ctx* ctx = new jgs2_ctx();
  ctx->c.device = device;
  // main stream at the highest priority: its latency-bound contact kernels are
  // scheduled ahead of the side stream's element-Hessian blocks
  int prio_lo = 0, prio_hi = 0;
  if (cudaSetDevice(device) != cudaSuccess || cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi) != cudaSuccess ||
      cudaStreamCreateWithPriority(&ctx->c.stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess) {
    fprintf(stderr, "jgs2_create: %s\n", cudaGetErrorString(cudaGetLastError()));
    delete ctx;
    return nullptr;
  }
  try {
    Ctx& C = ctx->c;
    C.partials = C.alloc<double>((size_t)R_NSLOTS * kMaxPartials);
    C.counters = C.alloc<unsigned>(R_NSLOTS);
    C.res = C.alloc<double>(R_NSLOTS);
    JGS2_CUDA(cudaMemset(C.counters, 0, R_NSLOTS * sizeof(unsigned)));
    JGS2_CUDA(cudaMemset(C.res, 0, R_NSLOTS * sizeof(double)));
    JGS2_CUDA(cudaMallocHost(&C.h_res, 8 * R_NSLOTS * sizeof(double)));
    C.tpart = C.alloc<double>(2 * (size_t)kTrialBatch * kMaxPartials);
    C.tres = C.alloc<double>(2 * kTrialBatch);
    C.tflags = C.alloc<int>(kTrialBatch);
    C.hess_count = C.alloc<int>(2);
    JGS2_CUDA(cudaStreamCreateWithPriority(&C.stream2, cudaStreamNonBlocking, prio_lo));
    JGS2_CUDA(cudaEventCreateWithFlags(&C.ev_fork, cudaEventDisableTiming));
    JGS2_CUDA(cudaEventCreateWithFlags(&C.ev_join, cudaEventDisableTiming));
    JGS2_CUDA(cudaStreamCreateWithFlags(&C.solve_side, cudaStreamNonBlocking));
    JGS2_CUDA(cudaStreamCreateWithFlags(&C.vp_stream, cudaStreamNonBlocking));
    JGS2_CUDA(cudaEventCreateWithFlags(&C.ev_vfork, cudaEventDisableTiming));
    JGS2_CUDA(cudaEventCreateWithFlags(&C.ev_vjoin, cudaEventDisableTiming));
    JGS2_CUDA(cudaEventCreateWithFlags(&C.ev_sfork, cudaEventDisableTiming));
    JGS2_CUDA(cudaEventCreateWithFlags(&C.ev_sjoin, cudaEventDisableTiming));
    cudaFuncSetAttribute(k_mplus_project, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kProjSmemBytes);
    cudaFuncSetAttribute(k_mplus_full, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kHessSmemBytes);
    cudaFuncSetAttribute(k_element_mplus, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kHessSmemBytes);

  } catch (const std::exception& e) {
    fprintf(stderr, "jgs2_create: %s\n", e.what());
    delete ctx;
    return nullptr;
  }
  return ctx;
}

jgs2_ctx* jgs2_create_on_stream(int32_t device, void* stream) {
  jgs2_ctx* ctx = jgs2_create(device);
  if (ctx && stream) {  // run on the caller's stream (not destroyed with the context)
    cudaStreamSynchronize(ctx->c.stream);
    cudaStreamDestroy(ctx->c.stream);
    ctx->c.stream = static_cast<cudaStream_t>(stream);
    ctx->c.own_stream = false;
  }
  return ctx;
}

int32_t jgs2_nccl_unique_id(uint8_t* id128) {
  if (!id128) return JGS2_E_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return JGS2_E_CUDA;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id128, &id, sizeof(id));
  return JGS2_OK;
}

namespace {
void check_comm_args(Ctx& C, int32_t world, int32_t rank) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(JGS2_E_ARG, "invalid world/rank");
  if (C.comm) throw Error(JGS2_E_ARG, "communicator already set");
  if (C.fac.ready || C.have_pre) throw Error(JGS2_E_ARG, "set the communicator before the factor and precompute");
}
}  // namespace

int32_t jgs2_set_comm_nccl(jgs2_ctx* ctx, int32_t world, int32_t rank, const uint8_t* id128) {
  return guarded(ctx, [&](Ctx& C) {
    check_comm_args(C, world, rank);
    if (!id128) throw Error(JGS2_E_ARG, "null unique id");
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    auto* nc = new NcclComm();
    nc->rank = rank;
    nc->world = world;
    nc->owned = true;
    ncclResult_t r = ncclCommInitRank(&nc->c, world, id, rank);
    if (r != ncclSuccess) {
      delete nc;
      throw Error(JGS2_E_CUDA, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    C.comm = nc;
  });
}

int32_t jgs2_set_comm_nccl_handle(jgs2_ctx* ctx, int32_t world, int32_t rank, void* nccl_comm) {
  return guarded(ctx, [&](Ctx& C) {
    check_comm_args(C, world, rank);
    if (!nccl_comm) throw Error(JGS2_E_ARG, "null ncclComm_t");
    auto* nc = new NcclComm();
    nc->rank = rank;
    nc->world = world;
    nc->c = static_cast<ncclComm_t>(nccl_comm);
    C.comm = nc;
  });
}

int32_t jgs2_set_comm_host(jgs2_ctx* ctx, int32_t world, int32_t rank, jgs2_allreduce_fn fn, void* user) {
  return guarded(ctx, [&](Ctx& C) {
    check_comm_args(C, world, rank);
    if (!fn) throw Error(JGS2_E_ARG, "null all-reduce callback");
    auto* hc = new HostComm();
    hc->rank = rank;
    hc->world = world;
    hc->fn = fn;
    hc->user = user;
    C.comm = hc;
  });
}

int32_t jgs2_set_partition(jgs2_ctx* ctx, int64_t v_begin, int64_t v_end) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.have_model) throw Error(JGS2_E_ARG, "set the model first");
    if (C.fac.ready || C.have_pre) throw Error(JGS2_E_ARG, "set the partition before the factor and precompute");
    if (C.mode != 0) throw Error(JGS2_E_ARG, "the partitioned solve runs Jacobi sweeps only");
    auto bv = std::find(C.body_v.begin(), C.body_v.end(), (int)v_begin);
    auto ev = std::find(C.body_v.begin(), C.body_v.end(), (int)v_end);
    if (v_begin < 0 || v_end > C.nv || v_begin >= v_end || bv == C.body_v.end() || ev == C.body_v.end())
      throw Error(JGS2_E_ARG, "partition must cover whole bodies (vertex ids at body boundaries)");
    int b0 = (int)(bv - C.body_v.begin()), b1 = (int)(ev - C.body_v.begin());
    C.own_v0 = (int)v_begin;
    C.own_v1 = (int)v_end;
    C.own_e0 = C.body_e[b0];
    C.own_e1 = C.body_e[b1];
    C.chunk_own0 = C.chunk_first_e[b0];
    C.chunk_own1 = C.chunk_first_e[b1];
    C.vchunk_own0 = C.chunk_first_v[b0];
    C.vchunk_own1 = C.chunk_first_v[b1];
    std::vector<int> freel;
    for (int v = C.own_v0; v < C.own_v1; ++v)
      if (!C.h_fixed[v]) freel.push_back(v);
    C.nfree = (int)freel.size();
    C.free_list = C.upload(freel.data(), freel.size());
    C.partitioned = C.own_v0 != 0 || C.own_v1 != C.nv || (C.comm && C.comm->world > 1);
    // rotations of other ranks' vertices stay zero (jgs2_get_rotations sums)
    JGS2_CUDA(cudaMemsetAsync(C.R, 0, 9 * (size_t)C.nv * sizeof(double), C.stream));
    C.sync();
  });
}

void jgs2_destroy(jgs2_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  delete ctx;
}

const char* jgs2_last_error(const jgs2_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

// ============================================================= setup
int32_t jgs2_set_model(jgs2_ctx* ctx, const jgs2_model* md) {
  return guarded(ctx, [&](Ctx& C) {
    if (!md || md->nv <= 0 || md->ne < 0) throw Error(JGS2_E_ARG, "invalid model sizes");
    if (C.have_model) throw Error(JGS2_E_ARG, "model already set (create a new context)");
    C.nv = (int)md->nv;
    C.ne = (int)md->ne;
    const int nv = C.nv, ne = C.ne;
    C.norm_scale = md->norm_scale;
    C.h_tets.assign(md->tets, md->tets + 4 * (size_t)ne);
    std::vector<int4> t4(ne);
    for (int e = 0; e < ne; ++e) {
      for (int a = 0; a < 4; ++a) {
        int64_t w = md->tets[4 * (size_t)e + a];
        if (w < 0 || w >= nv) throw Error(JGS2_E_ARG, "element references a vertex out of range");
      }
      t4[e] = make_int4((int)md->tets[4 * (size_t)e], (int)md->tets[4 * (size_t)e + 1],
                        (int)md->tets[4 * (size_t)e + 2], (int)md->tets[4 * (size_t)e + 3]);
    }
    C.tets = C.upload(t4.data(), ne);
    C.dminv = C.upload(md->dm_inv, 9 * (size_t)ne);
    std::vector<double4> ep(ne);
    for (int e = 0; e < ne; ++e)
      ep[e] = make_double4(md->volumes[e], md->mu[e], md->lam[e], md->elem_qmass[e]);
    C.eprops = C.upload(ep.data(), ne);
    // incidence CSR, ascending element id per vertex
    std::vector<int> cnt(nv + 1, 0), inc(4 * (size_t)ne);
    for (size_t k = 0; k < 4 * (size_t)ne; ++k) cnt[md->tets[k] + 1]++;
    for (int v = 0; v < nv; ++v) cnt[v + 1] += cnt[v];
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int e = 0; e < ne; ++e)
      for (int a = 0; a < 4; ++a) inc[fill[md->tets[4 * (size_t)e + a]]++] = 4 * e + a;
    C.inc_ptr = C.upload(cnt.data(), nv + 1);
    C.inc = C.upload(inc.data(), 4 * (size_t)ne);
    C.mass = C.upload(md->masses, nv);
    C.h_fixed.assign(md->fixed_mask, md->fixed_mask + nv);
    C.fixed = C.upload(md->fixed_mask, nv);
    C.h_rest.assign(md->rest_positions, md->rest_positions + 3 * (size_t)nv);
    C.rest = C.upload(md->rest_positions, 3 * (size_t)nv);
    std::vector<int> freel;
    for (int v = 0; v < nv; ++v)
      if (!md->fixed_mask[v]) freel.push_back(v);
    C.nfree = (int)freel.size();
    C.free_list = C.upload(freel.data(), freel.size());
    C.x = C.alloc<double>(3 * (size_t)nv);
    C.z = C.alloc<double>(3 * (size_t)nv);
    C.R = C.alloc<double>(9 * (size_t)nv);
    C.gasm = C.alloc<double>(3 * (size_t)nv);
    C.b = C.alloc<double>(3 * (size_t)std::max(C.nfree, 1));
    C.q = C.alloc<double>(3 * (size_t)std::max(C.nfree, 1));
    C.delta = C.alloc<double>(3 * (size_t)nv);
    C.dx = C.alloc<double>(3 * (size_t)nv);
    C.alpha0 = C.alloc<double>(nv);
    C.kacc = C.alloc<int>(nv);
    JGS2_CUDA(cudaMemsetAsync(C.delta, 0, 3 * (size_t)nv * sizeof(double), C.stream));
    JGS2_CUDA(cudaMemsetAsync(C.dx, 0, 3 * (size_t)nv * sizeof(double), C.stream));
    contact_setup(C, md);
    // body boundaries (bodies are numbered consecutively in vertex and element
    // ids, as Model concatenates them, assembly.py:40-116) and the chunk table
    C.body_v.assign(1, 0);
    C.body_e.assign(1, 0);
    bool monotone = md->vertex_body != nullptr;
    for (int v = 1; v < nv && monotone; ++v) monotone = md->vertex_body[v] >= md->vertex_body[v - 1];
    if (monotone) {
      for (int v = 1; v < nv; ++v)
        if (md->vertex_body[v] != md->vertex_body[v - 1]) C.body_v.push_back(v);
      int b = 0;
      for (int e = 0; e < ne; ++e) {  // first element of each body
        int64_t eb = md->vertex_body[md->tets[4 * (size_t)e]];
        while (b + 1 < (int)C.body_v.size() && eb >= md->vertex_body[C.body_v[b + 1]]) {
          C.body_e.push_back(e);
          ++b;
        }
        for (int a = 1; a < 4 && monotone; ++a) monotone = md->vertex_body[md->tets[4 * (size_t)e + a]] == eb;
        if (e > 0 && eb < md->vertex_body[md->tets[4 * (size_t)(e - 1)]]) monotone = false;
      }
      while (C.body_e.size() < C.body_v.size()) C.body_e.push_back(ne);
    }
    if (!monotone) {  // one block: no partitioning possible
      C.body_v.assign(1, 0);
      C.body_e.assign(1, 0);
    }
    C.body_v.push_back(nv);
    C.body_e.push_back(ne);
    std::vector<int2> ch;
    std::vector<int> ech_first(C.body_e.size()), vch_first(C.body_v.size());
    for (size_t b = 0; b + 1 < C.body_e.size(); ++b) {
      ech_first[b] = (int)ch.size();
      for (int e = C.body_e[b]; e < C.body_e[b + 1]; e += kChunkE)
        ch.push_back(make_int2(e, std::min(e + kChunkE, C.body_e[b + 1])));
    }
    ech_first.back() = (int)ch.size();
    C.nchunk_e = (int)ch.size();
    for (size_t b = 0; b + 1 < C.body_v.size(); ++b) {
      vch_first[b] = (int)ch.size();
      for (int v = C.body_v[b]; v < C.body_v[b + 1]; v += kChunkV)
        ch.push_back(make_int2(v, std::min(v + kChunkV, C.body_v[b + 1])));
    }
    vch_first.back() = (int)ch.size();
    C.nchunk_v = (int)ch.size() - C.nchunk_e;
    C.chunk_first_e = ech_first;
    C.chunk_first_v = vch_first;
    C.chunks = C.upload(ch.data(), ch.size());
    C.cpart = C.alloc<double>((size_t)(kTrials + 1) * ch.size());
    C.own_v0 = 0; C.own_v1 = nv; C.own_e0 = 0; C.own_e1 = ne;
    C.chunk_own0 = 0; C.chunk_own1 = C.nchunk_e;
    C.vchunk_own0 = C.nchunk_e; C.vchunk_own1 = C.nchunk_e + C.nchunk_v;
    C.have_model = true;
    C.sync();
  });
}

int32_t jgs2_set_precompute(jgs2_ctx* ctx, const jgs2_precompute* p, const jgs2_config* cfg) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.have_model) throw Error(JGS2_E_ARG, "set the model first");
    if (!cfg) throw Error(JGS2_E_ARG, "null config");
    if (C.have_pre) throw Error(JGS2_E_ARG, "precompute already set");
    C.tol_dx = cfg->tol_dx;
    C.max_outer = cfg->max_outer;
    C.local_line_search = cfg->local_line_search != 0;
    C.track_energy = cfg->track_energy != 0;
    C.max_halvings = cfg->max_halvings;
    C.alpha_floor = cfg->alpha_floor;
    if (cfg->mode != 0 && cfg->mode != 1) throw Error(JGS2_E_ARG, "mode must be 0 (jacobi) or 1 (gauss_seidel)");
    if (cfg->mode != 0 && C.partitioned) throw Error(JGS2_E_ARG, "the partitioned solve runs Jacobi sweeps only");
    C.mode = cfg->mode;
    if (C.tol_dx <= 0 || C.max_outer < 1 || C.max_halvings < 0)
      throw Error(JGS2_E_ARG, "invalid solver config");
    const int nv = C.nv;
    if (cfg->subspace != 0 && cfg->subspace != 1) throw Error(JGS2_E_ARG, "subspace must be 0 or 1");
    if (cfg->subspace == 1) {  // plain vertex block descent: no bases, no factor
      C.plain = true;
      C.smax = 0;
      if (!C.pos) {  // no factor: free-vertex marker for the update kernels (-1 fixed / other rank)
        std::vector<int> pos(nv, -1);
        int k = 0;
        for (int v = 0; v < nv; ++v)
          if (!C.h_fixed[v] && C.owns(v)) pos[v] = k++;
        C.pos = C.upload(pos.data(), nv);
      }
      C.nuniq = 0;
      C.nslots = 0;
      C.mplus_all = C.alloc<double>(45 * (size_t)std::max(C.ne, 1));
      C.hess_list_all = C.alloc<int>(2 * (size_t)std::max(C.ne, 1));
      C.ls_max = C.alloc<unsigned long long>(C.max_halvings + 2);
      C.ls_cnt = C.alloc<int>(C.max_halvings + 2);
      C.ls_final = C.alloc<int>(4);
      JGS2_CUDA(cudaMemsetAsync(C.ls_final, 0, 4 * sizeof(int), C.stream));
      C.have_pre = true;
      C.sync();
      return;
    }
    if (!p) throw Error(JGS2_E_ARG, "null precompute");
    const int64_t nb = p->n_bases;
    C.gmax = (int)std::max<int64_t>(p->gmax, 1);
    std::vector<int> bidx(nv, -1);
    for (int64_t k = 0; k < nb; ++k) {
      int64_t v = p->vertices[k];
      if (v < 0 || v >= nv) throw Error(JGS2_E_ARG, "basis vertex out of range");
      bidx[v] = (int)k;
    }
    for (int v = 0; v < nv; ++v)
      if (!C.h_fixed[v] && C.owns(v) && bidx[v] < 0)
        throw Error(JGS2_E_KEY, "free vertex " + std::to_string(v) + " has no basis");
    std::vector<double> gbar(9 * (size_t)nv, 0.0), grows(9 * (size_t)C.gmax * nv, 0.0);
    std::vector<int> group((size_t)C.gmax * nv, -1);
    int smax = 0;
    for (int v = 0; v < nv; ++v) {
      int k = bidx[v];
      if (k < 0 || C.h_fixed[v] || !C.owns(v)) continue;  // this rank's vertices
      smax = std::max<int>(smax, (int)(p->cub_ptr[k + 1] - p->cub_ptr[k]));
      for (int i = 0; i < 9; ++i) gbar[9 * (size_t)v + i] = p->gbar[9 * k + i];
      for (int g = 0; g < p->gmax; ++g) group[(size_t)C.gmax * v + g] = (int)p->group[p->gmax * k + g];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3 * p->gmax; ++c)
          grows[9 * (size_t)C.gmax * v + 3 * C.gmax * r + c] = p->gbar_rows[(3 * p->gmax) * (3 * k + r) + c];
    }
    C.smax = smax;
    C.gbar = C.upload(gbar.data(), gbar.size());
    C.group = C.upload(group.data(), group.size());
    C.grows = C.upload(grows.data(), grows.size());
    // cubature slots
    size_t ns = (size_t)nv * std::max(smax, 1);
    std::vector<int> cub_e(ns, -1);
    std::vector<double> cub_w(ns, 0.0), cub_rows(36 * ns, 0.0);
    std::vector<int4> cub_verts(ns, make_int4(0, 0, 0, 0));
    for (int v = 0; v < nv; ++v) {
      int k = bidx[v];
      if (k < 0 || C.h_fixed[v] || !C.owns(v)) continue;  // this rank's vertices
      const int64_t* keys = p->vrows_keys + p->vrows_ptr[k];
      int64_t nk = p->vrows_ptr[k + 1] - p->vrows_ptr[k];
      for (int64_t s = p->cub_ptr[k]; s < p->cub_ptr[k + 1]; ++s) {
        int slot = (int)(s - p->cub_ptr[k]);
        int64_t e = p->cub_elems[s];
        if (e < 0 || e >= C.ne) throw Error(JGS2_E_ARG, "cubature element out of range");
        size_t vs = (size_t)slot * nv + v;  // slot-major SoA (LocalArgs)
        cub_e[vs] = (int)e;
        cub_w[vs] = p->cub_weights[s];
        int cs[4];
        for (int a = 0; a < 4; ++a) {
          int64_t w = C.h_tets[4 * e + a];
          cs[a] = (int)w;
          const int64_t* it = std::lower_bound(keys, keys + nk, w);
          if (it == keys + nk || *it != w)
            throw Error(JGS2_E_KEY, "basis at vertex " + std::to_string(v) + " lacks rows for vertex " +
                                        std::to_string(w) + " of cubature element " + std::to_string(e));
          const double* blk = p->vrows + 9 * (p->vrows_ptr[k] + (it - keys));
          for (int i = 0; i < 9; ++i) cub_rows[((size_t)slot * 36 + 9 * a + i) * nv + v] = blk[i];
        }
        cub_verts[vs] = make_int4(cs[0], cs[1], cs[2], cs[3]);
      }
    }
    std::vector<int> uniq;
    for (int e : cub_e)
      if (e >= 0) uniq.push_back(e);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    C.nuniq = (int)uniq.size();
    std::vector<int> cub_u(ns, -1);
    for (size_t i = 0; i < ns; ++i)
      if (cub_e[i] >= 0) cub_u[i] = (int)(std::lower_bound(uniq.begin(), uniq.end(), cub_e[i]) - uniq.begin());
    C.cub_u = C.upload(cub_u.data(), ns);
    C.cub_w = C.upload(cub_w.data(), ns);
    C.cub_rows = C.upload(cub_rows.data(), 36 * ns);
    C.cub_verts = C.upload(cub_verts.data(), ns);
    C.uniq = C.upload(uniq.data(), uniq.size());
    C.nslots = 0;
    for (int e : cub_e) C.nslots += (e >= 0);
    C.mplus = C.alloc<double>(45 * (size_t)std::max(C.nuniq, 1));
    C.hess_list = C.alloc<int>(2 * (size_t)std::max(C.nuniq, 1));
    C.crest = C.alloc<double>(9 * (size_t)nv);
    JGS2_CUDA(cudaMemsetAsync(C.crest, 0, 9 * (size_t)nv * sizeof(double), C.stream));
    C.ls_max = C.alloc<unsigned long long>(C.max_halvings + 2);
    C.ls_cnt = C.alloc<int>(C.max_halvings + 2);
    C.ls_final = C.alloc<int>(4);
    JGS2_CUDA(cudaMemsetAsync(C.ls_final, 0, 4 * sizeof(int), C.stream));
    // retained rows CSR (contact coupling rows, local_solver.py:85-112): only
    // surface vertices can be pair members, so only their bases are kept.
    if (contact_active(C)) {
      std::vector<int> vptr(nv + 1, 0), vkeys;
      std::vector<double> vrows;
      for (int v = 0; v < nv; ++v) {
        int k = bidx[v];
        if (k >= 0 && C.h_surface[v]) {
          for (int64_t q = p->vrows_ptr[k]; q < p->vrows_ptr[k + 1]; ++q) {
            vkeys.push_back((int)p->vrows_keys[q]);
            vrows.insert(vrows.end(), p->vrows + 9 * q, p->vrows + 9 * q + 9);
          }
        }
        vptr[v + 1] = (int)vkeys.size();
      }
      C.vr_ptr = C.upload(vptr.data(), vptr.size());
      C.vr_keys = C.upload(vkeys.data(), vkeys.size());
      C.vr_rows = C.upload(vrows.data(), vrows.size());
    }
    // rest constant C_v with identity rotations and rest element Hessians
    if (C.nuniq > 0) {
      DevModel m = devmodel(C);
      // pos is needed by devmodel consumers only after factoring; not used here
      launch_element_mplus(C.nuniq, C.uniq, C.rest, C.tets, C.dminv, C.eprops, C.mplus, C.hess_count,
                           C.hess_list, C.stream);
      C.check_launch();
      double* Rid = nullptr;
      JGS2_CUDA(cudaMallocAsync(&Rid, 9 * (size_t)nv * sizeof(double), C.stream));
      k_fill_identity<<<grid_for(nv), kBlock, 0, C.stream>>>(nv, Rid);
      C.check_launch();
      LocalArgs a = localargs(C);
      a.R = Rid;
      k_rest_constant<<<grid_for(C.nfree, 128), 128, 0, C.stream>>>(m, a, C.crest);
      C.check_launch();
      JGS2_CUDA(cudaFreeAsync(Rid, C.stream));
    }
    C.have_pre = true;
    C.sync();
  });
}

int32_t jgs2_set_colors(jgs2_ctx* ctx, const int64_t* colors) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.have_model) throw Error(JGS2_E_ARG, "model not set");
    int64_t cmax = -1;
    for (int v = 0; v < C.nv; ++v) {
      if (colors[v] < 0) throw Error(JGS2_E_ARG, "negative colour");
      cmax = std::max<int64_t>(cmax, colors[v]);
    }
    std::vector<int> cnt(cmax + 2, 0);
    for (int v = 0; v < C.nv; ++v)
      if (!C.h_fixed[v]) cnt[colors[v] + 1]++;
    std::vector<int> ptr(1, 0);  // non-empty colour groups only (local_solver.py:298-303)
    std::vector<int> verts;
    for (int64_t c = 0; c <= cmax; ++c) {
      if (cnt[c + 1] == 0) continue;
      for (int v = 0; v < C.nv; ++v)
        if (!C.h_fixed[v] && colors[v] == c) verts.push_back(v);
      ptr.push_back((int)verts.size());
    }
    C.color_ptr = ptr;
    C.color_verts = verts.empty() ? nullptr : C.upload(verts.data(), verts.size());
    if (C.gs_gsq) C.gs_gsq = C.alloc<double>(std::max<size_t>(ptr.size(), 1));
  });
}

int32_t jgs2_set_ordering(jgs2_ctx* ctx, int32_t ordering) {
  return guarded(ctx, [&](Ctx& C) {
    if (ordering != 0 && ordering != 1) throw Error(JGS2_E_ARG, "ordering must be 0 (geometric) or 1 (METIS)");
    if (C.fac.ready) throw Error(JGS2_E_ARG, "factor already built");
    C.ordering = ordering;
  });
}

int32_t jgs2_set_hess_overlap(jgs2_ctx* ctx, int32_t blocks_per_sm) {
  return guarded(ctx, [&](Ctx& C) {
    if (blocks_per_sm < 0 || blocks_per_sm > 16) throw Error(JGS2_E_ARG, "blocks_per_sm must be in [0, 16]");
    C.hess_overlap = blocks_per_sm;
  });
}

int32_t jgs2_factor_rest(jgs2_ctx* ctx, double h_ref, int32_t leaf_size, jgs2_factor_info* info) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.have_model) throw Error(JGS2_E_ARG, "set the model first");
    if (!(h_ref > 0)) throw Error(JGS2_E_ARG, "h_ref must be positive");
    if (C.fac.ready) throw Error(JGS2_E_ARG, "factor already built");
    factor_build(C, h_ref, leaf_size > 0 ? leaf_size : 32);
    if (info) {
      info->n_free = C.fac.nfree;
      info->nnz_dof = C.fac.sym.nnz_dof;
      info->nfronts = C.fac.nfronts;
      info->nlevels = C.fac.nlevels;
      info->max_front = C.fac.max_nf;
      info->factor_seconds = C.fac.seconds;
      info->ordering = C.fac.ordering_metis ? 1 : 0;
    }
  });
}

int32_t jgs2_factor_blocks(jgs2_ctx* ctx, int64_t nblocks, const int64_t* brow, const int64_t* bcol,
                           const double* bval, int32_t leaf_size, jgs2_factor_info* info) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.have_model) throw Error(JGS2_E_ARG, "set the model first");
    if (C.fac.ready) throw Error(JGS2_E_ARG, "factor already built");
    BlockInput in{nblocks, brow, bcol, bval};
    factor_build(C, 1.0, leaf_size > 0 ? leaf_size : 32, &in);
    if (info) {
      info->n_free = C.fac.nfree;
      info->nnz_dof = C.fac.sym.nnz_dof;
      info->nfronts = C.fac.nfronts;
      info->nlevels = C.fac.nlevels;
      info->max_front = C.fac.max_nf;
      info->factor_seconds = C.fac.seconds;
      info->ordering = C.fac.ordering_metis ? 1 : 0;
    }
  });
}

// ============================================================= state
int32_t jgs2_set_state(jgs2_ctx* ctx, const double* x, const double* z, double h) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.have_model) throw Error(JGS2_E_ARG, "model not set");
    if (!(h > 0)) throw Error(JGS2_E_ARG, "h must be positive");
    size_t n = 3 * (size_t)C.nv * sizeof(double);
    if (x) JGS2_CUDA(cudaMemcpyAsync(C.x, x, n, cudaMemcpyHostToDevice, C.stream));
    if (z) JGS2_CUDA(cudaMemcpyAsync(C.z, z, n, cudaMemcpyHostToDevice, C.stream));
    C.h = h;
    C.sync();
  });
}

int32_t jgs2_set_x(jgs2_ctx* ctx, const double* x) {
  return guarded(ctx, [&](Ctx& C) {
    JGS2_CUDA(cudaMemcpyAsync(C.x, x, 3 * (size_t)C.nv * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    C.sync();
  });
}

int32_t jgs2_get_x(jgs2_ctx* ctx, double* x) {
  return guarded(ctx, [&](Ctx& C) {
    JGS2_CUDA(cudaMemcpyAsync(x, C.x, 3 * (size_t)C.nv * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    C.sync();
  });
}

int32_t jgs2_get_dx(jgs2_ctx* ctx, double* dx) {
  return guarded(ctx, [&](Ctx& C) {
    JGS2_CUDA(cudaMemcpyAsync(dx, C.dx, 3 * (size_t)C.nv * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    C.sync();
  });
}

int32_t jgs2_set_rotations(jgs2_ctx* ctx, const double* R) {
  return guarded(ctx, [&](Ctx& C) {
    JGS2_CUDA(cudaMemcpyAsync(C.R, R, 9 * (size_t)C.nv * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    C.rot_valid = true;
    C.sync();
  });
}

int32_t jgs2_get_rotations(jgs2_ctx* ctx, double* R) {
  return guarded(ctx, [&](Ctx& C) {
    if (C.partitioned) {  // each rank holds its own vertices' rotations: sum the slices
      size_t n9 = 9 * (size_t)C.nv;
      double* t = nullptr;
      JGS2_CUDA(cudaMallocAsync(&t, n9 * sizeof(double), C.stream));
      JGS2_CUDA(cudaMemsetAsync(t, 0, n9 * sizeof(double), C.stream));
      size_t o = 9 * (size_t)C.own_v0, n = 9 * (size_t)(C.own_v1 - C.own_v0);
      JGS2_CUDA(cudaMemcpyAsync(t + o, C.R + o, n * sizeof(double), cudaMemcpyDeviceToDevice, C.stream));
      C.allreduce(t, n9, CT_F64, CO_SUM);
      JGS2_CUDA(cudaMemcpyAsync(R, t, n9 * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
      JGS2_CUDA(cudaFreeAsync(t, C.stream));
      C.sync();
      return;
    }
    JGS2_CUDA(cudaMemcpyAsync(R, C.R, 9 * (size_t)C.nv * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    C.sync();
  });
}

// ============================================================= hot path
int32_t jgs2_rotations(jgs2_ctx* ctx) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.have_model) throw Error(JGS2_E_ARG, "model not set");
    vertex_pass(C, true);
    C.sync();
  });
}

int32_t jgs2_sweep(jgs2_ctx* ctx, int32_t refresh_rotations, jgs2_sweep_info* info) {
  return guarded(ctx, [&](Ctx& C) { sweep_core(C, refresh_rotations != 0, info); });
}

int32_t jgs2_sweep_host(jgs2_ctx* ctx, const double* x, const double* z, double h,
                        const double* rotations, double* x_out, double* dx_out,
                        jgs2_sweep_info* info) {
  return guarded(ctx, [&](Ctx& C) {
    size_t n = 3 * (size_t)C.nv * sizeof(double);
    if (!(h > 0)) throw Error(JGS2_E_ARG, "h must be positive");
    JGS2_CUDA(cudaMemcpyAsync(C.x, x, n, cudaMemcpyHostToDevice, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(C.z, z, n, cudaMemcpyHostToDevice, C.stream));
    C.h = h;
    if (rotations) {
      JGS2_CUDA(cudaMemcpyAsync(C.R, rotations, 3 * n, cudaMemcpyHostToDevice, C.stream));
      C.rot_valid = true;
    }
    sweep_core(C, rotations == nullptr, info);
    if (x_out) JGS2_CUDA(cudaMemcpyAsync(x_out, C.x, n, cudaMemcpyDeviceToHost, C.stream));
    if (dx_out) JGS2_CUDA(cudaMemcpyAsync(dx_out, C.dx, n, cudaMemcpyDeviceToHost, C.stream));
    C.sync();
  });
}

int32_t jgs2_outer_solve(jgs2_ctx* ctx, double* dx_norms, double* grad_norms, double* energies,
                         double* max_local_steps, int64_t* activations, int32_t* iterations,
                         int32_t* converged) {
  return guarded(ctx, [&](Ctx& C) {
    int it = 0;
    bool conv = false;
    for (; it < C.max_outer;) {
      jgs2_sweep_info inf;
      sweep_core(C, true, &inf);
      if (dx_norms) dx_norms[it] = inf.dx_norm;
      if (grad_norms) grad_norms[it] = inf.grad_norm;
      if (energies) energies[it] = inf.energy;
      if (max_local_steps) max_local_steps[it] = inf.max_local_step;
      if (activations) activations[it] = inf.line_search_activations;
      ++it;
      if (inf.dx_norm < C.tol_dx) { conv = true; break; }
    }
    if (iterations) *iterations = it;
    if (converged) *converged = conv ? 1 : 0;
  });
}

// ============================================================= frame driver
// compute_z + initialize_step (assembly.py:165-180, harness.py:130-134) and
// step_velocity_update (assembly.py:346-351) on device-resident state.
namespace {
__global__ void k_compute_z(int nv, const double* xp, const double* v, double h, double g0, double g1,
                            double g2, const uint8_t* fixed, double* z, double* dz) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  double g[3] = {g0, g1, g2};
  for (int c = 0; c < 3; ++c) {
    double zc = fixed[i] ? xp[3 * i + c] : (xp[3 * i + c] + h * v[3 * i + c]) + (h * h) * g[c];
    z[3 * i + c] = zc;
    dz[3 * i + c] = zc - xp[3 * i + c];
  }
}
__global__ void k_init_x(int nv, const double* xp, const double* dz, double cap, double* x) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * nv) return;
  x[i] = xp[i] + cap * dz[i];
}
__global__ void k_velocity(int nv, double h, const double* x, double* xp, double* v) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * nv) return;
  v[i] = (x[i] - xp[i]) / h;
  xp[i] = x[i];
}
}  // namespace

int32_t jgs2_set_frame_state(jgs2_ctx* ctx, const double* x_prev, const double* v, double h,
                             const double* gravity) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.have_model) throw Error(JGS2_E_ARG, "model not set");
    if (!(h > 0)) throw Error(JGS2_E_ARG, "h must be positive");
    size_t n = 3 * (size_t)C.nv;
    if (!C.xprev) { C.xprev = C.alloc<double>(n); C.vel = C.alloc<double>(n); C.dz = C.alloc<double>(n); }
    if (!C.xprev0) { C.xprev0 = C.alloc<double>(n); C.vel0 = C.alloc<double>(n); }
    JGS2_CUDA(cudaMemcpyAsync(C.xprev, x_prev, n * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(C.vel, v, n * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(C.xprev0, C.xprev, n * sizeof(double), cudaMemcpyDeviceToDevice, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(C.vel0, C.vel, n * sizeof(double), cudaMemcpyDeviceToDevice, C.stream));
    for (int c = 0; c < 3; ++c) C.gravity[c] = gravity ? gravity[c] : 0.0;
    C.h = h;
    C.sync();
  });
}

int32_t jgs2_frame_begin(jgs2_ctx* ctx, double* cap_out) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.xprev) throw Error(JGS2_E_ARG, "frame state not set");
    k_compute_z<<<grid_for(C.nv), kBlock, 0, C.stream>>>(C.nv, C.xprev, C.vel, C.h, C.gravity[0],
                                                         C.gravity[1], C.gravity[2], C.fixed, C.z, C.dz);
    C.check_launch();
    double cap = 1.0;
    if (contact_active(C)) {
      C.phase_begin(10, 0.0);
      cap = contact_step_cap(C, C.xprev, C.dz);
      C.phase_end();
    }
    k_init_x<<<grid_for(3 * (int64_t)C.nv), kBlock, 0, C.stream>>>(C.nv, C.xprev, C.dz, cap, C.x);
    C.check_launch();
    C.sync();
    if (cap_out) *cap_out = cap;
  });
}

int32_t jgs2_frame_reset(jgs2_ctx* ctx) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.xprev0) throw Error(JGS2_E_ARG, "frame state not set");
    size_t n = 3 * (size_t)C.nv * sizeof(double);
    JGS2_CUDA(cudaMemcpyAsync(C.xprev, C.xprev0, n, cudaMemcpyDeviceToDevice, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(C.vel, C.vel0, n, cudaMemcpyDeviceToDevice, C.stream));
  });
}

int32_t jgs2_frame_end(jgs2_ctx* ctx) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.xprev) throw Error(JGS2_E_ARG, "frame state not set");
    k_velocity<<<grid_for(3 * (int64_t)C.nv), kBlock, 0, C.stream>>>(C.nv, C.h, C.x, C.xprev, C.vel);
    C.check_launch();
  });
}

// One whole timestep from HOST buffers (harness.py:187-211 per frame:
// compute_z, initialize_step, outer_solve to tol_dx, velocity update): the
// frame state (x_prev, v) goes h2d, the step runs on the device, and the
// new (x_prev, v) come back d2h. x_prev_out / v_out may alias the inputs.
int32_t jgs2_timestep_host(jgs2_ctx* ctx, const double* x_prev, const double* v, double h,
                           const double* gravity, double* x_prev_out, double* v_out,
                           int32_t* iterations, int32_t* converged) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.have_model) throw Error(JGS2_E_ARG, "model not set");
    if (!(h > 0)) throw Error(JGS2_E_ARG, "h must be positive");
    if (!x_prev || !v) throw Error(JGS2_E_ARG, "x_prev and v are required");
    size_t n = 3 * (size_t)C.nv;
    if (!C.xprev) { C.xprev = C.alloc<double>(n); C.vel = C.alloc<double>(n); C.dz = C.alloc<double>(n); }
    JGS2_CUDA(cudaMemcpyAsync(C.xprev, x_prev, n * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(C.vel, v, n * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    for (int c = 0; c < 3; ++c) C.gravity[c] = gravity ? gravity[c] : 0.0;
    C.h = h;
    k_compute_z<<<grid_for(C.nv), kBlock, 0, C.stream>>>(C.nv, C.xprev, C.vel, C.h, C.gravity[0],
                                                         C.gravity[1], C.gravity[2], C.fixed, C.z, C.dz);
    C.check_launch();
    double cap = 1.0;
    if (contact_active(C)) {
      C.phase_begin(10, 0.0);
      cap = contact_step_cap(C, C.xprev, C.dz);
      C.phase_end();
    }
    k_init_x<<<grid_for(3 * (int64_t)C.nv), kBlock, 0, C.stream>>>(C.nv, C.xprev, C.dz, cap, C.x);
    C.check_launch();
    int it = 0;
    bool conv = false;
    while (it < C.max_outer) {
      jgs2_sweep_info inf;
      sweep_core(C, true, &inf);
      ++it;
      if (inf.dx_norm < C.tol_dx) { conv = true; break; }
    }
    k_velocity<<<grid_for(3 * (int64_t)C.nv), kBlock, 0, C.stream>>>(C.nv, C.h, C.x, C.xprev, C.vel);
    C.check_launch();
    if (x_prev_out) JGS2_CUDA(cudaMemcpyAsync(x_prev_out, C.xprev, n * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    if (v_out) JGS2_CUDA(cudaMemcpyAsync(v_out, C.vel, n * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    C.sync();
    if (iterations) *iterations = it;
    if (converged) *converged = conv ? 1 : 0;
  });
}

int32_t jgs2_get_frame_state(jgs2_ctx* ctx, double* x_prev, double* v) {
  return guarded(ctx, [&](Ctx& C) {
    size_t n = 3 * (size_t)C.nv * sizeof(double);
    if (x_prev) JGS2_CUDA(cudaMemcpyAsync(x_prev, C.xprev, n, cudaMemcpyDeviceToHost, C.stream));
    if (v) JGS2_CUDA(cudaMemcpyAsync(v, C.vel, n, cudaMemcpyDeviceToHost, C.stream));
    C.sync();
  });
}

// ============================================================= per-kernel entries
int32_t jgs2_total_energy(jgs2_ctx* ctx, const double* x, double* energy) {
  return guarded(ctx, [&](Ctx& C) {
    if (x) JGS2_CUDA(cudaMemcpyAsync(C.x, x, 3 * (size_t)C.nv * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    if (contact_active(C)) contact_find_pairs(C, C.x, nullptr, 0.0);
    launch_energy(C, nullptr, 0.0, R_ENERGY);
    JGS2_CUDA(cudaMemcpyAsync(C.h_res, C.res, R_NSLOTS * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    C.sync();
    if (contact_active(C) && contact_infeasible(C)) throw Error(JGS2_E_INFEASIBLE, "barrier distance <= 0");
    *energy = C.h_res[R_ENERGY];
  });
}

int32_t jgs2_assembled_field(jgs2_ctx* ctx, double* g) {
  return guarded(ctx, [&](Ctx& C) {
    if (contact_active(C)) contact_find_pairs(C, C.x, nullptr, 0.0);
    vertex_pass(C, false);
    if (contact_active(C)) contact_add_gradients(C);
    JGS2_CUDA(cudaMemcpyAsync(g, C.gasm, 3 * (size_t)C.nv * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    C.sync();
  });
}

int32_t jgs2_reduced_collect(jgs2_ctx* ctx, const double* R, const double* g, double* q) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.fac.ready) throw Error(JGS2_E_ARG, "rest factor not built");
    size_t n = 3 * (size_t)C.nv * sizeof(double);
    JGS2_CUDA(cudaMemcpyAsync(C.R, R, 3 * n, cudaMemcpyHostToDevice, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(C.gasm, g, n, cudaMemcpyHostToDevice, C.stream));
    C.rot_valid = true;
    collect(C);
    std::vector<double> b(3 * (size_t)std::max(C.nfree, 1)), out(3 * (size_t)C.nv, 0.0);
    std::vector<int> pos(C.nv);
    JGS2_CUDA(cudaMemcpyAsync(b.data(), C.q, 3 * (size_t)C.nfree * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(pos.data(), C.pos, C.nv * sizeof(int), cudaMemcpyDeviceToHost, C.stream));
    C.sync();
    for (int v = 0; v < C.nv; ++v)
      if (pos[v] >= 0)
        for (int c = 0; c < 3; ++c) out[3 * (size_t)v + c] = b[3 * (size_t)pos[v] + c];
    memcpy(q, out.data(), n);
  });
}

static void debug_systems(Ctx& C, double* a, double* g, double* corr) {
  require_ready(C);
  if (!C.rot_valid) throw Error(JGS2_E_ARG, "rotations not set");
  if (contact_active(C)) contact_find_pairs(C, C.x, nullptr, 0.0);
  vertex_pass(C, false);
  if (contact_active(C)) contact_add_gradients(C);
  collect(C);
  size_t n9 = 9 * (size_t)C.nv;
  double *dA = nullptr, *dg = nullptr, *dc = nullptr;
  JGS2_CUDA(cudaMallocAsync(&dA, n9 * sizeof(double), C.stream));
  JGS2_CUDA(cudaMallocAsync(&dg, n9 * sizeof(double), C.stream));
  JGS2_CUDA(cudaMallocAsync(&dc, n9 * sizeof(double), C.stream));
  JGS2_CUDA(cudaMemsetAsync(dA, 0, n9 * sizeof(double), C.stream));
  JGS2_CUDA(cudaMemsetAsync(dg, 0, n9 * sizeof(double), C.stream));
  JGS2_CUDA(cudaMemsetAsync(dc, 0, n9 * sizeof(double), C.stream));
  local_systems(C, dA, dg, dc);
  if (a) JGS2_CUDA(cudaMemcpyAsync(a, dA, n9 * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  if (g) JGS2_CUDA(cudaMemcpyAsync(g, dg, 3 * (size_t)C.nv * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  if (corr) JGS2_CUDA(cudaMemcpyAsync(corr, dc, n9 * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
  JGS2_CUDA(cudaFreeAsync(dA, C.stream));
  JGS2_CUDA(cudaFreeAsync(dg, C.stream));
  JGS2_CUDA(cudaFreeAsync(dc, C.stream));
  C.sync();
}

int32_t jgs2_sampled_corrections(jgs2_ctx* ctx, double* corr) {
  return guarded(ctx, [&](Ctx& C) { debug_systems(C, nullptr, nullptr, corr); });
}

int32_t jgs2_reduced_systems(jgs2_ctx* ctx, double* a, double* g) {
  return guarded(ctx, [&](Ctx& C) { debug_systems(C, a, g, nullptr); });
}

int32_t jgs2_local_step(jgs2_ctx* ctx, double* delta, double* alpha, int64_t* activations) {
  return guarded(ctx, [&](Ctx& C) {
    require_ready(C);
    if (!C.rot_valid) throw Error(JGS2_E_ARG, "rotations not set");
    if (contact_active(C)) contact_find_pairs(C, C.x, nullptr, 0.0);
    vertex_pass(C, false);
    if (contact_active(C)) contact_add_gradients(C);
    collect(C);
    local_systems(C, nullptr, nullptr, nullptr);
    DevModel m = devmodel(C);
    k_ls_final<<<1, 1, 0, C.stream>>>(C.max_halvings, C.alpha_floor, C.ls_cnt, C.ls_max, C.ls_final);
    C.check_launch();
    double* dal = nullptr;
    JGS2_CUDA(cudaMallocAsync(&dal, (size_t)C.nv * sizeof(double), C.stream));
    k_alpha_out<<<grid_for(C.nv), kBlock, 0, C.stream>>>(m, C.alpha0, C.kacc, C.ls_final, C.local_line_search ? 1 : 0,
                                                         C.max_halvings, C.alpha_floor, dal);
    C.check_launch();
    int lsf[3] = {0, 0, 0};
    if (delta) JGS2_CUDA(cudaMemcpyAsync(delta, C.delta, 3 * (size_t)C.nv * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    if (alpha) JGS2_CUDA(cudaMemcpyAsync(alpha, dal, (size_t)C.nv * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(lsf, C.ls_final, 3 * sizeof(int), cudaMemcpyDeviceToHost, C.stream));
    JGS2_CUDA(cudaFreeAsync(dal, C.stream));
    C.sync();
    if (activations) *activations = C.local_line_search ? lsf[2] : 0;
  });
}

int32_t jgs2_factor_fill(jgs2_ctx* ctx, int64_t* out) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.fac.ready) throw Error(JGS2_E_ARG, "rest factor not built");
    const Symbolic& S = C.fac.sym;
    const int n = S.n;
    // the factored free-vertex graph (vertex adjacency through elements)
    // node ids of the symbolic graph: node = perm[pos]; pos = h_pos[v]
    std::vector<int> node_of(C.nv, -1);
    for (int v = 0; v < C.nv; ++v)
      if (C.fac.h_pos[v] >= 0) node_of[v] = S.perm[C.fac.h_pos[v]];
    std::vector<std::vector<int>> nb(n);
    for (int e = 0; e < C.ne; ++e) {
      const int64_t* t = &C.h_tets[4 * (size_t)e];
      for (int a = 0; a < 4; ++a) {
        int na = node_of[t[a]];
        if (na < 0) continue;
        for (int b = 0; b < 4; ++b) {
          int nbb = node_of[t[b]];
          if (nbb >= 0 && nbb != na) nb[na].push_back(nbb);
        }
      }
    }
    std::vector<int64_t> ptr(n + 1, 0);
    std::vector<int32_t> adj;
    for (int i = 0; i < n; ++i) {
      auto& s = nb[i];
      std::sort(s.begin(), s.end());
      s.erase(std::unique(s.begin(), s.end()), s.end());
      adj.insert(adj.end(), s.begin(), s.end());
      ptr[i + 1] = (int64_t)adj.size();
    }
    auto dof = [n](int64_t lv) { return 9 * (lv - n) + 6 * (int64_t)n; };  // 3x3 blocks, lower
    std::vector<int32_t> pnd(S.perm.begin(), S.perm.end()), pm(n);
    int64_t nd_exact = chol_nnz(n, ptr.data(), adj.data(), pnd.data());
    metis_nd(n, ptr.data(), adj.data(), pm.data());
    int64_t metis_exact = chol_nnz(n, ptr.data(), adj.data(), pm.data());
    out[0] = S.nnz_dof;        // the solve's supernodal storage (dense diagonal blocks)
    out[1] = dof(nd_exact);    // exact Cholesky fill of the same ordering
    out[2] = dof(metis_exact); // exact Cholesky fill of METIS nested dissection
  });
}

// ---- scalable precompute (selinv.cuh, train.cuh)
int32_t jgs2_selected_inverse(jgs2_ctx* ctx, double* seconds) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.fac.ready) throw Error(JGS2_E_ARG, "rest factor not built");
    auto t0 = std::chrono::steady_clock::now();
    selected_inverse(C);
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

int32_t jgs2_inverse_blocks(jgs2_ctx* ctx, int64_t n, const int64_t* v, const int64_t* w, double* out,
                            int32_t* found) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.fac.Z) throw Error(JGS2_E_ARG, "selected inverse not computed");
    if (n <= 0) return;
    int64_t *dv = nullptr, *dw = nullptr;
    double* dout = nullptr;
    int* dfound = nullptr;
    JGS2_CUDA(cudaMallocAsync(&dv, n * sizeof(int64_t), C.stream));
    JGS2_CUDA(cudaMallocAsync(&dw, n * sizeof(int64_t), C.stream));
    JGS2_CUDA(cudaMallocAsync(&dout, 9 * n * sizeof(double), C.stream));
    JGS2_CUDA(cudaMallocAsync(&dfound, n * sizeof(int), C.stream));
    JGS2_CUDA(cudaMemcpyAsync(dv, v, n * sizeof(int64_t), cudaMemcpyHostToDevice, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(dw, w, n * sizeof(int64_t), cudaMemcpyHostToDevice, C.stream));
    k_inverse_blocks<<<grid_for(n), kBlock, 0, C.stream>>>(selinv_dev(C), (int)n, dv, dw, dout, dfound);
    C.check_launch();
    JGS2_CUDA(cudaMemcpyAsync(out, dout, 9 * n * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(found, dfound, n * sizeof(int), cudaMemcpyDeviceToHost, C.stream));
    for (void* p : {(void*)dv, (void*)dw, (void*)dout, (void*)dfound}) JGS2_CUDA(cudaFreeAsync(p, C.stream));
    C.sync();
  });
}

int32_t jgs2_stencil_gradients(jgs2_ctx* ctx, const double* x, const double* z, double h, double* out) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.have_model) throw Error(JGS2_E_ARG, "model not set");
    size_t n = 3 * (size_t)C.nv;
    double *dx = nullptr, *dz = nullptr, *dout = nullptr;
    JGS2_CUDA(cudaMallocAsync(&dx, n * sizeof(double), C.stream));
    JGS2_CUDA(cudaMallocAsync(&dz, n * sizeof(double), C.stream));
    JGS2_CUDA(cudaMallocAsync(&dout, 12 * (size_t)C.ne * sizeof(double), C.stream));
    JGS2_CUDA(cudaMemcpyAsync(dx, x, n * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(dz, z, n * sizeof(double), cudaMemcpyHostToDevice, C.stream));
    k_stencil_grads<<<grid_for(C.ne), kBlock, 0, C.stream>>>(devmodel(C), dx, dz, h, dout);
    C.check_launch();
    JGS2_CUDA(cudaMemcpyAsync(out, dout, 12 * (size_t)C.ne * sizeof(double), cudaMemcpyDeviceToHost, C.stream));
    for (void* p : {(void*)dx, (void*)dz, (void*)dout}) JGS2_CUDA(cudaFreeAsync(p, C.stream));
    C.sync();
  });
}

int32_t jgs2_precompute_train(jgs2_ctx* ctx, const jgs2_train_params* p, int64_t* sizes) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.fac.Z) throw Error(JGS2_E_ARG, "selected inverse not computed");
    if (!p || p->n_poses < 0 || (p->n_poses > 0 && (!p->pose_grads || !p->pose_solves)))
      throw Error(JGS2_E_ARG, "invalid training inputs");
    TrainParams P{p->n_poses, p->candidates_per_round, p->max_size, p->target_residual, p->seed,
                  p->pose_grads, p->pose_solves};
    C.train = std::make_shared<TrainOut>();
    train_all_host(C, P, *C.train);
    if (sizes) {
      sizes[0] = (int64_t)C.train->vertices.size();
      sizes[1] = (int64_t)C.train->vr_keys.size();
      sizes[2] = (int64_t)C.train->cub_elems.size();
    }
  });
}

int32_t jgs2_precompute_export(jgs2_ctx* ctx, int64_t* vertices, double* gbar, int64_t* vrows_ptr,
                               int64_t* vrows_keys, double* vrows, int64_t* cub_ptr, int64_t* cub_elems,
                               double* cub_weights, double* residual, uint8_t* converged) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.train) throw Error(JGS2_E_ARG, "jgs2_precompute_train first");
    const TrainOut& T = *C.train;
    auto cp = [](auto* dst, const auto& v) { if (dst && !v.empty()) memcpy(dst, v.data(), v.size() * sizeof(v[0])); };
    cp(vertices, T.vertices); cp(gbar, T.gbar); cp(vrows_ptr, T.vr_ptr); cp(vrows_keys, T.vr_keys);
    cp(vrows, T.vrows); cp(cub_ptr, T.cub_ptr); cp(cub_elems, T.cub_elems); cp(cub_weights, T.cub_w);
    cp(residual, T.residual); cp(converged, T.converged);
  });
}

int32_t jgs2_find_pairs(jgs2_ctx* ctx, double* rows, int64_t capacity, int64_t* count) {
  return guarded(ctx, [&](Ctx& C) {
    if (!contact_active(C)) { *count = 0; return; }
    contact_find_pairs(C, C.x, nullptr, 0.0);
    C.sync();
    *count = C.npairs;
    if (C.npairs > capacity) throw Error(JGS2_E_ARG, "pair capacity too small");
    if (C.npairs)
      JGS2_CUDA(cudaMemcpy(rows, C.pairs, (size_t)C.npairs * kPairRow * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int32_t jgs2_last_kernel_launches(jgs2_ctx* ctx, int64_t* launches) {
  if (!ctx || !launches) return JGS2_E_ARG;
  *launches = ctx->c.launches;
  return JGS2_OK;
}

// ============================================================= measurement
int32_t jgs2_profile(jgs2_ctx* ctx, int32_t enable) {
  return guarded(ctx, [&](Ctx& C) { C.sync(); C.profiling = enable != 0; });
}

int32_t jgs2_phase_stats(jgs2_ctx* ctx, double* ms, int64_t* launches, double* bytes) {
  return guarded(ctx, [&](Ctx& C) {
    C.sync();
    for (int p = 0; p < Ctx::kPhases; ++p) {
      if (ms) ms[p] = C.phase_ms[p];
      if (launches) launches[p] = C.phase_launch[p];
      if (bytes) bytes[p] = C.phase_bytes[p];
    }
  });
}

int32_t jgs2_phase_reset(jgs2_ctx* ctx) {
  return guarded(ctx, [&](Ctx& C) {
    C.sync();
    for (int p = 0; p < Ctx::kPhases; ++p) { C.phase_ms[p] = 0; C.phase_launch[p] = 0; C.phase_bytes[p] = 0; }
  });
}

int32_t jgs2_timer_start(jgs2_ctx* ctx) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.tstart) { JGS2_CUDA(cudaEventCreate(&C.tstart)); JGS2_CUDA(cudaEventCreate(&C.tstop)); }
    JGS2_CUDA(cudaEventRecord(C.tstart, C.stream));
    cudaProfilerStart();  // profiler range = the timed window (ncu --profile-from-start off)
  });
}

int32_t jgs2_timer_stop(jgs2_ctx* ctx, double* ms) {
  return guarded(ctx, [&](Ctx& C) {
    if (!C.tstart) throw Error(JGS2_E_ARG, "timer not started");
    JGS2_CUDA(cudaEventRecord(C.tstop, C.stream));
    JGS2_CUDA(cudaEventSynchronize(C.tstop));
    cudaProfilerStop();
    float f = 0.f;
    JGS2_CUDA(cudaEventElapsedTime(&f, C.tstart, C.tstop));
    *ms = f;
  });
}

void* jgs2_pinned_alloc(int64_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, (size_t)std::max<int64_t>(bytes, 1)) != cudaSuccess) return nullptr;
  return p;
}

void jgs2_pinned_free(void* p) {
  if (p) cudaFreeHost(p);
}

int32_t jgs2_step_cap(jgs2_ctx* ctx, const double* x, const double* dx, double* cap) {
  return guarded(ctx, [&](Ctx& C) {
    *cap = 1.0;
    if (!contact_active(C)) return;
    // own scratch (x, dx), so a device-resident frame in flight (C.x) is untouched
    size_t n = 3 * (size_t)C.nv * sizeof(double);
    if (!C.cap_x) {
      C.cap_x = C.alloc<double>(3 * (size_t)C.nv);
      C.cap_dx = C.alloc<double>(3 * (size_t)C.nv);
    }
    JGS2_CUDA(cudaMemcpyAsync(C.cap_x, x, n, cudaMemcpyHostToDevice, C.stream));
    JGS2_CUDA(cudaMemcpyAsync(C.cap_dx, dx, n, cudaMemcpyHostToDevice, C.stream));
    *cap = contact_step_cap(C, C.cap_x, C.cap_dx);
    C.sync();
  });
}

// ============================================================= symbolic (host only)
jgs2_sym* jgs2_sym_build(int64_t n, const int64_t* adj_ptr, const int32_t* adj, const double* coords,
                         int32_t leaf_size) {
  try {
    jgs2_sym* s = new jgs2_sym();
    build_symbolic((int)n, adj_ptr, adj, coords, leaf_size, s->s);
    return s;
  } catch (...) {
    return nullptr;
  }
}

int32_t jgs2_sym_sizes(const jgs2_sym* s, int64_t* sizes) {
  if (!s || !sizes) return JGS2_E_ARG;
  sizes[0] = s->s.nfronts;
  sizes[1] = (int64_t)s->s.struct_pos.size();
  sizes[2] = s->s.nlevels;
  sizes[3] = s->s.nnz_dof;
  return JGS2_OK;
}

int32_t jgs2_sym_export(const jgs2_sym* s, int32_t* perm, int32_t* parent, int32_t* col_begin,
                        int32_t* col_end, int64_t* struct_ptr, int32_t* struct_pos, int32_t* level) {
  if (!s) return JGS2_E_ARG;
  const Symbolic& S = s->s;
  if (perm) std::copy(S.perm.begin(), S.perm.end(), perm);
  if (parent) std::copy(S.parent.begin(), S.parent.end(), parent);
  if (col_begin) std::copy(S.col_begin.begin(), S.col_begin.end(), col_begin);
  if (col_end) std::copy(S.col_end.begin(), S.col_end.end(), col_end);
  if (struct_ptr) std::copy(S.struct_ptr.begin(), S.struct_ptr.end(), struct_ptr);
  if (struct_pos) std::copy(S.struct_pos.begin(), S.struct_pos.end(), struct_pos);
  if (level) std::copy(S.level.begin(), S.level.end(), level);
  return JGS2_OK;
}

void jgs2_sym_free(jgs2_sym* s) { delete s; }

}  // extern "C"
