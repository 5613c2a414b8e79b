/* jgs2.h -- C ABI of the B200-native JGS2 runtime iteration (sm_100a).
 *
 * Drop-in boundary for the reference package's hot path
 *   tetsolve.local_solver.LocalSolver.sweep / .outer_solve
 *   (/root/reference/pkg/src/tetsolve/local_solver.py:606-655, 688-721)
 * in subspace="corotated_cubature", mode="jacobi".  The reference is pure
 * Python with no FFI of its own; these entry points are what its
 * LocalSolver would bind (see INTEGRATION.md for the ctypes stub).
 *
 * Conventions: plain pointers and sizes only; host arrays are caller-owned
 * and copied; the context owns all device memory and one CUDA stream.
 * Every call returns 0 on success or a negative JGS2_E* code; the message
 * is available from jgs2_last_error().  No exceptions cross the ABI.
 * FP64 values, int64 indices (numpy default), row-major 3x3 blocks.
 * Deterministic: ordered gathers, no floating-point atomics.
 */
#ifndef JGS2_H
#define JGS2_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JGS2_OK 0
#define JGS2_E_ARG -1        /* invalid argument / state (ValueError) */
#define JGS2_E_CUDA -2       /* CUDA runtime / library failure */
#define JGS2_E_FACTOR -3     /* rest Hessian not SPD (PrecomputeError) */
#define JGS2_E_KEY -4        /* basis lacks rows of a cubature element (KeyError) */
#define JGS2_E_INFEASIBLE -5 /* barrier distance <= 0 at the sweep start (FeasibilityError) */
#define JGS2_E_NODEV -6      /* no CUDA device */

typedef struct jgs2_ctx jgs2_ctx;

/* Static scene data: the reference Model arrays (assembly.py:40-116). */
typedef struct jgs2_model {
  int64_t nv, ne;
  const double* rest_positions; /* nv*3 (Hbar is built at rest, subspace.py:48-57) */
  const int64_t* tets;          /* ne*4 */
  const double* dm_inv;         /* ne*9 */
  const double* volumes;        /* ne */
  const double* mu;             /* ne */
  const double* lam;            /* ne */
  const double* elem_qmass;     /* ne  (rho V / 4, assembly.py:82-84) */
  const double* masses;         /* nv */
  const uint8_t* fixed_mask;    /* nv */
  double norm_scale;            /* normalization.scale (assembly.py:112-116) */
  /* contact (contact.py:216-240); n_planes/n_surface_* may be 0 */
  int32_t has_barrier;
  double dhat, kappa;
  int64_t n_planes;
  const double* plane_points;   /* n_planes*3 */
  const double* plane_normals;  /* n_planes*3 (unit) */
  int64_t n_bodies;
  int64_t n_surface_vertices, n_surface_tris;
  const int64_t* surface_vertices; /* ascending */
  const int64_t* surface_tris;     /* n_surface_tris*3 */
  const int64_t* vertex_body;      /* nv */
  const int64_t* surface_tri_body; /* n_surface_tris */
} jgs2_model;

/* Precompute (harness.prepare, harness.py:57-107) in flat CSR form. */
typedef struct jgs2_precompute {
  int64_t n_bases, gmax;
  const int64_t* vertices;   /* n_bases, ascending free vertex ids */
  const double* gbar;        /* n_bases*9 */
  const int64_t* group;      /* n_bases*gmax, -1 padded */
  const double* gbar_rows;   /* n_bases*3*(3*gmax) row-major */
  const int64_t* vrows_ptr;  /* n_bases+1 */
  const int64_t* vrows_keys; /* retained vertex ids, ascending per basis */
  const double* vrows;       /* nnz*9 */
  const int64_t* cub_ptr;    /* n_bases+1 */
  const int64_t* cub_elems;
  const double* cub_weights;
} jgs2_precompute;

/* SolverConfig subset on the path (local_solver.py:38-56). */
typedef struct jgs2_config {
  double tol_dx;
  int32_t max_outer;
  int32_t local_line_search;
  int32_t track_energy;
  int32_t max_halvings;
  double alpha_floor;
  int32_t mode;            /* 0 jacobi, 1 gauss_seidel (local_solver.py:627-649) */
  int32_t subspace;        /* 0 corotated_cubature, 1 none (plain vertex block descent,
                              local_solver.py:325-353, 472-522; jgs2_set_precompute then
                              takes pre = NULL and no factor is needed) */
} jgs2_config;

/* sweep() info dict (local_solver.py:613-614, 654) + extras. */
typedef struct jgs2_sweep_info {
  int64_t line_search_activations;
  double max_local_step;
  double grad_norm;
  double grad_sq;
  double dx_norm;          /* normalization.scale * |dx| (assembly.py:118-120) */
  double energy;           /* total_energy at the new x (track_energy) */
  int32_t halvings;        /* global backtrack halvings */
  int32_t n_pairs;         /* active pairs at the sweep start */
  int32_t n_indefinite;    /* cubature elements whose Hessian needed projection */
  int32_t pad_;
  double gamma;            /* accepted global step fraction (cap * 2^-halvings) */
  double cap;              /* feasibility cap of the sweep (1 without contact) */
} jgs2_sweep_info;

typedef struct jgs2_factor_info {
  int64_t n_free;          /* factored (free) vertices */
  int64_t nnz_dof;         /* stored lower-triangular entries (DOF units) */
  int64_t nfronts;
  int64_t nlevels;
  int64_t max_front;       /* largest front order (DOFs) */
  double factor_seconds;
  int64_t ordering;        /* 1 METIS nested dissection (default), 0 geometric nested dissection */
} jgs2_factor_info;

/* ---- lifecycle ------------------------------------------------------- */
jgs2_ctx* jgs2_create(int32_t device);
void jgs2_destroy(jgs2_ctx* ctx);
const char* jgs2_last_error(const jgs2_ctx* ctx);
int32_t jgs2_device_count(void);

/* ---- setup (LocalSolver.__init__, local_solver.py:217-240) ------------ */
int32_t jgs2_set_model(jgs2_ctx* ctx, const jgs2_model* model);
int32_t jgs2_set_precompute(jgs2_ctx* ctx, const jgs2_precompute* pre, const jgs2_config* cfg);
/* Vertex colours for the Gauss-Seidel schedule (Model.colors, greedy
 * first-fit in ascending vertex id, mesh.py:164-178; nv entries): free
 * vertices are updated colour by colour, ascending (local_solver.py:298-303). */
int32_t jgs2_set_colors(jgs2_ctx* ctx, const int64_t* colors);
/* Fill-reducing ordering of the next factorization: 1 = METIS nested
 * dissection (cusolverSpXcsrmetisndHost) with an elimination-tree front tree,
 * fronts amalgamated up to leaf_size vertices (the default); 0 = geometric
 * nested dissection with leaves of leaf_size vertices (the scalable
 * precompute's large fronts). */
int32_t jgs2_set_ordering(jgs2_ctx* ctx, int32_t ordering);
/* Schedule of the element Hessians (no reference counterpart; a tuning knob):
 * blocks_per_sm > 0 runs them on a side stream under the factor solve, capped
 * at that many resident blocks per SM (default 1, or JGS2_HESS_OVERLAP);
 * 0 runs them just before the local systems. Results are identical. */
int32_t jgs2_set_hess_overlap(jgs2_ctx* ctx, int32_t blocks_per_sm);
/* Rest Hessian M/h^2 + PSD elastic, Dirichlet-eliminated, factored on the
 * device (replaces subspace.rest_factorization, subspace.py:126-130). */
int32_t jgs2_factor_rest(jgs2_ctx* ctx, double h_ref, int32_t leaf_size, jgs2_factor_info* info);

/* Factor a caller-supplied rest Hessian given as 3x3 blocks (row vertex,
 * column vertex, row-major values) over the free vertices -- e.g. the very
 * matrix the reference factored with SuperLU (harness.py:76-77). Blocks
 * touching fixed vertices are ignored (their rows are identity). */
int32_t jgs2_factor_blocks(jgs2_ctx* ctx, int64_t nblocks, const int64_t* brow, const int64_t* bcol,
                           const double* bval, int32_t leaf_size, jgs2_factor_info* info);

/* Fill of the factor: out[0] = stored supernodal entries (DOF units, the
 * bytes the solve streams), out[1] = exact Cholesky fill of the factor's own
 * ordering, out[2] = exact fill of METIS nested dissection
 * (cusolverSpXcsrmetisndHost) of the whole graph. */
int32_t jgs2_factor_fill(jgs2_ctx* ctx, int64_t* out);

/* ---- state ----------------------------------------------------------- */
int32_t jgs2_set_state(jgs2_ctx* ctx, const double* x, const double* z, double h);
int32_t jgs2_set_x(jgs2_ctx* ctx, const double* x);
int32_t jgs2_get_x(jgs2_ctx* ctx, double* x);
int32_t jgs2_get_dx(jgs2_ctx* ctx, double* dx);
int32_t jgs2_set_rotations(jgs2_ctx* ctx, const double* rotations /* nv*9 */);
int32_t jgs2_get_rotations(jgs2_ctx* ctx, double* rotations);

/* ---- hot path -------------------------------------------------------- */
/* vertex_rotations(model, x) on the device state (subspace.py:206-231). */
int32_t jgs2_rotations(jgs2_ctx* ctx);
/* One Jacobi sweep on the device state (LocalSolver.sweep,
 * local_solver.py:606-655). refresh_rotations != 0 recomputes the vertex
 * rotations at x first, fused with the assembled-field pass (one
 * outer_solve iteration, local_solver.py:699-703); 0 uses the context's
 * current rotations. */
int32_t jgs2_sweep(jgs2_ctx* ctx, int32_t refresh_rotations, jgs2_sweep_info* info);
/* End-to-end sweep from HOST buffers: x, z in; x, dx out
 * (h2d of x,z and d2h of x,dx inside the call). rotations may be NULL
 * (then computed on device from x, as outer_solve does). */
int32_t jgs2_sweep_host(jgs2_ctx* ctx, const double* x, const double* z, double h,
                        const double* rotations, double* x_out, double* dx_out,
                        jgs2_sweep_info* info);
/* outer_solve (local_solver.py:688-721) on the device state. Per-iteration
 * arrays have capacity max_outer; returns iterations in *iterations. */
int32_t jgs2_outer_solve(jgs2_ctx* ctx, double* dx_norms, double* grad_norms, double* energies,
                         double* max_local_steps, int64_t* activations, int32_t* iterations,
                         int32_t* converged);

/* ---- frame driver (device-resident timesteps) ------------------------- */
/* x_prev, v host arrays (nv*3), gravity[3]. */
int32_t jgs2_set_frame_state(jgs2_ctx* ctx, const double* x_prev, const double* v, double h,
                             const double* gravity);
/* z = x_prev + h v + h^2 g (fixed: z = x_prev), x = x_prev + cap (z - x_prev)
 * with cap = feasibility_step_cap (assembly.py:165-180, harness.py:130-134). */
int32_t jgs2_frame_begin(jgs2_ctx* ctx, double* cap);
/* restore the frame state saved by jgs2_set_frame_state (device copy) */
int32_t jgs2_frame_reset(jgs2_ctx* ctx);
/* v = (x - x_prev) / h; x_prev = x (assembly.py:346-351). */
int32_t jgs2_frame_end(jgs2_ctx* ctx);
int32_t jgs2_get_frame_state(jgs2_ctx* ctx, double* x_prev, double* v);
/* One timestep from HOST buffers, as harness.run does per frame
 * (harness.py:187-211: compute_z, initialize_step with the feasibility cap,
 * outer_solve to tol_dx, step_velocity_update): x_prev, v (nv*3) in, the new
 * x_prev (= x) and v out (outputs may alias inputs); gravity[3] may be NULL. */
int32_t jgs2_timestep_host(jgs2_ctx* ctx, const double* x_prev, const double* v, double h,
                           const double* gravity, double* x_prev_out, double* v_out,
                           int32_t* iterations, int32_t* converged);

/* ---- per-kernel entry points (parity tests; device state in/out) ------- */
int32_t jgs2_total_energy(jgs2_ctx* ctx, const double* x, double* energy);
int32_t jgs2_assembled_field(jgs2_ctx* ctx, double* g_asm /* nv*3 */);
int32_t jgs2_reduced_collect(jgs2_ctx* ctx, const double* rotations, const double* g_asm,
                             double* q /* nv*3 */);
int32_t jgs2_sampled_corrections(jgs2_ctx* ctx, double* corr /* nv*9, free rows */);
int32_t jgs2_reduced_systems(jgs2_ctx* ctx, double* a /* nv*9 */, double* g /* nv*3 */);
/* Local steps at the device state (x, z, h, rotations): delta = A^-1 (-g)
 * per vertex (nv*3; _solve_batch, local_solver.py:580-588), the local
 * search's final step fraction alpha (nv; _line_search + _alpha_caps,
 * local_solver.py:450-470, 530-553; 1 for fixed vertices) and the
 * activation count (vertices not accepted at alpha0). */
int32_t jgs2_local_step(jgs2_ctx* ctx, double* delta, double* alpha, int64_t* activations);
/* Active pairs at the device x: rows of 10 doubles
 * (kind, vertex, tri0, tri1, tri2, plane, d, bary0, bary1, bary2). */
int32_t jgs2_find_pairs(jgs2_ctx* ctx, double* rows, int64_t capacity, int64_t* count);
int32_t jgs2_last_kernel_launches(jgs2_ctx* ctx, int64_t* launches);

/* ---- measurement ------------------------------------------------------ */
#define JGS2_NPHASES 11
/* phases: 0 vertex pass (rotations + assembled field), 1 collect rhs,
 * 2 factor solve (forward + backward), 3 cubature element Hessians,
 * 4 local systems + line search, 5 energy evaluations, 6 update/finalize,
 * 7 contact pairs at x (detection, pair terms, gradients), 8 sweep
 * feasibility cap, 9 backtracking barrier trials (candidates + energies),
 * 10 per-frame initial-guess feasibility cap. */
int32_t jgs2_profile(jgs2_ctx* ctx, int32_t enable);
/* accumulated device ms (CUDA events on the context stream), launch
 * counts and algorithmic bytes per phase since the last reset */
int32_t jgs2_phase_stats(jgs2_ctx* ctx, double* ms, int64_t* launches, double* bytes);
int32_t jgs2_phase_reset(jgs2_ctx* ctx);
/* CUDA-event stopwatch on the context stream; the window is also a
 * cudaProfilerStart/Stop range (ncu --profile-from-start off) */
int32_t jgs2_timer_start(jgs2_ctx* ctx);
int32_t jgs2_timer_stop(jgs2_ctx* ctx, double* ms);
/* pinned host buffers for the end-to-end path */
void* jgs2_pinned_alloc(int64_t bytes);
void jgs2_pinned_free(void* p);
/* feasibility_step_cap(model, x, dx) (assembly.py:263-291) on host arrays,
 * for the frame driver's initialize_step (harness.py:130-134) */
int32_t jgs2_step_cap(jgs2_ctx* ctx, const double* x, const double* dx, double* cap);

/* ---- partitioned solve (multi-GPU) ------------------------
 * One context per GPU, one process per GPU. Each rank owns a contiguous
 * range of whole bodies (vertex ids [v_begin, v_end), its elements): it
 * factors and solves its bodies' blocks of the block-diagonal rest Hessian
 * (the exact collect, local_solver.py:115-126), and runs the vertex pass,
 * element Hessians and local systems of its vertices. Per sweep the ranks
 * all-reduce the local-search counters, dx (its owner's rows, zeros
 * elsewhere), and per-chunk partial sums of the trial energies and grad_sq;
 * contact detection, the feasibility cap and the backtracking decisions
 * run replicated on identical data. Results are bit-identical to one GPU.
 * Call order: create -> set_model -> set_comm_* -> set_partition ->
 * factor_* -> set_precompute. Jacobi mode only. */
/* all-reduce callback for jgs2_set_comm_host: reduce host_buf (count
 * elements; dtype 0 f64, 1 i32, 2 u64; op 0 sum, 1 max) in place across all
 * ranks; return 0 on success */
typedef int32_t (*jgs2_allreduce_fn)(void* host_buf, int64_t count, int32_t dtype, int32_t op, void* user);
/* ncclGetUniqueId (128 bytes), to be broadcast from rank 0 */
int32_t jgs2_nccl_unique_id(uint8_t* id128);
/* NCCL communicator created by the context (ncclCommInitRank) */
int32_t jgs2_set_comm_nccl(jgs2_ctx* ctx, int32_t world, int32_t rank, const uint8_t* id128);
/* caller-owned ncclComm_t (not destroyed by the context) */
int32_t jgs2_set_comm_nccl_handle(jgs2_ctx* ctx, int32_t world, int32_t rank, void* nccl_comm);
/* host-callback collectives (tests: ranks sharing one GPU over gloo) */
int32_t jgs2_set_comm_host(jgs2_ctx* ctx, int32_t world, int32_t rank, jgs2_allreduce_fn fn, void* user);
/* own vertices [v_begin, v_end): must start and end at body boundaries */
int32_t jgs2_set_partition(jgs2_ctx* ctx, int64_t v_begin, int64_t v_end);
/* context on a caller-provided CUDA stream (cudaStream_t; NULL = own) */
jgs2_ctx* jgs2_create_on_stream(int32_t device, void* stream);

/* ---- scalable precompute (replaces harness.prepare's
 * subspace.precompute_bases + retain_rows + cubature.train_all,
 * harness.py:57-107, subspace.py:133-203, cubature.py:113-291) ------------
 * Call order on a context with the model set and the rest factor built
 * (jgs2_factor_rest): jgs2_selected_inverse -> (training inputs) ->
 * jgs2_precompute_train -> jgs2_precompute_export. */
/* Hbar^-1 on the factor's pattern (Takahashi equations, cuBLAS per front) */
int32_t jgs2_selected_inverse(jgs2_ctx* ctx, double* seconds);
/* (Hbar^-1)_{w v} 3x3 blocks (row-major) for n vertex pairs; found[k] = 0
 * when (v, w) is not adjacent in the filled graph */
int32_t jgs2_inverse_blocks(jgs2_ctx* ctx, int64_t n, const int64_t* v, const int64_t* w, double* out,
                            int32_t* found);
/* element stencil gradients at x (cubature.stencil_gradients,
 * cubature.py:37-60): out[ne*12], vertex-major element DOFs */
int32_t jgs2_stencil_gradients(jgs2_ctx* ctx, const double* x, const double* z, double h, double* out);
typedef struct jgs2_train_params {
  int32_t n_poses;              /* T training poses (cubature.build_training_set) */
  int32_t candidates_per_round; /* 32 */
  int32_t max_size;             /* 6 */
  int32_t pad_;
  double target_residual;       /* 0.01 */
  uint64_t seed;
  const double* pose_grads;     /* T*ne*12 stencil gradients per pose */
  const double* pose_solves;    /* T*nv*3: Hbar^-1 applied to each pose's assembled gradient */
} jgs2_train_params;
/* bases + cubature sets of every free vertex; sizes = [n_bases, retained
 * rows, cubature elements] */
int32_t jgs2_precompute_train(jgs2_ctx* ctx, const jgs2_train_params* params, int64_t* sizes);
/* the jgs2_precompute layout (gbar_rows = gbar, group = the vertex; Jacobi
 * sub-problems, harness.py:66-69) plus per-vertex training residual and
 * converged flag */
int32_t jgs2_precompute_export(jgs2_ctx* ctx, int64_t* vertices, double* gbar, int64_t* vrows_ptr,
                               int64_t* vrows_keys, double* vrows, int64_t* cub_ptr, int64_t* cub_elems,
                               double* cub_weights, double* residual, uint8_t* converged);

/* ---- symbolic analysis (host only; no device needed) ------------------ */
typedef struct jgs2_sym jgs2_sym;
jgs2_sym* jgs2_sym_build(int64_t n, const int64_t* adj_ptr, const int32_t* adj,
                         const double* coords, int32_t leaf_size);
/* sizes[0]=nfronts, [1]=struct entries, [2]=nlevels, [3]=nnz_dof */
int32_t jgs2_sym_sizes(const jgs2_sym* s, int64_t* sizes);
int32_t jgs2_sym_export(const jgs2_sym* s, int32_t* perm, int32_t* parent, int32_t* col_begin,
                        int32_t* col_end, int64_t* struct_ptr, int32_t* struct_pos,
                        int32_t* level);
void jgs2_sym_free(jgs2_sym* s);

#ifdef __cplusplus
}
#endif
#endif /* JGS2_H */
