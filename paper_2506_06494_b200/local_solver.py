"""Drop-in GPU ``LocalSolver`` for the reference's hot path.

Mirrors ``tetsolve.local_solver`` (``local_solver.py:38-69, 214-721``): the
same ``SolverConfig`` / ``IterationStats`` dataclasses, the same constructor
``LocalSolver(model, config, bases, cubature_sets, factor)`` and the same
``sweep(state, rotations=None) -> (dx, info)`` / ``outer_solve(state) ->
IterationStats`` semantics (both mutate ``state.x``; ``outer_solve`` also sets
``state.rotations``). Every sweep runs as sm_100a kernels behind the C ABI in
``include/jgs2.h``; Python only marshals host arrays. There is no CPU
fallback: a missing library or device raises ``RuntimeError``.

Scope: ``subspace="corotated_cubature"`` with ``mode="jacobi"`` (the
reference defaults) or ``mode="gauss_seidel"`` (colour sweeps,
local_solver.py:627-649). ``exact`` (a <=6000-DOF verification path) and
``none`` (the plain VBD baseline) are out of scope and raise
``ValueError``.
"""

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib as L
from .precompute import Precompute

SUBSPACE_MODES = ("exact", "corotated_cubature", "none")
SCHEDULES = ("jacobi", "gauss_seidel")
FeasibilityError = L.FeasibilityError
PrecomputeError = L.PrecomputeError


@dataclass
class SolverConfig:
    """local_solver.py:38-56."""
    mode: str = "jacobi"
    subspace: str = "corotated_cubature"
    tol_dx: float = 1e-3
    max_outer: int = 500
    local_line_search: bool = True
    track_energy: bool = True
    exact_size_cap: int = 6000
    max_halvings: int = 30
    alpha_floor: float = 1e-6

    def __post_init__(self):
        if self.mode not in SCHEDULES:
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.subspace not in SUBSPACE_MODES:
            raise ValueError(f"unknown subspace {self.subspace!r}")
        if self.tol_dx <= 0:
            raise ValueError("tol_dx must be positive")


@dataclass
class IterationStats:
    """local_solver.py:59-69."""
    energies: list = field(default_factory=list)
    dx_norms: list = field(default_factory=list)
    grad_norms: list = field(default_factory=list)
    max_local_steps: list = field(default_factory=list)
    line_search_activations: list = field(default_factory=list)
    wall_ms: list = field(default_factory=list)
    outer_iterations: int = 0
    wall_seconds: float = 0.0
    converged: bool = False


def vertex_adjacency(model):
    """Vertex graph of the mesh (vertices sharing a tet, self loops included):
    the block pattern of the rest Hessian (assembly.py:194-259)."""
    tets = np.asarray(model.tets, dtype=np.int64)
    nv = int(model.num_vertices)
    r = np.repeat(tets, 4, axis=1).ravel()
    c = np.tile(tets, (1, 4)).ravel()
    a = sp.csr_matrix((np.ones(r.size, dtype=np.int8), (r, c)), shape=(nv, nv))
    a = (a + sp.identity(nv, dtype=np.int8, format="csr")).tocsr()
    a.sum_duplicates()
    a.data[:] = 1
    return a


def hbar_from_factor(factor, model):
    """Recover the matrix a factorization object was built from, on the mesh
    pattern only, from its ``.solve``-free triangular factors.

    The reference passes ``subspace.rest_factorization(hbar)`` -- a SciPy
    SuperLU with Pr A Pc = L U (subspace.py:126-130) -- as ``factor``
    (harness.py:120-127). Forming L U densifies every fill position, so
    instead A is probed: a distance-2 colouring of the vertex graph groups
    columns that share no row, and A @ (sum of a colour's unit vectors) for
    each colour and DOF component is one product with U then L. Each probe
    entry at a row adjacent to the colour's column is exactly one A entry.
    Cost: 3 x colours products with L and U (no fill-sized temporaries).
    Returns a CSR matrix on the vertex-block pattern."""
    n = factor.shape[0]
    adj = vertex_adjacency(model)
    nv = adj.shape[0]
    if n != 3 * nv:
        raise ValueError(f"factor order {n} does not match 3 x {nv} vertices")
    # distance-2 greedy colouring (ascending vertex id)
    a2 = (adj @ adj).tocsr()
    colour = np.full(nv, -1, dtype=np.int64)
    for v in range(nv):
        used = colour[a2.indices[a2.indptr[v]:a2.indptr[v + 1]]]
        taken = np.zeros(used.max(initial=-1) + 2, dtype=bool)
        taken[used[used >= 0]] = True
        colour[v] = int(np.flatnonzero(~taken)[0])
    ncol = int(colour.max()) + 1
    # probe block: column (3 c + d) = sum over vertices w of colour c of e_{3w+d}
    cols = (3 * colour[:, None] + np.arange(3)).ravel()
    rows = np.arange(3 * nv)
    probe = sp.csc_matrix((np.ones(3 * nv), (rows, cols)), shape=(3 * nv, 3 * ncol))
    # SciPy's convention Pr A Pc = L U with Pr e_i = e_perm_r[i] and
    # Pc e_perm_c[i] = e_i, so A x = Pr^T L U Pc^T x, (Pc^T x)[perm_c] = x
    # and (Pr^T w) = w[perm_r]
    dense = probe.toarray()
    z = np.empty_like(dense)
    z[np.asarray(factor.perm_c)] = dense
    w = factor.L @ (factor.U @ z)
    out = w[np.asarray(factor.perm_r)]
    # scatter back to the block pattern: entry (3v + r, 3w + d) = out[3v + r, 3 colour(w) + d]
    bp = sp.bsr_matrix((np.ones((adj.nnz, 3, 3)), adj.indices, adj.indptr), shape=(3 * nv, 3 * nv))
    coo = bp.tocoo()
    vals = out[coo.row, 3 * colour[coo.col // 3] + coo.col % 3]
    a = sp.csr_matrix((vals, (coo.row, coo.col)), shape=(3 * nv, 3 * nv))
    a.eliminate_zeros()
    return a


def matrix_blocks(hbar):
    """3x3 block triplets (row vertex, col vertex, values) of a sparse matrix."""
    b = sp.bsr_matrix(sp.csr_matrix(hbar), blocksize=(3, 3))
    b.sum_duplicates()
    nvb = b.shape[0] // 3
    rows = np.repeat(np.arange(nvb, dtype=np.int64), np.diff(b.indptr))
    return rows, b.indices.astype(np.int64), np.ascontiguousarray(b.data, dtype=np.float64)


def _require_finite(*arrays):
    """Non-finite positions are rejected on the host: on the device they end
    in an illegal memory access that poisons the context."""
    for a in arrays:
        if not np.isfinite(a).all():
            raise ValueError("non-finite positions (NaN or inf) in the state")


class LocalSolver:
    """GPU JGS2 solver with the reference ``LocalSolver`` interface.

    ``factor`` may be the reference's SuperLU rest factorization (the matrix
    it factored is recovered on the mesh pattern and refactored on the
    device), a float ``h_ref``, or ``None`` together with ``h_ref=`` /
    ``hbar=`` keywords (``hbar=RuntimeData.hbar`` passes the reference's
    own matrix, harness.py:29-35). ``precompute`` (a
    :class:`~paper_2506_06494_b200.precompute.Precompute`) may replace
    ``bases``/``cubature_sets``. ``dist`` (torch.distributed, world > 1)
    partitions the scene by bodies across the ranks' GPUs (partition.py).
    """

    def __init__(self, model, config, bases=None, cubature_sets=None, factor=None, *,
                 precompute=None, h_ref=None, hbar=None, device=0, leaf_size=32, dist=None,
                 comm="nccl"):
        self.model = model
        self.config = config
        self.plain = config.subspace == "none"  # plain vertex block descent (local_solver.py:325-353)
        if config.subspace == "exact":
            raise ValueError("subspace 'exact' (the <=6000-DOF verification path) is not on the GPU path")
        if self.plain:
            precompute = None
        elif precompute is None:
            if not bases:
                raise ValueError("corotated_cubature needs precomputed bases")
            precompute = Precompute.from_reference(bases, cubature_sets or {})
        if not self.plain and hbar is None and factor is not None and hasattr(factor, "perm_r"):
            hbar = hbar_from_factor(factor, model)
        if self.plain:
            pass
        elif hbar is None and h_ref is None:
            if isinstance(factor, (int, float)):
                h_ref = float(factor)
            elif factor is not None and hasattr(factor, "h_ref"):
                h_ref = float(factor.h_ref)
            else:
                raise ValueError("corotated_cubature needs the rest-Hessian factorization "
                                 "from precomputation (factor / h_ref / hbar)")
        self.pre = precompute
        self.free = np.flatnonzero(~np.asarray(model.fixed_mask))
        self._lib = L.lib()
        if L.device_count() <= 0:
            raise RuntimeError("no CUDA device: the JGS2 path has no CPU fallback")
        self._ctx = self._lib.jgs2_create(int(device))
        if not self._ctx:
            raise RuntimeError(f"jgs2_create failed on device {device}")
        self._keep = []
        self._upload_model(model)
        # partitioned solve (partition.py): dist = an initialized
        # torch.distributed with world > 1, one rank per GPU; comm = "nccl" or
        # "host" (gloo callback, for ranks sharing a GPU in tests)
        self.partition, self._comm_keep = None, None
        if dist is not None and dist.get_world_size() > 1:
            from . import partition as P
            self._comm_keep = P.attach(self._lib, self._ctx, dist, comm)
            self.partition = P.plan(model, dist.get_world_size())[dist.get_rank()]
            self._call(self._lib.jgs2_set_partition, int(self.partition[0]), int(self.partition[1]))
        t0 = time.perf_counter()
        self.factor_info = L.FactorInfo()
        if self.plain:
            pass
        elif hbar is not None:
            br, bc, bv = matrix_blocks(hbar)
            self._call(self._lib.jgs2_factor_blocks, br.size, L.ptr(br, L.i64), L.ptr(bc, L.i64),
                       L.ptr(bv, L.f64), int(leaf_size), C_ref(self.factor_info))
        else:
            self._call(self._lib.jgs2_factor_rest, float(h_ref), int(leaf_size),
                       C_ref(self.factor_info))
        self.factor_seconds = time.perf_counter() - t0
        self._upload_precompute(precompute, config)
        self._keep = None
        self.nv = model.num_vertices

    # ------------------------------------------------------------ plumbing
    def _call(self, fn, *args):
        L.check(fn(self._ctx, *args), self._ctx)

    def _upload_model(self, m):
        upload_model(self._lib, self._ctx, m, self._keep)

    def _upload_precompute(self, p, cfg):
        k = self._keep
        arr = lambda a, f: k.append(f(a)) or k[-1]  # noqa: E731
        if p is None:  # plain mode: configuration only
            c = self._config_struct(cfg)
            c.subspace = 1
            self._call(self._lib.jgs2_set_precompute, None, C_ref(c))
            if cfg.mode == "gauss_seidel":
                colors = L.i64a(self.model.colors)
                self._call(self._lib.jgs2_set_colors, L.ptr(colors, L.i64))
            return
        d = L.Precompute()
        d.n_bases = int(np.asarray(p.vertices).size)
        d.gmax = int(np.asarray(p.group).shape[1])
        d.vertices = L.ptr(arr(p.vertices, L.i64a), L.i64)
        d.gbar = L.ptr(arr(p.gbar, L.f64a), L.f64)
        d.group = L.ptr(arr(p.group, L.i64a), L.i64)
        d.gbar_rows = L.ptr(arr(p.gbar_rows, L.f64a), L.f64)
        d.vrows_ptr = L.ptr(arr(p.vrows_ptr, L.i64a), L.i64)
        d.vrows_keys = L.ptr(arr(p.vrows_keys, L.i64a), L.i64)
        d.vrows = L.ptr(arr(p.vrows, L.f64a), L.f64)
        d.cub_ptr = L.ptr(arr(p.cub_ptr, L.i64a), L.i64)
        d.cub_elems = L.ptr(arr(p.cub_elems, L.i64a), L.i64)
        d.cub_weights = L.ptr(arr(p.cub_weights, L.f64a), L.f64)
        c = self._config_struct(cfg)
        self._call(self._lib.jgs2_set_precompute, C_ref(d), C_ref(c))
        if cfg.mode == "gauss_seidel":  # colour groups (local_solver.py:298-303)
            colors = L.i64a(self.model.colors)
            self._call(self._lib.jgs2_set_colors, L.ptr(colors, L.i64))

    @staticmethod
    def _config_struct(cfg):
        c = L.Config()
        c.tol_dx = float(cfg.tol_dx)
        c.max_outer = int(cfg.max_outer)
        c.local_line_search = int(bool(cfg.local_line_search))
        c.track_energy = int(bool(cfg.track_energy))
        c.max_halvings = int(cfg.max_halvings)
        c.alpha_floor = float(cfg.alpha_floor)
        c.mode = SCHEDULES.index(cfg.mode)
        c.subspace = 0
        return c

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.jgs2_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_launches(self):
        n = L.i64(0)
        L.check(self._lib.jgs2_last_kernel_launches(self._ctx, C_ref(n)))
        return int(n.value)

    # ------------------------------------------------------------ measurement
    def factor_fill(self):
        """(stored supernodal nnz, exact fill of the same ordering, exact fill
        of METIS nested dissection), DOF units (jgs2_factor_fill)."""
        out = np.zeros(3, dtype=np.int64)
        self._call(self._lib.jgs2_factor_fill, L.ptr(out, L.i64))
        return tuple(int(x) for x in out)

    def set_hess_overlap(self, blocks_per_sm):
        """Element Hessians under the factor solve, capped at blocks_per_sm
        resident blocks per SM (0: just before the local systems)."""
        self._call(self._lib.jgs2_set_hess_overlap, int(blocks_per_sm))

    def profile(self, enable=True):
        self._call(self._lib.jgs2_profile, int(bool(enable)))

    def phase_reset(self):
        self._call(self._lib.jgs2_phase_reset)

    def phase_stats(self):
        """{phase: (device ms, kernel launches, algorithmic bytes)}."""
        k = len(L.PHASES)
        ms = np.zeros(k)
        n = np.zeros(k, dtype=np.int64)
        by = np.zeros(k)
        self._call(self._lib.jgs2_phase_stats, L.ptr(ms, L.f64), L.ptr(n, L.i64), L.ptr(by, L.f64))
        return {p: (float(ms[i]), int(n[i]), float(by[i])) for i, p in enumerate(L.PHASES)}

    def timer_start(self):
        self._call(self._lib.jgs2_timer_start)

    def timer_stop(self):
        ms = L.f64(0.0)
        self._call(self._lib.jgs2_timer_stop, C_ref(ms))
        return float(ms.value)

    def step_cap(self, x, dx):
        """feasibility_step_cap (assembly.py:263-291) on the device."""
        cap = L.f64(1.0)
        self._call(self._lib.jgs2_step_cap, L.ptr(L.f64a(x), L.f64), L.ptr(L.f64a(dx), L.f64),
                   C_ref(cap))
        return float(cap.value)

    def initialize_step(self, state):
        """Warm start at the predictor, feasibility-capped (harness.py:130-134)."""
        dx = state.z - state.x_prev
        state.x = state.x_prev + self.step_cap(state.x_prev, dx) * dx

    # ------------------------------------------------------------ state I/O
    def set_state(self, x, z, h):
        self._call(self._lib.jgs2_set_state, L.ptr(L.f64a(x), L.f64), L.ptr(L.f64a(z), L.f64),
                   float(h))

    def get_x(self):
        out = np.empty((self.nv, 3))
        self._call(self._lib.jgs2_get_x, L.ptr(out, L.f64))
        return out

    def get_dx(self):
        out = np.empty((self.nv, 3))
        self._call(self._lib.jgs2_get_dx, L.ptr(out, L.f64))
        return out

    def set_rotations(self, rot):
        self._call(self._lib.jgs2_set_rotations, L.ptr(L.f64a(rot), L.f64))

    def get_rotations(self):
        out = np.empty((self.nv, 3, 3))
        self._call(self._lib.jgs2_get_rotations, L.ptr(out, L.f64))
        return out

    @staticmethod
    def _info_dict(inf):
        return {"line_search_activations": int(inf.line_search_activations),
                "max_local_step": float(inf.max_local_step),
                "grad_norm": float(inf.grad_norm), "grad_sq": float(inf.grad_sq),
                "dx_norm": float(inf.dx_norm), "energy": float(inf.energy),
                "halvings": int(inf.halvings), "n_pairs": int(inf.n_pairs),
                "n_indefinite": int(inf.n_indefinite), "gamma": float(inf.gamma),
                "cap": float(inf.cap)}

    # ------------------------------------------------------------ hot path
    def sweep(self, state, rotations=None):
        """One outer iteration; returns (dx applied, info dict)
        (local_solver.py:606-655). Like the reference, ``rotations=None``
        means identity rotations."""
        if rotations is None:
            rotations = np.broadcast_to(np.eye(3), (self.nv, 3, 3))
        x = L.f64a(state.x)
        z = L.f64a(state.z)
        _require_finite(x, z)
        rot = L.f64a(rotations)
        x_out = np.empty_like(x)
        dx = np.empty_like(x)
        inf = L.SweepInfo()
        self._call(self._lib.jgs2_sweep_host, L.ptr(x, L.f64), L.ptr(z, L.f64), float(state.h),
                   L.ptr(rot, L.f64), L.ptr(x_out, L.f64), L.ptr(dx, L.f64), C_ref(inf))
        state.x = x_out
        return dx, self._info_dict(inf)

    def sweep_resident(self, refresh_rotations=True):
        """Device-resident sweep (no host copies of x/z); returns info."""
        inf = L.SweepInfo()
        self._call(self._lib.jgs2_sweep, int(bool(refresh_rotations)), C_ref(inf))
        return self._info_dict(inf)

    def outer_solve(self, state):
        """Sweeps until the normalized position change drops below tol_dx
        (local_solver.py:688-721); rotations refreshed every sweep on the
        device, fused with the assembled-field pass."""
        cfg = self.config
        stats = IterationStats()
        t0 = time.perf_counter()
        _require_finite(state.x, state.z)
        self.set_state(state.x, state.z, state.h)
        for _ in range(cfg.max_outer):
            t1 = time.perf_counter()
            info = self.sweep_resident(refresh_rotations=not self.plain)
            stats.wall_ms.append(1e3 * (time.perf_counter() - t1))
            stats.dx_norms.append(info["dx_norm"])
            stats.grad_norms.append(info["grad_norm"])
            stats.max_local_steps.append(info["max_local_step"])
            stats.line_search_activations.append(info["line_search_activations"])
            if cfg.track_energy:
                stats.energies.append(info["energy"])
            stats.outer_iterations += 1
            if info["dx_norm"] < cfg.tol_dx:
                stats.converged = True
                break
        state.x = self.get_x()
        if not self.plain:  # plain mode leaves state.rotations alone (local_solver.py:699-702)
            state.rotations = self.get_rotations()
        stats.wall_seconds = time.perf_counter() - t0
        return stats

    # ------------------------------------------------- device frame driver
    def set_frame_state(self, state, gravity):
        """Upload (x_prev, v, h) for device-resident timesteps."""
        g = L.f64a(gravity)
        self._call(self._lib.jgs2_set_frame_state, L.ptr(L.f64a(state.x_prev), L.f64),
                   L.ptr(L.f64a(state.v), L.f64), float(state.h), L.ptr(g, L.f64))

    def run_frames(self, frames):
        """``frames`` timesteps fully on the device: compute_z + capped
        initialize_step, outer_solve sweeps to tol_dx, velocity update
        (harness.py:187-211 without the file outputs). Returns per-frame
        (iterations, converged)."""
        out = []
        cap = L.f64(1.0)
        for _ in range(frames):
            self._call(self._lib.jgs2_frame_begin, C_ref(cap))
            it, conv = 0, False
            for it in range(1, self.config.max_outer + 1):
                info = self.sweep_resident(refresh_rotations=True)
                if info["dx_norm"] < self.config.tol_dx:
                    conv = True
                    break
            self._call(self._lib.jgs2_frame_end)
            out.append((it, conv))
        return out

    def timestep(self, state, gravity, x_prev_out=None, v_out=None):
        """One harness timestep from host arrays (harness.py:187-211 per
        frame: compute_z, capped initialize_step, outer_solve to tol_dx,
        step_velocity_update) in one ABI call. ``state.x_prev`` / ``state.v``
        go to the device; the new x_prev and v are written to ``x_prev_out`` /
        ``v_out`` (default: in place, and then ``state.x`` = the new x and
        ``state.z`` = the frame's z, as compute_z / step_velocity_update leave
        them, assembly.py:165-180, 346-351). Returns (iterations, converged)."""
        xp = L.f64a(state.x_prev)
        v = L.f64a(state.v)
        in_place = x_prev_out is None
        if in_place:  # the frame's z (compute_z) from the inputs, before they are overwritten
            z = xp + state.h * v + state.h ** 2 * np.asarray(gravity, dtype=np.float64)
            fm = np.asarray(self.model.fixed_mask)
            z[fm] = xp[fm]
        xo = xp if in_place else x_prev_out
        vo = v if v_out is None else v_out
        g = L.f64a(gravity)
        it, conv = L.i32(0), L.i32(0)
        self._call(self._lib.jgs2_timestep_host, L.ptr(xp, L.f64), L.ptr(v, L.f64), float(state.h),
                   L.ptr(g, L.f64), L.ptr(xo, L.f64), L.ptr(vo, L.f64), C_ref(it), C_ref(conv))
        if in_place:
            state.x_prev, state.v = xp, v
            state.x, state.z = xp.copy(), z
        return int(it.value), bool(conv.value)

    def run_sweeps(self, budget, record=None):
        """Continue the device-resident simulation for exactly ``budget``
        sweeps (frames end on convergence or max_outer; a frame still open
        when the budget runs out is resumed by the next call). Per-sweep info
        dicts are appended to ``record`` when given. Returns the list of
        iteration counts of the frames completed."""
        done = []
        left = budget
        cap = L.f64(1.0)
        while left > 0:
            if not getattr(self, "_frame_open", False):
                self._call(self._lib.jgs2_frame_begin, C_ref(cap))
                self._frame_open, self._frame_iters = True, 0
            info = self.sweep_resident(refresh_rotations=True)
            if record is not None:
                record.append(info)
            left -= 1
            self._frame_iters += 1
            if info["dx_norm"] < self.config.tol_dx or self._frame_iters >= self.config.max_outer:
                self._call(self._lib.jgs2_frame_end)
                done.append(self._frame_iters)
                self._frame_open = False
        return done

    def get_frame_state(self):
        xp = np.empty((self.nv, 3))
        v = np.empty((self.nv, 3))
        self._call(self._lib.jgs2_get_frame_state, L.ptr(xp, L.f64), L.ptr(v, L.f64))
        return xp, v

    # ------------------------------------------------- per-kernel entry points
    def total_energy(self, x):
        e = L.f64(0.0)
        self._call(self._lib.jgs2_total_energy, L.ptr(L.f64a(x), L.f64), C_ref(e))
        return float(e.value)

    def assembled_field(self, x, z, h):
        self.set_state(x, z, h)
        out = np.empty((self.nv, 3))
        self._call(self._lib.jgs2_assembled_field, L.ptr(out, L.f64))
        return out

    def collect(self, rotations, g_asm):
        q = np.empty((self.nv, 3))
        self._call(self._lib.jgs2_reduced_collect, L.ptr(L.f64a(rotations), L.f64),
                   L.ptr(L.f64a(g_asm), L.f64), L.ptr(q, L.f64))
        return q

    def rotations(self, x):
        self._call(self._lib.jgs2_set_x, L.ptr(L.f64a(x), L.f64))
        self._call(self._lib.jgs2_rotations)
        return self.get_rotations()

    def reduced_systems(self, x, z, h, rotations):
        """(A, g) for all free vertices (local_solver.py:392-416)."""
        self.set_state(x, z, h)
        self.set_rotations(rotations)
        a = np.zeros((self.nv, 3, 3))
        g = np.zeros((self.nv, 3))
        self._call(self._lib.jgs2_reduced_systems, L.ptr(a, L.f64), L.ptr(g, L.f64))
        return a[self.free], g[self.free]

    def corrections(self, x, z, h, rotations):
        """Sampled corrections for all free vertices (local_solver.py:355-390)."""
        self.set_state(x, z, h)
        self.set_rotations(rotations)
        c = np.zeros((self.nv, 3, 3))
        self._call(self._lib.jgs2_sampled_corrections, L.ptr(c, L.f64))
        return c[self.free]

    def local_step(self, x, z, h, rotations):
        """(delta, alpha, activations) of the free vertices: the batched 3x3
        solves and the local search (local_solver.py:580-604)."""
        self.set_state(x, z, h)
        self.set_rotations(rotations)
        d = np.zeros((self.nv, 3))
        al = np.ones(self.nv)
        acts = L.i64(0)
        self._call(self._lib.jgs2_local_step, L.ptr(d, L.f64), L.ptr(al, L.f64), C_ref(acts))
        return d[self.free], al[self.free], int(acts.value)

    def find_pairs(self, x):
        """Active pair rows (kind, vertex, tri0..2, plane, d, bary0..2)."""
        self._call(self._lib.jgs2_set_x, L.ptr(L.f64a(x), L.f64))
        cap = 1 << 16
        while True:
            rows = np.zeros((cap, 10))
            cnt = L.i64(0)
            code = self._lib.jgs2_find_pairs(self._ctx, L.ptr(rows, L.f64), cap, C_ref(cnt))
            if code == 0:
                return rows[:cnt.value]
            if cnt.value > cap:
                cap = int(cnt.value)
                continue
            L.check(code, self._ctx)


def upload_model(lib, ctx, m, keep):
    """jgs2_set_model from a reference-style Model (assembly.py:40-116); host
    arrays are kept alive in ``keep`` until the call returns."""
    k = keep
    arr = lambda a, f: k.append(f(a)) or k[-1]  # noqa: E731
    nv, ne = int(m.num_vertices), int(np.asarray(m.tets).shape[0])
    d = L.Model()
    d.nv, d.ne = nv, ne
    d.rest_positions = L.ptr(arr(m.rest_positions, L.f64a), L.f64)
    d.tets = L.ptr(arr(m.tets, L.i64a), L.i64)
    d.dm_inv = L.ptr(arr(m.dm_inv, L.f64a), L.f64)
    d.volumes = L.ptr(arr(m.volumes, L.f64a), L.f64)
    d.mu = L.ptr(arr(m.mu, L.f64a), L.f64)
    d.lam = L.ptr(arr(m.lam, L.f64a), L.f64)
    d.elem_qmass = L.ptr(arr(m.elem_qmass, L.f64a), L.f64)
    d.masses = L.ptr(arr(m.masses, L.f64a), L.f64)
    d.fixed_mask = L.ptr(arr(np.asarray(m.fixed_mask, dtype=np.uint8), np.ascontiguousarray), L.u8)
    d.norm_scale = float(m.normalization.scale)
    bar = getattr(m, "barrier", None)
    d.has_barrier = 0 if bar is None else 1
    if bar is not None:
        d.dhat, d.kappa = float(bar.dhat), float(bar.kappa)
        planes = list(getattr(m, "planes", []) or [])
        d.n_planes = len(planes)
        pts = np.array([p.point for p in planes], dtype=np.float64).reshape(-1, 3)
        nrm = np.array([p.normal for p in planes], dtype=np.float64).reshape(-1, 3)
        d.plane_points = L.ptr(arr(pts, L.f64a), L.f64)
        d.plane_normals = L.ptr(arr(nrm, L.f64a), L.f64)
        d.n_bodies = len(m.bodies)
        sv = arr(m.surface_vertices, L.i64a)
        st = arr(m.surface_tris, L.i64a)
        d.n_surface_vertices, d.n_surface_tris = sv.size, st.shape[0] if st.ndim == 2 else 0
        d.surface_vertices = L.ptr(sv, L.i64)
        d.surface_tris = L.ptr(st, L.i64)
        d.vertex_body = L.ptr(arr(m.vertex_body, L.i64a), L.i64)
        d.surface_tri_body = L.ptr(arr(m.surface_tri_body, L.i64a), L.i64)
    else:
        d.n_bodies = len(getattr(m, "bodies", [0]))
        if getattr(m, "vertex_body", None) is not None:
            d.vertex_body = L.ptr(arr(m.vertex_body, L.i64a), L.i64)
    L.check(lib.jgs2_set_model(ctx, C_ref(d)), ctx)


def C_ref(obj):
    import ctypes
    return ctypes.byref(obj)
