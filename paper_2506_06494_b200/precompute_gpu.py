"""Scalable precompute on the device: bases and cubature
sets for every free vertex from one factorization of the rest Hessian.

Replaces ``harness.prepare``'s precompute (harness.py:57-107):
``subspace.rest_hessian`` / ``rest_factorization`` (subspace.py:48-57,
126-130) -> the device supernodal Cholesky (jgs2_factor_rest);
``precompute_bases`` + ``retain_rows`` (subspace.py:133-203) -> the
selected inverse of H-bar on the factor's pattern (jgs2_selected_inverse,
selinv.cuh), which holds every block the bases read; ``rest_eigenmodes``
(subspace.py:240-267) -> ARPACK shift-invert with the device solve as the
inverse operator (same start vector, v0 = default_rng(0)); the training set
(cubature.py:63-80) -> device stencil gradients per pose; ``train_all``
(cubature.py:279-291) -> train.cuh (greedy selection + Lawson-Hanson NNLS per
vertex, OpenMP over the factor's fronts).

The reference keeps a dense N x 3 column per vertex (O(N^2) memory, dense
3N-column solve); it cannot run past ~50K tets. The bases here
equal the reference's (tests/test_gpu_precompute.py pins them to the
reference's own C1 bases); the cubature candidate pool is restricted to the
elements of the vertex's front (see train.cuh), so the cubature sets differ
from the reference's random global draws.
"""

import ctypes as C
import time

import numpy as np

from . import _lib as L
from .local_solver import upload_model
from .precompute import Precompute


def scalable_precompute(model, h_ref, *, max_size=6, training_poses=2, amplitude_fraction=0.02,
                        target_residual=0.01, candidates_per_round=32, seed=0, device=0, leaf_size=512):
    """(Precompute, info) for ``model`` at time step ``h_ref`` (the cubature
    settings are CubatureConfig's, scene.py:42-47)."""
    import scipy.sparse.linalg as spla
    lib = L.lib()
    if L.device_count() <= 0:
        raise RuntimeError("no CUDA device: the precompute has no CPU fallback")
    ctx = lib.jgs2_create(int(device))
    if not ctx:
        raise RuntimeError("jgs2_create failed")
    info = {}
    try:
        keep = []
        upload_model(lib, ctx, model, keep)
        t0 = time.perf_counter()
        fi = L.FactorInfo()
        # geometric nested dissection with large leaves: each vertex's front (the
        # rows the selected inverse provides, the cubature pool) is its leaf cell
        L.check(lib.jgs2_set_ordering(ctx, 0), ctx)
        L.check(lib.jgs2_factor_rest(ctx, float(h_ref), int(leaf_size), C.byref(fi)), ctx)
        info["factor_s"] = time.perf_counter() - t0
        info["nnz_L"] = int(fi.nnz_dof)
        sel = L.f64(0.0)
        L.check(lib.jgs2_selected_inverse(ctx, C.byref(sel)), ctx)
        info["selected_inverse_s"] = float(sel.value)
        nv = int(model.num_vertices)
        free = ~np.asarray(model.fixed_mask, dtype=bool)
        rid = np.ascontiguousarray(np.broadcast_to(np.eye(3), (nv, 3, 3)))
        calls = [0]

        def solve_full(g):
            """H-bar^-1 g (fixed rows zero): the device collect with R = I."""
            g = np.ascontiguousarray(g, dtype=np.float64).reshape(nv, 3)
            q = np.empty((nv, 3))
            L.check(lib.jgs2_reduced_collect(ctx, L.ptr(rid, L.f64), L.ptr(g, L.f64), L.ptr(q, L.f64)), ctx)
            calls[0] += 1
            return q

        # rest eigenmodes (subspace.rest_eigenmodes, subspace.py:240-267)
        t0 = time.perf_counter()
        fdofs = np.flatnonzero(np.repeat(free, 3))
        nf = fdofs.size
        k = min(int(training_poses), nf - 2)

        def opinv(xf):
            g = np.zeros(3 * nv)
            g[fdofs] = xf
            return solve_full(g).ravel()[fdofs]

        class _Unused(spla.LinearOperator):  # shift-invert uses only OPinv
            def __init__(self):
                super().__init__(np.float64, (nf, nf))

            def _matvec(self, x):
                raise RuntimeError("not used in shift-invert mode")

        v0 = np.random.default_rng(0).standard_normal(nf)
        vals, vecs = spla.eigsh(_Unused(), k=k, sigma=0, which="LM", v0=v0,
                                OPinv=spla.LinearOperator((nf, nf), matvec=opinv, dtype=np.float64))
        order = np.argsort(vals)
        vecs = vecs[:, order]
        modes = np.zeros((3 * nv, k))
        modes[fdofs] = vecs
        mdiag = np.repeat(np.asarray(model.masses, dtype=np.float64), 3)
        for j in range(k):
            mn = np.sqrt(modes[:, j] @ (mdiag * modes[:, j]))
            if mn > 0:
                modes[:, j] /= mn
        info["eigen_s"] = time.perf_counter() - t0
        info["eigenvalues"] = [float(v) for v in np.sort(vals)]
        # training set (cubature.build_training_set, cubature.py:63-80) and the
        # per-pose adjoint solves H-bar^-1 g_t
        t0 = time.perf_counter()
        rest = np.ascontiguousarray(model.rest_positions, dtype=np.float64)
        diag = float(np.linalg.norm(rest.max(axis=0) - rest.min(axis=0)))
        tets = np.asarray(model.tets, dtype=np.int64)
        ne = tets.shape[0]
        grads, solves = [], []
        for j in range(k):
            disp = modes[:, j].reshape(-1, 3)
            peak = np.linalg.norm(disp, axis=1).max()
            if peak <= 0:
                continue
            disp = disp * (amplitude_fraction * diag / peak)
            x = np.ascontiguousarray(rest + disp)
            sg = np.empty((ne, 12))
            L.check(lib.jgs2_stencil_gradients(ctx, L.ptr(x, L.f64), L.ptr(rest, L.f64), float(h_ref),
                                               L.ptr(sg, L.f64)), ctx)
            gsc = np.zeros((nv, 3))
            np.add.at(gsc, tets.ravel(), sg.reshape(-1, 3))
            grads.append(sg)
            solves.append(solve_full(gsc))
        T = len(grads)
        G = np.ascontiguousarray(np.stack(grads) if T else np.zeros((0, ne, 12)))
        Z = np.ascontiguousarray(np.stack(solves) if T else np.zeros((0, nv, 3)))
        info["training_s"] = time.perf_counter() - t0
        # bases + cubature (train.cuh)
        t0 = time.perf_counter()
        prm = L.TrainParams()
        prm.n_poses, prm.candidates_per_round, prm.max_size = T, int(candidates_per_round), int(max_size)
        prm.target_residual, prm.seed = float(target_residual), int(seed)
        prm.pose_grads, prm.pose_solves = L.ptr(G, L.f64), L.ptr(Z, L.f64)
        sizes = np.zeros(3, dtype=np.int64)
        L.check(lib.jgs2_precompute_train(ctx, C.byref(prm), L.ptr(sizes, L.i64)), ctx)
        nb, nk, nc = (int(x) for x in sizes)
        out = {"vertices": np.empty(nb, np.int64), "gbar": np.empty((nb, 3, 3)),
               "vrows_ptr": np.empty(nb + 1, np.int64), "vrows_keys": np.empty(nk, np.int64),
               "vrows": np.empty((nk, 3, 3)), "cub_ptr": np.empty(nb + 1, np.int64),
               "cub_elems": np.empty(nc, np.int64), "cub_weights": np.empty(nc),
               "residual": np.empty(nb), "converged": np.empty(nb, np.uint8)}
        L.check(lib.jgs2_precompute_export(
            ctx, L.ptr(out["vertices"], L.i64), L.ptr(out["gbar"], L.f64), L.ptr(out["vrows_ptr"], L.i64),
            L.ptr(out["vrows_keys"], L.i64), L.ptr(out["vrows"], L.f64), L.ptr(out["cub_ptr"], L.i64),
            L.ptr(out["cub_elems"], L.i64), L.ptr(out["cub_weights"], L.f64), L.ptr(out["residual"], L.f64),
            L.ptr(out["converged"], L.u8)), ctx)
        info["train_s"] = time.perf_counter() - t0
        info["solves"] = calls[0]
        info["n_poses"] = T
        info["residual_median"] = float(np.median(out["residual"])) if nb else 0.0
        info["converged_fraction"] = float(out["converged"].mean()) if nb else 1.0
        info["mean_cubature_size"] = float(np.diff(out["cub_ptr"]).mean()) if nb else 0.0
        pre = Precompute(vertices=out["vertices"], gbar=out["gbar"], group=out["vertices"][:, None].copy(),
                         gbar_rows=out["gbar"].copy(), vrows_ptr=out["vrows_ptr"],
                         vrows_keys=out["vrows_keys"], vrows=out["vrows"], cub_ptr=out["cub_ptr"],
                         cub_elems=out["cub_elems"], cub_weights=out["cub_weights"])
        info["residual"] = out["residual"]
        info["converged"] = out["converged"].astype(bool)
        return pre, info
    finally:
        lib.jgs2_destroy(ctx)


def inverse_blocks(ctx_lib, ctx, v, w):
    """(Hbar^-1)_{w v} blocks and found flags for vertex pairs (tests)."""
    v = np.ascontiguousarray(v, dtype=np.int64)
    w = np.ascontiguousarray(w, dtype=np.int64)
    out = np.empty((v.size, 3, 3))
    found = np.empty(v.size, dtype=np.int32)
    L.check(ctx_lib.jgs2_inverse_blocks(ctx, v.size, L.ptr(v, L.i64), L.ptr(w, L.i64), L.ptr(out, L.f64),
                                        L.ptr(found, L.i32)), ctx)
    return out, found.astype(bool)
