"""ctypes binding of the C ABI in ``include/jgs2.h`` (``lib/libjgs2.so``).

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, constructing a solver raises ``RuntimeError``.
"""

import ctypes as C
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libjgs2.so"

i32, i64, f64, u8 = C.c_int32, C.c_int64, C.c_double, C.c_uint8
P = C.POINTER

EXPORTS = (
    "jgs2_create", "jgs2_destroy", "jgs2_last_error", "jgs2_device_count",
    "jgs2_set_model", "jgs2_set_precompute", "jgs2_factor_rest", "jgs2_factor_blocks",
    "jgs2_set_colors", "jgs2_set_state", "jgs2_set_x", "jgs2_get_x", "jgs2_get_dx", "jgs2_set_rotations",
    "jgs2_get_rotations", "jgs2_rotations", "jgs2_sweep", "jgs2_sweep_host",
    "jgs2_outer_solve", "jgs2_total_energy", "jgs2_assembled_field", "jgs2_reduced_collect",
    "jgs2_sampled_corrections", "jgs2_reduced_systems", "jgs2_local_step", "jgs2_find_pairs",
    "jgs2_last_kernel_launches", "jgs2_sym_build", "jgs2_sym_sizes", "jgs2_sym_export",
    "jgs2_sym_free", "jgs2_profile", "jgs2_phase_stats", "jgs2_phase_reset", "jgs2_timer_start",
    "jgs2_timer_stop", "jgs2_pinned_alloc", "jgs2_pinned_free", "jgs2_step_cap",
    "jgs2_set_frame_state", "jgs2_frame_begin", "jgs2_frame_end", "jgs2_get_frame_state",
    "jgs2_frame_reset", "jgs2_timestep_host", "jgs2_nccl_unique_id", "jgs2_set_comm_nccl",
    "jgs2_set_comm_nccl_handle", "jgs2_set_comm_host", "jgs2_set_partition", "jgs2_create_on_stream",
    "jgs2_selected_inverse", "jgs2_inverse_blocks", "jgs2_stencil_gradients", "jgs2_precompute_train",
    "jgs2_precompute_export", "jgs2_factor_fill", "jgs2_set_ordering", "jgs2_set_hess_overlap",
)
PHASES = ("vertex_pass", "collect_rhs", "factor_solve", "cubature_hessians", "local_systems",
          "energy", "update", "contact_pairs", "contact_cap", "contact_trials", "frame_cap")


def pinned_array(shape, dtype=np.float64):
    """numpy view of page-locked host memory (freed with the returned owner)."""
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    p = lib().jgs2_pinned_alloc(n)
    if not p:
        raise RuntimeError("cudaMallocHost failed")
    buf = (C.c_char * n).from_address(p)
    arr = np.frombuffer(buf, dtype=dtype).reshape(shape)

    class _Owner:
        def __del__(self):
            try:
                lib().jgs2_pinned_free(p)
            except Exception:
                pass
    return arr, _Owner()


class Model(C.Structure):
    _fields_ = [("nv", i64), ("ne", i64), ("rest_positions", P(f64)), ("tets", P(i64)),
                ("dm_inv", P(f64)), ("volumes", P(f64)), ("mu", P(f64)), ("lam", P(f64)),
                ("elem_qmass", P(f64)), ("masses", P(f64)), ("fixed_mask", P(u8)),
                ("norm_scale", f64), ("has_barrier", i32), ("dhat", f64), ("kappa", f64),
                ("n_planes", i64), ("plane_points", P(f64)), ("plane_normals", P(f64)),
                ("n_bodies", i64), ("n_surface_vertices", i64), ("n_surface_tris", i64),
                ("surface_vertices", P(i64)), ("surface_tris", P(i64)), ("vertex_body", P(i64)),
                ("surface_tri_body", P(i64))]


class Precompute(C.Structure):
    _fields_ = [("n_bases", i64), ("gmax", i64), ("vertices", P(i64)), ("gbar", P(f64)),
                ("group", P(i64)), ("gbar_rows", P(f64)), ("vrows_ptr", P(i64)),
                ("vrows_keys", P(i64)), ("vrows", P(f64)), ("cub_ptr", P(i64)),
                ("cub_elems", P(i64)), ("cub_weights", P(f64))]


class Config(C.Structure):
    _fields_ = [("tol_dx", f64), ("max_outer", i32), ("local_line_search", i32),
                ("track_energy", i32), ("max_halvings", i32), ("alpha_floor", f64),
                ("mode", i32), ("subspace", i32)]


class SweepInfo(C.Structure):
    _fields_ = [("line_search_activations", i64), ("max_local_step", f64), ("grad_norm", f64),
                ("grad_sq", f64), ("dx_norm", f64), ("energy", f64), ("halvings", i32),
                ("n_pairs", i32), ("n_indefinite", i32), ("pad_", i32), ("gamma", f64), ("cap", f64)]


class TrainParams(C.Structure):
    _fields_ = [("n_poses", i32), ("candidates_per_round", i32), ("max_size", i32), ("pad_", i32),
                ("target_residual", f64), ("seed", C.c_uint64), ("pose_grads", P(f64)),
                ("pose_solves", P(f64))]


class FactorInfo(C.Structure):
    _fields_ = [("n_free", i64), ("nnz_dof", i64), ("nfronts", i64), ("nlevels", i64),
                ("max_front", i64), ("factor_seconds", f64), ("ordering", i64)]


_lib = None


def lib():
    """Load libjgs2.so (once) and declare prototypes. Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                           "`python paper_2506_06494_b200/build.py` (no CPU fallback exists)")
    L = C.CDLL(str(LIB_PATH))
    vp = C.c_void_p
    sig = {
        "jgs2_create": (vp, [i32]),
        "jgs2_destroy": (None, [vp]),
        "jgs2_last_error": (C.c_char_p, [vp]),
        "jgs2_device_count": (i32, []),
        "jgs2_set_model": (i32, [vp, P(Model)]),
        "jgs2_set_precompute": (i32, [vp, P(Precompute), P(Config)]),
        "jgs2_factor_rest": (i32, [vp, f64, i32, P(FactorInfo)]),
        "jgs2_factor_blocks": (i32, [vp, i64, P(i64), P(i64), P(f64), i32, P(FactorInfo)]),
        "jgs2_set_colors": (i32, [vp, P(i64)]),
        "jgs2_set_state": (i32, [vp, P(f64), P(f64), f64]),
        "jgs2_set_x": (i32, [vp, P(f64)]),
        "jgs2_get_x": (i32, [vp, P(f64)]),
        "jgs2_get_dx": (i32, [vp, P(f64)]),
        "jgs2_set_rotations": (i32, [vp, P(f64)]),
        "jgs2_get_rotations": (i32, [vp, P(f64)]),
        "jgs2_rotations": (i32, [vp]),
        "jgs2_sweep": (i32, [vp, i32, P(SweepInfo)]),
        "jgs2_sweep_host": (i32, [vp, P(f64), P(f64), f64, P(f64), P(f64), P(f64), P(SweepInfo)]),
        "jgs2_outer_solve": (i32, [vp, P(f64), P(f64), P(f64), P(f64), P(i64), P(i32), P(i32)]),
        "jgs2_total_energy": (i32, [vp, P(f64), P(f64)]),
        "jgs2_assembled_field": (i32, [vp, P(f64)]),
        "jgs2_reduced_collect": (i32, [vp, P(f64), P(f64), P(f64)]),
        "jgs2_sampled_corrections": (i32, [vp, P(f64)]),
        "jgs2_reduced_systems": (i32, [vp, P(f64), P(f64)]),
        "jgs2_local_step": (i32, [vp, P(f64), P(f64), P(i64)]),
        "jgs2_find_pairs": (i32, [vp, P(f64), i64, P(i64)]),
        "jgs2_last_kernel_launches": (i32, [vp, P(i64)]),
        "jgs2_sym_build": (vp, [i64, P(i64), P(i32), P(f64), i32]),
        "jgs2_sym_sizes": (i32, [vp, P(i64)]),
        "jgs2_sym_export": (i32, [vp, P(i32), P(i32), P(i32), P(i32), P(i64), P(i32), P(i32)]),
        "jgs2_sym_free": (None, [vp]),
        "jgs2_profile": (i32, [vp, i32]),
        "jgs2_phase_stats": (i32, [vp, P(f64), P(i64), P(f64)]),
        "jgs2_phase_reset": (i32, [vp]),
        "jgs2_timer_start": (i32, [vp]),
        "jgs2_timer_stop": (i32, [vp, P(f64)]),
        "jgs2_pinned_alloc": (vp, [i64]),
        "jgs2_pinned_free": (None, [vp]),
        "jgs2_step_cap": (i32, [vp, P(f64), P(f64), P(f64)]),
        "jgs2_set_frame_state": (i32, [vp, P(f64), P(f64), f64, P(f64)]),
        "jgs2_frame_begin": (i32, [vp, P(f64)]),
        "jgs2_frame_end": (i32, [vp]),
        "jgs2_frame_reset": (i32, [vp]),
        "jgs2_get_frame_state": (i32, [vp, P(f64), P(f64)]),
        "jgs2_timestep_host": (i32, [vp, P(f64), P(f64), f64, P(f64), P(f64), P(f64), P(i32), P(i32)]),
        "jgs2_nccl_unique_id": (i32, [P(u8)]),
        "jgs2_set_comm_nccl": (i32, [vp, i32, i32, P(u8)]),
        "jgs2_set_comm_nccl_handle": (i32, [vp, i32, i32, vp]),
        "jgs2_set_comm_host": (i32, [vp, i32, i32, vp, vp]),
        "jgs2_set_partition": (i32, [vp, i64, i64]),
        "jgs2_create_on_stream": (vp, [i32, vp]),
        "jgs2_selected_inverse": (i32, [vp, P(f64)]),
        "jgs2_factor_fill": (i32, [vp, P(i64)]),
        "jgs2_set_ordering": (i32, [vp, i32]),
        "jgs2_set_hess_overlap": (i32, [vp, i32]),
        "jgs2_inverse_blocks": (i32, [vp, i64, P(i64), P(i64), P(f64), P(i32)]),
        "jgs2_stencil_gradients": (i32, [vp, P(f64), P(f64), f64, P(f64)]),
        "jgs2_precompute_train": (i32, [vp, P(TrainParams), P(i64)]),
        "jgs2_precompute_export": (i32, [vp, P(i64), P(f64), P(i64), P(i64), P(f64), P(i64), P(i64), P(f64),
                                         P(f64), P(u8)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def ptr(a, ctype):
    """Pointer into a contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    return a.ctypes.data_as(P(ctype))


def f64a(a, shape=None):
    out = np.ascontiguousarray(a, dtype=np.float64)
    return out.reshape(shape) if shape is not None else out


def i64a(a):
    return np.ascontiguousarray(a, dtype=np.int64)


ERRORS = {-1: ValueError, -2: RuntimeError, -3: RuntimeError, -4: KeyError, -5: RuntimeError,
          -6: RuntimeError}


def _reference_base(module, name):
    """The reference's own exception class when ``tetsolve`` is importable
    (energy.py:14, subspace.py:29), so a caller's ``except
    energy.FeasibilityError`` also catches the GPU path's error; else
    Exception."""
    try:
        import importlib
        return getattr(importlib.import_module(f"tetsolve.{module}"), name)
    except Exception:
        return Exception


class FeasibilityError(_reference_base("energy", "FeasibilityError")):
    """A barrier distance reached <= 0 (reference energy.FeasibilityError)."""


class PrecomputeError(_reference_base("subspace", "PrecomputeError")):
    """Rest Hessian factorization failed (reference subspace.PrecomputeError)."""


def check(code, ctx=None):
    if code == 0:
        return
    msg = lib().jgs2_last_error(ctx).decode() if ctx else f"error {code}"
    if code == -5:
        raise FeasibilityError(msg)
    if code == -3:
        raise PrecomputeError(msg)
    raise ERRORS.get(code, RuntimeError)(msg)


def device_count():
    return int(lib().jgs2_device_count())
