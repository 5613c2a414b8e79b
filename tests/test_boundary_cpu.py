"""Host side of the drop-in boundary (no GPU): the factor argument, the
reference-object adapter and the exception identities."""

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import jgs2_oracle as orc
from paper_2506_06494_b200.local_solver import hbar_from_factor, vertex_adjacency
from paper_2506_06494_b200.precompute import Precompute
from helpers import reference_objects, scene_inputs


@pytest.mark.parametrize("name", ("beam", "two_body", "c1"))
def test_hbar_recovered_from_superlu_on_mesh_pattern(golden, name):
    # the reference passes subspace.rest_factorization(hbar) (a SuperLU,
    # subspace.py:126-130) as `factor`; the matrix comes back on the mesh's
    # vertex-block pattern, without the fill of L U
    g = golden(name)
    model, _, h = scene_inputs(g)
    hb = orc.rest_hessian(model, h).tocsr()
    a = hbar_from_factor(spla.splu(hb.tocsc()), model)
    assert abs(a - hb).max() <= 1e-14 * abs(hb).max()
    assert a.nnz <= 9 * vertex_adjacency(model).nnz  # the mesh block pattern, no fill


def test_reference_objects_round_trip(golden):
    g = golden("two_body")
    _, pre, _ = scene_inputs(g)
    bases, sets = reference_objects(pre)
    back = Precompute.from_reference(bases, sets)
    for key in ("vertices", "gbar", "vrows_ptr", "vrows_keys", "vrows", "cub_ptr", "cub_elems",
                "cub_weights"):
        np.testing.assert_array_equal(np.asarray(back[key]), np.asarray(pre[key]))


def test_exceptions_are_the_references_when_importable():
    from paper_2506_06494_b200 import _lib
    try:
        import tetsolve.energy as energy
        import tetsolve.subspace as subspace
    except Exception:
        pytest.skip("tetsolve not importable here")
    assert issubclass(_lib.FeasibilityError, energy.FeasibilityError)
    assert issubclass(_lib.PrecomputeError, subspace.PrecomputeError)
