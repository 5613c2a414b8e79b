"""On-disk formats against files the reference's own
writers produced (tests/golden/make_io_goldens.py): byte-identical output,
and the reference's precompute cache loads into the GPU path's Precompute."""
from pathlib import Path

import numpy as np
import pytest

from paper_2506_06494_b200 import formats
from paper_2506_06494_b200.model import Model
from paper_2506_06494_b200.precompute import KEYS, Precompute

IO = Path(__file__).resolve().parent / "golden" / "io"


def test_metrics_csv_is_byte_identical(tmp_path):
    rows = [(1, 0, "jgs2_cubature", 1.2345678901234567e3, 0.1, 2.5e-7, 12.3456789),
            (1, 1, "jgs2_cubature", float("nan"), 1e-300, 3.0, 0.0),
            (2, 0, "jgs2_cubature", -4.0, 7.0e-4, 1.0 / 3.0, 1234567.891)]
    formats.write_metrics(tmp_path / "metrics.csv", rows)
    assert (tmp_path / "metrics.csv").read_bytes() == (IO / "metrics.csv").read_bytes()
    back = formats.read_metrics(IO / "metrics.csv")
    assert back[0][:3] == (1, 0, "jgs2_cubature") and np.isnan(back[1][3])
    assert back[2][5] == 1.0 / 3.0


def test_obj_and_node_ele_are_byte_identical(golden, tmp_path):
    g = golden("beam")
    model = Model.from_arrays(g)
    x = g["frame_x_final"][0]
    formats.export_obj(tmp_path / "f.obj", x, model.surface_tris)
    assert (tmp_path / "f.obj").read_bytes() == (IO / "beam_frame.obj").read_bytes()
    formats.save_mesh(model.tets, x, tmp_path / "b.node", tmp_path / "b.ele")
    assert (tmp_path / "b.node").read_bytes() == (IO / "beam_body0.node").read_bytes()
    assert (tmp_path / "b.ele").read_bytes() == (IO / "beam_body0.ele").read_bytes()


def test_reference_precompute_cache_loads(golden):
    # the cache written by subspace.save_bases / cubature.save_cubature holds the
    # same precompute the beam golden recorded from harness.prepare
    pre, info = formats.load_precompute_cache(IO / "beam_bases.npz", IO / "beam_cubature.npz")
    ref = Precompute.from_arrays(golden("beam"))
    for k in KEYS:
        a, b = np.asarray(getattr(pre, k)), np.asarray(getattr(ref, k))
        assert a.shape == b.shape, k
        assert np.array_equal(a, b), k
    assert info["mode"] == "jacobi" and info["h_ref"] > 0
