"""Fixtures for the on-disk formats, written by the REFERENCE's own writers.

Build container only (imports /root/reference). Writes tests/golden/io/:
  * beam_bases.npz / beam_cubature.npz: subspace.save_bases and
    cubature.save_cubature of harness.prepare(beam) (the precompute cache);
  * beam_frame.obj, beam_body0.node/.ele: mesh.export_obj / mesh.save_mesh of
    the golden beam frame-1 final positions;
  * metrics.csv: harness._write_metrics on fixed rows (incl. a NaN energy).
Usage: PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_io_goldens.py
"""
import os
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
os.environ.setdefault("TETSOLVE_CACHE_DIR", "/tmp/tetsolve_cache_io")

import numpy as np  # noqa: E402

from tetsolve import harness, subspace, cubature, mesh as meshlib  # noqa: E402
from tetsolve.scene import parse_scene  # noqa: E402

OUT = Path(__file__).resolve().parent / "io"


def main():
    OUT.mkdir(exist_ok=True)
    scene = parse_scene(REF / "scenes" / "beam.toml")
    model = harness.build_model(scene)
    rt = harness.prepare(model, scene, use_cache=False, seed=scene.seed)
    subspace.save_bases(OUT / "beam_bases.npz", rt.bases, rt.info)
    cubature.save_cubature(OUT / "beam_cubature.npz", rt.cubature_sets)
    g = np.load(Path(__file__).resolve().parent / "beam.npz")
    x = g["frame_x_final"][0]
    meshlib.export_obj(OUT / "beam_frame.obj", x, model.surface_tris)
    body = model.bodies[0]
    sl = slice(body.vertex_offset, body.vertex_offset + body.mesh.num_vertices)
    meshlib.save_mesh(body.mesh, OUT / "beam_body0.node", OUT / "beam_body0.ele", positions=x[sl])
    rows = [(1, 0, "jgs2_cubature", 1.2345678901234567e3, 0.1, 2.5e-7, 12.3456789),
            (1, 1, "jgs2_cubature", float("nan"), 1e-300, 3.0, 0.0),
            (2, 0, "jgs2_cubature", -4.0, 7.0e-4, 1.0 / 3.0, 1234567.891)]
    harness._write_metrics(OUT / "metrics.csv", rows)
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
