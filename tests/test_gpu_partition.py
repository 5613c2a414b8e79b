"""Partitioned solve on the GPU (partition.py): two ranks, each
owning half of the tank's bodies, exchange through the host-callback
collectives over gloo (the pool has one GPU per call, so both ranks share
cuda:0; their kernels never wait on one another -- every exchange is a
host-side all-reduce). The result must be bit-identical to one process
solving the whole scene: the same positions, iteration counts and
halvings."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(name, frames, sweeps, dist=None):
    from paper_2506_06494_b200 import scenes
    from paper_2506_06494_b200.local_solver import LocalSolver, SolverConfig
    from paper_2506_06494_b200.model import SystemState
    from paper_2506_06494_b200.precompute import Precompute
    m, st, h, _ = scenes.build(name)
    pre = Precompute.injected(m, h, samples=6, seed=0)
    s = LocalSolver(m, SolverConfig(tol_dx=m.tol_dx, max_outer=200), precompute=pre, h_ref=h,
                    dist=dist, comm="host")
    out = {"part": s.partition}
    # host-buffer sweeps (the reference's sweep(state, rotations) call)
    a = SystemState(x=st.x.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
    infos = []
    for _ in range(sweeps):
        _, info = s.sweep(a, s.rotations(a.x))
        infos.append((info["line_search_activations"], info["halvings"], info["grad_norm"],
                      info["energy"], info["n_indefinite"]))
    out["sweep_x"], out["sweep_info"] = a.x, infos
    out["rot"] = s.get_rotations()
    # device-resident frames (compute_z, capped predictor, sweeps to tol_dx, velocity update)
    init = SystemState(x=st.x_prev.copy(), x_prev=st.x_prev.copy(), v=st.v.copy(), z=st.z.copy(), h=h)
    s.set_frame_state(init, m.gravity)
    out["frames"] = s.run_frames(frames)
    out["frame_x"] = s.get_x()
    s.close()
    return out


def _worker(rank, world, port, name, frames, sweeps, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = _run(name, frames, sweeps, dist)
    np.savez(f"{path}_{rank}.npz", sweep_x=out["sweep_x"], frame_x=out["frame_x"], rot=out["rot"],
             sweep_info=np.array(out["sweep_info"]), frames=np.array(out["frames"]),
             part=np.array(out["part"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("name,frames,sweeps", [("c4s8", 2, 3), ("c4t6", 1, 2)])
def test_two_ranks_bit_identical_to_one(tmp_path, name, frames, sweeps):
    ref = _run(name, frames, sweeps)
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, frames, sweeps, str(tmp_path / "r")),
             nprocs=world, join=True)
    parts = []
    for r in range(world):
        with np.load(tmp_path / f"r_{r}.npz") as d:
            got = {k: d[k] for k in d.files}
        parts.append(tuple(got["part"]))
        np.testing.assert_array_equal(got["sweep_x"], ref["sweep_x"])
        np.testing.assert_array_equal(got["sweep_info"], np.array(ref["sweep_info"]))
        np.testing.assert_array_equal(got["rot"], ref["rot"])
        np.testing.assert_array_equal(got["frames"], np.array(ref["frames"]))
        np.testing.assert_array_equal(got["frame_x"], ref["frame_x"])
    assert parts[0][0] == 0 and parts[0][1] == parts[1][0] and parts[0][1] < parts[1][1]


def test_nccl_communicator_single_rank():
    """The NCCL back-end end to end on one rank (world 1: the collectives
    are NCCL calls on the context stream); matches the plain solver."""
    import ctypes as C
    from paper_2506_06494_b200 import _lib as L
    lib = L.lib()
    uid = (C.c_uint8 * 128)()
    assert lib.jgs2_nccl_unique_id(uid) == 0
    ctx = lib.jgs2_create(0)
    try:
        assert lib.jgs2_set_comm_nccl(ctx, 1, 0, uid) == 0, lib.jgs2_last_error(ctx)
    finally:
        lib.jgs2_destroy(ctx)
