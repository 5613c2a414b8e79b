"""Host side of the partitioned multi-GPU solve (partition.py) on CPU:
the body partition plan and the gloo all-reduce callback, world_size 2."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

from paper_2506_06494_b200 import partition, scenes  # noqa: E402


@pytest.fixture(scope="module")
def tank():
    return scenes.build("c4s6")[0]


def test_body_ranges_cover_the_mesh(tank):
    r = partition.body_ranges(tank)
    assert len(r) == 10 and r[0][0] == 0 and r[-1][1] == tank.num_vertices
    assert all(a < b for a, b in r) and all(r[k][1] == r[k + 1][0] for k in range(9))
    vb = np.asarray(tank.vertex_body)
    assert all(np.all(vb[a:b] == vb[a]) for a, b in r)


@pytest.mark.parametrize("world", (1, 2, 3, 4, 8, 10))
def test_plan_is_contiguous_whole_bodies_and_balanced(tank, world):
    bodies = partition.body_ranges(tank)
    p = partition.plan(tank, world)
    assert len(p) == world and p[0][0] == 0 and p[-1][1] == tank.num_vertices
    starts = {a for a, _ in bodies} | {tank.num_vertices}
    assert all(a in starts and b in starts and a < b for a, b in p)
    assert all(p[k][1] == p[k + 1][0] for k in range(world - 1))
    cost = partition.body_costs(tank, bodies)
    per_rank = [sum(c for (a, _), c in zip(bodies, cost) if lo <= a < hi) for lo, hi in p]
    # optimal contiguous split: no better than the largest single body or the mean
    assert max(per_rank) <= max(cost.max(), cost.sum() / world) * (1 + 1e-12) + cost.max()


def test_plan_rejects_more_ranks_than_bodies(tank):
    with pytest.raises(ValueError):
        partition.plan(tank, 11)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import ctypes as C
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h = partition.HostAllReduce(dist)
    # exactly what the C side passes: a raw buffer, dtype / op codes
    f = np.array([0.0, 1.5, 0.0]) if rank == 0 else np.array([2.25, 0.0, -0.0])
    i = np.array([rank + 1, 10 * rank], dtype=np.int32)
    bits = np.array([0.5, 0.25 * (rank + 1)]).view(np.int64)  # u64 max of non-negative doubles
    rc = [h.fn(a.ctypes.data_as(C.c_void_p), a.size, code, op, None)
          for a, code, op in ((f, 0, 0), (i, 1, 0), (bits, 2, 1))]
    out[rank] = (rc, f.tolist(), i.tolist(), bits.view(np.float64).tolist(), h.calls)
    dist.destroy_process_group()


def test_host_allreduce_callback_two_ranks():
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        rc, f, i, mx, calls = res[r]
        assert rc == [0, 0, 0] and calls == 3
        assert f == [2.25, 1.5, 0.0]       # owner's value + zeros: exact
        assert i == [3, 10]
        assert mx == [0.5, 0.5]
