"""N>1 bench plumbing (replicas) on CPU: world_size-2 gloo."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    from paper_2506_06494_b200 import replicas
    w, r, local, dist = replicas.setup()
    assert (w, r, local) == (world, rank, rank) and dist is not None
    replicas.barrier(dist)
    # rank r did 10 * (r + 1) sweeps in (r + 1) seconds
    units, secs = 10.0 * (rank + 1), float(rank + 1)
    out[rank] = (replicas.max_over_ranks(dist, secs), replicas.sum_over_ranks(dist, units),
                 replicas.job_throughput(dist, units, secs))
    dist.destroy_process_group()


def test_two_rank_timing_is_max_and_work_is_summed():
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        mx, tot, thr = res[r]
        assert mx == 2.0            # slowest rank's device time
        assert tot == 30.0          # all ranks' sweeps
        assert thr == pytest.approx(15.0)


def test_single_process_is_identity(monkeypatch):
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    from paper_2506_06494_b200 import replicas
    w, r, local, dist = replicas.setup()
    assert (w, r, local, dist) == (1, 0, 0, None)
    assert replicas.job_throughput(None, 50, 2.0) == 25.0
