"""Multi-GPU driver plumbing for ``bench.py --gpus N``.

The path runs as independent replicas: one process per GPU (torchrun), each
with its own context and scene, no data-path collective. Only the timing
crosses ranks: the device time of the timed window is the max over ranks,
and the whole-job throughput is the sum of the ranks' work over that time.
``torch.distributed`` is plumbing here (NCCL on GPUs, gloo in the CPU tests).
"""

import os


def setup():
    """(world, rank, local_rank, dist or None) from the torchrun environment."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world <= 1:
        return world, rank, local, None
    import torch
    import torch.distributed as dist
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        dist.init_process_group("gloo")
    return world, rank, local, dist


def _device(dist):
    import torch
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def barrier(dist):
    if dist is None:
        return
    import torch
    dist.barrier()
    if torch.cuda.is_available():
        torch.cuda.synchronize()


def max_over_ranks(dist, value):
    """max of a float over all ranks (every rank gets it)."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, value):
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device(dist))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def job_throughput(dist, units, seconds):
    """Whole-job rate: all ranks' units over the slowest rank's time."""
    total = sum_over_ranks(dist, units)
    slowest = max_over_ranks(dist, seconds)
    return total / slowest if slowest > 0 else 0.0
