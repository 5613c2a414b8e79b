"""Partitioned multi-GPU solve: host side.

One process per GPU (torchrun). The rest Hessian H-bar is block diagonal
across bodies (no elastic coupling between bodies, assembly.py:194-259), so
each rank owns a contiguous range of whole bodies: it factors and solves its
bodies' blocks (the exact collect, local_solver.py:115-126) and runs the
vertex pass, element Hessians and local systems of its vertices. The data
path exchanges (all in the C ABI, on the context stream) are

* the local search's per-round counters (int sum, max) -- the halving rounds
  are global (local_solver.py:539-553);
* dx (its owner's rows, zeros elsewhere; a sum is exact);
* per-chunk partial sums of the trial energies and of grad_sq, combined in
  a fixed chunk order (partition.cuh) -- bit-identical to one GPU.

Contact detection, the feasibility cap and every backtracking decision run
replicated on identical data. This module plans the body ranges and builds
the collective back-end: NCCL (production) or a host callback over a
torch.distributed gloo group (tests: ranks sharing one GPU).
"""

import ctypes as C

import numpy as np

from . import _lib as L


def body_ranges(model):
    """[(v_begin, v_end)] per body (bodies are consecutive vertex ranges,
    assembly.py:40-116); one range if the model's bodies are not ordered."""
    vb = np.asarray(getattr(model, "vertex_body", np.zeros(model.num_vertices, dtype=np.int64)))
    nv = int(model.num_vertices)
    if nv == 0 or np.any(np.diff(vb) < 0):
        return [(0, nv)]
    cuts = np.flatnonzero(np.diff(vb) != 0) + 1
    edges = np.r_[0, cuts, nv].astype(np.int64)
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]


def body_costs(model, ranges):
    """Per-body work proxy: elements^1.2 (element passes are linear, the
    factor's nnz grows ~ne^1.36 under nested dissection)."""
    tets = np.asarray(model.tets)
    vb0 = np.array([a for a, _ in ranges])
    owner = np.searchsorted(vb0, tets[:, 0], side="right") - 1
    ne = np.bincount(owner, minlength=len(ranges)).astype(np.float64)
    return ne ** 1.2


def plan(model, world):
    """Contiguous split of the bodies over ``world`` ranks minimizing the
    largest per-rank cost (exact DP). Returns [(v_begin, v_end)] per rank."""
    ranges = body_ranges(model)
    nb = len(ranges)
    if world > nb:
        raise ValueError(f"{world} ranks for {nb} bodies: the partition is by whole bodies")
    cost = body_costs(model, ranges)
    pre = np.r_[0.0, np.cumsum(cost)]
    inf = float("inf")
    best = np.full((world + 1, nb + 1), inf)
    cut = np.zeros((world + 1, nb + 1), dtype=np.int64)
    best[0, 0] = 0.0
    for p in range(1, world + 1):
        for j in range(p, nb + 1):
            for i in range(p - 1, j):
                v = max(best[p - 1, i], pre[j] - pre[i])
                if v < best[p, j]:
                    best[p, j], cut[p, j] = v, i
    bounds, j = [nb], nb
    for p in range(world, 0, -1):
        j = int(cut[p, j])
        bounds.append(j)
    bounds = bounds[::-1]
    return [(ranges[a][0], ranges[b - 1][1]) for a, b in zip(bounds[:-1], bounds[1:])]


# ------------------------------------------------------------ collectives
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p)
_DTYPES = {0: np.float64, 1: np.int32, 2: np.int64}  # u64 maxima are bit patterns of
# non-negative doubles: their order is the int64 order


class HostAllReduce:
    """jgs2_allreduce_fn over a torch.distributed (gloo) group: the C side
    stages the device buffer in pinned memory and calls back here."""

    def __init__(self, dist, group=None):
        self.dist, self.group = dist, group
        self.fn = ALLREDUCE_FN(self._call)  # keep the trampoline alive
        self.calls = 0

    def reduce(self, arr, op):
        import torch
        t = torch.from_numpy(arr)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM if op == 0 else self.dist.ReduceOp.MAX,
                             group=self.group)
        self.calls += 1

    def _call(self, buf, count, dtype, op, user):
        try:
            dt = np.dtype(_DTYPES[int(dtype)])
            raw = (C.c_char * (int(count) * dt.itemsize)).from_address(buf)
            self.reduce(np.frombuffer(raw, dtype=dt), int(op))
            return 0
        except Exception:
            return -1


def attach(lib, ctx, dist, kind="nccl"):
    """Give a context its communicator: ``"nccl"`` (rank 0's unique id
    broadcast over ``dist``) or ``"host"`` (HostAllReduce over ``dist``).
    Returns an object the caller must keep alive (the host callback)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    if kind == "host":
        h = HostAllReduce(dist)
        L.check(lib.jgs2_set_comm_host(ctx, world, rank, C.cast(h.fn, C.c_void_p), None), ctx)
        return h
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        L.check(lib.jgs2_nccl_unique_id(uid))
    box = [bytes(uid) if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
    L.check(lib.jgs2_set_comm_nccl(ctx, world, rank, uid), ctx)
    return None
