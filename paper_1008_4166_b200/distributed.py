"""Multi-GPU plumbing: one process per GPU, an NCCL communicator owned by the
native library (hjb_comm_init), bootstrapped over torch.distributed.

The data path (block exchange per step, rotation all-reduce per sweep,
final gather) runs inside hjb_solve over NCCL; torch.distributed only
broadcasts the 128-byte NCCL unique id (any backend, e.g. gloo).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def ring_ranks_of_gpu(p: int, world: int, g: int):
    """Ring workers hosted by GPU g: contiguous [g*p//world, (g+1)*p//world)
    (csrc/solver.cu, wlo())."""
    return range(g * p // world, (g + 1) * p // world)


def gpu_of_worker(p: int, world: int, q: int) -> int:
    for g in range(world):
        if q in ring_ranks_of_gpu(p, world, g):
            return g
    raise ValueError(q)


def exchange_plan(strategy: str, p: int, world: int, sweeps: int = 1):
    """Per step, the block transfers that cross a GPU boundary: list of
    (src_gpu, dst_gpu, block) derived from the reference's StepPlans
    (strategies.py:75-136).  Everything else is an index remap."""
    from .strategies import schedule_arrays
    _, plans = schedule_arrays(strategy, p, sweeps)
    out = []
    for step in plans:
        xf = []
        for q, (snd_rnk, snd_blk, rcv_rnk, rcv_blk) in enumerate(step):
            src, dst = gpu_of_worker(p, world, q), gpu_of_worker(p, world, int(snd_rnk))
            if src != dst:
                xf.append((src, dst, int(snd_blk)))
        out.append(xf)
    return out


class Comm:
    """Handle passed as SolverConfig.comm."""

    def __init__(self, handle, rank, world):
        self.handle = handle
        self.rank = rank
        self.world = world

    @classmethod
    def create(cls, rank: int, world: int, device: int):
        import torch.distributed as dist
        L = _lib.lib()
        buf = (C.c_char * 128)()
        if rank == 0:
            _lib.check(L.hjb_comm_unique_id(buf))
        obj = [bytes(buf) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = (C.c_char * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _lib.check(L.hjb_comm_init(uid, world, rank, device, C.byref(h)))
        return cls(h.value, rank, world)

    def close(self):
        if self.handle:
            _lib.lib().hjb_comm_destroy(self.handle)
            self.handle = None
