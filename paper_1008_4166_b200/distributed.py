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


def exchange_plan(strategy: str, p: int, world: int, rank: int, sweeps: int = 1):
    """The native multi-GPU transfer plan of GPU ``rank`` (hjb_exchange_plan,
    the same code hjb_solve runs): per step a list of (0-based block, peer,
    send?) for the block columns that cross a GPU boundary."""
    from .strategies import steps_per_sweep, strategy_code
    steps = steps_per_sweep(strategy, p) * sweeps
    mx = 2 * p
    out = np.zeros((max(steps, 1), mx, 3), np.int32)
    cnt = np.zeros(max(steps, 1), np.int32)
    _lib.check(_lib.lib().hjb_exchange_plan(strategy_code(strategy), p, world, rank, sweeps, mx,
                                            out.ctypes.data, cnt.ctypes.data))
    return [[(int(b), int(pe), bool(sd)) for b, pe, sd in out[s, :cnt[s]]] for s in range(steps)]


def block_owners(strategy: str, p: int, world: int, sweeps: int):
    """GPU holding each 0-based block after ``sweeps`` sweeps (hjb_block_owners,
    the map hjb_solve gathers G_out from; parallel.py:299-301)."""
    from .strategies import strategy_code
    out = np.zeros(2 * p, np.int32)
    _lib.check(_lib.lib().hjb_block_owners(strategy_code(strategy), p, world, sweeps, out.ctypes.data))
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
