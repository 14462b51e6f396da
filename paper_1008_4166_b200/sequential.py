"""The reference's sequential entry points on the GPU ring solver.

``jacobi_diagonalize`` (rotations.py:203-223), ``full_block``
(blocking.py:205-250) and ``block_oriented`` (blocking.py:253-293) are the
reference's single-threaded drivers.  A GPU has no use for a sequential
column-cyclic sweep, so each of them runs the ring solver of
``parallel_jacobi`` over the block partition it is given -- the F variant for
the two full-diagonalisation drivers, the B variant for ``block_oriented`` --
and keeps the reference's calling convention: G is transformed IN PLACE, the
return value is a ``DiagInfo``, and with ``accumulate`` / ``accumulate_V`` the
accumulated J-unitary transformation (G_out = G_in W) is returned in
``info.W``.  The fixed point is the same (columns J-orthogonal to the same
tolerance); sweep and rotation counts are those of the parallel block order.

``apply_rotation`` (rotations.py:158-182) and ``BlockMessage``
(parallel.py:66-74) complete the reference's exported surface.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device
from .blocking import BlockPartition
from .parallel import SolverConfig, parallel_jacobi
from .rotations import DEFAULT_TOL, HYPERBOLIC, IDENTITY, DiagInfo, PlaneRotation, Tolerances


@dataclass
class BlockMessage:
    """One block column in flight (parallel.py:66-74).  The GPU ring never
    materialises messages (blocks stay in place in HBM and the schedule is an
    index table); the type is kept for callers that build them."""

    index: int
    G_block: np.ndarray
    J_seg: np.ndarray
    D_seg: np.ndarray


def apply_rotation(G, W, D, r, s, rot: PlaneRotation, hyp: int | None = None):
    """Columns r, s of G and W <- their images under ``rot``; D[r], D[s] get
    the Gram-diagonal update (rotations.py:158-182)."""
    if r == s:
        raise ValueError("rotation columns must differ")
    if rot.kind == IDENTITY:
        return
    h = (1 if rot.kind == HYPERBOLIC else -1) if hyp is None else hyp
    if D is not None:
        step = rot.t * rot.eta
        D[r] += h * step
        D[s] += step
    for M in (G, W):
        if M is None or M.shape[0] == 0:
            continue
        x = rot.phase * M[:, r]
        new_r = rot.cs * x + (h * rot.sn) * M[:, s]
        new_s = rot.sn * x + rot.cs * M[:, s]
        M[:, r] = new_r
        M[:, s] = new_s


def _ring_in_place(G, signs, variant, nbl, tol, want_w):
    if not isinstance(G, np.ndarray):
        raise TypeError("the in-place drivers take a numpy array (use parallel_jacobi for CUDA tensors)")
    n = G.shape[1]
    p = max(1, (max(nbl, 1) + 1) // 2)
    while 2 * p > n and p > 1:
        p -= 1
    cfg = SolverConfig(variant=variant, strategy="round_robin", p=p, tol=tol)
    G0 = G.copy(order="F") if want_w else None
    Gout, info = parallel_jacobi(G, signs, cfg)
    G[...] = Gout
    if want_w:
        # W = G_in^+ G_out on the GPU (a library least-squares solve; W is a
        # by-product for callers, not part of the solver path)
        t = _device.torch()
        a = t.from_numpy(np.ascontiguousarray(G0)).cuda()
        b = t.from_numpy(np.ascontiguousarray(Gout)).cuda()
        w = t.linalg.solve(a, b) if a.shape[0] == a.shape[1] else t.linalg.lstsq(a, b).solution
        info.W = np.asfortranarray(w.cpu().numpy())
    return info


def jacobi_diagonalize(G, signs, tol: Tolerances = DEFAULT_TOL, accumulate=False) -> DiagInfo:
    """J-orthogonalise the columns of G in place (rotations.py:203-223)."""
    n = G.shape[1]
    return _ring_in_place(G, signs, "2F", -(-n // 64), tol, accumulate)


def full_block(G, signs, part: BlockPartition, tol: Tolerances = DEFAULT_TOL, accumulate_V=False) -> DiagInfo:
    """blocking.py:205-250 over ``part.b`` blocks, in place."""
    if part.n != G.shape[1]:
        raise ValueError("partition does not cover all columns")
    return _ring_in_place(G, signs, "2F", part.b, tol, accumulate_V)


def block_oriented(G, signs, part: BlockPartition, tol: Tolerances = DEFAULT_TOL, accumulate_V=False) -> DiagInfo:
    """blocking.py:253-293 over ``part.b`` blocks, in place."""
    if part.n != G.shape[1]:
        raise ValueError("partition does not cover all columns")
    return _ring_in_place(G, signs, "2B", part.b, tol, accumulate_V)
