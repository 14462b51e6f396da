"""The ring solver on B200: drop-in for the reference's
``parallel_jacobi(G, signs, SolverConfig)`` (pkg/src/hjacobi/parallel.py:255-309).

Variants (parallel.py:43, 150-174).  ``2F`` / ``3F``: F pre-pass, structured
pair factor, every pivot diagonalised until a sweep applies no rotation.
``2B`` / ``3B``: no pre-pass, dense pair factor, one annihilation cycle per
step (all pairs of the pivot at the first step of a sweep, the cross pairs of
the two blocks afterwards).  The reference's three-level variants (3F / 3B)
block the pivot's inner level into ``inner_n_t``-column sub-blocks; on the
GPU the inner level is ALWAYS blocked -- the Jacobi kernel runs the
reference's ring ordering over register-resident column sub-blocks, one warp
per sub-block pair (csrc/jacobi.cu) -- so 3F runs the same kernels as 2F and
3B the same as 2B; ``inner_n_t`` is validated but the sub-block width is the
kernel's.

The ring of p workers is not a set of threads here: every worker's block pair
of a step is one item of a batched GPU launch (Gram -> pivot -> update), and
the ring exchange is a column-index remap on one GPU and an NCCL send/recv of
the blocks crossing a GPU boundary on several.  The whole
sweep loop runs in native code (libhjb200.so, hjb_solve).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .core import as_matrix, as_signs
from .rotations import DEFAULT_TOL, DiagInfo, Tolerances
from .strategies import MODULUS, normalize_strategy, strategy_code

VARIANTS = ("2F", "2B", "3F", "3B")
SUPPORTED_VARIANTS = VARIANTS
MAX_BLOCK_WIDTH = 128  # widest block column of the GPU kernels (pivot order 256)


def effective_p(n: int, p: int) -> int:
    """Ring workers actually used: ``p`` unless its blocks (n / 2p columns,
    parallel.py:266) would be wider than the kernels' 128 columns; then the
    smallest p whose blocks fit.  The reference has no such limit; a finer
    partition is the same algorithm with more, narrower blocks."""
    need = -(-n // (2 * MAX_BLOCK_WIDTH))
    return max(p, need)


@dataclass(frozen=True)
class SolverConfig:
    """Same fields and validation as parallel.py:46-62, plus the B200 knobs
    ``device`` (CUDA ordinal, default current), ``comm`` (multi-GPU handle
    from ``paper_1008_4166_b200.distributed``), ``phase_times``,
    ``gather_root`` (multi-GPU: only rank 0 receives G_out) and the
    checkpoint/resume pair ``first_sweep`` / ``sweep_count`` (G is the state
    after sweep first_sweep-1; run sweep_count sweeps, 0 = to convergence).
    The state at a sweep boundary is (G, sweep index): the ring layout is
    data-independent (strategies.py:58-136) and D is recomputed."""

    variant: str
    strategy: str = MODULUS
    p: int = 1
    inner_n_t: int = 32
    tol: Tolerances = DEFAULT_TOL
    channel_timeout: float = 120.0
    device: int | None = None
    comm: object = None
    phase_times: bool = False
    gather_root: bool = False
    first_sweep: int = 1
    sweep_count: int = 0
    tail_split: bool = True   # False: HJB_FLAG_NO_TAIL_SPLIT (one Jacobi launch per step)

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")
        object.__setattr__(self, "strategy", normalize_strategy(self.strategy))
        if self.p < 1:
            raise ValueError("p must be >= 1")
        if self.inner_n_t < 1:
            raise ValueError("inner_n_t must be >= 1")
        if self.first_sweep < 1 or self.sweep_count < 0:
            raise ValueError("first_sweep must be >= 1 and sweep_count >= 0")


def _info_from(res: _lib.Result, p_eff=None) -> DiagInfo:
    stats = {k: getattr(res, k) for k, _ in _lib.Result._fields_}
    if p_eff is not None:
        stats["p_effective"] = p_eff
    return DiagInfo(sweeps=res.sweeps, rotations=res.rotations, big_rotations=res.big_rotations,
                    max_abs_t=res.max_abs_t, converged=bool(res.converged), stats=stats)


def _problem(cfg: SolverConfig, m, n, ld, cx, mem, gin, gout, signs, device, stream):
    pr = _lib.Problem()
    pr.dtype = _lib.HJB_C128 if cx else _lib.HJB_F64
    pr.memspace = mem
    pr.m, pr.n, pr.ldg = m, n, ld
    pr.G_in, pr.G_out = gin, gout
    pr.signs = signs.ctypes.data
    pr.p = effective_p(n, cfg.p)
    pr.strategy = strategy_code(cfg.strategy)
    pr.orth_tol = cfg.tol.orth_tol if cfg.tol.orth_tol is not None else -1.0
    pr.quad_tol = cfg.tol.quad_tol if cfg.tol.quad_tol is not None else -1.0
    pr.max_sweeps = cfg.tol.max_sweeps
    pr.device = device
    pr.stream = stream
    pr.comm = cfg.comm.handle if cfg.comm is not None else None
    pr.flags = (_lib.HJB_FLAG_PHASE_TIMES if cfg.phase_times else 0) | \
        (_lib.HJB_FLAG_GATHER_ROOT if cfg.gather_root else 0) | \
        (_lib.HJB_FLAG_VARIANT_B if cfg.variant in ("2B", "3B") else 0) | \
        (0 if cfg.tail_split else _lib.HJB_FLAG_NO_TAIL_SPLIT)
    pr.first_sweep = cfg.first_sweep
    pr.sweep_count = cfg.sweep_count
    return pr


def parallel_jacobi(G, signs, config: SolverConfig):
    """Diagonalize (A = G^* G, J) with p ring workers; returns (G_out, info).

    ``G`` may be a host array (returned G_out is a new Fortran-ordered numpy
    array; the input is left untouched, parallel.py:271/299) or a CUDA tensor
    (G_out is a new column-major CUDA tensor).  Same column order as G
    (parallel.py:299-301).  Non-convergence sets ``info.converged = False``.
    Raises ValueError, PivotDefinitenessError, DefinitenessError like the
    reference.
    """
    L = _lib.lib()
    res = _lib.Result()
    if _device.is_cuda_tensor(G):
        t = _device.torch()
        Gd, m, n = _device.as_device_colmajor(G)
        s = as_signs(signs.cpu().numpy() if hasattr(signs, "cpu") else signs, n)
        out = _device.empty_colmajor(m, n, Gd.dtype, Gd.device)
        dev = Gd.device.index
        st = t.cuda.current_stream(Gd.device).cuda_stream
        pr = _problem(config, m, n, m, Gd.is_complex(), _lib.HJB_DEVICE, Gd.data_ptr(), out.data_ptr(),
                      s, dev, st)
        rc = L.hjb_solve(C.byref(pr), C.byref(res))
        _lib.check(rc, res)
        return out, _info_from(res, pr.p)
    A = as_matrix(G)
    m, n = A.shape
    s = as_signs(signs, n)
    dev = config.device
    if dev is None:
        dev = _device.torch().cuda.current_device() if L.hjb_device_count() > 0 else 0
    try:  # page-locked result: full-speed D2H (falls back to pageable memory)
        out = _device.pinned_host_colmajor(m, n, A.dtype)
    except Exception:
        out = np.empty((m, n), dtype=A.dtype, order="F")
    pr = _problem(config, m, n, m, np.iscomplexobj(A), _lib.HJB_HOST, A.ctypes.data, out.ctypes.data, s,
                  dev, None)
    rc = L.hjb_solve(C.byref(pr), C.byref(res))
    _lib.check(rc, res)
    return out, _info_from(res, pr.p)


def solve_device(Gd, signs_np, config: SolverConfig, out=None, stream=None):
    """Low-overhead entry for resident device data (bench / distributed):
    Gd column-major CUDA tensor (ld = m); writes the result into ``out``
    (may be ``Gd`` itself for an in-place solve).  Returns the raw
    ``_lib.Result``."""
    t = _device.torch()
    m, n = Gd.shape
    out = Gd if out is None else out
    st = stream if stream is not None else t.cuda.current_stream(Gd.device).cuda_stream
    pr = _problem(config, m, n, Gd.stride(1), Gd.is_complex(), _lib.HJB_DEVICE, Gd.data_ptr(),
                  out.data_ptr(), signs_np, Gd.device.index, st)
    res = _lib.Result()
    _lib.check(_lib.lib().hjb_solve(C.byref(pr), C.byref(res)), res)
    return res
