"""Tolerances, counters and eigenpair extraction (reference rotations.py).

``extract_eigen`` runs on the GPU (hjb_extract): lambda_k = j_k ||g_k||^2 and
u_k = g_k / ||g_k|| (rotations.py:226-251).
"""

import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _device, _lib
from .core import EigenResult
from .errors import StructuralError

EPS = float(np.finfo(np.float64).eps)


@dataclass(frozen=True)
class Tolerances:
    """Thresholds of the sweep loop (rotations.py:56-83)."""

    orth_tol: float | None = None
    quad_tol: float | None = None
    max_sweeps: int = 30

    def __post_init__(self):
        if self.max_sweeps < 1:
            raise ValueError("max_sweeps must be >= 1")
        for v in (self.orth_tol, self.quad_tol):
            if v is not None and v <= 0:
                raise ValueError("tolerances must be positive")

    def orth(self, m):
        return self.orth_tol if self.orth_tol is not None else math.sqrt(m) * EPS

    def quad(self, n):
        return self.quad_tol if self.quad_tol is not None else n * EPS

    def with_max_sweeps(self, max_sweeps):
        return replace(self, max_sweeps=max_sweeps)


DEFAULT_TOL = Tolerances()


@dataclass
class DiagInfo:
    """Aggregate result of a diagonalization driver (rotations.py:107-121),
    plus the device counters of the B200 run in ``stats``."""

    sweeps: int = 0
    rotations: int = 0
    big_rotations: int = 0
    max_abs_t: float = 0.0
    converged: bool = False
    W: object = None
    stats: dict = field(default_factory=dict)


def extract_eigen(G_final, signs, col_perm=None, sort_descending=False):
    """Read eigenpairs off a converged factor on the GPU (rotations.py:226-251).

    ``G_final`` is a host array or a CUDA tensor (column-major); the result
    lives where the input lived.  ``col_perm`` maps current column positions
    to original indices; ``sort_descending`` re-sorts stably by eigenvalue.
    Raises StructuralError on a zero column.
    """
    torch = _device.torch()
    host = not _device.is_cuda_tensor(G_final)
    Gd, m, n = _device.as_device_colmajor(G_final)
    cx = Gd.is_complex()
    dt = _lib.HJB_C128 if cx else _lib.HJB_F64
    sd = _device.signs_to_device(signs, n, Gd.device)
    st = torch.cuda.current_stream(Gd.device).cuda_stream
    L = _lib.lib()
    lam = torch.empty(n, dtype=torch.float64, device=Gd.device)
    U = _device.empty_colmajor(m, n, Gd.dtype, Gd.device)
    rc = L.hjb_extract(dt, m, n, Gd.data_ptr(), m, sd.data_ptr(), lam.data_ptr(), U.data_ptr(), m, None, st)
    if rc == _lib.HJB_CHOL_FAIL:
        raise StructuralError("zero-norm column: factor is rank deficient")
    _lib.check(rc)
    perm = None
    if col_perm is not None or sort_descending:
        lam_h = lam.cpu().numpy()
        order = np.arange(n)
        if col_perm is not None:
            cp = np.asarray(col_perm)
            order = np.empty(n, np.int64)
            order[cp] = np.arange(n)          # out[col_perm[c]] = in[c]
            lam_h = lam_h[order]
        if sort_descending:
            o2 = np.argsort(-lam_h, kind="stable")
            order = order[o2]
        perm = torch.as_tensor(np.ascontiguousarray(order, np.int64), device=Gd.device)
        rc = L.hjb_extract(dt, m, n, Gd.data_ptr(), m, sd.data_ptr(), lam.data_ptr(), U.data_ptr(), m,
                           perm.data_ptr(), st)
        _lib.check(rc)
    if host:
        return EigenResult(eigenvalues=lam.cpu().numpy(), eigenvectors=_device.to_host(U))
    return EigenResult(eigenvalues=lam, eigenvectors=U)
