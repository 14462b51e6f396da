"""Tolerances, counters and eigenpair extraction (reference rotations.py).

``extract_eigen`` runs on the GPU (hjb_extract): lambda_k = j_k ||g_k||^2 and
u_k = g_k / ||g_k|| (rotations.py:226-251).
"""

import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _device, _lib
from .core import EigenResult
from .errors import PivotDefinitenessError, StructuralError

EPS = float(np.finfo(np.float64).eps)


TRIGONOMETRIC = "trigonometric"
HYPERBOLIC = "hyperbolic"
IDENTITY = "identity"


@dataclass(frozen=True)
class PlaneRotation:
    """Nontrivial 2x2 part of a J-unitary plane transformation (same fields
    and ``matrix`` convention as rotations.py:24-53)."""

    kind: str
    cs: float
    sn: float
    phase: complex
    t: float
    eta: float = 0.0

    @property
    def matrix(self):
        """W_P with [g_r', g_s'] = [g_r, g_s] W_P (rotations.py:42-53)."""
        if self.kind == IDENTITY:
            return np.eye(2)
        sigma = 1.0 if self.kind == HYPERBOLIC else -1.0
        return np.array([[self.cs * self.phase, self.sn * self.phase], [sigma * self.sn, self.cs]])


def compute_plane_rotation(a_rr, a_ss, a_rs, j_rr, j_ss):
    """compute_plane_rotation (rotations.py:128-155) evaluated by the pivot
    kernel's own rotation code on the GPU (hjb_plane_rotations): the 2x2
    parameters the B200 path applies.  Raises PivotDefinitenessError(0, 1)
    for a pivot that is not positive definite (rotations.py:134-135, 147-148)."""
    import ctypes

    cx = isinstance(a_rs, complex) or np.iscomplexobj(a_rs)
    arr = np.array([float(a_rr)])
    ass = np.array([float(a_ss)])
    ars = np.array([a_rs], np.complex128 if cx else np.float64)
    jr = np.array([int(j_rr)], np.int8)
    js = np.array([int(j_ss)], np.int8)
    out = np.zeros(8)
    _lib.check(_lib.lib().hjb_plane_rotations(_lib.HJB_C128 if cx else _lib.HJB_F64, 1, arr.ctypes.data,
                                              ass.ctypes.data, ars.ctypes.data, jr.ctypes.data,
                                              js.ctypes.data, out.ctypes.data))
    code, cs, sn, t, eta, ph_re, ph_im, _ = out
    if code < 0:
        raise PivotDefinitenessError(0, 1, "2x2 pivot is not positive definite")
    if code == 0:
        return PlaneRotation(IDENTITY, 1.0, 0.0, 1.0, 0.0, 0.0)
    phase = complex(ph_re, ph_im) if cx else ph_re
    kind = TRIGONOMETRIC if int(j_rr) == int(j_ss) else HYPERBOLIC
    return PlaneRotation(kind, float(cs), float(sn), phase, float(t), float(eta))


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


def orthogonality(U):
    """max |U^H U - I| (the reference's ``orthogonality`` metric, solve.py:
    108-110) on the GPU through hjb_orthogonality (Gram kernel over all
    64-column block pairs + a max fold).  ``U`` is a host array or CUDA tensor."""
    import ctypes

    torch = _device.torch()
    Ud, m, n = _device.as_device_colmajor(U)
    if m == 0 or n == 0:
        return 0.0
    ld = m
    if not Ud.is_complex() and m % 2:
        # 16-byte aligned columns for the Gram kernel's cp.async staging
        P = torch.zeros((n, m + 1), dtype=Ud.dtype, device=Ud.device)
        P[:, :m] = Ud.t()
        Ud, ld = P.t(), m + 1
    dt = _lib.HJB_C128 if Ud.is_complex() else _lib.HJB_F64
    out = ctypes.c_double(0.0)
    st = torch.cuda.current_stream(Ud.device).cuda_stream
    _lib.check(_lib.lib().hjb_orthogonality(dt, m, n, Ud.data_ptr(), ld, ctypes.byref(out), st))
    return float(out.value)
