"""Host front end: Hermitian indefinite factorisation H = G J G^* and helpers.

This is the pre-processing step before the hot path,
kept on the host like the reference's (pkg/src/hjacobi/factorization.py).
The reference factorises with Bunch-Parlett complete pivoting
(factorization.py:62-144); BASELINE.json's cfg4 asks for Bunch-Kaufman, which
is what LAPACK's ?hetrf/?sytrf implement (via scipy.linalg.ldl).  Each 2x2
pivot block is diagonalised in closed form and the columns scaled by
sqrt(|eigenvalue|) exactly as factorization.py:131-143, so the signature ends
up in J.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from .core import as_matrix, as_signs
from .errors import RankDeficiencyError, SingularMatrixError


@dataclass
class FactoredForm:
    """Factor pair (G, J) with row permutation P and inertia ordering P1
    (factorization.py:20-29): (P H P^T)[i, j] == H[P[i], P[j]]."""

    G: np.ndarray
    J: np.ndarray
    P: np.ndarray
    P1: np.ndarray


def _eigh2(a, b, c):
    """Eigenvalues and an orthonormal eigenvector matrix of the 2x2 Hermitian
    pivot block [[a, b], [conj(b), c]] of the LDL^* factor (LAPACK's
    symmetric eigensolver on the tiny block; any orthonormal basis serves the
    column scaling below)."""
    blk = np.array([[a, b], [np.conj(b), c]])
    w, Q = np.linalg.eigh(blk)
    return float(w[0]), float(w[1]), Q


def factorize_hermitian_indefinite(H, herm_rtol=1e-10):
    """H = G J G^* by Bunch-Kaufman (LAPACK ?hetrf via scipy.linalg.ldl)
    followed by the 2x2 spectral scaling of factorization.py:131-143.

    The L factor of scipy's ldl already absorbs the pivoting, so G satisfies
    H = G J G^* with P = identity.  Raises SingularMatrixError on a zero
    pivot, ValueError if H is not Hermitian.
    """
    from scipy.linalg import ldl

    H = as_matrix(H)
    n = H.shape[0]
    if H.shape[1] != n:
        raise ValueError("H must be square")
    if n and not np.allclose(H, H.conj().T, rtol=herm_rtol, atol=herm_rtol * np.abs(H).max()):
        raise ValueError("H is not Hermitian")
    A = (H + H.conj().T) / 2
    lu, d, _perm = ldl(A, lower=True, hermitian=True)
    scale = np.abs(A).max() if n else 0.0
    tiny = 64.0 * n * np.finfo(np.float64).eps * scale
    G = np.array(lu, dtype=A.dtype, order="F")
    J = np.empty(n, np.int8)
    k = 0
    while k < n:
        if k + 1 < n and d[k + 1, k] != 0:
            lam1, lam2, Q = _eigh2(d[k, k].real, d[k, k + 1], d[k + 1, k + 1].real)
            if min(abs(lam1), abs(lam2)) <= tiny:
                raise SingularMatrixError("zero pivot: H is numerically singular; supply a factor directly")
            S = Q @ np.diag([math.sqrt(abs(lam1)), math.sqrt(abs(lam2))])
            G[:, k:k + 2] = G[:, k:k + 2] @ S.astype(G.dtype)
            J[k], J[k + 1] = (1 if lam1 >= 0 else -1), (1 if lam2 >= 0 else -1)
            k += 2
        else:
            dk = d[k, k].real
            if abs(dk) <= tiny:
                raise SingularMatrixError("zero pivot: H is numerically singular; supply a factor directly")
            G[:, k] *= math.sqrt(abs(dk))
            J[k] = 1 if dk >= 0 else -1
            k += 1
    return FactoredForm(G=np.asfortranarray(G), J=J, P=np.arange(n), P1=np.arange(n))


def order_by_inertia(f: FactoredForm) -> FactoredForm:
    """Columns with sign +1 first, then the -1 columns, each group in its
    original order; P1 records where every column came from
    (factorization.py:147-153)."""
    pos, neg = np.flatnonzero(f.J != -1), np.flatnonzero(f.J == -1)
    take = np.concatenate([pos, neg])
    return replace(f, G=np.asfortranarray(f.G[:, take]), J=f.J[take], P1=f.P1[take])


def scaled_condition(A):
    """kappa_2 of D^-1/2 A D^-1/2 with D = diag(A), from a symmetric
    eigensolver on the host (factorization.py:156-168; a diagnostic for a
    Gram matrix that is already on the host -- ``scaled_condition_factor``
    is the GPU form used by ``solve_hermitian``)."""
    A = as_matrix(A)
    diag = np.real(np.diagonal(A))
    if diag.size and diag.min() <= 0:
        raise ValueError("scaled_condition requires a strictly positive diagonal")
    r = np.reciprocal(np.sqrt(diag))
    As = (A * r[:, None]) * r[None, :]
    ev = np.abs(np.linalg.eigvalsh(0.5 * (As + As.conj().T)))
    return math.inf if ev.size and ev.min() == 0.0 else float(ev.max() / ev.min()) if ev.size else 1.0


def scaled_condition_factor(G) -> float:
    """kappa(A_s) of A = G^H G scaled to unit diagonal (factorization.py:156-168,
    the metric of solve.py:85) WITHOUT the host n x n eigvalsh: the scaled Gram
    is G_s^H G_s with G_s = G diag(||g_k||)^-1, so its eigenvalues are the
    squared singular values of G_s -- the squared column norms the one-sided
    Jacobi solver itself leaves for J = +I (all rotations trigonometric).  The
    ring solver runs on the GPU over 64-column blocks; G may be a host array
    or a CUDA tensor."""
    from . import _device
    from .parallel import SolverConfig, parallel_jacobi
    from .rotations import Tolerances

    torch = _device.torch()
    if _device.is_cuda_tensor(G):
        Gd = G
    else:
        A = as_matrix(G)
        Gd = torch.from_numpy(np.ascontiguousarray(A.T)).to("cuda").t()
    n = Gd.shape[1]
    if n == 0:
        return 1.0
    d = (Gd.real ** 2 + Gd.imag ** 2).sum(dim=0) if Gd.is_complex() else (Gd * Gd).sum(dim=0)
    if bool((d <= 0).any()):
        raise ValueError("scaled_condition requires a strictly positive diagonal")
    Gs = (Gd / torch.sqrt(d).to(Gd.dtype)[None, :]).t().contiguous().t()  # column-major
    p = max(1, n // 128)
    while 2 * p > n and p > 1:
        p -= 1
    eps = float(np.finfo(np.float64).eps)
    cfg = SolverConfig(variant="2F", strategy="round_robin", p=p, tol=Tolerances(orth_tol=n * eps))
    Gout, _ = parallel_jacobi(Gs, np.ones(n, np.int8), cfg)
    w = (Gout.real ** 2 + Gout.imag ** 2).sum(dim=0) if Gout.is_complex() else (Gout * Gout).sum(dim=0)
    lo, hi = float(w.min()), float(w.max())
    return math.inf if lo == 0.0 else hi / lo


def accept_external_factor(G, J) -> FactoredForm:
    """A caller-supplied factor pair taken as is, after the reference's checks
    (factorization.py:171-189): at least as many rows as columns, a valid sign
    vector, no zero column, full column rank (Cholesky of the Gram)."""
    G = as_matrix(G)
    rows, cols = G.shape
    if cols > rows:
        raise ValueError("factor must have at least as many rows as columns")
    signs = as_signs(J, cols)
    gram = G.conj().T @ G
    try:
        np.linalg.cholesky(gram)
    except np.linalg.LinAlgError as exc:
        raise RankDeficiencyError("supplied factor is rank deficient") from exc
    if cols and np.real(np.diagonal(gram)).min() == 0.0:
        raise RankDeficiencyError("supplied factor has a zero column")
    ident_r, ident_c = np.arange(rows), np.arange(cols)
    return FactoredForm(G=G, J=signs, P=ident_r, P1=ident_c)
