"""Host front end (CPU): Bunch-Kaufman + 2x2 spectral scaling reproduces
H = G J G^* with the right inertia (the reference's criterion 2,
test_acceptance.py:80-104, restated on our own generator)."""

import numpy as np
import pytest

import paper_1008_4166_b200 as P
from paper_1008_4166_b200 import workloads

EPS = np.finfo(np.float64).eps


@pytest.mark.parametrize("n,cplx", [(5, False), (20, True), (100, False), (100, True)])
def test_factorization_reconstructs_and_keeps_inertia(rng, n, cplx):
    for _ in range(5):
        A = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
        H = (A + A.conj().T) / 2
        f = P.factorize_hermitian_indefinite(H)
        R = f.G @ np.diag(f.J.astype(float)) @ f.G.conj().T
        assert np.abs(H[np.ix_(f.P, f.P)] - R).max() <= 50 * n * EPS * np.abs(H).max()
        assert int(np.sum(f.J > 0)) == int(np.sum(np.linalg.eigvalsh(H) > 0))
        g = P.order_by_inertia(f)
        assert np.all(np.diff((g.J == -1).astype(int)) >= 0)


def test_factorization_rejects_non_hermitian_and_singular(rng):
    with pytest.raises(ValueError):
        P.factorize_hermitian_indefinite(rng.standard_normal((4, 4)))
    with pytest.raises(P.SingularMatrixError):
        P.factorize_hermitian_indefinite(np.zeros((3, 3)))


def test_cfg4_generator_small():
    w = workloads.cfg4(n=128, b=16)
    R = w.G @ np.diag(w.J.astype(float)) @ w.G.conj().T
    assert np.abs(R - w.H).max() <= 1e-12 * np.abs(w.H).max() * 128
    assert w.G.dtype == np.complex128 and w.p == 4
    assert int(np.sum(w.J < 0)) == 64
