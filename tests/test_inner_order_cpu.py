"""The GPU pivot kernel's warp-block inner order (oracle WBlockState,
pivot.cu HJB_WBLOCK): every round is a set of disjoint pairs over all column
positions, every pair of columns meets in every sweep, and the order is a
valid one-sided J-Jacobi order (converges to the same eigenvalues as the
reference's cyclic order, _kernels.py:41-52)."""

import numpy as np
import pytest

import oracle as O
from oracle import jjacobi as OJ


@pytest.mark.parametrize("nmax,nw", [(32, 1), (32, 2), (64, 2), (64, 4), (128, 2), (128, 4), (128, 8),
                                     (256, 4), (256, 8), (256, 16)])
def test_wblock_rounds_cover_all_pairs(nmax, nw):
    st = OJ.WBlockState(nmax, nw)
    for _ in range(3):  # the arrangement persists across sweeps
        tab = st.sweep_table()
        assert tab.shape == (nmax, nmax // 2, 2)
        seen = set()
        for rnd in tab:
            assert sorted(rnd.reshape(-1).tolist()) == list(range(nmax))  # disjoint, all positions
            seen.update((min(r, s), max(r, s)) for r, s in rnd.tolist())
        assert len(seen) == nmax * (nmax - 1) // 2


@pytest.mark.parametrize("cplx", [False, True])
def test_wblock_diagonalize_matches_cyclic(cplx):
    rng = np.random.default_rng(11)
    n = 64
    G = rng.standard_normal((96, n)) + (1j * rng.standard_normal((96, n)) if cplx else 0)
    J = np.array([1] * 40 + [-1] * 24, np.int8)
    R0 = O.chol_upper(O.gram(G))
    out = {}
    for order in ("cyclic", "wblock:64:2", "wblock:128:4"):  # 128: half the positions are padding
        R = R0.copy(order="F")
        W, sw, nrot, *_ , conv = O.diagonalize(R, J, order=order)
        assert conv
        out[order] = (np.sort(J * O.column_norms2(R)), sw)
        Jf = np.diag(J.astype(float))
        assert np.abs(W.conj().T @ Jf @ W - Jf).max() <= 64 * n * O.EPS * np.linalg.norm(W, 2) ** 2
    ref = out["cyclic"][0]
    for order, (lam, sw) in out.items():
        assert np.max(np.abs(lam - ref) / np.abs(ref)) <= 1e-12
        assert abs(sw - out["cyclic"][1]) <= 2


@pytest.mark.parametrize("nmax,c,w,spw", [(32, 1, 4, 4), (32, 2, 4, 2), (64, 2, 4, 4), (64, 4, 4, 2),
                                          (128, 4, 8, 2), (128, 8, 4, 2), (128, 4, 4, 4), (256, 8, 8, 2),
                                          (256, 4, 8, 4), (256, 16, 4, 2)])
def test_ring_of_rings_rounds_cover_all_pairs(nmax, c, w, spw):
    """Jacobi kernel order (jacobi.cu, oracle RingOfRings): N - 1 rounds of
    N/2 disjoint pairs per inner sweep, every pair exactly once, for the
    shapes the library instantiates; the layout persists across sweeps."""
    st = OJ.RingOfRings(nmax, c, w, spw)
    for _ in range(4):  # odd and even sweeps (the stepper's direction alternates)
        tab = st.sweep_table()
        assert tab.shape == (nmax - 1, nmax // 2, 2)
        seen = set()
        for rnd in tab:
            assert sorted(rnd.reshape(-1).tolist()) == list(range(nmax))
            seen.update((min(r, s), max(r, s)) for r, s in rnd.tolist())
        assert len(seen) == nmax * (nmax - 1) // 2


@pytest.mark.parametrize("cplx", [False, True])
def test_ring_of_rings_diagonalize_matches_cyclic(cplx):
    rng = np.random.default_rng(12)
    n = 64
    G = rng.standard_normal((96, n)) + (1j * rng.standard_normal((96, n)) if cplx else 0)
    J = np.array([1] * 40 + [-1] * 24, np.int8)
    R0 = O.chol_upper(O.gram(G))
    out = {}
    for order in ("cyclic", "ror:64:2:4:4", "ror:64:4:4:2", "ror:128:8:4:2"):  # 128: padding columns
        R = R0.copy(order="F")
        W, sw, nrot, *_, conv = O.diagonalize(R, J, order=order)
        assert conv
        out[order] = (np.sort(J * O.column_norms2(R)), sw)
        Jf = np.diag(J.astype(float))
        assert np.abs(W.conj().T @ Jf @ W - Jf).max() <= 64 * n * O.EPS * np.linalg.norm(W, 2) ** 2
    ref = out["cyclic"][0]
    for order, (lam, sw) in out.items():
        assert np.max(np.abs(lam - ref) / np.abs(ref)) <= 1e-12
        assert abs(sw - out["cyclic"][1]) <= 2
