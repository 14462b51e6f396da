import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

# the oracle's numba cache must live somewhere writable
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(ROOT, ".numba_cache"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def pytest_sessionstart(session):
    """A fresh checkout has no libhjb200.so (built artefacts stay out of
    history): build it once (nvcc cross-compiles sm_100a without a GPU, about
    two minutes) so the library tests do not fail on "not built".  An existing
    library is left alone (a copied tree has unreliable mtimes; rebuild with
    ``python -m paper_1008_4166_b200.build`` or ``__graft_entry__.build()``)."""
    try:
        from paper_1008_4166_b200 import build as b
        if not os.environ.get("HJB_LIB") and not os.path.exists(b.OUT):
            b.build(force=True)
    except Exception as exc:  # the tests that need the library will say so loudly
        sys.stderr.write(f"conftest: library build skipped/failed: {exc}\n")


@pytest.fixture
def rng():
    # the reference suite's seed (pkg/tests/conftest.py:5-7)
    return np.random.default_rng(20240817)


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def random_full_rank(rng, m, n, complex_scalars=False):
    while True:
        G = rng.standard_normal((m, n))
        if complex_scalars:
            G = G + 1j * rng.standard_normal((m, n))
        if np.linalg.matrix_rank(G) == n:
            return np.asfortranarray(G)


def small_solve_cases():
    z = golden("small_solves.npz")
    ms = z["max_sweeps"]
    out = []
    k = 0
    while f"c{k}_G" in z:
        meta = z[f"c{k}_meta"]
        out.append(dict(
            k=k, G=z[f"c{k}_G"], J=z[f"c{k}_J"], Gout=z[f"c{k}_Gout"],
            p=int(meta[0]), strategy="modulus" if meta[1] else "round_robin",
            orth_tol=None if meta[2] < 0 else float(meta[2]),
            sweeps=int(meta[3]), rotations=int(meta[4]), big=int(meta[5]),
            max_t=float(meta[6]), converged=bool(meta[7]), max_sweeps=int(ms[k])))
        k += 1
    return out
