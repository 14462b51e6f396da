"""Seeded synthetic inputs for the BASELINE.json configurations.

No public benchmark suite is involved: BASELINE.json defines the inputs, and
SURVEY.md section 8(d) fixes the generator conventions (numpy
``default_rng``, C-order draw, then column-major).  The same generator feeds
the oracle, the parity tests and ``bench.py``.

``n`` may be overridden to get a smaller instance drawn the same way (used
for parity proxies that the CPU oracle finishes in seconds).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Workload:
    name: str
    G: np.ndarray          # m x n, float64 or complex128, column-major
    J: np.ndarray          # int8 +-1, length n
    b: int                 # block width
    p: int                 # ring workers = n / (2b)
    description: str

    @property
    def n(self):
        return self.G.shape[1]

    @property
    def m(self):
        return self.G.shape[0]

    @property
    def orth_tol(self):
        # BASELINE: tol = n * eps, mapped to Tolerances(orth_tol=n*eps)
        #
        return self.n * float(np.finfo(np.float64).eps)


def _inertia(G, J):
    # factorization.py:147-153 applied to both sides
    idx = np.argsort(J == -1, kind="stable")
    return np.asfortranarray(G[:, idx]), np.ascontiguousarray(J[idx])


def cfg1(n=512, b=32):
    """Real N(0,1) from seed 0; J = +1 x 3n/4, -1 x n/4; block width 32."""
    G = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
    npos = (3 * n) // 4
    J = np.array([1] * npos + [-1] * (n - npos), np.int8)
    return Workload("cfg1", G, J, b, n // (2 * b),
                    f"real f64 {n}x{n} N(0,1) seed 0, J +{npos}/-{n - npos}, b={b}")


def cfg2(n=2048, b=64):
    """Complex, re/im iid N(0,1/2) from seed 1; J half/half; b = 64."""
    r = np.random.default_rng(1)
    re = r.standard_normal((n, n))
    im = r.standard_normal((n, n))
    G = np.asfortranarray((re + 1j * im) * math.sqrt(0.5))
    J = np.array([1] * (n // 2) + [-1] * (n - n // 2), np.int8)
    return Workload("cfg2", G, J, b, n // (2 * b),
                    f"complex128 {n}x{n} N(0,1/2) seed 1, J half/half, b={b}")


def cfg3(n=4096, b=64):
    """Graded real G = B diag(10^-u), u ~ U[0,8] (seed 2); J = -1 w.p. 0.3
    (seed 3), inertia-ordered; b = 64 (BASELINE leaves b open; reference
    nt_outer default, solve.py:34)."""
    r = np.random.default_rng(2)
    B = r.standard_normal((n, n))
    u = r.uniform(0.0, 8.0, n)
    G = B * (10.0 ** (-u))[None, :]
    J = np.where(np.random.default_rng(3).random(n) < 0.3, -1, 1).astype(np.int8)
    G, J = _inertia(G, J)
    return Workload("cfg3", G, J, b, n // (2 * b),
                    f"graded real {n}x{n}, seed 2/3, P(-1)=0.3, b={b}")


def cfg4_hermitian(n=8192):
    """H = Q diag(lam) Q^*: Q from QR of a complex Gaussian (seed 4),
    lam_k = s_k 10^-v_k, v ~ U[0,6], s_k = -1 on half the indices."""
    r = np.random.default_rng(4)
    X = (r.standard_normal((n, n)) + 1j * r.standard_normal((n, n))) * math.sqrt(0.5)
    Q, _ = np.linalg.qr(X)
    v = r.uniform(0.0, 6.0, n)
    s = np.ones(n)
    s[r.permutation(n)[: n // 2]] = -1.0
    lam = s * 10.0 ** (-v)
    H = (Q * lam[None, :]) @ Q.conj().T
    return (H + H.conj().T) / 2, lam


def cfg4(n=8192, b=64):
    """Prescribed spectrum, factorised on the host by Bunch-Kaufman + 2x2
    spectral scaling (factorization.py), inertia ordered; b = 64."""
    from .factorization import factorize_hermitian_indefinite, order_by_inertia
    H, lam = cfg4_hermitian(n)
    f = order_by_inertia(factorize_hermitian_indefinite(H))
    w = Workload("cfg4", np.asfortranarray(f.G), np.ascontiguousarray(f.J), b, n // (2 * b),
                 f"complex128 prescribed spectrum n={n}, Bunch-Kaufman factor, b={b}")
    w.H, w.lam = H, np.sort(lam)
    return w


def cfg5r(n=32768, b=128):
    G = np.asfortranarray(np.random.default_rng(5).standard_normal((n, n)))
    J = np.array([1] * (n // 2) + [-1] * (n - n // 2), np.int8)
    return Workload("cfg5r", G, J, b, n // (2 * b),
                    f"real f64 {n}x{n} seed 5, J half/half, b={b}")


def cfg5c(n=16384, b=128):
    r = np.random.default_rng(6)
    re = r.standard_normal((n, n))
    im = r.standard_normal((n, n))
    G = np.asfortranarray((re + 1j * im) * math.sqrt(0.5))
    J = np.array([1] * (n // 2) + [-1] * (n - n // 2), np.int8)
    return Workload("cfg5c", G, J, b, n // (2 * b),
                    f"complex128 {n}x{n} seed 6, J half/half, b={b}")


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5r": cfg5r, "cfg5c": cfg5c}


def make(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)


def algorithmic_flops(m, b, complex_, pairs_updated, pairs_visited,
                      prepass_updated, prepass_visited):
    """c*[2mb^2 (pairs+nbl Grams) + 8mb^2 (updated pairs)
    + 2mb^2 (updated pre-pass blocks)], c = 4 for complex."""
    c = 4.0 if complex_ else 1.0
    mb2 = float(m) * b * b
    return c * (2 * mb2 * (pairs_visited + prepass_visited)
                + 8 * mb2 * pairs_updated + 2 * mb2 * prepass_updated)
