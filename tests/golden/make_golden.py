"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (the reference is only present there):

    OPENBLAS_NUM_THREADS=1 NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden.py

It imports ``hjacobi`` from ``/root/reference/pkg/src`` (read-only) and writes
small ``.npz`` fixtures next to this script.  The fixtures travel with the
repo; nothing at test time reads ``/root/reference``.  BLAS threads are pinned
to 1 because the reference's bits depend on BLAS threading.
"""

import json
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import hjacobi  # noqa: E402
from hjacobi import errors as herr  # noqa: E402
from hjacobi.blocking import chol_upper, structured_cholesky  # noqa: E402
from hjacobi.core import column_norms_squared, gram  # noqa: E402
from hjacobi.parallel import SolverConfig, parallel_jacobi  # noqa: E402
from hjacobi.rotations import Tolerances, jacobi_diagonalize  # noqa: E402
from hjacobi.strategies import (  # noqa: E402
    generate_sweep_schedule, init_strategy, step_fn, steps_per_sweep)

from paper_1008_4166_b200 import workloads  # noqa: E402

EPS = np.finfo(np.float64).eps


def schedules():
    out = {}
    for strategy in ("modulus", "round_robin"):
        for p in list(range(1, 9)) + [16, 32, 64]:
            sweeps = 3 if p <= 32 else 2
            lay = np.array(generate_sweep_schedule(strategy, p, sweeps=sweeps), np.int32)
            # plans from the steppers themselves
            states = [init_strategy(q, 2 * p) for q in range(p)]
            fn = step_fn(strategy)
            plans = []
            for sweep in range(1, sweeps + 1):
                for st in states:
                    st.nsweep = sweep
                for _ in range(steps_per_sweep(strategy, p)):
                    row = []
                    for st in states:
                        pl = fn(st, p)
                        row.append((pl.snd_rnk, pl.snd_blk, pl.rcv_rnk, pl.rcv_blk))
                    plans.append(row)
            out[f"{strategy}_p{p}_layouts"] = lay
            out[f"{strategy}_p{p}_plans"] = np.array(plans, np.int32)
    np.savez_compressed(os.path.join(HERE, "schedules.npz"), **out)


def random_full_rank(rng, m, n, cplx):
    while True:
        G = rng.standard_normal((m, n))
        if cplx:
            G = G + 1j * rng.standard_normal((m, n))
        if np.linalg.matrix_rank(G) == n:
            return np.asfortranarray(G)


def small_solves():
    """Whole-path cases with full G_out stored."""
    cases = []
    rng = np.random.default_rng(20240817)
    specs = [
        # (m, n, n_neg, complex, p, strategy, orth_tol)
        (20, 20, 7, False, 1, "round_robin", None),
        (20, 20, 7, False, 2, "round_robin", None),
        (20, 20, 7, False, 3, "round_robin", None),   # ragged blocks 4,4,3,3,3,3
        (20, 20, 7, False, 3, "modulus", None),
        (48, 48, 19, True, 2, "round_robin", None),
        (48, 48, 19, True, 3, "modulus", None),
        (48, 48, 19, True, 4, "round_robin", 48 * EPS),
        (64, 64, 16, False, 4, "round_robin", 64 * EPS),
        (64, 64, 32, True, 2, "modulus", 64 * EPS),
        (80, 64, 20, False, 4, "round_robin", 64 * EPS),  # rectangular m > n
        (30, 30, 0, False, 3, "round_robin", None),       # definite J (all trig)
        (30, 30, 30, True, 3, "modulus", None),           # all -1
    ]
    out = {}
    for k, (m, n, nneg, cplx, p, strat, otol) in enumerate(specs):
        G = random_full_rank(rng, m, n, cplx)
        J = np.array([1] * (n - nneg) + [-1] * nneg, np.int8)
        tol = Tolerances(orth_tol=otol)
        Gout, info = parallel_jacobi(G.copy(order="F"), J.copy(),
                                     SolverConfig(variant="2F", strategy=strat, p=p, tol=tol))
        out[f"c{k}_G"] = G
        out[f"c{k}_J"] = J
        out[f"c{k}_Gout"] = Gout
        out[f"c{k}_meta"] = np.array([p, 1 if strat == "modulus" else 0,
                                      otol if otol is not None else -1.0,
                                      info.sweeps, info.rotations, info.big_rotations,
                                      info.max_abs_t, int(info.converged)], np.float64)
    # orthogonal input: zero rotations, 1 sweep, exact column order (test_parallel.py:72-89)
    G = np.asfortranarray(np.diag(np.arange(1.0, 13.0)))
    J = np.ones(12, np.int8)
    Gout, info = parallel_jacobi(G.copy(order="F"), J, SolverConfig(variant="2F", p=3))
    k = len(specs)
    out[f"c{k}_G"], out[f"c{k}_J"], out[f"c{k}_Gout"] = G, J, Gout
    # SolverConfig's default strategy is modulus (parallel.py:49)
    out[f"c{k}_meta"] = np.array([3, 1, -1.0, info.sweeps, info.rotations,
                                  info.big_rotations, info.max_abs_t, int(info.converged)])
    # non-convergence flag (test_parallel.py:100-104)
    rng2 = np.random.default_rng(99)
    G = random_full_rank(rng2, 24, 24, False)
    J = np.array([1] * 15 + [-1] * 9, np.int8)
    Gout, info = parallel_jacobi(G.copy(order="F"), J.copy(),
                                 SolverConfig(variant="2F", p=2, tol=Tolerances(max_sweeps=1)))
    k += 1
    out[f"c{k}_G"], out[f"c{k}_J"], out[f"c{k}_Gout"] = G, J, Gout
    out[f"c{k}_meta"] = np.array([2, 1, -1.0, info.sweeps, info.rotations,
                                  info.big_rotations, info.max_abs_t, int(info.converged)])
    out["max_sweeps"] = np.array([30] * (len(specs) + 1) + [1])
    np.savez_compressed(os.path.join(HERE, "small_solves.npz"), **out)


def config_proxies():
    """Eigenvalues + counters of the BASELINE configs at full size (cfg1) and
    at reduced n with the same generators (cfg2/cfg3/cfg5 proxies)."""
    out = {}
    runs = [
        ("cfg1", {}),
        ("cfg2", {"n": 512, "b": 32}),
        ("cfg3", {"n": 512, "b": 32}),
        ("cfg5r", {"n": 512, "b": 64}),
        ("cfg5r", {"n": 1024, "b": 128}),
        ("cfg5c", {"n": 1024, "b": 128}),
    ]
    meta = {}
    for name, kw in runs:
        w = workloads.make(name, **kw)
        tol = Tolerances(orth_tol=w.orth_tol)
        Gout, info = parallel_jacobi(w.G.copy(order="F"), w.J.copy(),
                                     SolverConfig(variant="2F", strategy="round_robin",
                                                  p=w.p, tol=tol))
        lam = w.J * column_norms_squared(Gout)
        key = f"{name}_n{w.n}_b{w.b}"
        out[key + "_lam"] = lam
        out[key + "_colsum"] = Gout.sum(axis=0)
        out[key + "_info"] = np.array([info.sweeps, info.rotations, info.big_rotations,
                                       info.max_abs_t, int(info.converged)], np.float64)
        meta[key] = dict(name=name, **kw)
        print(key, info.sweeps, info.rotations, flush=True)
    np.savez_compressed(os.path.join(HERE, "config_proxies.npz"), **out)
    with open(os.path.join(HERE, "config_proxies.json"), "w") as f:
        json.dump(meta, f, indent=1)


def fullsize():
    """BASELINE cfg2 (n=2048) and cfg3 (n=4096) at FULL size with the
    reference itself (2F, round-robin, p = n/(2b) worker threads, orth_tol =
    n eps), plus the cfg5 sweep-count proxies at n = 4096, b = 128 (SURVEY.md
    8(d) cfg5 oracle item iii).  Stored per column: lambda = J ||g||^2 and
    the column sums of G_out; per run: DiagInfo and the wall time.  G_out
    itself (64-128 MiB) is not stored.  kappa(G_s) (factorization.py:156-168)
    of the input is stored for the per-eigenvalue bound."""
    import time
    from hjacobi.factorization import scaled_condition
    which = os.environ.get("HJB_FULLSIZE", "cfg2,cfg3,cfg5r_p,cfg5c_p").split(",")
    runs = {"cfg2": ("cfg2", {}), "cfg3": ("cfg3", {}),
            "cfg5r_p": ("cfg5r", {"n": 4096, "b": 128}), "cfg5c_p": ("cfg5c", {"n": 4096, "b": 128})}
    for tag in which:
        name, kw = runs[tag]
        w = workloads.make(name, **kw)
        tol = Tolerances(orth_tol=w.orth_tol)
        t0 = time.perf_counter()
        Gout, info = parallel_jacobi(w.G.copy(order="F"), w.J.copy(),
                                     SolverConfig(variant="2F", strategy="round_robin",
                                                  p=w.p, tol=tol))
        wall = time.perf_counter() - t0
        kappa = np.sqrt(scaled_condition(gram(w.G)))
        key = f"{name}_n{w.n}_b{w.b}"
        out = {key + "_lam": w.J * column_norms_squared(Gout),
               key + "_colsum": Gout.sum(axis=0),
               key + "_info": np.array([info.sweeps, info.rotations, info.big_rotations,
                                        info.max_abs_t, int(info.converged), wall, kappa,
                                        os.cpu_count()], np.float64)}
        np.savez_compressed(os.path.join(HERE, f"fullsize_{key}.npz"), **out)
        print(key, info.sweeps, info.rotations, f"{wall:.1f}s", f"kappa {kappa:.3e}", flush=True)


def variants():
    """The other reference variants on small seeded inputs: 3F / 2B / 3B
    through parallel_jacobi (parallel.py:150-174) and the sequential drivers
    seq / seqF / seqB through run_solver (solve.py:44-64).  Stored: the input,
    lambda = J ||g||^2 per column of G_out, DiagInfo, kappa(G_s)."""
    from hjacobi.factorization import scaled_condition
    from hjacobi.solve import SolveOptions, run_solver
    rng = np.random.default_rng(777)
    specs = [
        # (m, n, n_neg, complex, graded, p, strategy, variants)
        (256, 256, 96, False, False, 4, "round_robin", ("2F", "3F", "2B", "3B")),
        (256, 192, 64, True, False, 3, "modulus", ("2F", "3F", "2B", "3B")),
        (256, 256, 77, False, True, 2, "round_robin", ("3F", "2B", "3B")),
        (160, 128, 40, True, False, 2, "round_robin", ("2B", "3F")),
        (100, 90, 33, False, False, 3, "modulus", ("2B", "3B")),     # ragged blocks of 15
    ]
    out, meta = {}, {}
    for k, (m, n, nneg, cplx, graded, p, strat, vs) in enumerate(specs):
        G = random_full_rank(rng, m, n, cplx)
        if graded:
            G = np.asfortranarray(G * 10.0 ** (-rng.uniform(0, 6, n)))
        J = np.array([1] * (n - nneg) + [-1] * nneg, np.int8)
        out[f"v{k}_G"], out[f"v{k}_J"] = G, J
        kappa = float(np.sqrt(scaled_condition(gram(G))))
        meta[f"v{k}"] = dict(m=m, n=n, p=p, strategy=strat, variants=list(vs), kappa=kappa, orth_tol=n * EPS)
        for v in vs:
            Gout, info = parallel_jacobi(G.copy(order="F"), J.copy(),
                                         SolverConfig(variant=v, strategy=strat, p=p,
                                                      tol=Tolerances(orth_tol=n * EPS)))
            out[f"v{k}_{v}_lam"] = J * column_norms_squared(Gout)
            out[f"v{k}_{v}_info"] = np.array([info.sweeps, info.rotations, info.big_rotations,
                                             info.max_abs_t, int(info.converged)], np.float64)
            print(f"v{k}", v, info.sweeps, info.rotations, info.converged, flush=True)
    # sequential drivers
    G = random_full_rank(rng, 128, 128, False)
    J = np.array([1] * 80 + [-1] * 48, np.int8)
    out["s_G"], out["s_J"] = G, J
    meta["s"] = dict(n=128, nt_outer=32, kappa=float(np.sqrt(scaled_condition(gram(G)))), orth_tol=128 * EPS)
    for v in ("seq", "seqF", "seqB"):
        Gout, info = run_solver(G.copy(order="F"), J.copy(),
                                SolveOptions(variant=v, nt_outer=32, tol=Tolerances(orth_tol=128 * EPS)))
        out[f"s_{v}_lam"] = J * column_norms_squared(Gout)
        out[f"s_{v}_info"] = np.array([info.sweeps, info.rotations, info.big_rotations,
                                       info.max_abs_t, int(info.converged)], np.float64)
        print("s", v, info.sweeps, info.rotations, info.converged, flush=True)
    np.savez_compressed(os.path.join(HERE, "variants.npz"), **out)
    with open(os.path.join(HERE, "variants.json"), "w") as f:
        json.dump(meta, f, indent=1)


def matio():
    """HJAC files written by the reference's own writer (matio.py:26-37, 65-71)."""
    from hjacobi.matio import write_matrix, write_signs
    rng = np.random.default_rng(4242)
    A = np.asfortranarray(rng.standard_normal((5, 3)))
    Z = np.asfortranarray(rng.standard_normal((4, 6)) + 1j * rng.standard_normal((4, 6)))
    write_matrix(os.path.join(HERE, "hjac_real.bin"), A)
    write_matrix(os.path.join(HERE, "hjac_cplx.bin"), Z)
    write_matrix(os.path.join(HERE, "hjac_real.txt"), A, text=True)
    write_matrix(os.path.join(HERE, "hjac_cplx.txt"), Z, text=True)
    write_signs(os.path.join(HERE, "hjac_signs.txt"), np.array([1, -1, 1, 1, -1, -1], np.int8))
    np.savez(os.path.join(HERE, "hjac_expected.npz"), A=A, Z=Z)


def kernels():
    """Pivot-level pins: structured Cholesky and jacobi_diagonalize."""
    out = {}
    rng = np.random.default_rng(66)
    for k in range(6):
        n_i = int(rng.integers(1, 33))
        n_j = int(rng.integers(1, 33))
        cplx = k % 2 == 1
        lam_i = rng.uniform(0.5, 4.0, n_i)
        lam_j = rng.uniform(0.5, 4.0, n_j)
        B = rng.standard_normal((n_i, n_j))
        if cplx:
            B = B + 1j * rng.standard_normal((n_i, n_j))
        B *= 0.6 * np.sqrt(lam_i.min() * lam_j.min()) / np.linalg.norm(B, 2)
        R = structured_cholesky(lam_i, B, lam_j)
        out[f"sc{k}_lam_i"], out[f"sc{k}_lam_j"], out[f"sc{k}_A"], out[f"sc{k}_R"] = lam_i, lam_j, B, R
    for k, (n, nneg, cplx) in enumerate([(6, 0, False), (10, 5, False), (16, 6, True),
                                         (64, 16, False), (64, 32, True)]):
        G = random_full_rank(rng, n, n, cplx)
        J = np.array([1] * (n - nneg) + [-1] * nneg, np.int8)
        R = chol_upper(gram(G))
        R0 = R.copy()
        info = jacobi_diagonalize(R, J, Tolerances(), accumulate=True)
        out[f"jd{k}_R0"], out[f"jd{k}_J"], out[f"jd{k}_R"], out[f"jd{k}_W"] = R0, J, R, info.W
        out[f"jd{k}_info"] = np.array([info.sweeps, info.rotations, info.big_rotations,
                                       info.max_abs_t, int(info.converged)])
    # error-path pins: exception type raised by the reference
    errs = {}
    G = random_full_rank(rng, 16, 16, False)
    G[:, 5] = G[:, 2]
    try:
        parallel_jacobi(G, np.ones(16, np.int8), SolverConfig(variant="2F", p=2))
        errs["duplicate_column"] = "none"
    except Exception as e:  # the reference's re-raise (parallel.py:298) can itself fail
        errs["duplicate_column"] = [type(e).__name__, type(e.__cause__).__name__]
    G = random_full_rank(rng, 16, 16, False)
    G[:, 3] = 0.0
    try:
        parallel_jacobi(G, np.ones(16, np.int8), SolverConfig(variant="2F", p=2))
        errs["zero_column"] = "none"
    except Exception as e:
        errs["zero_column"] = [type(e).__name__, type(e.__cause__).__name__]
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    with open(os.path.join(HERE, "errors.json"), "w") as f:
        json.dump(errs, f, indent=1)


if __name__ == "__main__":
    with open(os.path.join(HERE, "provenance.json"), "w") as f:
        import numba
        json.dump({"reference": REF, "hjacobi": hjacobi.__version__,
                   "numpy": np.__version__, "numba": numba.__version__,
                   "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
                   "numba_enabled": hjacobi.NUMBA_ENABLED}, f, indent=1)
    which = sys.argv[1:] or ["schedules", "kernels", "small_solves", "config_proxies"]
    for name in which:
        globals()[name]()
