"""Randomised GPU-vs-oracle sweep over small shapes: both dtypes, both variants,
both orderings, ragged blocks down to width 1, tall and square factors,
definite and indefinite J.  Prints one line per failure and a summary.
    python tools/fuzz_gpu.py [--cases 200] [--seed 0]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_1008_4166_b200 as P

EPS = np.finfo(float).eps


def run(cases, seed):
    rng = np.random.default_rng(seed)
    bad = 0
    for k in range(cases):
        n = int(rng.integers(2, 150))
        p = int(rng.integers(1, max(2, min(6, n // 2) + 1)))
        while 2 * p > n:
            p -= 1
        m = n + int(rng.integers(0, 40))
        cx = bool(rng.integers(0, 2))
        variant = "2F" if rng.integers(0, 2) else "2B"
        strat = "round_robin" if rng.integers(0, 2) else "modulus"
        nneg = int(rng.integers(0, n + 1))
        G = rng.standard_normal((m, n)) + (1j * rng.standard_normal((m, n)) if cx else 0)
        if rng.integers(0, 3) == 0:
            G = G * 10.0 ** (-rng.uniform(0, 4, n))
        G = np.asfortranarray(G)
        J = np.array([1] * (n - nneg) + [-1] * nneg, np.int8)
        tol = n * EPS
        desc = f"case {k}: n={n} m={m} p={p} cx={cx} {variant} {strat} nneg={nneg}"
        try:
            if variant == "2F":
                ref_G, ri = O.parallel_jacobi_2f(G, J, p, strat, orth_tol=tol)
            else:
                ref_G, ri = O.parallel_jacobi_2b(G, J, p, strat, orth_tol=tol)
        except Exception as e:  # the oracle itself rejects the input (indefinite pivot): the GPU must raise too
            try:
                P.parallel_jacobi(G, J, P.SolverConfig(variant=variant, strategy=strat, p=p, tol=P.Tolerances(orth_tol=tol)))
                print("FAIL (oracle raised", type(e).__name__, "GPU did not)", desc, flush=True)
                bad += 1
            except Exception:
                pass
            continue
        try:
            Gout, info = P.parallel_jacobi(G, J, P.SolverConfig(variant=variant, strategy=strat, p=p,
                                                                tol=P.Tolerances(orth_tol=tol)))
        except Exception as e:
            print("FAIL (GPU raised", type(e).__name__, e, ")", desc, flush=True)
            bad += 1
            continue
        ref = np.sort(J * O.column_norms2(ref_G))
        got = np.sort(J * np.sum(np.abs(np.asarray(Gout)) ** 2, axis=0))
        kappa = np.sqrt(O.scaled_condition(O.gram(G)))
        rel = np.max(np.abs(got - ref) / np.abs(ref))
        slack = 1 if variant == "2F" else 2
        ok = info.converged == ri.converged and rel <= 64 * n * EPS * kappa and abs(info.sweeps - ri.sweeps) <= slack + 1
        if not ok:
            print("FAIL", desc, "rel", rel, "bound", 64 * n * EPS * kappa, "sweeps", info.sweeps, ri.sweeps,
                  "conv", info.converged, ri.converged, flush=True)
            bad += 1
    return bad


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    nbad = run(a.cases, a.seed)
    print(f"fuzz: {a.cases} cases, {nbad} failures", flush=True)
    sys.exit(1 if nbad else 0)
