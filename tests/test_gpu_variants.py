"""GPU parity of the other reference variants (3F / 2B / 3B through
parallel_jacobi, seq / seqF / seqB through run_solver) against goldens the
reference itself produced (tests/golden/make_golden.py variants ->
variants.npz), plus the B step against the oracle's 2B restatement."""
import json
import os

import numpy as np
import pytest

import paper_1008_4166_b200 as pkg
from conftest import GOLDEN

pytestmark = pytest.mark.gpu
EPS = float(np.finfo(np.float64).eps)


def _load():
    return np.load(os.path.join(GOLDEN, "variants.npz")), json.load(open(os.path.join(GOLDEN, "variants.json")))


def _cases():
    _, meta = _load()
    return [(k, v) for k in sorted(meta) if k != "s" for v in meta[k]["variants"]]


@pytest.mark.parametrize("key,variant", _cases())
def test_variant_matches_reference(key, variant):
    """Per-eigenvalue relative error <= 64 n eps kappa(G_s) against the
    reference run of the SAME variant, converged, and the sweep count within
    +-1 for the F variants.  The B variants apply one annihilation cycle per
    step, so their sweep count depends on the pair order inside the cycle
    (the reference's is sequential column-cyclic, _kernels.py:41-52; the GPU's
    is the parallel ring order): +-2."""
    z, meta = _load()
    mt = meta[key]
    G, J = z[key + "_G"], z[key + "_J"]
    cfg = pkg.SolverConfig(variant=variant, strategy=mt["strategy"], p=mt["p"],
                           tol=pkg.Tolerances(orth_tol=mt["orth_tol"]))
    Gout, info = pkg.parallel_jacobi(G, J, cfg)
    ref_info = z[f"{key}_{variant}_info"]
    ref = np.sort(z[f"{key}_{variant}_lam"])
    got = np.sort(J * np.sum(np.abs(np.asarray(Gout)) ** 2, axis=0))
    rel = np.max(np.abs(got - ref) / np.abs(ref))
    bound = 64 * mt["n"] * EPS * mt["kappa"]
    assert info.converged
    assert rel <= bound, (key, variant, rel, bound)
    slack = 1 if variant.endswith("F") else 2
    assert abs(info.sweeps - int(ref_info[0])) <= slack, (key, variant, info.sweeps, ref_info[0])
    if variant.endswith("B"):
        assert info.stats["prepass_visited"] == 0  # no F pre-pass (parallel.py:229-230)
        # one cycle per step: far fewer rotations than the F variants
        assert info.rotations < 4 * int(ref_info[1])


@pytest.mark.parametrize("variant", ["seq", "seqF", "seqB"])
def test_sequential_drivers_map_to_the_ring(variant):
    """run_solver with the sequential variants (solve.py:47-56) returns the
    same eigenvalues as the reference's sequential drivers."""
    z, meta = _load()
    mt = meta["s"]
    G, J = z["s_G"], z["s_J"]
    opts = pkg.SolveOptions(variant=variant, nt_outer=mt["nt_outer"], tol=pkg.Tolerances(orth_tol=mt["orth_tol"]))
    Gout, info = pkg.run_solver(G, J, opts)
    ref = np.sort(z[f"s_{variant}_lam"])
    got = np.sort(J * np.sum(np.abs(np.asarray(Gout)) ** 2, axis=0))
    assert info.converged
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= 64 * mt["n"] * EPS * mt["kappa"]


def test_b_variant_matches_oracle_2b():
    """GPU 2B against the oracle's 2B restatement on a fresh seeded input."""
    import oracle as O
    rng = np.random.default_rng(5)
    n = 192
    G = np.asfortranarray(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    J = np.array([1] * 100 + [-1] * 92, np.int8)
    tol = n * EPS
    ref_G, ref_info = O.parallel_jacobi_2b(G, J, 3, "round_robin", orth_tol=tol)
    Gout, info = pkg.parallel_jacobi(G, J, pkg.SolverConfig(variant="2B", strategy="round_robin", p=3,
                                                           tol=pkg.Tolerances(orth_tol=tol)))
    ref = np.sort(J * O.column_norms2(ref_G))
    got = np.sort(J * np.sum(np.abs(np.asarray(Gout)) ** 2, axis=0))
    kappa = np.sqrt(O.scaled_condition(O.gram(G)))
    assert info.converged and abs(info.sweeps - ref_info.sweeps) <= 2
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= 64 * n * EPS * kappa


def test_default_options_beyond_256_columns():
    """solve_hermitian(H) with the reference's default SolveOptions (variant
    'seq', p = 1; solve.py:29-41) works for n > 256: the ring uses as many
    workers as the 128-column kernels need (parallel.effective_p)."""
    rng = np.random.default_rng(11)
    n = 300
    A = rng.standard_normal((n, n))
    H = (A + A.T) / 2
    res, metrics = pkg.solve_hermitian(H)
    ref = np.sort(np.linalg.eigvalsh(H))[::-1]
    assert metrics["converged"]
    assert np.max(np.abs(np.sort(res.eigenvalues)[::-1] - ref)) <= 1e-10 * np.abs(ref).max()
    assert metrics["residual"] <= 1e-12 and metrics["orthogonality"] <= 64 * n * EPS
    G = np.asfortranarray(rng.standard_normal((600, 600)))
    _, info = pkg.parallel_jacobi(G, np.ones(600, np.int8), pkg.SolverConfig(variant="2F", p=1))
    assert info.converged and info.stats["p_effective"] == 3


def test_in_place_sequential_entry_points():
    """jacobi_diagonalize / full_block / block_oriented (rotations.py:203-223,
    blocking.py:205-293): in place, DiagInfo, W with G_in W = G_out, the
    reference's eigenvalues."""
    z, meta = _load()
    mt = meta["s"]
    J = z["s_J"]
    tol = pkg.Tolerances(orth_tol=mt["orth_tol"])
    bound = 64 * mt["n"] * EPS * mt["kappa"]
    part = pkg.greedy_partition(mt["n"], mt["nt_outer"])
    for fn, key, kw in ((lambda G: pkg.jacobi_diagonalize(G, J, tol, accumulate=True), "seq", {}),
                        (lambda G: pkg.full_block(G, J, part, tol, accumulate_V=True), "seqF", {}),
                        (lambda G: pkg.block_oriented(G, J, part, tol), "seqB", {})):
        G0 = z["s_G"].copy(order="F")
        G = G0.copy(order="F")
        info = fn(G)
        ref = np.sort(z[f"s_{key}_lam"])
        got = np.sort(J * np.sum(G * G, axis=0))
        assert info.converged and np.max(np.abs(got - ref) / np.abs(ref)) <= bound, key
        if info.W is not None:
            assert np.max(np.abs(G0 @ info.W - G)) <= 1e-9 * np.abs(G).max()
            Jm = np.diag(J.astype(float))   # W is J-unitary (test_rotations.py:201-209)
            assert np.max(np.abs(info.W.T @ Jm @ info.W - Jm)) <= 64 * mt["n"] * EPS * np.max(np.abs(info.W)) ** 2 * mt["kappa"]


def test_apply_rotation_contract():
    """compute_plane_rotation + apply_rotation annihilate the pivot's
    off-diagonal Gram entry (rotations.py:128-182; test_rotations.py:41-58)."""
    rng = np.random.default_rng(3)
    for cx, (jr, js) in ((False, (1, 1)), (True, (1, -1)), (True, (-1, -1))):
        G = rng.standard_normal((8, 2)) + (1j * rng.standard_normal((8, 2)) if cx else 0)
        if jr != js:
            G[:, 1] *= 0.3   # keep the hyperbolic pivot definite
        A = G.conj().T @ G
        rot = pkg.compute_plane_rotation(A[0, 0].real, A[1, 1].real, A[0, 1], jr, js)
        D = np.array([A[0, 0].real, A[1, 1].real])
        W = np.eye(2, dtype=G.dtype)
        pkg.apply_rotation(G, W, D, 0, 1, rot)
        A2 = G.conj().T @ G
        assert abs(A2[0, 1]) <= 32 * EPS * np.sqrt(A2[0, 0].real * A2[1, 1].real)
        assert np.allclose(D, [A2[0, 0].real, A2[1, 1].real], rtol=1e-13)


def test_scaled_condition_on_the_gpu():
    """kappa(A_s) from the solver itself (factorization.scaled_condition_factor)
    equals the reference's eigvalsh-based value (factorization.py:156-168)."""
    rng = np.random.default_rng(8)
    for cx in (False, True):
        G = rng.standard_normal((200, 160)) + (1j * rng.standard_normal((200, 160)) if cx else 0)
        G = G * 10.0 ** (-rng.uniform(0, 5, 160))
        ref = pkg.scaled_condition(G.conj().T @ G)
        got = pkg.scaled_condition_factor(np.asfortranarray(G))
        assert abs(got - ref) <= 1e-9 * ref, (got, ref)


def test_read_matrix_pinned(tmp_path):
    rng = np.random.default_rng(1)
    Z = np.asfortranarray(rng.standard_normal((33, 7)) + 1j * rng.standard_normal((33, 7)))
    pkg.write_matrix(tmp_path / "z.bin", Z)
    out = pkg.read_matrix_pinned(tmp_path / "z.bin")
    assert out.flags.f_contiguous and np.array_equal(out, Z)


@pytest.mark.parametrize("cx", [False, True], ids=["f64", "c128"])
@pytest.mark.parametrize("n,m,p,variant,strategy", [
    (96, 100, 3, "2F", "round_robin"),    # b = 16: the order-32 pivot instance, m > n
    (130, 131, 2, "2F", "round_robin"),   # ragged blocks 33/33/32/32 -> order-128 instance, odd m
    (260, 260, 2, "2F", "modulus"),       # b = 65 -> order-256 instance with padding
    (130, 131, 2, "2B", "round_robin"),
    (260, 260, 2, "2B", "round_robin"),
    (96, 100, 3, "2B", "modulus"),
])
def test_ragged_shapes_every_kernel_instance(cx, n, m, p, variant, strategy):
    """Odd row counts, ragged and padded blocks through every pivot-order
    instance of the factor / Jacobi / update kernels, both variants, against
    the oracle's restatement of the same variant."""
    import oracle as O
    rng = np.random.default_rng(n + m + p)
    G = rng.standard_normal((m, n)) + (1j * rng.standard_normal((m, n)) if cx else 0)
    G = np.asfortranarray(G)
    J = np.array([1] * (n - n // 3) + [-1] * (n // 3), np.int8)
    tol = n * EPS
    if variant == "2F":
        ref_G, ref_info = O.parallel_jacobi_2f(G, J, p, strategy, orth_tol=tol)
    else:
        ref_G, ref_info = O.parallel_jacobi_2b(G, J, p, strategy, orth_tol=tol)
    Gout, info = pkg.parallel_jacobi(G, J, pkg.SolverConfig(variant=variant, strategy=strategy, p=p,
                                                           tol=pkg.Tolerances(orth_tol=tol)))
    ref = np.sort(J * O.column_norms2(ref_G))
    got = np.sort(J * np.sum(np.abs(np.asarray(Gout)) ** 2, axis=0))
    kappa = np.sqrt(O.scaled_condition(O.gram(G)))
    assert info.converged and abs(info.sweeps - ref_info.sweeps) <= (1 if variant == "2F" else 2)
    assert np.max(np.abs(got - ref) / np.abs(ref)) <= 64 * n * EPS * kappa
    # column order is preserved (parallel.py:299-301): every output column keeps its sign's inertia count
    res = pkg.extract_eigen(Gout, J)
    lam = res.eigenvalues.cpu().numpy() if hasattr(res.eigenvalues, "cpu") else np.asarray(res.eigenvalues)
    assert np.all(np.sign(lam) == J)


def test_tail_split_is_bitwise_neutral():
    """A step with more pivots than resident Jacobi clusters splits its last,
    mostly empty wave onto a second stream (solver.cu run_phase).  Same
    arithmetic: G_out is bitwise equal to the single-launch run."""
    import torch
    from paper_1008_4166_b200 import parallel as par
    rng = np.random.default_rng(21)
    p, b, m = 20, 66, 700          # 20 pivots of order 132 -> the order-256 complex instance (18 resident)
    n = 2 * p * b
    G = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    # m < n would be rank deficient: use a tall factor instead
    m = n + 8
    G = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    J = np.array([1] * (n // 2) + [-1] * (n - n // 2), np.int8)
    Gd = torch.from_numpy(np.ascontiguousarray(G.T)).cuda().t()
    outs, res = [], []
    for split in (True, False):
        cfg = pkg.SolverConfig(variant="2F", strategy="round_robin", p=p, tol=pkg.Tolerances(orth_tol=n * EPS),
                               tail_split=split, sweep_count=2)
        out = torch.empty_like(Gd.t()).t()
        res.append(par.solve_device(Gd, J, cfg, out=out))
        outs.append(out)
    assert res[0].tail_splits > 0 and res[1].tail_splits == 0
    assert res[0].rotations == res[1].rotations
    assert torch.equal(outs[0], outs[1])


def test_randomised_shapes_against_the_oracle():
    """60 seeded random small problems (tools/fuzz_gpu.py: both dtypes, variants
    and orderings, ragged blocks down to width 1, graded columns, any inertia)
    agree with the oracle; 300 more were run once per round (profiles/)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "fuzz_gpu", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "fuzz_gpu.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.run(60, 7) == 0


def test_c_example_runs_on_the_gpu(tmp_path):
    """examples/solve_c.c (plain C caller of the ABI) solves its problem."""
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    libdir = os.path.join(root, "paper_1008_4166_b200")
    exe = str(tmp_path / "solve_c")
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(root, "include"), os.path.join(root, "examples", "solve_c.c"),
                    "-o", exe, "-L", libdir, "-l:libhjb200.so", f"-Wl,-rpath,{libdir}", "-lm"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "converged 1" in r.stdout, (r.stdout, r.stderr)
