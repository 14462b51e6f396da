"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import json
import math
import os

import numpy as np
import pytest

import oracle as O
from conftest import GOLDEN, golden, small_solve_cases
from paper_1008_4166_b200 import workloads

EPS = np.finfo(np.float64).eps


@pytest.mark.parametrize("strategy", ["modulus", "round_robin"])
@pytest.mark.parametrize("p", list(range(1, 9)) + [16, 32, 64])
def test_schedule_bit_exact(strategy, p):
    z = golden("schedules.npz")
    lay = z[f"{strategy}_p{p}_layouts"]
    plans = z[f"{strategy}_p{p}_plans"]
    sweeps = lay.shape[0] // O.steps_per_sweep(strategy, p)
    got = np.array(O.sweep_schedule(strategy, p, sweeps), np.int32)
    assert np.array_equal(got, lay)
    ring = O.RingSchedule(strategy, p)
    gp = []
    for sweep in range(1, sweeps + 1):
        for _ in range(O.steps_per_sweep(strategy, p)):
            gp.append(ring.advance(sweep))
    assert np.array_equal(np.array(gp, np.int32), plans)


@pytest.mark.parametrize("case", small_solve_cases(), ids=lambda c: f"c{c['k']}")
def test_small_solves_bit_exact(case):
    Gout, info = O.parallel_jacobi_2f(case["G"], case["J"], case["p"], case["strategy"],
                                      orth_tol=case["orth_tol"], max_sweeps=case["max_sweeps"])
    assert np.array_equal(Gout, case["Gout"])
    assert info.sweeps == case["sweeps"]
    assert info.rotations == case["rotations"]
    assert info.big_rotations == case["big"]
    assert info.max_abs_t == case["max_t"]
    assert info.converged == case["converged"]


def test_structured_cholesky_and_diagonalize_bit_exact():
    z = golden("kernels.npz")
    for k in range(6):
        R = O.structured_cholesky(z[f"sc{k}_lam_i"], z[f"sc{k}_A"], z[f"sc{k}_lam_j"])
        assert np.array_equal(R, z[f"sc{k}_R"])
    for k in range(5):
        R = z[f"jd{k}_R0"].copy(order="F")
        W, sweeps, nrot, nbig, mt, conv = O.diagonalize(R, z[f"jd{k}_J"])
        info = z[f"jd{k}_info"]
        assert np.array_equal(R, z[f"jd{k}_R"]) and np.array_equal(W, z[f"jd{k}_W"])
        assert (sweeps, nrot, nbig, mt, conv) == (info[0], info[1], info[2], info[3], bool(info[4]))


def test_cfg1_full_size_bit_exact():
    z = golden("config_proxies.npz")
    w = workloads.cfg1()
    Gout, info = O.parallel_jacobi_2f(w.G, w.J, w.p, "round_robin", orth_tol=w.orth_tol,
                                      threads=4)
    key = "cfg1_n512_b32"
    assert np.array_equal(w.J * O.column_norms2(Gout), z[key + "_lam"])
    assert np.array_equal(Gout.sum(axis=0), z[key + "_colsum"])
    assert info.sweeps == 13 and info.rotations == int(z[key + "_info"][1])


def test_tournament_inner_order_within_tolerance():
    """The GPU's inner order vs the pinned cyclic one: outer sweeps within
    +-1 and eigenvalues within the north_star bound."""
    z = golden("config_proxies.npz")
    w = workloads.cfg3(n=512, b=32)
    Gout, info = O.parallel_jacobi_2f(w.G, w.J, w.p, "round_robin", orth_tol=w.orth_tol,
                                      inner_order="tournament", threads=4)
    key = "cfg3_n512_b32"
    ref = np.sort(z[key + "_lam"])
    lam = np.sort(w.J * O.column_norms2(Gout))
    kappa = math.sqrt(O.scaled_condition(O.gram(w.G)))
    assert np.all(np.abs(lam - ref) <= 64 * w.n * EPS * kappa * np.abs(ref))
    assert abs(info.sweeps - int(z[key + "_info"][0])) <= 1


def test_tournament_pairs_cover_each_pair_once():
    for n in (1, 2, 3, 7, 8, 64, 65):
        seen = {}
        for rnd in O.tournament_pairs(n):
            cols = [c for pr in rnd for c in pr]
            assert len(cols) == len(set(cols))
            for pr in rnd:
                assert pr[0] < pr[1] < n
                seen[pr] = seen.get(pr, 0) + 1
        assert len(seen) == n * (n - 1) // 2 and set(seen.values()) <= {1}


def test_reference_error_behaviour_recorded():
    errs = json.load(open(os.path.join(GOLDEN, "errors.json")))
    # a zero column surfaces as DefinitenessError (pre-pass Cholesky fails)
    assert errs["zero_column"][0] == "DefinitenessError"
    G = np.asfortranarray(np.random.default_rng(3).standard_normal((16, 16)))
    G[:, 3] = 0.0
    with pytest.raises(O.CholeskyFailure):
        O.parallel_jacobi_2f(G, np.ones(16, np.int8), 2, "modulus")


def test_oracle_2b_matches_reference_variants():
    """The 2B restatement (oracle.parallel_jacobi_2b; parallel.py:160-174,
    199-200) against the reference's own 2B runs (tests/golden/variants.npz):
    same sweeps and rotation counts, eigenvalues to rounding."""
    import json
    z = np.load(os.path.join(GOLDEN, "variants.npz"))
    meta = json.load(open(os.path.join(GOLDEN, "variants.json")))
    for key in ("v0", "v1", "v3", "v4"):
        mt = meta[key]
        G, J = z[key + "_G"], z[key + "_J"]
        Gout, info = O.parallel_jacobi_2b(G, J, mt["p"], mt["strategy"], orth_tol=mt["orth_tol"])
        ref_info = z[key + "_2B_info"]
        lam = J * O.column_norms2(Gout)
        ref = z[key + "_2B_lam"]
        assert info.converged and info.sweeps == int(ref_info[0]), (key, info.sweeps, ref_info)
        assert info.rotations == int(ref_info[1]), (key, info.rotations, ref_info)
        assert np.max(np.abs(lam - ref) / np.abs(ref)) <= 1e-12, key
