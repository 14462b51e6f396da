"""CPU-side checks of the native library: it loads, exports every symbol the
C header declares, its ring schedule is bit-exact with the reference's, and
argument validation matches the reference's ValueErrors.  No GPU needed."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
import paper_1008_4166_b200 as P
from paper_1008_4166_b200 import _lib, strategies


def header_symbols():
    src = open(os.path.join(ROOT, "include", "hjb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(hjb_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 14
    for name in syms:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, name
    assert L.hjb_version() == 2


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("strategy", ["modulus", "round_robin"])
@pytest.mark.parametrize("p", list(range(1, 9)) + [16, 32, 64])
def test_native_schedule_bit_exact(strategy, p):
    z = golden("schedules.npz")
    lay_ref = z[f"{strategy}_p{p}_layouts"]
    plans_ref = z[f"{strategy}_p{p}_plans"]
    sweeps = lay_ref.shape[0] // strategies.steps_per_sweep(strategy, p)
    lay, plans = strategies.schedule_arrays(strategy, p, sweeps)
    assert np.array_equal(lay, lay_ref)
    assert np.array_equal(plans, plans_ref)


def test_schedule_period_two_sweeps():
    """Layouts repeat every 2 sweeps for the config sizes."""
    for strategy in ("modulus", "round_robin"):
        for p in (8, 16, 32, 64, 128):
            lay, _ = strategies.schedule_arrays(strategy, p, 4)
            s = strategies.steps_per_sweep(strategy, p)
            assert np.array_equal(lay[:2 * s], lay[2 * s:])


def test_steps_per_sweep_native():
    L = _lib.lib()
    assert L.hjb_steps_per_sweep(0, 3) == 6 and L.hjb_steps_per_sweep(1, 3) == 5
    assert L.hjb_steps_per_sweep(1, 0) == -1


def test_validation_errors_match_reference():
    rng = np.random.default_rng(0)
    G = rng.standard_normal((4, 4))
    J = np.ones(4, np.int8)
    with pytest.raises(ValueError):
        P.SolverConfig(variant="4X")
    with pytest.raises(ValueError):
        P.SolverConfig(variant="2F", p=0)
    assert P.SolverConfig(variant="2F", strategy="rr").strategy == "round_robin"
    with pytest.raises(ValueError):  # parallel.py:264-265
        P.parallel_jacobi(G, J, P.SolverConfig(variant="2F", p=3))
    with pytest.raises(ValueError):
        P.parallel_jacobi(G, np.array([1, 2, 1, 1]), P.SolverConfig(variant="2F", p=1))
    for v in ("2F", "3F", "2B", "3B"):  # every reference variant is accepted (parallel.py:43)
        assert P.SolverConfig(variant=v).variant == v
    assert P.SolveOptions().variant == "seq"  # the reference's default (solve.py:31)
    from paper_1008_4166_b200.parallel import effective_p
    assert effective_p(256, 1) == 1 and effective_p(257, 1) == 2 and effective_p(32768, 128) == 128
    assert effective_p(600, 1) == 3 and effective_p(600, 5) == 5


def test_uniform_partition_matches_reference_rule():
    part = P.uniform_partition(20, 6)
    assert part.sizes == (4, 4, 3, 3, 3, 3) and part.offsets[-1] == 20
    with pytest.raises(ValueError):
        P.uniform_partition(3, 4)


def test_generate_sweep_schedule_surface():
    lay = P.generate_sweep_schedule("rr", 3, 1)
    assert len(lay) == 5 and lay[0] == [(1, 6), (2, 5), (3, 4)]


def test_orthogonality_argument_validation():
    """hjb_orthogonality rejects bad arguments before touching a device, and an
    empty U has orthogonality 0 (solve.py:108-110 returns 0.0 for U.size == 0)."""
    import ctypes

    L = _lib.lib()
    out = ctypes.c_double(-1.0)
    dummy = ctypes.c_void_p(16)  # never dereferenced on these paths
    assert L.hjb_orthogonality(_lib.HJB_F64, 4, 4, None, 4, ctypes.byref(out), None) == _lib.HJB_EINVAL
    assert L.hjb_orthogonality(_lib.HJB_F64, 4, 4, dummy, 3, ctypes.byref(out), None) == _lib.HJB_EINVAL
    assert L.hjb_orthogonality(_lib.HJB_F64, 5, 4, dummy, 5, ctypes.byref(out), None) == _lib.HJB_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.HJB_EINVAL)
    assert L.hjb_orthogonality(_lib.HJB_C128, 4, 0, dummy, 4, ctypes.byref(out), None) == _lib.HJB_OK
    assert out.value == 0.0


def test_native_partition_matches_reference_rule():
    """hjb_partition (the partition hjb_solve uses) == blocking.py:63-68 as
    restated by the oracle, for ragged and exact splits."""
    import oracle as O
    for n in (1, 7, 20, 64, 100, 2048, 4097):
        for nbl in (1, 2, 3, 6, 16, 64):
            if nbl > n:
                with pytest.raises(ValueError):
                    P.uniform_partition(n, nbl)
                continue
            assert list(P.uniform_partition(n, nbl).sizes) == O.uniform_sizes(n, nbl)
    assert P.greedy_partition(10, 4).sizes == (4, 4, 2) and P.num_blocks(10, 4) == 3


def test_header_is_plain_c_and_the_c_example_links(tmp_path):
    """include/hjb200.h is a C header (plain pointers and sizes, no C++ / torch
    types): examples/solve_c.c compiles as C99 with -Werror and links against
    the built library; every symbol the header declares resolves.  Without a
    GPU the program stops at hjb_device_count() (exit 2, "no CPU fallback")."""
    import re
    import shutil
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    libdir = os.path.join(root, "paper_1008_4166_b200")
    exe = str(tmp_path / "solve_c")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(root, "include"),
                    os.path.join(root, "examples", "solve_c.c"), "-o", exe, "-L", libdir, "-l:libhjb200.so",
                    f"-Wl,-rpath,{libdir}", "-lm"], check=True)
    header = open(os.path.join(root, "include", "hjb200.h")).read()
    declared = set(re.findall(r"^(?:int|const char \*)\s*(hjb_\w+)\(", header, re.M))
    assert declared and declared <= set(_lib.SIGNATURES), declared - set(_lib.SIGNATURES)
    if _lib.lib().hjb_device_count() < 1:
        r = subprocess.run([exe], capture_output=True, text=True)
        assert r.returncode == 2 and "no CPU fallback" in r.stderr
