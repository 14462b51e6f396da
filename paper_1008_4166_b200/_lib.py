"""ctypes binding of libhjb200.so (include/hjb200.h).

The product path has no CPU fallback: if the shared library is missing or
cannot be loaded, every entry point raises ``RuntimeError`` (call
``paper_1008_4166_b200.build.build()`` or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HJB_LIB") or os.path.join(HERE, "libhjb200.so")

HJB_OK, HJB_EINVAL, HJB_PIVOT_INDEFINITE, HJB_CHOL_FAIL, HJB_ECUDA, HJB_ENCCL, HJB_ENOMEM = range(7)
HJB_F64, HJB_C128 = 0, 1
HJB_MODULUS, HJB_ROUND_ROBIN = 0, 1
HJB_HOST, HJB_DEVICE = 0, 1
HJB_FLAG_PHASE_TIMES = 1
HJB_FLAG_GATHER_ROOT = 4
HJB_FLAG_VARIANT_B = 8
HJB_FLAG_NO_TAIL_SPLIT = 16
ST_N = 8


class Problem(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("memspace", C.c_int32),
        ("m", C.c_int64), ("n", C.c_int64), ("ldg", C.c_int64),
        ("G_in", C.c_void_p), ("G_out", C.c_void_p), ("signs", C.c_void_p),
        ("p", C.c_int32), ("strategy", C.c_int32),
        ("orth_tol", C.c_double), ("quad_tol", C.c_double),
        ("max_sweeps", C.c_int32), ("device", C.c_int32),
        ("stream", C.c_void_p), ("comm", C.c_void_p), ("flags", C.c_int32),
        ("first_sweep", C.c_int32), ("sweep_count", C.c_int32),
    ]


class Result(C.Structure):
    _fields_ = [
        ("sweeps", C.c_int32), ("converged", C.c_int32),
        ("rotations", C.c_int64), ("big_rotations", C.c_int64),
        ("max_abs_t", C.c_double),
        ("fail_rank", C.c_int32), ("fail_r", C.c_int32), ("fail_s", C.c_int32),
        ("pairs_visited", C.c_int64), ("pairs_updated", C.c_int64),
        ("prepass_visited", C.c_int64), ("prepass_updated", C.c_int64),
        ("fallbacks", C.c_int64),
        ("t_total_ms", C.c_double), ("t_gram_ms", C.c_double), ("t_pivot_ms", C.c_double),
        ("t_update_ms", C.c_double), ("t_exchange_ms", C.c_double),
        ("exchange_bytes", C.c_int64),
        ("cluster_size", C.c_int32), ("gram_splits", C.c_int32),
        ("inner_sweeps", C.c_int64), ("inner_pair_visits", C.c_int64),
        ("kernel_launches", C.c_int64), ("tail_splits", C.c_int64),
    ]


# name -> (restype, argtypes); every symbol include/hjb200.h declares
SIGNATURES = {
    "hjb_version": (C.c_int, []),
    "hjb_last_error": (C.c_char_p, []),
    "hjb_device_count": (C.c_int, []),
    "hjb_solve": (C.c_int, [C.POINTER(Problem), C.POINTER(Result)]),
    "hjb_schedule": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "hjb_steps_per_sweep": (C.c_int, [C.c_int32, C.c_int32]),
    "hjb_partition": (C.c_int, [C.c_int64, C.c_int32, C.c_void_p]),
    "hjb_extract": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "hjb_orthogonality": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                    C.POINTER(C.c_double), C.c_void_p]),
    "hjb_gram": (C.c_int, [C.c_int32, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                           C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hjb_pivot": (C.c_int, [C.c_int32, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                            C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                            C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "hjb_pivot_ld": (C.c_int, [C.c_int32]),
    "hjb_jacobi": (C.c_int, [C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                             C.c_double, C.c_double, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]),
    "hjb_plane_rotations": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]),
    "hjb_pivot_set_profile": (C.c_int, [C.c_void_p]),
    "hjb_tune": (C.c_int, [C.c_int32, C.c_int32]),
    "hjb_pivot_occupancy": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "hjb_inner_order": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    "hjb_pivot_order": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                 C.POINTER(C.c_int32)]),
    "hjb_update": (C.c_int, [C.c_int32, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32,
                             C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hjb_exchange_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_void_p, C.c_void_p]),
    "hjb_block_owners": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    "hjb_comm_unique_id": (C.c_int, [C.c_void_p]),
    "hjb_comm_init": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "hjb_comm_destroy": (C.c_int, [C.c_void_p]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """The loaded library; raises RuntimeError if it is not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is not built; run `python -m paper_1008_4166_b200.build` "
                        "(there is no CPU fallback)")
                L = C.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                if L.hjb_version() != 2:
                    raise RuntimeError("libhjb200.so ABI version mismatch")
                # tuning overrides for experiments (0 = the library's heuristic)
                nt, cl = int(os.environ.get("HJB_PIVOT_THREADS", 0)), int(os.environ.get("HJB_PIVOT_CLUSTER", 0))
                if nt or cl:
                    L.hjb_tune(nt, cl)
                _lib = L
    return _lib


def last_error() -> str:
    msg = lib().hjb_last_error()
    return msg.decode() if msg else ""


def check(rc: int, res: Result | None = None):
    """Map an hjb_status to the reference's exception types
    (errors.py:10-44; parallel.py:296-298 prefixes the worker rank)."""
    if rc == HJB_OK:
        return
    msg = last_error()
    if rc == HJB_EINVAL:
        raise ValueError(msg)
    if rc == HJB_PIVOT_INDEFINITE:
        r = res.fail_r if res is not None else -1
        s = res.fail_s if res is not None else -1
        raise errors.PivotDefinitenessError(r, s, msg)
    if rc == HJB_CHOL_FAIL:
        raise errors.DefinitenessError(msg)
    if rc == HJB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)
