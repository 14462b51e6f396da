"""Ring orderings (reference strategies.py): the schedule itself is generated
by the native library (csrc/schedule.cpp, exported as hjb_schedule), which is
what the solver replays; this module is the Python surface over it."""

import numpy as np

from . import _lib

MODULUS = "modulus"
ROUND_ROBIN = "round_robin"
STRATEGIES = (MODULUS, ROUND_ROBIN)


def normalize_strategy(name: str) -> str:
    """strategies.py:19-24."""
    alias = {"rr": ROUND_ROBIN, "round-robin": ROUND_ROBIN}
    name = alias.get(name, name)
    if name not in STRATEGIES:
        raise ValueError(f"unknown strategy {name!r}")
    return name


def strategy_code(name: str) -> int:
    return _lib.HJB_MODULUS if normalize_strategy(name) == MODULUS else _lib.HJB_ROUND_ROBIN


def steps_per_sweep(strategy: str, p: int) -> int:
    """strategies.py:27-28."""
    return 2 * p if normalize_strategy(strategy) == MODULUS else 2 * p - 1


def schedule_arrays(strategy: str, p: int, sweeps: int = 1):
    """(layouts int32 [steps, p, 2], plans int32 [steps, p, 4]) from the
    native ring schedule; plans are (snd_rnk, snd_blk, rcv_rnk, rcv_blk)."""
    if p < 1:
        raise ValueError("p must be >= 1")
    steps = steps_per_sweep(strategy, p) * sweeps
    lay = np.zeros((steps, p, 2), np.int32)
    plans = np.zeros((steps, p, 4), np.int32)
    _lib.check(_lib.lib().hjb_schedule(strategy_code(strategy), p, sweeps,
                                       lay.ctypes.data, plans.ctypes.data))
    return lay, plans


def generate_sweep_schedule(strategy: str, p: int, sweeps: int = 1):
    """Global layouts per step, as strategies.py:143-176 (list of lists of
    (i_blk, j_blk) per rank); raises on collisions like the reference."""
    lay, _ = schedule_arrays(strategy, p, sweeps)
    nbl = 2 * p
    out = []
    for step in lay:
        layout = [tuple(int(v) for v in pr) for pr in step]
        if sorted(b for pr in layout for b in pr) != list(range(1, nbl + 1)):
            raise RuntimeError(f"block collision in layout {layout}")
        out.append(layout)
    return out
