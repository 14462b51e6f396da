"""Block-column partitions of the 2F driver (API of the reference's
blocking.py:18-68).  ``uniform_partition`` is the native one hjb_solve uses
(hjb_partition, csrc/solver.cu), so the Python view of the blocks is the GPU's
by construction; the other helpers are index arithmetic on top of it."""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from . import _lib


@dataclass(frozen=True)
class BlockPartition:
    """Widths of consecutive column blocks; ``offsets[i]`` is where block i
    starts and ``offsets[-1]`` the column count (reference blocking.py:18-45)."""

    sizes: tuple
    offsets: tuple = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        sizes = tuple(int(s) for s in self.sizes)
        if not sizes or min(sizes) < 1:
            raise ValueError("all block sizes must be >= 1")
        object.__setattr__(self, "sizes", sizes)
        object.__setattr__(self, "offsets", (0, *itertools.accumulate(sizes)))

    @property
    def b(self) -> int:
        return len(self.sizes)

    @property
    def n(self) -> int:
        return self.offsets[-1]

    def columns(self, i):
        return slice(self.offsets[i], self.offsets[i + 1])


def num_blocks(n: int, n_t: int) -> int:
    """Blocks of target width n_t covering n columns (blocking.py:48-52)."""
    if min(n, n_t) < 1:
        raise ValueError("n and n_t must be >= 1")
    return (n + n_t - 1) // n_t


def greedy_partition(n: int, n_t: int) -> BlockPartition:
    """Width n_t everywhere but a shorter remainder block at the end
    (blocking.py:55-60)."""
    full, rem = divmod(n, n_t) if n >= 1 and n_t >= 1 else (0, 0)
    num_blocks(n, n_t)  # validation
    return BlockPartition((n_t,) * full + ((rem,) if rem else ()))


def uniform_partition(n: int, b: int) -> BlockPartition:
    """b blocks of near-equal width, the wider ones first (blocking.py:63-68;
    parallel.py:266) -- computed by the library (hjb_partition)."""
    if not 1 <= b <= n:
        raise ValueError(f"need 1 <= b <= n, got b={b}, n={n}")
    off = np.zeros(b + 1, np.int64)
    _lib.check(_lib.lib().hjb_partition(n, b, off.ctypes.data))
    return BlockPartition(tuple(np.diff(off).tolist()))
