"""Block partitions (reference blocking.py:18-68): pure index bookkeeping."""

from dataclasses import dataclass


@dataclass(frozen=True)
class BlockPartition:
    """Block-column sizes and their offsets (blocking.py:18-45)."""

    sizes: tuple

    def __post_init__(self):
        if any(s < 1 for s in self.sizes):
            raise ValueError("all block sizes must be >= 1")

    @property
    def b(self) -> int:
        return len(self.sizes)

    @property
    def n(self) -> int:
        return sum(self.sizes)

    @property
    def offsets(self):
        out = [0]
        for s in self.sizes:
            out.append(out[-1] + s)
        return tuple(out)

    def columns(self, i):
        off = self.offsets
        return slice(off[i], off[i + 1])


def num_blocks(n: int, n_t: int) -> int:
    """ceil(n / n_t) (blocking.py:48-52)."""
    if n < 1 or n_t < 1:
        raise ValueError("n and n_t must be >= 1")
    return -(-n // n_t)


def greedy_partition(n: int, n_t: int) -> BlockPartition:
    b = num_blocks(n, n_t)
    last = (n - 1) % n_t + 1
    return BlockPartition(tuple([n_t] * (b - 1) + [last]))


def uniform_partition(n: int, b: int) -> BlockPartition:
    """b blocks whose sizes differ by at most one, larger first
    (blocking.py:63-68); the partition the 2F driver uses (parallel.py:266)."""
    if not 1 <= b <= n:
        raise ValueError(f"need 1 <= b <= n, got b={b}, n={n}")
    n_min, b_r = divmod(n, b)
    return BlockPartition(tuple([n_min + 1] * b_r + [n_min] * (b - b_r)))
