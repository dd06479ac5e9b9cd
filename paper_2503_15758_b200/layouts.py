"""Cyclic token layouts over a Pr x Pc device grid — the reference's square
layouts (pkg/src/attn2d/layouts.py:1-69) generalised to rectangles, plus the
ring's mirrored halves (strategies/ring.py:27-38).

Rank (r, c) has global rank r*Pc + c (the reference's ProcGrid.rank,
mesh.py:64-65).  With P = Pr*Pc:

* column-major (input/output layout): (r, c) owns tokens {x + P i},
  x = r + Pr c                                   (layouts.py COLUMN_MAJOR);
* row-major (keys/values after the permutation): (r, c) holds {y + P i},
  y = c + Pc r                                   (layouts.py ROW_MAJOR);
* row-gathered: all-gathering the column-major shards along grid row r gives
  the query rows {r + Pr t}; in all-gather order block c' holds
  r + Pr c' + P i, i.e. an affine-blocked index map (bases r + Pr c', stride P);
* col-gathered: all-gathering the row-major shards along column c gives the
  keys {c + Pc t}; block r' holds c + Pc r' + P i.

For Pr == Pc these are exactly the reference's four forms; the permutation
x -> (x div Pc, x mod Pc) is the reference's mirror transpose (r,c)->(c,r).
"""

from __future__ import annotations

from dataclasses import dataclass
from math import isqrt

import numpy as np

from .errors import ConfigError
from .ops import TokenIndex


@dataclass(frozen=True)
class Grid2D:
    pr: int
    pc: int

    def __post_init__(self):
        if self.pr < 1 or self.pc < 1:
            raise ConfigError(f"grid needs positive sides, got {self.pr}x{self.pc}")

    @classmethod
    def square(cls, p: int) -> "Grid2D":
        s = isqrt(p)
        if s * s != p:
            raise ConfigError(f"2d strategies need a square processor count, got p={p}")
        return cls(s, s)

    @property
    def p(self) -> int:
        return self.pr * self.pc

    def rank(self, r: int, c: int) -> int:
        return r * self.pc + c

    def coord(self, rank: int) -> tuple[int, int]:
        return rank // self.pc, rank % self.pc

    def coords(self):
        return [(r, c) for r in range(self.pr) for c in range(self.pc)]

    def row_ranks(self, r: int) -> list[int]:
        return [self.rank(r, c) for c in range(self.pc)]

    def col_ranks(self, c: int) -> list[int]:
        return [self.rank(r, c) for r in range(self.pr)]

    # residues of the cyclic deal
    def residue(self, r: int, c: int) -> int:
        return r + self.pr * c

    def kv_residue(self, r: int, c: int) -> int:
        return c + self.pc * r

    def kv_dest(self, r: int, c: int) -> int:
        """Rank that holds this rank's keys/values after the permutation."""
        x = self.residue(r, c)
        return self.rank(x // self.pc, x % self.pc)

    def kv_src(self, r: int, c: int) -> int:
        """Rank whose keys/values this rank holds after the permutation."""
        y = self.kv_residue(r, c)
        return self.rank(y % self.pr, y // self.pr)

    # index sets
    def check_n(self, n: int) -> int:
        if n % self.p:
            raise ConfigError(f"p={self.p} does not divide n={n}")
        return n // self.p

    def owned(self, n: int, r: int, c: int) -> np.ndarray:
        return np.arange(self.residue(r, c), n, self.p, dtype=np.int64)

    def kv_owned(self, n: int, r: int, c: int) -> np.ndarray:
        return np.arange(self.kv_residue(r, c), n, self.p, dtype=np.int64)

    def q_gathered(self, n: int, r: int) -> TokenIndex:
        L = self.check_n(n)
        return TokenIndex.blocked([r + self.pr * cc for cc in range(self.pc)], self.p, L)

    def k_gathered(self, n: int, c: int) -> TokenIndex:
        L = self.check_n(n)
        return TokenIndex.blocked([c + self.pc * rr for rr in range(self.pr)], self.p, L)


def ring_block_indices(n: int, p: int, rank: int) -> np.ndarray:
    """TE load-balanced ring rows: front block `rank` and the mirrored back
    block (strategies/ring.py:27-38)."""
    if p == 1:
        return np.arange(n, dtype=np.int64)
    if n % (2 * p):
        raise ConfigError(f"ring layout needs 2*p={2 * p} to divide n={n}")
    c = n // (2 * p)
    front = np.arange(rank * c, (rank + 1) * c, dtype=np.int64)
    back = np.arange(n // 2 + (p - 1 - rank) * c, n // 2 + (p - rank) * c, dtype=np.int64)
    return np.concatenate([front, back])


def ring_index(n: int, p: int, rank: int) -> TokenIndex:
    if p == 1:
        return TokenIndex.contiguous(n)
    c = n // (2 * p)
    return TokenIndex.blocked([rank * c, n // 2 + (p - 1 - rank) * c], 1, c)
