"""Row partition of X across ranks (rows are independent, one global reduction).

Host-side logic only (no GPU): which contiguous block of the global X a rank owns.  Theta is keyed
by the GLOBAL row index, so the sum over ranks of the rank-local sketches is the sketch of the
whole X for ANY partition."""
from __future__ import annotations


def row_block(m_global: int, world: int, rank: int) -> tuple[int, int]:
    """(row_offset, m_local) of `rank` for a strong-scaling split of m_global rows."""
    if world < 1 or not 0 <= rank < world or m_global < 0:
        raise ValueError("bad partition arguments")
    base, rem = divmod(m_global, world)
    m_local = base + (1 if rank < rem else 0)
    return rank * base + min(rank, rem), m_local


def weak_block(m_per_rank: int, world: int, rank: int) -> tuple[int, int, int]:
    """(row_offset, m_local, m_global) when every rank owns m_per_rank rows (weak scaling)."""
    if world < 1 or not 0 <= rank < world or m_per_rank < 0:
        raise ValueError("bad partition arguments")
    return rank * m_per_rank, m_per_rank, m_per_rank * world
