"""Row-slab partition for the multi-GPU path (host logic).

Rank r of P owns interior rows [row_begin, row_end) of an ny-row grid.  Slabs consist of whole
units of `unit` rows (tile rows for the hierarchical method, 16-row blocks for the classic
kernel), so no tile straddles two ranks and the iteration is identical for every P
(DESIGN.md §3 reading c18).  Units are spread as evenly as possible (sizes differ by <= 1 unit).
"""
from __future__ import annotations


def slab(ny: int, unit: int, rank: int, nranks: int) -> tuple[int, int]:
    if not (0 <= rank < nranks) or unit < 1 or ny < 1:
        raise ValueError("bad slab request")
    units = (ny + unit - 1) // unit
    if units < nranks:
        raise ValueError(f"{ny} rows in units of {unit} cannot feed {nranks} ranks")
    b = (units * rank // nranks) * unit
    e = min((units * (rank + 1) // nranks) * unit, ny)
    return b, e


def neighbours(rank: int, nranks: int) -> tuple[int | None, int | None]:
    """(rank owning the rows below, rank owning the rows above) or None at the global ring."""
    return (rank - 1 if rank > 0 else None, rank + 1 if rank < nranks - 1 else None)
