"""Column sharding of Y = A X across GPUs.

Every operation of the reference multiply (proj/src/kernels.cpp:27-62) acts
on one feature column j independently, so rank r of N holds a full replica of
the uploaded CBM and multiplies its own contiguous column slab of X; the
slabs of Y are bit-identical to the corresponding columns of the 1-GPU
result and no collective is needed for A.X itself. Slabs are multiples of 4
columns (16-byte rows for the LDG.128 lanes) where the width allows.
"""
from __future__ import annotations

from . import column_slab as _native_slab


def column_slab(d: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) columns of `rank`: contiguous, balanced in units of 4 columns
    (the library's cbm_b200_column_slab, so every rank and the single-process
    cbm_b200_spmm_sharded agree on the partition)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("column_slab: bad rank/world")
    return _native_slab(d, world, rank)


def all_slabs(d: int, world: int) -> list[tuple[int, int]]:
    return [column_slab(d, world, r) for r in range(world)]
