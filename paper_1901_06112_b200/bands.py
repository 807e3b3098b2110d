"""Row-band planning (pure host logic, no device work).

Two uses, both driven by the R-row vertical halo of the separable kernel:

* within one GPU, when the (m0+1)(n+1) horizontally-filtered planes of the
  whole image exceed the HBM budget (cfg 5: 67 M px x 1105 planes x 4 B =
  296 GB > 180 GB), K2/K3 run band by band; band b's K2 covers its output
  rows plus R virtual rows on each side (rows outside the image replicate
  the border row, so K3 never clamps);
* across GPUs, rank g owns the rows [g*H/G, (g+1)*H/G) and receives
  R (+ patch radius) input rows from each neighbour (``parallel.py``).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Band:
    out0: int      # first output row
    out_rows: int  # output rows
    hp0: int       # first virtual row of the horizontal-pass planes (out0 - R, may be < 0)
    hp_rows: int   # rows of planes: out_rows + 2R virtual rows


def band_for(out0: int, out_rows: int, H: int, R: int) -> Band:
    return Band(out0, out_rows, out0 - R, out_rows + 2 * R)


def plan_bands(H: int, R: int, row_bytes: int, budget_bytes: int, max_bands: int | None = None) -> list[Band]:
    """Split rows [0, H) into the fewest near-equal bands whose plane buffer
    (hp_rows * row_bytes) fits in ``budget_bytes``."""
    if H < 1 or R < 0 or row_bytes < 1:
        raise ValueError("bad band geometry")
    max_rows = budget_bytes // row_bytes
    if max_rows >= H + 2 * R:
        return [band_for(0, H, H, R)]
    out_max = max_rows - 2 * R
    if out_max < 1:
        raise MemoryError(f"plane buffer budget {budget_bytes} B cannot hold one band "
                          f"({2 * R + 1} rows x {row_bytes} B)")
    nb = -(-H // out_max)
    if max_bands is not None:
        nb = max(nb, max_bands)
    bands = []
    base, rem = divmod(H, nb)
    r = 0
    for b in range(nb):
        rows = base + (1 if b < rem else 0)
        bands.append(band_for(r, rows, H, R))
        r += rows
    return bands


def shard_rows(H: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [lo, hi) owned by ``rank`` in a ``world``-way row-band split."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, rem = divmod(H, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def halo_rows(lo: int, hi: int, H: int, halo: int) -> tuple[int, int]:
    """Input rows a shard needs: its own rows plus ``halo`` on each side,
    clipped to the image (edge replication happens inside the kernels)."""
    return max(0, lo - halo), min(H, hi + halo)
