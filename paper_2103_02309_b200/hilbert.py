"""3-D Hilbert keys (J. Skilling, "Programming the Hilbert curve", AIP Conf.
Proc. 707, 2004: AxesToTranspose + bit interleave).

Mirror of the reference's key function (/root/reference/pkg/src/tetray/
hilbert.py:14-73) -- same grid, same key for every cell -- used by
``tetmesh.reorder`` to sort points and tets along the curve.
"""

from __future__ import annotations

import numpy as np


def _axes_to_transpose(x: list[np.ndarray], order: int) -> None:
    """In-place Skilling transform of three uint32 coordinate arrays."""
    top = np.uint32(1 << (order - 1))
    q = top
    while q > 1:
        mask = np.uint32(q - 1)
        for i in range(3):
            flip = (x[i] & q) != 0
            # where bit q of x[i] is set: invert low bits of x[0];
            # otherwise exchange the low bits of x[0] and x[i]
            x[0] = np.where(flip, x[0] ^ mask, x[0])
            swap = np.where(flip, np.uint32(0), (x[0] ^ x[i]) & mask)
            x[0] ^= swap
            x[i] ^= swap
        q = np.uint32(q >> 1)
    # Gray code
    x[1] ^= x[0]
    x[2] ^= x[1]
    acc = np.zeros_like(x[0])
    q = top
    while q > 1:
        acc = np.where((x[2] & q) != 0, acc ^ np.uint32(q - 1), acc)
        q = np.uint32(q >> 1)
    for i in range(3):
        x[i] ^= acc


def hilbert_keys(cells: np.ndarray, order: int) -> np.ndarray:
    """uint64 Hilbert key of each (n, 3) integer grid cell in [0, 2**order)."""
    cells = np.asarray(cells)
    if cells.ndim != 2 or cells.shape[1] != 3:
        raise ValueError("cells must have shape (n, 3)")
    if order < 1 or order > 20:
        raise ValueError("order must be in 1..20")
    lim = 1 << order
    if cells.min(initial=0) < 0 or cells.max(initial=0) >= lim:
        raise ValueError(f"grid coordinates must be in [0, {lim})")
    x = [np.ascontiguousarray(cells[:, i]).astype(np.uint32) for i in range(3)]
    _axes_to_transpose(x, order)
    # interleave: bit b of axis 0 is the most significant of each triple
    key = np.zeros(len(cells), dtype=np.uint64)
    for b in range(order - 1, -1, -1):
        triple = (
            (((x[0] >> np.uint32(b)) & np.uint32(1)).astype(np.uint64) << np.uint64(2))
            | (((x[1] >> np.uint32(b)) & np.uint32(1)).astype(np.uint64) << np.uint64(1))
            | ((x[2] >> np.uint32(b)) & np.uint32(1)).astype(np.uint64)
        )
        key = (key << np.uint64(3)) | triple
    return key


def hilbert_index(cell, order: int) -> int:
    return int(hilbert_keys(np.asarray(cell, dtype=np.int64)[None, :], order)[0])


def quantize(points: np.ndarray, lo, hi, order: int = 10) -> np.ndarray:
    """Cells of the 2**order grid spanning [lo, hi] (hilbert.py:66-73 semantics)."""
    points = np.asarray(points, dtype=np.float64)
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    extent = np.where(hi > lo, hi - lo, 1.0)
    scaled = ((points - lo) / extent) * ((1 << order) - 1)
    return np.clip(np.floor(scaled).astype(np.int64), 0, (1 << order) - 1)
