"""3-D Hilbert-curve keys for the locality reorder.

The keys are the reference's (``tetray.hilbert``, hilbert.py:14-73: Skilling's
transpose construction on a 2**order grid, axis 0 most significant) -- the
reorder permutation, and with it every tet id the GPU returns, depends on
them bit for bit.  The arithmetic runs natively (``tb_hilbert_keys`` /
``tb_hilbert_quantize`` in csrc/host_mesh.cpp, host code, no GPU needed);
this module checks arguments and shapes.
"""

from __future__ import annotations

import numpy as np

from ._lib import addr, check, lib

MAX_ORDER = 20


def _cells_array(cells) -> np.ndarray:
    a = np.asarray(cells)
    if a.ndim != 2 or a.shape[1] != 3:
        raise ValueError(f"expected an (n, 3) array of grid cells, got shape {a.shape}")
    return np.ascontiguousarray(a, dtype=np.int64)


def hilbert_keys(cells, order: int) -> np.ndarray:
    """uint64 key per (n, 3) integer cell of the 2**order grid."""
    if not 1 <= int(order) <= MAX_ORDER:
        raise ValueError(f"order {order} outside 1..{MAX_ORDER}")
    c = _cells_array(cells)
    side = 1 << int(order)
    if c.size and (int(c.min()) < 0 or int(c.max()) >= side):
        raise ValueError(f"cells must lie in [0, {side}) for order {order}")
    keys = np.empty(len(c), dtype=np.uint64)
    if len(c):
        check(lib.tb_hilbert_keys(addr(c), len(c), int(order), addr(keys)), "tb_hilbert_keys")
    return keys


def hilbert_index(cell, order: int) -> int:
    """Key of a single cell."""
    return int(hilbert_keys(np.reshape(np.asarray(cell, dtype=np.int64), (1, 3)), order)[0])


def quantize(points, lo, hi, order: int = 10) -> np.ndarray:
    """(n, 3) cells of the 2**order grid spanning the box [lo, hi]; a flat
    axis (hi <= lo) maps to extent 1, out-of-box points clamp to the border."""
    if not 1 <= int(order) <= MAX_ORDER:
        raise ValueError(f"order {order} outside 1..{MAX_ORDER}")
    p = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    box = [np.ascontiguousarray(np.broadcast_to(np.asarray(b, dtype=np.float64), (3,))) for b in (lo, hi)]
    cells = np.empty((len(p), 3), dtype=np.int64)
    if len(p):
        check(lib.tb_hilbert_quantize(addr(p), len(p), addr(box[0]), addr(box[1]), int(order), addr(cells)),
              "tb_hilbert_quantize")
    return cells
