"""Locate the installed reference package (oracle/_ref/site, built by
oracle/build_ref.sh -- git-ignored, shipped to the GPU box with the repo
snapshot).  Test infrastructure: nothing here reads /root/reference."""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_SITE = ROOT / "oracle" / "_ref" / "site"
REF_PKG = ROOT / "oracle" / "_ref" / "pkg"
REF_SCENES = ROOT / "oracle" / "_ref" / "scenes"


def have_ref() -> bool:
    return (REF_SITE / "tetray" / "batch.py").exists()


def import_tetray():
    """The unmodified reference package (its own compiled _kernels included)."""
    if str(REF_SITE) not in sys.path:
        sys.path.insert(0, str(REF_SITE))
    import tetray

    if not Path(tetray.__file__).resolve().is_relative_to(REF_SITE.resolve()):
        raise ImportError(f"tetray resolved to {tetray.__file__}, not the oracle/_ref install")
    return tetray


def ref_cast_full(mesh, o, d, st, threads: int | None = None, chunk: int = 1 << 16):
    """The reference's batch.cast_rays (its compiled kernels + the batch
    epilogue, batch.py:39-80) over a thread pool -- the checker for the
    full-size parity tests.  Returns (status, cf, tet, visited, triangle, t,
    tet_back)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import_tetray()
    from tetray import batch

    n = len(st)
    bounds = list(range(0, n, chunk)) + [n]

    def one(i):
        a, b = bounds[i], bounds[i + 1]
        h = batch.cast_rays(mesh, o[a:b], d[a:b], st[a:b])
        return h.status, h.cf, h.tet_front, h.visited, h.triangle, h.t, h.tet_back

    with ThreadPoolExecutor(max_workers=threads or os.cpu_count() or 1) as pool:
        parts = list(pool.map(one, range(len(bounds) - 1)))
    return [np.concatenate([p[k] for p in parts]) for k in range(7)]


# The fused epilogue reproduces numpy 2.3's einsum("ij,ij->i") reduction order
# ((p0 + p2) + p1, traverse.cuh einsum3) bit for bit.  The reference's batch
# epilogue runs live on whatever numpy the box has: a numpy whose einsum sums
# in another order moves t by an ulp on a few % of rays.  Then t is held to
# the north-star contract instead (1e-5 relative), so a numpy bump cannot
# read as a kernel regression; every other array stays bit-exact.
EINSUM_PINNED_NUMPY = "2.3."
T_RTOL = 1e-5
HIT_NAMES = ("status", "cf", "tet", "visited", "triangle", "t", "tet_back")


def hits_mismatch(got, exp) -> dict:
    """Per-array mismatch counts of the 7 hit arrays (``t`` compared within
    T_RTOL when the live numpy is not the einsum-pinned one)."""
    import numpy as np

    bad = {}
    for name, g, e in zip(HIT_NAMES, got, exp):
        g, e = np.asarray(g), np.asarray(e)
        if g.shape != e.shape:
            bad[name] = f"shape {g.shape} != {e.shape}"
            continue
        same = g == e
        if g.dtype.kind == "f":
            same |= np.isnan(g) & np.isnan(e)
        neq = ~same
        if name == "t" and neq.any() and not np.__version__.startswith(EINSUM_PINNED_NUMPY):
            fin = np.isfinite(e) & np.isfinite(g)
            rel = np.abs(g[fin] - e[fin]) / np.maximum(np.abs(e[fin]), 1e-30)
            neq = neq & ~fin
            neq[np.nonzero(fin)[0][rel > T_RTOL]] = True
        bad[name] = int(np.count_nonzero(neq))
    return bad
