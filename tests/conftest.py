"""Shared fixtures: golden meshes and ray sets.

Golden data (tests/golden/) was produced by the unmodified reference
(tests/golden/make_golden.py); nothing here reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2103_02309_b200.tetmesh import (  # noqa: E402
    CompactMesh,
    SceneTriangleSoup,
    _records_from_tables,
)

GOLDEN = ROOT / "tests" / "golden"
FIXTURES = ("box1", "box4", "pane4", "region4", "open_box4", "model")
RAY_SEEDS = {"box4": 100, "pane4": 101, "region4": 102, "model": 103, "open_box4": 104, "box1": 105}
PANE_OCC = [(0, 2, (1, 1), (3, 3))]
REGION_OCC = [(axis, k, (1, 1), (3, 3)) for axis in range(3) for k in (1, 3)]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libtetb200.so")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


HAS_GPU = _has_gpu()


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN / "golden_small.npz")


@pytest.fixture(scope="session")
def digests():
    return json.loads((GOLDEN / "golden_digests.json").read_text())


def golden_mesh(g, name: str, layout: str = "tet20") -> CompactMesh:
    sv = g[f"{name}/side_verts"]
    sn = g[f"{name}/side_neighbors"]
    return CompactMesh(
        layout=layout,
        points=g[f"{name}/points"],
        records=_records_from_tables(layout, sv, sn),
        side_verts=sv,
        side_neighbors=sn,
        cf_triangle=g[f"{name}/cf_triangle"],
        cf_tets=g[f"{name}/cf_tets"],
        cf_verts=g[f"{name}/cf_verts"],
        source_tet=int(g[f"{name}/source_tet"]),
        soup=SceneTriangleSoup(
            vertices=g[f"{name}/soup_vertices"],
            triangles=g[f"{name}/soup_triangles"],
            material_ids=g[f"{name}/soup_material_ids"],
        ),
    )


@pytest.fixture(scope="session")
def meshes(golden):
    return {name: golden_mesh(golden, name) for name in FIXTURES}


def digest(*arrays) -> str:
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def mesh_digest(m) -> str:
    return digest(m.points, m.side_verts, m.side_neighbors, m.cf_triangle, m.cf_tets, m.cf_verts, m.records_u32(),
                  m.soup.vertices, m.soup.triangles, np.array([m.source_tet]))
