"""Build a bench scene with the REFERENCE's own pipeline and save it in the
reference's own .npz format (test infrastructure; never the product path).

    PYTHONPATH=oracle/_ref/site python oracle/make_ref_scene.py --grid 55 --layout tet20 --scheme hilbert

Pipeline, all from the unmodified reference installed by oracle/build_ref.sh:
tools/gen_model_mesh.py at GRID (pkg/tools/gen_model_mesh.py:25-63,76-91)
-> TetGen/OBJ files -> ingestion.parse_tetgen / load_obj /
associate_constrained_faces -> tetmesh.encode -> tetmesh.reorder
(render.py:150-163 does the same) -> cli.save_compact (cli.py:249-265).
The bench's reference arm loads the file with cli.load_compact
(cli.py:268-290), so that process never maps this repo's CUDA library.
The output is byte-identical to the mesh bench.py builds natively (pinned by
the mesh digests in tests/golden/golden_digests.json, which the same
pipeline produced).
"""

from __future__ import annotations

import argparse
import contextlib
import importlib.util
import io
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = HERE / "_ref"
SCENES = REF / "scenes"


def scene_path(grid: int, layout: str, scheme: str) -> Path:
    return SCENES / f"blob{grid}_{layout}_{scheme}.npz"


def build(grid: int, layout: str, scheme: str) -> Path:
    from tetray.cli import save_compact
    from tetray.ingestion import associate_constrained_faces, load_obj, parse_tetgen
    from tetray.tetmesh import encode, reorder

    spec = importlib.util.spec_from_file_location("gen_model_mesh", REF / "pkg" / "tools" / "gen_model_mesh.py")
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    gen.GRID = grid
    with tempfile.TemporaryDirectory() as tmp:
        gen.ROOT = Path(tmp)
        with contextlib.redirect_stdout(io.StringIO()):
            gen.main()
        data = Path(tmp) / "data" / "model"
        raw = parse_tetgen(data / "blob.1")
        soup = load_obj(data / "blob.obj")
    faces = np.array([cf.vertex_ids for cf in raw.constrained_faces], dtype=np.int64)
    tri_ids = associate_constrained_faces(raw.points, faces, soup, tolerance=1e-9)
    for cf, tid in zip(raw.constrained_faces, tri_ids):
        cf.triangle_id = int(tid)
    mesh = reorder(encode(raw, layout, soup), scheme)
    SCENES.mkdir(parents=True, exist_ok=True)
    out = scene_path(grid, layout, scheme)
    tmp_out = out.with_suffix(".tmp.npz")
    save_compact(mesh, tmp_out)
    tmp_out.replace(out)
    return out


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=55)
    ap.add_argument("--layout", default="tet20")
    ap.add_argument("--scheme", default="hilbert")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    out = scene_path(a.grid, a.layout, a.scheme)
    if out.exists() and not a.force:
        return 0
    import tetray

    if not str(Path(tetray.__file__).resolve()).startswith(str(REF.resolve())):
        raise SystemExit(f"tetray must come from {REF}/site (got {tetray.__file__})")
    t0 = time.perf_counter()
    build(a.grid, a.layout, a.scheme)
    print(f"wrote {out} ({out.stat().st_size >> 20} MiB) in {time.perf_counter() - t0:.0f}s", file=sys.stderr)
    return 0


if __name__ == "__main__":
    sys.exit(main())
