"""The drop-in claim, exercised through the UNMODIFIED reference.

The reference package is installed under oracle/_ref/site by
oracle/build_ref.sh (git-ignored, shipped to the GPU box).  Here its own
batch layer (/root/reference/pkg/src/tetray/batch.py:39-159) is driven with
``kernels=paper_2103_02309_b200.kernels`` and compared with the same calls on
the reference's own compiled kernels, on meshes built by the reference's own
ingestion/encode; and the reference's own test suite (tests/test_kernels.py,
tests/test_acceptance.py, ...) runs with the CUDA module registered as its
compiled and active backend (tests/ref_suite_plugin.py).
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from refpkg import REF_PKG, REF_SITE, ROOT, have_ref, import_tetray

pytestmark = pytest.mark.skipif(not have_ref(), reason="oracle/_ref/site missing: run oracle/build_ref.sh")

PANE_OCC = [(0, 2, (1, 1), (3, 3))]
REGION_OCC = [(axis, k, (1, 1), (3, 3)) for axis in range(3) for k in (1, 3)]
LAYOUTS = ("tet32", "tet20", "tet16")


def _interior_rays(mesh, n, seed):
    """The reference conftest's ray sampler (pkg/tests/conftest.py:61-73)."""
    rng = np.random.default_rng(seed)
    ti = rng.integers(0, mesh.n_tets, n).astype(np.int32)
    bary = rng.dirichlet(np.ones(4) * 4.0, n)
    pts = mesh.points.astype(np.float64)
    o = np.einsum("ij,ijk->ik", bary, pts[mesh.side_verts[ti]])
    d = rng.normal(size=(n, 3))
    return o.astype(np.float32), d.astype(np.float32), ti


@pytest.fixture(scope="module")
def ref():
    return import_tetray()


@pytest.fixture(scope="module")
def ref_meshes(ref):
    """Fixtures built by the reference's own code (pkg/tests/conftest.py:21-58)."""
    from tetray.ingestion import associate_constrained_faces, build_box_fixture, load_obj, parse_tetgen
    from tetray.tetmesh import encode

    def fx(n=4, occluders=(), walls="constrained"):
        raw, soup = build_box_fixture(n, occluders=occluders, walls=walls)
        return encode(raw, "tet20", soup)

    data = REF_PKG / "data" / "model"
    raw = parse_tetgen(data / "blob.1")
    soup = load_obj(data / "blob.obj")
    faces = np.array([cf.vertex_ids for cf in raw.constrained_faces], dtype=np.int64)
    for cf, tid in zip(raw.constrained_faces, associate_constrained_faces(raw.points, faces, soup, tolerance=1e-9)):
        cf.triangle_id = int(tid)
    return {"box4": fx(), "pane4": fx(occluders=PANE_OCC), "region4": fx(occluders=REGION_OCC),
            "open_box4": fx(walls="open"), "model": encode(raw, "tet20", soup)}


def test_reference_install_is_the_compiled_reference(ref):
    from tetray import backend

    assert backend.active_backend() == "compiled"
    assert Path(backend.get_kernels("compiled").__file__).resolve().is_relative_to(REF_SITE.resolve())


def test_plugin_registers_the_cuda_module():
    """CPU: the suite plugin swaps the reference's backend (no kernel runs)."""
    code = ("import ref_suite_plugin, types; ref_suite_plugin.pytest_configure(types.SimpleNamespace("
            "addinivalue_line=lambda *a: None)); from tetray import backend; k = backend.get_kernels(); "
            "print(k.__name__, k.BACKEND_NAME, backend.get_kernels('compiled') is k)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(REF_SITE), str(ROOT / "tests"), str(ROOT)]),
               TETB200_REF_SITE=str(REF_SITE))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.split() == ["paper_2103_02309_b200.kernels", "cuda", "True"]


def _hits(h):
    return [h.status, h.cf, h.triangle, h.t, h.tet_front, h.tet_back, h.visited]


@pytest.mark.gpu
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("name", ("box4", "pane4", "region4", "open_box4", "model"))
def test_reference_batch_cast_rays_with_cuda_kernels(ref, ref_meshes, name, layout):
    from tetray import backend, batch
    from tetray.tetmesh import relayout

    import paper_2103_02309_b200.kernels as cuda

    mesh = relayout(ref_meshes[name], layout)
    o, d, st = _interior_rays(mesh, 10_000, 200 + len(name))
    got = batch.cast_rays(mesh, o, d, st, kernels=cuda)
    exp = batch.cast_rays(mesh, o, d, st, kernels=backend.get_kernels("compiled"))
    for f, a, b in zip(("status", "cf", "triangle", "t", "tet_front", "tet_back", "visited"), _hits(got), _hits(exp)):
        assert a.dtype == b.dtype, f
        assert np.array_equal(a, b), f


@pytest.mark.gpu
@pytest.mark.parametrize("layout", LAYOUTS)
def test_reference_batch_cast_rays_visits_with_cuda_kernels(ref, ref_meshes, layout):
    from tetray import backend, batch
    from tetray.tetmesh import relayout

    import paper_2103_02309_b200.kernels as cuda

    for name in ("region4", "model"):
        mesh = relayout(ref_meshes[name], layout)
        o, d, st = _interior_rays(mesh, 3000, 41)
        hg, vg, og = batch.cast_rays_visits(mesh, o, d, st, kernels=cuda)
        he, ve, oe = batch.cast_rays_visits(mesh, o, d, st, kernels=backend.get_kernels("compiled"))
        assert np.array_equal(og, oe) and np.array_equal(vg, ve)
        for a, b in zip(_hits(hg), _hits(he)):
            assert np.array_equal(a, b)


@pytest.mark.gpu
def test_reference_batch_locate_and_shadow_with_cuda_kernels(ref, ref_meshes):
    from tetray import backend, batch

    import paper_2103_02309_b200.kernels as cuda

    K = backend.get_kernels("compiled")
    rng = np.random.default_rng(43)
    for name in ("region4", "pane4", "model"):
        mesh = ref_meshes[name]
        lo, hi = mesh.points.min(0) - 0.5, mesh.points.max(0) + 0.5
        q = rng.uniform(lo, hi, size=(5000, 3))  # includes outside points
        tg, vg = batch.locate_points(mesh, q, kernels=cuda)
        te, ve = batch.locate_points(mesh, q, kernels=K)
        assert np.array_equal(tg, te) and np.array_equal(vg, ve)
        assert (tg == -1).any() and (tg >= 0).any()
        light = lo + (hi - lo) * np.array([0.31, 0.72, 0.76])
        lt, _ = batch.locate_points(mesh, light[None], kernels=K)
        inside = te >= 0
        og, wg = batch.shadow_rays(mesh, q[inside], light, te[inside], int(lt[0]), kernels=cuda)
        oe, we = batch.shadow_rays(mesh, q[inside], light, te[inside], int(lt[0]), kernels=K)
        assert np.array_equal(og, oe) and np.array_equal(wg, we)


@pytest.mark.gpu
def test_reference_test_suite_runs_on_the_cuda_backend():
    """The reference's whole test suite, unmodified, with the CUDA module as
    its compiled and active backend: test_kernels.py becomes "pure-python
    reference vs CUDA" (bit-exact), and every acceptance criterion
    (test_acceptance.py:54-370, incl. 2 oracle equivalence, 3 layout
    equivalence, 9 point location, 10 shadow/secondary correctness through the
    renderer's 4-thread tile pool) runs its batch calls on the GPU."""
    if not (REF_PKG / "tests" / "test_acceptance.py").exists():
        pytest.skip("oracle/_ref/pkg missing: run oracle/build_ref.sh")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(REF_SITE), str(ROOT / "tests"), str(ROOT)]),
               TETB200_REF_SITE=str(REF_SITE))
    env.pop("TETRAY_PURE", None)
    cmd = [sys.executable, "-m", "pytest", "-q", "-s", "-p", "ref_suite_plugin", "-p", "no:cacheprovider",
           "--rootdir", str(REF_PKG), "-c", os.devnull, str(REF_PKG / "tests")]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=1800, cwd=str(REF_PKG))
    log = out.stdout + "\n" + out.stderr
    if (ROOT / "gpurun_out").is_dir():
        (ROOT / "gpurun_out" / "ref_suite_cuda.log").write_text(log)
    assert "tetray backend swapped" in log or "passed" in log
    assert out.returncode == 0, log[-6000:]
    acc = re.findall(r"ACCEPTANCE\s+(\d+) (PASS|FAIL)", log)
    assert sorted(int(c) for c, s in acc if s == "PASS") == list(range(1, 11)), acc
    m = re.search(r"(\d+) passed", log)
    assert m and int(m.group(1)) >= 200, log[-3000:]
