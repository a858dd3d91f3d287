"""The C-ABI boundary without a GPU: the library loads, exports every entry
point include/tetb200.h declares, and fails loudly (error code + message,
no crash) instead of falling back to the CPU."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from conftest import HAS_GPU, ROOT


def _declared():
    text = (ROOT / "include" / "tetb200.h").read_text()
    return sorted(set(re.findall(r"\b(tb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2103_02309_b200 import _lib

    names = _declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(_lib.lib, name), name
    assert set(names) == set(_lib.EXPORTED)


def test_abi_version_and_errors():
    from paper_2103_02309_b200._lib import lib

    assert lib.tb_abi_version() == 1
    assert lib.tb_mesh_destroy(None) == 0
    rc = lib.tb_cast_rays(None, 1, None, None, None, None, None, None, None, None, None, None, None)
    assert rc == -1
    assert b"NULL" in lib.tb_last_error()


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure path")
def test_mesh_create_fails_loudly_without_gpu(meshes):
    from paper_2103_02309_b200._lib import TetB200Error
    from paper_2103_02309_b200.device import DeviceMesh

    with pytest.raises(TetB200Error):
        DeviceMesh(meshes["box4"], device=0)


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure path")
def test_kernel_module_has_no_cpu_fallback(meshes):
    from paper_2103_02309_b200 import kernels
    from paper_2103_02309_b200._lib import TetB200Error

    m = meshes["box4"]
    import numpy as np

    with pytest.raises(TetB200Error):
        kernels.cast_rays(m, np.zeros((1, 3), np.float32), np.ones((1, 3), np.float32), np.zeros(1, np.int32))


def test_header_cites_reference_interfaces():
    text = (ROOT / "include" / "tetb200.h").read_text()
    for cite in ("_kernels.pyx:271-370", "_kernels.pyx:416-492", "_kernels.pyx:527-614", "batch.py:57-71",
                 "traversal.py:484-511"):
        assert cite in text


def test_oracle_library_loads():
    from oracle import pyoracle

    L = pyoracle.lib()
    for name in ("to_cast_rays", "to_sctp_cast_rays", "to_locate_points", "to_shadow_rays", "to_mt_t"):
        assert hasattr(L, name)


def test_no_oracle_import_in_product():
    for p in (ROOT / "paper_2103_02309_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p


def test_schedule_setter_roundtrip_and_validation():
    from paper_2103_02309_b200 import _lib

    mode0, k0 = _lib.get_schedule()
    try:
        _lib.set_schedule("compact", 8)
        assert _lib.get_schedule() == (3, 8)
        _lib.set_schedule(None, 24)  # leaves the mode alone
        assert _lib.get_schedule() == (3, 24)
        with pytest.raises(_lib.TetB200Error):
            _lib.set_schedule(9)
        assert _lib.lib.tb_set_schedule(-1, 0) != 0
        assert _lib.get_schedule() == (3, 24)
    finally:
        _lib.set_schedule(mode0, k0)


def test_binned_pieces_rule():
    """tb_binned_pieces: the binned schedule splits into two pieces of whole
    262144-ray sorting segments only when the batch spans two or more of
    them; a negative count is rejected (host logic, no GPU)."""
    from paper_2103_02309_b200._lib import lib

    seg = 262144
    assert lib.tb_binned_pieces(-1) == -1
    for n, want in ((0, 1), (1, 1), (seg, 1), (seg + 1, 2), (2 * seg, 2), (16_777_216, 2)):
        assert lib.tb_binned_pieces(n) == want, n


def test_cast_rays_sched_validates_arguments():
    from paper_2103_02309_b200._lib import lib

    args = (None,) * 10
    assert lib.tb_cast_rays_sched(None, 1, *args, 0, None) == -1
    assert b"NULL" in lib.tb_last_error()
    fake = ctypes.c_void_p(1)  # never dereferenced: the schedule is checked first
    assert lib.tb_cast_rays_sched(fake, 1, *args, 9, None) == -1
    assert b"schedule" in lib.tb_last_error()


def test_probe_gather_validates_arguments():
    from paper_2103_02309_b200._lib import lib

    assert lib.tb_probe_gather(None, 1, 0, None, None) == -1
    assert b"NULL" in lib.tb_last_error()


@pytest.mark.gpu
def test_probe_gather_runs_per_layout(golden):
    """tb_probe_gather (the L2 gather roof bench.py reports) runs on every
    point-array layout and refuses TetMesh-80, which has none."""
    import torch

    from conftest import golden_mesh
    from paper_2103_02309_b200._lib import lib
    from paper_2103_02309_b200.device import device_mesh
    from paper_2103_02309_b200.tetmesh import relayout

    base = golden_mesh(golden, "box4", "tet32")
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    for layout in ("tet32", "tet20", "tet16"):
        dm = device_mesh(relayout(base, layout))
        assert lib.tb_probe_gather(dm.handle, 100_003, 7, sink.data_ptr(), None) == 0, lib.tb_last_error()
        assert lib.tb_probe_gather(dm.handle, -1, 7, sink.data_ptr(), None) == -1
    torch.cuda.synchronize()
    dm80 = device_mesh(base, layout="tet80")
    assert lib.tb_probe_gather(dm80.handle, 10, 7, sink.data_ptr(), None) != 0
    assert b"layout" in lib.tb_last_error()


@pytest.mark.gpu
def test_device_mesh_outlives_its_host_mesh(golden):
    """A DeviceMesh stays valid after the host mesh it was uploaded from is
    collected (the cache entry goes, the device copy stays while held)."""
    import gc

    import numpy as np

    from conftest import golden_mesh
    from paper_2103_02309_b200.device import device_mesh
    from paper_2103_02309_b200.tetmesh import relayout
    from paper_2103_02309_b200.trace import trace

    import torch

    base = golden_mesh(golden, "box4", "tet32")
    dm = device_mesh(relayout(base, "tet16"))  # the relayouted host mesh dies here
    gc.collect()
    n = 64
    o = torch.full((n, 3), 0.5, dtype=torch.float32, device="cuda") + torch.rand(n, 3, device="cuda")
    d = torch.randn(n, 3, device="cuda")
    from paper_2103_02309_b200.trace import locate

    st, _ = locate(dm, o.double(), torch.full((n,), base.source_tet, dtype=torch.int32, device="cuda"))
    res = trace(dm, o, d, st.clamp(min=0))
    torch.cuda.synchronize()
    assert int(res.status.max()) <= 1
    dm.close()
    from paper_2103_02309_b200._lib import TetB200Error

    with pytest.raises(TetB200Error):
        trace(dm, o, d, st.clamp(min=0))


def test_multi_gpu_entry_points_validate_arguments():
    """tb_trace_multi / tb_mesh_replicate / tb_cast_epilogue reject bad
    arguments before touching a device (runs without a GPU)."""
    import ctypes

    from paper_2103_02309_b200._lib import lib

    nulls = (None,) * 10
    assert lib.tb_trace_multi(0, None, 16, 16, *nulls, None) == -1
    assert b"n_meshes" in lib.tb_last_error()
    assert lib.tb_trace_multi(65, None, 16, 16, *nulls, None) == -1
    out = ctypes.c_void_p()
    assert lib.tb_mesh_replicate(None, 0, ctypes.byref(out)) == -1
    assert b"NULL" in lib.tb_last_error()
    assert lib.tb_cast_epilogue(None, 1, *(None,) * 7, None) == -1


def test_fastcall_extension_is_built_and_bound():
    """The per-tile fast path of kernels.cast_rays (csrc/fastcall.c) is built
    with the library and bound to the same libtetb200.so the ctypes path uses."""
    from paper_2103_02309_b200 import kernels

    assert kernels._fastcall is not None
    assert kernels._fastcall.__file__.startswith(str(ROOT / "paper_2103_02309_b200"))


def test_fastcall_declines_other_layouts_and_checks_arguments():
    """cast4 returns None (the caller takes the general path) for anything but
    contiguous float32 (n, 3) / int32 (n,) inputs, and raises what the ctypes
    path raises: ValueError on a length mismatch, IndexError on a start tet
    outside the mesh, TetB200Error from the C ABI (here: a NULL mesh handle)."""
    import numpy as np

    from paper_2103_02309_b200 import kernels
    from paper_2103_02309_b200._lib import TetB200Error

    f = kernels._fastcall.cast4
    o = np.zeros((4, 3), np.float32)
    d = np.ones((4, 3), np.float32)
    st = np.zeros(4, np.int32)
    assert f(0, 10, o.astype(np.float64), d, st) is None
    assert f(0, 10, o, d[::2].repeat(2, 0)[:, :2], st) is None
    assert f(0, 10, o, d, st.astype(np.int64)) is None
    assert f(0, 10, np.asfortranarray(np.zeros((4, 3), np.float32)), d, st) is None  # F-order
    with pytest.raises(ValueError, match="length mismatch"):
        f(0, 10, o[:3], d, st)
    with pytest.raises(IndexError, match=r"start\[2\] = 10"):
        f(0, 10, o, d, np.array([0, 1, 10, 2], np.int32))
    with pytest.raises(TetB200Error, match="NULL"):
        f(0, 10, o, d, st)
    status, cf, tet, visited = f(0, 10, o[:0], d[:0], st[:0])
    assert status.dtype == np.uint8 and cf.dtype == tet.dtype == visited.dtype == np.int32 and len(status) == 0


def test_ordered_cast_validates_arguments():
    from paper_2103_02309_b200._lib import lib

    assert lib.tb_cast_block_size() == 128
    rc = lib.tb_cast_rays_ordered(None, 1, None, None, None, None, 1, None, None, None, None, None, None, None, None)
    assert rc != 0 and b"NULL" in lib.tb_last_error()
