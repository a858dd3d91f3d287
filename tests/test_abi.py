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
