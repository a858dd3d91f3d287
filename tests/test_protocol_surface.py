"""The kernel module is a drop-in for the reference's backend protocol
(backend.get_kernels, /root/reference/pkg/src/tetray/backend.py:35-45): the
same module-level names and the same call signatures as the reference's
kernel modules (_kernels.pyx:15-19,271,416,527; pure twin _kernels_py.py).
CPU only: no kernel is called."""

from __future__ import annotations

import importlib.util
import inspect
from pathlib import Path

import pytest

from refpkg import REF_SITE

# the installed reference (oracle/_ref/site, shipped to the GPU box)
REF_PURE = REF_SITE / "tetray" / "_kernels_py.py"
PROTOCOL = {
    "cast_rays": ["mesh", "o32", "d32", "start", "visits_sink"],
    "locate_points": ["mesh", "q", "hints"],
    "shadow_rays": ["mesh", "p", "light", "p_tet", "light_tet", "eps"],
}


def _params(fn):
    return [(p.name, p.default) for p in inspect.signature(fn).parameters.values()]


def test_module_constants_and_functions():
    from paper_2103_02309_b200 import kernels as K

    assert K.BACKEND_NAME == "cuda"
    assert (K.STATUS_MISS, K.STATUS_HIT, K.STATUS_ERROR) == (0, 1, 2)
    for name, params in PROTOCOL.items():
        assert [p for p, _ in _params(getattr(K, name))] == params, name
    assert dict(_params(K.cast_rays))["visits_sink"] is None
    assert dict(_params(K.shadow_rays))["eps"] == 1e-4


@pytest.mark.skipif(not REF_PURE.exists(), reason="oracle/_ref/site missing: run oracle/build_ref.sh")
def test_signatures_equal_the_reference_kernel_module():
    spec = importlib.util.spec_from_file_location("ref_kernels_py", REF_PURE)
    ref = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ref)
    from paper_2103_02309_b200 import kernels as K

    for name in ("STATUS_MISS", "STATUS_HIT", "STATUS_ERROR"):
        assert getattr(K, name) == getattr(ref, name)
    for name in PROTOCOL:
        assert _params(getattr(K, name)) == _params(getattr(ref, name)), name


def test_batch_mirror_signatures():
    """The batch layer mirror takes the reference's arguments (batch.py:39-160)."""
    from paper_2103_02309_b200 import batch

    for name in ("cast_rays", "cast_rays_visits", "locate_points", "shadow_rays"):
        params = [p for p, _ in _params(getattr(batch, name))]
        assert params[0] == "mesh" and "kernels" in params, (name, params)


@pytest.mark.skipif(not REF_PURE.exists(), reason="oracle/_ref/site missing: run oracle/build_ref.sh")
def test_batch_mirror_matches_reference_batch_signatures():
    import subprocess
    import sys

    code = (f"import sys, inspect, json; sys.path.insert(0, {str(REF_SITE)!r}); import tetray.batch as b; "
            "print(json.dumps({n: [p.name for p in inspect.signature(getattr(b, n)).parameters.values()] "
            "for n in ('cast_rays', 'cast_rays_visits', 'locate_points', 'shadow_rays')}))")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    if out.returncode != 0:
        pytest.skip(f"reference batch module not importable here: {out.stderr[-200:]}")
    import json

    from paper_2103_02309_b200 import batch

    ref = json.loads(out.stdout.strip().splitlines()[-1])
    for name, params in ref.items():
        assert [p for p, _ in _params(getattr(batch, name))] == params, name
