"""pytest plugin: run the reference's OWN test suite with the CUDA module as
its compiled backend.

    PYTHONPATH=oracle/_ref/site:tests:. python -m pytest -p ref_suite_plugin oracle/_ref/pkg/tests

The reference selects kernels through ``tetray.backend``
(/root/reference/pkg/src/tetray/backend.py:20-45): ``_compiled`` is what
``get_kernels("compiled")`` returns and ``_active`` what every
``batch.*`` / ``render`` call uses when no ``kernels=`` is passed
(batch.py:48,91,142,155; render.py:467).  This plugin points both at
``paper_2103_02309_b200.kernels`` before collection -- the registration a
maintainer would add -- so, unmodified:

* test_kernels.py compares the reference's pure-python kernels with the
  CUDA module (its "compiled vs pure" parity suite, bit-exact);
* test_acceptance.py, test_render.py, test_bench.py, ... run every batch
  and render call on the GPU (the renderer's 16x16-tile thread pool calls
  ``cast_rays`` concurrently on one mesh, render.py:538-541).

Test infrastructure only (used by tests/test_reference_dropin.py).
"""

from __future__ import annotations

import os


def pytest_configure(config):
    import tetray
    from tetray import backend

    import paper_2103_02309_b200.kernels as cuda

    site = os.environ.get("TETB200_REF_SITE")
    if site and not os.path.abspath(tetray.__file__).startswith(os.path.abspath(site)):
        raise RuntimeError(f"tetray imported from {tetray.__file__}, expected under {site}")
    backend._compiled = cuda
    backend._active = cuda
    config.addinivalue_line("markers", "cuda_backend: reference suite running on paper_2103_02309_b200.kernels")


def pytest_report_header(config):
    from tetray import backend

    k = backend.get_kernels()
    return f"tetray backend swapped: active = {k.__name__} (BACKEND_NAME={getattr(k, 'BACKEND_NAME', '?')})"
