"""bench.py's driver contract on CPU: the reference arm (the reference's own
compiled kernels on the host cores) prints one JSON line with the keys the
driver reads.  The GPU arm's line is exercised by the round-end bench run."""

from __future__ import annotations

import json
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.timeout(600)
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "2",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["tets_visited_per_ray"]["mean"] == pytest.approx(4.49, abs=0.01)
    # the reference arm runs the reference only: its own compiled kernels, not this repo's CUDA library
    assert not any("libtetb200" in so for so in d["native_so_loaded"]), d["native_so_loaded"]
    assert any(so.startswith("oracle/_ref/") for so in d["native_so_loaded"])
    # both arms describe the workload with the same config dict
    sys.path.insert(0, str(ROOT))
    import bench

    assert d["config"] == bench.config_dict(bench.CONFIGS[1], 1)


@pytest.mark.timeout(300)
def test_gpus_flag_launches_ranks_and_fails_loudly_without_gpus():
    """--gpus 2 outside torchrun relaunches under torch.distributed.run; with
    fewer visible GPUs than ranks every rank exits with the reason."""
    import torch

    if torch.cuda.device_count() >= 2:
        pytest.skip("enough GPUs here: the multi-GPU bench is exercised on the box")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode != 0
    assert "torch.distributed.run" in out.stderr and "visible GPU" in out.stderr, out.stderr[-2000:]


def test_bench_rejects_short_warmup():
    out = subprocess.run([sys.executable, "bench.py", "--warmup", "2"], cwd=ROOT, capture_output=True, text=True,
                         timeout=120)
    assert out.returncode != 0 and "warmup" in out.stderr


def test_roofline_is_the_binding_pipe_of_the_committed_sass():
    """`roofline` = achieved walk steps against max(issue, 2 x ALU-pipe SASS)
    per warp-step from profiles/sass_step_counts.json (regenerated per build);
    the ALU pipe binds for every 2-D walk layout."""
    sys.path.insert(0, str(ROOT))
    import bench

    for layout in ("tet16", "tet20", "tet32"):
        r = bench.issue_roof(layout, "lane", walk_steps=1e9, kern_s=1e-3, clk_mhz=1965.0, sms=148)
        assert r["bound"] == "alu_pipe", (layout, r)
        assert r["cycles_per_warp_step"] == 2 * r["alu_per_step"] > r["sass_per_step"]
        peak = 148 * 4 * 1965e6 * 32 / r["cycles_per_warp_step"]
        assert r["frac"] == pytest.approx(1e12 / peak)
        assert r["issue_frac"] < r["frac"]
    assert bench.issue_roof("tet20", "lane", 1e9, 1e-3, None, 148) is None  # no clock sample: no roof


def test_incoherent_walk_reports_the_l1_data_pipe_when_it_binds():
    """Config 4's binned walk: the L1 data-pipe roof (ncu wavefronts per
    launch over the live time, peak = SMs x 1 wavefront per SM cycle x clock)
    binds over the ALU-pipe roof, which rides along; walks without a wavefront
    count keep the ALU-pipe roof."""
    sys.path.insert(0, str(ROOT))
    import bench

    wf = bench.pipes_of("cfg4/tet16")["l1tex_lsu_wavefronts_per_launch"]
    l1 = bench.l1_pipe_roof("cfg4/tet16", kern_s=4.62e-3, clk_mhz=1965.0, sms=148)
    assert l1["frac"] == pytest.approx(wf / 4.62e-3 / (148 * 1.0 * 1965e6), rel=1e-3)
    alu = bench.issue_roof("tet16", "binned", walk_steps=16_777_216 * 64.0, kern_s=4.62e-3, clk_mhz=1965.0, sms=148)
    r = bench.binding_roof(alu, l1)
    assert r["bound"] == "l1_data_pipe" and r["roofline_alu_pipe"]["bound"] == "alu_pipe"
    assert 0.5 < r["frac"] < 1.0 and r["frac"] > alu["frac"]
    assert bench.l1_pipe_roof("cfg2/tet20", 1.7e-4, 1965.0, 148) is None
    assert bench.binding_roof(alu, None) is alu


def test_profiles_carry_traffic_and_pipes_for_every_bench_config():
    sys.path.insert(0, str(ROOT))
    import bench

    for c, cfg in bench.CONFIGS.items():
        assert bench.traffic_of(f"cfg{c}/{cfg['layout']}"), c
    for key in ("cfg2/tet20", "cfg3/tet16", "cfg4/tet16", "cfg5/tet32"):
        p = bench.pipes_of(key)
        assert p and 0 < p["alu_pipe_pct"] <= 100 and 0 < p["l1tex_lsu_wavefronts_pct"] <= 100, key


def test_hits_mismatch_holds_t_to_the_contract_only_off_the_pinned_numpy(monkeypatch):
    import numpy as np

    import refpkg

    a = [np.arange(4, dtype=np.int32)] * 5 + [np.array([1.0, np.inf, 2.0, 3.0])] + [np.arange(4, dtype=np.int32)]
    b = [x.copy() for x in a]
    b[5][2] = 2.0 * (1 + 4e-6)  # 4e-6 relative: an einsum-order ulp drift is far smaller
    assert refpkg.hits_mismatch(a, b)["t"] == 1  # pinned numpy: bit-exact required
    monkeypatch.setattr(refpkg, "EINSUM_PINNED_NUMPY", "0.0.")
    assert refpkg.hits_mismatch(a, b)["t"] == 0  # other numpy: within 1e-5 relative
    b[5][3] = 3.1
    assert refpkg.hits_mismatch(a, b)["t"] == 1
    b[1] = b[1] + 1
    assert refpkg.hits_mismatch(a, b)["cf"] == 4  # every other array stays bit-exact
