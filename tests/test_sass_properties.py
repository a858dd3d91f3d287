"""Static checks of the built sm_100a walk loops (cuobjdump, no GPU needed) --
the machine-code analogue of the reference's acceptance criteria 6 and 7
(test_acceptance.py:220-286: a bounded flop count per step, one point fetch
per step) plus the exactness rule of SURVEY A.1 (no FMA contraction)."""

from __future__ import annotations

import re
import shutil
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, str(ROOT / "tools"))

pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not installed")

LIB = ROOT / "paper_2103_02309_b200" / "libtetb200.so"


@pytest.fixture(scope="module")
def loops():
    import sass_steps as S

    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    out = {}
    for name, ins in S.functions(sass):
        m = re.search(r"11cast_kernelILi(\d+)ELb0ELb0", name)  # device-ray path, validated mesh
        if m:
            ls = S.walk_loops(ins)
            out[int(m.group(1))] = [re.sub(r"^@!?U?P\w+\s+", "", s) for _, s in ls[0]]
    return out


def test_every_layout_has_a_walk_loop(loops):
    assert set(loops) == {16, 20, 32, 80}


@pytest.mark.parametrize("layout,rec_loads", [(16, ["LDG.E.128"]), (20, ["LDG.E", "LDG.E.128"]),
                                              (32, ["LDG.E.128", "LDG.E.128"])])
def test_one_record_and_one_point_fetch_per_step(loops, layout, rec_loads):
    """Acceptance 7 (one point fetch per step): the step loads the record
    (Tet16 one 16 B, Tet20 4 B + 16 B, Tet32 2 x 16 B) and exactly one 16 B
    point copy -- nothing else."""
    body = loops[layout]
    loads = sorted(o.split()[0].replace(".CONSTANT", "") for o in body if o.startswith("LDG"))
    assert loads == sorted(rec_loads + ["LDG.E.128"]), loads


@pytest.mark.parametrize("layout", (16, 20, 32, 80))
def test_no_fma_contraction_in_the_walk(loops, layout):
    """the reference is built with -ffp-contract=off; an FFMA in
    the step would change results on tie-heavy meshes."""
    assert not [o for o in loops[layout] if o.startswith(("FFMA", "DFMA", "HFMA"))]


@pytest.mark.parametrize("layout", (16, 20, 32))
def test_flops_per_step(loops, layout):
    """Acceptance 6 counts 7 mul + 5 add per step for the lazy Python
    Algorithm 1; the kernel evaluates all three face products eagerly
    (branch-free, 2 more FMUL) and multiplies by sgn (1 FMUL): 10 FMUL +
    5 FADD, no divides, no fp64."""
    body = loops[layout]
    fmul = sum(o.startswith("FMUL") for o in body)
    fadd = sum(o.startswith("FADD") for o in body)
    assert fmul == 10 and fadd == 5, (fmul, fadd)
    assert not [o for o in body if o.startswith(("MUFU", "DMUL", "DADD", "FCHK"))]


@pytest.mark.parametrize("layout", (16, 20, 32, 80))
def test_no_local_memory_in_the_walk(loops, layout):
    assert not [o for o in loops[layout] if o.startswith(("LDL", "STL"))]
