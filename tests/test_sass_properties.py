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


def _walks(pattern):
    import sass_steps as S

    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    out = {}
    for name, ins in S.functions(sass):
        m = re.search(pattern, name)
        if m:
            ls = S.walk_loops(ins)
            out[int(m.group(1))] = [[re.sub(r"^@!?U?P\w+\s+", "", s) for _, s in lp] for lp in (ls[0], ls[-1])]
    return out


@pytest.fixture(scope="module")
def walks():
    """cast_kernel<L, validated, device rays, no scatter, no gather>: its
    single-step walk loop and its 8x unrolled one (the hot loop)."""
    return _walks(r"11cast_kernelILi(\d+)ELb0ELb0ELb0ELb0E")


@pytest.fixture(scope="module")
def loops(walks):
    return {k: v[0] for k, v in walks.items()}


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


def _written(body):
    """Registers written inside a loop body (first operand of each instruction)."""
    out = set()
    for o in body:
        parts = o.split(None, 1)
        if len(parts) == 2:
            m = re.match(r"(R\d+)", parts[1])
            if m:
                out.add(m.group(1))
    return out


@pytest.mark.parametrize("layout", (16, 20, 32, 80))
def test_no_fma_contraction_in_the_walk(loops, layout):
    """the reference is built with -ffp-contract=off; a contracted
    multiply-add in the step would change results on tie-heavy meshes.  The
    one FFMA per step is the projection's y1 + sgn * q.z, whose factor sgn is
    the ray's +-1 (an exact product, so one rounding either way): it must take
    a loop-invariant register as a factor, and no packed FFMA2 may appear."""
    body = loops[layout]
    assert not [o for o in body if o.startswith(("FFMA2", "DFMA", "HFMA"))]
    ffma = [o for o in body if o.startswith("FFMA")]
    assert len(ffma) == 1, ffma
    regs = re.findall(r"-?(R\d+)", ffma[0].split(None, 1)[1])
    invariant = [r for r in regs[1:3] if r not in _written(body)]
    assert invariant, (ffma[0], "no loop-invariant factor")


@pytest.mark.parametrize("layout", (16, 20, 32))
def test_flops_per_step(loops, layout):
    """Acceptance 6 counts 7 mul + 5 add per step for the lazy Python
    Algorithm 1; the kernel evaluates all three face products eagerly
    (branch-free, 2 more muls) and multiplies by sgn (1 mul): 10 multiplies
    and 5 adds, here as packed pairs (FMUL2 / FADD2 = 2 each) and the one
    sign FFMA (1 + 1), no divides, no fp64."""
    body = loops[layout]
    ops = [o.split()[0] for o in body]
    mul = ops.count("FMUL") + 2 * ops.count("FMUL2") + ops.count("FFMA")
    add = ops.count("FADD") + 2 * ops.count("FADD2") + ops.count("FFMA")
    assert mul == 10 and add == 5, (mul, add)
    assert not [o for o in body if o.startswith(("MUFU", "DMUL", "DADD", "FCHK"))]


@pytest.mark.parametrize("layout", (16, 20, 80))
def test_no_local_memory_in_the_walk(walks, layout):
    """The 10-blocks-per-SM walks (48 registers) keep the whole step in
    registers, in the single-step and in the unrolled loop."""
    for body in walks[layout]:
        assert not [o for o in body if o.startswith(("LDL", "STL"))]


def test_latency_bound_walks_spill_at_most_two_loads_per_step(walks):
    """Tet32 and the direction-binned (gather) walks run 12 blocks per SM (40
    registers, cast_min_blocks): r02 A/B measured that residency worth more
    than the few reloads it costs (config 5 +5 %, config 4 +2.6 %).  Bound it:
    no spill stores in the unrolled loop, at most two local reloads per step."""
    gathered = _walks(r"11cast_kernelILi(\d+)ELb0ELb0ELb1ELb1E")
    for layout, (one, big) in [(32, walks[32])] + sorted(gathered.items()):
        steps = sum(o.startswith("LDG") for o in big) // max(1, sum(o.startswith("LDG") for o in one))
        assert not [o for o in big if o.startswith("STL")], layout
        assert sum(o.startswith("LDL") for o in big) <= 2 * steps, layout
