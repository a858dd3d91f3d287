#!/usr/bin/env python
"""Per-step SASS instruction mix of the traversal kernels' walk loops.

    python tools/sass_steps.py [libtetb200.so] [-o profiles/sass_step_counts.json]

Finds, in each cast/compact kernel, the innermost backward branch that
contains the per-step loads (the walk loop: record load -> xor -> point
load -> Algorithm 1 -> next_ref), and counts its instructions by the pipe
that executes them on sm_100a.  The counts feed bench.py's ALU-pipe
roofline (ALU ops per ray-step) and document every step-level experiment.

Pipe classes (sm_100a, following ncu's pipe names): ALU = integer/logic
compares, selects, shifts, min/max, LEA; FMA = FP32 mul/add/fma and IMAD*
(fmaheavy); LSU = global/shared/local memory; CBU = branches/barriers;
other = everything else.  VIADD is counted under ALU (conservative: ncu
shows it on neither FMA counter in r01 captures).
"""

from __future__ import annotations

import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

ALU = ("ISETP", "FSETP", "DSETP", "LOP3", "LOP", "SEL", "FSEL", "PLOP3", "IMNMX", "VIMNMX", "FMNMX", "LEA",
       "SHF", "PRMT", "IADD3", "VIADD", "FLO", "POPC", "BREV", "IABS", "P2R", "R2P", "ISCADD", "SGXT", "BMSK")
FMA = ("FMUL", "FADD", "FFMA", "IMAD", "IMUL", "FMNMX3", "FMUL2", "FADD2", "FFMA2")
LSU = ("LDG", "STG", "LDS", "STS", "LDL", "STL", "LD", "ST", "ATOM", "ATOMS", "RED", "LDC")
CBU = ("BRA", "EXIT", "BSSY", "BSYNC", "BAR", "WARPSYNC", "RET", "CALL", "BREAK", "JMP")


def classify(op: str) -> str:
    base = op.split(".")[0]
    if base in FMA:
        return "fma"
    if base in ALU:
        return "alu"
    if base in LSU:
        return "lsu"
    if base in CBU:
        return "cbu"
    return "other"


def functions(sass: str):
    for part in re.split(r"\n\s+Function : ", sass)[1:]:
        name = part.split("\n", 1)[0].strip()
        ins = []
        for line in part.split("\n"):
            m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        yield name, ins


def walk_loops(ins):
    """Backward-branch loop bodies holding the per-step loads (>= 2 LDG and
    >= 3 FSETP), smallest first: the single-step walk loop, then unrolled
    copies (k steps = k times its loads)."""
    addr = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, s) in enumerate(ins):
        m = re.search(r"BRA .*?0x([0-9a-f]+)", s)
        if not m:
            continue
        t = int(m.group(1), 16)
        if t >= a or t not in addr:
            continue
        body = ins[addr[t]:i + 1]
        ops = [re.sub(r"^@!?U?P\w+\s+", "", x) for _, x in body]
        if sum(o.startswith("LDG") for o in ops) >= 2 and sum(o.startswith("FSETP") for o in ops) >= 3:
            loops.append(body)
    return sorted(loops, key=len)


def mix_of(body, steps=1):
    mix = {"total": 0, "alu": 0, "fma": 0, "lsu": 0, "cbu": 0, "other": 0}
    for _, s in body:
        op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0]
        mix[classify(op)] += 1
        mix["total"] += 1
    return {k: round(v / steps, 2) for k, v in mix.items()}


def main(argv):
    lib = ROOT / "paper_2103_02309_b200" / "libtetb200.so"
    out = None
    args = list(argv)
    if "-o" in args:
        k = args.index("-o")
        out = Path(args[k + 1])
        del args[k:k + 2]
    if args:
        lib = Path(args[0])
    sass = subprocess.run(["cuobjdump", "-sass", str(lib)], capture_output=True, text=True, check=True).stdout
    res = {}
    for name, ins in functions(sass):
        m = re.search(r"(cast_kernel|cast_compact_kernel|sctp_kernel|shadow_kernel)ILi(\d+)E(?:Li\d+E)?(Lb[01]E)?"
                      r"((?:Lb[01]E)*)", name)
        if not m:
            continue
        if "Lb1E" in m.group(4):  # host-ray / scatter / gather variants: the device-ray kernel is the reference
            continue
        key = f"{m.group(1)}<{m.group(2)}{'' if not m.group(3) else (', clamp' if m.group(3) == 'Lb1E' else ', validated')}>"
        if key in res:
            continue
        loops = walk_loops(ins)
        if not loops:
            continue
        one = loops[0]
        n_ld = sum(re.sub(r"^@!?U?P\w+\s+", "", x).startswith("LDG") for _, x in one)
        # exactness guard: the walk's fp32 arithmetic is mul/add with explicit
        # rounding; a contracted FFMA / FFMA2 in a walk step breaks bit-exactness.
        # Checked on the single-step loop of every cast walk and the unrolled
        # loop of cast_kernel (the shadow / ScTP steps and the compact kernels'
        # refill hold IEEE divisions, whose expansions use FFMA legitimately).
        # The one intended FFMA per step is project_perm's y1 + sgn * q.z (an
        # exact product): a step with more, or any FFMA2, was contracted.
        checked = [one] + ([loops[-1]] if key.startswith("cast_kernel") else [])
        for body in checked:
            steps = max(1, sum(re.sub(r"^@!?U?P\w+\s+", "", x).startswith("LDG") for _, x in body) //
                        max(1, sum(re.sub(r"^@!?U?P\w+\s+", "", x).startswith("LDG") for _, x in one)))
            ffma = [x for _, x in body if re.search(r"\bFFMA\b", x)]
            ffma2 = [x for _, x in body if re.search(r"\bFFMA2\b", x)]
            if key.startswith("cast") and (ffma2 or len(ffma) > steps):
                raise SystemExit(f"{key}: contracted FFMA in the walk loop: {(ffma2 + ffma)[:3]}")
        entry = {"single_step": mix_of(one)}
        big = loops[-1]
        k = sum(re.sub(r"^@!?U?P\w+\s+", "", x).startswith("LDG") for _, x in big) // max(n_ld, 1)
        if k > 1 and key.startswith("cast_kernel"):
            entry[f"unrolled_x{k}_per_step"] = mix_of(big, k)
        res[key] = entry
    text = json.dumps({"_source": f"cuobjdump -sass {lib.name}; tools/sass_steps.py (walk-loop body per step)",
                       **dict(sorted(res.items()))}, indent=1)
    if out:
        out.write_text(text + "\n")
    print(text)


if __name__ == "__main__":
    main(sys.argv[1:])
