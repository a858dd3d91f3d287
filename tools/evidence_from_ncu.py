#!/usr/bin/env python
"""Regenerate profiles/pipe_util.json and profiles/traffic.json from one
`ncu --set full` capture of each config's timed walk (tools/gpu_r02_final.sh).

    python tools/evidence_from_ncu.py TAG cfg2/tet20=prof_cfg2.ncu-rep cfg4/tet16=prof_cfg4.ncu-rep ...

Reads the raw page of each report here (ncu -i ... --page raw --csv) and
writes, per key, the walk's pipe and memory utilisation (pipe_util.json, what
bench.py's `ncu_pipes` reports) and its DRAM bytes per launch (traffic.json,
bench.py's `traffic`; ncu flushes the caches before the replayed launch, so
this is the cold-L2 figure).  Keys not given keep their previous entries.
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "us": 1,
        "msecond": 1e3, "ms": 1e3, "second": 1e6}


def raw(path: str) -> dict:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    return [{k: (u[i], v[i]) for i, k in enumerate(h)} for v in rows[2:]]


def num(m: dict, key: str) -> float:
    unit, val = m[key]
    return float(val.replace(",", "")) * UNIT.get(unit, 1)


def main(argv):
    tag, pairs = argv[0], [a.split("=", 1) for a in argv[1:]]
    pp = os.path.join(ROOT, "profiles", "pipe_util.json")
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    pipes = json.load(open(pp)) if os.path.exists(pp) else {}
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    for key, path in pairs:
        ms = raw(path)  # one row per captured launch: a walk in pieces sums its launches
        m = ms[0]
        name = m["Kernel Name"][1] if "Kernel Name" in m else "?"
        pipes[key] = {
            "kernel": name.split("(")[0].replace("void <unnamed>::", ""),
            "alu_pipe_pct": round(num(m, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"), 1),
            "fma_pipe_pct": round(num(m, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"), 1),
            "l1tex_lsu_wavefronts_pct": round(
                num(m, "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"), 1),
            "achieved_occupancy_pct": round(num(m, "sm__warps_active.avg.pct_of_peak_sustained_active"), 1),
            "l1_hit_pct": round(num(m, "l1tex__t_sector_hit_rate.pct"), 1),
            "l2_hit_pct": round(num(m, "lts__t_sector_hit_rate.pct"), 1),
            "issue_active_pct": round(num(m, "smsp__issue_active.avg.pct_of_peak_sustained_active"), 1),
            "duration_us": round(sum(num(x, "gpu__time_duration.sum") for x in ms), 1),
        }
        if len(ms) > 1:
            pipes[key]["launches"] = len(ms)
        wf_key = "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg"
        if all(wf_key in x for x in ms):
            sms = num(m, "device__attribute_multiprocessor_count") if "device__attribute_multiprocessor_count" in m \
                else 148
            # L1 data-pipe wavefronts of the whole walk (launches summed) and
            # the pipe's peak per SM cycle (per-SM average over its utilisation
            # over the SM's elapsed cycles: 1.0 on sm_100)
            pipes[key]["l1tex_lsu_wavefronts_per_launch"] = int(sum(num(x, wf_key) for x in ms) * sms)
            pipes[key]["l1tex_lsu_wavefronts_peak_per_sm_cycle"] = round(
                num(m, wf_key) / (num(m, "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed") / 100)
                / num(m, "sm__cycles_elapsed.avg"), 3)
        traffic[key] = int(round(sum(num(x, "dram__bytes_read.sum") + num(x, "dram__bytes_write.sum")
                                     for x in ms), -5))
        print(key, pipes[key], traffic[key])
    pipes["_source"] = (f"ncu --set full --clock-control none of the timed walk per config (tools/gpu_r02_final.sh, "
                        f"gpurun_out/{tag}/prof_cfg*.ncu-rep), read by tools/evidence_from_ncu.py; % of peak "
                        "sustained (active cycles for the pipes and issue, elapsed for the L1 data pipe)")
    traffic["_source"] = (f"dram__bytes_read.sum + dram__bytes_write.sum of the timed walk's launch in one ncu --set "
                          f"full capture per config (gpurun_out/{tag}; ncu flushes caches before the replayed launch, "
                          "so this is the cold-L2 figure), tools/evidence_from_ncu.py")
    json.dump(dict(sorted(pipes.items())), open(pp, "w"), indent=1)
    json.dump(dict(sorted(traffic.items())), open(tp, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
