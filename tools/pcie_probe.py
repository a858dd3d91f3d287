#!/usr/bin/env python
"""Floor of the zero-copy end-to-end transport (config 2 sizes: 58 MB of rays
in, 60 MB of hits out per frame).  Builds tools/pcie_probe.cu with nvcc into
/tmp, then times (CUDA events, median of --reps):

  zc_read   kernel reads the input bytes from pinned host memory
  zc_write  kernel writes the output bytes to pinned host memory
  zc_both   both in one kernel (what tb_cast_rays_host does, minus the walk)
  ce_*      the copy engines: H2D, D2H, and both on two streams

    python tools/pcie_probe.py [--in-mb 58.06] [--out-mb 60.13] [--reps 20]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))


def build() -> ctypes.CDLL:
    so = "/tmp/pcie_probe.so"
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode",
                           "arch=compute_100a,code=sm_100a", os.path.join(HERE, "pcie_probe.cu"), "-o", so])
    lib = ctypes.CDLL(so)
    lib.pcie_move.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                              ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    lib.pcie_flagged.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    for f in (lib.pcie_bulk, lib.pcie_bulk_write):
        f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                      ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    return lib


def timed(fn, reps, stream):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return float(np.median(ms))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--in-mb", type=float, default=2_073_600 * 28 / 1e6)
    ap.add_argument("--out-mb", type=float, default=2_073_600 * 29 / 1e6)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--bulk", choices=("off", "device", "host"), default="off",
                    help="TMA bulk-copy probes on device buffers (a self-check) or on pinned host buffers")
    args = ap.parse_args()
    lib = build()
    dev = torch.device("cuda", 0)
    nin = int(args.in_mb * 1e6) // 16 * 16
    nout = int(args.out_mb * 1e6) // 16 * 16
    hin = torch.empty(nin, dtype=torch.uint8).pin_memory()
    hout = torch.empty(nout, dtype=torch.uint8).pin_memory()
    din = torch.empty(nin, dtype=torch.uint8, device=dev)
    dout = torch.empty(nout, dtype=torch.uint8, device=dev)
    sink = torch.zeros(16, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev)
    s2 = torch.cuda.Stream(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    rows = []

    def rec(name, ms, nbytes, **kw):
        row = {"probe": name, "ms": round(ms, 4), "GB_s": round(nbytes / ms / 1e6, 1), **kw}
        rows.append(row)
        print(json.dumps(row), flush=True)

    if args.bulk != "off":
        src, dst = (din, dout) if args.bulk == "device" else (hin, hout)
        g = sms * 2
        for name, fn, nb in (
                ("bulk_read", lambda: lib.pcie_bulk(src.data_ptr(), nin, None, 0, sink.data_ptr(), g, 256, 0,
                                                    s.cuda_stream), nin),
                ("bulk_read_zc_write", lambda: lib.pcie_bulk(src.data_ptr(), nin, dst.data_ptr(), nout,
                                                             sink.data_ptr(), g, 256, 1, s.cuda_stream), nin + nout),
                ("bulk_write", lambda: lib.pcie_bulk_write(None, 0, dst.data_ptr(), nout, sink.data_ptr(), g, 256, 0,
                                                           s.cuda_stream), nout),
                ("bulk_read_bulk_write", lambda: lib.pcie_bulk_write(src.data_ptr(), nin, dst.data_ptr(), nout,
                                                                     sink.data_ptr(), g, 256, 1, s.cuda_stream),
                 nin + nout)):
            rec(name, timed(fn, args.reps, s), nb, memory=args.bulk, grid=g, block=256)
        torch.cuda.synchronize()
        return
    for grid_mul, block in ((1, 256), (4, 256), (8, 256), (16, 256), (8, 128), (8, 512)):
        g = sms * grid_mul
        tag = {"grid": g, "block": block}
        rec("zc_read", timed(lambda: lib.pcie_move(hin.data_ptr(), nin, None, 0, sink.data_ptr(), g, block,
                                                   s.cuda_stream), args.reps, s), nin, **tag)
        rec("zc_write", timed(lambda: lib.pcie_move(None, 0, hout.data_ptr(), nout, sink.data_ptr(), g, block,
                                                    s.cuda_stream), args.reps, s), nout, **tag)
        rec("zc_both", timed(lambda: lib.pcie_move(hin.data_ptr(), nin, hout.data_ptr(), nout, sink.data_ptr(), g,
                                                   block, s.cuda_stream), args.reps, s), nin + nout, **tag)
    rec("ce_h2d", timed(lambda: din.copy_(hin, non_blocking=True), args.reps, s), nin)
    rec("ce_d2h", timed(lambda: hout.copy_(dout, non_blocking=True), args.reps, s), nout)

    def both():
        ev = torch.cuda.Event()
        ev.record(s)
        s2.wait_event(ev)
        din.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        s.wait_event(ev2)

    rec("ce_both", timed(both, args.reps, s), nin + nout)

    # mixed: one direction by the SMs (zero copy), the other by a copy engine
    # on a second stream, concurrently
    g = sms * 8

    def zc_read_ce_d2h():
        ev = torch.cuda.Event()
        ev.record(s)
        s2.wait_event(ev)
        lib.pcie_move(hin.data_ptr(), nin, None, 0, sink.data_ptr(), g, 256, s.cuda_stream)
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        s.wait_event(ev2)

    def ce_h2d_zc_write():
        ev = torch.cuda.Event()
        ev.record(s)
        s2.wait_event(ev)
        lib.pcie_move(None, 0, hout.data_ptr(), nout, sink.data_ptr(), g, 256, s.cuda_stream)
        with torch.cuda.stream(s2):
            din.copy_(hin, non_blocking=True)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        s.wait_event(ev2)

    rec("zc_read_ce_d2h", timed(zc_read_ce_d2h, args.reps, s), nin + nout, grid=g, block=256)

    # copy-engine H2D streamed into one running kernel by per-chunk flags
    nb = 2_073_600 // 128
    # 28 B in / 29 B out per ray; each block's share a whole number of 16 B words
    in_b, out_b = nb * (28 * 128 // 16) * 16, nb * (29 * 128 // 16) * 16
    hin2 = torch.empty(in_b, dtype=torch.uint8).pin_memory()
    hout2 = torch.empty(out_b, dtype=torch.uint8).pin_memory()
    stage = torch.empty(in_b, dtype=torch.uint8, device=dev)
    flag = torch.zeros(4, dtype=torch.int32, device=dev)
    vals = torch.arange(1, 4097, dtype=torch.int32).pin_memory()
    sinkf = torch.zeros(8, dtype=torch.int32, device=dev)
    evf, evj = torch.cuda.Event(), torch.cuda.Event()
    evf.record(s)
    evj.record(s)
    assert (in_b // 16) % nb == 0 and (out_b // 16) % nb == 0
    for chunk_blocks in (256, 512, 1024, 2048, 4096):
        for copies in (1, 3):
            fn = lambda: lib.pcie_flagged(hin2.data_ptr(), stage.data_ptr(), in_b, hout2.data_ptr(), out_b,
                                          flag.data_ptr(), vals.data_ptr(), nb, chunk_blocks, copies,
                                          sinkf.data_ptr(), s.cuda_stream, s2.cuda_stream, evf.cuda_event,
                                          evj.cuda_event)
            ms = timed(fn, args.reps, s)
            torch.cuda.synchronize()
            rec("ce_h2d_flagged_kernel_zc_write", ms, in_b + out_b, chunk_rays=chunk_blocks * 128, copies=copies,
                timeouts=int(sinkf[4].item()))
    rec("ce_h2d_zc_write", timed(ce_h2d_zc_write, args.reps, s), nin + nout, grid=g, block=256)


if __name__ == "__main__":
    main()
