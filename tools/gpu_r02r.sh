#!/bin/bash
# round-2: TMA bulk copies to / from pinned host memory (zero-copy transport probe).
# Device buffers first (self-check of the kernels), then host buffers, each in its own process.
TAG=${1:-r02r}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python tools/pcie_probe.py --bulk device --reps 10 > $OUT/bulk_device.jsonl 2> $OUT/bulk_device.err; echo "rc=$?" >> $OUT/bulk_device.err
timeout 300 python tools/pcie_probe.py --bulk host --reps 10 > $OUT/bulk_host.jsonl 2> $OUT/bulk_host.err; echo "rc=$?" >> $OUT/bulk_host.err
timeout 300 python tools/pcie_probe.py --reps 10 > $OUT/zc.jsonl 2> $OUT/zc.err
nvidia-smi -q | grep -i -A3 "xid\|retired" > $OUT/smi_after.txt 2>&1
echo done
