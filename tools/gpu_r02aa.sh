#!/bin/bash
# round-2: spatial sub-key inside the direction cells of the segmented binning (config 4, tile-ordered rays)
TAG=${1:-r02aa}; OUT=gpurun_out/$TAG; mkdir -p $OUT
BIN_TILES=1 BIN_KEYS="seg,cube4;seg,cube4,start>>6;seg,cube4,start>>8;seg,cube4,start>>10;seg,cube4,start>>12;seg,cube4,start>>14;cube4,start>>8" \
  timeout 1200 python tools/bin_probe.py --reps 5 > $OUT/bin_probe.jsonl 2> $OUT/bin_probe.err
echo done
