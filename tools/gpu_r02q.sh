#!/bin/bash
# round-2: TMA bulk L2 prefetch of the rays one residency wave ahead -- A/B
TAG=${1:-r02q}; OUT=gpurun_out/$TAG; mkdir -p $OUT
L="varlibs/base2.so varlibs/pf740.so varlibs/pf1480.so varlibs/pf2960.so"
AB_TILES=1 timeout 1200 python tools/ab_libs.py $L --configs 2,3,5 --reps 10 --rounds 3 > $OUT/ab.jsonl 2> $OUT/ab.err
echo done
