#!/bin/bash
# round-2: epilogue ray reload (registers), occupancy 12 blocks, 8x unrolled walk -- A/B vs base
TAG=${1:-r02k}; OUT=gpurun_out/$TAG; mkdir -p $OUT
L="varlibs/base.so varlibs/reload.so varlibs/reload12.so varlibs/u8.so varlibs/reload_u8.so"
AB_TILES=1 timeout 1200 python tools/ab_libs.py $L --configs 2,3,5 --reps 10 --rounds 3 > $OUT/ab.jsonl 2> $OUT/ab.err
AB_TILES=1 AB_SCHED=6 timeout 900 python tools/ab_libs.py $L --configs 4 --reps 5 --rounds 3 >> $OUT/ab.jsonl 2>> $OUT/ab.err
echo done
