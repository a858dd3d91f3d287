#!/bin/bash
# round-2: residency of the binned Tet20 walk (10 vs 12 blocks per SM)
TAG=${1:-r02t}; OUT=gpurun_out/$TAG; mkdir -p $OUT
L="varlibs/g20_12.so varlibs/g20_10.so"
AB_TILES=1 AB_SCHED=6 AB_SECONDARIES=1 timeout 900 python tools/ab_libs.py $L --configs 2 --reps 10 --rounds 3 > $OUT/ab.jsonl 2> $OUT/ab.err
AB_TILES=1 AB_SCHED=6 AB_LAYOUT=tet20 timeout 900 python tools/ab_libs.py $L --configs 4 --reps 5 --rounds 3 >> $OUT/ab.jsonl 2>> $OUT/ab.err
echo done
