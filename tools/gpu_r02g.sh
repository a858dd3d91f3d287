#!/bin/bash
TAG=${1:-r02g}; OUT=gpurun_out/$TAG; mkdir -p $OUT
AB_TILES=1 AB_SCHED=6 timeout 900 python tools/ab_libs.py varlibs/lib_base.so varlibs/lib_single.so --configs 4 --reps 5 --rounds 3 > $OUT/ab_single_cfg4.jsonl 2> $OUT/ab.err
AB_TILES=1 timeout 900 python tools/ab_libs.py varlibs/lib_base.so varlibs/lib_single.so --configs 2,3,5 --reps 10 --rounds 3 > $OUT/ab_single.jsonl 2>> $OUT/ab.err
echo done
