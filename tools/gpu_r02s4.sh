#!/bin/bash
# A/B: evict-first (ld/st.global.cs) ray I/O in the walk -- stores only / loads + stores
TAG=${1:-r02s4}; OUT=gpurun_out/$TAG; mkdir -p $OUT
L="varlibs/base.so varlibs/cs_st.so varlibs/cs.so"
AB_PRIMARY_SCHED=7 timeout 900 python tools/ab_libs.py $L --configs 2,3 --reps 10 --rounds 3 > $OUT/ab.jsonl 2> $OUT/ab.err
AB_TILES=1 AB_SCHED=6 timeout 900 python tools/ab_libs.py $L --configs 4 --reps 5 --rounds 3 >> $OUT/ab.jsonl 2>> $OUT/ab.err
AB_TILES=1 AB_SCHED=6 AB_SECONDARIES=1 timeout 900 python tools/ab_libs.py $L --configs 2 --reps 10 --rounds 3 >> $OUT/ab.jsonl 2>> $OUT/ab.err
echo done
