#!/bin/bash
# A/B round 2: evict-first ray I/O, hybrid (stores always; loads only for in-place walks) vs base
TAG=${1:-r02s5}; OUT=gpurun_out/$TAG; mkdir -p $OUT
L="varlibs/base.so varlibs/cs_hyb.so varlibs/cs.so varlibs/cs_st.so"
AB_PRIMARY_SCHED=7 timeout 900 python tools/ab_libs.py $L --configs 2,3 --reps 10 --rounds 5 > $OUT/ab.jsonl 2> $OUT/ab.err
AB_TILES=1 AB_SCHED=6 timeout 900 python tools/ab_libs.py $L --configs 4 --reps 5 --rounds 5 >> $OUT/ab.jsonl 2>> $OUT/ab.err
AB_TILES=1 AB_SCHED=6 AB_SECONDARIES=1 timeout 900 python tools/ab_libs.py $L --configs 2 --reps 10 --rounds 5 >> $OUT/ab.jsonl 2>> $OUT/ab.err
timeout 900 python tools/ab_libs.py varlibs/base.so varlibs/cs_hyb.so --configs 5 --reps 3 --rounds 3 >> $OUT/ab.jsonl 2>> $OUT/ab.err
echo done
