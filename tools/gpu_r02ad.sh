#!/bin/bash
# round-2: rank bits by xor3 / maj3 LOP3 (two levels shallower) -- parity (in-tree lib) + A/B
TAG=${1:-r02ad}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_cuda_parity.py tests/test_cuda_edge_cases.py tests/test_full_size_parity.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
L="varlibs/base4.so varlibs/rkl.so"
AB_TILES=1 timeout 1200 python tools/ab_libs.py $L --configs 2,3,5 --reps 10 --rounds 3 > $OUT/ab.jsonl 2> $OUT/ab.err
AB_TILES=1 AB_SCHED=6 timeout 900 python tools/ab_libs.py $L --configs 4 --reps 5 --rounds 3 >> $OUT/ab.jsonl 2>> $OUT/ab.err
AB_TILES=1 AB_SCHED=6 AB_SECONDARIES=1 timeout 900 python tools/ab_libs.py $L --configs 2 --reps 10 --rounds 3 >> $OUT/ab.jsonl 2>> $OUT/ab.err
echo done
