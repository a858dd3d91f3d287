#!/bin/bash
# round-2: packed f32x2 projection / Algorithm-1 products (FMUL2/FADD2) -- parity + A/B vs scalar
TAG=${1:-r02j}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_cuda_parity.py tests/test_cuda_edge_cases.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
AB_TILES=1 timeout 900 python tools/ab_libs.py varlibs/base.so varlibs/f32x2.so --configs 2,3,5 --reps 10 --rounds 3 > $OUT/ab.jsonl 2> $OUT/ab.err
AB_TILES=1 AB_SCHED=6 timeout 900 python tools/ab_libs.py varlibs/base.so varlibs/f32x2.so --configs 4 --reps 5 --rounds 3 >> $OUT/ab.jsonl 2>> $OUT/ab.err
echo done
