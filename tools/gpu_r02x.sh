#!/bin/bash
# round-2: Tet16 exit reference as one 3-input LOP3 -- parity + A/B; compute-sanitizer over the round-2 paths
TAG=${1:-r02x}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_cuda_parity.py tests/test_cuda_edge_cases.py tests/test_full_size_parity.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
L="varlibs/rk_alu.so varlibs/lop3.so"
AB_TILES=1 timeout 900 python tools/ab_libs.py $L --configs 3 --reps 10 --rounds 3 > $OUT/ab.jsonl 2> $OUT/ab.err
AB_TILES=1 AB_SCHED=6 timeout 900 python tools/ab_libs.py $L --configs 4 --reps 5 --rounds 3 >> $OUT/ab.jsonl 2>> $OUT/ab.err
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_cuda_parity.py tests/test_cuda_edge_cases.py -m gpu -q -p no:cacheprovider \
   -k "fastcall or golden or binned or host or upload_validation or schedules_identical_results" > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_cuda_parity.py -m gpu -q -p no:cacheprovider -k "binned_many_segments or fastcall" > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
echo done
