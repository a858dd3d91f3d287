#!/bin/bash
# round-2 compute-sanitizer pass over the host paths / schedules changed in r02
TAG=${1:-r02i}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_cuda_parity.py tests/test_cuda_edge_cases.py -m gpu -q -p no:cacheprovider \
   -k "concurrent or host or small_batch or frozen or upload_validation or schedules_identical_results or binned or config2_full" > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_multigpu_p2p.py -m gpu -q -p no:cacheprovider -k "trace_multi" > $OUT/memcheck_multi.log 2>&1; echo "rc=$?" >> $OUT/memcheck_multi.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_cuda_parity.py -m gpu -q -p no:cacheprovider -k "binned_many_segments or (schedules_identical_results and compact and tet20)" > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_cuda_parity.py -m gpu -q -p no:cacheprovider -k "binned_many_segments or (schedules_identical_results and compact and tet20)" > $OUT/synccheck.log 2>&1; echo "rc=$?" >> $OUT/synccheck.log
echo done
