#!/bin/bash
# round-2: C fast path of the per-tile protocol call -- drop-in tests + renderer-granularity A/B
TAG=${1:-r02w}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_reference_dropin.py tests/test_cuda_parity.py tests/test_cuda_edge_cases.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python tools/small_batch.py > $OUT/small_fast.json 2> $OUT/small.err
TETB200_NO_FASTCALL=1 timeout 600 python tools/small_batch.py > $OUT/small_ctypes.json 2>> $OUT/small.err
timeout 600 python tools/small_batch.py > $OUT/small_fast2.json 2>> $OUT/small.err
echo done
