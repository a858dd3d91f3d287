#!/bin/bash
# round-2: multi-chunk / ray-prefetch A/B + host-path overhead checks
TAG=${1:-r02c}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python tools/ab_libs.py varlibs/lib_base.so varlibs/lib_k2.so varlibs/lib_k2p.so varlibs/lib_k4p.so varlibs/lib_k8p.so --configs 2,3,5 --reps 10 --rounds 3 > $OUT/ab_chunks.jsonl 2> $OUT/ab_chunks.err
AB_SCHED=1 timeout 900 python tools/ab_libs.py varlibs/lib_base.so varlibs/lib_k2p.so varlibs/lib_k4p.so --configs 4 --reps 5 --rounds 3 > $OUT/ab_chunks_cfg4.jsonl 2>> $OUT/ab_chunks.err
timeout 900 python -m pytest tests/test_cuda_edge_cases.py tests/test_reference_dropin.py tests/test_cuda_parity.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python tools/small_batch.py > $OUT/small_batch.json 2> $OUT/small_batch.err
echo done
