#!/bin/bash
# round-2: schedule 7 "sampled" (capped one-ray-per-block pre-pass -> longest-first block order) -- tests + A/B
TAG=${1:-r02ao}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_cuda_parity.py -m gpu -q -x -k "sampled or schedule or block_order" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python tools/sched_ab.py --configs 2,3,5 --schedules lane,sampled --tiles --reps 20 > $OUT/sched.jsonl 2> $OUT/sched.err
for cap in 24 48; do TETB200_PROBE_CAP=$cap timeout 600 python tools/sched_ab.py --configs 2,3 --schedules lane,sampled --tiles --reps 20 | sed "s/^{/{\"cap\": $cap, /" >> $OUT/sched.jsonl 2>> $OUT/sched.err; done
echo done
