#!/bin/bash
# round-2: TetMesh-32A (neighbour-apex records) parity + layout A/B
TAG=${1:-r02e}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_cuda_parity.py tests/test_cuda_edge_cases.py -m gpu -q -x -k "tet32a or config2_full or schedules" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python tools/sched_ab.py --configs 2,3,5 --schedules lane --layouts tet20,tet16,tet32,tet32a --tiles --reps 10 > $OUT/layouts.jsonl 2> $OUT/layouts.err
timeout 900 python tools/sched_ab.py --configs 4 --schedules binned,lane --layouts tet16,tet20,tet32,tet32a --tiles --reps 5 > $OUT/layouts_cfg4.jsonl 2>> $OUT/layouts.err
echo done
