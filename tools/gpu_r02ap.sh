#!/bin/bash
# round-2: schedule "auto" = sampled longest-first for launches of <= 16 waves -- tests + bench lines
TAG=${1:-r02ap}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_cuda_parity.py tests/test_cuda_edge_cases.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-small-batch > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-small-batch --schedule lane --no-e2e --no-cfg4 --no-secondary --no-cpu-baseline > $OUT/bench_cfg2_lane.json 2> $OUT/bench_cfg2_lane.err
timeout 900 python bench.py --config 3 --steps 20 --warmup 5 --no-small-batch --no-e2e --no-cpu-baseline > $OUT/bench_cfg3.json 2> $OUT/bench_cfg3.err
echo done
