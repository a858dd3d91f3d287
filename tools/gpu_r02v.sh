#!/bin/bash
# round-2: default bench line (config 2) on the final build + its reference arm
TAG=${1:-r02v}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref_cfg2.json 2> $OUT/bench_ref_cfg2.err
echo done
