#!/bin/bash
# round-2 evidence pass on the final build: smoke, the whole -m gpu suite, the
# default bench line + reference arm, every config's bench line, the ncu launch
# list of the default line, one ncu --set full capture of each config's timed walk.
#   gpurun --timeout 4800 -- 'bash tools/gpu_r02_final.sh r02z'
TAG=${1:-r02z}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref_cfg2.json 2> $OUT/bench_ref_cfg2.err
for c in 1 3 4 5; do
  timeout 1200 python bench.py --config $c --steps 20 --warmup 5 --no-small-batch > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
timeout 900 python bench.py --impl reference --config 4 --steps 3 --warmup 3 > $OUT/bench_ref_cfg4.json 2> $OUT/bench_ref_cfg4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-l2-probe --no-small-batch --no-parity \
    > $OUT/ncu_launch_bench.log 2>&1
NO="--no-e2e --no-cpu-baseline --no-l2-probe --no-parity --no-small-batch"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cast_kernel -s 3 -c 1 -o $OUT/prof_cfg2 \
    python bench.py --steps 1 --warmup 3 $NO --no-secondary --no-cfg4 > $OUT/ncu_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:cast_kernel -s 3 -c 1 -o $OUT/prof_cfg3 \
    python bench.py --config 3 --steps 1 --warmup 3 $NO > $OUT/ncu_cfg3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cast_kernel -s 2 -c 1 -o $OUT/prof_cfg4 \
    python bench.py --config 4 --steps 1 --warmup 3 $NO > $OUT/ncu_cfg4.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:cast_kernel -s 3 -c 1 -o $OUT/prof_cfg5 \
    python bench.py --config 5 --steps 1 --warmup 3 $NO > $OUT/ncu_cfg5.log 2>&1
echo done
