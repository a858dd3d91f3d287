#!/bin/bash
# One gpurun pass: GPU tests, the default bench line, the reference arm,
# the ncu launch list and (optionally) one `ncu --set full` capture of the top kernel.
#   gpurun --timeout 3000 -- 'bash tools/gpu_check.sh r02a [full]'
TAG=${1:-run}
FULL=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --ignore=tests/test_full_size_parity.py --durations=15 \
    > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-l2-probe --no-small-batch --no-parity \
    > $OUT/ncu_launch_bench.log 2>&1
if [ "$FULL" = "full" ]; then
  timeout 3000 python -m pytest tests/test_full_size_parity.py -m gpu -q --durations=5 \
      > $OUT/pytest_full_size.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_full_size.log
fi
echo done
