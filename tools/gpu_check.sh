#!/bin/bash
# One gpurun pass: GPU tests, the default bench line, the reference arm,
# the ncu launch list and one `ncu --set full` capture of the top kernel.
#   gpurun --timeout 1500 -- 'bash tools/gpu_check.sh r01b'
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-l2-probe > $OUT/ncu_launch_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg4.csv \
    python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-l2-probe --no-parity \
    > $OUT/ncu_launch_bench_cfg4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cast_kernel -s 3 -c 1 -o $OUT/prof_cast \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe > $OUT/ncu_full.log 2>&1
if [ -f $OUT/prof_cast.ncu-rep ]; then
  python tools/ncu_summary.py $OUT/prof_cast.ncu-rep > $OUT/prof_cast_summary.txt 2>&1
  ncu -i $OUT/prof_cast.ncu-rep --page source --csv > $OUT/prof_cast_source.csv 2>/dev/null
fi
echo done
