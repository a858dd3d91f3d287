#!/bin/bash
# round-2 closing evidence on HEAD: compute-sanitizer over the split schedules
# (sampled head/tail on two streams, binned in two pieces), every config's bench
# line, the ncu launch list of the default line, ncu --set full of configs 2 and 4.
TAG=${1:-r02s3}; OUT=gpurun_out/$TAG; mkdir -p $OUT
SEL="sampled or binned or block_order or schedules_identical_results or trace_schedule_argument"
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_cuda_parity.py -m gpu -q -p no:cacheprovider \
   -k "$SEL" > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_cuda_parity.py -m gpu -q -p no:cacheprovider \
   -k "binned_many_segments or (sampled_schedule_matches_lane and tet20)" > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
for c in 1 3 5; do
  timeout 1200 python bench.py --config $c --steps 20 --warmup 5 --no-small-batch > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-l2-probe --no-small-batch --no-parity \
    > $OUT/ncu_launch_bench.log 2>&1
NO="--no-e2e --no-cpu-baseline --no-l2-probe --no-parity --no-small-batch"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cast_kernel -s 3 -c 1 -o $OUT/prof_cfg2 \
    python bench.py --steps 1 --warmup 3 $NO --no-secondary --no-cfg4 > $OUT/ncu_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cast_kernel -s 2 -c 2 -o $OUT/prof_cfg4 \
    python bench.py --config 4 --steps 1 --warmup 3 $NO > $OUT/ncu_cfg4.log 2>&1
echo done
