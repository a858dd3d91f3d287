#!/bin/bash
# round-2 measurement pass: default bench line, schedule A/B, per-config
# bench lines, DRAM traffic per config (ncu metrics), one full ncu capture.
#   gpurun --timeout 3600 -- 'bash tools/gpu_r02b.sh r02b'
TAG=${1:-r02b}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python tools/sched_ab.py --configs 2,3,5 --schedules lane,dynamic > $OUT/sched_ab.jsonl 2> $OUT/sched_ab.err
timeout 900 python tools/sched_ab.py --configs 4 --schedules binned,lane,dynamic --reps 10 > $OUT/sched_ab_cfg4.jsonl 2>> $OUT/sched_ab.err
for c in 1 3 4 5; do
  timeout 1200 python bench.py --config $c --steps 20 --warmup 5 --no-small-batch > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct
for c in 2 3 4 5; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:'cast_kernel|bin_' --csv --log-file $OUT/traffic_cfg$c.csv \
      python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-l2-probe --no-small-batch \
      --no-parity --no-secondary --no-cfg4 > $OUT/traffic_cfg$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cast_kernel -s 3 -c 1 -o $OUT/prof_cast \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe --no-small-batch --no-secondary \
    --no-cfg4 --no-parity > $OUT/ncu_full.log 2>&1
echo done
