#!/bin/bash
# round-2 evidence pass: every config's bench line, the reference arm per
# config, DRAM traffic of config 1 / config 5 (tet32), ncu full of configs 3 and 5.
TAG=${1:-r02h}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
for c in 1 3 4 5; do
  timeout 1200 python bench.py --config $c --steps 20 --warmup 5 --no-small-batch > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
for c in 2 4; do
  timeout 900 python bench.py --impl reference --config $c --steps 3 --warmup 3 > $OUT/bench_ref_cfg$c.json 2> $OUT/bench_ref_cfg$c.err
done
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none -k regex:'sctp_kernel' --csv --log-file $OUT/traffic_cfg1.csv \
    python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-l2-probe --no-small-batch --no-parity > $OUT/traffic_cfg1.log 2>&1
timeout 900 ncu --metrics $M --clock-control none -k regex:'cast_kernel' --csv --log-file $OUT/traffic_cfg5.csv \
    python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-l2-probe --no-small-batch --no-parity > $OUT/traffic_cfg5.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:cast_kernel -s 2 -c 1 -o $OUT/prof_cfg3 \
    python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe --no-parity --no-small-batch > $OUT/ncu_cfg3.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:cast_kernel -s 2 -c 1 -o $OUT/prof_cfg5 \
    python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe --no-parity --no-small-batch > $OUT/ncu_cfg5.log 2>&1
echo done
