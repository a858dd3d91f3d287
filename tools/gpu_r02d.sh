#!/bin/bash
# round-2: config-4 source-level ncu capture, config-1 traffic, host-path wait change
TAG=${1:-r02d}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python tools/small_batch.py > $OUT/small_batch.json 2> $OUT/small_batch.err
timeout 900 python -m pytest tests/test_cuda_parity.py tests/test_cuda_edge_cases.py -m gpu -q -x -k "host or concurrent or small_batch or frozen or shadow or locate" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-secondary --no-cfg4 --no-small-batch --no-cpu-baseline > $OUT/bench_e2e.json 2> $OUT/bench_e2e.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct
timeout 600 ncu --metrics $M --clock-control none -k regex:'sctp_kernel' --csv --log-file $OUT/traffic_cfg1.csv \
    python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-l2-probe --no-small-batch --no-parity > $OUT/traffic_cfg1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cast_kernel -s 2 -c 1 -o $OUT/prof_cfg4 \
    python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-probe --no-parity --no-small-batch > $OUT/ncu_cfg4.log 2>&1
if [ -f $OUT/prof_cfg4.ncu-rep ]; then
  ncu -i $OUT/prof_cfg4.ncu-rep --page source --csv > $OUT/prof_cfg4_source.csv 2>/dev/null
fi
echo done
