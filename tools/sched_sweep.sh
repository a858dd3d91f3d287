#!/bin/bash
# Ray-schedule sweep on one box:
#   tools/sched_sweep.sh OUT "configs" "sched:round[:compact_below_pct] ..." reps
OUT=${1:-gpurun_out/sched}; CFGS=${2:-"2 3 4"}; SCHEDS=${3:-"1:16 3:32 5:32:70"}; REPS=${4:-2}
mkdir -p $(dirname $OUT)
for r in $(seq $REPS); do for c in $CFGS; do for sr in $SCHEDS; do
  IFS=: read s k pct <<< "$sr"; pct=${pct:-70}
  TETB200_SCHED=$s TETB200_ROUND=$k TETB200_COMPACT_BELOW=$pct timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(dict(cfg=$c, sched=$s, round=$k, below=$pct, value=round(d['value'],1), kernel_ms=round(d['kernel_ms']['mean'],4), parity=d.get('parity'))))" >> $OUT.jsonl
done; done; done
