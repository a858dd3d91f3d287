#!/bin/bash
# Bench lines for every config on one box: tools/bench_all.sh TAG
TAG=${1:-run}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in 2 1 3 4 5; do
  timeout 1200 python bench.py --config $c > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_cfg2.json 2> $OUT/bench_ref.err
for c in 1 2 3 4 5; do python -c "
import json; d=json.load(open('$OUT/bench_cfg$c.json')); print($c, round(d['value']), 'e2e', round(d['e2e']['value']), 'issue', None if not d.get('roofline_issue') else round(d['roofline_issue']['frac'],3), d['parity'].get('bit_exact', d['parity'].get('traversal_bit_exact')), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
