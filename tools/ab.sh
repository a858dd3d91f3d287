#!/bin/bash
# A/B two builds of the library on the same box, interleaved: tools/ab.sh libA libB "configs" reps
A=$1; B=$2; CFGS=${3:-"2 3 4"}; REPS=${4:-2}
for r in $(seq $REPS); do for c in $CFGS; do for lib in $A $B; do
  TETB200_LIB=$PWD/$lib python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', $c, round(d['value']), round(d['kernel_ms']['mean'],4))"
done; done; done
