#!/bin/bash
# HEAD with evict-first ray I/O: smoke, the whole -m gpu suite, every config's bench line, reference arm
TAG=${1:-r02s6}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref_cfg2.json 2> $OUT/bench_ref_cfg2.err
for c in 1 3 4 5; do
  timeout 1200 python bench.py --config $c --steps 20 --warmup 5 --no-small-batch > $OUT/bench_cfg$c.json 2> $OUT/bench_cfg$c.err
done
echo done
