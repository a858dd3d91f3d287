#!/bin/bash
# closing confirmation on the final HEAD: smoke, whole -m gpu suite, default line, reference arm, config-4 line
TAG=${1:-r02s12}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref_cfg2.json 2> $OUT/bench_ref_cfg2.err
timeout 1200 python bench.py --config 4 --steps 20 --warmup 5 --no-small-batch > $OUT/bench_cfg4.json 2> $OUT/bench_cfg4.err
echo done
