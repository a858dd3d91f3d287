#!/bin/bash
# re-entry check of HEAD: smoke, the whole -m gpu suite, default bench line, reference arm, config-4 line
TAG=${1:-r02s2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ref_cfg2.json 2> $OUT/bench_ref_cfg2.err
timeout 1200 python bench.py --config 4 --steps 20 --warmup 5 --no-small-batch > $OUT/bench_cfg4.json 2> $OUT/bench_cfg4.err
echo done
