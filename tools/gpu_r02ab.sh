#!/bin/bash
# round-2: pipelined root epilogue of the P2P frame assembly -- two-rank tests + N=2/4 bench on the shared GPU
TAG=${1:-r02ab}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_multigpu_p2p.py -m gpu -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for N in 2 4; do
  TETB200_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps 10 --warmup 3 \
      --no-small-batch --no-cpu-baseline > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err
  echo "N=$N rc=$?" >> $OUT/rc.txt
done
echo done
