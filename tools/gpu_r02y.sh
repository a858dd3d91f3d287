#!/bin/bash
# round-2: the N>1 bench code path on the final build, ranks sharing the box's one GPU over gloo
# (P2P frame assembly into rank 0 through CUDA IPC; frame 0 checked against the reference digests)
TAG=${1:-r02y}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for N in 2 4; do
  TETB200_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps 10 --warmup 3 \
      --no-small-batch --no-cpu-baseline > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err
  echo "N=$N rc=$?" >> $OUT/rc.txt
done
echo done
