# round-2 GPU session script (gpurun runs it from the repo root on the box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02
O=gpurun_out/r02
nvidia-smi -L > $O/smi.txt 2>&1
timeout 600 python tools/small_batch.py > $O/small_batch.json 2> $O/small_batch.err
timeout 900 python tools/sched_ab.py --configs 2,3,5 --schedules lane,dynamic > $O/sched_ab.jsonl 2> $O/sched_ab.err
timeout 900 python -m pytest tests/test_cuda_parity.py tests/test_cuda_edge_cases.py tests/test_multigpu_p2p.py tests/test_reference_dropin.py -m gpu -q -p no:cacheprovider -x > $O/gputest.log 2>&1; echo "rc=$?" >> $O/gputest.log
