#!/bin/bash
# The N>1 bench path on a one-GPU box: two ranks time-sliced on cuda:0 (numbers meaningless), gloo host coordination.
mkdir -p gpurun_out
SS_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
   --master-port 29633 bench.py --gpus 2 --cells 60 --steps 2 --warmup 1 --no-cpu > gpurun_out/nproc2.log 2> gpurun_out/nproc2.err
echo "rc=$?" >> gpurun_out/nproc2.err
SS_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
   --master-port 29634 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/nproc2_ref.log 2>&1
echo "rc=$?" >> gpurun_out/nproc2_ref.log
tail -n 5 gpurun_out/nproc2.err; cat gpurun_out/nproc2.log; tail -c 600 gpurun_out/nproc2_ref.log
