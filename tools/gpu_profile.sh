#!/bin/bash
# ncu launch list + one full capture of the top kernel (1 GPU).
mkdir -p gpurun_out
ARGS=${BENCH_ARGS:-"--steps 2 --warmup 3 --no-cpu"}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
   --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch_bench.log 2>&1
echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-step_kernel} -s ${SKIP:-20} -c ${COUNT:-2} \
   -o gpurun_out/prof python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
ls -la gpurun_out
