#!/bin/bash
# Full measurement round (1 GPU): GPU tests, smoke, bench line, reference arm,
# ncu launch list + one full capture of the dominant kernel.
#   KREGEX (default tile_lean) selects the kernel for the full capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-fp64 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-tile_lean} -s 30 -c 1 \
   -o gpurun_out/prof python bench.py --steps 1 --warmup 3 --no-cpu --no-fp64 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
   -o gpurun_out/prof_f64 python tools/f64_probe.py > gpurun_out/ncu_f64.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log
cat gpurun_out/bench.log gpurun_out/bench_ref.log
