#!/bin/bash
# Full measurement round (1 GPU): GPU tests, smoke, bench line, reference arm,
# ncu launch list of the headline (fp64) bench, one full capture of the fp64
# headline kernel and one of the fp32 production kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/host.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/host.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-400m --no-extra > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_f64 -s 30 -c 1 \
   -o gpurun_out/prof_f64 python bench.py --steps 1 --warmup 3 --no-cpu --no-400m --no-extra > gpurun_out/ncu_f64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_lean -s 30 -c 1 \
   -o gpurun_out/prof_f32 python bench.py --precision f32 --steps 1 --warmup 3 --no-cpu --no-400m --no-extra > gpurun_out/ncu_f32.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.err
cat gpurun_out/bench.log gpurun_out/bench_ref.log
