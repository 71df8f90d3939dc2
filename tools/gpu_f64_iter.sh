#!/bin/bash
# fp64 kernel iteration (1 GPU): kernel tests, A/B bench of the variants, one ncu capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_f64_kernel.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pytest_f64.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f64.log
for v in ${VARIANTS:-0 1 2}; do
  SS_F64_VARIANT=$v timeout 300 python bench.py --no-extra --no-400m --no-cpu --steps 10 > gpurun_out/bench_v$v.log 2>&1
done
SS_F64_KERNEL=step timeout 300 python bench.py --no-extra --no-400m --no-cpu --steps 10 > gpurun_out/bench_step.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_f64 -s 20 -c 1 \
   -o gpurun_out/prof_f64new python bench.py --no-extra --no-400m --no-cpu --steps 1 --warmup 3 > gpurun_out/ncu_f64new.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
   --log-file gpurun_out/launches_f64.csv python bench.py --no-extra --no-400m --no-cpu --steps 1 --warmup 3 > /dev/null 2>&1
tail -n 3 gpurun_out/pytest_f64.log
for f in gpurun_out/bench_v*.log gpurun_out/bench_step.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print(d['value'], r['avg_launch_us'], r['frac'], r['kernel'])
" ; tail -2 $f | grep -v "^{"; done
