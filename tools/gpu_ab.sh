#!/bin/bash
# A/B of fp64 kernel variants (env pairs in $AB, ';'-separated), bench --no-extra each.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_f64_kernel.py -x -q > gpurun_out/pytest_f64.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f64.log
IFS=';' read -ra RUNS <<< "$AB"
i=0
for envs in "${RUNS[@]}"; do
  env $envs timeout 300 python bench.py --no-extra --no-400m --no-cpu --steps 10 ${BENCH_ARGS} > gpurun_out/ab_$i.log 2>&1
  python -c "
import json
for l in open('gpurun_out/ab_$i.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('$envs', round(d['value']/1e9,1), 'G/s', round(r['avg_launch_us'],2), 'us', round(r['frac'],3), r['kernel'])
"
  i=$((i+1))
done
tail -n 2 gpurun_out/pytest_f64.log
