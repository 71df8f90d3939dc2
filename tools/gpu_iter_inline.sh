#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_f64_kernel.py tests/test_gpu_api.py -x -q > gpurun_out/pytest_inl.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_inl.log
timeout 600 python bench.py --no-400m --no-cpu --steps 10 > gpurun_out/bench_inl.log 2>&1
tail -n 3 gpurun_out/pytest_inl.log
python - <<PY
import json
for l in open('gpurun_out/bench_inl.log'):
    if l.startswith('{'):
        d=json.loads(l); g=d['general_graph_format']; print('f64', round(d['value']/1e9,1), round(d['roofline']['avg_launch_us'],2), 'general', round(g['value']/1e9,1), round(g['roofline']['avg_launch_us'],2), g['roofline']['kernel'], g['roofline']['format'], 'e2e', round(d['e2e']['value']/1e9,1))
PY
