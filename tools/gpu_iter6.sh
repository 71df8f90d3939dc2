#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_energy_pairwise.py -x -q > gpurun_out/pytest_api.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_api.log
timeout 600 python bench.py --no-400m --no-cpu --steps 10 > gpurun_out/bench6.log 2>&1
tail -n 3 gpurun_out/pytest_api.log
python - <<PY
import json
for l in open('gpurun_out/bench6.log'):
    if l.startswith('{'):
        d=json.loads(l); print('f64', round(d['value']/1e9,1), 'e2e', round(d['e2e']['value']/1e9,1), 'f32', round(d['fp32_production']['value']/1e9,1), 'e2e', round(d['fp32_production']['e2e']['value']/1e9,1), 'general', round(d['general_graph_format']['value']/1e9,1))
PY
tail -3 gpurun_out/bench6.log | grep -v "^{"
