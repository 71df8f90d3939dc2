#!/bin/bash
# fp64 kernel A/B (variants, V read skipped), transfer rates, e2e breakdown
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_f64_kernel.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_f64.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f64.log
for v in 0 4 5 0; do
  SS_F64_VARIANT=$v timeout 300 python bench.py --no-extra --no-400m --no-cpu --steps 10 > gpurun_out/ab_v$v.log 2>&1
  python - <<PY
import json
for l in open('gpurun_out/ab_v$v.log'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('variant $v', round(d['value']/1e9,1), 'G/s', round(r['avg_launch_us'],2), 'us', round(r['frac'],3), 'e2e', round(d['e2e']['value']/1e9,1))
PY
done
timeout 300 python tools/xfer_probe.py > gpurun_out/xfer.log 2>&1
PREC=f64 timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_f64.log 2>&1
PREC=f32 timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_f32.log 2>&1
tail -n 2 gpurun_out/pytest_f64.log; cat gpurun_out/xfer.log gpurun_out/e2e_f64.log gpurun_out/e2e_f32.log
