#!/bin/bash
# fp64 RK4 on tile_f64_kernel: parity tests, integrator timings, small scenes, the reference's own tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_f64_kernel.py tests/test_gpu_api.py -x -q > gpurun_out/pytest_rk4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rk4.log
timeout 300 python tools/integ_probe.py > gpurun_out/integ.log 2>&1
timeout 300 python tools/small_bench.py > gpurun_out/small.log 2>&1
PRECS="f64 f32" REFTEST_TIMEOUT=1200 bash tools/reftests/run.sh > /dev/null 2>&1
tail -n 3 gpurun_out/pytest_rk4.log; cat gpurun_out/integ.log gpurun_out/small.log
tail -n 30 gpurun_out/reftests_f64.log; tail -n 15 gpurun_out/reftests_f32.log
