#!/bin/bash
# gpu suite + the reference's whole test suite against the GPU engine (f64, f32)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
PRECS="f64 f32" REFTEST_TIMEOUT=1200 bash tools/reftests/run.sh > /dev/null 2>&1
tail -n 5 gpurun_out/pytest_gpu4.log; grep -E "FAILED|passed|failed" gpurun_out/reftests_f64.log gpurun_out/reftests_f32.log
