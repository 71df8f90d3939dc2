#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_api.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_observables.py -x -q > gpurun_out/pytest_res.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_res.log
timeout 300 python tools/cluster_check.py > gpurun_out/cluster_check.log 2>&1
tail -n 3 gpurun_out/pytest_res.log; cat gpurun_out/cluster_check.log
