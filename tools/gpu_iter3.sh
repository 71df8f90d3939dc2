#!/bin/bash
# pairwise energies + fp64 RK4 tile stages: full gpu suite, then the reference's tests that failed before.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
REFTEST_PATHS="baseline/_ref/tests/test_engine.py baseline/_ref/tests/test_service.py baseline/_ref/tests/test_analysis.py" REFTEST_K="ivergence or Snapshots or energ" \
  PRECS=f64 REFTEST_TIMEOUT=600 bash tools/reftests/run.sh > /dev/null 2>&1
tail -n 15 gpurun_out/pytest_gpu3.log; tail -n 12 gpurun_out/reftests_f64.log
