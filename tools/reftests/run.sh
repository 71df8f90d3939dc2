#!/bin/bash
# Run the reference's own tests (copied into the git-ignored baseline/_ref/tests
# by tools/reftests/prepare.sh) against the B200 engine.  Output: gpurun_out/reftests_<prec>.log
# REFTEST_PATHS (default: the whole suite), REFTEST_K (a -k expression), PRECS (default f64).
mkdir -p gpurun_out
export NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=$PWD:$PWD/baseline/_ref
for prec in ${PRECS:-f64}; do
  SS_REFTEST_PRECISION=$prec timeout ${REFTEST_TIMEOUT:-1500} python -m pytest ${REFTEST_PATHS:-baseline/_ref/tests} \
     -p tools.reftests.gpu_backend_plugin -q -rfE -o addopts="" ${REFTEST_K:+-k "$REFTEST_K"} \
     > gpurun_out/reftests_$prec.log 2>&1
  echo "rc=$?" >> gpurun_out/reftests_$prec.log
  tail -n 40 gpurun_out/reftests_$prec.log
done
