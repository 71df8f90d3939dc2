#!/bin/bash
# One iteration on the GPU box: GPU tests, kernel-variant timings, optional ncu capture.
#   KB_VARIANTS="once:3,step2"  NCU_KERNEL=tile_once  NCU_VARIANT=once:3
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
VARIANTS=${KB_VARIANTS:-once:3,once:2,step2} timeout 600 python tools/kbench.py > gpurun_out/kbench.log 2>&1; echo "kbench rc=$?" >> gpurun_out/kbench.log
cat gpurun_out/kbench.log
if [ -n "$NCU_KERNEL" ]; then
  V=${NCU_VARIANT:-once:3}
  export SS_KERNEL=${V%%:*}; [ "$V" != "${V#*:}" ] && export SS_ONCE_MINB=${V#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$NCU_KERNEL -s 30 -c 1 \
     -o gpurun_out/prof_${SS_KERNEL} python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
fi
