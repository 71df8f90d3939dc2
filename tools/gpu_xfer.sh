#!/bin/bash
mkdir -p gpurun_out
for mb in 1 2 4 8 16; do SS_CHUNK_MB=$mb timeout 120 python tools/xfer_probe.py; done > gpurun_out/xfer_chunks.log 2>&1
for t in 2 4 8; do echo "omp $t"; OMP_NUM_THREADS=$t SS_CHUNK_MB=4 timeout 120 python tools/xfer_probe.py; done >> gpurun_out/xfer_chunks.log 2>&1
cat gpurun_out/xfer_chunks.log
