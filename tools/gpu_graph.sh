#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pt_graph.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_graph.log
tail -n 3 gpurun_out/pt_graph.log
for g in 1 0; do SS_GRAPH=$g MODES=default CELLS=20,30,42,91 timeout 400 python tools/wave_probe.py | sed "s/^/graph=$g /"; done
