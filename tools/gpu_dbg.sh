#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
for c in thacker dambreak tvb; do timeout 300 python tools/debug_parity.py $c 100 > gpurun_out/dbg_$c.log 2>&1; done
for L in 1 2 3; do L=$L timeout 300 python tools/debug_parity.py smoothmrab 10 > gpurun_out/dbg_smooth_L$L.log 2>&1; done
tail -3 gpurun_out/pytest_gpu.log
