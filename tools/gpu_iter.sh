#!/bin/bash
# Iteration loop on the GPU: tests, parity tracer, quick bench, K1 ncu capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
for c in thacker dambreak tvb; do timeout 300 python tools/debug_parity.py $c 100 > gpurun_out/dbg_$c.log 2>&1; done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench.log 2>&1
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rhs_update -s 40 -c 1 \
     -o gpurun_out/k1_full python bench.py --steps 1 --warmup 3 --base-n 640 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log | cut -c1-400
