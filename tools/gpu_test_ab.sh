#!/bin/bash
# GPU tests, then an A/B of library variants on the C5 bench (args: .so paths).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu_ab.sh "$@"
