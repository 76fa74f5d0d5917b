#!/bin/bash
# Parity tests on the default library, then same-box A/B (twice) of the library variants given as arguments.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/pytest_parity.log 2>&1; tail -3 gpurun_out/pytest_parity.log
if [ $# -gt 0 ]; then bash tools/gpu_ab.sh "$@"; bash tools/gpu_ab.sh "$@"; fi
