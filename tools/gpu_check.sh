#!/bin/bash
# One GPU round trip: build check, smoke, GPU tests, bench, ncu launch list + one full K1 capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 1 --warmup 3 --base-n 640 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rhs_update -s 40 -c 2 \
     -o gpurun_out/k1_full python bench.py --steps 1 --warmup 3 --base-n 640 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
fi
ls -la gpurun_out
