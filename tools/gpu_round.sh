#!/bin/bash
# Tests + A/B of the given variant libraries (twice, same box) + K1 level-4 ncu --set full capture
# and the launch list of the default library at full C5 size.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
if [ $# -gt 0 ]; then bash tools/gpu_ab.sh "$@"; bash tools/gpu_ab.sh "$@"; fi
if [ "${NCU:-1}" = "1" ]; then
  B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:"^(k_rhs_update|k_tvb)$" -s 62 -c 30 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_rhs_update$ -s 31 -c 1 \
     -o gpurun_out/k1_l4 $B > gpurun_out/ncu_k1_l4.log 2>&1
fi
ls gpurun_out
