#!/bin/bash
# Bench at order N=$1 (C5 full size) + ncu launch list + ncu --set full of one level-4 K1 launch.
mkdir -p gpurun_out
N=${1:-4}
timeout 600 python bench.py --order $N --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n$N.log 2>&1; tail -1 gpurun_out/bench_n$N.log | cut -c1-400
B="python bench.py --order $N --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_rhs_update" -s ${SKIP:-31} -c 1 \
   -o gpurun_out/k1_n$N $B > gpurun_out/ncu_k1_n$N.log 2>&1
ncu -i gpurun_out/k1_n$N.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/k1_n${N}_src.csv 2>/dev/null
ls gpurun_out | tail -3
