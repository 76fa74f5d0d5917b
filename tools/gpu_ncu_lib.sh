#!/bin/bash
# Launch list + ncu --set full of one K1 launch (SKIP = matching launches to skip) for the library $1 (default: in-tree), tag $2.
mkdir -p gpurun_out
LIB=${1:-paper_1403_1661_b200/libswe_b200.so}
TAG=${2:-k1}
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
SWE_LIB=$PWD/$LIB timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_rhs_update" -c 40 --csv \
   --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_launch_$TAG.log 2>&1
SWE_LIB=$PWD/$LIB timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_rhs_update" -s ${SKIP:-31} -c 1 \
   -o gpurun_out/k1_$TAG $B > gpurun_out/ncu_k1_$TAG.log 2>&1
ls gpurun_out
