#!/bin/bash
# Round profile capture (full-size C5, N=3, L=4): launch list with per-launch DRAM bytes, ncu --set full of
# K1 (level-4 and level-1 launches of macro step 3, AB3 active) and of one K2 launch.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"^(k_rhs_update|k_tvb|k_tvb_list)$" -s 62 -c 30 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_rhs_update$ -s 31 -c 1 \
   -o gpurun_out/k1_l4 $B > gpurun_out/ncu_k1_l4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_rhs_update$ -s 34 -c 1 \
   -o gpurun_out/k1_l1 $B > gpurun_out/ncu_k1_l1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_tvb(_list)?$" -s 30 -c 1 \
   -o gpurun_out/k2_l4 $B > gpurun_out/ncu_k2.log 2>&1
ls -la gpurun_out
