#!/bin/bash
# ncu --set full of one K1 launch (level 4 of macro step 3) of a library variant.
# usage: gpu_ncu_variant.sh LIB.so KERNEL_REGEX SKIP OUTNAME
mkdir -p gpurun_out
SWE_LIB=$PWD/$1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 \
   -o gpurun_out/$4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/$4.log 2>&1
tail -2 gpurun_out/$4.log
