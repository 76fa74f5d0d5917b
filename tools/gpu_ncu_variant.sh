#!/bin/bash
# ncu --set full of one K1 launch of a library variant / bench configuration.
# usage: gpu_ncu_variant.sh LIB.so KERNEL_REGEX SKIP OUTNAME [extra bench args]
mkdir -p gpurun_out
LIB=$1; RX=$2; SK=$3; OUT=$4; shift 4
SWE_LIB=$PWD/$LIB timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SK -c 1 \
   -o gpurun_out/$OUT python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 "$@" > gpurun_out/$OUT.log 2>&1
tail -2 gpurun_out/$OUT.log
