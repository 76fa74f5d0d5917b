#!/bin/bash
mkdir -p gpurun_out
for L in 2; do L=$L timeout 300 python tools/debug_parity.py smoothmrab 2 > gpurun_out/dbg_smooth_L$L.log 2>&1; done
