#!/bin/bash
# A/B the library variants given as arguments (paths of .so files) on the C5 bench (same box, in turn).
mkdir -p gpurun_out
for lib in "$@"; do
  tag=$(basename $lib .so)
  SWE_LIB=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 $BENCH_ARGS > gpurun_out/ab_$tag.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_$tag.log').read().strip().splitlines()[-1]);r=d['roofline'];print('$tag', '%.4e'%d['value'], round(r['achieved']), round(r['k1_launch_ms_avg'],4), round(r['k2_share_of_kernel_time'],4))" || tail -3 gpurun_out/ab_$tag.log
done
