#!/bin/bash
# A/B the library variants given as arguments (paths of .so files) on the C5 bench.
mkdir -p gpurun_out
for lib in "$@"; do
  tag=$(basename $lib .so)
  SWE_LIB=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 $BENCH_ARGS > gpurun_out/ab_$tag.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_$tag.log').read().strip().splitlines()[-1]);print('$tag', '%.3e'%d['value'], round(d['roofline']['achieved']), round(d['roofline']['k1_share_of_step'],3))" || tail -3 gpurun_out/ab_$tag.log
done
