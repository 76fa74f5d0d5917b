#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -rf -x > gpurun_out/pytest_gpu.log 2>&1
for mb in 3; do SWE_K1_MINB=$mb timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_mb$mb.log 2>&1; done
SWE_K1_MINB=${MB:-3} timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rhs_update -s 40 -c 1 \
     -o gpurun_out/k1_full python bench.py --steps 1 --warmup 3 --base-n 640 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
for mb in 3; do python -c "import json;d=json.loads(open('gpurun_out/bench_mb$mb.log').read().strip().splitlines()[-1]);print($mb, '%.3e'%d['value'], d['roofline']['achieved'], d['roofline']['k1_share_of_step'])"; done
