#!/bin/bash
# Round numbers: GPU tests, smoke, default bench, N = 2/4/5 and FP32 bench lines (C5 full size).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-300
for N in 2 4 5; do timeout 600 python bench.py --order $N --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_n$N.log 2>&1; done
timeout 600 python bench.py --precision 32 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_fp32.log 2>&1
for f in bench_n2 bench_n4 bench_n5 bench_fp32; do python -c "import json;d=json.loads(open('gpurun_out/$f.log').read().strip().splitlines()[-1]);r=d['roofline'];print('$f', '%.3e'%d['value'], round(r['frac'],3), round(r['step_frac'],3), round(r['k1_launch_ms_avg'],4))"; done
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_gpus2.log 2>&1; tail -1 gpurun_out/bench_gpus2.log | cut -c1-250
